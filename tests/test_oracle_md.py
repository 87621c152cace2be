"""Pins of oracle.md: velocity Verlet, kinetic
energy, outlier rule (Fig. 1)."""
import math

import numpy as np
import pytest

from oracle import allegro, md, weights_io
from synth import nh3, weights as sw


def test_harmonic_oscillator_closed_form():
    # one H atom in a harmonic well F = -k x: Verlet vs exact cos
    k = 2.0
    m = md.MASS_H
    omega = math.sqrt(k * md.KAPPA / m)
    box = np.array([1e6, 1e6, 1e6])
    x0 = box / 2 + np.array([0.1, 0.0, 0.0])
    fn = lambda p: (0.5 * k * np.sum((p - box / 2) ** 2), -k * (p - box / 2))
    dt = 0.05
    n = int(2 * math.pi / omega / dt)
    p, v, _, _ = md.verlet(fn, x0[None], np.zeros((1, 3)), np.array([0]), box, dt, n)
    exact = 0.1 * math.cos(omega * n * dt)
    assert abs((p[0, 0] - box[0] / 2) - exact) < 1e-3 * 0.1
    # energy error is O(dt^2): halving dt quarters the max deviation
    def max_err(dt):
        steps = int(20 / dt)
        _, _, _, log = md.verlet(fn, x0[None], np.zeros((1, 3)), np.array([0]), box, dt, steps)
        e = np.array([a + b for a, b in log])
        return np.abs(e - 0.5 * k * 0.01).max()
    r = max_err(0.2) / max_err(0.1)
    assert 3.6 < r < 4.4


def test_free_atom_and_wrap():
    box = np.array([5.0, 5.0, 5.0])
    fn = lambda p: (0.0, np.zeros_like(p))
    p, v, _, _ = md.verlet(fn, np.array([[4.9, 0.1, 2.5]]), np.array([[0.05, -0.05, 0.0]]), np.array([1]), box, 2.0, 10)
    np.testing.assert_allclose(p[0], [(4.9 + 1.0) % 5.0, (0.1 - 1.0) % 5.0, 2.5], atol=1e-12)
    assert np.all(p >= 0) and np.all(p < box)


def test_kinetic_energy_and_temperature_units():
    # KE = 1/2 m v^2 / kappa eV; T = 2 KE / (3 N k_B)
    v = np.array([[0.01, 0.0, 0.0]])
    ke = md.kinetic_energy(v, np.array([1]))
    assert abs(ke - 0.5 * 14.007 * 1e-4 * 103.6427) < 1e-6
    s = nh3.maxwell_boltzmann(nh3.nh3_box("fcc", (6, 6, 6)), 200.0)
    assert abs(md.temperature(s.vel, s.species) - 200.0) < 10.0
    p = (s.masses()[:, None] * s.vel).sum(0)
    assert np.abs(p).max() < 1e-12


def test_outlier_hand_examples():
    # all at mean -> 0; one at mean + 6 sigma -> 1; exactly 5 sigma -> 0
    F = np.array([[1.0, 0, 0]] * 10)
    assert md.count_outliers(F, 1.0, 0.5) == 0
    F2 = F.copy()
    F2[3] = [1.0 + 6 * 0.5, 0, 0]
    assert md.count_outliers(F2, 1.0, 0.5) == 1
    F3 = F.copy()
    F3[3] = [1.0 + 5 * 0.5, 0, 0]
    assert md.count_outliers(F3, 1.0, 0.5) == 0
    mean, std = md.force_baseline(np.array([[3.0, 4.0, 0.0], [0.0, 0.0, 1.0]]))
    assert mean == 3.0 and std == 2.0


@pytest.fixture(scope="module")
def c1_model(tmp_path_factory):
    path = str(tmp_path_factory.mktemp("w") / "c1.algw")
    sw.write(path, 2, 1, 5.0, sw.generate(2, 1, 0), sw.nbar_for(5.0), (0.05, 0.05), (0.0, 0.0))
    return weights_io.read(path)


def test_model_nve_time_reversal_momentum_and_dt2(c1_model):
    s = nh3.maxwell_boltzmann(nh3.nh3_box("fcc", (1, 1, 1)), 200.0)
    fn = lambda p: (lambda r: (r["energy"], r["forces"]))(allegro.energy_forces(c1_model, p, s.species, s.box))
    p1, v1, f1, log = md.verlet(fn, s.pos, s.vel, s.species, s.box, 1.0, 10)
    # time reversal
    p2, v2, _, _ = md.verlet(fn, p1, -v1, s.species, s.box, 1.0, 10, forces=f1)
    d = p2 - nh3.wrap_positions(s.pos, s.box)
    d -= s.box * np.round(d / s.box)
    assert np.abs(d).max() < 1e-10
    np.testing.assert_allclose(-v2, s.vel, atol=1e-10)
    # momentum conservation
    m = s.masses()[:, None]
    assert np.abs((m * v1).sum(0)).max() < 1e-10
    # NVE energy fluctuation scales as dt^2
    def fluct(dt):
        _, _, _, lg = md.verlet(fn, s.pos, s.vel, s.species, s.box, dt, int(8 / dt))
        e = np.array([a + b for a, b in lg])
        return e.max() - e.min()
    r = fluct(1.0) / fluct(0.5)
    assert 3.0 < r < 5.0


def test_nvt_reduces_to_nve_for_infinite_q(c1_model):
    s = nh3.maxwell_boltzmann(nh3.nh3_box("fcc", (1, 1, 1)), 200.0)
    fn = lambda p: (lambda r: (r["energy"], r["forces"]))(allegro.energy_forces(c1_model, p, s.species, s.box))
    p1, v1, _, _ = md.verlet(fn, s.pos, s.vel, s.species, s.box, 1.0, 3)
    p2, v2, _, xi, eta, _ = md.nvt_verlet(fn, s.pos, s.vel, s.species, s.box, 1.0, 3, 200.0, 1e12)
    np.testing.assert_allclose(p2, p1, atol=1e-12)
    np.testing.assert_allclose(v2, v1, atol=1e-12)
    assert abs(xi) < 1e-20


def test_nvt_fixed_point_first_quarter():
    # K exactly at g k_B T / 2 and xi = 0: the thermostat quarter-kick leaves xi = 0
    species = np.array([0, 1, 1])
    v = np.random.default_rng(0).standard_normal((3, 3))
    K = md.kinetic_energy(v, species)
    T = 2 * K / (3 * 3 * md.KB)
    g = 9
    Q = g * md.KB * T * 50.0**2
    vel, K2, xi, eta = md.nvt_half(v, species, K, 0.0, 0.0, 1.0, T, Q)
    assert xi == 0.0 and eta == 0.0 and np.array_equal(vel, v)


def test_nvt_conserved_quantity_dt2_and_thermalisation(c1_model):
    s = nh3.maxwell_boltzmann(nh3.nh3_box("fcc", (1, 1, 1)), 300.0)  # start hot, target 200 K
    fn = lambda p: (lambda r: (r["energy"], r["forces"]))(allegro.energy_forces(c1_model, p, s.species, s.box))

    def drift(dt):
        _, _, _, _, _, lg = md.nvt_verlet(fn, s.pos, s.vel, s.species, s.box, dt, int(6 / dt), 200.0, 20.0)
        h = np.array([c for _, _, c in lg])
        return h.max() - h.min(), lg

    d1, lg = drift(1.0)
    d2, _ = drift(0.5)
    assert 3.0 < d1 / d2 < 5.0  # extended energy conserved to O(dt^2)
    # the thermostat removes kinetic energy from the 300 K start
    assert lg[-1][1] < md.kinetic_energy(s.vel, s.species)
