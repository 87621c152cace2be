"""Pins of oracle.allegro (E, E_i, F) against what the mathematics fixes.

* F = -grad E (Eq. 1): central finite differences and an
  independent torch-autograd witness (tests/torch_witness.py).
* E(3) invariance: random rotations of isolated clusters, the 48
  cubic-group operations incl. inversion on periodic boxes, translations,
  permutations; zero net force.
* locality / extensivity: 2x2x2 replica -> E x 8, same forces.
* cutoff smoothness, envelope closed forms, c_SiLU by quadrature.
* pair-potential limit: W_env = 0 -> E = sum_e f(Z_i, Z_j, d), checked against
  an independent scalar code (plain loops).
"""
import itertools
import math

import numpy as np
import pytest
from scipy import integrate

from oracle import allegro, neighbors, weights_io
from synth import nh3, weights as sw

from . import torch_witness


def _model(tmp, L, lmax, r_c, seed=0, sigma=1.0, mutate=None):
    path = f"{tmp}/m_{L}_{lmax}_{r_c}_{seed}.algw"
    tensors = sw.generate(L, lmax, seed)
    if mutate:
        tensors = mutate(tensors)
    sw.write(path, L, lmax, r_c, tensors, sw.nbar_for(r_c), (sigma, 1.3 * sigma), (0.0, 0.0))
    return weights_io.read(path)


@pytest.fixture(scope="module")
def tmp(tmp_path_factory):
    return str(tmp_path_factory.mktemp("w"))


@pytest.fixture(scope="module")
def c1():
    return nh3.nh3_box("fcc", (1, 1, 1))


def _cluster(n_mol=3, box=40.0, seed=5):
    rng = np.random.default_rng(seed)
    pos, spc = [], []
    for m in range(n_mol):
        rot = nh3._quat_to_matrix(rng.standard_normal(4) / 1.0)
        q = rng.standard_normal(4)
        rot = nh3._quat_to_matrix(q / np.linalg.norm(q))
        ctr = np.array([box / 2] * 3) + rng.uniform(-2.5, 2.5, 3)
        pos.append(ctr + nh3.BODY @ rot.T)
        spc.append(nh3.BODY_SPECIES)
    return np.concatenate(pos), np.concatenate(spc), np.array([box] * 3)


def test_c_silu_quadrature():
    f = lambda z: (z / (1 + math.exp(-z))) ** 2 * math.exp(-z * z / 2) / math.sqrt(2 * math.pi)
    val, _ = integrate.quad(f, -40, 40, epsabs=1e-14, epsrel=1e-14)
    assert abs(val ** -0.5 - allegro.C_SILU) < 1e-9


def test_envelope_closed_form():
    rc = 5.0
    d = np.array([0.0, rc])
    np.testing.assert_allclose(allegro.envelope(d, rc), [1.0, 0.0], atol=1e-15)
    np.testing.assert_allclose(allegro.envelope_deriv(d, rc), [0.0, 0.0], atol=1e-15)
    # u''(r_c) = 0: second difference of u' at the cutoff
    # u''(r_c - h) ~ u'''(r_c) h -> 0 linearly in h
    v = lambda h: abs(allegro.envelope_deriv(np.array([rc - h]), rc)[0]) / h
    assert v(1e-5) < 1e-4 and v(1e-6) < v(1e-5) / 5
    dd = np.linspace(0.5, 4.9, 9)
    fd = (allegro.envelope(dd + 1e-6, rc) - allegro.envelope(dd - 1e-6, rc)) / 2e-6
    np.testing.assert_allclose(allegro.envelope_deriv(dd, rc), fd, atol=1e-8)
    freq = np.pi * np.arange(1, 9)
    fd = (allegro.bessel(dd + 1e-6, rc, freq) - allegro.bessel(dd - 1e-6, rc, freq)) / 2e-6
    np.testing.assert_allclose(allegro.bessel_deriv(dd, rc, freq), fd, atol=1e-7)


@pytest.mark.parametrize("L,lmax", [(2, 1), (3, 2)])
def test_forces_equal_finite_differences(tmp, c1, L, lmax):
    m = _model(tmp, L, lmax, 5.0)
    r = allegro.energy_forces(m, c1.pos, c1.species, c1.box)
    h = 1e-5
    rng = np.random.default_rng(0)
    coords = [(a, al) for a in range(c1.n) for al in range(3)]
    if L == 3:
        coords = [coords[q] for q in rng.choice(len(coords), 12, replace=False)]
    scale = np.abs(r["forces"]).max()
    for a, al in coords:
        p = c1.pos.copy()
        p[a, al] += h
        ep = allegro.energy_forces(m, p, c1.species, c1.box)["energy"]
        p[a, al] -= 2 * h
        em = allegro.energy_forces(m, p, c1.species, c1.box)["energy"]
        assert abs(-(ep - em) / (2 * h) - r["forces"][a, al]) <= 1e-7 * scale


@pytest.mark.parametrize("L,lmax", [(2, 1), (2, 2), (3, 0), (3, 1), (3, 2)])
def test_torch_autograd_witness(tmp, c1, L, lmax):
    m = _model(tmp, L, lmax, 5.0)
    r = allegro.energy_forces(m, c1.pos, c1.species, c1.box)
    pos = neighbors.wrap(c1.pos, c1.box)
    E, F = torch_witness.energy_forces(m, pos, c1.species, c1.box, r["edges"])
    assert abs(E - r["energy"]) <= 1e-12 * np.abs(r["e_atom"]).sum()
    np.testing.assert_allclose(r["forces"], F, atol=1e-12 * np.abs(F).max())


@pytest.mark.parametrize("L,lmax", [(2, 1), (3, 2)])
def test_net_force_zero_and_translation(tmp, c1, L, lmax):
    m = _model(tmp, L, lmax, 5.0)
    r = allegro.energy_forces(m, c1.pos, c1.species, c1.box)
    assert np.abs(r["forces"].sum(0)).max() < 1e-10
    r2 = allegro.energy_forces(m, c1.pos + np.array([1.3, -2.1, 7.7]), c1.species, c1.box)
    assert abs(r2["energy"] - r["energy"]) < 1e-11 * np.abs(r["e_atom"]).sum()
    np.testing.assert_allclose(r2["forces"], r["forces"], atol=1e-11)


def test_permutation(tmp, c1):
    m = _model(tmp, 2, 1, 5.0)
    r = allegro.energy_forces(m, c1.pos, c1.species, c1.box)
    perm = np.random.default_rng(3).permutation(c1.n)
    r2 = allegro.energy_forces(m, c1.pos[perm], c1.species[perm], c1.box)
    assert abs(r2["energy"] - r["energy"]) < 1e-11
    np.testing.assert_allclose(r2["forces"], r["forces"][perm], atol=1e-11)
    np.testing.assert_allclose(r2["e_atom"], r["e_atom"][perm], atol=1e-11)


@pytest.mark.parametrize("L,lmax", [(2, 1), (3, 1), (3, 2)])
def test_rotation_isolated_cluster(tmp, L, lmax):
    m = _model(tmp, L, lmax, 5.0)
    pos, spc, box = _cluster()
    r = allegro.energy_forces(m, pos, spc, box)
    rng = np.random.default_rng(7)
    from oracle import so3

    ctr = box / 2
    for _ in range(3):
        R = so3.random_rotation(rng)
        pr = (pos - ctr) @ R.T + ctr
        r2 = allegro.energy_forces(m, pr, spc, box)
        assert abs(r2["energy"] - r["energy"]) <= 1e-12 * np.abs(r["e_atom"]).sum()
        np.testing.assert_allclose(r2["forces"], r["forces"] @ R.T, atol=1e-12 * np.abs(r["forces"]).max())


def _cubic_ops():
    ops = []
    for perm in itertools.permutations(range(3)):
        for signs in itertools.product((1, -1), repeat=3):
            M = np.zeros((3, 3))
            for a in range(3):
                M[a, perm[a]] = signs[a]
            ops.append(M)
    return ops


@pytest.mark.parametrize("L,lmax", [(2, 1), (3, 2)])
def test_cubic_group_with_inversion(tmp, c1, L, lmax):
    m = _model(tmp, L, lmax, 5.0)
    r = allegro.energy_forces(m, c1.pos, c1.species, c1.box)
    ops = _cubic_ops()
    assert len(ops) == 48
    if L == 3:
        ops = [ops[q] for q in (0, 7, 13, 22, 35, 47)] + [-np.eye(3)]
    for M in ops:
        pr = neighbors.wrap(c1.pos @ M.T, c1.box)
        r2 = allegro.energy_forces(m, pr, c1.species, c1.box)
        assert abs(r2["energy"] - r["energy"]) <= 1e-12 * np.abs(r["e_atom"]).sum()
        np.testing.assert_allclose(r2["forces"], r["forces"] @ M.T, atol=1e-12 * np.abs(r["forces"]).max())


def test_extensivity_2x2x2(tmp, c1):
    m = _model(tmp, 2, 1, 5.0)
    r = allegro.energy_forces(m, c1.pos, c1.species, c1.box)
    big = nh3.replicate(c1, (2, 2, 2))
    r8 = allegro.energy_forces(m, big.pos, big.species, big.box)
    assert abs(r8["energy"] - 8 * r["energy"]) <= 1e-10 * np.abs(r8["e_atom"]).sum()
    np.testing.assert_allclose(r8["forces"], np.tile(r["forces"], (8, 1)), atol=1e-10)


def test_cutoff_smoothness(tmp):
    m = _model(tmp, 2, 1, 5.0)
    box = np.array([30.0, 30.0, 30.0])
    spc = np.array([1, 0])
    out = []
    for dd in (5.0 - 1e-6, 5.0, 5.0 + 1e-6):
        pos = np.array([[10.0, 10.0, 10.0], [10.0 + dd, 10.0, 10.0]])
        r = allegro.energy_forces(m, pos, spc, box)
        out.append((r["energy"], r["forces"][1, 0]))
    # E ~ (r_c - d)^3 near the cutoff (u is C^2): continuous to ~1e-16
    assert max(abs(e) for e, _ in out) < 1e-12
    assert max(abs(f) for _, f in out) < 1e-9


def _scalar_pair_energy(t, zi, zj, d, rc, nbar, sigma, L, n_s_list):
    """Independent scalar code for E_e(i -> j) with W_env = 0 (plain loops)."""
    x = d / rc
    u = 1 - 28 * x**6 + 48 * x**7 - 21 * x**8 if x < 1 else 0.0
    z = [1.0 if zi == 0 else 0.0, 1.0 if zi == 1 else 0.0, 1.0 if zj == 0 else 0.0, 1.0 if zj == 1 else 0.0]
    z += [u * (2 / rc) * math.sin(t["bessel_freq"][n] * d / rc) / d for n in range(8)]

    def lin(v, W, scale):
        return [sum(v[q] * W[q][k] for q in range(len(v))) * scale for k in range(len(W[0]))]

    silu = lambda a: a / (1 + math.exp(-a))
    c = 1.6765324703
    h = [silu(a) for a in lin(z, t["tb_w0"], 1 / math.sqrt(12))]
    h = [silu(a) for a in lin(h, t["tb_w1"], c / math.sqrt(32))]
    lat = [u * a for a in lin(h, t["tb_w2"], c / math.sqrt(64))]
    for k in range(L):
        Wl = t[f"lat_{k}"]
        fan = 128 + 32 * n_s_list[k]
        hh = lin(lat, Wl[:128], 1 / math.sqrt(fan))  # scalars s are exactly 0
        lat = [(2 * a + u * b) / math.sqrt(5) for a, b in zip(lat, hh)]
    e1 = lin(lat, t["out_w1"], 1 / math.sqrt(128))
    e = lin(e1, t["out_w2"], 1 / math.sqrt(32))[0]
    return sigma[zi] / math.sqrt(nbar) * e


def test_pair_potential_limit(tmp):
    def zero_env(tensors):
        return [(n, np.zeros_like(a) if n.startswith("env_") else a) for n, a in tensors]

    m = _model(tmp, 2, 1, 5.0, mutate=zero_env)
    box = np.array([30.0, 30.0, 30.0])
    spc = np.array([1, 0])
    for dd in (0.9, 1.7, 3.1, 4.6):
        pos = np.array([[10.0, 11.0, 12.0], [10.0 + dd, 11.0, 12.0]])
        r = allegro.energy_forces(m, pos, spc, box)
        E = lambda q: (
            _scalar_pair_energy(m.t, 1, 0, q, 5.0, m.nbar, m.sigma, 2, [2, 2])
            + _scalar_pair_energy(m.t, 0, 1, q, 5.0, m.nbar, m.sigma, 2, [2, 2])
        )
        assert abs(r["energy"] - E(dd)) < 1e-12 * max(1.0, abs(E(dd)))
        h = 1e-5
        f = -(E(dd + h) - E(dd - h)) / (2 * h)
        assert abs(r["forces"][1, 0] - f) < 1e-8
        assert abs(r["forces"][0, 0] + f) < 1e-8


def test_sampled_forces_match_full(tmp):
    m = _model(tmp, 2, 1, 5.0)
    s = nh3.nh3_box("fcc", (2, 2, 2))
    full = allegro.energy_forces(m, s.pos, s.species, s.box)
    atoms = np.array([0, 5, 77, 120])
    F, Ei, _ = allegro.sampled_forces(m, s.pos, s.species, s.box, atoms)
    np.testing.assert_allclose(F, full["forces"][atoms], atol=1e-12)
    np.testing.assert_allclose(Ei, full["e_atom"][atoms], atol=1e-12)
