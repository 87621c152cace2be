"""Pins of oracle/pimd.py (ring-polymer MD, reading D25) against closed forms, an independent
matrix exponential (scipy.linalg.expm), the classical limit P = 1 and energy conservation."""
import numpy as np
import pytest
from scipy.linalg import expm

from oracle import md, pimd

KB, HBAR = md.KB, pimd.HBAR


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8, 32])
def test_normal_modes_orthonormal_and_diagonalise_the_ring(P):
    C = pimd.normal_mode_matrix(P)
    np.testing.assert_allclose(C.T @ C, np.eye(P), atol=1e-13)
    S = np.roll(np.eye(P), 1, axis=1)  # cyclic shift
    A = 2 * np.eye(P) - S - S.T         # ring Laplacian: sum_j |q_j - q_j+1|^2 = q^T A q
    D = C.T @ A @ C
    lam = 4 * np.sin(np.arange(P) * np.pi / P) ** 2
    np.testing.assert_allclose(D, np.diag(lam), atol=1e-12)


def test_frequencies_closed_form():
    wp = pimd.omega_p(32, 200.0)
    assert abs(wp - 32 * 8.617333e-5 * 200.0 / 0.6582119569) < 1e-15
    w = pimd.mode_frequencies(32, wp)
    assert w[0] == 0 and abs(w[16] - 2 * wp) < 1e-12 and np.allclose(w[1:16], w[31:16:-1])


@pytest.mark.parametrize("P", [2, 3, 6])
def test_free_ring_step_equals_matrix_exponential(P):
    """V = 0: m dv/dt = -m w_P^2 A q per component; the exact flow is expm of the 2P x 2P
    generator -- an independent library routine."""
    rng = np.random.default_rng(P)
    q = rng.normal(size=(P, 2, 3))
    v = rng.normal(size=(P, 2, 3)) * 0.01
    wp, dt = 0.3, 0.7
    q1, v1 = pimd.free_ring_step(q, v, wp, dt)
    S = np.roll(np.eye(P), 1, axis=1)
    A = 2 * np.eye(P) - S - S.T
    G = np.block([[np.zeros((P, P)), np.eye(P)], [-wp * wp * A, np.zeros((P, P))]])
    U = expm(G * dt)
    for n in range(2):
        for d in range(3):
            y = U @ np.concatenate([q[:, n, d], v[:, n, d]])
            np.testing.assert_allclose(q1[:, n, d], y[:P], atol=1e-12)
            np.testing.assert_allclose(v1[:, n, d], y[P:], atol=1e-12)


def test_free_ring_conserves_energy_and_centroid_velocity():
    rng = np.random.default_rng(1)
    P, species = 8, np.array([0, 1, 0])
    q = rng.normal(size=(P, 3, 3)) * 0.1
    v = rng.normal(size=(P, 3, 3)) * 0.02
    wp = pimd.omega_p(P, 200.0)
    m = md.masses(species)[None, :, None]
    e = lambda q, v: float(0.5 * np.sum(m * v * v) / md.KAPPA) + pimd.spring_energy(q, species, wp)
    e0, vc0, qc0 = e(q, v), v.mean(axis=0), q.mean(axis=0)
    q1, v1 = pimd.free_ring_step(q, v, wp, 13.0)
    assert abs(e(q1, v1) - e0) < 1e-12 * max(1, abs(e0))
    np.testing.assert_allclose(v1.mean(axis=0), vc0, atol=1e-14)
    np.testing.assert_allclose(q1.mean(axis=0), qc0 + 13.0 * vc0, atol=1e-12)


def _harmonic(anchors, box, k=1.5):
    def fn(pos):
        d = pos - anchors
        d -= box * np.round(d / box)
        return 0.5 * k * float((d * d).sum()), -k * d
    return fn


def test_one_bead_is_classical_velocity_verlet():
    rng = np.random.default_rng(2)
    box = np.array([10.0, 11.0, 12.0])
    species = np.array([0, 1, 0, 0])
    x0 = rng.uniform(1, 9, size=(4, 3))
    v0 = rng.normal(size=(4, 3)) * 0.01
    fn = _harmonic(x0 + 0.2, box)
    q, v, f, _ = pimd.pimd(fn, x0[None], v0[None], species, box, 0.5, 300.0, 20)
    p2, v2, f2, _ = md.verlet(fn, x0, v0, species, box, 0.5, 20)
    np.testing.assert_allclose(pimd.wrap(q[0], box), p2, atol=1e-12)
    np.testing.assert_allclose(v[0], v2, atol=1e-13)


def test_rpmd_energy_conservation_is_second_order():
    """External harmonic wells + springs (P = 4): the drift of H_P over a fixed time scales as dt^2."""
    rng = np.random.default_rng(3)
    box = np.array([20.0, 20.0, 20.0])
    species = np.array([0, 1, 0])
    x0 = rng.uniform(5, 15, size=(3, 3))
    q0 = x0[None] + rng.normal(size=(4, 3, 3)) * 0.05
    v0 = rng.normal(size=(4, 3, 3)) * 0.02
    fn = _harmonic(x0, box, k=20.0)
    errs = []
    for dt, n in ((0.4, 50), (0.2, 100)):
        _, _, _, log = pimd.pimd(fn, q0, v0, species, box, dt, 200.0, n)
        h = np.array([r[3] for r in log])
        errs.append(np.abs(h - h[0]).max())
    assert 3.0 < errs[0] / errs[1] < 5.0


def test_time_reversal():
    rng = np.random.default_rng(4)
    box = np.array([20.0, 20.0, 20.0])
    species = np.array([1, 0])
    x0 = rng.uniform(5, 15, size=(2, 3))
    q0 = x0[None] + rng.normal(size=(3, 2, 3)) * 0.05
    v0 = rng.normal(size=(3, 2, 3)) * 0.02
    fn = _harmonic(x0, box, k=5.0)
    q1, v1, _, _ = pimd.pimd(fn, q0, v0, species, box, 0.5, 200.0, 10)
    q2, v2, _, _ = pimd.pimd(fn, q1, -v1, species, box, 0.5, 200.0, 10)
    np.testing.assert_allclose(q2, q0, atol=1e-10)
    np.testing.assert_allclose(-v2, v0, atol=1e-10)
