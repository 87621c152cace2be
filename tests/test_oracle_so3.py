"""Pins of oracle.so3 (real SH and W3j) against closed forms and invariants.

SURVEY.md §8(c) E3 and reading row 7; PAPER.md:129-130 (E(3) equivariance).
"""
import itertools
import math

import numpy as np
import pytest

from oracle import so3


def _unit(rng, n):
    v = rng.standard_normal((n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def test_sh_closed_form_on_axes():
    Y = so3.sh(np.array([[0.0, 0.0, 2.5]]), 2)[0]  # z axis, length irrelevant
    np.testing.assert_allclose(Y, [1, 0, math.sqrt(3), 0, 0, 0, math.sqrt(5), 0, 0], atol=1e-15)
    Y = so3.sh(np.array([[1.0, 0.0, 0.0]]), 2)[0]  # x axis
    np.testing.assert_allclose(
        Y, [1, 0, 0, math.sqrt(3), 0, 0, -math.sqrt(5) / 2, 0, math.sqrt(15) / 2], atol=1e-15
    )


def test_sh_component_normalised():
    rng = np.random.default_rng(0)
    Y = so3.sh(_unit(rng, 50) * 3.7, 2)
    for l in range(3):
        sl = slice(l * l, (l + 1) ** 2)
        np.testing.assert_allclose((Y[:, sl] ** 2).sum(1), 2 * l + 1, rtol=1e-14)


def test_sh_orthogonality_quadrature():
    # int Y_a Y_b dOmega / 4pi = delta_ab (component normalisation), exact
    # Gauss-Legendre x uniform-phi quadrature for degree <= 4
    xg, wg = np.polynomial.legendre.leggauss(8)
    phi = np.linspace(0, 2 * np.pi, 16, endpoint=False)
    ct, ph = np.meshgrid(xg, phi, indexing="ij")
    st = np.sqrt(1 - ct**2)
    pts = np.stack([st * np.cos(ph), st * np.sin(ph), ct], -1).reshape(-1, 3)
    w = (wg[:, None] * np.ones_like(phi)[None, :]).reshape(-1) * (2 * np.pi / 16) / (4 * np.pi)
    Y = so3.sh(pts, 2)
    G = (Y * w[:, None]).T @ Y
    np.testing.assert_allclose(G, np.eye(9), atol=1e-13)


def test_sh_grad_matches_finite_differences():
    rng = np.random.default_rng(1)
    r = rng.standard_normal((20, 3)) * 2
    g = so3.sh_grad(r, 2)
    h = 1e-6
    for a in range(3):
        e = np.zeros(3)
        e[a] = h
        fd = (so3.sh(r + e, 2) - so3.sh(r - e, 2)) / (2 * h)
        np.testing.assert_allclose(g[:, :, a], fd, atol=1e-8)


@pytest.mark.parametrize("l", [0, 1, 2])
def test_wigner_d_orthogonal_and_homomorphic(l):
    rng = np.random.default_rng(2)
    R1, R2 = so3.random_rotation(rng), so3.random_rotation(rng)
    D1, D2 = so3.wigner_d(l, R1), so3.wigner_d(l, R2)
    np.testing.assert_allclose(D1 @ D1.T, np.eye(2 * l + 1), atol=1e-13)
    np.testing.assert_allclose(so3.wigner_d(l, R1 @ R2), D1 @ D2, atol=1e-13)


TRIPLES = [t for t in itertools.product(range(3), repeat=3) if abs(t[0] - t[1]) <= t[2] <= t[0] + t[1]]


@pytest.mark.parametrize("l1,l2,l3", TRIPLES)
def test_w3j_invariant_normalised_signed(l1, l2, l3):
    W = so3.w3j(l1, l2, l3)
    assert abs(np.linalg.norm(W) - 1) < 1e-13
    rng = np.random.default_rng(3)
    for _ in range(3):
        R = so3.random_rotation(rng)
        D1, D2, D3 = (so3.wigner_d(l, R) for l in (l1, l2, l3))
        WR = np.einsum("abc,ai,bj,ck->ijk", W, D1, D2, D3)
        np.testing.assert_allclose(WR, W, atol=1e-12)
    flat = W.reshape(-1)
    assert flat[np.nonzero(np.abs(flat) > 1e-10)[0][0]] > 0


def test_w3j_closed_forms():
    np.testing.assert_allclose(so3.w3j(1, 1, 0)[:, :, 0], np.eye(3) / math.sqrt(3), atol=1e-14)
    for l in range(3):
        np.testing.assert_allclose(so3.w3j(0, l, l)[0], np.eye(2 * l + 1) / math.sqrt(2 * l + 1), atol=1e-14)
    # (1,1,1): Levi-Civita / sqrt6 in the stored (y, z, x) order
    eps = np.zeros((3, 3, 3))
    for (a, b, c), s in {(0, 1, 2): 1, (1, 2, 0): 1, (2, 0, 1): 1, (0, 2, 1): -1, (2, 1, 0): -1, (1, 0, 2): -1}.items():
        eps[a, b, c] = s
    np.testing.assert_allclose(so3.w3j(1, 1, 1), eps / math.sqrt(6), atol=1e-14)
    # (1,1,2): W[a,b,m] = +-(Hessian of P2_m / 2) / ||.||, P2 the harmonic
    # polynomials of E3; indices a,b in (y, z, x) order.
    s5, s15 = math.sqrt(5), math.sqrt(15)
    Q = np.zeros((5, 3, 3))  # in (x, y, z)
    Q[0][0, 1] = Q[0][1, 0] = s15 / 2
    Q[1][1, 2] = Q[1][2, 1] = s15 / 2
    Q[2] = np.diag([-1.0, -1.0, 2.0]) * s5 / 2
    Q[3][0, 2] = Q[3][2, 0] = s15 / 2
    Q[4] = np.diag([1.0, -1.0, 0.0]) * s15 / 2
    perm = [1, 2, 0]  # (y, z, x)
    W = np.transpose(Q[:, perm][:, :, perm], (1, 2, 0))
    W /= np.linalg.norm(W)
    W = W * np.sign(W.reshape(-1)[np.nonzero(np.abs(W.reshape(-1)) > 1e-12)[0][0]])
    np.testing.assert_allclose(so3.w3j(1, 1, 2), W, atol=1e-14)
    assert abs(so3.w3j(1, 1, 2)[0, 0, 2] - 1 / math.sqrt(30)) < 1e-14


@pytest.mark.parametrize("l1,l2,l3", [t for t in TRIPLES if sum(t) % 2 == 0])
def test_w3j_even_equals_gaunt_integral(l1, l2, l3):
    # for l1+l2+l3 even the invariant is proportional to the Gaunt integral
    # int Y^l1_a Y^l2_b Y^l3_c dOmega (exact quadrature, degree <= 6)
    xg, wg = np.polynomial.legendre.leggauss(10)
    nphi = 20
    phi = np.linspace(0, 2 * np.pi, nphi, endpoint=False)
    ct, ph = np.meshgrid(xg, phi, indexing="ij")
    st = np.sqrt(1 - ct**2)
    pts = np.stack([st * np.cos(ph), st * np.sin(ph), ct], -1).reshape(-1, 3)
    w = (wg[:, None] * np.ones(nphi)[None, :]).reshape(-1)
    Y = so3.sh(pts, 2)
    s = lambda l: slice(l * l, (l + 1) ** 2)
    G = np.einsum("p,pa,pb,pc->abc", w, Y[:, s(l1)], Y[:, s(l2)], Y[:, s(l3)])
    G /= np.linalg.norm(G)
    W = so3.w3j(l1, l2, l3)
    assert min(np.abs(G - W).max(), np.abs(G + W).max()) < 1e-12
