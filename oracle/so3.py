"""Real spherical harmonics and real Wigner-3j tables (oracle; test infrastructure only).

PAPER.md:129-130 (§2.1): Allegro's energy terms are E(3)-equivariant, built
from "tensors up to rank l and tensor products using their irreducible
representations".  The concrete basis is a reading (SURVEY.md §8(c) E3 and
reading row 7):

* component-normalised real SH (sum_m (Y^l_m)^2 = 2l+1), m = -l..l:
    Y^0 = 1
    Y^1 = sqrt3 (y, z, x)
    Y^2 = (sqrt15 xy, sqrt15 yz, sqrt5/2 (3z^2 - 1), sqrt15 xz, sqrt15/2 (x^2 - y^2))
  of the unit vector r_hat.  Written as Y^l = P_l(r)/|r|^l with P_l a harmonic
  polynomial, the gradient is dY/dr = grad P / d^l - l P r / d^(l+2).
* W3j^{l1 l2 l3}: the rotation-invariant tensor of Y^l1 (x) Y^l2 (x) Y^l3 --
  computed here by its *definition*: the common null vector of
  (D^l1(R) (x) D^l2(R) (x) D^l3(R) - I) over random rotations R, where D^l(R)
  is the matrix with Y^l(R r) = D^l(R) Y^l(r) (fitted by least squares on
  sample points).  Frobenius norm 1; global sign such that the first entry
  with |w| > 1e-10 in (m1, m2, m3) lexicographic order is positive.
"""
from __future__ import annotations

import functools
import math

import numpy as np

S3 = math.sqrt(3.0)
S5 = math.sqrt(5.0)
S15 = math.sqrt(15.0)


def sh_dim(lmax: int) -> int:
    return (lmax + 1) ** 2


def _poly(r: np.ndarray, l: int) -> np.ndarray:
    x, y, z = r[..., 0], r[..., 1], r[..., 2]
    if l == 0:
        return np.ones(r.shape[:-1] + (1,))
    if l == 1:
        return S3 * np.stack([y, z, x], axis=-1)
    if l == 2:
        return np.stack(
            [
                S15 * x * y,
                S15 * y * z,
                0.5 * S5 * (2 * z * z - x * x - y * y),
                S15 * x * z,
                0.5 * S15 * (x * x - y * y),
            ],
            axis=-1,
        )
    raise ValueError("l <= 2 only")


def _poly_grad(r: np.ndarray, l: int) -> np.ndarray:
    """d P_l[m] / d r_alpha  -> [..., 2l+1, 3]."""
    x, y, z = r[..., 0], r[..., 1], r[..., 2]
    zero = np.zeros_like(x)
    one = np.ones_like(x)
    if l == 0:
        return np.zeros(r.shape[:-1] + (1, 3))
    if l == 1:
        return S3 * np.stack(
            [np.stack([zero, one, zero], -1), np.stack([zero, zero, one], -1), np.stack([one, zero, zero], -1)],
            axis=-2,
        )
    if l == 2:
        rows = [
            S15 * np.stack([y, x, zero], -1),
            S15 * np.stack([zero, z, y], -1),
            0.5 * S5 * np.stack([-2 * x, -2 * y, 4 * z], -1),
            S15 * np.stack([z, zero, x], -1),
            0.5 * S15 * np.stack([2 * x, -2 * y, zero], -1),
        ]
        return np.stack(rows, axis=-2)
    raise ValueError("l <= 2 only")


def sh(r: np.ndarray, lmax: int) -> np.ndarray:
    """Y^l_m(r_hat) for l <= lmax, concatenated l-major -> [..., (lmax+1)^2]."""
    d = np.linalg.norm(r, axis=-1, keepdims=True)
    return np.concatenate([_poly(r, l) / d**l for l in range(lmax + 1)], axis=-1)


def sh_grad(r: np.ndarray, lmax: int) -> np.ndarray:
    """dY/dr (w.r.t. the un-normalised vector r) -> [..., (lmax+1)^2, 3]."""
    d = np.linalg.norm(r, axis=-1)
    out = []
    for l in range(lmax + 1):
        P = _poly(r, l)
        gP = _poly_grad(r, l)
        dl = d[..., None, None] ** l
        term2 = l * P[..., :, None] * r[..., None, :] / (d[..., None, None] ** (l + 2))
        out.append(gP / dl - term2)
    return np.concatenate(out, axis=-2)


def random_rotation(rng: np.random.Generator) -> np.ndarray:
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array(
        [
            [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
            [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
            [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
        ]
    )


def wigner_d(l: int, R: np.ndarray, n_samples: int = 64, seed: int = 1234) -> np.ndarray:
    """D^l(R) with Y^l(R r) = D^l(R) Y^l(r): least squares over sample points."""
    rng = np.random.default_rng(seed)
    pts = rng.standard_normal((n_samples, 3))
    pts /= np.linalg.norm(pts, axis=1, keepdims=True)
    A = _poly(pts, l)  # Y(r)   [S, 2l+1]
    B = _poly(pts @ R.T, l)  # Y(Rr)  [S, 2l+1]
    # B = A D^T  ->  D^T = lstsq(A, B)
    Dt, *_ = np.linalg.lstsq(A, B, rcond=None)
    return Dt.T


@functools.lru_cache(maxsize=None)
def w3j(l1: int, l2: int, l3: int) -> np.ndarray:
    """Real Wigner-3j tensor [2l1+1, 2l2+1, 2l3+1] (see module docstring)."""
    if not (abs(l1 - l2) <= l3 <= l1 + l2):
        raise ValueError("triangle rule violated")
    rng = np.random.default_rng(20230314)
    dims = (2 * l1 + 1, 2 * l2 + 1, 2 * l3 + 1)
    n = dims[0] * dims[1] * dims[2]
    blocks = []
    for _ in range(4):
        R = random_rotation(rng)
        K = np.kron(np.kron(wigner_d(l1, R), wigner_d(l2, R)), wigner_d(l3, R))
        blocks.append(K - np.eye(n))
    A = np.concatenate(blocks, axis=0)
    _, sv, vt = np.linalg.svd(A)
    if n > 1 and sv[-2] < 1e-6:
        raise RuntimeError("invariant subspace is not one-dimensional")
    if sv[-1] > 1e-9:
        raise RuntimeError("no invariant tensor found")
    w = vt[-1].reshape(dims)
    w /= np.linalg.norm(w)
    flat = w.reshape(-1)
    first = flat[np.nonzero(np.abs(flat) > 1e-10)[0][0]]
    if first < 0:
        w = -w
    w[np.abs(w) < 1e-14] = 0.0
    return w
