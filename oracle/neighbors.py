"""Image-aware full directed neighbour list (oracle; test infrastructure only).

Edge set (SURVEY.md §8(c) "Edges", readings rows 11-14):

    E = {(i, j, n) : n in Z^3, (i != j or n != 0), |r_j + n*L - r_i| <= r_c}

full and directed (Allegro's E_ij != E_ji), including several
images and self-images when L < 2 r_c (config C1).  Inclusion is decided by the
canonical fp64 formula of reading row 12 -- each operation rounded separately
(numpy never contracts to FMA):

    s = fl(n*L); x' = fl(x_j + s); delta = fl(x' - x_i);
    d2 = fl(fl(fl(dx^2) + fl(dy^2)) + fl(dz^2));  include iff d2 <= fl(r_c^2)

Two independent enumerations: ``brute_force`` (all pairs x all shifts, PAPER.md
has none -- SPEC.md:64/112's brute-force pin) and ``cell_list`` (the paper's
linked-list cell decomposition, §2.4).  Both return
(i, j, n) sorted lexicographically by (i, j, nx, ny, nz) -- the canonical row
order of reading row 13.
"""
from __future__ import annotations

import itertools
import math

import numpy as np


def wrap(pos: np.ndarray, box: np.ndarray) -> np.ndarray:
    """x <- x - L*floor(x/L); x == L -> 0 (reading row 17)."""
    out = pos - box * np.floor(pos / box)
    return np.where(out >= box, 0.0, out)


def canonical_d2(xi: np.ndarray, xj: np.ndarray, shift: np.ndarray, box: np.ndarray) -> np.ndarray:
    """Reading row 12, elementwise over broadcast arrays [..., 3]."""
    s = shift * box
    xp = xj + s
    d = xp - xi
    sq = d * d
    return (sq[..., 0] + sq[..., 1]) + sq[..., 2]


def _sort_edges(i, j, n):
    order = np.lexsort((n[:, 2], n[:, 1], n[:, 0], j, i))
    return i[order].astype(np.int64), j[order].astype(np.int64), n[order].astype(np.int64)


def max_shift(box: np.ndarray, r_cut: float) -> np.ndarray:
    """|n_alpha| <= ceil(r_c / L_alpha) + 1 covers every image within r_c."""
    return np.array([int(math.ceil(r_cut / L)) + 1 for L in box], dtype=np.int64)


def brute_force(pos: np.ndarray, box: np.ndarray, r_cut: float):
    """O(N^2 * images) enumeration; pos must already be wrapped."""
    n_atoms = pos.shape[0]
    m = max_shift(box, r_cut)
    shifts = np.array(
        list(itertools.product(*[range(-int(k), int(k) + 1) for k in m])), dtype=np.float64
    )  # [S, 3]
    rc2 = r_cut * r_cut
    I, J, N = [], [], []
    for i in range(n_atoms):
        # [N, S]
        d2 = canonical_d2(pos[i][None, None, :], pos[:, None, :], shifts[None, :, :], box)
        mask = d2 <= rc2
        zero = np.all(shifts == 0, axis=1)
        mask[i, zero] = False
        jj, ss = np.nonzero(mask)
        I.append(np.full(jj.shape, i))
        J.append(jj)
        N.append(shifts[ss])
    if not I:
        return np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros((0, 3), np.int64)
    return _sort_edges(np.concatenate(I), np.concatenate(J), np.concatenate(N).astype(np.int64))


def cell_list(pos: np.ndarray, box: np.ndarray, r_cut: float, centers=None):
    """Linked-cell search: periodic images within r_c of the box
    become ghosts; ghosts and atoms are binned into cells of edge >= r_c; each
    atom scans its 27 neighbouring cells.  pos must already be wrapped.
    ``centers``: optional subset of centre atoms whose rows are wanted."""
    n_atoms = pos.shape[0]
    m = max_shift(box, r_cut)
    margin = 1e-9 * max(1.0, float(np.max(box)))
    # ghosts: every image whose position lies within r_c (+margin) of the box
    gp, gj, gn = [pos], [np.arange(n_atoms)], [np.zeros((n_atoms, 3))]
    for shift in itertools.product(*[range(-int(k), int(k) + 1) for k in m]):
        if shift == (0, 0, 0):
            continue
        sh = np.array(shift, dtype=np.float64)
        xp = pos + sh * box
        inside = np.all((xp >= -r_cut - margin) & (xp < box + r_cut + margin), axis=1)
        idx = np.nonzero(inside)[0]
        gp.append(xp[idx])
        gj.append(idx)
        gn.append(np.tile(sh, (idx.size, 1)))
    gp = np.concatenate(gp)
    gj = np.concatenate(gj)
    gn = np.concatenate(gn)
    # cells over the extended region [-r_c - margin, L + r_c + margin)
    lo = -r_cut - margin
    ext = box + 2 * (r_cut + margin)
    ncell = np.maximum(1, np.floor(ext / r_cut).astype(np.int64))
    csize = ext / ncell
    cidx = np.clip(np.floor((gp - lo) / csize).astype(np.int64), 0, ncell - 1)
    lin = (cidx[:, 2] * ncell[1] + cidx[:, 1]) * ncell[0] + cidx[:, 0]
    order = np.argsort(lin, kind="stable")
    lin_sorted = lin[order]
    rc2 = r_cut * r_cut
    I, J, N = [], [], []
    it = range(n_atoms) if centers is None else np.asarray(centers)
    for i in it:
        ci = cidx[i]
        cand = []
        for d in itertools.product((-1, 0, 1), repeat=3):
            c = ci + np.array(d)
            if np.any(c < 0) or np.any(c >= ncell):
                continue
            key = (c[2] * ncell[1] + c[1]) * ncell[0] + c[0]
            a, b = np.searchsorted(lin_sorted, [key, key + 1])
            cand.append(order[a:b])
        cand = np.concatenate(cand) if cand else np.zeros(0, np.int64)
        if cand.size == 0:
            continue
        d2 = canonical_d2(pos[i][None, :], pos[gj[cand]], gn[cand], box)
        keep = d2 <= rc2
        self_img = (gj[cand] == i) & np.all(gn[cand] == 0, axis=1)
        keep &= ~self_img
        sel = cand[keep]
        I.append(np.full(sel.shape, i))
        J.append(gj[sel])
        N.append(gn[sel])
    if not I:
        return np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros((0, 3), np.int64)
    return _sort_edges(np.concatenate(I), np.concatenate(J), np.concatenate(N).astype(np.int64))


def edge_vectors(pos: np.ndarray, box: np.ndarray, i, j, n) -> np.ndarray:
    """r_e = (r_j + n*L) - r_i in fp64, rounded in the canonical order."""
    xp = pos[j] + n * box
    return xp - pos[i]
