"""Spatial domain decomposition of the force evaluation (oracle; test infrastructure only).

PAPER.md:187-191 (§2.4): globally scalable spatial decomposition with minimal
inter-domain exchange; SURVEY.md §8(e) gives the rules written out here:

* grid (px, py, pz); domain d owns the atoms whose wrapped coordinate lies in
  (c w, (c+1) w] per axis (w = L/p) -- an atom on an internal face belongs to the
  lower-index domain: owner = clamp(ceil(x/w) - 1, 0, p-1);
* the halo is built in three stages (x, y, z): in stage alpha every domain sends to
  its -alpha neighbour the local atoms (owned + ghosts of earlier stages) with
  x_alpha < lo + r_c and to its +alpha neighbour those with x_alpha >= hi - r_c,
  shifting the coordinate by +L / -L when the message wraps around the box
  (fl(x + fl(+-1 * L)), the canonical image of reading row 12);
* each domain evaluates the rows of its owned centres over its owned + ghost atoms;
  forces on ghosts are returned to their owners (ghost-force return).

The functions are written per domain (``stage_messages``, ``domain_rows``) so the
serial driver below and the multi-process gloo test share the same rules.
"""
from __future__ import annotations

import itertools
import math

import numpy as np

from . import allegro, neighbors


def grid_coords(rank: int, grid):
    px, py, _ = grid
    return np.array([rank % px, (rank // px) % py, rank // (px * py)])


def rank_of(coord, grid):
    px, py, _ = grid
    return int(coord[0] + px * (coord[1] + py * coord[2]))


def owner_coords(pos: np.ndarray, box: np.ndarray, grid) -> np.ndarray:
    w = box / np.asarray(grid)
    return np.clip(np.ceil(pos / w) - 1, 0, np.asarray(grid) - 1).astype(np.int64)


def domain_bounds(coord, box, grid):
    w = box / np.asarray(grid)
    lo = coord * w
    hi = np.where(coord == np.asarray(grid) - 1, box, (coord + 1) * w)
    return lo, hi


def stage_messages(local, axis, coord, box, grid, r_cut):
    """Messages of one halo stage from a domain's local atoms.

    local: dict(gid [n], species [n], pos [n,3], shift [n,3]); returns
    (to_minus, to_plus) with the same keys (copies, shifted when wrapping)."""
    lo, hi = domain_bounds(coord, box, grid)
    rc = r_cut * (1 + 1e-9) + 1e-9
    x = local["pos"][:, axis]
    out = []
    for sel, wrap, sgn in ((x < lo[axis] + rc, coord[axis] == 0, +1),
                           (x >= hi[axis] - rc, coord[axis] == grid[axis] - 1, -1)):
        idx = np.nonzero(sel)[0]
        msg = {k: v[idx].copy() for k, v in local.items()}
        if wrap:
            msg["pos"][:, axis] = msg["pos"][:, axis] + sgn * box[axis]
            msg["shift"][:, axis] += sgn
        msg["src"] = idx
        out.append(msg)
    return out


def neighbour_ranks(coord, axis, grid):
    lo = coord.copy()
    hi = coord.copy()
    lo[axis] = (coord[axis] - 1) % grid[axis]
    hi[axis] = (coord[axis] + 1) % grid[axis]
    return rank_of(lo, grid), rank_of(hi, grid)


def append(local, msg):
    return {k: np.concatenate([local[k], msg[k]]) for k in local}


def domain_rows(model, local, n_owned, r_cut):
    """Rows of the owned centres over the local atoms (no periodicity: ghosts carry
    their image shift).  Returns (e_atom [n_owned], edges (i, j, n) local, g [E,3])."""
    pos = local["pos"]
    rc2 = r_cut * r_cut
    I, J = [], []
    for i in range(n_owned):
        d = pos - pos[i]
        sq = d * d
        d2 = (sq[:, 0] + sq[:, 1]) + sq[:, 2]
        nb = np.nonzero(d2 <= rc2)[0]
        nb = nb[nb != i]
        # canonical row order (gid_j, shift)
        key = np.lexsort((local["shift"][nb, 2], local["shift"][nb, 1], local["shift"][nb, 0], local["gid"][nb]))
        nb = nb[key]
        I.append(np.full(nb.shape, i))
        J.append(nb)
    ei = np.concatenate(I) if I else np.zeros(0, np.int64)
    ej = np.concatenate(J) if J else np.zeros(0, np.int64)
    rvec = pos[ej] - pos[ei]
    spc = local["species"]
    e_loc, _, g = allegro._rows(model, rvec, spc[ei], spc[ej], ei, n_owned, spc[:n_owned])
    return e_loc + model.mu[spc[:n_owned]], (ei, ej), g


def decomposed_energy_forces(model, pos, species, box, grid):
    """Serial driver: all domains of ``grid`` in one process (SURVEY.md §4 "oracle
    runs P virtual domains").  Returns (energy, e_atom [N], forces [N,3], n_ghosts)."""
    box = np.asarray(box, dtype=np.float64)
    pos = neighbors.wrap(np.asarray(pos, dtype=np.float64), box)
    species = np.asarray(species)
    grid = tuple(int(g) for g in grid)
    P = int(np.prod(grid))
    own = owner_coords(pos, box, grid)
    locs, n_own = [], []
    for r in range(P):
        c = grid_coords(r, grid)
        idx = np.nonzero(np.all(own == c, axis=1))[0]
        locs.append(dict(gid=idx.astype(np.int64), species=species[idx], pos=pos[idx].copy(),
                         shift=np.zeros((idx.size, 3), np.int64)))
        n_own.append(idx.size)
    for axis in range(3):
        msgs = [stage_messages(locs[r], axis, grid_coords(r, grid), box, grid, model.r_max) for r in range(P)]
        new = []
        for r in range(P):
            rm, rp = neighbour_ranks(grid_coords(r, grid), axis, grid)
            # from the -neighbour: its "+" message; from the +neighbour: its "-" message
            loc = append(locs[r], {k: v for k, v in msgs[rm][1].items() if k != "src"})
            loc = append(loc, {k: v for k, v in msgs[rp][0].items() if k != "src"})
            new.append(loc)
        locs = new
    N = pos.shape[0]
    e_atom = np.zeros(N)
    forces = np.zeros((N, 3))
    n_ghosts = 0
    for r in range(P):
        loc = locs[r]
        n_ghosts += loc["gid"].size - n_own[r]
        e_loc, (ei, ej), g = domain_rows(model, loc, n_own[r], model.r_max)
        e_atom[loc["gid"][: n_own[r]]] = e_loc
        np.add.at(forces, loc["gid"][ei], g)
        np.add.at(forces, loc["gid"][ej], -g)  # ghosts: returned to their owners
    return float(e_atom.sum()), e_atom, forces, n_ghosts
