"""Seeded liquid-NH3 boxes shaped like the paper's ammonia runs.

Recipe (SURVEY.md §8(d) "Synthetic inputs", readings §8(c) rows 8, 17, 19):

* density 0.73 g/cm^3 -> rho_mol = 0.025813 molecules/A^3 (0.10325 atoms/A^3);
  the paper does not state its density; liquid NH3 near 200 K (PAPER.md:217,
  §3.2) is ~0.73 g/cm^3.
* rigid NH3: N-H 1.012 A, angle HNH 106.7 deg, body frame below.
* molecular centres (the N atom) on sc / bcc / fcc lattice sites of edge
  a = (sites / rho_mol)^(1/3); each molecule gets a Haar-random orientation from
  a normalised 4-D Gaussian quaternion drawn from ``default_rng(structure_seed)``,
  one draw per molecule in molecule order.
* atom order is molecule-major, gid = 4*mol + {0: N, 1..3: H}; molecules are
  numbered over lattice cells with x fastest, then y, then z, and the sites of a
  cell innermost.  Species: H = 0, N = 1 (atomic number ascending).
* positions wrapped into [0, L) per axis.
* velocities: Maxwell-Boltzmann at T (200 K) from
  ``default_rng(velocity_seed)``, centre-of-mass momentum removed.

No arithmetic of the method lives here.
"""
from __future__ import annotations

import dataclasses

import numpy as np

RHO_MOL = 0.025813  # molecules / A^3  (0.73 g/cm^3 / 17.031 g/mol * N_A)
SPECIES_H = 0
SPECIES_N = 1
MASS = {SPECIES_H: 1.008, SPECIES_N: 14.007}  # amu
KB_EV = 8.617333e-5  # eV / K
KAPPA = 9.648533e-3  # A fs^-2 per (eV A^-1 amu^-1)

# Body frame (A): N at the origin, three H at N-H = 1.012 A, HNH = 106.7 deg.
BODY = np.array(
    [
        [0.0, 0.0, 0.0],
        [0.93753, 0.0, -0.38103],
        [-0.46876, 0.81192, -0.38103],
        [-0.46876, -0.81192, -0.38103],
    ],
    dtype=np.float64,
)
BODY_SPECIES = np.array([SPECIES_N, SPECIES_H, SPECIES_H, SPECIES_H], dtype=np.int32)

LATTICE_SITES = {
    "sc": np.array([[0.0, 0.0, 0.0]]),
    "bcc": np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.5]]),
    "fcc": np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.0], [0.5, 0.0, 0.5], [0.0, 0.5, 0.5]]),
}


@dataclasses.dataclass
class System:
    """A periodic orthorhombic box of atoms (host arrays, fp64 state)."""

    pos: np.ndarray  # [N, 3] float64, A, wrapped into [0, L)
    species: np.ndarray  # [N] int32 (0 = H, 1 = N)
    box: np.ndarray  # [3] float64, A
    gid: np.ndarray  # [N] int32 global ids
    vel: np.ndarray | None = None  # [N, 3] float64, A/fs

    @property
    def n(self) -> int:
        return int(self.pos.shape[0])

    def masses(self) -> np.ndarray:
        return np.where(self.species == SPECIES_N, MASS[SPECIES_N], MASS[SPECIES_H])

    def copy(self) -> "System":
        return System(
            self.pos.copy(),
            self.species.copy(),
            self.box.copy(),
            self.gid.copy(),
            None if self.vel is None else self.vel.copy(),
        )


def lattice_constant(lattice: str) -> float:
    return (len(LATTICE_SITES[lattice]) / RHO_MOL) ** (1.0 / 3.0)


def _quat_to_matrix(q: np.ndarray) -> np.ndarray:
    w, x, y, z = q
    return np.array(
        [
            [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
            [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
            [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
        ]
    )


def wrap_positions(pos: np.ndarray, box: np.ndarray) -> np.ndarray:
    """x <- x - L*floor(x/L); x == L -> 0."""
    out = pos - box * np.floor(pos / box)
    out = np.where(out >= box, 0.0, out)
    return out


def nh3_box(lattice: str, cells, structure_seed: int = 1) -> System:
    """Liquid-NH3-density box of ``cells = (cx, cy, cz)`` lattice cells."""
    cx, cy, cz = (int(c) for c in cells)
    a = lattice_constant(lattice)
    sites = LATTICE_SITES[lattice]
    box = np.array([cx * a, cy * a, cz * a], dtype=np.float64)
    centres = []
    for iz in range(cz):
        for iy in range(cy):
            for ix in range(cx):
                for s in sites:
                    centres.append((np.array([ix, iy, iz], dtype=np.float64) + s) * a)
    centres = np.asarray(centres)
    n_mol = centres.shape[0]
    rng = np.random.default_rng(structure_seed)
    quats = rng.standard_normal((n_mol, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    pos = np.empty((n_mol * 4, 3))
    for m in range(n_mol):
        rot = _quat_to_matrix(quats[m])
        pos[4 * m : 4 * m + 4] = centres[m] + BODY @ rot.T
    pos = wrap_positions(pos, box)
    species = np.tile(BODY_SPECIES, n_mol).astype(np.int32)
    gid = np.arange(n_mol * 4, dtype=np.int32)
    return System(pos, species, box, gid)


def maxwell_boltzmann(system: System, temperature: float = 200.0, velocity_seed: int = 2) -> System:
    """Attach MB velocities at ``temperature`` (K) with zero total momentum."""
    rng = np.random.default_rng(velocity_seed)
    m = system.masses()
    std = np.sqrt(KB_EV * temperature * KAPPA / m)
    vel = rng.standard_normal((system.n, 3)) * std[:, None]
    p = (m[:, None] * vel).sum(axis=0)
    vel -= p / m.sum()
    out = system.copy()
    out.vel = vel
    return out


def replicate(system: System, reps) -> System:
    """Periodic replica of ``system`` tiled ``reps = (rx, ry, rz)`` times.

    Copy index runs x fastest; gid = copy * N + gid (C5's
    P-GPU box is a periodic replica of the P = 1 box)."""
    rx, ry, rz = (int(r) for r in reps)
    n = system.n
    pos, spc, gid, vel = [], [], [], []
    c = 0
    for iz in range(rz):
        for iy in range(ry):
            for ix in range(rx):
                pos.append(system.pos + system.box * np.array([ix, iy, iz], dtype=np.float64))
                spc.append(system.species)
                gid.append(system.gid + c * n)
                if system.vel is not None:
                    vel.append(system.vel)
                c += 1
    box = system.box * np.array([rx, ry, rz], dtype=np.float64)
    return System(
        np.concatenate(pos),
        np.concatenate(spc).astype(np.int32),
        box,
        np.concatenate(gid).astype(np.int32),
        np.concatenate(vel) if vel else None,
    )


def random_box(n: int, box, seed: int, species_frac_n: float = 0.25, min_dist: float = 0.0) -> System:
    """Uniform random atoms (test fixtures for the neighbour pins)."""
    rng = np.random.default_rng(seed)
    box = np.asarray(box, dtype=np.float64)
    pos = rng.random((n, 3)) * box
    species = (rng.random(n) < species_frac_n).astype(np.int32)
    return System(wrap_positions(pos, box), species, box, np.arange(n, dtype=np.int32))
