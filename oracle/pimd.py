"""Ring-polymer path-integral MD (oracle; test infrastructure only).

PAPER.md:419-429 (§5) runs PIMD "where each atom has 32 replicas that are harmonically coupled
together" and notes that "the major cost is computing the energy and forces for the atoms
within each replica".  The paper names no integrator; reading D25 -- ring-polymer
MD with

    H_P = sum_j [ sum_i m_i |v_ij|^2 / (2 kappa) + V(q_j) ] + sum_i sum_j m_i w_P^2 |q_ij - q_i,j+1|^2 / (2 kappa),
    w_P = P k_B T / hbar   (beads at temperature P T; j + 1 taken mod P),

integrated per step as: v += (dt/2) kappa F/m; exact free ring-polymer evolution over dt in the
normal modes of the ring; F_j = -grad V(q_j) for every bead; v += (dt/2) kappa F/m.  The normal
modes are the real orthonormal eigenvectors of the cyclic ring (C[j][k], j = bead, k = mode):

    C[j][0] = 1/sqrt(P);  C[j][k] = sqrt(2/P) cos(2 pi j k / P), 1 <= k < P/2;
    C[j][P/2] = (-1)^j / sqrt(P) (P even);  C[j][k] = sqrt(2/P) sin(2 pi j k / P), k > P/2,

with frequencies w_k = 2 w_P sin(k pi / P); mode k evolves as a harmonic oscillator
(k = 0, the centroid, as a free particle).  Units: A, fs, amu, eV; kappa as oracle/md.py.
"""
from __future__ import annotations

import numpy as np

from . import md
from .neighbors import wrap

HBAR = 0.6582119569  # eV fs


def normal_mode_matrix(P: int) -> np.ndarray:
    C = np.zeros((P, P))
    for j in range(P):
        for k in range(P):
            if k == 0:
                C[j, k] = 1.0 / np.sqrt(P)
            elif 2 * k < P:
                C[j, k] = np.sqrt(2.0 / P) * np.cos(2 * np.pi * j * k / P)
            elif 2 * k == P:
                C[j, k] = (-1.0) ** j / np.sqrt(P)
            else:
                C[j, k] = np.sqrt(2.0 / P) * np.sin(2 * np.pi * j * k / P)
    return C


def omega_p(P: int, T: float) -> float:
    return P * md.KB * T / HBAR


def mode_frequencies(P: int, wp: float) -> np.ndarray:
    return np.array([2.0 * wp * np.sin(k * np.pi / P) for k in range(P)])


def free_ring_step(q, v, wp, dt):
    """Exact evolution of the free ring polymer (springs only) over dt; q, v [P][N][3]."""
    P = q.shape[0]
    C = normal_mode_matrix(P)
    w = mode_frequencies(P, wp)
    xq = np.einsum("jk,jnd->knd", C, q)
    xv = np.einsum("jk,jnd->knd", C, v)
    nq, nv = np.empty_like(xq), np.empty_like(xv)
    for k in range(P):
        if k == 0:
            nq[k] = xq[k] + xv[k] * dt
            nv[k] = xv[k]
        else:
            c, s = np.cos(w[k] * dt), np.sin(w[k] * dt)
            nq[k] = xq[k] * c + xv[k] * s / w[k]
            nv[k] = -xq[k] * w[k] * s + xv[k] * c
    return np.einsum("jk,knd->jnd", C, nq), np.einsum("jk,knd->jnd", C, nv)


def spring_energy(q, species, wp) -> float:
    m = md.masses(species)
    d = q - np.roll(q, -1, axis=0)  # q_j - q_{j+1}
    return float(0.5 * wp * wp * np.sum(m[None, :, None] * d * d) / md.KAPPA)


def batch_forces(force_fn, q, box):
    """Every bead evaluated on its own (wrapped) copy: force_fn(pos) -> (energy, forces)."""
    es, fs = [], []
    for j in range(q.shape[0]):
        e, f = force_fn(wrap(q[j], box))
        es.append(e)
        fs.append(f)
    return np.array(es), np.array(fs)


def pimd(force_fn, q, v, species, box, dt, T, n_steps, forces=None):
    """n_steps of ring-polymer MD.  q, v [P][N][3] (q unwrapped).  Returns (q, v, forces,
    [(V_sum, K, E_spring, H)] per step)."""
    box = np.asarray(box, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64).copy()
    v = np.asarray(v, dtype=np.float64).copy()
    P = q.shape[0]
    wp = omega_p(P, T)
    m = md.masses(species)[None, :, None]
    if forces is None:
        _, forces = batch_forces(force_fn, q, box)
    log = []
    for _ in range(n_steps):
        v = v + 0.5 * dt * md.KAPPA * forces / m
        q, v = free_ring_step(q, v, wp, dt)
        es, forces = batch_forces(force_fn, q, box)
        v = v + 0.5 * dt * md.KAPPA * forces / m
        K = float(0.5 * np.sum(m * v * v) / md.KAPPA)
        Es = spring_energy(q, species, wp)
        log.append((float(es.sum()), K, Es, float(es.sum()) + K + Es))
    return q, v, forces, log
