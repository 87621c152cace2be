"""Velocity Verlet, kinetic energy and 5-sigma force outliers (oracle; test infrastructure only).

* Eq. 1 (§2.1): m_i d^2 r_i/dt^2 = f_i = -dE/dr_i.
* NVE "simply integrating the equations of motion" with dt = 2 fs
  (§3.2), as velocity Verlet exactly as SPEC.md:77:
      v <- v + (dt/2) kappa F/m;  r <- wrap(r + dt v);  F <- F(r);  v <- v + (dt/2) kappa F/m
  with kappa = 9.648533e-3 A fs^-2 per (eV A^-1 amu^-1); KE = 1/2 sum m v^2 / kappa (eV).
* NVT thermalisation (§3.2: "thermalized at a temperature of 200 K
  using NVT ensemble"): one Nose-Hoover thermostat variable xi (no chain --
  the paper names none), integrated by a symmetric Trotter split around the velocity-Verlet
  core (reading D23 in DESIGN.md):
      half(dt/2):  xi += (dt/4) G;  v *= exp(-xi dt/2);  eta += xi dt/2;  xi += (dt/4) G,
      G = (2 K - g k_B T) / Q,  g = 3N,  Q = g k_B T tau^2
  step: half; Verlet core; half.  Conserved: H' = E + K + Q xi^2 / 2 + g k_B T eta.
* 5-sigma outliers: "unphysically large force values (over 5 sigma)"
  (Fig. 1 caption): #{a : |F_a| > mean + k sigma}, strict
  inequality, mean/sigma = mean and population std of |F_a|
  over all atoms at step 0 (reading row 18).
"""
from __future__ import annotations

import numpy as np

from .neighbors import wrap

KAPPA = 9.648533e-3
KB = 8.617333e-5  # eV/K
MASS_H = 1.008
MASS_N = 14.007


def masses(species) -> np.ndarray:
    species = np.asarray(species)
    return np.where(species == 1, MASS_N, MASS_H).astype(np.float64)


def kinetic_energy(vel, species) -> float:
    m = masses(species)
    return float(0.5 * np.sum(m[:, None] * vel * vel) / KAPPA)


def temperature(vel, species) -> float:
    n = np.asarray(species).shape[0]
    return 2.0 * kinetic_energy(vel, species) / (3.0 * n * KB)


def verlet(force_fn, pos, vel, species, box, dt, n_steps, forces=None):
    """n_steps of velocity Verlet; force_fn(pos) -> (energy, forces).

    Exactly one force evaluation per step (forces cached).
    Returns (pos, vel, forces, [(e_pot, e_kin)] per step)."""
    box = np.asarray(box, dtype=np.float64)
    m = masses(species)[:, None]
    pos = wrap(np.asarray(pos, dtype=np.float64), box)
    vel = np.asarray(vel, dtype=np.float64).copy()
    if forces is None:
        _, forces = force_fn(pos)
    log = []
    for _ in range(n_steps):
        vel = vel + 0.5 * dt * KAPPA * forces / m
        pos = wrap(pos + dt * vel, box)
        e_pot, forces = force_fn(pos)
        vel = vel + 0.5 * dt * KAPPA * forces / m
        log.append((e_pot, kinetic_energy(vel, species)))
    return pos, vel, forces, log


def nvt_half(vel, species, K, xi, eta, dt, T, Q):
    """Thermostat propagation over dt/2 (see module docstring)."""
    g = 3 * len(species)
    kT = KB * T
    xi = xi + 0.25 * dt * (2.0 * K - g * kT) / Q
    s = np.exp(-xi * 0.5 * dt)
    vel = vel * s
    K = K * s * s
    eta = eta + xi * 0.5 * dt
    xi = xi + 0.25 * dt * (2.0 * K - g * kT) / Q
    return vel, K, xi, eta


def nvt_verlet(force_fn, pos, vel, species, box, dt, n_steps, T, tau, forces=None, xi=0.0, eta=0.0):
    """n_steps of Nose-Hoover NVT (one thermostat); tau in fs, Q = 3N k_B T tau^2.

    Returns (pos, vel, forces, xi, eta, [(e_pot, e_kin, conserved)] per step)."""
    box = np.asarray(box, dtype=np.float64)
    m = masses(species)[:, None]
    pos = wrap(np.asarray(pos, dtype=np.float64), box)
    vel = np.asarray(vel, dtype=np.float64).copy()
    g = 3 * len(species)
    Q = g * KB * T * tau * tau
    if forces is None:
        _, forces = force_fn(pos)
    log = []
    for _ in range(n_steps):
        K = kinetic_energy(vel, species)
        vel, K, xi, eta = nvt_half(vel, species, K, xi, eta, dt, T, Q)
        vel = vel + 0.5 * dt * KAPPA * forces / m
        pos = wrap(pos + dt * vel, box)
        e_pot, forces = force_fn(pos)
        vel = vel + 0.5 * dt * KAPPA * forces / m
        K = kinetic_energy(vel, species)
        vel, K, xi, eta = nvt_half(vel, species, K, xi, eta, dt, T, Q)
        conserved = e_pot + K + 0.5 * Q * xi * xi + g * KB * T * eta
        log.append((e_pot, K, conserved))
    return pos, vel, forces, xi, eta, log


def force_baseline(forces):
    """(mean, population std) of |F_a| (reading row 18)."""
    norms = np.linalg.norm(np.asarray(forces, dtype=np.float64), axis=1)
    return float(norms.mean()), float(norms.std())


def count_outliers(forces, mean, sigma, k=5.0) -> int:
    """#{a : |F_a| > mean + k*sigma}, strict."""
    norms = np.linalg.norm(np.asarray(forces, dtype=np.float64), axis=1)
    return int(np.sum(norms > mean + k * sigma))
