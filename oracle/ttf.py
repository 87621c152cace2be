"""Time-to-failure protocol and the fidelity-scaling fit (oracle; test infrastructure only).

* Protocol (§3.2): "thermalized at a temperature of 200 K using NVT
  ensemble for 1,000 steps.  We subsequently switch the ensemble to NVE and continue the
  simulation until it fails to determine t_failure", dt = 2 fs.
* "Fails" is not defined by the paper; the criteria are SPEC.md:459's (reading D24):
  non_finite (any position / velocity / force / energy), displacement_blowup (some atom
  drifts more than disp_max in one step: |dt v_half| > disp_max) and energy_drift
  (|E - E0| > drift_tol |E0|, E = E_pot + E_kin, checked every check_interval NVE steps, E0 at
  the start of NVE).  Outlier counts (Fig. 1) are recorded every
  outlier_interval steps against the force-norm mean / population std at NVE start and never
  trigger a failure.
* Fit (Eq. 4): t_failure = alpha N^(-beta); per N the mean of the
  uncensored failing steps (t_failure = the NVE step at which the
  failure is detected, so a failure in the first step is t = 1); ordinary least squares of ln t on ln N written out as sums
  (SPEC.md:474-476): slope = -beta, intercept = ln alpha, beta_stderr from the residual
  variance.
"""
from __future__ import annotations

import math

import numpy as np

from . import md
from .neighbors import wrap

CENSORED, NON_FINITE, DISPLACEMENT, ENERGY_DRIFT = 0, 1, 2, 3


class FitError(ValueError):
    pass


def detect_failure(pos, vel, forces, e_total, e0, step, check_interval, drift_tol, max_disp_step, disp_max):
    """The failure classifier of one NVE step (see module docstring).  max_disp_step is the
    largest single-atom drift |dt v_half| of this step.  Returns one of the reason codes."""
    arrays_finite = all(np.all(np.isfinite(np.asarray(a))) for a in (pos, vel, forces))
    if not arrays_finite or not math.isfinite(e_total):
        return NON_FINITE
    if disp_max > 0 and not (max_disp_step <= disp_max):
        return DISPLACEMENT
    if step % check_interval == 0 and abs(e_total - e0) > drift_tol * abs(e0):
        return ENERGY_DRIFT
    return CENSORED


def run_ttf(force_fn, pos, vel, species, box, dt, nvt_steps, T, tau, max_nve_steps, check_interval=100,
            drift_tol=0.1, disp_max=0.5, outlier_k=5.0, outlier_interval=1):
    """The protocol on the oracle model; force_fn(pos) -> (e_pot, forces).

    Returns dict(steps_survived, fail_step, reason, e0, e_last, f_mean, f_sigma, series)."""
    box = np.asarray(box, dtype=np.float64)
    m = md.masses(species)[:, None]
    pos = wrap(np.asarray(pos, dtype=np.float64), box)
    vel = np.asarray(vel, dtype=np.float64).copy()
    e_pot, forces = force_fn(pos)
    if nvt_steps > 0:
        pos, vel, forces, _, _, log = md.nvt_verlet(force_fn, pos, vel, species, box, dt, nvt_steps, T, tau,
                                                    forces=forces)
        e_pot = log[-1][0]
    e0 = e_pot + md.kinetic_energy(vel, species)
    f_mean, f_sigma = md.force_baseline(forces)
    series = []
    reason, s, e_last = CENSORED, 0, e0
    for s in range(1, max_nve_steps + 1):
        vel = vel + 0.5 * dt * md.KAPPA * forces / m
        max_disp = float(np.max(np.linalg.norm(dt * vel, axis=1))) if len(vel) else 0.0
        pos = wrap(pos + dt * vel, box)
        e_pot, forces = force_fn(pos)
        vel = vel + 0.5 * dt * md.KAPPA * forces / m
        e_tot = e_pot + md.kinetic_energy(vel, species)
        if s % check_interval == 0:
            e_last = e_tot
        reason = detect_failure(pos, vel, forces, e_tot, e0, s, check_interval, drift_tol, max_disp, disp_max)
        if reason == CENSORED and s % outlier_interval == 0:
            series.append(md.count_outliers(forces, f_mean, f_sigma, outlier_k))
        if reason != CENSORED:
            break
    return dict(steps_survived=s - 1 if reason else max_nve_steps, fail_step=s if reason else 0, reason=reason,
                e0=e0, e_last=e_last, f_mean=f_mean, f_sigma=f_sigma, series=series)


def fit_power_law(records):
    """records: iterable of (n_atoms, t_failure, reason) with t_failure the NVE step at which
    the failure was detected (>= 1).  Returns dict(alpha, beta, beta_stderr, r_squared,
    censored_count, sizes)."""
    by_n: dict[int, list[float]] = {}
    censored = 0
    for n, t, reason in records:
        if reason == CENSORED:
            censored += 1
            continue
        by_n.setdefault(int(n), []).append(float(t))
    sizes = sorted(by_n)
    if len(sizes) < 2:
        raise FitError("need >= 2 system sizes with an uncensored record")
    if any(t <= 0 for n in sizes for t in by_n[n]):
        raise FitError("t_failure must be positive")
    x = [math.log(n) for n in sizes]
    y = [math.log(sum(by_n[n]) / len(by_n[n])) for n in sizes]
    k = len(x)
    xm = sum(x) / k
    ym = sum(y) / k
    sxx = sum((xi - xm) ** 2 for xi in x)
    sxy = sum((xi - xm) * (yi - ym) for xi, yi in zip(x, y))
    slope = sxy / sxx
    intercept = ym - slope * xm
    resid = [yi - (intercept + slope * xi) for xi, yi in zip(x, y)]
    sse = sum(r * r for r in resid)
    syy = sum((yi - ym) ** 2 for yi in y)
    stderr = math.sqrt(sse / (k - 2) / sxx) if k > 2 else float("nan")
    r2 = 1.0 - sse / syy if syy > 0 else 1.0
    return dict(alpha=math.exp(intercept), beta=-slope, beta_stderr=stderr, r_squared=r2, censored_count=censored,
                sizes=sizes)
