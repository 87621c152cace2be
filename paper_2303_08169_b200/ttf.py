"""Host side of the time-to-failure harness (NEXT-2).

The dynamics run on the GPU (``Allegro.md_run_ttf`` -> ``md_run_ttf`` in include/allegro.h);
this module only aggregates the records and fits Eq. 4 of the paper:
t_failure = alpha N^(-beta), by least squares of ln(mean uncensored t) on ln N
(censored runs are excluded and counted).
"""
from __future__ import annotations

import numpy as np

CENSORED = 0


class FitError(ValueError):
    pass


def fit_power_law(records):
    """records: iterable of (n_atoms, t_failure, reason) -> dict(alpha, beta, beta_stderr,
    r_squared, censored_count, sizes, t_mean).  t_failure is the NVE step at which the failure
    was detected (md_run_ttf's fail_step, >= 1); censored records are excluded."""
    rec = [(int(n), float(t), int(r)) for n, t, r in records]
    censored = sum(1 for _, _, r in rec if r == CENSORED)
    sizes = np.array(sorted({n for n, _, r in rec if r != CENSORED}), dtype=np.float64)
    if sizes.size < 2:
        raise FitError("need >= 2 system sizes with an uncensored record")
    t_mean = np.array([np.mean([t for n, t, r in rec if n == s and r != CENSORED]) for s in sizes])
    if np.any(t_mean <= 0):
        raise FitError("t_failure must be positive (use the failing step, >= 1)")
    X = np.stack([np.ones_like(sizes), np.log(sizes)], axis=1)
    y = np.log(t_mean)
    coef, *_ = np.linalg.lstsq(X, y, rcond=None)
    resid = y - X @ coef
    dof = sizes.size - 2
    cov = (resid @ resid / dof) * np.linalg.inv(X.T @ X) if dof > 0 else np.full((2, 2), np.nan)
    ss_tot = float(((y - y.mean()) ** 2).sum())
    return {"alpha": float(np.exp(coef[0])), "beta": float(-coef[1]), "beta_stderr": float(np.sqrt(cov[1, 1])),
            "r_squared": 1.0 - float(resid @ resid) / ss_tot if ss_tot > 0 else 1.0, "censored_count": censored,
            "sizes": sizes.astype(int).tolist(), "t_mean": t_mean.tolist()}
