"""Pins of oracle/ttf.py (time-to-failure protocol and Eq. 4 fit) against hand cases,
closed forms and an independent library regression (scipy.stats.linregress)."""
import math

import numpy as np
import pytest
from scipy import stats

from oracle import md, ttf
from synth import configs, nh3


def _healthy(n=4):
    return np.zeros((n, 3)), np.zeros((n, 3)), np.ones((n, 3))


def test_detect_failure_hand_cases():
    p, v, f = _healthy()
    assert ttf.detect_failure(p, v, f, -10.0, -10.0, 100, 100, 0.1, 0.01, 0.5) == ttf.CENSORED
    f2 = f.copy()
    f2[1, 2] = np.nan
    assert ttf.detect_failure(p, v, f2, -10.0, -10.0, 1, 100, 0.1, 0.01, 0.5) == ttf.NON_FINITE
    assert ttf.detect_failure(p, v, f, float("inf"), -10.0, 1, 100, 0.1, 0.01, 0.5) == ttf.NON_FINITE
    # one atom moved 0.6 A in one step with a 0.5 A limit; the limit itself is allowed
    assert ttf.detect_failure(p, v, f, -10.0, -10.0, 3, 100, 0.1, 0.6, 0.5) == ttf.DISPLACEMENT
    assert ttf.detect_failure(p, v, f, -10.0, -10.0, 3, 100, 0.1, 0.5, 0.5) == ttf.CENSORED
    assert ttf.detect_failure(p, v, f, -10.0, -10.0, 3, 100, 0.1, 9.0, 0.0) == ttf.CENSORED  # disabled
    # drift of 2x the tolerance: a failure only at a check step
    assert ttf.detect_failure(p, v, f, -12.0, -10.0, 200, 100, 0.1, 0.0, 0.5) == ttf.ENERGY_DRIFT
    assert ttf.detect_failure(p, v, f, -12.0, -10.0, 201, 100, 0.1, 0.0, 0.5) == ttf.CENSORED
    # exactly at the tolerance is not a failure (strict)
    assert ttf.detect_failure(p, v, f, -11.0, -10.0, 100, 100, 0.1, 0.0, 0.5) == ttf.CENSORED
    # non-finite wins over the other criteria
    assert ttf.detect_failure(p, v, f2, -12.0, -10.0, 100, 100, 0.1, 9.0, 0.5) == ttf.NON_FINITE


def test_fit_exact_power_law():
    """Noise-free t = 1e6 N^-0.29 (the paper's Allegro exponent, Fig. 2) -> exact recovery."""
    rec = [(n, 1e6 * n ** -0.29, ttf.ENERGY_DRIFT) for n in (432, 864, 1728)]
    r = ttf.fit_power_law(rec)
    assert abs(r["beta"] - 0.29) < 1e-9
    assert abs(r["alpha"] / 1e6 - 1) < 1e-6
    assert r["r_squared"] > 1 - 1e-12


def test_fit_constant_and_censoring():
    rec = [(n, 500.0, ttf.NON_FINITE) for n in (100, 200, 400)] + [(800, 10 ** 6, ttf.CENSORED)]
    r = ttf.fit_power_law(rec)
    assert abs(r["beta"]) < 1e-12 and r["censored_count"] == 1 and r["sizes"] == [100, 200, 400]
    with pytest.raises(ttf.FitError):
        ttf.fit_power_law([(100, 5.0, 1), (100, 7.0, 3), (200, 9.0, 0)])


def test_fit_mean_over_seeds_and_library_regression():
    """Per-N mean of the uncensored records, then OLS in log-log == scipy's linregress."""
    rng = np.random.default_rng(7)
    sizes = [256, 512, 1024, 2048, 4096, 8192]
    rec = [(n, float(rng.uniform(50, 5000)), int(rng.integers(1, 4))) for n in sizes for _ in range(10)]
    r = ttf.fit_power_law(rec)
    means = [np.mean([t for m, t, _ in rec if m == n]) for n in sizes]
    lr = stats.linregress(np.log(sizes), np.log(means))
    assert abs(r["beta"] + lr.slope) < 1e-12
    assert abs(math.log(r["alpha"]) - lr.intercept) < 1e-12
    assert abs(r["beta_stderr"] - lr.stderr) < 1e-12
    assert abs(r["r_squared"] - lr.rvalue ** 2) < 1e-12


def test_fit_recovers_known_beta_within_two_stderr():
    """Monte Carlo: noisy log-linear data with beta = 0.14 (Allegro-Legato,
    Fig. 2); the 2-stderr interval covers the truth in about 95 % of trials (t-dist, 18 dof)."""
    rng = np.random.default_rng(11)
    sizes = np.geomspace(400, 40000, 20).astype(int)
    hits = 0
    for _ in range(200):
        t = 3e4 * sizes ** -0.14 * np.exp(rng.normal(0, 0.2, sizes.size))
        r = ttf.fit_power_law([(n, tt, ttf.ENERGY_DRIFT) for n, tt in zip(sizes, t)])
        hits += abs(r["beta"] - 0.14) <= 2 * r["beta_stderr"]
    assert hits >= 180  # 2 sigma of t(18 dof) ~ 93.9 %; binomial margin


def _harmonic(box, anchors, k=2.0):
    def fn(pos):
        d = pos - anchors
        d -= box * np.round(d / box)
        return 0.5 * k * float((d * d).sum()), -k * d
    return fn


def test_harness_neutral_on_a_stable_potential():
    """SPEC.md:486 harness neutrality: harmonic wells (a stable force field) never trigger a
    failure; with the limits tightened the same trajectory fails on the criterion hit first."""
    s = nh3.maxwell_boltzmann(nh3.nh3_box("fcc", (1, 1, 1)), 200.0)
    fn = _harmonic(s.box, s.pos.copy())
    r = ttf.run_ttf(fn, s.pos, s.vel, s.species, s.box, 1.0, 20, 200.0, 50.0, 200, check_interval=10)
    assert r["reason"] == ttf.CENSORED and r["steps_survived"] == 200 and len(r["series"]) == 200
    r = ttf.run_ttf(fn, s.pos, s.vel, s.species, s.box, 1.0, 0, 200.0, 50.0, 200, check_interval=10,
                    drift_tol=1e-14)
    assert r["reason"] == ttf.ENERGY_DRIFT and r["fail_step"] == 10 and r["steps_survived"] == 9
    r = ttf.run_ttf(fn, s.pos, s.vel, s.species, s.box, 1.0, 0, 200.0, 50.0, 200, disp_max=1e-4)
    assert r["reason"] == ttf.DISPLACEMENT and r["fail_step"] == 1 and r["series"] == []


def test_unstable_force_field_fails():
    """An inverted harmonic well (runaway) fails by displacement blow-up or drift."""
    s = nh3.maxwell_boltzmann(nh3.nh3_box("fcc", (1, 1, 1)), 200.0)
    fn = _harmonic(s.box, s.pos.copy() + 0.05, k=-50.0)
    r = ttf.run_ttf(fn, s.pos, s.vel, s.species, s.box, 2.0, 0, 200.0, 50.0, 10000, check_interval=10)
    assert r["reason"] in (ttf.DISPLACEMENT, ttf.ENERGY_DRIFT) and r["fail_step"] < 10000


def test_fit_rejects_nonpositive_times():
    with pytest.raises(ttf.FitError):
        ttf.fit_power_law([(100, 0.0, ttf.DISPLACEMENT), (200, 3.0, ttf.DISPLACEMENT)])


def test_product_fit_matches_oracle_fit():
    """The package's host-side fit (numpy lstsq) and the oracle's written-out sums agree."""
    from paper_2303_08169_b200 import ttf as pttf

    rng = np.random.default_rng(3)
    rec = [(n, float(rng.integers(1, 9000)), int(rng.integers(0, 4))) for n in (128, 432, 1024, 2000) for _ in range(10)]
    a, b = ttf.fit_power_law(rec), pttf.fit_power_law(rec)
    for k in ("alpha", "beta", "beta_stderr", "r_squared"):
        assert abs(a[k] - b[k]) <= 1e-9 * max(1.0, abs(a[k])), k
    assert a["censored_count"] == b["censored_count"] and a["sizes"] == b["sizes"]
