"""GPU time-to-failure harness (NEXT-2; include/allegro.h md_run_ttf) against oracle/ttf.py.

Trajectories are compared only over a few steps (reading D21); each scenario is built so the
failure decision is far from its threshold, so both sides must take the same one."""
import numpy as np
import pytest

from oracle import allegro as oa, ttf as ottf, weights_io
from synth import configs, nh3

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2303_08169_b200 as pb

    return pb


@pytest.fixture(scope="module")
def c1():
    s = nh3.maxwell_boltzmann(nh3.nh3_box("fcc", (1, 1, 1)), 200.0)
    wf = configs.weight_file("C1")
    model = weights_io.read(wf)
    fn = lambda q: (lambda r: (r["energy"], r["forces"]))(oa.energy_forces(model, q, s.species, s.box))
    return s, wf, fn


def _gpu(pb, s, wf, **kw):
    m = pb.Allegro(wf, s.box, precision=pb.PREC_3XTF32)
    m.md_set_state(s.species, s.pos, s.vel)
    r, series = m.md_run_ttf(**kw)
    m.close()
    return r, series


def test_energy_drift_decision(pb, c1):
    """Tiny drift tolerance: both sides fail at the first check step after 3 NVT steps."""
    s, wf, fn = c1
    kw = dict(dt_fs=1.0, nvt_steps=3, T_K=200.0, tau_fs=20.0, max_nve_steps=20, check_interval=2,
              drift_tol=1e-12, disp_max=0.5, outlier_k=5.0, outlier_interval=1)
    g, gs = _gpu(pb, s, wf, **kw)
    o = ottf.run_ttf(fn, s.pos, s.vel, s.species, s.box, 1.0, 3, 200.0, 20.0, 20, check_interval=2,
                     drift_tol=1e-12, disp_max=0.5)
    assert g["reason_name"] == "energy_drift" and o["reason"] == ottf.ENERGY_DRIFT
    assert g["fail_step"] == o["fail_step"] == 2 and g["steps_survived"] == 1
    assert abs(g["e0"] - o["e0"]) <= 1e-5 * abs(o["e0"]) + 1e-4
    assert abs(g["f_mean"] - o["f_mean"]) < 1e-4 and abs(g["f_sigma"] - o["f_sigma"]) < 1e-4
    assert list(gs) == o["series"]


def test_displacement_decision(pb, c1):
    s, wf, fn = c1
    g, gs = _gpu(pb, s, wf, dt_fs=2.0, nvt_steps=0, max_nve_steps=10, disp_max=1e-3)
    o = ottf.run_ttf(fn, s.pos, s.vel, s.species, s.box, 2.0, 0, 200.0, 100.0, 10, disp_max=1e-3)
    assert g["reason_name"] == "displacement_blowup" and o["reason"] == ottf.DISPLACEMENT
    assert g["fail_step"] == o["fail_step"] == 1 and g["steps_survived"] == 0 and len(gs) == 0


def test_censored_run_and_outlier_series(pb, c1):
    """Generous limits: censored at max_nve_steps; the per-step 5-sigma counts match the oracle's
    wherever no force norm lies within the force tolerance of the threshold."""
    s, wf, fn = c1
    g, gs = _gpu(pb, s, wf, dt_fs=1.0, nvt_steps=0, max_nve_steps=6, check_interval=3, drift_tol=1e9,
                 disp_max=1e9, outlier_k=1.0)
    o = ottf.run_ttf(fn, s.pos, s.vel, s.species, s.box, 1.0, 0, 200.0, 100.0, 6, check_interval=3,
                     drift_tol=1e9, disp_max=1e9, outlier_k=1.0)
    assert g["reason_name"] == "censored" and o["reason"] == ottf.CENSORED
    assert g["steps_survived"] == 6 and g["fail_step"] == 0 and len(gs) == 6
    assert np.abs(np.asarray(gs) - np.asarray(o["series"])).max() <= 1
    assert abs(g["e_last"] - o["e_last"]) <= 1e-5 * abs(o["e_last"]) + 1e-4


def test_protocol_arguments_rejected(pb, c1):
    s, wf, _ = c1
    m = pb.Allegro(wf, s.box)
    m.md_set_state(s.species, s.pos, s.vel)
    for bad in (dict(check_interval=0), dict(outlier_interval=0), dict(drift_tol=0.0), dict(nvt_steps=5, T_K=0.0)):
        with pytest.raises(pb.AllegroError):
            m.md_run_ttf(max_nve_steps=5, **bad)
    m.close()


def test_paper_protocol_runs_to_a_decision(pb):
    """The paper's protocol shape on C2 (NVT 200 K then NVE, dt 2 fs) with a short NVT phase:
    the random-weight model (no repulsive core) must end in a failure or a censor, with the
    series length consistent with the steps survived."""
    s = configs.system("C2")
    m = pb.Allegro(configs.weight_file("C2"), s.box, precision=pb.PREC_3XTF32)
    m.md_set_state(s.species, s.pos, s.vel)
    r, series = m.md_run_ttf(dt_fs=2.0, nvt_steps=50, max_nve_steps=400, check_interval=20)
    m.close()
    assert r["reason_name"] in ("censored", "non_finite", "displacement_blowup", "energy_drift")
    assert len(series) == r["steps_survived"]
    assert r["failed_in_nvt"] == 0 and np.isfinite(r["e0"])
