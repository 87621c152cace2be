"""GPU replica batches and ring-polymer MD (NEXT-3) against the oracle (oracle/pimd.py).

* A batch of replicas evaluated in one pass equals, replica by replica, the oracle and the
  single-replica GPU evaluation (bit for bit: edges never cross replicas, rows and sums are
  the single evaluation's).
* A few PIMD steps (P = 4, C1 geometry) follow the oracle's trajectory (reading D21: short
  horizons only); H_P bookkeeping matches the oracle's."""
import numpy as np
import pytest

from oracle import allegro as oa, pimd as opimd, weights_io
from synth import configs, nh3

pytestmark = pytest.mark.gpu
E_TOL, F_TOL = 1e-5, 1e-4


@pytest.fixture(scope="module")
def pb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2303_08169_b200 as pb

    return pb


def _beads(s, P, seed, sigma=0.05):
    rng = np.random.default_rng(seed)
    q = s.pos[None] + rng.normal(size=(P, s.n, 3)) * sigma
    v = s.vel[None] + rng.normal(size=(P, s.n, 3)) * 0.005
    return q, v


@pytest.mark.parametrize("cfg,P", [("C1", 3), ("C2", 4)])
def test_batch_matches_oracle_and_single(pb, cfg, P):
    s = configs.system(cfg)
    wf = configs.weight_file(cfg)
    model = weights_io.read(wf)
    q, _ = _beads(s, P, 5)
    m = pb.Allegro(wf, s.box, precision=pb.PREC_3XTF32)
    e_rep, e_atom, F = m.compute_energy_forces_batch(q, s.species)
    for j in range(P):
        ref = oa.energy_forces(model, q[j], s.species, s.box)
        norm = np.abs(ref["e_atom"]).sum()
        assert abs(e_rep[j] - ref["energy"]) <= E_TOL * norm
        assert np.abs(e_atom[j] - ref["e_atom"]).max() <= E_TOL * np.abs(ref["e_atom"]).max()
        assert np.abs(F[j] - ref["forces"]).max() <= F_TOL
        e1, ea1, f1 = m.compute_energy_forces(q[j], s.species)
        assert e1 == e_rep[j] and np.array_equal(ea1, e_atom[j]) and np.array_equal(f1, F[j])
    m.close()


def test_pimd_steps_follow_oracle(pb):
    s = nh3.maxwell_boltzmann(nh3.nh3_box("fcc", (1, 1, 1)), 200.0)
    wf = configs.weight_file("C1")
    model = weights_io.read(wf)
    P, T, dt = 4, 200.0, 0.25
    q0, v0 = _beads(s, P, 7)
    m = pb.Allegro(wf, s.box, precision=pb.PREC_3XTF32)
    m.pimd_set_state(s.species, q0, v0, T)
    reps = [m.pimd_step(1, dt) for _ in range(3)]
    q, v, f, e = m.pimd_get_state()
    fn = lambda x: (lambda r: (r["energy"], r["forces"]))(oa.energy_forces(model, x, s.species, s.box))
    qo, vo, fo, log = opimd.pimd(fn, q0, v0, s.species, s.box, dt, T, 3)
    assert np.abs(q - qo).max() < 1e-6 and np.abs(v - vo).max() < 1e-5
    assert np.abs(f - fo).max() < F_TOL
    Vs, K, Es, H = log[-1]
    r = reps[-1]
    assert abs(r.e_pot_mean * P - Vs) <= E_TOL * max(1.0, abs(Vs)) + 1e-4
    assert abs(r.e_kin - K) <= 1e-6 * max(1.0, K) and abs(r.e_spring - Es) <= 1e-6 * max(1.0, Es)
    assert abs(r.omega_p - opimd.omega_p(P, T)) < 1e-15
    assert abs(e.sum() - Vs) <= E_TOL * max(1.0, abs(Vs)) + 1e-4
    m.close()


def test_pimd_one_bead_equals_md(pb):
    """P = 1 is classical velocity Verlet: the PIMD path and md_step agree."""
    s = nh3.maxwell_boltzmann(nh3.nh3_box("fcc", (1, 1, 1)), 200.0)
    wf = configs.weight_file("C1")
    m = pb.Allegro(wf, s.box, precision=pb.PREC_3XTF32)
    m.pimd_set_state(s.species, s.pos[None], s.vel[None], 200.0)
    m.pimd_step(4, 0.5)
    q, v, f, _ = m.pimd_get_state()
    m.md_set_state(s.species, s.pos, s.vel)
    m.md_step(4, 0.5)
    p2, v2, f2 = m.md_get_state()
    dq = q[0] - p2
    dq -= s.box * np.round(dq / s.box)
    assert np.abs(dq).max() < 1e-9 and np.abs(v[0] - v2).max() < 1e-9 and np.abs(f[0] - f2).max() < 1e-9
    m.close()


def test_pimd_rejects_bad_state(pb):
    s = nh3.maxwell_boltzmann(nh3.nh3_box("fcc", (1, 1, 1)), 200.0)
    m = pb.Allegro(configs.weight_file("C1"), s.box)
    with pytest.raises(pb.AllegroError):
        m.pimd_step(1, 0.5)  # before pimd_set_state
    with pytest.raises(pb.AllegroError):
        m.pimd_set_state(s.species, np.zeros((65, s.n, 3)), np.zeros((65, s.n, 3)), 200.0)
    m.close()
