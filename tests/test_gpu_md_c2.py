"""C2 (BASELINE.json configs[1]: liquid NH3, 1,024 atoms, 2-layer lmax=2) molecular dynamics on
the GPU against the fp64 oracle.

* NVE at dt = 2 fs (§3.2) from the 200 K start: the GPU state every 100 steps
  is re-evaluated by the oracle (trajectories are chaotic, so parity is per evaluation of the
  same snapshot: reading D21).  Bars: D20 for the energy; forces D26 = 1e-4 eV/A x max(1,
  RMS|F|_oracle) -- reading row 10 fixes the 1e-4 eV/A bar at the calibration scale RMS|F| = 1
  eV/A, and the random-weight liquid heats, raising RMS|F| above that scale.
* NVE energy conservation at small dt over the first 10 fs, gated by the velocity-Verlet error
  bound: for a harmonic mode the shadow Hamiltonian differs from H by (dt^2 / 8) kappa F^2 / m,
  so |H(t) - H(0)| <= 2 (dt^2 / 8) max_t sum_i kappa |F_i|^2 / m_i (both end points), and a
  factor 2 for anharmonicity; plus the dt^2 scaling of the fluctuation.  The
  window is short on purpose: the random-weight model has no repulsive core, atoms approach
  each other within ~50 fs, the forces (~1/d as d -> 0) grow by two orders of magnitude and no
  fixed dt resolves the motion any more (a 50-fs window at dt = 0.5 fs measured 42 eV/atom of
  drift against a 28 eV/atom bound on a B200; reported in DESIGN.md §3, not a GPU defect --
  the snapshots stay within D20/D26 of the oracle throughout).
"""
import numpy as np
import pytest

from oracle import allegro as oa, md as omd, weights_io
from synth import configs

pytestmark = pytest.mark.gpu

E_TOL = 1e-5
F_TOL = 1e-4


@pytest.fixture(scope="module")
def pb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2303_08169_b200 as pb

    return pb


def test_c2_nve_snapshot_parity_every_100_steps(pb):
    s = configs.system("C2")
    wf = configs.weight_file("C2")
    model = weights_io.read(wf)
    m = pb.Allegro(wf, s.box)
    m.md_set_state(s.species, s.pos, s.vel)
    rep = m.md_step(0, 2.0)
    for step in (0, 100, 200):
        if step:
            rep = m.md_step(100, 2.0)
            assert rep.steps_done == 100
        p, v, f = m.md_get_state()
        ref = oa.energy_forces(model, p, s.species, s.box)
        rms = float(np.sqrt((ref["forces"] ** 2).sum(1).mean()))
        err = float(np.abs(f - ref["forces"]).max())
        print(f"C2 NVE step {step}: T = {rep.temperature:.0f} K, RMS|F| = {rms:.3g}, max|dF| = {err:.3g} eV/A")
        assert err <= F_TOL * max(1.0, rms)
        assert abs(rep.e_pot - ref["energy"]) <= E_TOL * np.abs(ref["e_atom"]).sum()


def _run(m, s, dt, n):
    m.md_set_state(s.species, s.pos, s.vel)
    inv_m = np.where(s.species == 1, 1.0 / omd.MASS_N, 1.0 / omd.MASS_H)
    e, fm = [], 0.0
    for _ in range(n):
        r = m.md_step(1, dt)
        e.append(r.e_total)
        f = m.md_get_state()[2]
        fm = max(fm, float(omd.KAPPA * ((f**2).sum(1) * inv_m).sum()))
    e = np.array(e)
    return e, fm


def test_c2_nve_energy_conservation_small_dt(pb):
    s = configs.system("C2")
    m = pb.Allegro(configs.weight_file("C2"), s.box)
    e_a, fm_a = _run(m, s, 0.5, 20)
    e_b, fm_b = _run(m, s, 0.25, 40)
    for e, fm, dt in ((e_a, fm_a, 0.5), (e_b, fm_b, 0.25)):
        bound = 4.0 * dt * dt / 8.0 * fm
        drift = np.abs(e - e[0]).max()
        print(f"C2 NVE over 10 fs at dt = {dt}: max|E - E0| = {drift:.3g} eV ({drift / s.n:.3g} eV/atom), "
              f"Verlet bound {bound:.3g} eV")
        assert drift <= bound
    ratio = (e_a.max() - e_a.min()) / (e_b.max() - e_b.min())
    print(f"fluctuation ratio dt 0.5 / 0.25 = {ratio:.2f}")
    assert 3.0 < ratio < 5.0
