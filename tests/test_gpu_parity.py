"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Bars (BASELINE.json north_star; SURVEY.md §8(c) reading row 20):
* neighbour lists bit-exact as sorted (i_gid, j_gid, shift) sets;
* energy: |dE| / sum_a |E_a - mu| <= 1e-5 and max_a |dE_a| <= 1e-5 max_a |E_a|;
* forces: max_{a,alpha} |dF| <= 1e-4 eV/A (sigma calibrated so RMS|F| = 1 eV/A).
"""
import numpy as np
import pytest

from oracle import allegro as oa, md as omd, neighbors as onb, weights_io
from synth import configs, nh3, weights as sw

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


def _edge_set(i, j, s):
    return sorted(zip(np.asarray(i).tolist(), np.asarray(j).tolist(), map(tuple, np.asarray(s).tolist())))


def _check_energy_forces(ref, e_tot, e_atom, F, atoms=None):
    ea = ref["e_atom"] if atoms is None else ref["e_atom"][atoms]
    fa = ref["forces"] if atoms is None else ref["forces"][atoms]
    if atoms is None:
        norm = np.abs(ea).sum()
        assert abs(e_tot - ref["energy"]) <= E_TOL * norm, (e_tot, ref["energy"])
    assert np.abs(e_atom - ea).max() <= E_TOL * np.abs(ea).max()
    err = np.abs(F - fa).max()
    assert err <= F_TOL, err
    return err


def _model_file(tmp_path, L, lmax, rc, sigma):
    path = str(tmp_path / f"m{L}{lmax}.algw")
    sw.write(path, L, lmax, rc, sw.generate(L, lmax, 0), sw.nbar_for(rc), (sigma, sigma), (0.0, 0.0))
    return path


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_edges_bit_exact(pb, cfg):
    c = configs.CONFIGS[cfg]
    s = configs.system(cfg)
    m = pb.Allegro(configs.weight_file(cfg), s.box)
    m.compute_energy_forces(s.pos, s.species)
    gi, gj, gs = m.get_edges()
    ri, rj, rn = onb.cell_list(onb.wrap(s.pos, s.box), s.box, c.r_cut)
    assert _edge_set(gi, gj, gs) == _edge_set(ri, rj, rn)
    # canonical row order: by centre, then (j_gid, shift)
    order = np.lexsort((gs[:, 2], gs[:, 1], gs[:, 0], gj, gi))
    assert np.array_equal(order, np.arange(len(gi)))


@pytest.mark.parametrize("seed", range(12))
def test_edges_random_boxes_incl_multi_image(pb, tmp_path, seed):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(1, 200))
    rc = 5.0
    lo = 0.7 * rc if seed % 2 == 0 else 2.5 * rc
    box = rng.uniform(lo, lo + 2 * rc, size=3)
    s = nh3.random_box(n, box, seed)
    m = pb.Allegro(_model_file(tmp_path, 2, 1, rc, 1.0), box)
    m.compute_energy_forces(s.pos, s.species)
    gi, gj, gs = m.get_edges()
    ri, rj, rn = onb.brute_force(onb.wrap(s.pos, box), box, rc)
    assert _edge_set(gi, gj, gs) == _edge_set(ri, rj, rn)


@pytest.mark.parametrize("M,N,K", [(1000, 32, 16), (4097, 128, 128), (300, 64, 224), (129, 16, 32), (5000, 192, 128),
                                   (777, 96, 96), (3001, 32, 96), (2050, 64, 32), (517, 32, 64)])
def test_gemm_kernels(pb, M, N, K):
    """Both contraction kernels against an fp64 matmul (ragged M, all N/K shapes used)."""
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = rng.uniform(-1.7, 1.7, (K, N)).astype(np.float32)
    ref = A.astype(np.float64) @ W.astype(np.float64)
    scale = np.abs(A).astype(np.float64) @ np.abs(W).astype(np.float64)
    for prec in (pb.PREC_FP32, pb.PREC_3XTF32):
        C = pb.debug_gemm(A, W, prec)
        err = np.abs(C - ref) / scale
        assert err.max() < 5e-6, (prec, err.max())


PRECS = ["fp32", "3xtf32"]


def _prec(pb, name):
    return pb.PREC_FP32 if name == "fp32" else pb.PREC_3XTF32


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_energy_forces_parity(pb, cfg, prec):
    s = configs.system(cfg)
    wf = configs.weight_file(cfg)
    model = weights_io.read(wf)
    ref = oa.energy_forces(model, s.pos, s.species, s.box)
    m = pb.Allegro(wf, s.box, precision=_prec(pb, prec))
    e, ea, F = m.compute_energy_forces(s.pos, s.species)
    err = _check_energy_forces(ref, e, ea, F)
    # per-edge dE/dr_e in the same (canonical) order
    g = m.get_edge_grad()
    assert np.abs(g - ref["g"]).max() <= F_TOL
    print(f"{cfg}: max|dF| = {err:.3g} eV/A, E = {e:.6f} vs {ref['energy']:.6f}")


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("L,lmax", [(2, 1), (2, 2), (3, 0), (3, 1), (3, 2)])
def test_every_architecture_on_c1_geometry(pb, tmp_path, L, lmax, prec):
    s = configs.system("C1")
    wf = _model_file(tmp_path, L, lmax, 5.0, 3.0)
    ref = oa.energy_forces(weights_io.read(wf), s.pos, s.species, s.box)
    m = pb.Allegro(wf, s.box, precision=_prec(pb, prec))
    e, ea, F = m.compute_energy_forces(s.pos, s.species)
    _check_energy_forces(ref, e, ea, F * 1.0)


@pytest.mark.parametrize("cfg,prec", [("C3", "fp32"), ("C3", "3xtf32"), ("C4", "3xtf32"), ("C5", "3xtf32")])
def test_full_size_sampled(pb, cfg, prec):
    """C3 (110,592 atoms, the paper's l=2 model), C4 (884,736 atoms, many chunks) and C5
    (500,000 atoms, the bench workload) at full size in the bench's launch configuration.  The
    oracle evaluates >= 64 sampled rows -- the first and last row of every model chunk plus
    random rows -- and the GPU's rows are compared edge by edge: the edge set (bit-exact),
    each edge's dE/dr_e, and E_i; exact forces on 3 atoms need the rows of all their
    neighbours (oracle.sampled_forces)."""
    s = configs.system(cfg)
    wf = configs.weight_file(cfg)
    model = weights_io.read(wf)
    m = pb.Allegro(wf, s.box, precision=_prec(pb, prec), n_atoms=s.n)
    e, ea, F = m.compute_energy_forces(s.pos, s.species)
    starts = m.chunk_starts()
    ends = np.append(starts[1:], s.n) - 1
    rng = np.random.default_rng(11)
    rows = np.unique(np.concatenate([starts, ends, rng.choice(s.n, 64, replace=False)]))
    assert rows.size >= 64 and (cfg != "C4" or starts.size > 1)
    gi, gj, gs, gg = m.get_row_edges(rows)
    ref = oa.energy_forces(model, s.pos, s.species, s.box, centers=rows)
    ri, rj, rn = ref["edges"]
    assert _edge_set(gi, gj, gs) == _edge_set(ri, rj, rn)
    og = np.lexsort((gs[:, 2], gs[:, 1], gs[:, 0], gj, gi))
    orf = np.lexsort((rn[:, 2], rn[:, 1], rn[:, 0], rj, ri))
    assert np.abs(gg[og] - ref["g"][orf]).max() <= F_TOL
    assert np.abs(ea[rows] - ref["e_atom"][rows]).max() <= E_TOL * np.abs(ea).max()
    atoms = np.array([rows[0], rows[rows.size // 2], rows[-1]])
    Fo, Eo, _ = oa.sampled_forces(model, s.pos, s.species, s.box, atoms)
    assert np.abs(F[atoms] - Fo).max() <= F_TOL
    # properties at any size: zero net force
    assert np.abs(F.sum(0)).max() < 1e-6 * s.n
    print(f"{cfg} {prec}: {starts.size} chunks, {rows.size} rows / {gi.size} edges checked")


def test_deterministic_and_device_pointers(pb):
    import torch

    s = configs.system("C2")
    m = pb.Allegro(configs.weight_file("C2"), s.box)
    e1, a1, F1 = m.compute_energy_forces(s.pos, s.species)
    e2, a2, F2 = m.compute_energy_forces(s.pos, s.species)
    assert e1 == e2 and np.array_equal(F1, F2) and np.array_equal(a1, a2)
    pos = torch.tensor(s.pos, device="cuda")
    spc = torch.tensor(s.species, device="cuda", dtype=torch.int32)
    e3, a3, F3 = m.compute_energy_forces(pos, spc)
    assert e3 == e1 and np.array_equal(F3.cpu().numpy(), F1)


def test_translation_and_replica(pb):
    s = configs.system("C1")
    wf = configs.weight_file("C1")
    m = pb.Allegro(wf, s.box)
    e, _, F = m.compute_energy_forces(s.pos, s.species)
    big = nh3.replicate(s, (2, 2, 2))
    m8 = pb.Allegro(wf, big.box)
    e8, _, F8 = m8.compute_energy_forces(big.pos, big.species)
    assert abs(e8 - 8 * e) <= 1e-5 * abs(8 * e) + 1e-5
    assert np.abs(F8 - np.tile(F, (8, 1))).max() <= 1e-5


def test_edge_cases(pb, tmp_path):
    wf = _model_file(tmp_path, 2, 1, 5.0, 1.0)
    box = np.array([30.0, 30.0, 30.0])
    m = pb.Allegro(wf, box)
    # isolated atoms: no edges, E = mu = 0, F = 0
    pos = np.array([[1.0, 1.0, 1.0], [15.0, 15.0, 15.0]])
    e, ea, F = m.compute_energy_forces(pos, np.array([0, 1]))
    assert e == 0.0 and np.all(F == 0)
    # species outside {0,1} and non-finite positions are rejected
    with pytest.raises(pb.AllegroError) as ex:
        m.compute_energy_forces(pos, np.array([0, 2]))
    assert ex.value.code == pb.E_ARG
    with pytest.raises(pb.AllegroError) as ex:
        m.compute_energy_forces(np.array([[np.nan, 1.0, 1.0], [2.0, 2.0, 2.0]]), np.array([0, 1]))
    assert ex.value.code == pb.E_ARG
    # positions outside the box are wrapped
    e1, _, F1 = m.compute_energy_forces(pos + np.array([30.0, -30.0, 60.0]), np.array([0, 1]))
    assert e1 == 0.0


def test_md_snapshot_parity_and_outliers(pb):
    """C1: 10 NVE steps at dt = 2 fs on the GPU; the final snapshot is re-evaluated by
    the oracle (trajectories are chaotic, so parity is per evaluation: reading row 21)."""
    s = configs.system("C1")
    wf = configs.weight_file("C1")
    model = weights_io.read(wf)
    m = pb.Allegro(wf, s.box)
    m.md_set_state(s.species, s.pos, s.vel)
    p0, v0, f0 = m.md_get_state()
    ref0 = oa.energy_forces(model, s.pos, s.species, s.box)
    assert np.abs(f0 - ref0["forces"]).max() <= F_TOL
    mean0, sig0 = m.md_force_baseline()
    rep = m.md_step(10, 2.0)
    assert rep.steps_done == 10
    p, v, f = m.md_get_state()
    assert np.all(p >= 0) and np.all(p < s.box)
    ref = oa.energy_forces(model, p, s.species, s.box)
    assert np.abs(f - ref["forces"]).max() <= F_TOL
    assert abs(rep.e_pot - ref["energy"]) <= E_TOL * np.abs(ref["e_atom"]).sum()
    # one oracle Verlet step from the same state agrees with one GPU step
    m.md_set_state(s.species, p, v)
    m.md_step(1, 2.0)
    p1, v1, _ = m.md_get_state()
    fn = lambda q: (lambda r: (r["energy"], r["forces"]))(oa.energy_forces(model, q, s.species, s.box))
    po, vo, _, _ = omd.verlet(fn, p, v, s.species, s.box, 2.0, 1)
    dp = p1 - po
    dp -= s.box * np.round(dp / s.box)
    # the GPU forces differ from the oracle's by <= F_TOL: bound the resulting kick
    dv_tol = 2.0 * omd.KAPPA * F_TOL / omd.MASS_H
    assert np.abs(v1 - vo).max() <= dv_tol and np.abs(dp).max() <= 2.0 * dv_tol + 1e-12
    # outlier count (integer): bit-exact against the count on the same forces
    for k in (0.5, 1.0, 2.0, 5.0):
        assert m.md_count_outliers(mean0, sig0, k) == omd.count_outliers(f1 := m.md_get_state()[2], mean0, sig0, k)
    mo, so = omd.force_baseline(f1)
    mg, sg = m.md_force_baseline()
    assert abs(mo - mg) < 1e-12 * max(1, mo) and abs(so - sg) < 1e-10 * max(1, so)


def test_md_energy_conservation_dt2_c2(pb):
    """C2 (1,024 atoms): the NVE energy error of the GPU integrator + forces scales as dt^2
    (velocity Verlet is second order).  Short windows: the random-weight
    landscape has no repulsive core, so long 2-fs runs may collapse (reported, not gated)."""
    s = configs.system("C2")
    m = pb.Allegro(configs.weight_file("C2"), s.box)

    def fluct(dt, t_total=5.0):
        m.md_set_state(s.species, s.pos, s.vel)
        e = []
        for _ in range(int(round(t_total / dt))):
            e.append(m.md_step(1, dt).e_total)
        return max(e) - min(e)

    f1, f2 = fluct(0.5), fluct(0.25)
    print(f"C2 energy fluctuation over 5 fs: dt=0.5 -> {f1:.3g} eV, dt=0.25 -> {f2:.3g} eV, ratio {f1 / f2:.2f}")
    assert 3.0 < f1 / f2 < 5.0


def test_md_step_host_matches_device(pb):
    """md_step_host (host-resident state, the e2e path) == md_step on the device."""
    s = configs.system("C1")
    wf = configs.weight_file("C1")
    m = pb.Allegro(wf, s.box)
    m.md_set_state(s.species, s.pos, s.vel)
    p0, v0, f0 = m.md_get_state()
    m.md_step(3, 2.0)
    pd, vd, fd = m.md_get_state()
    m.md_set_state(s.species, s.pos, s.vel)
    p, v, f = p0.copy(), v0.copy(), f0.copy()
    spc = s.species.astype(np.int32)
    for _ in range(3):
        m.md_step_host(spc, p, v, f, 1, 2.0)
    assert np.array_equal(p, pd) and np.array_equal(v, vd) and np.array_equal(f, fd)
    # the caller's arrays must hold the local count (capacity, include/allegro.h)
    with pytest.raises(pb.AllegroError) as ex:
        m.md_step_host(spc, p[:-1].copy(), v, f, 1, 2.0)
    assert ex.value.code == pb.E_ARG


def test_profiler_counts_launches(pb):
    s = configs.system("C1")
    m = pb.Allegro(configs.weight_file("C1"), s.box)
    m.md_set_state(s.species, s.pos, s.vel)
    m.profile(True)
    m.md_step(2, 2.0)
    prof = m.profile_read()
    assert m.launch_count() == sum(v[3] for v in prof.values()) > 20
    assert prof["gemm"][3] > 0 and prof["gemm"][0] > 0 and prof["gemm"][1] > 0
    # 2 layers x 2 steps: layer 0 runs the fused TP + TP-linear kernels (3xTF32 default), layer 1 the TP kernels
    # and layer 1 (the last) the fused last-layer kernel (forward + read-out + reverse)
    assert prof["tp_lin_fwd"][3] == prof["gamma"][3] == prof["tp_lin_bwd"][3] == prof["env_adj"][3] == 2
    assert prof["last_layer"][3] == 2 and prof["tp_fwd"][3] == prof["tp_bwd"][3] == prof["energy"][3] == 0


def test_nvt_step_matches_oracle(pb):
    """Nose-Hoover NVT (NEXT-1): 3 GPU steps vs the oracle's nvt_verlet from the
    same state (bounded by the force tolerance), and the extended energy is conserved."""
    s = nh3.maxwell_boltzmann(nh3.nh3_box("fcc", (1, 1, 1)), 300.0)
    wf = configs.weight_file("C1")
    model = weights_io.read(wf)
    m = pb.Allegro(wf, s.box, precision=pb.PREC_3XTF32)
    m.md_set_state(s.species, s.pos, s.vel)
    m.md_set_thermostat(200.0, 20.0)
    m.md_set_state(s.species, s.pos, s.vel)  # Q uses the state size
    reps = [m.md_step(1, 1.0) for _ in range(3)]
    p, v, f = m.md_get_state()
    fn = lambda q: (lambda r: (r["energy"], r["forces"]))(oa.energy_forces(model, q, s.species, s.box))
    po, vo, fo, xi, eta, lg = omd.nvt_verlet(fn, s.pos, s.vel, s.species, s.box, 1.0, 3, 200.0, 20.0)
    dp = p - po
    dp -= s.box * np.round(dp / s.box)
    assert np.abs(dp).max() < 1e-6 and np.abs(v - vo).max() < 1e-5
    assert abs(reps[-1].xi - xi) < 1e-6 * max(1.0, abs(xi))
    assert abs(reps[-1].e_conserved - lg[-1][2]) < 1e-3
    h = [r.e_conserved for r in reps]
    assert max(h) - min(h) < 1e-2


def test_repeated_evaluations_bit_identical(pb):
    """The whole 3xTF32 path is deterministic: 25 evaluations of C2 (many pipelined tiles per
    CTA through every fused epilogue) give bit-identical energies and forces."""
    s = configs.system("C2")
    m = pb.Allegro(configs.weight_file("C2"), s.box, precision=pb.PREC_3XTF32)
    e0, ea0, f0 = m.compute_energy_forces(s.pos, s.species)
    for _ in range(25):
        e, ea, f = m.compute_energy_forces(s.pos, s.species)
        assert e == e0 and np.array_equal(ea, ea0) and np.array_equal(f, f0)
    m.close()


def test_resnet_contraction_deterministic(pb):
    """The two-operand resnet contraction (x | s) W with the aux save, X = x, ragged M, two
    co-scheduled N-tiles: repeated launches are bit-identical and within 3xTF32 accuracy."""
    rng = np.random.default_rng(2)
    M, N, K, K1 = 90198, 128, 224, 128
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    u = rng.uniform(0, 1, M).astype(np.float32)
    code = 3 | (K1 << 8)  # EPI_RESID with columns [K1, K) from the second operand
    c0, a0 = pb.debug_gemm_epi(A, W, code, X=A, u=u, want_aux=True)
    exact = 0.75 * (A.astype(np.float64) @ W.astype(np.float64))
    assert np.abs(a0 - exact).max() <= 2e-5 * np.abs(exact).max()
    want_c = 0.5 * A[:, :128].astype(np.float64) + 0.25 * u[:, None] * exact
    assert np.abs(c0 - want_c).max() <= 2e-5 * np.abs(want_c).max()
    for _ in range(8):
        c, a = pb.debug_gemm_epi(A, W, code, X=A, u=u, want_aux=True)
        assert np.array_equal(c, c0) and np.array_equal(a, a0)


@pytest.mark.parametrize("cfg", ["C1", "C5"])
def test_fused_tp_linear_matches_unfused(pb, cfg, monkeypatch):
    """The fused kernels against the unfused path: the last layer in one kernel (k_last) is
    bit-identical; the fused TP + TP-linear forward (same FMA order, same 3xTF32 contraction) gives
    bit-identical energies; the fused backward re-associates the Gamma-bar row sum (per edge,
    then over the row) and the merged x-bar contraction scales A rows before the TF32 split, so
    forces agree to rounding.  C1 (2, 1) and the bench's C5 (3, 1)."""
    s = configs.system(cfg)
    wf = configs.weight_file(cfg)
    m = pb.Allegro(wf, s.box, precision=pb.PREC_3XTF32, n_atoms=s.n)
    monkeypatch.setenv("ALLEGRO_FUSED_TP", "0")
    monkeypatch.setenv("ALLEGRO_FUSED_TP_BWD", "0")
    monkeypatch.setenv("ALLEGRO_FUSED_LAST", "0")
    monkeypatch.setenv("ALLEGRO_MERGE_XBAR", "0")
    e0, ea0, f0 = m.compute_energy_forces(s.pos, s.species)
    # the fused last layer alone: the same arithmetic in the same order (bit-identical)
    monkeypatch.setenv("ALLEGRO_FUSED_LAST", "1")
    eL, eaL, fL = m.compute_energy_forces(s.pos, s.species)
    assert eL == e0 and np.array_equal(eaL, ea0) and np.array_equal(fL, f0)
    monkeypatch.setenv("ALLEGRO_FUSED_TP", "1")
    monkeypatch.setenv("ALLEGRO_FUSED_TP_BWD", "1")
    monkeypatch.setenv("ALLEGRO_MERGE_XBAR", "1")
    m.profile(True)
    e1, ea1, f1 = m.compute_energy_forces(s.pos, s.species)
    assert m.profile_read()["tp_lin_fwd"][3] > 0
    m.profile(False)
    print(f"{cfg}: fused vs unfused bitwise: E {e1 == e0}, F {np.array_equal(f1, f0)}, "
          f"max|dF| = {np.abs(f1 - f0).max():.3g}")
    assert e1 == e0 and np.array_equal(ea1, ea0)
    # re-association only: the fused path may spend at most a tenth of the force parity budget
    # (D26: 1e-4 eV/A x max(1, RMS|F|)) relative to the unfused one (C5 measured 1.4e-6 eV/A)
    rms = float(np.sqrt((f0**2).sum(1).mean()))
    assert np.abs(f1 - f0).max() <= 1e-5 * max(1.0, rms)
