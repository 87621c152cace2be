"""GPU edge cases through the C ABI (SURVEY.md §8(b) conventions, §8(c) reading rows 12 and 14).

* pairs at EXACTLY d^2 = fl(r_c^2) (integer Pythagorean offsets, exact in fp64) and pairs a
  few ulps either side of it: the GPU's canonical no-FMA fp64 rule (D12) must give
  the oracle's brute-force set bit for bit, including the image edges at exactly r_c (D14)
  and both directions of every pair (D22);
* coincident atoms (d = 0) give a non-finite result -> ALLEGRO_E_NONFINITE (SPEC.md:78,
  never masked);
* a domain edge below r_c + skin with world_size > 1 -> ALLEGRO_E_GEOMETRY;
* single-pass TF32: reported, not gated (SURVEY.md §8(c) acceptance, App. C).
"""
import numpy as np
import pytest

from oracle import allegro as oa, neighbors as onb, weights_io
from synth import configs, weights as sw

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2303_08169_b200 as pb

    return pb


def _model_file(tmp_path, L, lmax, rc, sigma=1.0):
    path = str(tmp_path / f"m{L}{lmax}_{rc:g}.algw")
    sw.write(path, L, lmax, rc, sw.generate(L, lmax, 0), sw.nbar_for(rc), (sigma, sigma), (0.0, 0.0))
    return path


def _edge_set(i, j, s):
    return sorted(zip(np.asarray(i).tolist(), np.asarray(j).tolist(), map(tuple, np.asarray(s).tolist())))


def _check_edges(pb, wf, pos, species, box, rc):
    m = pb.Allegro(wf, box)
    m.compute_energy_forces(pos, species)
    gi, gj, gs = m.get_edges()
    ri, rj, rn = onb.brute_force(onb.wrap(pos, box), box, rc)
    assert _edge_set(gi, gj, gs) == _edge_set(ri, rj, rn)
    return m, len(gi)


@pytest.mark.parametrize("seed", range(4))
def test_pairs_at_exactly_rc(pb, tmp_path, seed):
    """Atoms on an integer lattice: offsets (3, 4, 0), (0, 0, 5), ... are exactly r_c = 5 in fp64
    (fl(d^2) = 25 = fl(r_c^2): included), (4, 4, 2) is 6 (excluded); box 10 puts images at
    exactly r_c too (a pair 5 apart along x is an edge twice: n = 0 and n = -1)."""
    rng = np.random.default_rng(900 + seed)
    rc = 5.0
    box = np.array([10.0, 10.0, 12.0]) if seed % 2 else np.array([10.0, 11.0, 13.0])
    pts = set()
    while len(pts) < 24:
        pts.add(tuple(int(v) for v in rng.integers(0, [10, 10, 12])))
    pos = np.array(sorted(pts), dtype=np.float64) + 0.5  # k + 0.5 is exact; differences stay integers
    species = rng.integers(0, 2, pos.shape[0])
    wf = _model_file(tmp_path, 2, 1, rc)
    m, n_e = _check_edges(pb, wf, pos, species, box, rc)
    # the set really has boundary pairs: count d == r_c edges in the oracle's list
    ri, rj, rn = onb.brute_force(onb.wrap(pos, box), box, rc)
    d = np.linalg.norm(onb.edge_vectors(onb.wrap(pos, box), box, ri, rj, rn), axis=1)
    assert np.sum(d == rc) >= 4
    # the energy / forces at the boundary: u(r_c) = 0 -> those edges contribute exactly 0
    ref = oa.energy_forces(weights_io.read(wf), pos, species, box)
    e, ea, F = m.compute_energy_forces(pos, species)
    assert np.abs(F - ref["forces"]).max() <= 1e-4
    assert np.abs(ea - ref["e_atom"]).max() <= 1e-5 * max(np.abs(ref["e_atom"]).max(), 1e-12)


@pytest.mark.parametrize("seed", range(4))
def test_pairs_within_ulps_of_rc(pb, tmp_path, seed):
    """Neighbours placed at r_c (1 + k eps) for k in -4..4 along random directions: fl(d^2)
    falls on both sides of fl(r_c^2) depending on the last bits, so only the canonical
    formula reproduces the oracle's decision for every pair and both directions."""
    rng = np.random.default_rng(950 + seed)
    rc = 6.0
    box = np.array([40.0, 40.0, 40.0])
    pos = []
    for k in range(-4, 5):
        for _ in range(3):
            a = rng.uniform(8.0, 32.0, 3)
            u = rng.standard_normal(3)
            u /= np.linalg.norm(u)
            b = a + rc * (1.0 + k * np.finfo(np.float64).eps) * u
            pos += [a, b]
    pos = np.array(pos)
    species = rng.integers(0, 2, pos.shape[0])
    wf = _model_file(tmp_path, 2, 1, rc)
    _check_edges(pb, wf, pos, species, box, rc)


def test_coincident_atoms_nonfinite(pb, tmp_path):
    """d = 0 between two distinct atoms: r_hat and B(d) are undefined, the result is non-finite
    and must be reported as ALLEGRO_E_NONFINITE, not masked."""
    wf = _model_file(tmp_path, 2, 1, 5.0)
    box = np.array([20.0, 20.0, 20.0])
    pos = np.array([[5.0, 5.0, 5.0], [5.0, 5.0, 5.0], [7.0, 5.0, 5.0]])
    m = pb.Allegro(wf, box)
    with pytest.raises(pb.AllegroError) as ex:
        m.compute_energy_forces(pos, np.array([0, 1, 0]))
    assert ex.value.code == pb.E_NONFINITE
    with pytest.raises(pb.AllegroError) as ex:
        m.md_set_state(np.array([0, 1, 0]), pos, np.zeros_like(pos))
    assert ex.value.code == pb.E_NONFINITE
    # the ctx stays usable
    e, _, F = m.compute_energy_forces(pos[[0, 2]], np.array([0, 0]))
    assert np.isfinite(e) and np.all(np.isfinite(F))


def test_domain_smaller_than_cutoff_geometry_error(pb, tmp_path):
    """world_size 2 on grid (2, 1, 1) with a 10 A box: the domain edge 5 A < r_c = 6 A.  The
    check runs before any NCCL call, so one GPU suffices."""
    wf = configs.weight_file("C2")
    with pytest.raises(pb.AllegroError) as ex:
        pb.Allegro(wf, np.array([10.0, 30.0, 30.0]), rank=0, world_size=2, nccl_id=b"\0" * 128, grid=(2, 1, 1))
    assert ex.value.code == pb.E_GEOMETRY
    with pytest.raises(pb.AllegroError) as ex:
        pb.Allegro(wf, np.array([30.0, 30.0, 30.0]), precision=pb.PREC_BF16X3)
    assert ex.value.code == pb.E_ARG


def test_single_pass_tf32_reported_not_gated(pb):
    """ALLEGRO_PREC_TF32 runs one tcgen05 pass (a_hi w_hi): reported, not gated (App. C predicts
    ~30x over the force bound).  Only sanity is asserted: finite, and far closer to the oracle
    than the force scale."""
    s = configs.system("C2")
    wf = configs.weight_file("C2")
    ref = oa.energy_forces(weights_io.read(wf), s.pos, s.species, s.box)
    m = pb.Allegro(wf, s.box, precision=pb.PREC_TF32)
    e, ea, F = m.compute_energy_forces(s.pos, s.species)
    err = np.abs(F - ref["forces"]).max()
    rel_e = abs(e - ref["energy"]) / np.abs(ref["e_atom"]).sum()
    print(f"TF32 single pass on C2: max|dF| = {err:.3g} eV/A (bar 1e-4), rel dE = {rel_e:.3g} (bar 1e-5)")
    assert np.all(np.isfinite(F)) and err < 0.1


def test_skin_edges_contribute_exact_zeros(pb):
    """NEXT-4: a neighbour-list skin adds edges with r_c < d <= r_c + skin; the
    envelope makes u = u' = 0 there, so x = w = V = 0 on them and their g is exactly 0 (§8(c)
    "exact zero beyond r_c").  Energies and per-atom energies with skin 0.5 A equal skin 0 bit for
    bit; the forces' lane-strided edge reductions (force gather, Gamma-bar row sums) hand the
    same nonzero terms to different lanes once zeros are interleaved, so they agree to fp32
    re-association (measured on a B200: energies bitwise, forces not)."""
    s = configs.system("C2")
    wf = configs.weight_file("C2")
    m0 = pb.Allegro(wf, s.box)
    m1 = pb.Allegro(wf, s.box, skin=0.5)
    e0, a0, f0 = m0.compute_energy_forces(s.pos, s.species)
    e1, a1, f1 = m1.compute_energy_forces(s.pos, s.species)
    assert len(m1.get_edges()[0]) > 1.2 * len(m0.get_edges()[0])
    assert e1 == e0 and np.array_equal(a1, a0)
    rms = float(np.sqrt((f0**2).sum(1).mean()))
    err = float(np.abs(f1 - f0).max())
    print(f"skin 0.5 vs 0: max|dF| = {err:.3g} eV/A (RMS|F| = {rms:.3g})")
    assert err <= 1e-6 * max(1.0, rms)
