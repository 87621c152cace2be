"""Pins of the spatial decomposition rules (oracle/domains.py):
P virtual domains reproduce P = 1 -- per-atom energies bit for bit
(same edges, same canonical row order), forces to rounding; the lower-index tie rule
(SPEC.md:544); ghost completeness."""
import numpy as np
import pytest

from oracle import allegro, domains, weights_io
from synth import nh3, weights as sw


@pytest.fixture(scope="module")
def model(tmp_path_factory):
    path = str(tmp_path_factory.mktemp("w") / "m.algw")
    sw.write(path, 2, 1, 5.0, sw.generate(2, 1, 0), sw.nbar_for(5.0), (1.5, 1.5), (0.0, 0.0))
    return weights_io.read(path)


@pytest.fixture(scope="module")
def box8():
    return nh3.nh3_box("fcc", (2, 2, 2))  # 128 atoms, L = 10.74 A: domains of 5.37 A >= r_c


@pytest.fixture(scope="module")
def ref(model, box8):
    return allegro.energy_forces(model, box8.pos, box8.species, box8.box)


@pytest.mark.parametrize("grid", [(2, 1, 1), (1, 2, 1), (1, 1, 2), (2, 2, 1), (2, 2, 2)])
def test_decomposition_equals_single_domain(model, box8, ref, grid):
    E, ea, F, n_ghost = domains.decomposed_energy_forces(model, box8.pos, box8.species, box8.box, grid)
    assert np.array_equal(ea, ref["e_atom"])  # identical rows => identical fp64 E_i
    np.testing.assert_allclose(F, ref["forces"], atol=1e-12)
    assert abs(E - ref["energy"]) < 1e-10
    assert n_ghost > 0


def test_owner_tie_rule_lower_index():
    box = np.array([10.0, 10.0, 10.0])
    pos = np.array([[5.0, 1.0, 1.0], [5.0 + 1e-12, 1.0, 1.0], [0.0, 10.0 - 1e-12, 0.0], [10.0 - 1e-13, 5.0, 5.0]])
    own = domains.owner_coords(pos, box, (2, 2, 2))
    assert own.tolist() == [[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 0, 0]]


def test_halo_is_complete_for_every_domain(model, box8):
    # every neighbour (with its image shift) of every owned centre is present locally
    from oracle import neighbors

    grid = (2, 2, 2)
    pos = neighbors.wrap(box8.pos, box8.box)
    ei, ej, en = neighbors.cell_list(pos, box8.box, model.r_max)
    want = set(zip(ei.tolist(), ej.tolist(), map(tuple, en.tolist())))
    got = set()
    own = domains.owner_coords(pos, box8.box, grid)
    for r in range(8):
        c = domains.grid_coords(r, grid)
        idx = np.nonzero(np.all(own == c, axis=1))[0]
        loc = dict(gid=idx.astype(np.int64), species=box8.species[idx], pos=pos[idx].copy(),
                   shift=np.zeros((idx.size, 3), np.int64))
        # serial halo for this one domain (messages from all domains each stage)
        locs = []
        for q in range(8):
            cq = domains.grid_coords(q, grid)
            iq = np.nonzero(np.all(own == cq, axis=1))[0]
            locs.append(dict(gid=iq.astype(np.int64), species=box8.species[iq], pos=pos[iq].copy(),
                             shift=np.zeros((iq.size, 3), np.int64)))
        for axis in range(3):
            msgs = [domains.stage_messages(locs[q], axis, domains.grid_coords(q, grid), box8.box, grid, model.r_max)
                    for q in range(8)]
            new = []
            for q in range(8):
                rm, rp = domains.neighbour_ranks(domains.grid_coords(q, grid), axis, grid)
                l2 = domains.append(locs[q], {k: v for k, v in msgs[rm][1].items() if k != "src"})
                l2 = domains.append(l2, {k: v for k, v in msgs[rp][0].items() if k != "src"})
                new.append(l2)
            locs = new
        loc = locs[r]
        n_own = idx.size
        _, (li, lj), _ = domains.domain_rows(model, loc, n_own, model.r_max)
        for a, b in zip(li.tolist(), lj.tolist()):
            got.add((int(loc["gid"][a]), int(loc["gid"][b]), tuple(int(x) for x in loc["shift"][b])))
    assert got == want
