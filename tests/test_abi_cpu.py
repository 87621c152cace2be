"""CPU-side checks of the C-ABI library (no GPU needed): it loads, exports every
symbol include/allegro.h declares, and its own derivations (W3j tables, Table 2
parameter counts, TP paths) agree with the oracle's independent ones."""
import itertools
import os
import re

import numpy as np
import pytest

import paper_2303_08169_b200 as pb
from oracle import irreps, so3

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "allegro.h")).read()
    names = set(re.findall(r"^\s*(?:int|void|const char\*|int64_t)\s+(\w+)\s*\(", hdr, re.M))
    assert "allegro_create" in names and "md_step" in names and len(names) >= 14
    for n in names:
        assert hasattr(pb._lib, n), n
    assert set(pb.EXPORTED) == names


@pytest.mark.parametrize("l1,l2,l3", [t for t in itertools.product(range(3), repeat=3)
                                      if abs(t[0] - t[1]) <= t[2] <= t[0] + t[1]])
def test_library_w3j_equals_oracle(l1, l2, l3):
    np.testing.assert_allclose(pb.w3j_table(l1, l2, l3), so3.w3j(l1, l2, l3), atol=1e-13)


@pytest.mark.parametrize("L,lmax", [(2, 1), (2, 2), (3, 0), (3, 1), (3, 2)])
def test_library_arch_equals_oracle(L, lmax):
    assert pb.param_count(L, lmax) == irreps.param_count(L, lmax)
    assert pb.layer_paths(L, lmax) == [(len(s.paths), s.n_scalar) for s in irreps.layer_specs(L, lmax)]


def test_version_and_create_errors(tmp_path):
    assert "sm_100a" in pb.version()
    with pytest.raises(pb.AllegroError) as e:
        pb.Allegro(str(tmp_path / "missing.algw"), [10, 10, 10])
    assert e.value.code in (pb.E_WEIGHTS, pb.E_CUDA)
    with pytest.raises(pb.AllegroError) as e:
        pb.Allegro(str(tmp_path / "missing.algw"), [10, -1, 10])
    assert e.value.code == pb.E_ARG
