"""Pins of oracle.irreps: Table 2's printed parameter counts."""
import pytest

from oracle import irreps as I
from synth import weights as sw


@pytest.mark.parametrize(
    "lmax,count",
    [(0, 95656), (1, 133544), (2, 183720)],  # Table 2
)
def test_table2_parameter_counts(lmax, count):
    assert I.param_count(3, lmax) == count


def test_baseline_config_counts():
    assert I.param_count(2, 1) == 94632  # C1
    assert I.param_count(2, 2) == 123304  # C2


def test_c3_layer0_paths_app_b():
    spec = I.layer_specs(3, 2)[0]
    names = [(I.irrep_name(a), I.irrep_name(b), I.irrep_name(c)) for a, b, c in spec.paths]
    assert names == [
        ("0e", "0e", "0e"), ("1o", "1o", "0e"), ("2e", "2e", "0e"),
        ("1o", "1o", "1e"), ("2e", "2e", "1e"),
        ("0e", "1o", "1o"), ("1o", "0e", "1o"), ("1o", "2e", "1o"), ("2e", "1o", "1o"),
        ("0e", "2e", "2e"), ("1o", "1o", "2e"), ("2e", "0e", "2e"), ("2e", "2e", "2e"),
        ("1o", "2e", "2o"), ("2e", "1o", "2o"),
    ]


@pytest.mark.parametrize("key", list(sw.ARCH))
def test_weight_file_table_matches_derivation(key):
    specs = I.layer_specs(*key)
    assert tuple((len(s.paths), s.n_scalar) for s in specs) == sw.ARCH[key]
    n = sum(int(__import__("numpy").prod(shape)) for _, shape in sw.tensor_list(*key))
    assert n == I.param_count(*key)
