"""Pins of oracle.neighbors against brute force, worked examples and closed forms.

SPEC.md:64/112 (cell-list pair set == brute force on 100 random configs),
SPEC.md:53-55/62-63 (worked examples), reading rows 12-14/17 of SURVEY.md §8(c).
"""
import itertools

import numpy as np
import pytest

from oracle import neighbors as nb
from synth import nh3


def _as_set(i, j, n):
    return set(zip(i.tolist(), j.tolist(), map(tuple, n.tolist())))


def test_worked_example_exact_cutoff_included():
    # d == r_c exactly is included (<=)
    box = np.array([10.0, 10.0, 10.0])
    pos = np.array([[1.0, 1.0, 1.0], [4.0, 1.0, 1.0]])
    i, j, n = nb.brute_force(pos, box, 3.0)
    assert _as_set(i, j, n) == {(0, 1, (0, 0, 0)), (1, 0, (0, 0, 0))}
    i, j, n = nb.brute_force(pos, box, 2.999999)
    assert len(i) == 0


def test_worked_example_periodic_image():
    box = np.array([10.0, 10.0, 10.0])
    pos = np.array([[0.5, 5.0, 5.0], [9.5, 5.0, 5.0]])
    i, j, n = nb.cell_list(pos, box, 1.5)
    assert _as_set(i, j, n) == {(0, 1, (-1, 0, 0)), (1, 0, (1, 0, 0))}
    rv = nb.edge_vectors(pos, box, i, j, n)
    np.testing.assert_allclose(np.linalg.norm(rv, axis=1), [1.0, 1.0])


def test_self_images_closed_form():
    # one atom in a cube of edge 2, r_c = 3: self-images n != 0 with 2|n| <= 3,
    # i.e. |n|^2 <= 2.25 -> 6 faces + 12 edges = 18
    box = np.array([2.0, 2.0, 2.0])
    pos = np.array([[0.3, 1.1, 1.7]])
    for fn in (nb.brute_force, nb.cell_list):
        i, j, n = fn(pos, box, 3.0)
        assert len(i) == 18
        assert sorted(map(tuple, n.tolist())) == sorted(
            s for s in itertools.product((-1, 0, 1), repeat=3) if 0 < sum(x * x for x in s) <= 2
        )


def test_wrap_examples():
    box = np.array([5.0, 5.0, 5.0])
    pos = np.array([[-0.5, 5.0, 12.25], [-1e-17, 4.999999, 0.0]])
    w = nb.wrap(pos, box)
    assert np.all(w >= 0) and np.all(w < box)
    np.testing.assert_allclose(w[0], [4.5, 0.0, 2.25])
    assert w[1, 0] == 0.0  # x - L*floor(x/L) rounds to L -> 0 (reading row 17)


@pytest.mark.parametrize("seed", range(100))
def test_cell_list_equals_brute_force(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 129))
    r_c = float(rng.uniform(1.0, 4.0))
    # a third of the boxes are smaller than 2 r_c along some axis (multi-image)
    lo = 0.6 * r_c if seed % 3 == 0 else 2.2 * r_c
    box = rng.uniform(lo, lo + 3 * r_c, size=3)
    pos = nb.wrap(rng.random((n, 3)) * box, box)
    a = nb.brute_force(pos, box, r_c)
    b = nb.cell_list(pos, box, r_c)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_c1_multi_image_and_symmetry():
    s = nh3.nh3_box("fcc", (1, 1, 1))
    assert s.box[0] < 2 * 5.0  # C1 is a multi-image box (SURVEY finding 3)
    i, j, n = nb.cell_list(s.pos, s.box, 5.0)
    edges = _as_set(i, j, n)
    # the directed list is closed under reversal (i, j, n) -> (j, i, -n)
    assert all((b, a, tuple(-x for x in s_)) in edges for a, b, s_ in edges)
    # several images of the same pair occur
    pairs = {}
    for a, b, _ in edges:
        pairs[(a, b)] = pairs.get((a, b), 0) + 1
    assert max(pairs.values()) > 1


def test_extensive_edge_count():
    s = nh3.nh3_box("fcc", (1, 1, 1))
    big = nh3.replicate(s, (2, 2, 2))
    i1, _, _ = nb.cell_list(s.pos, s.box, 5.0)
    i8, _, _ = nb.cell_list(big.pos, big.box, 5.0)
    assert len(i8) == 8 * len(i1)


def test_centers_subset_rows_match_full():
    s = nh3.nh3_box("fcc", (2, 2, 2))
    full = nb.cell_list(s.pos, s.box, 6.0)
    centers = np.array([3, 17, 40])
    sub = nb.cell_list(s.pos, s.box, 6.0, centers)
    mask = np.isin(full[0], centers)
    for x, y in zip(full, sub):
        np.testing.assert_array_equal(x[mask], y)
