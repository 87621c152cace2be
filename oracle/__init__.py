"""fp64 CPU oracle for the Allegro-Legato NNQMD hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import anything under ``oracle/``.  The product
path (``paper_2303_08169_b200``) never does, and shares no code with it.

What it computes (§2.1, Eq. 1 at PAPER.md:119-121 and the Allegro
summary at PAPER.md:128-131; full reading in SURVEY.md §8(c) E1-E9):

* ``oracle.neighbors``  image-aware full directed edge set (brute force + cell list)
* ``oracle.so3``        real spherical harmonics, their gradients, real W3j tables
* ``oracle.irreps``     o3_full irreps / TP paths per layer, parameter counts
* ``oracle.weights_io`` reader of the weight file (own reader)
* ``oracle.allegro``    E, E_i and F = -dE/dr by a hand-written reverse mode
* ``oracle.md``         velocity Verlet, kinetic energy, 5-sigma outlier count

Everything is plain numpy fp64; loops over centre-atom batches only bound memory
(E = sum_i E_i and each E_i depends only on its own row of edges).

Parity status: every function is pinned by ``tests/test_oracle_*.py`` against
brute force, closed forms, finite differences, symmetry invariants, Table 2's
parameter counts or an independent scalar code.  The ABSOLUTE values of E and F
are *parity unpinned* against the paper: the paper prints no energies/forces
(no weights exist); they are pinned only by the invariants above.
"""
