"""Characterise the wrong rows of the nondeterministic stacked resnet contraction (diagnostics)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("ALG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2303_08169_b200 as pb  # noqa: E402

rng = np.random.default_rng(2)
M, N, K, K1 = 300001, 128, 224, 128
A = rng.standard_normal((M, K)).astype(np.float32)
W = rng.uniform(-1, 1, (K, N)).astype(np.float32)
u = rng.uniform(0, 1, M).astype(np.float32)
X = A[:, :128].copy()
code = 3 | (K1 << 8)
exact_aux = 0.75 * (A.astype(np.float64) @ W.astype(np.float64))
ref_c, ref_a = pb.debug_gemm_epi(A, W, code, X=X, u=u, want_aux=True)
print("ref aux err vs exact", np.abs(ref_a - exact_aux).max() / np.abs(exact_aux).max())
for it in range(8):
    c, a = pb.debug_gemm_epi(A, W, code, X=X, u=u, want_aux=True)
    bad = np.argwhere(a != ref_a)
    if len(bad):
        e1 = np.abs(a - exact_aux)[a != ref_a].max()
        e0 = np.abs(ref_a - exact_aux)[a != ref_a].max()
        print("  this-run err at bad elems", e1, "ref err there", e0, "scale", np.abs(exact_aux).max())
    if len(bad) == 0:
        print("run", it, "ok")
        continue
    rows = np.unique(bad[:, 0])
    cols = np.unique(bad[:, 1])
    print("run", it, "bad elems", len(bad), "rows", rows[:10], "cols", cols[:16], "...", cols[-4:])
    r = rows[0]
    cb = bad[bad[:, 0] == r][:, 1]
    # candidate explanations for row r: stale values from another row? zero?
    v = a[r, cb]
    print("  row", r, "tile", r // 128, "lane", r % 128, "sample got", v[:4], "want", exact_aux[r, cb][:4])
    for rr in (r - 128, r + 128, r - 256, r + 256, r ^ 1):
        if 0 <= rr < M:
            print("   vs row", rr, np.abs(a[rr, cb] - v).max() if len(cb) else None)
    print("  zero?", np.abs(v).max())
