"""Minimal reproducer of the nondeterministic resnet contraction (diagnostics)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("ALG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2303_08169_b200 as pb  # noqa: E402

rng = np.random.default_rng(2)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
M, N, K, K1 = int(os.environ.get("M_ROWS", 300001)), 128, 224, 128
A = rng.standard_normal((M, K)).astype(np.float32)
W = rng.uniform(-1, 1, (K, N)).astype(np.float32)
u = rng.uniform(0, 1, M).astype(np.float32)
for xs in ("self", "copy"):
    X = A if xs == "self" else A[:, :128].copy()
    code = 3 | (K1 << 8)
    ref, ra = pb.debug_gemm_epi(A, W, code, X=X, u=u, want_aux=True)
    bad, worst, rows = 0, 0, set()
    for _ in range(reps):
        c, a = pb.debug_gemm_epi(A, W, code, X=X, u=u, want_aux=True)
        d = (c != ref) | (a != ra)
        if d.any():
            bad += 1
            worst = max(worst, int(d.sum()))
            rows.update(np.nonzero(d.any(axis=1))[0][:8].tolist())
    print(os.environ.get("TAG", ""), f"X={xs}: nondeterministic {bad}/{reps} (max {worst} elements) rows {sorted(rows)[:12]}",
          flush=True)
