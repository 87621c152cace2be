"""Determinism of the two-operand (A | A2) contraction with the resnet epilogue (diagnostics)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("ALG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2303_08169_b200 as pb  # noqa: E402

rng = np.random.default_rng(2)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for (M, N, K, K1, epi) in [(90198, 128, 224, 128, 3), (90198, 128, 224, 0, 3), (90198, 128, 224, 128, 4), (90198, 128, 192, 128, 3),
                          (90198, 128, 224, 128, 0), (90198, 64, 224, 128, 3), (300001, 128, 224, 128, 3)]:
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    X = rng.standard_normal((M, N)).astype(np.float32)
    u = rng.uniform(0, 1, M).astype(np.float32)
    code = epi | (K1 << 8)
    if K1 == N:  # X = the first operand (x of the resnet update): pass A's own buffer
        X = A
    ref, ra = pb.debug_gemm_epi(A, W, code, X=X, u=u, want_aux=True)
    exact = 0.75 * (A.astype(np.float64) @ W.astype(np.float64))
    bad, worst = 0, 0
    for _ in range(reps):
        c, a = pb.debug_gemm_epi(A, W, code, X=X, u=u, want_aux=True)
        d = int((c != ref).sum() + (a != ra).sum())
        bad += d > 0
        worst = max(worst, d)
    print(f"M={M} N={N} K={K} K1={K1} epi={epi}: nondeterministic {bad}/{reps} (max {worst} elements), "
          f"aux err {np.abs(ra - exact).max() / np.abs(exact).max():.1e}", flush=True)
