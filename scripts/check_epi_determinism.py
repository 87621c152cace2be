"""Repeat each fused-epilogue contraction and compare outputs bit for bit (diagnostics)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("ALG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2303_08169_b200 as pb  # noqa: E402

rng = np.random.default_rng(1)
M = 200003
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for epi in range(9):
    for N, K in [(32, 64), (64, 128), (128, 128)]:
        A = rng.standard_normal((M, K)).astype(np.float32)
        W = rng.uniform(-1, 1, (K, N)).astype(np.float32)
        X = rng.standard_normal((M, N)).astype(np.float32)
        u = rng.uniform(0, 1, M).astype(np.float32)
        C0 = rng.standard_normal((M, N)).astype(np.float32)
        ref, ra = pb.debug_gemm_epi(A, W, epi, X=X, u=u, C=C0, want_aux=True)
        bad = 0
        for _ in range(reps):
            c, a = pb.debug_gemm_epi(A, W, epi, X=X, u=u, C=C0, want_aux=True)
            bad += int(not (np.array_equal(c, ref) and np.array_equal(a, ra)))
        print(f"epi={epi} N={N} K={K} nondeterministic={bad}/{reps}", flush=True)
