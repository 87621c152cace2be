"""Repeat tensor-core contractions and compare the outputs bit for bit (diagnostics)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("ALG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2303_08169_b200 as pb  # noqa: E402

rng = np.random.default_rng(0)
M = 300000
for N, K in [(32, 32), (32, 64), (32, 96), (64, 32), (64, 128), (96, 32), (128, 64), (128, 128), (192, 128), (128, 224)]:
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    ref = pb.debug_gemm(A, W, pb.PREC_3XTF32)
    bad = 0
    for it in range(15):
        C = pb.debug_gemm(A, W, pb.PREC_3XTF32)
        bad += int(not np.array_equal(C, ref))
    exact = A.astype(np.float64) @ W.astype(np.float64)
    err = np.abs(ref - exact).max() / np.abs(exact).max()
    print(f"N={N} K={K} nondeterministic={bad}/15 relerr={err:.2e}", flush=True)
