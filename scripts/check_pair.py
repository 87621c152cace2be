"""CTA-pair contraction (cta_group::2) vs the sibling-CTA path on the N-split shapes: the two runs
(ALLEGRO_TC_PAIR=1 / 0, one process each) must agree.  usage: python scripts/check_pair.py out.npz"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2303_08169_b200 as pb

rng = np.random.default_rng(5)
res = {}
for M, K, K1 in ((1000, 192, 0), (5 * 128 + 37, 256, 128), (300_001, 192, 128), (77, 192, 0)):
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = (rng.standard_normal((K, 128)) / np.sqrt(K)).astype(np.float32)
    X = rng.standard_normal((M, 128)).astype(np.float32)
    u = rng.uniform(0, 1, M).astype(np.float32)
    c, a = pb.debug_gemm_epi(A, W, 3 | (K1 << 8), X=X, u=u, want_aux=True)
    ref = 0.75 * (A.astype(np.float64) @ W.astype(np.float64))
    res[f"c_{M}_{K}_{K1}"] = c
    res[f"a_{M}_{K}_{K1}"] = a
    print(M, K, K1, "aux vs fp64 max rel", float(np.abs(a - ref).max() / np.abs(ref).max()), flush=True)
np.savez(sys.argv[1], **res)
