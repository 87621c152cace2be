"""Where does a C5 contraction's time go (round-2 shapes)?  Diagnostic variants of k_tc_gemm
(tc_gemm.cuh diag bits): 0 production; 1 no MMAs; 2 no epilogue global traffic; 4 one MMA per
K-step instead of three (3xTF32 -> 1 pass).  M = one C5 chunk (5.2 M edge rows).  Results of the
diagnostic variants are wrong by design; only their times matter."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08169_b200 as pb  # noqa: E402

M = 5_200_000
for N, K, epi in [(128, 192, 3), (128, 256, 3), (64, 128, 5), (64, 128, 0), (128, 128, 0)]:
    out = {"N": N, "K": K, "epi": epi}
    for name, diag in (("prod", 0), ("no_mma", 1), ("no_epi_io", 2), ("1mma", 4), ("no_mma_no_io", 3)):
        ms = pb.debug_gemm_bench(M, N, K, epi, iters=5, diag=diag)
        out[name] = round(ms, 4)
        out[name + "_gbs"] = round(4.0 * M * (K + N * (2 if epi in (3,) else 1) + (N if epi == 3 else 0)) / ms / 1e6, 1)
    print(json.dumps(out), flush=True)
