"""Where does a contraction's time go?  Diagnostic variants of k_tc_gemm (tc_gemm.cuh diag bits):
0 production; 1 no MMAs; 2 no epilogue global traffic; 4 one MMA per K-step; 8 the three 3xTF32
products into three separate accumulators (independent MMAs).  Results of 4/8 are wrong by design."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08169_b200 as pb  # noqa: E402

M = 4 * 1024 * 1024
for N, K, epi in [(32, 96, 0), (32, 64, 0), (64, 128, 0), (128, 128, 0), (128, 64, 2), (128, 128, 4)]:
    out = {"N": N, "K": K, "epi": epi}
    for name, hook, diag in (("stack", 1, 0), ("3mma", -1, 0), ("no_mma", -1, 1), ("no_epi_io", -1, 2),
                             ("1mma", -1, 4), ("3mma_3acc", -1, 8)):
        if diag == 8 and N > 64:
            continue
        ms = pb.debug_gemm_bench(M, N, K, epi, iters=5, tma_store=hook, diag=diag)
        out[name] = round(ms, 4)
    print(json.dumps(out), flush=True)
