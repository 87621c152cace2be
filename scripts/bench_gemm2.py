"""Microbenchmark of the small-K / SiLU-epilogue contraction shapes (diagnostics)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08169_b200 as pb
M = 5 * 1024 * 1024
for N, K, epi, name in [(64, 32, 1, "silu_n64k32"), (64, 32, 0, "store_n64k32"), (32, 16, 1, "silu_n32k16"),
                        (64, 128, 8, "dsilu_n64k128"), (64, 128, 0, "store_n64k128"), (128, 64, 2, "umul"),
                        (32, 64, 0, "store_n32k64")]:
    aux = epi in (1, 2, 3)
    x = epi in (3, 4, 7, 8)
    byt = 4.0 * M * (K + N * (1 + aux + x))
    out = {"shape": name}
    for diag in (0, 1, 2):
        ms = pb.debug_gemm_bench(M, N, K, epi, iters=5, diag=diag)
        out[f"d{diag}"] = round(ms, 3)
    out["GBs"] = round(byt / 1e6 / out["d0"], 1)
    print(json.dumps(out), flush=True)
