"""Microbenchmark of the contraction kernels on representative C5 shapes (diagnostics)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08169_b200 as pb
M = 4 * 1024 * 1024
shapes = [(128, 128, 0, "store"), (128, 128, 3, "resid"), (128, 192, 3, "latent"), (64, 128, 0, "env64"),
          (32, 32, 0, "n32k32"), (128, 64, 2, "umul")]
for N, K, epi, name in shapes:
    byt = 4.0 * M * (K + N * (1 + (epi in (2, 3)) + (epi == 3)))
    out = {"shape": name, "N": N, "K": K}
    ms = pb.debug_gemm_bench(M, N, K, epi, precision=pb.PREC_FP32, iters=5)
    out["simt_ms"] = round(ms, 3)
    for ts in (0, 1):
        for st in (2, 3, 4):
            for diag in (0, 1, 2):
                try:
                    ms = pb.debug_gemm_bench(M, N, K, epi, iters=5, tma_store=ts, max_stages=st, diag=diag)
                    out[f"tc_ts{ts}_st{st}_d{diag}"] = round(ms, 3)
                except Exception as e:
                    out[f"tc_ts{ts}_st{st}_d{diag}"] = str(e)[:40]
    out["bytes_GB"] = round(byt / 1e9, 3)
    out["best_tc_gbs"] = round(byt / 1e6 / min(v for k, v in out.items() if k.startswith("tc_") and k.endswith("d0") and isinstance(v, float)), 1)
    print(json.dumps(out), flush=True)
