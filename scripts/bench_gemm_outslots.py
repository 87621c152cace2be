import sys, json
sys.path.insert(0, '.')
import paper_2303_08169_b200 as pb
M = 5_200_000
out = {}
for N, K, epi in [(128, 64, 3), (64, 64, 3), (64, 128, 3)]:
    out[f"{N}_{K}_{epi}"] = [round(pb.debug_gemm_bench(M, N, K, epi, iters=5, diag=d), 4) for d in (0, 2)]
print(json.dumps(out))
