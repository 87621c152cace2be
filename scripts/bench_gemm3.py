"""Stacked-vs-three-MMA comparison of the C5 contraction shapes (tcgen05 3xTF32 GEMM; diagnostics).

Prints one JSON line per shape: ms per launch and algorithmic GB/s for each max_stages."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08169_b200 as pb  # noqa: E402

M = 4 * 1024 * 1024
# (N, K, epi) of the C5 step (bench.py "shapes"); epi ids from csrc/gemm.cuh
SHAPES = [(32, 64, 0), (32, 96, 0), (32, 32, 0), (64, 32, 1), (64, 32, 0), (96, 32, 0), (64, 128, 0),
          (64, 128, 5), (128, 64, 2), (128, 128, 4), (128, 64, 6), (64, 32, 7), (64, 128, 8), (32, 64, 8)]
for N, K, epi in SHAPES:
    aux = epi in (1, 2, 3)
    x = epi in (3, 4, 6, 7, 8)
    byt = 4.0 * M * (K + N * (1 + aux + x))
    out = {"N": N, "K": K, "epi": epi}
    # tma_store hook: 1 = production, -1 = stacked hi/lo MMAs disabled, >= 2 = accumulator ring cap
    for rep in range(2):  # alternate the two variants to cancel drift
        for name, hook in (("stacked", 1), ("three_mma", -1)):
            ms = pb.debug_gemm_bench(M, N, K, epi, iters=5, max_stages=4, tma_store=hook)
            out[f"{name}_gbs_{rep}"] = round(byt / 1e6 / ms, 1)
    print(json.dumps(out), flush=True)
