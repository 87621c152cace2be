"""Run contraction shapes once each (for an ncu --set full capture of k_tc_gemm).
usage: python scripts/ncu_gemm_shapes.py N,K,epi [N,K,epi ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08169_b200 as pb  # noqa: E402

M = 4 * 1024 * 1024
shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(32, 96, 0), (128, 128, 4)]
for N, K, epi in shapes:
    print(N, K, epi, pb.debug_gemm_bench(M, N, K, epi, iters=1))
