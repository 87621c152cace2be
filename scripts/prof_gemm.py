"""Run one tcgen05 GEMM shape a few times (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08169_b200 as pb
N, K, epi = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
print(pb.debug_gemm_bench(2 * 1024 * 1024, N, K, epi, iters=2))
