// tc_gemm.cuh -- tcgen05 / TMEM / TMA tensor-core GEMM in split precision (3xTF32) for
// the per-edge contractions (ALLEGRO_PREC_3XTF32).  Same epilogues as gemm.cuh.
//
// Single-pass TF32 misses the force bound by ~30x; 3xTF32
// (a = a_hi + a_lo, w = w_hi + w_lo, a w ~ a_hi w_lo + a_lo w_hi + a_hi w_hi) keeps the
// error at the fp32 level.  W is pre-split and pre-swizzled on the host once per weight.
#pragma once
#include <cuda.h>

#include <vector>

#include "gemm.cuh"

namespace allegro {

// A weight W [K][N] prepared for the tensor-core path: per N-tile an SMEM image
// [hi | lo], each [K/32 blocks][N_t rows][128 B, SWIZZLE_128B] of W^T (K-major).
struct TcWeight {
  int K = 0, N = 0, N_t = 0, n_tiles = 0;
  size_t tile_bytes = 0;  // bytes of one N-tile image (hi + lo)
  float* dev = nullptr;   // n_tiles images, contiguous
};

// Build (host) and upload a TcWeight from row-major fp32 W [K][N].
TcWeight tc_prepare_weight(const std::vector<float>& W, int K, int N, std::vector<void*>& owned);

// C = epi(A W) on the tensor cores.  g.W is ignored; K % 32 == 0 (pad), N % 16 == 0.
void tc_gemm(const GemmArgs& g, const TcWeight& w, cudaStream_t st, Profiler* prof);

// fp32 tensor map (rank 2 or 3; dims / box innermost first; strides in bytes of dims 1..rank-1),
// SWIZZLE_128B (the innermost box extent must be 32 fp32), zero fill out of bounds.
CUtensorMap tc_map_f32(const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                       const uint32_t* box);

// Launch tuning / diagnostics (defaults are the production configuration).
struct TcTuning {
  int tma_store = 1;   // TMA-store epilogue when N_t % 32 == 0
  int store_hint = 0;  // L2 evict_first policy on the TMA stores
  int max_stages = 4;  // A-stage ring depth cap
  int max_acc = 4;     // TMEM accumulator ring depth cap (>= 2)
  int stack = 0;       // stacked hi/lo MMAs for N_t in {32, 64} (off: nondeterministic under load)
  int diag = 0;        // bit0: skip MMAs, bit1: skip the epilogue's global traffic
};
extern TcTuning g_tc_tuning;

// tcgen05 contraction modes: 3xTF32 (parity / production) and single-pass TF32 (reported only)
inline bool tc_mode(int precision) { return precision == 1 /*ALLEGRO_PREC_3XTF32*/ || precision == 3 /*ALLEGRO_PREC_TF32*/; }

// Host-side split used for the weights (exposed for tests): hi = fp32 with the low
// 13 mantissa bits cleared (exactly representable in TF32), lo = fp32(x - hi).
float tf32_hi(float x);

}  // namespace allegro
