// tp_fused.cuh -- host entry of the fused tensor product + TP-linear kernel (tp_fused.cu).
#pragma once
#include <cuda_runtime.h>

#include "arch.cuh"
#include "layer.cuh"
#include "prof.cuh"

namespace allegro {

// One layer k < L-1 of one chunk: inputs V^k (per in irrep, [E][dim][C]) or, for k = 0, w
// ([E][NW], the w_edge columns) and Y ([E][DSH]); Gamma [n_c][DSH][C] (k_gamma); outputs
// V^{k+1} per out irrep and the scalar paths s = T_0e ([E][n_s C]).  All chunk-local.
struct TplIO {
  ChunkPtrs ch;
  const int32_t* cidx = nullptr;  // global edge -> centre (local atom index)
  const float* G = nullptr;
  const float* Y = nullptr;
  const float* w = nullptr;
  const float* vin[kMaxIr] = {};
  float* vout[kMaxIr] = {};
  float* s = nullptr;
  const float* wimg[kMaxIr] = {};  // TP-linear weight images (tc_prepare_weight, N_t = 32)
  size_t wbytes[kMaxIr] = {};
  double tp_fma_per_edge = 0;      // algorithmic TP FMAs of the layer per edge (profiling)
};

// Backward of one layer k < L-1 (same chunk): inputs V-bar^{k+1} per out irrep, s-bar, V^k (or w,
// Y for k = 0), Gamma; outputs V-bar^k per in irrep (k >= 1) or the w_edge columns of w-bar and
// Y-bar (k = 0, accumulated), and gp [E][DSH][C], each edge's term of Gamma-bar (k_env_adj sums it).
struct TpbIO {
  ChunkPtrs ch;
  const int32_t* cidx = nullptr;
  const float* G = nullptr;
  const float* Y = nullptr;
  const float* w = nullptr;
  const float* vin[kMaxIr] = {};
  const float* vbar_in[kMaxIr] = {};
  const float* sbar = nullptr;
  float* vbar_out[kMaxIr] = {};
  float* wbar = nullptr;
  float* ybar = nullptr;
  float* gp = nullptr;
  const float* wimg[kMaxIr] = {};  // TP-linear^T weight images (N_t = n_to C, K = C)
  size_t wbytes[kMaxIr] = {};
  double tp_fma_per_edge = 0;
};

bool tpl_fwd_supported(int NL, int LMAX, int K);
void tpl_fwd(int NL, int LMAX, int K, const TplIO& io, cudaStream_t st, Profiler* prof);
void tpl_bwd(int NL, int LMAX, int K, const TpbIO& io, cudaStream_t st, Profiler* prof);

}  // namespace allegro
