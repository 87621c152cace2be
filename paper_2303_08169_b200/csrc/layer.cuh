// layer.cuh -- compile-time view of one Allegro layer (arch.cuh's LayerArch) used by the per-edge
// kernels of model.cu and tp_fused.cu, and the chunk descriptor they share.
#pragma once
#include "arch.cuh"
#include "common.cuh"

namespace allegro {

template <int NL, int LMAX, int K>
struct Arch {
  static constexpr LayerArch A = layer_arch(NL, LMAX, K);
  static constexpr int DSH = (LMAX + 1) * (LMAX + 1);
  static constexpr int NENV = LMAX + 1;
  static constexpr int NW = kC * NENV * (K == 0 ? 2 : 1);
  static constexpr int ENV_OFF = K == 0 ? kC * NENV : 0;  // column offset of the env chunk in w
  static constexpr int DIN = A.dim_in;
  static constexpr int DT = A.dim_T;
  static constexpr int t_base(int o) {
    int b = 0;
    for (int q = 0; q < o; ++q) b += ir_dim(A.out.v[q]) * A.n_to[q] * kC;
    return b;
  }
  static constexpr int v_base(int i) {
    int b = 0;
    for (int q = 0; q < i; ++q) b += ir_dim(A.in.v[q]) * kC;
    return b;
  }
};

__host__ __device__ constexpr int lm_l(int m) { return m == 0 ? 0 : (m < 4 ? 1 : 2); }

// model chunk: complete CSR rows of consecutive centre atoms (model.cu)
struct ChunkPtrs {
  int64_t a0, n_c;  // first centre atom, number of centres
  int64_t e0, n_e;  // first edge, number of edges
};



}  // namespace allegro
