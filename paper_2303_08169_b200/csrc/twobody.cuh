// twobody.cuh -- host entry of the fused geometry + two-body MLP kernels (twobody.cu).
#pragma once
#include <cuda_runtime.h>

#include "ctx.cuh"
#include "geom.cuh"
#include "layer.cuh"
#include "prof.cuh"

namespace allegro {

// Forward over one chunk: reads positions / edges, writes u [E], Y [E][DSH], x0 [E][128] and, when
// the pointers are set, a1 [E][32], a2 [E][64], m [E][128] for the unfused reverse.
struct TbIO {
  ChunkPtrs ch;
  GeomParams gp;
  const double* apos = nullptr;
  const int32_t* cidx = nullptr;
  const int32_t* nbr = nullptr;
  const int32_t* aspec = nullptr;
  const int32_t* species = nullptr;
  const float* w0 = nullptr;  // W0 fp32 [16][32]
  const Wt* w1 = nullptr;     // W1 [32][64] (tensor-core image)
  const Wt* w2 = nullptr;     // W2 [64][128]
  float* u = nullptr;
  float* Y = nullptr;
  float* x0 = nullptr;
  float* a1 = nullptr;
  float* a2 = nullptr;
  float* m = nullptr;
};

void tb_fwd(const TbIO& io, cudaStream_t st, Profiler* prof);

// Reverse over the same chunk (TbIO: geometry inputs, w0, w1; its outputs are not used): x-bar0
// [E][128] (the latent gradient after layer 0), u-bar [E] (complete: <x-bar0, m> included), Y-bar
// [E][DSH] in; g [E][4] out.
struct TbbIO {
  const Wt* w2t = nullptr;  // W2^T [128][64]
  const Wt* w1t = nullptr;  // W1^T [64][32]
  const float* xbar = nullptr;
  const float* ubar = nullptr;
  const float* ybar = nullptr;
  float* g = nullptr;
  const int32_t* rev = nullptr;  // [E] reverse edge (global index) or -1
  float* gT = nullptr;           // [E][4] g scattered to the reverse edge's slot
};

void tb_bwd(const TbIO& io, const TbbIO& bo, cudaStream_t st, Profiler* prof);

}  // namespace allegro
