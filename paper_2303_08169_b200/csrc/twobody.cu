// twobody.cu -- the edge geometry (E1-E3) and the two-body MLP (E4-E5) of SURVEY.md §8(c) in ONE
// kernel per direction, the MLP's contractions on the tcgen05 tensor cores (3xTF32):
//
//   forward   r_e, d, u(d), B(d) u, Y(r_hat); a1 = z W0 / sqrt 12 (z = [onehot Z_i, onehot Z_j, u B]);
//             a2 = SiLU(a1) W1 c / sqrt 32;  m = SiLU(a2) W2 c / sqrt 64;  x0 = u m
//   reverse   (k_tb_bwd, below) recomputes a1, a2, m from the geometry and runs the chain transposed
//
// so a1, a2 (and in the reverse ab2, ab1, m) never reach HBM.  Arithmetic and order are those of
// k_geom + the two contractions of the unfused path (same 3xTF32 split and MMA sequence), so the
// forward is bit-identical to it.
//
// Tiles of 128 edges (one MMA row per edge).  Warps 0-7: two groups of four "row" warps (thread =
// edge row, TMEM lane quarter = warp & 3) taking alternate tiles; warp 8: TMEM allocator and MMA
// issuer.  TMEM per group (256 columns): A1 [0, 64) and D1 [64, 128), A2 [128, 256), then D2 [0, 128)
// over A1 / D1 once both are consumed.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "ctx.cuh"
#include "geom.cuh"
#include "layer.cuh"
#include "tc_gemm.cuh"
#include "tc_ptx.cuh"
#include "twobody.cuh"

namespace allegro {
namespace {

constexpr int kRows = 128;
constexpr int kTbThreads = 32 * 9;
constexpr int kBox = 32 * 128;  // [32 rows x 32 fp32] staging box
constexpr float kCSiluTb = 1.6765324703f;

__device__ __forceinline__ float sigm_tb(float t) { return __fdividef(1.f, 1.f + exp2f(-1.4426950408889634f * t)); }
__device__ __forceinline__ float silu_tb(float t) { return t * sigm_tb(t); }

struct TbParams {
  ChunkPtrs ch;
  GeomParams gp;
  const double* apos;
  const int32_t* cidx;
  const int32_t* nbr;
  const int32_t* aspec;
  const int32_t* species;
  const float* w0;  // [16][32] fp32 (rows 0..11)
  float s0, s1, s2;  // 1/sqrt 12, c/sqrt 32, c/sqrt 64
  const float* w1img;
  const float* w2img;
  uint32_t w1bytes, w2bytes;
  float* u;
  float* Y;
  float* x0;
  float* a1;  // optional (the unfused reverse needs a1, a2 and m)
  float* a2;
  float* m;
  int n_tiles;
};

// split 32 fp32 values into TF32 hi / lo and store both into TMEM (32x32b, this warp's lane quarter)
__device__ __forceinline__ void split_store(uint32_t taddr, const float* x) {
  uint32_t hi[32], lo[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const uint32_t h = __float_as_uint(x[c]) & 0xffffe000u;
    hi[c] = h;
    lo[c] = __float_as_uint(x[c] - __uint_as_float(h));
  }
  tmem_st32(taddr, hi);
  tmem_st32(taddr + 32, lo);
}

// 3xTF32 MMAs of one K-block (32 fp32 of K): A (hi, lo) from TMEM columns ahi / ahi + 32, W from the
// SMEM image block (hi rows, then lo rows N * 128 bytes later), D in TMEM
__device__ __forceinline__ void mma_kblock(uint32_t L, uint32_t d, uint32_t ahi, uint64_t dkb, uint32_t N,
                                           uint32_t idesc, bool first) {
  const uint32_t alo = ahi + 32;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint64_t dwh = dkb + (uint64_t)(k * 2);
    const uint64_t dwl = dwh + (uint64_t)((N * 128) >> 4);
    mma_tf32_ts_w(L, d, ahi + 8 * k, dwl, idesc, (!first || k) ? 1u : 0u);
    mma_tf32_ts_w(L, d, alo + 8 * k, dwh, idesc, 1u);
    mma_tf32_ts_w(L, d, ahi + 8 * k, dwh, idesc, 1u);
  }
}

__device__ __forceinline__ uint32_t idesc_n(uint32_t N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((uint32_t)(kRows >> 4) << 24);
}

// the geometry of one edge and its first two-body layer, exactly as k_geom (model.cu)
__device__ __forceinline__ void geom_row(const TbParams& p, const float (*sw)[32], int64_t e, float& uu, float* y,
                                         float* a1) {
  const int64_t ge = p.ch.e0 + e;
  const int32_t i = p.cidx[ge], a = p.nbr[ge];
  float r[3];
  edge_vec(p.apos, i, a, r);
  const float d = sqrtf(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  const float x = d * p.gp.inv_rc;
  uu = 0.f;
  if (x < 1.f) {
    const float x2 = x * x, x3 = x2 * x, x6 = x3 * x3;
    uu = 1.f - 28.f * x6 + 48.f * x6 * x - 21.f * x6 * x2;
  }
  const int zi = p.species[i], zj = p.aspec[a];
  const float pre = 2.f * p.gp.inv_rc / d;
  float zb[kNB];
#pragma unroll
  for (int q = 0; q < kNB; ++q) zb[q] = uu * pre * sinf(p.gp.freq[q] * d * p.gp.inv_rc);
  const float4* s4 = reinterpret_cast<const float4*>(&sw[0][0]);
#pragma unroll
  for (int c4 = 0; c4 < 8; ++c4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (zi < 2) acc = s4[zi * 8 + c4];
    if (zj < 2) {
      const float4 b = s4[(2 + zj) * 8 + c4];
      acc = make_float4(acc.x + b.x, acc.y + b.y, acc.z + b.z, acc.w + b.w);
    }
#pragma unroll
    for (int q = 0; q < kNB; ++q) {
      const float4 wq = s4[(4 + q) * 8 + c4];
      acc = make_float4(fmaf(zb[q], wq.x, acc.x), fmaf(zb[q], wq.y, acc.y), fmaf(zb[q], wq.z, acc.z),
                        fmaf(zb[q], wq.w, acc.w));
    }
    a1[4 * c4 + 0] = p.s0 * acc.x;
    a1[4 * c4 + 1] = p.s0 * acc.y;
    a1[4 * c4 + 2] = p.s0 * acc.z;
    a1[4 * c4 + 3] = p.s0 * acc.w;
  }
  const float inv = 1.f / d;
  const float nv[3] = {r[0] * inv, r[1] * inv, r[2] * inv};
  sh_eval(nv, y, p.gp.lmax);
}

// one [32 rows x 32 fp32] box of this warp's rows (thread = row) through a swizzled SMEM slot
__device__ __forceinline__ void store_box(unsigned char* slot, const CUtensorMap* map, int col, int row0, const float* v,
                                          int lane) {
#pragma unroll
  for (int c4 = 0; c4 < 8; ++c4)
    *reinterpret_cast<float4*>(slot + lane * 128 + ((c4 ^ (lane & 7)) << 4)) =
        make_float4(v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2], v[4 * c4 + 3]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(map, col, row0, slot);
    bulk_commit();
  }
}

struct TbMaps {
  CUtensorMap x0, a1, a2, m;  // [E][128], [E][32], [E][64], [E][128]
};

__global__ void __launch_bounds__(kTbThreads, 1) k_tb_fwd(const __grid_constant__ TbMaps maps, const TbParams p) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* base = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  unsigned char* w1s = base;                               // W1 image (K 32 x N 64, hi | lo)
  unsigned char* w2s = w1s + ((p.w1bytes + 1023u) & ~1023u);  // W2 image (K 64 x N 128)
  unsigned char* slots = w2s + ((p.w2bytes + 1023u) & ~1023u);  // [8 warps][2][4 KB]
  float(*sw)[32] = reinterpret_cast<float(*)[32]>(slots + 16 * kBox);  // W0 rows [12][32]
  uint64_t* bars = reinterpret_cast<uint64_t*>(slots + 16 * kBox + 12 * 32 * 4 + 512);
  uint64_t* a1_full = bars;      // [2] per group
  uint64_t* d1_full = bars + 2;  // [2]
  uint64_t* a2_full = bars + 4;  // [2]
  uint64_t* d2_full = bars + 6;  // [2]
  uint64_t* w_full = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = threadIdx.x; t < 12 * 32; t += blockDim.x) sw[t / 32][t % 32] = p.w0[t];
  if (threadIdx.x == 0) {
    for (int g = 0; g < 2; ++g)
      mbar_init(a1_full + g, 4), mbar_init(d1_full + g, 1), mbar_init(a2_full + g, 4), mbar_init(d2_full + g, 1);
    mbar_init(w_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_my = p.n_tiles > (int)blockIdx.x ? (p.n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  if (warp == 8) {
    // ---------------- MMA issuer: per tile MMA1 (K 32 -> N 64) then MMA2 (K 64 -> N 128) ----------------
    if (lane == 0) {
      mbar_expect_tx(w_full, p.w1bytes + p.w2bytes);
      bulk_load(w1s, p.w1img, p.w1bytes, w_full);
      bulk_load(w2s, p.w2img, p.w2bytes, w_full);
    }
    mbar_wait(w_full, 0);
    tc_fence_after();
    __syncwarp();
    const uint32_t L = elect_leader();
    const uint64_t dw1 = sdesc(smem_u32(w1s)), dw2 = sdesc(smem_u32(w2s));
    for (int t = 0; t < n_my; ++t) {
      const int g = t & 1;
      const uint32_t ph = (uint32_t)(t >> 1) & 1u;
      const uint32_t b = tmem + 256u * g;
      mbar_wait(a1_full + g, ph);
      __syncwarp();
      tc_fence_after();
      mma_kblock(L, b + 64, b, dw1, 64, idesc_n(64), true);
      mma_commit_w(L, d1_full + g);
      mbar_wait(a2_full + g, ph);
      __syncwarp();
      tc_fence_after();
      mma_kblock(L, b, b + 128, dw2, 128, idesc_n(128), true);
      mma_kblock(L, b, b + 192, dw2 + (uint64_t)((2 * 128 * 128) >> 4), 128, idesc_n(128), false);
      mma_commit_w(L, d2_full + g);
    }
  } else {
    // ---------------- row warps: two groups of four, alternate tiles ----------------
    const int g = warp >> 2, q = warp & 3;
    const uint32_t b = tmem + 256u * g + ((uint32_t)(q * 32) << 16);
    int n_st = 0;
    for (int t = g; t < n_my; t += 2) {
      const uint32_t ph = (uint32_t)(t >> 1) & 1u;
      const int64_t e0 = (int64_t)((int)blockIdx.x + t * (int)gridDim.x) * kRows;
      const int64_t e = e0 + q * 32 + lane;
      const bool valid = e < p.ch.n_e;
      float uu = 0.f, y[9], a[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) a[c] = 0.f;
      if (valid) {
        geom_row(p, sw, e, uu, y, a);
        p.u[e] = uu;
        if (p.gp.dsh == 4) reinterpret_cast<float4*>(p.Y)[e] = make_float4(y[0], y[1], y[2], y[3]);
        else
          for (int k = 0; k < p.gp.dsh; ++k) p.Y[e * p.gp.dsh + k] = y[k];
      }
      unsigned char* slot0 = slots + (size_t)(2 * warp) * kBox;
      auto next_slot = [&]() -> unsigned char* {  // the slot used two stores ago has been read
        unsigned char* s = slot0 + (size_t)(n_st & 1) * kBox;
        if (n_st >= 2) {
          if (lane == 0) bulk_wait_read1();
          __syncwarp();
        }
        ++n_st;
        return s;
      };
      if (p.a1) store_box(next_slot(), &maps.a1, 0, (int)(e0 + q * 32), a, lane);
      // A1 = SiLU(a1) (the contraction applies SiLU to its operand on load)
#pragma unroll
      for (int c = 0; c < 32; ++c) a[c] = silu_tb(a[c]);
      tc_fence_after();
      split_store(b, a);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a1_full + g);
      // a2 = s1 D1; A2 = SiLU(a2) (two K-blocks)
      mbar_wait(d1_full + g, ph);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[32];
        tmem_ld32(b + 64 + 32 * h, v);
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = p.s1 * v[c];
        if (p.a2) store_box(next_slot(), &maps.a2, 32 * h, (int)(e0 + q * 32), v, lane);
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = silu_tb(v[c]);
        split_store(b + 128 + 64 * h, v);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a2_full + g);
      // m = s2 D2, x0 = u m
      mbar_wait(d2_full + g, ph);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        float v[32];
        tmem_ld32(b + 32 * h, v);
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = p.s2 * v[c];
        if (p.m) store_box(next_slot(), &maps.m, 32 * h, (int)(e0 + q * 32), v, lane);
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = uu * v[c];
        store_box(next_slot(), &maps.x0, 32 * h, (int)(e0 + q * 32), v, lane);
      }
      tc_fence_before();
      __syncwarp();
    }
    if (lane == 0) bulk_wait0();
  }
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

CUtensorMap map_rows(const float* ptr, int64_t rows, int cols) {
  const uint64_t dims[2] = {(uint64_t)cols, (uint64_t)rows};
  const uint64_t strides[1] = {(uint64_t)cols * 4};
  const uint32_t box[2] = {32, 32};
  return tc_map_f32(ptr, 2, dims, strides, box);
}

}  // namespace

void tb_fwd(const TbIO& io, cudaStream_t st, Profiler* prof) {
  const int64_t E = io.ch.n_e;
  if (E <= 0) return;
  if (io.w1->tc.N_t != 64 || io.w1->tc.n_tiles != 1 || io.w2->tc.N_t != 128 || io.w2->tc.n_tiles != 1)
    throw CudaError("tb_fwd: unexpected two-body weight images");
  TbParams p;
  std::memset(&p, 0, sizeof(p));
  p.ch = io.ch;
  p.gp = io.gp;
  p.apos = io.apos;
  p.cidx = io.cidx;
  p.nbr = io.nbr;
  p.aspec = io.aspec;
  p.species = io.species;
  p.w0 = io.w0;
  p.s0 = 1.f / std::sqrt(12.f);
  p.s1 = kCSiluTb / std::sqrt(32.f);
  p.s2 = kCSiluTb / std::sqrt(64.f);
  p.w1img = io.w1->tc.dev;
  p.w2img = io.w2->tc.dev;
  p.w1bytes = (uint32_t)io.w1->tc.tile_bytes;
  p.w2bytes = (uint32_t)io.w2->tc.tile_bytes;
  p.u = io.u;
  p.Y = io.Y;
  p.x0 = io.x0;
  p.a1 = io.a1;
  p.a2 = io.a2;
  p.m = io.m;
  p.n_tiles = (int)((E + kRows - 1) / kRows);
  TbMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  maps.x0 = map_rows(io.x0, E, 128);
  if (io.a1) maps.a1 = map_rows(io.a1, E, 32);
  if (io.a2) maps.a2 = map_rows(io.a2, E, 64);
  if (io.m) maps.m = map_rows(io.m, E, 128);
  const size_t smem = 1024 + ((p.w1bytes + 1023) & ~1023u) + ((p.w2bytes + 1023) & ~1023u) + 16 * kBox + 12 * 32 * 4 +
                      512 + 256;
  int dev = 0;
  ALG_CUDA(cudaGetDevice(&dev));
  static bool attr[64] = {};
  static int nsm[64] = {};
  if (!attr[dev]) {
    ALG_CUDA(cudaFuncSetAttribute(k_tb_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    ALG_CUDA(cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev));
    attr[dev] = true;
  }
  const int grid = std::max(1, std::min(p.n_tiles, nsm[dev]));
  {
    // algorithmic: the two contractions (2 M N K each) + geometry; bytes: positions / indices in,
    // u, Y, x0 (+ a1, a2, m when the unfused reverse needs them) out
    const double flops = 2.0 * E * (32.0 * 64 + 64.0 * 128);
    const double bytes = (double)E * (8 + 2 * 24 + 4 + 4.0 * p.gp.dsh + 512 + (io.a1 ? 128 : 0) + (io.a2 ? 256 : 0) +
                                      (io.m ? 512 : 0));
    ProfScope ps_(prof, st, PK_TWOBODY, flops, bytes, "two-body fwd (fused)");
    k_tb_fwd<<<grid, kTbThreads, smem, st>>>(maps, p);
  }
  ALG_LAUNCH_CHECK();
  if (std::getenv("ALLEGRO_SYNC_CHECK")) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) throw CudaError(std::string("k_tb_fwd: ") + cudaGetErrorString(e));
  }
}

}  // namespace allegro
