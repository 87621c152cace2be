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
#include <mutex>
#include <string>

#include "ctx.cuh"
#include "geom.cuh"
#include "layer.cuh"
#include "tc_gemm.cuh"
#include "tc_ptx.cuh"
#include "twobody.cuh"

namespace allegro {
namespace {

std::mutex g_attr_mu;  // guards the per-device attribute tables of the launchers below

constexpr int kRows = 128;
constexpr int kTbThreads = 32 * 9;
constexpr int kBox = 32 * 128;  // [32 rows x 32 fp32] staging box
constexpr float kCSiluTb = 1.6765324703f;

// exp2f(x) is MUFU.EX2 for x >= -126 plus a denormal-result fix-up below; 1 + 2^x rounds to 1 there
// anyway, so the bare ex2.approx.ftz gives the same sigmoid bits with three fewer instructions
__device__ __forceinline__ float sigm_tb(float t) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-1.4426950408889634f * t));
  return __fdividef(1.f, 1.f + e);
}
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

// the geometry of one edge and its first two-body layer, exactly as k_geom (model.cu); s4 = W0 rows
// 0..11 as float4 (SMEM in the forward, global / L1 broadcast in the reverse); Y only when y != nullptr
template <bool kY>
__device__ __forceinline__ void geom_row(const TbParams& p, const float4* s4, int32_t i, int32_t a, float& uu, float* y,
                                         float* a1, float* r) {
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
  if constexpr (kY) {
    const float inv = 1.f / d;
    const float nv[3] = {r[0] * inv, r[1] * inv, r[2] * inv};
    sh_eval(nv, y, p.gp.lmax);
  }
}

__device__ __forceinline__ void prefetch_l1(const void* ptr) { asm volatile("prefetch.global.L1 [%0];" ::"l"(ptr)); }

// The edge endpoints of a group's NEXT tile are loaded one tile ahead, and once they have arrived the
// positions / species they point at are prefetched into L1: the dependent index -> position gather
// is otherwise exposed on every tile (the row warps are few; their latency is the kernel's bound).
struct NextIdx {
  int32_t i = 0, a = 0;
  __device__ __forceinline__ void load(const TbParams& p, int64_t e) {
    if (e < p.ch.n_e) i = __ldg(p.cidx + p.ch.e0 + e), a = __ldg(p.nbr + p.ch.e0 + e);
  }
  __device__ __forceinline__ void prefetch(const TbParams& p) const {
    prefetch_l1(p.apos + (int64_t)i * 3);
    prefetch_l1(p.apos + (int64_t)a * 3);
    prefetch_l1(p.species + i);
    prefetch_l1(p.aspec + a);
  }
};

__device__ __forceinline__ int64_t tile_row(int t, int qw, int lane) {
  return (int64_t)((int)blockIdx.x + t * (int)gridDim.x) * kRows + qw * 32 + lane;
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
    NextIdx nx;
    if (g < n_my) nx.load(p, tile_row(g, q, lane));
    for (int t = g; t < n_my; t += 2) {
      const uint32_t ph = (uint32_t)(t >> 1) & 1u;
      const int64_t e0 = (int64_t)((int)blockIdx.x + t * (int)gridDim.x) * kRows;
      const int64_t e = e0 + q * 32 + lane;
      const bool valid = e < p.ch.n_e;
      const int32_t ci = nx.i, ca = nx.a;
      if (t + 2 < n_my) nx.load(p, tile_row(t + 2, q, lane));
      float uu = 0.f, y[9], a[32], r[3];
#pragma unroll
      for (int c = 0; c < 32; ++c) a[c] = 0.f;
      if (valid) {
        geom_row<true>(p, reinterpret_cast<const float4*>(&sw[0][0]), ci, ca, uu, y, a, r);
        p.u[e] = uu;
        if (p.gp.dsh == 4) reinterpret_cast<float4*>(p.Y)[e] = make_float4(y[0], y[1], y[2], y[3]);
        else
#pragma unroll
          for (int k = 0; k < 9; ++k)
            if (k < p.gp.dsh) p.Y[e * p.gp.dsh + k] = y[k];
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
      if (t + 2 < n_my) nx.prefetch(p);
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

// ---------------------------------------------------------------------------------------------
// Reverse: per 128-edge tile (thread = edge row), with a1 and a2 recomputed from the geometry:
//   ab2 = u (s2 xbar0 W2^T) dsilu(a2);  ab1 = (s1 ab2 W1^T) dsilu(a1);  zbar = ab1 W0[Bessel]^T;
//   g = geometry adjoint (geom_bwd_tail, shared with k_geom_bwd)
// -- the arithmetic and order of the unfused reverse (two EPI_DSILU contractions + k_geom_bwd), so
// g is bit-identical to it.  The u-gradient <xbar0, m> stays in layer 0's env^T epilogue (ubar in).
// Warps 0-7: two groups of four row warps, alternate tiles; warps 8 / 9: MMA issuer of group 0 / 1.
// TMEM per group (256 columns): A1 [0, 64), D1 [64, 128) (kept: a2 = s1 D1 is re-read for dsilu),
// xbar0 K-blocks {0, 1} then {2, 3} split into [128, 256), D3 [0, 64) (A1 consumed), A4 (ab2 split)
// [128, 256), D4 [64, 96) (D1 read by then).  xbar0 arrives by per-warp TMA boxes, one tile ahead.
struct TbbParams {
  TbParams f;      // geometry inputs and the forward weights (f.w1img: W1)
  const float* w2t_img;  // W2^T [128][64] image (N 64, 4 K-blocks)
  const float* w1t_img;  // W1^T [64][32] image (N 32, 2 K-blocks)
  uint32_t w2t_bytes, w1t_bytes;
  float s3, s4;    // c / sqrt 64, c / sqrt 32
  const float* ubar;
  const float* ybar;
  float* g;
  const int32_t* rev;
  float* gT;
};

__device__ __forceinline__ float dsilu_tb(float t) {
  const float s = sigm_tb(t);
  return s * (1.f + t * (1.f - s));
}

// split 32 fp32 values read from a swizzled [32 rows x 32 fp32] SMEM box (this thread's row) into TMEM
__device__ __forceinline__ void split_box(uint32_t taddr, const unsigned char* box, int lane) {
  float x[32];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float4 v = *reinterpret_cast<const float4*>(box + lane * 128 + ((c ^ (lane & 7)) << 4));
    x[4 * c] = v.x, x[4 * c + 1] = v.y, x[4 * c + 2] = v.z, x[4 * c + 3] = v.w;
  }
  split_store(taddr, x);
}

__global__ void __launch_bounds__(32 * 8, 1) k_tb_bwd(const __grid_constant__ CUtensorMap map_xbar, const TbbParams q) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  const TbParams& p = q.f;
  // no alignment slack: the dynamic window starts 1024-aligned (after the reserved 1 KB) -- checked
  if (smem_u32(smem_dyn) & 1023u) __trap();
  unsigned char* w1s = smem_dyn;
  unsigned char* w2ts = w1s + ((p.w1bytes + 1023u) & ~1023u);
  unsigned char* w1ts = w2ts + ((q.w2t_bytes + 1023u) & ~1023u);
  unsigned char* slots = w1ts + ((q.w1t_bytes + 1023u) & ~1023u);  // [8 warps][4 K-blocks][4 KB]
  float(*sw)[32] = reinterpret_cast<float(*)[32]>(slots + 32 * kBox);      // W0 rows 0..11 [12][32]
  float(*swt)[kNB] = reinterpret_cast<float(*)[kNB]>(slots + 32 * kBox + 12 * 32 * 4);  // W0 rows 4..11^T [32][8]
  uint64_t* bars = reinterpret_cast<uint64_t*>(slots + 32 * kBox + 12 * 32 * 4 + 32 * kNB * 4);
  uint64_t* a1_full = bars;        // [2]
  uint64_t* d1_full = bars + 2;    // [2]
  uint64_t* x3a_full = bars + 4;   // [2]
  uint64_t* x3a_empty = bars + 6;  // [2]
  uint64_t* x3b_full = bars + 8;   // [2]
  uint64_t* d3_full = bars + 10;   // [2]
  uint64_t* a4_full = bars + 12;   // [2]
  uint64_t* d4_full = bars + 14;   // [2]
  uint64_t* xb_full = bars + 16;   // [8] per row warp
  uint64_t* w_full = bars + 24;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 25);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = threadIdx.x; t < 12 * 32; t += blockDim.x) sw[t / 32][t % 32] = p.w0[t];
  for (int t = threadIdx.x; t < kNB * 32; t += blockDim.x) swt[t % 32][t / 32] = p.w0[4 * 32 + t];
  if (threadIdx.x == 0) {
    for (int g = 0; g < 2; ++g) {
      mbar_init(a1_full + g, 4), mbar_init(d1_full + g, 1), mbar_init(x3a_full + g, 4), mbar_init(x3a_empty + g, 1);
      mbar_init(x3b_full + g, 4), mbar_init(d3_full + g, 1), mbar_init(a4_full + g, 4), mbar_init(d4_full + g, 1);
    }
    for (int w = 0; w < 8; ++w) mbar_init(xb_full + w, 1);
    mbar_init(w_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_my = p.n_tiles > (int)blockIdx.x ? (p.n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  {
    // ---------------- row warps (warp 0 of each group also issues the group's MMAs) ----------------
    if (warp == 0 && lane == 0) {
      mbar_expect_tx(w_full, p.w1bytes + q.w2t_bytes + q.w1t_bytes);
      bulk_load(w1s, p.w1img, p.w1bytes, w_full);
      bulk_load(w2ts, q.w2t_img, q.w2t_bytes, w_full);
      bulk_load(w1ts, q.w1t_img, q.w1t_bytes, w_full);
    }
    const int g = warp >> 2, qw = warp & 3;
    const bool issuer = qw == 0;
    const uint32_t bm = tmem + 256u * g;  // the group's TMEM base (lane 0) for the MMAs
    uint32_t L = 0;
    if (issuer) {
      mbar_wait(w_full, 0);
      tc_fence_after();
      __syncwarp();
      L = elect_leader();
    }
    const uint64_t dw1 = sdesc(smem_u32(w1s)), dw2t = sdesc(smem_u32(w2ts)), dw1t = sdesc(smem_u32(w1ts));
    const uint64_t kb64 = (uint64_t)((2 * 64 * 128) >> 4), kb32 = (uint64_t)((2 * 32 * 128) >> 4);
    const uint32_t b = tmem + 256u * g + ((uint32_t)(qw * 32) << 16);
    unsigned char* myslots = slots + (size_t)(4 * warp) * kBox;
    auto load_xbar = [&](int t) {  // this warp's 32 rows of tile t: four [32 x 32] boxes
      if (lane == 0 && t < n_my) {
        const int row0 = ((int)blockIdx.x + t * (int)gridDim.x) * kRows + qw * 32;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(xb_full + warp, 4 * kBox);
        for (int kb = 0; kb < 4; ++kb) tma_load_2d(myslots + kb * kBox, &map_xbar, 32 * kb, row0, xb_full + warp);
      }
    };
    load_xbar(g);
    NextIdx nx;
    if (g < n_my) nx.load(p, tile_row(g, qw, lane));
    for (int t = g; t < n_my; t += 2) {
      const uint32_t ph = (uint32_t)(t >> 1) & 1u;
      const int64_t e = tile_row(t, qw, lane);
      const bool valid = e < p.ch.n_e;
      const int32_t ci = nx.i, ca = nx.a;
      if (t + 2 < n_my) nx.load(p, tile_row(t + 2, qw, lane));
      float uu = 0.f, a1[32], x[32], r[3] = {0.f, 0.f, 0.f}, ub = 0.f, yb[9];
      int32_t rv = -1;
#pragma unroll
      for (int c = 0; c < 32; ++c) a1[c] = 0.f;
      if (valid) {
        ub = __ldg(q.ubar + e);  // consumed at the end of the tile: in flight across the MMA chain
        rv = __ldg(q.rev + p.ch.e0 + e);
        load_ybar(q.ybar, e, p.gp.dsh, yb);
        geom_row<false>(p, reinterpret_cast<const float4*>(&sw[0][0]), ci, ca, uu, nullptr, a1, r);
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) {  // SiLU(a1) for MMA1 and dsilu(a1) for ab1, one sigmoid each
        const float sg = sigm_tb(a1[c]);
        x[c] = a1[c] * sg;
        a1[c] = sg * (1.f + a1[c] * (1.f - sg));
      }
      tc_fence_after();
      split_store(b, x);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a1_full + g);
      if (issuer) {
        mbar_wait(a1_full + g, ph);
        tc_fence_after();
        mma_kblock(L, bm + 64, bm, dw1, 64, idesc_n(64), true);  // D1 = SiLU(a1) W1
        mma_commit_w(L, d1_full + g);
      }
      // xbar0 K-blocks 0, 1 -> [128, 256) (free: the previous tile's MMA4 completed)
      mbar_wait(xb_full + warp, ph);
      split_box(b + 128, myslots, lane);
      split_box(b + 192, myslots + kBox, lane);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(x3a_full + g);
      if (issuer) {
        mbar_wait(d1_full + g, ph);  // MMA1 done: D3 may overwrite A1
        mbar_wait(x3a_full + g, ph);
        tc_fence_after();
        mma_kblock(L, bm, bm + 128, dw2t, 64, idesc_n(64), true);  // D3 = xbar0 W2^T, K-blocks 0, 1
        mma_kblock(L, bm, bm + 192, dw2t + kb64, 64, idesc_n(64), false);
        mma_commit_w(L, x3a_empty + g);
      }
      mbar_wait(x3a_empty + g, ph);
      tc_fence_after();
      split_box(b + 128, myslots + 2 * kBox, lane);
      split_box(b + 192, myslots + 3 * kBox, lane);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(x3b_full + g);
      if (issuer) {
        mbar_wait(x3b_full + g, ph);
        tc_fence_after();
        mma_kblock(L, bm, bm + 128, dw2t + 2 * kb64, 64, idesc_n(64), false);  // K-blocks 2, 3
        mma_kblock(L, bm, bm + 192, dw2t + 3 * kb64, 64, idesc_n(64), false);
        mma_commit_w(L, d3_full + g);
      }
      load_xbar(t + 2);  // the slots are read: fetch the group's next tile
      if (t + 2 < n_my) nx.prefetch(p);
      // ab2 = u (s3 D3) dsilu(a2), a2 = s1 D1 -> A4 [128, 256)
      mbar_wait(d3_full + g, ph);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float d1[32], d3[32];
        tmem_ld32(b + 64 + 32 * h, d1);
        tmem_ld32(b + 32 * h, d3);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float a2 = p.s1 * d1[c];
          x[c] = uu * (q.s3 * d3[c]) * dsilu_tb(a2);
        }
        split_store(b + 128 + 64 * h, x);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a4_full + g);
      if (issuer) {
        mbar_wait(a4_full + g, ph);
        tc_fence_after();
        mma_kblock(L, bm + 64, bm + 128, dw1t, 32, idesc_n(32), true);  // D4 = ab2 W1^T
        mma_kblock(L, bm + 64, bm + 192, dw1t + kb32, 32, idesc_n(32), false);
        mma_commit_w(L, d4_full + g);
      }
      // ab1 = (s4 D4) dsilu(a1); zbar; g
      mbar_wait(d4_full + g, ph);
      tc_fence_after();
      tmem_ld32(b + 64, x);
      tc_fence_before();
      if (valid) {
        float zbar[kNB];
#pragma unroll
        for (int k = 0; k < kNB; ++k) zbar[k] = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float ab1 = 1.f * (q.s4 * x[j]) * a1[j];  // a1[j] holds dsilu(a1_j)
          const float4* wj = reinterpret_cast<const float4*>(&swt[j][0]);
#pragma unroll
          for (int h = 0; h < kNB / 4; ++h) {
            const float4 w4 = wj[h];
            zbar[4 * h] = fmaf(ab1, w4.x, zbar[4 * h]);
            zbar[4 * h + 1] = fmaf(ab1, w4.y, zbar[4 * h + 1]);
            zbar[4 * h + 2] = fmaf(ab1, w4.z, zbar[4 * h + 2]);
            zbar[4 * h + 3] = fmaf(ab1, w4.w, zbar[4 * h + 3]);
          }
        }
        geom_bwd_tail(p.gp, r, ub, yb, p.s0, zbar, q.g, p.ch.e0 + e, rv, q.gT);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------------------------
// k_tb_bwd2: the same reverse with each row's columns split over TWO warps per lane quarter (16 row
// warps = 2 groups x 8): the kernel is bound by the row warps' ALU issue (35 % issue-active with 8
// warps), and TMEM holds only two tiles' chains, so more warps must share a tile's rows.  Warp
// j = 0..7 of group g: lane quarter j & 3, column half hf = j >> 2.  Each computes the geometry
// (duplicated), its 16 columns of a1 / dsilu(a1) / ab1, its two x-bar0 K-blocks and its 32 columns
// of ab2; the zbar chain (j = 0..31, the unfused order) runs j < 16 in the hf = 0 warp, which hands
// its partial sums to the hf = 1 warp through shared memory, which finishes the chain and the
// geometry adjoint.  Bit-identical to k_tb_bwd.
__device__ __forceinline__ void geom_core(const TbParams& p, int32_t i, int32_t a, float* r, float& uu, float* zb,
                                          int& zi, int& zj) {
  edge_vec(p.apos, i, a, r);
  const float d = sqrtf(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  const float x = d * p.gp.inv_rc;
  uu = 0.f;
  if (x < 1.f) {
    const float x2 = x * x, x3 = x2 * x, x6 = x3 * x3;
    uu = 1.f - 28.f * x6 + 48.f * x6 * x - 21.f * x6 * x2;
  }
  zi = p.species[i], zj = p.aspec[a];
  const float pre = 2.f * p.gp.inv_rc / d;
#pragma unroll
  for (int q = 0; q < kNB; ++q) zb[q] = uu * pre * sinf(p.gp.freq[q] * d * p.gp.inv_rc);
}

// columns 16 hf .. 16 hf + 15 of a1 (the arithmetic of geom_row, per 4-column group)
__device__ __forceinline__ void a1_half(const TbParams& p, const float4* s4, int hf, const float* zb, int zi, int zj,
                                        float* a1) {
#pragma unroll
  for (int k4 = 0; k4 < 4; ++k4) {
    const int c4 = 4 * hf + k4;
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
    a1[4 * k4 + 0] = p.s0 * acc.x;
    a1[4 * k4 + 1] = p.s0 * acc.y;
    a1[4 * k4 + 2] = p.s0 * acc.z;
    a1[4 * k4 + 3] = p.s0 * acc.w;
  }
}

__device__ __forceinline__ void split_store16(uint32_t taddr_hi, uint32_t taddr_lo, const float* x) {
  uint32_t hi[16], lo[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const uint32_t h = __float_as_uint(x[c]) & 0xffffe000u;
    hi[c] = h;
    lo[c] = __float_as_uint(x[c] - __uint_as_float(h));
  }
  tmem_st16(taddr_hi, hi);
  tmem_st16(taddr_lo, lo);
}

// one swizzled [32 x 32] box row -> hi / lo TMEM (two 16-column halves: register budget)
__device__ __forceinline__ void split_box16(uint32_t taddr, const unsigned char* box, int lane) {
#pragma unroll
  for (int hc = 0; hc < 2; ++hc) {
    float x[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = 4 * hc + k;
      const float4 v = *reinterpret_cast<const float4*>(box + lane * 128 + ((c ^ (lane & 7)) << 4));
      x[4 * k] = v.x, x[4 * k + 1] = v.y, x[4 * k + 2] = v.z, x[4 * k + 3] = v.w;
    }
    split_store16(taddr + 16 * hc, taddr + 32 + 16 * hc, x);
  }
}

constexpr int kTb2Warps = 16;

__global__ void __launch_bounds__(32 * kTb2Warps, 1) k_tb_bwd2(const __grid_constant__ CUtensorMap map_xbar,
                                                              const TbbParams q) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  const TbParams& p = q.f;
  if (smem_u32(smem_dyn) & 1023u) __trap();
  unsigned char* w1s = smem_dyn;
  unsigned char* w2ts = w1s + ((p.w1bytes + 1023u) & ~1023u);
  unsigned char* w1ts = w2ts + ((q.w2t_bytes + 1023u) & ~1023u);
  unsigned char* slots = w1ts + ((q.w1t_bytes + 1023u) & ~1023u);  // [16 warps][2 K-blocks][4 KB]
  float(*sw)[32] = reinterpret_cast<float(*)[32]>(slots + 32 * kBox);
  float(*swt)[kNB] = reinterpret_cast<float(*)[kNB]>(slots + 32 * kBox + 12 * 32 * 4);
  uint64_t* bars = reinterpret_cast<uint64_t*>(slots + 32 * kBox + 12 * 32 * 4 + 32 * kNB * 4);
  uint64_t* a1_full = bars;        // [2]
  uint64_t* d1_full = bars + 2;    // [2]
  uint64_t* x3a_full = bars + 4;   // [2]
  uint64_t* x3a_empty = bars + 6;  // [2]
  uint64_t* x3b_full = bars + 8;   // [2]
  uint64_t* d3_full = bars + 10;   // [2]
  uint64_t* a4_full = bars + 12;   // [2]
  uint64_t* d4_full = bars + 14;   // [2]
  uint64_t* xb_full = bars + 16;   // [16] per row warp
  uint64_t* w_full = bars + 32;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 33);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = threadIdx.x; t < 12 * 32; t += blockDim.x) sw[t / 32][t % 32] = p.w0[t];
  for (int t = threadIdx.x; t < kNB * 32; t += blockDim.x) swt[t % 32][t / 32] = p.w0[4 * 32 + t];
  if (threadIdx.x == 0) {
    for (int g = 0; g < 2; ++g) {
      mbar_init(a1_full + g, 8), mbar_init(d1_full + g, 1), mbar_init(x3a_full + g, 8), mbar_init(x3a_empty + g, 1);
      mbar_init(x3b_full + g, 8), mbar_init(d3_full + g, 1), mbar_init(a4_full + g, 8), mbar_init(d4_full + g, 1);
    }
    for (int w = 0; w < kTb2Warps; ++w) mbar_init(xb_full + w, 1);
    mbar_init(w_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_my = p.n_tiles > (int)blockIdx.x ? (p.n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  if (warp == 0 && lane == 0) {
    mbar_expect_tx(w_full, p.w1bytes + q.w2t_bytes + q.w1t_bytes);
    bulk_load(w1s, p.w1img, p.w1bytes, w_full);
    bulk_load(w2ts, q.w2t_img, q.w2t_bytes, w_full);
    bulk_load(w1ts, q.w1t_img, q.w1t_bytes, w_full);
  }
  const int g = warp >> 3, j8 = warp & 7, qw = j8 & 3, hf = j8 >> 2;
  const bool issuer = j8 == 0;
  const uint32_t bm = tmem + 256u * g;
  uint32_t L = 0;
  if (issuer) {
    mbar_wait(w_full, 0);
    tc_fence_after();
    __syncwarp();
    L = elect_leader();
  }
  const uint64_t dw1 = sdesc(smem_u32(w1s)), dw2t = sdesc(smem_u32(w2ts)), dw1t = sdesc(smem_u32(w1ts));
  const uint64_t kb64 = (uint64_t)((2 * 64 * 128) >> 4), kb32 = (uint64_t)((2 * 32 * 128) >> 4);
  const uint32_t b = bm + ((uint32_t)(qw * 32) << 16);
  unsigned char* myslots = slots + (size_t)(2 * warp) * kBox;
  // the zbar hand-off (hf = 0 -> hf = 1 warp of the same quarter) uses the hf = 0 warp's first slot
  float* zhand = reinterpret_cast<float*>(slots + (size_t)(2 * (8 * g + qw)) * kBox) + lane * kNB;
  const int pair_bar = 1 + 4 * g + qw;  // named barrier of the (hf = 0, hf = 1) warp pair
  auto load_xbar = [&](int t) {  // this warp's 32 rows of tile t: K-blocks hf and 2 + hf
    if (lane == 0 && t < n_my) {
      const int row0 = ((int)blockIdx.x + t * (int)gridDim.x) * kRows + qw * 32;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(xb_full + warp, 2 * kBox);
      tma_load_2d(myslots, &map_xbar, 32 * hf, row0, xb_full + warp);
      tma_load_2d(myslots + kBox, &map_xbar, 32 * (2 + hf), row0, xb_full + warp);
    }
  };
  auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory"); };
  load_xbar(g);
  NextIdx nx;
  if (g < n_my) nx.load(p, tile_row(g, qw, lane));
  for (int t = g; t < n_my; t += 2) {
    const uint32_t ph = (uint32_t)(t >> 1) & 1u;
    const int64_t e = tile_row(t, qw, lane);
    const bool valid = e < p.ch.n_e;
    const int32_t ci = nx.i, ca = nx.a;
    if (t + 2 < n_my) nx.load(p, tile_row(t + 2, qw, lane));
    float uu = 0.f, da1[16], x[16], r[3] = {0.f, 0.f, 0.f}, ub = 0.f, yb[9];
    int32_t rv = -1;
#pragma unroll
    for (int c = 0; c < 16; ++c) da1[c] = 0.f;
    if (valid) {
      if (hf == 1) {  // the geometry adjoint's inputs, in flight across the MMA chain
        ub = __ldg(q.ubar + e);
        rv = __ldg(q.rev + p.ch.e0 + e);
        load_ybar(q.ybar, e, p.gp.dsh, yb);
      }
      float zb[kNB];
      int zi, zj;
      geom_core(p, ci, ca, r, uu, zb, zi, zj);
      a1_half(p, reinterpret_cast<const float4*>(&sw[0][0]), hf, zb, zi, zj, da1);
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) {  // SiLU(a1) for MMA1 and dsilu(a1) for ab1, one sigmoid each
      const float sg = sigm_tb(da1[c]);
      x[c] = da1[c] * sg;
      da1[c] = sg * (1.f + da1[c] * (1.f - sg));
    }
    tc_fence_after();
    split_store16(b + 16 * hf, b + 32 + 16 * hf, x);
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(a1_full + g);
    if (issuer) {
      mbar_wait(a1_full + g, ph);
      tc_fence_after();
      mma_kblock(L, bm + 64, bm, dw1, 64, idesc_n(64), true);  // D1 = SiLU(a1) W1
      mma_commit_w(L, d1_full + g);
    }
    // xbar0 K-block hf -> [128 + 64 hf, ...) (free: the previous tile's MMA4 completed)
    mbar_wait(xb_full + warp, ph);
    split_box16(b + 128 + 64 * hf, myslots, lane);
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(x3a_full + g);
    if (issuer) {
      mbar_wait(d1_full + g, ph);  // MMA1 done: D3 may overwrite A1
      mbar_wait(x3a_full + g, ph);
      tc_fence_after();
      mma_kblock(L, bm, bm + 128, dw2t, 64, idesc_n(64), true);  // D3 = xbar0 W2^T, K-blocks 0, 1
      mma_kblock(L, bm, bm + 192, dw2t + kb64, 64, idesc_n(64), false);
      mma_commit_w(L, x3a_empty + g);
    }
    mbar_wait(x3a_empty + g, ph);
    tc_fence_after();
    split_box16(b + 128 + 64 * hf, myslots + kBox, lane);  // K-block 2 + hf
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(x3b_full + g);
    if (issuer) {
      mbar_wait(x3b_full + g, ph);
      tc_fence_after();
      mma_kblock(L, bm, bm + 128, dw2t + 2 * kb64, 64, idesc_n(64), false);  // K-blocks 2, 3
      mma_kblock(L, bm, bm + 192, dw2t + 3 * kb64, 64, idesc_n(64), false);
      mma_commit_w(L, d3_full + g);
    }
    if (hf == 1) {  // the hf = 0 warp's slots carry the zbar hand-off: it refills them later
      load_xbar(t + 2);
    }
    if (t + 2 < n_my) nx.prefetch(p);
    // ab2 columns 32 hf .. 32 hf + 31 = u (s3 D3) dsilu(s1 D1) -> A4 K-block hf
    mbar_wait(d3_full + g, ph);
    tc_fence_after();
#pragma unroll
    for (int hc = 0; hc < 2; ++hc) {
      float d1[16], d3[16];
      tmem_ld16(b + 64 + 32 * hf + 16 * hc, d1);
      tmem_ld16(b + 32 * hf + 16 * hc, d3);
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float a2 = p.s1 * d1[c];
        x[c] = uu * (q.s3 * d3[c]) * dsilu_tb(a2);
      }
      split_store16(b + 128 + 64 * hf + 16 * hc, b + 128 + 64 * hf + 32 + 16 * hc, x);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(a4_full + g);
    if (issuer) {
      mbar_wait(a4_full + g, ph);
      tc_fence_after();
      mma_kblock(L, bm + 64, bm + 128, dw1t, 32, idesc_n(32), true);  // D4 = ab2 W1^T
      mma_kblock(L, bm + 64, bm + 192, dw1t + kb32, 32, idesc_n(32), false);
      mma_commit_w(L, d4_full + g);
    }
    // ab1 columns 16 hf .. 16 hf + 15 = (s4 D4) dsilu(a1); the zbar chain over j in order
    mbar_wait(d4_full + g, ph);
    tc_fence_after();
    tmem_ld16(b + 64 + 16 * hf, x);
    tc_fence_before();
    float zbar[kNB];
    if (hf == 1) {
      pair_sync();  // the hf = 0 warp's partial sums are in shared memory
#pragma unroll
      for (int k = 0; k < kNB; ++k) zbar[k] = zhand[k];
      pair_sync();  // read: the hf = 0 warp may refill its slots
    } else {
#pragma unroll
      for (int k = 0; k < kNB; ++k) zbar[k] = 0.f;
    }
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const int j = 16 * hf + jj;
      const float ab1 = 1.f * (q.s4 * x[jj]) * da1[jj];
      const float4* wj = reinterpret_cast<const float4*>(&swt[j][0]);
#pragma unroll
      for (int h = 0; h < kNB / 4; ++h) {
        const float4 w4 = wj[h];
        zbar[4 * h] = fmaf(ab1, w4.x, zbar[4 * h]);
        zbar[4 * h + 1] = fmaf(ab1, w4.y, zbar[4 * h + 1]);
        zbar[4 * h + 2] = fmaf(ab1, w4.z, zbar[4 * h + 2]);
        zbar[4 * h + 3] = fmaf(ab1, w4.w, zbar[4 * h + 3]);
      }
    }
    if (hf == 0) {
#pragma unroll
      for (int k = 0; k < kNB; ++k) zhand[k] = zbar[k];
      pair_sync();
      pair_sync();
      load_xbar(t + 2);
    } else if (valid) {
      geom_bwd_tail(p.gp, r, ub, yb, p.s0, zbar, q.g, p.ch.e0 + e, rv, q.gT);
    }
    __syncwarp();
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// k_tb_fwd2: the forward with each row's columns over two warps per lane quarter (16 row warps,
// 2 groups x 8; see k_tb_bwd2): warp (q, hf) computes the geometry, a1 columns 16 hf .. + 15, a2
// columns 32 hf .. + 31 and x^0 columns 64 hf .. + 63; hf = 0 writes u, hf = 1 writes Y.  Used when
// nothing but u, Y and x^0 is stored (the fused reverse recomputes a1, a2); bit-identical to k_tb_fwd.
__global__ void __launch_bounds__(32 * 16, 1) k_tb_fwd2(const __grid_constant__ TbMaps maps, const TbParams p) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* base = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  unsigned char* w1s = base;
  unsigned char* w2s = w1s + ((p.w1bytes + 1023u) & ~1023u);
  unsigned char* slots = w2s + ((p.w2bytes + 1023u) & ~1023u);  // [16 warps][2][4 KB]
  float(*sw)[32] = reinterpret_cast<float(*)[32]>(slots + 32 * kBox);
  uint64_t* bars = reinterpret_cast<uint64_t*>(slots + 32 * kBox + 12 * 32 * 4 + 512);
  uint64_t* a1_full = bars;      // [2]
  uint64_t* d1_full = bars + 2;  // [2]
  uint64_t* a2_full = bars + 4;  // [2]
  uint64_t* d2_full = bars + 6;  // [2]
  uint64_t* w_full = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = threadIdx.x; t < 12 * 32; t += blockDim.x) sw[t / 32][t % 32] = p.w0[t];
  if (threadIdx.x == 0) {
    for (int g = 0; g < 2; ++g)
      mbar_init(a1_full + g, 8), mbar_init(d1_full + g, 1), mbar_init(a2_full + g, 8), mbar_init(d2_full + g, 1);
    mbar_init(w_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_my = p.n_tiles > (int)blockIdx.x ? (p.n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  if (warp == 0 && lane == 0) {
    mbar_expect_tx(w_full, p.w1bytes + p.w2bytes);
    bulk_load(w1s, p.w1img, p.w1bytes, w_full);
    bulk_load(w2s, p.w2img, p.w2bytes, w_full);
  }
  const int g = warp >> 3, j8 = warp & 7, q = j8 & 3, hf = j8 >> 2;
  const bool issuer = j8 == 0;
  const uint32_t bm = tmem + 256u * g;
  const uint32_t b = bm + ((uint32_t)(q * 32) << 16);
  uint32_t L = 0;
  if (issuer) {
    mbar_wait(w_full, 0);
    tc_fence_after();
    __syncwarp();
    L = elect_leader();
  }
  const uint64_t dw1 = sdesc(smem_u32(w1s)), dw2 = sdesc(smem_u32(w2s));
  int n_st = 0;
  unsigned char* slot0 = slots + (size_t)(2 * warp) * kBox;
  NextIdx nx;
  if (g < n_my) nx.load(p, tile_row(g, q, lane));
  for (int t = g; t < n_my; t += 2) {
    const uint32_t ph = (uint32_t)(t >> 1) & 1u;
    const int64_t e0 = (int64_t)((int)blockIdx.x + t * (int)gridDim.x) * kRows;
    const int64_t e = e0 + q * 32 + lane;
    const bool valid = e < p.ch.n_e;
    const int32_t ci = nx.i, ca = nx.a;
    if (t + 2 < n_my) nx.load(p, tile_row(t + 2, q, lane));
    float uu = 0.f, a[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) a[c] = 0.f;
    if (valid) {
      float r[3], zb[kNB];
      int zi, zj;
      geom_core(p, ci, ca, r, uu, zb, zi, zj);
      a1_half(p, reinterpret_cast<const float4*>(&sw[0][0]), hf, zb, zi, zj, a);
      if (hf == 0) {
        p.u[e] = uu;
      } else {  // Y(r_hat), as geom_row
        const float d = sqrtf(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
        const float inv = 1.f / d;
        const float nv[3] = {r[0] * inv, r[1] * inv, r[2] * inv};
        float y[9];
        sh_eval(nv, y, p.gp.lmax);
        if (p.gp.dsh == 4) reinterpret_cast<float4*>(p.Y)[e] = make_float4(y[0], y[1], y[2], y[3]);
        else
#pragma unroll
          for (int k = 0; k < 9; ++k)
            if (k < p.gp.dsh) p.Y[e * p.gp.dsh + k] = y[k];
      }
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) a[c] = silu_tb(a[c]);
    tc_fence_after();
    split_store16(b + 16 * hf, b + 32 + 16 * hf, a);
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(a1_full + g);
    if (issuer) {
      mbar_wait(a1_full + g, ph);
      tc_fence_after();
      mma_kblock(L, bm + 64, bm, dw1, 64, idesc_n(64), true);
      mma_commit_w(L, d1_full + g);
    }
    if (t + 2 < n_my) nx.prefetch(p);
    // a2 columns 32 hf .. + 31 = s1 D1; A2 K-block hf = SiLU(a2)
    mbar_wait(d1_full + g, ph);
    tc_fence_after();
#pragma unroll
    for (int hc = 0; hc < 2; ++hc) {
      float v[16];
      tmem_ld16(b + 64 + 32 * hf + 16 * hc, v);
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = silu_tb(p.s1 * v[c]);
      split_store16(b + 128 + 64 * hf + 16 * hc, b + 128 + 64 * hf + 32 + 16 * hc, v);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(a2_full + g);
    if (issuer) {
      mbar_wait(a2_full + g, ph);
      tc_fence_after();
      mma_kblock(L, bm, bm + 128, dw2, 128, idesc_n(128), true);
      mma_kblock(L, bm, bm + 192, dw2 + (uint64_t)((2 * 128 * 128) >> 4), 128, idesc_n(128), false);
      mma_commit_w(L, d2_full + g);
    }
    // x^0 columns 64 hf .. + 63 = u (s2 D2)
    mbar_wait(d2_full + g, ph);
    tc_fence_after();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float v[32];
      tmem_ld32(b + 64 * hf + 32 * h, v);
#pragma unroll
      for (int c = 0; c < 32; ++c) v[c] = uu * (p.s2 * v[c]);
      unsigned char* sl = slot0 + (size_t)(n_st & 1) * kBox;  // the slot used two stores ago has been read
      if (n_st >= 2) {
        if (lane == 0) bulk_wait_read1();
        __syncwarp();
      }
      ++n_st;
      store_box(sl, &maps.x0, 64 * hf + 32 * h, (int)(e0 + q * 32), v, lane);
    }
    tc_fence_before();
    __syncwarp();
  }
  if (lane == 0) bulk_wait0();
  __syncthreads();
  if (warp == 0) {
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
  const size_t smem2 = 1024 + ((p.w1bytes + 1023) & ~1023u) + ((p.w2bytes + 1023) & ~1023u) + 32 * kBox +
                       12 * 32 * 4 + 512 + 256;
  // two warps per lane quarter when only u, Y and x^0 leave the kernel (A/B: ALLEGRO_TB_FWD_SPLIT=1;
  // off: 11.8-12.0 vs 10.4-10.5 ms per C5 step same box, the duplicated geometry costs more than the
  // extra warps win here)
  static const bool split_env = [] {
    const char* e = std::getenv("ALLEGRO_TB_FWD_SPLIT");
    return e && std::atoi(e) != 0;
  }();
  const bool split2 = split_env && !io.a1 && !io.a2 && !io.m;
  int dev = 0;
  ALG_CUDA(cudaGetDevice(&dev));
  static bool attr[64] = {};
  static int nsm[64] = {};
  if (dev < 0 || dev >= 64) throw CudaError("device ordinal out of range");
  {
    std::lock_guard<std::mutex> lk_(g_attr_mu);  // per-device function attributes, set once (thread-safe)
    if (!attr[dev]) {
      ALG_CUDA(cudaFuncSetAttribute(k_tb_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      ALG_CUDA(cudaFuncSetAttribute(k_tb_fwd2, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      ALG_CUDA(cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev));
      attr[dev] = true;
    }
  }
  const int grid = std::max(1, std::min(p.n_tiles, nsm[dev]));
  {
    // algorithmic: the two contractions (2 M N K each) + geometry; bytes: positions / indices in,
    // u, Y, x0 (+ a1, a2, m when the unfused reverse needs them) out
    const double flops = 2.0 * E * (32.0 * 64 + 64.0 * 128);
    const double bytes = (double)E * (8 + 2 * 24 + 4 + 4.0 * p.gp.dsh + 512 + (io.a1 ? 128 : 0) + (io.a2 ? 256 : 0) +
                                      (io.m ? 512 : 0));
    ProfScope ps_(prof, st, PK_TWOBODY, flops, bytes, "two-body fwd (fused)");
    if (split2) k_tb_fwd2<<<grid, 32 * 16, smem2, st>>>(maps, p);
    else k_tb_fwd<<<grid, kTbThreads, smem, st>>>(maps, p);
  }
  ALG_LAUNCH_CHECK();
  if (std::getenv("ALLEGRO_SYNC_CHECK")) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) throw CudaError(std::string("k_tb_fwd: ") + cudaGetErrorString(e));
  }
}

void tb_bwd(const TbIO& io, const TbbIO& bo, cudaStream_t st, Profiler* prof) {
  const int64_t E = io.ch.n_e;
  if (E <= 0) return;
  if (io.w1->tc.N_t != 64 || io.w1->tc.n_tiles != 1 || bo.w2t->tc.N_t != 64 || bo.w2t->tc.n_tiles != 1 ||
      bo.w2t->tc.K != 128 || bo.w1t->tc.N_t != 32 || bo.w1t->tc.n_tiles != 1 || bo.w1t->tc.K != 64)
    throw CudaError("tb_bwd: unexpected two-body weight images");
  TbbParams q;
  std::memset(&q, 0, sizeof(q));
  TbParams& p = q.f;
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
  p.w1img = io.w1->tc.dev;
  p.w1bytes = (uint32_t)io.w1->tc.tile_bytes;
  p.n_tiles = (int)((E + kRows - 1) / kRows);
  q.w2t_img = bo.w2t->tc.dev;
  q.w1t_img = bo.w1t->tc.dev;
  q.w2t_bytes = (uint32_t)bo.w2t->tc.tile_bytes;
  q.w1t_bytes = (uint32_t)bo.w1t->tc.tile_bytes;
  q.s3 = kCSiluTb / std::sqrt(64.f);
  q.s4 = kCSiluTb / std::sqrt(32.f);
  q.ubar = bo.ubar;
  q.ybar = bo.ybar;
  q.g = bo.g;
  q.rev = bo.rev;
  q.gT = bo.gT;
  const CUtensorMap mx = map_rows(bo.xbar, E, 128);
  const size_t smem = ((p.w1bytes + 1023) & ~1023u) + ((q.w2t_bytes + 1023) & ~1023u) +
                      ((q.w1t_bytes + 1023) & ~1023u) + 32 * kBox + 12 * 32 * 4 + 32 * kNB * 4 + 512;
  int dev = 0;
  ALG_CUDA(cudaGetDevice(&dev));
  static const bool split2 = [] {  // A/B switch: each row's columns over two warps (default)
    const char* e = std::getenv("ALLEGRO_TB_BWD_SPLIT");
    return !e || std::atoi(e) != 0;
  }();
  static bool attr[64] = {};
  static int nsm[64] = {};
  if (dev < 0 || dev >= 64) throw CudaError("device ordinal out of range");
  {
    std::lock_guard<std::mutex> lk_(g_attr_mu);  // per-device function attributes, set once (thread-safe)
    if (!attr[dev]) {
      ALG_CUDA(cudaFuncSetAttribute(k_tb_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      ALG_CUDA(cudaFuncSetAttribute(k_tb_bwd2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      ALG_CUDA(cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev));
      attr[dev] = true;
    }
  }
  const int grid = std::max(1, std::min(p.n_tiles, nsm[dev]));
  {
    // algorithmic: three contractions (MMA1 recompute, x-bar W2^T, ab2 W1^T); bytes: x-bar0, u-bar,
    // Y-bar, positions / indices in, g out
    const double flops = 2.0 * E * (32.0 * 64 + 128.0 * 64 + 64.0 * 32);
    const double bytes = (double)E * (8 + 2 * 24 + 512 + 4 + 4.0 * p.gp.dsh + 16);
    ProfScope ps_(prof, st, PK_TWOBODY_BWD, flops, bytes, "two-body bwd (fused)");
    if (split2) k_tb_bwd2<<<grid, 32 * kTb2Warps, smem, st>>>(mx, q);
    else k_tb_bwd<<<grid, 32 * 8, smem, st>>>(mx, q);
  }
  ALG_LAUNCH_CHECK();
  if (std::getenv("ALLEGRO_SYNC_CHECK")) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) throw CudaError(std::string("k_tb_bwd: ") + cudaGetErrorString(e));
  }
}

}  // namespace allegro
