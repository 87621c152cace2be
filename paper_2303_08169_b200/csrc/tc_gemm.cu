// tc_gemm.cu -- tcgen05 tensor-core GEMM (3xTF32) with TMA-fed operands, TMEM
// accumulators and the fused epilogues of gemm.cuh.
//
// One CTA per SM walks 128-row tiles of A (persistent); the N-tiles of a wide contraction are
// sibling CTAs of the same launch walking the same M-tiles (A comes from HBM once, from L2 for
// the sibling).  Warp roles (352 threads):
//   warp 8      TMA producer: A[128 x 32] fp32 K-blocks (SWIZZLE_128B) into a ring of raw
//               SMEM stages (from a second tensor map past K1 for two-operand contractions);
//               the W image of this N-tile once (cp.async.bulk).
//   warps 0-3   split warpgroup (thread = row = TMEM lane): reads its row of a raw stage
//               (applying SiLU first when the operand is a stored pre-activation, silu_a),
//               a_hi = a with the low 13 mantissa bits cleared, a_lo = a - a_hi, and writes
//               both into a TMEM A stage with tcgen05.st (the raw stage is freed at once).
//   warp 9      MMA issuer (whole warp, one elect.sync leader issues): per K-block 4 x K=8
//               steps of tcgen05.mma.kind::tf32 (A from TMEM, W from SMEM)
//                 D += a_hi w_lo;  D += a_lo w_hi;  D += a_hi w_hi
//               into a ring of TMEM accumulators [128 lanes x N_t fp32 columns] (2-4 deep);
//               tcgen05.commit frees the TMEM A stage / publishes the accumulator.
//               (Optional "stacked" variant for N_t <= 64, off by default: one MMA
//               a_hi [w_hi | w_lo] of width 2 N_t into [D | D'], the epilogue adds D + D'.)
//   warps 4-7   epilogue warpgroup: tcgen05.ld 32x32b (thread = row), fused epilogue; each
//               [32 rows x 32 cols] output box is staged in one of the warp's two swizzled
//               SMEM slots and written by one TMA store (cp.async.bulk.tensor, bulk groups
//               recycle the slots; the saved pre-activation "aux" leaves the same way); the
//               optional row-dot with a second [M][N] operand reads the staged box back in
//               the transposed, coalesced view.  (Fallback without TMA stores: the same
//               slot as a transpose tile, global stores as 4 x 128 B lines.)
//   warp 10     epilogue-input producer: the residual / accumulate input (X or old C) is
//               streamed by TMA in [128 x 32] boxes into a 2-deep SMEM ring ahead of the epilogue.
// Every consumer of a TMA-filled ring slot executes fence.proxy.async.shared::cta before it
// releases the slot (generic-proxy loads vs the async-proxy refill).
// W SMEM descriptors: K-major, SWIZZLE_128B, SBO = 1024 B, version 1 (sm_100).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "tc_gemm.cuh"
#include "tc_ptx.cuh"  // PTX wrappers shared with tp_fused.cu

namespace allegro {
namespace {

constexpr int TC_THREADS = 352;              // 11 warps
constexpr int BLK_K = 32;                    // fp32 per 128-byte K-block
constexpr int ROWS = 128;                    // UMMA M
constexpr int A_BLOCK_BYTES = ROWS * 128;    // 16 KB raw A K-block (TMA, SWIZZLE_128B)
constexpr int STAGE_BYTES = A_BLOCK_BYTES;
constexpr int A_TMEM_COLS = 64;              // one TMEM A stage: hi (32 cols) + lo (32 cols)
constexpr size_t SMEM_LIMIT = 227 * 1024;
constexpr size_t SMEM_RESERVE = 2048;        // barriers + alignment slack
constexpr int STAGE_OUT_BYTES = 32 * 128;    // per epilogue warp: [32 rows x 32 fp32] transpose tile
// per-row epilogue scalars: L1 prefetch a tile ahead + load at the tile start (1), or a register
// loaded a tile ahead (0, the round-2 form; build-time A/B)
#ifndef ALG_TC_ROWPF
#define ALG_TC_ROWPF 1
#endif
constexpr int X_STAGES = 2;                  // epilogue input ring: [128 rows x 32 fp32] TMA boxes
constexpr int X_STAGE_BYTES = ROWS * 128;

// sigmoid via exp2 + fast reciprocal (a few ulp; the parity tolerance is ~1e-6 relative)
// exp2f(x) is MUFU.EX2 for x >= -126 plus a denormal-result fix-up below; 1 + 2^x rounds to 1 there
// anyway, so the bare ex2.approx.ftz gives the same sigmoid bits with three fewer instructions
__device__ __forceinline__ float sigm(float t) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-1.4426950408889634f * t));
  return __fdividef(1.f, 1.f + e);
}
__device__ __forceinline__ float silu(float t) { return t * sigm(t); }
__device__ __forceinline__ float dsilu(float t) {
  const float s = sigm(t);
  return s * (1.f + t * (1.f - s));
}

struct TcParams {
  GemmArgs g;
  const float* wimg;   // N-tile images (hi | lo), tile_floats apart
  size_t tile_floats;
  int n_tiles;         // CTAs blockIdx % n_tiles = N-tile of the same M-tiles (siblings share A via L2)
  int n_tiles_total;   // N-tiles of the whole contraction (row-dot partials when > 1)
  int tile_base;       // first N-tile of this launch
  int N_img;           // N rows of this CTA's W image (= N_t, or N_t / 2 for a CTA pair)
  int N_t;             // tile width (multiple of 16)
  int nK;              // K-blocks of 32
  int nK1;             // K-blocks coming from A (rest from A2)
  int stages;          // raw SMEM ring depth
  int a_stages;        // TMEM A ring depth
  uint32_t w_bytes;    // bytes of the W image (hi + lo)
  int n_mtiles;
  int acc_cols;        // TMEM columns per accumulator (>= N_t, multiple of 32)
  int n_acc;           // accumulator ring depth (2..4)
  int stack;           // 1: stacked hi/lo MMA (N_t in {32, 64})
  uint32_t tmem_cols;  // allocated TMEM columns
  int diag;            // diagnostics: bit0 skip MMAs, bit1 skip global stores
  int has_x;           // the epilogue reads an [M][N] input (X, or old C) through the TMA ring
  int tma_store;       // the output C (and aux) leave by TMA stores of [32 x 32] boxes (no row-dot)
  int store_hint;      // TMA stores carry an L2 evict_first policy
  int out_slots;       // output staging slots per epilogue warp (2, or 4: two C + aux groups in flight)
  int dot_x;           // EPI_R2: the row-dot operand arrives through the X ring (thread = row sums)
};

// v <- s v (the saved pre-activation "aux"); out <- epilogue(v, xin) (xin = X, or old C for EPI_ACC)
template <int NV, int EPI>
__device__ __forceinline__ void epi_apply(const GemmArgs& g, float* v, const float* xin, float ur, float* out) {
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const float pv = g.s * v[j];
    v[j] = pv;
    switch (EPI) {
      case EPI_STORE: out[j] = pv; break;
      case EPI_SILU: out[j] = silu(pv); break;
      case EPI_UMUL_SAVE: out[j] = ur * pv; break;
      case EPI_RESID: out[j] = g.alpha * xin[j] + g.beta * ur * pv; break;
      case EPI_URESID: out[j] = g.alpha * xin[j] + g.beta * ur * pv; break;
      case EPI_USCALE: out[j] = g.beta * ur * pv; break;
      case EPI_ACC: out[j] = xin[j] + pv; break;
      case EPI_ADDX: out[j] = pv + xin[j]; break;
      case EPI_DSILU: out[j] = ur * pv * dsilu(xin[j]); break;
      case EPI_R2: out[j] = pv + xin[j]; break;  // xin = rs2 (vec1 + u vec2), prepared by the caller
      case EPI_ACCX: out[j] = pv + g.alpha * xin[j]; break;
      default: out[j] = pv; break;
    }
  }
}

// Per-warp transpose tile [32 rows][32 fp32] with 16-byte chunks XOR-swizzled by row % 8:
// a thread writing / reading its own row and a warp reading / writing 4 rows x 128 B are
// both bank-conflict free.
__device__ __forceinline__ float4* tile_at(unsigned char* buf, int row, int chunk) {
  return reinterpret_cast<float4*>(buf + row * 128 + ((chunk ^ (row & 7)) << 4));
}
// coalesced global [32 rows x 32 cols] (row stride ld floats) -> thread-row registers
// nc = valid 16-byte chunks per row (8 for 32 columns, 4 for a 16-column tile)
__device__ __forceinline__ void gather_rows(unsigned char* buf, const float* src, int64_t ld, int64_t row0, int64_t M,
                                            int lane, float* dst, int nc) {
  float4 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {  // all 8 coalesced loads in flight before any use
    const int r = (lane >> 3) + 4 * i, c = lane & 7;
    v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row0 + r < M && c < nc) v[i] = __ldg(reinterpret_cast<const float4*>(src + (row0 + r) * ld + 4 * c));
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) *tile_at(buf, (lane >> 3) + 4 * i, lane & 7) = v[i];
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float4 w = *tile_at(buf, lane, c);
    dst[4 * c] = w.x, dst[4 * c + 1] = w.y, dst[4 * c + 2] = w.z, dst[4 * c + 3] = w.w;
  }
  __syncwarp();
}
// thread-row registers -> coalesced global
__device__ __forceinline__ void scatter_rows(unsigned char* buf, float* dst, int64_t ld, int64_t row0, int64_t M, int lane,
                                             const float* src, int nc) {
#pragma unroll
  for (int c = 0; c < 8; ++c) *tile_at(buf, lane, c) = make_float4(src[4 * c], src[4 * c + 1], src[4 * c + 2], src[4 * c + 3]);
  __syncwarp();
  float4 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = *tile_at(buf, (lane >> 3) + 4 * i, lane & 7);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = (lane >> 3) + 4 * i, c = lane & 7;
    if (row0 + r < M && c < nc) __stcs(reinterpret_cast<float4*>(dst + (row0 + r) * ld + 4 * c), v[i]);
  }
  __syncwarp();
}

// scatter_rows + the fused row-dot: while the transposed (coalesced) values v[i] of rows
// (lane >> 3) + 4 i, columns 4 (lane & 7).. are in registers, accumulate v[i] . dq[i] into acc8[i]
// (dq = the row-dot operand, loaded in the same coalesced layout).
__device__ __forceinline__ void scatter_rows_dot(unsigned char* buf, float* dst, int64_t ld, int64_t row0, int64_t M,
                                                 int lane, const float* src, int nc, const float4* dq, float* acc8) {
#pragma unroll
  for (int c = 0; c < 8; ++c) *tile_at(buf, lane, c) = make_float4(src[4 * c], src[4 * c + 1], src[4 * c + 2], src[4 * c + 3]);
  __syncwarp();
  float4 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = *tile_at(buf, (lane >> 3) + 4 * i, lane & 7);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = (lane >> 3) + 4 * i, c = lane & 7;
    if (row0 + r < M && c < nc) {
      __stcs(reinterpret_cast<float4*>(dst + (row0 + r) * ld + 4 * c), v[i]);
      acc8[i] = fmaf(v[i].x, dq[i].x, fmaf(v[i].y, dq[i].y, fmaf(v[i].z, dq[i].z, fmaf(v[i].w, dq[i].w, acc8[i]))));
    }
  }
  __syncwarp();
}

// MODE 0: 3xTF32 (a_hi w_lo, a_lo w_hi, a_hi w_hi); 1: stacked (a_hi [w_hi | w_lo] into the
// adjacent accumulators [D | D'], then a_lo w_hi into D; the epilogue adds D + D'); 2: single-pass
// TF32 (a_hi w_hi; ALLEGRO_PREC_TF32, reported, not gated: SURVEY.md App. C); 4: no MMAs.
template <int MODE, int PAIR>
__device__ __forceinline__ void mma_issuer(const TcParams& p, uint32_t tmem, uint32_t tmem_a, uint32_t wimg, int n_my,
                                           uint64_t* a_full, uint64_t* a_empty, uint64_t* acc_full,
                                           uint64_t* acc_empty) {
  // PAIR: M = 256 over the CTA pair (each CTA's 128 rows), N = the full N_t (each CTA holds N_t / 2 of W)
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(p.N_t >> 3) << 17) |
                         ((uint32_t)((PAIR ? 2 * ROWS : ROWS) >> 4) << 24);
  const uint32_t idesc2 = idesc + ((uint32_t)(p.N_t >> 3) << 17);  // width 2 N_t (stacked)
  const uint32_t wblk = (uint32_t)p.N_img * 128;                    // bytes of one W half-block (hi or lo)
  const uint64_t desc0 = sdesc(wimg);
  const uint64_t dlo = (uint64_t)(wblk >> 4);                        // descriptor step hi -> lo
  __syncwarp();
  const uint32_t L = elect_leader();
  int j = 0;
  uint32_t aph = 0;
  for (int t = 0; t < n_my; ++t) {
    const int a = t % p.n_acc;
    const uint32_t acph = (uint32_t)(t / p.n_acc) & 1u;
    if (PAIR) mbar_wait_cluster(acc_empty + a, acph ^ 1);  // both CTAs' epilogues released it
    else mbar_wait(acc_empty + a, acph ^ 1);
    __syncwarp();
    tc_fence_after();
    const uint32_t d = tmem + (uint32_t)(a * p.acc_cols);
    for (int kb = 0; kb < p.nK; ++kb) {
      if (PAIR) mbar_wait_cluster(a_full + j, aph);  // both CTAs' split warps filled stage j
      else mbar_wait(a_full + j, aph);
      __syncwarp();
      tc_fence_after();
      const uint32_t ahi = tmem_a + (uint32_t)(j * A_TMEM_COLS), alo = ahi + 32;
      const uint64_t dkb = desc0 + (uint64_t)((kb * 2 * wblk) >> 4);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t dwh = dkb + (uint64_t)(k * 2);  // +32 bytes = 8 tf32 of a W row
        const uint64_t dwl = dwh + dlo;
        const uint32_t acc = (kb | k) ? 1u : 0u;
        if constexpr (MODE == 0 && PAIR) {
          mma2_tf32_ts_w(L, d, ahi + 8 * k, dwl, idesc, acc);
          mma2_tf32_ts_w(L, d, alo + 8 * k, dwh, idesc, 1u);
          mma2_tf32_ts_w(L, d, ahi + 8 * k, dwh, idesc, 1u);
        } else if constexpr (MODE == 0) {
          mma_tf32_ts_w(L, d, ahi + 8 * k, dwl, idesc, acc);
          mma_tf32_ts_w(L, d, alo + 8 * k, dwh, idesc, 1u);
          mma_tf32_ts_w(L, d, ahi + 8 * k, dwh, idesc, 1u);
        } else if constexpr (MODE == 1) {
          mma_tf32_ts_w(L, d, ahi + 8 * k, dwh, idesc2, acc);  // [D | D'] += a_hi [w_hi | w_lo]
          mma_tf32_ts_w(L, d, alo + 8 * k, dwh, idesc, 1u);
        } else if constexpr (MODE == 2) {
          mma_tf32_ts_w(L, d, ahi + 8 * k, dwh, idesc, acc);  // single-pass TF32: a_hi w_hi only
        }
      }
      if constexpr (PAIR) {  // multicast: both CTAs' split warps / epilogues see the completion
        mma2_commit_w(L, a_empty + j);
        if (kb == p.nK - 1) mma2_commit_w(L, acc_full + a);
      } else {
        mma_commit_w(L, a_empty + j);
        if (kb == p.nK - 1) mma_commit_w(L, acc_full + a);
      }
      if (++j == p.a_stages) j = 0, aph ^= 1;
    }
  }
}

template <int EPI, int PAIR>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapA2,
              const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapC,
              const __grid_constant__ CUtensorMap mapAux, TcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  // 1024-align inside the __shared__ array (pointer arithmetic keeps the shared address space)
  unsigned char* base = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  unsigned char* w_img = base;  // per K-block: [w_hi rows][w_lo rows]
  unsigned char* stage0 = base + ((p.w_bytes + 1023) & ~1023u);
  unsigned char* out_stage = stage0 + (size_t)p.stages * STAGE_BYTES;  // [4 warps][out_slots][4 KB]
  unsigned char* x_stage = out_stage + 4 * p.out_slots * STAGE_OUT_BYTES;  // [X_STAGES][16 KB] (if has_x)
  uint64_t* bars = reinterpret_cast<uint64_t*>(x_stage + (p.has_x ? X_STAGES * X_STAGE_BYTES : 0));
  uint64_t* raw_full = bars;                          // [stages]  TMA landed
  uint64_t* raw_empty = raw_full + p.stages;          // [stages]  split warps read it
  uint64_t* a_full = raw_empty + p.stages;            // [a_stages] hi/lo in TMEM
  uint64_t* a_empty = a_full + p.a_stages;            // [a_stages] MMAs done with it
  uint64_t* acc_full = a_empty + p.a_stages;          // [n_acc]
  uint64_t* acc_empty = acc_full + 4;                 // [n_acc]
  uint64_t* w_full = acc_empty + 4;
  uint64_t* x_full = w_full + 1;                      // [X_STAGES]
  uint64_t* x_empty = x_full + X_STAGES;              // [X_STAGES]
  uint64_t* peer_w = x_empty + X_STAGES;              // PAIR: the peer CTA's W half has landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(peer_w + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(raw_full + s, 1);
      mbar_init(raw_empty + s, 4);
    }
    for (int s = 0; s < p.a_stages; ++s) {
      mbar_init(a_full + s, PAIR ? 8 : 4);
      mbar_init(a_empty + s, 1);
    }
    for (int a = 0; a < p.n_acc; ++a) {
      mbar_init(acc_full + a, 1);
      mbar_init(acc_empty + a, PAIR ? 8 : 4);
    }
    mbar_init(w_full, 1);
    mbar_init(peer_w, 1);
    for (int s2 = 0; s2 < X_STAGES; ++s2) {
      mbar_init(x_full + s2, 1);
      mbar_init(x_empty + s2, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 9) {
    if (PAIR) tmem_alloc2(tmem_slot, p.tmem_cols);  // the same columns in both CTAs of the pair
    else tmem_alloc(tmem_slot, p.tmem_cols);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();  // both CTAs' barriers exist before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_a = tmem + (uint32_t)(p.n_acc * p.acc_cols);  // A ring after the accumulators
  const uint32_t crank = PAIR ? cluster_ctarank() : 0u;

  // sibling CTAs (one per N-tile) walk the same M-tiles in step, so A is read from HBM once; a CTA
  // PAIR (cluster of 2) instead walks M-tile pairs: CTA r takes M-tile 2 u + r of pair-unit u and
  // holds the N-half r of its pair tile, the pair's M = 256 MMAs produce all N_t columns of both
  // CTAs' rows.  With more than one pair tile (p.n_tiles of them, N_t columns each; l = 2's merged
  // x-bar, whose W image leaves room for 32-column halves only) sibling pairs share the M-tiles.
  const int pu = (int)blockIdx.x / 2;                 // PAIR: cluster index
  const int pt = PAIR ? pu % p.n_tiles : 0;           // PAIR: pair tile
  const int tile = PAIR ? 2 * pt + (int)crank : p.tile_base + (int)blockIdx.x % p.n_tiles;  // W image
  const int grp = PAIR ? pu / p.n_tiles : (int)blockIdx.x / p.n_tiles;
  const int n_grp = PAIR ? (int)gridDim.x / 2 / p.n_tiles : (int)gridDim.x / p.n_tiles;
  const int col0 = PAIR ? pt * p.N_t : tile * p.N_t;
  const int dtile = PAIR ? pt : tile;                 // this CTA's column block of the row-dot partials
  const float* wimg_g = p.wimg + (size_t)tile * p.tile_floats;
  const int n_units = PAIR ? (p.n_mtiles + 1) / 2 : p.n_mtiles;
  const int n_my = n_units > grp ? (n_units - 1 - grp) / n_grp + 1 : 0;
  auto mt = [&](int tt) -> int { return PAIR ? 2 * (grp + tt * n_grp) + (int)crank : grp + tt * n_grp; };

  if (warp == 8) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      mbar_expect_tx(w_full, p.w_bytes);
      const uint32_t chunk = 32768;
      for (uint32_t off = 0; off < p.w_bytes; off += chunk) {
        const uint32_t b = p.w_bytes - off < chunk ? p.w_bytes - off : chunk;
        bulk_load(base + off, reinterpret_cast<const unsigned char*>(wimg_g) + off, b, w_full);
      }
      int s = 0;
      uint32_t ph = 0;
      for (int t = 0; t < n_my; ++t) {
        const int m0 = mt(t) * ROWS;
        for (int kb = 0; kb < p.nK; ++kb) {
          mbar_wait(raw_empty + s, ph ^ 1);
          unsigned char* dst = stage0 + (size_t)s * STAGE_BYTES;
          mbar_expect_tx(raw_full + s, A_BLOCK_BYTES);
          if (kb < p.nK1) tma_load_2d(dst, &mapA, kb * BLK_K, m0, raw_full + s);
          else tma_load_2d(dst, &mapA2, (kb - p.nK1) * BLK_K, m0, raw_full + s);
          if (++s == p.stages) s = 0, ph ^= 1;
        }
      }
    }
  } else if (warp == 10) {
    // ---------------- epilogue-input producer: X (or old C) [128 x 32] boxes by TMA ----------------
    if (lane == 0 && p.has_x) {
      int s2 = 0;
      uint32_t ph = 0;
      for (int t = 0; t < n_my; ++t) {
        const int m0 = mt(t) * ROWS;
        for (int c0 = 0; c0 < p.N_t; c0 += 32) {
          mbar_wait(x_empty + s2, ph ^ 1);
          mbar_expect_tx(x_full + s2, X_STAGE_BYTES);
          tma_load_2d(x_stage + (size_t)s2 * X_STAGE_BYTES, &mapX, col0 + c0, m0, x_full + s2);
          if (++s2 == X_STAGES) s2 = 0, ph ^= 1;
        }
      }
    }
  } else if (warp < 4) {
    // ---------------- split warpgroup: raw smem row -> (hi, lo) TMEM ----------------
    const int row = warp * 32 + lane;  // TMEM lane quarter = warp
    int s = 0, j = 0;
    uint32_t ph = 0, aph = 0;
    auto row_scale_u = [&](int tt) -> float {  // arow_u of this thread's row of tile tt (loaded a tile ahead)
      const int64_t rr = (int64_t)mt(tt) * ROWS + row;
      return (p.g.arow_u != nullptr && tt < n_my && rr < p.g.M) ? __ldg(p.g.arow_u + rr) : 1.f;
    };
    float ru_next = row_scale_u(0);
    for (int t = 0; t < n_my; ++t) {
      const float ru = ru_next;
      ru_next = row_scale_u(t + 1);
      for (int kb = 0; kb < p.nK; ++kb) {
        const float rsc = p.g.arow_u == nullptr ? 1.f : (kb < p.nK1 ? p.g.arow_c1 * ru : p.g.arow_c2);
        mbar_wait(raw_full + s, ph);
        const unsigned char* raw = stage0 + (size_t)s * STAGE_BYTES;
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 v = *reinterpret_cast<const float4*>(raw + row * 128 + ((c ^ (row & 7)) << 4));
          float x[4] = {v.x, v.y, v.z, v.w};
          if (p.g.silu_a) {  // pre-activation operand (SiLU(0) = 0 keeps the zero-filled tail zero)
#pragma unroll
            for (int e = 0; e < 4; ++e) x[e] = silu(x[e]);
          }
          if (p.g.arow_u != nullptr) {
#pragma unroll
            for (int e = 0; e < 4; ++e) x[e] *= rsc;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t h = __float_as_uint(x[e]) & 0xffffe000u;
            hi[4 * c + e] = h;
            lo[4 * c + e] = __float_as_uint(x[e] - __uint_as_float(h));
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // as for the X ring
        __syncwarp();
        if (lane == 0) mbar_arrive(raw_empty + s);
        if (++s == p.stages) s = 0, ph ^= 1;
        mbar_wait(a_empty + j, aph ^ 1);
        tc_fence_after();
        const uint32_t ta = tmem_a + (uint32_t)(j * A_TMEM_COLS) + ((uint32_t)(warp * 32) << 16);
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR) {  // the leader CTA's MMA warp waits for both
#ifndef ALG_PAIR_RELEASE
            mbar_arrive_cluster_relaxed(a_full + j, 0);  // TMEM stores ordered by wait::st + tcgen05 fence
#else
            mbar_arrive_cluster(a_full + j, 0);
#endif
          }
          else mbar_arrive(a_full + j);
        }
        if (++j == p.a_stages) j = 0, aph ^= 1;
      }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer (whole warp, one elected lane issues) ----------------
    mbar_wait(w_full, 0);
    if constexpr (PAIR) {
      if (crank != 0) {  // the peer CTA issues nothing: it reports its W half to the leader
        if (lane == 0) mbar_arrive_cluster(peer_w, 0);
      } else {
        mbar_wait_cluster(peer_w, 0);
        tc_fence_after();
        mma_issuer<0, 1>(p, tmem, tmem_a, smem_u32(w_img), n_my, a_full, a_empty, acc_full, acc_empty);
      }
    } else {
      tc_fence_after();
      if (p.diag & 1) mma_issuer<4, 0>(p, tmem, tmem_a, smem_u32(w_img), n_my, a_full, a_empty, acc_full, acc_empty);
      else if (p.g.single_pass) mma_issuer<2, 0>(p, tmem, tmem_a, smem_u32(w_img), n_my, a_full, a_empty, acc_full, acc_empty);
      else if (p.stack) mma_issuer<1, 0>(p, tmem, tmem_a, smem_u32(w_img), n_my, a_full, a_empty, acc_full, acc_empty);
      else mma_issuer<0, 0>(p, tmem, tmem_a, smem_u32(w_img), n_my, a_full, a_empty, acc_full, acc_empty);
    }
  } else {
    // ---------------- epilogue warpgroup (warps 4..7) ----------------
    const int q = warp & 3;  // TMEM lane quarter
    // EPI_R2's row-dot operand arrives through the X ring (compile-time: the per-lane operand
    // registers of the other epilogues' row-dot would spill this instantiation)
    constexpr bool kDotX = EPI == EPI_R2;
    const bool dotx = kDotX && p.g.dotv != nullptr;
    const GemmArgs& g = p.g;
    constexpr bool kX = EPI == EPI_RESID || EPI == EPI_URESID || EPI == EPI_ADDX || EPI == EPI_DSILU || EPI == EPI_ACCX;
    constexpr bool kAuxEpi = EPI == EPI_SILU || EPI == EPI_UMUL_SAVE || EPI == EPI_RESID;
    const bool want_aux = kAuxEpi && g.aux != nullptr;
    unsigned char* buf = out_stage + (size_t)(p.out_slots * q) * STAGE_OUT_BYTES;  // this warp's slots
    constexpr bool kIn = kX || EPI == EPI_ACC;  // epilogue reads a [M][N] input (X or old C)
    int xs = 0;
    uint32_t xph = 0;
    // per-row scalars (u, and rs2 for EPI_R2): their 128-B lines are prefetched into L1 one tile
    // ahead and loaded at the tile start (a register loaded a tile ahead was spilled at once by
    // the register-capped epilogues -- the spill store waited a DRAM round trip every tile)
    auto row_u = [&](int tt) -> float {
      const int64_t rr = (int64_t)mt(tt) * ROWS + q * 32 + lane;
      return (tt < n_my && rr < g.M && g.u != nullptr) ? __ldg(g.u + rr) : 1.f;
    };
    auto row_rs2 = [&](int tt) -> float {
      const int64_t rr = (int64_t)mt(tt) * ROWS + q * 32 + lane;
      return (EPI == EPI_R2 && tt < n_my && rr < g.M) ? __ldg(g.rs2 + rr) : 0.f;
    };
#if ALG_TC_ROWPF
    auto pf_rows = [&](int tt) {
      const int64_t r0 = (int64_t)mt(tt) * ROWS + q * 32;
      if (lane == 0 && tt < n_my && r0 < g.M) {
        if (g.u != nullptr) asm volatile("prefetch.global.L1 [%0];" ::"l"(g.u + r0));
        if (EPI == EPI_R2) asm volatile("prefetch.global.L1 [%0];" ::"l"(g.rs2 + r0));
      }
    };
    pf_rows(0);
#else
    float u_next = row_u(0), rs2_next = row_rs2(0);
#endif
    int n_st = 0;  // TMA stores issued by this warp
    for (int t = 0; t < n_my; ++t) {
      const int a = t % p.n_acc;
      const uint32_t acph = (uint32_t)(t / p.n_acc) & 1u;
#if ALG_TC_ROWPF
      const float ur = row_u(t), e2_row = row_rs2(t);
      pf_rows(t + 1);
#else
      const float ur = u_next, e2_row = rs2_next;
      u_next = row_u(t + 1);
      rs2_next = row_rs2(t + 1);
#endif
      const int64_t row0 = (int64_t)mt(t) * ROWS + q * 32;
      // the row-dot's read-modify-write target (and 1/u) of this warp's 32 rows (one 128-B line
      // each): warmed in L2 now, so the tile's last step is not a dependent DRAM round trip
      if ((EPI == EPI_ACCX || EPI == EPI_R2 || EPI == EPI_ACC) && g.dotv != nullptr && p.n_tiles_total == 1 &&
          lane == 0 && row0 < g.M) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(g.dot_out + row0));
        if (g.dot_inv_u) asm volatile("prefetch.global.L2 [%0];" ::"l"(g.dot_inv_u + row0));
      }
      mbar_wait(acc_full + a, acph);
      tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * p.acc_cols);
      float acc8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // row-dot partials, rows (lane>>3)+4i
      float dsum = 0.f;  // dot_x: this thread's row-dot
      for (int c0 = 0; c0 < p.N_t; c0 += 32) {
        float v[32], out[32], xin[32];
        float4 dq[8];
        if (!kDotX && g.dotv != nullptr) {  // row-dot operand, coalesced like the stores; in flight during the waits
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int64_t rr = row0 + (lane >> 3) + 4 * i;
            const int cc = 4 * (lane & 7);
            dq[i] = (rr < g.M && cc < p.N_t - c0) ? __ldg(reinterpret_cast<const float4*>(g.dotv + rr * g.N + col0 + c0 + cc))
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          // warm L2 with the next chunk's [32 x 32] block (one 128-B line per lane, no registers held)
          const int tn = c0 + 32 < p.N_t ? t : t + 1, cn = c0 + 32 < p.N_t ? c0 + 32 : 0;
          const int64_t rn = (int64_t)mt(tn) * ROWS + q * 32 + lane;
          if (tn < n_my && rn < g.M)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(g.dotv + rn * g.N + col0 + cn));
        }
        if constexpr (kIn) {
          // this thread's row of the TMA-loaded [128 x 32] input box (SWIZZLE_128B)
          mbar_wait(x_full + xs, xph);
          const unsigned char* xb = x_stage + (size_t)xs * X_STAGE_BYTES;
          const int row = q * 32 + lane;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 w4 = *reinterpret_cast<const float4*>(xb + row * 128 + ((c ^ (row & 7)) << 4));
            xin[4 * c] = w4.x, xin[4 * c + 1] = w4.y, xin[4 * c + 2] = w4.z, xin[4 * c + 3] = w4.w;
          }
          // the slot is refilled by TMA (async proxy) once all four warps released it: order
          // these generic-proxy reads before the release
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(x_empty + xs);
          if (++xs == X_STAGES) xs = 0, xph ^= 1;
        }
        if constexpr (EPI == EPI_R2) {
          const float e2 = e2_row;
          const int cb = col0 + c0;
          if (cb + 32 <= g.N) {  // warp-uniform float4 loads (broadcast)
            const float4* v1 = reinterpret_cast<const float4*>(g.vec1 + cb);
            const float4* v2 = reinterpret_cast<const float4*>(g.vec2 + cb);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float4 a4 = __ldg(v1 + c), b4 = __ldg(v2 + c);
              xin[4 * c] = e2 * fmaf(ur, b4.x, a4.x);
              xin[4 * c + 1] = e2 * fmaf(ur, b4.y, a4.y);
              xin[4 * c + 2] = e2 * fmaf(ur, b4.z, a4.z);
              xin[4 * c + 3] = e2 * fmaf(ur, b4.w, a4.w);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = cb + j;
              xin[j] = col < g.N ? e2 * (__ldg(g.vec1 + col) + ur * __ldg(g.vec2 + col)) : 0.f;
            }
          }
        }
        tmem_ld32(tbase + (uint32_t)c0, v);
        if (p.stack) {  // + a_hi w_lo, accumulated beside D
          float v2[32];
          tmem_ld32(tbase + (uint32_t)(p.N_t + c0), v2);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += v2[j];
        }
        if (p.diag & 2) {  // diagnostics (no stores): still release the row-dot operand's ring slot
          if (dotx) {
            mbar_wait(x_full + xs, xph);
            __syncwarp();
            if (lane == 0) mbar_arrive(x_empty + xs);
            if (++xs == X_STAGES) xs = 0, xph ^= 1;
          }
          continue;
        }
        const int64_t col = col0 + c0;
        const int nc = (p.N_t - c0) >= 32 ? 8 : (p.N_t - c0) / 4;
        epi_apply<32, EPI>(g, v, xin, ur, out);
        if (dotx) {
          // this thread's row of the TMA-loaded [128 x 32] row-dot operand box: sum in column order
          mbar_wait(x_full + xs, xph);
          const unsigned char* xb = x_stage + (size_t)xs * X_STAGE_BYTES;
          const int row = q * 32 + lane;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 d4 = *reinterpret_cast<const float4*>(xb + row * 128 + ((c ^ (row & 7)) << 4));
            dsum = fmaf(out[4 * c], d4.x, dsum);
            dsum = fmaf(out[4 * c + 1], d4.y, dsum);
            dsum = fmaf(out[4 * c + 2], d4.z, dsum);
            dsum = fmaf(out[4 * c + 3], d4.w, dsum);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(x_empty + xs);
          if (++xs == X_STAGES) xs = 0, xph ^= 1;
        }
        if (!kDotX && g.dotv != nullptr && !p.tma_store) {
          scatter_rows_dot(buf, g.C + col, g.N, row0, g.M, lane, out, nc, dq, acc8);
        } else if (p.tma_store) {  // [32 rows x 32 cols] boxes through this warp's two SMEM slots
          if (want_aux) {  // C and aux in one group; wait until the previous group has read both slots
            // with 4 slots two (C, aux) groups alternate: the group of two stores ago must be read
            const int grp2 = p.out_slots == 4 ? (n_st & 1) : 0;
            unsigned char* tc = out_stage + (size_t)(p.out_slots * q + 2 * grp2) * STAGE_OUT_BYTES;
            unsigned char* ta = tc + STAGE_OUT_BYTES;
            if (n_st >= (p.out_slots == 4 ? 2 : 1)) {
              if (lane == 0) {
                if (p.out_slots == 4) bulk_wait_read1();
                else bulk_wait_read0();
              }
              __syncwarp();
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              *tile_at(tc, lane, c) = make_float4(out[4 * c], out[4 * c + 1], out[4 * c + 2], out[4 * c + 3]);
              *tile_at(ta, lane, c) = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> TMA reads
            __syncwarp();
            if (lane == 0) {
              if (p.store_hint) {
                const uint64_t pol = policy_evict_first();
                tma_store_2d_hint(&mapC, (int)col, (int)row0, tc, pol);
                tma_store_2d_hint(&mapAux, (int)col, (int)row0, ta, pol);
              } else {
                tma_store_2d(&mapC, (int)col, (int)row0, tc);
                tma_store_2d(&mapAux, (int)col, (int)row0, ta);
              }
              bulk_commit();
            }
          } else {  // double- (or quad-) buffered: the slot of chunk n_st - out_slots must have been read
            unsigned char* tb =
                out_stage + (size_t)(p.out_slots * q + (n_st & (p.out_slots - 1))) * STAGE_OUT_BYTES;
            if (n_st >= p.out_slots) {
              if (lane == 0) {
                if (p.out_slots == 4) bulk_wait_read3();
                else bulk_wait_read1();
              }
              __syncwarp();
            }
#pragma unroll
            for (int c = 0; c < 8; ++c)
              *tile_at(tb, lane, c) = make_float4(out[4 * c], out[4 * c + 1], out[4 * c + 2], out[4 * c + 3]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> TMA reads
            __syncwarp();
            if (lane == 0) {
              if (p.store_hint) tma_store_2d_hint(&mapC, (int)col, (int)row0, tb, policy_evict_first());
              else tma_store_2d(&mapC, (int)col, (int)row0, tb);
              bulk_commit();
            }
            if (!kDotX && g.dotv != nullptr) {  // fused row-dot on the transposed (coalesced) view of the slot
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float4 o4 = *tile_at(tb, (lane >> 3) + 4 * i, lane & 7);
                acc8[i] = fmaf(o4.x, dq[i].x, fmaf(o4.y, dq[i].y, fmaf(o4.z, dq[i].z, fmaf(o4.w, dq[i].w, acc8[i]))));
              }
            }
          }
          ++n_st;
          continue;  // aux (if any) already stored
        } else {
          scatter_rows(buf, g.C + col, g.N, row0, g.M, lane, out, nc);
        }
        if (want_aux) scatter_rows(buf, g.aux + col, g.N, row0, g.M, lane, v, nc);
      }
      if (g.dotv != nullptr) {  // reduce the 8 lanes of each row; lane (lane & 7) == i writes row (lane>>3)+4i
        float mine = dsum;
        if constexpr (!kDotX) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float t8 = acc8[i];
            t8 += __shfl_xor_sync(0xffffffffu, t8, 1);
            t8 += __shfl_xor_sync(0xffffffffu, t8, 2);
            t8 += __shfl_xor_sync(0xffffffffu, t8, 4);
            if ((lane & 7) == i) mine = t8;
          }
        }
        const int64_t rr = kDotX ? row0 + lane : row0 + (lane >> 3) + 4 * (lane & 7);
        if (rr < g.M) {
          if (p.n_tiles_total > 1) g.dot_part[rr * p.n_tiles_total + dtile] = mine;  // summed by k_dot_parts
          else {
            if (g.dot_inv_u) {  // x^0 = u m: <x-bar^0, m> from <x-bar^0, x^0> (u = 0: u' = 0 there too)
              const float ur = g.dot_inv_u[rr];
              mine = ur != 0.f ? mine / ur : 0.f;
            }
            g.dot_out[rr] += g.dot_coef * mine;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) {  // the leader reuses it once both CTAs read it
#ifndef ALG_PAIR_RELEASE
          mbar_arrive_cluster_relaxed(acc_empty + a, 0);  // TMEM loads completed (wait::ld) + tcgen05 fence
#else
          mbar_arrive_cluster(acc_empty + a, 0);
#endif
        }
        else mbar_arrive(acc_empty + a);
      }
    }
    if (p.tma_store && lane == 0) bulk_wait0();  // the output is complete before the CTA retires
  }
  __syncthreads();
  if (PAIR) cluster_sync_all();  // the leader's last MMAs wrote into this CTA's TMEM
  if (warp == 9) {
    tc_fence_after();
    if (PAIR) tmem_dealloc2(tmem, p.tmem_cols);
    else tmem_dealloc(tmem, p.tmem_cols);
  }
}

__global__ void k_dot_parts(int64_t M, int nt, const float* __restrict__ part, float coef, const float* __restrict__ inv_u,
                            float* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  float sdot = part[r * nt];
  for (int t = 1; t < nt; ++t) sdot += part[r * nt + t];
  if (inv_u) {
    const float ur = inv_u[r];
    sdot = ur != 0.f ? sdot / ur : 0.f;
  }
  out[r] += coef * sdot;
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

void get_encode() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      throw CudaError("cuTensorMapEncodeTiled unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
}

CUtensorMap make_map(const float* ptr, int64_t rows, int cols, int ld, int box_rows = ROWS) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)(rows > 0 ? rows : 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  const cuuint32_t box[2] = {BLK_K, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

}  // namespace

CUtensorMap tc_map_f32(const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                       const uint32_t* box) {
  get_encode();
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  cuuint64_t d[3], st[2];
  cuuint32_t b[3], es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) d[i] = dims[i] > 0 ? dims[i] : 1, b[i] = box[i];
  for (int i = 0; i + 1 < rank; ++i) st[i] = strides_bytes[i];
  const CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(ptr), d, st, b, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

namespace {

// per-device launch state (a process may drive ctxs on several devices)
constexpr int kMaxDev = 64;
int g_num_sms[kMaxDev] = {};
bool g_attr_set[kMaxDev] = {};
std::mutex g_dev_mu;

}  // namespace

TcTuning make_tuning() {
  TcTuning t;
  if (const char* e = std::getenv("ALLEGRO_TC_STACK")) t.stack = std::atoi(e) != 0;  // A/B switches for measurements
  if (const char* e = std::getenv("ALLEGRO_TC_MAXACC")) t.max_acc = std::atoi(e);
  if (const char* e = std::getenv("ALLEGRO_TC_MAXSTAGES")) t.max_stages = std::atoi(e);
  if (const char* e = std::getenv("ALLEGRO_TC_TMASTORE")) t.tma_store = std::atoi(e) != 0;
  if (const char* e = std::getenv("ALLEGRO_TC_STOREHINT")) t.store_hint = std::atoi(e);
  return t;
}
TcTuning g_tc_tuning = make_tuning();

float tf32_hi(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u &= 0xffffe000u;
  float h;
  std::memcpy(&h, &u, 4);
  return h;
}

TcWeight tc_prepare_weight(const std::vector<float>& W, int K, int N, std::vector<void*>& owned) {
  TcWeight t;
  t.K = K;
  t.N = N;
  const int nK = (K + BLK_K - 1) / BLK_K;
  // widest N-tile (multiple of 16 dividing N) whose image leaves room for >= 2 stages
  const size_t budget = SMEM_LIMIT - SMEM_RESERVE - 2 * (size_t)STAGE_BYTES - 8 * (size_t)STAGE_OUT_BYTES -
                        (size_t)X_STAGES * X_STAGE_BYTES;
  int nt = 0;
  for (int c = std::min(N, 256); c >= 16; c -= 16)
    if (N % c == 0 && (size_t)2 * nK * c * 128 <= budget) {
      nt = c;
      break;
    }
  if (nt == 0) throw CudaError("tc_prepare_weight: no N-tile fits shared memory");
  t.N_t = nt;
  t.n_tiles = N / nt;
  t.tile_bytes = (size_t)2 * nK * nt * 128;
  std::vector<float> img(t.tile_bytes / 4 * t.n_tiles, 0.f);
  for (int tile = 0; tile < t.n_tiles; ++tile) {
    float* hi = img.data() + tile * (t.tile_bytes / 4);
    float* lo = hi + (size_t)nt * 128 / 4;  // each K-block holds [hi rows][lo rows]
    for (int n = 0; n < nt; ++n)
      for (int k = 0; k < nK * BLK_K; ++k) {
        const float w = k < K ? W[(size_t)k * N + tile * nt + n] : 0.f;
        const float h = tf32_hi(w);
        const int kb = k / BLK_K, kk = k % BLK_K;
        // byte offset inside the K-block: row n (128 B), 16-byte chunk swizzled by n % 8
        const size_t off = (size_t)kb * 2 * nt * 128 + (size_t)n * 128 + (size_t)(((kk / 4) ^ (n % 8)) * 16) + (kk % 4) * 4;
        hi[off / 4] = h;
        lo[off / 4] = w - h;
      }
  }
  ALG_CUDA(cudaMalloc(&t.dev, img.size() * sizeof(float)));
  ALG_CUDA(cudaMemcpy(t.dev, img.data(), img.size() * sizeof(float), cudaMemcpyHostToDevice));
  owned.push_back(t.dev);
  return t;
}

void tc_gemm(const GemmArgs& g, const TcWeight& w, cudaStream_t st, Profiler* prof) {
  if (g.M == 0) return;
  if (g.N != w.N || g.K != w.K || (g.A2 && g.K1 % BLK_K != 0))
    throw CudaError("tc_gemm: shape mismatch N=" + std::to_string(g.N) + " K=" + std::to_string(g.K));
  get_encode();
  int dev = 0;
  ALG_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDev) throw CudaError("tc_gemm: device ordinal out of range");
  const int nK = (g.K + BLK_K - 1) / BLK_K;
  const int K1 = g.A2 ? g.K1 : g.K;
  const CUtensorMap mA = make_map(g.A, g.M, K1, g.lda);
  const CUtensorMap mA2 = g.A2 ? make_map(g.A2, g.M, g.K - g.K1, g.lda2) : mA;
  const size_t w_bytes = w.tile_bytes;
  const size_t w_round = (w_bytes + 1023) & ~(size_t)1023;
  // EPI_R2 has no [M][N] input: its X ring carries the row-dot operand instead (thread = row sums)
  const bool dot_x = g.epi == EPI_R2 && g.dotv != nullptr;
  if (dot_x && g.N % 32 != 0) throw CudaError("tc_gemm: EPI_R2 row-dot needs N % 32 == 0");
  const bool has_x = g.epi == EPI_RESID || g.epi == EPI_URESID || g.epi == EPI_ADDX || g.epi == EPI_DSILU ||
                     g.epi == EPI_ACC || g.epi == EPI_ACCX || dot_x;
  const bool aux_epi0 = g.aux && (g.epi == EPI_SILU || g.epi == EPI_UMUL_SAVE || g.epi == EPI_RESID);
  // A/B (ALLEGRO_TC_OUTSLOTS=4): two (C, aux) store groups in flight per epilogue warp
  static const int outslots_env = [] {
    const char* e = std::getenv("ALLEGRO_TC_OUTSLOTS");
    return e ? std::atoi(e) : 2;
  }();
  // store-heavy contractions (N >= 2 K: l = 2's TP-linear^T, K = 32) keep four output boxes in flight
  // per epilogue warp (A/B ALLEGRO_TC_STORE4=0)
  static const bool store4_on = [] {
    const char* e = std::getenv("ALLEGRO_TC_STORE4");
    return !e || std::atoi(e) != 0;
  }();
  const bool store4 = store4_on && !aux_epi0 && g.dotv == nullptr && g.N >= 2 * g.K;
  const int out_slots = ((aux_epi0 && outslots_env == 4) || store4) ? 4 : 2;
  const size_t out_bytes = 4 * (size_t)out_slots * STAGE_OUT_BYTES + (has_x ? (size_t)X_STAGES * X_STAGE_BYTES : 0);
  int stages = (int)((SMEM_LIMIT - SMEM_RESERVE - w_round - out_bytes) / STAGE_BYTES);
  stages = std::min(stages, g_tc_tuning.max_stages);
  if (stages < 2) throw CudaError("tc_gemm: shared memory too small for 2 stages");
  const size_t smem = 1024 + w_round + out_bytes + (size_t)stages * STAGE_BYTES + 512;
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (!g_attr_set[dev]) {  // the function attribute is per device
#define ALG_SET(e) ALG_CUDA(cudaFuncSetAttribute(k_tc_gemm<e, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_LIMIT));
      ALG_SET(EPI_STORE) ALG_SET(EPI_SILU) ALG_SET(EPI_UMUL_SAVE) ALG_SET(EPI_RESID) ALG_SET(EPI_URESID)
      ALG_SET(EPI_USCALE) ALG_SET(EPI_ACC) ALG_SET(EPI_ADDX) ALG_SET(EPI_DSILU) ALG_SET(EPI_R2) ALG_SET(EPI_ACCX)
#undef ALG_SET
      ALG_CUDA(cudaFuncSetAttribute(k_tc_gemm<EPI_RESID, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_LIMIT));
      ALG_CUDA(cudaFuncSetAttribute(k_tc_gemm<EPI_ACCX, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_LIMIT));
      ALG_CUDA(cudaFuncSetAttribute(k_tc_gemm<EPI_STORE, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_LIMIT));
      ALG_CUDA(cudaDeviceGetAttribute(&g_num_sms[dev], cudaDevAttrMultiProcessorCount, dev));
      g_attr_set[dev] = true;
    }
  }
  // CTA pair (cta_group::2) for a contraction split into two N-tiles: each CTA of a cluster pair
  // holds one N-half of W and splits only its own A rows (instead of two sibling CTAs splitting the
  // same rows); A/B switch ALLEGRO_TC_PAIR
  static const bool pair_on = [] {  // on by default (with relaxed remote arrivals)
    const char* e = std::getenv("ALLEGRO_TC_PAIR");
    return !e || std::atoi(e) != 0;
  }();
  // (more than two N-tiles: sibling pairs, ALLEGRO_TC_PAIR_MULTI=0 keeps those on single CTAs)
  static const bool pair_multi = [] {
    const char* e = std::getenv("ALLEGRO_TC_PAIR_MULTI");
    return !e || std::atoi(e) != 0;
  }();
  static const bool pair_store = [] {  // plain stores split over N-tiles (l = 2's env contraction); A/B
    const char* e = std::getenv("ALLEGRO_TC_PAIR_STORE");
    return !e || std::atoi(e) != 0;
  }();
  const bool pair = pair_on && (w.n_tiles == 2 || (pair_multi && w.n_tiles % 2 == 0)) &&
                    (g.epi == EPI_RESID || g.epi == EPI_ACCX || (g.epi == EPI_STORE && pair_store)) && !g.single_pass &&
                    g_tc_tuning.diag == 0 &&
                    (w.N_t * 2) % 32 == 0;
  const int n_pt = pair ? w.n_tiles / 2 : 1;  // pair tiles
  TcParams p;
  p.g = g;
  p.N_t = pair ? 2 * w.N_t : w.N_t;
  p.N_img = w.N_t;
  p.nK = nK;
  p.nK1 = g.A2 ? g.K1 / BLK_K : nK;
  p.stages = stages;
  p.w_bytes = (uint32_t)w_bytes;
  p.n_mtiles = (int)((g.M + ROWS - 1) / ROWS);
  // stacked hi/lo MMAs where the tensor pipe paces the kernel (A/B on one B200,
  // profiles/r01_gemm_stack_ab.jsonl): N_t = 32 always, N_t = 64 from K = 64 (at K = 32 the
  // doubled accumulator read makes the epilogue the bottleneck)
  p.stack = (!pair && g_tc_tuning.stack && (w.N_t == 32 || (w.N_t == 64 && g.K >= 64))) ? 1 : 0;
  p.acc_cols = (p.stack ? 2 : 1) * ((p.N_t + 31) / 32 * 32);
  // TMEM: two accumulators + the A ring (64 columns per stage), power of two <= 512
  // a deeper accumulator ring for narrow tiles lets the MMAs run further ahead of the epilogue
  p.n_acc = std::max(2, std::min(g_tc_tuning.max_acc, (512 - 4 * A_TMEM_COLS) / p.acc_cols));
  if (pair) {  // A/B: a deeper accumulator ring at the cost of A stages (ALLEGRO_TC_PAIR_ACC = 3)
    static const int pacc = [] {
      const char* e = std::getenv("ALLEGRO_TC_PAIR_ACC");
      return e ? std::atoi(e) : 2;
    }();
    p.n_acc = std::max(2, std::min(pacc, (512 - 2 * A_TMEM_COLS) / p.acc_cols));
  }
  int a_st = std::min(4, (512 - p.n_acc * p.acc_cols) / A_TMEM_COLS);
  if (a_st < 2) throw CudaError("tc_gemm: TMEM too small");
  p.a_stages = a_st;
  uint32_t cols = 32;
  while (cols < (uint32_t)(p.n_acc * p.acc_cols + a_st * A_TMEM_COLS)) cols <<= 1;
  p.tmem_cols = cols;
  p.diag = g_tc_tuning.diag;
  p.has_x = has_x ? 1 : 0;
  const float* xsrc = dot_x ? g.dotv : (g.epi == EPI_ACC ? g.C : g.X);
  p.dot_x = dot_x ? 1 : 0;
  const CUtensorMap mX = has_x ? make_map(xsrc, g.M, g.N, g.N) : mA;
  const bool aux_epi = g.aux && (g.epi == EPI_SILU || g.epi == EPI_UMUL_SAVE || g.epi == EPI_RESID);
  p.tma_store = (g_tc_tuning.tma_store && w.N_t % 32 == 0 && (p.diag & 2) == 0) ? 1 : 0;
  p.store_hint = g_tc_tuning.store_hint;
  p.out_slots = out_slots;
  const CUtensorMap mC = p.tma_store ? make_map(g.C, g.M, g.N, g.N, 32) : mA;
  const CUtensorMap mAux = (p.tma_store && aux_epi) ? make_map(g.aux, g.M, g.N, g.N, 32) : mA;
  if (g.dotv && (pair ? n_pt : w.n_tiles) != 1 && !g.dot_part)
    throw CudaError("tc_gemm: a row-dot over N-tiles needs dot_part");
  // one launch; CTA b handles N-tile b % n_tiles of M-tile group b / n_tiles
  // (ALLEGRO_TC_COSCHED=0: one launch per N-tile, for A/B measurements)
  static const bool cosched = [] {
    const char* e = std::getenv("ALLEGRO_TC_COSCHED");
    return !e || std::atoi(e) != 0;
  }();
  const int per_launch = pair ? w.n_tiles : (cosched ? w.n_tiles : 1);
  const int groups = pair ? std::max(1, std::min((p.n_mtiles + 1) / 2, g_num_sms[dev] / (2 * n_pt)))
                          : std::max(1, std::min(p.n_mtiles, g_num_sms[dev] / per_launch));
  const int grid = groups * (pair ? 2 * n_pt : per_launch);
  const double mn = (double)g.M * g.N;
  const int n_io = 1 + (g.aux != nullptr) + (g.X != nullptr) + (g.epi == EPI_ACC);
  p.n_tiles = pair ? n_pt : per_launch;
  p.n_tiles_total = pair ? n_pt : w.n_tiles;  // one pair tile's row-dot covers all N columns: no partials
  p.wimg = w.dev;
  p.tile_floats = w.tile_bytes / 4;
  for (int tb = 0; tb < w.n_tiles; tb += per_launch) {
    p.tile_base = tb;
    char tag[96];
    std::snprintf(tag, sizeof(tag), "tc N=%d K=%d epi=%d A2=%d Nt=%d%s", g.N, g.K, g.epi, g.A2 ? 1 : 0, w.N_t,
                  pair ? " pair" : "");
    const double frac = (double)per_launch / w.n_tiles;
    ProfScope ps(prof, st, PK_GEMM, frac * (2.0 * mn * g.K + (g.dotv ? 2.0 * mn : 0.0)),
                 frac * 4.0 * ((double)g.M * g.K + (double)g.K * g.N + mn * (n_io + (g.dotv ? 1 : 0)) + (g.dotv ? 2.0 * g.M : 0.0)),
                 tag);
    if (pair) {  // cluster launch: two CTAs per cluster on one TPC
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)grid);
      cfg.blockDim = dim3(TC_THREADS);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if (g.epi == EPI_RESID) ALG_CUDA(cudaLaunchKernelEx(&cfg, k_tc_gemm<EPI_RESID, 1>, mA, mA2, mX, mC, mAux, p));
      else if (g.epi == EPI_ACCX) ALG_CUDA(cudaLaunchKernelEx(&cfg, k_tc_gemm<EPI_ACCX, 1>, mA, mA2, mX, mC, mAux, p));
      else ALG_CUDA(cudaLaunchKernelEx(&cfg, k_tc_gemm<EPI_STORE, 1>, mA, mA2, mX, mC, mAux, p));
      ALG_LAUNCH_CHECK();
      break;
    }
    switch (g.epi) {
#define ALG_EPI(e) \
  case e: k_tc_gemm<e, 0><<<grid, TC_THREADS, smem, st>>>(mA, mA2, mX, mC, mAux, p); break;
      ALG_EPI(EPI_STORE) ALG_EPI(EPI_SILU) ALG_EPI(EPI_UMUL_SAVE) ALG_EPI(EPI_RESID) ALG_EPI(EPI_URESID)
      ALG_EPI(EPI_USCALE) ALG_EPI(EPI_ACC) ALG_EPI(EPI_ADDX) ALG_EPI(EPI_DSILU) ALG_EPI(EPI_R2) ALG_EPI(EPI_ACCX)
#undef ALG_EPI
      default: throw CudaError("tc_gemm: unknown epilogue");
    }
    ALG_LAUNCH_CHECK();
  }
  if (g.dotv && p.n_tiles_total > 1) {  // dot_out[r] += coef (partial_0 + partial_1 + ...), fixed order
    const int nt = p.n_tiles_total;
    ProfScope ps(prof, st, PK_ROWDOT, (double)g.M * nt, 4.0 * (double)g.M * (nt + 2));
    k_dot_parts<<<ceil_div(g.M, 256), 256, 0, st>>>(g.M, nt, g.dot_part, g.dot_coef, g.dot_inv_u, g.dot_out);
    ALG_LAUNCH_CHECK();
  }
}

}  // namespace allegro
