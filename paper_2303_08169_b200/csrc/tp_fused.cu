// tp_fused.cu -- the tensor product (A8) and the TP-linear channel mix (A9) of one layer in ONE
// kernel: the "uuu" product is computed straight into tensor memory, one MMA row per thread, and
// multiplied by the TP-linear weights on the tcgen05 tensor cores (3xTF32), so T never reaches HBM
// (only its scalar paths s, which the latent update reads).
//
//   T_e[c, p, m3] = sqrt(2 l_o + 1) sum_{m1, m2} W3j[m1, m2, m3] V_e[c, ir1, m1] Gamma_i[c, ir2, m2]
//   V^{k+1}_e[v, o, m] = sum_{p -> o} sum_c T_e[c, p, m] W^k_p[c, v] / sqrt(C n_{->o})
// (§2.1, "tensor products using their irreducible representations"; concrete
// reading SURVEY.md §8(c) E6, D1/D7).  Gamma_i (the environment sum, a segmented
// reduction over the CSR row of i) is formed beforehand by k_gamma (model.cu).
//
// Layout of one 32-edge tile (edges e0 .. e0+31 of the chunk) for out irrep o of dim d:
//   MMA rows r = 32 m3 + e (m-major), so TMEM lane quarter q holds one m3 for all 32 edges;
//   A[r][(p, c)] = T_e[c, p, m3] (K = n_{->o} 32), B = W_o (K x 32, the GEMM path's pre-split
//   image), D[r][v] in TMEM -> V^{k+1}_o[e0 + e][m3][v] by a 3-D TMA store of [32 e x 32 v].
// Warp roles (704 threads, one CTA per SM, persistent over tiles):
//   warps 0-15 TP warps: thread = MMA row (lane quarter w & 3), 8 channels per warp (w >> 2): per
//              (o, p) K-block the warps assigned to o compute T for their m3 from the tile's inputs
//              in SMEM, split it into TF32 hi / lo and tcgen05.st both into a TMEM A stage (the
//              scalar irrep's T also leaves as s).  Irreps are spread over the four quarters (base).
//              (Four warps with 32 channels each were latency-bound: one warp per SMSP, 4.5 us per
//              tile; sixteen warps with 8 channels each: 17 + 16 ms per C5 step for layers 0, 1.)
//   warps 16-19 epilogue: tcgen05.ld of D (thread = row), scale, SMEM box, TMA store.
//   warp 20    producer: the tile's centre indices (coalesced loads), then TMA loads of its V^k
//              rows (or w_edge for layer 0) and bulk copies of Y and of the Gamma rows of its
//              centre atoms into a ring of input stages.
//   warp 21    TMEM allocator and MMA issuer (one elected lane): D += a_hi w_lo + a_lo w_hi +
//              a_hi w_hi per K-step of 8, A from TMEM, W from SMEM.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "ctx.cuh"
#include "layer.cuh"
#include "tc_gemm.cuh"
#include "tc_ptx.cuh"
#include "tp_fused.cuh"

namespace allegro {
namespace {

std::mutex g_attr_mu;  // guards the per-device attribute tables of the launchers below

constexpr int kTile = 32;           // edges per tile
constexpr int kTpWarps = 16;        // TP warps: 4 lane quarters x 4 channel groups
constexpr int kProdWarp = kTpWarps + 4;
constexpr int kMmaWarp = kTpWarps + 5;
constexpr int kThreads = 32 * (kTpWarps + 6);  // 22 warps
constexpr int kATm = 64;            // TMEM columns of one A stage (hi 32 | lo 32)
// TMEM of k_tpl_fwd: kAccBufs accumulator sets (NO x 32 columns each) + the A ring (64 columns per
// stage); build-time A/B (ALG_TPF_ACCBUFS / ALG_TPF_ASTAGES)
#ifndef ALG_TPF_ACCBUFS
#define ALG_TPF_ACCBUFS 2
#endif
#ifndef ALG_TPF_ASTAGES
#define ALG_TPF_ASTAGES 4
#endif
constexpr int kAccBufs = ALG_TPF_ACCBUFS;
constexpr int kAStages = ALG_TPF_ASTAGES;  // TMEM A ring depth
constexpr int kBoxBytes = 32 * 128; // one [32 x 32 fp32] TMA box
constexpr size_t kSmemLimit = 227 * 1024;

template <int NL, int LMAX, int K>
struct Fz {
  using AR = Arch<NL, LMAX, K>;
  static constexpr LayerArch A = AR::A;
  static constexpr int NO = A.out.n;
  static constexpr int NI = A.in.n;
  static constexpr int DSH = AR::DSH;
  static constexpr int dim(int o) { return ir_dim(A.out.v[o]); }
  static constexpr int nto(int o) { return A.n_to[o]; }
  static constexpr bool scalar(int o) { return A.out.v[o].l == 0 && A.out.v[o].p == 1; }
  static constexpr int path_of(int o, int p) {
    for (int q = 0; q < A.n_paths; ++q)
      if (A.out_idx[q] == o && A.out_local[q] == p) return q;
    return -1;
  }
  // K-block (A stage) index of (o, p) within a tile
  static constexpr int kb_of(int o, int p) {
    int b = 0;
    for (int q = 0; q < o; ++q) b += nto(q);
    return b + p;
  }
  static constexpr int n_kb() { return kb_of(NO, 0); }
  // lane quarter of m3 = 0 of irrep o: a greedy spread of the K-block work over the four warps
  static constexpr int base(int o) {
    int load[4] = {0, 0, 0, 0};
    int b_of[kMaxIr] = {};
    bool done[kMaxIr] = {};
    for (int it = 0; it < NO; ++it) {
      int pick = -1;  // heaviest unassigned irrep first
      for (int q = 0; q < NO; ++q)
        if (!done[q] && (pick < 0 || dim(q) * nto(q) > dim(pick) * nto(pick))) pick = q;
      int best = 0, best_cost = 1 << 30;
      for (int b = 0; b < 4; ++b) {
        int cost = 0;
        for (int m = 0; m < dim(pick); ++m) cost = cost > load[(b + m) % 4] + nto(pick) ? cost : load[(b + m) % 4] + nto(pick);
        if (cost < best_cost) best_cost = cost, best = b;
      }
      for (int m = 0; m < dim(pick); ++m) load[(best + m) % 4] += nto(pick);
      b_of[pick] = best;
      done[pick] = true;
    }
    return b_of[o];
  }
  // warp holding m3 = 0 of the scalar irrep (its T values are s)
  static constexpr int s_warp() {
    for (int o = 0; o < NO; ++o)
      if (scalar(o)) return base(o);
    return -1;
  }
  // input stage layout (bytes): V^k per in irrep (K >= 1) or w_edge per l (K = 0), Y, Gamma, header
  static constexpr int in_rows(int i) { return kTile * ir_dim(A.in.v[i]); }
  static constexpr int v_off(int i) {
    int b = 0;
    for (int q = 0; q < i; ++q) b += in_rows(q) * 128;
    return b;
  }
  static constexpr int wv_bytes() { return K == 0 ? AR::NENV * kBoxBytes : v_off(NI); }
  static constexpr int y_off() { return wv_bytes(); }
  static constexpr int g_off() { return y_off() + (K == 0 ? kTile * DSH * 4 : 0); }
  static constexpr int GA = 32;  // Gamma rows staged per tile (atoms); a wider span reads the rest from L2
  static constexpr int g_bytes() { return GA * DSH * 128; }
  static constexpr int h_off() { return g_off() + g_bytes(); }
  static constexpr int stage_bytes() { return (h_off() + 256 + 1023) / 1024 * 1024; }
  static constexpr int acc_cols() { return NO * 32; }
};

struct TplParams {
  int64_t n_e;          // edges of the chunk
  int64_t e0g, a0;      // first global edge / centre atom of the chunk
  const int32_t* cidx;  // [global edges] centre atom (local atom index)
  const float* G;       // [n_c][DSH][C]
  const float* Y;       // [E][DSH]
  float* s;             // [E][n_s C] scalar paths of T
  const float* wimg[kMaxIr];
  uint32_t wbytes[kMaxIr];
  float scale[kMaxIr];
  int n_tiles;
  int stages;           // input ring depth
  int diag;             // diagnostics (ALLEGRO_TPL_DIAG): bit0 no Gamma copy, bit1 no V/w loads, bit2 no TP
                        // reads, bit3 no output stores, bit4 no s stores, bit5 no MMAs
};

struct TplMaps {
  CUtensorMap in[kMaxIr];   // V^k per in irrep [E*dim][32] (K >= 1) or w [E][NW] (K = 0, in[0])
  CUtensorMap out[kMaxIr];  // V^{k+1} per out irrep, 3-D [E][dim][32]
};

template <int NL, int LMAX, int K>
__global__ void __launch_bounds__(kThreads, 1) k_tpl_fwd(const __grid_constant__ TplMaps maps, const TplParams p) {
  using F = Fz<NL, LMAX, K>;
  using AR = typename F::AR;
  constexpr LayerArch A = F::A;
  constexpr int NO = F::NO, DSH = F::DSH, NKB = F::n_kb();
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* base = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  uint32_t woff[kMaxIr + 1];
  woff[0] = 0;
#pragma unroll
  for (int o = 0; o < kMaxIr; ++o) woff[o + 1] = woff[o] + (o < NO ? p.wbytes[o] : 0u);
  unsigned char* w_img = base;
  unsigned char* stage0 = base + ((woff[NO] + 1023u) & ~1023u);
  unsigned char* epi = stage0 + (size_t)p.stages * F::stage_bytes();  // [4 warps][2][4 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi + 8 * kBoxBytes);
  uint64_t* in_full = bars;
  uint64_t* in_empty = in_full + 4;
  uint64_t* a_full = in_empty + 4;
  uint64_t* a_empty = a_full + kAStages;
  uint64_t* acc_full = a_empty + kAStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* w_full = acc_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_full + 1);
  static_assert(kAccBufs >= 1 && kAccBufs <= 2 && kAccBufs * F::acc_cols() + kAStages * kATm <= 512, "TMEM budget");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) mbar_init(in_full + s, 1), mbar_init(in_empty + s, kTpWarps);
    for (int s = 0; s < kAStages; ++s) mbar_init(a_full + s, kTpWarps), mbar_init(a_empty + s, 1);
    for (int b = 0; b < kAccBufs; ++b) mbar_init(acc_full + b, 1), mbar_init(acc_empty + b, 4);
    mbar_init(w_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_a = tmem + (uint32_t)(kAccBufs * F::acc_cols());  // A ring after the accumulator sets
  const int n_my = p.n_tiles > (int)blockIdx.x ? (p.n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  if (warp == kProdWarp) {
    // ---------------- producer ----------------
    if (lane == 0) {
      mbar_expect_tx(w_full, woff[NO]);
      for (int o = 0; o < NO; ++o) bulk_load(w_img + woff[o], p.wimg[o], p.wbytes[o], w_full);
    }
    int s = 0;
    uint32_t ph = 0;
    // centre indices of tile t (the load for tile t + 1 is issued before tile t waits for its stage)
    auto load_ci = [&](int t) -> int {
      const int64_t e0 = (int64_t)((int)blockIdx.x + t * (int)gridDim.x) * kTile;
      return (t < n_my && e0 + lane < p.n_e) ? __ldg(p.cidx + p.e0g + e0 + lane) - (int)p.a0 : 0;
    };
    int ci_next = load_ci(0);
    for (int t = 0; t < n_my; ++t) {
      const int64_t e0 = (int64_t)((int)blockIdx.x + t * (int)gridDim.x) * kTile;
      const int nv = (int)(p.n_e - e0 < kTile ? p.n_e - e0 : kTile);
      const int ci = ci_next;
      ci_next = load_ci(t + 1);
      mbar_wait(in_empty + s, ph ^ 1);
      unsigned char* st = stage0 + (size_t)s * F::stage_bytes();
      int* hdr = reinterpret_cast<int*>(st + F::h_off());
      const int a_lo = __shfl_sync(0xffffffffu, ci, 0);
      const int a_hi = __shfl_sync(0xffffffffu, ci, nv - 1);
      hdr[lane] = lane < nv ? ci - a_lo : 0;  // Gamma row block of this edge's centre
      if (lane == 0) hdr[32] = nv, hdr[33] = a_lo;
      __syncwarp();
      if (lane == 0) {
        const int span = a_hi - a_lo + 1;
        const uint32_t gbytes = (uint32_t)(span < F::GA ? span : F::GA) * DSH * 128;
        uint32_t bytes = (p.diag & 1) ? 0u : gbytes;
        if (!(p.diag & 2)) {
          if constexpr (K == 0) bytes += AR::NENV * kBoxBytes + (uint32_t)nv * DSH * 4;
          else bytes += (uint32_t)F::v_off(F::NI);
        }
        mbar_expect_tx(in_full + s, bytes);
        if (p.diag & 2) {
        } else if constexpr (K == 0) {
#pragma unroll
          for (int l = 0; l < AR::NENV; ++l) tma_load_2d(st + l * kBoxBytes, &maps.in[0], 32 * l, (int)e0, in_full + s);
          bulk_load(st + F::y_off(), p.Y + e0 * DSH, (uint32_t)nv * DSH * 4, in_full + s);
        } else {
          // compile-time loop: a runtime index into the constexpr arch would read host-only data
          static_for<F::NI>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int dim = ir_dim(A.in.v[i]);
            tma_load_2d(st + F::v_off(i), &maps.in[i], 0, (int)(e0 * dim), in_full + s);
          });
        }
        if (!(p.diag & 1)) bulk_load(st + F::g_off(), p.G + (int64_t)a_lo * DSH * 32, gbytes, in_full + s);
      }
      if (++s == p.stages) s = 0, ph ^= 1;
    }
  } else if (warp < kTpWarps) {
    // ---------------- TP warps: thread = MMA row (m3, e), 8 channels per warp ----------------
    const int qw = warp & 3;                 // TMEM lane quarter
    const int cg = warp >> 2;                // channel group: channels 8 cg .. 8 cg + 7
    int s = 0, j = 0;
    uint32_t ph = 0, aph = 0;
    for (int t = 0; t < n_my; ++t) {
      const int64_t e0 = (int64_t)((int)blockIdx.x + t * (int)gridDim.x) * kTile;
      mbar_wait(in_full + s, ph);
      const unsigned char* st = stage0 + (size_t)s * F::stage_bytes();
      const int* hdr = reinterpret_cast<const int*>(st + F::h_off());
      const int e = lane;
      const int nv = hdr[32];
      const int ga = hdr[e];  // Gamma row block (valid edges; 0 for the padding rows)
      // staged rows, or (a tile spanning more than GA atoms: atoms without edges in between) L2
      const unsigned char* gb = ga < F::GA ? st + F::g_off() + (size_t)ga * DSH * 128
                                           : reinterpret_cast<const unsigned char*>(p.G + (int64_t)(hdr[33] + ga) * DSH * 32);
      // layer 0: this row's Y (DSH = 4) as one 16-B load (scalar loads at a 16-B lane stride were
      // 4-way shared-memory bank conflicts: 8 % of the kernel's shared wavefronts)
      [[maybe_unused]] float yrow[4] = {0.f, 0.f, 0.f, 0.f};
      if constexpr (K == 0) {
        static_assert(DSH == 4, "the fused TP forward is built for lmax = 1");
        const float4 y4 = *reinterpret_cast<const float4*>(st + F::y_off() + e * 16);
        yrow[0] = y4.x, yrow[1] = y4.y, yrow[2] = y4.z, yrow[3] = y4.w;
      }
      static_for<NO>([&](auto O) {
        constexpr int o = decltype(O)::value;
        constexpr int D3 = F::dim(o);
        constexpr int B0 = F::base(o);
        const int m3 = (qw - B0 + 4) & 3;
        static_for<F::nto(o)>([&](auto P) {
          constexpr int pl = decltype(P)::value;
          constexpr int q = F::path_of(o, pl);
          constexpr int L1 = A.path[q].a.l, L2 = A.path[q].b.l, LO = A.path[q].o.l;
          constexpr int D1 = 2 * L1 + 1, D2 = 2 * L2 + 1;
          mbar_wait(a_empty + j, aph ^ 1);
          if (m3 < D3) {
            float acc[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] = 0.f;
            static_for<D3>([&](auto M3) {
              constexpr int mm3 = decltype(M3)::value;
              if (m3 == mm3 && !(p.diag & 4)) {
                static_for<D1 * D2>([&](auto I) {
                  constexpr int m1 = decltype(I)::value / D2, m2 = decltype(I)::value % D2;
                  constexpr float cf = (float)(csqrt(2.0 * LO + 1.0) * W3j<L1, L2, LO>::t.v[(m1 * D2 + m2) * (2 * LO + 1) + mm3]);
                  if constexpr (cf != 0.f) {
                    const unsigned char* grow = gb + (A.sh_off[q] + m2) * 128;
                    if constexpr (K == 0) {
                      constexpr int mv = A.in_off[q] + m1;  // V0[m] = w_edge[l(m)] Y[m]
                      const float yv = yrow[mv];
                      const unsigned char* vrow = st + lm_l(mv) * kBoxBytes + e * 128;
#pragma unroll
                      for (int h = 0; h < 2; ++h) {
                        const int c4 = 2 * cg + h;
                        const float4 v = *reinterpret_cast<const float4*>(vrow + ((c4 ^ (e & 7)) << 4));
                        const float4 g = *reinterpret_cast<const float4*>(grow + (c4 << 4));
                        acc[4 * h + 0] = fmaf(cf * (v.x * yv), g.x, acc[4 * h + 0]);
                        acc[4 * h + 1] = fmaf(cf * (v.y * yv), g.y, acc[4 * h + 1]);
                        acc[4 * h + 2] = fmaf(cf * (v.z * yv), g.z, acc[4 * h + 2]);
                        acc[4 * h + 3] = fmaf(cf * (v.w * yv), g.w, acc[4 * h + 3]);
                      }
                    } else {
                      constexpr int ii = A.in.index(A.path[q].a);
                      const int r = e * D1 + m1;
                      const unsigned char* vrow = st + F::v_off(ii) + r * 128;
#pragma unroll
                      for (int h = 0; h < 2; ++h) {
                        const int c4 = 2 * cg + h;
                        const float4 v = *reinterpret_cast<const float4*>(vrow + ((c4 ^ (r & 7)) << 4));
                        const float4 g = *reinterpret_cast<const float4*>(grow + (c4 << 4));
                        acc[4 * h + 0] = fmaf(cf * v.x, g.x, acc[4 * h + 0]);
                        acc[4 * h + 1] = fmaf(cf * v.y, g.y, acc[4 * h + 1]);
                        acc[4 * h + 2] = fmaf(cf * v.z, g.z, acc[4 * h + 2]);
                        acc[4 * h + 3] = fmaf(cf * v.w, g.w, acc[4 * h + 3]);
                      }
                    }
                  }
                });
              }
            });
            if constexpr (F::scalar(o)) {
              // s = the scalar paths of T, [E][n_s 32]: this thread's 8 channels (32 B) of row e0 + e
              if (m3 == 0 && e < nv && !(p.diag & 16)) {
                float4* dst = reinterpret_cast<float4*>(p.s + (e0 + e) * (A.n_s * 32) + pl * 32 + 8 * cg);
                __stcs(dst, make_float4(acc[0], acc[1], acc[2], acc[3]));
                __stcs(dst + 1, make_float4(acc[4], acc[5], acc[6], acc[7]));
              }
            }
            uint32_t hi[8], lo[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint32_t h = __float_as_uint(acc[c]) & 0xffffe000u;
              hi[c] = h;
              lo[c] = __float_as_uint(acc[c] - __uint_as_float(h));
            }
            tc_fence_after();
            const uint32_t ta = tmem_a + (uint32_t)(j * kATm + 8 * cg) + ((uint32_t)(qw * 32) << 16);
            tmem_st8(ta, hi);
            tmem_st8(ta + 32, lo);
            tmem_st_wait();
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(a_full + j);
          if (++j == kAStages) j = 0, aph ^= 1;
        });
      });
      // the stage is refilled by TMA (async proxy): order these generic reads first
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(in_empty + s);
      if (++s == p.stages) s = 0, ph ^= 1;
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer ----------------
    mbar_wait(w_full, 0);
    tc_fence_after();
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(32 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t wblk = 32 * 128;  // one W half-block (hi or lo) of a K-block
    __syncwarp();
    const uint32_t L = elect_leader();
    int j = 0;
    uint32_t aph = 0;
    for (int t = 0; t < n_my; ++t) {
      const int buf = t % kAccBufs;
      mbar_wait(acc_empty + buf, ((uint32_t)(t / kAccBufs) & 1u) ^ 1u);
      __syncwarp();
      tc_fence_after();
      static_for<NO>([&](auto O) {
        constexpr int o = decltype(O)::value;
        const uint32_t d = tmem + (uint32_t)(buf * F::acc_cols() + 32 * o);
        const uint64_t desc_o = sdesc(smem_u32(w_img + woff[o]));
        static_for<F::nto(o)>([&](auto P) {
          constexpr int pl = decltype(P)::value;
          mbar_wait(a_full + j, aph);
          __syncwarp();
          tc_fence_after();
          const uint32_t ahi = tmem_a + (uint32_t)(j * kATm), alo = ahi + 32;
          const uint64_t dkb = desc_o + (uint64_t)((pl * 2 * wblk) >> 4);
#pragma unroll
          for (int k = 0; k < 4 && !(p.diag & 32); ++k) {
            const uint64_t dwh = dkb + (uint64_t)(k * 2);
            const uint64_t dwl = dwh + (uint64_t)(wblk >> 4);
            mma_tf32_ts_w(L, d, ahi + 8 * k, dwl, idesc, (pl | k) ? 1u : 0u);
            mma_tf32_ts_w(L, d, alo + 8 * k, dwh, idesc, 1u);
            mma_tf32_ts_w(L, d, ahi + 8 * k, dwh, idesc, 1u);
          }
          mma_commit_w(L, a_empty + j);
          if (++j == kAStages) j = 0, aph ^= 1;
        });
      });
      mma_commit_w(L, acc_full + buf);
    }
  } else {
    // ---------------- epilogue (warps 4-7): D -> V^{k+1} ----------------
    const int qd = warp & 3;  // TMEM lane quarter (warps 16-19)
    int n_st = 0;
    for (int t = 0; t < n_my; ++t) {
      const int64_t e0 = (int64_t)((int)blockIdx.x + t * (int)gridDim.x) * kTile;
      const int buf = t % kAccBufs;
      mbar_wait(acc_full + buf, (uint32_t)(t / kAccBufs) & 1u);
      tc_fence_after();
      static_for<NO>([&](auto O) {
        constexpr int o = decltype(O)::value;
        constexpr int B0 = F::base(o);
        const int m3 = (qd - B0 + 4) & 3;
        if (m3 < F::dim(o)) {
          float v[32];
          tmem_ld32(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(buf * F::acc_cols() + 32 * o), v);
          unsigned char* box = epi + (size_t)(2 * qd + (n_st & 1)) * kBoxBytes;
          if (n_st >= 2) {
            if (lane == 0) bulk_wait_read1();
            __syncwarp();
          }
          const float sc = p.scale[o];
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4)
            *reinterpret_cast<float4*>(box + lane * 128 + ((c4 ^ (lane & 7)) << 4)) =
                make_float4(sc * v[4 * c4], sc * v[4 * c4 + 1], sc * v[4 * c4 + 2], sc * v[4 * c4 + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0 && !(p.diag & 8)) {
            tma_store_3d(&maps.out[o], 0, m3, (int)e0, box);
            bulk_commit();
          }
          ++n_st;
        }
      });
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + buf);
    }
    if (lane == 0) bulk_wait0();
  }
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int NL, int LMAX, int K>
void launch(const TplIO& io, cudaStream_t st, Profiler* prof) {
  using F = Fz<NL, LMAX, K>;
  constexpr LayerArch A = F::A;
  const int64_t E = io.ch.n_e;
  if (E <= 0) return;
  TplMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  TplParams p;
  std::memset(&p, 0, sizeof(p));
  p.n_e = E;
  p.e0g = io.ch.e0;
  p.a0 = io.ch.a0;
  p.cidx = io.cidx;
  p.G = io.G;
  p.Y = io.Y;
  p.s = io.s;
  p.n_tiles = (int)((E + kTile - 1) / kTile);
  if (const char* d = std::getenv("ALLEGRO_TPL_DIAG")) p.diag = std::atoi(d);
  uint32_t wsum = 0;
  for (int o = 0; o < F::NO; ++o) {
    p.wimg[o] = io.wimg[o];
    p.wbytes[o] = (uint32_t)io.wbytes[o];
    if (io.wbytes[o] != (size_t)F::nto(o) * 2 * 32 * 128) throw CudaError("tpl_fwd: unexpected TP-linear weight image");
    p.scale[o] = 1.f / std::sqrt((float)(kC * F::nto(o)));
    wsum += p.wbytes[o];
    const uint64_t dims[3] = {32, (uint64_t)F::dim(o), (uint64_t)E};
    const uint64_t strides[2] = {128, (uint64_t)F::dim(o) * 128};
    const uint32_t box[3] = {32, 1, 32};
    maps.out[o] = tc_map_f32(io.vout[o], 3, dims, strides, box);
  }
  if constexpr (K == 0) {
    const uint64_t dims[2] = {(uint64_t)Arch<NL, LMAX, K>::NW, (uint64_t)E};
    const uint64_t strides[1] = {(uint64_t)Arch<NL, LMAX, K>::NW * 4};
    const uint32_t box[2] = {32, 32};
    maps.in[0] = tc_map_f32(io.w, 2, dims, strides, box);
  } else {
    for (int i = 0; i < F::NI; ++i) {
      const uint64_t dims[2] = {32, (uint64_t)E * ir_dim(A.in.v[i])};
      const uint64_t strides[1] = {128};
      const uint32_t box[2] = {32, (uint32_t)F::in_rows(i)};
      maps.in[i] = tc_map_f32(io.vin[i], 2, dims, strides, box);
    }
  }
  if (std::getenv("ALLEGRO_SYNC_CHECK")) {
    std::fprintf(stderr, "[tpl_fwd K=%d] E=%lld e0g=%lld a0=%lld n_c=%lld G=%p Y=%p w=%p s=%p\n", K, (long long)E,
                 (long long)io.ch.e0, (long long)io.ch.a0, (long long)io.ch.n_c, (const void*)io.G, (const void*)io.Y,
                 (const void*)io.w, (void*)io.s);
    for (int i = 0; i < F::NI; ++i) std::fprintf(stderr, "  vin[%d]=%p rows=%d\n", i, (const void*)io.vin[i], F::in_rows(i));
    for (int o = 0; o < F::NO; ++o)
      std::fprintf(stderr, "  vout[%d]=%p wimg=%p wbytes=%zu\n", o, (void*)io.vout[o], (const void*)io.wimg[o], io.wbytes[o]);
  }
  const size_t fixed = 1024 + ((wsum + 1023) / 1024) * 1024 + 8 * kBoxBytes + 512;
  int stages = (int)std::min<size_t>(4, (kSmemLimit - fixed) / F::stage_bytes());
  if (stages < 2) throw CudaError("tpl_fwd: shared memory too small for two input stages");
  p.stages = stages;
  const size_t smem = fixed + (size_t)stages * F::stage_bytes();
  int dev = 0;
  ALG_CUDA(cudaGetDevice(&dev));
  static bool attr[64] = {};
  static int nsm[64] = {};
  if (dev < 0 || dev >= 64) throw CudaError("device ordinal out of range");
  {
    std::lock_guard<std::mutex> lk_(g_attr_mu);  // per-device function attributes, set once (thread-safe)
    if (!attr[dev]) {
      ALG_CUDA(cudaFuncSetAttribute(k_tpl_fwd<NL, LMAX, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemLimit));
      ALG_CUDA(cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev));
      attr[dev] = true;
    }
  }
  const int grid = std::max(1, std::min(p.n_tiles, nsm[dev]));
  {
    char tag[48];
    std::snprintf(tag, sizeof(tag), "tpl_fwd layer=%d", K);
    // algorithmic work: the TP FMAs (CUDA cores) + the TP-linear MACs (tensor cores), per edge
    double mac = 0;
    for (int o = 0; o < F::NO; ++o) mac += (double)F::dim(o) * F::nto(o) * kC * kC;
    const double flops = (double)E * (2.0 * io.tp_fma_per_edge + 2.0 * mac);
    double bytes = 0;
    for (int i = 0; i < F::NI; ++i) bytes += K == 0 ? 0.0 : (double)ir_dim(A.in.v[i]) * 128;
    if (K == 0) bytes += Arch<NL, LMAX, K>::NENV * 128 + F::DSH * 4;
    for (int o = 0; o < F::NO; ++o) bytes += (double)F::dim(o) * 128;
    bytes += (double)A.n_s * 128 + 4;  // s, cidx
    ProfScope ps_(prof, st, PK_TPL_FWD, flops, bytes * E, tag);
    k_tpl_fwd<NL, LMAX, K><<<grid, kThreads, smem, st>>>(maps, p);
  }
  ALG_LAUNCH_CHECK();
  if (std::getenv("ALLEGRO_SYNC_CHECK")) {  // diagnostics: attribute a fault to this launch
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess)
      throw CudaError(std::string("k_tpl_fwd layer ") + std::to_string(K) + ": " + cudaGetErrorString(e));
  }
}

// ====================================================================== backward
// One layer k < L-1, per 32-edge tile:
//   T-bar_o = V-bar^{k+1}_o W_o^T / sqrt(C n_{->o})  (+ s-bar on the scalar paths)    tcgen05 (3xTF32)
//   then per edge (warp per edge, lane = channel) the TP adjoint of k_tp_bwd (model.cu):
//   V-bar^k (k >= 1) or w-bar_edge and Y-bar (k = 0), and the edge's term of Gamma-bar_i (to HBM;
//   k_env_adj sums it over the row in edge order and applies the environment adjoint).
// T-bar never reaches HBM.  Warp roles (704 threads):
//   warps 0-11  TP adjoint (lane = channel) from the T-bar tile in SMEM and the tile's inputs
//   warps 12-15 split: V-bar rows (TMA boxes, one per (o, m3)) -> TF32 hi / lo -> TMEM A stage
//   warps 16-19 T-bar copy: tcgen05.ld of D (thread = row), scale, + s-bar, -> SMEM tile
//   warp 20     producer (TMA / bulk loads), warp 21 TMEM allocator + MMA issuer
// TP warps of k_tpl_bwd per layer (build-time A/B): layer 0 (w (x) Y inputs, w-bar / Y-bar outputs)
// is TP-warp-bound and takes 16 (one edge per warp per T-bar half); layer >= 1 is closer to its HBM
// bound and runs faster with 12 (more registers per thread for the rest)
#ifndef ALG_TPB_WARPS0
#define ALG_TPB_WARPS0 16
#endif
#ifndef ALG_TPB_WARPS1
#define ALG_TPB_WARPS1 12
#endif
template <int K>
struct BW {
  static constexpr int Tp = K == 0 ? ALG_TPB_WARPS0 : ALG_TPB_WARPS1;
  static constexpr int Split0 = Tp;
  static constexpr int Copy0 = Tp + 4;
  static constexpr int Prod = Tp + 8;   // ring B producer (the TP inputs)
  static constexpr int Mma = Tp + 9;
  static constexpr int ProdA = Tp + 10; // ring A producer (the MMA chain's V-bar / s-bar boxes) + W images
  static constexpr int Threads = 32 * (Tp + 11);
};
constexpr int kBAStages = 3;
constexpr int kBGA = 8;  // Gamma rows staged per tile (atoms); wider spans read from L2

template <int NL, int LMAX, int K>
struct Bz {
  using F = Fz<NL, LMAX, K>;
  using AR = Arch<NL, LMAX, K>;
  static constexpr LayerArch A = AR::A;
  static constexpr int NO = A.out.n, NI = A.in.n, DSH = AR::DSH, DT = A.dim_T, DIN = A.dim_in;
  static constexpr int col_off(int o) {
    int b = 0;
    for (int q = 0; q < o; ++q) b += A.n_to[q] * 32;
    return b;
  }
  static constexpr int acc_cols() { return col_off(NO); }
  static constexpr int vb_off(int o) {
    int b = 0;
    for (int q = 0; q < o; ++q) b += ir_dim(A.out.v[q]) * kBoxBytes;
    return b;
  }
  // ring A stage (split / MMA / copy chain): V-bar^{k+1} boxes, one per (irrep, m3), then s-bar boxes
  static constexpr int sb_off() { return vb_off(NO); }
  static constexpr int a_bytes() { return sb_off() + A.n_s * kBoxBytes; }
  // ring B stage (the TP warps): V^k per in irrep (k >= 1) or w_edge boxes + Y + old Y-bar (k = 0),
  // the Gamma rows of the tile's centres, and the header (centre slots, edge count, first centre)
  static constexpr int v_off(int i) { return F::v_off(i); }
  static constexpr int y_off() { return AR::NENV * kBoxBytes; }
  static constexpr int yb_off() { return y_off() + kTile * DSH * 4; }
  static constexpr int g_off() { return K == 0 ? yb_off() + kTile * DSH * 4 : F::v_off(NI); }
  static constexpr int h_off() { return g_off() + kBGA * DSH * 128; }
  static constexpr int b_bytes() { return (h_off() + 256 + 1023) / 1024 * 1024; }
  static constexpr int b_tma_bytes() { return K == 0 ? AR::NENV * kBoxBytes : F::v_off(NI); }
  static constexpr int tb_bytes() { return kTile * DT * 128; }  // two 16-edge halves, double-buffered in turn
};

template <int NL, int LMAX, int K>
constexpr double DSH_bytes() { return 2.0 * Arch<NL, LMAX, K>::DSH * 4; }

struct TpbParams {
  int64_t n_e, e0g, a0;
  const int32_t* cidx;
  const float* G;
  const float* Y;
  float* vbo[kMaxIr];  // V-bar^k per in irrep (k >= 1)
  float* wbar;         // [E][NW] (k = 0: the w_edge columns)
  float* ybar;         // [E][DSH] (k = 0)
  float* gp;           // [E][DSH][C]
  const float* wimg[kMaxIr];
  uint32_t wbytes[kMaxIr];
  float scale[kMaxIr];
  int n_tiles, sa, sb;  // ring depths
  int rr;               // TP warps take the tile's edges round-robin across both T-bar halves
  int diag;             // timing diagnostics (ALLEGRO_TPB_DIAG, wrong results): bit0 TP warps skip the
                        // edge work, bit1 copy warps skip the TMEM reads / T-bar stores
};

struct TpbMaps {
  CUtensorMap vb[kMaxIr];  // V-bar^{k+1} per out irrep, 3-D [E][dim][32], box [32 e][1][32 c]
  CUtensorMap sb;          // s-bar [E][n_s 32], box [32 e][32 c]
  CUtensorMap in[kMaxIr];  // V^k per in irrep (k >= 1) or w [E][NW] (k = 0, in[0])
};

template <int NL, int LMAX, int K>
__global__ void __launch_bounds__(BW<K>::Threads, 1) k_tpl_bwd(const __grid_constant__ TpbMaps maps, const TpbParams p) {
  constexpr int kBTp = BW<K>::Tp, kBSplit0 = BW<K>::Split0, kBCopy0 = BW<K>::Copy0, kBProd = BW<K>::Prod,
                kBMma = BW<K>::Mma, kBProdA = BW<K>::ProdA;
  using B = Bz<NL, LMAX, K>;
  using F = Fz<NL, LMAX, K>;
  using AR = Arch<NL, LMAX, K>;
  constexpr LayerArch A = B::A;
  constexpr int NO = B::NO, DSH = B::DSH, DT = B::DT, DIN = B::DIN;
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* base = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  uint32_t woff[kMaxIr + 1];
  woff[0] = 0;
#pragma unroll
  for (int o = 0; o < kMaxIr; ++o) woff[o + 1] = woff[o] + (o < NO ? p.wbytes[o] : 0u);
  unsigned char* w_img = base;
  unsigned char* ringA = base + ((woff[NO] + 1023u) & ~1023u);
  unsigned char* ringB = ringA + (size_t)p.sa * B::a_bytes();
  unsigned char* tbt = ringB + (size_t)p.sb * B::b_bytes();
  uint64_t* bars = reinterpret_cast<uint64_t*>(tbt + B::tb_bytes());
  uint64_t* in_full = bars;           // [4] ring A: the tile's V-bar and s-bar boxes
  uint64_t* in_empty = in_full + 4;   // [4] released by the split and copy warps
  uint64_t* a_full = in_empty + 4;
  uint64_t* a_empty = a_full + kBAStages;
  uint64_t* acc_full = a_empty + kBAStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* tb_full = acc_empty + 2;  // [2] T-bar halves (edges 0-15, 16-31)
  uint64_t* tb_empty = tb_full + 2;   // [2]
  uint64_t* w_full = tb_empty + 2;
  uint64_t* in_full_b = w_full + 1;   // [4] ring B: the TP inputs
  uint64_t* in_empty_b = in_full_b + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(in_empty_b + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.sa; ++s) mbar_init(in_full + s, 1), mbar_init(in_empty + s, 8);
    for (int s = 0; s < p.sb; ++s) mbar_init(in_full_b + s, 1), mbar_init(in_empty_b + s, kBTp);
    for (int s = 0; s < kBAStages; ++s) mbar_init(a_full + s, 4), mbar_init(a_empty + s, 1);
    for (int b = 0; b < 2; ++b) mbar_init(acc_full + b, 1), mbar_init(acc_empty + b, 4);
    for (int h = 0; h < 2; ++h) mbar_init(tb_full + h, 4), mbar_init(tb_empty + h, kBTp);
    mbar_init(w_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kBMma) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_a = tmem + 2u * B::acc_cols();
  const int n_my = p.n_tiles > (int)blockIdx.x ? (p.n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto tile_e0 = [&](int t) -> int64_t { return (int64_t)((int)blockIdx.x + t * (int)gridDim.x) * kTile; };

  if (warp == kBProdA) {
    // ---------------- ring A producer: the MMA chain's operands (and the W images) ----------------
    if (lane == 0) {
      mbar_expect_tx(w_full, woff[NO]);
      for (int o = 0; o < NO; ++o) bulk_load(w_img + woff[o], p.wimg[o], p.wbytes[o], w_full);
      int s = 0;
      uint32_t ph = 0;
      for (int t = 0; t < n_my; ++t) {
        const int64_t e0 = tile_e0(t);
        mbar_wait(in_empty + s, ph ^ 1);
        unsigned char* st = ringA + (size_t)s * B::a_bytes();
        mbar_expect_tx(in_full + s, (uint32_t)B::a_bytes());
        static_for<NO>([&](auto O) {
          constexpr int o = decltype(O)::value;
          static_for<ir_dim(A.out.v[o])>([&](auto M) {
            constexpr int m = decltype(M)::value;
            tma_load_3d(st + B::vb_off(o) + m * kBoxBytes, &maps.vb[o], 0, m, (int)e0, in_full + s);
          });
        });
        for (int q = 0; q < A.n_s; ++q) tma_load_2d(st + B::sb_off() + q * kBoxBytes, &maps.sb, 32 * q, (int)e0, in_full + s);
        if (++s == p.sa) s = 0, ph ^= 1;
      }
    }
  } else if (warp == kBProd) {
    // ---------------- ring B producer: the TP inputs ----------------
    int s = 0;
    uint32_t ph = 0;
    auto load_ci = [&](int t) -> int {
      const int64_t e0 = tile_e0(t);
      return (t < n_my && e0 + lane < p.n_e) ? __ldg(p.cidx + p.e0g + e0 + lane) - (int)p.a0 : 0;
    };
    int ci_next = load_ci(0);
    for (int t = 0; t < n_my; ++t) {
      const int64_t e0 = tile_e0(t);
      const int nv = (int)(p.n_e - e0 < kTile ? p.n_e - e0 : kTile);
      const int ci = ci_next;
      ci_next = load_ci(t + 1);
      mbar_wait(in_empty_b + s, ph ^ 1);
      unsigned char* st = ringB + (size_t)s * B::b_bytes();
      int* hdr = reinterpret_cast<int*>(st + B::h_off());
      const int a_lo = __shfl_sync(0xffffffffu, ci, 0);
      const int a_hi = __shfl_sync(0xffffffffu, ci, nv - 1);
      hdr[lane] = lane < nv ? ci - a_lo : 0;
      if (lane == 0) hdr[32] = nv, hdr[33] = a_lo;
      __syncwarp();
      if (lane == 0) {
        const int span = a_hi - a_lo + 1;
        const uint32_t gbytes = (uint32_t)(span < kBGA ? span : kBGA) * DSH * 128;
        mbar_expect_tx(in_full_b + s, (uint32_t)B::b_tma_bytes() + gbytes + (K == 0 ? 2u * (uint32_t)nv * DSH * 4 : 0u));
        if constexpr (K == 0) {
#pragma unroll
          for (int l = 0; l < AR::NENV; ++l) tma_load_2d(st + l * kBoxBytes, &maps.in[0], 32 * l, (int)e0, in_full_b + s);
          bulk_load(st + B::y_off(), p.Y + e0 * DSH, (uint32_t)nv * DSH * 4, in_full_b + s);
          bulk_load(st + B::yb_off(), p.ybar + e0 * DSH, (uint32_t)nv * DSH * 4, in_full_b + s);
        } else {
          static_for<B::NI>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int dim = ir_dim(A.in.v[i]);
            tma_load_2d(st + B::v_off(i), &maps.in[i], 0, (int)(e0 * dim), in_full_b + s);
          });
        }
        bulk_load(st + B::g_off(), p.G + (int64_t)a_lo * DSH * 32, gbytes, in_full_b + s);
      }
      if (++s == p.sb) s = 0, ph ^= 1;
    }
  } else if (warp >= kBSplit0 && warp < kBSplit0 + 4) {
    // ---------------- split: V-bar rows -> TF32 hi / lo in TMEM ----------------
    const int qw = warp & 3;
    int s = 0, j = 0;
    uint32_t ph = 0, aph = 0;
    for (int t = 0; t < n_my; ++t) {
      mbar_wait(in_full + s, ph);
      const unsigned char* st = ringA + (size_t)s * B::a_bytes();
      static_for<NO>([&](auto O) {
        constexpr int o = decltype(O)::value;
        constexpr int B0 = F::base(o);
        const int m3 = (qw - B0 + 4) & 3;
        mbar_wait(a_empty + j, aph ^ 1);
        if (m3 < F::dim(o)) {
          const unsigned char* row = st + B::vb_off(o) + m3 * kBoxBytes + lane * 128;
          const uint32_t ta = tmem_a + (uint32_t)(j * kATm) + ((uint32_t)(qw * 32) << 16);
          tc_fence_after();
#pragma unroll
          for (int hc = 0; hc < 2; ++hc) {  // two 16-column chunks (register budget of 16 TP warps)
            uint32_t hi[16], lo[16];
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const int cc = 4 * hc + c4;
              const float4 v = *reinterpret_cast<const float4*>(row + ((cc ^ (lane & 7)) << 4));
              const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t h = __float_as_uint(x[q]) & 0xffffe000u;
                hi[4 * c4 + q] = h;
                lo[4 * c4 + q] = __float_as_uint(x[q] - __uint_as_float(h));
              }
            }
            tmem_st16(ta + 16 * hc, hi);
            tmem_st16(ta + 32 + 16 * hc, lo);
          }
          tmem_st_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full + j);
        if (++j == kBAStages) j = 0, aph ^= 1;
      });
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(in_empty + s);
      if (++s == p.sa) s = 0, ph ^= 1;
    }
  } else if (warp == kBMma) {
    // ---------------- MMA issuer: D_o = A_o W_o^T ----------------
    mbar_wait(w_full, 0);
    tc_fence_after();
    __syncwarp();
    const uint32_t L = elect_leader();
    int j = 0;
    uint32_t aph = 0;
    for (int t = 0; t < n_my; ++t) {
      const int buf = t & 1;
      mbar_wait(acc_empty + buf, ((uint32_t)(t >> 1) & 1u) ^ 1u);
      __syncwarp();
      tc_fence_after();
      static_for<NO>([&](auto O) {
        constexpr int o = decltype(O)::value;
        constexpr uint32_t N = (uint32_t)A.n_to[o] * 32;
        constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t d = tmem + (uint32_t)(buf * B::acc_cols() + B::col_off(o));
        const uint64_t desc_o = sdesc(smem_u32(w_img + woff[o]));
        mbar_wait(a_full + j, aph);
        __syncwarp();
        tc_fence_after();
        const uint32_t ahi = tmem_a + (uint32_t)(j * kATm), alo = ahi + 32;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t dwh = desc_o + (uint64_t)(k * 2);
          const uint64_t dwl = dwh + (uint64_t)((N * 128) >> 4);
          mma_tf32_ts_w(L, d, ahi + 8 * k, dwl, idesc, k ? 1u : 0u);
          mma_tf32_ts_w(L, d, alo + 8 * k, dwh, idesc, 1u);
          mma_tf32_ts_w(L, d, ahi + 8 * k, dwh, idesc, 1u);
        }
        mma_commit_w(L, a_empty + j);
        if (++j == kBAStages) j = 0, aph ^= 1;
      });
      mma_commit_w(L, acc_full + buf);
    }
  } else if (warp >= kBCopy0 && warp < kBCopy0 + 4) {
    // ---------------- T-bar copy: TMEM rows -> SMEM tile [e][t][c] (+ s-bar) ----------------
    const int qw = warp & 3;
    int s = 0;
    uint32_t ph = 0;
    for (int t = 0; t < n_my; ++t) {
      const int buf = t & 1;
      mbar_wait(acc_full + buf, (uint32_t)(t >> 1) & 1u);
      tc_fence_after();
      mbar_wait(in_full + s, ph);                      // (complete: its s-bar boxes are read here)
      const unsigned char* st = ringA + (size_t)s * B::a_bytes();
      const int e = lane;
      // two passes over the accumulator: edges 0-15 into half 0, then 16-31 into half 1, so that the
      // TP warps work on one half while the other is refilled
      for (int h = 0; h < 2; ++h) {
        mbar_wait(tb_empty + h, ((uint32_t)t & 1u) ^ 1u);  // the TP warps are done with this half
        const bool mine = (e >> 4) == h;
        static_for<NO>([&](auto O) {
          constexpr int o = decltype(O)::value;
          constexpr int B0 = F::base(o);
          const int m3 = (qw - B0 + 4) & 3;
          if (m3 < F::dim(o) && !(p.diag & 2)) {
            static_for<A.n_to[o]>([&](auto P) {
              constexpr int pl = decltype(P)::value;
              constexpr int q = F::path_of(o, pl);
#pragma unroll
              for (int hc = 0; hc < 2; ++hc) {  // 16-column chunks (register budget of 16 TP warps)
                float v[16];
                tmem_ld16(tmem + ((uint32_t)(qw * 32) << 16) +
                              (uint32_t)(buf * B::acc_cols() + B::col_off(o) + 32 * pl + 16 * hc),
                          v);
                if (mine) {
                  const float sc = p.scale[o];
                  const int row = (e & 15) * DT + A.t_off[q] + m3;
                  unsigned char* dst = tbt + (size_t)h * (B::tb_bytes() / 2) + (size_t)row * 128;
                  const unsigned char* sbr = st + B::sb_off() + pl * kBoxBytes + e * 128;
#pragma unroll
                  for (int c4 = 0; c4 < 4; ++c4) {
                    const int cc = 4 * hc + c4;
                    float4 w4 = make_float4(sc * v[4 * c4], sc * v[4 * c4 + 1], sc * v[4 * c4 + 2], sc * v[4 * c4 + 3]);
                    if constexpr (F::scalar(o)) {  // T-bar of the scalar paths += s-bar (same order as EPI_ADDX)
                      const float4 a4 = *reinterpret_cast<const float4*>(sbr + ((cc ^ (e & 7)) << 4));
                      w4 = make_float4(w4.x + a4.x, w4.y + a4.y, w4.z + a4.z, w4.w + a4.w);
                    }
                    *reinterpret_cast<float4*>(dst + ((cc ^ (row & 7)) << 4)) = w4;
                  }
                }
              }
            });
          }
        });
        __syncwarp();
        if (lane == 0) mbar_arrive(tb_full + h);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + buf);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(in_empty + s);
      if (++s == p.sa) s = 0, ph ^= 1;
    }
  } else if (warp < kBTp) {
    // ---------------- TP adjoint: warp per edge, lane = channel ----------------
    const int c = lane;
    int s = 0;
    uint32_t ph = 0;
    for (int t = 0; t < n_my; ++t) {
      const int64_t e0 = tile_e0(t);
      mbar_wait(in_full_b + s, ph);
      const unsigned char* st = ringB + (size_t)s * B::b_bytes();
      const int* hdr = reinterpret_cast<const int*>(st + B::h_off());
      const int nv = hdr[32], a_lo = hdr[33];
      // the tile's 32 edges over the kBTp warps round-robin across both T-bar halves (with 12 warps:
      // edges w, w + 12, w + 24, three rounds instead of two per half; with 16: one edge per half); a
      // warp releases half 0 when it moves to its first half-1 edge (every warp has edges in both)
      mbar_wait(tb_full + 0, (uint32_t)t & 1u);
      bool in_h1 = false;
      for (int r = 0; r < 4; ++r) {
        int e;
        if (p.rr) {  // round-robin over the whole tile (default)
          e = warp + r * kBTp;
          if (e >= 2 * 16) break;
        } else {  // A/B: each half in turn, edges 16 h + w (+ 12)
          e = 16 * (r >> 1) + warp + (r & 1) * kBTp;
          if (e >= 16 * (r >> 1) + 16) continue;
        }
        const int h = e >> 4;
        if (h == 1 && !in_h1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(tb_empty + 0);
          mbar_wait(tb_full + 1, (uint32_t)t & 1u);
          in_h1 = true;
        }
        if (e >= nv || (p.diag & 1)) continue;
        const unsigned char* tbh = tbt + (size_t)h * (B::tb_bytes() / 2);
        {
        const int ga = hdr[e];
        const float* gsrc = ga < kBGA ? reinterpret_cast<const float*>(st + B::g_off() + (size_t)ga * DSH * 128)
                                      : p.G + (int64_t)(a_lo + ga) * DSH * 32;
        float G[DSH], tb[DT], v[DIN], vb[DIN], gp[DSH];
#pragma unroll
        for (int m = 0; m < DSH; ++m) G[m] = gsrc[m * 32 + c], gp[m] = 0.f;
#pragma unroll
        for (int q = 0; q < DT; ++q) {
          const int row = (e & 15) * DT + q;
          tb[q] = *reinterpret_cast<const float*>(tbh + row * 128 + ((((c >> 2) ^ (row & 7))) << 4) + (c & 3) * 4);
        }
        [[maybe_unused]] float we[AR::NENV], yv[DSH];
        if constexpr (K == 0) {
#pragma unroll
          for (int l = 0; l < AR::NENV; ++l)
            we[l] = *reinterpret_cast<const float*>(st + l * kBoxBytes + e * 128 + (((c >> 2) ^ (e & 7)) << 4) + (c & 3) * 4);
#pragma unroll
          for (int m = 0; m < DSH; ++m) yv[m] = reinterpret_cast<const float*>(st + B::y_off())[e * DSH + m];
#pragma unroll
          for (int m = 0; m < DSH; ++m) v[m] = we[lm_l(m)] * yv[m];
        } else {
          static_for<B::NI>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int dim = ir_dim(A.in.v[i]);
            constexpr int off = A.in.off(i);
#pragma unroll
            for (int m = 0; m < dim; ++m) {
              const int row = e * dim + m;
              v[off + m] = *reinterpret_cast<const float*>(st + B::v_off(i) + row * 128 + ((((c >> 2) ^ (row & 7))) << 4) + (c & 3) * 4);
            }
          });
        }
#pragma unroll
        for (int q = 0; q < DIN; ++q) vb[q] = 0.f;
        static_for<A.n_paths>([&](auto Q) {
          constexpr int q = decltype(Q)::value;
          constexpr int L1 = A.path[q].a.l, L2 = A.path[q].b.l, LO = A.path[q].o.l;
          constexpr int D2 = 2 * L2 + 1, D3 = 2 * LO + 1;
          constexpr double alpha = csqrt(2.0 * LO + 1.0);
          static_for<(2 * L1 + 1) * D2 * D3>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int m1 = i / (D2 * D3), m2 = (i / D3) % D2, m3 = i % D3;
            constexpr float cf = (float)(alpha * W3j<L1, L2, LO>::t.v[i]);
            constexpr int it = A.t_off[q] + m3, iv = A.in_off[q] + m1, ig = A.sh_off[q] + m2;
            if constexpr (cf != 0.f) {
              const float ct = cf * tb[it];
              vb[iv] = fmaf(ct, G[ig], vb[iv]);
              gp[ig] = fmaf(ct, v[iv], gp[ig]);
            }
          });
        });
        const int64_t ge = e0 + e;
        if constexpr (K == 0) {
          // V0 = w_edge (x) Y:  w-bar_edge[l] = sum_m vb[m] Y[m];  Y-bar[m] += sum_c vb[m] w_edge[l(m)]
          float wb[AR::NENV], prod[DSH];
#pragma unroll
          for (int l = 0; l < AR::NENV; ++l) wb[l] = 0.f;
#pragma unroll
          for (int m = 0; m < DSH; ++m) {
            wb[lm_l(m)] = fmaf(vb[m], yv[m], wb[lm_l(m)]);
            prod[m] = vb[m] * we[lm_l(m)];
          }
          int mq;
          const float sm = warp_sum_multi<DSH>(prod, lane, &mq);
#pragma unroll
          for (int l = 0; l < AR::NENV; ++l) p.wbar[ge * AR::NW + l * 32 + c] = wb[l];
          constexpr int LP = DSH <= 1 ? 0 : DSH <= 2 ? 1 : DSH <= 4 ? 2 : DSH <= 8 ? 3 : 4;
          if (mq < DSH && (lane & ((1 << (5 - LP)) - 1)) == 0)  // old Y-bar staged by the producer
            p.ybar[ge * DSH + mq] = reinterpret_cast<const float*>(st + B::yb_off())[e * DSH + mq] + sm;
        } else {
          static_for<B::NI>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int dim = ir_dim(A.in.v[i]);
            constexpr int off = A.in.off(i);
#pragma unroll
            for (int m = 0; m < dim; ++m) p.vbo[i][(ge * dim + m) * 32 + c] = vb[off + m];
          });
        }
#pragma unroll
        for (int m = 0; m < DSH; ++m) p.gp[(ge * DSH + m) * 32 + c] = gp[m];
      }
      }
      static_assert(kBTp > 8 && kBTp <= 16, "every TP warp needs an edge in each T-bar half");
      __syncwarp();
      if (lane == 0) mbar_arrive(tb_empty + 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(in_empty_b + s);
      if (++s == p.sb) s = 0, ph ^= 1;
    }
  }
  __syncthreads();
  if (warp == kBMma) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int NL, int LMAX, int K>
void launch_bwd(const TpbIO& io, cudaStream_t st, Profiler* prof) {
  using B = Bz<NL, LMAX, K>;
  using F = Fz<NL, LMAX, K>;
  constexpr LayerArch A = B::A;
  const int64_t E = io.ch.n_e;
  if (E <= 0) return;
  TpbMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  TpbParams p;
  std::memset(&p, 0, sizeof(p));
  p.n_e = E;
  p.e0g = io.ch.e0;
  p.a0 = io.ch.a0;
  p.cidx = io.cidx;
  p.G = io.G;
  p.Y = io.Y;
  for (int i = 0; i < B::NI; ++i) p.vbo[i] = io.vbar_out[i];
  p.wbar = io.wbar;
  p.ybar = io.ybar;
  p.gp = io.gp;
  p.n_tiles = (int)((E + kTile - 1) / kTile);
  uint32_t wsum = 0;
  for (int o = 0; o < B::NO; ++o) {
    p.wimg[o] = io.wimg[o];
    p.wbytes[o] = (uint32_t)io.wbytes[o];
    if (io.wbytes[o] != (size_t)F::nto(o) * 32 * 2 * 128) throw CudaError("tpl_bwd: unexpected TP-linear^T weight image");
    p.scale[o] = 1.f / std::sqrt((float)(kC * F::nto(o)));
    wsum += p.wbytes[o];
    const uint64_t dims[3] = {32, (uint64_t)F::dim(o), (uint64_t)E};
    const uint64_t strides[2] = {128, (uint64_t)F::dim(o) * 128};
    const uint32_t box[3] = {32, 1, 32};
    maps.vb[o] = tc_map_f32(io.vbar_in[o], 3, dims, strides, box);
  }
  {
    const uint64_t dims[2] = {(uint64_t)A.n_s * 32, (uint64_t)E};
    const uint64_t strides[1] = {(uint64_t)A.n_s * 128};
    const uint32_t box[2] = {32, 32};
    maps.sb = tc_map_f32(io.sbar, 2, dims, strides, box);
  }
  if constexpr (K == 0) {
    const uint64_t dims[2] = {(uint64_t)Arch<NL, LMAX, K>::NW, (uint64_t)E};
    const uint64_t strides[1] = {(uint64_t)Arch<NL, LMAX, K>::NW * 4};
    const uint32_t box[2] = {32, 32};
    maps.in[0] = tc_map_f32(io.w, 2, dims, strides, box);
  } else {
    for (int i = 0; i < B::NI; ++i) {
      const uint64_t dims[2] = {32, (uint64_t)E * ir_dim(A.in.v[i])};
      const uint64_t strides[1] = {128};
      const uint32_t box[2] = {32, (uint32_t)F::in_rows(i)};
      maps.in[i] = tc_map_f32(io.vin[i], 2, dims, strides, box);
    }
  }
  const size_t fixed = 1024 + ((wsum + 1023) / 1024) * 1024 + B::tb_bytes() + 512 + 2 * (size_t)B::b_bytes();
  // ring B: two stages; ring A (the latency-critical MMA chain) as deep as the rest allows (<= 4)
  const int sa = (int)std::min<size_t>(4, (kSmemLimit - fixed) / B::a_bytes());
  if (sa < 2) throw CudaError("tpl_bwd: shared memory too small for two stages per ring");
  p.sa = sa;
  p.sb = 2;
  {
    static const int rr = [] {
      const char* e = std::getenv("ALLEGRO_TPB_RR");
      return (!e || std::atoi(e) != 0) ? 1 : 0;
    }();
    p.rr = rr;
    const char* dg = std::getenv("ALLEGRO_TPB_DIAG");
    p.diag = dg ? std::atoi(dg) : 0;
  }
  const size_t smem = fixed + (size_t)sa * B::a_bytes();
  if (std::getenv("ALLEGRO_TPB_INFO"))
    std::fprintf(stderr, "[tpl_bwd K=%d] W %u B, ring A %d x %d B, ring B %d x %d B, T-bar %d B, smem %zu B\n", K,
                 wsum, sa, B::a_bytes(), p.sb, B::b_bytes(), B::tb_bytes(), smem);
  int dev = 0;
  ALG_CUDA(cudaGetDevice(&dev));
  static bool attr[64] = {};
  static int nsm[64] = {};
  if (dev < 0 || dev >= 64) throw CudaError("device ordinal out of range");
  {
    std::lock_guard<std::mutex> lk_(g_attr_mu);  // per-device function attributes, set once (thread-safe)
    if (!attr[dev]) {
      ALG_CUDA(cudaFuncSetAttribute(k_tpl_bwd<NL, LMAX, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemLimit));
      ALG_CUDA(cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev));
      attr[dev] = true;
    }
  }
  const int grid = std::max(1, std::min(p.n_tiles, nsm[dev]));
  {
    char tag[48];
    std::snprintf(tag, sizeof(tag), "tpl_bwd layer=%d", K);
    double mac = 0;
    for (int o = 0; o < B::NO; ++o) mac += (double)F::dim(o) * F::nto(o) * kC * kC;
    const double flops = (double)E * (2.0 * 2.0 * io.tp_fma_per_edge + 2.0 * mac);
    double bytes = 0;
    for (int o = 0; o < B::NO; ++o) bytes += (double)F::dim(o) * 128;       // V-bar^{k+1}
    bytes += (double)A.n_s * 128 + 4;                                        // s-bar, cidx
    if (K == 0) bytes += Arch<NL, LMAX, K>::NENV * 128 * 2 + DSH_bytes<NL, LMAX, K>();  // w_edge in, w-bar out, Y, Y-bar
    else bytes += 2.0 * A.dim_in * 128;                                      // V^k in, V-bar^k out
    bytes += (double)B::DSH * 128;                                           // Gamma-bar terms out
    ProfScope ps_(prof, st, PK_TPL_BWD, flops, bytes * E, tag);
    k_tpl_bwd<NL, LMAX, K><<<grid, BW<K>::Threads, smem, st>>>(maps, p);
  }
  ALG_LAUNCH_CHECK();
  if (std::getenv("ALLEGRO_SYNC_CHECK")) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess)
      throw CudaError(std::string("k_tpl_bwd layer ") + std::to_string(K) + ": " + cudaGetErrorString(e));
  }
}

}  // namespace

bool tpl_fwd_supported(int NL, int LMAX, int K) { return LMAX == 1 && K < NL - 1 && (NL == 2 || NL == 3); }

void tpl_bwd(int NL, int LMAX, int K, const TpbIO& io, cudaStream_t st, Profiler* prof) {
#define ALG_TPB(nl, lm, k) \
  if (NL == nl && LMAX == lm && K == k) return launch_bwd<nl, lm, k>(io, st, prof);
  ALG_TPB(2, 1, 0)
  ALG_TPB(3, 1, 0) ALG_TPB(3, 1, 1)
#undef ALG_TPB
  throw CudaError("tpl_bwd: no fused kernel for this layer");
}

void tpl_fwd(int NL, int LMAX, int K, const TplIO& io, cudaStream_t st, Profiler* prof) {
#define ALG_TPL(nl, lm, k) \
  if (NL == nl && LMAX == lm && K == k) return launch<nl, lm, k>(io, st, prof);
  ALG_TPL(2, 1, 0)
  ALG_TPL(3, 1, 0) ALG_TPL(3, 1, 1)
#undef ALG_TPL
  throw CudaError("tpl_fwd: no fused kernel for this layer");
}

}  // namespace allegro
