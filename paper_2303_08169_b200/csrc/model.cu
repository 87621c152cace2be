// model.cu -- the Allegro energy and its analytic forces on the GPU.
//
// PAPER.md:128-131 (§2.1) and Eq. 1; concrete model = SURVEY.md
// §8(c) E1-E9.  Centre atoms are processed in chunks of complete CSR
// rows (each E_i depends on its own row only), so every segmented reduction (Gamma_i,
// its adjoint, E_i) stays inside one warp and is done in a fixed order: the result is
// deterministic and independent of the chunking.
//
// Per chunk (E edges, fp32 row-major [E][width] activations):
//   K3  k_geom        r_e (fp64 difference -> fp32), u(d), B(d) u, Y(r_hat)       E1-E3
//   A5  3 GEMMs       two-body MLP 16(12) -> 32 -> 64 -> 128, x0 = u MLP           E4-E5
//   per layer k:
//   A6  GEMM          w = x^k W_env / sqrt(D)                                      E6
//   A7+A8 k_tp_fwd    Gamma_i (warp per centre, lane = channel) and the "uuu" TP  E6
//   A9  GEMMs         V^{k+1} per out irrep; x^{k+1} = a x^k + b u [x^k,s] W_lat   E6
//   A10 k_energy      E_e = x^L . w_out, E_i = sigma nbar^-1/2 sum E_e + mu      E7-E8
//   A11 reverse mode  the same chain transposed (W^T GEMMs, k_tp_bwd), k_geom_bwd E9
// then over all atoms:
//   A12 k_force_warp  F_a = sum_{e in row a} (g_e - gT_e), gT_e = g_rev(e), fixed-order warp sum (fp64)
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>

#include "ctx.cuh"
#include "gemm.cuh"
#include "geom.cuh"
#include "layer.cuh"
#include "tp_fused.cuh"
#include "twobody.cuh"

namespace allegro {
namespace {

constexpr float kCSilu = 1.6765324703f;  // E[SiLU(z)^2]^-1/2 (reading row 5)
constexpr float kResA = 0.89442719099991588f;  // 2/sqrt5
constexpr float kResB = 0.44721359549995794f;  // 1/sqrt5

// ----------------------------------------------------------------- K3 geometry (helpers: geom.cuh)
// The first two-body layer is folded in (E4): a1 = (1/sqrt 12) z W0 with z = [onehot(Z_i),
// onehot(Z_j), u B(d)] never leaves registers -- two selected rows of W0 plus eight Bessel rows.
__global__ void __launch_bounds__(256) k_geom(ChunkPtrs ch, GeomParams gp, const double* __restrict__ apos,
                                              const int32_t* __restrict__ cidx, const int32_t* __restrict__ nbr,
                                              const int32_t* __restrict__ aspec, const int32_t* __restrict__ species,
                                              const float* __restrict__ w0, float s0, float* __restrict__ a1,
                                              float* __restrict__ Y, float* __restrict__ u) {
  __shared__ __align__(16) float sw[12][32];  // W0 rows 0..11 ([K = 12][N = 32]); read as broadcast float4
  __shared__ float4 stile[256 * 8];           // the block's a1 rows, 16-B chunks XOR-swizzled by row % 8
  for (int t = threadIdx.x; t < 12 * 32; t += blockDim.x) sw[t / 32][t % 32] = w0[t];
  __syncthreads();
  const int64_t e0 = (int64_t)blockIdx.x * blockDim.x;
  const int row = threadIdx.x;
  const int64_t e = e0 + row;
  if (e < ch.n_e) {
    const int64_t ge = ch.e0 + e;
    const int32_t i = cidx[ge], a = nbr[ge];
    float r[3];
    edge_vec(apos, i, a, r);
    const float d = sqrtf(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    const float x = d * gp.inv_rc;
    float uu = 0.f;
    if (x < 1.f) {
      const float x2 = x * x, x3 = x2 * x, x6 = x3 * x3;
      uu = 1.f - 28.f * x6 + 48.f * x6 * x - 21.f * x6 * x2;
    }
    u[e] = uu;
    const int zi = species[i], zj = aspec[a];
    const float pre = 2.f * gp.inv_rc / d;
    float zb[kNB];
#pragma unroll
    for (int q = 0; q < kNB; ++q) zb[q] = uu * pre * sinf(gp.freq[q] * d * gp.inv_rc);
    // a1 = s0 (z W0): one-hot rows first, then the Bessel rows in k order; W0 is read as
    // broadcast float4, the row goes to SMEM and leaves the block as coalesced 16-B stores
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
      stile[row * 8 + (c4 ^ (row & 7))] = make_float4(s0 * acc.x, s0 * acc.y, s0 * acc.z, s0 * acc.w);
    }
    const float inv = 1.f / d;
    const float nv[3] = {r[0] * inv, r[1] * inv, r[2] * inv};
    float y[9];
    sh_eval(nv, y, gp.lmax);
    if (gp.dsh == 4) {
      reinterpret_cast<float4*>(Y)[e] = make_float4(y[0], y[1], y[2], y[3]);
    } else {
      for (int q = 0; q < gp.dsh; ++q) Y[e * gp.dsh + q] = y[q];
    }
  }
  __syncthreads();
  const int rows = ch.n_e - e0 < 256 ? (int)(ch.n_e - e0) : 256;
  float4* dst = reinterpret_cast<float4*>(a1 + e0 * 32);
  for (int f = threadIdx.x; f < rows * 8; f += 256) {
    const int rr = f >> 3, c = f & 7;
    dst[f] = stile[rr * 8 + (c ^ (rr & 7))];
  }
}

// ----------------------------------------------------------------- A7+A8 TP forward
struct TpArgs {
  ChunkPtrs ch;
  const int32_t* row_ptr;
  const float* w;      // [E][NW] layer weights (env chunk at ENV_OFF)
  const float* Y;      // [E][DSH]
  const float* V;      // layer-K V store (K >= 1)
  float* T;            // T scratch (per out irrep [E][dim][n_to][C])
  float* G;            // [n_c][DSH][C]
  const float* Tb[kMaxIr];  // backward: T-bar per out irrep
  float* Vb;           // backward: V-bar store of layer K (K >= 1)
  float* wbar;         // backward: [E][NW]
  float* ybar;         // backward: [E][DSH] accumulated
  const float* gp;     // fused backward: [E][DSH][C] per-edge Gamma-bar terms
  int64_t e_cap;
  float inv_sqrt_nbar;
};

// Per-edge operands of the TP kernels.  Every edge loop below is software-pipelined: the
// loads of edge e+1 are issued before edge e is computed and stored (the stores of edge e
// may alias the next loads as far as the compiler knows, so without this every edge costs
// a full DRAM round trip per warp -- ncu: long-scoreboard stalls, 58 % of HBM).
template <int NL, int LMAX, int K>
struct VIn {
  using AR = Arch<NL, LMAX, K>;
  static constexpr int NY = K == 0 ? AR::DSH : 1;
  static constexpr int NE = K == 0 ? AR::NENV : 1;
  static constexpr int NV = K == 0 ? 1 : AR::DIN;
  float y[NY], we[NE], v[NV];
};

template <int NL, int LMAX, int K>
__device__ __forceinline__ void fetch_v(const TpArgs& t, int64_t e, int lane, VIn<NL, LMAX, K>& in) {
  using AR = Arch<NL, LMAX, K>;
  if constexpr (K == 0) {
#pragma unroll
    for (int m = 0; m < AR::DSH; ++m) in.y[m] = t.Y[e * AR::DSH + m];
#pragma unroll
    for (int l = 0; l < AR::NENV; ++l) in.we[l] = t.w[e * AR::NW + l * kC + lane];
  } else {
    static_for<AR::A.in.n>([&](auto I) {
      constexpr int ii = decltype(I)::value;
      constexpr int dim = ir_dim(AR::A.in.v[ii]);
      constexpr int off = AR::A.in.off(ii);
      constexpr int vbase = AR::v_base(ii);
      const float* src = t.V + (int64_t)vbase * t.e_cap + e * dim * kC + lane;
#pragma unroll
      for (int m = 0; m < dim; ++m) in.v[off + m] = src[m * kC];
    });
  }
}

// V of layer K from the fetched operands (K = 0: V0 = w_edge (x) Y)
template <int NL, int LMAX, int K>
__device__ __forceinline__ void expand_v(const VIn<NL, LMAX, K>& in, float* v) {
  using AR = Arch<NL, LMAX, K>;
  if constexpr (K == 0) {
#pragma unroll
    for (int m = 0; m < AR::DSH; ++m) v[m] = in.we[lm_l(m)] * in.y[m];
  } else {
#pragma unroll
    for (int m = 0; m < AR::DIN; ++m) v[m] = in.v[m];
  }
}

// w_env chunk and Y of one edge (the environment sum and its adjoint)
template <int NL, int LMAX, int K>
struct EnvIn {
  float y[Arch<NL, LMAX, K>::DSH], we[Arch<NL, LMAX, K>::NENV];
};

template <int NL, int LMAX, int K>
__device__ __forceinline__ void fetch_env(const TpArgs& t, int64_t e, int lane, EnvIn<NL, LMAX, K>& in) {
  using AR = Arch<NL, LMAX, K>;
#pragma unroll
  for (int m = 0; m < AR::DSH; ++m) in.y[m] = t.Y[e * AR::DSH + m];
#pragma unroll
  for (int l = 0; l < AR::NENV; ++l) in.we[l] = t.w[e * AR::NW + AR::ENV_OFF + l * kC + lane];
}

// L2 prefetch of edge e's per-edge blocks (each lane one 128-B line of a [dim][32] block): issued
// a fixed number of edges ahead of the register pipeline, holds no registers.  Measured on C5
// (profiles/r01_tp_prefetch_ab.jsonl): k_tp_fwd 46.9 -> 44.6 ms per step at distance 2; in
// k_tp_bwd it raises the register count (72 -> 96) and nets nothing, so it is off there.
#ifndef ALG_LAST_BATCH
#define ALG_LAST_BATCH 4  // k_last's per-edge loop: edges per batch of loads in flight
#endif
#ifndef ALG_ENV_BATCH
#define ALG_ENV_BATCH 4  // environment adjoint: edges per batch of loads in flight (1 = one edge ahead)
#endif
#ifndef ALG_GBAR_BATCH
#define ALG_GBAR_BATCH 8  // Gamma-bar row sum in k_env_adj: edges per batch (1 = one edge ahead)
#endif
#ifndef ALG_GAMMA_BATCH
#define ALG_GAMMA_BATCH 8  // Gamma_i: edges per batch of loads in flight (1 = the one-edge-ahead pipeline)
#endif
#ifndef ALG_TP_PFD_FWD
#define ALG_TP_PFD_FWD 2
#endif
#ifndef ALG_TP_PFD_BWD
#define ALG_TP_PFD_BWD 0
#endif
__device__ __forceinline__ void pf_lines(const float* base, int nlines, int lane) {
  if (lane < nlines) asm volatile("prefetch.global.L2 [%0];" ::"l"(base + lane * kC));
}

// L2 prefetch of edge e's environment operands: the w_env rows (lanes 0 .. NENV-1), the Y and Y-bar
// lines (the next two lanes); issued a few edges ahead of the register pipeline of the row loops,
// it holds no registers (the row kernels have one edge of loads in flight per warp otherwise)
#ifndef ALG_ROW_PFD
#define ALG_ROW_PFD 3
#endif
template <int NL, int LMAX, int K>
__device__ __forceinline__ void prefetch_env(const TpArgs& t, int64_t e, int lane, bool ybar) {
  using AR = Arch<NL, LMAX, K>;
  const float* p = nullptr;
  if (lane < AR::NENV) p = t.w + e * AR::NW + AR::ENV_OFF + lane * kC;
  else if (lane == AR::NENV) p = t.Y + e * AR::DSH;
  else if (lane == AR::NENV + 1 && ybar) p = t.ybar + e * AR::DSH;
  if (p) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <int NL, int LMAX, int K, bool TB>
__device__ __forceinline__ void prefetch_edge(const TpArgs& t, int64_t e, int lane) {
  using AR = Arch<NL, LMAX, K>;
  if constexpr (K == 0) {
    pf_lines(t.w + e * AR::NW, AR::NENV, lane);
  } else {
    static_for<AR::A.in.n>([&](auto I) {
      constexpr int ii = decltype(I)::value;
      constexpr int dim = ir_dim(AR::A.in.v[ii]);
      pf_lines(t.V + (int64_t)AR::v_base(ii) * t.e_cap + e * dim * kC, dim, lane);
    });
  }
  if constexpr (TB) {
    static_for<AR::A.out.n>([&](auto O) {
      constexpr int o = decltype(O)::value;
      constexpr int dim = ir_dim(AR::A.out.v[o]);
      constexpr int nto = AR::A.n_to[o];
      pf_lines(t.Tb[o] + e * dim * nto * kC, dim * nto, lane);
    });
  }
}

// one prefetch per lane per edge: lane i owns line i of the edge's V (or w) blocks followed by its
// T-bar blocks; a base pointer and a per-edge stride are all it holds across the edge loop
struct PfPlan {
  const float* base = nullptr;
  int64_t stride = 0;
};

template <int NL, int LMAX, int K>
__device__ __forceinline__ PfPlan pf_plan_bwd(const TpArgs& t, int lane) {
  using AR = Arch<NL, LMAX, K>;
  PfPlan pl;
  int first = 0;
  auto take = [&](const float* blk, int nlines, int64_t stride) {
    if (lane >= first && lane < first + nlines) pl.base = blk + (lane - first) * kC, pl.stride = stride;
    first += nlines;
  };
  if constexpr (K == 0) {
    take(t.w, AR::NENV, AR::NW);
  } else {
    static_for<AR::A.in.n>([&](auto I) {
      constexpr int ii = decltype(I)::value;
      constexpr int dim = ir_dim(AR::A.in.v[ii]);
      take(t.V + (int64_t)AR::v_base(ii) * t.e_cap, dim, dim * kC);
    });
  }
  static_for<AR::A.out.n>([&](auto O) {
    constexpr int o = decltype(O)::value;
    constexpr int dim = ir_dim(AR::A.out.v[o]);
    constexpr int nto = AR::A.n_to[o];
    take(t.Tb[o], dim * nto, dim * nto * kC);
  });
  return pl;
}

// lanes that own the butterfly total of value mm (warp_sum_multi<DSH>)
template <int DSH>
__device__ __forceinline__ bool owns_total(int lane, int mm) {
  constexpr int LP = DSH <= 1 ? 0 : DSH <= 2 ? 1 : DSH <= 4 ? 2 : DSH <= 8 ? 3 : 4;
  return mm < DSH && (lane & ((1 << (5 - LP)) - 1)) == 0;
}

// GAMMA_ONLY: only the environment sums Gamma_i (k_gamma; the fused TP + TP-linear kernel of
// tp_fused.cu does the rest)
template <int NL, int LMAX, int K, bool GAMMA_ONLY = false>
__global__ void __launch_bounds__(128) k_tp_fwd(TpArgs t) {
  using AR = Arch<NL, LMAX, K>;
  constexpr LayerArch A = AR::A;
  const int lane = threadIdx.x & 31;
  const int64_t ii = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ii >= t.ch.n_c) return;
  const int64_t r0 = t.row_ptr[t.ch.a0 + ii] - t.ch.e0, r1 = t.row_ptr[t.ch.a0 + ii + 1] - t.ch.e0;
  float G[AR::DSH];
#pragma unroll
  for (int m = 0; m < AR::DSH; ++m) G[m] = 0.f;
  if (r1 > r0) {
#if ALG_GAMMA_BATCH > 1
    // ALG_GAMMA_BATCH edges' loads in flight at once (the row's edges are summed in edge order as
    // before): the one-edge-ahead pipeline left the warp waiting one L2 round trip per edge
    for (int64_t e0 = r0; e0 < r1; e0 += ALG_GAMMA_BATCH) {
      EnvIn<NL, LMAX, K> buf[ALG_GAMMA_BATCH];
#pragma unroll
      for (int j = 0; j < ALG_GAMMA_BATCH; ++j)
        if (e0 + j < r1) fetch_env<NL, LMAX, K>(t, e0 + j, lane, buf[j]);
      {  // warm L2 with the next batch: lane -> (edge, line), NENV w lines + the Y line per edge
        constexpr int kL = AR::NENV + 1;
        const int j = lane / kL, part = lane % kL;
        const int64_t en = e0 + ALG_GAMMA_BATCH + j;
        if (j < ALG_GAMMA_BATCH && en < r1) {
          const float* pf = part < AR::NENV ? t.w + en * AR::NW + AR::ENV_OFF + part * kC : t.Y + en * AR::DSH;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pf));
        }
      }
#pragma unroll
      for (int j = 0; j < ALG_GAMMA_BATCH; ++j)
        if (e0 + j < r1) {
#pragma unroll
          for (int m = 0; m < AR::DSH; ++m) G[m] = fmaf(buf[j].we[lm_l(m)], buf[j].y[m], G[m]);
        }
    }
#else
    EnvIn<NL, LMAX, K> nx;
    fetch_env<NL, LMAX, K>(t, r0, lane, nx);
    for (int64_t e = r1 - 1 < r0 + ALG_ROW_PFD ? r1 - 1 : r0 + ALG_ROW_PFD; e > r0; --e)
      prefetch_env<NL, LMAX, K>(t, e, lane, false);
    for (int64_t e = r0; e < r1; ++e) {
      const EnvIn<NL, LMAX, K> cur = nx;
      fetch_env<NL, LMAX, K>(t, e + 1 < r1 ? e + 1 : e, lane, nx);
      if (e + 1 + ALG_ROW_PFD < r1) prefetch_env<NL, LMAX, K>(t, e + 1 + ALG_ROW_PFD, lane, false);
#pragma unroll
      for (int m = 0; m < AR::DSH; ++m) G[m] = fmaf(cur.we[lm_l(m)], cur.y[m], G[m]);
    }
#endif
  }
#pragma unroll
  for (int m = 0; m < AR::DSH; ++m) {
    G[m] *= t.inv_sqrt_nbar;
    t.G[(ii * AR::DSH + m) * kC + lane] = G[m];
  }
  if (GAMMA_ONLY || r1 <= r0) return;
  VIn<NL, LMAX, K> nx;
  fetch_v<NL, LMAX, K>(t, r0, lane, nx);
  for (int64_t e = r0; e < r1; ++e) {
    float v[AR::DIN];
    expand_v<NL, LMAX, K>(nx, v);
    fetch_v<NL, LMAX, K>(t, e + 1 < r1 ? e + 1 : e, lane, nx);
    if constexpr (ALG_TP_PFD_FWD > 0)
      if (e + ALG_TP_PFD_FWD < r1) prefetch_edge<NL, LMAX, K, false>(t, e + ALG_TP_PFD_FWD, lane);
    float T[AR::DT];
#pragma unroll
    for (int q = 0; q < AR::DT; ++q) T[q] = 0.f;
    static_for<A.n_paths>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      constexpr int L1 = AR::A.path[q].a.l, L2 = AR::A.path[q].b.l, LO = AR::A.path[q].o.l;
      constexpr int D2 = 2 * L2 + 1, D3 = 2 * LO + 1;
      constexpr double alpha = csqrt(2.0 * LO + 1.0);
      static_for<(2 * L1 + 1) * D2 * D3>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int m1 = i / (D2 * D3), m2 = (i / D3) % D2, m3 = i % D3;
        constexpr float c = (float)(alpha * W3j<L1, L2, LO>::t.v[i]);
        constexpr int it = AR::A.t_off[q] + m3, iv = AR::A.in_off[q] + m1, ig = AR::A.sh_off[q] + m2;
        if constexpr (c != 0.f) T[it] = fmaf(c * v[iv], G[ig], T[it]);
      });
    });
    static_for<A.n_paths>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      constexpr int o = AR::A.out_idx[q];
      constexpr int dim = ir_dim(AR::A.out.v[o]);
      constexpr int nto = AR::A.n_to[o];
      constexpr int ol = AR::A.out_local[q];
      constexpr int toff = AR::A.t_off[q];
      constexpr int tbase = AR::t_base(o);
      float* dst = t.T + (int64_t)tbase * t.e_cap + (e * dim * nto + ol) * kC + lane;
#pragma unroll
      for (int m = 0; m < dim; ++m) dst[m * nto * kC] = T[toff + m];
    });
  }
}

// ----------------------------------------------------------------- A11 TP backward
template <int NL, int LMAX, int K>
struct BwdIn {
  VIn<NL, LMAX, K> v;
  float tb[Arch<NL, LMAX, K>::DT];
  float yb_old;  // K = 0: this lane's Y-bar total slot (read-modify-write)
};

template <int NL, int LMAX, int K>
__device__ __forceinline__ void fetch_bwd(const TpArgs& t, int64_t e, int lane, int mm, BwdIn<NL, LMAX, K>& in) {
  using AR = Arch<NL, LMAX, K>;
  fetch_v<NL, LMAX, K>(t, e, lane, in.v);
  static_for<AR::A.n_paths>([&](auto Q) {
    constexpr int q = decltype(Q)::value;
    constexpr int o = AR::A.out_idx[q];
    constexpr int dim = ir_dim(AR::A.out.v[o]);
    constexpr int nto = AR::A.n_to[o];
    constexpr int ol = AR::A.out_local[q];
    constexpr int toff = AR::A.t_off[q];
    const float* src = t.Tb[o] + (e * dim * nto + ol) * kC + lane;
#pragma unroll
    for (int m = 0; m < dim; ++m) in.tb[toff + m] = src[m * nto * kC];
  });
  if constexpr (K == 0) in.yb_old = owns_total<AR::DSH>(lane, mm) ? t.ybar[e * AR::DSH + mm] : 0.f;
}

// environment adjoint of one CSR row: w_env-bar and Y-bar from the complete Gamma-bar_i
template <int NL, int LMAX, int K>
__device__ __forceinline__ void env_adjoint(const TpArgs& t, int64_t r0, int64_t r1, int lane, int mm,
                                            const float (&Gb)[Arch<NL, LMAX, K>::DSH]) {
  using AR = Arch<NL, LMAX, K>;
  struct EnvB {
    EnvIn<NL, LMAX, K> env;
    float yb_old;
  };
  auto fetch_envb = [&](int64_t e, EnvB& in) {
    fetch_env<NL, LMAX, K>(t, e, lane, in.env);
    in.yb_old = owns_total<AR::DSH>(lane, mm) ? t.ybar[e * AR::DSH + mm] : 0.f;
  };
  auto adjoint_edge = [&](int64_t e, const EnvB& cur) {  // w_env-bar and Y-bar of one edge
    float wb[AR::NENV];
#pragma unroll
    for (int l = 0; l < AR::NENV; ++l) wb[l] = 0.f;
    float prod[AR::DSH];
#pragma unroll
    for (int m = 0; m < AR::DSH; ++m) {
      wb[lm_l(m)] = fmaf(Gb[m], cur.env.y[m], wb[lm_l(m)]);
      prod[m] = Gb[m] * cur.env.we[lm_l(m)];
    }
    int mq;
    const float s = warp_sum_multi<AR::DSH>(prod, lane, &mq);
#pragma unroll
    for (int l = 0; l < AR::NENV; ++l) t.wbar[e * AR::NW + AR::ENV_OFF + l * kC + lane] = t.inv_sqrt_nbar * wb[l];
    if (owns_total<AR::DSH>(lane, mm)) t.ybar[e * AR::DSH + mm] = cur.yb_old + t.inv_sqrt_nbar * s;
  };
#if ALG_ENV_BATCH > 1
  // ALG_ENV_BATCH edges' inputs in flight at once (each edge's outputs depend on that edge only)
  for (int64_t e0 = r0; e0 < r1; e0 += ALG_ENV_BATCH) {
    EnvB buf[ALG_ENV_BATCH];
#pragma unroll
    for (int j = 0; j < ALG_ENV_BATCH; ++j)
      if (e0 + j < r1) fetch_envb(e0 + j, buf[j]);
    {  // warm L2 with the next batch: lane -> (edge, line): NENV w lines, Y, Y-bar
      constexpr int kL = AR::NENV + 2;
      const int j = lane / kL, part = lane % kL;
      const int64_t en2 = e0 + ALG_ENV_BATCH + j;
      if (j < ALG_ENV_BATCH && en2 < r1) {
        const float* pf = part < AR::NENV ? t.w + en2 * AR::NW + AR::ENV_OFF + part * kC
                                          : (part == AR::NENV ? t.Y + en2 * AR::DSH : t.ybar + en2 * AR::DSH);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pf));
      }
    }
#pragma unroll
    for (int j = 0; j < ALG_ENV_BATCH; ++j)
      if (e0 + j < r1) adjoint_edge(e0 + j, buf[j]);
  }
#else
  EnvB en;
  fetch_envb(r0, en);
  for (int64_t e = r1 - 1 < r0 + ALG_ROW_PFD ? r1 - 1 : r0 + ALG_ROW_PFD; e > r0; --e)
    prefetch_env<NL, LMAX, K>(t, e, lane, true);
  for (int64_t e = r0; e < r1; ++e) {  // pipelined one edge ahead (+ L2 prefetch further ahead)
    const EnvB cur = en;
    fetch_envb(e + 1 < r1 ? e + 1 : e, en);
    if (e + 1 + ALG_ROW_PFD < r1) prefetch_env<NL, LMAX, K>(t, e + 1 + ALG_ROW_PFD, lane, true);
    adjoint_edge(e, cur);
  }
#endif
}

template <int NL, int LMAX, int K>
__global__ void __launch_bounds__(128) k_tp_bwd(TpArgs t) {
  using AR = Arch<NL, LMAX, K>;
  constexpr LayerArch A = AR::A;
  const int lane = threadIdx.x & 31;
  const int64_t ii = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ii >= t.ch.n_c) return;
  const int64_t r0 = t.row_ptr[t.ch.a0 + ii] - t.ch.e0, r1 = t.row_ptr[t.ch.a0 + ii + 1] - t.ch.e0;
  if (r1 <= r0) return;  // no edges: Gamma-bar = 0, nothing to write
  constexpr int LP = AR::DSH <= 1 ? 0 : AR::DSH <= 2 ? 1 : AR::DSH <= 4 ? 2 : AR::DSH <= 8 ? 3 : 4;
  const int mm = lane >> (5 - LP);  // value index of this lane's butterfly total
  float G[AR::DSH], Gb[AR::DSH];
#pragma unroll
  for (int m = 0; m < AR::DSH; ++m) {
    G[m] = t.G[(ii * AR::DSH + m) * kC + lane];
    Gb[m] = 0.f;
  }
  BwdIn<NL, LMAX, K> nx;
  fetch_bwd<NL, LMAX, K>(t, r0, lane, mm, nx);
  [[maybe_unused]] const PfPlan pf = ALG_TP_PFD_BWD > 0 ? pf_plan_bwd<NL, LMAX, K>(t, lane) : PfPlan{};
  for (int64_t e = r0; e < r1; ++e) {
    const BwdIn<NL, LMAX, K> cur = nx;
    fetch_bwd<NL, LMAX, K>(t, e + 1 < r1 ? e + 1 : e, lane, mm, nx);
    if constexpr (ALG_TP_PFD_BWD > 0)
      if (pf.base != nullptr && e + ALG_TP_PFD_BWD < r1)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pf.base + (e + ALG_TP_PFD_BWD) * pf.stride));
    float v[AR::DIN], vb[AR::DIN];
    expand_v<NL, LMAX, K>(cur.v, v);
#pragma unroll
    for (int q = 0; q < AR::DIN; ++q) vb[q] = 0.f;
    static_for<A.n_paths>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      constexpr int L1 = AR::A.path[q].a.l, L2 = AR::A.path[q].b.l, LO = AR::A.path[q].o.l;
      constexpr int D2 = 2 * L2 + 1, D3 = 2 * LO + 1;
      constexpr double alpha = csqrt(2.0 * LO + 1.0);
      static_for<(2 * L1 + 1) * D2 * D3>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int m1 = i / (D2 * D3), m2 = (i / D3) % D2, m3 = i % D3;
        constexpr float c = (float)(alpha * W3j<L1, L2, LO>::t.v[i]);
        constexpr int it = AR::A.t_off[q] + m3, iv = AR::A.in_off[q] + m1, ig = AR::A.sh_off[q] + m2;
        if constexpr (c != 0.f) {
          const float ct = c * cur.tb[it];
          vb[iv] = fmaf(ct, G[ig], vb[iv]);
          Gb[ig] = fmaf(ct, v[iv], Gb[ig]);
        }
      });
    });
    if constexpr (K == 0) {
      // V0 = w_edge (x) Y:  wbar_edge[l] = sum_m vb[m] Y[m];  Ybar[m] += sum_c vb[m] w_edge[l]
      float wb[AR::NENV];
#pragma unroll
      for (int l = 0; l < AR::NENV; ++l) wb[l] = 0.f;
      float prod[AR::DSH];
#pragma unroll
      for (int m = 0; m < AR::DSH; ++m) {
        wb[lm_l(m)] = fmaf(vb[m], cur.v.y[m], wb[lm_l(m)]);
        prod[m] = vb[m] * cur.v.we[lm_l(m)];
      }
      int mq;
      const float s = warp_sum_multi<AR::DSH>(prod, lane, &mq);
#pragma unroll
      for (int l = 0; l < AR::NENV; ++l) t.wbar[e * AR::NW + l * kC + lane] = wb[l];
      if (owns_total<AR::DSH>(lane, mm)) t.ybar[e * AR::DSH + mm] = cur.yb_old + s;
    } else {
      static_for<AR::A.in.n>([&](auto I) {
        constexpr int ii2 = decltype(I)::value;
        constexpr int dim = ir_dim(AR::A.in.v[ii2]);
        constexpr int off = AR::A.in.off(ii2);
        constexpr int vbase = AR::v_base(ii2);
        float* dst = t.Vb + (int64_t)vbase * t.e_cap + e * dim * kC + lane;
#pragma unroll
        for (int m = 0; m < dim; ++m) dst[m * kC] = vb[off + m];
      });
    }
  }
  env_adjoint<NL, LMAX, K>(t, r0, r1, lane, mm, Gb);
}

// Fused backward path (tp_fused.cu): Gamma-bar_i = sum over the row, in edge order, of the
// per-edge terms gp that k_tpl_bwd wrote, then the environment adjoint of the row.
template <int NL, int LMAX, int K>
__global__ void __launch_bounds__(128) k_env_adj(TpArgs t) {
  using AR = Arch<NL, LMAX, K>;
  const int lane = threadIdx.x & 31;
  const int64_t ii = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ii >= t.ch.n_c) return;
  const int64_t r0 = t.row_ptr[t.ch.a0 + ii] - t.ch.e0, r1 = t.row_ptr[t.ch.a0 + ii + 1] - t.ch.e0;
  if (r1 <= r0) return;
  constexpr int LP = AR::DSH <= 1 ? 0 : AR::DSH <= 2 ? 1 : AR::DSH <= 4 ? 2 : AR::DSH <= 8 ? 3 : 4;
  const int mm = lane >> (5 - LP);
  float Gb[AR::DSH];
#pragma unroll
  for (int m = 0; m < AR::DSH; ++m) Gb[m] = 0.f;
#if ALG_GBAR_BATCH > 1
  for (int64_t e0 = r0; e0 < r1; e0 += ALG_GBAR_BATCH) {  // loads of ALG_GBAR_BATCH edges in flight
    float buf[ALG_GBAR_BATCH][AR::DSH];
#pragma unroll
    for (int j = 0; j < ALG_GBAR_BATCH; ++j)
#pragma unroll
      for (int m = 0; m < AR::DSH; ++m) buf[j][m] = e0 + j < r1 ? t.gp[((e0 + j) * AR::DSH + m) * kC + lane] : 0.f;
    {  // warm L2 with the next batch: lane -> (edge, m line)
      const int j = lane / AR::DSH, m = lane % AR::DSH;
      const int64_t en2 = e0 + ALG_GBAR_BATCH + j;
      if (j < ALG_GBAR_BATCH && en2 < r1) asm volatile("prefetch.global.L2 [%0];" ::"l"(t.gp + (en2 * AR::DSH + m) * kC));
    }
#pragma unroll
    for (int j = 0; j < ALG_GBAR_BATCH; ++j)
      if (e0 + j < r1) {  // the row's edges in order, as before
#pragma unroll
        for (int m = 0; m < AR::DSH; ++m) Gb[m] += buf[j][m];
      }
  }
#else
  float nx[AR::DSH];
#pragma unroll
  for (int m = 0; m < AR::DSH; ++m) nx[m] = t.gp[(r0 * AR::DSH + m) * kC + lane];
  for (int64_t e = r0 + 1; e < r1 && e <= r0 + ALG_ROW_PFD; ++e)
    if (lane < AR::DSH) asm volatile("prefetch.global.L2 [%0];" ::"l"(t.gp + (e * AR::DSH + lane) * kC));
  for (int64_t e = r0; e < r1; ++e) {  // pipelined one edge ahead (+ L2 prefetch further ahead)
    float cur[AR::DSH];
#pragma unroll
    for (int m = 0; m < AR::DSH; ++m) cur[m] = nx[m];
    const int64_t en = e + 1 < r1 ? e + 1 : e;
    if (lane < AR::DSH && e + 1 + ALG_ROW_PFD < r1)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(t.gp + ((e + 1 + ALG_ROW_PFD) * AR::DSH + lane) * kC));
#pragma unroll
    for (int m = 0; m < AR::DSH; ++m) nx[m] = t.gp[(en * AR::DSH + m) * kC + lane];
#pragma unroll
    for (int m = 0; m < AR::DSH; ++m) Gb[m] += cur[m];
  }
#endif
  env_adjoint<NL, LMAX, K>(t, r0, r1, lane, mm, Gb);
}

// ----------------------------------------------------------------- the last layer, fused
// Layer L-1 has only scalar outputs (T = s) and no TP-linear, and its latent update is folded into
// the read-out (below), so its whole forward + reverse is per CSR row: one warp per centre computes
// Gamma_i, then per edge s (the TP), E_e, u-bar and E-bar (as k_energy_last), s-bar = T-bar and the
// TP adjoint (V-bar^{L-1}, Gamma-bar in registers), and finally the environment adjoint of the row.
// Same arithmetic in the same order as k_tp_fwd<L-1> + k_energy_last + k_tp_bwd<L-1> (bit-identical),
// without their T, s-bar, Gamma and second V round trips through HBM.
struct LastArgs {
  TpArgs t;
  const int32_t* species;
  const float* x;     // x^{L-1} [E][D]
  const float* u;     // [E]
  const float* wout;  // [D]
  const float* q;     // [fan_lat]: x rows, then the scalar rows (path, c)
  double* e_atom;
  float* ubar;
  float* ebar;
  double s0, s1, mu0, mu1;
  float ra, sf;
};

template <int NL, int LMAX>
__global__ void __launch_bounds__(128) k_last(LastArgs a) {
  constexpr int K = NL - 1;
  using AR = Arch<NL, LMAX, K>;
  constexpr LayerArch A = AR::A;
  constexpr int NS = A.n_s;  // every path of the last layer is scalar
  static_assert(NS == A.n_paths && NS <= 3, "last layer: scalar paths only, <= 96 channels");
  static_assert(A.t_off[NS > 1 ? NS - 1 : 0] == (NS > 1 ? NS - 1 : 0), "last layer: T index = path index");
  const TpArgs& t = a.t;
  const int lane = threadIdx.x & 31;
  const int64_t ii = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ii >= t.ch.n_c) return;
  const int64_t at = t.ch.a0 + ii;
  const int64_t r0 = t.row_ptr[at] - t.ch.e0, r1 = t.row_ptr[at + 1] - t.ch.e0;
  const int z = a.species[at];
  const double sig = z == 0 ? a.s0 : a.s1;
  if (r1 <= r0) {
    if (lane == 0) a.e_atom[at] = z == 0 ? a.mu0 : a.mu1;  // sig nbar^-1/2 * 0 + mu
    return;
  }
  // Gamma_i (as k_tp_fwd)
  float G[AR::DSH];
#pragma unroll
  for (int m = 0; m < AR::DSH; ++m) G[m] = 0.f;
  for (int64_t e0 = r0; e0 < r1; e0 += ALG_GAMMA_BATCH) {  // batches of loads in flight, edge order kept
    EnvIn<NL, LMAX, K> buf[ALG_GAMMA_BATCH];
#pragma unroll
    for (int j = 0; j < ALG_GAMMA_BATCH; ++j)
      if (e0 + j < r1) fetch_env<NL, LMAX, K>(t, e0 + j, lane, buf[j]);
#pragma unroll
    for (int j = 0; j < ALG_GAMMA_BATCH; ++j)
      if (e0 + j < r1) {
#pragma unroll
        for (int m = 0; m < AR::DSH; ++m) G[m] = fmaf(buf[j].we[lm_l(m)], buf[j].y[m], G[m]);
      }
  }
#pragma unroll
  for (int m = 0; m < AR::DSH; ++m) G[m] *= t.inv_sqrt_nbar;
  // read-out constants (as k_energy_last)
  const float eb = (float)sig * t.inv_sqrt_nbar;
  const float4 w4 = reinterpret_cast<const float4*>(a.wout)[lane];
  const float4 q4 = reinterpret_cast<const float4*>(a.q)[lane];
  float qs[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) qs[k] = k < NS ? a.q[128 + lane + 32 * k] : 0.f;
  float acc = 0.f, Gb[AR::DSH];
#pragma unroll
  for (int m = 0; m < AR::DSH; ++m) Gb[m] = 0.f;
  struct In {
    VIn<NL, LMAX, K> v;
    float4 x4;
    float ue;
  };
  auto fetch = [&](int64_t e, In& in) {
    fetch_v<NL, LMAX, K>(t, e, lane, in.v);
    in.x4 = reinterpret_cast<const float4*>(a.x + e * kD)[lane];
    in.ue = a.u[e];
  };
  auto pf = [&](int64_t e) {  // V rows (lanes 0 .. DIN-1) and the x row (4 lines) of edge e
    const float* q = nullptr;
    if (lane < AR::DIN) {
      int ii2 = 0, m = lane;
      static_for<A.in.n>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int dim = ir_dim(A.in.v[i]);
        constexpr int off = A.in.off(i);
        if (lane >= off && lane < off + dim) ii2 = AR::v_base(i), m = lane - off, q = t.V + (int64_t)ii2 * t.e_cap + (e * dim + m) * kC;
      });
    } else if (lane < AR::DIN + 4) {
      q = a.x + e * kD + (lane - AR::DIN) * 32;
    }
    if (q) asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
  };
  // the row's edges in order (E_e sum, Gamma-bar), ALG_LAST_BATCH edges' inputs in flight at once
  auto process = [&](int64_t e, const In& cur) {
    float v[AR::DIN];
    expand_v<NL, LMAX, K>(cur.v, v);
    // T = s (scalar outputs only)
    float T[AR::DT];
#pragma unroll
    for (int q = 0; q < AR::DT; ++q) T[q] = 0.f;
    static_for<A.n_paths>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      constexpr int L1 = A.path[q].a.l, L2 = A.path[q].b.l, LO = A.path[q].o.l;
      constexpr int D2 = 2 * L2 + 1, D3 = 2 * LO + 1;
      constexpr double alpha = csqrt(2.0 * LO + 1.0);
      static_for<(2 * L1 + 1) * D2 * D3>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int m1 = i / (D2 * D3), m2 = (i / D3) % D2, m3 = i % D3;
        constexpr float c = (float)(alpha * W3j<L1, L2, LO>::t.v[i]);
        constexpr int it = A.t_off[q] + m3, iv = A.in_off[q] + m1, ig = A.sh_off[q] + m2;
        if constexpr (c != 0.f) T[it] = fmaf(c * v[iv], G[ig], T[it]);
      });
    });
    // E_e = a (x.w_out) + (b u / sqrt(fan)) ([x, s].q)
    const float4 x4 = cur.x4;
    float d1 = x4.x * w4.x;
    d1 = fmaf(x4.y, w4.y, d1);
    d1 = fmaf(x4.z, w4.z, d1);
    d1 = fmaf(x4.w, w4.w, d1);
    float d2 = x4.x * q4.x;
    d2 = fmaf(x4.y, q4.y, d2);
    d2 = fmaf(x4.z, q4.z, d2);
    d2 = fmaf(x4.w, q4.w, d2);
#pragma unroll
    for (int k = 0; k < 3; ++k) d2 = fmaf(k < NS ? T[k < NS ? k : 0] : 0.f, qs[k], d2);  // qs = 0 beyond NS
    d1 = warp_sum(d1);
    d2 = warp_sum(d2);
    acc += a.ra * d1 + a.sf * cur.ue * d2;
    if (lane == 0) {
      a.ubar[e] = eb * a.sf * d2;
      a.ebar[e] = eb;
    }
    // T-bar = s-bar = E-bar u (b / sqrt(fan)) q_s; the TP adjoint (as k_tp_bwd)
    float tb[AR::DT];
#pragma unroll
    for (int q = 0; q < AR::DT; ++q) tb[q] = 0.f;
#pragma unroll
    for (int k = 0; k < NS; ++k) tb[k] = eb * cur.ue * a.sf * qs[k];
    float vb[AR::DIN];
#pragma unroll
    for (int q = 0; q < AR::DIN; ++q) vb[q] = 0.f;
    static_for<A.n_paths>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      constexpr int L1 = A.path[q].a.l, L2 = A.path[q].b.l, LO = A.path[q].o.l;
      constexpr int D2 = 2 * L2 + 1, D3 = 2 * LO + 1;
      constexpr double alpha = csqrt(2.0 * LO + 1.0);
      static_for<(2 * L1 + 1) * D2 * D3>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int m1 = i / (D2 * D3), m2 = (i / D3) % D2, m3 = i % D3;
        constexpr float c = (float)(alpha * W3j<L1, L2, LO>::t.v[i]);
        constexpr int it = A.t_off[q] + m3, iv = A.in_off[q] + m1, ig = A.sh_off[q] + m2;
        if constexpr (c != 0.f) {
          const float ct = c * tb[it];
          vb[iv] = fmaf(ct, G[ig], vb[iv]);
          Gb[ig] = fmaf(ct, v[iv], Gb[ig]);
        }
      });
    });
    static_for<A.in.n>([&](auto I) {
      constexpr int ii2 = decltype(I)::value;
      constexpr int dim = ir_dim(A.in.v[ii2]);
      constexpr int off = A.in.off(ii2);
      constexpr int vbase = AR::v_base(ii2);
      float* dst = t.Vb + (int64_t)vbase * t.e_cap + e * dim * kC + lane;
#pragma unroll
      for (int m = 0; m < dim; ++m) dst[m * kC] = vb[off + m];
    });
  };
  for (int64_t e = r0 + ALG_LAST_BATCH; e < r1 && e < r0 + 2 * ALG_LAST_BATCH; ++e) pf(e);
  for (int64_t e0 = r0; e0 < r1; e0 += ALG_LAST_BATCH) {
    In buf[ALG_LAST_BATCH];
#pragma unroll
    for (int j = 0; j < ALG_LAST_BATCH; ++j)
      if (e0 + j < r1) fetch(e0 + j, buf[j]);
#pragma unroll
    for (int j = 0; j < ALG_LAST_BATCH; ++j)  // warm L2 two batches ahead
      if (e0 + 2 * ALG_LAST_BATCH + j < r1) pf(e0 + 2 * ALG_LAST_BATCH + j);
#pragma unroll
    for (int j = 0; j < ALG_LAST_BATCH; ++j)
      if (e0 + j < r1) process(e0 + j, buf[j]);
  }
  if (lane == 0) a.e_atom[at] = sig * (double)t.inv_sqrt_nbar * (double)acc + (z == 0 ? a.mu0 : a.mu1);
  constexpr int LP = AR::DSH <= 1 ? 0 : AR::DSH <= 2 ? 1 : AR::DSH <= 4 ? 2 : AR::DSH <= 8 ? 3 : 4;
  env_adjoint<NL, LMAX, K>(t, r0, r1, lane, lane >> (5 - LP), Gb);
}

void last_dispatch(int NL, int LMAX, const LastArgs& a, cudaStream_t st, Profiler* prof, const LayerInfo& L) {
  const unsigned blocks = (unsigned)((a.t.ch.n_c * 32 + 127) / 128);
  if (blocks == 0) return;
  const double E = (double)a.t.ch.n_e;
  const int dsh = (LMAX + 1) * (LMAX + 1);
  const double vin = (double)L.A.dim_in * kC, nenv = LMAX + 1;
  // algorithmic: Gamma + TP + adjoint FMAs and the read-out dots; bytes: w_env + Y twice (Gamma, env
  // adjoint), V, x, u in; V-bar, w-bar, Y-bar, u-bar, E-bar out
  const double flops = E * (kC * 2.0 * (3.0 * L.tp_nnz + 3.0 * dsh) + 6.0 * 128);
  const double bytes = 4.0 * E * (2.0 * (nenv * kC + dsh) + vin + 128 + 1 + vin + nenv * kC + 2.0 * dsh + 2);
  {
    ProfScope ps_(prof, st, PK_LAST, flops, bytes, "last layer (fused)");
#define ALG_LAST(nl, lm) \
  if (NL == nl && LMAX == lm) k_last<nl, lm><<<blocks, 128, 0, st>>>(a);
    ALG_LAST(2, 1) ALG_LAST(2, 2) ALG_LAST(3, 0) ALG_LAST(3, 1) ALG_LAST(3, 2)
#undef ALG_LAST
  }
  ALG_LAUNCH_CHECK();
}

// ----------------------------------------------------------------- A10 energies
// Last layer folded into the linear read-out: with w_out = W_o1 W_o2 / sqrt(D 32)
// and q = W_lat(L-1) w_out (all linear),
//   E_e = a (x.w_out) + (b u / sqrt(fan)) ([x, s].q)            (x = x^{L-1}, s = its scalars)
// and the reverse mode of the last layer is rank one per edge:
//   ubar = Ebar (b / sqrt(fan)) [x, s].q,  sbar = Ebar u (b / sqrt(fan)) q_s,
//   xbar^{L-1} = Ebar (a w_out + u (b / sqrt(fan)) q_x)  (applied in the env^T GEMM epilogue).
__global__ void k_energy_last(ChunkPtrs ch, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ species,
                              const float* __restrict__ x, const float* __restrict__ sc, int nsc,
                              const float* __restrict__ u, const float* __restrict__ wout,
                              const float* __restrict__ q, double* __restrict__ e_atom, float* __restrict__ ubar,
                              float* __restrict__ sbar, float* __restrict__ ebar, double s0, double s1, double mu0,
                              double mu1, float inv_sqrt_nbar, float ra, float sf) {
  const int lane = threadIdx.x & 31;
  const int64_t ii = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ii >= ch.n_c) return;
  const int64_t at = ch.a0 + ii;
  const int64_t r0 = row_ptr[at] - ch.e0, r1 = row_ptr[at + 1] - ch.e0;
  const int z = species[at];
  const double sig = z == 0 ? s0 : s1;
  const float eb = (float)sig * inv_sqrt_nbar;
  const float4 w4 = reinterpret_cast<const float4*>(wout)[lane];
  const float4 q4 = reinterpret_cast<const float4*>(q)[lane];
  float qs[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) qs[k] = (lane + 32 * k < nsc) ? q[128 + lane + 32 * k] : 0.f;
  float acc = 0.f;
  // pipelined one edge ahead (see the TP kernels)
  auto fetch = [&](int64_t e, float4& x4, float* sv, float& ue) {
    x4 = reinterpret_cast<const float4*>(x + e * kD)[lane];
#pragma unroll
    for (int k = 0; k < 3; ++k) sv[k] = (lane + 32 * k < nsc) ? sc[e * nsc + lane + 32 * k] : 0.f;
    ue = u[e];
  };
  float4 xn;
  float sn[3], un = 0.f;
  if (r1 > r0) fetch(r0, xn, sn, un);
  for (int64_t e = r0; e < r1; ++e) {
    const float4 x4 = xn;
    const float s3[3] = {sn[0], sn[1], sn[2]};
    const float ue = un;
    fetch(e + 1 < r1 ? e + 1 : e, xn, sn, un);
    float d1 = x4.x * w4.x;
    d1 = fmaf(x4.y, w4.y, d1);
    d1 = fmaf(x4.z, w4.z, d1);
    d1 = fmaf(x4.w, w4.w, d1);
    float d2 = x4.x * q4.x;
    d2 = fmaf(x4.y, q4.y, d2);
    d2 = fmaf(x4.z, q4.z, d2);
    d2 = fmaf(x4.w, q4.w, d2);
#pragma unroll
    for (int k = 0; k < 3; ++k) d2 = fmaf(s3[k], qs[k], d2);  // qs = 0 beyond nsc
    d1 = warp_sum(d1);
    d2 = warp_sum(d2);
    acc += ra * d1 + sf * ue * d2;
    if (lane == 0) {
      ubar[e] = eb * sf * d2;
      ebar[e] = eb;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (lane + 32 * k < nsc) sbar[e * nsc + lane + 32 * k] = eb * ue * sf * qs[k];
  }
  if (lane == 0) e_atom[at] = sig * (double)inv_sqrt_nbar * (double)acc + (z == 0 ? mu0 : mu1);
}

// ubar[e] += coef <P[e], Q[e]> over 128 (warp per edge)
__global__ void k_rowdot(int64_t E, const float* __restrict__ P, const float* __restrict__ Q, float coef,
                         const float* __restrict__ inv_u, float* __restrict__ ubar) {
  const int lane = threadIdx.x & 31;
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (e >= E) return;
  const float4 p = reinterpret_cast<const float4*>(P + e * kD)[lane];
  const float4 q = reinterpret_cast<const float4*>(Q + e * kD)[lane];
  float s = warp_sum(p.x * q.x + p.y * q.y + p.z * q.z + p.w * q.w);
  if (inv_u) {  // x^0 = u m: <x-bar^0, m> = <x-bar^0, x^0> / u (u = 0: u' = 0 there, the term drops)
    const float ur = inv_u[e];
    s = ur != 0.f ? s / ur : 0.f;
  }
  if (lane == 0) ubar[e] += coef * s;
}

// ----------------------------------------------------------------- E9 geometry reverse
// zbar (Bessel part) = s0 ab1 W0[4..11]^T is formed here from ab1 (the first two-body layer's
// reverse, folded in like its forward in k_geom); the one-hot rows carry no gradient.
__global__ void __launch_bounds__(256) k_geom_bwd(ChunkPtrs ch, GeomParams gp, const double* __restrict__ apos,
                                                  const int32_t* __restrict__ cidx, const int32_t* __restrict__ nbr,
                                                  const float* __restrict__ ubar, const float* __restrict__ w0, float s0,
                                                  const float* __restrict__ ab1, const float* __restrict__ ybar,
                                                  float* __restrict__ g, const int32_t* __restrict__ rev,
                                                  float* __restrict__ gT) {
  __shared__ __align__(16) float swt[32][kNB];  // W0 Bessel rows 4..11, transposed: [j][q], broadcast float4 reads
  __shared__ float4 stile[256 * 8];             // the block's ab1 rows (coalesced load), XOR-swizzled by row % 8
  for (int t = threadIdx.x; t < kNB * 32; t += blockDim.x) swt[t % 32][t / 32] = w0[4 * 32 + t];
  const int64_t e0 = (int64_t)blockIdx.x * blockDim.x;
  {
    const int rows = ch.n_e - e0 < 256 ? (int)(ch.n_e - e0) : 256;
    const float4* src = reinterpret_cast<const float4*>(ab1 + e0 * 32);
    for (int f = threadIdx.x; f < rows * 8; f += 256) {
      const int rr = f >> 3, c = f & 7;
      stile[rr * 8 + (c ^ (rr & 7))] = src[f];
    }
  }
  __syncthreads();
  const int row = threadIdx.x;
  const int64_t e = e0 + row;
  if (e >= ch.n_e) return;
  float zbar[kNB];
#pragma unroll
  for (int q = 0; q < kNB; ++q) zbar[q] = 0.f;
  {
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4) {
      const float4 v = stile[row * 8 + (c4 ^ (row & 7))];
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float4* wj = reinterpret_cast<const float4*>(&swt[4 * c4 + t][0]);
#pragma unroll
        for (int h = 0; h < kNB / 4; ++h) {
          const float4 w4 = wj[h];
          zbar[4 * h] = fmaf(vv[t], w4.x, zbar[4 * h]);
          zbar[4 * h + 1] = fmaf(vv[t], w4.y, zbar[4 * h + 1]);
          zbar[4 * h + 2] = fmaf(vv[t], w4.z, zbar[4 * h + 2]);
          zbar[4 * h + 3] = fmaf(vv[t], w4.w, zbar[4 * h + 3]);
        }
      }
    }
  }
  const int64_t ge = ch.e0 + e;
  float r[3], yb[9];
  edge_vec(apos, cidx[ge], nbr[ge], r);
  load_ybar(ybar, e, gp.dsh, yb);
  geom_bwd_tail(gp, r, ubar[e], yb, s0, zbar, g, ge, __ldg(rev + ge), gT);
}

// A/B switch: the producer of g scatters it to the reverse edge's slot (default) or the force gather
// gathers it through rev
bool force_scatter() {
  static const bool on = [] {
    const char* e = std::getenv("ALLEGRO_FORCE_SCATTER");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// ----------------------------------------------------------------- A12 force gather
// A/B variant without the producer-side scatter (ALLEGRO_FORCE_SCATTER=0): the reverse operand is
// gathered through rev (a dependent index -> 16-B gather round trip per edge); same sums, same order.
__global__ void k_force_warp_rev(int64_t n, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ rev,
                                 const float* __restrict__ g, const long long* __restrict__ acc,
                                 double* __restrict__ F, int* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (a >= n) return;
  double f[3] = {0, 0, 0};
  const int64_t r0 = row_ptr[a], r1 = row_ptr[a + 1];
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (int64_t base = r0; base < r1; base += 128) {
    int32_t rr[4];
    float4 a4[4], b4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t e = base + lane + 32 * k;
      rr[k] = e < r1 ? __ldg(rev + e) : -1;
      a4[k] = e < r1 ? __ldg(g4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) b4[k] = rr[k] >= 0 ? __ldg(g4 + rr[k]) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (base + lane + 32 * k < r1) {
        f[0] += (double)a4[k].x - (double)b4[k].x;
        f[1] += (double)a4[k].y - (double)b4[k].y;
        f[2] += (double)a4[k].z - (double)b4[k].z;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int d = 0; d < 3; ++d) f[d] += __shfl_xor_sync(0xffffffffu, f[d], o);
  if (lane == 0) {
    bool bad = false;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double v = f[d] + (acc != nullptr ? (double)acc[a * 3 + d] * (1.0 / kFixScale) : 0.0);
      F[a * 3 + d] = v;
      bad = bad || !isfinite(v);
    }
    if (bad) atomicOr(flags + 2, 1);
  }
}

// Warp per atom: the lanes stride the atom's CSR row and the fp64 partial sums are combined by a
// fixed butterfly, so the result is deterministic (and independent of the chunking).
// F_a = sum_{e in row a} (g_e - g_rev(e)) (+ the returned ghost forces).  g_rev(e) is read from gT[e]
// (= g[rev[e]], or 0 without a reverse edge), which the producer of g scattered, so both operands
// stream sequentially: no dependent index -> gather round trip.
__global__ void k_force_warp(int64_t n, const int32_t* __restrict__ row_ptr, const float* __restrict__ g,
                             const float* __restrict__ gT, const long long* __restrict__ acc, double* __restrict__ F,
                             int* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (a >= n) return;
  double f[3] = {0, 0, 0};
  const int64_t r0 = row_ptr[a], r1 = row_ptr[a + 1];
  const float4* g4 = reinterpret_cast<const float4*>(g);
  // Four edges per lane per round, all loads in flight before the first use (each lane adds its
  // edges in the order r0 + lane, + 32, + 64, ...); gT is packed [E][3] (12 B per edge)
  for (int64_t base = r0; base < r1; base += 128) {
    float4 a4[4];
    float3 b4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t e = base + lane + 32 * k;
      a4[k] = e < r1 ? __ldg(g4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
      b4[k] = e < r1 ? make_float3(__ldg(gT + 3 * e), __ldg(gT + 3 * e + 1), __ldg(gT + 3 * e + 2))
                     : make_float3(0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (base + lane + 32 * k < r1) {
        f[0] += (double)a4[k].x - (double)b4[k].x;
        f[1] += (double)a4[k].y - (double)b4[k].y;
        f[2] += (double)a4[k].z - (double)b4[k].z;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int d = 0; d < 3; ++d) f[d] += __shfl_xor_sync(0xffffffffu, f[d], o);
  if (lane == 0) {
    bool bad = false;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      // multi-GPU: -g of edges that point at images of a, returned by the reverse halo
      const double v = f[d] + (acc != nullptr ? (double)acc[a * 3 + d] * (1.0 / kFixScale) : 0.0);
      F[a * 3 + d] = v;
      bad = bad || !isfinite(v);
    }
    if (bad) atomicOr(flags + 2, 1);
  }
}

// ----------------------------------------------------------------- dispatch
template <int NL, int LMAX, int K>
void launch_tp(int mode, const TpArgs& t, cudaStream_t st, Profiler* prof, double flops, double bytes) {
  const unsigned blocks = (unsigned)((t.ch.n_c * 32 + 127) / 128);
  if (blocks == 0) return;
  {
    char tag[48];
    static const char* names[4] = {"tp_fwd", "tp_bwd", "gamma", "env_adj"};
    static const int kinds[4] = {PK_TP_FWD, PK_TP_BWD, PK_GAMMA, PK_ENV_ADJ};
    std::snprintf(tag, sizeof(tag), "%s layer=%d", names[mode], K);
    ProfScope ps_(prof, st, kinds[mode], flops, bytes, tag);
    if (mode == 0) k_tp_fwd<NL, LMAX, K><<<blocks, 128, 0, st>>>(t);
    else if (mode == 1) k_tp_bwd<NL, LMAX, K><<<blocks, 128, 0, st>>>(t);
    else if (mode == 2) k_tp_fwd<NL, LMAX, K, true><<<blocks, 128, 0, st>>>(t);
    else k_env_adj<NL, LMAX, K><<<blocks, 128, 0, st>>>(t);
  }
  ALG_LAUNCH_CHECK();
  if (mode >= 2 && std::getenv("ALLEGRO_SYNC_CHECK")) ALG_CUDA(cudaStreamSynchronize(st));
}

// Algorithmic work of the TP kernels per edge: forward = Gamma sum
// (DSH FMA) + TP (nnz FMA) per channel; backward = 2 nnz FMA + env adjoint.  Bytes:
// the per-edge operands the method reads/writes once (w, Y, V in; T out / T-bar, V,
// w, Y in; w-bar, Y-bar, V-bar out), fp32.
// mode 0: TP forward (Gamma + T), 1: TP backward, 2: Gamma only, 3: Gamma-bar row sums + environment
// adjoint (2 and 3: the fused path of tp_fused.cu)
void tp_dispatch(int NL, int LMAX, int K, int mode, const TpArgs& t, cudaStream_t st, Profiler* prof,
                 const LayerInfo& L) {
  const double E = (double)t.ch.n_e;
  const int dsh = (LMAX + 1) * (LMAX + 1);
  const double vin = K == 0 ? 0.0 : (double)L.A.dim_in * kC;
  const double nenv = LMAX + 1;
  const double flops = mode == 0   ? E * kC * 2.0 * (L.tp_nnz + dsh)
                       : mode == 1 ? E * kC * 2.0 * (2.0 * L.tp_nnz + 2 * dsh)
                       : mode == 2 ? E * kC * 2.0 * dsh
                                   : E * kC * (dsh + 4.0 * dsh);
  const double bytes = mode == 0   ? 4.0 * E * (L.nw + dsh + vin + (double)L.A.dim_T * kC)
                       : mode == 1 ? 4.0 * E * ((double)L.A.dim_T * kC + 2.0 * vin + 2.0 * L.nw + 2.0 * dsh)
                       : mode == 2 ? 4.0 * E * (nenv * kC + dsh) + 4.0 * t.ch.n_c * dsh * kC
                                   : 4.0 * E * (dsh * kC + 2.0 * nenv * kC + 3.0 * dsh);
#define ALG_TP(nl, lm, k) \
  if (NL == nl && LMAX == lm && K == k) return launch_tp<nl, lm, k>(mode, t, st, prof, flops, bytes);
  ALG_TP(2, 1, 0) ALG_TP(2, 1, 1)
  ALG_TP(2, 2, 0) ALG_TP(2, 2, 1)
  ALG_TP(3, 0, 0) ALG_TP(3, 0, 1) ALG_TP(3, 0, 2)
  ALG_TP(3, 1, 0) ALG_TP(3, 1, 1) ALG_TP(3, 1, 2)
  ALG_TP(3, 2, 0) ALG_TP(3, 2, 1) ALG_TP(3, 2, 2)
#undef ALG_TP
  throw CudaError("no TP kernel for this architecture");
}

// CUDA-core fp32 (parity reference mode) or tcgen05 3xTF32 (tensor cores)
__global__ void k_count_diff(const float* a, const float* b, int64_t n, unsigned long long* cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && __float_as_uint(a[i]) != __float_as_uint(b[i])) atomicAdd(cnt, 1ull);
}

void run_gemm(const Model& M, const GemmArgs& g_in, const Wt& w, cudaStream_t st, Profiler* prof) {
  GemmArgs g = g_in;
  g.single_pass = M.precision == ALLEGRO_PREC_TF32 ? 1 : 0;
  static const bool fuse_dot = [] {  // A/B switch for measurements (default: fused)
    const char* e = std::getenv("ALLEGRO_FUSE_ROWDOT");
    return !e || std::atoi(e) != 0;
  }();
  static const bool verify = std::getenv("ALLEGRO_VERIFY_GEMM") != nullptr;  // diagnostics: rerun and compare
  if (verify && tc_mode(M.precision) && g.epi != EPI_ACC && g.epi != EPI_R2 && !g.dotv && g.M > 0) {
    tc_gemm(g, w.tc, st, prof);
    float* tmp = nullptr;
    unsigned long long* cnt = nullptr;
    const size_t n = (size_t)g.M * g.N;
    ALG_CUDA(cudaMallocAsync(&tmp, n * sizeof(float), st));
    ALG_CUDA(cudaMallocAsync(&cnt, sizeof(unsigned long long), st));
    ALG_CUDA(cudaMemcpyAsync(tmp, g.C, n * sizeof(float), cudaMemcpyDeviceToDevice, st));
    ALG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
    tc_gemm(g, w.tc, st, prof);
    k_count_diff<<<ceil_div((int64_t)n, 256), 256, 0, st>>>(tmp, g.C, (int64_t)n, cnt);
    unsigned long long h = 0;
    ALG_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
    ALG_CUDA(cudaStreamSynchronize(st));
    if (h) std::fprintf(stderr, "[verify] gemm M=%lld N=%d K=%d epi=%d lda=%d A2=%d: %llu elements differ\n",
                        (long long)g.M, g.N, g.K, g.epi, g.lda, g.A2 ? 1 : 0, h);
    ALG_CUDA(cudaFreeAsync(tmp, st));
    ALG_CUDA(cudaFreeAsync(cnt, st));
    return;
  }
  // (measured: fused into EPI_ACC it is cost-neutral against the separate pass; into EPI_R2 it
  // was 2-3 ms slower with the STG epilogue and is 2 ms faster with the TMA-store epilogue)
  static const bool fuse_r2 = [] {  // A/B switch: the row-dot fused into the EPI_R2 epilogue too
    const char* e = std::getenv("ALLEGRO_FUSE_R2");
    return !e || std::atoi(e) != 0;
  }();
  if (tc_mode(M.precision) &&
      (!g.dotv || (g.dot_part && fuse_dot) || (fuse_dot && w.tc.n_tiles == 1 && (fuse_r2 || g.epi != EPI_R2)))) {
    tc_gemm(g, w.tc, st, prof);  // the row-dot (if any) is fused into the epilogue
    return;
  }
  GemmArgs g0 = g;
  g0.dotv = nullptr;
  if (tc_mode(M.precision)) tc_gemm(g0, w.tc, st, prof);
  else gemm(g0, st, prof);
  // fp32 reference mode, or an output split over N-tiles (a fused dot would need an
  // order-dependent cross-CTA sum): a separate row-dot over the finished output
  if (g.dotv && g.M > 0) {
    if (g.N != kD) throw CudaError("row-dot over N != 128");
    {
      ProfScope ps_(prof, st, PK_ROWDOT, 2.0 * 128 * g.M, (double)g.M * 1024);
      k_rowdot<<<ceil_div(g.M * 32, 256), 256, 0, st>>>(g.M, g.dotv, g.C, g.dot_coef, g.dot_inv_u, g.dot_out);
    }
    ALG_LAUNCH_CHECK();
  }
}

size_t floats_per_edge(const Model& M) {
  const int dsh = (M.lmax + 1) * (M.lmax + 1);
  size_t f = 32 + 64 + 128 + 1 + dsh + 2 * 128;  // a1, a2, m, u, Y, x (two buffers)
  size_t tmax = 0, vmax = 0, nwmax = 0, nsmax = 0;
  for (int k = 0; k < M.n_layers; ++k) {
    const LayerInfo& L = M.L[k];
    f += L.nw + 128;
    if (k >= 1) f += (size_t)L.A.dim_in * kC;
    tmax = std::max(tmax, (size_t)L.A.dim_T * kC);
    vmax = std::max(vmax, (size_t)L.A.dim_in * kC);
    nwmax = std::max(nwmax, (size_t)L.nw);
    nsmax = std::max(nsmax, (size_t)L.A.n_s * kC);
  }
  f += tmax + 2 * 128 + nsmax + 2 * vmax + nwmax + dsh + 1 + 64 + 32 + 1;
  f += dsh * kC + 4;  // gp (fused backward), row-dot partials
  return f;
}

void reserve_ws(allegro_ctx* c, size_t e_cap, size_t a_cap) {
  Workspace& w = c->ws;
  const Model& M = c->model;
  const int dsh = (M.lmax + 1) * (M.lmax + 1);
  w.a1.reserve(e_cap * 32);
  w.a2.reserve(e_cap * 64);
  w.m.reserve(e_cap * 128);
  w.u.reserve(e_cap);
  w.Y.reserve(e_cap * dsh);
  w.xa.reserve(e_cap * 128);
  w.xb.reserve(e_cap * 128);
  size_t tmax = 0, vmax = 0, nwmax = 0, nsmax = 0;
  for (int k = 0; k < M.n_layers; ++k) {
    const LayerInfo& L = M.L[k];
    w.w[k].reserve(e_cap * L.nw);
    w.h[k].reserve(e_cap * 128);
    if (k >= 1) w.V[k].reserve(e_cap * L.A.dim_in * kC);
    w.G[k].reserve(a_cap * dsh * kC);
    tmax = std::max(tmax, (size_t)L.A.dim_T * kC);
    vmax = std::max(vmax, (size_t)L.A.dim_in * kC);
    nwmax = std::max(nwmax, (size_t)L.nw);
    nsmax = std::max(nsmax, (size_t)L.A.n_s * kC);
  }
  w.T.reserve(e_cap * tmax);
  w.xbar_a.reserve(e_cap * 128);
  w.xbar_b.reserve(e_cap * 128);
  w.sbar.reserve(e_cap * nsmax);
  w.vbar_a.reserve(e_cap * vmax);
  w.vbar_b.reserve(e_cap * vmax);
  w.wbar.reserve(e_cap * nwmax);
  w.ybar.reserve(e_cap * dsh);
  w.ubar.reserve(e_cap);
  w.ab2.reserve(e_cap * 64);
  w.ab1.reserve(e_cap * 32);
  w.ebar.reserve(e_cap);
  w.gp.reserve(e_cap * dsh * kC);
  w.dotp.reserve(e_cap * 4);  // row-dot partials of a contraction split over N-tiles
  w.e_cap = e_cap;
  w.a_cap = a_cap;
}

void run_chunk(allegro_ctx* c, const ChunkPtrs& ch) {
  const Model& M = c->model;
  Workspace& w = c->ws;
  cudaStream_t st = c->stream;
  const int64_t E = ch.n_e;
  const int64_t ecap = (int64_t)w.e_cap;
  const int dsh = (M.lmax + 1) * (M.lmax + 1);
  const float inv_sqrt_nbar = (float)(1.0 / std::sqrt(M.nbar));
  GeomParams gp;
  gp.rc = (float)M.r_max;
  gp.inv_rc = (float)(1.0 / M.r_max);
  for (int q = 0; q < kNB; ++q) gp.freq[q] = M.w.bessel[q];
  gp.lmax = M.lmax;
  gp.dsh = dsh;
  const char* f2_env = std::getenv("ALLEGRO_FUSED_2B");  // A/B switch: geometry + two-body MLP in one kernel
  const int f2_mask = (f2_env ? std::atoi(f2_env) : 3) * (M.precision == ALLEGRO_PREC_3XTF32 ? 1 : 0);
  const bool fused_2b = f2_mask & 1, fused_2b_bwd = (f2_mask >> 1) & 1;  // bit 0: forward, bit 1: reverse
  if (E > 0 && !fused_2b) {
    {
      ProfScope ps_(&c->prof, st, PK_GEOM, 0, (double)E * (8 + 128 + 4 * dsh + 4));
      k_geom<<<ceil_div(E, 256), 256, 0, st>>>(ch, gp, c->apos.p, c->cidx.p, c->nbr.p, c->aspec.p, c->species.p,
                                             M.w.tb_w0.f, 1.f / std::sqrt(12.f), w.a1.p, w.Y.p, w.u.p);
    }
    ALG_LAUNCH_CHECK();
  }
  const Wt* last_w = nullptr;
  auto G = [&](const float* A, int lda, const Wt& Wm, int N, int K, float* C, float s, int epi) {
    last_w = &Wm;
    const float* W = Wm.f;
    GemmArgs g;
    g.M = E;
    g.N = N;
    g.K = K;
    g.A = A;
    g.lda = lda;
    g.W = W;
    g.C = C;
    g.s = s;
    g.epi = epi;
    return g;
  };
  // ---- two-body MLP (E4, E5) ----
  TbIO tbio;
  {
    TbIO& io = tbio;
    io.ch = ch;
    io.gp = gp;
    io.apos = c->apos.p;
    io.cidx = c->cidx.p;
    io.nbr = c->nbr.p;
    io.aspec = c->aspec.p;
    io.species = c->species.p;
    io.w0 = M.w.tb_w0.f;
    io.w1 = &M.w.tb_w1;
    io.w2 = &M.w.tb_w2;
    io.u = w.u.p;
    io.Y = w.Y.p;
    io.x0 = w.m.p;  // x^0 = u m in its own buffer (kept for the reverse's row-dot; m is not stored)
    io.a1 = fused_2b_bwd ? nullptr : w.a1.p;  // the fused reverse recomputes a1, a2
    io.a2 = fused_2b_bwd ? nullptr : w.a2.p;
    io.m = nullptr;
  }
  if (fused_2b) {
    tb_fwd(tbio, st, &c->prof);
  } else {
    // only the pre-activations a1, a2 are stored (the reverse pass needs them); the next
    // contraction applies SiLU to its operand on load instead of reading a stored h = SiLU(a)
    // (a1 = z W0 / sqrt 12 was formed by k_geom)
    GemmArgs g = G(w.a1.p, 32, M.w.tb_w1, 64, 32, w.a2.p, kCSilu / std::sqrt(32.f), EPI_STORE);
    g.silu_a = 1;
    run_gemm(M, g, *last_w, st, &c->prof);
    g = G(w.a2.p, 64, M.w.tb_w2, 128, 64, w.m.p, kCSilu / std::sqrt(64.f), EPI_UMUL_SAVE);
    g.silu_a = 1;
    g.aux = nullptr;
    g.u = w.u.p;
    run_gemm(M, g, *last_w, st, &c->prof);
  }
  float* x = w.m.p;  // x^0 (never overwritten: the latent updates alternate between xa and xb)
  float* xn = w.xa.p;
  TpArgs tp{};
  tp.ch = ch;
  tp.row_ptr = c->row_ptr.p;
  tp.Y = w.Y.p;
  tp.T = w.T.p;
  tp.e_cap = ecap;
  tp.inv_sqrt_nbar = inv_sqrt_nbar;
  const unsigned warp_blocks = (unsigned)((ch.n_c * 32 + 127) / 128);
  const char* fl_env = std::getenv("ALLEGRO_FUSED_LAST");  // A/B switch: the last layer in one kernel
  const bool fused_last = !fl_env || std::atoi(fl_env) != 0;
  // ---- layers (E6) ----
  for (int k = 0; k < M.n_layers; ++k) {
    const LayerInfo& L = M.L[k];
    {
      GemmArgs g = G(x, 128, M.w.env[k], L.nw, 128, w.w[k].p, 1.f / std::sqrt(128.f), EPI_STORE);
      run_gemm(M, g, *last_w, st, &c->prof);
    }
    tp.w = w.w[k].p;
    tp.V = k >= 1 ? w.V[k].p : nullptr;
    tp.G = w.G[k].p;
    const char* fz_env = std::getenv("ALLEGRO_FUSED_TP");  // A/B switch (default: fused where built)
    const int fz_mask = fz_env ? std::atoi(fz_env) : -1;  // bit k: fuse layer k (0: none)
    const bool fused = ((fz_mask >> k) & 1) && M.precision == ALLEGRO_PREC_3XTF32 &&
                       tpl_fwd_supported(M.n_layers, M.lmax, k);
    if (fused) {
      tp_dispatch(M.n_layers, M.lmax, k, 2, tp, st, &c->prof, L);  // Gamma_i
      TplIO io;
      io.ch = ch;
      io.cidx = c->cidx.p;
      io.G = w.G[k].p;
      io.Y = w.Y.p;
      io.w = w.w[k].p;
      for (int i = 0; i < L.A.in.n; ++i) io.vin[i] = k >= 1 ? w.V[k].p + (int64_t)L.v_base[i] * ecap : nullptr;
      for (int o = 0; o < L.A.out.n; ++o) {
        io.vout[o] = w.V[k + 1].p + (int64_t)M.L[k + 1].v_base[o] * ecap;
        io.wimg[o] = M.w.lin[k][o].tc.dev;
        io.wbytes[o] = M.w.lin[k][o].tc.tile_bytes;
      }
      io.s = w.T.p;  // T_0e = s, [E][n_s C] (the latent update's second operand)
      io.tp_fma_per_edge = (double)L.tp_nnz * kC;
      tpl_fwd(M.n_layers, M.lmax, k, io, st, &c->prof);
    } else if (!(k == M.n_layers - 1 && fused_last)) {  // (the fused last layer forms Gamma and s itself)
      tp_dispatch(M.n_layers, M.lmax, k, 0, tp, st, &c->prof, L);
    }
    if (k < M.n_layers - 1 && !fused) {
      for (int o = 0; o < L.A.out.n; ++o) {
        const int dim = ir_dim(L.A.out.v[o]);
        GemmArgs g = G(w.T.p + (int64_t)L.t_base[o] * ecap, L.A.n_to[o] * kC, M.w.lin[k][o], kC, L.A.n_to[o] * kC,
                       w.V[k + 1].p + (int64_t)M.L[k + 1].v_base[o] * ecap, 1.f / std::sqrt((float)(kC * L.A.n_to[o])),
                       EPI_STORE);
        g.M = E * dim;
        run_gemm(M, g, *last_w, st, &c->prof);
      }
    }
    if (k == M.n_layers - 1) break;  // the last latent update is folded into the read-out (k_energy_last)
    GemmArgs g = G(x, 128, M.w.lat[k], 128, L.fan_lat, xn, 1.f / std::sqrt((float)L.fan_lat), EPI_RESID);
    g.K1 = 128;
    g.A2 = w.T.p;  // T_0e = the scalars s, [E][n_s C] in (q, c) order
    g.lda2 = L.A.n_s * kC;
    g.aux = w.h[k].p;
    g.X = x;
    g.u = w.u.p;
    g.alpha = kResA;
    g.beta = kResB;
    run_gemm(M, g, *last_w, st, &c->prof);
    float* done = x;
    x = xn;
    xn = done == w.m.p ? w.xb.p : done;
  }
  // ---- energies (E7, E8) and the rank-one reverse mode of the last layer ----
  float* xb = w.xbar_a.p;
  float* xbn = w.xbar_b.p;
  const LayerInfo& LL = M.L[M.n_layers - 1];
  const int nsc_last = LL.A.n_s * kC;
  if (nsc_last > 3 * 32) throw CudaError("k_energy_last holds at most 96 last-layer scalar channels (lmax <= 2)");
  const float sf_last = kResB / std::sqrt((float)LL.fan_lat);
  if (warp_blocks && !fused_last) {
    {
      ProfScope ps_(&c->prof, st, PK_ENERGY, 6.0 * 128 * E, (double)E * (512 + 8.0 * nsc_last + 16));
      k_energy_last<<<warp_blocks, 128, 0, st>>>(ch, c->row_ptr.p, c->species.p, x, w.T.p, nsc_last, w.u.p, M.w.wout,
                                                 M.w.q_last, c->e_atom.p, w.ubar.p, w.sbar.p, w.ebar.p, M.sigma[0],
                                                 M.sigma[1], M.mu[0], M.mu[1], inv_sqrt_nbar, kResA, sf_last);
    }
    ALG_LAUNCH_CHECK();
  }
  // ---- reverse mode (E9) ----
  ALG_CUDA(cudaMemsetAsync(w.ybar.p, 0, sizeof(float) * E * dsh, st));
  float* vb = w.vbar_a.p;   // V-bar^{k+1} (input to layer k)
  float* vbn = w.vbar_b.p;  // V-bar^k (output of layer k)
  for (int k = M.n_layers - 1; k >= 0; --k) {
    const LayerInfo& L = M.L[k];
    const bool last = k == M.n_layers - 1;
    const float sl = 1.f / std::sqrt((float)L.fan_lat);
    // merged x-bar contraction (3xTF32): the latent transpose and the env transpose of this layer
    // accumulate in ONE contraction over K = 128 + nw (A = [b u x-bar^{k+1} / sqrt(fan) | w-bar / sqrt(D)],
    // rows scaled before the TF32 split), so the partial x-bar^k never round-trips HBM
    const char* mx_env = std::getenv("ALLEGRO_MERGE_XBAR");
    const bool merge_x = !last && M.precision == ALLEGRO_PREC_3XTF32 && (!mx_env || std::atoi(mx_env) != 0);
    if (!last) {
      GemmArgs g;
      if (!merge_x) {
        g = G(xb, 128, M.w.latT_x[k], 128, 128, xbn, sl, EPI_URESID);
        g.X = xb;
        g.u = w.u.p;
        g.alpha = kResA;
        g.beta = kResB;
        run_gemm(M, g, *last_w, st, &c->prof);
      }
      g = G(xb, 128, M.w.latT_s[k], L.A.n_s * kC, 128, w.sbar.p, sl, EPI_USCALE);
      g.u = w.u.p;
      g.beta = kResB;
      run_gemm(M, g, *last_w, st, &c->prof);
    }
    tp.w = w.w[k].p;
    tp.V = k >= 1 ? w.V[k].p : nullptr;
    tp.G = w.G[k].p;
    tp.wbar = w.wbar.p;
    tp.ybar = w.ybar.p;
    tp.Vb = vbn;
    const char* fb_env = std::getenv("ALLEGRO_FUSED_TP_BWD");  // A/B switch (bit k: fuse layer k)
    const int fb_mask = fb_env ? std::atoi(fb_env) : -1;
    const bool fused_bwd = ((fb_mask >> k) & 1) && M.precision == ALLEGRO_PREC_3XTF32 &&
                           tpl_fwd_supported(M.n_layers, M.lmax, k);
    if (fused_bwd) {
      TpbIO io;
      io.ch = ch;
      io.cidx = c->cidx.p;
      io.G = w.G[k].p;
      io.Y = w.Y.p;
      io.w = w.w[k].p;
      for (int i = 0; i < L.A.in.n; ++i) {
        io.vin[i] = k >= 1 ? w.V[k].p + (int64_t)L.v_base[i] * ecap : nullptr;
        io.vbar_out[i] = k >= 1 ? vbn + (int64_t)L.v_base[i] * ecap : nullptr;
      }
      for (int o = 0; o < L.A.out.n; ++o) {
        io.vbar_in[o] = vb + (int64_t)M.L[k + 1].v_base[o] * ecap;
        io.wimg[o] = M.w.linT[k][o].tc.dev;
        io.wbytes[o] = M.w.linT[k][o].tc.tile_bytes;
      }
      io.sbar = w.sbar.p;
      io.wbar = w.wbar.p;
      io.ybar = w.ybar.p;
      io.gp = w.gp.p;
      io.tp_fma_per_edge = (double)L.tp_nnz * kC;
      tpl_bwd(M.n_layers, M.lmax, k, io, st, &c->prof);
      tp.gp = w.gp.p;
      tp_dispatch(M.n_layers, M.lmax, k, 3, tp, st, &c->prof, L);  // Gamma-bar + environment adjoint
    } else if (k == M.n_layers - 1 && fused_last) {
      LastArgs la;
      la.t = tp;
      la.species = c->species.p;
      la.x = x;
      la.u = w.u.p;
      la.wout = M.w.wout;
      la.q = M.w.q_last;
      la.e_atom = c->e_atom.p;
      la.ubar = w.ubar.p;
      la.ebar = w.ebar.p;
      la.s0 = M.sigma[0], la.s1 = M.sigma[1], la.mu0 = M.mu[0], la.mu1 = M.mu[1];
      la.ra = kResA;
      la.sf = sf_last;
      last_dispatch(M.n_layers, M.lmax, la, st, &c->prof, L);
    } else if (k == M.n_layers - 1) {
      tp.Tb[0] = w.sbar.p;  // last layer: out = {0e}, T-bar = s-bar
    } else {
      for (int o = 0; o < L.A.out.n; ++o) {
        const int dim = ir_dim(L.A.out.v[o]);
        float* dst = w.T.p + (int64_t)L.t_base[o] * ecap;
        GemmArgs g = G(vb + (int64_t)M.L[k + 1].v_base[o] * ecap, kC, M.w.linT[k][o], L.A.n_to[o] * kC, kC, dst,
                       1.f / std::sqrt((float)(kC * L.A.n_to[o])), EPI_STORE);
        g.M = E * dim;
        if (L.A.out.v[o].l == 0 && L.A.out.v[o].p == 1) {
          g.epi = EPI_ADDX;
          g.X = w.sbar.p;
        }
        run_gemm(M, g, *last_w, st, &c->prof);
        tp.Tb[o] = dst;
      }
    }
    if (!fused_bwd && !(last && fused_last)) tp_dispatch(M.n_layers, M.lmax, k, 1, tp, st, &c->prof, L);
    if (merge_x) {
      GemmArgs g = G(xb, 128, M.w.latenvT[k], 128, 128 + L.nw, xbn, 1.f, EPI_ACCX);
      g.K1 = 128;
      g.A2 = w.wbar.p;
      g.lda2 = L.nw;
      g.arow_u = w.u.p;
      g.arow_c1 = kResB * sl;
      g.arow_c2 = 1.f / std::sqrt(128.f);
      g.X = xb;
      g.alpha = kResA;
      g.dotv = k >= 1 ? w.h[k - 1].p : w.m.p;  // k = 0: x^0, divided by u per row
      g.dot_inv_u = k >= 1 ? nullptr : w.u.p;
      g.dot_coef = k >= 1 ? kResB : 1.f;
      g.dot_out = w.ubar.p;
      g.dot_part = w.dotp.p;
      run_gemm(M, g, *last_w, st, &c->prof);
    } else {
      GemmArgs g = G(w.wbar.p, L.nw, M.w.envT[k], 128, L.nw, xbn, 1.f / std::sqrt(128.f), last ? EPI_R2 : EPI_ACC);
      if (last) {  // xbar^{L-1} = env^T part + Ebar (a w_out + u (b/sqrt(fan)) q_x)
        g.rs2 = w.ebar.p;
        g.u = w.u.p;
        g.vec1 = M.w.r2_vec1;
        g.vec2 = M.w.r2_vec2;
      }
      // xbar^k is complete here: fuse the u-gradient of the update that produced x^k,
      // ubar += (1/sqrt5) <xbar^k, h^{k-1}> (latent resnet) or <xbar^0, m> (two-body x^0 = u m)
      g.dotv = k >= 1 ? w.h[k - 1].p : w.m.p;  // k = 0: x^0, divided by u per row
      g.dot_inv_u = k >= 1 ? nullptr : w.u.p;
      g.dot_coef = k >= 1 ? kResB : 1.f;
      g.dot_out = w.ubar.p;
      run_gemm(M, g, *last_w, st, &c->prof);
    }
    std::swap(xb, xbn);
    std::swap(vb, vbn);
  }
  // ---- two-body reverse (its u-gradient row-dot ran in layer 0's env^T epilogue) ----
  if (fused_2b_bwd) {
    TbbIO bo;
    bo.w2t = &M.w.tb_w2T;
    bo.w1t = &M.w.tb_w1T;
    bo.xbar = xb;
    bo.ubar = w.ubar.p;
    bo.ybar = w.ybar.p;
    bo.g = c->g.p;
    bo.rev = c->rev.p;
    bo.gT = force_scatter() ? c->gT.p : nullptr;
    tb_bwd(tbio, bo, st, &c->prof);
    return;
  }
  {
    GemmArgs g = G(xb, 128, M.w.tb_w2T, 64, 128, w.ab2.p, kCSilu / std::sqrt(64.f), EPI_DSILU);
    g.X = w.a2.p;
    g.u = w.u.p;
    run_gemm(M, g, *last_w, st, &c->prof);
    g = G(w.ab2.p, 64, M.w.tb_w1T, 32, 64, w.ab1.p, kCSilu / std::sqrt(32.f), EPI_DSILU);
    g.X = w.a1.p;
    run_gemm(M, g, *last_w, st, &c->prof);
    // (ab1 W0^T is formed inside k_geom_bwd)
  }
  if (E > 0) {
    {
      ProfScope ps_(&c->prof, st, PK_GEOM_BWD, 0, (double)E * (8 + 4 + 128 + 4 * dsh + 16));
      k_geom_bwd<<<ceil_div(E, 256), 256, 0, st>>>(ch, gp, c->apos.p, c->cidx.p, c->nbr.p, w.ubar.p, M.w.tb_w0.f,
                                                 1.f / std::sqrt(12.f), w.ab1.p, w.ybar.p, c->g.p, c->rev.p,
                                                 force_scatter() ? c->gT.p : nullptr);
    }
    ALG_LAUNCH_CHECK();
  }
}

}  // namespace

void compute_forces(allegro_ctx* c, bool defer_e) {
  cudaStream_t st = c->stream;
  const int64_t n = c->n;
  const int64_t E = c->n_edges;
  c->e_atom.reserve(n + 1);
  c->frc.reserve(3 * n + 3);
  // chunk plan: complete rows, at most e_cap edges per chunk
  const size_t fpe = floats_per_edge(c->model);
  size_t e_cap = std::max<size_t>(4096, c->ws_budget_bytes / (fpe * sizeof(float)));
  e_cap = std::min<size_t>(e_cap, (size_t)std::max<int64_t>(E, 4096));
  std::vector<ChunkPtrs> chunks;
  int64_t a = 0;
  size_t a_cap = 1;
  if ((size_t)E <= e_cap) {  // one chunk: no need for the row offsets on the host
    chunks.push_back(ChunkPtrs{0, n, 0, E});
    a_cap = std::max<size_t>(1, n);
    a = n;
  } else {
    c->h_row_ptr.resize(n + 1);
    ALG_CUDA(cudaMemcpyAsync(c->h_row_ptr.data(), c->row_ptr.p, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost,
                             st));
    ALG_CUDA(cudaStreamSynchronize(st));
  }
  while (a < n) {
    int64_t b = a;
    while (b < n && (b == a || (size_t)(c->h_row_ptr[b + 1] - c->h_row_ptr[a]) <= e_cap)) ++b;
    ChunkPtrs ch{a, b - a, c->h_row_ptr[a], (int64_t)c->h_row_ptr[b] - c->h_row_ptr[a]};
    if ((size_t)ch.n_e > e_cap) e_cap = ch.n_e;  // a single row larger than the cap
    a_cap = std::max<size_t>(a_cap, ch.n_c);
    chunks.push_back(ch);
    a = b;
  }
  reserve_ws(c, e_cap, a_cap);
  c->chunk_a0.clear();
  for (const ChunkPtrs& ch : chunks) c->chunk_a0.push_back(ch.a0);
  for (const ChunkPtrs& ch : chunks) run_chunk(c, ch);
  ALG_CUDA(cudaMemsetAsync(c->flags.p + 2, 0, sizeof(int), st));
  if (c->dom.multi) ghost_force_return(c);
  if (n > 0) {
    {
      // algorithmic: g_e, g_rev (12 B each); + rev (4 B) on the gather variant
      ProfScope ps_(&c->prof, st, PK_FORCE, 0, 24.0 * n + 8.0 * n + (force_scatter() ? 24.0 : 28.0) * E);
      if (force_scatter())
        k_force_warp<<<ceil_div(n * 32, 256), 256, 0, st>>>(n, c->row_ptr.p, c->g.p, c->gT.p,
                                                          c->dom.multi ? c->dom.acc.p : nullptr, c->frc.p, c->flags.p);
      else
        k_force_warp_rev<<<ceil_div(n * 32, 256), 256, 0, st>>>(n, c->row_ptr.p, c->rev.p, c->g.p,
                                                              c->dom.multi ? c->dom.acc.p : nullptr, c->frc.p,
                                                              c->flags.p);
    }
    ALG_LAUNCH_CHECK();
  }
  if (defer_e) {  // md_run: fetched (multi-GPU: allreduced) together with the finite flag (all_finite)
    sum_e_atom_async(c);
    c->e_pot_pending = true;
  } else {
    c->e_pot = allreduce_sum(c, sum_e_atom(c));
  }
}

}  // namespace allegro
