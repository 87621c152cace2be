// gemm.cu -- CUDA-core fp32 tiled GEMM with fused epilogues (ALLEGRO_PREC_FP32, the
// parity mode).  BM = 128 rows x BN columns per CTA, BK = 16, 256 threads, each
// thread owns 8 rows x BN/16 columns (rows ty + 16 i, columns tx + 16 j: broadcast
// A reads, conflict-free W reads from shared memory); the next K tile is prefetched
// into registers while the current one is multiplied.
#include "gemm.cuh"

namespace allegro {
namespace {

constexpr int BM = 128, BK = 16, NT = 256;

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

template <int BN>
__global__ void __launch_bounds__(NT) k_gemm(GemmArgs g) {
  constexpr int TN = BN / 16;
  __shared__ float As[2][BK][BM + 4];
  __shared__ float Ws[2][BK][BN];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t row0 = (int64_t)blockIdx.x * BM;
  const int col0 = blockIdx.y * BN;
  // A tile loader: thread -> (row tid/2, k offset (tid%2)*8), two float4
  const int la_r = tid >> 1, la_k = (tid & 1) * 8;
  const int64_t a_row = row0 + la_r;
  const bool a_ok = a_row < g.M;
  float4 ra[2];
  float rw[(BK * BN + NT - 1) / NT];
  auto load_tile = [&](int k0) {
    const float* src;
    int kk = k0 + la_k;
    if (g.A2 != nullptr && kk >= g.K1) src = g.A2 + a_row * g.lda2 + (kk - g.K1);
    else src = g.A + a_row * g.lda + kk;
    if (a_ok) {
      ra[0] = *reinterpret_cast<const float4*>(src);
      ra[1] = *reinterpret_cast<const float4*>(src + 4);
      if (g.silu_a) {
#pragma unroll
        for (int q = 0; q < 2; ++q) ra[q] = make_float4(silu(ra[q].x), silu(ra[q].y), silu(ra[q].z), silu(ra[q].w));
      }
    } else {
      ra[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      ra[1] = ra[0];
    }
#pragma unroll
    for (int q = 0; q < (BK * BN + NT - 1) / NT; ++q) {
      const int idx = tid + q * NT;
      if (idx < BK * BN) rw[q] = g.W[(int64_t)(k0 + idx / BN) * g.N + col0 + (idx % BN)];
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) As[buf][la_k + q][la_r] = reinterpret_cast<const float*>(&ra[0])[q];
#pragma unroll
    for (int q = 0; q < 4; ++q) As[buf][la_k + 4 + q][la_r] = reinterpret_cast<const float*>(&ra[1])[q];
#pragma unroll
    for (int q = 0; q < (BK * BN + NT - 1) / NT; ++q) {
      const int idx = tid + q * NT;
      if (idx < BK * BN) Ws[buf][idx / BN][idx % BN] = rw[q];
    }
  };
  float acc[8][TN];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
  const int nk = g.K / BK;
  load_tile(0);
  store_tile(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load_tile((kt + 1) * BK);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[8], b[TN];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[buf][k][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Ws[buf][k][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (kt + 1 < nk) store_tile(buf ^ 1);
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = row0 + ty + 16 * i;
    if (r >= g.M) continue;
    const float ur = (g.u != nullptr) ? g.u[r] : 1.f;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t o = r * g.N + col0 + tx + 16 * j;
      const float p = g.s * acc[i][j];
      switch (g.epi) {
        case EPI_STORE: g.C[o] = p; break;
        case EPI_SILU: g.aux[o] = p; g.C[o] = silu(p); break;
        case EPI_UMUL_SAVE:
          if (g.aux) g.aux[o] = p;  // (the model passes none: x^0 = u m keeps m recoverable)
          g.C[o] = ur * p;
          break;
        case EPI_RESID: g.aux[o] = p; g.C[o] = g.alpha * g.X[o] + g.beta * ur * p; break;
        case EPI_URESID: g.C[o] = g.alpha * g.X[o] + g.beta * ur * p; break;
        case EPI_USCALE: g.C[o] = g.beta * ur * p; break;
        case EPI_ACC: g.C[o] += p; break;
        case EPI_ADDX: g.C[o] = p + g.X[o]; break;
        case EPI_DSILU: g.C[o] = ur * p * dsilu(g.X[o]); break;
        case EPI_R2: {
          const int col = col0 + tx + 16 * j;
          g.C[o] = p + g.rs2[r] * (g.vec1[col] + ur * g.vec2[col]);
          break;
        }
        default: break;
      }
    }
  }
}

}  // namespace

void gemm(const GemmArgs& g, cudaStream_t st, Profiler* prof) {
  if (g.M == 0) return;
  // algorithmic work: 2 M N K flops; A, W read, C written (+ aux written, X read)
  const double mn = (double)g.M * g.N;
  const int n_io = 1 + (g.aux != nullptr) + (g.X != nullptr) + (g.epi == EPI_ACC);
  ProfScope ps(prof, st, PK_GEMM, 2.0 * mn * g.K, 4.0 * ((double)g.M * g.K + (double)g.K * g.N + mn * n_io));
  if (g.K % BK != 0 || g.N % 16 != 0 || (g.A2 && g.K1 % BK != 0))
    throw CudaError("gemm: unsupported shape N=" + std::to_string(g.N) + " K=" + std::to_string(g.K));
  const unsigned gx = (unsigned)((g.M + BM - 1) / BM);
  if (g.N % 128 == 0) {
    k_gemm<128><<<dim3(gx, g.N / 128), NT, 0, st>>>(g);
  } else if (g.N % 96 == 0) {
    k_gemm<96><<<dim3(gx, g.N / 96), NT, 0, st>>>(g);
  } else if (g.N % 64 == 0) {
    k_gemm<64><<<dim3(gx, g.N / 64), NT, 0, st>>>(g);
  } else if (g.N % 32 == 0) {
    k_gemm<32><<<dim3(gx, g.N / 32), NT, 0, st>>>(g);
  } else {
    k_gemm<16><<<dim3(gx, g.N / 16), NT, 0, st>>>(g);
  }
  ALG_LAUNCH_CHECK();
}

}  // namespace allegro
