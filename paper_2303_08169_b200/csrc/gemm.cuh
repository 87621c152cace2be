// gemm.cuh -- per-edge dense contractions C[M x N] = epi(A[M x K] W[K x N]).
// The only dense GEMMs of the method: the
// two-body MLP, env-embed, TP-linear and latent linears and their input-gradient
// (W^T) counterparts.  M = edges (or edges x irrep dim), K, N <= 224.
#pragma once
#include "common.cuh"
#include "prof.cuh"

namespace allegro {

enum GemmEpi : int {
  EPI_STORE = 0,      // C = s acc
  EPI_SILU = 1,       // aux = s acc; C = SiLU(aux)
  EPI_UMUL_SAVE = 2,  // aux = s acc; C = u[r] aux
  EPI_RESID = 3,      // aux = s acc; C = alpha X + beta u[r] aux
  EPI_URESID = 4,     // C = alpha X + beta u[r] s acc
  EPI_USCALE = 5,     // C = beta u[r] s acc
  EPI_ACC = 6,        // C += s acc
  EPI_ADDX = 7,       // C = s acc + X
  EPI_DSILU = 8,      // C = (u ? u[r] : 1) s acc SiLU'(X)
  EPI_R2 = 9,         // C = s acc + rs2[r] (vec1[col] + u[r] vec2[col])   (rank-2 affine term)
  EPI_ACCX = 10,      // C = s acc + alpha X   (the latent-transpose + env-transpose contraction, one K)
};

struct GemmArgs {
  int64_t M = 0;
  int N = 0, K = 0;
  const float* A = nullptr;  // row-major, columns [0, K1)
  int lda = 0;
  const float* A2 = nullptr;  // row-major, columns [K1, K) (nullptr: A has all K)
  int lda2 = 0;
  int K1 = 0;
  const float* W = nullptr;  // [K][N] row-major
  float* C = nullptr;        // [M][N]
  float* aux = nullptr;      // [M][N]
  const float* X = nullptr;  // [M][N]
  const float* u = nullptr;  // [M]
  const float* rs2 = nullptr;   // [M]   (EPI_R2)
  const float* vec1 = nullptr;  // [N]   (EPI_R2)
  const float* vec2 = nullptr;  // [N]   (EPI_R2)
  // optional fused row-dot (the u-gradient of a residual update): dot_out[r] += dot_coef <C[r], dotv[r]>
  // over the N output columns (3xTF32 path: in the epilogue; fp32 path: a separate kernel)
  const float* dotv = nullptr;  // [M][N]
  float* dot_out = nullptr;     // [M]
  float dot_coef = 0.f;
  const float* dot_inv_u = nullptr;  // [M] if set: the row-dot of row r is divided by u[r] (0 where u = 0)
  float s = 1.f, alpha = 0.f, beta = 0.f;
  int epi = EPI_STORE;
  int silu_a = 0;  // A holds pre-activations: the contraction multiplies SiLU(A) (applied on load)
  int single_pass = 0;  // tcgen05 path: one TF32 MMA (a_hi w_hi) instead of 3xTF32 (ALLEGRO_PREC_TF32)
  // tcgen05 path: A rows scaled before the hi/lo split -- columns [0, K1) by arow_c1 * arow_u[r],
  // columns [K1, K) by arow_c2 (two contractions of different scale in one accumulator)
  const float* arow_u = nullptr;
  float arow_c1 = 1.f, arow_c2 = 1.f;
  // row-dot of an output split over N-tiles: each tile writes its partial to dot_part[r][tile] and
  // the host adds dot_out[r] += dot_coef sum_tile dot_part[r][tile] (fixed order) after the launch
  float* dot_part = nullptr;
};

void gemm(const GemmArgs& g, cudaStream_t st, Profiler* prof);

}  // namespace allegro
