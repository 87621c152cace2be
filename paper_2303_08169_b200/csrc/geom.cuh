// geom.cuh -- per-edge geometry of the model (E1-E3 of SURVEY.md §8(c)): the edge vector (canonical
// fp64 difference, then fp32), the component-normalised real spherical harmonics, and the
// parameters of the envelope / Bessel basis.  Shared by model.cu and twobody.cu.
#pragma once
#include <cstdint>

#include "arch.cuh"

namespace allegro {

// (a plain aggregate with external linkage: the fused two-body kernel takes it across TUs)
struct GeomParams {
  float rc, inv_rc;
  float freq[kNB];
  int lmax, dsh;
};

namespace {

__device__ __forceinline__ void sh_eval(const float n[3], float* Y, int lmax) {
  // component-normalised real SH (E3), m = -l..l; l = 1 stored (y, z, x)
  const float s3 = 1.7320508075688772f, s5 = 2.2360679774997896f, s15 = 3.8729833462074170f;
  Y[0] = 1.f;
  if (lmax >= 1) {
    Y[1] = s3 * n[1];
    Y[2] = s3 * n[2];
    Y[3] = s3 * n[0];
  }
  if (lmax >= 2) {
    Y[4] = s15 * n[0] * n[1];
    Y[5] = s15 * n[1] * n[2];
    Y[6] = 0.5f * s5 * (2.f * n[2] * n[2] - n[0] * n[0] - n[1] * n[1]);
    Y[7] = s15 * n[0] * n[2];
    Y[8] = 0.5f * s15 * (n[0] * n[0] - n[1] * n[1]);
  }
}

__device__ __forceinline__ void edge_vec(const double* __restrict__ apos, int32_t i, int32_t a, float r[3]) {
#pragma unroll
  for (int d = 0; d < 3; ++d) r[d] = (float)__dsub_rn(apos[(int64_t)a * 3 + d], apos[(int64_t)i * 3 + d]);
}


}  // namespace
}  // namespace allegro
