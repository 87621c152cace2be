// geom.cuh -- per-edge geometry of the model (E1-E3 of SURVEY.md §8(c)): the edge vector (canonical
// fp64 difference, then fp32), the component-normalised real spherical harmonics, and the
// parameters of the envelope / Bessel basis.  Shared by model.cu and twobody.cu.
#pragma once
#include <cstdint>

#include "arch.cuh"
#include "layer.cuh"

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


// Y-bar of edge e (chunk-local) into registers (the first dsh entries)
__device__ __forceinline__ void load_ybar(const float* __restrict__ ybar, int64_t e, int dsh, float* yb) {
  if (dsh == 4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(ybar) + e);
    yb[0] = v.x, yb[1] = v.y, yb[2] = v.z, yb[3] = v.w;
  } else {
#pragma unroll
    for (int k = 0; k < 9; ++k)
      if (k < dsh) yb[k] = __ldg(ybar + e * dsh + k);
  }
}

// The geometry adjoint of one edge (global index ge, edge vector r), given zbar = ab1 W0[Bessel
// rows]^T, its u-bar and Y-bar: the u / B chain rule, the envelope derivative and the Y-bar term;
// writes g [E][4] (shared by k_geom_bwd and the fused two-body reverse, so both give the same bits).
// rr = rev[ge]: g is also stored at gT[rr] (the reverse edge's slot, [E][3] packed), or gT[ge] = 0
// when the edge has no reverse (rev is an involution, so every gT slot has exactly one writer).
__device__ __forceinline__ void geom_bwd_tail(const GeomParams& gp, const float r[3], float ub, const float* yb,
                                              float s0, const float* zbar, float* __restrict__ g, int64_t ge,
                                              int32_t rr, float* __restrict__ gT) {
  const float d = sqrtf(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  const float inv = 1.f / d;
  const float n[3] = {r[0] * inv, r[1] * inv, r[2] * inv};
  const float x = d * gp.inv_rc;
  float uu = 0.f, du = 0.f;
  if (x < 1.f) {
    const float x2 = x * x, x3 = x2 * x, x5 = x3 * x2, x6 = x3 * x3;
    uu = 1.f - 28.f * x6 + 48.f * x6 * x - 21.f * x6 * x2;
    du = -168.f * gp.inv_rc * x5 * (1.f - x) * (1.f - x);
  }
  float db = 0.f;
  const float pre = 2.f * gp.inv_rc;
#pragma unroll
  for (int q = 0; q < kNB; ++q) {
    const float k = gp.freq[q] * gp.inv_rc;
    float sn, cs;
    sincosf(k * d, &sn, &cs);
    const float B = pre * sn * inv;
    const float dB = pre * (k * cs * inv - sn * inv * inv);
    const float zb = s0 * zbar[q];
    ub = fmaf(zb, B, ub);
    db = fmaf(uu * zb, dB, db);
  }
  db = fmaf(ub, du, db);
  float gx = db * n[0], gy = db * n[1], gz = db * n[2];
  // sum_m Ybar[m] dY_m/dr,  dY^l/dr = (grad P_l(n) - l Y^l n) / d
  if (gp.lmax >= 1) {
    const float s3 = 1.7320508075688772f;
    const float b1 = yb[1], b2 = yb[2], b3 = yb[3];
    const float dot1 = b1 * n[1] + b2 * n[2] + b3 * n[0];  // sum_m yb_m Y_m / sqrt3
    gx += s3 * inv * (b3 - dot1 * n[0]);
    gy += s3 * inv * (b1 - dot1 * n[1]);
    gz += s3 * inv * (b2 - dot1 * n[2]);
    if (gp.lmax >= 2) {
      const float s5 = 2.2360679774997896f, s15 = 3.8729833462074170f;
      const float c0 = yb[4], c1 = yb[5], c2 = yb[6], c3 = yb[7], c4 = yb[8];
      float Y2[5] = {s15 * n[0] * n[1], s15 * n[1] * n[2], 0.5f * s5 * (2.f * n[2] * n[2] - n[0] * n[0] - n[1] * n[1]),
                     s15 * n[0] * n[2], 0.5f * s15 * (n[0] * n[0] - n[1] * n[1])};
      const float sy = c0 * Y2[0] + c1 * Y2[1] + c2 * Y2[2] + c3 * Y2[3] + c4 * Y2[4];
      // grad P2 at n
      const float px = s15 * (c0 * n[1] + c3 * n[2]) + 0.5f * s5 * c2 * (-2.f * n[0]) + 0.5f * s15 * c4 * (2.f * n[0]);
      const float py = s15 * (c0 * n[0] + c1 * n[2]) + 0.5f * s5 * c2 * (-2.f * n[1]) + 0.5f * s15 * c4 * (-2.f * n[1]);
      const float pz = s15 * (c1 * n[1] + c3 * n[0]) + 0.5f * s5 * c2 * (4.f * n[2]);
      gx += inv * (px - 2.f * sy * n[0]);
      gy += inv * (py - 2.f * sy * n[1]);
      gz += inv * (pz - 2.f * sy * n[2]);
    }
  }
  const float4 g4 = make_float4(gx, gy, gz, 0.f);
  reinterpret_cast<float4*>(g)[ge] = g4;
  if (gT != nullptr) {  // packed [E][3]: the force gather reads 12 B per edge from it
    const int64_t t = 3 * (rr >= 0 ? (int64_t)rr : ge);
    gT[t] = rr >= 0 ? gx : 0.f;
    gT[t + 1] = rr >= 0 ? gy : 0.f;
    gT[t + 2] = rr >= 0 ? gz : 0.f;
  }
}

}  // namespace
}  // namespace allegro
