// md.cu -- velocity Verlet, kinetic energy, force statistics and the 5-sigma outlier
// count, plus deterministic fp64 reductions.
//
// Eq. 1 integrated under NVE with dt = 2 fs;
// velocity Verlet as SPEC.md:77:
//   v += (dt/2) kappa F/m;  r = wrap(r + dt v);  F = F(r);  v += (dt/2) kappa F/m
// kappa = 9.648533e-3 A fs^-2 per (eV A^-1 amu^-1); KE = 1/2 sum m v^2 / kappa (eV).
// Outliers (Fig. 1 caption): #{a : |F_a| > mean + k sigma}, strict
// (SPEC.md:452/457).
#include "ctx.cuh"

namespace allegro {
namespace {

constexpr double kKappa = 9.648533e-3;
constexpr double kMassH = 1.008, kMassN = 14.007;
constexpr int kRedThreads = 1024;

__device__ __forceinline__ double mass_of(int z) { return z == 1 ? kMassN : kMassH; }

// disp_max2 > 0: flag (blowup) when the drift |dt v| of an atom exceeds sqrt(disp_max2)
// (time-to-failure harness, "displacement_blowup")
__global__ void k_kick_drift(double* __restrict__ pos, double* __restrict__ vel, const double* __restrict__ frc,
                             const int32_t* __restrict__ species, int64_t n, double dt, double Lx, double Ly, double Lz,
                             double disp_max2, int* __restrict__ blowup) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  const double m = mass_of(species[a]);
  const double L[3] = {Lx, Ly, Lz};
  double d2 = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double v = vel[a * 3 + d] + 0.5 * dt * kKappa * frc[a * 3 + d] / m;
    vel[a * 3 + d] = v;
    d2 += (dt * v) * (dt * v);
    const double x = pos[a * 3 + d] + dt * v;
    double y = __dsub_rn(x, __dmul_rn(L[d], floor(__ddiv_rn(x, L[d]))));
    if (y >= L[d]) y = 0.0;
    pos[a * 3 + d] = y;
  }
  if (disp_max2 > 0.0 && !(d2 <= disp_max2)) atomicOr(blowup, 1);
}

__global__ void k_kick(double* __restrict__ vel, const double* __restrict__ frc, const int32_t* __restrict__ species,
                       int64_t n, double dt) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  const double m = mass_of(species[a]);
#pragma unroll
  for (int d = 0; d < 3; ++d) vel[a * 3 + d] += 0.5 * dt * kKappa * frc[a * 3 + d] / m;
}

__global__ void k_scale(double* __restrict__ vel, int64_t n3, double s) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a < n3) vel[a] *= s;
}

// Single-block fixed-order reduction of f(a) over a < n (deterministic).
template <typename F>
__device__ void block_reduce_sum(int64_t n, F f, double* out) {
  __shared__ double sm[kRedThreads];
  double s = 0.0;
  for (int64_t a = threadIdx.x; a < n; a += kRedThreads) s += f(a);
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = kRedThreads / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

__global__ void k_sum(const double* __restrict__ x, int64_t n, double* out) {
  block_reduce_sum(n, [&](int64_t a) { return x[a]; }, out);
}

__global__ void k_ke(const double* __restrict__ vel, const int32_t* __restrict__ species, int64_t n, double* out) {
  block_reduce_sum(
      n,
      [&](int64_t a) {
        const double v2 = vel[a * 3] * vel[a * 3] + vel[a * 3 + 1] * vel[a * 3 + 1] + vel[a * 3 + 2] * vel[a * 3 + 2];
        return 0.5 * mass_of(species[a]) * v2 / kKappa;
      },
      out);
}

__device__ __forceinline__ double fnorm(const double* F, int64_t a) {
  return sqrt(F[a * 3] * F[a * 3] + F[a * 3 + 1] * F[a * 3 + 1] + F[a * 3 + 2] * F[a * 3 + 2]);
}

__global__ void k_fnorm_sum(const double* __restrict__ F, int64_t n, double* out) {
  block_reduce_sum(n, [&](int64_t a) { return fnorm(F, a); }, out);
}

__global__ void k_fnorm_var(const double* __restrict__ F, int64_t n, const double* mean_sum, double* out) {
  const double mean = *mean_sum / (double)n;
  block_reduce_sum(
      n,
      [&](int64_t a) {
        const double d = fnorm(F, a) - mean;
        return d * d;
      },
      out);
}

__global__ void k_outliers(const double* __restrict__ F, int64_t n, double thr, unsigned long long* count) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool hit = a < n && fnorm(F, a) > thr;
  const unsigned b = __ballot_sync(0xffffffffu, hit);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(count, (unsigned long long)__popc(b));
}

__global__ void k_finite3(const double* __restrict__ x, int64_t n, int* flag) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= 3 * n) return;
  if (!isfinite(x[a])) atomicOr(flag, 1);
}

double fetch(allegro_ctx* c, const double* d) {
  double h = 0;
  ALG_CUDA(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  ALG_CUDA(cudaStreamSynchronize(c->stream));
  return h;
}

}  // namespace

void md_half_kick_drift(allegro_ctx* c, double dt) {
  if (c->n == 0) return;
  {
    ProfScope ps_(&c->prof, c->stream, PK_VERLET, 0, 124.0 * c->n);
    k_kick_drift<<<ceil_div(c->n, 256), 256, 0, c->stream>>>(c->pos.p, c->vel.p, c->frc.p, c->species.p, c->n, dt,
                                                           c->box[0], c->box[1], c->box[2], c->disp_max2,
                                                           c->flags.p + 4);
  }
  ALG_LAUNCH_CHECK();
}

void md_half_kick(allegro_ctx* c, double dt) {
  if (c->n == 0) return;
  {
    ProfScope ps_(&c->prof, c->stream, PK_VERLET, 0, 76.0 * c->n);
    k_kick<<<ceil_div(c->n, 256), 256, 0, c->stream>>>(c->vel.p, c->frc.p, c->species.p, c->n, dt);
  }
  ALG_LAUNCH_CHECK();
}

void md_scale_velocities(allegro_ctx* c, double s) {
  if (c->n == 0) return;
  {
    ProfScope ps_(&c->prof, c->stream, PK_VERLET, 0, 48.0 * c->n);
    k_scale<<<ceil_div(3 * c->n, 256), 256, 0, c->stream>>>(c->vel.p, 3 * c->n, s);
  }
  ALG_LAUNCH_CHECK();
}

double md_kinetic(allegro_ctx* c) {
  c->red.reserve(8);
  {
    ProfScope ps_(&c->prof, c->stream, PK_REDUCE, 0, 28.0 * c->n);
    k_ke<<<1, kRedThreads, 0, c->stream>>>(c->vel.p, c->species.p, c->n, c->red.p);
  }
  ALG_LAUNCH_CHECK();
  return allreduce_sum(c, fetch(c, c->red.p));
}

void sum_e_atom_async(allegro_ctx* c) {
  c->red.reserve(8);
  {
    ProfScope ps_(&c->prof, c->stream, PK_REDUCE, 0, 8.0 * c->n);
    k_sum<<<1, kRedThreads, 0, c->stream>>>(c->e_atom.p, c->n, c->red.p + 1);
  }
  ALG_LAUNCH_CHECK();
}

double sum_e_atom(allegro_ctx* c) {
  sum_e_atom_async(c);
  return fetch(c, c->red.p + 1);
}

void force_stats(allegro_ctx* c, double* mean, double* sigma) {
  c->red.reserve(8);
  const double n_tot = (double)allreduce_sum_i64(c, c->n);
  if (n_tot == 0) {
    *mean = *sigma = 0;
    return;
  }
  if (c->n == 0) {  // this rank owns nothing: still take part in the two reductions
    const double m = allreduce_sum(c, 0.0) / n_tot;
    *mean = m;
    *sigma = std::sqrt(allreduce_sum(c, 0.0) / n_tot);
    return;
  }
  {
    ProfScope ps_(&c->prof, c->stream, PK_REDUCE, 0, 24.0 * c->n);
    k_fnorm_sum<<<1, kRedThreads, 0, c->stream>>>(c->frc.p, c->n, c->red.p + 2);
  }
  ALG_LAUNCH_CHECK();
  {
    ProfScope ps_(&c->prof, c->stream, PK_REDUCE, 0, 24.0 * c->n);
    k_fnorm_var<<<1, kRedThreads, 0, c->stream>>>(c->frc.p, c->n, c->red.p + 2, c->red.p + 3);
  }
  ALG_LAUNCH_CHECK();
  // two passes: the global mean first, then the population variance about it
  const double mean_g = allreduce_sum(c, fetch(c, c->red.p + 2)) / n_tot;
  const double mean_l = fetch(c, c->red.p + 2) / (double)c->n;
  // k_fnorm_var used the local mean: shift to the global mean: sum (x - m_g)^2 = S_l + n (m_l - m_g)^2
  const double var_l = fetch(c, c->red.p + 3) + (double)c->n * (mean_l - mean_g) * (mean_l - mean_g);
  *mean = mean_g;
  *sigma = std::sqrt(allreduce_sum(c, var_l) / n_tot);
}

int64_t count_outliers(allegro_ctx* c, double thr) {
  c->red.reserve(8);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(c->red.p + 4);
  ALG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), c->stream));
  if (c->n > 0) {
    {
      ProfScope ps_(&c->prof, c->stream, PK_REDUCE, 0, 24.0 * c->n);
      k_outliers<<<ceil_div(c->n, 256), 256, 0, c->stream>>>(c->frc.p, c->n, thr, cnt);
    }
    ALG_LAUNCH_CHECK();
  }
  unsigned long long h = 0;
  ALG_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  ALG_CUDA(cudaStreamSynchronize(c->stream));
  return allreduce_sum_i64(c, (int64_t)h);
}

bool all_finite(allegro_ctx* c) {
  // flags[2] is set by the force gather; also check velocities
  if (c->n > 0 && c->md_ready) {
    {
      ProfScope ps_(&c->prof, c->stream, PK_REDUCE, 0, 24.0 * c->n);
      k_finite3<<<ceil_div(3 * c->n, 256), 256, 0, c->stream>>>(c->vel.p, c->n, c->flags.p + 2);
    }
    ALG_LAUNCH_CHECK();
  }
  int f = 0;
  if (c->dom.multi && c->e_pot_pending) {  // one packed allreduce + one host read per step
    allreduce_e_flag(c, c->red.p + 1, c->flags.p + 2, &c->e_pot, &f);
    c->e_pot_pending = false;
    return f == 0 && std::isfinite(c->e_pot);
  }
  ALG_CUDA(cudaMemcpyAsync(&f, c->flags.p + 2, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  if (c->e_pot_pending) ALG_CUDA(cudaMemcpyAsync(&c->e_pot, c->red.p + 1, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  ALG_CUDA(cudaStreamSynchronize(c->stream));
  c->e_pot_pending = false;
  f = allreduce_max_i32(c, f);
  return f == 0 && std::isfinite(c->e_pot);
}

bool check_inputs(allegro_ctx* c) {
  int f = 0;
  ALG_CUDA(cudaMemcpyAsync(&f, c->flags.p + 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  ALG_CUDA(cudaStreamSynchronize(c->stream));
  return allreduce_max_i32(c, f) == 0;
}

}  // namespace allegro
