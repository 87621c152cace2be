// pimd.cu -- replica batches and ring-polymer path-integral MD (NEXT-3 of SURVEY.md §8(f)).
//
// PAPER.md:419-429 (§5): PIMD "where each atom has 32 replicas that are harmonically coupled
// together ... the major cost is computing the energy and forces for the atoms within each
// replica".  The paper gives no integrator; reading D25: ring-polymer MD in the
// convention H_P = sum_j [K_j + V(q_j)] + sum_i sum_j m_i w_P^2 |q_ij - q_i,j+1|^2 / 2,
// w_P = P k_B T / hbar (beads at temperature P T), integrated as
//   v += (dt/2) kappa F/m;  exact free ring-polymer evolution over dt in normal modes;
//   F = -grad V(q_j) for all beads (one batched evaluation);  v += (dt/2) kappa F/m.
// Normal modes (real orthogonal basis of the cyclic ring, C[j][k], j = bead, k = mode):
//   C[j][0] = 1/sqrt(P);  C[j][k] = sqrt(2/P) cos(2 pi j k / P) for 1 <= k < P/2;
//   C[j][P/2] = (-1)^j / sqrt(P) (P even);  C[j][k] = sqrt(2/P) sin(2 pi j k / P) for k > P/2;
//   w_k = 2 w_P sin(k pi / P).
// The batched force evaluation is the single-replica path with the cells keyed by replica
// (neighbor.cu CellGeom::n_per): every replica's edges, rows and sums are exactly those of a
// single evaluation of that replica.
#include <cmath>
#include <vector>

#include "ctx.cuh"

namespace allegro {
namespace {

constexpr double kKappaP = 9.648533e-3;   // A fs^-2 per (eV A^-1 amu^-1)
constexpr double kKB = 8.617333e-5;       // eV / K
constexpr double kHbar = 0.6582119569;    // eV fs
constexpr int kMaxBeads = 64;
constexpr int kRed = 1024;

__device__ __forceinline__ double bead_mass(int z) { return z == 1 ? 14.007 : 1.008; }

__global__ void k_iota_mod(int32_t* __restrict__ gid, int64_t n, int64_t n_per) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a < n) gid[a] = (int32_t)(a % n_per);
}

__global__ void k_rep_species(const int32_t* __restrict__ s, int32_t* __restrict__ out, int64_t n, int64_t n_per) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a < n) out[a] = s[a % n_per];
}

// one block per replica: fixed-order sum of e_atom over the replica's atoms
__global__ void k_segment_sum(const double* __restrict__ x, int64_t len, double* __restrict__ out) {
  __shared__ double sm[kRed];
  const double* base = x + (int64_t)blockIdx.x * len;
  double s = 0.0;
  for (int64_t a = threadIdx.x; a < len; a += kRed) s += base[a];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = kRed / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}

// exact free ring-polymer evolution over dt: thread = (atom i, component d)
// mode[3k..3k+2] = (cos w_k dt, sin w_k dt, w_k)
__global__ void k_pimd_free(double* __restrict__ q, double* __restrict__ v, int64_t n_per, int P,
                            const double* __restrict__ C, const double* __restrict__ mode, double dt) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 3 * n_per) return;
  const int64_t stride = 3 * n_per;
  double xq[kMaxBeads], xv[kMaxBeads];
  for (int k = 0; k < P; ++k) {
    double a = 0.0, b = 0.0;
    for (int j = 0; j < P; ++j) {
      a += C[j * P + k] * q[j * stride + t];
      b += C[j * P + k] * v[j * stride + t];
    }
    const double cs = mode[3 * k], sn = mode[3 * k + 1], w = mode[3 * k + 2];
    if (w == 0.0) {
      xq[k] = a + b * dt;
      xv[k] = b;
    } else {
      xq[k] = a * cs + b * (sn / w);
      xv[k] = -a * w * sn + b * cs;
    }
  }
  for (int j = 0; j < P; ++j) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < P; ++k) {
      a += C[j * P + k] * xq[k];
      b += C[j * P + k] * xv[k];
    }
    q[j * stride + t] = a;
    v[j * stride + t] = b;
  }
}

// spring energy sum_i sum_j m_i w_P^2 |q_ij - q_i,j+1|^2 / (2 kappa)  (eV), fixed order
__global__ void k_pimd_spring(const double* __restrict__ q, const int32_t* __restrict__ species, int64_t n_per, int P,
                              double wp2, double* __restrict__ out) {
  __shared__ double sm[kRed];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n_per; i += kRed) {
    double acc = 0.0;
    for (int j = 0; j < P; ++j) {
      const int jn = (j + 1) % P;
      for (int d = 0; d < 3; ++d) {
        const double dx = q[((int64_t)j * n_per + i) * 3 + d] - q[((int64_t)jn * n_per + i) * 3 + d];
        acc += dx * dx;
      }
    }
    s += 0.5 * bead_mass(species[i]) * wp2 * acc / kKappaP;
  }
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = kRed / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

double fetch1(allegro_ctx* c, const double* d) {
  double h = 0;
  ALG_CUDA(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  ALG_CUDA(cudaStreamSynchronize(c->stream));
  return h;
}

}  // namespace

void set_replicas(allegro_ctx* c, int64_t n_rep, int64_t n_per, const int32_t* species_dev_per) {
  c->n_rep = n_rep;
  c->n_per = n_per;
  const int64_t n = n_rep * n_per;
  {
    ProfScope ps_(&c->prof, c->stream, PK_WRAP, 0, 8.0 * n);
    k_iota_mod<<<ceil_div(std::max<int64_t>(n, 1), 256), 256, 0, c->stream>>>(c->gid.p, n, n_per);
    if (species_dev_per)
      k_rep_species<<<ceil_div(std::max<int64_t>(n, 1), 256), 256, 0, c->stream>>>(species_dev_per, c->species.p, n,
                                                                                    n_per);
  }
  ALG_LAUNCH_CHECK();
}

void replica_energies(allegro_ctx* c) {
  c->e_rep.reserve(c->n_rep + 1);
  {
    ProfScope ps_(&c->prof, c->stream, PK_REDUCE, 0, 8.0 * c->n);
    k_segment_sum<<<(unsigned)c->n_rep, kRed, 0, c->stream>>>(c->e_atom.p, c->n_per, c->e_rep.p);
  }
  ALG_LAUNCH_CHECK();
}

void pimd_setup_modes(allegro_ctx* c, int P) {
  if (P < 1 || P > kMaxBeads) throw std::invalid_argument("n_beads must be in [1, 64]");
  std::vector<double> C((size_t)P * P);
  for (int j = 0; j < P; ++j)
    for (int k = 0; k < P; ++k) {
      double v;
      if (k == 0) v = 1.0 / std::sqrt((double)P);
      else if (2 * k < P) v = std::sqrt(2.0 / P) * std::cos(2.0 * M_PI * j * k / P);
      else if (2 * k == P) v = ((j % 2) ? -1.0 : 1.0) / std::sqrt((double)P);
      else v = std::sqrt(2.0 / P) * std::sin(2.0 * M_PI * j * k / P);
      C[(size_t)j * P + k] = v;
    }
  c->pimd_c.reserve(C.size());
  ALG_CUDA(cudaMemcpyAsync(c->pimd_c.p, C.data(), sizeof(double) * C.size(), cudaMemcpyHostToDevice, c->stream));
  ALG_CUDA(cudaStreamSynchronize(c->stream));
}

double pimd_omega_p(allegro_ctx* c) { return (double)c->n_rep * kKB * c->pimd_T / kHbar; }  // 1/fs

void pimd_free_step(allegro_ctx* c, double dt) {
  const int P = (int)c->n_rep;
  const double wp = pimd_omega_p(c);
  std::vector<double> mode((size_t)3 * P);
  for (int k = 0; k < P; ++k) {
    const double w = 2.0 * wp * std::sin(k * M_PI / P);
    mode[3 * k] = std::cos(w * dt);
    mode[3 * k + 1] = std::sin(w * dt);
    mode[3 * k + 2] = k == 0 ? 0.0 : w;
  }
  c->pimd_mode.reserve(mode.size());
  ALG_CUDA(cudaMemcpyAsync(c->pimd_mode.p, mode.data(), sizeof(double) * mode.size(), cudaMemcpyHostToDevice,
                           c->stream));
  {
    ProfScope ps_(&c->prof, c->stream, PK_VERLET, 2.0 * 2 * P * P * 3.0 * c->n_per, 48.0 * c->n);
    k_pimd_free<<<ceil_div(3 * c->n_per, 128), 128, 0, c->stream>>>(c->pq.p, c->vel.p, c->n_per, P, c->pimd_c.p,
                                                                    c->pimd_mode.p, dt);
  }
  ALG_LAUNCH_CHECK();
  ALG_CUDA(cudaStreamSynchronize(c->stream));  // the host mode table is reused next step
}

double pimd_spring_energy(allegro_ctx* c) {
  c->red.reserve(8);
  const double wp = pimd_omega_p(c);
  {
    ProfScope ps_(&c->prof, c->stream, PK_REDUCE, 0, 24.0 * c->n);
    k_pimd_spring<<<1, kRed, 0, c->stream>>>(c->pq.p, c->species.p, c->n_per, (int)c->n_rep, wp * wp, c->red.p + 5);
  }
  ALG_LAUNCH_CHECK();
  return fetch1(c, c->red.p + 5);
}

}  // namespace allegro
