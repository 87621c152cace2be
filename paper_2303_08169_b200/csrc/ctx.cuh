// ctx.cuh -- the runtime state behind the opaque allegro_ctx, and the internal entry
// points of each subsystem (neighbour build, model, MD).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/allegro.h"
#include "arch.cuh"
#include "common.cuh"
#include "prof.cuh"
#include "tc_gemm.cuh"
#include "comm.cuh"

namespace allegro {

struct WeightsError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct GeometryError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Device buffer that only grows (capacity in elements of T).
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;
  void reserve(size_t n) {
    if (n <= cap) return;
    if (p) cudaFree(p);
    p = nullptr;
    size_t c = n + n / 4 + 64;
    if (cudaMalloc(&p, c * sizeof(T)) != cudaSuccess) {
      cap = 0;
      p = nullptr;
      cudaGetLastError();
      throw CudaError("OOM: cudaMalloc of " + std::to_string(c * sizeof(T)) + " bytes");
    }
    cap = c;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Runtime view of the compile-time layer architecture (same constexpr derivation).
struct LayerInfo {
  LayerArch A;
  int nw;              // env-embed outputs: C * n_env * (2 if k == 0 else 1)
  int fan_lat;         // D + C * n_s
  int t_base[kMaxIr];  // per out irrep: offset (floats per edge) of T_o in the T scratch
  int v_base[kMaxIr];  // per in irrep: offset (floats per edge) of V_ir in the V store of this layer
  int tp_nnz;          // non-zero W3j entries summed over the layer's paths (FMAs per edge-channel)
};

// One GEMM weight W [K][N]: fp32 row-major (CUDA-core path) and, in 3xTF32 mode, the
// pre-split / pre-swizzled tensor-core image.
struct Wt {
  float* f = nullptr;
  TcWeight tc;
  int K = 0, N = 0;
};

struct DevWeights {
  Wt tb_w0;   // [16][32], rows 12..15 zero
  Wt tb_w1;   // [32][64]
  Wt tb_w2;   // [64][128]
  Wt tb_w0T;  // [32][16]
  Wt tb_w1T;  // [64][32]
  Wt tb_w2T;  // [128][64]
  Wt env[kMaxLayers];             // [128][nw]  columns in [chunk][l][c] order
  Wt envT[kMaxLayers];            // [nw][128]
  Wt lin[kMaxLayers][kMaxIr];     // [n_to*C][C]   rows (path_local, c)
  Wt linT[kMaxLayers][kMaxIr];    // [C][n_to*C]
  Wt lat[kMaxLayers];             // [128 + n_s*C][128], scalar rows in (q, c) order
  Wt latT_x[kMaxLayers];          // [128][128]
  Wt latT_s[kMaxLayers];          // [128][n_s*C]
  Wt latenvT[kMaxLayers];         // [128 + nw][128]: latT_x stacked over envT (the merged x-bar contraction)
  float* wout = nullptr;          // [128] = W_o1 W_o2 / (sqrt(128) sqrt(32))
  // last layer folded into the linear read-out: q = W_lat(L-1) w_out
  float* q_last = nullptr;        // [fan_lat(L-1)] device row order (x rows, then scalar rows (q, c))
  float* r2_vec1 = nullptr;       // [128] a w_out
  float* r2_vec2 = nullptr;       // [128] (b / sqrt(fan)) q_x
  float bessel[kNB] = {};
  std::vector<void*> owned;
};

struct Model {
  int n_layers = 0, lmax = 0;
  int precision = ALLEGRO_PREC_FP32;
  double r_max = 0, nbar = 0, sigma[2] = {1, 1}, mu[2] = {0, 0};
  LayerInfo L[kMaxLayers];
  DevWeights w;
};

// Per-chunk activation workspace (fp32, row-major [E_cap][width]).
struct Workspace {
  size_t e_cap = 0, a_cap = 0;
  DBuf<float> z, a1, h1, a2, h2, m, u, Y;
  DBuf<float> xa, xb;
  DBuf<float> w[kMaxLayers], h[kMaxLayers], V[kMaxLayers], G[kMaxLayers];
  DBuf<float> T;
  DBuf<float> xbar_a, xbar_b, sbar, vbar_a, vbar_b, wbar, ybar, ubar, zbar, ab2, ab1, ee, ebar, gp, dotp;
};

// Spatial domain decomposition (§2.4).
struct HaloStage {
  int64_t n_send[2] = {0, 0};   // to the -/+ neighbour
  int64_t n_recv[2] = {0, 0};   // from the -/+ neighbour
  int64_t recv_base[2] = {0, 0};  // first atom index of the ghosts received from -/+
  DBuf<int32_t> send_idx[2];    // local atom indices sent to -/+
};

struct Domain {
  bool multi = false;           // world_size > 1
  int rank = 0, size = 1;
  int P[3] = {1, 1, 1}, c[3] = {0, 0, 0};
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, w[3] = {0, 0, 0};
  int nbr[3][2] = {};           // ranks of the -/+ neighbours per axis
  ncclComm_t comm = nullptr;
  HaloStage st[3];
  DBuf<unsigned char> sendbuf[2], recvbuf[2];
  DBuf<int32_t> flag, pos_idx;
  DBuf<long long> acc;          // [n + G][3] fixed-point ghost-force accumulators
  DBuf<long long> cnt;          // scratch counts
  DBuf<long long> hs;           // halo message-path state (domain.cu: n_cur, overflow, per-stage counts)
  double cap_scale = 1.0;       // halo message capacity scale (doubled on overflow, on every rank;
                                // ALLEGRO_HALO_CAP_SCALE sets the start, a test hook)
  DBuf<long long> ms;           // migration message-path state (owned count, stayers, overflow)
  DBuf<unsigned char> mstage;   // migration stayers staging (MigAtom)
  DBuf<double> red;             // allreduce scratch
  // migration / halo scratch (per ctx, so ctxs on different devices or threads never share it)
  DBuf<double> tpos, tvel;
  DBuf<int32_t> tgid, tspec, f0, f1, f2, i0, i1, i2;
};

}  // namespace allegro

struct allegro_ctx {
  std::string err;
  allegro_params prm{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  double box[3] = {0, 0, 0};
  double r_cut = 0, skin = 0;
  allegro::Model model;

  // ---- atoms (owned first, then ghosts) ----
  int64_t n = 0;        // owned (this rank)
  int64_t n_global = 0; // atoms in the whole box (md state)
  int64_t n_ghost = 0;  // ghosts of the last build
  int64_t n_rep = 1;    // replica batch (PIMD beads): n = n_rep * n_per, replica-major
  int64_t n_per = 0;
  allegro::DBuf<double> pos, vel, frc;       // [n][3] owned state (fp64)
  allegro::DBuf<int32_t> species, gid;       // [n]
  allegro::DBuf<double> apos;                // [n + G][3] canonical image positions
  allegro::DBuf<int32_t> aowner, ashift, agid, aspec;  // [n + G] (aowner = -1 for remote ghosts)
  allegro::DBuf<int32_t> gcount, goff;       // ghost count / offsets per owned atom
  // ---- cells ----
  int ncell[3] = {0, 0, 0};
  double cell_lo[3] = {0, 0, 0}, cell_size[3] = {0, 0, 0};
  allegro::DBuf<int32_t> ccount, cstart, cslot, csorted;
  allegro::DBuf<double4> cpos;  // positions in cell order (x, y, z, pad)
  // ---- edges (CSR by owned centre, canonical row order) ----
  int max_nb = 256;
  int64_t n_edges = 0;
  allegro::DBuf<int32_t> nb_count, nb_pad, row_ptr, nbr, cidx, rev;
  allegro::DBuf<unsigned long long> key_pad, key;
  allegro::DBuf<float> g;                    // [E][4] dE/dr_e (x, y, z, pad)
  allegro::DBuf<float> gT;                   // [E][3] gT[e] = g[rev[e]] (0 without a reverse edge), scattered by
                                             // the producer of g so the force gather streams both arrays
  std::vector<int32_t> h_row_ptr;
  std::vector<int64_t> chunk_a0;             // first centre atom of each model chunk (last evaluation)
  // ---- scalars / flags ----
  allegro::DBuf<int> flags;                  // [0] overflow max count, [1] bad input, [2] non-finite
  allegro::DBuf<double> red;                 // reduction scratch
  allegro::DBuf<double> e_atom;              // [n]
  allegro::DBuf<int32_t> scan_tmp;
  allegro::DBuf<int32_t> scan_lv[8];          // exclusive_scan block sums per recursion level
  allegro::Workspace ws;
  size_t ws_budget_bytes = 0;
  // ---- MD ----
  bool md_ready = false;
  int64_t md_steps = 0, n_rebuilds = 0;
  double e_pot = 0;
  bool e_pot_pending = false;  // e_pot is in red[1] on the device (read by all_finite)
  double f_mean0 = 0, f_sigma0 = 0;  // step-0 outlier baseline
  // Nose-Hoover NVT (one thermostat; D23): off when tau <= 0
  bool nvt = false;
  double nvt_T = 0, nvt_tau = 0, nvt_Q = 0, nvt_xi = 0, nvt_eta = 0;
  double disp_max2 = 0;  // time-to-failure harness: squared single-step displacement limit (0 = off)
  // ring-polymer PIMD (NEXT-3; D25): unwrapped bead state, replica-major [P][N][3]
  bool pimd_ready = false;
  int64_t pimd_steps = 0;
  double pimd_T = 0;
  allegro::DBuf<double> pq, pv, pimd_c, pimd_mode, e_rep;  // C [P][P]; per mode (cos, sin, w); [P]
  bool baseline_set = false;
  allegro::Profiler prof;
  allegro::Domain dom;
};

namespace allegro {

// weights.cu
void load_model(allegro_ctx* c, const char* path);
void free_model(Model& m);

// scan.cu: out[i] = sum_{j<i} in[j] (int32), out[n] = total; returns total (host sync)
void exclusive_scan(allegro_ctx* c, const int32_t* in, int32_t* out, int64_t n);

// neighbor.cu: wrap owned positions, build ghosts, cells, CSR edges and reverse index.
void build_neighbors(allegro_ctx* c);
void wrap_positions(allegro_ctx* c);

// model.cu: energies and forces for the current edge list -> c->frc, c->e_atom, c->e_pot
void compute_forces(allegro_ctx* c, bool defer_e = false);  // defer_e: e_pot read by all_finite

// domain.cu (world_size > 1)
void domain_setup(allegro_ctx* c, const void* nccl_id);
void domain_teardown(allegro_ctx* c);
void migrate(allegro_ctx* c);
bool all_owned(allegro_ctx* c);          // every owned atom lies in this rank's domain (collective)
void halo_exchange(allegro_ctx* c);     // fills apos/agid/aspec/ashift for owned + ghosts
void ghost_force_return(allegro_ctx* c);  // accumulates ghost forces and returns them to owners
double allreduce_sum(allegro_ctx* c, double v);
void allreduce_e_flag(allegro_ctx* c, const double* d_e, const int* d_flag, double* e, int* flag);
int64_t allreduce_sum_i64(allegro_ctx* c, int64_t v);
int allreduce_max_i32(allegro_ctx* c, int v);
void select_owned(allegro_ctx* c, int64_t n_global, const int32_t* species, const double* pos, const double* vel);
void gather_state(allegro_ctx* c, int64_t n_global, double* pos, double* vel, double* forces);
constexpr double kFixScale = 4294967296.0;  // 2^32: fixed-point ghost forces (exact, order independent)

// md.cu
void md_half_kick_drift(allegro_ctx* c, double dt);
void md_half_kick(allegro_ctx* c, double dt);
void md_scale_velocities(allegro_ctx* c, double s);
double md_kinetic(allegro_ctx* c);
void force_stats(allegro_ctx* c, double* mean, double* sigma);
int64_t count_outliers(allegro_ctx* c, double thr);
bool all_finite(allegro_ctx* c);
double sum_e_atom(allegro_ctx* c);
void sum_e_atom_async(allegro_ctx* c);  // the sum into red[1] without reading it
bool check_inputs(allegro_ctx* c);

// pimd.cu (replica batches, ring-polymer MD; world_size == 1)
void set_replicas(allegro_ctx* c, int64_t n_rep, int64_t n_per, const int32_t* species_dev_per);
void replica_energies(allegro_ctx* c);  // c->e_rep[r] = sum of e_atom over replica r
void pimd_setup_modes(allegro_ctx* c, int P);
void pimd_free_step(allegro_ctx* c, double dt);
double pimd_spring_energy(allegro_ctx* c);
double pimd_omega_p(allegro_ctx* c);

}  // namespace allegro
