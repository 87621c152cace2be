/*
 * allegro.h -- C ABI of the B200-native Allegro-Legato NNQMD hot path.
 *
 * One MD step of the paper's method: the energy and analytic forces of a
 * strictly local E(3)-equivariant Allegro model, then a velocity-Verlet update.
 *
 *   Eq. 1 (§2.1):  m_i d^2 r_i / dt^2 = f_i = -dE/dr_i
 *   Allegro (§2.1): E = sum of pairwise embedding energies
 *       E_ij within a finite cutoff, equivariant to E(3), tensors up to rank l
 *       and tensor products of irreps.  The concrete model is the reading
 *       written out in SURVEY.md §8(c) E1-E9.
 *   NVE integration at dt = 2 fs (§3.2); velocity Verlet as
 *       SPEC.md:77.
 *   5-sigma force outliers (Fig. 1 caption).
 *   Neighbour lists by linked-list cells (§2.4), here on device.
 *
 * Conventions (all calls):
 *   - Every call returns int status: 0 = ALLEGRO_OK, < 0 = an ALLEGRO_E_* code.
 *     No C++ exception crosses the ABI.  allegro_last_error() gives a message.
 *   - Units: positions A, velocities A/fs, time fs, energies eV, forces eV/A,
 *     masses amu (H 1.008, N 14.007).  Species: 0 = H, 1 = N.
 *   - Arrays are caller-owned.  `where` selects host (ALLEGRO_HOST) or device
 *     (ALLEGRO_DEVICE, CUDA global memory on the ctx's device) pointers for the
 *     per-atom arrays of allegro_compute_energy_forces; device pointers are used
 *     with zero copy.  No pointer is retained after a call returns.
 *   - Layouts: pos / forces / vel are row-major [n][3] float64; gid, species
 *     are int32 [n]; e_atom is float64 [n].
 *   - Positions outside the box are wrapped into [0, L), not
 *     rejected.  Non-finite inputs -> ALLEGRO_E_ARG; species outside {0,1} ->
 *     ALLEGRO_E_ARG; a non-finite result -> ALLEGRO_E_NONFINITE (never masked,
 *     SPEC.md:78).
 *   - Determinism: results are bit-identical across repeated runs at a fixed
 *     world size and precision (fixed-order reductions, no float atomics).
 *   - Threading: one ctx per rank; calls on a ctx are not thread-safe.  With
 *     world_size > 1 every call that takes a ctx is collective.
 */
#ifndef ALLEGRO_B200_H
#define ALLEGRO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct allegro_ctx allegro_ctx; /* opaque; owns all device work buffers */

enum {
  ALLEGRO_OK = 0,
  ALLEGRO_E_ARG = -1,       /* bad argument (NULL, size, non-finite input, species) */
  ALLEGRO_E_GEOMETRY = -2,  /* domain smaller than r_c + skin with world_size > 1 */
  ALLEGRO_E_NONFINITE = -3, /* a non-finite energy / force / velocity was produced */
  ALLEGRO_E_WEIGHTS = -4,   /* weight file unreadable or inconsistent with its header */
  ALLEGRO_E_CUDA = -5,      /* CUDA runtime error */
  ALLEGRO_E_NCCL = -6,      /* NCCL error */
  ALLEGRO_E_OOM = -7,       /* device allocation failed */
  ALLEGRO_E_STATE = -8      /* call out of order (e.g. md_step before md_set_state) */
};

enum { ALLEGRO_HOST = 0, ALLEGRO_DEVICE = 1 };

/* Arithmetic of the per-edge MLP contractions (the only dense GEMMs).
 *   3XTF32  tcgen05 kind::tf32 in split precision (a_hi w_hi + a_hi w_lo + a_lo w_hi):
 *           fp32-level accuracy; the production and parity mode (the binding's default).
 *   FP32    CUDA-core fp32 FMA: the second parity gate (reference arithmetic).
 *   TF32    tcgen05, one pass (a_hi w_hi): fast, outside the force bound by ~30x (App. C);
 *           reported, not gated.
 *   BF16X3, BF16: reserved; allegro_create returns ALLEGRO_E_ARG (not built: the unfused
 *           contractions are HBM-bound, so halving their operand precision buys nothing). */
enum {
  ALLEGRO_PREC_FP32 = 0,
  ALLEGRO_PREC_3XTF32 = 1,
  ALLEGRO_PREC_BF16X3 = 2,
  ALLEGRO_PREC_TF32 = 3,
  ALLEGRO_PREC_BF16 = 4
};

typedef struct {
  const char* weights_path; /* weight file (synth/weights.py layout): header L, lmax, C, D,
                               widths, n_basis, n_species, p, r_max, nbar, sigma_Z, mu_Z */
  double r_cut;             /* A; must equal the file's r_max (else ALLEGRO_E_WEIGHTS); <= 0: take the file's */
  double skin;              /* A; 0 = rebuild the neighbour list every step (the paper: P:246) */
  double box[3];            /* orthorhombic periodic box edges, A */
  int64_t n_atoms_global;   /* atoms in the whole box */
  int device;               /* CUDA ordinal for this rank */
  int rank, world_size;     /* 1 GPU: 0, 1 */
  const void* nccl_unique_id; /* 128-byte ncclUniqueId broadcast by the caller; NULL if world_size == 1 */
  int grid[3];              /* domain grid px,py,pz (product == world_size); {0,0,0} = auto */
  int precision;            /* ALLEGRO_PREC_* (0 = FP32 for a zeroed struct; ALLEGRO_PREC_3XTF32 is production) */
  void* cuda_stream;        /* cudaStream_t to run on (e.g. torch's current stream); NULL = ctx-owned stream.
                               Device pointers passed to the calls are read / written on this stream: the
                               caller orders their producers / consumers with it (e.g. pass torch's current
                               stream, or synchronise before the call); every call that returns results to
                               the host synchronises the stream before it returns. */
} allegro_params;

/* Create a ctx: reads and validates the weight file (tensor shapes and the parameter
 * count are re-derived from the irreps rules; Table 2), uploads fp32
 * weights, and sizes buffers.  Collective over ranks.  On failure *out is NULL and
 * allegro_last_error(NULL) describes the error (thread-local). */
int allegro_create(const allegro_params* p, allegro_ctx** out);
void allegro_destroy(allegro_ctx* ctx);
const char* allegro_last_error(const allegro_ctx* ctx);

/* One force evaluation (Eq. 1).
 *   n        owned atoms passed by this rank (world_size 1: all atoms)
 *   where    ALLEGRO_HOST or ALLEGRO_DEVICE for gid/species/pos/e_atom/forces
 *   gid      [n] global ids (NULL: 0..n-1); identify atoms in the canonical row order
 *   species  [n] 0 = H, 1 = N
 *   pos      [n][3] A (wrapped internally)
 *   box      [3] A, or NULL = the box given at create
 *   e_total  out, host double, eV (all ranks)
 *   e_atom   out [n] eV, or NULL
 *   forces   out [n][3] eV/A
 * Returns ALLEGRO_E_NONFINITE if any output is non-finite. */
int allegro_compute_energy_forces(allegro_ctx* ctx, int64_t n, int where, const int32_t* gid,
                                  const int32_t* species, const double* pos, const double* box,
                                  double* e_total, double* e_atom, double* forces);

/* MD state lives on the device inside ctx.  set/get take GLOBAL host arrays
 * [n_global] (species, pos [n][3] A, vel [n][3] A/fs); set computes the initial forces.
 * With world_size > 1 every rank passes the same global arrays and keeps the atoms of its
 * domain (atom index = gid); get gathers the global state on rank 0 (other ranks' output
 * arrays are not written).  Collective. */
int md_set_state(allegro_ctx* ctx, int64_t n_global, const int32_t* species, const double* pos,
                 const double* vel);
int md_get_state(allegro_ctx* ctx, int64_t n_global, double* pos, double* vel, double* forces);

typedef struct {
  int64_t steps_done;
  double e_pot, e_kin, e_total, temperature; /* eV, eV, eV, K after the last step */
  int64_t n_outliers_last;                   /* outliers of the last step vs the step-0 baseline */
  int64_t n_edges, n_rebuilds;                /* edges summed over ranks */
  int64_t n_local;                           /* atoms this rank owns after the call */
  double xi;                                 /* Nose-Hoover friction (1/fs); 0 under NVE */
  double e_conserved;                        /* NVE: e_total; NVT: e_total + Q xi^2/2 + 3N k_B T eta */
} md_report;

/* NVT thermalisation (§3.2: 200 K NVT before NVE): one Nose-Hoover
 * thermostat, Q = 3N k_B T tau^2, symmetric split around the Verlet core
 * (D23).  tau_fs <= 0 switches back to NVE.  Takes effect for the following
 * md_step calls; md_set_state resets xi and eta. */
int md_set_thermostat(allegro_ctx* ctx, double T_target_K, double tau_fs);

/* n_steps of velocity Verlet at dt (fs): exactly one
 * force evaluation per step, forces cached.  Stops at the first non-finite value and
 * returns ALLEGRO_E_NONFINITE with steps_done set.  out may be NULL. */
int md_step(allegro_ctx* ctx, int64_t n_steps, double dt_fs, md_report* out);

/* Time-to-failure harness (NEXT-2 of SURVEY.md §8(f); §3.2 and Eq. 4).
 * The paper's protocol: NVT at 200 K for 1,000 steps, then NVE "until it fails"; the paper
 * does not define failure, so the criteria are SPEC.md:459's (D24):
 *   non_finite           a non-finite energy / force / velocity (every step),
 *   displacement_blowup  some atom drifts more than disp_max A in one step (every step),
 *   energy_drift         |E - E0| > drift_tol |E0| with E = E_pot + E_kin, checked every
 *                        check_interval NVE steps (E0 at the start of NVE).
 * Outliers (Fig. 1: |F_a| > mean + k sigma of the force norms at NVE start)
 * are recorded every outlier_interval steps but never trigger a failure. */
typedef struct {
  int64_t nvt_steps;        /* NVT steps before NVE (paper 1,000); 0 = start in NVE */
  double T_K, tau_fs;       /* NVT target (paper 200 K) and time constant (D23) */
  int64_t max_nve_steps;    /* censoring cap */
  int64_t check_interval;   /* energy-drift check cadence (SPEC: 100) */
  double drift_tol;         /* relative energy drift (SPEC: 0.1) */
  double disp_max;          /* single-step displacement limit, A; <= 0 disables */
  double outlier_k;         /* outlier threshold in sigmas (paper: 5) */
  int64_t outlier_interval; /* outlier-count cadence in NVE steps (>= 1) */
} md_ttf_protocol;

enum { ALLEGRO_TTF_CENSORED = 0, ALLEGRO_TTF_NONFINITE = 1, ALLEGRO_TTF_DISPLACEMENT = 2, ALLEGRO_TTF_ENERGY_DRIFT = 3 };

typedef struct {
  int64_t steps_survived; /* NVE steps completed before the failing one; max_nve_steps if censored */
  int64_t fail_step;      /* 1-based NVE step at which failure was detected; 0 if censored */
  int reason;             /* ALLEGRO_TTF_* */
  int failed_in_nvt;      /* 1: non-finite during thermalisation (NVE never started) */
  double e0, e_last;      /* E_pot + E_kin at NVE start and at the last drift check, eV */
  double f_mean, f_sigma; /* outlier baseline at NVE start, eV/A */
  int64_t n_series;       /* outlier counts written to the caller's series */
} md_ttf_result;

/* Runs the protocol from the current MD state (md_set_state first); the state afterwards is
 * the state at failure.  series (caller-owned, series_cap entries, may be NULL if 0) receives
 * the global outlier count every outlier_interval NVE steps.  Collective when world_size > 1.
 * Errors: ALLEGRO_E_ARG (bad protocol), ALLEGRO_E_STATE; a failure of the dynamics is a result
 * (reason), not an error. */
int md_run_ttf(allegro_ctx* ctx, double dt_fs, const md_ttf_protocol* protocol, int64_t* series, int64_t series_cap,
               md_ttf_result* out);

/* ---- Replica batches and ring-polymer PIMD (NEXT-3; §5; D25) ----
 * A batch of n_rep independent copies ("replicas", PIMD beads) of one n_per-atom system in
 * the box given at create, evaluated in ONE pass of the kernels: cells and edges are keyed by
 * replica, so replica r's energy and forces are exactly those of a single evaluation of it.
 * world_size must be 1.  pos / forces: [n_rep][n_per][3] A, eV/A (replica-major); species
 * [n_per] (shared by all replicas); e_rep [n_rep] eV; e_atom [n_rep * n_per] or NULL.
 * where = ALLEGRO_HOST / ALLEGRO_DEVICE for every array. */
int allegro_compute_energy_forces_batch(allegro_ctx* ctx, int64_t n_rep, int64_t n_per, int where,
                                        const int32_t* species, const double* pos, double* e_rep, double* e_atom,
                                        double* forces);

/* Ring-polymer MD: P = n_beads (1..64) beads per atom at physical temperature T_K, RPMD
 * Hamiltonian H_P = sum_j [K_j + V(q_j)] + sum_i sum_j m_i w_P^2 |q_ij - q_i,j+1|^2 / 2 with
 * w_P = P k_B T / hbar; each step: half kick with the bead forces, exact free ring-polymer
 * evolution in normal modes over dt, one batched force evaluation of all beads, half kick.
 * No thermostat (microcanonical RPMD).  Host arrays: species [n_per], pos / vel
 * [n_beads][n_per][3] (A, A/fs; positions are kept unwrapped so the springs see bead
 * differences, the force evaluation wraps a copy). */
int pimd_set_state(allegro_ctx* ctx, int64_t n_beads, int64_t n_per, const int32_t* species, const double* pos,
                   const double* vel, double T_K);
typedef struct {
  int64_t steps_done;
  double e_pot_mean;        /* (1/P) sum_j V(q_j), eV */
  double e_spring;          /* ring-polymer spring energy, eV */
  double e_kin;             /* kinetic energy of all beads, eV */
  double h_conserved;       /* sum_j V(q_j) + e_kin + e_spring (RPMD Hamiltonian), eV */
  double temperature_beads; /* 2 e_kin / (3 N P k_B), K (equals P T at equilibrium) */
  double omega_p;           /* P k_B T / hbar, 1/fs */
  int64_t n_edges;          /* edges of all beads */
} pimd_report;
int pimd_step(allegro_ctx* ctx, int64_t n_steps, double dt_fs, pimd_report* out);
/* host arrays [n_beads][n_per][3] (pos unwrapped) and e_rep [n_beads]; any may be NULL */
int pimd_get_state(allegro_ctx* ctx, double* pos, double* vel, double* forces, double* e_rep);

/* End-to-end variant of md_step for HOST-resident state (the e2e measurement of bench.py):
 * copies species [n], pos/vel/forces [n][3] (forces = F at pos, e.g. from the previous call
 * or from md_get_state) host -> device, runs n_steps exactly as md_step, and writes pos, vel
 * and forces (and, with world_size > 1, species) back into the caller's arrays (device ->
 * host).  n must equal the number of atoms this rank owns (allegro_local_count; all atoms on
 * one GPU).  capacity (>= n) is the number of rows the caller's arrays hold: with
 * world_size > 1 migration may change the local count (out->n_local returns it); if it
 * exceeds capacity nothing is copied back and ALLEGRO_E_ARG is returned (the state stays on
 * the device: md_get_local_state).  Pinned host memory makes the copies asynchronous. */
int md_step_host(allegro_ctx* ctx, int64_t n, int64_t capacity, int32_t* species, double* pos, double* vel,
                 double* forces, int64_t n_steps, double dt_fs, md_report* out);

/* Count atoms with |F_a| > mean + k*sigma (strict) for the current
 * forces.  Collective. */
int md_count_outliers(allegro_ctx* ctx, double mean, double sigma, double k, int64_t* count);
/* mean and population std of |F_a| over all atoms for the current forces */
int md_force_baseline(allegro_ctx* ctx, double* mean, double* sigma);

/* Test hook: the current edge list (of the last force evaluation) as (i_gid, j_gid, shift),
 * in the canonical row order (row by centre, within a row by (j_gid, nx, ny, nz)).
 * capacity: entries available in the output arrays; *n_edges receives the count
 * (ALLEGRO_E_ARG if capacity is too small; outputs may be NULL to query the count). */
int allegro_get_edges(allegro_ctx* ctx, int64_t capacity, int64_t* n_edges, int32_t* i_gid,
                      int32_t* j_gid, int8_t* shift);

/* Test hook: per-edge dE/dr_e [E][3] (fp32 widened to double) of the last evaluation,
 * in the edge order of allegro_get_edges. */
int allegro_get_edge_grad(allegro_ctx* ctx, int64_t capacity, double* g);

/* Test hook: the edges of selected rows (owned local atom indices `rows`, in that order; each
 * row in canonical order) as (i_gid, j_gid, shift) and their dE/dr_e [.][3] (g may be NULL).
 * *n_out receives the edge count; all outputs NULL = query.  ALLEGRO_E_ARG if capacity is too
 * small or a row is out of range. */
int allegro_get_row_edges(allegro_ctx* ctx, int64_t n_rows, const int64_t* rows, int64_t capacity, int64_t* n_out,
                          int32_t* i_gid, int32_t* j_gid, int8_t* shift, double* g);
/* Test hook: the first centre atom of each chunk of complete CSR rows the model ran in at the
 * last evaluation (chunks bound the per-edge workspace; results do not depend on them). */
int allegro_chunk_starts(allegro_ctx* ctx, int64_t capacity, int64_t* n_chunks, int64_t* first_atom);

/* world_size > 1: rank 0 creates the 128-byte NCCL unique id and broadcasts it (e.g. with
 * torch.distributed) to every rank's allegro_params.nccl_unique_id. */
int allegro_nccl_unique_id(void* out128);
/* atoms owned by this rank (its spatial domain) */
int64_t allegro_local_count(const allegro_ctx* ctx);
/* this rank's owned MD state (host arrays with room for `capacity` atoms; any may be NULL) */
int md_get_local_state(allegro_ctx* ctx, int64_t capacity, int64_t* n_local, int32_t* species, int32_t* gid,
                       double* pos, double* vel, double* forces);

/* Per-kernel-class accounting.  Every launch of the library is counted;
 * with profiling enabled each launch is also bracketed by CUDA events on the stream it is
 * launched on and its ALGORITHMIC flops / DRAM bytes are accumulated.
 * allegro_profile(ctx, 1) synchronises the stream, resets all totals and the launch counter
 * and starts recording; allegro_profile(ctx, 0) stops recording (no synchronisation) and
 * keeps the totals readable.  Kinds are 0 .. allegro_profile_kinds()-1. */
int allegro_profile(allegro_ctx* ctx, int enable);
int allegro_profile_read(allegro_ctx* ctx, int kind, double* time_ms, double* flops, double* bytes,
                         int64_t* launches);
int64_t allegro_launch_count(allegro_ctx* ctx); /* launches since the last allegro_profile(ctx, 1) */
/* per-shape detail entry idx (0..): name, time, algorithmic bytes, launches; ALLEGRO_E_ARG past the end */
int allegro_profile_detail(allegro_ctx* ctx, int idx, char* name, int name_cap, double* time_ms, double* bytes,
                           int64_t* launches);

/* Test hook: one GEMM C[M][N] = A[M][K] W[K][N] (row-major fp32 HOST arrays) on device
 * `device` with the given ALLEGRO_PREC_* contraction kernel (CUDA-core or tcgen05). */
int allegro_debug_gemm(int device, int precision, int64_t M, int N, int K, const float* A, const float* W, float* C);

/* Test hook: time `iters` launches of one contraction shape on device buffers (CUDA events);
 * epi = internal epilogue id; tma_store / max_stages / diag tune the tcgen05 kernel. */
/* test hook: one contraction with epilogue `epi` (csrc/gemm.cuh ids, s = 0.75); X, u may be NULL; C is the
 * old C on input (EPI_ACC) and the result on output; aux (may be NULL) receives the saved pre-activation */
int allegro_debug_gemm_epi(int device, int precision, int64_t M, int N, int K, int epi, const float* A, const float* W,
                           const float* X, const float* u, float* C, float* aux);
int allegro_debug_gemm_bench(int device, int precision, int64_t M, int N, int K, int epi, int iters, int tma_store,
                             int max_stages, int diag, double* ms_per_iter);

/* Host-only helpers (no GPU needed): this library's own derivations. */
int allegro_profile_kinds(void);
const char* allegro_profile_kind_name(int kind);
/* real W3j^{l1 l2 l3} table (l <= 2) into out[(2l1+1)(2l2+1)(2l3+1)] */
int allegro_w3j_table(int l1, int l2, int l3, double* out);
/* parameter count of the (n_layers, lmax) model with C=32, D=128 (Table 2) */
int64_t allegro_param_count(int n_layers, int lmax);
/* per-layer (#paths, #scalar paths) of (n_layers, lmax): out[2*k], out[2*k+1] */
int allegro_layer_paths(int n_layers, int lmax, int* out);
/* algorithmic forward work per edge of the (n_layers, lmax) model: out[0] =
 * dense-contraction MACs (two-body, env-embed, TP-linear of all but the last layer, latent,
 * edge-energy), out[1] = tensor-product FMAs (non-zero W3j entries x channels).  The step does
 * the forward plus the input-gradient reverse: 2x the MACs and 3x the TP FMAs. */
int allegro_work_per_edge(int n_layers, int lmax, double* out);
const char* allegro_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ALLEGRO_B200_H */
