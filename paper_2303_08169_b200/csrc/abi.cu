// abi.cu -- the extern "C" boundary declared in include/allegro.h.  Argument checking,
// host <-> device marshalling and error mapping only; every step of the method runs
// in the kernels of neighbor.cu, model.cu and md.cu.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "gemm.cuh"
#include "tc_gemm.cuh"

using namespace allegro;

namespace {

thread_local std::string g_create_err;

int fail(allegro_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  else g_create_err = msg;
  return code;
}

template <typename F>
int guarded(allegro_ctx* c, F&& f) {
  try {
    return f();
  } catch (const WeightsError& e) {
    return fail(c, ALLEGRO_E_WEIGHTS, e.what());
  } catch (const GeometryError& e) {
    return fail(c, ALLEGRO_E_GEOMETRY, e.what());
  } catch (const NcclError& e) {
    return fail(c, ALLEGRO_E_NCCL, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(c, ALLEGRO_E_ARG, e.what());
  } catch (const CudaError& e) {
    const std::string m = e.what();
    return fail(c, m.rfind("OOM", 0) == 0 ? ALLEGRO_E_OOM : ALLEGRO_E_CUDA, m);
  } catch (const std::exception& e) {
    return fail(c, ALLEGRO_E_CUDA, e.what());
  } catch (...) {
    return fail(c, ALLEGRO_E_CUDA, "unknown error");
  }
}

__global__ void k_iota(int32_t* x, int64_t n) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a < n) x[a] = (int32_t)a;
}

void reserve_atoms(allegro_ctx* c, int64_t n) {
  c->pos.reserve(3 * n + 3);
  c->vel.reserve(3 * n + 3);
  c->frc.reserve(3 * n + 3);
  c->species.reserve(n + 1);
  c->gid.reserve(n + 1);
  c->e_atom.reserve(n + 1);
}

bool debug_on() {
  static const bool on = std::getenv("ALLEGRO_DEBUG") != nullptr;
  return on;
}

int evaluate(allegro_ctx* c, bool check_domain = false) {
  ALG_CUDA(cudaMemsetAsync(c->flags.p, 0, 4 * sizeof(int), c->stream));
  wrap_positions(c);
  if (!check_inputs(c)) return fail(c, ALLEGRO_E_ARG, "non-finite position or species outside {0, 1}");
  if (check_domain && c->dom.multi && !all_owned(c))
    return fail(c, ALLEGRO_E_ARG, "an atom passed to this rank lies outside its spatial domain");
  build_neighbors(c);
  compute_forces(c);
  if (debug_on())
    std::fprintf(stderr, "[allegro rank %d] n=%lld ghosts=%lld edges=%lld e_pot=%.9g max_nb=%d\n", c->dom.rank,
                 (long long)c->n, (long long)c->n_ghost, (long long)c->n_edges, c->e_pot, c->max_nb);
  if (!all_finite(c)) return fail(c, ALLEGRO_E_NONFINITE, "non-finite energy or force");
  return ALLEGRO_OK;
}

bool box_ok(const double* b) {
  for (int d = 0; d < 3; ++d)
    if (!(std::isfinite(b[d]) && b[d] > 0)) return false;
  return true;
}

}  // namespace

extern "C" {

const char* allegro_version(void) { return "allegro-b200 0.1 (sm_100a)"; }

const char* allegro_last_error(const allegro_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

int allegro_create(const allegro_params* p, allegro_ctx** out) {
  if (!out) return fail(nullptr, ALLEGRO_E_ARG, "out is NULL");
  *out = nullptr;
  if (!p || !p->weights_path) return fail(nullptr, ALLEGRO_E_ARG, "params or weights_path is NULL");
  if (!box_ok(p->box)) return fail(nullptr, ALLEGRO_E_ARG, "box must be three finite positive lengths");
  if (p->world_size < 1 || p->rank < 0 || p->rank >= p->world_size)
    return fail(nullptr, ALLEGRO_E_ARG, "rank / world_size out of range");
  if (p->precision != ALLEGRO_PREC_FP32 && p->precision != ALLEGRO_PREC_3XTF32 && p->precision != ALLEGRO_PREC_TF32)
    return fail(nullptr, ALLEGRO_E_ARG,
                "built precisions: ALLEGRO_PREC_3XTF32 (default), ALLEGRO_PREC_FP32, ALLEGRO_PREC_TF32; "
                "the bf16 modes are reserved");
  if (!(p->skin >= 0 && std::isfinite(p->skin))) return fail(nullptr, ALLEGRO_E_ARG, "skin must be >= 0");
  allegro_ctx* c = new allegro_ctx();
  c->prm = *p;
  int rc = guarded(nullptr, [&]() -> int {
    ALG_CUDA(cudaSetDevice(p->device));
    c->device = p->device;
    if (p->cuda_stream) {
      c->stream = (cudaStream_t)p->cuda_stream;
    } else {
      ALG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    load_model(c, p->weights_path);
    if (p->r_cut > 0 && std::fabs(p->r_cut - c->model.r_max) > 1e-12)
      throw WeightsError("r_cut differs from the weight file's r_max");
    c->r_cut = c->model.r_max;
    c->skin = p->skin;
    for (int d = 0; d < 3; ++d) c->box[d] = p->box[d];
    c->flags.reserve(8);
    c->red.reserve(8);
    domain_setup(c, p->nccl_unique_id);
    size_t free_b = 0, total_b = 0;
    ALG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    // per-chunk activation workspace: half the free memory, capped (ALLEGRO_WS_GB overrides the cap)
    static const size_t ws_cap = [] {
      const char* e = std::getenv("ALLEGRO_WS_GB");
      return (size_t)(e ? std::atof(e) : 80.0) << 30;  // 80 GB: two C5-size ctxs still fit one B200
    }();
    c->ws_budget_bytes = std::min<size_t>(free_b / 2, ws_cap);
    if (p->n_atoms_global > 0) reserve_atoms(c, p->n_atoms_global);
    return ALLEGRO_OK;
  });
  if (rc != ALLEGRO_OK) {
    allegro_destroy(c);
    return rc;
  }
  *out = c;
  return ALLEGRO_OK;
}

void allegro_destroy(allegro_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  free_model(c->model);
  domain_teardown(c);
  c->aspec.release();
  c->pq.release();
  c->pimd_c.release();
  c->pimd_mode.release();
  c->e_rep.release();
  c->pos.release();
  c->vel.release();
  c->frc.release();
  c->species.release();
  c->gid.release();
  c->apos.release();
  c->aowner.release();
  c->ashift.release();
  c->agid.release();
  c->gcount.release();
  c->goff.release();
  c->ccount.release();
  c->cstart.release();
  c->cslot.release();
  c->csorted.release();
  c->cpos.release();
  c->nb_count.release();
  c->nb_pad.release();
  c->row_ptr.release();
  c->nbr.release();
  c->cidx.release();
  c->rev.release();
  c->key_pad.release();
  c->key.release();
  c->g.release();
  c->gT.release();
  c->flags.release();
  c->red.release();
  c->e_atom.release();
  c->scan_tmp.release();
  for (auto& b : c->scan_lv) b.release();
  Workspace& w = c->ws;
  for (DBuf<float>* b : {&w.z, &w.a1, &w.h1, &w.a2, &w.h2, &w.m, &w.u, &w.Y, &w.xa, &w.xb, &w.T, &w.xbar_a, &w.xbar_b,
                         &w.sbar, &w.vbar_a, &w.vbar_b, &w.wbar, &w.ybar, &w.ubar, &w.zbar, &w.ab2, &w.ab1, &w.ee, &w.ebar, &w.gp, &w.dotp})
    b->release();
  for (int k = 0; k < kMaxLayers; ++k) {
    w.w[k].release();
    w.h[k].release();
    w.V[k].release();
    w.G[k].release();
  }
  c->prof.destroy();
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int allegro_compute_energy_forces(allegro_ctx* c, int64_t n, int where, const int32_t* gid, const int32_t* species,
                                  const double* pos, const double* box, double* e_total, double* e_atom, double* forces) {
  if (!c) return fail(nullptr, ALLEGRO_E_ARG, "ctx is NULL");
  if (n < 0 || !species || !pos || !e_total || !forces) return fail(c, ALLEGRO_E_ARG, "NULL argument or n < 0");
  if (where != ALLEGRO_HOST && where != ALLEGRO_DEVICE) return fail(c, ALLEGRO_E_ARG, "where must be HOST or DEVICE");
  if (box && !box_ok(box)) return fail(c, ALLEGRO_E_ARG, "box must be three finite positive lengths");
  if (c->dom.multi && !gid) return fail(c, ALLEGRO_E_ARG, "world_size > 1 needs the global ids of the owned atoms");
  if (c->dom.multi && box) return fail(c, ALLEGRO_E_ARG, "the box is fixed at create when world_size > 1");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    if (box)
      for (int d = 0; d < 3; ++d) c->box[d] = box[d];
    c->n = n;
    c->n_rep = 1, c->n_per = n;
    c->pimd_ready = false;
    reserve_atoms(c, n);
    const cudaMemcpyKind kin = where == ALLEGRO_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    const cudaMemcpyKind kout = where == ALLEGRO_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (n > 0) {
      ALG_CUDA(cudaMemcpyAsync(c->pos.p, pos, sizeof(double) * 3 * n, kin, c->stream));
      ALG_CUDA(cudaMemcpyAsync(c->species.p, species, sizeof(int32_t) * n, kin, c->stream));
      if (gid) {
        ALG_CUDA(cudaMemcpyAsync(c->gid.p, gid, sizeof(int32_t) * n, kin, c->stream));
      } else {
        {
          ProfScope ps_(&c->prof, c->stream, PK_WRAP, 0, 4.0 * n);
          k_iota<<<ceil_div(n, 256), 256, 0, c->stream>>>(c->gid.p, n);
        }
        ALG_LAUNCH_CHECK();
      }
    }
    c->md_ready = false;
    const int rc = evaluate(c, /*check_domain=*/true);
    *e_total = c->e_pot;
    if (n > 0) {
      ALG_CUDA(cudaMemcpyAsync(forces, c->frc.p, sizeof(double) * 3 * n, kout, c->stream));
      if (e_atom) ALG_CUDA(cudaMemcpyAsync(e_atom, c->e_atom.p, sizeof(double) * n, kout, c->stream));
    }
    ALG_CUDA(cudaStreamSynchronize(c->stream));
    c->prof.flush_if_large();
    return rc;
  });
}

int md_set_state(allegro_ctx* c, int64_t n, const int32_t* species, const double* pos, const double* vel) {
  if (!c) return fail(nullptr, ALLEGRO_E_ARG, "ctx is NULL");
  if (n <= 0 || !species || !pos || !vel) return fail(c, ALLEGRO_E_ARG, "NULL argument or n <= 0");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    c->n_rep = 1, c->n_per = 0;
    c->pimd_ready = false;
    if (c->dom.multi) {
      select_owned(c, n, species, pos, vel);  // this rank's domain, in gid order
    } else {
      c->n = n;
      reserve_atoms(c, n);
      ALG_CUDA(cudaMemcpyAsync(c->pos.p, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
      ALG_CUDA(cudaMemcpyAsync(c->vel.p, vel, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
      ALG_CUDA(cudaMemcpyAsync(c->species.p, species, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
      {
        ProfScope ps_(&c->prof, c->stream, PK_WRAP, 0, 4.0 * n);
        k_iota<<<ceil_div(n, 256), 256, 0, c->stream>>>(c->gid.p, n);
      }
      ALG_LAUNCH_CHECK();
    }
    c->n_global = n;
    c->md_ready = false;
    const int rc = evaluate(c);
    if (rc != ALLEGRO_OK) return rc;
    force_stats(c, &c->f_mean0, &c->f_sigma0);
    c->baseline_set = true;
    c->nvt_xi = c->nvt_eta = 0.0;
    if (c->nvt) c->nvt_Q = 3.0 * (double)c->n_global * 8.617333e-5 * c->nvt_T * c->nvt_tau * c->nvt_tau;
    c->md_ready = true;
    c->md_steps = 0;
    return ALLEGRO_OK;
  });
}

int md_get_state(allegro_ctx* c, int64_t n, double* pos, double* vel, double* forces) {
  if (!c) return fail(nullptr, ALLEGRO_E_ARG, "ctx is NULL");
  if (!c->md_ready) return fail(c, ALLEGRO_E_STATE, "md_set_state has not been called");
  if (n != c->n_global) return fail(c, ALLEGRO_E_ARG, "n differs from the state size");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    if (c->dom.multi) {
      gather_state(c, n, pos, vel, forces);
      return ALLEGRO_OK;
    }
    if (pos) ALG_CUDA(cudaMemcpyAsync(pos, c->pos.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
    if (vel) ALG_CUDA(cudaMemcpyAsync(vel, c->vel.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
    if (forces) ALG_CUDA(cudaMemcpyAsync(forces, c->frc.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaStreamSynchronize(c->stream));
    return ALLEGRO_OK;
  });
}

// Nose-Hoover thermostat over dt/2 (D23; same split as oracle/md.py nvt_half)
static void nvt_half(allegro_ctx* c, double& K, double dt) {
  const double g = 3.0 * (double)c->n_global, kT = 8.617333e-5 * c->nvt_T;
  c->nvt_xi += 0.25 * dt * (2.0 * K - g * kT) / c->nvt_Q;
  const double s = std::exp(-c->nvt_xi * 0.5 * dt);
  md_scale_velocities(c, s);
  K *= s * s;
  c->nvt_eta += c->nvt_xi * 0.5 * dt;
  c->nvt_xi += 0.25 * dt * (2.0 * K - g * kT) / c->nvt_Q;
}

static int md_run(allegro_ctx* c, int64_t n_steps, double dt, md_report* out) {
  {
    int rc = ALLEGRO_OK;
    int64_t done = 0;
    for (; done < n_steps; ++done) {
      if (c->nvt) {
        double K = md_kinetic(c);
        nvt_half(c, K, dt);
      }
      md_half_kick_drift(c, dt);
      if (c->dom.multi) migrate(c);
      ALG_CUDA(cudaMemsetAsync(c->flags.p, 0, 4 * sizeof(int), c->stream));
      build_neighbors(c);
      compute_forces(c, /*defer_e=*/true);  // e_pot arrives with the finite check below
      md_half_kick(c, dt);
      if (c->nvt) {
        double K = md_kinetic(c);
        nvt_half(c, K, dt);
      }
      if (!all_finite(c)) {
        rc = fail(c, ALLEGRO_E_NONFINITE, "non-finite energy, force or velocity at step " + std::to_string(c->md_steps + 1));
        ++done;
        ++c->md_steps;
        break;
      }
      ++c->md_steps;
      c->prof.flush_if_large();
    }
    if (out) {
      out->steps_done = done;
      out->e_pot = c->e_pot;
      out->e_kin = md_kinetic(c);
      out->e_total = out->e_pot + out->e_kin;
      out->xi = c->nvt ? c->nvt_xi : 0.0;
      out->e_conserved = out->e_total;
      if (c->nvt)
        out->e_conserved += 0.5 * c->nvt_Q * c->nvt_xi * c->nvt_xi +
                            3.0 * (double)c->n_global * 8.617333e-5 * c->nvt_T * c->nvt_eta;
      out->temperature = 2.0 * out->e_kin / (3.0 * (double)c->n_global * 8.617333e-5);
      out->n_outliers_last = count_outliers(c, c->f_mean0 + 5.0 * c->f_sigma0);
      out->n_edges = allreduce_sum_i64(c, c->n_edges);
      out->n_local = c->n;
      out->n_rebuilds = c->n_rebuilds;
    }
    c->prof.flush_if_large();
    return rc;
  }
}

int md_step(allegro_ctx* c, int64_t n_steps, double dt, md_report* out) {
  if (!c) return fail(nullptr, ALLEGRO_E_ARG, "ctx is NULL");
  if (!c->md_ready) return fail(c, ALLEGRO_E_STATE, "md_set_state has not been called");
  if (n_steps < 0 || !(dt > 0 && std::isfinite(dt))) return fail(c, ALLEGRO_E_ARG, "bad n_steps or dt");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    return md_run(c, n_steps, dt, out);
  });
}

int md_step_host(allegro_ctx* c, int64_t n, int64_t capacity, int32_t* species, double* pos, double* vel,
                 double* forces, int64_t n_steps, double dt, md_report* out) {
  if (!c) return fail(nullptr, ALLEGRO_E_ARG, "ctx is NULL");
  if (!c->md_ready) return fail(c, ALLEGRO_E_STATE, "md_set_state has not been called");
  if (n != c->n || !species || !pos || !vel || !forces) return fail(c, ALLEGRO_E_ARG, "bad arrays or n (local count)");
  if (capacity < n) return fail(c, ALLEGRO_E_ARG, "capacity < n");
  if (n_steps < 0 || !(dt > 0 && std::isfinite(dt))) return fail(c, ALLEGRO_E_ARG, "bad n_steps or dt");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    ALG_CUDA(cudaMemcpyAsync(c->species.p, species, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
    ALG_CUDA(cudaMemcpyAsync(c->pos.p, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
    ALG_CUDA(cudaMemcpyAsync(c->vel.p, vel, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
    ALG_CUDA(cudaMemcpyAsync(c->frc.p, forces, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
    const int rc = md_run(c, n_steps, dt, out);
    // multi-GPU: the local count may change by migration; the caller's arrays hold `capacity` rows
    const int64_t nn = c->n;
    if (nn > capacity) {
      ALG_CUDA(cudaStreamSynchronize(c->stream));
      return fail(c, ALLEGRO_E_ARG,
                  "local count after migration (" + std::to_string(nn) + ") exceeds capacity; the state stays on "
                  "the device (md_get_local_state)");
    }
    if (c->dom.multi) {
      ALG_CUDA(cudaMemcpyAsync(species, c->species.p, sizeof(int32_t) * nn, cudaMemcpyDeviceToHost, c->stream));
    }
    ALG_CUDA(cudaMemcpyAsync(pos, c->pos.p, sizeof(double) * 3 * nn, cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaMemcpyAsync(vel, c->vel.p, sizeof(double) * 3 * nn, cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaMemcpyAsync(forces, c->frc.p, sizeof(double) * 3 * nn, cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaStreamSynchronize(c->stream));
    return rc;
  });
}

int md_set_thermostat(allegro_ctx* c, double T_target, double tau_fs) {
  if (!c) return fail(nullptr, ALLEGRO_E_ARG, "ctx is NULL");
  if (!(std::isfinite(T_target) && std::isfinite(tau_fs)) || (tau_fs > 0 && T_target <= 0))
    return fail(c, ALLEGRO_E_ARG, "bad thermostat parameters");
  c->nvt = tau_fs > 0;
  c->nvt_T = T_target;
  c->nvt_tau = tau_fs;
  c->nvt_xi = c->nvt_eta = 0.0;
  c->nvt_Q = c->nvt ? 3.0 * (double)c->n_global * 8.617333e-5 * T_target * tau_fs * tau_fs : 0.0;
  return ALLEGRO_OK;
}

int md_run_ttf(allegro_ctx* c, double dt, const md_ttf_protocol* pr, int64_t* series, int64_t series_cap,
               md_ttf_result* out) {
  if (!c) return fail(nullptr, ALLEGRO_E_ARG, "ctx is NULL");
  if (!c->md_ready) return fail(c, ALLEGRO_E_STATE, "md_set_state has not been called");
  if (!pr || !out || !(dt > 0 && std::isfinite(dt)) || pr->nvt_steps < 0 || pr->max_nve_steps < 0 ||
      pr->check_interval < 1 || pr->outlier_interval < 1 || series_cap < 0 || (series_cap > 0 && !series) ||
      !(pr->drift_tol > 0) || (pr->nvt_steps > 0 && !(pr->T_K > 0 && pr->tau_fs > 0)))
    return fail(c, ALLEGRO_E_ARG, "bad time-to-failure protocol");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    std::memset(out, 0, sizeof(*out));
    // (1) NVT thermalisation (1,000 steps at 200 K)
    if (pr->nvt_steps > 0) {
      const int rc0 = md_set_thermostat(c, pr->T_K, pr->tau_fs);
      if (rc0 != ALLEGRO_OK) return rc0;
      const int rc = md_run(c, pr->nvt_steps, dt, nullptr);
      c->nvt = false;
      if (rc == ALLEGRO_E_NONFINITE) {  // failed before NVE started
        out->reason = ALLEGRO_TTF_NONFINITE;
        out->failed_in_nvt = 1;
        return ALLEGRO_OK;
      }
      if (rc != ALLEGRO_OK) return rc;
    }
    c->nvt = false;
    // (2) NVE until failure ("continue the simulation until it fails")
    out->e0 = c->e_pot + md_kinetic(c);
    out->e_last = out->e0;
    force_stats(c, &out->f_mean, &out->f_sigma);
    const double thr = out->f_mean + pr->outlier_k * out->f_sigma;
    c->disp_max2 = pr->disp_max > 0 ? pr->disp_max * pr->disp_max : 0.0;
    int64_t s = 1;
    int rc = ALLEGRO_OK;
    for (; s <= pr->max_nve_steps; ++s) {
      ALG_CUDA(cudaMemsetAsync(c->flags.p + 4, 0, sizeof(int), c->stream));
      rc = md_run(c, 1, dt, nullptr);
      if (rc == ALLEGRO_E_NONFINITE) {
        out->reason = ALLEGRO_TTF_NONFINITE;
        rc = ALLEGRO_OK;
        break;
      }
      if (rc != ALLEGRO_OK) break;
      int blow = 0;
      ALG_CUDA(cudaMemcpyAsync(&blow, c->flags.p + 4, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      ALG_CUDA(cudaStreamSynchronize(c->stream));
      if (allreduce_max_i32(c, blow)) {
        out->reason = ALLEGRO_TTF_DISPLACEMENT;
        break;
      }
      if (s % pr->check_interval == 0) {
        out->e_last = c->e_pot + md_kinetic(c);
        if (std::fabs(out->e_last - out->e0) > pr->drift_tol * std::fabs(out->e0)) {
          out->reason = ALLEGRO_TTF_ENERGY_DRIFT;
          break;
        }
      }
      if (s % pr->outlier_interval == 0 && out->n_series < series_cap)  // steps that did not fail
        series[out->n_series++] = count_outliers(c, thr);
    }
    c->disp_max2 = 0.0;
    out->fail_step = out->reason ? s : 0;
    out->steps_survived = out->reason ? s - 1 : pr->max_nve_steps;
    return rc;
  });
}

int allegro_compute_energy_forces_batch(allegro_ctx* c, int64_t n_rep, int64_t n_per, int where, const int32_t* species,
                                        const double* pos, double* e_rep, double* e_atom, double* forces) {
  if (!c) return fail(nullptr, ALLEGRO_E_ARG, "ctx is NULL");
  if (n_rep < 1 || n_per < 1 || !species || !pos || !e_rep || !forces)
    return fail(c, ALLEGRO_E_ARG, "NULL argument or n_rep / n_per < 1");
  if (where != ALLEGRO_HOST && where != ALLEGRO_DEVICE) return fail(c, ALLEGRO_E_ARG, "where must be HOST or DEVICE");
  if (c->dom.multi) return fail(c, ALLEGRO_E_ARG, "replica batches need world_size == 1");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    const int64_t n = n_rep * n_per;
    c->n = n;
    reserve_atoms(c, n);
    const cudaMemcpyKind kin = where == ALLEGRO_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    const cudaMemcpyKind kout = where == ALLEGRO_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    ALG_CUDA(cudaMemcpyAsync(c->pos.p, pos, sizeof(double) * 3 * n, kin, c->stream));
    ALG_CUDA(cudaMemcpyAsync(c->species.p, species, sizeof(int32_t) * n_per, kin, c->stream));
    set_replicas(c, n_rep, n_per, c->species.p);  // in place: replica 0 is the source
    c->md_ready = false;
    c->pimd_ready = false;
    const int rc = evaluate(c);
    replica_energies(c);
    ALG_CUDA(cudaMemcpyAsync(e_rep, c->e_rep.p, sizeof(double) * n_rep, kout, c->stream));
    ALG_CUDA(cudaMemcpyAsync(forces, c->frc.p, sizeof(double) * 3 * n, kout, c->stream));
    if (e_atom) ALG_CUDA(cudaMemcpyAsync(e_atom, c->e_atom.p, sizeof(double) * n, kout, c->stream));
    ALG_CUDA(cudaStreamSynchronize(c->stream));
    c->prof.flush_if_large();
    return rc;
  });
}

int pimd_set_state(allegro_ctx* c, int64_t n_beads, int64_t n_per, const int32_t* species, const double* pos,
                   const double* vel, double T_K) {
  if (!c) return fail(nullptr, ALLEGRO_E_ARG, "ctx is NULL");
  if (n_beads < 1 || n_beads > 64 || n_per < 1 || !species || !pos || !vel || !(T_K > 0 && std::isfinite(T_K)))
    return fail(c, ALLEGRO_E_ARG, "bad PIMD state (1 <= n_beads <= 64, n_per >= 1, T > 0)");
  if (c->dom.multi) return fail(c, ALLEGRO_E_ARG, "PIMD needs world_size == 1");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    const int64_t n = n_beads * n_per;
    c->n = n;
    c->n_global = n;
    reserve_atoms(c, n);
    c->pq.reserve(3 * n);
    ALG_CUDA(cudaMemcpyAsync(c->pq.p, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
    ALG_CUDA(cudaMemcpyAsync(c->pos.p, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
    ALG_CUDA(cudaMemcpyAsync(c->vel.p, vel, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
    ALG_CUDA(cudaMemcpyAsync(c->species.p, species, sizeof(int32_t) * n_per, cudaMemcpyHostToDevice, c->stream));
    set_replicas(c, n_beads, n_per, c->species.p);
    c->pimd_T = T_K;
    pimd_setup_modes(c, (int)n_beads);
    c->md_ready = false;
    c->pimd_ready = false;
    const int rc = evaluate(c);
    if (rc != ALLEGRO_OK) return rc;
    c->pimd_ready = true;
    c->pimd_steps = 0;
    return ALLEGRO_OK;
  });
}

static void pimd_fill_report(allegro_ctx* c, int64_t done, pimd_report* out) {
  out->steps_done = done;
  out->e_pot_mean = c->e_pot / (double)c->n_rep;
  out->e_kin = md_kinetic(c);
  out->e_spring = pimd_spring_energy(c);
  out->h_conserved = c->e_pot + out->e_kin + out->e_spring;
  out->temperature_beads = 2.0 * out->e_kin / (3.0 * (double)c->n * 8.617333e-5);
  out->omega_p = pimd_omega_p(c);
  out->n_edges = c->n_edges;
}

int pimd_step(allegro_ctx* c, int64_t n_steps, double dt, pimd_report* out) {
  if (!c) return fail(nullptr, ALLEGRO_E_ARG, "ctx is NULL");
  if (!c->pimd_ready) return fail(c, ALLEGRO_E_STATE, "pimd_set_state has not been called");
  if (n_steps < 0 || !(dt > 0 && std::isfinite(dt))) return fail(c, ALLEGRO_E_ARG, "bad n_steps or dt");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    int64_t done = 0;
    int rc = ALLEGRO_OK;
    for (; done < n_steps; ++done) {
      md_half_kick(c, dt);
      pimd_free_step(c, dt);
      ALG_CUDA(cudaMemcpyAsync(c->pos.p, c->pq.p, sizeof(double) * 3 * c->n, cudaMemcpyDeviceToDevice, c->stream));
      rc = evaluate(c);  // wraps the working copy; pq stays unwrapped (the springs need it)
      if (rc != ALLEGRO_OK) {
        ++done;
        break;
      }
      md_half_kick(c, dt);
      if (!all_finite(c)) {
        rc = fail(c, ALLEGRO_E_NONFINITE, "non-finite velocity at PIMD step " + std::to_string(c->pimd_steps + 1));
        ++done;
        ++c->pimd_steps;
        break;
      }
      ++c->pimd_steps;
      c->prof.flush_if_large();
    }
    if (out) pimd_fill_report(c, done, out);
    c->prof.flush_if_large();
    return rc;
  });
}

int pimd_get_state(allegro_ctx* c, double* pos, double* vel, double* forces, double* e_rep) {
  if (!c) return fail(nullptr, ALLEGRO_E_ARG, "ctx is NULL");
  if (!c->pimd_ready) return fail(c, ALLEGRO_E_STATE, "pimd_set_state has not been called");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    const int64_t n = c->n;
    if (pos) ALG_CUDA(cudaMemcpyAsync(pos, c->pq.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
    if (vel) ALG_CUDA(cudaMemcpyAsync(vel, c->vel.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
    if (forces) ALG_CUDA(cudaMemcpyAsync(forces, c->frc.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
    if (e_rep) {
      replica_energies(c);
      ALG_CUDA(cudaMemcpyAsync(e_rep, c->e_rep.p, sizeof(double) * c->n_rep, cudaMemcpyDeviceToHost, c->stream));
    }
    ALG_CUDA(cudaStreamSynchronize(c->stream));
    return ALLEGRO_OK;
  });
}

int allegro_nccl_unique_id(void* out128) {
  if (!out128) return fail(nullptr, ALLEGRO_E_ARG, "out is NULL");
  return guarded(nullptr, [&]() -> int {
    ncclUniqueId id;
    ALG_NCCL(NcclApi::get().GetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return ALLEGRO_OK;
  });
}

int64_t allegro_local_count(const allegro_ctx* c) { return c ? c->n : -1; }

int md_get_local_state(allegro_ctx* c, int64_t capacity, int64_t* n_local, int32_t* species, int32_t* gid, double* pos,
                       double* vel, double* forces) {
  if (!c || !n_local) return fail(c, ALLEGRO_E_ARG, "NULL argument");
  if (!c->md_ready) return fail(c, ALLEGRO_E_STATE, "md_set_state has not been called");
  *n_local = c->n;
  if (capacity < c->n) return fail(c, ALLEGRO_E_ARG, "capacity too small");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    const int64_t n = c->n;
    if (species) ALG_CUDA(cudaMemcpyAsync(species, c->species.p, 4 * n, cudaMemcpyDeviceToHost, c->stream));
    if (gid) ALG_CUDA(cudaMemcpyAsync(gid, c->gid.p, 4 * n, cudaMemcpyDeviceToHost, c->stream));
    if (pos) ALG_CUDA(cudaMemcpyAsync(pos, c->pos.p, 24 * n, cudaMemcpyDeviceToHost, c->stream));
    if (vel) ALG_CUDA(cudaMemcpyAsync(vel, c->vel.p, 24 * n, cudaMemcpyDeviceToHost, c->stream));
    if (forces) ALG_CUDA(cudaMemcpyAsync(forces, c->frc.p, 24 * n, cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaStreamSynchronize(c->stream));
    return ALLEGRO_OK;
  });
}

int allegro_profile(allegro_ctx* c, int enable) {
  if (!c) return fail(nullptr, ALLEGRO_E_ARG, "ctx is NULL");
  return guarded(c, [&]() -> int {
    if (!enable) {  // stop recording; the totals stay readable (no synchronisation)
      c->prof.on = false;
      return ALLEGRO_OK;
    }
    ALG_CUDA(cudaSetDevice(c->device));
    ALG_CUDA(cudaStreamSynchronize(c->stream));
    c->prof.reset();
    c->prof.on = true;
    return ALLEGRO_OK;
  });
}

int allegro_profile_read(allegro_ctx* c, int kind, double* ms, double* flops, double* bytes, int64_t* launches) {
  if (!c || kind < 0 || kind >= PK_COUNT) return fail(c, ALLEGRO_E_ARG, "bad ctx or kind");
  c->prof.flush();
  if (ms) *ms = c->prof.ms[kind];
  if (flops) *flops = c->prof.flops[kind];
  if (bytes) *bytes = c->prof.bytes[kind];
  if (launches) *launches = c->prof.count[kind];
  return ALLEGRO_OK;
}

int64_t allegro_launch_count(allegro_ctx* c) { return c ? c->prof.launches : -1; }

int allegro_profile_detail(allegro_ctx* c, int idx, char* name, int name_cap, double* time_ms, double* bytes,
                           int64_t* launches) {
  if (!c) return fail(nullptr, ALLEGRO_E_ARG, "ctx is NULL");
  c->prof.flush();
  if (idx < 0 || idx >= (int)c->prof.tags.size()) return ALLEGRO_E_ARG;
  if (name && name_cap > 0) std::snprintf(name, name_cap, "%s", c->prof.tags[idx].c_str());
  if (time_ms) *time_ms = c->prof.tag_ms[idx];
  if (bytes) *bytes = c->prof.tag_bytes[idx];
  if (launches) *launches = c->prof.tag_n[idx];
  return ALLEGRO_OK;
}

int allegro_profile_kinds(void) { return PK_COUNT; }

const char* allegro_profile_kind_name(int kind) { return prof_name(kind); }

int md_count_outliers(allegro_ctx* c, double mean, double sigma, double k, int64_t* count) {
  if (!c || !count) return fail(c, ALLEGRO_E_ARG, "NULL argument");
  if (!(std::isfinite(mean) && std::isfinite(sigma) && std::isfinite(k)))
    return fail(c, ALLEGRO_E_ARG, "non-finite threshold");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    *count = count_outliers(c, mean + k * sigma);
    return ALLEGRO_OK;
  });
}

int md_force_baseline(allegro_ctx* c, double* mean, double* sigma) {
  if (!c || !mean || !sigma) return fail(c, ALLEGRO_E_ARG, "NULL argument");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    force_stats(c, mean, sigma);
    return ALLEGRO_OK;
  });
}

int allegro_get_edges(allegro_ctx* c, int64_t capacity, int64_t* n_edges, int32_t* i_gid, int32_t* j_gid, int8_t* shift) {
  if (!c || !n_edges) return fail(c, ALLEGRO_E_ARG, "NULL argument");
  *n_edges = c->n_edges;
  if (!i_gid && !j_gid && !shift) return ALLEGRO_OK;
  if (capacity < c->n_edges) return fail(c, ALLEGRO_E_ARG, "capacity too small");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    const int64_t E = c->n_edges, na = c->n + c->n_ghost;
    std::vector<int32_t> cidx(E), nbr(E), gid(c->n), agid(na), ash(na);
    ALG_CUDA(cudaMemcpyAsync(cidx.data(), c->cidx.p, 4 * E, cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaMemcpyAsync(nbr.data(), c->nbr.p, 4 * E, cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaMemcpyAsync(gid.data(), c->gid.p, 4 * c->n, cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaMemcpyAsync(agid.data(), c->agid.p, 4 * na, cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaMemcpyAsync(ash.data(), c->ashift.p, 4 * na, cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaStreamSynchronize(c->stream));
    for (int64_t e = 0; e < E; ++e) {
      if (i_gid) i_gid[e] = gid[cidx[e]];
      if (j_gid) j_gid[e] = agid[nbr[e]];
      if (shift) {
        const int32_t s = ash[nbr[e]];
        shift[3 * e] = (int8_t)((s & 0xff) - 128);
        shift[3 * e + 1] = (int8_t)(((s >> 8) & 0xff) - 128);
        shift[3 * e + 2] = (int8_t)(((s >> 16) & 0xff) - 128);
      }
    }
    return ALLEGRO_OK;
  });
}

int allegro_get_row_edges(allegro_ctx* c, int64_t n_rows, const int64_t* rows, int64_t capacity, int64_t* n_out,
                          int32_t* i_gid, int32_t* j_gid, int8_t* shift, double* g) {
  if (!c || !n_out || (n_rows > 0 && !rows) || n_rows < 0) return fail(c, ALLEGRO_E_ARG, "NULL argument");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    const int64_t n = c->n, na = c->n + c->n_ghost;
    for (int64_t r = 0; r < n_rows; ++r)
      if (rows[r] < 0 || rows[r] >= n) return fail(c, ALLEGRO_E_ARG, "row outside the owned atoms");
    std::vector<int32_t> rp(n + 1), gid(n), agid(na), ash(na);
    ALG_CUDA(cudaMemcpyAsync(rp.data(), c->row_ptr.p, 4 * (n + 1), cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaMemcpyAsync(gid.data(), c->gid.p, 4 * n, cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaMemcpyAsync(agid.data(), c->agid.p, 4 * na, cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaMemcpyAsync(ash.data(), c->ashift.p, 4 * na, cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaStreamSynchronize(c->stream));
    int64_t tot = 0;
    for (int64_t r = 0; r < n_rows; ++r) tot += rp[rows[r] + 1] - rp[rows[r]];
    *n_out = tot;
    if (!i_gid && !j_gid && !shift && !g) return ALLEGRO_OK;
    if (capacity < tot) return fail(c, ALLEGRO_E_ARG, "capacity too small");
    int64_t o = 0;
    for (int64_t r = 0; r < n_rows; ++r) {
      const int64_t e0 = rp[rows[r]], ne = rp[rows[r] + 1] - e0;
      std::vector<int32_t> nb(ne);
      std::vector<float> gg(4 * ne);
      if (ne > 0) {
        ALG_CUDA(cudaMemcpyAsync(nb.data(), c->nbr.p + e0, 4 * ne, cudaMemcpyDeviceToHost, c->stream));
        ALG_CUDA(cudaMemcpyAsync(gg.data(), c->g.p + 4 * e0, 16 * ne, cudaMemcpyDeviceToHost, c->stream));
        ALG_CUDA(cudaStreamSynchronize(c->stream));
      }
      for (int64_t e = 0; e < ne; ++e, ++o) {
        if (i_gid) i_gid[o] = gid[rows[r]];
        if (j_gid) j_gid[o] = agid[nb[e]];
        if (shift) {
          const int32_t sh = ash[nb[e]];
          shift[3 * o] = (int8_t)((sh & 0xff) - 128);
          shift[3 * o + 1] = (int8_t)(((sh >> 8) & 0xff) - 128);
          shift[3 * o + 2] = (int8_t)(((sh >> 16) & 0xff) - 128);
        }
        if (g)
          for (int d = 0; d < 3; ++d) g[3 * o + d] = gg[4 * e + d];
      }
    }
    return ALLEGRO_OK;
  });
}

int allegro_chunk_starts(allegro_ctx* c, int64_t capacity, int64_t* n_chunks, int64_t* first_atom) {
  if (!c || !n_chunks) return fail(c, ALLEGRO_E_ARG, "NULL argument");
  *n_chunks = (int64_t)c->chunk_a0.size();
  if (!first_atom) return ALLEGRO_OK;
  if (capacity < *n_chunks) return fail(c, ALLEGRO_E_ARG, "capacity too small");
  for (size_t k = 0; k < c->chunk_a0.size(); ++k) first_atom[k] = c->chunk_a0[k];
  return ALLEGRO_OK;
}

int allegro_get_edge_grad(allegro_ctx* c, int64_t capacity, double* g) {
  if (!c || !g) return fail(c, ALLEGRO_E_ARG, "NULL argument");
  if (capacity < c->n_edges) return fail(c, ALLEGRO_E_ARG, "capacity too small");
  return guarded(c, [&]() -> int {
    ALG_CUDA(cudaSetDevice(c->device));
    std::vector<float> h(4 * c->n_edges);  // device layout [E][4]
    ALG_CUDA(cudaMemcpyAsync(h.data(), c->g.p, sizeof(float) * h.size(), cudaMemcpyDeviceToHost, c->stream));
    ALG_CUDA(cudaStreamSynchronize(c->stream));
    for (int64_t e = 0; e < c->n_edges; ++e)
      for (int d = 0; d < 3; ++d) g[e * 3 + d] = h[e * 4 + d];
    return ALLEGRO_OK;
  });
}

int allegro_debug_gemm(int device, int precision, int64_t M, int N, int K, const float* A, const float* W, float* C) {
  if (!A || !W || !C || M < 0 || N <= 0 || K <= 0) return fail(nullptr, ALLEGRO_E_ARG, "bad gemm arguments");
  return guarded(nullptr, [&]() -> int {
    ALG_CUDA(cudaSetDevice(device));
    std::vector<void*> owned;
    std::vector<float> w(W, W + (size_t)K * N);
    float *dA = nullptr, *dW = nullptr, *dC = nullptr;
    ALG_CUDA(cudaMalloc(&dA, sizeof(float) * (M * K + 4)));
    ALG_CUDA(cudaMalloc(&dW, sizeof(float) * K * N));
    ALG_CUDA(cudaMalloc(&dC, sizeof(float) * (M * N + 4)));
    ALG_CUDA(cudaMemcpy(dA, A, sizeof(float) * M * K, cudaMemcpyHostToDevice));
    ALG_CUDA(cudaMemcpy(dW, W, sizeof(float) * K * N, cudaMemcpyHostToDevice));
    GemmArgs g;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = dA;
    g.lda = K;
    g.W = dW;
    g.C = dC;
    if (tc_mode(precision)) {
      g.single_pass = precision == ALLEGRO_PREC_TF32 ? 1 : 0;
      TcWeight t = tc_prepare_weight(w, K, N, owned);
      tc_gemm(g, t, 0, nullptr);
    } else {
      gemm(g, 0, nullptr);
    }
    ALG_CUDA(cudaDeviceSynchronize());
    ALG_CUDA(cudaMemcpy(C, dC, sizeof(float) * M * N, cudaMemcpyDeviceToHost));
    cudaFree(dA);
    cudaFree(dW);
    cudaFree(dC);
    for (void* p : owned) cudaFree(p);
    return ALLEGRO_OK;
  });
}

int allegro_debug_gemm_epi(int device, int precision, int64_t M, int N, int K, int epi, const float* A, const float* W,
                           const float* X, const float* u, float* C, float* aux) {
  if (!A || !W || !C || M < 0 || N <= 0 || K <= 0 || (epi & 0xff) > EPI_DSILU)
    return fail(nullptr, ALLEGRO_E_ARG, "bad gemm arguments");
  return guarded(nullptr, [&]() -> int {
    ALG_CUDA(cudaSetDevice(device));
    std::vector<void*> owned;
    std::vector<float> w(W, W + (size_t)K * N);
    auto up = [&](const float* h, size_t n) -> float* {
      float* d = nullptr;
      ALG_CUDA(cudaMalloc(&d, sizeof(float) * (n + 4)));
      if (h) ALG_CUDA(cudaMemcpy(d, h, sizeof(float) * n, cudaMemcpyHostToDevice));
      owned.push_back(d);
      return d;
    };
    GemmArgs g;
    g.M = M;
    g.N = N;
    g.K = K;
    const int K1 = (epi >> 8) & 0xffff;  // > 0: columns [K1, K) come from a separate array (the A2 path)
    epi &= 0xff;
    if (K1 > 0) {
      std::vector<float> a1((size_t)M * K1), a2((size_t)M * (K - K1));
      for (int64_t r = 0; r < M; ++r)
        for (int k = 0; k < K; ++k)
          (k < K1 ? a1[(size_t)r * K1 + k] : a2[(size_t)r * (K - K1) + k - K1]) = A[(size_t)r * K + k];
      g.A = up(a1.data(), a1.size());
      g.lda = K1;
      g.A2 = up(a2.data(), a2.size());
      g.lda2 = K - K1;
      g.K1 = K1;
    } else {
      g.A = up(A, (size_t)M * K);
      g.lda = K;
    }
    g.W = up(W, (size_t)K * N);
    g.C = up(C, (size_t)M * N);  // old C (EPI_ACC)
    g.epi = epi;
    g.alpha = 0.5f;
    g.beta = 0.25f;
    if (X == A && K1 == N) g.X = g.A;  // the resnet case: X is the first operand itself
    else if (X) g.X = up(X, (size_t)M * N);
    if (u) g.u = up(u, (size_t)M);
    float* daux = aux ? up(nullptr, (size_t)M * N) : nullptr;
    g.aux = daux;
    g.s = 0.75f;
    if (precision == ALLEGRO_PREC_3XTF32) {
      TcWeight t = tc_prepare_weight(w, K, N, owned);
      tc_gemm(g, t, 0, nullptr);
    } else {
      gemm(g, 0, nullptr);
    }
    ALG_CUDA(cudaDeviceSynchronize());
    ALG_CUDA(cudaMemcpy(C, g.C, sizeof(float) * M * N, cudaMemcpyDeviceToHost));
    if (aux) ALG_CUDA(cudaMemcpy(aux, daux, sizeof(float) * M * N, cudaMemcpyDeviceToHost));
    for (void* p : owned) cudaFree(p);
    return ALLEGRO_OK;
  });
}

int allegro_debug_gemm_bench(int device, int precision, int64_t M, int N, int K, int epi, int iters, int tma_store,
                             int max_stages, int diag, double* ms_per_iter) {
  if (!ms_per_iter || M <= 0 || N <= 0 || K <= 0 || iters <= 0) return fail(nullptr, ALLEGRO_E_ARG, "bad arguments");
  return guarded(nullptr, [&]() -> int {
    ALG_CUDA(cudaSetDevice(device));
    std::vector<void*> owned;
    std::vector<float> w((size_t)K * N);
    for (size_t i = 0; i < w.size(); ++i) w[i] = (float)((i * 2654435761u) % 1000) / 1000.f - 0.5f;
    float *dA = nullptr, *dW = nullptr, *dC = nullptr, *dX = nullptr, *dAux = nullptr, *du = nullptr;
    ALG_CUDA(cudaMalloc(&dA, sizeof(float) * M * K));
    ALG_CUDA(cudaMalloc(&dW, sizeof(float) * K * N));
    ALG_CUDA(cudaMalloc(&dC, sizeof(float) * M * N));
    ALG_CUDA(cudaMalloc(&dX, sizeof(float) * M * N));
    ALG_CUDA(cudaMalloc(&dAux, sizeof(float) * M * N));
    ALG_CUDA(cudaMalloc(&du, sizeof(float) * M));
    ALG_CUDA(cudaMemset(dA, 0, sizeof(float) * M * K));
    ALG_CUDA(cudaMemset(dX, 0, sizeof(float) * M * N));
    ALG_CUDA(cudaMemset(du, 0, sizeof(float) * M));
    ALG_CUDA(cudaMemcpy(dW, w.data(), sizeof(float) * K * N, cudaMemcpyHostToDevice));
    GemmArgs g;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = dA;
    g.lda = K;
    g.W = dW;
    g.C = dC;
    g.epi = epi;
    if (epi == EPI_RESID || epi == EPI_SILU || epi == EPI_UMUL_SAVE) g.aux = dAux;
    if (epi == EPI_RESID || epi == EPI_URESID || epi == EPI_ADDX || epi == EPI_DSILU) g.X = dX;
    if (epi == EPI_RESID || epi == EPI_URESID || epi == EPI_UMUL_SAVE || epi == EPI_USCALE) g.u = du;
    const TcTuning saved = g_tc_tuning;
    g_tc_tuning.tma_store = tma_store;
    if (tma_store >= 2) g_tc_tuning.max_acc = tma_store;  // test hook: >= 2 sets the accumulator ring cap
    if (tma_store < 0) g_tc_tuning.stack = 0;             // test hook: < 0 disables the stacked MMAs
    g_tc_tuning.max_stages = max_stages;
    g_tc_tuning.diag = diag;
    TcWeight t;
    if (precision == ALLEGRO_PREC_3XTF32) t = tc_prepare_weight(w, K, N, owned);
    auto run = [&]() {
      if (precision == ALLEGRO_PREC_3XTF32) tc_gemm(g, t, 0, nullptr);
      else gemm(g, 0, nullptr);
    };
    run();
    ALG_CUDA(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, 0);
    for (int i = 0; i < iters; ++i) run();
    cudaEventRecord(e1, 0);
    ALG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *ms_per_iter = ms / iters;
    g_tc_tuning = saved;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (void* q : {(void*)dA, (void*)dW, (void*)dC, (void*)dX, (void*)dAux, (void*)du}) cudaFree(q);
    for (void* q : owned) cudaFree(q);
    return ALLEGRO_OK;
  });
}

int allegro_w3j_table(int l1, int l2, int l3, double* out) {
  if (!out || l1 < 0 || l2 < 0 || l3 < 0 || l1 > 2 || l2 > 2 || l3 > 2) return ALLEGRO_E_ARG;
  if (!(std::abs(l1 - l2) <= l3 && l3 <= l1 + l2)) return ALLEGRO_E_ARG;
  const int d2 = 2 * l2 + 1, d3 = 2 * l3 + 1;
  for (int a = 0; a < 2 * l1 + 1; ++a)
    for (int b = 0; b < d2; ++b)
      for (int c = 0; c < d3; ++c) out[(a * d2 + b) * d3 + c] = w3j_value(l1, l2, l3, a, b, c);
  return ALLEGRO_OK;
}

int64_t allegro_param_count(int n_layers, int lmax) {
  if (n_layers < 1 || n_layers > kMaxLayers || lmax < 0 || lmax > 2) return -1;
  return param_count(n_layers, lmax);
}

int allegro_layer_paths(int n_layers, int lmax, int* out) {
  if (!out || n_layers < 1 || n_layers > kMaxLayers || lmax < 0 || lmax > 2) return ALLEGRO_E_ARG;
  for (int k = 0; k < n_layers; ++k) {
    const LayerArch A = layer_arch(n_layers, lmax, k);
    out[2 * k] = A.n_paths;
    out[2 * k + 1] = A.n_s;
  }
  return ALLEGRO_OK;
}

int allegro_work_per_edge(int n_layers, int lmax, double* out) {
  if (!out || n_layers < 1 || n_layers > kMaxLayers || lmax < 0 || lmax > 2) return ALLEGRO_E_ARG;
  const int n_env = lmax + 1;
  double mac = 12 * 32 + 32 * 64 + 64 * 128;  // two-body MLP
  double tp = 0;
  for (int k = 0; k < n_layers; ++k) {
    const LayerArch A = layer_arch(n_layers, lmax, k);
    mac += (double)kD * kC * n_env * (k == 0 ? 2 : 1);  // env embed
    if (k < n_layers - 1)                              // TP-linear (the last layer's output is unused)
      for (int o = 0; o < A.out.n; ++o) mac += (double)ir_dim(A.out.v[o]) * A.n_to[o] * kC * kC;
    mac += (double)(kD + kC * A.n_s) * kD;              // latent update
    for (int q = 0; q < A.n_paths; ++q) {               // TP: non-zero W3j entries x channels
      const int l1 = A.path[q].a.l, l2 = A.path[q].b.l, l3 = A.path[q].o.l;
      for (int m1 = 0; m1 < 2 * l1 + 1; ++m1)
        for (int m2 = 0; m2 < 2 * l2 + 1; ++m2)
          for (int m3 = 0; m3 < 2 * l3 + 1; ++m3) tp += w3j_value(l1, l2, l3, m1, m2, m3) != 0.0 ? kC : 0;
    }
  }
  mac += kD * 32 + 32;  // edge-energy MLP
  out[0] = mac;
  out[1] = tp;
  return ALLEGRO_OK;
}

}  // extern "C"
