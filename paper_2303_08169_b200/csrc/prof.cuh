// prof.cuh -- per-kernel-class launch accounting: every launch of this library goes
// through a ProfScope, which counts it and (when profiling is enabled) brackets it
// with CUDA events on the launching stream and adds the ALGORITHMIC work of that
// launch (flops / DRAM bytes the method must move).  bench.py reads
// the totals to report the live roofline of the dominant kernel.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <string>
#include <vector>

namespace allegro {

enum ProfKind : int {
  PK_WRAP = 0,
  PK_GHOST,
  PK_CELL,
  PK_EDGE,
  PK_SCAN,
  PK_GEOM,
  PK_GEMM,
  PK_TP_FWD,
  PK_TP_BWD,
  PK_ENERGY,
  PK_ROWDOT,
  PK_GEOM_BWD,
  PK_FORCE,
  PK_VERLET,
  PK_REDUCE,
  PK_HALO,
  PK_GAMMA,     // environment sums Gamma_i (fused path)
  PK_TPL_FWD,   // fused TP + TP-linear (tcgen05), forward
  PK_TPL_BWD,   // fused TP-linear^T + TP adjoint (tcgen05), backward
  PK_ENV_ADJ,   // Gamma-bar row sums + environment adjoint (fused path)
  PK_LAST,      // last layer forward + read-out + reverse, one warp per row
  PK_TWOBODY,   // fused geometry + two-body MLP (tcgen05), forward
  PK_TWOBODY_BWD,  // fused two-body MLP reverse + geometry adjoint (tcgen05)
  PK_COUNT
};

inline const char* prof_name(int k) {
  static const char* names[PK_COUNT] = {"wrap", "ghost", "cell", "edge_build", "scan", "geom", "gemm", "tp_fwd",
                                        "tp_bwd", "energy", "rowdot", "geom_bwd", "force_gather", "verlet", "reduce", "halo", "gamma", "tp_lin_fwd", "tp_lin_bwd", "env_adj", "last_layer", "twobody", "twobody_bwd"};
  return (k >= 0 && k < PK_COUNT) ? names[k] : "?";
}

struct Profiler {
  bool on = false;
  long long launches = 0;
  double ms[PK_COUNT] = {}, flops[PK_COUNT] = {}, bytes[PK_COUNT] = {};
  long long count[PK_COUNT] = {};
  struct Rec {
    int kind;
    cudaEvent_t a, b;
    double flops, bytes;
    int tag;  // index into tags (-1: none)
  };
  // optional per-shape detail (e.g. "gemm N=128 K=192 epi=3 M=..."): time, bytes, launches
  std::vector<std::string> tags;
  std::map<std::string, int> tag_id;
  std::vector<double> tag_ms, tag_bytes;
  std::vector<long long> tag_n;
  int tag_of(const std::string& t) {
    auto it = tag_id.find(t);
    if (it != tag_id.end()) return it->second;
    const int id = (int)tags.size();
    tags.push_back(t);
    tag_id[t] = id;
    tag_ms.push_back(0), tag_bytes.push_back(0), tag_n.push_back(0);
    return id;
  }
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;

  cudaEvent_t ev() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  void reset() {
    flush();
    launches = 0;
    for (int k = 0; k < PK_COUNT; ++k) ms[k] = flops[k] = bytes[k] = 0, count[k] = 0;
    tags.clear(), tag_id.clear(), tag_ms.clear(), tag_bytes.clear(), tag_n.clear();
  }
  // accumulate completed records (call after a stream synchronisation)
  void flush() {
    for (Rec& r : pending) {
      cudaEventSynchronize(r.b);
      float t = 0;
      cudaEventElapsedTime(&t, r.a, r.b);
      ms[r.kind] += t;
      flops[r.kind] += r.flops;
      bytes[r.kind] += r.bytes;
      count[r.kind] += 1;
      if (r.tag >= 0) tag_ms[r.tag] += t, tag_bytes[r.tag] += r.bytes, tag_n[r.tag] += 1;
      pool.push_back(r.a);
      pool.push_back(r.b);
    }
    pending.clear();
  }
  // the per-call paths defer the host-side reading of event pairs until the totals are read
  // (allegro_profile_read): reading ~1,000 pairs after every MD step left the GPU idle for
  // milliseconds inside the timed region of small boxes
  void flush_if_large() {
    if (pending.size() > 200000) flush();
  }
  void destroy() {
    flush();
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
    pool.clear();
  }
};

struct ProfScope {
  Profiler* p;
  cudaStream_t st;
  ProfScope(Profiler* prof, cudaStream_t s, int kind, double flops = 0, double bytes = 0, const char* tag = nullptr)
      : p(prof), st(s) {
    if (!p) return;
    ++p->launches;
    if (p->on) {
      Profiler::Rec r{kind, p->ev(), p->ev(), flops, bytes, tag ? p->tag_of(tag) : -1};
      cudaEventRecord(r.a, st);
      p->pending.push_back(r);
    }
  }
  ~ProfScope() {
    if (p && p->on) cudaEventRecord(p->pending.back().b, st);
  }
};

}  // namespace allegro
