// weights.cu -- this library's own reader of the weight file (layout: synth/weights.py;
// "the file is the contract", SURVEY.md §8(c) reading row 9) and the device-side
// fp32 weight layouts of the CUDA path.
//
// The file stores the paper's architecture (Table 2; SURVEY.md
// App. A) in fp64.  The reader re-derives every tensor shape and the parameter
// count from arch.cuh and rejects a file that disagrees (ALLEGRO_E_WEIGHTS).
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <stdexcept>

#include "ctx.cuh"

namespace allegro {

namespace {

struct HostTensor {
  std::vector<int> shape;
  std::vector<double> v;
  int rows() const { return shape.size() == 2 ? shape[0] : 1; }
  int cols() const { return shape.size() == 2 ? shape[1] : shape[0]; }
  double at(int r, int c) const { return v[(size_t)r * cols() + c]; }
};

template <typename T>
T rd(const std::vector<char>& b, size_t& off) {
  if (off + sizeof(T) > b.size()) throw WeightsError("weight file truncated");
  T x;
  std::memcpy(&x, b.data() + off, sizeof(T));
  off += sizeof(T);
  return x;
}

float* upload(DevWeights& w, const std::vector<float>& h) {
  float* d = nullptr;
  ALG_CUDA(cudaMalloc(&d, h.size() * sizeof(float)));
  ALG_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
  w.owned.push_back(d);
  return d;
}

Wt make_wt(DevWeights& w, const std::vector<float>& h, int K, int N, bool tc) {
  Wt t;
  t.K = K;
  t.N = N;
  t.f = upload(w, h);
  if (tc) t.tc = tc_prepare_weight(h, K, N, w.owned);
  return t;
}

std::vector<float> transpose(const std::vector<float>& a, int rows, int cols) {
  std::vector<float> t((size_t)rows * cols);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) t[(size_t)c * rows + r] = a[(size_t)r * cols + c];
  return t;
}

}  // namespace

void free_model(Model& m) {
  for (void* p : m.w.owned) cudaFree(p);
  m.w.owned.clear();
}

void load_model(allegro_ctx* c, const char* path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw WeightsError(std::string("cannot open weight file ") + (path ? path : "(null)"));
  std::vector<char> b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  size_t off = 0;
  if (b.size() < 8 || std::memcmp(b.data(), "ALGW", 4) != 0) throw WeightsError("bad magic");
  off = 4;
  if (rd<int32_t>(b, off) != 1) throw WeightsError("unsupported weight-file version");
  int32_t hdr[12];
  for (int i = 0; i < 12; ++i) hdr[i] = rd<int32_t>(b, off);
  const int L = hdr[0], lmax = hdr[1], C = hdr[2], D = hdr[3], nb = hdr[4], ns = hdr[5], p = hdr[6];
  const int t0 = hdr[7], t1 = hdr[8], t2 = hdr[9], eh = hdr[10], nt = hdr[11];
  double dh[6];
  for (int i = 0; i < 6; ++i) dh[i] = rd<double>(b, off);
  const bool supported = (L == 2 && (lmax == 1 || lmax == 2)) || (L == 3 && lmax >= 0 && lmax <= 2);
  if (!supported) throw WeightsError("unsupported (n_layers, lmax) = (" + std::to_string(L) + ", " + std::to_string(lmax) + ")");
  if (C != kC || D != kD || nb != kNB || ns != 2 || p != 6 || t0 != 32 || t1 != 64 || t2 != 128 || eh != 32)
    throw WeightsError("weight-file widths differ from the architecture this library implements (App. A)");
  std::map<std::string, HostTensor> T;
  int64_t total = 0;
  for (int q = 0; q < nt; ++q) {
    if (off + 32 > b.size()) throw WeightsError("weight file truncated");
    std::string name(b.data() + off, strnlen(b.data() + off, 32));
    off += 32;
    HostTensor t;
    const int nd = rd<int32_t>(b, off);
    if (nd < 1 || nd > 2) throw WeightsError("bad tensor rank");
    size_t cnt = 1;
    for (int i = 0; i < nd; ++i) {
      t.shape.push_back(rd<int32_t>(b, off));
      cnt *= (size_t)t.shape.back();
    }
    t.v.resize(cnt);
    if (off + cnt * 8 > b.size()) throw WeightsError("weight file truncated");
    std::memcpy(t.v.data(), b.data() + off, cnt * 8);
    off += cnt * 8;
    total += (int64_t)cnt;
    T[name] = std::move(t);
  }
  if (total != param_count(L, lmax)) throw WeightsError("parameter count differs from Table 2 derivation");
  auto need = [&](const std::string& n, int r, int cc) -> const HostTensor& {
    auto it = T.find(n);
    if (it == T.end()) throw WeightsError("missing tensor " + n);
    const HostTensor& t = it->second;
    if (t.rows() != r || t.cols() != cc) throw WeightsError("tensor " + n + " has the wrong shape");
    return t;
  };

  Model& M = c->model;
  free_model(M);
  M.precision = c->prm.precision;
  M.n_layers = L;
  M.lmax = lmax;
  M.r_max = dh[0];
  M.nbar = dh[1];
  M.sigma[0] = dh[2];
  M.sigma[1] = dh[3];
  M.mu[0] = dh[4];
  M.mu[1] = dh[5];
  const int n_env = lmax + 1;
  DevWeights& W = M.w;
  const bool tc = tc_mode(M.precision);

  const HostTensor& bf = need("bessel_freq", 1, kNB);
  for (int i = 0; i < kNB; ++i) W.bessel[i] = (float)bf.v[i];
  // two-body: W0 padded to 16 input rows (z is padded to 16 on device)
  {
    const HostTensor& w0 = need("tb_w0", 12, 32);
    std::vector<float> h(16 * 32, 0.f);
    for (int r = 0; r < 12; ++r)
      for (int q = 0; q < 32; ++q) h[r * 32 + q] = (float)w0.at(r, q);
    W.tb_w0 = make_wt(W, h, 16, 32, tc);
    W.tb_w0T = make_wt(W, transpose(h, 16, 32), 32, 16, tc);
    const HostTensor& w1 = need("tb_w1", 32, 64);
    std::vector<float> h1(w1.v.begin(), w1.v.end());
    W.tb_w1 = make_wt(W, h1, 32, 64, tc);
    W.tb_w1T = make_wt(W, transpose(h1, 32, 64), 64, 32, tc);
    const HostTensor& w2 = need("tb_w2", 64, 128);
    std::vector<float> h2(w2.v.begin(), w2.v.end());
    W.tb_w2 = make_wt(W, h2, 64, 128, tc);
    W.tb_w2T = make_wt(W, transpose(h2, 64, 128), 128, 64, tc);
  }
  for (int k = 0; k < L; ++k) {
    LayerInfo& li = M.L[k];
    li.A = layer_arch(L, lmax, k);
    const LayerArch& A = li.A;
    li.nw = C * n_env * (k == 0 ? 2 : 1);
    li.fan_lat = D + C * A.n_s;
    // env: file columns [chunk][c][l] -> device [chunk][l][c]
    const HostTensor& we = need("env_" + std::to_string(k), D, li.nw);
    std::vector<float> h((size_t)D * li.nw);
    const int n_chunk = k == 0 ? 2 : 1;
    for (int r = 0; r < D; ++r)
      for (int ch = 0; ch < n_chunk; ++ch)
        for (int cc = 0; cc < C; ++cc)
          for (int l = 0; l < n_env; ++l)
            h[(size_t)r * li.nw + ch * C * n_env + l * C + cc] = (float)we.at(r, ch * C * n_env + cc * n_env + l);
    W.env[k] = make_wt(W, h, D, li.nw, tc);
    W.envT[k] = make_wt(W, transpose(h, D, li.nw), li.nw, D, tc);
    // TP-linear per out irrep: rows (path_local, c)
    int np_found = 0;
    while (T.count("tplin_" + std::to_string(k) + "_" + std::to_string(np_found))) ++np_found;
    if (np_found != A.n_paths) throw WeightsError("layer " + std::to_string(k) + ": TP-linear count differs from the derived paths");
    int tb = 0;
    for (int o = 0; o < A.out.n; ++o) {
      li.t_base[o] = tb;
      tb += ir_dim(A.out.v[o]) * A.n_to[o] * C;
      std::vector<float> lw((size_t)A.n_to[o] * C * C);
      for (int q = 0; q < A.n_paths; ++q) {
        if (A.out_idx[q] != o) continue;
        const HostTensor& wp = need("tplin_" + std::to_string(k) + "_" + std::to_string(q), C, C);
        for (int cc = 0; cc < C; ++cc)
          for (int v = 0; v < C; ++v) lw[((size_t)A.out_local[q] * C + cc) * C + v] = (float)wp.at(cc, v);
      }
      W.lin[k][o] = make_wt(W, lw, A.n_to[o] * C, C, tc);
      W.linT[k][o] = make_wt(W, transpose(lw, A.n_to[o] * C, C), C, A.n_to[o] * C, tc);
    }
    li.tp_nnz = 0;
    for (int q = 0; q < A.n_paths; ++q) {
      const int l1 = A.path[q].a.l, l2 = A.path[q].b.l, l3 = A.path[q].o.l;
      for (int a = 0; a < 2 * l1 + 1; ++a)
        for (int b2 = 0; b2 < 2 * l2 + 1; ++b2)
          for (int c3 = 0; c3 < 2 * l3 + 1; ++c3) li.tp_nnz += w3j_value(l1, l2, l3, a, b2, c3) != 0.0;
    }
    int vb = 0;
    for (int i = 0; i < A.in.n; ++i) {
      li.v_base[i] = vb;
      vb += ir_dim(A.in.v[i]) * C;
    }
    // latent: scalar rows file (c*n_s + q) -> device (q*C + c)
    const HostTensor& wl = need("lat_" + std::to_string(k), li.fan_lat, D);
    std::vector<float> hl((size_t)li.fan_lat * D);
    for (int r = 0; r < D; ++r)
      for (int q = 0; q < D; ++q) hl[(size_t)r * D + q] = (float)wl.at(r, q);
    for (int cc = 0; cc < C; ++cc)
      for (int s = 0; s < A.n_s; ++s)
        for (int q = 0; q < D; ++q) hl[(size_t)(D + s * C + cc) * D + q] = (float)wl.at(D + cc * A.n_s + s, q);
    W.lat[k] = make_wt(W, hl, li.fan_lat, D, tc);
    std::vector<float> hx(hl.begin(), hl.begin() + (size_t)D * D);
    std::vector<float> hs(hl.begin() + (size_t)D * D, hl.end());
    W.latT_x[k] = make_wt(W, transpose(hx, D, D), D, D, tc);
    {  // [latT_x; envT] stacked along K: x-bar^k = a x-bar^{k+1} + [b u x-bar^{k+1} / sqrt(fan) | w-bar / sqrt(D)] W
      std::vector<float> st = transpose(hx, D, D);
      const std::vector<float> et = transpose(h, D, li.nw);
      st.insert(st.end(), et.begin(), et.end());
      W.latenvT[k] = make_wt(W, st, D + li.nw, D, tc);
    }
    W.latT_s[k] = make_wt(W, transpose(hs, C * A.n_s, D), D, C * A.n_s, tc);
  }
  {
    const HostTensor& o1 = need("out_w1", D, 32);
    const HostTensor& o2 = need("out_w2", 32, 1);
    std::vector<float> wo(D);
    for (int r = 0; r < D; ++r) {
      double s = 0;
      for (int q = 0; q < 32; ++q) s += o1.at(r, q) * o2.at(q, 0);
      wo[r] = (float)(s / (std::sqrt(128.0) * std::sqrt(32.0)));
    }
    W.wout = upload(W, wo);
    // q = W_lat(L-1) w_out in the device row order of lat (x rows, then scalar rows (q, c))
    const LayerInfo& last = M.L[L - 1];
    const HostTensor& wl = need("lat_" + std::to_string(L - 1), last.fan_lat, D);
    std::vector<double> wod(D);
    for (int r = 0; r < D; ++r) {
      double s = 0;
      for (int q = 0; q < 32; ++q) s += o1.at(r, q) * o2.at(q, 0);
      wod[r] = s / (std::sqrt(128.0) * std::sqrt(32.0));
    }
    std::vector<float> q(last.fan_lat);
    auto qrow = [&](int file_row) {
      double s = 0;
      for (int v = 0; v < D; ++v) s += wl.at(file_row, v) * wod[v];
      return s;
    };
    for (int r = 0; r < D; ++r) q[r] = (float)qrow(r);
    for (int cc = 0; cc < C; ++cc)
      for (int s2 = 0; s2 < last.A.n_s; ++s2) q[D + s2 * C + cc] = (float)qrow(D + cc * last.A.n_s + s2);
    W.q_last = upload(W, q);
    const double a = 2.0 / std::sqrt(5.0), b = 1.0 / std::sqrt(5.0), sf = b / std::sqrt((double)last.fan_lat);
    std::vector<float> v1(D), v2(D);
    for (int r = 0; r < D; ++r) {
      v1[r] = (float)(a * wod[r]);
      v2[r] = (float)(sf * qrow(r));
    }
    W.r2_vec1 = upload(W, v1);
    W.r2_vec2 = upload(W, v2);
  }
}

}  // namespace allegro
