// arch.cuh -- compile-time architecture of the Allegro model: irreps, tensor-product
// paths and real Wigner-3j tables.  This library's OWN derivation (it shares no code
// with oracle/; the test suite compares the two).
//
// PAPER.md:129-130 (§2.1): E(3)-equivariant energy built from "tensors up to rank l
// and tensor products using their irreducible representations".  Concrete reading:
// SURVEY.md §8(c) E3/E6 and reading row 7; architecture pinned by Table 2's
// parameter counts:
//   * irreps (l, p), ordered by l ascending, even before odd; SH irreps (l, (-1)^l);
//   * path (ir1 x ir2 -> ir_o) iff p1 p2 = p_o and |l1-l2| <= l_o <= l1+l2;
//   * o3_full: every reachable irrep with l <= lmax, last layer 0e only, then
//     backward pruning of irreps no later path uses; path order for o, ir1, ir2.
//
// W3j is built here from Cartesian tensors (NOT the oracle's numerical null space):
// l = 1 components are the axis vectors in the stored (y, z, x) order, l = 2
// components the symmetric traceless matrices Q_m with Y^2_m(r) = r^T Q_m r for
// the component-normalised basis.  The invariant trilinear forms
//   (0,l,l): full contraction;  (1,1,1): eps_ijk a_i b_j c_k;
//   (1,1,2) and permutations: v^T Q w;  (1,2,2) and permutations: eps_ijk v_i (Q Q')_jk;
//   (2,2,2): tr(Q Q' Q'')
// are SO(3)-invariant and non-zero, hence equal W3j up to scale (the coupling is
// multiplicity free); normalised to Frobenius norm 1 with the first non-zero entry
// (lexicographic m1, m2, m3) positive -- the convention of reading row 7.
#pragma once
#include <cstdint>

namespace allegro {

constexpr int kC = 32;     // channels (App. A)
constexpr int kD = 128;    // latent width
constexpr int kNB = 8;     // Bessel functions
constexpr int kMaxIr = 6;  // l <= 2, both parities
constexpr int kMaxPaths = 20;
constexpr int kMaxLayers = 4;

struct Irrep {
  int l = 0;
  int p = 1;
};
constexpr bool ir_eq(Irrep a, Irrep b) { return a.l == b.l && a.p == b.p; }
constexpr int ir_dim(Irrep a) { return 2 * a.l + 1; }
constexpr int iabs_c(int x) { return x < 0 ? -x : x; }
constexpr bool tp_allowed(Irrep a, Irrep b, Irrep o) {
  return a.p * b.p == o.p && iabs_c(a.l - b.l) <= o.l && o.l <= a.l + b.l;
}

struct IrList {
  int n = 0;
  Irrep v[kMaxIr] = {};
  constexpr int index(Irrep a) const {
    for (int i = 0; i < n; ++i)
      if (ir_eq(v[i], a)) return i;
    return -1;
  }
  constexpr int off(int i) const {
    int o = 0;
    for (int q = 0; q < i; ++q) o += ir_dim(v[q]);
    return o;
  }
  constexpr int dim() const { return off(n); }
  constexpr void push(Irrep a) { v[n++] = a; }
};

constexpr IrList sh_irreps(int lmax) {
  IrList s;
  for (int l = 0; l <= lmax; ++l) s.push(Irrep{l, (l % 2 == 0) ? 1 : -1});
  return s;
}
constexpr IrList all_irreps(int lmax) {
  IrList s;
  for (int l = 0; l <= lmax; ++l) {
    s.push(Irrep{l, 1});
    s.push(Irrep{l, -1});
  }
  return s;
}

struct Path {
  Irrep a, b, o;
};

struct LayerArch {
  IrList in, out, sh;
  int n_paths = 0;
  Path path[kMaxPaths] = {};
  int dim_in = 0;   // sum of in irrep dims (V per channel)
  int dim_sh = 0;   // (lmax+1)^2
  int dim_T = 0;    // sum over paths of out dims (T per channel)
  int n_s = 0;      // scalar (0e) paths
  int t_off[kMaxPaths] = {};
  int in_off[kMaxPaths] = {};
  int sh_off[kMaxPaths] = {};
  int out_idx[kMaxPaths] = {};
  int out_local[kMaxPaths] = {};
  int n_to[kMaxIr] = {};
};

constexpr LayerArch layer_arch(int n_layers, int lmax, int k) {
  const IrList sh = sh_irreps(lmax);
  const IrList all = all_irreps(lmax);
  IrList ins[kMaxLayers + 1] = {};
  IrList outs[kMaxLayers] = {};
  ins[0] = sh;
  for (int q = 0; q < n_layers; ++q) {
    IrList o;
    if (q == n_layers - 1) {
      o.push(Irrep{0, 1});
    } else {
      for (int c = 0; c < all.n; ++c) {
        bool ok = false;
        for (int a = 0; a < ins[q].n; ++a)
          for (int b = 0; b < sh.n; ++b) ok = ok || tp_allowed(ins[q].v[a], sh.v[b], all.v[c]);
        if (ok) o.push(all.v[c]);
      }
    }
    outs[q] = o;
    ins[q + 1] = o;
  }
  for (int q = n_layers - 2; q >= 0; --q) {
    IrList kept;
    for (int i = 0; i < outs[q].n; ++i) {
      bool used = false;
      for (int b = 0; b < sh.n; ++b)
        for (int o = 0; o < outs[q + 1].n; ++o) used = used || tp_allowed(outs[q].v[i], sh.v[b], outs[q + 1].v[o]);
      if (used) kept.push(outs[q].v[i]);
    }
    outs[q] = kept;
    ins[q + 1] = kept;
  }
  LayerArch A;
  A.in = ins[k];
  A.out = outs[k];
  A.sh = sh;
  A.dim_in = A.in.dim();
  A.dim_sh = sh.dim();
  for (int o = 0; o < A.out.n; ++o)
    for (int a = 0; a < A.in.n; ++a)
      for (int b = 0; b < sh.n; ++b)
        if (tp_allowed(A.in.v[a], sh.v[b], A.out.v[o])) {
          const int q = A.n_paths++;
          A.path[q] = Path{A.in.v[a], sh.v[b], A.out.v[o]};
          A.t_off[q] = A.dim_T;
          A.dim_T += ir_dim(A.out.v[o]);
          A.in_off[q] = A.in.off(a);
          A.sh_off[q] = sh.off(b);
          A.out_idx[q] = o;
          A.out_local[q] = A.n_to[o]++;
          if (A.out.v[o].l == 0 && A.out.v[o].p == 1) ++A.n_s;
        }
  return A;
}

constexpr int64_t param_count(int n_layers, int lmax) {
  const int n_env = lmax + 1;
  int64_t t = kNB;                       // Bessel frequencies
  t += 12 * 32 + 32 * 64 + 64 * 128;     // two-body MLP
  for (int k = 0; k < n_layers; ++k) {
    const LayerArch A = layer_arch(n_layers, lmax, k);
    t += (int64_t)kD * kC * n_env * (k == 0 ? 2 : 1);  // env embed
    t += (int64_t)A.n_paths * kC * kC;                 // TP-linear
    t += (int64_t)(kD + kC * A.n_s) * kD;              // latent
  }
  t += kD * 32 + 32;                     // edge energy MLP
  return t;
}

// ------------------------------------------------------------------ real W3j
constexpr double csqrt(double x) {
  if (x <= 0) return 0;
  double r = x > 1 ? x : 1;
  for (int i = 0; i < 64; ++i) {
    const double nr = 0.5 * (r + x / r);
    if (nr == r) break;
    r = nr;
  }
  return r;
}
constexpr double kH15 = csqrt(15.0) / 2;
constexpr double kH5 = csqrt(5.0) / 2;
// l = 1 basis vector m in (y, z, x) order; component i in (x, y, z)
constexpr double cvec(int m, int i) { return (m == 0 && i == 1) || (m == 1 && i == 2) || (m == 2 && i == 0) ? 1.0 : 0.0; }
// l = 2 symmetric traceless matrices, Y^2_m(r) = r^T Q_m r
constexpr double cmat(int m, int i, int j) {
  const double h15 = kH15, h5 = kH5;
  switch (m) {
    case 0: return ((i == 0 && j == 1) || (i == 1 && j == 0)) ? h15 : 0.0;
    case 1: return ((i == 1 && j == 2) || (i == 2 && j == 1)) ? h15 : 0.0;
    case 2: return i != j ? 0.0 : (i == 2 ? 2 * h5 : -h5);
    case 3: return ((i == 0 && j == 2) || (i == 2 && j == 0)) ? h15 : 0.0;
    default: return i != j ? 0.0 : (i == 0 ? h15 : (i == 1 ? -h15 : 0.0));
  }
}
constexpr double ceps(int i, int j, int k) {
  if (i == j || j == k || i == k) return 0.0;
  return ((i == 0 && j == 1) || (i == 1 && j == 2) || (i == 2 && j == 0)) ? 1.0 : -1.0;
}
constexpr double qq(int m, int n, int j, int k) {  // (Q_m Q_n)_jk
  double s = 0;
  for (int t = 0; t < 3; ++t) s += cmat(m, j, t) * cmat(n, t, k);
  return s;
}
// unnormalised invariant trilinear form
constexpr double w3j_raw(int l1, int l2, int l3, int m1, int m2, int m3) {
  const int ls[3] = {l1, l2, l3};
  const int ms[3] = {m1, m2, m3};
  int n0 = 0, n1 = 0, n2 = 0;
  for (int q = 0; q < 3; ++q) n0 += ls[q] == 0, n1 += ls[q] == 1, n2 += ls[q] == 2;
  if (n0 == 3) return 1.0;
  if (n0 == 1) {  // (0, l, l) in any order: contraction of the other two
    int a = -1, b = -1;
    for (int q = 0; q < 3; ++q)
      if (ls[q] != 0) (a < 0 ? a : b) = q;
    if (ls[a] != ls[b]) return 0.0;
    double s = 0;
    if (ls[a] == 1)
      for (int i = 0; i < 3; ++i) s += cvec(ms[a], i) * cvec(ms[b], i);
    else
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) s += cmat(ms[a], i, j) * cmat(ms[b], i, j);
    return s;
  }
  if (n1 == 3) {
    double s = 0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) s += ceps(i, j, k) * cvec(m1, i) * cvec(m2, j) * cvec(m3, k);
    return s;
  }
  if (n1 == 2 && n2 == 1) {  // v^T Q w
    int v = -1, w = -1, q2 = -1;
    for (int q = 0; q < 3; ++q) {
      if (ls[q] == 2) q2 = q;
      else (v < 0 ? v : w) = q;
    }
    double s = 0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) s += cvec(ms[v], i) * cmat(ms[q2], i, j) * cvec(ms[w], j);
    return s;
  }
  if (n1 == 1 && n2 == 2) {  // eps_ijk v_i (Q Q')_jk
    int v = -1, qa = -1, qb = -1;
    for (int q = 0; q < 3; ++q) {
      if (ls[q] == 1) v = q;
      else (qa < 0 ? qa : qb) = q;
    }
    double s = 0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) s += ceps(i, j, k) * cvec(ms[v], i) * qq(ms[qa], ms[qb], j, k);
    return s;
  }
  if (n2 == 3) {
    double s = 0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) s += cmat(m1, i, j) * cmat(m2, j, k) * cmat(m3, k, i);
    return s;
  }
  return 0.0;  // other combinations (e.g. (0,1,2)) violate the triangle rule
}

template <int N>
struct DArr {
  double v[N > 0 ? N : 1] = {};
};

// Normalised table of (l1, l2, l3), flattened (m1, m2, m3) row-major.
template <int N>
constexpr DArr<N> w3j_table(int l1, int l2, int l3) {
  const int d2 = 2 * l2 + 1, d3 = 2 * l3 + 1;
  DArr<N> t;
  double nrm = 0, first = 0;
  for (int i = 0; i < N; ++i) {
    const double r = w3j_raw(l1, l2, l3, i / (d2 * d3), (i / d3) % d2, i % d3);
    t.v[i] = (r < 1e-12 && r > -1e-12) ? 0.0 : r;
    nrm += t.v[i] * t.v[i];
    if (first == 0 && t.v[i] != 0) first = t.v[i];
  }
  const double s = (first < 0 ? -1.0 : 1.0) / csqrt(nrm);
  for (int i = 0; i < N; ++i) t.v[i] *= s;
  return t;
}

template <int L1, int L2, int L3>
struct W3j {
  static constexpr int N = (2 * L1 + 1) * (2 * L2 + 1) * (2 * L3 + 1);
  static constexpr DArr<N> t = w3j_table<N>(L1, L2, L3);
};

// host-side value (same derivation; used by the allegro_w3j_table test hook)
inline double w3j_value(int l1, int l2, int l3, int m1, int m2, int m3) {
  const int d2 = 2 * l2 + 1, d3 = 2 * l3 + 1, n = (2 * l1 + 1) * d2 * d3;
  double nrm = 0, first = 0;
  for (int i = 0; i < n; ++i) {
    double r = w3j_raw(l1, l2, l3, i / (d2 * d3), (i / d3) % d2, i % d3);
    if (r < 1e-12 && r > -1e-12) r = 0.0;
    nrm += r * r;
    if (first == 0 && r != 0) first = r;
  }
  double v = w3j_raw(l1, l2, l3, m1, m2, m3);
  if (v < 1e-12 && v > -1e-12) return 0.0;
  return (first < 0 ? -v : v) / csqrt(nrm);
}

}  // namespace allegro
