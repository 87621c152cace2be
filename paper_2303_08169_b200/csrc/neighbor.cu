// neighbor.cu -- device neighbour machinery: wrap, periodic-image ghosts, linked-cell
// binning (counting sort), full directed CSR edge list in canonical row order, and
// the reverse-edge index used by the deterministic force gather.
//
// PAPER.md:187-189 (§2.4): "locally efficient linked-list decomposition and
// subsequent neighborlist construction to achieve the O(N) computational
// complexity" -- built on the CPU in the paper; here on the GPU.
// Edge set, inclusion rule and order: SURVEY.md §8(c) "Edges" and reading rows
// 11-14, 17:
//   E = {(i, j, n) : (i != j or n != 0), |r_j + n L - r_i| <= r_c}, full, directed,
//   multi-image; include iff d2 <= fl(r_c^2) with
//   s = fl(n L), x' = fl(x_j + s), delta = fl(x' - x_i), d2 = fl(fl(dx^2 + dy^2) + dz^2)
//   evaluated with explicit round-to-nearest intrinsics (no FMA contraction), so the
//   set is bit-identical to the oracle's for identical fp64 inputs.
//   Row order: by centre, then (gid_j, nx, ny, nz) ascending.
#include <algorithm>
#include <cmath>
#include <mutex>

#include "ctx.cuh"

namespace allegro {
namespace {

__device__ __forceinline__ int32_t pack_shift(int nx, int ny, int nz) {
  return (nx + 128) | ((ny + 128) << 8) | ((nz + 128) << 16);
}
__device__ __forceinline__ void unpack_shift(int32_t s, int& nx, int& ny, int& nz) {
  nx = (s & 0xff) - 128;
  ny = ((s >> 8) & 0xff) - 128;
  nz = ((s >> 16) & 0xff) - 128;
}
__device__ __forceinline__ unsigned long long edge_key(int32_t gid, int32_t packed) {
  int nx, ny, nz;
  unpack_shift(packed, nx, ny, nz);
  return ((unsigned long long)(uint32_t)gid << 24) | ((unsigned long long)(nx + 128) << 16) |
         ((unsigned long long)(ny + 128) << 8) | (unsigned long long)(nz + 128);
}

// x <- x - L floor(x/L); x >= L -> 0 (reading row 17); flags[1] |= bad input
__global__ void k_wrap(double* __restrict__ pos, const int32_t* __restrict__ species, int64_t n, double Lx, double Ly,
                       double Lz, int* __restrict__ flags) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  const double L[3] = {Lx, Ly, Lz};
  bool bad = species[a] < 0 || species[a] > 1;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double x = pos[a * 3 + d];
    if (!isfinite(x)) {
      bad = true;
      continue;
    }
    double y = __dsub_rn(x, __dmul_rn(L[d], floor(__ddiv_rn(x, L[d]))));
    if (y >= L[d]) y = 0.0;
    pos[a * 3 + d] = y;
  }
  if (bad) atomicOr(flags + 1, 1);
}

struct GhostGeom {
  double L[3], lo[3], hi[3];
  int m[3];
};

__device__ __forceinline__ bool image_inside(const double* x, const GhostGeom& g, int nx, int ny, int nz, double* xp) {
  const int n3[3] = {nx, ny, nz};
  bool in = true;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    xp[d] = __dadd_rn(x[d], __dmul_rn((double)n3[d], g.L[d]));
    in = in && xp[d] >= g.lo[d] && xp[d] < g.hi[d];
  }
  return in;
}

__global__ void k_ghost_count(const double* __restrict__ pos, int64_t n, GhostGeom g, int32_t* __restrict__ cnt) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  const double x[3] = {pos[a * 3], pos[a * 3 + 1], pos[a * 3 + 2]};
  int c = 0;
  double xp[3];
  for (int nz = -g.m[2]; nz <= g.m[2]; ++nz)
    for (int ny = -g.m[1]; ny <= g.m[1]; ++ny)
      for (int nx = -g.m[0]; nx <= g.m[0]; ++nx) {
        if (nx == 0 && ny == 0 && nz == 0) continue;
        c += image_inside(x, g, nx, ny, nz, xp);
      }
  cnt[a] = c;
}

__global__ void k_ghost_fill(const double* __restrict__ pos, const int32_t* __restrict__ gid,
                             const int32_t* __restrict__ spec, int64_t n, GhostGeom g, const int32_t* __restrict__ off,
                             double* __restrict__ apos, int32_t* __restrict__ aowner, int32_t* __restrict__ ashift,
                             int32_t* __restrict__ agid, int32_t* __restrict__ aspec) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  const double x[3] = {pos[a * 3], pos[a * 3 + 1], pos[a * 3 + 2]};
  apos[a * 3] = x[0];
  apos[a * 3 + 1] = x[1];
  apos[a * 3 + 2] = x[2];
  aowner[a] = (int32_t)a;
  ashift[a] = pack_shift(0, 0, 0);
  agid[a] = gid[a];
  aspec[a] = spec[a];
  int64_t o = n + off[a];
  double xp[3];
  for (int nz = -g.m[2]; nz <= g.m[2]; ++nz)
    for (int ny = -g.m[1]; ny <= g.m[1]; ++ny)
      for (int nx = -g.m[0]; nx <= g.m[0]; ++nx) {
        if (nx == 0 && ny == 0 && nz == 0) continue;
        if (!image_inside(x, g, nx, ny, nz, xp)) continue;
        apos[o * 3] = xp[0];
        apos[o * 3 + 1] = xp[1];
        apos[o * 3 + 2] = xp[2];
        aowner[o] = (int32_t)a;
        ashift[o] = pack_shift(nx, ny, nz);
        agid[o] = gid[a];
        aspec[o] = spec[a];
        ++o;
      }
}

struct CellGeom {
  double lo[3], inv[3];
  int n[3];
  // replica batches (PIMD beads, NEXT-3): atom a belongs to replica owner(a) / n_per and the
  // cells of replica r are [r * ncell_rep, (r + 1) * ncell_rep), so edges never cross
  // replicas; n_per = 0: one replica
  int64_t n_per;
  int ncell_rep;
};

__device__ __forceinline__ int64_t cell_base(const CellGeom& c, int64_t owner) {
  return c.n_per > 0 ? (owner / c.n_per) * (int64_t)c.ncell_rep : 0;
}

__device__ __forceinline__ int cell_coord(double x, const CellGeom& c, int d) {
  int q = (int)floor((x - c.lo[d]) * c.inv[d]);
  return q < 0 ? 0 : (q >= c.n[d] ? c.n[d] - 1 : q);
}

__global__ void k_cell_count(const double* __restrict__ apos, const int32_t* __restrict__ aowner, int64_t na, CellGeom cg,
                             int32_t* __restrict__ ccount, int32_t* __restrict__ cslot) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= na) return;
  const int cx = cell_coord(apos[a * 3], cg, 0), cy = cell_coord(apos[a * 3 + 1], cg, 1),
            cz = cell_coord(apos[a * 3 + 2], cg, 2);
  const int64_t c = cell_base(cg, aowner[a]) + (cz * cg.n[1] + cy) * cg.n[0] + cx;
  cslot[a] = atomicAdd(ccount + c, 1);
}

__global__ void k_cell_fill(const double* __restrict__ apos, const int32_t* __restrict__ aowner, int64_t na, CellGeom cg,
                            const int32_t* __restrict__ cstart, const int32_t* __restrict__ cslot,
                            int32_t* __restrict__ sorted, double4* __restrict__ spos) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= na) return;
  const double x = apos[a * 3], y = apos[a * 3 + 1], z = apos[a * 3 + 2];
  const int cx = cell_coord(x, cg, 0), cy = cell_coord(y, cg, 1), cz = cell_coord(z, cg, 2);
  const int64_t c = cell_base(cg, aowner[a]) + (cz * cg.n[1] + cy) * cg.n[0] + cx;
  const int t = cstart[c] + cslot[a];
  sorted[t] = (int32_t)a;
  spos[t] = make_double4(x, y, z, 0.0);  // cell-ordered copy: the edge build reads candidates contiguously
}

constexpr int kEdgeWarps = 4;

// One warp per owned centre: scan the 27 neighbouring cells, keep candidates with the
// canonical fp64 test, rank-sort the row by key out of shared memory.
__global__ void __launch_bounds__(kEdgeWarps * 32) k_edge_build(const double* __restrict__ apos, int64_t n, CellGeom cg,
                                                                 const int32_t* __restrict__ cstart,
                                                                 const int32_t* __restrict__ sorted,
                                                                 const double4* __restrict__ spos,
                                                                 const int32_t* __restrict__ ashift,
                                                                 const int32_t* __restrict__ agid, double rc2, int max_nb,
                                                                 int32_t* __restrict__ nb_count, int32_t* __restrict__ nb_pad,
                                                                 unsigned long long* __restrict__ key_pad,
                                                                 int* __restrict__ flags) {
  extern __shared__ unsigned char smem_raw[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* sk = reinterpret_cast<unsigned long long*>(smem_raw) + (size_t)wid * max_nb;
  int32_t* si = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned long long*>(smem_raw) + (size_t)kEdgeWarps * max_nb) +
                (size_t)wid * max_nb;
  const int64_t i = (int64_t)blockIdx.x * kEdgeWarps + wid;
  if (i >= n) return;
  const double xi = apos[i * 3], yi = apos[i * 3 + 1], zi = apos[i * 3 + 2];
  const int cx = cell_coord(xi, cg, 0), cy = cell_coord(yi, cg, 1), cz = cell_coord(zi, cg, 2);
  const int64_t cb = cell_base(cg, i);
  // lane l < 27 owns neighbour cell l (dz, dy, dx in -1..1, x fastest); the warp scans the
  // cells' candidate counts and then walks the concatenated candidate list 32 at a time, so the
  // loads of one pass are independent of the previous pass (no cstart -> sorted chain per cell)
  int s0 = 0, nc = 0;
  if (lane < 27) {
    const int x = cx + lane % 3 - 1, y = cy + (lane / 3) % 3 - 1, z = cz + lane / 9 - 1;
    if (x >= 0 && x < cg.n[0] && y >= 0 && y < cg.n[1] && z >= 0 && z < cg.n[2]) {
      const int64_t c = cb + (z * cg.n[1] + y) * cg.n[0] + x;
      s0 = cstart[c];
      nc = cstart[c + 1] - s0;
    }
  }
  int off = nc;  // inclusive scan of the counts
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, off, d);
    if (lane >= d) off += o;
  }
  const int total = __shfl_sync(0xffffffffu, off, 31);
  off -= nc;  // exclusive
  int cnt = 0;
  for (int k0 = 0; k0 < total; k0 += 32) {
    const int k = k0 + lane;
    // the cell holding candidate k: the last lane j with off[j] <= k (off is non-decreasing)
    int j = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int oj = __shfl_sync(0xffffffffu, off, j + step);
      if (j + step < 27 && oj <= k) j += step;
    }
    const int sj = __shfl_sync(0xffffffffu, s0, j), oj = __shfl_sync(0xffffffffu, off, j);
    bool inc = false;
    int32_t a = -1;
    if (k < total) {
      const int t = sj + (k - oj);
      a = sorted[t];
      const double4 pa = spos[t];
      const double dxv = __dsub_rn(pa.x, xi);
      const double dyv = __dsub_rn(pa.y, yi);
      const double dzv = __dsub_rn(pa.z, zi);
      const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dxv, dxv), __dmul_rn(dyv, dyv)), __dmul_rn(dzv, dzv));
      inc = (d2 <= rc2) && ((int64_t)a != i);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, inc);
    const int slot = cnt + __popc(bal & ((1u << lane) - 1u));
    if (inc && slot < max_nb) {
      sk[slot] = edge_key(agid[a], ashift[a]);
      si[slot] = a;
    }
    cnt += __popc(bal);
  }
  if (cnt > max_nb) {
    if (lane == 0) atomicMax(flags, cnt);
    cnt = max_nb;
  }
  __syncwarp();
  // rank sort by key (keys are unique per row; ties would be broken by candidate order): each
  // lane ranks four of the row's entries against all of them, reading keys as SMEM broadcasts
  for (int t0 = 0; t0 < cnt; t0 += 128) {
    unsigned long long kr[4];
    int rk[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int t = t0 + 32 * r + lane;
      kr[r] = t < cnt ? sk[t] : ~0ull;
      rk[r] = 0;
    }
    for (int m = 0; m < cnt; ++m) {
      const unsigned long long km = sk[m];
#pragma unroll
      for (int r = 0; r < 4; ++r) rk[r] += (km < kr[r]) || (km == kr[r] && m < t0 + 32 * r + lane);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int t = t0 + 32 * r + lane;
      if (t < cnt) {
        nb_pad[i * max_nb + rk[r]] = si[t];
        key_pad[i * max_nb + rk[r]] = kr[r];
      }
    }
  }
  if (lane == 0) nb_count[i] = cnt;
}

__global__ void k_edge_compact(int64_t n, int max_nb, const int32_t* __restrict__ nb_count, const int32_t* __restrict__ nb_pad,
                               const unsigned long long* __restrict__ key_pad, const int32_t* __restrict__ row_ptr,
                               int32_t* __restrict__ nbr, unsigned long long* __restrict__ key, int32_t* __restrict__ cidx) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int c = nb_count[i];
  const int64_t r = row_ptr[i];
  for (int t = lane; t < c; t += 32) {
    nbr[r + t] = nb_pad[i * max_nb + t];
    key[r + t] = key_pad[i * max_nb + t];
    cidx[r + t] = (int32_t)i;
  }
}

// rev[e] = index of (j, i, -n) in row owner(j), or -1 (measure-zero asymmetry at d == r_c)
__global__ void k_edge_rev(int64_t E, int64_t n_owned_only, const int32_t* __restrict__ cidx, const int32_t* __restrict__ nbr,
                           const int32_t* __restrict__ aowner, const int32_t* __restrict__ ashift,
                           const int32_t* __restrict__ gid, const int32_t* __restrict__ row_ptr,
                           const unsigned long long* __restrict__ key, int32_t* __restrict__ rev) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int32_t i = cidx[e], a = nbr[e];
  if (n_owned_only > 0 && a >= n_owned_only) {  // multi-GPU: ghost neighbours go through the reverse halo
    rev[e] = -1;
    return;
  }
  const int32_t o = aowner[a];
  int nx, ny, nz;
  unpack_shift(ashift[a], nx, ny, nz);
  const unsigned long long want = edge_key(gid[i], pack_shift(-nx, -ny, -nz));
  int lo = row_ptr[o], hi = row_ptr[o + 1] - 1, found = -1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const unsigned long long k = key[mid];
    if (k == want) {
      found = mid;
      break;
    }
    if (k < want) lo = mid + 1;
    else hi = mid - 1;
  }
  rev[e] = found;
}

}  // namespace

void wrap_positions(allegro_ctx* c) {
  if (c->n == 0) return;
  {
    ProfScope ps_(&c->prof, c->stream, PK_WRAP, 0, 52.0 * c->n);
    k_wrap<<<ceil_div(c->n, 256), 256, 0, c->stream>>>(c->pos.p, c->species.p, c->n, c->box[0], c->box[1], c->box[2],
                                                     c->flags.p);
  }
  ALG_LAUNCH_CHECK();
}

void build_neighbors(allegro_ctx* c) {
  cudaStream_t st = c->stream;
  const int64_t n = c->n;
  const double rc = c->r_cut + c->skin;
  // ---- ghosts: periodic images within r_c of the box (1 GPU) or the NCCL halo ----
  GhostGeom gg;
  for (int d = 0; d < 3; ++d) {
    const double L = c->box[d];
    const double margin = 1e-9 * std::max(1.0, L);
    gg.L[d] = L;
    const double lo = c->dom.multi ? c->dom.lo[d] : 0.0, hi = c->dom.multi ? c->dom.hi[d] : L;
    gg.lo[d] = lo - rc - margin;
    gg.hi[d] = hi + rc + margin;
    gg.m[d] = (int)std::ceil(rc / L) + 1;
  }
  if (c->dom.multi) {
    halo_exchange(c);
  } else {
    c->gcount.reserve(n + 1);
    c->goff.reserve(n + 1);
    {
      ProfScope ps_(&c->prof, st, PK_GHOST, 0, 28.0 * n);
      k_ghost_count<<<ceil_div(std::max<int64_t>(n, 1), 256), 256, 0, st>>>(c->pos.p, n, gg, c->gcount.p);
    }
    ALG_LAUNCH_CHECK();
    exclusive_scan(c, c->gcount.p, c->goff.p, n);
    int32_t G = 0;
    ALG_CUDA(cudaMemcpyAsync(&G, c->goff.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    ALG_CUDA(cudaStreamSynchronize(st));
    c->n_ghost = G;
    const int64_t na0 = n + G;
    c->apos.reserve(3 * na0);
    c->aowner.reserve(na0);
    c->ashift.reserve(na0);
    c->agid.reserve(na0);
    c->aspec.reserve(na0);
    {
      ProfScope ps_(&c->prof, st, PK_GHOST, 0, 24.0 * n + 44.0 * (n + G));
      k_ghost_fill<<<ceil_div(std::max<int64_t>(n, 1), 256), 256, 0, st>>>(c->pos.p, c->gid.p, c->species.p, n, gg,
                                                                           c->goff.p, c->apos.p, c->aowner.p,
                                                                           c->ashift.p, c->agid.p, c->aspec.p);
    }
    ALG_LAUNCH_CHECK();
  }
  const int64_t na = n + c->n_ghost;
  // ---- cells of edge >= rc (1 + 1e-9) over [lo, hi) ----
  CellGeom cg;
  int64_t ncells = 1;
  for (int d = 0; d < 3; ++d) {
    const double ext = gg.hi[d] - gg.lo[d];
    int nc = (int)std::floor(ext / (rc * (1.0 + 1e-9)));
    nc = std::max(1, std::min(nc, 1024));
    cg.n[d] = nc;
    cg.lo[d] = gg.lo[d];
    cg.inv[d] = nc / ext;
    c->ncell[d] = nc;
    ncells *= nc;
  }
  if (c->n_rep > 1 && c->dom.multi) throw std::invalid_argument("replica batches need world_size == 1");
  cg.n_per = c->n_rep > 1 ? c->n_per : 0;
  cg.ncell_rep = (int)ncells;
  ncells *= std::max<int64_t>(c->n_rep, 1);
  c->ccount.reserve(ncells + 1);
  c->cstart.reserve(ncells + 1);
  c->cslot.reserve(na);
  c->csorted.reserve(na);
  c->cpos.reserve(na);
  ALG_CUDA(cudaMemsetAsync(c->ccount.p, 0, sizeof(int32_t) * (ncells + 1), st));
  {
    ProfScope ps_(&c->prof, st, PK_CELL, 0, 28.0 * na);
    k_cell_count<<<ceil_div(na, 256), 256, 0, st>>>(c->apos.p, c->aowner.p, na, cg, c->ccount.p, c->cslot.p);
  }
  ALG_LAUNCH_CHECK();
  exclusive_scan(c, c->ccount.p, c->cstart.p, ncells);
  {
    ProfScope ps_(&c->prof, st, PK_CELL, 0, 68.0 * na);
    k_cell_fill<<<ceil_div(na, 256), 256, 0, st>>>(c->apos.p, c->aowner.p, na, cg, c->cstart.p, c->cslot.p,
                                                 c->csorted.p, c->cpos.p);
  }
  ALG_LAUNCH_CHECK();
  // ---- edges ----
  const double rc2 = rc * rc;
  c->nb_count.reserve(n + 1);
  c->row_ptr.reserve(n + 1);
  int32_t E = 0;
  for (;;) {
    c->nb_pad.reserve((size_t)n * c->max_nb);
    c->key_pad.reserve((size_t)n * c->max_nb);
    ALG_CUDA(cudaMemsetAsync(c->flags.p, 0, sizeof(int), st));
    const size_t smem = (size_t)kEdgeWarps * c->max_nb * (sizeof(unsigned long long) + sizeof(int32_t));
    if (smem > 48 * 1024) {  // the attribute is per device: set once to the limit (the launch passes its own size)
      int dev = 0;
      ALG_CUDA(cudaGetDevice(&dev));
      if (dev < 0 || dev >= 64) throw CudaError("device ordinal out of range");
      static bool attr[64] = {};
      static std::mutex mu;
      std::lock_guard<std::mutex> lk(mu);
      if (!attr[dev]) {
        ALG_CUDA(cudaFuncSetAttribute(k_edge_build, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr[dev] = true;
      }
    }
    if (n > 0) {
      {
        ProfScope ps_(&c->prof, st, PK_EDGE, 0, 28.0 * n);
        k_edge_build<<<ceil_div(n, kEdgeWarps), kEdgeWarps * 32, smem, st>>>(
          c->apos.p, n, cg, c->cstart.p, c->csorted.p, c->cpos.p, c->ashift.p, c->agid.p, rc2, c->max_nb, c->nb_count.p, c->nb_pad.p,
          c->key_pad.p, c->flags.p);
      }
      ALG_LAUNCH_CHECK();
    }
    // the row offsets are scanned before the overflow check so that one host read brings both
    // (a rebuild after an overflow rescans)
    exclusive_scan(c, c->nb_count.p, c->row_ptr.p, n);
    int over = 0;
    ALG_CUDA(cudaMemcpyAsync(&over, c->flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    ALG_CUDA(cudaMemcpyAsync(&E, c->row_ptr.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    ALG_CUDA(cudaStreamSynchronize(st));
    if (over <= c->max_nb) break;
    int nm = c->max_nb;
    while (nm < over) nm *= 2;
    if (nm > 4096) throw CudaError("neighbour count exceeds 4096 per atom");
    c->max_nb = nm;
  }
  c->n_edges = E;
  c->nbr.reserve(E + 1);
  c->key.reserve(E + 1);
  c->cidx.reserve(E + 1);
  c->rev.reserve(E + 1);
  c->g.reserve(4 * (size_t)E + 4);  // [E][4] (x, y, z, pad)
  c->gT.reserve(3 * (size_t)E + 4);
  if (n > 0) {
    {
      ProfScope ps_(&c->prof, st, PK_EDGE, 0, 4.0 * n);
      k_edge_compact<<<ceil_div(n * 32, 256), 256, 0, st>>>(n, c->max_nb, c->nb_count.p, c->nb_pad.p, c->key_pad.p,
                                                         c->row_ptr.p, c->nbr.p, c->key.p, c->cidx.p);
    }
    ALG_LAUNCH_CHECK();
  }
  if (E > 0) {
    {
      ProfScope ps_(&c->prof, st, PK_EDGE, 0, 16.0 * E);
      k_edge_rev<<<ceil_div(E, 256), 256, 0, st>>>(E, c->dom.multi ? n : 0, c->cidx.p, c->nbr.p, c->aowner.p,
                                                 c->ashift.p, c->gid.p, c->row_ptr.p, c->key.p, c->rev.p);
    }
    ALG_LAUNCH_CHECK();
  }
  c->n_rebuilds++;
}

}  // namespace allegro
