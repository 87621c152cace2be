// scan.cu -- exclusive prefix sum of int32 counts (cell counts, ghost counts,
// neighbour counts -> CSR offsets).  Three-phase block scan, recursive over the
// block sums; deterministic.
#include "ctx.cuh"

namespace allegro {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int block_exclusive(int v, int* smem, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < kScanThreads / 32 ? smem[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kScanThreads / 32) smem[lane] = s;
  }
  __syncthreads();
  const int warp_off = wid > 0 ? smem[wid - 1] : 0;
  *total = smem[kScanThreads / 32 - 1];
  return warp_off + x - v;
}

__global__ void scan_tiles(const int32_t* __restrict__ in, int32_t* __restrict__ out, int32_t* __restrict__ sums, int64_t n) {
  __shared__ int smem[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int v[kScanItems];
  int s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? in[base + i] : 0;
    s += v[i];
  }
  int total;
  int run = block_exclusive(s, smem, &total);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (threadIdx.x == 0 && sums) sums[blockIdx.x] = total;
}

__global__ void scan_add(int32_t* __restrict__ out, const int32_t* __restrict__ offs, int64_t n) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  const int o = offs[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) out[base + i] += o;
}

__global__ void scan_total(const int32_t* in, int32_t* out, int64_t n) {
  // out[n] = out[n-1] + in[n-1]
  if (n > 0) out[n] = out[n - 1] + in[n - 1];
  else out[0] = 0;
}

// Small inputs (the halo / migration flags, cell and ghost counts of a few-thousand-atom domain) in
// ONE launch: a 1024-thread block walks the input in 4,096-element chunks with a running carry and
// also writes the total out[n].  Multi-GPU steps run ~14 scans; the three-phase scan's four
// launches each cost more than the data (0.35 ms per CP step at 4 GPUs).
constexpr int kSmallThreads = 1024;
constexpr int64_t kSmallMax = 1 << 16;

__global__ void __launch_bounds__(kSmallThreads) scan_small(const int32_t* __restrict__ in, int32_t* __restrict__ out,
                                                             int64_t n) {
  __shared__ int smem[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int carry = 0;
  for (int64_t c0 = 0; c0 < n; c0 += kSmallThreads * kScanItems) {
    const int64_t base = c0 + (int64_t)threadIdx.x * kScanItems;
    int v[kScanItems];
    int s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      v[i] = (base + i < n) ? in[base + i] : 0;
      s += v[i];
    }
    int x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) smem[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = smem[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      smem[lane] = w;
    }
    __syncthreads();
    int run = carry + (wid > 0 ? smem[wid - 1] : 0) + x - s;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      if (base + i < n) out[base + i] = run;
      run += v[i];
    }
    carry += smem[31];
    __syncthreads();  // smem is rewritten by the next chunk
  }
  if (threadIdx.x == 0) out[n] = carry;
}

void scan_rec(cudaStream_t st, const int32_t* in, int32_t* out, int64_t n, DBuf<int32_t>* tmp, int level, Profiler* prof) {
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles <= 1) {
    ProfScope ps_(prof, st, PK_SCAN, 0, 8.0 * n);
    scan_tiles<<<1, kScanThreads, 0, st>>>(in, out, nullptr, n);
    ALG_LAUNCH_CHECK();
    return;
  }
  // block sums for this level live in tmp[level]
  tmp[level].reserve(2 * tiles + 2);
  int32_t* sums = tmp[level].p;
  int32_t* offs = sums + tiles + 1;
  {
    ProfScope ps_(prof, st, PK_SCAN, 0, 8.0 * n);
    scan_tiles<<<(unsigned)tiles, kScanThreads, 0, st>>>(in, out, sums, n);
  }
  ALG_LAUNCH_CHECK();
  scan_rec(st, sums, offs, tiles, tmp, level + 1, prof);
  {
    ProfScope ps_(prof, st, PK_SCAN, 0, 8.0 * n);
    scan_add<<<(unsigned)tiles, kScanThreads, 0, st>>>(out, offs, n);
  }
  ALG_LAUNCH_CHECK();
}

}  // namespace

void exclusive_scan(allegro_ctx* c, const int32_t* in, int32_t* out, int64_t n) {
  if (n <= kSmallMax) {  // out[0..n] (total included) in one launch
    ProfScope ps_(&c->prof, c->stream, PK_SCAN, 0, 8.0 * n);
    scan_small<<<1, kSmallThreads, 0, c->stream>>>(in, out, n);
    ALG_LAUNCH_CHECK();
    return;
  }
  scan_rec(c->stream, in, out, n, c->scan_lv, 0, &c->prof);  // per-ctx scratch (one device each)
  ProfScope ps_(&c->prof, c->stream, PK_SCAN, 0, 0);
  scan_total<<<1, 1, 0, c->stream>>>(in, out, n);
  ALG_LAUNCH_CHECK();
}

}  // namespace allegro
