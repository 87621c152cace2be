// tc_gemm.cu -- tcgen05 tensor-core GEMM (3xTF32) with TMA-fed operands, TMEM
// accumulators and the fused epilogues of gemm.cuh.
//
// One CTA per SM walks 128-row tiles of A (persistent).  Warp roles (256 threads):
//   warp 0      TMA producer: A[128 x 32] fp32 K-blocks (SWIZZLE_128B) into a ring of
//               stages; the W image of this N-tile once (cp.async.bulk).
//   warps 2-3   split workers: a_hi = a with the low 13 mantissa bits cleared (in place),
//               a_lo = a - a_hi into the stage's lo buffer; fence.proxy.async; arrive.
//   warp 1      MMA issuer (one lane): per K-block 4 x K=8 steps of
//               tcgen05.mma.kind::tf32  D += a_hi w_lo;  D += a_lo w_hi;  D += a_hi w_hi
//               into one of two TMEM accumulators [128 lanes x N_t fp32 columns];
//               tcgen05.commit frees the stage / publishes the accumulator.
//   warps 4-7   epilogue warpgroup: tcgen05.ld 32x32b (thread = row), fused epilogue,
//               vectorised stores; releases the accumulator.
// SMEM descriptors: K-major, SWIZZLE_128B, SBO = 1024 B, version 1 (sm_100).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

#include "tc_gemm.cuh"

namespace allegro {
namespace {

constexpr int TC_THREADS = 256;
constexpr int BLK_K = 32;                    // fp32 per 128-byte K-block
constexpr int ROWS = 128;                    // UMMA M
constexpr int A_BLOCK_BYTES = ROWS * 128;    // 16 KB
constexpr int STAGE_BYTES = 2 * A_BLOCK_BYTES;
constexpr size_t SMEM_LIMIT = 227 * 1024;
constexpr size_t SMEM_RESERVE = 2048;        // barriers + alignment slack

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// K-major SWIZZLE_128B smem matrix descriptor (sm_100 "version 1")
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}

__device__ __forceinline__ float silu(float t) { return t / (1.f + __expf(-t)); }
__device__ __forceinline__ float dsilu(float t) {
  const float s = 1.f / (1.f + __expf(-t));
  return s * (1.f + t * (1.f - s));
}

struct TcParams {
  GemmArgs g;
  const float* wimg;   // this launch's N-tile image (hi | lo)
  int col0;            // first output column of the N-tile
  int N_t;             // tile width (multiple of 16)
  int nK;              // K-blocks of 32
  int nK1;             // K-blocks coming from A (rest from A2)
  int stages;
  uint32_t w_bytes;    // bytes of the W image (hi + lo)
  int n_mtiles;
};

__global__ void __launch_bounds__(TC_THREADS, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapA2, TcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  // 1024-align the dynamic smem base (SWIZZLE_128B atoms)
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  unsigned char* w_hi = base;
  unsigned char* w_lo = base + p.w_bytes / 2;
  unsigned char* stage0 = base + ((p.w_bytes + 1023) & ~1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage0 + (size_t)p.stages * STAGE_BYTES);
  uint64_t* full = bars;                    // [stages] TMA landed
  uint64_t* split = bars + p.stages;        // [stages] hi/lo written
  uint64_t* empty = bars + 2 * p.stages;    // [stages] MMAs done with the stage
  uint64_t* acc_full = bars + 3 * p.stages; // [2]
  uint64_t* acc_empty = acc_full + 2;       // [2]
  uint64_t* w_full = acc_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int acc_cols = p.N_t;
  uint32_t tmem_cols = 32;
  while (tmem_cols < 2u * acc_cols) tmem_cols <<= 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(split + s, 64);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(acc_full + a, 1);
      mbar_init(acc_empty + a, 4);
    }
    mbar_init(w_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int n_my = p.n_mtiles > (int)blockIdx.x ? (p.n_mtiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      mbar_expect_tx(w_full, p.w_bytes);
      const uint32_t chunk = 32768;
      for (uint32_t off = 0; off < p.w_bytes; off += chunk) {
        const uint32_t b = p.w_bytes - off < chunk ? p.w_bytes - off : chunk;
        bulk_load(base + off, reinterpret_cast<const unsigned char*>(p.wimg) + off, b, w_full);
      }
      int s = 0;
      uint32_t ph = 0;
      for (int t = 0; t < n_my; ++t) {
        const int m0 = ((int)blockIdx.x + t * (int)gridDim.x) * ROWS;
        for (int kb = 0; kb < p.nK; ++kb) {
          mbar_wait(empty + s, ph ^ 1);
          unsigned char* dst = stage0 + (size_t)s * STAGE_BYTES;
          mbar_expect_tx(full + s, A_BLOCK_BYTES);
          if (kb < p.nK1) tma_load_2d(dst, &mapA, kb * BLK_K, m0, full + s);
          else tma_load_2d(dst, &mapA2, (kb - p.nK1) * BLK_K, m0, full + s);
          if (++s == p.stages) s = 0, ph ^= 1;
        }
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ---------------- split workers ----------------
    const int t64 = threadIdx.x - 64;
    int s = 0;
    uint32_t ph = 0;
    for (int t = 0; t < n_my; ++t) {
      for (int kb = 0; kb < p.nK; ++kb) {
        mbar_wait(full + s, ph);
        float4* hi = reinterpret_cast<float4*>(stage0 + (size_t)s * STAGE_BYTES);
        float4* lo = reinterpret_cast<float4*>(stage0 + (size_t)s * STAGE_BYTES + A_BLOCK_BYTES);
#pragma unroll 4
        for (int i = t64; i < A_BLOCK_BYTES / 16; i += 64) {
          float4 v = hi[i];
          float4 h, l;
          h.x = __uint_as_float(__float_as_uint(v.x) & 0xffffe000u);
          h.y = __uint_as_float(__float_as_uint(v.y) & 0xffffe000u);
          h.z = __uint_as_float(__float_as_uint(v.z) & 0xffffe000u);
          h.w = __uint_as_float(__float_as_uint(v.w) & 0xffffe000u);
          l.x = v.x - h.x;
          l.y = v.y - h.y;
          l.z = v.z - h.z;
          l.w = v.w - h.w;
          hi[i] = h;
          lo[i] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(split + s);
        if (++s == p.stages) s = 0, ph ^= 1;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(p.N_t >> 3) << 17) | ((uint32_t)(ROWS >> 4) << 24);
    mbar_wait(w_full, 0);
    tc_fence_after();
    const uint32_t whi = smem_u32(w_hi), wlo = smem_u32(w_lo);
    const uint32_t wblk = (uint32_t)p.N_t * 128;  // bytes of one W K-block
    int s = 0;
    uint32_t ph = 0;
    for (int t = 0; t < n_my; ++t) {
      const int a = t & 1;
      const uint32_t aph = (t >> 1) & 1;
      mbar_wait(acc_empty + a, aph ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(a * acc_cols);
      for (int kb = 0; kb < p.nK; ++kb) {
        mbar_wait(split + s, ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t ahi = smem_u32(stage0 + (size_t)s * STAGE_BYTES);
          const uint32_t alo = ahi + A_BLOCK_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t ko = k * 32;
            const uint64_t dah = sdesc(ahi + ko), dal = sdesc(alo + ko);
            const uint64_t dwh = sdesc(whi + kb * wblk + ko), dwl = sdesc(wlo + kb * wblk + ko);
            mma_tf32(d, dah, dwl, idesc, (kb | k) ? 1u : 0u);
            mma_tf32(d, dal, dwh, idesc, 1u);
            mma_tf32(d, dah, dwh, idesc, 1u);
          }
          mma_commit(empty + s);
          if (kb == p.nK - 1) mma_commit(acc_full + a);
        }
        __syncwarp();
        if (++s == p.stages) s = 0, ph ^= 1;
      }
    }
  } else {
    // ---------------- epilogue warpgroup (warps 4..7) ----------------
    const int q = warp & 3;  // TMEM lane quarter
    const int row_in_tile = q * 32 + lane;
    const GemmArgs& g = p.g;
    for (int t = 0; t < n_my; ++t) {
      const int a = t & 1;
      const uint32_t aph = (t >> 1) & 1;
      mbar_wait(acc_full + a, aph);
      tc_fence_after();
      const int64_t r = (int64_t)((int)blockIdx.x + t * (int)gridDim.x) * ROWS + row_in_tile;
      const bool ok = r < g.M;
      const float ur = (ok && g.u != nullptr) ? g.u[r] : 1.f;
      for (int c0 = 0; c0 < p.N_t; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * acc_cols + c0), v);
        if (!ok) continue;
        const int64_t o = r * g.N + p.col0 + c0;
        float out[16];
        float xin[16];
        if (g.X != nullptr) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 x4 = reinterpret_cast<const float4*>(g.X + o)[j];
            xin[4 * j] = x4.x, xin[4 * j + 1] = x4.y, xin[4 * j + 2] = x4.z, xin[4 * j + 3] = x4.w;
          }
        }
        float cold[16];
        if (g.epi == EPI_ACC) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 c4 = reinterpret_cast<const float4*>(g.C + o)[j];
            cold[4 * j] = c4.x, cold[4 * j + 1] = c4.y, cold[4 * j + 2] = c4.z, cold[4 * j + 3] = c4.w;
          }
        }
        float aux[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float pv = g.s * v[j];
          aux[j] = pv;
          switch (g.epi) {
            case EPI_STORE: out[j] = pv; break;
            case EPI_SILU: out[j] = silu(pv); break;
            case EPI_UMUL_SAVE: out[j] = ur * pv; break;
            case EPI_RESID: out[j] = g.alpha * xin[j] + g.beta * ur * pv; break;
            case EPI_URESID: out[j] = g.alpha * xin[j] + g.beta * ur * pv; break;
            case EPI_USCALE: out[j] = g.beta * ur * pv; break;
            case EPI_ACC: out[j] = cold[j] + pv; break;
            case EPI_ADDX: out[j] = pv + xin[j]; break;
            case EPI_DSILU: out[j] = ur * pv * dsilu(xin[j]); break;
            default: out[j] = pv; break;
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          reinterpret_cast<float4*>(g.C + o)[j] = make_float4(out[4 * j], out[4 * j + 1], out[4 * j + 2], out[4 * j + 3]);
        if (g.aux != nullptr && (g.epi == EPI_SILU || g.epi == EPI_UMUL_SAVE || g.epi == EPI_RESID)) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            reinterpret_cast<float4*>(g.aux + o)[j] = make_float4(aux[4 * j], aux[4 * j + 1], aux[4 * j + 2], aux[4 * j + 3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + a);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

void get_encode() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      throw CudaError("cuTensorMapEncodeTiled unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
}

CUtensorMap make_map(const float* ptr, int64_t rows, int cols, int ld) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)(rows > 0 ? rows : 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  const cuuint32_t box[2] = {BLK_K, ROWS};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

int g_num_sms = 0;

}  // namespace

float tf32_hi(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u &= 0xffffe000u;
  float h;
  std::memcpy(&h, &u, 4);
  return h;
}

TcWeight tc_prepare_weight(const std::vector<float>& W, int K, int N, std::vector<void*>& owned) {
  TcWeight t;
  t.K = K;
  t.N = N;
  const int nK = (K + BLK_K - 1) / BLK_K;
  // widest N-tile (multiple of 16 dividing N) whose image leaves room for >= 2 stages
  const size_t budget = SMEM_LIMIT - SMEM_RESERVE - 2 * (size_t)STAGE_BYTES;
  int nt = 0;
  for (int c = std::min(N, 256); c >= 16; c -= 16)
    if (N % c == 0 && (size_t)2 * nK * c * 128 <= budget) {
      nt = c;
      break;
    }
  if (nt == 0) throw CudaError("tc_prepare_weight: no N-tile fits shared memory");
  t.N_t = nt;
  t.n_tiles = N / nt;
  t.tile_bytes = (size_t)2 * nK * nt * 128;
  std::vector<float> img(t.tile_bytes / 4 * t.n_tiles, 0.f);
  for (int tile = 0; tile < t.n_tiles; ++tile) {
    float* hi = img.data() + tile * (t.tile_bytes / 4);
    float* lo = hi + t.tile_bytes / 8;
    for (int n = 0; n < nt; ++n)
      for (int k = 0; k < nK * BLK_K; ++k) {
        const float w = k < K ? W[(size_t)k * N + tile * nt + n] : 0.f;
        const float h = tf32_hi(w);
        const int kb = k / BLK_K, kk = k % BLK_K;
        // byte offset inside the K-block: row n (128 B), 16-byte chunk swizzled by n % 8
        const size_t off = (size_t)kb * nt * 128 + (size_t)n * 128 + (size_t)(((kk / 4) ^ (n % 8)) * 16) + (kk % 4) * 4;
        hi[off / 4] = h;
        lo[off / 4] = w - h;
      }
  }
  ALG_CUDA(cudaMalloc(&t.dev, img.size() * sizeof(float)));
  ALG_CUDA(cudaMemcpy(t.dev, img.data(), img.size() * sizeof(float), cudaMemcpyHostToDevice));
  owned.push_back(t.dev);
  return t;
}

void tc_gemm(const GemmArgs& g, const TcWeight& w, cudaStream_t st, Profiler* prof) {
  if (g.M == 0) return;
  if (g.N != w.N || g.K != w.K || (g.A2 && g.K1 % BLK_K != 0))
    throw CudaError("tc_gemm: shape mismatch N=" + std::to_string(g.N) + " K=" + std::to_string(g.K));
  get_encode();
  if (g_num_sms == 0) {
    int dev;
    ALG_CUDA(cudaGetDevice(&dev));
    ALG_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int nK = (g.K + BLK_K - 1) / BLK_K;
  const int K1 = g.A2 ? g.K1 : g.K;
  const CUtensorMap mA = make_map(g.A, g.M, K1, g.lda);
  const CUtensorMap mA2 = g.A2 ? make_map(g.A2, g.M, g.K - g.K1, g.lda2) : mA;
  const size_t w_bytes = w.tile_bytes;
  const size_t w_round = (w_bytes + 1023) & ~(size_t)1023;
  int stages = (int)((SMEM_LIMIT - SMEM_RESERVE - w_round) / STAGE_BYTES);
  stages = std::max(2, std::min(stages, 4));
  const size_t smem = 1024 + w_round + (size_t)stages * STAGE_BYTES + 256;
  static bool attr_set = false;
  if (!attr_set) {
    ALG_CUDA(cudaFuncSetAttribute(k_tc_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_LIMIT));
    attr_set = true;
  }
  TcParams p;
  p.g = g;
  p.N_t = w.N_t;
  p.nK = nK;
  p.nK1 = g.A2 ? g.K1 / BLK_K : nK;
  p.stages = stages;
  p.w_bytes = (uint32_t)w_bytes;
  p.n_mtiles = (int)((g.M + ROWS - 1) / ROWS);
  const int grid = std::min(p.n_mtiles, g_num_sms);
  const double mn = (double)g.M * g.N;
  const int n_io = 1 + (g.aux != nullptr) + (g.X != nullptr) + (g.epi == EPI_ACC);
  for (int tile = 0; tile < w.n_tiles; ++tile) {
    p.col0 = tile * w.N_t;
    p.wimg = w.dev + tile * (w.tile_bytes / 4);
    ProfScope ps(prof, st, PK_GEMM, 2.0 * mn * g.K / w.n_tiles,
                 4.0 * ((double)g.M * g.K + (double)g.K * g.N + mn * n_io) / w.n_tiles);
    k_tc_gemm<<<grid, TC_THREADS, smem, st>>>(mA, mA2, p);
    ALG_LAUNCH_CHECK();
  }
}

}  // namespace allegro
