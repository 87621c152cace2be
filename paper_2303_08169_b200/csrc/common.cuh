// common.cuh -- small device/host utilities shared by the kernels of this library.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>

namespace allegro {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define ALG_CUDA(expr)                                                                      \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess)                                                                  \
      throw ::allegro::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e) + " @" + \
                                 __FILE__ + ":" + std::to_string(__LINE__));                \
  } while (0)

#define ALG_LAUNCH_CHECK() ALG_CUDA(cudaGetLastError())

// Compile-time loop: f(std::integral_constant<int, I>) for I = 0..N-1.
template <typename F, int... I>
__host__ __device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, typename F>
__host__ __device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum each of NV values over the warp; the total of value m ends in lane (m << (5 - log2 P))
// (P = NV rounded up to a power of two).  Reduce-scatter butterfly: ~P + 5 - log2 P shuffles
// instead of 5 NV.  Returns the total this lane holds and writes its value index to *m_out.
template <int NV>
__device__ __forceinline__ float warp_sum_multi(const float* in, int lane, int* m_out) {
  constexpr int P = NV <= 1 ? 1 : NV <= 2 ? 2 : NV <= 4 ? 4 : NV <= 8 ? 8 : 16;
  constexpr int LP = P == 1 ? 0 : P == 2 ? 1 : P == 4 ? 2 : P == 8 ? 3 : 4;
  float v[P];
#pragma unroll
  for (int i = 0; i < P; ++i) v[i] = i < NV ? in[i] : 0.f;
  static_for<5>([&](auto S) {
    constexpr int st = decltype(S)::value;  // stage: offset 16 >> st
    constexpr int o = 16 >> st;
    constexpr int cnt = (st < LP) ? (P >> st) : 1;
    if constexpr (cnt > 1) {
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < cnt / 2; ++i) {
        const float send = upper ? v[i] : v[i + cnt / 2];
        const float keep = upper ? v[i + cnt / 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  });
  *m_out = lane >> (5 - LP);
  return v[0];
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace allegro
