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

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace allegro
