// Shared helpers for the EGN sm_100a kernels: status/error plumbing and
// small device utilities.  Every ABI entry point returns 0 or a nonzero
// status and records a thread-local message readable via egn_last_error().
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/egn_b200.h"

namespace egn {

void set_error(const char* fmt, ...);

inline cudaStream_t as_stream(egn_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Check the launch that was just issued; on failure record the message.
inline int check_launch(const char* what) {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(err));
    return 1;
  }
  return 0;
}

#define EGN_REQUIRE(cond, ...)   \
  do {                           \
    if (!(cond)) {               \
      ::egn::set_error(__VA_ARGS__); \
      return 2;                  \
    }                            \
  } while (0)

inline int grid_for(int64_t n, int threads, int64_t cap = 148 * 32) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

constexpr int kNumSMs = 148;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Radial basis constants (basis.py:23-32): centres c_k = k * step with
// step = cutoff/(K-1) (np.linspace), c = [0] when K == 1; gamma = (K/cutoff)^2.
struct RbfParams {
  float gamma;
  float step;
};
inline RbfParams rbf_params(int k, double cutoff) {
  RbfParams p;
  p.gamma = static_cast<float>((k / cutoff) * (k / cutoff));
  p.step = k > 1 ? static_cast<float>(cutoff / (k - 1)) : 0.0f;
  return p;
}

}  // namespace egn
