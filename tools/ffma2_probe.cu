// FFMA vs FFMA2 (packed fp32, sm_100a) throughput probe: 8 independent accumulator chains per
// thread, 148 x 8 CTAs of 256 threads.  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/ffma2 tools/ffma2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void scalar_k(float* out, int iters, float a, float b) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  float x = a + threadIdx.x * 1e-6f, y = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], x, y);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void packed_k(float* out, int iters, float a, float b) {
  float2 acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + 2 * i, threadIdx.x * 1e-3f + 2 * i + 1);
  const float x = a + threadIdx.x * 1e-6f;
  const float2 y = make_float2(b, b);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = __ffma2_rn(acc[i], make_float2(x, x), y);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  float* d;
  cudaMalloc(&d, blocks * threads * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    for (int which = 0; which < 2; ++which) {
      cudaEventRecord(e0);
      if (which == 0) scalar_k<<<blocks, threads>>>(d, iters, 0.999f, 1e-3f);
      else packed_k<<<blocks, threads>>>(d, iters, 0.999f, 1e-3f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fma = double(blocks) * threads * iters * 16;
      if (rep) printf("%s: %.3f ms, %.1f TFLOP/s fp32\n", which ? "FFMA2" : "FFMA ", ms, 2 * fma / ms / 1e9);
    }
  }
  return 0;
}
