// Throughput of warp-level mma.sync m16n8k8 tf32 (fp32 accumulate) on this GPU:
// every warp issues independent MMAs on register operands (no memory traffic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/mmasync_probe tools/mmasync_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void k(float* out, int iters) {
  uint32_t a[4], b[2];
  float c[8][4];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
  for (int j = 0; j < 8; ++j)
    for (int i = 0; i < 4; ++i) c[j][i] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
  }
  float s = 0.f;
  for (int j = 0; j < 8; ++j)
    for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  float* d;
  cudaMalloc(&d, 4);
  for (int warps : {4, 8, 16}) {
    const int iters = 4096;
    k<<<148 * 4, warps * 32>>>(d, iters);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<148 * 4, warps * 32>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * 16 * 8 * 8 * 8.0 * iters * warps * 148 * 4;
    printf("warps/CTA %2d: %.1f TFLOP/s tf32 mma.sync (%s)\n", warps, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
