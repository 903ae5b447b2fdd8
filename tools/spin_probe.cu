// Does a warp slow down when the other warps of its CTA spin in mbarrier.try_wait?
// Warp 0 runs a fixed ALU + shared-store loop; warps 1..n-1 wait on a barrier that
// only completes when warp 0 is done.  Prints warp 0's cycles for several n.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/spin_probe tools/spin_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int HINT>
__global__ void probe(long long* out, int iters) {
  __shared__ __align__(8) uint64_t bar;
  __shared__ float buf[32 * 33 * 4];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    float x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      x = x * 1.0001f + 0.5f;
      buf[threadIdx.x * 33 + (i & 31)] = x;
      __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = static_cast<long long>(x);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar)) : "memory");
    }
  } else {
    if (HINT) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0, %1;\n\t@!p bra W;\n\t}" ::"r"(
              su32(&bar)),
          "r"(HINT)
          : "memory");
    } else {
      asm volatile(
          "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
              su32(&bar))
          : "memory");
    }
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  for (int threads : {32, 64, 128, 256, 448}) {
    for (int hint = 0; hint < 2; ++hint) {
      long long h[2];
      if (hint) {
        probe<1000000><<<148, threads>>>(d, 4096);
        probe<1000000><<<148, threads>>>(d, 4096);
      } else {
        probe<0><<<148, threads>>>(d, 4096);
        probe<0><<<148, threads>>>(d, 4096);
      }
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("warps %2d hint %d : %.1f cycles per iteration\n", threads / 32, hint, double(h[0]) / 4096);
    }
  }
  return 0;
}
