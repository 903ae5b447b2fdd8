// Per-launch cost of a persistent-style kernel vs its dynamic shared memory size
// and TMEM allocation (148 CTAs, back-to-back launches, CUDA-event timed).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/launch_probe tools/launch_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <bool TMEM>
__global__ void k(int* out) {
  extern __shared__ uint8_t sm[];
  __shared__ uint32_t tb;
  if (TMEM) {
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(&tb))));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
  }
  if (threadIdx.x == 0 && out == nullptr) sm[0] = 1;
}

template <bool TMEM>
void run(int smem, int threads) {
  auto f = k<TMEM>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int i = 0; i < 10; ++i) f<<<148, threads, smem>>>(reinterpret_cast<int*>(1));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 200; ++i) f<<<148, threads, smem>>>(reinterpret_cast<int*>(1));
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("smem %6d threads %3d tmem %d : %.2f us per launch (%s)\n", smem, threads, TMEM ? 1 : 0, ms * 1000 / 200,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  for (int s : {0, 100000, 200000, 232000}) {
    run<false>(s, 448);
    run<true>(s, 448);
  }
  return 0;
}
