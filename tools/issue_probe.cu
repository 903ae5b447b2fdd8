// Cost of one MMA-issuer loop iteration as written in the GEMM / triplet kernels:
// mbarrier wait (already complete) -> tcgen05 fence -> elect -> 12 x tcgen05.mma ->
// tcgen05.commit, measured with clock64 over many iterations (single CTA), with
// variants that drop pieces of the iteration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/issue_probe tools/issue_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t kdesc(uint32_t s) {
  return static_cast<uint64_t>((s >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

template <int MODE>  // 0 full; 1 no mma; 2 no commit; 3 no fence; 4 no wait
__global__ void probe(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tb;
  if (threadIdx.x < 32) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (4u << 17) | (4u << 24);  // M=64 N=32
    const uint32_t a = su32(sm), b = su32(sm + 16384);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (MODE != 4) {
        // bar[0] phase 0 was never arrived on: wait for parity 1 returns immediately
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                su32(&bar[0]))
            : "memory");
      }
      if (MODE != 3) asm volatile("tcgen05.fence::after_thread_sync;");
      if (elect_one()) {
        if (MODE != 1) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
#pragma unroll
            for (int t = 0; t < 3; ++t) {
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                  "l"(kdesc(a + 32 * k)), "l"(kdesc(b + 32 * k)), "r"(idesc), "r"(1u));
            }
          }
        }
        if (MODE != 2)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           su32(&bar[1]))
                       : "memory");
      }
      __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

template <int MODE>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 8);
  auto k = probe<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k<<<1, 128, 70000>>>(d, 64);
  k<<<1, 128, 70000>>>(d, 256);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %.1f cycles per iteration (%s)\n", name, h / 256.0, cudaGetErrorString(e));
}

int main() {
  run<0>("full (wait+fence+12mma+commit)");
  run<1>("no mma");
  run<2>("no commit");
  run<3>("no fence");
  run<4>("no wait");
  return 0;
}
