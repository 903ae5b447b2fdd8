// Where does an M = 64 tcgen05.mma (cta_group::1, kind::tf32) put its accumulator
// rows in TMEM?  A[r, 0] = r + 1 (K-major SW128 in shared memory), B[n, 0] = 1 +
// 100 n, everything else 0, so D[r, n] = (r + 1)(1 + 100 n).  All 128 lanes x 8
// columns are read back and printed as "lane: values".
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/tmem_m64_probe tools/tmem_m64_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t kdesc(const void* p) {
  return static_cast<uint64_t>((su32(p) >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}
__device__ __forceinline__ int sw(int r, int k) { return (r / 8) * 256 + (r % 8) * 32 + (((k / 4) ^ (r % 8)) * 4) + (k % 4); }

template <int M>
__global__ void probe(float* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  float* sm = reinterpret_cast<float*>(raw + ((1024u - (su32(raw) & 1023u)) & 1023u));
  float* A = sm;           // M rows x 32 (one SW128 slab)
  float* B = sm + 128 * 32; // 8 rows
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) sm[i] = 0.f;
  __syncthreads();
  if (threadIdx.x < M) A[sw(threadIdx.x, 0)] = threadIdx.x + 1.f;
  if (threadIdx.x < 8) B[sw(threadIdx.x, 0)] = 1.f + 100.f * threadIdx.x;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tb;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 17) | (static_cast<uint32_t>(M >> 4) << 24);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tm), "l"(kdesc(A)), "l"(kdesc(B)), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(su32(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(tm + (static_cast<uint32_t>(w * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 8; ++i) out[(w * 32 + lane) * 8 + i] = __uint_as_float(r[i]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 8 * 4);
  for (int M : {64, 128}) {
    cudaMemset(d, 0, 128 * 8 * 4);
    auto k = M == 64 ? probe<64> : probe<128>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
    k<<<1, 128, 40 * 1024>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    float h[128 * 8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("M=%d (%s): lane -> D[row, n=0..3]\n", M, cudaGetErrorString(e));
    for (int l = 0; l < 128; ++l) {
      if (h[l * 8] != 0.f || h[l * 8 + 1] != 0.f || l % 16 == 0)
        printf("  lane %3d: %8.0f %8.0f %8.0f %8.0f\n", l, h[l * 8], h[l * 8 + 1], h[l * 8 + 2], h[l * 8 + 3]);
    }
  }
  return 0;
}
