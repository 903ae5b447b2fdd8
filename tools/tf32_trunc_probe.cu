// Does kind::tf32 tcgen05.mma truncate or round the fp32 operand bits below the tf32
// mantissa?  A[0, 0] = 1 + 2^-11 + 2^-12 (bits below tf32 precision), B[0, 0] = 1, all
// else 0, K = 8:  D[0, 0] = 1 (truncation) or 1 + 2^-10 (round to nearest).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/tf32_trunc_probe tools/tf32_trunc_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t kdesc(const void* p) {
  return static_cast<uint64_t>((su32(p) >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

__global__ void probe(float a00, float* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  float* sm = reinterpret_cast<float*>(raw + ((1024u - (su32(raw) & 1023u)) & 1023u));
  float* A = sm;            // 128 rows x 32 (SW128 K-major; row 0 granule 0 unswizzled)
  float* B = sm + 128 * 32; // 8 rows
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 136 * 32; i += blockDim.x) sm[i] = 0.f;
  __syncthreads();
  if (threadIdx.x == 0) {
    A[0] = a00;
    B[0] = 1.f;
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
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 17) | (8u << 24);  // M=128 N=8
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tm), "l"(kdesc(A)), "l"(kdesc(B)), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(su32(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (threadIdx.x == 0) out[0] = __uint_as_float(r);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
  float* d;
  cudaMalloc(&d, 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  const float vals[4] = {1.0f + 0.00048828125f + 0.000244140625f,   // 1 + 2^-11 + 2^-12
                         1.0f + 0.000732421875f + 0.0000001192092896f, // just above
                         -(1.0f + 0.00048828125f + 0.000244140625f), 1.0f + 0.0009765625f};
  for (float a : vals) {
    probe<<<1, 128, 40 * 1024>>>(a, d);
    cudaError_t e = cudaDeviceSynchronize();
    float h;
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("A = %.10f -> D = %.10f  (trunc %.10f)  %s\n", a, h, (double)__builtin_bit_cast(float, __builtin_bit_cast(unsigned, a) & 0xffffe000u), cudaGetErrorString(e));
  }
  return 0;
}
