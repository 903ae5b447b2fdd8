// Microbenchmark: cycles per tcgen05.mma (M = 128, cta_group::1) for the operand
// kinds/sources the GEMM can use.  Single CTA; thread 0 issues R back-to-back MMAs
// into one accumulator, commits, waits, reads clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/mma_probe tools/mma_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t kdesc(const void* p) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((su32(p) >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__device__ __forceinline__ uint64_t mndesc(const void* p) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((su32(p) >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(4096 >> 4) << 16;
  d |= static_cast<uint64_t>(512 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(1) << 61;
  return d;
}

// mode 0: tf32 A,B smem; 1: tf32 A TMEM; 2: bf16 A,B smem; 3: bf16 A TMEM; 4: tf32 A TMEM, B MN-major;
// 5: tf32 SS, B MN-major; 6: tf32 A TMEM, K-major B with per-step descriptor advance
template <int MODE, int N, int LOAD>
__global__ void probe(long long* out, int reps, int distinct_d) {
  __shared__ volatile int stop;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  uint8_t* base = sm + ((1024u - (su32(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 1.0f + 0.001f * (i % 977);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (LOAD && threadIdx.x >= 32) {
    const int w = threadIdx.x >> 5;
    float4* buf = reinterpret_cast<float4*>(base + 40960 + (w - 1) * 4096);
    float acc = 0.f;
    long long n = 0;
    while (!stop) {
      if (LOAD == 3) {
        // spin on an mbarrier phase that never completes (like idle role warps)
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(su32(&bar2)) : "memory");
        if (ok) acc += 1.f;
      } else if (LOAD == 1) {
#pragma unroll 8
        for (int i = 0; i < 64; ++i) {
          float4 v = buf[(threadIdx.x & 31) + (i & 7) * 32];
          acc += v.x;
          buf[(threadIdx.x & 31) + ((i + 3) & 7) * 32] = make_float4(acc, acc, acc, acc);
        }
      } else {
        const uint32_t ta = tm + 384 + (static_cast<uint32_t>(w * 32) << 16);
        uint32_t r = __float_as_uint(acc);
#pragma unroll 4
        for (int i = 0; i < 16; ++i)
          asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(ta + (i & 3) * 16), "r"(r) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      ++n;
    }
    if (acc == 12345.f) out[2] = n;
  }
  if (threadIdx.x == 0) {
    const bool tf = MODE < 2 || MODE >= 4;
    const uint32_t fmt = tf ? 2u : 1u;  // tf32 = 2 (kind::tf32), bf16 = 1 (kind::f16)
    const uint32_t bmn = (MODE == 4 || MODE == 5) ? 1u : 0u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (bmn << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
                           (static_cast<uint32_t>(128 >> 4) << 24);
    const uint64_t da = kdesc(base);
    const uint64_t db = bmn ? mndesc(base + 32768) : kdesc(base + 32768);
    const uint32_t ta = tm + 256;
    long long t0 = clock64();
    for (int i = 0; i < reps; ++i) {
      const uint32_t d = distinct_d ? tm + (i & 1) * 128 : tm;
      const uint32_t acc = i > 1 ? 1u : 0u;
      if (MODE == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      if (MODE == 1 || MODE == 4)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(d), "r"(ta), "l"(db), "r"(idesc), "r"(acc));
      if (MODE == 5)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      if (MODE == 6)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(d), "r"(ta + (i & 3) * 8), "l"(kdesc(base + 32768 + (i & 3) * 32)), "r"(idesc), "r"(acc));
      if (MODE == 2)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      if (MODE == 3)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(d), "r"(ta), "l"(db), "r"(idesc), "r"(acc));
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
            su32(&bar))
        : "memory");
    long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int MODE, int N, int LOAD = 0>
void run(const char* name, int grid = 1) {
  long long* d;
  cudaMalloc(&d, 16);
  auto k = probe<MODE, N, LOAD>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int dd = 0; dd < 2; ++dd) {
    long long h[2];
    const int reps = 256;
    k<<<grid, LOAD == 3 ? 448 : 128, 70000>>>(d, reps, dd);  // warm
    k<<<grid, LOAD == 3 ? 448 : 128, 70000>>>(d, reps, dd);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-22s L%d N=%3d distinct_d=%d : issue %.1f cyc/mma, complete %.1f cyc/mma  (%s)\n", name, LOAD, N, dd,
           double(h[0]) / reps, double(h[1]) / reps, cudaGetErrorString(e));
  }
  cudaFree(d);
}

int main() {
  run<0, 64>("tf32 SS");
  run<0, 128>("tf32 SS");
  run<0, 256>("tf32 SS");
  run<1, 64>("tf32 TS(A in TMEM)");
  run<1, 128>("tf32 TS(A in TMEM)");
  run<2, 64>("bf16 SS");
  run<2, 128>("bf16 SS");
  run<2, 256>("bf16 SS");
  run<3, 128>("bf16 TS(A in TMEM)");
  run<4, 64>("tf32 TS B MN-major");
  run<5, 64>("tf32 SS B MN-major");
  run<4, 128>("tf32 TS B MN-major");
  run<6, 64>("tf32 TS desc advance");
  run<1, 64, 3>("tf32 TS +spinners");
  run<1, 64>("tf32 TS grid148", 148);
  run<0, 128>("tf32 SS grid148", 148);
  run<0, 64, 1>("tf32 SS +smem load");
  run<1, 64, 1>("tf32 TS +smem load");
  run<1, 64, 2>("tf32 TS +tmem st load");
  run<0, 128, 1>("tf32 SS +smem load");
  return 0;
}
