// Cycles per k-block of the GEMM's MMA-issuer loop in isolation (one CTA, no producer /
// split / epilogue): per k-block 4 k8-steps x 3 tcgen05.mma (M=128, N=64, A from TMEM,
// B hi/lo K-major SW128 in shared memory), a window commit every W k8-steps and an
// operand-slot commit per k-block.  Variants change W, the operand sources and whether
// the per-window commits are issued, to see which part of the loop costs time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/mma_loop_probe tools/mma_loop_probe.cu
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
__device__ __forceinline__ void mma_ta(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
}

// MODE bit0: A from smem (SS) instead of TMEM; bit1: no window commits; bit2: same B for all
// three products; bit3: N = 128
template <int MODE>
__global__ void probe(long long* out, int kblocks, int win) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar[8];
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.f;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tb;
  constexpr int N = (MODE & 8) ? 128 : 64;
  if (threadIdx.x < 32) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24);
    const uint32_t bs = su32(sm + 65536);
    long long t0 = clock64();
    int wpos = 0, fc = 0;
    for (int kb = 0; kb < kblocks; ++kb) {
      const int o = kb & 1;
      const uint32_t bhi = bs + o * 16384, blo = bhi + 8192;
      const uint32_t ta = tm + 256 + o * 64;
      const uint32_t as = su32(sm + o * 32768);
      for (int k = 0; k < 4; ++k) {
        const bool fstart = wpos == 0;
        const uint32_t tacc = tm + (fc & 1) * N;
        const bool fend = ++wpos == win;
        if (elect_one()) {
          const uint64_t dh = kdesc(bhi + k * 32), dl = (MODE & 4) ? dh : kdesc(blo + k * 32);
          if (MODE & 1) {
            mma_ss(tacc, kdesc(as + 16384 + k * 32), dh, idesc, fstart ? 0u : 1u);
            mma_ss(tacc, kdesc(as + k * 32), dl, idesc, 1u);
            mma_ss(tacc, kdesc(as + k * 32), dh, idesc, 1u);
          } else {
            mma_ta(tacc, ta + 32 + k * 8, dh, idesc, fstart ? 0u : 1u);
            mma_ta(tacc, ta + k * 8, dl, idesc, 1u);
            mma_ta(tacc, ta + k * 8, dh, idesc, 1u);
          }
          if (fend && !(MODE & 2)) commit(&bar[2 + (fc & 1)]);
        }
        __syncwarp();
        if (fend) { wpos = 0; ++fc; }
      }
      if (elect_one()) commit(&bar[o]);
      __syncwarp();
    }
    long long t1 = clock64();
    if (elect_one()) commit(&bar[4]);
    __syncwarp();
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(su32(&bar[4])) : "memory");
    long long t2 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int MODE>
void run(const char* name, int win) {
  long long* d;
  cudaMalloc(&d, 16);
  auto k = probe<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int kb = 256;
  k<<<1, 128, 100 * 1024>>>(d, kb, win);
  k<<<1, 128, 100 * 1024>>>(d, kb, win);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-34s win=%2d: issue %6.1f, complete %6.1f cycles per k-block (12 MMAs) (%s)\n", name, win, double(h[0]) / kb,
         double(h[1]) / kb, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("TS, hi/lo B, window commits", 2);
  run<0>("TS, hi/lo B, window commits", 4);
  run<2>("TS, hi/lo B, no window commits", 2);
  run<4>("TS, one B, window commits", 2);
  run<1>("SS, hi/lo B, window commits", 2);
  run<3>("SS, hi/lo B, no window commits", 2);
  run<8>("TS N=128, window commits", 2);
  run<10>("TS N=128, no window commits", 2);
  run<9>("SS N=128, window commits", 2);
  return 0;
}
