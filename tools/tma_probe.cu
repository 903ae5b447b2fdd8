// TMA streaming probe: 148 persistent CTAs stream a [M][128] fp32 array (30 MB at M = 58,644)
// through a ring of 16 KB shared-memory slots, as the tcgen05 GEMM's A operand does, and report
// the achieved rate.  Patterns: "kblock" = the GEMM's boxes ([128 rows][32 floats] SW128, four per
// 128-row tile, each row read in four 128-byte pieces), "rows" = the same bytes as contiguous
// 16 KB boxes (32 whole rows each).  Ring depth R in 16 KB slots.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/tma_probe tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}

template <int R>
__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap map, int tiles, int row0, int mode,
                                                 float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = sm + ((1024u - (su32(sm) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[R], empty[R];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < R; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t it = 0;
  float acc = 0.f;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    for (int kb = 0; kb < 4; ++kb, ++it) {
      const int slot = it % R;
      if (warp == 0) {
        if (threadIdx.x == 0) {
          wait(&empty[slot], ((it / R) & 1) ^ 1);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[slot])), "r"(16384)
                       : "memory");
          int c0, c1;
          if (mode == 0) { c0 = kb * 32; c1 = row0 + t * 128; }          // [128 rows][32] at column kb*32
          else { c0 = 0; c1 = (row0 + t * 128) * 4 + kb * 128; }           // 128 quarter-rows = 32 whole rows
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                  su32(s + slot * 16384)),
              "l"(&map), "r"(su32(&full[slot])), "r"(c0), "r"(c1)
              : "memory");
        }
        __syncwarp();
      } else {
        wait(&full[slot], (it / R) & 1);
        acc += reinterpret_cast<const float*>(s + slot * 16384)[threadIdx.x & 31];
        __syncwarp();
        if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[slot])) : "memory");
      }
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int R>
float run(EncFn enc, float* buf, int64_t total_rows, int M, int mode, int l2promo) {
  CUtensorMap map;
  cuuint64_t dims[2], strides[1];
  cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
  if (mode == 0) { dims[0] = 128; dims[1] = total_rows; strides[0] = 512; }
  else { dims[0] = 32; dims[1] = total_rows * 4; strides[0] = 128; }
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B,
                   l2promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                : (l2promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B),
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); return -1; }
  const int smem = R * 16384 + 1024;
  auto k = stream<R>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tiles = M / 128;
  const int chunks = static_cast<int>(total_rows / M);
  for (int i = 0; i < 3; ++i) k<<<148, 64, smem>>>(map, tiles, (i % chunks) * M, mode, nullptr);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 16;
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) k<<<148, 64, smem>>>(map, tiles, ((i + 3) % chunks) * M, mode, nullptr);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double us = ms * 1000.0 / reps;
  const double gb = static_cast<double>(tiles) * 128 * 512 / 1e9;
  printf("mode %-6s R=%2d promo=%d M=%7d: %7.1f us per launch  %6.0f GB/s  (%s)\n", mode ? "rows" : "kblock", R, l2promo,
         M, us, gb / (us * 1e-6), cudaGetErrorString(cudaGetLastError()));
  return static_cast<float>(us);
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncFn enc = reinterpret_cast<EncFn>(p);
  const int64_t total_rows = 1 << 21;  // 1 GB: consecutive launches read different 30 MB chunks (cold L2)
  float* buf;
  cudaMalloc(&buf, total_rows * 512);
  cudaMemset(buf, 0, total_rows * 512);
  for (int M : {58624, 234496}) {
    for (int mode : {0, 1}) {
      for (int promo : {0, 2}) {
        run<4>(enc, buf, total_rows, M, mode, promo);
        run<8>(enc, buf, total_rows, M, mode, promo);
        run<12>(enc, buf, total_rows, M, mode, promo);
      }
    }
  }
  return 0;
}
