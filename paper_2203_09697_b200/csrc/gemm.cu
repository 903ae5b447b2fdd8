// Dense fp32-accurate GEMM on the 5th-generation tensor cores (tcgen05, TMEM, TMA).
//
//   C[M, N] = sum_s A_s[M, K_s] . B_s[N, K_s]^T   (+ fused epilogue)
//
// Used for every M = N_e (or N_v) sized product of the model (linear(),
// egn/tape.py:104-119): A rows are activations (row-major, K contiguous),
// B rows are weights stored (out, in) exactly as the reference stores them.
//
// Precision: the parity target is 1e-4 relative in fp32 (TF32 alone moves the
// forces by ~1e-3), so each operand is split x = hi + lo
// with hi = rna_tf32(x), lo = x - hi, and the product is formed as
// A_hi B_hi + A_hi B_lo + A_lo B_hi (3 x kind::tf32 MMAs, error ~2^-21).
//
// Structure (one 128-row tile per CTA, 128 threads):
//   * thread 0 issues TMA loads (SWIZZLE_128B, 32 fp32 = 128 B per row) of the
//     A and B k-blocks into a 2-stage ring guarded by mbarriers,
//   * all threads split the landed stage into hi/lo buffers (same swizzled
//     layout, so the split is elementwise),
//   * thread 0 issues 4 k-steps x 3 tcgen05.mma (M=128, N=BN, K=8) into a TMEM
//     accumulator and commits to an mbarrier that frees the stage,
//   * the epilogue warps read TMEM (tcgen05.ld 32x32b, thread = row) and apply
//     bias / residual / gathered-row add / SiLU / gate before storing.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace egn {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 32;                 // fp32 elements per 128-byte swizzled row
constexpr int kStages = 2;
constexpr int kThreads = 128;

enum Epi : int {
  EPI_BIAS = 1,        // C += bias[n]
  EPI_RESID = 2,       // C += R[m, n]
  EPI_GATHER = 4,      // C += G[idx[m], n]
  EPI_SILU_OUT2 = 8,   // out2 = silu(C)          (C stored to out)
  EPI_MUL_AUX = 16,    // out2 = C; C *= Aux[m, n]
  EPI_DSILU_AUX = 32,  // C *= silu'(Aux[m, n])
};

struct Params {
  int64_t M;
  int N, nseg, k0, k1;      // K extents of the (up to) two segments
  const float* bias;
  const float* resid;
  int64_t ldr;
  const float* gsrc;
  const int32_t* gidx;
  int64_t ldg;
  const float* aux;
  int64_t ldaux;
  int flags;
  float* out;
  int64_t ldo;
  float* out2;
  int64_t ldo2;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ uint64_t sw128_kmajor_desc(const void* smem_tile) {
  // start address >> 4 | LBO (unused for swizzled K-major) = 1 | SBO = 1024 B (8 rows x 128 B)
  // | version 1 (bits 46-47) | layout SWIZZLE_128B = 2 (bits 61-63)
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_u32(smem_tile) >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap mapA0, const __grid_constant__ CUtensorMap mapB0,
                   const __grid_constant__ CUtensorMap mapA1, const __grid_constant__ CUtensorMap mapB1,
                   Params P) {
  constexpr int A_BYTES = BM * BK * 4;        // 16 KB
  constexpr int B_BYTES = BN * BK * 4;
  constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;  // raw/hi + lo for A and B
  constexpr uint32_t TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ __align__(8) uint64_t free_bar[kStages];
  __shared__ __align__(8) uint64_t done_bar;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int n0 = blockIdx.y * BN;
  const int nk0 = (P.k0 + BK - 1) / BK;
  const int nk = nk0 + (P.nseg > 1 ? (P.k1 + BK - 1) / BK : 0);

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&free_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  auto stage_ptr = [&](int s) { return smem + s * STAGE; };
  auto issue_load = [&](int kb, int s) {
    uint8_t* st = stage_ptr(s);
    mbar_expect_tx(&full_bar[s], A_BYTES + B_BYTES);
    if (kb < nk0) {
      tma_load_2d(st, &mapA0, &full_bar[s], kb * BK, static_cast<int>(m0));
      tma_load_2d(st + 2 * A_BYTES, &mapB0, &full_bar[s], kb * BK, n0);
    } else {
      const int kk = (kb - nk0) * BK;
      tma_load_2d(st, &mapA1, &full_bar[s], kk, static_cast<int>(m0));
      tma_load_2d(st + 2 * A_BYTES, &mapB1, &full_bar[s], kk, n0);
    }
  };
  if (tid == 0) {
    for (int kb = 0; kb < (nk < kStages ? nk : kStages); ++kb) issue_load(kb, kb);
  }
  // instruction descriptor: D f32, A/B tf32, K-major both, N = BN, M = 128
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                         (static_cast<uint32_t>(BM >> 4) << 24);
  for (int kb = 0; kb < nk; ++kb) {
    const int s = kb % kStages;
    const uint32_t ph = (kb / kStages) & 1;
    mbar_wait(&full_bar[s], ph);
    // split: raw -> hi (in place), lo (second buffer); A then B
    uint8_t* st = stage_ptr(s);
    {
      float4* a = reinterpret_cast<float4*>(st);
      float4* alo = reinterpret_cast<float4*>(st + A_BYTES);
      for (int i = tid; i < A_BYTES / 16; i += kThreads) {
        float4 v = a[i], h;
        h.x = tf32_rna(v.x); h.y = tf32_rna(v.y); h.z = tf32_rna(v.z); h.w = tf32_rna(v.w);
        a[i] = h;
        alo[i] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
      }
      float4* b = reinterpret_cast<float4*>(st + 2 * A_BYTES);
      float4* blo = reinterpret_cast<float4*>(st + 2 * A_BYTES + B_BYTES);
      for (int i = tid; i < B_BYTES / 16; i += kThreads) {
        float4 v = b[i], h;
        h.x = tf32_rna(v.x); h.y = tf32_rna(v.y); h.z = tf32_rna(v.z); h.w = tf32_rna(v.w);
        b[i] = h;
        blo[i] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint8_t* ahi = st;
      const uint8_t* alo = st + A_BYTES;
      const uint8_t* bhi = st + 2 * A_BYTES;
      const uint8_t* blo = st + 2 * A_BYTES + B_BYTES;
#pragma unroll
      for (int k = 0; k < BK / 8; ++k) {
        const int off = k * 32;  // 8 tf32 = 32 bytes along the swizzled row
        const uint64_t dah = sw128_kmajor_desc(ahi + off), dal = sw128_kmajor_desc(alo + off);
        const uint64_t dbh = sw128_kmajor_desc(bhi + off), dbl = sw128_kmajor_desc(blo + off);
        const uint32_t acc0 = (kb > 0 || k > 0) ? 1u : 0u;
        mma_tf32(tmem, dal, dbh, idesc, acc0);  // small terms first
        mma_tf32(tmem, dah, dbl, idesc, 1u);
        mma_tf32(tmem, dah, dbh, idesc, 1u);
      }
      mma_commit(&free_bar[s]);
      if (kb + kStages < nk) {
        mbar_wait(&free_bar[s], ph);
        issue_load(kb + kStages, s);
      }
    }
  }
  if (tid == 0) mma_commit(&done_bar);
  mbar_wait(&done_bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");

  // ---------------- epilogue: thread = row (TMEM lane), 16 columns per load
  const int64_t row = m0 + warp * 32 + lane;
  const bool rok = row < P.M;
  const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  int64_t grow = 0;
  if ((P.flags & EPI_GATHER) && rok) grow = P.gidx[row];
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(lane_base + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (!rok) continue;
    const int cbase = n0 + c0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int col = cbase + i;
      if (col >= P.N) break;
      float v = __uint_as_float(r[i]);
      if (P.flags & EPI_BIAS) v += P.bias[col];
      if (P.flags & EPI_RESID) v += P.resid[row * P.ldr + col];
      if (P.flags & EPI_GATHER) v += P.gsrc[grow * P.ldg + col];
      if (P.flags & EPI_DSILU_AUX) {
        const float hx = P.aux[row * P.ldaux + col];
        const float sg = 1.f / (1.f + __expf(-hx));
        v *= sg * (1.f + hx * (1.f - sg));
      }
      if (P.flags & EPI_MUL_AUX) {
        P.out2[row * P.ldo2 + col] = v;
        v *= P.aux[row * P.ldaux + col];
      }
      P.out[row * P.ldo + col] = v;
      if (P.flags & EPI_SILU_OUT2) P.out2[row * P.ldo2 + col] = v / (1.f + __expf(-v));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// rows x cols fp32 row-major (cols contiguous, row stride ld elements); box = box_rows x 32
static int make_map(CUtensorMap* map, const float* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  EncodeFn enc = get_encode();
  EGN_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  EGN_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, "GEMM operand must be 16-byte aligned");
  EGN_REQUIRE((ld * 4) % 16 == 0, "GEMM operand row stride must be a multiple of 16 bytes");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 4)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  EGN_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return 0;
}

template <int BN>
static int launch(const CUtensorMap& a0, const CUtensorMap& b0, const CUtensorMap& a1, const CUtensorMap& b1,
                  const Params& P, cudaStream_t st) {
  constexpr int STAGE = 2 * BM * BK * 4 + 2 * BN * BK * 4;
  const size_t smem = static_cast<size_t>(kStages) * STAGE + 1024;
  auto kern = gemm_tf32x3_kernel<BN>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured = true;
  }
  dim3 grid(static_cast<unsigned>((P.M + BM - 1) / BM), static_cast<unsigned>((P.N + BN - 1) / BN));
  kern<<<grid, kThreads, smem, st>>>(a0, b0, a1, b1, P);
  return check_launch("gemm_tf32x3");
}

}  // namespace gemm
}  // namespace egn

using namespace egn;

extern "C" int egn_gemm(int64_t M, int N, int nseg, const float* a0, int64_t lda0, const float* b0, int64_t ldb0,
                        int k0, const float* a1, int64_t lda1, const float* b1, int64_t ldb1, int k1,
                        const float* bias, const float* resid, int64_t ldr, const float* gsrc, const int32_t* gidx,
                        int64_t ldg, const float* aux, int64_t ldaux, int flags, float* out, int64_t ldo,
                        float* out2, int64_t ldo2, egn_stream_t stream) {
  using namespace egn::gemm;
  EGN_REQUIRE(nseg == 1 || nseg == 2, "nseg must be 1 or 2");
  EGN_REQUIRE(N >= 16 && N % 16 == 0, "GEMM N must be a positive multiple of 16 (got %d)", N);
  EGN_REQUIRE(k0 > 0 && k0 % 4 == 0 && (nseg == 1 || (k1 > 0 && k1 % 4 == 0)), "GEMM K must be a multiple of 4");
  if (M == 0) return 0;
  Params P{M, N, nseg, k0, nseg > 1 ? k1 : 0, bias, resid, ldr, gsrc, gidx, ldg, aux, ldaux, flags, out, ldo, out2,
           ldo2};
  const int BNsel = N <= 64 ? 64 : (N <= 128 ? 128 : 256);
  CUtensorMap ma0, mb0, ma1, mb1;
  if (int rc = make_map(&ma0, a0, M, k0, lda0, BM)) return rc;
  if (int rc = make_map(&mb0, b0, N, k0, ldb0, BNsel)) return rc;
  if (nseg > 1) {
    if (int rc = make_map(&ma1, a1, M, k1, lda1, BM)) return rc;
    if (int rc = make_map(&mb1, b1, N, k1, ldb1, BNsel)) return rc;
  } else {
    ma1 = ma0;
    mb1 = mb0;
  }
  cudaStream_t st = as_stream(stream);
  if (BNsel == 64) return launch<64>(ma0, mb0, ma1, mb1, P, st);
  if (BNsel == 128) return launch<128>(ma0, mb0, ma1, mb1, P, st);
  return launch<256>(ma0, mb0, ma1, mb1, P, st);
}
