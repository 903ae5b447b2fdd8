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
constexpr int kStages = 3;
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
  int kb_per_split;        // split-K: k-blocks per blockIdx.z (0 = all)
  int64_t split_stride;    // split-K: elements between partial outputs
  long long* trace;        // debug timeline (EGN_GEMM_TRACE), CTA 0 only
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
// MN-major tf32 operands must use SWIZZLE_128B_BASE32B (layout type 1, CuTe
// Layout_MN_SW128_32B_Atom): 128-byte rows hold 32 consecutive MN elements of one
// k, swizzled in 32-byte chunks over 4-row (512 B) atoms; TMA writes it with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.  LBO = 4096 B between 32-element MN groups
// (one TMA box of 32 k-rows each), SBO = 512 B between 4-row k groups.
__device__ __forceinline__ uint64_t sw128_mnmajor_desc(const void* smem_tile) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_u32(smem_tile) >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(4096 >> 4) << 16;
  d |= static_cast<uint64_t>(512 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(1) << 61;
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

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

template <int N>
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

#define EGN_TRACE(role, idx)                                                            \
  do {                                                                                  \
    if (P.trace && blockIdx.x == 0 && (idx) < 64 && ((threadIdx.x & 31) == 0)) {        \
      long long t_;                                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
      P.trace[(role) * 64 + (idx)] = t_;                                                \
    }                                                                                   \
  } while (0)

// Persistent, warp-specialised 3xTF32 GEMM (BN = 64 output columns per tile).
//   warp 0       : TMA producer (S-deep ring of raw fp32 A/B k-blocks)
//   warp 1       : MMA issuer (one elected thread)
//   warps 2..5   : split each landed k-block into hi (in place) / lo buffers
//   warps 6..13  : two accumulator groups of 4 warps; group = tile parity, so one
//                  group's epilogue overlaps the other group's main loop.
//                  TMEM lane quarter = warp % 4.
// Accuracy: the big term A_hi.B_hi goes to a fresh TMEM tile every kFlush k-steps
// (double buffered per group) that the group adds into fp32 registers, so the
// tensor core's truncating accumulation spans kFlush steps only; the small terms
// (A_lo.B_hi, A_hi.B_lo, ~2^-11 smaller) accumulate in TMEM over the whole K range.
constexpr int kFlush = 2;

template <int BN, bool AMN, bool BMN>
__global__ void __launch_bounds__(448, 1)
gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap mapA0, const __grid_constant__ CUtensorMap mapB0,
                   const __grid_constant__ CUtensorMap mapA1, const __grid_constant__ CUtensorMap mapB1,
                   Params P, int tiles_n, int splits, int total_items) {
  static_assert(BN == 64, "tile width");
  constexpr int A_BYTES = BM * BK * 4;  // 16 KB
  constexpr int B_BYTES = BN * BK * 4;  // 8 KB
  constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  constexpr int S = 3;
  constexpr uint32_t TMEM_COLS = 512;  // 2 groups x (big[2] + small) x 64
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for SWIZZLE_128B by offsetting the __shared__ array itself
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* stile_all = reinterpret_cast<float*>(smem + S * STAGE);  // 8 warps x [32][33]
  __shared__ __align__(8) uint64_t full_bar[S], conv_bar[S], empty_bar[S];
  __shared__ __align__(8) uint64_t accf_bar[2][2], acce_bar[2][2], small_bar[2];
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nk0 = (P.k0 + BK - 1) / BK;
  const int nk_all = nk0 + (P.nseg > 1 ? (P.k1 + BK - 1) / BK : 0);
  const int kbps = P.kb_per_split > 0 ? P.kb_per_split : nk_all;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&conv_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int gr = 0; gr < 2; ++gr) {
      for (int b = 0; b < 2; ++b) {
        mbar_init(&accf_bar[gr][b], 1);
        mbar_init(&acce_bar[gr][b], 4);
      }
      mbar_init(&small_bar[gr], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  auto item_coords = [&](int item, int64_t& m0, int& n0, int& kbeg, int& nk) {
    const int z = item % splits;
    const int rest = item / splits;
    const int nt = rest % tiles_n;
    const int mt = rest / tiles_n;
    m0 = static_cast<int64_t>(mt) * BM;
    n0 = nt * BN;
    kbeg = z * kbps;
    nk = max(0, min(kbps, nk_all - kbeg));
    return z;
  };

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      uint32_t it = 0;
      for (int item = blockIdx.x; item < total_items; item += gridDim.x) {
        int64_t m0;
        int n0, kbeg, nk;
        item_coords(item, m0, n0, kbeg, nk);
        for (int kbl = 0; kbl < nk; ++kbl, ++it) {
          const int s = it % S;
          mbar_wait(&empty_bar[s], ((it / S) & 1) ^ 1);
          EGN_TRACE(0, it);
          uint8_t* st = smem + s * STAGE;
          mbar_expect_tx(&full_bar[s], A_BYTES + B_BYTES);
          const int kb = kbeg + kbl;
          const bool first = kb < nk0;
          const int kk = (first ? kb : kb - nk0) * BK;
          const CUtensorMap* ma = first ? &mapA0 : &mapA1;
          const CUtensorMap* mb = first ? &mapB0 : &mapB1;
          if (AMN) {
#pragma unroll
            for (int i = 0; i < BM / 32; ++i)
              tma_load_2d(st + i * 4096, ma, &full_bar[s], static_cast<int>(m0) + 32 * i, kk);
          } else {
            tma_load_2d(st, ma, &full_bar[s], kk, static_cast<int>(m0));
          }
          if (BMN) {
#pragma unroll
            for (int i = 0; i < BN / 32; ++i) tma_load_2d(st + 2 * A_BYTES + i * 4096, mb, &full_bar[s], n0 + 32 * i, kk);
          } else {
            tma_load_2d(st + 2 * A_BYTES, mb, &full_bar[s], kk, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((AMN ? 1u : 0u) << 15) |
                             ((BMN ? 1u : 0u) << 16) | (static_cast<uint32_t>(BN >> 3) << 17) |
                             (static_cast<uint32_t>(BM >> 4) << 24);
      uint32_t it = 0, t = 0;
      uint32_t fc[2] = {0, 0};  // flush counter per group
      for (int item = blockIdx.x; item < total_items; item += gridDim.x, ++t) {
        int64_t m0;
        int n0, kbeg, nk;
        item_coords(item, m0, n0, kbeg, nk);
        const int gr = t & 1;
        const uint32_t tg = tmem + gr * (3 * BN);
        const uint32_t t_small = tg + 2 * BN;
        mbar_wait(&small_bar[gr], ((t >> 1) & 1) ^ 1);  // this group's previous tile drained
        asm volatile("tcgen05.fence::after_thread_sync;");
        uint32_t b = 0, tbig = tg;
        for (int kbl = 0; kbl < nk; ++kbl, ++it) {
          const int s = it % S;
          mbar_wait(&conv_bar[s], (it / S) & 1);
          EGN_TRACE(1, it);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint8_t* st = smem + s * STAGE;
          const uint8_t* ahi = st;
          const uint8_t* alo = st + A_BYTES;
          const uint8_t* bhi = st + 2 * A_BYTES;
          const uint8_t* blo = st + 2 * A_BYTES + B_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            const int oa = AMN ? k * 1024 : k * 32;
            const int ob = BMN ? k * 1024 : k * 32;
            const uint64_t dah = AMN ? sw128_mnmajor_desc(ahi + oa) : sw128_kmajor_desc(ahi + oa);
            const uint64_t dal = AMN ? sw128_mnmajor_desc(alo + oa) : sw128_kmajor_desc(alo + oa);
            const uint64_t dbh = BMN ? sw128_mnmajor_desc(bhi + ob) : sw128_kmajor_desc(bhi + ob);
            const uint64_t dbl = BMN ? sw128_mnmajor_desc(blo + ob) : sw128_kmajor_desc(blo + ob);
            const bool fstart = (k % kFlush) == 0;
            if (fstart) {
              b = fc[gr] & 1;
              mbar_wait(&acce_bar[gr][b], ((fc[gr] >> 1) & 1) ^ 1);
              asm volatile("tcgen05.fence::after_thread_sync;");
              tbig = tg + b * BN;
            }
            const uint32_t first_small = (kbl == 0 && k == 0) ? 0u : 1u;
            mma_tf32(t_small, dal, dbh, idesc, first_small);
            mma_tf32(t_small, dah, dbl, idesc, 1u);
            mma_tf32(tbig, dah, dbh, idesc, fstart ? 0u : 1u);
            if ((k % kFlush) == kFlush - 1) {
              mma_commit(&accf_bar[gr][b]);
              ++fc[gr];
            }
          }
          mma_commit(&empty_bar[s]);
        }
      }
    }
  } else if (warp < 6) {
    // ---------------- hi/lo split of each landed k-block (128 threads)
    const int ct = tid - 64;
    uint32_t it = 0;
    for (int item = blockIdx.x; item < total_items; item += gridDim.x) {
      int64_t m0;
      int n0, kbeg, nk;
      item_coords(item, m0, n0, kbeg, nk);
      for (int kbl = 0; kbl < nk; ++kbl, ++it) {
        const int s = it % S;
        mbar_wait(&full_bar[s], (it / S) & 1);
        if (ct == 0) EGN_TRACE(2, it);
        uint8_t* st = smem + s * STAGE;
        float4* a = reinterpret_cast<float4*>(st);
        float4* alo = reinterpret_cast<float4*>(st + A_BYTES);
#pragma unroll 4
        for (int i = ct; i < A_BYTES / 16; i += 128) {
          const float4 v = a[i];
          float4 h;
          h.x = tf32_rna(v.x); h.y = tf32_rna(v.y); h.z = tf32_rna(v.z); h.w = tf32_rna(v.w);
          a[i] = h;
          alo[i] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        }
        float4* bb = reinterpret_cast<float4*>(st + 2 * A_BYTES);
        float4* blo = reinterpret_cast<float4*>(st + 2 * A_BYTES + B_BYTES);
#pragma unroll 4
        for (int i = ct; i < B_BYTES / 16; i += 128) {
          const float4 v = bb[i];
          float4 h;
          h.x = tf32_rna(v.x); h.y = tf32_rna(v.y); h.z = tf32_rna(v.z); h.w = tf32_rna(v.w);
          bb[i] = h;
          blo[i] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        named_bar_sync(1, 128);
        if (ct == 0) {
          EGN_TRACE(3, it);
          mbar_arrive(&conv_bar[s]);
        }
      }
    }
  } else {
    // ---------------- accumulator groups + epilogue (thread = tile row)
    const int gr = (warp - 6) >> 2;
    const int q = warp & 3;  // TMEM lane quarter == this warp's 32 tile rows
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t tg = tmem + gr * (3 * BN) + lane_off;
    float* stile = stile_all + (warp - 6) * (32 * 33);
    const int opkind = (P.flags & EPI_RESID) ? 1 : ((P.flags & EPI_GATHER) ? 2 : ((P.flags & (EPI_DSILU_AUX | EPI_MUL_AUX)) ? 3 : 0));
    uint32_t fcount = 0;
    uint32_t t = 0;
    for (int item = blockIdx.x; item < total_items; item += gridDim.x, ++t) {
      if ((t & 1) != static_cast<uint32_t>(gr)) continue;
      if (q == 0 && gr == 0) EGN_TRACE(7, t);
      int64_t m0;
      int n0, kbeg, nk;
      const int z = item_coords(item, m0, n0, kbeg, nk);
      const int64_t rbase = m0 + q * 32;
      float acc[BN];
#pragma unroll
      for (int i = 0; i < BN; ++i) acc[i] = 0.f;
      const int nflush = nk * (BK / 8) / kFlush;
      for (int j = 0; j < nflush; ++j, ++fcount) {
        const uint32_t b = fcount & 1;
        mbar_wait(&accf_bar[gr][b], (fcount >> 1) & 1);
        if (q == 0 && gr == 0) EGN_TRACE(5, fcount);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t base = tg + b * BN;
#pragma unroll
        for (int c = 0; c < BN; c += 16) {
          float v[16];
          tmem_ld16<16>(base + c, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[c + i] += v[i];
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&acce_bar[gr][b]);
      }
      if (nflush > 0) {
#pragma unroll
        for (int c = 0; c < BN; c += 16) {
          float v[16];
          tmem_ld16<16>(tg + 2 * BN + c, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[c + i] += v[i];
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&small_bar[gr]);
      if (q == 0 && gr == 0) EGN_TRACE(6, t);
      // epilogue: per 32-column chunk, transpose through smem; lanes over columns,
      // operand loads batched 8 rows deep
      float* out_base = P.out + static_cast<int64_t>(z) * P.split_stride;
      const int nrows = P.M - rbase < 32 ? static_cast<int>(P.M - rbase) : 32;
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 32) {
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 32; ++i) stile[lane * 33 + i] = acc[c0 + i];
        __syncwarp();
        const int col = n0 + c0 + lane;
        if (col >= P.N) continue;
        const float bv = (P.flags & EPI_BIAS) ? P.bias[col] : 0.f;
        const float* sv = stile + lane;
        float* dst = out_base + rbase * P.ldo + col;
        float* dst2 = P.out2 ? P.out2 + rbase * P.ldo2 + col : nullptr;
        const int64_t ldo = P.ldo, ldo2 = P.ldo2;
        const bool silu2 = P.flags & EPI_SILU_OUT2;
        for (int r0 = 0; r0 < nrows; r0 += 8) {
          float o[8];
          if (opkind) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int64_t row = rbase + r0 + i;
              o[i] = 0.f;
              if (r0 + i < nrows)
                o[i] = opkind == 1 ? P.resid[row * P.ldr + col]
                     : opkind == 2 ? P.gsrc[static_cast<int64_t>(P.gidx[row]) * P.ldg + col]
                                   : P.aux[row * P.ldaux + col];
            }
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = r0 + i;
            if (rr >= nrows) break;
            float v = sv[rr * 33] + bv;
            if (opkind == 1 || opkind == 2) v += o[i];
            if (P.flags & EPI_DSILU_AUX) {
              const float sg = 1.f / (1.f + __expf(-o[i]));
              v *= sg * (1.f + o[i] * (1.f - sg));
            }
            if (P.flags & EPI_MUL_AUX) {
              dst2[rr * ldo2] = v;
              v *= o[i];
            }
            dst[rr * ldo] = v;
            if (silu2) dst2[rr * ldo2] = v / (1.f + __expf(-v));
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
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

// 2-D fp32 tensor map: `outer` rows of `inner` contiguous elements (row stride ld elements);
// box = 32 (inner, 128 B) x box_outer, SWIZZLE_128B, zero fill out of bounds.
static int make_map(CUtensorMap* map, const float* ptr, int64_t outer, int64_t inner, int64_t ld, int box_outer,
                    bool mn_major = false) {
  EncodeFn enc = get_encode();
  EGN_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  EGN_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, "GEMM operand must be 16-byte aligned");
  EGN_REQUIRE((ld * 4) % 16 == 0, "GEMM operand row stride must be a multiple of 16 bytes");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 4)};
  cuuint32_t box[2] = {32u, static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  EGN_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return 0;
}

template <int BN, bool AMN, bool BMN>
static int launch(const CUtensorMap& a0, const CUtensorMap& b0, const CUtensorMap& a1, const CUtensorMap& b1,
                  const Params& P, int splits, cudaStream_t st) {
  constexpr int STAGE = 2 * BM * BK * 4 + 2 * BN * BK * 4;
  const size_t smem = static_cast<size_t>(3) * STAGE + 8 * 32 * 33 * 4 + 1024;
  auto kern = gemm_tf32x3_kernel<BN, AMN, BMN>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured = true;
  }
  const int tiles_m = static_cast<int>((P.M + BM - 1) / BM);
  const int tiles_n = (P.N + BN - 1) / BN;
  const int total = tiles_m * tiles_n * splits;
  const int grid = std::min(total, kNumSMs);
  if (getenv("EGN_GEMM_TRACE")) {  // debug timeline of CTA 0 (ns since its first event)
    Params Q = P;
    long long* d = nullptr;
    cudaMalloc(&d, 8 * 64 * sizeof(long long));
    cudaMemset(d, 0, 8 * 64 * sizeof(long long));
    Q.trace = d;
    kern<<<grid, 448, smem, st>>>(a0, b0, a1, b1, Q, tiles_n, splits, total);
    long long h[8 * 64];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d);
    long long t0 = h[0];
    const char* names[8] = {"prod_issue", "mma_conv_ok", "conv_full_ok", "conv_done", "-", "acc0_flush", "epi0_start",
                            "tile0_begin"};
    for (int r = 0; r < 8; ++r) {
      printf("%-14s", names[r]);
      for (int i = 0; i < 24; ++i) printf(" %7lld", h[r * 64 + i] ? (h[r * 64 + i] - t0) : -1);
      printf("\n");
    }
    fflush(stdout);
    return check_launch("gemm_tf32x3");
  }
  kern<<<grid, 448, smem, st>>>(a0, b0, a1, b1, P, tiles_n, splits, total);
  return check_launch("gemm_tf32x3");
}

template <bool AMN, bool BMN>
static int launch_bn(int, const CUtensorMap& a0, const CUtensorMap& b0, const CUtensorMap& a1,
                     const CUtensorMap& b1, const Params& P, int splits, cudaStream_t st) {
  return launch<64, AMN, BMN>(a0, b0, a1, b1, P, splits, st);
}

__global__ void reduce_splits_kernel(const float* __restrict__ part, int splits, int64_t len, float* __restrict__ out,
                                     int accumulate) {
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * 32; base < len; base += static_cast<int64_t>(gridDim.x) * 32) {
    const int64_t i = base + lane;
    float s0 = 0.f, s1 = 0.f;
    if (i < len) {
      int z = w;
      for (; z + 8 < splits; z += 16) {
        s0 += part[z * len + i];
        s1 += part[(z + 8) * len + i];
      }
      if (z < splits) s0 += part[z * len + i];
    }
    red[w][lane] = s0 + s1;
    __syncthreads();
    if (w == 0 && i < len) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) s += red[k][lane];
      out[i] = accumulate ? out[i] + s : s;
    }
    __syncthreads();
  }
}

static void wgrad_split(int64_t krows, int M, int N, int* splits, int* kbps) {
  const int BNsel = 64;
  const int tiles = static_cast<int>(((M + BM - 1) / BM) * ((N + BNsel - 1) / BNsel));
  const int nk = static_cast<int>((krows + BK - 1) / BK);
  int want = std::max(1, kNumSMs / tiles);      // one wave of CTAs
  want = std::min(want, std::max(1, nk / 8));   // >= 8 k-blocks per CTA
  *kbps = (nk + want - 1) / want;
  *splits = (nk + *kbps - 1) / *kbps;
}

}  // namespace gemm
}  // namespace egn

using namespace egn;

extern "C" int egn_gemm(int64_t M, int N, int nseg, const float* a0, int64_t lda0, const float* b0, int64_t ldb0,
                        int k0, const float* a1, int64_t lda1, const float* b1, int64_t ldb1, int k1,
                        const float* bias, const float* resid, int64_t ldr, const float* gsrc, const int32_t* gidx,
                        int64_t ldg, const float* aux, int64_t ldaux, int flags, float* out, int64_t ldo,
                        float* out2, int64_t ldo2, int b_mn, egn_stream_t stream) {
  using namespace egn::gemm;
  EGN_REQUIRE(nseg == 1 || nseg == 2, "nseg must be 1 or 2");
  EGN_REQUIRE(N >= 16 && N % 16 == 0, "GEMM N must be a positive multiple of 16 (got %d)", N);
  EGN_REQUIRE(k0 > 0 && k0 % 4 == 0 && (nseg == 1 || (k1 > 0 && k1 % 4 == 0)), "GEMM K must be a multiple of 4");
  if (M == 0) return 0;
  Params P{M, N, nseg, k0, nseg > 1 ? k1 : 0, bias, resid, ldr, gsrc, gidx, ldg, aux, ldaux, flags, out, ldo, out2,
           ldo2, 0, 0};
  const int BNsel = 64;
  CUtensorMap ma0, mb0, ma1, mb1;
  // A: K-major [M, K]; B: K-major [N, K] (weights (out, in)) or MN-major [K, N] (b_mn)
  if (int rc = make_map(&ma0, a0, M, k0, lda0, BM)) return rc;
  if (int rc = b_mn ? make_map(&mb0, b0, k0, N, ldb0, BK, true) : make_map(&mb0, b0, N, k0, ldb0, BNsel)) return rc;
  if (nseg > 1) {
    if (int rc = make_map(&ma1, a1, M, k1, lda1, BM)) return rc;
    if (int rc = b_mn ? make_map(&mb1, b1, k1, N, ldb1, BK, true) : make_map(&mb1, b1, N, k1, ldb1, BNsel)) return rc;
  } else {
    ma1 = ma0;
    mb1 = mb0;
  }
  cudaStream_t st = as_stream(stream);
  if (b_mn) return launch_bn<false, true>(BNsel, ma0, mb0, ma1, mb1, P, 1, st);
  return launch_bn<false, false>(BNsel, ma0, mb0, ma1, mb1, P, 1, st);
}

extern "C" int64_t egn_gemm_wgrad_workspace_bytes(int64_t krows, int M, int N) {
  int splits, kbps;
  egn::gemm::wgrad_split(krows, M, N, &splits, &kbps);
  return static_cast<int64_t>(splits) * M * N * 4;
}

extern "C" int egn_gemm_wgrad(int64_t krows, int M, int N, const float* g, int64_t ldg, const float* x,
                              int64_t ldx, float* out, int accumulate, void* workspace, egn_stream_t stream) {
  using namespace egn::gemm;
  EGN_REQUIRE(M >= 1 && N >= 16 && N % 16 == 0, "wgrad needs N % 16 == 0 (got %d)", N);
  cudaStream_t st = as_stream(stream);
  if (krows == 0) {
    if (!accumulate) cudaMemsetAsync(out, 0, sizeof(float) * M * N, st);
    return check_launch("gemm_wgrad_empty");
  }
  int splits, kbps;
  wgrad_split(krows, M, N, &splits, &kbps);
  const int BNsel = 64;
  float* part = reinterpret_cast<float*>(workspace);
  Params P{M, N, 1, static_cast<int>(krows), 0, nullptr, nullptr, 0, nullptr, nullptr, 0, nullptr, 0, 0,
           part, N, nullptr, 0, kbps, static_cast<int64_t>(M) * N};
  CUtensorMap ma, mb;
  // A = g^T: g is [krows, M] with M contiguous (MN-major); B = x^T likewise
  if (int rc = make_map(&ma, g, krows, M, ldg, BK, true)) return rc;
  if (int rc = make_map(&mb, x, krows, N, ldx, BK, true)) return rc;
  if (int rc = launch_bn<true, true>(BNsel, ma, mb, ma, mb, P, splits, st)) return rc;
  const int64_t len = static_cast<int64_t>(M) * N;
  reduce_splits_kernel<<<static_cast<int>(std::min<int64_t>((len + 31) / 32, 4096)), 256, 0, st>>>(part, splits, len, out, accumulate);
  return check_launch("gemm_wgrad_reduce");
}
