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
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace egn {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 32;                 // fp32 elements per 128-byte swizzled row

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
  int flush_steps;         // k-steps (of 8) per TMEM->register flush (0 = whole tile)
  int tma_out;             // single-output epilogues store through mapOut (TMA)
  float* gsum_part;        // wgrad: per-split column sums of g (rows of A), [splits][M], or null
  int mcast;               // 1: CTA pairs (cluster of 2) share each A k-block by TMA multicast
  int64_t split_stride;    // split-K: elements between partial outputs
  long long* trace;        // debug timeline (EGN_GEMM_TRACE), CTA 0 only
  int dbg;                 // EGN_GEMM_DBG experiments: 4 no TMEM reads, 16 no B loads, 32 no A loads (n0 > 0);
                           // with -DEGN_GEMM_ABLATE also 1 no MMA, 2 no split math, 8 no B_lo math
  int op_tma;              // (with store_warp) residual / aux rows arrive by TMA through mapOp
  int store_warp;          // (with tma_out) a dedicated warp issues the TMA stores
};

// Stage-ablation switches in the k-block loops cost ~4% at the XL widths even
// when off, so they are compiled in only with -DEGN_GEMM_ABLATE.
#ifdef EGN_GEMM_ABLATE
constexpr bool kAblate = true;
#else
constexpr bool kAblate = false;
#endif

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
#ifdef EGN_WAIT_HINT
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(EGN_WAIT_HINT)
#else
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
#endif
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(c2), "r"(smem_u32(src))
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
__device__ __forceinline__ uint64_t sw128_kmajor_desc_u(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}
__device__ __forceinline__ uint64_t sw128_mnmajor_desc_u(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(4096 >> 4) << 16) |
         (static_cast<uint64_t>(512 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(1) << 61);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
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
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_));                                 \
      P.trace[(role) * 64 + (idx)] = t_;                                                \
    }                                                                                   \
  } while (0)

// Persistent, warp-specialised 3xTF32 GEMM, 128 x BN output tiles (BN = 64 or 128).
//   warp 0       : TMA producer: raw fp32 A/B k-blocks into a kTmaRing-deep ring
//   warp 1       : MMA issuer (whole warp walks the loop, one elected lane issues)
//   warps 2..5   : split each landed k-block: the raw tiles are the tf32 hi parts (the
//                  tensor core truncates), so A rows (thread = row) give A_lo = a - trunc(a)
//                  to a TMEM slot (tcgen05.st) and B gives B_lo to a shared operand slot
//                  (same swizzled layout, elementwise).  Weight gradients (MN-major A)
//                  put A_hi = rna(a) and A_lo into TMEM instead.  kOpRing operand slots.
//   warps 6..13  : accumulator warps: two groups of 4 (BN 64, group = tile parity) or one
//                  group of 8 (BN 128, warp = lane quarter x column half).
//   warp 14      : store warp (TMA stores of finished tiles, operand-row prefetch).
//   warp 15      : (BLO instantiations, egn_gemm_blo) loads the precomputed lo tile of the
//                  weight B into the operand slot by TMA; the split warps then form A_lo only.
// Per k-step: A_lo.B_hi (A from TMEM), A_hi.B_lo and A_hi.B_hi (A from the TMA slot); the
// MMA commit releases the TMA slot and the operand slot.
// Accuracy: the tensor core accumulates with truncation, a bias that grows with
// the number of k-steps summed in TMEM.  The products of each k-block (small ones
// first) go to a TMEM window tile (kAccBufs buffers per group) that is restarted every
// P.flush_steps k-steps; the group adds each finished window into fp32 registers (round
// to nearest).
// TMEM columns: [0, 384) accumulator windows; [384, 384 + 64 kOpRing) A operand slots
// (A_lo at +0; weight gradients: A_hi at +0, A_lo at +32).
// Epilogue: each warp owns a [2 chunks][32 rows][32 cols] fp32 staging buffer (16-byte
// granules XOR-swizzled by row, the TMA SWIZZLE_128B layout) that receives the operand rows
// (residual / gathered rows / aux); thread = row combines in place, then the store warp
// TMA-stores it.
constexpr int kEpiWarp = 2 * 32 * 32 * 4;  // 8 KB per accumulator warp
constexpr int EW = 64;                     // output columns per accumulator warp
// Per-tile-width configuration.  BN = 64: two accumulator groups of 4 warps (tile
// parity), each warp 32 rows x 64 columns.  BN = 128 (N % 128 == 0): one group of 8
// warps, warp = (row quarter, column half); one A k-block feeds N = 128 MMAs, which
// run at twice the N = 64 rate per output column.
// TRUNC (activation x weight products): the operand slot holds B_lo only (the raw tiles are
// the hi parts), which leaves room for a deeper TMA ring.
template <int BN, bool TRUNC = false>
struct Cfg {
  static constexpr int kTmaRing = TRUNC ? (BN == 64 ? 6 : 4) : (BN == 64 ? 5 : 3);
  static constexpr int kOpRing = 2;
  static constexpr int kAccBufs = BN == 64 ? 2 : 3;  // TMEM window buffers per group
  static constexpr int kGroups = BN == 64 ? 2 : 1;
  static constexpr int kTmaSlot = BM * BK * 4 + BN * BK * 4;  // raw A + raw B k-block
  static constexpr int kOpSlot = (TRUNC ? 1 : 2) * BN * BK * 4;  // B lo (+ B hi)
  static constexpr size_t kSmem =
      static_cast<size_t>(kTmaRing) * kTmaSlot + kOpRing * kOpSlot + 8 * kEpiWarp + 1024;
  static_assert(kGroups * kAccBufs * BN + 64 * kOpRing <= 512, "TMEM columns");
  static_assert(kSmem <= 232448, "shared memory");
};

__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
      "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
      "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}
// round-to-nearest (ties away) to tf32 with integer ops: add half an ulp of the
// 10-bit mantissa to the magnitude bits and clear the 13 low bits
__device__ __forceinline__ float tf32_rna_int(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}
// lo part for the truncation split: x - trunc_tf32(x).  RNA: itself rounded to nearest tf32
// so that the tensor core's truncation of it is exact -- an unbiased ~2^-21 |x| error instead
// of a one-signed ~2^-20 |x| one (worst model-gradient error 2.2e-5 with RNA on both lo
// parts, 6.7e-5 without, for ~1% of step time).
template <bool RNA>
__device__ __forceinline__ float tf32_lo_trunc(float x) {
  const float lo = x - __uint_as_float(__float_as_uint(x) & 0xffffe000u);
  return RNA ? tf32_rna_int(lo) : lo;
}
__device__ __forceinline__ float dsilu(float o) {
  const float sg = __fdividef(1.f, 1.f + __expf(-o));
  return sg * (1.f + o * (1.f - sg));
}
// element (r, c) of a [32][32] epilogue chunk (granule swizzled by row)
__device__ __forceinline__ int epi_idx(int r, int c) { return r * 32 + ((((c >> 2) ^ (r & 7))) << 2) + (c & 3); }

template <bool AMN, bool BMN, int BN, bool BLO = false>
__global__ void __launch_bounds__(512, 1)
gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap mapA0, const __grid_constant__ CUtensorMap mapB0,
                   const __grid_constant__ CUtensorMap mapA1, const __grid_constant__ CUtensorMap mapB1,
                   const __grid_constant__ CUtensorMap mapOut, const __grid_constant__ CUtensorMap mapOut2,
                   const __grid_constant__ CUtensorMap mapOp, const __grid_constant__ CUtensorMap mapBlo0,
                   const __grid_constant__ CUtensorMap mapBlo1, Params P,
                   int tiles_n, int splits, int total_items) {
  constexpr int A_BYTES = BM * BK * 4;  // 16 KB raw A k-block
  using C = Cfg<BN, true>;
  constexpr int kTmaRing = C::kTmaRing, kOpRing = C::kOpRing, kAccBufs = C::kAccBufs, kGroups = C::kGroups;
  constexpr int kTmaSlot = C::kTmaSlot, kOpSlot = C::kOpSlot;
  constexpr int B_BYTES = BN * BK * 4;  // 8 / 16 KB
  constexpr uint32_t TMEM_COLS = 512;
  constexpr uint32_t A_TMEM = kGroups * kAccBufs * BN;  // 384
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1024-byte alignment for SWIZZLE_128B by offsetting the __shared__ array itself
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* opring = smem + kTmaRing * kTmaSlot;
  float* epi_all = reinterpret_cast<float*>(opring + kOpRing * kOpSlot);
  __shared__ __align__(8) uint64_t tma_full[kTmaRing], tma_empty[kTmaRing], op_full[kOpRing], op_empty[kOpRing];
  __shared__ __align__(8) uint64_t blo_full[kOpRing];  // B_lo tile of the operand slot landed (BLO)
  __shared__ __align__(8) uint64_t accf_bar[kGroups][kAccBufs], acce_bar[kGroups][kAccBufs];
  // store warp hand-off per group: results staged (epi_full), staging read by the TMA store
  // (buf_free), next tile's operand rows landed in the staging buffers (op_bar)
  __shared__ __align__(8) uint64_t epi_full[kGroups], buf_free[kGroups], op_bar[kGroups];
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nk0 = (P.k0 + BK - 1) / BK;
  const int nk_all = nk0 + (P.nseg > 1 ? (P.k1 + BK - 1) / BK : 0);
  const int kbps = P.kb_per_split > 0 ? P.kb_per_split : nk_all;
  if (P.trace && tid == 0) {
    long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    P.trace[1024 + 4 * blockIdx.x] = g;
  }

  const uint32_t crank = P.mcast ? cluster_rank() : 0;
  // Truncation split (activation x weight products, K-major A): the tensor core reads fp32
  // operands as tf32 by truncation (tools/tf32_trunc_probe.cu), so the raw TMA tiles serve as
  // the hi parts (A_hi B_hi and A_hi B_lo read A from shared memory); the split warps only
  // form lo = x - trunc(x) (A_lo to TMEM, B_lo to shared memory) and the TMA slot stays until
  // the k-block's MMAs complete.  Weight gradients (MN-major A read by the split warps) keep
  // the rna hi / lo split of A in TMEM and truncate B only.
  constexpr bool trunc = true;
  constexpr bool trunc_a = !AMN;
  if (tid == 0) {
    // descriptor fetches off the critical path (the output map is first used at the end of a tile)
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA0) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB0) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA1) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB1) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapOut) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapOp) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapOut2) : "memory");
    if (BLO) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapBlo0) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapBlo1) : "memory");
    }
    for (int s = 0; s < kTmaRing; ++s) {
      mbar_init(&tma_full[s], 1);
      // the multicast leader reuses slot s only after both CTAs' split warps released it
      mbar_init(&tma_empty[s], (P.mcast && crank == 0) ? 2 : 1);
    }
    for (int s = 0; s < kOpRing; ++s) {
      mbar_init(&op_full[s], 1);
      mbar_init(&op_empty[s], 1);
      mbar_init(&blo_full[s], 1);
    }
    for (int gr = 0; gr < kGroups; ++gr) {
      for (int b = 0; b < kAccBufs; ++b) {
        mbar_init(&accf_bar[gr][b], 1);
        mbar_init(&acce_bar[gr][b], 8 / kGroups);  // every warp of the group drains
      }
      mbar_init(&epi_full[gr], 8 / kGroups);
      mbar_init(&buf_free[gr], 1);
      mbar_init(&op_bar[gr], 1);
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
  if (P.mcast) cluster_sync();  // the peer's barriers exist before any multicast / remote arrive
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
    uint32_t it = 0;
    for (int item = blockIdx.x; item < total_items; item += gridDim.x) {
      int64_t m0;
      int n0, kbeg, nk;
      item_coords(item, m0, n0, kbeg, nk);
      for (int kbl = 0; kbl < nk; ++kbl, ++it) {
        const int s = it % kTmaRing;
        mbar_wait(&tma_empty[s], ((it / kTmaRing) & 1) ^ 1);
        EGN_TRACE(0, it);
        if (elect_one()) {
          uint8_t* st = smem + s * kTmaSlot;
          const bool skip_b = P.dbg & 16, skip_a = (P.dbg & 32) && (n0 != 0);
          if (skip_a && skip_b) mbar_arrive(&tma_full[s]);
          else mbar_expect_tx(&tma_full[s], (skip_a ? 0 : A_BYTES) + (skip_b ? 0 : B_BYTES));
          const int kb = kbeg + kbl;
          const bool first = kb < nk0;
          const int kk = (first ? kb : kb - nk0) * BK;
          const CUtensorMap* ma = first ? &mapA0 : &mapA1;
          const CUtensorMap* mb = first ? &mapB0 : &mapB1;
          if (skip_a) {
          } else if (AMN) {
            tma_load_2d(st, ma, &tma_full[s], static_cast<int>(m0), kk);  // [32 k][128 m], unswizzled
          } else if (!P.mcast) {
            tma_load_2d(st, ma, &tma_full[s], kk, static_cast<int>(m0));  // [128 m][32 k], SW128
          } else if (crank == 0) {
            // both CTAs of the pair work on this m-tile: one L2 read, delivered to both
            tma_load_2d_mc(st, ma, &tma_full[s], kk, static_cast<int>(m0), 0x3);
          }
          if (skip_b) {
          } else if (BMN) {
#pragma unroll
            for (int i = 0; i < BN / 32; ++i) tma_load_2d(st + A_BYTES + i * 4096, mb, &tma_full[s], n0 + 32 * i, kk);
          } else {
            tma_load_2d(st + A_BYTES, mb, &tma_full[s], kk, n0);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((BMN ? 1u : 0u) << 16) |
                           (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(BM >> 4) << 24);
    uint32_t it = 0, t = 0;
    uint32_t fc0 = 0, fc1 = 0;  // window counters per accumulator group
    uint32_t wtr = 0;           // (trace) windows started
    for (int item = blockIdx.x; item < total_items; item += gridDim.x, ++t) {
      int64_t m0;
      int n0, kbeg, nk;
      item_coords(item, m0, n0, kbeg, nk);
      const int gr = kGroups == 2 ? static_cast<int>(t & 1) : 0;
      uint32_t& fc = gr ? fc1 : fc0;
      const uint32_t tg = tmem + gr * (kAccBufs * BN);
      uint32_t tacc = tg, bsel = 0;
      const int nsteps = nk * (BK / 8);
      const int win = P.flush_steps > 0 ? P.flush_steps : nsteps;
      int j = 0, wpos = 0;
      for (int kbl = 0; kbl < nk; ++kbl, ++it) {
        const int o = it % kOpRing;
        mbar_wait(&op_full[o], (it / kOpRing) & 1);
        if constexpr (BLO) mbar_wait(&blo_full[o], (it / kOpRing) & 1);
        EGN_TRACE(1, it);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t bhi = smem_u32(opring + o * kOpSlot);
        const uint32_t blo = bhi + B_BYTES;
        const uint32_t ta = tmem + A_TMEM + o * 64;
        if (trunc) {
          // raw A / B in the TMA slot are the hi parts; B_lo at the operand slot, A_lo in TMEM
          const int s = it % kTmaRing;
          const uint32_t araw = smem_u32(smem + s * kTmaSlot);
          const uint32_t braw = araw + A_BYTES;
          const uint32_t bl = bhi;  // B_lo
          const bool fstart = wpos == 0;
          if (fstart) {
            bsel = fc % kAccBufs;
            mbar_wait(&acce_bar[gr][bsel], ((fc / kAccBufs) & 1) ^ 1);
            EGN_TRACE(12, wtr);
            ++wtr;
            asm volatile("tcgen05.fence::after_thread_sync;");
            tacc = tg + bsel * BN;
          }
          j += BK / 8;
          wpos += BK / 8;
          const bool fend = (wpos >= win) || (j == nsteps);
          if (elect_one()) {
            // A_lo / A_hi: TMEM columns [0, 32) / shared-memory raw tile (trunc_a), or TMEM
            // [32, 64) / [0, 32) (rna split of an MN-major A)
            if (!(kAblate && (P.dbg & 1))) {  // (ablation bit 1: no MMAs, commits only)
#pragma unroll
            for (int k = 0; k < BK / 8; ++k) {  // small terms first
              const uint32_t ob = BMN ? k * 1024 : k * 32;
              const uint64_t db = BMN ? sw128_mnmajor_desc_u(braw + ob) : sw128_kmajor_desc_u(braw + ob);
              const uint64_t dl = BMN ? sw128_mnmajor_desc_u(bl + ob) : sw128_kmajor_desc_u(bl + ob);
              if (trunc_a) {
                mma_tf32_ta(tacc, ta + k * 8, db, idesc, (fstart && k == 0) ? 0u : 1u);  // A_lo B_hi
                mma_tf32(tacc, sw128_kmajor_desc_u(araw + k * 32), dl, idesc, 1u);      // A_hi B_lo
              } else {
                mma_tf32_ta(tacc, ta + 32 + k * 8, db, idesc, (fstart && k == 0) ? 0u : 1u);
                mma_tf32_ta(tacc, ta + k * 8, dl, idesc, 1u);
              }
            }
#pragma unroll
            for (int k = 0; k < BK / 8; ++k) {
              const uint32_t ob = BMN ? k * 1024 : k * 32;
              const uint64_t db = BMN ? sw128_mnmajor_desc_u(braw + ob) : sw128_kmajor_desc_u(braw + ob);
              if (trunc_a) mma_tf32(tacc, sw128_kmajor_desc_u(araw + k * 32), db, idesc, 1u);  // A_hi B_hi
              else mma_tf32_ta(tacc, ta + k * 8, db, idesc, 1u);
            }
            }
            if (fend) mma_commit(&accf_bar[gr][bsel]);
            mma_commit(&tma_empty[s]);  // the raw tiles are free once these MMAs completed
          }
          __syncwarp();
          if (fend) {
            ++fc;
            wpos = 0;
          }
        }
        EGN_TRACE(4, it);
        if (elect_one()) mma_commit(&op_empty[o]);
        __syncwarp();
      }
    }
  } else if (warp < 6) {
    // ---------------- split (128 threads): raw TMA slot -> operand slot, release
    const int ct = tid - 64;
    const int q = warp & 3;
    const int r = q * 32 + lane;  // A row of this thread == its TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    uint32_t it = 0;
    for (int item = blockIdx.x; item < total_items; item += gridDim.x) {
      int64_t m0;
      int n0, kbeg, nk;
      const int z = item_coords(item, m0, n0, kbeg, nk);
      float gs = 0.f;  // wgrad: sum over this split's rows of A row r (= column r of g)
      for (int kbl = 0; kbl < nk; ++kbl, ++it) {
        const int s = it % kTmaRing;
        const int o = it % kOpRing;
        mbar_wait(&tma_full[s], (it / kTmaRing) & 1);
        if (ct == 0) EGN_TRACE(2, it);
        mbar_wait(&op_empty[o], ((it / kOpRing) & 1) ^ 1);
        if (ct == 0) EGN_TRACE(11, it);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint8_t* st = smem + s * kTmaSlot;
        const uint32_t ta = tmem + lane_off + A_TMEM + o * 64;
        if (trunc && !(kAblate && (P.dbg & 2))) {  // (ablation bit 2: no split math)
          // lo = x - trunc_tf32(x) only (the raw tiles are the hi parts)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (!trunc_a) break;
            float lo[16];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const int gran = h * 4 + g;
              const float4 v = *reinterpret_cast<const float4*>(st + r * 128 + ((gran ^ (r & 7)) << 4));
              lo[g * 4 + 0] = tf32_lo_trunc<true>(v.x);
              lo[g * 4 + 1] = tf32_lo_trunc<true>(v.y);
              lo[g * 4 + 2] = tf32_lo_trunc<true>(v.z);
              lo[g * 4 + 3] = tf32_lo_trunc<true>(v.w);
            }
            tmem_st16(ta + h * 16, lo);
          }
          if (!trunc_a) {  // MN-major A: rna hi / lo into TMEM columns [0, 32) / [32, 64)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              float hi[16], lo[16];
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                const float* col = reinterpret_cast<const float*>(st) + r;
                const float4 v = make_float4(col[(h * 16 + g * 4 + 0) * BM], col[(h * 16 + g * 4 + 1) * BM],
                                             col[(h * 16 + g * 4 + 2) * BM], col[(h * 16 + g * 4 + 3) * BM]);
                gs += (v.x + v.y) + (v.z + v.w);
                hi[g * 4 + 0] = tf32_rna_int(v.x);
                hi[g * 4 + 1] = tf32_rna_int(v.y);
                hi[g * 4 + 2] = tf32_rna_int(v.z);
                hi[g * 4 + 3] = tf32_rna_int(v.w);
                lo[g * 4 + 0] = v.x - hi[g * 4 + 0];
                lo[g * 4 + 1] = v.y - hi[g * 4 + 1];
                lo[g * 4 + 2] = v.z - hi[g * 4 + 2];
                lo[g * 4 + 3] = v.w - hi[g * 4 + 3];
              }
              tmem_st16(ta + h * 16, hi);
              tmem_st16(ta + 32 + h * 16, lo);
            }
          }
          const float4* braw = reinterpret_cast<const float4*>(st + A_BYTES);
          float4* bl = reinterpret_cast<float4*>(opring + o * kOpSlot);
#pragma unroll
          for (int i = (BLO || (kAblate && (P.dbg & 8))) ? B_BYTES / 16 : ct; i < B_BYTES / 16; i += 128) {
            const float4 v = braw[i];
            bl[i] = make_float4(tf32_lo_trunc<true>(v.x), tf32_lo_trunc<true>(v.y), tf32_lo_trunc<true>(v.z),
                                tf32_lo_trunc<true>(v.w));
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        named_bar_sync(1, 128);
        if (ct == 0) {
          EGN_TRACE(3, it);
          if (!trunc) {  // (truncation split: the MMA commit releases the raw tiles)
            mbar_arrive(&tma_empty[s]);
            if (P.mcast && crank == 1) mbar_arrive_remote(&tma_empty[s], 0);
          }
          mbar_arrive(&op_full[o]);
        }
      }
      if (AMN && P.gsum_part != nullptr && n0 == 0 && m0 + r < P.M) P.gsum_part[z * P.M + m0 + r] = gs;
    }
  } else if (warp < 14) {
    // ---------------- accumulator groups + epilogue (thread = tile row)
    const int gr = kGroups == 2 ? (warp - 6) >> 2 : 0;
    const int chalf = kGroups == 2 ? 0 : (warp - 6) >> 2;  // this warp's 64-column half of the tile
    const int q = warp & 3;  // TMEM lane quarter == this warp's 32 tile rows
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t tg = tmem + gr * (kAccBufs * BN) + lane_off + chalf * EW;
    float* ebuf = epi_all + (warp - 6) * (2 * 32 * 32);
    const int opkind = (P.flags & EPI_RESID) ? 1 : ((P.flags & EPI_GATHER) ? 2 : ((P.flags & (EPI_DSILU_AUX | EPI_MUL_AUX)) ? 3 : 0));
    uint32_t fcount = 0;
    uint32_t t = 0;
    for (int item = blockIdx.x; item < total_items; item += gridDim.x, ++t) {
      if (kGroups == 2 && (t & 1) != static_cast<uint32_t>(gr)) continue;
      if (q == 0 && gr == 0 && chalf == 0) EGN_TRACE(7, t);
      int64_t m0;
      int n0, kbeg, nk;
      const int z = item_coords(item, m0, n0, kbeg, nk);
      n0 += chalf * EW;  // this warp's columns
      const int64_t rbase = m0 + q * 32;
      const int nrows = P.M - rbase < 32 ? static_cast<int>(P.M - rbase) : 32;
      const uint32_t u = t / kGroups;  // this group's tile count
      // with TMA stores the staging buffer is free once the store warp saw the previous
      // store read it; operand rows by TMA are loaded by the store warp itself
      const bool sw = P.tma_out && P.store_warp;
      const bool op_async = opkind && !(sw && P.op_tma);
      // staged outputs per tile (out, out2) = store-warp hand-offs per tile
      const uint32_t nout = (P.flags & (EPI_SILU_OUT2 | EPI_MUL_AUX)) ? 2u : 1u;
      if (sw) {
        if (op_async) mbar_wait(&buf_free[gr], ((u * nout) & 1) ^ 1);
      } else if (lane == 0) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // own previous store
      }
      __syncwarp();
      if (q == 0 && gr == 0 && chalf == 0) EGN_TRACE(15, t);
      // prefetch this warp's operand rows into the swizzled buffer (16 B cp.async,
      // two rows per instruction), overlapped with the main loop
      if (op_async) {
        int32_t gi = 0;
        if (opkind == 2 && lane < nrows) gi = P.gidx[rbase + lane];
        const int half = lane >> 4, gcol = lane & 15;  // 16 granules = 64 columns per row
        const int ch = gcol >> 3, g = gcol & 7;
        for (int rr = half; rr < 32; rr += 2) {
          const int32_t grow = __shfl_sync(0xffffffffu, gi, rr);
          if (rr < nrows && n0 + gcol * 4 < P.N) {
            const int64_t row = rbase + rr;
            const float* src = opkind == 1 ? P.resid + row * P.ldr
                             : opkind == 2 ? P.gsrc + static_cast<int64_t>(grow) * P.ldg
                                           : P.aux + row * P.ldaux;
            float* dst = ebuf + ch * 1024 + rr * 32 + ((g ^ (rr & 7)) << 2);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src + n0 + gcol * 4)
                         : "memory");
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
      float acc[EW];
#pragma unroll
      for (int i = 0; i < EW; ++i) acc[i] = 0.f;
      const int nsteps = nk * (BK / 8);
      const int win = P.flush_steps > 0 ? P.flush_steps : nsteps;
      const int nflush = nsteps > 0 ? (nsteps + win - 1) / win : 0;
      for (int j = 0; j < nflush; ++j, ++fcount) {
        const uint32_t b = fcount % kAccBufs;
        mbar_wait(&accf_bar[gr][b], (fcount / kAccBufs) & 1);
        if (q == 0 && gr == 0 && chalf == 0) EGN_TRACE(5, fcount);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t base = tg + b * BN;
#pragma unroll
        for (int c = 0; c < EW; c += 16) {
          if (P.dbg & 4) break;
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
      if (q == 0 && gr == 0 && chalf == 0) EGN_TRACE(6, t);
      if (P.tma_out && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapOut) : "memory");
      if (op_async) asm volatile("cp.async.wait_all;" ::: "memory");
      else if (opkind) mbar_wait(&op_bar[gr], u & 1);
      else if (sw) mbar_wait(&buf_free[gr], ((u * nout) & 1) ^ 1);
      __syncwarp();
      if (q == 0 && gr == 0 && chalf == 0) EGN_TRACE(8, t);
      // thread = row: combine with the operand in place.  Variant loops are
      // hoisted so each unrolled body is branch-free; an additive bias is applied
      // in the copy-out (lane = column), a bias under a product here.
      const int fl = P.flags;
      const bool has_bias = fl & EPI_BIAS;
      const int variant = opkind == 0 ? 0 : (fl & (EPI_RESID | EPI_GATHER)) ? 1 : (fl & EPI_DSILU_AUX) ? 2 : 3;
#define EGN_SLOT(c4) reinterpret_cast<float4*>(ebuf + ((c4) >> 3) * 1024 + epi_idx(lane, ((c4) & 7) * 4))
#define EGN_ACC4(c4) make_float4(acc[(c4) * 4], acc[(c4) * 4 + 1], acc[(c4) * 4 + 2], acc[(c4) * 4 + 3])
      const bool silu2 = fl & EPI_SILU_OUT2;
      const bool tma_store = P.tma_out;  // two outputs only with the store warp
      if (tma_store && has_bias && variant <= 1) {
        // bias here (the TMA store has no lane = column pass); broadcast loads, 16 B
        // when the bias vector is aligned
        const bool b16 = (reinterpret_cast<uintptr_t>(P.bias) & 15) == 0;
#pragma unroll
        for (int c4 = 0; c4 < EW / 4; ++c4) {
          const int col = min(n0 + c4 * 4, P.N - 4);
          const float4 bv = b16 ? __ldg(reinterpret_cast<const float4*>(P.bias + col))
                                : make_float4(__ldg(P.bias + col), __ldg(P.bias + col + 1), __ldg(P.bias + col + 2),
                                              __ldg(P.bias + col + 3));
          float4 a = EGN_ACC4(c4);
          if (variant == 1) {
            const float4 o = *EGN_SLOT(c4);
            a.x += o.x; a.y += o.y; a.z += o.z; a.w += o.w;
          }
          *EGN_SLOT(c4) = make_float4(a.x + bv.x, a.y + bv.y, a.z + bv.z, a.w + bv.w);
        }
      } else if (variant == 0) {
#pragma unroll
        for (int c4 = 0; c4 < EW / 4; ++c4) *EGN_SLOT(c4) = EGN_ACC4(c4);
      } else if (variant == 1) {
#pragma unroll
        for (int c4 = 0; c4 < EW / 4; ++c4) {
          const float4 o = *EGN_SLOT(c4);
          const float4 a = EGN_ACC4(c4);
          *EGN_SLOT(c4) = make_float4(a.x + o.x, a.y + o.y, a.z + o.z, a.w + o.w);
        }
      } else {
        const bool dsl = variant == 2;
#pragma unroll
        for (int c4 = 0; c4 < EW / 4; ++c4) {
          const float4 o = *EGN_SLOT(c4);
          float4 a = EGN_ACC4(c4);
          const int col = n0 + c4 * 4;
          if (has_bias && col < P.N) {
            a.x += __ldg(P.bias + col); a.y += __ldg(P.bias + col + 1);
            a.z += __ldg(P.bias + col + 2); a.w += __ldg(P.bias + col + 3);
          }
          const float4 f = dsl ? make_float4(dsilu(o.x), dsilu(o.y), dsilu(o.z), dsilu(o.w)) : o;
          *EGN_SLOT(c4) = make_float4(a.x * f.x, a.y * f.y, a.z * f.z, a.w * f.w);
        }
      }
      if (tma_store) {
        if (q == 0 && gr == 0 && chalf == 0) EGN_TRACE(13, t);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (q == 0 && gr == 0 && chalf == 0) EGN_TRACE(14, t);
        if (lane == 0) {
          if (sw) {
            mbar_arrive(&epi_full[gr]);  // the store warp takes it from here
          } else {  // (single output only)
            // [split][M][N] output map: rows >= M clip per split
            tma_store_3d(&mapOut, ebuf, n0, static_cast<int>(rbase), z);
            if (n0 + 32 < P.N) tma_store_3d(&mapOut, ebuf + 1024, n0 + 32, static_cast<int>(rbase), z);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        if (sw && nout == 2) {
          // second output through the same staging buffer once the first store read it:
          // silu(out) in place, or the pre-gate value
          mbar_wait(&buf_free[gr], (u * 2) & 1);
          if (silu2) {
#pragma unroll
            for (int c4 = 0; c4 < EW / 4; ++c4) {
              const float4 v = *EGN_SLOT(c4);
              *EGN_SLOT(c4) = make_float4(__fdividef(v.x, 1.f + __expf(-v.x)), __fdividef(v.y, 1.f + __expf(-v.y)),
                                          __fdividef(v.z, 1.f + __expf(-v.z)), __fdividef(v.w, 1.f + __expf(-v.w)));
            }
          } else {
#pragma unroll
            for (int c4 = 0; c4 < EW / 4; ++c4) {
              float4 a = EGN_ACC4(c4);
              if (has_bias) {
                const int col = min(n0 + c4 * 4, P.N - 4);
                a.x += __ldg(P.bias + col); a.y += __ldg(P.bias + col + 1);
                a.z += __ldg(P.bias + col + 2); a.w += __ldg(P.bias + col + 3);
              }
              *EGN_SLOT(c4) = a;
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&epi_full[gr]);
        }
        if (q == 0 && gr == 0 && chalf == 0) EGN_TRACE(9, t);
        continue;
      }
      __syncwarp();
      if (q == 0 && gr == 0 && chalf == 0) EGN_TRACE(9, t);
      float* out_base = P.out + static_cast<int64_t>(z) * P.split_stride;
      const int64_t ldo = P.ldo, ldo2 = P.ldo2;
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        const int col = n0 + ch * 32 + lane;
        if (col < P.N) {
          const float b = (variant <= 1 && has_bias) ? __ldg(P.bias + col) : 0.f;
          const float* src = ebuf + ch * 1024;
          float* dst = out_base + rbase * ldo + col;
          if (!silu2) {
#pragma unroll 8
            for (int rr = 0; rr < nrows; ++rr) dst[rr * ldo] = src[epi_idx(rr, lane)] + b;
          } else {
            float* dst2 = P.out2 + rbase * ldo2 + col;
#pragma unroll 4
            for (int rr = 0; rr < nrows; ++rr) {
              const float v = src[epi_idx(rr, lane)] + b;
              dst[rr * ldo] = v;
              dst2[rr * ldo2] = __fdividef(v, 1.f + __expf(-v));
            }
          }
        }
      }
      if (q == 0 && gr == 0 && chalf == 0) EGN_TRACE(10, t);
      if (variant == 3) {
        // out2 = the pre-gate value acc + bias: second pass through the buffer
        __syncwarp();
#pragma unroll
        for (int c4 = 0; c4 < EW / 4; ++c4) *EGN_SLOT(c4) = EGN_ACC4(c4);
        __syncwarp();
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          const int col = n0 + ch * 32 + lane;
          if (col < P.N) {
            const float b = has_bias ? __ldg(P.bias + col) : 0.f;
            const float* src = ebuf + ch * 1024;
            float* dst2 = P.out2 + rbase * ldo2 + col;
#pragma unroll 8
            for (int rr = 0; rr < nrows; ++rr) dst2[rr * ldo2] = src[epi_idx(rr, lane)] + b;
          }
        }
      }
#undef EGN_SLOT
#undef EGN_ACC4
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp == 15) {
    // ---------------- B_lo loader (BLO): the precomputed lo tile of each k-block into the
    // operand slot, once the MMAs that read the slot's previous contents completed
    if constexpr (BLO) {
      uint32_t it = 0;
      for (int item = blockIdx.x; item < total_items; item += gridDim.x) {
        int64_t m0;
        int n0, kbeg, nk;
        item_coords(item, m0, n0, kbeg, nk);
        for (int kbl = 0; kbl < nk; ++kbl, ++it) {
          const int o = it % kOpRing;
          mbar_wait(&op_empty[o], ((it / kOpRing) & 1) ^ 1);
          if (elect_one()) {
            mbar_expect_tx(&blo_full[o], B_BYTES);
            const int kb = kbeg + kbl;
            const bool first = kb < nk0;
            const int kk = (first ? kb : kb - nk0) * BK;
            const CUtensorMap* mb = first ? &mapBlo0 : &mapBlo1;
            uint8_t* dst = opring + o * kOpSlot;
            if (BMN) {
#pragma unroll
              for (int i = 0; i < BN / 32; ++i) tma_load_2d(dst + i * 4096, mb, &blo_full[o], n0 + 32 * i, kk);
            } else {
              tma_load_2d(dst, mb, &blo_full[o], kk, n0);
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (P.tma_out && P.store_warp) {
    // ---------------- store warp: TMA-stores each finished tile from the staging
    // buffers, then refills them with the operand rows of the group's next tile
    const int opkind = (P.flags & EPI_RESID) ? 1 : ((P.flags & (EPI_DSILU_AUX | EPI_MUL_AUX)) ? 3 : 0);
    const bool op_tma = P.op_tma && opkind && !(P.flags & EPI_GATHER);
    const uint32_t nout = (P.flags & (EPI_SILU_OUT2 | EPI_MUL_AUX)) ? 2u : 1u;
    constexpr int kWarps = 8 / kGroups;
    // staging buffer (g, w) belongs to epilogue warp 6 + g * kWarps + w: rows of its TMEM
    // lane quarter (warp % 4), columns of its half (one-group layout)
    auto warp_box = [&](int item, int g, int w, int64_t& rb, int& nn, int& z) {
      int64_t m0;
      int n0, kbeg, nk;
      z = item_coords(item, m0, n0, kbeg, nk);
      const int ew = g * kWarps + w;
      rb = m0 + ((6 + ew) & 3) * 32;
      nn = n0 + (kGroups == 2 ? 0 : (ew >> 2) * EW);
    };
    auto prefetch = [&](int item, int g) {
      if (!op_tma || item >= total_items) return;
      if (elect_one()) {
        uint32_t bytes = 0;
        for (int w = 0; w < kWarps; ++w) {
          int64_t rb;
          int nn, z;
          warp_box(item, g, w, rb, nn, z);
          bytes += (nn + 32 < P.N ? 2u : 1u) * 4096u;
        }
        mbar_expect_tx(&op_bar[g], bytes);
        for (int w = 0; w < kWarps; ++w) {
          int64_t rb;
          int nn, z;
          warp_box(item, g, w, rb, nn, z);
          float* eb = epi_all + (g * kWarps + w) * (2 * 32 * 32);
          tma_load_2d(eb, &mapOp, &op_bar[g], nn, static_cast<int>(rb));
          if (nn + 32 < P.N) tma_load_2d(eb + 1024, &mapOp, &op_bar[g], nn + 32, static_cast<int>(rb));
        }
      }
      __syncwarp();
    };
    for (int g = 0; g < kGroups; ++g) prefetch(blockIdx.x + g * gridDim.x, g);
    uint32_t t = 0;
    for (int item = blockIdx.x; item < total_items; item += gridDim.x, ++t) {
      const int g = kGroups == 2 ? static_cast<int>(t & 1) : 0;
      const uint32_t u = t / kGroups;
      for (uint32_t pass = 0; pass < nout; ++pass) {
        mbar_wait(&epi_full[g], (u * nout + pass) & 1);
        const CUtensorMap* mo = pass ? &mapOut2 : &mapOut;
        if (elect_one()) {
          for (int w = 0; w < kWarps; ++w) {
            int64_t rb;
            int nn, z;
            warp_box(item, g, w, rb, nn, z);
            const float* eb = epi_all + (g * kWarps + w) * (2 * 32 * 32);
            // [split][M][N] output map: rows >= M clip per split
            tma_store_3d(mo, eb, nn, static_cast<int>(rb), z);
            if (nn + 32 < P.N) tma_store_3d(mo, eb + 1024, nn + 32, static_cast<int>(rb), z);
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          mbar_arrive(&buf_free[g]);
        }
        __syncwarp();
      }
      prefetch(item + kGroups * gridDim.x, g);
    }
    if (elect_one()) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  if (P.trace && tid == 32) {
    long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    P.trace[1025 + 4 * blockIdx.x] = g;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (P.trace && tid == 32) {
    long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    P.trace[1026 + 4 * blockIdx.x] = g;
  }
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
  if (P.mcast) cluster_sync();  // no CTA leaves while its peer may still signal it
  if (P.trace && tid == 32) {
    long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    P.trace[1027 + 4 * blockIdx.x] = g;
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

// 2-D fp32 tensor maps (`outer` rows of `inner` contiguous elements, row stride ld),
// zero fill out of bounds:
//   kMapK     : box 32 (inner, 128 B) x box_outer, SWIZZLE_128B (K-major MMA operand)
//   kMapMN    : box 32 x box_outer, SWIZZLE_128B_ATOM_32B (MN-major MMA operand)
//   kMapPlain : box BM (inner) x box_outer, no swizzle (MN-major A, read by threads)
enum MapKind { kMapK, kMapMN, kMapPlain };
static int make_map(CUtensorMap* map, const float* ptr, int64_t outer, int64_t inner, int64_t ld, int box_outer,
                    MapKind kind) {
  EncodeFn enc = get_encode();
  EGN_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  EGN_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, "GEMM operand must be 16-byte aligned");
  EGN_REQUIRE((ld * 4) % 16 == 0, "GEMM operand row stride must be a multiple of 16 bytes");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 4)};
  cuuint32_t box[2] = {kind == kMapPlain ? static_cast<cuuint32_t>(BM) : 32u, static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle swz = kind == kMapK    ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : kind == kMapMN ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                                  : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  EGN_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return 0;
}

constexpr int kGemmThreads = 480;     // 14 role warps + the store warp
constexpr int kGemmThreadsBlo = 512;  // + the B_lo loader (BLO instantiations)

// Output map [splits][M][N] (row stride ld, split stride M * ld), box 32 x 32 x 1,
// SWIZZLE_128B: the epilogue buffer layout (16-byte granules XOR row % 8).
static int make_out_map(CUtensorMap* map, const float* ptr, int64_t M, int N, int64_t ld, int splits) {
  EncodeFn enc = get_encode();
  EGN_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(splits)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld * 4), static_cast<cuuint64_t>(M * ld * 4)};
  cuuint32_t box[3] = {32u, 32u, 1u};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  EGN_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (output) failed (%d)", static_cast<int>(r));
  return 0;
}

// TMA stores need a 16-byte aligned base and row stride
static bool out_map_ok(const float* out, int64_t ldo) {
  return (reinterpret_cast<uintptr_t>(out) & 15) == 0 && (ldo * 4) % 16 == 0;
}

template <bool AMN, bool BMN, int BN, bool BLO = false>
static int launch(const CUtensorMap& a0, const CUtensorMap& b0, const CUtensorMap& a1, const CUtensorMap& b1,
                  const CUtensorMap& mo, const CUtensorMap& mo2, const CUtensorMap& mop, const Params& P, int splits,
                  cudaStream_t st, const CUtensorMap* bl0 = nullptr, const CUtensorMap* bl1 = nullptr) {
  const CUtensorMap& mbl0 = bl0 ? *bl0 : b0;
  const CUtensorMap& mbl1 = bl1 ? *bl1 : b1;
  const size_t smem = Cfg<BN, true>::kSmem;
  auto kern = gemm_tf32x3_kernel<AMN, BMN, BN, BLO>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured = true;
  }
  const int tiles_m = static_cast<int>((P.M + BM - 1) / BM);
  const int tiles_n = (P.N + BN - 1) / BN;
  const int total = tiles_m * tiles_n * splits;
  int grid = std::min(total, kNumSMs);
  // CTA pairs over the two 64-column halves of a 128-column product share A by multicast
  // Opt-in (EGN_GEMM_MCAST=1): measured slower at C2 shapes (the pair runs in lockstep and the
  // loader is latency-, not L2-bandwidth-bound), kept for the wider XL products.
  static const bool mc_enabled = [] { const char* e = std::getenv("EGN_GEMM_MCAST"); return e && e[0] == '1'; }();
  if (false && mc_enabled && tiles_n == 2) {  // multicast retired: the truncation split releases TMA slots from the MMA warp
    static int max_clusters = -1;
    if (max_clusters < 0) {
      cudaLaunchConfig_t qc = {};
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = 2;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      qc.gridDim = dim3(kNumSMs, 1, 1);
      qc.blockDim = dim3(kGemmThreads, 1, 1);
      qc.dynamicSmemBytes = smem;
      qc.attrs = qa;
      qc.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &qc) != cudaSuccess) {
        cudaGetLastError();
        max_clusters = 0;
      }
    }
    if (max_clusters > 0) {
      Params Q = P;
      Q.mcast = 1;
      grid = std::min(total, 2 * max_clusters) & ~1;
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(grid, 1, 1);
      cfg.blockDim = dim3(BLO ? kGemmThreadsBlo : kGemmThreads, 1, 1);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, kern, a0, b0, a1, b1, mo, mo2, mop, mbl0, mbl1, Q, tiles_n, splits, total);
      return check_launch("gemm_tf32x3_mc");
    }
  }
  if (getenv("EGN_GEMM_TRACE")) {  // debug timeline of CTA 0 (SM cycles since its first event)
    Params Q = P;
    long long* d = nullptr;
    cudaMalloc(&d, (1024 + 4 * kNumSMs) * sizeof(long long));
    cudaMemset(d, 0, (1024 + 4 * kNumSMs) * sizeof(long long));
    static_assert(16 * 64 <= 1024, "trace rows");
    Q.trace = d;
    kern<<<grid, BLO ? kGemmThreadsBlo : kGemmThreads, smem, st>>>(a0, b0, a1, b1, mo, mo2, mop, mbl0, mbl1, Q, tiles_n, splits, total);
    long long h[1024 + 4 * kNumSMs];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    {
      long long g0 = h[1024], g1 = 0;
      for (int c = 0; c < grid; ++c) g0 = std::min(g0, h[1024 + 4 * c]);
      printf("cta entry/alloc/done/exit (us after first entry):");
      for (int c = 0; c < grid; c += 8) {
        printf("\n  %3d: %5.1f %5.1f %5.1f %5.1f", c, (h[1024 + 4 * c] - g0) * 1e-3, (h[1025 + 4 * c] - g0) * 1e-3,
               (h[1026 + 4 * c] - g0) * 1e-3, (h[1027 + 4 * c] - g0) * 1e-3);
      }
      for (int c = 0; c < grid; ++c) g1 = std::max(g1, h[1027 + 4 * c]);
      printf("\n  kernel span %.1f us\n", (g1 - g0) * 1e-3);
    }
    cudaFree(d);
    long long t0 = h[0];
    const char* names[16] = {"prod_issue", "mma_conv_ok", "conv_full_ok", "conv_done", "mma_issued", "acc0_flush",
                             "epi0_start", "tile0_begin", "epi0_opwait", "epi0_rows", "epi0_out", "conv_op_ok",
                             "mma_win_ok", "epi_combined", "epi_fenced", "epi_bufok"};
    for (int r = 0; r < 16; ++r) {
      printf("%-14s", names[r]);
      for (int i = 0; i < 30; ++i) printf(" %6lld", h[r * 64 + i] ? (h[r * 64 + i] - t0) / 100 : -1);
      printf("\n");
    }
    fflush(stdout);
    return check_launch("gemm_tf32x3");
  }
  static const int dbg = [] { const char* e = std::getenv("EGN_GEMM_DBG"); return e ? std::atoi(e) : 0; }();
  if (dbg) {
    Params Q = P;
    Q.dbg = dbg;
    kern<<<grid, BLO ? kGemmThreadsBlo : kGemmThreads, smem, st>>>(a0, b0, a1, b1, mo, mo2, mop, mbl0, mbl1, Q, tiles_n, splits, total);
    return check_launch("gemm_tf32x3");
  }
  kern<<<grid, BLO ? kGemmThreadsBlo : kGemmThreads, smem, st>>>(a0, b0, a1, b1, mo, mo2, mop, mbl0, mbl1, P, tiles_n, splits,
                                                                    total);
  return check_launch("gemm_tf32x3");
}

// ---------------------------------------------------------------- small-M products
// Node-level products (M = atoms, a few thousand rows) fill too few 128-row tcgen05 tiles to
// hide the pipeline latency; they run as a SIMT fp32 GEMM (32 x 64 tiles, thread = 4 x 4
// outputs, K in 32-wide shared-memory slabs, next slab prefetched into registers) with the
// same fused epilogue.  fp32 FMA in fixed order.  Up to 4096 rows (C2 node products, 2,560
// rows, stay here; the 5,298-row C1 edge products measured 4% faster per step on tcgen05 beside
// the side-stream work).
constexpr int kSimtM = 32, kSimtN = 64, kSimtK = 32;
static int64_t g_simt_max_m = [] { const char* e = std::getenv("EGN_GEMM_SIMT_MAX_M"); return e ? std::atoll(e) : 4096LL; }();
// ... and at most this many multiply-adds: the XL node products (640 x 1536 x 2048) take 4-5x
// longer on the CUDA cores than one partial wave of 128 x 64 tcgen05 tiles with their long K loop
constexpr int64_t kSimtMaxWork = int64_t(1) << 28;

// 32 x 64 tile per 128-thread CTA (thread = 4 x 4 outputs); the next K slab is fetched into
// registers while the current one is multiplied out of shared memory.
template <bool BMN>
__global__ void __launch_bounds__(128) gemm_simt_kernel(int64_t M, int N, int nseg, const float* __restrict__ a0,
                                                        int64_t lda0, const float* __restrict__ b0, int64_t ldb0,
                                                        int k0, const float* __restrict__ a1, int64_t lda1,
                                                        const float* __restrict__ b1, int64_t ldb1, int k1,
                                                        Params P) {
  __shared__ __align__(16) float As[kSimtK][kSimtM + 4];  // [k][m]
  __shared__ __align__(16) float Bs[kSimtK][kSimtN + 4];  // [k][n]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;  // ty 0..7 (4 rows), tx 0..15 (4 cols)
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kSimtM;
  const int n0 = blockIdx.y * kSimtN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  // slab loaders: A 32 x 32 (2 float4 / thread), B 64 x 32 (4 float4 / thread)
  auto load = [&](int sg, int kk, float4 (&ra)[2], float4 (&rb)[4]) {
    const float* A = sg ? a1 : a0;
    const float* B = sg ? b1 : b0;
    const int64_t lda = sg ? lda1 : lda0, ldb = sg ? ldb1 : ldb0;
    const int K = sg ? k1 : k0;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int row = (tid >> 3) + 16 * i, kq = (tid & 7) * 4;
      ra[i] = (m0 + row < M && kk + kq < K) ? __ldg(reinterpret_cast<const float4*>(A + (m0 + row) * lda + kk + kq))
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (!BMN) {
        const int row = (tid >> 3) + 16 * i, kq = (tid & 7) * 4;
        rb[i] = (n0 + row < N && kk + kq < K)
                    ? __ldg(reinterpret_cast<const float4*>(B + static_cast<int64_t>(n0 + row) * ldb + kk + kq))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        const int k = (tid >> 4) + 8 * i, nq = (tid & 15) * 4;
        rb[i] = (kk + k < K && n0 + nq < N)
                    ? __ldg(reinterpret_cast<const float4*>(B + static_cast<int64_t>(kk + k) * ldb + n0 + nq))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  };
  auto stash = [&](const float4 (&ra)[2], const float4 (&rb)[4]) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int row = (tid >> 3) + 16 * i, kq = (tid & 7) * 4;
      As[kq][row] = ra[i].x; As[kq + 1][row] = ra[i].y; As[kq + 2][row] = ra[i].z; As[kq + 3][row] = ra[i].w;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (!BMN) {
        const int row = (tid >> 3) + 16 * i, kq = (tid & 7) * 4;
        Bs[kq][row] = rb[i].x; Bs[kq + 1][row] = rb[i].y; Bs[kq + 2][row] = rb[i].z; Bs[kq + 3][row] = rb[i].w;
      } else {
        const int k = (tid >> 4) + 8 * i, nq = (tid & 15) * 4;
        *reinterpret_cast<float4*>(&Bs[k][nq]) = rb[i];
      }
    }
  };
  // flattened slab sequence over both segments
  const int ns0 = (k0 + kSimtK - 1) / kSimtK, ns = ns0 + (nseg > 1 ? (k1 + kSimtK - 1) / kSimtK : 0);
  float4 ra[2], rb[4];
  if (ns > 0) load(0, 0, ra, rb);
  for (int sl = 0; sl < ns; ++sl) {
    __syncthreads();  // previous slab consumed
    stash(ra, rb);
    __syncthreads();
    if (sl + 1 < ns) {
      const int nx = sl + 1;
      load(nx < ns0 ? 0 : 1, (nx < ns0 ? nx : nx - ns0) * kSimtK, ra, rb);  // next slab in flight
    }
#pragma unroll 8
    for (int k = 0; k < kSimtK; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
  }
  const int fl = P.flags;
  const int n = n0 + tx * 4;
  if (n >= N) return;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) break;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[j] = acc[i][j];
      if (fl & EPI_BIAS) v[j] += __ldg(P.bias + n + j);
      if (fl & EPI_RESID) v[j] += P.resid[m * P.ldr + n + j];
      if (fl & EPI_GATHER) v[j] += P.gsrc[static_cast<int64_t>(P.gidx[m]) * P.ldg + n + j];
    }
    float o[4], o2[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      o[j] = v[j];
      o2[j] = 0.f;
      if (fl & EPI_DSILU_AUX) o[j] = v[j] * dsilu(P.aux[m * P.ldaux + n + j]);
      if (fl & EPI_MUL_AUX) {
        o2[j] = v[j];
        o[j] = v[j] * P.aux[m * P.ldaux + n + j];
      }
      if (fl & EPI_SILU_OUT2) o2[j] = __fdividef(v[j], 1.f + __expf(-v[j]));
    }
    *reinterpret_cast<float4*>(P.out + m * P.ldo + n) = make_float4(o[0], o[1], o[2], o[3]);
    if (fl & (EPI_MUL_AUX | EPI_SILU_OUT2))
      *reinterpret_cast<float4*>(P.out2 + m * P.ldo2 + n) = make_float4(o2[0], o2[1], o2[2], o2[3]);
  }
}

// Whole-panel variant for K <= kPanelMaxK (the node products: K = 64 / 128 / 128 + 64).  The
// slab kernel above waits one L2/DRAM latency per 32-wide K slab with one warp per SM
// sub-partition; here every 16 B chunk of the CTA's A panel [32 x K] and B panel [64 x K]
// (or [K x 64]) is put in flight at once with cp.async (zero-filled past M / N), the
// epilogue operands are loaded into registers behind them, and PS x 128 threads split K in PS
// parts (fixed-order combine through shared memory).  PS = 4 when the grid is under half a wave
// (C1's 256-row node products: 16 CTAs, step 0.87 -> 0.85 ms); PS = 2 otherwise (4 measured
// 10.1 -> 11.7 us per call on the 160-CTA C2 node products).  (One bulk copy per row through the
// TMA engine measured slower: ~80 small copies per CTA serialise in the copy engine.)
constexpr int kPanelMaxK = 256;
constexpr int kPanelMaxSplit = 4;  // K parts (128 threads each): 2, or 4 when the grid is under half a wave
__device__ __forceinline__ void cp16_zfill(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
// Shared-memory row pitch (floats) for K-contiguous panels: pitch / 4 odd, so the eight
// 16 B reads of a quarter warp (eight consecutive rows) hit eight distinct bank quads.
__host__ __device__ __forceinline__ int panel_pitch(int K) { return ((K / 4) & 1) ? K + 8 : K + 4; }
static size_t panel_smem(int K, bool b_mn) {
  const int kp = panel_pitch(K);
  const size_t panels = static_cast<size_t>(kSimtM) * kp + (b_mn ? static_cast<size_t>(K) * (kSimtN + 4)
                                                                 : static_cast<size_t>(kSimtN) * kp);
  return sizeof(float) * std::max<size_t>(panels, kPanelMaxSplit * 4 * 4 * 128);  // >= the combine exchange
}

// CTA tile 32 x 64: thread (ty, tx) of each K part owns rows ty + 8 i (i < 4) and columns
// tx + 16 j (tx * 4 + j when BMN).
template <bool BMN, int PS>
__global__ void __launch_bounds__(128 * PS) gemm_simt_panel_kernel(int64_t M, int N, int nseg, const float* __restrict__ a0,
                                                              int64_t lda0, const float* __restrict__ b0,
                                                              int64_t ldb0, int k0, const float* __restrict__ a1,
                                                              int64_t lda1, const float* __restrict__ b1,
                                                              int64_t ldb1, int k1, Params P) {
  constexpr int kPanelSplit = PS, kPanelThreads = 128 * PS, kPanelRows = 4 / PS;
  extern __shared__ __align__(16) float psm[];
  const int K = k0 + (nseg > 1 ? k1 : 0);
  const int kp = panel_pitch(K);
  float* As = psm;                // [32][kp]     (m, k)
  float* Bs = psm + kSimtM * kp;  // [64][kp] (n, k)  or  [K][68] (k, n) when BMN
  const int tid = threadIdx.x, h = tid >> 7, t = tid & 127, tx = t & 15, ty = t >> 4;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kSimtM;
  const int n0 = blockIdx.y * kSimtN;
  const int kq = K / 4;  // 16 B chunks per K row
  // ---- issue the panels
  for (int c = tid; c < kSimtM * kq; c += kPanelThreads) {
    const int r = c / kq, k = (c - r * kq) * 4;
    const bool ok = m0 + r < M;
    const float* src = k < k0 ? a0 + (ok ? (m0 + r) * lda0 : 0) + k : a1 + (ok ? (m0 + r) * lda1 : 0) + (k - k0);
    cp16_zfill(As + r * kp + k, src, ok);
  }
  if (!BMN) {
    for (int c = tid; c < kSimtN * kq; c += kPanelThreads) {
      const int r = c / kq, k = (c - r * kq) * 4;
      const bool ok = n0 + r < N;
      const int64_t n = ok ? n0 + r : 0;
      const float* src = k < k0 ? b0 + n * ldb0 + k : b1 + n * ldb1 + (k - k0);
      cp16_zfill(Bs + r * kp + k, src, ok);
    }
  } else {
    for (int c = tid; c < K * (kSimtN / 4); c += kPanelThreads) {
      const int k = c >> 4, nq = (c & 15) * 4;
      const bool ok = n0 + nq < N;
      const float* src = k < k0 ? b0 + static_cast<int64_t>(k) * ldb0 + (ok ? n0 + nq : 0)
                                : b1 + static_cast<int64_t>(k - k0) * ldb1 + (ok ? n0 + nq : 0);
      cp16_zfill(Bs + k * (kSimtN + 4) + nq, src, ok);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  // ---- epilogue operands of the outputs this thread finishes (rows ty + 8 i, i = kPanelRows h + ii)
  const int fl = P.flags;
  auto ncol = [&](int j) { return BMN ? n0 + tx * 4 + j : n0 + tx + 16 * j; };
  float add[kPanelRows][4], aux[kPanelRows][4];
#pragma unroll
  for (int ii = 0; ii < kPanelRows; ++ii) {
    const int64_t m = m0 + ty + 8 * (kPanelRows * h + ii);
    const bool okm = m < M;
    const int64_t gr = (okm && (fl & EPI_GATHER)) ? static_cast<int64_t>(P.gidx[m]) : 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = ncol(j);
      const bool ok = okm && n < N;
      float v = 0.f;
      if (ok && (fl & EPI_BIAS)) v += __ldg(P.bias + n);
      if (ok && (fl & EPI_RESID)) v += P.resid[m * P.ldr + n];
      if (ok && (fl & EPI_GATHER)) v += P.gsrc[gr * P.ldg + n];
      add[ii][j] = v;
      aux[ii][j] = (ok && (fl & (EPI_DSILU_AUX | EPI_MUL_AUX))) ? P.aux[m * P.ldaux + n] : 0.f;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  // ---- this part's share of K (multiples of 4)
  const int kb = (K / 4) * h / kPanelSplit * 4, ke = (K / 4) * (h + 1) / kPanelSplit * 4;
  // PS == 2 (wave-filling grids, C2's node products): scalar FFMA (FFMA2 measured +0.2% C2 step);
  // PS == 4 (small grids, C1): packed FFMA2 (C1 step 0.845 -> 0.817 ms)
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  if constexpr (PS == 2) {
#pragma unroll 2
    for (int k = kb; k < ke; k += 4) {
      float4 a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = *reinterpret_cast<const float4*>(As + (ty + 8 * i) * kp + k);
      if (!BMN) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 b = *reinterpret_cast<const float4*>(Bs + (tx + 16 * j) * kp + k);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            acc[i][j] = fmaf(a[i].x, b.x, acc[i][j]);
            acc[i][j] = fmaf(a[i].y, b.y, acc[i][j]);
            acc[i][j] = fmaf(a[i].z, b.z, acc[i][j]);
            acc[i][j] = fmaf(a[i].w, b.w, acc[i][j]);
          }
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float4 b = *reinterpret_cast<const float4*>(Bs + (k + kk) * (kSimtN + 4) + tx * 4);
          const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float av = kk == 0 ? a[i].x : kk == 1 ? a[i].y : kk == 2 ? a[i].z : a[i].w;
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av, bv[j], acc[i][j]);
          }
        }
      }
    }
  } else {
    // packed FFMA2 accumulators: K-major B pairs even / odd k (two partial sums per output,
    // added at the end); MN-major B pairs adjacent columns (the same per-element order as FFMA)
    float2 acc2[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc2[i][j] = make_float2(0.f, 0.f);
#pragma unroll 2
    for (int k = kb; k < ke; k += 4) {
      float4 a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = *reinterpret_cast<const float4*>(As + (ty + 8 * i) * kp + k);
      if (!BMN) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 b = *reinterpret_cast<const float4*>(Bs + (tx + 16 * j) * kp + k);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            acc2[i][j] = __ffma2_rn(make_float2(a[i].x, a[i].y), make_float2(b.x, b.y), acc2[i][j]);
            acc2[i][j] = __ffma2_rn(make_float2(a[i].z, a[i].w), make_float2(b.z, b.w), acc2[i][j]);
          }
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float4 b = *reinterpret_cast<const float4*>(Bs + (k + kk) * (kSimtN + 4) + tx * 4);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float av = kk == 0 ? a[i].x : kk == 1 ? a[i].y : kk == 2 ? a[i].z : a[i].w;
            const float2 av2 = make_float2(av, av);
            // columns (0, 1) and (2, 3) of the thread: acc2[i][0] / acc2[i][1] hold them packed
            acc2[i][0] = __ffma2_rn(av2, make_float2(b.x, b.y), acc2[i][0]);
            acc2[i][1] = __ffma2_rn(av2, make_float2(b.z, b.w), acc2[i][1]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (!BMN) {
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = acc2[i][j].x + acc2[i][j].y;
      } else {
        acc[i][0] = acc2[i][0].x;
        acc[i][1] = acc2[i][0].y;
        acc[i][2] = acc2[i][1].x;
        acc[i][3] = acc2[i][1].y;
      }
    }
  }
  // ---- combine the parts: every part parks its 16 partial sums, then part h adds the
  // kPanelSplit partials of its rows in K order (the same order for every element)
  __syncthreads();  // panels consumed
  float* xch = psm;  // [kPanelSplit parts][4 rows][4][128 threads]
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) xch[((h * 4 + i) * 4 + j) * 128 + t] = acc[i][j];
  __syncthreads();
#pragma unroll
  for (int ii = 0; ii < kPanelRows; ++ii) {
    const int i = kPanelRows * h + ii;
    const int64_t m = m0 + ty + 8 * i;
    if (m >= M) continue;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float sum = xch[(i * 4 + j) * 128 + t];
#pragma unroll
      for (int p = 1; p < kPanelSplit; ++p) sum += xch[((p * 4 + i) * 4 + j) * 128 + t];
      v[j] = sum + add[ii][j];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = ncol(j);
      if (n >= N) continue;
      float o = v[j], o2 = 0.f;
      if (fl & EPI_DSILU_AUX) o = v[j] * dsilu(aux[ii][j]);
      if (fl & EPI_MUL_AUX) {
        o2 = v[j];
        o = v[j] * aux[ii][j];
      }
      if (fl & EPI_SILU_OUT2) o2 = __fdividef(v[j], 1.f + __expf(-v[j]));
      P.out[m * P.ldo + n] = o;
      if (fl & (EPI_MUL_AUX | EPI_SILU_OUT2)) P.out2[m * P.ldo2 + n] = o2;
    }
  }
}

// Weight gradient over few rows (node rows): out[z][m][n] = sum_{r in split z} g[r][m] x[r][n]
// as an fp32 SIMT product (32 x 64 output tile per 128-thread CTA, 32-row slabs, next slab
// prefetched into registers), plus the split's column sums of g (n-block 0 only); the
// partials are summed by reduce_splits_kernel in fixed order.
__global__ void __launch_bounds__(128) wgrad_simt_kernel(int64_t R, int M, int N, const float* __restrict__ g,
                                                         int64_t ldg, const float* __restrict__ x, int64_t ldx,
                                                         int rows_per_split, float* __restrict__ part,
                                                         float* __restrict__ gpart) {
  __shared__ __align__(16) float As[kSimtK][kSimtM + 4];  // [r][m]
  __shared__ __align__(16) float Bs[kSimtK][kSimtN + 4];  // [r][n]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int tiles_m = (M + kSimtM - 1) / kSimtM;
  const int m0 = (blockIdx.x % tiles_m) * kSimtM;
  const int n0 = (blockIdx.x / tiles_m) * kSimtN;
  const int z = blockIdx.y;
  const int64_t r_beg = static_cast<int64_t>(z) * rows_per_split;
  const int64_t r_end = r_beg + rows_per_split < R ? r_beg + rows_per_split : R;
  float acc[4][4], cs[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  auto load = [&](int64_t r0, float4 (&ra)[2], float4 (&rb)[4]) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {  // g slab [32 r][32 m]
      const int r = (tid >> 3) + 16 * i, mq = (tid & 7) * 4;
      ra[i] = (r0 + r < r_end && m0 + mq < M) ? __ldg(reinterpret_cast<const float4*>(g + (r0 + r) * ldg + m0 + mq))
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // x slab [32 r][64 n]
      const int r = (tid >> 4) + 8 * i, nq = (tid & 15) * 4;
      rb[i] = (r0 + r < r_end && n0 + nq < N) ? __ldg(reinterpret_cast<const float4*>(x + (r0 + r) * ldx + n0 + nq))
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  float4 ra[2], rb[4];
  if (r_beg < r_end) load(r_beg, ra, rb);
  for (int64_t r0 = r_beg; r0 < r_end; r0 += kSimtK) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i) *reinterpret_cast<float4*>(&As[(tid >> 3) + 16 * i][(tid & 7) * 4]) = ra[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) *reinterpret_cast<float4*>(&Bs[(tid >> 4) + 8 * i][(tid & 15) * 4]) = rb[i];
    __syncthreads();
    if (r0 + kSimtK < r_end) load(r0 + kSimtK, ra, rb);
#pragma unroll 8
    for (int k = 0; k < kSimtK; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        cs[i] += av[i];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
    }
  }
  float* out = part + static_cast<int64_t>(z) * M * N;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    const int n = n0 + tx * 4;
    if (m < M && n < N) *reinterpret_cast<float4*>(out + static_cast<int64_t>(m) * N + n) =
        make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    if (gpart != nullptr && n0 == 0 && tx == 0 && m < M) gpart[static_cast<int64_t>(z) * M + m] = cs[i];
  }
}

// Whole-panel variant of wgrad_simt_kernel for splits of at most kPanelMaxRows rows: the
// split's g [rows x 32] and x [rows x 64] panels are put in flight at once (cp.async), and
// 256 threads take half the rows each, combined low rows first.
constexpr int kPanelMaxRows = 128;
__global__ void __launch_bounds__(256) wgrad_simt_panel_kernel(int64_t R, int M, int N, const float* __restrict__ g,
                                                               int64_t ldg, const float* __restrict__ x, int64_t ldx,
                                                               int rows_per_split, float* __restrict__ part,
                                                               float* __restrict__ gpart) {
  extern __shared__ __align__(16) float psm[];
  float(*Gs)[kSimtM + 4] = reinterpret_cast<float(*)[kSimtM + 4]>(psm);                                  // [r][m]
  float(*Xs)[kSimtN + 4] = reinterpret_cast<float(*)[kSimtN + 4]>(psm + kPanelMaxRows * (kSimtM + 4));  // [r][n]
  const int tid = threadIdx.x, h = tid >> 7, t = tid & 127, tx = t & 15, ty = t >> 4;
  const int tiles_m = (M + kSimtM - 1) / kSimtM;
  const int m0 = (blockIdx.x % tiles_m) * kSimtM;
  const int n0 = (blockIdx.x / tiles_m) * kSimtN;
  const int z = blockIdx.y;
  const int64_t r_beg = static_cast<int64_t>(z) * rows_per_split;
  const int64_t r_end = r_beg + rows_per_split < R ? r_beg + rows_per_split : R;
  const int rows = r_end > r_beg ? static_cast<int>(r_end - r_beg) : 0;
  for (int c = tid; c < rows * (kSimtM / 4); c += 256) {
    const int r = c >> 3, mq = (c & 7) * 4;
    const bool ok = m0 + mq < M;
    cp16_zfill(&Gs[r][mq], g + (r_beg + r) * ldg + (ok ? m0 + mq : 0), ok);
  }
  for (int c = tid; c < rows * (kSimtN / 4); c += 256) {
    const int r = c >> 4, nq = (c & 15) * 4;
    const bool ok = n0 + nq < N;
    cp16_zfill(&Xs[r][nq], x + (r_beg + r) * ldx + (ok ? n0 + nq : 0), ok);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const int rh = rows / 2;
  const int rb = h ? rh : 0, re = h ? rows : rh;
  float acc[4][4], cs[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  // packed FFMA2 over column pairs (j, j + 1): per element the same fma sequence as FFMA
  float2 acc2[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc2[i][0] = acc2[i][1] = make_float2(0.f, 0.f);
#pragma unroll 4
  for (int r = rb; r < re; ++r) {
    const float4 a = *reinterpret_cast<const float4*>(&Gs[r][ty * 4]);
    const float4 b = *reinterpret_cast<const float4*>(&Xs[r][tx * 4]);
    const float av[4] = {a.x, a.y, a.z, a.w};
    const float2 b01 = make_float2(b.x, b.y), b23 = make_float2(b.z, b.w);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      cs[i] += av[i];
      const float2 a2 = make_float2(av[i], av[i]);
      acc2[i][0] = __ffma2_rn(a2, b01, acc2[i][0]);
      acc2[i][1] = __ffma2_rn(a2, b23, acc2[i][1]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    acc[i][0] = acc2[i][0].x;
    acc[i][1] = acc2[i][0].y;
    acc[i][2] = acc2[i][1].x;
    acc[i][3] = acc2[i][1].y;
  }
  __syncthreads();  // panels consumed
  float* xch = &Gs[0][0];  // [2 halves][2 rows][5][128 threads] (4 products + column sum)
#pragma unroll
  for (int ii = 0; ii < 2; ++ii) {
#pragma unroll
    for (int j = 0; j < 4; ++j) xch[((h * 2 + ii) * 5 + j) * 128 + t] = h ? acc[ii][j] : acc[2 + ii][j];
    xch[((h * 2 + ii) * 5 + 4) * 128 + t] = h ? cs[ii] : cs[2 + ii];
  }
  __syncthreads();
  float* out = part + static_cast<int64_t>(z) * M * N;
#pragma unroll
  for (int ii = 0; ii < 2; ++ii) {
    const int i = 2 * h + ii;
    const int m = m0 + ty * 4 + i;
    const int n = n0 + tx * 4;
    const float* o = xch + (((1 - h) * 2 + ii) * 5) * 128 + t;
    float v[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const float mine = j < 4 ? (h ? acc[2 + ii][j] : acc[ii][j]) : (h ? cs[2 + ii] : cs[ii]);
      v[j] = h ? o[j * 128] + mine : mine + o[j * 128];
    }
    if (m < M && n < N) *reinterpret_cast<float4*>(out + static_cast<int64_t>(m) * N + n) = make_float4(v[0], v[1], v[2], v[3]);
    if (gpart != nullptr && n0 == 0 && tx == 0 && m < M) gpart[static_cast<int64_t>(z) * M + m] = v[4];
  }
}

// Fixed-order sum of the split-K partials: elements [0, len) of the [splits][M][N]
// matrix partials go to out (row stride ldo), elements [len, len + mg) of the
// [splits][M] column-sum partials go to gout.
__global__ void reduce_splits_kernel(const float* __restrict__ part, int splits, int64_t len, int n,
                                     float* __restrict__ out, int64_t ldo, const float* __restrict__ gpart, int mg,
                                     float* __restrict__ gout, int accumulate) {
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t total = len + mg;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * 32; base < total;
       base += static_cast<int64_t>(gridDim.x) * 32) {
    const int64_t i = base + lane;
    const bool second = i >= len;
    const float* src = second ? gpart + (i - len) : part + i;
    const int64_t stride = second ? mg : len;
    float s0 = 0.f, s1 = 0.f;
    if (i < total) {
      int z = w;
      for (; z + 8 < splits; z += 16) {
        s0 += src[z * stride];
        s1 += src[(z + 8) * stride];
      }
      if (z < splits) s0 += src[z * stride];
    }
    red[w][lane] = s0 + s1;
    __syncthreads();
    if (w == 0 && i < total) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) s += red[k][lane];
      float* dst = second ? gout + (i - len) : out + (i / n) * ldo + (i % n);
      *dst = accumulate ? *dst + s : s;
    }
    __syncthreads();
  }
}

// Tile width: 128 columns (N = 128 MMAs, one A k-block per 128 x 128 tile, store warp)
// when N allows and there is at least a wave of such tiles; else 64 (two accumulator
// groups, more CTAs for small products).
// 128-wide tiles also whenever they alone fill a wave (wide XL products: N = 128 MMAs halve
// the per-k-block issue and split work per output; 64-wide tiles measured 31% tensor-pipe busy
// at 14,792 x 2048 x 2048).
static int tile_n(int64_t M, int N) {
  const int64_t tiles128 = (M + BM - 1) / BM * ((N + 127) / 128);
  if (N >= 256 && tiles128 >= 2 * kNumSMs) return 128;  // (a partial last n tile is clipped like with 64)
  return (N % 128 == 0 && M >= static_cast<int64_t>(kNumSMs) * BM) ? 128 : 64;
}
static int wgrad_tile_n(int64_t krows, int N, int M = 0) {
  const int64_t tiles128 = static_cast<int64_t>((M + BM - 1) / BM) * ((N + 127) / 128);
  // wide products: 128-wide tiles once they fill half a wave (one K range each, no split)
  if (N >= 256 && tiles128 >= kNumSMs / 2) return 128;
  return (N % 128 == 0 && krows >= static_cast<int64_t>(kNumSMs) * 8 * BK) ? 128 : 64;
}

static void wgrad_split(int64_t krows, int M, int N, int* splits, int* kbps) {
  const int BN = wgrad_tile_n(krows, N, M);
  const int tiles = static_cast<int>(((M + BM - 1) / BM) * ((N + BN - 1) / BN));
  const int nk = static_cast<int>((krows + BK - 1) / BK);
  if (nk == 0) {  // no rows: nothing to split (the entry point zero-fills the output)
    *kbps = *splits = 1;
    return;
  }
  int want = std::max(1, kNumSMs / tiles);      // one wave of CTAs
  want = std::min(want, std::max(1, nk / 4));   // >= 4 k-blocks per CTA
  *kbps = (nk + want - 1) / want;
  *splits = (nk + *kbps - 1) / *kbps;
}

// k-steps (of 8) per TMEM->register flush: one k-block for K <= 512 (small products first,
// see the MMA issuer), four for longer K (the XL products: 5% faster, still within the 2e-6
// GEMM tolerance).  EGN_GEMM_FLUSH (long K) / EGN_GEMM_FLUSH_SHORT override for precision
// experiments (values that are not multiples of 4 use the per-k8 interleaved order).
static int flush_window(bool long_k) {
  static const int lw = [] { const char* e = std::getenv("EGN_GEMM_FLUSH"); return e ? std::atoi(e) : 16; }();
  static const int sw = [] { const char* e = std::getenv("EGN_GEMM_FLUSH_SHORT"); return e ? std::atoi(e) : 4; }();
  return long_k ? lw : sw;
}

}  // namespace gemm
}  // namespace egn

using namespace egn;

extern "C" int egn_gemm_blo(int64_t M, int N, int nseg, const float* a0, int64_t lda0, const float* b0,
                            int64_t ldb0, int k0, const float* a1, int64_t lda1, const float* b1, int64_t ldb1, int k1,
                            const float* bias, const float* resid, int64_t ldr, const float* gsrc,
                            const int32_t* gidx, int64_t ldg, const float* aux, int64_t ldaux, int flags, float* out,
                            int64_t ldo, float* out2, int64_t ldo2, int b_mn, const float* b0_lo, int64_t ldb0_lo,
                            const float* b1_lo, int64_t ldb1_lo, egn_stream_t stream);

extern "C" int egn_gemm(int64_t M, int N, int nseg, const float* a0, int64_t lda0, const float* b0, int64_t ldb0,
                        int k0, const float* a1, int64_t lda1, const float* b1, int64_t ldb1, int k1,
                        const float* bias, const float* resid, int64_t ldr, const float* gsrc, const int32_t* gidx,
                        int64_t ldg, const float* aux, int64_t ldaux, int flags, float* out, int64_t ldo,
                        float* out2, int64_t ldo2, int b_mn, egn_stream_t stream) {
  return egn_gemm_blo(M, N, nseg, a0, lda0, b0, ldb0, k0, a1, lda1, b1, ldb1, k1, bias, resid, ldr, gsrc, gidx, ldg,
                      aux, ldaux, flags, out, ldo, out2, ldo2, b_mn, nullptr, 0, nullptr, 0, stream);
}

// The lo parts x - trunc_tf32(x) (tf32-rounded, as the split warps form them) of a [rows, cols]
// row-strided array, for egn_gemm_blo's B_lo operands.
namespace egn {
namespace gemm {
__global__ void tf32_lo_kernel(const float* __restrict__ x, int64_t rows, int cols, int64_t ldx, float* __restrict__ lo,
                               int64_t ldl) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols;
    const int c = static_cast<int>(i - r * cols);
    lo[r * ldl + c] = tf32_lo_trunc<true>(x[r * ldx + c]);
  }
}
}  // namespace gemm
}  // namespace egn

extern "C" int egn_tf32_lo(const float* x, int64_t rows, int cols, int64_t ldx, float* lo, int64_t ldl,
                           egn_stream_t stream) {
  if (rows == 0 || cols == 0) return 0;
  egn::gemm::tf32_lo_kernel<<<grid_for(rows * cols, 256), 256, 0, as_stream(stream)>>>(x, rows, cols, ldx, lo, ldl);
  return check_launch("tf32_lo");
}

extern "C" int egn_gemm_blo(int64_t M, int N, int nseg, const float* a0, int64_t lda0, const float* b0,
                            int64_t ldb0, int k0, const float* a1, int64_t lda1, const float* b1, int64_t ldb1, int k1,
                            const float* bias, const float* resid, int64_t ldr, const float* gsrc,
                            const int32_t* gidx, int64_t ldg, const float* aux, int64_t ldaux, int flags, float* out,
                            int64_t ldo, float* out2, int64_t ldo2, int b_mn, const float* b0_lo, int64_t ldb0_lo,
                            const float* b1_lo, int64_t ldb1_lo, egn_stream_t stream) {
  using namespace egn::gemm;
  EGN_REQUIRE(nseg == 1 || nseg == 2, "nseg must be 1 or 2");
  EGN_REQUIRE(N >= 16 && N % 16 == 0, "GEMM N must be a positive multiple of 16 (got %d)", N);
  EGN_REQUIRE(k0 > 0 && k0 % 4 == 0 && (nseg == 1 || (k1 > 0 && k1 % 4 == 0)), "GEMM K must be a multiple of 4");
  if (M == 0) return 0;
  Params P{M, N, nseg, k0, nseg > 1 ? k1 : 0, bias, resid, ldr, gsrc, gidx, ldg, aux, ldaux, flags, out, ldo, out2,
           ldo2, 0, 0};
  // small M (at most ~half a wave of 128-row tiles): SIMT fp32 path
  const bool al = (reinterpret_cast<uintptr_t>(a0) & 15) == 0 && lda0 % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(b0) & 15) == 0 && ldb0 % 4 == 0 &&
                  (nseg == 1 || ((reinterpret_cast<uintptr_t>(a1) & 15) == 0 && lda1 % 4 == 0 &&
                                 (reinterpret_cast<uintptr_t>(b1) & 15) == 0 && ldb1 % 4 == 0));
  const int64_t work = M * static_cast<int64_t>(N) * (k0 + (nseg > 1 ? k1 : 0));
  if (M <= g_simt_max_m && work <= kSimtMaxWork && al && (reinterpret_cast<uintptr_t>(out) & 15) == 0 && ldo % 4 == 0 &&
      (!(flags & (EPI_MUL_AUX | EPI_SILU_OUT2)) || ((reinterpret_cast<uintptr_t>(out2) & 15) == 0 && ldo2 % 4 == 0))) {
    const dim3 grid(static_cast<unsigned>((M + kSimtM - 1) / kSimtM), static_cast<unsigned>((N + kSimtN - 1) / kSimtN));
    cudaStream_t st = as_stream(stream);
    const int K = k0 + (nseg > 1 ? k1 : 0);
    // EGN_GEMM_PANEL=0 keeps the slab kernel (for comparison)
    static const bool panel = [] { const char* e = std::getenv("EGN_GEMM_PANEL"); return !(e && e[0] == '0'); }();
    if (panel && K <= kPanelMaxK) {
      static const bool attr = [] {
        const int mx = static_cast<int>(std::max(panel_smem(kPanelMaxK, false), panel_smem(kPanelMaxK, true)));
        cudaFuncSetAttribute(gemm_simt_panel_kernel<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(gemm_simt_panel_kernel<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(gemm_simt_panel_kernel<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(gemm_simt_panel_kernel<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        return true;
      }();
      (void)attr;
      const size_t sm = panel_smem(K, b_mn);
      const bool wide = static_cast<int64_t>(grid.x) * grid.y < kNumSMs / 2;
#define EGN_PANEL(BM_, PS_) \
  gemm_simt_panel_kernel<BM_, PS_><<<grid, 128 * PS_, sm, st>>>(M, N, nseg, a0, lda0, b0, ldb0, k0, a1, lda1, b1, ldb1, k1, P)
      if (b_mn) { if (wide) EGN_PANEL(true, 4); else EGN_PANEL(true, 2); }
      else { if (wide) EGN_PANEL(false, 4); else EGN_PANEL(false, 2); }
#undef EGN_PANEL
      return check_launch("gemm_simt_panel");
    }
    if (b_mn) gemm_simt_kernel<true><<<grid, 128, 0, st>>>(M, N, nseg, a0, lda0, b0, ldb0, k0, a1, lda1, b1, ldb1, k1, P);
    else gemm_simt_kernel<false><<<grid, 128, 0, st>>>(M, N, nseg, a0, lda0, b0, ldb0, k0, a1, lda1, b1, ldb1, k1, P);
    return check_launch("gemm_simt");
  }
  P.flush_steps = (k0 + (nseg > 1 ? k1 : 0)) > 512 ? flush_window(true) : flush_window(false);
  CUtensorMap ma0, mb0, ma1, mb1;
  const int BN = tile_n(M, N);
  // store warp for every tile width (EGN_GEMM_SW64=0 keeps the BN = 64 accumulator groups
  // issuing their own stores, for comparison)
  static const bool sw64 = [] { const char* e = std::getenv("EGN_GEMM_SW64"); return !(e && e[0] == '0'); }();
  P.store_warp = BN == 128 || sw64;
  // A: K-major [M, K]; B: K-major [N, K] (weights (out, in)) or MN-major [K, N] (b_mn)
  if (int rc = make_map(&ma0, a0, M, k0, lda0, BM, kMapK)) return rc;
  if (int rc = b_mn ? make_map(&mb0, b0, k0, N, ldb0, BK, kMapMN) : make_map(&mb0, b0, N, k0, ldb0, BN, kMapK)) return rc;
  // precomputed B_lo (both segments, 16-byte aligned rows): loaded by TMA instead of formed by
  // the split warps (same values, bit-identical products)
  CUtensorMap mbl0 = mb0, mbl1 = mb0;
  const bool blo = b0_lo != nullptr && (nseg == 1 || b1_lo != nullptr) &&
                   (reinterpret_cast<uintptr_t>(b0_lo) & 15) == 0 && ldb0_lo % 4 == 0 &&
                   (nseg == 1 || ((reinterpret_cast<uintptr_t>(b1_lo) & 15) == 0 && ldb1_lo % 4 == 0));
  if (blo) {
    if (int rc = b_mn ? make_map(&mbl0, b0_lo, k0, N, ldb0_lo, BK, kMapMN) : make_map(&mbl0, b0_lo, N, k0, ldb0_lo, BN, kMapK))
      return rc;
    if (nseg > 1)
      if (int rc = b_mn ? make_map(&mbl1, b1_lo, k1, N, ldb1_lo, BK, kMapMN) : make_map(&mbl1, b1_lo, N, k1, ldb1_lo, BN, kMapK))
        return rc;
  }
  if (nseg > 1) {
    if (int rc = make_map(&ma1, a1, M, k1, lda1, BM, kMapK)) return rc;
    if (int rc = b_mn ? make_map(&mb1, b1, k1, N, ldb1, BK, kMapMN) : make_map(&mb1, b1, N, k1, ldb1, BN, kMapK)) return rc;
  } else {
    ma1 = ma0;
    mb1 = mb0;
  }
  CUtensorMap mo = ma0;
  static const bool no_tma_out = std::getenv("EGN_GEMM_NO_TMA_OUT") != nullptr;
  CUtensorMap mo2 = ma0;
  // two outputs (SiLU / gate) go through TMA only with the store warp (it sequences the
  // two stores through one staging buffer)
  const bool two_out = flags & (EPI_SILU_OUT2 | EPI_MUL_AUX);
  if (!no_tma_out && out_map_ok(out, ldo) && (!two_out || (P.store_warp && out_map_ok(out2, ldo2)))) {
    if (int rc = make_out_map(&mo, out, M, N, ldo, 1)) return rc;
    if (two_out)
      if (int rc = make_out_map(&mo2, out2, M, N, ldo2, 1)) return rc;
    P.tma_out = 1;
  }
  // residual / aux rows by TMA into the staging buffers (the store warp loads them)
  CUtensorMap mop = ma0;
  const float* opnd = (flags & EPI_RESID) ? resid
                      : ((flags & (EPI_DSILU_AUX | EPI_MUL_AUX)) && !(flags & EPI_GATHER)) ? aux : nullptr;
  const int64_t ldop = (flags & EPI_RESID) ? ldr : ldaux;
  if (P.tma_out && P.store_warp && opnd != nullptr && out_map_ok(opnd, ldop)) {
    if (int rc = make_map(&mop, opnd, M, N, ldop, 32, kMapK)) return rc;
    P.op_tma = 1;
  }
  cudaStream_t st = as_stream(stream);
#define EGN_GEMM_LAUNCH(BMN_, BN_)                                                                        \
  return blo ? launch<false, BMN_, BN_, true>(ma0, mb0, ma1, mb1, mo, mo2, mop, P, 1, st, &mbl0, &mbl1)   \
             : launch<false, BMN_, BN_, false>(ma0, mb0, ma1, mb1, mo, mo2, mop, P, 1, st, &mbl0, &mbl1)
  if (BN == 128) {
    if (b_mn) EGN_GEMM_LAUNCH(true, 128);
    EGN_GEMM_LAUNCH(false, 128);
  }
  if (b_mn) EGN_GEMM_LAUNCH(true, 64);
  EGN_GEMM_LAUNCH(false, 64);
#undef EGN_GEMM_LAUNCH
}

extern "C" int64_t egn_gemm_simt_max_m(int64_t value) {
  const int64_t old = egn::gemm::g_simt_max_m;
  if (value >= 0) egn::gemm::g_simt_max_m = value;
  return old;
}

extern "C" int64_t egn_gemm_wgrad_workspace_bytes(int64_t krows, int M, int N) {
  int splits, kbps;
  egn::gemm::wgrad_split(krows, M, N, &splits, &kbps);
  return static_cast<int64_t>(splits) * M * N * 4 + static_cast<int64_t>(splits) * M * 4;
}

extern "C" int egn_gemm_wgrad(int64_t krows, int M, int N, const float* g, int64_t ldg, const float* x,
                              int64_t ldx, float* out, int64_t ldo, float* g_colsum, int accumulate,
                              void* workspace, egn_stream_t stream) {
  using namespace egn::gemm;
  EGN_REQUIRE(M >= 1 && N >= 16 && N % 16 == 0, "wgrad needs N % 16 == 0 (got %d)", N);
  EGN_REQUIRE(ldo >= N, "wgrad output row stride must be >= N");
  cudaStream_t st = as_stream(stream);
  if (krows == 0) {
    if (!accumulate) {
      cudaMemset2DAsync(out, sizeof(float) * ldo, 0, sizeof(float) * N, M, st);
      if (g_colsum) cudaMemsetAsync(g_colsum, 0, sizeof(float) * M, st);
    }
    return check_launch("gemm_wgrad_empty");
  }
  int splits, kbps;
  wgrad_split(krows, M, N, &splits, &kbps);
  float* part = reinterpret_cast<float*>(workspace);
  if (krows <= g_simt_max_m && krows * static_cast<int64_t>(M) * N <= kSimtMaxWork &&
      (reinterpret_cast<uintptr_t>(g) & 15) == 0 && ldg % 4 == 0 &&
      (reinterpret_cast<uintptr_t>(x) & 15) == 0 && ldx % 4 == 0 && M % 4 == 0) {
    // few rows: SIMT fp32 partials over the same split plan (workspace sized by wgrad_split)
    const int rps = static_cast<int>((krows + splits - 1) / splits);
    float* gpart_s = part + static_cast<int64_t>(splits) * M * N;
    const dim3 grid(static_cast<unsigned>(((M + kSimtM - 1) / kSimtM) * ((N + kSimtN - 1) / kSimtN)),
                    static_cast<unsigned>(splits));
    static const bool panel = [] { const char* e = std::getenv("EGN_GEMM_PANEL"); return !(e && e[0] == '0'); }();
    if (panel && rps <= kPanelMaxRows) {
      constexpr int sm = kPanelMaxRows * (kSimtM + 4 + kSimtN + 4) * static_cast<int>(sizeof(float));
      static const bool attr = [] {
        cudaFuncSetAttribute(wgrad_simt_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        return true;
      }();
      (void)attr;
      wgrad_simt_panel_kernel<<<grid, 256, sm, st>>>(krows, M, N, g, ldg, x, ldx, rps, part,
                                                     g_colsum ? gpart_s : nullptr);
    } else {
      wgrad_simt_kernel<<<grid, 128, 0, st>>>(krows, M, N, g, ldg, x, ldx, rps, part, g_colsum ? gpart_s : nullptr);
    }
    if (check_launch("gemm_wgrad_simt")) return 1;
    const int64_t len = static_cast<int64_t>(M) * N;
    const int mg = g_colsum ? M : 0;
    reduce_splits_kernel<<<static_cast<int>(std::min<int64_t>((len + mg + 31) / 32, 4096)), 256, 0, st>>>(
        part, splits, len, N, out, ldo, gpart_s, mg, g_colsum, accumulate);
    return check_launch("gemm_wgrad_reduce");
  }
  Params P{M, N, 1, static_cast<int>(krows), 0, nullptr, nullptr, 0, nullptr, nullptr, 0, nullptr, 0, 0,
           part, N, nullptr, 0, kbps, flush_window(true), 0, nullptr, 0, static_cast<int64_t>(M) * N};
  CUtensorMap ma, mb;
  // A = g^T: g is [krows, M] with M contiguous (MN-major); B = x^T likewise
  if (int rc = make_map(&ma, g, krows, M, ldg, BK, kMapPlain)) return rc;
  if (int rc = make_map(&mb, x, krows, N, ldx, BK, kMapMN)) return rc;
  CUtensorMap mo = ma;
  const bool wide = wgrad_tile_n(krows, N, M) == 128;
  P.store_warp = 1;
  if (splits == 1 && !accumulate && out_map_ok(out, ldo)) {
    // one K range per tile: the tiles go straight to the output (no partial buffer, no
    // reduction pass), the column sums straight to g_colsum
    P.out = out;
    P.ldo = ldo;
    if (int rc = make_out_map(&mo, out, M, N, ldo, 1)) return rc;
    P.tma_out = 1;
    P.gsum_part = g_colsum;
    return wide ? launch<true, true, 128>(ma, mb, ma, mb, mo, ma, ma, P, 1, st)
                : launch<true, true, 64>(ma, mb, ma, mb, mo, ma, ma, P, 1, st);
  }
  if (out_map_ok(part, N)) {
    if (int rc = make_out_map(&mo, part, M, N, N, splits)) return rc;
    P.tma_out = 1;
  }
  float* gpart = part + static_cast<int64_t>(splits) * M * N;
  P.gsum_part = g_colsum ? gpart : nullptr;
  const int rc = wide ? launch<true, true, 128>(ma, mb, ma, mb, mo, ma, ma, P, splits, st)
                      : launch<true, true, 64>(ma, mb, ma, mb, mo, ma, ma, P, splits, st);
  if (rc) return rc;
  const int64_t len = static_cast<int64_t>(M) * N;
  const int mg = g_colsum ? M : 0;
  reduce_splits_kernel<<<static_cast<int>(std::min<int64_t>((len + mg + 31) / 32, 4096)), 256, 0, st>>>(
      part, splits, len, N, out, ldo, gpart, mg, g_colsum, accumulate);
  return check_launch("gemm_wgrad_reduce");
}
