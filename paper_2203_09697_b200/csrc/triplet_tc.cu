// Triplet-interaction forward on the 5th-generation tensor cores (tcgen05).
//
// For centre atom j with n out-edges (rows p) and their reverses rq = rev(off_j+q)
// (the in-edges k->j), the forward of egn_triplet_fwd is
//
//   S[off_j+p, c] = sum_{q != p} sum_l T_l(u_p . u_q) * Y[q, l, c],
//   Y[q, l, c]    = X[rq, c] * sum_k rbf_k(d_q) W[k, l, c]
//
// (record_tu, egn/engine.py:136-148, after the algebraic reorder of DESIGN.md 4.1).
// Per centre that is one GEMM with one K = 8 step per in-edge q (l padded to 8):
//
//   D[c, p] = sum_q A_q[c, 0..7] . B_q[p, 0..7],  A_q = Y[q, :, c]^T,  B_q = T(x_pq) (0 if p == q)
//
// M = channel block (64 or 128 channels), N = rows p (<= 256 per pass), fp32-accurate
// through the 3xTF32 split (A_lo.B_hi + A_hi.B_lo + A_hi.B_hi).
//
// Warp roles (416 threads, persistent CTAs over centres):
//   warps 0-7 : operand builders -- per slab of 4 in-edges they write A (thread = channel:
//               X gather, rbf, W column in registers) and B (Chebyshev table of the
//               centre's angles) as hi/lo in the K-major SWIZZLE_128B layout;
//   warp 8    : MMA issuer (one elected lane), D double-buffered in TMEM per pass;
//   warps 9-12: epilogue -- TMEM -> registers -> S rows (lanes = channels, coalesced).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"

namespace egn {
namespace tc {

constexpr int kBuilders = 256;             // warps 0-7
constexpr int kMmaWarp = kBuilders / 32;   // warp 8
constexpr int kThreads = kBuilders + 32 + 128;  // + MMA warp + 4 epilogue warps
constexpr int kQChunk = 64;                // in-edges whose X rows are staged at once
constexpr int kMaxDeg = 1024;  // centre geometry staged in shared memory
constexpr int kMaxNB = 256;    // rows p per pass (MMA N)
constexpr int kMaxK = 8;

struct Args {
  const int64_t* edge_ptr;
  const int32_t* rev;
  const float4* geo;
  int64_t nv;
  const float* X;
  const float* W;
  float* S;
  int K, L, ld, c0;  // channel block [c0, c0 + M) of rows with stride ld
  float gamma, step;
  int nbmax, nslot, gcap;  // rows per pass (TMEM columns per buffer), ring slots, staged degree cap
  int min_n;               // centres with n <= min_n are left to the CUDA-core small-degree kernel
  long long* trace;        // debug timeline (EGN_TC_TRACE): CTA 0, [role][centre]
  int qchunk;              // in-edges staged per X/rbf chunk (power of two, multiple of 4)
};
#define TC_TRACE(role, idx)                                                            \
  do {                                                                                 \
    if (a.trace && blockIdx.x == 0 && (idx) < 32 && (threadIdx.x & 31) == 0) {         \
      long long t_;                                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                           \
      a.trace[(role) * 32 + (idx)] = t_;                                               \
    }                                                                                  \
  } while (0)

template <int M>
__global__ void __launch_bounds__(kThreads, 1) fwd_kernel(Args a) {
  constexpr int A_BYTES = M * 128;
  extern __shared__ __align__(16) uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  const int B_BYTES = a.nbmax * 128;
  const int SLOT = 2 * A_BYTES + 2 * B_BYTES;
  uint8_t* ring = sm;
  float4* U = reinterpret_cast<float4*>(sm + a.nslot * SLOT);  // [gcap] centre out-edge geometry
  int32_t* RQ = reinterpret_cast<int32_t*>(U + a.gcap);        // [gcap] in-edge ids
  float* XS = reinterpret_cast<float*>(RQ + a.gcap);           // [kQChunk][M] staged X rows
  float* RB = XS + a.qchunk * M;                               // [qchunk][kMaxK] rbf values
  __shared__ __align__(8) uint64_t full[4], empty[4], dfull[2], dempty[2];
  __shared__ uint32_t tbase;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NS = a.nslot;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&dfull[b], 1);
      mbar_init(&dempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t tcols = 32;
  while (tcols < 2u * a.nbmax) tcols <<= 1;
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  if (tid == 0) TC_TRACE(7, 0);

  if (warp < kBuilders / 32) {
    // ------------------------------------------------ builders
    // thread -> channel c (fixed), k-steps j = jt, jt + JS, ... of each slab
    constexpr int JS = kBuilders / M;  // 4 (M = 64) or 2 (M = 128)
    const int c = tid % M, jt = tid / M;
    float w[kMaxK][8];
#pragma unroll
    for (int k = 0; k < kMaxK; ++k)
#pragma unroll
      for (int l = 0; l < 8; ++l)
        w[k][l] = (k < a.K && l < a.L) ? a.W[(static_cast<int64_t>(k) * a.L + l) * a.ld + a.c0 + c] : 0.f;
    uint32_t it = 0;
    int ci = -1;
    for (int64_t j = blockIdx.x; j < a.nv; j += gridDim.x) {
      const int64_t off = a.edge_ptr[j];
      const int n = static_cast<int>(a.edge_ptr[j + 1] - off);
      if (n <= 0 || n <= a.min_n) continue;
      ++ci;
      if (tid == 0) TC_TRACE(0, ci);
      named_sync(1, kBuilders);  // previous centre's readers of U/RQ are done
      for (int q = tid; q < n; q += kBuilders) {
        U[q] = a.geo[off + q];
        RQ[q] = a.rev[off + q];
      }
      named_sync(1, kBuilders);
      if (tid == 0) TC_TRACE(1, ci);
      const int nslab = (n + 3) >> 2;
      for (int p0 = 0; p0 < n; p0 += kMaxNB) {
        const int np = min(kMaxNB, n - p0);
        const int nb = (np + 15) & ~15;
        for (int s = 0; s < nslab; ++s, ++it) {
          if ((s & (a.qchunk / 4 - 1)) == 0) {
            // stage X rows and rbf values of the next qchunk in-edges (coalesced rows)
            const int q0 = 4 * s, nq = min(a.qchunk, n - q0);
            named_sync(1, kBuilders);
            for (int i = tid; i < nq * (M / 4); i += kBuilders) {
              const int qq = i / (M / 4), c4 = i - qq * (M / 4);
              *reinterpret_cast<float4*>(XS + qq * M + 4 * c4) = __ldg(reinterpret_cast<const float4*>(
                  a.X + static_cast<int64_t>(RQ[q0 + qq]) * a.ld + a.c0 + 4 * c4));
            }
            for (int i = tid; i < nq * kMaxK; i += kBuilders) {
              const int qq = i / kMaxK, k = i - qq * kMaxK;
              const float dd = U[q0 + qq].w - a.step * k;
              RB[i] = k < a.K ? __expf(-a.gamma * dd * dd) : 0.f;
            }
            named_sync(1, kBuilders);
          }
          const int slot = it % NS;
          mbar_wait(&empty[slot], ((it / NS) & 1) ^ 1);
          uint8_t* ahi = ring + slot * SLOT;
          uint8_t* alo = ahi + A_BYTES;
          uint8_t* bhi = alo + A_BYTES;
          uint8_t* blo = bhi + B_BYTES;
          // A: Y[q, l, c] for the slab's 4 in-edges
#pragma unroll
          for (int jj = 0; jj < 4 / JS; ++jj) {
            const int js = jt + jj * JS;
            const int q = 4 * s + js;
            const int qq = q & (a.qchunk - 1);
            float y[8];
            if (q < n) {
              const float x = XS[qq * M + c];
              float rb[kMaxK];
#pragma unroll
              for (int k = 0; k < kMaxK; ++k) rb[k] = RB[qq * kMaxK + k];
#pragma unroll
              for (int l = 0; l < 8; ++l) {
                float r = 0.f;
#pragma unroll
                for (int k = 0; k < kMaxK; ++k) r = fmaf(rb[k], w[k][l], r);
                y[l] = x * r;
              }
            } else {
#pragma unroll
              for (int l = 0; l < 8; ++l) y[l] = 0.f;
            }
            put8(ahi, alo, c, js, y);
          }
          // B: Chebyshev T_l(u_p . u_q), zero on the diagonal and in padding
          for (int idx = tid; idx < nb * 4; idx += kBuilders) {
            const int pr = idx >> 2, js = idx & 3;
            const int p = p0 + pr, q = 4 * s + js;
            float t[8];
            if (pr < np && q < n && p != q) {
              const float4 up = U[p], uq = U[q];
              const float xx = up.x * uq.x + up.y * uq.y + up.z * uq.z;
              t[0] = 1.f;
              t[1] = xx;
#pragma unroll
              for (int l = 2; l < 8; ++l) t[l] = 2.f * xx * t[l - 1] - t[l - 2];
#pragma unroll
              for (int l = 0; l < 8; ++l)
                if (l >= a.L) t[l] = 0.f;
            } else {
#pragma unroll
              for (int l = 0; l < 8; ++l) t[l] = 0.f;
            }
            put8(bhi, blo, pr, js, t);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          named_sync(1, kBuilders);
          if (tid == 0) mbar_arrive(&full[slot]);
        }
      }
      if (tid == 0) TC_TRACE(2, ci);
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------ MMA issuer
    uint32_t it = 0, pass = 0;
    int ci = -1;
    for (int64_t j = blockIdx.x; j < a.nv; j += gridDim.x) {
      const int64_t off = a.edge_ptr[j];
      const int n = static_cast<int>(a.edge_ptr[j + 1] - off);
      if (n <= 0 || n <= a.min_n) continue;
      ++ci;
      const int nslab = (n + 3) >> 2;
      for (int p0 = 0; p0 < n; p0 += kMaxNB, ++pass) {
        const int nb = (min(kMaxNB, n - p0) + 15) & ~15;
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(nb >> 3) << 17) |
                               (static_cast<uint32_t>(M >> 4) << 24);
        const uint32_t b = pass & 1;
        mbar_wait(&dempty[b], ((pass >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem + b * a.nbmax;
        for (int s = 0; s < nslab; ++s, ++it) {
          const int slot = it % NS;
          mbar_wait(&full[slot], (it / NS) & 1);
          if (s == 0) TC_TRACE(3, ci);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t ahi = su32(ring + slot * SLOT);
          const uint32_t alo = ahi + A_BYTES, bhi = alo + A_BYTES, blo = bhi + B_BYTES;
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t acc = (s == 0 && k == 0) ? 0u : 1u;
              mma_tf32(d, kdesc(alo + 32 * k), kdesc(bhi + 32 * k), idesc, acc);
              mma_tf32(d, kdesc(ahi + 32 * k), kdesc(blo + 32 * k), idesc, 1u);
              mma_tf32(d, kdesc(ahi + 32 * k), kdesc(bhi + 32 * k), idesc, 1u);
            }
            mma_commit(&empty[slot]);
            if (s == nslab - 1) mma_commit(&dfull[b]);
          }
          __syncwarp();
        }
        TC_TRACE(4, ci);
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 5..8)
    const int qd = warp & 3;  // TMEM lane quarter
    // M = 128: row c = 32 qd + lane; M = 64: row c = 16 qd + lane (lanes 0..15)
    const int c = M == 128 ? 32 * qd + lane : 16 * qd + lane;
    const bool active = M == 128 || lane < 16;
    uint32_t pass = 0;
    int ci = -1;
    for (int64_t j = blockIdx.x; j < a.nv; j += gridDim.x) {
      const int64_t off = a.edge_ptr[j];
      const int n = static_cast<int>(a.edge_ptr[j + 1] - off);
      if (n <= 0 || n <= a.min_n) continue;
      ++ci;
      for (int p0 = 0; p0 < n; p0 += kMaxNB, ++pass) {
        const int np = min(kMaxNB, n - p0);
        const uint32_t b = pass & 1;
        mbar_wait(&dfull[b], (pass >> 1) & 1);
        if (qd == 1) TC_TRACE(5, ci);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t taddr = tmem + b * a.nbmax + (static_cast<uint32_t>(qd * 32) << 16);
        float* dst = a.S + (off + p0) * a.ld + a.c0 + c;
        for (int cb = 0; cb < np; cb += 16) {
          uint32_t r[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
              : "r"(taddr + cb));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (active) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (cb + i < np) dst[static_cast<int64_t>(cb + i) * a.ld] = __uint_as_float(r[i]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&dempty[b]);
        if (qd == 1) TC_TRACE(6, ci);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == kMmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
}

}  // namespace tc

// ---------------------------------------------------------------------------
// host side (called from egn_triplet_fwd)
// ---------------------------------------------------------------------------
bool tc_fwd_supported(int K, int L, int dg, int max_degree) {
  static const bool enabled = [] {
    const char* e = std::getenv("EGN_TRIPLET_TC");
    return !(e && e[0] == '0');
  }();
  return enabled && K >= 1 && K <= tc::kMaxK && L >= 1 && L <= 8 && dg % 64 == 0 && max_degree >= 0 &&
         max_degree <= tc::kMaxDeg;
}

int tc_fwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, int max_degree,
           const float* X, const float* W, int K, int L, int dg, RbfParams rp, float* S, int min_n,
           cudaStream_t st) {
  const int nbmax = std::max(16, (std::min(max_degree, tc::kMaxNB) + 15) & ~15);
  for (int c0 = 0; c0 < dg; c0 += 128) {
    const int M = (dg - c0) >= 128 ? 128 : 64;
    const int slot = 2 * M * 128 + 2 * nbmax * 128;
    const int gcap = std::max(4, (max_degree + 3) & ~3);
    // ring depth 2-3 slots; the X/rbf staging chunk shrinks until everything fits
    int qchunk = tc::kQChunk;
    auto stage_bytes = [&](int qc) { return gcap * 20 + qc * (M + tc::kMaxK) * 4; };
    int nslot = 3;
    while (nslot > 2 && static_cast<size_t>(nslot) * slot + stage_bytes(qchunk) + 1024 > 72 * 1024) --nslot;
    while (qchunk > 4 && static_cast<size_t>(nslot) * slot + stage_bytes(qchunk) + 1024 > 225 * 1024) qchunk >>= 1;
    const size_t smem = static_cast<size_t>(nslot) * slot + stage_bytes(qchunk) + 1024;
    EGN_REQUIRE(smem <= 227 * 1024, "triplet_fwd_tc: %zu bytes of shared memory (max degree %d)", smem, max_degree);
    static long long* trace = nullptr;
    const bool tracing = std::getenv("EGN_TC_TRACE") != nullptr;
    if (tracing && !trace) cudaMalloc(&trace, 8 * 32 * sizeof(long long));
    if (tracing) cudaMemsetAsync(trace, 0, 8 * 32 * sizeof(long long), st);
    tc::Args a{edge_ptr, rev, geo, nv, X, W, S, K, L, dg, c0, rp.gamma, rp.step, nbmax, nslot, gcap, min_n,
               tracing ? trace : nullptr, qchunk};
    auto kern = M == 128 ? tc::fwd_kernel<128> : tc::fwd_kernel<64>;
    // host-side launch configuration is cached per (kernel, shared-memory size)
    static size_t configured[2] = {0, 0};
    static int occ[2] = {1, 1};
    const int ki = M == 128 ? 1 : 0;
    if (configured[ki] != smem) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[ki], kern, tc::kThreads, smem);
      configured[ki] = smem;
    }
    int per_sm = occ[ki];
    uint32_t tcols = 32;
    while (tcols < 2u * nbmax) tcols <<= 1;
    per_sm = std::max(1, std::min<int>(per_sm, 512 / tcols));  // TMEM: 512 columns per SM
    const int grid = static_cast<int>(std::min<int64_t>(nv, static_cast<int64_t>(kNumSMs) * per_sm));
    kern<<<grid, tc::kThreads, smem, st>>>(a);
    if (int rc = check_launch("triplet_fwd_tc")) return rc;
    if (tracing) {
      long long h[8 * 32];
      cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const char* names[8] = {"b_centre", "b_geo", "b_done", "mma_first", "mma_done", "epi_full", "epi_done",
                              "start"};
      std::printf("tc fwd trace CTA 0 (us after start), grid %d, smem %zu, per_sm %d\n", grid, smem, per_sm);
      for (int r = 0; r < 7; ++r) {
        std::printf("%-10s", names[r]);
        for (int i = 0; i < 12; ++i) std::printf(" %7.2f", h[r * 32 + i] ? (h[r * 32 + i] - h[7 * 32]) * 1e-3 : -1.0);
        std::printf("\n");
      }
    }
    if (M == 64) break;
  }
  return 0;
}

}  // namespace egn
