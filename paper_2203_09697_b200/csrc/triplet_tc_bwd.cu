// Triplet-interaction backward on the tensor cores (tcgen05), for large centres.
//
// Adjoint of the forward of triplet_tc.cu (record_tu VJPs, egn/tape.py gather /
// segment_sum / linear / angular_sbf, after the reorder of DESIGN.md 4.1).  Per
// centre j with n out-edges, S_bar rows p and in-edges rq = rev(off_j + q):
//
//   Ybar[q, l, c] = sum_{p != q} T_l(x_pq) S_bar[p, c]                  (kernel y)
//     X_bar[rq, c]   = sum_l Ybar[q, l, c] Rw[q, l, c]
//     W_bar[k, l, c] += rbf_k(d_q) Ybar[q, l, c] X[rq, c]
//     d_bar[q]       = sum_{k,l,c} rbf_k'(d_q) W[k, l, c] Ybar[q, l, c] X[rq, c]
//   Tbar[p, q, l] = sum_c S_bar[p, c] Y[q, l, c],  Y = X[rq] * Rw      (kernel a)
//     g_pq = sum_l Tbar[p, q, l] T_l'(x_pq)  ->  u_bar_p += g u_q,  u_bar_q += g u_p
//     edge_grad[off + i].xyz += (u_bar_i - (u_bar_i . u_i) u_i) / d_i
//
// Both are per-centre GEMMs in 3xTF32 with one K = 8 step per 8 rows p (kernel y,
// D[c, (q,l)], M = channel block) or per 8 channels (kernel a, D[p, (q,l)], M = 128
// rows p).  Same warp roles as the forward: 8 builder warps, 1 MMA warp, 4 epilogue
// warps; centre geometry is double-buffered and handed over with an mbarrier.
// Deterministic: per-q/per-edge sums are fixed-order, W_bar partials per CTA are
// reduced in block order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"

namespace egn {
namespace tcb {

using namespace egn::tc;

constexpr int kBuilders = 256;
constexpr int kMmaWarp = 8;
constexpr int kThreads = kBuilders + 32 + 128;
constexpr int kNQ = 16;  // in-edges per pass: N = 8 kNQ = 128 columns (q, l)
constexpr int kMaxK = 8;

struct Args {
  const int64_t* edge_ptr;
  const int32_t* rev;
  const float4* geo;
  int64_t nv;
  const float* X;
  const float* W;
  const float* Sbar;
  float* Xbar;
  float4* edge_grad;
  float* Wpart;  // kernel y: [grid][K][L][M]
  int K, L, ld, c0, dg;
  float gamma, step;
  int nslot, gcap, min_n;
};

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// common prologue: barriers, TMEM (2 buffers x 128 columns)
struct Sync {
  uint64_t full[4], empty[4], dfull[2], dempty[2], gfull[2], gfree[2];
  uint32_t tbase;
};

__device__ __forceinline__ void init_sync(Sync& sy, int nslot) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < nslot; ++s) {
      mbar_init(&sy.full[s], 1);
      mbar_init(&sy.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sy.dfull[b], 1);
      mbar_init(&sy.dempty[b], 4);
      mbar_init(&sy.gfull[b], 1);
      mbar_init(&sy.gfree[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if ((threadIdx.x >> 5) == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&sy.tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
}

__device__ __forceinline__ void mma_slab(uint32_t d, uint32_t ahi, uint32_t alo, uint32_t bhi, uint32_t blo,
                                         uint32_t idesc, bool first) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    mma_tf32(d, kdesc(alo + 32 * k), kdesc(bhi + 32 * k), idesc, (first && k == 0) ? 0u : 1u);
    mma_tf32(d, kdesc(ahi + 32 * k), kdesc(blo + 32 * k), idesc, 1u);
    mma_tf32(d, kdesc(ahi + 32 * k), kdesc(bhi + 32 * k), idesc, 1u);
  }
}

// Builders stage centre geometry into buffer (ci & 1) once the epilogue released it.
__device__ __forceinline__ void stage_geometry(const Args& a, Sync& sy, float4* U2, int32_t* RQ2, int ci,
                                               int64_t off, int n) {
  const int b = ci & 1;
  mbar_wait(&sy.gfree[b], ((ci >> 1) & 1) ^ 1);
  float4* U = U2 + b * a.gcap;
  int32_t* RQ = RQ2 + b * a.gcap;
  for (int q = threadIdx.x; q < n; q += kBuilders) {
    U[q] = a.geo[off + q];
    RQ[q] = a.rev[off + q];
  }
  named_sync(1, kBuilders);
  if (threadIdx.x == 0) mbar_arrive(&sy.gfull[b]);
}

// ============================================================================
// kernel y: Ybar = T^T S_bar per channel block, epilogue X_bar / W_bar / d_bar
// ============================================================================
template <int M>
__global__ void __launch_bounds__(kThreads, 1) y_kernel(Args a) {
  constexpr int A_BYTES = M * 128;
  constexpr int B_BYTES = 8 * kNQ * 128;
  constexpr int SLOT = 2 * A_BYTES + 2 * B_BYTES;
  extern __shared__ __align__(16) uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  uint8_t* ring = sm;
  float4* U2 = reinterpret_cast<float4*>(sm + a.nslot * SLOT);
  int32_t* RQ2 = reinterpret_cast<int32_t*>(U2 + 2 * a.gcap);
  float* Ws = reinterpret_cast<float*>(RQ2 + 2 * a.gcap);  // [kMaxK][8][M]
  __shared__ float DP[4][kNQ];
  __shared__ Sync sy;
  init_sync(sy, a.nslot);
  const uint32_t tmem = sy.tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NS = a.nslot;

  if (warp < kBuilders / 32) {
    // ------------------------------------------------ builders
    for (int i = tid; i < kMaxK * 8 * M; i += kBuilders) {
      const int k = i / (8 * M), l = (i / M) % 8, c = i % M;
      Ws[i] = (k < a.K && l < a.L) ? a.W[(static_cast<int64_t>(k) * a.L + l) * a.ld + a.c0 + c] : 0.f;
    }
    uint32_t it = 0;
    int ci = -1;
    for (int64_t j = blockIdx.x; j < a.nv; j += gridDim.x) {
      const int64_t off = a.edge_ptr[j];
      const int n = static_cast<int>(a.edge_ptr[j + 1] - off);
      if (n <= 0 || n <= a.min_n) continue;
      ++ci;
      stage_geometry(a, sy, U2, RQ2, ci, off, n);
      const float4* U = U2 + (ci & 1) * a.gcap;
      const int nslab = (n + 31) >> 5;
      for (int q0 = 0; q0 < n; q0 += kNQ) {
        const int nq = min(kNQ, n - q0);
        const int nqp = (nq + 1) & ~1;
        for (int s = 0; s < nslab; ++s, ++it) {
          const int slot = it % NS;
          mbar_wait(&sy.empty[slot], ((it / NS) & 1) ^ 1);
          uint8_t* ahi = ring + slot * SLOT;
          uint8_t* alo = ahi + A_BYTES;
          uint8_t* bhi = alo + A_BYTES;
          uint8_t* blo = bhi + B_BYTES;
          // A[c, p] = S_bar[off + p, c0 + c], 8 rows p per k-step
          for (int idx = tid; idx < M * 4; idx += kBuilders) {
            const int c = idx % M, pg = idx / M;
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int p = 32 * s + 8 * pg + i;
              v[i] = p < n ? __ldg(a.Sbar + (off + p) * a.ld + a.c0 + c) : 0.f;
            }
            put8(ahi, alo, c, pg, v);
          }
          // B[(q, l), p] = T_l(x_pq) (0 for p == q and in padding)
          for (int idx = tid; idx < nqp * 4; idx += kBuilders) {
            const int qi = idx >> 2, pg = idx & 3;
            const int q = q0 + qi;
            float t[8][8];  // [l][i]
            const float4 uq = U[min(q, n - 1)];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int p = 32 * s + 8 * pg + i;
              if (qi < nq && p < n && p != q) {
                const float4 up = U[p];
                const float xx = up.x * uq.x + up.y * uq.y + up.z * uq.z;
                float tm2 = 1.f, tm1 = xx;
                t[0][i] = 1.f;
                t[1][i] = xx;
#pragma unroll
                for (int l = 2; l < 8; ++l) {
                  const float tn = 2.f * xx * tm1 - tm2;
                  t[l][i] = tn;
                  tm2 = tm1;
                  tm1 = tn;
                }
#pragma unroll
                for (int l = 0; l < 8; ++l)
                  if (l >= a.L) t[l][i] = 0.f;
              } else {
#pragma unroll
                for (int l = 0; l < 8; ++l) t[l][i] = 0.f;
              }
            }
#pragma unroll
            for (int l = 0; l < 8; ++l) put8(bhi, blo, 8 * qi + l, pg, t[l]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          named_sync(1, kBuilders);
          if (tid == 0) mbar_arrive(&sy.full[slot]);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------ MMA issuer
    uint32_t it = 0, pass = 0;
    for (int64_t j = blockIdx.x; j < a.nv; j += gridDim.x) {
      const int64_t off = a.edge_ptr[j];
      const int n = static_cast<int>(a.edge_ptr[j + 1] - off);
      if (n <= 0 || n <= a.min_n) continue;
      const int nslab = (n + 31) >> 5;
      for (int q0 = 0; q0 < n; q0 += kNQ, ++pass) {
        const int nqp = (min(kNQ, n - q0) + 1) & ~1;
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(nqp) << 17) |
                               (static_cast<uint32_t>(M >> 4) << 24);  // N = 8 nqp -> N >> 3 = nqp
        const uint32_t b = pass & 1;
        mbar_wait(&sy.dempty[b], ((pass >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem + b * 128;
        for (int s = 0; s < nslab; ++s, ++it) {
          const int slot = it % NS;
          mbar_wait(&sy.full[slot], (it / NS) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t ahi = su32(ring + slot * SLOT);
          if (elect_one()) {
            mma_slab(d, ahi, ahi + A_BYTES, ahi + 2 * A_BYTES, ahi + 2 * A_BYTES + B_BYTES, idesc, s == 0);
            mma_commit(&sy.empty[slot]);
            if (s == nslab - 1) mma_commit(&sy.dfull[b]);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (thread = channel)
    const int qd = warp & 3;
    const int c = M == 128 ? 32 * qd + lane : 16 * qd + lane;
    const bool active = M == 128 || lane < 16;
    float wacc[kMaxK][8];
#pragma unroll
    for (int k = 0; k < kMaxK; ++k)
#pragma unroll
      for (int l = 0; l < 8; ++l) wacc[k][l] = 0.f;
    uint32_t pass = 0;
    int ci = -1;
    for (int64_t j = blockIdx.x; j < a.nv; j += gridDim.x) {
      const int64_t off = a.edge_ptr[j];
      const int n = static_cast<int>(a.edge_ptr[j + 1] - off);
      if (n <= 0 || n <= a.min_n) continue;
      ++ci;
      const int gb = ci & 1;
      mbar_wait(&sy.gfull[gb], (ci >> 1) & 1);
      const float4* U = U2 + gb * a.gcap;
      const int32_t* RQ = RQ2 + gb * a.gcap;
      for (int q0 = 0; q0 < n; q0 += kNQ, ++pass) {
        const int nq = min(kNQ, n - q0);
        const uint32_t b = pass & 1;
        mbar_wait(&sy.dfull[b], (pass >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t taddr = tmem + b * 128 + (static_cast<uint32_t>(qd * 32) << 16);
        for (int qi = 0; qi < nq; ++qi) {
          float yb[8];
          tmem_ld8(taddr + 8 * qi, yb);
          const int q = q0 + qi;
          const float d = U[q].w;
          float rb[kMaxK], rbd[kMaxK];
#pragma unroll
          for (int k = 0; k < kMaxK; ++k) {
            const float dd = d - a.step * k;
            rb[k] = k < a.K ? __expf(-a.gamma * dd * dd) : 0.f;
            rbd[k] = -2.f * a.gamma * dd * rb[k];
          }
          float dsum = 0.f;
          if (active) {
            const int64_t row = static_cast<int64_t>(RQ[q]) * a.ld + a.c0 + c;
            const float x = __ldg(a.X + row);
            float xb = 0.f;
#pragma unroll
            for (int l = 0; l < 8; ++l) {
              if (l >= a.L) break;
              float rw = 0.f, rwd = 0.f;
#pragma unroll
              for (int k = 0; k < kMaxK; ++k) {
                const float wv = Ws[(k * 8 + l) * M + c];
                rw = fmaf(rb[k], wv, rw);
                rwd = fmaf(rbd[k], wv, rwd);
              }
              xb = fmaf(yb[l], rw, xb);
              const float rbar = yb[l] * x;
              dsum = fmaf(rwd, rbar, dsum);
#pragma unroll
              for (int k = 0; k < kMaxK; ++k) wacc[k][l] = fmaf(rb[k], rbar, wacc[k][l]);
            }
            a.Xbar[row] = xb;
          }
          dsum = warp_sum(dsum);
          if (lane == 0) DP[qd][qi] = dsum;
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&sy.dempty[b]);
        named_sync(2, 128);
        const int t = tid - (kBuilders + 32);
        if (t < nq) {
          const float s = (DP[0][t] + DP[1][t]) + (DP[2][t] + DP[3][t]);
          a.edge_grad[off + q0 + t].w += s;
        }
        named_sync(2, 128);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sy.gfree[gb]);
    }
    if (active) {
      float* part = a.Wpart + static_cast<int64_t>(blockIdx.x) * a.K * a.L * M;
#pragma unroll
      for (int k = 0; k < kMaxK; ++k)
#pragma unroll
        for (int l = 0; l < 8; ++l)
          if (k < a.K && l < a.L) part[(k * a.L + l) * M + c] = wacc[k][l];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == kMmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// W_bar[(k L + l) ld + c0 + c] += sum over blocks of part[b][k][l][c] (fixed block order)
__global__ void wbar_reduce_kernel(const float* __restrict__ part, int nblocks, int KL, int M, int ld, int c0,
                                   float* __restrict__ Wbar) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= KL * M) return;
  float s = 0.f;
  for (int b = 0; b < nblocks; ++b) s += part[static_cast<int64_t>(b) * KL * M + i];
  const int kl = i / M, c = i % M;
  Wbar[static_cast<int64_t>(kl) * ld + c0 + c] += s;
}

// ============================================================================
// kernel a: Tbar = S_bar Y^T over all channels, epilogue angle adjoints
// ============================================================================
__global__ void __launch_bounds__(kThreads, 1) a_kernel(Args a) {
  constexpr int M = 128;
  constexpr int A_BYTES = M * 128;
  constexpr int B_BYTES = 8 * kNQ * 128;
  constexpr int SLOT = 2 * A_BYTES + 2 * B_BYTES;
  extern __shared__ __align__(16) uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  uint8_t* ring = sm;
  float4* U2 = reinterpret_cast<float4*>(sm + a.nslot * SLOT);
  int32_t* RQ2 = reinterpret_cast<int32_t*>(U2 + 2 * a.gcap);
  float* UB = reinterpret_cast<float*>(RQ2 + 2 * a.gcap);  // [gcap][3] u_bar of the epilogue's centre
  __shared__ float CP[4][kNQ][3];
  __shared__ Sync sy;
  init_sync(sy, a.nslot);
  const uint32_t tmem = sy.tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NS = a.nslot;
  const int nch = a.dg >> 5;  // channel slabs

  if (warp < kBuilders / 32) {
    // ------------------------------------------------ builders
    uint32_t it = 0;
    int ci = -1;
    for (int64_t j = blockIdx.x; j < a.nv; j += gridDim.x) {
      const int64_t off = a.edge_ptr[j];
      const int n = static_cast<int>(a.edge_ptr[j + 1] - off);
      if (n <= 0 || n <= a.min_n) continue;
      ++ci;
      stage_geometry(a, sy, U2, RQ2, ci, off, n);
      const float4* U = U2 + (ci & 1) * a.gcap;
      const int32_t* RQ = RQ2 + (ci & 1) * a.gcap;
      for (int p0 = 0; p0 < n; p0 += M) {
        const int np = min(M, n - p0);
        for (int q0 = 0; q0 < n; q0 += kNQ) {
          const int nq = min(kNQ, n - q0);
          const int nqp = (nq + 1) & ~1;
          for (int s = 0; s < nch; ++s, ++it) {
            const int slot = it % NS;
            mbar_wait(&sy.empty[slot], ((it / NS) & 1) ^ 1);
            uint8_t* ahi = ring + slot * SLOT;
            uint8_t* alo = ahi + A_BYTES;
            uint8_t* bhi = alo + A_BYTES;
            uint8_t* blo = bhi + B_BYTES;
            const int cs = 32 * s;
            // A[p, c] = S_bar[off + p0 + p, cs + c]
            for (int idx = tid; idx < M * 4; idx += kBuilders) {
              const int p = idx >> 2, cg = idx & 3;
              float v[8];
              if (p < np) {
                const float4* src = reinterpret_cast<const float4*>(a.Sbar + (off + p0 + p) * a.ld + cs + 8 * cg);
                const float4 v0 = __ldg(src), v1 = __ldg(src + 1);
                v[0] = v0.x; v[1] = v0.y; v[2] = v0.z; v[3] = v0.w;
                v[4] = v1.x; v[5] = v1.y; v[6] = v1.z; v[7] = v1.w;
              } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = 0.f;
              }
              put8(ahi, alo, p, cg, v);
            }
            // B[(q, l), c] = Y[q, l, c] = X[rq, c] sum_k rbf_k(d_q) W[k, l, c]; task = (q, channel
            // group of 8, pair of l)
            for (int idx = tid; idx < nqp * 16; idx += kBuilders) {
              const int qi = idx >> 4, cg = (idx >> 2) & 3, lp = idx & 3;
              const int q = q0 + qi;
              float y0[8], y1[8];
              if (qi < nq) {
                const float d = U[q].w;
                float rb[kMaxK];
#pragma unroll
                for (int k = 0; k < kMaxK; ++k) {
                  const float dd = d - a.step * k;
                  rb[k] = k < a.K ? __expf(-a.gamma * dd * dd) : 0.f;
                }
                const float4* xs =
                    reinterpret_cast<const float4*>(a.X + static_cast<int64_t>(RQ[q]) * a.ld + cs + 8 * cg);
                const float4 x0 = __ldg(xs), x1 = __ldg(xs + 1);
                const float xv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
                const int l0 = 2 * lp;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  float r0 = 0.f, r1 = 0.f;
#pragma unroll
                  for (int k = 0; k < kMaxK; ++k) {
                    if (k < a.K) {
                      if (l0 < a.L) r0 = fmaf(rb[k], __ldg(a.W + (k * a.L + l0) * a.ld + cs + 8 * cg + i), r0);
                      if (l0 + 1 < a.L)
                        r1 = fmaf(rb[k], __ldg(a.W + (k * a.L + l0 + 1) * a.ld + cs + 8 * cg + i), r1);
                    }
                  }
                  y0[i] = xv[i] * r0;
                  y1[i] = xv[i] * r1;
                }
              } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) y0[i] = y1[i] = 0.f;
              }
              put8(bhi, blo, 8 * qi + 2 * lp, cg, y0);
              put8(bhi, blo, 8 * qi + 2 * lp + 1, cg, y1);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            named_sync(1, kBuilders);
            if (tid == 0) mbar_arrive(&sy.full[slot]);
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------ MMA issuer
    uint32_t it = 0, pass = 0;
    for (int64_t j = blockIdx.x; j < a.nv; j += gridDim.x) {
      const int64_t off = a.edge_ptr[j];
      const int n = static_cast<int>(a.edge_ptr[j + 1] - off);
      if (n <= 0 || n <= a.min_n) continue;
      for (int p0 = 0; p0 < n; p0 += M) {
        for (int q0 = 0; q0 < n; q0 += kNQ, ++pass) {
          const int nqp = (min(kNQ, n - q0) + 1) & ~1;
          const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(nqp) << 17) |
                                 (static_cast<uint32_t>(M >> 4) << 24);
          const uint32_t b = pass & 1;
          mbar_wait(&sy.dempty[b], ((pass >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t d = tmem + b * 128;
          for (int s = 0; s < nch; ++s, ++it) {
            const int slot = it % NS;
            mbar_wait(&sy.full[slot], (it / NS) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t ahi = su32(ring + slot * SLOT);
            if (elect_one()) {
              mma_slab(d, ahi, ahi + A_BYTES, ahi + 2 * A_BYTES, ahi + 2 * A_BYTES + B_BYTES, idesc, s == 0);
              mma_commit(&sy.empty[slot]);
              if (s == nch - 1) mma_commit(&sy.dfull[b]);
            }
            __syncwarp();
          }
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (thread = row p)
    const int qd = warp & 3;
    const int t = tid - (kBuilders + 32);
    uint32_t pass = 0;
    int ci = -1;
    for (int64_t j = blockIdx.x; j < a.nv; j += gridDim.x) {
      const int64_t off = a.edge_ptr[j];
      const int n = static_cast<int>(a.edge_ptr[j + 1] - off);
      if (n <= 0 || n <= a.min_n) continue;
      ++ci;
      const int gb = ci & 1;
      mbar_wait(&sy.gfull[gb], (ci >> 1) & 1);
      const float4* U = U2 + gb * a.gcap;
      for (int i = t; i < 3 * n; i += 128) UB[i] = 0.f;
      named_sync(2, 128);
      for (int p0 = 0; p0 < n; p0 += M) {
        const int p = p0 + 32 * qd + lane;
        const bool pv = p < n;
        const float4 up = U[pv ? p : 0];
        float ub0 = 0.f, ub1 = 0.f, ub2 = 0.f;
        for (int q0 = 0; q0 < n; q0 += kNQ, ++pass) {
          const int nq = min(kNQ, n - q0);
          const uint32_t b = pass & 1;
          mbar_wait(&sy.dfull[b], (pass >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t taddr = tmem + b * 128 + (static_cast<uint32_t>(qd * 32) << 16);
          for (int qi = 0; qi < nq; ++qi) {
            float tb[8];
            tmem_ld8(taddr + 8 * qi, tb);
            const int q = q0 + qi;
            float g = 0.f;
            const float4 uq = U[q];
            if (pv && p != q) {
              const float x = up.x * uq.x + up.y * uq.y + up.z * uq.z;
              // T_l'(x) = l U_{l-1}(x), U_0 = 1, U_1 = 2x, U_{m+1} = 2x U_m - U_{m-1}
              float um2 = 1.f, um1 = 2.f * x;
              g = tb[1];
              if (a.L > 2) g = fmaf(2.f * um1, tb[2], g);
#pragma unroll
              for (int l = 3; l < 8; ++l) {
                if (l >= a.L) break;
                const float un = 2.f * x * um1 - um2;
                g = fmaf(static_cast<float>(l) * un, tb[l], g);
                um2 = um1;
                um1 = un;
              }
            }
            ub0 = fmaf(g, uq.x, ub0);
            ub1 = fmaf(g, uq.y, ub1);
            ub2 = fmaf(g, uq.z, ub2);
            const float c0 = warp_sum(g * up.x), c1 = warp_sum(g * up.y), c2 = warp_sum(g * up.z);
            if (lane == 0) {
              CP[qd][qi][0] = c0;
              CP[qd][qi][1] = c1;
              CP[qd][qi][2] = c2;
            }
          }
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mbar_arrive(&sy.dempty[b]);
          named_sync(2, 128);
          if (t < 3 * nq) {
            const int qi = t / 3, comp = t % 3;
            UB[3 * (q0 + qi) + comp] += (CP[0][qi][comp] + CP[1][qi][comp]) + (CP[2][qi][comp] + CP[3][qi][comp]);
          }
          named_sync(2, 128);
        }
        if (pv) {
          UB[3 * p + 0] += ub0;
          UB[3 * p + 1] += ub1;
          UB[3 * p + 2] += ub2;
        }
        named_sync(2, 128);
      }
      // unit-vector adjoint -> edge vector adjoint of every out-edge of the centre
      for (int i = t; i < n; i += 128) {
        const float4 u = U[i];
        const float bx = UB[3 * i], by = UB[3 * i + 1], bz = UB[3 * i + 2];
        const float pr = bx * u.x + by * u.y + bz * u.z;
        const float inv = 1.f / u.w;
        float4 eg = a.edge_grad[off + i];
        eg.x += (bx - pr * u.x) * inv;
        eg.y += (by - pr * u.y) * inv;
        eg.z += (bz - pr * u.z) * inv;
        a.edge_grad[off + i] = eg;
      }
      named_sync(2, 128);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sy.gfree[gb]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == kMmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

}  // namespace tcb

// ---------------------------------------------------------------------------
// host side (called from egn_triplet_bwd)
// ---------------------------------------------------------------------------
bool tc_bwd_supported(int K, int L, int dg, int max_degree) {
  static const bool enabled = [] {
    const char* e = std::getenv("EGN_TRIPLET_TC");
    return !(e && e[0] == '0');
  }();
  return enabled && K >= 1 && K <= tcb::kMaxK && L >= 2 && L <= 8 && dg % 64 == 0 && max_degree >= 0 &&
         max_degree <= 1024;
}

static int tc_bwd_grid(int64_t nv) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(nv, kNumSMs))); }

int64_t tc_bwd_workspace_bytes(int64_t nv, int K, int L) {
  return static_cast<int64_t>(tc_bwd_grid(nv)) * K * L * 128 * 4;
}

int tc_bwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, int max_degree,
           const float* X, const float* W, int K, int L, int dg, RbfParams rp, const float* Sbar, float* Xbar,
           float* Wbar, float4* edge_grad, void* ws, int min_n, cudaStream_t st) {
  const int gcap = std::max(4, (max_degree + 3) & ~3);
  const int grid = tc_bwd_grid(nv);
  float* part = reinterpret_cast<float*>(ws);
  // kernel y per channel block of 128 (or a final 64)
  for (int c0 = 0; c0 < dg; c0 += 128) {
    const int M = (dg - c0) >= 128 ? 128 : 64;
    const int slot = 2 * M * 128 + 2 * 8 * tcb::kNQ * 128;
    const size_t fixed = static_cast<size_t>(gcap) * 2 * 20 + tcb::kMaxK * 8 * M * 4 + 1024;
    int nslot = 3;
    while (nslot > 2 && nslot * static_cast<size_t>(slot) + fixed > 200 * 1024) --nslot;
    const size_t smem = nslot * static_cast<size_t>(slot) + fixed;
    EGN_REQUIRE(smem <= 227 * 1024, "triplet_bwd_tc: %zu bytes of shared memory", smem);
    tcb::Args a{edge_ptr, rev, geo, nv, X, W, Sbar, Xbar, edge_grad, part, K, L, dg, c0, dg,
                rp.gamma, rp.step, nslot, gcap, min_n};
    auto kern = M == 128 ? tcb::y_kernel<128> : tcb::y_kernel<64>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<grid, tcb::kThreads, smem, st>>>(a);
    if (int rc = check_launch("triplet_bwd_tc_y")) return rc;
    tcb::wbar_reduce_kernel<<<(K * L * M + 255) / 256, 256, 0, st>>>(part, grid, K * L, M, dg, c0, Wbar);
    if (int rc = check_launch("triplet_bwd_tc_wbar")) return rc;
    if (M == 64) break;
  }
  {
    const int slot = 2 * 128 * 128 + 2 * 8 * tcb::kNQ * 128;
    const size_t fixed = static_cast<size_t>(gcap) * (2 * 20 + 12) + 1024;
    int nslot = 3;
    while (nslot > 2 && nslot * static_cast<size_t>(slot) + fixed > 200 * 1024) --nslot;
    const size_t smem = nslot * static_cast<size_t>(slot) + fixed;
    EGN_REQUIRE(smem <= 227 * 1024, "triplet_bwd_tc: %zu bytes of shared memory", smem);
    tcb::Args a{edge_ptr, rev, geo, nv, X, W, Sbar, Xbar, edge_grad, part, K, L, dg, 0, dg,
                rp.gamma, rp.step, nslot, gcap, min_n};
    cudaFuncSetAttribute(tcb::a_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    tcb::a_kernel<<<grid, tcb::kThreads, smem, st>>>(a);
    if (int rc = check_launch("triplet_bwd_tc_angles")) return rc;
  }
  return 0;
}

}  // namespace egn
