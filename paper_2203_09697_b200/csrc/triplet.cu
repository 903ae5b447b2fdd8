// Triplet interaction (TU + TA) forward and backward for sm_100a.
//
// Reference: record_tu, egn/engine.py:118-149, and the tape VJPs it implies
// (gather/segment_sum tape.py:129-154, linear :104-119, angular_sbf
// :231-242, triplet_angles :185-195).
//
// Centre-tile formulation.  Edges are sorted by (src, recv), so the
// out-edges of centre atom j are the contiguous rows [off_j, off_j + n).
// Triplet ((k->j), (j->i)) with out-edge p = (j->i) and in-edge
// rq = rev(off_j + q) = (k->j) exists for every ordered pair q != p of j's
// out-edges, and all of j's triplets form one n x n block minus its
// diagonal (enumerate_triplets, graph.py:106-139).  Hence
//   * the segment_sum over id3_ji is a reduction inside the tile (no atomics),
//   * every use of an edge as id3_kj lies in the tile of its receiver, so the
//     adjoint scatter to id3_kj is tile-local as well,
//   * the angle only needs the two out-edge unit vectors u_p, u_q of the
//     tile: cos(alpha) = x_pq = u_p . u_q and cos(l alpha) = T_l(x_pq)
//     (Chebyshev), and the SBF radial factor rbf(d_kj) uses d_q = d_rq.
// The per-triplet SBF gate sbf_t W^T factorises per in-edge:
//   g_sbf_t = sum_l T_l(x_pq) Rw[rq, l, :],  Rw[e, l, c] = sum_k rbf_k(d_e) W[k, l, c],
// and Q[q, l, c] = X[rq, c] Rw[rq, l, c] is built once per tile in shared
// memory.  Per triplet the kernel then spends L * dg FMAs; nothing per
// triplet ever touches HBM.
//
// Backward per centre (two phases, see the backward section):
//   Qbar[q,l,c] = sum_p T_l(x_pq) Sbar[p,c]                 -> X_bar, W_bar, dd_q
//   xbar(p,q)   = sum_l T_l'(x_pq) sum_c Sbar[p,c] Q[q,l,c]  -> dE/dv_p, dE/dv_q
// with dE/dv_q += xbar (u_p - x u_q) / d_q, the gradient of x_pq w.r.t. the
// edge vector v_q; using d cos(l a)/dx = T_l'(x) = l U_{l-1}(x) avoids the
// atan2 singularity and equals the reference's zero subgradient at
// collinear triplets (both factors vanish there).
#include <algorithm>

#include <cstdlib>
#include <string>

#include "common.cuh"

namespace egn {

constexpr int kThreads = 128;
constexpr int kMaxL = 8;
constexpr int kMaxK = 16;

// Triplet window (graph-parallel "reference" schedule, egn/partition.py:28-37): the launch
// covers centres [0, nv) and keeps only the triplets whose centre-local index
// k = p (n - 1) + (q < p ? q : q - 1) (the (out, in) order of enumerate_triplets) is >= first_lo
// at centre 0 and < last_hi at centre nv - 1, so a contiguous split_range shard of the
// triplet list is reproduced exactly even when it cuts through a centre's tile.
struct TripWin {
  int64_t first_lo, last_hi;
};
__device__ __forceinline__ bool in_window(const TripWin& w, int64_t j, int64_t nv, int n, int p, int q) {
  const int64_t k = static_cast<int64_t>(p) * (n - 1) + (q < p ? q : q - 1);
  return (j != 0 || k >= w.first_lo) && (j != nv - 1 || k < w.last_hi);
}

template <int CW, int GC>
struct ChanMap {
  static constexpr int VW = CW < 4 ? CW : 4;
  static constexpr int DP = CW * GC;
  // channel of slot i for channel-group cg: VW-wide chunks interleaved so
  // that one warp-wide vector load covers a contiguous 16*GC-byte span.
  __device__ __forceinline__ static int chan(int cg, int i) {
    return (i / VW) * (VW * GC) + cg * VW + (i % VW);
  }
};

template <int VW>
__device__ __forceinline__ void load_vec(const float* p, float* v) {
  if constexpr (VW == 4) {
    float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else if constexpr (VW == 2) {
    float2 t = *reinterpret_cast<const float2*>(p);
    v[0] = t.x; v[1] = t.y;
  } else {
    v[0] = p[0];
  }
}

// Shared-memory carve-up common to both kernels (floats, 16B aligned pieces).
struct TileLayout {
  int qt;      // q rows per tile
  int k, l, dp;
  int off_rb, off_w, off_q, off_x;  // float offsets
  int total;
  __host__ __device__ static int up4(int x) { return (x + 3) & ~3; }
  __host__ __device__ TileLayout(int qt_, int k_, int l_, int dp_, int extra_rows)
      : qt(qt_), k(k_), l(l_), dp(dp_) {
    int o = 4 * qt;              // Us (float4 per row)
    off_rb = o; o += up4(qt * k);  // rbf of tile rows
    off_w = o; o += up4(k * l * dp);
    off_q = o; o += up4(qt * l * dp);
    off_x = o; o += up4(extra_rows);  // kernel-specific extra
    total = o;
  }
};

__device__ __forceinline__ float rbf_val(float d, int k, RbfParams rp) {
  float dd = d - rp.step * k;
  return __expf(-rp.gamma * dd * dd);
}

// Build the tile: Us[t] = geo[off+q0+t], Rb[t][k] = rbf_k(d), Qs[t][l][c] = X[rq][c] * Rw.
template <int CW, int GC>
__device__ __forceinline__ void build_tile(const TileLayout& Ly, float* sm, const float4* __restrict__ geo,
                                           const int32_t* __restrict__ rev, const float* __restrict__ X,
                                           int64_t off, int q0, int nq, int dg, RbfParams rp) {
  using CM = ChanMap<CW, GC>;
  constexpr int DP = CM::DP;
  const int tid = threadIdx.x;
  float4* Us = reinterpret_cast<float4*>(sm);
  float* Rb = sm + Ly.off_rb;
  const float* Wsm = sm + Ly.off_w;
  float* Qs = sm + Ly.off_q;
  const int K = Ly.k, L = Ly.l;
  if (tid < nq) Us[tid] = geo[off + q0 + tid];
  for (int idx = tid; idx < nq * K; idx += kThreads) {
    int t = idx / K, k = idx - t * K;
    Rb[idx] = rbf_val(geo[off + q0 + t].w, k, rp);
  }
  __syncthreads();
  for (int idx = tid; idx < nq * DP; idx += kThreads) {
    int t = idx / DP, c = idx - t * DP;
    float xv = 0.f;
    if (c < dg) xv = X[static_cast<int64_t>(rev[off + q0 + t]) * dg + c];
    const float* rb = Rb + t * K;
    for (int l = 0; l < L; ++l) {
      float s = 0.f;
      for (int k = 0; k < K; ++k) s = fmaf(rb[k], Wsm[(k * L + l) * DP + c], s);
      Qs[(t * L + l) * DP + c] = xv * s;
    }
  }
  __syncthreads();
}

template <int CW, int GC>
__device__ __forceinline__ void load_weights(float* Wsm, const float* __restrict__ W, int K, int L, int dg) {
  constexpr int DP = CW * GC;
  for (int idx = threadIdx.x; idx < K * L * DP; idx += kThreads) {
    int kl = idx / DP, c = idx - kl * DP;
    Wsm[idx] = c < dg ? W[kl * dg + c] : 0.f;
  }
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
template <int CW, int GC, int R>
__global__ void __launch_bounds__(kThreads)
triplet_fwd_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ rev,
                   const float4* __restrict__ geo, int64_t nv, const float* __restrict__ X,
                   const float* __restrict__ W, int K, int L, int dg, int qt, RbfParams rp,
                   float* __restrict__ S, int min_n, TripWin win) {
  using CM = ChanMap<CW, GC>;
  constexpr int GP = kThreads / GC, VW = CM::VW, DP = CM::DP;
  extern __shared__ __align__(16) float sm[];
  TileLayout Ly(qt, K, L, DP, 0);
  const float4* Us = reinterpret_cast<const float4*>(sm);
  const float* Qs = sm + Ly.off_q;
  const int tid = threadIdx.x, cg = tid % GC, pg = tid / GC;

  load_weights<CW, GC>(sm + Ly.off_w, W, K, L, dg);
  // (the first tile build synchronises before Wsm is read)

  for (int64_t j = blockIdx.x; j < nv; j += gridDim.x) {
    const int64_t off = edge_ptr[j];
    const int n = static_cast<int>(edge_ptr[j + 1] - off);
    if (n == 0 || n <= min_n) continue;  // centres with n <= min_n run on the fast path
    for (int p0 = 0; p0 < n; p0 += GP * R) {
      const int reff = min(R, (n - p0 + GP - 1) / GP);  // CTA-uniform
      float4 up[R];
      int pidx[R];
      float acc[R][CW];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        pidx[r] = p0 + pg + GP * r;
        up[r] = (r < reff && pidx[r] < n) ? geo[off + pidx[r]] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < CW; ++i) acc[r][i] = 0.f;
      }
      for (int q0 = 0; q0 < n; q0 += qt) {
        const int nq = min(qt, n - q0);
        __syncthreads();
        build_tile<CW, GC>(Ly, sm, geo, rev, X, off, q0, nq, dg, rp);
        for (int t = 0; t < nq; ++t) {
          const float4 uq = Us[t];
          const int qg = q0 + t;
          float x2[R], tc[R], tp[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            float x = up[r].x * uq.x + up[r].y * uq.y + up[r].z * uq.z;
            float m = (pidx[r] != qg && in_window(win, j, nv, n, pidx[r], qg)) ? 1.f : 0.f;
            x2[r] = 2.f * x;
            tc[r] = m;       // T_0
            tp[r] = m * x;   // T_{-1} = T_1 = x
          }
          const float* qrow = Qs + t * L * DP;
          for (int l = 0; l < L; ++l) {
            float qv[CW];
#pragma unroll
            for (int i = 0; i < CW; i += VW) load_vec<VW>(qrow + l * DP + CM::chan(cg, i), qv + i);
#pragma unroll
            for (int r = 0; r < R; ++r) {
              if (r < reff) {
#pragma unroll
                for (int i = 0; i < CW; ++i) acc[r][i] = fmaf(tc[r], qv[i], acc[r][i]);
              }
              float tn = fmaf(x2[r], tc[r], -tp[r]);
              tp[r] = tc[r];
              tc[r] = tn;
            }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r < reff && pidx[r] < n) {
          float* dst = S + (off + pidx[r]) * dg;
#pragma unroll
          for (int i = 0; i < CW; ++i) {
            int c = CM::chan(cg, i);
            if (c < dg) dst[c] = acc[r][i];
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------
// Two phases per centre, both atomic-free and deterministic:
//  Phase 1 (rows p, like the forward; Q tiles in smem):
//     xbar(p,q) = sum_l T_l'(x_pq) sum_c Sbar[p,c] Q[q,l,c]
//     row part of dE/dv_p  += xbar(p,q) (u_q - x u_p)        (registers)
//     column part of dE/dv_q += xbar(p,q) (u_p - x u_q)      (XB tile in smem,
//                                                             summed by column owners)
//  Phase 2 (rows q; Sbar tiles in smem):
//     Qbar[q,l,c] = sum_p T_l(x_pq) Sbar[p,c]
//     X_bar[rq,c] = sum_l Qbar[q,l,c] Rw[rq,l,c],  R_bar = Qbar * X[rq]
//     W_bar[k,l,c] += sum_q rbf_k(d_q) R_bar[q,l,c],  dd_q = sum R_bar * dRw/dd
// Cost: ~2x the forward's FMAs.
struct BwdLayout {
  int us, rb, w, qs, sbs, wb, up, xb, rbs, fs, total;
  __host__ __device__ BwdLayout(int qt, int K, int L, int DP, int GP, int PB, int nmax) {
    auto up4 = TileLayout::up4;
    int o = 0;
    us = o; o += 4 * qt;
    rb = o; o += up4(qt * K);
    w = o; o += up4(K * L * DP);
    qs = o; o += up4((qt > GP ? qt : GP) * L * DP);  // Q tile (phase 1) / R_bar staging (phase 2)
    sbs = o; o += up4(qt * DP);
    wb = o; o += up4(K * L * DP);
    up = o; o += 4 * PB;
    xb = o; o += up4(PB * qt);
    rbs = o; o += up4(GP * K);
    fs = o; o += 4 * nmax;
    total = o;
  }
};

template <int CW, int GC, int R1>
__global__ void __launch_bounds__(kThreads)
triplet_bwd_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ rev,
                   const float4* __restrict__ geo, int64_t nv, const float* __restrict__ X,
                   const float* __restrict__ W, int K, int L, int dg, int qt, int nmax, int min_n, RbfParams rp,
                   const float* __restrict__ Sbar, float* __restrict__ Xbar,
                   float* __restrict__ wbar_part, float4* __restrict__ edge_grad, TripWin win) {
  using CM = ChanMap<CW, GC>;
  constexpr int GP = kThreads / GC, VW = CM::VW, DP = CM::DP, PB = GP * R1;
  extern __shared__ __align__(16) float sm[];
  const BwdLayout B(qt, K, L, DP, GP, PB, nmax);
  TileLayout Ly(qt, K, L, DP, 0);  // for build_tile: Us at 0, Rb, W, Qs offsets must match B
  float4* Us = reinterpret_cast<float4*>(sm + B.us);
  const float* Wsm = sm + B.w;
  float* Qs = sm + B.qs;
  float* Rst = sm + B.qs;
  float* Sbs = sm + B.sbs;
  float* Wb = sm + B.wb;
  float4* Up = reinterpret_cast<float4*>(sm + B.up);
  float* XB = sm + B.xb;
  float* Rbs = sm + B.rbs;
  float4* Fs = reinterpret_cast<float4*>(sm + B.fs);
  const int tid = threadIdx.x, cg = tid % GC, pg = tid / GC;

  load_weights<CW, GC>(sm + B.w, W, K, L, dg);
  for (int idx = tid; idx < K * L * DP; idx += kThreads) Wb[idx] = 0.f;

  for (int64_t j = blockIdx.x; j < nv; j += gridDim.x) {
    const int64_t off = edge_ptr[j];
    const int n = static_cast<int>(edge_ptr[j + 1] - off);
    if (n <= min_n) continue;  // handled by the fast path
    if (n < 2) {
      // no triplets at this centre: its in-edge (if any) gets a zero X_bar row
      if (n == 1) {
        const int64_t r0 = rev[off];
        for (int c = tid; c < dg; c += kThreads) Xbar[r0 * dg + c] = 0.f;
      }
      continue;
    }
    __syncthreads();  // previous centre finished with every buffer
    for (int i = tid; i < n; i += kThreads) Fs[i] = make_float4(0.f, 0.f, 0.f, 0.f);

    // ------------------------------ phase 1 ------------------------------
    for (int p0 = 0; p0 < n; p0 += PB) {
      const int reff = min(R1, (n - p0 + GP - 1) / GP);
      float4 up[R1];
      int pidx[R1];
      float sb[R1][CW];
      float fr[R1][3];
#pragma unroll
      for (int r = 0; r < R1; ++r) {
        pidx[r] = p0 + pg + GP * r;
        const bool ok = r < reff && pidx[r] < n;
        up[r] = ok ? geo[off + pidx[r]] : make_float4(0.f, 0.f, 0.f, 1.f);
#pragma unroll
        for (int i = 0; i < CW; ++i) {
          const int c = CM::chan(cg, i);
          sb[r][i] = (ok && c < dg) ? Sbar[(off + pidx[r]) * dg + c] : 0.f;
        }
        fr[r][0] = fr[r][1] = fr[r][2] = 0.f;
        if (cg == 0) Up[pg + GP * r] = up[r];
      }
      for (int q0 = 0; q0 < n; q0 += qt) {
        const int nq = min(qt, n - q0);
        __syncthreads();
        build_tile<CW, GC>(Ly, sm, geo, rev, X, off, q0, nq, dg, rp);
        for (int t = 0; t < nq; ++t) {
          const float4 uq = Us[t];
          const int qg = q0 + t;
          float x[R1], x2[R1], uc[R1], um[R1], s[R1];
#pragma unroll
          for (int r = 0; r < R1; ++r) {
            x[r] = up[r].x * uq.x + up[r].y * uq.y + up[r].z * uq.z;
            x2[r] = 2.f * x[r];
            uc[r] = 0.f;  // U_{l-1} at l = 0
            um[r] = 0.f;
            s[r] = 0.f;
          }
          const float* qrow = Qs + t * L * DP;
#pragma unroll
          for (int l = 0; l < kMaxL; ++l) {
            if (l < L) {
              float qv[CW];
#pragma unroll
              for (int i = 0; i < CW; i += VW) load_vec<VW>(qrow + l * DP + CM::chan(cg, i), qv + i);
#pragma unroll
              for (int r = 0; r < R1; ++r) {
                if (r < reff) {
                  float d = 0.f;
#pragma unroll
                  for (int i = 0; i < CW; ++i) d = fmaf(sb[r][i], qv[i], d);
                  s[r] = fmaf(static_cast<float>(l) * uc[r], d, s[r]);
                }
                const float un = (l == 0) ? 1.f : fmaf(x2[r], uc[r], -um[r]);
                um[r] = uc[r];
                uc[r] = un;
              }
            }
          }
#pragma unroll
          for (int r = 0; r < R1; ++r) {
            if (r < reff) {
              float v = s[r];
#pragma unroll
              for (int o = GC / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
              v = (pidx[r] < n && pidx[r] != qg && in_window(win, j, nv, n, pidx[r], qg)) ? v : 0.f;
              fr[r][0] = fmaf(v, uq.x - x[r] * up[r].x, fr[r][0]);
              fr[r][1] = fmaf(v, uq.y - x[r] * up[r].y, fr[r][1]);
              fr[r][2] = fmaf(v, uq.z - x[r] * up[r].z, fr[r][2]);
              if (cg == 0) XB[(pg + GP * r) * qt + t] = v;
            } else if (cg == 0) {
              XB[(pg + GP * r) * qt + t] = 0.f;
            }
          }
        }
        __syncthreads();
        // column owners: dE/dv_q += sum_p xbar(p,q) (u_p - x u_q), rows in fixed order
        const int rows = min(PB, n - p0);
        for (int t = tid; t < nq; t += kThreads) {
          const float4 uq = Us[t];
          float cx = 0.f, cy = 0.f, cz = 0.f;
          for (int ri = 0; ri < rows; ++ri) {
            const float4 u = Up[ri];
            const float xv = XB[ri * qt + t];
            const float x = u.x * uq.x + u.y * uq.y + u.z * uq.z;
            cx = fmaf(xv, u.x - x * uq.x, cx);
            cy = fmaf(xv, u.y - x * uq.y, cy);
            cz = fmaf(xv, u.z - x * uq.z, cz);
          }
          float4 f = Fs[q0 + t];
          f.x += cx;
          f.y += cy;
          f.z += cz;
          Fs[q0 + t] = f;
        }
      }
      __syncthreads();
      if (cg == 0) {
#pragma unroll
        for (int r = 0; r < R1; ++r) {
          if (r < reff && pidx[r] < n) {
            float4 f = Fs[pidx[r]];
            f.x += fr[r][0];
            f.y += fr[r][1];
            f.z += fr[r][2];
            Fs[pidx[r]] = f;
          }
        }
      }
    }

    // ------------------------------ phase 2 ------------------------------
    for (int b0 = 0; b0 < n; b0 += GP) {
      const int q = b0 + pg;
      const bool valid = q < n;
      const float4 uq = valid ? geo[off + q] : make_float4(0.f, 0.f, 0.f, 1.f);
      float qb[kMaxL][CW];
#pragma unroll
      for (int l = 0; l < kMaxL; ++l)
#pragma unroll
        for (int i = 0; i < CW; ++i) qb[l][i] = 0.f;
      for (int p0 = 0; p0 < n; p0 += qt) {
        const int np = min(qt, n - p0);
        __syncthreads();
        if (tid < np) Us[tid] = geo[off + p0 + tid];
        for (int idx = tid; idx < np * DP; idx += kThreads) {
          const int t = idx / DP, c = idx - t * DP;
          Sbs[idx] = c < dg ? Sbar[(off + p0 + t) * dg + c] : 0.f;
        }
        __syncthreads();
        for (int t = 0; t < np; ++t) {
          const float4 up = Us[t];
          const float x = up.x * uq.x + up.y * uq.y + up.z * uq.z;
          const float m = (p0 + t != q && in_window(win, j, nv, n, p0 + t, q)) ? 1.f : 0.f;
          float sbp[CW];
#pragma unroll
          for (int i = 0; i < CW; i += VW) load_vec<VW>(Sbs + t * DP + CM::chan(cg, i), sbp + i);
          const float x2 = 2.f * x;
          float tc = m, tp = m * x;
#pragma unroll
          for (int l = 0; l < kMaxL; ++l) {
            if (l < L) {
#pragma unroll
              for (int i = 0; i < CW; ++i) qb[l][i] = fmaf(tc, sbp[i], qb[l][i]);
              const float tn = fmaf(x2, tc, -tp);
              tp = tc;
              tc = tn;
            }
          }
        }
      }
      // ---- row epilogue ----
      const int64_t rq = valid ? static_cast<int64_t>(rev[off + q]) : 0;
      float xo[CW], xb[CW];
#pragma unroll
      for (int i = 0; i < CW; ++i) {
        const int c = CM::chan(cg, i);
        xo[i] = (valid && c < dg) ? X[rq * dg + c] : 0.f;
        xb[i] = 0.f;
      }
      float rbo[kMaxK], rdo[kMaxK];  // rbf_k(d_q), d rbf_k / dd
#pragma unroll
      for (int k = 0; k < kMaxK; ++k) {
        rbo[k] = k < K ? rbf_val(uq.w, k, rp) : 0.f;
        rdo[k] = -2.f * rp.gamma * (uq.w - rp.step * k) * rbo[k];
      }
      float dd = 0.f;
      __syncthreads();  // Rst (aliases the Q tile) is free
#pragma unroll
      for (int l = 0; l < kMaxL; ++l) {
        if (l < L) {
#pragma unroll
          for (int i = 0; i < CW; ++i) {
            const int c = CM::chan(cg, i);
            float rw = 0.f, rwd = 0.f;
#pragma unroll
            for (int k = 0; k < kMaxK; ++k) {
              if (k < K) {
                const float w = Wsm[(k * L + l) * DP + c];
                rw = fmaf(rbo[k], w, rw);
                rwd = fmaf(rdo[k], w, rwd);
              }
            }
            xb[i] = fmaf(qb[l][i], rw, xb[i]);
            const float rbar = qb[l][i] * xo[i];
            dd = fmaf(rbar, rwd, dd);
            Rst[(pg * L + l) * DP + c] = valid ? rbar : 0.f;
          }
        }
      }
      if (cg == 0) {
#pragma unroll
        for (int k = 0; k < kMaxK; ++k)
          if (k < K) Rbs[pg * K + k] = valid ? rbo[k] : 0.f;
      }
#pragma unroll
      for (int o = GC / 2; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
      if (valid) {
#pragma unroll
        for (int i = 0; i < CW; ++i) {
          const int c = CM::chan(cg, i);
          if (c < dg) Xbar[rq * dg + c] = xb[i];
        }
        if (cg == 0) {
          const float inv = 1.f / uq.w;
          const float4 f = Fs[q];
          float4 g = edge_grad[off + q];
          g.x += f.x * inv;
          g.y += f.y * inv;
          g.z += f.z * inv;
          g.w += dd;
          edge_grad[off + q] = g;
        }
      }
      __syncthreads();
      // W_bar[k,l,c] += sum_rows rbf_k(row) R_bar[row,l,c]   (thread-owned (l,c): no atomics)
      const int rows = min(GP, n - b0);
      for (int idx = tid; idx < L * DP; idx += kThreads) {
        for (int k = 0; k < K; ++k) {
          float s = Wb[k * L * DP + idx];
          for (int r = 0; r < rows; ++r) s = fmaf(Rbs[r * K + k], Rst[r * L * DP + idx], s);
          Wb[k * L * DP + idx] = s;
        }
      }
    }
  }
  __syncthreads();
  float* dst = wbar_part + static_cast<int64_t>(blockIdx.x) * K * L * dg;
  for (int idx = tid; idx < K * L * dg; idx += kThreads) {
    const int kl = idx / dg, c = idx - kl * dg;
    dst[idx] = Wb[kl * DP + c];
  }
}

__global__ void reduce_partials_kernel(const float* __restrict__ part, int nparts, int64_t len,
                                       float* __restrict__ out, int accumulate) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < nparts; ++p) s += part[p * len + i];
    out[i] = accumulate ? out[i] + s : s;
  }
}

// fast path (triplet_fast.cu): centres with deg <= 64 and (K, L) = (6, 7)
bool fast_supported(int K, int L, int dg);
int fast_fwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, const float* X,
             const float* W, int K, int L, int dg, RbfParams rp, float* S, cudaStream_t st, int mode = 0,
             const float* rtab = nullptr);
int64_t fast_bwd_workspace_bytes(int64_t nv, int64_t ne, int K, int L, int dg);
int fast_bwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, int64_t ne,
             const float* X, const float* W, int K, int L, int dg, RbfParams rp, const float* Sbar, float* Xbar,
             float* Wbar, float4* edge_grad, void* ws, cudaStream_t st, int phases, int mode = 0,
             const float* rtab = nullptr, const float* dtab = nullptr);
constexpr int kFastMaxDeg = 64;
// spherical-harmonic factorised path (triplet_sh.cu): O(deg) per edge
bool sh_supported(int K, int L, int dg);
int64_t sh_fwd_workspace_bytes(int64_t nv, int max_degree, int K, int L, int dg);
int sh_fwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, int max_degree, const float* X,
           const float* W, int K, int L, int dg, RbfParams rp, float cutoff, int mode, float* S, void* ws, int min_n,
           cudaStream_t st, const float* rtab = nullptr);
int64_t sh_bwd_workspace_bytes(int64_t nv, int64_t ne, int max_degree, int K, int L, int dg);
int64_t sh_radial_table_floats(int64_t ne, int mode);
int sh_radial_table(const float4* geo, int64_t ne, float cutoff, int mode, float* tab, float* dtab, cudaStream_t st);
int sh_bwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, int64_t ne, int max_degree,
           const float* X, const float* W, int K, int L, int dg, RbfParams rp, float cutoff, int mode,
           const float* Sbar, float* Xbar, float* Wbar, float4* edge_grad, void* ws, int min_n, int accumulate,
           cudaStream_t st, const float* rtab = nullptr,
           const float* drtab = nullptr);

// Path selection (egn_triplet_path): 0 = auto (deg <= 64: pairwise centre tiles; larger centres:
// the linear-in-degree spherical-harmonic kernels), 1 = spherical-harmonic kernels for every
// centre, 2 = pairwise only (centre tiles + tensor-core kernels for deg > 64).  EGN_TRIPLET_PATH
// (auto / sh / pairwise) sets the initial value; EGN_TRIPLET_TC_ALL=1 forces the tensor path.
static int g_triplet_path = [] {
  const char* e = std::getenv("EGN_TRIPLET_PATH");
  if (!e) return 0;
  const std::string v(e);
  return v == "sh" ? 1 : (v == "pairwise" ? 2 : 0);
}();
bool tc_fwd_supported(int K, int L, int dg, int max_degree);
bool tc_bwd_supported(int K, int L, int dg, int max_degree);
int64_t tc_bwd_workspace_bytes(int64_t nv, int K, int L);
int tc_bwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, int max_degree,
           const float* X, const float* W, int K, int L, int dg, RbfParams rp, const float* Sbar, float* Xbar,
           float* Wbar, float4* edge_grad, void* ws, int min_n, cudaStream_t st);
int tc_fwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, int max_degree,
           const float* X, const float* W, int K, int L, int dg, RbfParams rp, float* S, int min_n,
           cudaStream_t st);

// Debug: per-triplet summand P[t, c] in (out, in) order.
__global__ void triplet_terms_kernel(const int64_t* __restrict__ edge_ptr,
                                     const int32_t* __restrict__ rev,
                                     const float4* __restrict__ geo,
                                     const int64_t* __restrict__ tri_ptr, int64_t nv,
                                     const float* __restrict__ X, const float* __restrict__ W,
                                     int K, int L, int dg, RbfParams rp, float* __restrict__ P) {
  for (int64_t j = blockIdx.x; j < nv; j += gridDim.x) {
    int64_t off = edge_ptr[j];
    int64_t n = edge_ptr[j + 1] - off;
    if (n < 2) continue;
    int64_t t0 = tri_ptr[j];
    int64_t cnt = n * (n - 1) * dg;
    for (int64_t k = threadIdx.x; k < cnt; k += blockDim.x) {
      int64_t tt = k / dg;
      int c = static_cast<int>(k - tt * dg);
      int64_t p = tt / (n - 1);
      int64_t r = tt - p * (n - 1);
      int64_t q = r < p ? r : r + 1;
      float4 a = geo[off + p], b = geo[off + q];
      float x = a.x * b.x + a.y * b.y + a.z * b.z;
      int64_t rq = rev[off + q];
      float tc = 1.f, tp = x, g = 0.f;
      for (int l = 0; l < L; ++l) {
        float rw = 0.f;
        for (int kk = 0; kk < K; ++kk) rw = fmaf(rbf_val(b.w, kk, rp), W[(kk * L + l) * dg + c], rw);
        g = fmaf(tc, rw, g);
        float tn = 2.f * x * tc - tp;
        tp = tc;
        tc = tn;
      }
      P[(t0 + tt) * dg + c] = X[rq * dg + c] * g;
    }
  }
}

// ---------------------------------------------------------------------------
// host dispatch
// ---------------------------------------------------------------------------
static int pick_qt(int K, int L, int DP, int extra_floats, int budget_bytes) {
  int fixed = 4 * (K * L * DP + extra_floats) + 64;
  int per_row = 4 * (L * DP + 4 + K);
  int qt = (budget_bytes - fixed) / per_row;
  if (qt > 32) qt = 32;
  if (qt < 4) qt = 4;
  return qt;
}

template <int CW, int GC, int R>
static int launch_fwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv,
                      const float* X, const float* W, int K, int L, int dg, RbfParams rp, float* S,
                      int min_n, cudaStream_t st, TripWin win = TripWin{0, INT64_MAX}) {
  constexpr int DP = CW * GC;
  int qt = pick_qt(K, L, DP, 0, 48 * 1024);
  TileLayout Ly(qt, K, L, DP, 0);
  size_t smem = static_cast<size_t>(Ly.total) * 4;
  auto kern = triplet_fwd_kernel<CW, GC, R>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = std::min<int64_t>(nv, static_cast<int64_t>(kNumSMs) * per_sm * 4);
  kern<<<static_cast<int>(grid), kThreads, smem, st>>>(edge_ptr, rev, geo, nv, X, W, K, L, dg, qt, rp, S, min_n,
                                                       win);
  return check_launch("triplet_fwd");
}

template <int CW, int GC, int R>
static int launch_bwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv,
                      const float* X, const float* W, int K, int L, int dg, int max_deg, RbfParams rp,
                      const float* Sbar, float* Xbar, float* Wbar, float4* edge_grad, void* ws,
                      int min_n, int accumulate, cudaStream_t st, TripWin win = TripWin{0, INT64_MAX}) {
  constexpr int DP = CW * GC, GP = kThreads / GC, PB = GP * R;
  EGN_REQUIRE(max_deg >= 0, "triplet backward needs the maximum centre degree");
  const int nmax = max_deg > 2 ? max_deg : 2;
  // pick the largest tile (<= 32 rows) that keeps shared memory under ~100 KB
  int qt = 32;
  while (qt > 4 && BwdLayout(qt, K, L, DP, GP, PB, nmax).total * 4 > 100 * 1024) qt -= 4;
  const size_t smem = static_cast<size_t>(BwdLayout(qt, K, L, DP, GP, PB, nmax).total) * 4;
  EGN_REQUIRE(smem <= 227 * 1024, "triplet backward needs %zu bytes of shared memory (max degree %d)", smem, max_deg);
  auto kern = triplet_bwd_kernel<CW, GC, R>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 4) per_sm = 4;
  const int grid = static_cast<int>(std::min<int64_t>(nv, static_cast<int64_t>(kNumSMs) * per_sm));
  float* part = reinterpret_cast<float*>(ws);
  kern<<<grid, kThreads, smem, st>>>(edge_ptr, rev, geo, nv, X, W, K, L, dg, qt, nmax, min_n, rp, Sbar, Xbar, part,
                                     edge_grad, win);
  if (check_launch("triplet_bwd")) return 1;
  const int64_t len = static_cast<int64_t>(K) * L * dg;
  reduce_partials_kernel<<<grid_for(len, 256), 256, 0, st>>>(part, grid, len, Wbar, accumulate);
  return check_launch("triplet_bwd_reduce");
}

}  // namespace egn

using namespace egn;


static int check_dims(int K, int L, int dg) {
  EGN_REQUIRE(K >= 1 && K <= 16, "k_rbf must be in [1, 16], got %d", K);
  EGN_REQUIRE(L >= 1 && L <= kMaxL, "l_sbf must be in [1, %d], got %d", kMaxL, L);
  EGN_REQUIRE(dg >= 1 && dg <= 256, "triplet width must be in [1, 256], got %d", dg);
  return 0;
}

extern "C" {

static int64_t align256(int64_t b) { return (b + 255) / 256 * 256; }

int64_t egn_triplet_fwd_basis_workspace_bytes(int64_t num_nodes, int64_t num_edges, int max_degree, int k_rbf,
                                              int l_sbf, int dg, int basis) {
  if (basis == 0) return egn_triplet_fwd_workspace_bytes(num_nodes, max_degree, k_rbf, l_sbf, dg);
  if (!sh_supported(k_rbf, l_sbf, dg) || max_degree < 0) return 0;
  // per-chunk moments, then the edges' radial table
  return align256(sh_fwd_workspace_bytes(num_nodes, max_degree, k_rbf, l_sbf, dg)) +
         sh_radial_table_floats(num_edges, basis) * 4;
}

int64_t egn_triplet_bwd_basis_workspace_bytes(int64_t num_nodes, int64_t num_edges, int max_degree, int k_rbf,
                                              int l_sbf, int dg, int basis) {
  const int64_t b = egn_triplet_bwd_workspace_bytes(num_nodes, num_edges, max_degree, k_rbf, l_sbf, dg);
  if (basis == 0) return b;
  return align256(b) + 2 * align256(sh_radial_table_floats(num_edges, basis) * 4);  // radial values, d-derivatives
}

int64_t egn_triplet_fwd_workspace_bytes(int64_t num_nodes, int max_degree, int k_rbf, int l_sbf, int dg) {
  // only the spherical-harmonic path needs one (its per-chunk moments)
  const bool fast_covers = g_triplet_path == 0 && fast_supported(k_rbf, l_sbf, dg) && max_degree <= kFastMaxDeg;
  if (!sh_supported(k_rbf, l_sbf, dg) || max_degree < 0 || g_triplet_path == 2 || fast_covers) return 0;
  return sh_fwd_workspace_bytes(num_nodes, max_degree, k_rbf, l_sbf, dg);
}

int egn_triplet_fwd(const int64_t* edge_ptr, const int32_t* rev, const float* geo,
                    int64_t num_nodes, int max_degree, const float* X, const float* W, int k_rbf,
                    int l_sbf, int dg, double cutoff, float* S, void* workspace, egn_stream_t stream) {
  if (int rc = check_dims(k_rbf, l_sbf, dg)) return rc;
  if (num_nodes == 0) return 0;
  RbfParams rp = rbf_params(k_rbf, cutoff);
  const float4* g4 = reinterpret_cast<const float4*>(geo);
  cudaStream_t st = as_stream(stream);
  // centres with deg <= 64: CUDA-core centre-tile kernel (triplet_fast.cu); larger
  // centres: tensor-core kernel (triplet_tc.cu) when the degree bound is known, else
  // the generic CUDA-core kernel
  int min_n = 0;
  static const bool tc_all = [] { const char* e = std::getenv("EGN_TRIPLET_TC_ALL"); return e && e[0] == '1'; }();
  const bool use_sh = !tc_all && g_triplet_path != 2 && sh_supported(k_rbf, l_sbf, dg) && max_degree >= 0 &&
                      workspace != nullptr;
  if (fast_supported(k_rbf, l_sbf, dg) && !(tc_all && tc_fwd_supported(k_rbf, l_sbf, dg, max_degree)) &&
      !(use_sh && g_triplet_path == 1)) {
    if (int rc = fast_fwd(edge_ptr, rev, g4, num_nodes, X, W, k_rbf, l_sbf, dg, rp, S, st)) return rc;
    if (max_degree >= 0 && max_degree <= kFastMaxDeg) return 0;
    min_n = kFastMaxDeg;
  }
  if (use_sh)
    return sh_fwd(edge_ptr, rev, g4, num_nodes, max_degree, X, W, k_rbf, l_sbf, dg, rp, static_cast<float>(cutoff), 0,
                  S, workspace, min_n, st);
  if (tc_fwd_supported(k_rbf, l_sbf, dg, max_degree))
    return tc_fwd(edge_ptr, rev, g4, num_nodes, max_degree, X, W, k_rbf, l_sbf, dg, rp, S, min_n, st);
#define EGN_FWD(CW, GC, R) \
  return launch_fwd<CW, GC, R>(edge_ptr, rev, g4, num_nodes, X, W, k_rbf, l_sbf, dg, rp, S, min_n, st)
  if (dg <= 4) EGN_FWD(4, 1, 1);
  if (dg <= 8) EGN_FWD(8, 1, 1);
  if (dg <= 16) EGN_FWD(8, 2, 2);
  if (dg <= 32) EGN_FWD(8, 4, 2);
  if (dg <= 64) EGN_FWD(8, 8, 4);
  if (dg <= 128) EGN_FWD(8, 16, 4);
  EGN_FWD(8, 32, 4);
#undef EGN_FWD
}

static int64_t generic_ws_bytes(int64_t num_nodes, int k_rbf, int l_sbf, int dg) {
  int64_t grid = std::min<int64_t>(std::max<int64_t>(num_nodes, 1), static_cast<int64_t>(kNumSMs) * 4);
  return grid * k_rbf * l_sbf * dg * 4;
}

static int64_t fast_ws_bytes(int64_t num_nodes, int64_t num_edges, int k_rbf, int l_sbf, int dg) {
  return fast_supported(k_rbf, l_sbf, dg) ? fast_bwd_workspace_bytes(num_nodes, num_edges, k_rbf, l_sbf, dg) : 0;
}

int64_t egn_triplet_bwd_workspace_bytes(int64_t num_nodes, int64_t num_edges, int max_degree, int k_rbf, int l_sbf,
                                        int dg) {
  return generic_ws_bytes(num_nodes, k_rbf, l_sbf, dg) + fast_ws_bytes(num_nodes, num_edges, k_rbf, l_sbf, dg) +
         tc_bwd_workspace_bytes(num_nodes, k_rbf, l_sbf) +
         (sh_supported(k_rbf, l_sbf, dg) && max_degree >= 0
              ? sh_bwd_workspace_bytes(num_nodes, num_edges, max_degree, k_rbf, l_sbf, dg)
              : 0);
}

int egn_triplet_bwd(const int64_t* edge_ptr, const int32_t* rev, const float* geo,
                    int64_t num_nodes, int64_t num_edges, int max_degree, const float* X, const float* W,
                    int k_rbf, int l_sbf, int dg, double cutoff, const float* S_bar, float* X_bar,
                    float* W_bar, float* edge_grad, void* workspace, egn_stream_t stream) {
  return egn_triplet_bwd_ex(edge_ptr, rev, geo, num_nodes, num_edges, max_degree, X, W, k_rbf, l_sbf, dg, cutoff,
                            S_bar, X_bar, W_bar, edge_grad, 3, workspace, stream);
}

int egn_triplet_bwd_ex(const int64_t* edge_ptr, const int32_t* rev, const float* geo, int64_t num_nodes,
                       int64_t num_edges, int max_degree, const float* X, const float* W, int k_rbf, int l_sbf,
                       int dg, double cutoff, const float* S_bar, float* X_bar, float* W_bar, float* edge_grad,
                       int phases, void* workspace, egn_stream_t stream) {
  if (int rc = check_dims(k_rbf, l_sbf, dg)) return rc;
  EGN_REQUIRE(phases >= 1 && phases <= 3, "phases must be 1, 2 or 3");
  cudaStream_t st = as_stream(stream);
  static const bool tc_all = [] { const char* e = std::getenv("EGN_TRIPLET_TC_ALL"); return e && e[0] == '1'; }();
  // the angle phase exists only on the small-degree fast path (bw1); elsewhere phase 2 does all
  const bool split_ok = g_triplet_path != 1 && fast_supported(k_rbf, l_sbf, dg) && !tc_all;
  if (!split_ok) {
    if (phases == 1) return 0;
    phases = 3;
  }
  if (num_nodes == 0) {
    if (!(phases & 2)) return 0;
    cudaMemsetAsync(W_bar, 0, sizeof(float) * k_rbf * l_sbf * dg, st);
    return check_launch("triplet_bwd_empty");
  }
  RbfParams rp = rbf_params(k_rbf, cutoff);
  const float4* g4 = reinterpret_cast<const float4*>(geo);
  float4* eg = reinterpret_cast<float4*>(edge_grad);
  int min_n = 0, accumulate = 0;
  const bool use_sh = !tc_all && g_triplet_path != 2 && sh_supported(k_rbf, l_sbf, dg) && max_degree >= 0;
  if (fast_supported(k_rbf, l_sbf, dg) && !(tc_all && tc_bwd_supported(k_rbf, l_sbf, dg, max_degree)) &&
      !(use_sh && g_triplet_path == 1)) {
    char* fws = reinterpret_cast<char*>(workspace) + generic_ws_bytes(num_nodes, k_rbf, l_sbf, dg);
    if (int rc = fast_bwd(edge_ptr, rev, g4, num_nodes, num_edges, X, W, k_rbf, l_sbf, dg, rp, S_bar, X_bar,
                          W_bar, eg, fws, st, phases))
      return rc;
    if (!(phases & 2)) return 0;  // angle phase only
    if (max_degree >= 0 && max_degree <= kFastMaxDeg) return 0;
    min_n = kFastMaxDeg;
    accumulate = 1;
  }
  if (use_sh) {
    char* sws = reinterpret_cast<char*>(workspace) + generic_ws_bytes(num_nodes, k_rbf, l_sbf, dg) +
                fast_ws_bytes(num_nodes, num_edges, k_rbf, l_sbf, dg) + tc_bwd_workspace_bytes(num_nodes, k_rbf, l_sbf);
    return sh_bwd(edge_ptr, rev, g4, num_nodes, num_edges, max_degree, X, W, k_rbf, l_sbf, dg, rp,
                  static_cast<float>(cutoff), 0, S_bar, X_bar, W_bar, eg, sws, min_n, accumulate, st);
  }
  // centres above the small-degree kernel's range: tensor-core backward (triplet_tc_bwd.cu)
  if (tc_bwd_supported(k_rbf, l_sbf, dg, max_degree)) {
    if (!accumulate) cudaMemsetAsync(W_bar, 0, sizeof(float) * k_rbf * l_sbf * dg, st);
    char* tws = reinterpret_cast<char*>(workspace) + generic_ws_bytes(num_nodes, k_rbf, l_sbf, dg) +
                fast_ws_bytes(num_nodes, num_edges, k_rbf, l_sbf, dg);
    return tc_bwd(edge_ptr, rev, g4, num_nodes, max_degree, X, W, k_rbf, l_sbf, dg, rp, S_bar, X_bar, W_bar, eg,
                  tws, min_n, st);
  }
#define EGN_BWD(CW, GC, R) \
  return launch_bwd<CW, GC, R>(edge_ptr, rev, g4, num_nodes, X, W, k_rbf, l_sbf, dg, max_degree, rp, S_bar, X_bar, \
                               W_bar, eg, workspace, min_n, accumulate, st)
  if (dg <= 4) EGN_BWD(4, 1, 1);
  if (dg <= 8) EGN_BWD(8, 1, 1);
  if (dg <= 16) EGN_BWD(8, 2, 2);
  if (dg <= 32) EGN_BWD(8, 4, 2);
  if (dg <= 64) EGN_BWD(8, 8, 4);
  if (dg <= 128) EGN_BWD(8, 16, 4);
  EGN_BWD(8, 32, 4);
#undef EGN_BWD
}

int egn_triplet_path(int mode) {
  const int old = g_triplet_path;
  if (mode >= 0 && mode <= 2) g_triplet_path = mode;
  return old;
}

// DimeNet++ / GemNet bases: basis 1 = GemNet CBF (radial Bessel basis of
// d_kj x Y_l0(angle)), 2 = DimeNet SBF (sqrt(2/c^3)/|j_{l+1}(z_ln)| u(d/c) j_l(z_ln d/c) Y_l0(angle));
// centres of degree <= 64 on the pairwise kernels (triplet_fast.cu MODE 1 / 2), the rest on the
// spherical-harmonic kernels (their A table absorbs the Y_l0 normalisation)
int egn_triplet_fwd_basis(const int64_t* edge_ptr, const int32_t* rev, const float* geo, int64_t num_nodes,
                          int64_t num_edges, int max_degree, const float* X, const float* W, int k_rbf, int l_sbf,
                          int dg, double cutoff, int basis, float* S, void* workspace, egn_stream_t stream) {
  if (basis == 0)
    return egn_triplet_fwd(edge_ptr, rev, geo, num_nodes, max_degree, X, W, k_rbf, l_sbf, dg, cutoff, S, workspace,
                           stream);
  if (int rc = check_dims(k_rbf, l_sbf, dg)) return rc;
  EGN_REQUIRE(basis == 1 || basis == 2, "basis must be 0, 1 or 2");
  EGN_REQUIRE(sh_supported(k_rbf, l_sbf, dg), "the bessel bases need k_rbf = 6, l_sbf = 7");
  EGN_REQUIRE(max_degree >= 0 && workspace != nullptr, "the bessel bases need max_degree and a workspace");
  if (num_nodes == 0) return 0;
  cudaStream_t st = as_stream(stream);
  const float4* g4 = reinterpret_cast<const float4*>(geo);
  float* tab = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) +
                                        align256(sh_fwd_workspace_bytes(num_nodes, max_degree, k_rbf, l_sbf, dg)));
  if (int rc = sh_radial_table(g4, num_edges, static_cast<float>(cutoff), basis, tab, nullptr, st)) return rc;
  int min_n = 0;
  if (g_triplet_path != 1 && fast_supported(k_rbf, l_sbf, dg)) {
    // both bases on the pairwise small-degree kernels (Legendre angular rows, radial rows from
    // the table: MODE 1 k-only, MODE 2 (k, l)); the spherical-harmonic kernels take the centres
    // above their range
    if (int rc = fast_fwd(edge_ptr, rev, g4, num_nodes, X, W, k_rbf, l_sbf, dg, rbf_params(k_rbf, cutoff), S, st,
                          basis, tab))
      return rc;
    if (max_degree <= kFastMaxDeg) return 0;
    min_n = kFastMaxDeg;
  }
  return sh_fwd(edge_ptr, rev, g4, num_nodes, max_degree, X, W, k_rbf, l_sbf, dg, rbf_params(k_rbf, cutoff),
                static_cast<float>(cutoff), basis, S, workspace, min_n, st, tab);
}

int egn_triplet_bwd_basis_ex(const int64_t* edge_ptr, const int32_t* rev, const float* geo, int64_t num_nodes,
                             int64_t num_edges, int max_degree, const float* X, const float* W, int k_rbf, int l_sbf,
                             int dg, double cutoff, int basis, int phases, const float* S_bar, float* X_bar,
                             float* W_bar, float* edge_grad, void* workspace, egn_stream_t stream);

int egn_triplet_bwd_basis(const int64_t* edge_ptr, const int32_t* rev, const float* geo, int64_t num_nodes,
                          int64_t num_edges, int max_degree, const float* X, const float* W, int k_rbf, int l_sbf,
                          int dg, double cutoff, int basis, const float* S_bar, float* X_bar, float* W_bar,
                          float* edge_grad, void* workspace, egn_stream_t stream) {
  return egn_triplet_bwd_basis_ex(edge_ptr, rev, geo, num_nodes, num_edges, max_degree, X, W, k_rbf, l_sbf, dg,
                                  cutoff, basis, 3, S_bar, X_bar, W_bar, edge_grad, workspace, stream);
}

int64_t egn_triplet_bwd_angle_workspace_bytes(int64_t num_edges, int basis) {
  return sh_radial_table_floats(num_edges, basis) * 4;
}

int egn_triplet_bwd_basis_ex(const int64_t* edge_ptr, const int32_t* rev, const float* geo, int64_t num_nodes,
                             int64_t num_edges, int max_degree, const float* X, const float* W, int k_rbf, int l_sbf,
                             int dg, double cutoff, int basis, int phases, const float* S_bar, float* X_bar,
                             float* W_bar, float* edge_grad, void* workspace, egn_stream_t stream) {
  if (basis == 0)
    return egn_triplet_bwd_ex(edge_ptr, rev, geo, num_nodes, num_edges, max_degree, X, W, k_rbf, l_sbf, dg, cutoff,
                              S_bar, X_bar, W_bar, edge_grad, phases, workspace, stream);
  EGN_REQUIRE(phases >= 1 && phases <= 3, "phases must be 1, 2 or 3");
  // the angle phase splits off only on the small-degree kernels
  const bool split_ok = g_triplet_path != 1 && fast_supported(k_rbf, l_sbf, dg);
  if (!split_ok) {
    if (phases == 1) return 0;
    phases = 3;
  }
  if (phases == 1) {  // own radial table in its own workspace (egn_triplet_bwd_angle_workspace_bytes)
    if (int rc = check_dims(k_rbf, l_sbf, dg)) return rc;
    if (num_nodes == 0) return 0;
    cudaStream_t st = as_stream(stream);
    const float4* g4 = reinterpret_cast<const float4*>(geo);
    float* tab = reinterpret_cast<float*>(workspace);
    if (int rc = sh_radial_table(g4, num_edges, static_cast<float>(cutoff), basis, tab, nullptr, st)) return rc;
    return fast_bwd(edge_ptr, rev, g4, num_nodes, num_edges, X, W, k_rbf, l_sbf, dg, rbf_params(k_rbf, cutoff), S_bar,
                    X_bar, W_bar, reinterpret_cast<float4*>(edge_grad), nullptr, st, 1, basis, tab, nullptr);
  }
  if (int rc = check_dims(k_rbf, l_sbf, dg)) return rc;
  EGN_REQUIRE(basis == 1 || basis == 2, "basis must be 0, 1 or 2");
  EGN_REQUIRE(sh_supported(k_rbf, l_sbf, dg), "the bessel bases need k_rbf = 6, l_sbf = 7");
  EGN_REQUIRE(max_degree >= 0, "the bessel bases need max_degree");
  cudaStream_t st = as_stream(stream);
  if (num_nodes == 0) {
    cudaMemsetAsync(W_bar, 0, sizeof(float) * k_rbf * l_sbf * dg, st);
    return check_launch("triplet_bwd_basis_empty");
  }
  char* sws = reinterpret_cast<char*>(workspace) + generic_ws_bytes(num_nodes, k_rbf, l_sbf, dg) +
              fast_ws_bytes(num_nodes, num_edges, k_rbf, l_sbf, dg) + tc_bwd_workspace_bytes(num_nodes, k_rbf, l_sbf);
  const float4* g4 = reinterpret_cast<const float4*>(geo);
  char* tb = reinterpret_cast<char*>(workspace) +
             align256(egn_triplet_bwd_workspace_bytes(num_nodes, num_edges, max_degree, k_rbf, l_sbf, dg));
  float* tab = reinterpret_cast<float*>(tb);
  float* dtab = reinterpret_cast<float*>(tb + align256(sh_radial_table_floats(num_edges, basis) * 4));
  if (int rc = sh_radial_table(g4, num_edges, static_cast<float>(cutoff), basis, tab, dtab, st)) return rc;
  int min_n = 0, accumulate = 0;
  if (g_triplet_path != 1 && fast_supported(k_rbf, l_sbf, dg)) {  // as egn_triplet_fwd_basis
    char* fws = reinterpret_cast<char*>(workspace) + generic_ws_bytes(num_nodes, k_rbf, l_sbf, dg);
    if (int rc = fast_bwd(edge_ptr, rev, g4, num_nodes, num_edges, X, W, k_rbf, l_sbf, dg, rbf_params(k_rbf, cutoff),
                          S_bar, X_bar, W_bar, reinterpret_cast<float4*>(edge_grad), fws, st, phases, basis, tab, dtab))
      return rc;
    if (max_degree <= kFastMaxDeg) return 0;
    min_n = kFastMaxDeg;
    accumulate = 1;
  }
  return sh_bwd(edge_ptr, rev, g4, num_nodes, num_edges, max_degree, X, W, k_rbf, l_sbf, dg, rbf_params(k_rbf, cutoff),
                static_cast<float>(cutoff), basis, S_bar, X_bar, W_bar, reinterpret_cast<float4*>(edge_grad), sws,
                min_n, accumulate, st, tab, dtab);
}

int egn_triplet_fwd_window(const int64_t* edge_ptr, const int32_t* rev, const float* geo, int64_t num_nodes,
                           int64_t first_lo, int64_t last_hi, const float* X, const float* W, int k_rbf, int l_sbf,
                           int dg, double cutoff, float* S, egn_stream_t stream) {
  if (int rc = check_dims(k_rbf, l_sbf, dg)) return rc;
  if (num_nodes == 0) return 0;
  RbfParams rp = rbf_params(k_rbf, cutoff);
  const float4* g4 = reinterpret_cast<const float4*>(geo);
  cudaStream_t st = as_stream(stream);
  const TripWin win{first_lo, last_hi};
#define EGN_FWD(CW, GC, R) \
  return launch_fwd<CW, GC, R>(edge_ptr, rev, g4, num_nodes, X, W, k_rbf, l_sbf, dg, rp, S, -1, st, win)
  if (dg <= 4) EGN_FWD(4, 1, 1);
  if (dg <= 8) EGN_FWD(8, 1, 1);
  if (dg <= 16) EGN_FWD(8, 2, 2);
  if (dg <= 32) EGN_FWD(8, 4, 2);
  if (dg <= 64) EGN_FWD(8, 8, 4);
  if (dg <= 128) EGN_FWD(8, 16, 4);
  EGN_FWD(8, 32, 4);
#undef EGN_FWD
}

int egn_triplet_bwd_window(const int64_t* edge_ptr, const int32_t* rev, const float* geo, int64_t num_nodes,
                           int64_t first_lo, int64_t last_hi, int max_degree, const float* X, const float* W,
                           int k_rbf, int l_sbf, int dg, double cutoff, const float* S_bar, float* X_bar,
                           float* W_bar, float* edge_grad, void* workspace, egn_stream_t stream) {
  if (int rc = check_dims(k_rbf, l_sbf, dg)) return rc;
  cudaStream_t st = as_stream(stream);
  if (num_nodes == 0) {
    cudaMemsetAsync(W_bar, 0, sizeof(float) * k_rbf * l_sbf * dg, st);
    return check_launch("triplet_bwd_window_empty");
  }
  RbfParams rp = rbf_params(k_rbf, cutoff);
  const float4* g4 = reinterpret_cast<const float4*>(geo);
  float4* eg = reinterpret_cast<float4*>(edge_grad);
  const TripWin win{first_lo, last_hi};
#define EGN_BWD(CW, GC, R) \
  return launch_bwd<CW, GC, R>(edge_ptr, rev, g4, num_nodes, X, W, k_rbf, l_sbf, dg, max_degree, rp, S_bar, X_bar, \
                               W_bar, eg, workspace, -1, 0, st, win)
  if (dg <= 4) EGN_BWD(4, 1, 1);
  if (dg <= 8) EGN_BWD(8, 1, 1);
  if (dg <= 16) EGN_BWD(8, 2, 2);
  if (dg <= 32) EGN_BWD(8, 4, 2);
  if (dg <= 64) EGN_BWD(8, 8, 4);
  if (dg <= 128) EGN_BWD(8, 16, 4);
  EGN_BWD(8, 32, 4);
#undef EGN_BWD
}

int egn_triplet_terms(const int64_t* edge_ptr, const int32_t* rev, const float* geo,
                      const int64_t* tri_ptr, int64_t num_nodes, const float* X, const float* W,
                      int k_rbf, int l_sbf, int dg, double cutoff, float* P, egn_stream_t stream) {
  EGN_REQUIRE(k_rbf >= 1 && l_sbf >= 1 && dg >= 1, "bad dims");
  if (num_nodes == 0) return 0;
  int grid = static_cast<int>(num_nodes < 65535 ? num_nodes : 65535);
  triplet_terms_kernel<<<grid, 256, 0, as_stream(stream)>>>(
      edge_ptr, rev, reinterpret_cast<const float4*>(geo), tri_ptr, num_nodes, X, W, k_rbf, l_sbf,
      dg, rbf_params(k_rbf, cutoff), P);
  return check_launch("triplet_terms");
}

}  // extern "C"
