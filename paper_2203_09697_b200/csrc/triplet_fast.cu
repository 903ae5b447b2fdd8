// Fast path of the triplet interaction for centres with deg(j) <= 64 and the
// model's basis sizes known at compile time (K = 6 radial, L = 7 angular).
//
// Same mathematics as triplet.cu (see the derivation there and DESIGN.md);
// the work per centre is reorganised as small dense products so that the
// inner loops are pure FFMA with register blocking:
//
//   forward   S[p, c]      = sum_{(q,l)} C[(q,l), p] * Q[(q,l), c]
//             C[(q,l), p]  = T_l(x_pq) (0 on the diagonal)         -- Chebyshev table
//             Q[(q,l), c]  = X[rq, c] * sum_k rbf_k(d_q) W[k, l, c]  -- gate table
//   backward  (kernel bw1)  xbar(p, q) = sum_c Sbar[p, c] sum_l T_l'(x_pq) Q[(q,l), c]
//             -> dE/dv_p, dE/dv_q (row / column passes over an XB tile)
//             (kernel bw2)  Qbar[(q,l), c] = sum_p C[(q,l), p] Sbar[p, c]
//             -> X_bar[rq], R_bar -> W_bar partials, dd_q partials
//
// Threads: 128 = 16 row groups x 8 channel groups; a thread owns rows
// {rg, rg+16, rg+32, rg+48} (first TMR of them) and channels
// {4cg..4cg+3, 32+4cg..32+4cg+3} of a 64-channel block, so every shared
// load is a 128-bit vector that 8 (or 16) lanes share.
#include <algorithm>

#include "common.cuh"

namespace egn {
namespace fast {

constexpr int kT = 128;
constexpr int kN = 64;    // max centre degree on this path
constexpr int kCB = 64;   // channels per block
constexpr int kQC = 8;    // q rows per table chunk (forward / bw1)

__device__ __forceinline__ int chan(int cg, int i) { return i < 4 ? cg * 4 + i : 32 + cg * 4 + (i - 4); }
// permuted row slot: thread group rg reads rows rg, rg+16, rg+32, rg+48 as one float4
__device__ __forceinline__ int rslot(int p) { return (p & 15) * 4 + (p >> 4); }

// packed fp32 FMA (FFMA2, sm_100a: two lanes of fp32 per instruction, twice the FFMA rate):
// c + a * b on both halves with a scalar a broadcast.  Per half it is the same fma.rn as
// fmaf, so a loop rewritten on it gives bit-identical results.
__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) { return __ffma2_rn(make_float2(a, a), b, c); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
constexpr int kLP = 4;  // L = 7 angular orders as 4 pairs (the 8th is zero)

__device__ __forceinline__ float rbf1(float d, int k, RbfParams rp) {
  const float dd = d - rp.step * k;
  return __expf(-rp.gamma * dd * dd);
}

// Basis MODE of the pairwise kernels: 0 = the reference's Gaussian rbf x cos(l a) = T_l(x);
// 1 = GemNet-T's CBF: radial Bessel basis e_k(d) (rows of the per-call radial table, stride 8,
// triplet_sh.cu radial_table_kernel) x Y_l0(a) = sqrt((2l+1)/4pi) P_l(x).
// MODE 2 = DimeNet++'s SBF: radial part sqrt(2/c^3)/|j_{l+1}(z_lk)| u(d/c) j_l(z_lk d/c) depends on
// (k, l) (table rows of 44 floats, [k][l]) x the same Y_l0 angular rows as MODE 1.
// Radial rows per in-edge in shared memory (rb_stride floats): MODE 0 / 1 K values; MODE 2 the
// K x L values as [k][8] (LMAJOR = false: l pairs adjacent, for the gate products) or [l][8]
// (LMAJOR = true: k pairs adjacent, for bw2's weight-gradient epilogue), zero padded.
template <int K, int L, int MODE>
constexpr int rb_stride() { return MODE == 2 ? 8 * (K > L ? K : L) : K; }

template <int K, int MODE = 0, bool LMAJOR = false>
__device__ __forceinline__ void load_center(float4* Us, float* Rb, const float4* __restrict__ geo, int64_t off,
                                            int n, RbfParams rp, const float* __restrict__ rtab = nullptr,
                                            float* DRb = nullptr, const float* __restrict__ dtab = nullptr) {
  for (int i = threadIdx.x; i < n; i += kT) Us[i] = geo[off + i];
  if constexpr (MODE == 2) {
    constexpr int L = 7, RS = rb_stride<K, 7, 2>(), TS = 44;  // sh radial table row (rad_stride<2>)
    for (int i = threadIdx.x; i < n * RS; i += kT) {
      const int q = i / RS, r = i - q * RS;
      const int k = LMAJOR ? (r & 7) : (r >> 3), l = LMAJOR ? (r >> 3) : (r & 7);
      const bool ok = k < K && l < L;
      Rb[i] = ok ? __ldg(rtab + (off + q) * TS + k * L + l) : 0.f;
      if (DRb) DRb[i] = ok ? __ldg(dtab + (off + q) * TS + k * L + l) : 0.f;
    }
  } else {
    for (int i = threadIdx.x; i < n * K; i += kT) {
      const int q = i / K, k = i - q * K;
      if constexpr (MODE == 0) {
        Rb[i] = rbf1(geo[off + q].w, k, rp);
      } else {
        Rb[i] = __ldg(rtab + (off + q) * 8 + k);
        if (DRb) DRb[i] = __ldg(dtab + (off + q) * 8 + k);
      }
    }
  }
}

// angular factor f_l(x) of the basis (masked by m) and the contraction sum_l f_l'(x) z_l
__constant__ float c_ynorm[8] = {0.28209479177387814f, 0.4886025119029199f, 0.6307831305050401f,
                                 0.7463526651802308f, 0.8462843753216345f, 0.9356025796273888f,
                                 1.0171072362820548f, 1.0925484305920792f};  // sqrt((2l+1)/(4 pi))
template <int L, int MODE>
__device__ __forceinline__ void angular_row(float x, float m, float (&f)[L]) {
  if constexpr (MODE == 0) {  // T_l(x) = cos(l a)
    float tp = m * x, tc = m;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      f[l] = tc;
      const float tn = fmaf(2.f * x, tc, -tp);
      tp = tc;
      tc = tn;
    }
  } else {  // Y_l0: P_{l+1} = (2l+1)/(l+1) x P_l - l/(l+1) P_{l-1} (constant coefficients, no division)
    float pm = 0.f, pc = m;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      f[l] = c_ynorm[l] * pc;
      const float a = static_cast<float>(2 * l + 1) / static_cast<float>(l + 1);
      const float b = static_cast<float>(l) / static_cast<float>(l + 1);
      const float pn = fmaf(a * x, pc, -b * pm);
      pm = pc;
      pc = pn;
    }
  }
}
template <int L, int MODE, typename ZF>
__device__ __forceinline__ float angular_dcontract(float x, ZF z) {
  float v = 0.f;
  if constexpr (MODE == 0) {  // T_l' = l U_{l-1}
    float um = 0.f, uc = 1.f;
#pragma unroll
    for (int l = 1; l < L; ++l) {
      v = fmaf(static_cast<float>(l) * uc, z(l), v);
      const float un = fmaf(2.f * x, uc, -um);
      um = uc;
      uc = un;
    }
  } else {  // P_{l+1}' = P_{l-1}' + (2l+1) P_l
    float pm = 1.f, pc = x;     // P_0, P_1
    float dm = 0.f, dc = 1.f;   // P_0', P_1'
#pragma unroll
    for (int l = 1; l < L; ++l) {
      v = fmaf(c_ynorm[l] * dc, z(l), v);
      const float dn = fmaf(static_cast<float>(2 * l + 1), pc, dm);
      const float a = static_cast<float>(2 * l + 1) / static_cast<float>(l + 1);
      const float b = static_cast<float>(l) / static_cast<float>(l + 1);
      const float pn = fmaf(a * x, pc, -b * pm);
      dm = dc;
      dc = dn;
      pm = pc;
      pc = pn;
    }
  }
  return v;
}

// Q chunk: rows (t, l) for t < nq (row stride RS floats), natural channel order; thread
// (cq = tid & 63, half = tid >> 6)
// X rows of chunk [q0, q0 + nq) for this thread (t = half + 2 i): issued one chunk ahead, so
// the gathers are in flight during the previous chunk's contraction
__device__ __forceinline__ void load_x(float (&xs)[kQC / 2], const int32_t* __restrict__ rev,
                                       const float* __restrict__ X, int64_t off, int q0, int nq, int dg, int c0) {
  const int cq = threadIdx.x & 63, half = threadIdx.x >> 6;
  const int c = c0 + cq;
#pragma unroll
  for (int i = 0; i < kQC / 2; ++i) {
    const int t = half + 2 * i;
    xs[i] = (t < nq && c < dg) ? __ldg(X + static_cast<int64_t>(rev[off + q0 + t]) * dg + c) : 0.f;
  }
}

template <int K, int L, int RS = kCB, int MODE = 0>
__device__ __forceinline__ void build_q(float* Qs, const float2 (&wreg)[K][kLP], const float* Rb,
                                        const float (&xs)[kQC / 2], int q0, int nq) {
  const int cq = threadIdx.x & 63, half = threadIdx.x >> 6;
#pragma unroll
  for (int i = 0; i < kQC / 2; ++i) {
    const int t = half + 2 * i;
    if (t >= nq) break;
    const float xv = xs[i];
    float2 s[kLP];
#pragma unroll
    for (int lp = 0; lp < kLP; ++lp) s[lp] = make_float2(0.f, 0.f);
    if constexpr (MODE == 2) {  // radial (k, l) rows [k][8]: the l pairs are the packed operands
      const float* rb = Rb + (q0 + t) * rb_stride<K, L, 2>();
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int lp = 0; lp < kLP; ++lp)
          s[lp] = ffma2(*reinterpret_cast<const float2*>(rb + k * 8 + 2 * lp), wreg[k][lp], s[lp]);
    } else {
      const float* rb = Rb + (q0 + t) * K;
      float r[K];
#pragma unroll
      for (int k = 0; k < K; ++k) r[k] = rb[k];
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int lp = 0; lp < kLP; ++lp) s[lp] = ffma2(r[k], wreg[k][lp], s[lp]);
    }
#pragma unroll
    for (int l = 0; l < L; ++l) Qs[(t * L + l) * RS + cq] = xv * ((l & 1) ? s[l >> 1].y : s[l >> 1].x);
  }
}

// Chebyshev chunk Ct[(t,l)][slot(p)] = T_l(x_pq) or T_l'(x_pq), masked on p == q / p >= n.
// slot(p) = (p % RG) * 4 + p / RG for rows = 4 RG, RG in {4, 8, 16} (RG = 16: rslot): row group g reads its rows
// g, g + RG, g + 2 RG, g + 3 RG as one float4.
template <int L, bool DERIV, int MODE = 0>
__device__ __forceinline__ void build_c(float* Ct, const float4* Us, int n, int rows, int q0, int nq, int RG = 16) {
  for (int i = threadIdx.x; i < nq * rows; i += kT) {
    const int t = i / rows, p = i - t * rows;
    const int q = q0 + t;
    const bool ok = p < n && p != q;
    float4 a = Us[q];
    float4 b = ok ? Us[p] : a;
    const float x = a.x * b.x + a.y * b.y + a.z * b.z;
    const float m = ok ? 1.f : 0.f;
    float* dst = Ct + t * L * kCB + (p & (RG - 1)) * 4 + (RG == 16 ? p >> 4 : (RG == 8 ? p >> 3 : p >> 2));
    if (!DERIV) {
      float f[L];
      angular_row<L, MODE>(x, m, f);
#pragma unroll
      for (int l = 0; l < L; ++l) dst[l * kCB] = f[l];
    } else {
      // T_l'(x) = l U_{l-1}(x)
      float um = 0.f, uc = 0.f;
#pragma unroll
      for (int l = 0; l < L; ++l) {
        dst[l * kCB] = m * static_cast<float>(l) * uc;
        const float un = (l == 0) ? 1.f : fmaf(2.f * x, uc, -um);
        um = uc;
        uc = un;
      }
    }
  }
}

// k-split micro kernel: this thread takes kk = ks, ks + KS, ... (KS thread sets share the chunk)
template <int TMR>
__device__ __forceinline__ void micro(const float* __restrict__ A, const float* __restrict__ B, int nkk,
                                      int rg, int cg, float2 (&acc)[4][4], int ks = 0, int KS = 1) {
#pragma unroll 4
  for (int kk = ks; kk < nkk; kk += KS) {
    const float4 a = *reinterpret_cast<const float4*>(A + kk * kCB + rg * 4);
    const float4 b0 = *reinterpret_cast<const float4*>(B + kk * kCB + cg * 4);
    const float4 b1 = *reinterpret_cast<const float4*>(B + kk * kCB + 32 + cg * 4);
    const float av[4] = {a.x, a.y, a.z, a.w};
    const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                          make_float2(b1.z, b1.w)};
#pragma unroll
    for (int r = 0; r < TMR; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[r][i] = ffma2(av[r], bv[i], acc[r][i]);
  }
}

template <int K, int L>
__device__ __forceinline__ void load_wreg(float2 (&wreg)[K][kLP], const float* __restrict__ W, int dg, int c) {
  static_assert(L <= 2 * kLP, "L <= 8");
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int lp = 0; lp < kLP; ++lp) {
      const int l0 = 2 * lp, l1 = 2 * lp + 1;
      wreg[k][lp] = make_float2(c < dg && l0 < L ? W[(k * L + l0) * dg + c] : 0.f,
                                c < dg && l1 < L ? W[(k * L + l1) * dg + c] : 0.f);
    }
}

// Rows [off, off + n) x channels [c0, c0 + 64) of a row-major [*, dg] array into dst[p * stride + c]
// (zero past dg).  16-byte cp.async when dg % 4 == 0 (rows 16-byte aligned, a granule is wholly in
// or out of range): every request of the CTA is in flight at once instead of one load latency per
// element.  The caller runs stage_wait() before the barrier that publishes dst.
__device__ __forceinline__ void stage_rows(float* dst, int stride, const float* __restrict__ src, int64_t off, int n,
                                           int dg, int c0) {
  if ((dg & 3) == 0) {
    for (int i = threadIdx.x; i < n * (kCB / 4); i += kT) {
      const int p = i >> 4, c = (i & 15) * 4;
      const bool ok = c0 + c < dg;
      const float* g = ok ? src + (off + p) * dg + c0 + c : src;
      const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst + p * stride + c));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(g), "r"(ok ? 16 : 0) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  } else {
    for (int i = threadIdx.x; i < n * kCB; i += kT) {
      const int p = i >> 6, c = i & 63;
      dst[p * stride + c] = c0 + c < dg ? src[(off + p) * dg + c0 + c] : 0.f;
    }
  }
}
__device__ __forceinline__ void stage_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---------------------------------------------------------------------------
template <int K, int L, int MINB = 4, int MODE = 0>
__global__ void __launch_bounds__(kT, MINB)
fwd_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ rev,
           const float4* __restrict__ geo, int64_t nv, const float* __restrict__ X,
           const float* __restrict__ W, int dg, RbfParams rp, float* __restrict__ S,
           const float* __restrict__ rtab) {
  __shared__ float4 Us[kN];
  __shared__ __align__(16) float Rb[kN * rb_stride<K, L, MODE>()];
  __shared__ __align__(16) float Ct[kQC * L * kCB];
  __shared__ __align__(16) float Qs[kQC * L * kCB];
  const int tid = threadIdx.x;
  for (int64_t j = blockIdx.x; j < nv; j += gridDim.x) {
    const int64_t off = edge_ptr[j];
    const int n = static_cast<int>(edge_ptr[j + 1] - off);
    if (n == 0 || n > kN) continue;
    // Small centres: RG = 4 / 8 row groups of 4 rows (16 / 32 rows), and the 128 threads split
    // the (q, l) reduction KS = 4 / 2 ways (thread set ks takes kk = ks mod KS), partials combined
    // in shared memory at the end in fixed order.  A 4 x 8 thread tile reads 3 float4 per 16 FFMA2
    // (a 2 x 8 tile needed 3 per 8: shared-memory bound).  Larger centres: 16 groups, tmr rows each.
    const int RG = n <= 16 ? 4 : (n <= 32 ? 8 : 16);
    const int KS = 128 / (RG * 8);
    const int tpg = RG * 8;
    const int ks = tid / tpg, w = tid - ks * tpg;
    const int cg = w & 7, rg = w >> 3;
    const int tmr = KS > 1 ? 4 : (n + 15) >> 4;
    const int rows = RG == 16 ? tmr * 16 : 4 * RG;
    __syncthreads();
    load_center<K, MODE>(Us, Rb, geo, off, n, rp, rtab);
    for (int c0 = 0; c0 < dg; c0 += kCB) {
      float2 wreg[K][kLP];
      load_wreg<K, L>(wreg, W, dg, c0 + (tid & 63));
      float2 acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[r][i] = make_float2(0.f, 0.f);
      float xs[kQC / 2];
      load_x(xs, rev, X, off, 0, min(kQC, n), dg, c0);
      for (int q0 = 0; q0 < n; q0 += kQC) {
        const int nq = min(kQC, n - q0);
        __syncthreads();
        build_q<K, L, kCB, MODE>(Qs, wreg, Rb, xs, q0, nq);
        build_c<L, false, MODE>(Ct, Us, n, rows, q0, nq, RG);
        __syncthreads();
        if (q0 + kQC < n) load_x(xs, rev, X, off, q0 + kQC, min(kQC, n - q0 - kQC), dg, c0);
        const int nkk = nq * L;
        if (KS > 1) {
          micro<4>(Ct, Qs, nkk, rg, cg, acc, ks, KS);
        } else {
          switch (tmr) {
            case 3: micro<3>(Ct, Qs, nkk, rg, cg, acc); break;
            default: micro<4>(Ct, Qs, nkk, rg, cg, acc); break;
          }
        }
      }
      if (KS > 1) {
        // combine the k-split partials: set ks > 0 parks its tile in Ct (layout [set][value][w],
        // conflict-free), set 0 adds them in set order
        __syncthreads();
        if (ks > 0) {
          float* red = Ct + (ks - 1) * 32 * tpg + w;
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              red[(r * 8 + 2 * i) * tpg] = acc[r][i].x;
              red[(r * 8 + 2 * i + 1) * tpg] = acc[r][i].y;
            }
        }
        __syncthreads();
        if (ks == 0) {
          for (int o = 1; o < KS; ++o) {
            const float* red = Ct + (o - 1) * 32 * tpg + w;
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                acc[r][i].x += red[(r * 8 + 2 * i) * tpg];
                acc[r][i].y += red[(r * 8 + 2 * i + 1) * tpg];
              }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int p = rg + RG * r;
        if (ks == 0 && r < tmr && p < n) {
          float* dst = S + (off + p) * dg + c0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int c = chan(cg, i);
            if (c0 + c < dg) dst[c] = (i & 1) ? acc[r][i >> 1].y : acc[r][i >> 1].x;
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// bw1: xbar(p, q) = sum_l T_l'(x_pq) Z[(q,l), p],  Z[(q,l), p] = sum_c Q[(q,l), c] Sbar[p, c]
// Per (centre, 8-in-edge chunk, 64-channel block), Z is a small GEMM whose thread tile is one
// in-edge q x all l x PP rows p (rows interleaved over the threads so shared-memory rows
// of Sbar spread over the banks); xbar accumulates in shared memory, one owner per (p, q).
// Then the row / column pass turns xbar into dE/dv (edge_grad.xyz += F / d).
constexpr int kSbStride = kCB + 4;  // padded Sbar / Q rows (bank spread for 16-byte loads)
// Row-pair layout of S-bar for PP >= 2: pair pr = 16 h + g holds rows a = 32 h + g and a + 16
// (the two rows one FFMA2 updates) interleaved per channel, [pr][c][2] at stride kPairStride:
// a float4 load gives (a, a + 16) at channels c and c + 1, already the packed operand pairs (no
// register moves to pair rows that came from two loads).  Same footprint as [kN][kSbStride].
constexpr int kPairStride = 2 * kCB + 8;  // 136 floats: 4 pairs of a warp on distinct banks
static_assert(kN / 2 * kPairStride == kN * kSbStride, "pair layout footprint");

// rows [off, off + n) of S-bar, channels [c0, c0 + 64), into the pair layout (np pairs); every
// global load of the thread is issued before its stores
__device__ __forceinline__ void stage_pairs(float* dst, const float* __restrict__ src, int64_t off, int n, int np,
                                            int dg, int c0) {
  auto load4 = [&](int row, int c) -> float4 {
    if (row >= n) return make_float4(0.f, 0.f, 0.f, 0.f);
    const float* g = src + (off + row) * dg + c0 + c;
    if ((dg & 3) == 0) return c0 + c < dg ? __ldg(reinterpret_cast<const float4*>(g)) : make_float4(0.f, 0.f, 0.f, 0.f);
    return make_float4(c0 + c < dg ? __ldg(g) : 0.f, c0 + c + 1 < dg ? __ldg(g + 1) : 0.f,
                       c0 + c + 2 < dg ? __ldg(g + 2) : 0.f, c0 + c + 3 < dg ? __ldg(g + 3) : 0.f);
  };
  constexpr int kIt = (kN / 2) * (kCB / 4) / kT;  // 4
  float4 va[kIt], vb[kIt];
  if (np * (kCB / 4) <= kT) {  // one granule pair per thread
    const int pr = threadIdx.x >> 4, c = (threadIdx.x & 15) * 4;
    if (pr < np) {
      const int ra = (pr >> 4) * 32 + (pr & 15);
      const float4 a = load4(ra, c), b = load4(ra + 16, c);
      float4* d = reinterpret_cast<float4*>(dst + pr * kPairStride + 2 * c);
      d[0] = make_float4(a.x, b.x, a.y, b.y);
      d[1] = make_float4(a.z, b.z, a.w, b.w);
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < kIt; ++k) {
    const int i = threadIdx.x + k * kT;
    const int pr = i >> 4, c = (i & 15) * 4;
    const int ra = (pr >> 4) * 32 + (pr & 15);
    if (pr < np) {
      va[k] = load4(ra, c);
      vb[k] = load4(ra + 16, c);
    }
  }
#pragma unroll
  for (int k = 0; k < kIt; ++k) {
    const int i = threadIdx.x + k * kT;
    const int pr = i >> 4, c = (i & 15) * 4;
    if (pr < np) {
      float4* d = reinterpret_cast<float4*>(dst + pr * kPairStride + 2 * c);
      d[0] = make_float4(va[k].x, vb[k].x, va[k].y, vb[k].y);
      d[1] = make_float4(va[k].z, vb[k].z, va[k].w, vb[k].w);
    }
  }
}

template <int K, int L, int PP, int MODE = 0>
__device__ __forceinline__ void bw1_tile(const float* Qs, const float* Sb, const float4* Us, float* XB, int n, int q0,
                                         int nq, int G) {
  // warp = 8 in-edges q x 4 row groups: a Q-row load is 8 distinct 16-byte rows (one wavefront,
  // conflict-free at stride 7 x 68 floats) and an S-bar load 4 (one wavefront); G = 16 row groups
  const int tid = threadIdx.x, lane = tid & 31;
  const int t = lane & 7, pg = (lane >> 3) + 4 * (tid >> 5);
  if (t >= nq) return;
  // Z[(q, l), p] for l >= 1 (T_0' = 0: the l = 0 row is never needed).  Packed accumulators:
  // row pairs (p_i, p_i+1) for PP >= 2 (bit-identical to the scalar loop), even / odd channel
  // halves for PP = 1.
  constexpr int PH = PP >= 2 ? PP / 2 : 1;
  float2 acc2[L][PH];
#pragma unroll
  for (int l = 1; l < L; ++l)
#pragma unroll
    for (int i = 0; i < PH; ++i) acc2[l][i] = make_float2(0.f, 0.f);
  const float* qrow = Qs + (t * L) * kSbStride;
  if constexpr (PP >= 2) {
    // S-bar in the row-pair layout (stage_pairs): pair i of this thread = rows (pg + 32 i, + 16)
#pragma unroll 2
    for (int c = 0; c < kCB; c += 4) {
      float4 s0[PH], s1[PH];
#pragma unroll
      for (int i = 0; i < PH; ++i) {
        const float* sp = Sb + (16 * i + pg) * kPairStride + 2 * c;
        s0[i] = *reinterpret_cast<const float4*>(sp);
        s1[i] = *reinterpret_cast<const float4*>(sp + 4);
      }
#pragma unroll
      for (int l = 1; l < L; ++l) {
        const float4 qv = *reinterpret_cast<const float4*>(qrow + l * kSbStride + c);
#pragma unroll
        for (int i = 0; i < PH; ++i) {
          acc2[l][i] = ffma2(qv.x, make_float2(s0[i].x, s0[i].y), acc2[l][i]);
          acc2[l][i] = ffma2(qv.y, make_float2(s0[i].z, s0[i].w), acc2[l][i]);
          acc2[l][i] = ffma2(qv.z, make_float2(s1[i].x, s1[i].y), acc2[l][i]);
          acc2[l][i] = ffma2(qv.w, make_float2(s1[i].z, s1[i].w), acc2[l][i]);
        }
      }
    }
  } else {
#pragma unroll 4
    for (int c = 0; c < kCB; c += 4) {
      const float4 sv = *reinterpret_cast<const float4*>(Sb + pg * kSbStride + c);
#pragma unroll
      for (int l = 1; l < L; ++l) {
        const float4 qv = *reinterpret_cast<const float4*>(qrow + l * kSbStride + c);
        acc2[l][0] = ffma2(make_float2(qv.x, qv.y), make_float2(sv.x, sv.y), acc2[l][0]);
        acc2[l][0] = ffma2(make_float2(qv.z, qv.w), make_float2(sv.z, sv.w), acc2[l][0]);
      }
    }
  }
  auto zval = [&](int l, int i) -> float {
    if (PP >= 2) return (i & 1) ? acc2[l][i >> 1].y : acc2[l][i >> 1].x;
    return acc2[l][0].x + acc2[l][0].y;
  };

  const int q = q0 + t;
  const float4 uq = Us[q];
#pragma unroll
  for (int i = 0; i < PP; ++i) {
    const int p = pg + G * i;
    if (p >= n || p == q) continue;
    const float4 up = Us[p];
    const float x = up.x * uq.x + up.y * uq.y + up.z * uq.z;
    // sum_l f_l'(x) Z_l
    const float v = angular_dcontract<L, MODE>(x, [&](int l) { return zval(l, i); });
    XB[p * (kN + 1) + q] += v;  // single owner per (p, q), ordered over channel blocks
  }
}

template <int K, int L, int MINB = 4, int MODE = 0>
__global__ void __launch_bounds__(kT, MINB)
bw1_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ rev,
           const float4* __restrict__ geo, int64_t nv, const float* __restrict__ X,
           const float* __restrict__ W, int dg, RbfParams rp, const float* __restrict__ Sbar,
           float4* __restrict__ edge_grad, const float* __restrict__ rtab) {
  extern __shared__ __align__(16) float bsm[];
  float4* Us = reinterpret_cast<float4*>(bsm);             // [kN]
  float* Rb = bsm + 4 * kN;                                 // [kN * K]
  float* Qs = Rb + ((kN * rb_stride<K, L, MODE>() + 3) & ~3);  // [kQC * L][kSbStride]
  float* Sb = Qs + kQC * L * kSbStride;                     // [kN][kSbStride]
  float* XB = Sb + kN * kSbStride;                          // [kN][kN + 1]
  const int tid = threadIdx.x;
  for (int64_t j = blockIdx.x; j < nv; j += gridDim.x) {
    const int64_t off = edge_ptr[j];
    const int n = static_cast<int>(edge_ptr[j + 1] - off);
    if (n < 2 || n > kN) continue;
    __syncthreads();
    load_center<K, MODE>(Us, Rb, geo, off, n, rp, rtab);
    for (int i = tid; i < n * (kN + 1); i += kT) XB[i] = 0.f;
    // thread tile: PP rows p = pg + 16 i of one in-edge q (bw1_tile)
    const int PP = n <= 16 ? 1 : (n <= 32 ? 2 : 4);
    const int G = 16;
    for (int c0 = 0; c0 < dg; c0 += kCB) {
      __syncthreads();
      if (PP == 1) stage_rows(Sb, kSbStride, Sbar, off, n, dg, c0);
      else stage_pairs(Sb, Sbar, off, n, PP == 2 ? 16 : 32, dg, c0);
      float2 wreg[K][kLP];
      load_wreg<K, L>(wreg, W, dg, c0 + (tid & 63));
      float xs[kQC / 2];
      load_x(xs, rev, X, off, 0, min(kQC, n), dg, c0);
      for (int q0 = 0; q0 < n; q0 += kQC) {
        const int nq = min(kQC, n - q0);
        if (q0 == 0) stage_wait();
        __syncthreads();
        build_q<K, L, kSbStride, MODE>(Qs, wreg, Rb, xs, q0, nq);
        __syncthreads();
        if (q0 + kQC < n) load_x(xs, rev, X, off, q0 + kQC, min(kQC, n - q0 - kQC), dg, c0);
        switch (PP) {
          case 1: bw1_tile<K, L, 1, MODE>(Qs, Sb, Us, XB, n, q0, nq, G); break;
          case 2: bw1_tile<K, L, 2, MODE>(Qs, Sb, Us, XB, n, q0, nq, G); break;
          default: bw1_tile<K, L, 4, MODE>(Qs, Sb, Us, XB, n, q0, nq, G); break;
        }
      }
    }
    __syncthreads();
    // dE/dv_e for every out-edge e of the centre: four lanes per e take the partners o = sub,
    // sub + 4, ... (rows then columns), combined by a fixed shuffle tree.  Every thread runs the
    // same number of rounds so the shuffles see full warps.
    for (int base = 0; base < n * 4; base += kT) {
      const int i = base + tid, e = i >> 2, sub = i & 3;
      const bool live = e < n;
      const float4 ue = Us[live ? e : 0];
      float fx = 0.f, fy = 0.f, fz = 0.f;
      if (live) {
        for (int o = sub; o < n; o += 4) {
          if (o == e) continue;
          const float4 uo = Us[o];
          const float x = ue.x * uo.x + ue.y * uo.y + ue.z * uo.z;
          const float v = XB[e * (kN + 1) + o] + XB[o * (kN + 1) + e];
          fx = fmaf(v, uo.x - x * ue.x, fx);
          fy = fmaf(v, uo.y - x * ue.y, fy);
          fz = fmaf(v, uo.z - x * ue.z, fz);
        }
      }
#pragma unroll
      for (int m = 1; m < 4; m <<= 1) {
        fx += __shfl_xor_sync(0xffffffffu, fx, m);
        fy += __shfl_xor_sync(0xffffffffu, fy, m);
        fz += __shfl_xor_sync(0xffffffffu, fz, m);
      }
      // x, y, z only (4-byte accesses): bw2 may update .w of the same edge concurrently when
      // the angle phase runs on its own stream (egn_triplet_bwd_ex phases)
      if (live && sub < 3) {
        const float f = sub == 0 ? fx : (sub == 1 ? fy : fz);
        reinterpret_cast<float*>(edge_grad + off + e)[sub] += f / ue.w;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// bw2: Qbar = C^T Sbar per (centre, 64-channel block); X_bar, W_bar partials, dd partials.
// grid = (centre CTAs, channel blocks).  The in-edges q of a centre go in batches of TQ = 16
// (or 8 for a short tail).  Main loop: thread (rg, cg) owns row q = qb0 + rg, all L and
// TQ/2 channels, Qbar accumulated over the out-edges p.  The batch's Qbar is staged in shared
// memory; the epilogue then runs one thread per channel (two halves splitting the rows), so
// the gate weights W[:, :, c] sit in registers and the chain rule folds through
// v_k = sum_l Qbar_l W[k, l, c]:
//   X_bar = sum_k rbf_k v_k,  dd = sum_c X sum_k rbf_k' v_k,  W_bar[k, l, c] += rbf_k X Qbar_l
// W_bar accumulates in registers for the CTA's whole life (one partial per CTA).
template <int L, int TQ>
__device__ __forceinline__ void bw2_main(const float* Cb, const float* Sb, int n, float* QB) {
  constexpr int CG = kT / TQ;           // channel groups: 8 (TQ 16) or 16 (TQ 8)
  constexpr int CPT = kCB / CG;         // channels per thread: 8 or 4
  const int tid = threadIdx.x, cg = tid % CG, rg = tid / CG;
  float2 acc[L][CPT / 2];
#pragma unroll
  for (int l = 0; l < L; ++l)
#pragma unroll
    for (int i = 0; i < CPT / 2; ++i) acc[l][i] = make_float2(0.f, 0.f);
#pragma unroll 2
  for (int p = 0; p < n; ++p) {
    const float4 a0 = *reinterpret_cast<const float4*>(Cb + (p * TQ + rg) * 8);
    const float4 a1 = *reinterpret_cast<const float4*>(Cb + (p * TQ + rg) * 8 + 4);
    const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    float bv[CPT];
    {
      const float4 b0 = *reinterpret_cast<const float4*>(Sb + p * kCB + cg * 4);
      bv[0] = b0.x; bv[1] = b0.y; bv[2] = b0.z; bv[3] = b0.w;
    }
    if (CPT == 8) {
      const float4 b1 = *reinterpret_cast<const float4*>(Sb + p * kCB + 32 + cg * 4);
      bv[4 % CPT] = b1.x; bv[5 % CPT] = b1.y; bv[6 % CPT] = b1.z; bv[7 % CPT] = b1.w;
    }
#pragma unroll
    for (int l = 0; l < L; ++l)
#pragma unroll
      for (int i = 0; i < CPT / 2; ++i) acc[l][i] = ffma2(av[l], make_float2(bv[2 * i], bv[2 * i + 1]), acc[l][i]);
  }
  __syncthreads();  // every Cb read done: QB aliases it
#pragma unroll
  for (int l = 0; l < L; ++l) {
    float* row = QB + (rg * L + l) * kCB;
    *reinterpret_cast<float4*>(row + cg * 4) = make_float4(acc[l][0].x, acc[l][0].y, acc[l][1].x, acc[l][1].y);
    if (CPT == 8)
      *reinterpret_cast<float4*>(row + 32 + cg * 4) =
          make_float4(acc[l][2 % (CPT / 2)].x, acc[l][2 % (CPT / 2)].y, acc[l][3 % (CPT / 2)].x,
                      acc[l][3 % (CPT / 2)].y);
  }
}

template <int K, int L, int MINB = 3, int MODE = 0>
__global__ void __launch_bounds__(kT, MINB)
bw2_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ rev,
           const float4* __restrict__ geo, int64_t nv, const float* __restrict__ X,
           const float* __restrict__ W, int dg, RbfParams rp, const float* __restrict__ Sbar,
           float* __restrict__ Xbar, float* __restrict__ wbar_part, float* __restrict__ dd_part,
           int64_t num_edges, float4* __restrict__ edge_grad, const float* __restrict__ rtab,
           const float* __restrict__ dtab) {
  static_assert(L <= 8, "L <= 8");
  extern __shared__ __align__(16) float dsm[];
  float4* Us = reinterpret_cast<float4*>(dsm);      // [64]
  constexpr int RBS = rb_stride<K, L, MODE>();       // radial row per in-edge (MODE 2: [l][8 k])
  float* Rb = dsm + 4 * kN;                          // [64 * RBS]
  float* Cb = Rb + ((kN * RBS + 3) & ~3);            // [p][TQ q][8 l]; QB [TQ][L][64] aliases it
  float* Sb = Cb + kN * 16 * 8;                      // Sbar rows of the centre, this channel block
  float* Wsm = Sb + kN * kCB;                        // W[k, l, c0 + c]
  float* DD = Wsm + K * L * kCB;                     // [16][2] dd partial per row and warp
  float* DRb = DD + 32;                               // [64 * RBS] radial d-derivatives (MODE 1, 2)
  int* Rv = reinterpret_cast<int*>(DRb + kN * RBS);    // [64] rev of the centre's edges
  const int tid = threadIdx.x;
  const int c = tid & (kCB - 1), h = tid >> 6;       // epilogue: channel, row half
  const int64_t c0 = static_cast<int64_t>(blockIdx.y) * kCB;
  const bool cok = c0 + c < dg;
  for (int i = tid; i < K * L * kCB; i += kT) {
    const int kl = i / kCB, cc = i - kl * kCB;
    Wsm[i] = c0 + cc < dg ? W[kl * dg + c0 + cc] : 0.f;
  }
  static_assert(K % 2 == 0, "K pairs");
  constexpr int KP = K / 2;
  float2 wb[KP][L];  // W_bar[2 kp, l], W_bar[2 kp + 1, l]
#pragma unroll
  for (int k = 0; k < KP; ++k)
#pragma unroll
    for (int l = 0; l < L; ++l) wb[k][l] = make_float2(0.f, 0.f);
  for (int64_t j = blockIdx.x; j < nv; j += gridDim.x) {
    const int64_t off = edge_ptr[j];
    const int n = static_cast<int>(edge_ptr[j + 1] - off);
    if (n > kN || n == 0) continue;
    if (n == 1) {
      const int64_t r0 = rev[off];
      if (tid < kCB && cok) Xbar[r0 * dg + c0 + tid] = 0.f;
      if (tid == 0 && gridDim.y > 1) dd_part[blockIdx.y * num_edges + off] = 0.f;
      continue;
    }
    __syncthreads();
    stage_rows(Sb, kCB, Sbar, off, n, dg, static_cast<int>(c0));
    for (int i = tid; i < n; i += kT) Rv[i] = rev[off + i];
    load_center<K, MODE, true>(Us, Rb, geo, off, n, rp, rtab, MODE == 0 ? nullptr : DRb, dtab);
    for (int qb0 = 0; qb0 < n; qb0 += 16) {
      const int nr = min(16, n - qb0);
      const int TQ = nr <= 8 ? 8 : 16;
      if (qb0 == 0) stage_wait();
      __syncthreads();
      // X rows of this thread's epilogue rows (row indices from shared memory: one global
      // latency), in flight during the table build and the main loop
      float xo[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = h + 2 * i;
        xo[i] = (r < nr && cok) ? __ldg(X + static_cast<int64_t>(Rv[qb0 + r]) * dg + c0 + c) : 0.f;
      }
      // Cb[p][g][l] = T_l(x_{p, qb0+g}) (masked on p == q and q >= n)
      for (int i = tid; i < n * TQ; i += kT) {
        const int p = i / TQ, g = i - p * TQ;
        const int q = qb0 + g;
        const bool ok = q < n && p != q;
        const float4 a = Us[p];
        const float4 b = ok ? Us[q] : a;
        const float x = a.x * b.x + a.y * b.y + a.z * b.z;
        const float m = ok ? 1.f : 0.f;
        float f[L], t[8];
        angular_row<L, MODE>(x, m, f);
#pragma unroll
        for (int l = 0; l < 8; ++l) t[l] = l < L ? f[l] : 0.f;
        float4* dst = reinterpret_cast<float4*>(Cb + (p * TQ + g) * 8);
        dst[0] = make_float4(t[0], t[1], t[2], t[3]);
        dst[1] = make_float4(t[4], t[5], t[6], t[7]);
      }
      __syncthreads();
      if (TQ == 8) bw2_main<L, 8>(Cb, Sb, n, Cb);
      else bw2_main<L, 16>(Cb, Sb, n, Cb);
      __syncthreads();
      // epilogue: thread (c, h) takes rows h, h + 2, ... of the batch
      float2 wr[KP][L];
#pragma unroll
      for (int k = 0; k < KP; ++k)
#pragma unroll
        for (int l = 0; l < L; ++l)
          wr[k][l] = make_float2(Wsm[(2 * k * L + l) * kCB + c], Wsm[((2 * k + 1) * L + l) * kCB + c]);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = h + 2 * i;
        if (r >= nr) break;
        const int q = qb0 + r;
        float qv[L];
#pragma unroll
        for (int l = 0; l < L; ++l) qv[l] = Cb[(r * L + l) * kCB + c];
        if constexpr (MODE == 2) {
          // radial rows [l][8 k] (k pairs packed): X_bar = sum_kl R W Qbar, dd = X sum_kl R' W Qbar,
          // W_bar[k, l] += R X Qbar_l
          const float* rr = Rb + q * RBS;
          const float* dr = DRb + q * RBS;
          const float x = xo[i];
          float2 xb2 = make_float2(0.f, 0.f), ds2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int l = 0; l < L; ++l) {
            const float rbar = qv[l] * x;
#pragma unroll
            for (int k = 0; k < KP; ++k) {
              const float2 r2 = *reinterpret_cast<const float2*>(rr + l * 8 + 2 * k);
              const float2 d2 = *reinterpret_cast<const float2*>(dr + l * 8 + 2 * k);
              const float2 wq = ffma2(qv[l], wr[k][l], make_float2(0.f, 0.f));
              xb2 = ffma2(r2, wq, xb2);
              ds2 = ffma2(d2, wq, ds2);
              wb[k][l] = ffma2(rbar, r2, wb[k][l]);
            }
          }
          if (cok) Xbar[static_cast<int64_t>(Rv[q]) * dg + c0 + c] = xb2.x + xb2.y;
          float dd = (ds2.x + ds2.y) * x;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
          if ((tid & 31) == 0) DD[r * 2 + ((tid >> 5) & 1)] = dd;
          continue;
        }
        const float d = Us[q].w;
        float rb[K];
        float2 v2[KP], rb2[KP];
#pragma unroll
        for (int k = 0; k < K; ++k) rb[k] = Rb[q * K + k];
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          rb2[k] = make_float2(rb[2 * k], rb[2 * k + 1]);
          v2[k] = make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < KP; ++k)
#pragma unroll
          for (int l = 0; l < L; ++l) v2[k] = ffma2(qv[l], wr[k][l], v2[k]);
        float xb = 0.f, ds = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const float vk = (k & 1) ? v2[k >> 1].y : v2[k >> 1].x;
          xb = fmaf(rb[k], vk, xb);
          const float drb = MODE == 0 ? -2.f * rp.gamma * (d - rp.step * k) * rb[k] : DRb[q * K + k];
          ds = fmaf(drb, vk, ds);
        }
        if (cok) Xbar[static_cast<int64_t>(Rv[q]) * dg + c0 + c] = xb;
        const float x = xo[i];
#pragma unroll
        for (int l = 0; l < L; ++l) {
          const float rbar = qv[l] * x;
#pragma unroll
          for (int k = 0; k < KP; ++k) wb[k][l] = ffma2(rbar, rb2[k], wb[k][l]);
        }
        float dd = ds * x;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
        if ((tid & 31) == 0) DD[r * 2 + ((tid >> 5) & 1)] = dd;
      }
      __syncthreads();
      if (tid < nr) {
        const float dd = DD[tid * 2] + DD[tid * 2 + 1];
        if (gridDim.y == 1) reinterpret_cast<float*>(edge_grad + off + qb0 + tid)[3] += dd;  // final value
        else dd_part[blockIdx.y * num_edges + off + qb0 + tid] = dd;
      }
    }
  }
  // combine the two row halves (fixed order), one partial per CTA:
  // layout [gridDim.y][gridDim.x][K*L*64]
  __syncthreads();
  if (h == 1) {
#pragma unroll
    for (int k = 0; k < KP; ++k)
#pragma unroll
      for (int l = 0; l < L; ++l) {
        Cb[(2 * k * L + l) * kCB + c] = wb[k][l].x;
        Cb[((2 * k + 1) * L + l) * kCB + c] = wb[k][l].y;
      }
  }
  __syncthreads();
  if (h == 0) {
    float* dst = wbar_part + (static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * (K * L * kCB);
#pragma unroll
    for (int k = 0; k < KP; ++k)
#pragma unroll
      for (int l = 0; l < L; ++l) {
        dst[(2 * k * L + l) * kCB + c] = wb[k][l].x + Cb[(2 * k * L + l) * kCB + c];
        dst[((2 * k + 1) * L + l) * kCB + c] = wb[k][l].y + Cb[((2 * k + 1) * L + l) * kCB + c];
      }
  }
}

// W_bar[k,l,c] = sum over x-CTAs of the partials of channel block c / 64; 32 outputs per
// block, kRW warps split the partials (eight loads in flight per thread), fixed-order combine
constexpr int kRW = 32;
__global__ void __launch_bounds__(kRW * 32) reduce_wbar_kernel(const float* __restrict__ part, int gx, int K, int L,
                                                               int dg, float* __restrict__ out) {
  __shared__ float red[kRW][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int total = K * L * dg;
  const int i = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (i < total) {
    const int kl = i / dg, c = i - kl * dg;
    const int cb = c / kCB, cc = c - cb * kCB;
    const int64_t st = K * L * kCB;
    const float* src = part + static_cast<int64_t>(cb) * gx * st + kl * kCB + cc;
    int x = w;
    for (; x + 7 * kRW < gx; x += 8 * kRW) {
      float a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = src[static_cast<int64_t>(x + u * kRW) * st];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += a[u];
    }
    for (; x < gx; x += kRW) s += src[static_cast<int64_t>(x) * st];
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && i < total) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < kRW; ++k) t += red[k][lane];
    out[i] = t;
  }
}

// edge_grad[e].w += sum over channel blocks of dd partials (only centres handled here, n <= 64)
__global__ void add_dd_kernel(const int64_t* __restrict__ edge_ptr, int64_t nv, const float* __restrict__ dd_part,
                              int ncb, int64_t ne, float4* __restrict__ edge_grad) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = edge_ptr[v], e1 = edge_ptr[v + 1];
    if (e1 - e0 < 2 || e1 - e0 > kN) continue;
    for (int64_t e = e0; e < e1; ++e) {
      float s = 0.f;
      for (int b = 0; b < ncb; ++b) s += dd_part[b * ne + e];
      reinterpret_cast<float*>(edge_grad + e)[3] += s;  // .w only (see bw1)
    }
  }
}

}  // namespace fast

// ---------------------------------------------------------------------------
// host side (called from triplet.cu's ABI functions)
// ---------------------------------------------------------------------------
bool fast_supported(int K, int L, int dg) { return K == 6 && L == 7 && dg >= 32; }

// mode 0: the reference's Gaussian rbf x T_l basis; mode 1: GemNet-T's CBF (rtab / dtab = the
// per-call radial table of triplet_sh.cu and its d-derivative, 8 floats per edge)
int fast_fwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, const float* X,
             const float* W, int K, int L, int dg, RbfParams rp, float* S, cudaStream_t st, int mode,
             const float* rtab) {
  // 4 CTAs per SM (128 registers): 5 or 6 (96 / 80 registers, spilling) measured 12% / 36% slower
  auto kern = mode == 2 ? fast::fwd_kernel<6, 7, 4, 2> : (mode == 1 ? fast::fwd_kernel<6, 7, 4, 1> : fast::fwd_kernel<6, 7>);
  // one centre per CTA: no tail imbalance from static round-robin over unequal degrees
  const int grid = static_cast<int>(std::min<int64_t>(nv, 1 << 30));
  kern<<<grid, fast::kT, 0, st>>>(edge_ptr, rev, geo, nv, X, W, dg, rp, S, rtab);
  return check_launch("triplet_fwd_fast");
}

int64_t fast_bwd_workspace_bytes(int64_t nv, int64_t ne, int K, int L, int dg) {
  const int64_t ncb = (dg + fast::kCB - 1) / fast::kCB;
  const int64_t gx = std::min<int64_t>(std::max<int64_t>(nv, 1), kNumSMs * 3);
  return (ncb * gx * K * L * fast::kCB + ncb * std::max<int64_t>(ne, 1)) * 4;
}

template <typename F>
static void fast_set_smem(F kern, size_t smem, bool& configured) {
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured = true;
  }
}

// phases: 1 = bw1 (the angle adjoint: edge_grad.xyz), 2 = bw2 + reductions (X_bar, W_bar,
// edge_grad.w), 3 = both.  The two touch disjoint outputs, so they may run on two streams.
int fast_bwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, int64_t ne,
             const float* X, const float* W, int K, int L, int dg, RbfParams rp, const float* Sbar, float* Xbar,
             float* Wbar, float4* edge_grad, void* ws, cudaStream_t st, int phases, int mode, const float* rtab,
             const float* dtab) {
  const int ncb = (dg + fast::kCB - 1) / fast::kCB;
  if (phases & 1) {
    const int grid = static_cast<int>(std::min<int64_t>(nv, 1 << 30));
    const int rbs = mode == 2 ? fast::rb_stride<6, 7, 2>() : 6;
    const size_t smem1 = (4 * fast::kN + ((fast::kN * rbs + 3) & ~3) + fast::kQC * 7 * fast::kSbStride +
                          fast::kN * fast::kSbStride + fast::kN * (fast::kN + 1)) *
                         sizeof(float);
    static bool c10 = false, c11 = false, c12 = false;  // 3 CTAs per SM: 168 registers, no spills (4: 128, spilling, 1% slower)
    if (mode == 2) {
      auto kern = fast::bw1_kernel<6, 7, 3, 2>;
      fast_set_smem(kern, smem1, c12);
      kern<<<grid, fast::kT, smem1, st>>>(edge_ptr, rev, geo, nv, X, W, dg, rp, Sbar, edge_grad, rtab);
    } else if (mode == 1) {
      auto kern = fast::bw1_kernel<6, 7, 3, 1>;
      fast_set_smem(kern, smem1, c11);
      kern<<<grid, fast::kT, smem1, st>>>(edge_ptr, rev, geo, nv, X, W, dg, rp, Sbar, edge_grad, rtab);
    } else {
      auto kern = fast::bw1_kernel<6, 7, 3>;
      fast_set_smem(kern, smem1, c10);
      kern<<<grid, fast::kT, smem1, st>>>(edge_ptr, rev, geo, nv, X, W, dg, rp, Sbar, edge_grad, nullptr);
    }
    if (check_launch("triplet_bw1_fast")) return 1;
  }
  if (!(phases & 2)) return 0;
  const int gx = static_cast<int>(std::min<int64_t>(nv, static_cast<int64_t>(kNumSMs) * 3));
  float* wpart = reinterpret_cast<float*>(ws);
  float* ddpart = wpart + static_cast<int64_t>(ncb) * gx * K * L * fast::kCB;
  const int rbs2 = mode == 2 ? fast::rb_stride<6, 7, 2>() : 6;
  const size_t smem = (4 * fast::kN + ((fast::kN * rbs2 + 3) & ~3) + fast::kN * 128 + fast::kN * fast::kCB +
                       6 * 7 * fast::kCB + 32 + fast::kN * rbs2 + fast::kN) * sizeof(float);
  static bool c20 = false, c21 = false, c22 = false;
  if (mode == 2) {  // 2 CTAs per SM (the (k, l) radial rows and their derivatives in shared memory)
    auto k2 = fast::bw2_kernel<6, 7, 2, 2>;
    fast_set_smem(k2, smem, c22);
    k2<<<dim3(gx, ncb), fast::kT, smem, st>>>(edge_ptr, rev, geo, nv, X, W, dg, rp, Sbar, Xbar, wpart, ddpart, ne,
                                              edge_grad, rtab, dtab);
  } else if (mode == 1) {
    auto k2 = fast::bw2_kernel<6, 7, 3, 1>;
    fast_set_smem(k2, smem, c21);
    k2<<<dim3(gx, ncb), fast::kT, smem, st>>>(edge_ptr, rev, geo, nv, X, W, dg, rp, Sbar, Xbar, wpart, ddpart, ne,
                                              edge_grad, rtab, dtab);
  } else {
    auto k2 = fast::bw2_kernel<6, 7>;
    fast_set_smem(k2, smem, c20);
    k2<<<dim3(gx, ncb), fast::kT, smem, st>>>(edge_ptr, rev, geo, nv, X, W, dg, rp, Sbar, Xbar, wpart, ddpart, ne,
                                              edge_grad, nullptr, nullptr);
  }
  if (check_launch("triplet_bw2_fast")) return 1;
  fast::reduce_wbar_kernel<<<static_cast<int>((static_cast<int64_t>(K) * L * dg + 31) / 32), fast::kRW * 32, 0, st>>>(
      wpart, gx, K, L, dg, Wbar);
  if (check_launch("triplet_bw2_reduce")) return 1;
  if (ncb == 1) return 0;  // bw2 added dE/dd directly
  fast::add_dd_kernel<<<grid_for(nv, 128), 128, 0, st>>>(edge_ptr, nv, ddpart, ncb, ne, edge_grad);
  return check_launch("triplet_bw_dd");
}

}  // namespace egn
