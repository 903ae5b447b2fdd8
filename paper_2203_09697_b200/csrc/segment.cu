// Edge/node aggregation, basis, force head, geometry adjoints and the SGD
// update.  All reductions are gather-form over sorted CSR rows (no global
// atomics), so results are deterministic and match the reference's
// ascending-edge accumulation order (receiver_plan, engine.py:78-90).
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace egn {

// ---------------------------------------------------------------- basis
__global__ void rbf_kernel(const float4* __restrict__ geo, int64_t ne, int K, RbfParams rp,
                           float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ne * K;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = i / K;
    int k = static_cast<int>(i - e * K);
    float dd = geo[e].w - rp.step * k;
    out[i] = __expf(-rp.gamma * dd * dd);
  }
}

// SBF rows for every triplet (debug / parity): (t, k*L+l) = rbf_k(d_q) T_l(x_pq).
__global__ void sbf_kernel(const float4* __restrict__ geo, const int64_t* __restrict__ edge_ptr,
                           const int64_t* __restrict__ tri_ptr, int64_t nv, int K, int L,
                           RbfParams rp, float* __restrict__ out) {
  for (int64_t j = blockIdx.x; j < nv; j += gridDim.x) {
    int64_t off = edge_ptr[j];
    int64_t n = edge_ptr[j + 1] - off;
    if (n < 2) continue;
    int64_t t0 = tri_ptr[j];
    for (int64_t k = threadIdx.x; k < n * (n - 1); k += blockDim.x) {
      int64_t p = k / (n - 1);
      int64_t r = k - p * (n - 1);
      int64_t q = r < p ? r : r + 1;
      float4 a = geo[off + p], b = geo[off + q];
      float x = a.x * b.x + a.y * b.y + a.z * b.z;
      float* row = out + (t0 + k) * K * L;
      for (int kk = 0; kk < K; ++kk) {
        float dd = b.w - rp.step * kk;
        float rb = __expf(-rp.gamma * dd * dd);
        float tc = 1.f, tp = x;
        for (int l = 0; l < L; ++l) {
          row[kk * L + l] = rb * tc;
          float tn = 2.f * x * tc - tp;
          tp = tc;
          tc = tn;
        }
      }
    }
  }
}

// ---------------------------------------------------------------- aggregation
// One warp per node; lanes over channels; in-edges of v are rev(out-edges of v)
// in ascending edge order.
__global__ void aggregate_in_edges_kernel(const int64_t* __restrict__ edge_ptr,
                                          const int32_t* __restrict__ rev, int64_t nv,
                                          const float* __restrict__ x, int64_t ldx, int d,
                                          float* __restrict__ out) {
  int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < nv; v += nwarps) {
    int64_t e0 = edge_ptr[v], e1 = edge_ptr[v + 1];
    for (int c0 = 0; c0 < d; c0 += 128) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int64_t e = e0; e < e1; ++e) {
        const float* row = x + static_cast<int64_t>(rev[e]) * ldx;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int c = c0 + u * 32 + lane;
          if (c < d) acc[u] += row[c];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int c = c0 + u * 32 + lane;
        if (c < d) out[v * d + c] = acc[u];
      }
    }
  }
}

// 16-byte path (d % 4 == 0, aligned rows): lane = 4 consecutive columns of a 128-column chunk,
// the segment's reverse-edge indices fetched 32 at a time, 4 rows in flight per lane.
__global__ void aggregate_in_edges_v4_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ rev,
                                             int64_t nv, const float* __restrict__ x, int64_t ldx, int d,
                                             float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < nv; v += nwarps) {
    const int64_t e0 = edge_ptr[v], e1 = edge_ptr[v + 1];
    for (int c0 = 0; c0 < d; c0 += 128) {
      const int c = c0 + lane * 4;
      const bool on = c < d;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int64_t b = e0; b < e1; b += 32) {
        const int nb = static_cast<int>(e1 - b < 32 ? e1 - b : 32);
        const int32_t my = lane < nb ? rev[b + lane] : 0;
        int j = 0;
        for (; j + 8 <= nb; j += 8) {  // 8 rows in flight per lane (a node has ~25 in-edges at C2)
          float4 t[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int32_t r = __shfl_sync(0xffffffffu, my, j + u);
            t[u] = on ? __ldg(reinterpret_cast<const float4*>(x + static_cast<int64_t>(r) * ldx + c))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {  // same order as the scalar path: edge after edge
            acc.x += t[u].x; acc.y += t[u].y; acc.z += t[u].z; acc.w += t[u].w;
          }
        }
        for (; j + 4 <= nb; j += 4) {
          float4 t[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int32_t r = __shfl_sync(0xffffffffu, my, j + u);
            t[u] = on ? __ldg(reinterpret_cast<const float4*>(x + static_cast<int64_t>(r) * ldx + c))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            acc.x += t[u].x; acc.y += t[u].y; acc.z += t[u].z; acc.w += t[u].w;
          }
        }
        for (; j < nb; ++j) {
          const int32_t r = __shfl_sync(0xffffffffu, my, j);
          if (on) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(x + static_cast<int64_t>(r) * ldx + c));
            acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
          }
        }
      }
      if (on) *reinterpret_cast<float4*>(out + v * d + c) = acc;
    }
  }
}

__global__ void gather_rows_kernel(const int32_t* __restrict__ idx, int64_t rows,
                                   const float* __restrict__ x, int64_t ldx, int d,
                                   float* __restrict__ out, int64_t ldo, int accumulate) {
  int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const float* src = x + static_cast<int64_t>(idx[r]) * ldx;
    float* dst = out + r * ldo;
    for (int c = lane; c < d; c += 32) dst[c] = accumulate ? dst[c] + src[c] : src[c];
  }
}

// out[dst[r]] (+)= x[src[r]]; destinations are distinct within one call (no races).
__global__ void scatter_rows_kernel(const int32_t* __restrict__ dst, const int32_t* __restrict__ src, int64_t rows,
                                    const float* __restrict__ x, int64_t ldx, int d, float* __restrict__ out,
                                    int64_t ldo, int accumulate) {
  int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const float* s = x + static_cast<int64_t>(src[r]) * ldx;
    float* o = out + static_cast<int64_t>(dst[r]) * ldo;
    for (int c = lane; c < d; c += 32) o[c] = accumulate ? o[c] + s[c] : s[c];
  }
}

// One CTA per (graph, 128-channel chunk); deterministic tree over nodes.
__global__ void graph_sum_kernel(const int64_t* __restrict__ graph_ptr, int64_t ng,
                                 const float* __restrict__ x, int d, float* __restrict__ out) {
  __shared__ float red[8][32];
  int chunks = (d + 31) / 32;
  for (int64_t item = blockIdx.x; item < ng * chunks; item += gridDim.x) {
    int64_t g = item / chunks;
    int c = static_cast<int>(item - g * chunks) * 32 + (threadIdx.x & 31);
    int row = threadIdx.x >> 5;  // 8 row lanes
    float s = 0.f;
    if (c < d)
      for (int64_t v = graph_ptr[g] + row; v < graph_ptr[g + 1]; v += 8) s += x[v * d + c];
    red[row][threadIdx.x & 31] = s;
    __syncthreads();
    if (row == 0 && c < d) {
      float t = 0.f;
#pragma unroll
      for (int r = 0; r < 8; ++r) t += red[r][threadIdx.x & 31];
      out[g * d + c] = t;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- force head
// scale[e] = m_e . w  (warp per edge)
__global__ void edge_dot_kernel(const float* __restrict__ m, int64_t ne, int d,
                                const float* __restrict__ w, float* __restrict__ scale) {
  int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t e = warp; e < ne; e += nwarps) {
    float s = 0.f;
    for (int c = lane; c < d; c += 32) s = fmaf(m[e * d + c], w[c], s);
    s = warp_sum(s);
    if (lane == 0) scale[e] = s;
  }
}

// forces[v] = sum over in-edges e of v of scale[e] u_e: warp per node, lanes over the in-edges
// (32 at a time), fixed butterfly reduction
__global__ void force_gather_warp_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ rev,
                                         const float4* __restrict__ geo, int64_t nv, const float* __restrict__ scale,
                                         float* __restrict__ forces) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < nv; v += nwarps) {
    float fx = 0.f, fy = 0.f, fz = 0.f;
    for (int64_t e = edge_ptr[v] + lane; e < edge_ptr[v + 1]; e += 32) {
      const int64_t ie = rev[e];
      const float sc = scale[ie];
      const float4 g = geo[ie];
      fx = fmaf(sc, g.x, fx);
      fy = fmaf(sc, g.y, fy);
      fz = fmaf(sc, g.z, fz);
    }
    fx = warp_sum(fx);
    fy = warp_sum(fy);
    fz = warp_sum(fz);
    if (lane == 0) {
      forces[3 * v + 0] = fx;
      forces[3 * v + 1] = fy;
      forces[3 * v + 2] = fz;
    }
  }
}

// Adjoint of the force head, lane group per edge (LPE = d / 4 lanes, float4 columns), two
// edges in flight: m_bar += sbar w, edge_grad += unit-vector adjoint, w_bar partial per CTA
// (fixed-order sum over the CTA's lane groups).  sbar = f_bar[recv] . u.
template <int LPE, int U = 4>
__global__ void __launch_bounds__(256) force_bwd_group_kernel(const int32_t* __restrict__ recv,
                                                              const float4* __restrict__ geo, int64_t ne,
                                                              const float* __restrict__ m, int d,
                                                              const float* __restrict__ w,
                                                              const float* __restrict__ scale,
                                                              const float* __restrict__ fbar,
                                                              float* __restrict__ mbar, float* __restrict__ wpart,
                                                              float4* __restrict__ edge_grad) {
  constexpr int EPW = 32 / LPE;
  __shared__ float red[8 * EPW][4 * LPE];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / LPE, gl = lane % LPE;
  const float4 wv = make_float4(__ldg(w + gl * 4), __ldg(w + gl * 4 + 1), __ldg(w + gl * 4 + 2), __ldg(w + gl * 4 + 3));
  float4 wacc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int64_t slots = static_cast<int64_t>(gridDim.x) * 8 * EPW;
  const int64_t my = (static_cast<int64_t>(blockIdx.x) * 8 + warp) * EPW + grp;
  for (int64_t e0 = my; e0 - grp < ne; e0 += U * slots) {  // U edges in flight per lane group
    float4 g[U], mv[U], mb[U];
    float sb[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * slots;
      ok[u] = e < ne;
      const int64_t ec = ok[u] ? e : 0;
      g[u] = geo[ec];
      const int64_t v = recv[ec];
      sb[u] = ok[u] ? (fbar[3 * v] * g[u].x + fbar[3 * v + 1] * g[u].y + fbar[3 * v + 2] * g[u].z) : 0.f;
      mv[u] = ok[u] ? __ldg(reinterpret_cast<const float4*>(m + ec * d) + gl) : make_float4(0.f, 0.f, 0.f, 0.f);
      mb[u] = ok[u] ? reinterpret_cast<const float4*>(mbar + ec * d)[gl] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!ok[u]) continue;
      const int64_t e = e0 + u * slots;
      const float s = sb[u];
      reinterpret_cast<float4*>(mbar + e * d)[gl] =
          make_float4(fmaf(s, wv.x, mb[u].x), fmaf(s, wv.y, mb[u].y), fmaf(s, wv.z, mb[u].z), fmaf(s, wv.w, mb[u].w));
      wacc.x = fmaf(s, mv[u].x, wacc.x);
      wacc.y = fmaf(s, mv[u].y, wacc.y);
      wacc.z = fmaf(s, mv[u].z, wacc.z);
      wacc.w = fmaf(s, mv[u].w, wacc.w);
      if (gl == 0) {
        const int64_t v = recv[e];
        const float bx = fbar[3 * v], by = fbar[3 * v + 1], bz = fbar[3 * v + 2];
        const float sc = scale[e];
        // units_bar = scale * fbar; d(unit)/d(v) adjoint: (ub - (ub.u) u) / d
        const float ux = sc * bx, uy = sc * by, uz = sc * bz;
        const float pr = ux * g[u].x + uy * g[u].y + uz * g[u].z;
        const float inv = 1.f / g[u].w;
        float4 eg = edge_grad[e];
        eg.x += (ux - pr * g[u].x) * inv;
        eg.y += (uy - pr * g[u].y) * inv;
        eg.z += (uz - pr * g[u].z) * inv;
        edge_grad[e] = eg;
      }
    }
  }
  *reinterpret_cast<float4*>(&red[warp * EPW + grp][gl * 4]) = wacc;
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += 256) {
    float t = 0.f;
#pragma unroll
    for (int r = 0; r < 8 * EPW; ++r) t += red[r][c];
    wpart[blockIdx.x * static_cast<int64_t>(d) + c] = t;
  }
}

// Adjoint of the force head, warp per edge, columns [c0, c0 + 512) of the edge
// features (launched once per 512-column chunk; the geometry term on chunk 0).
__global__ void force_bwd_kernel(const int32_t* __restrict__ recv, const float4* __restrict__ geo,
                                 int64_t ne, const float* __restrict__ m, int d, int c0,
                                 const float* __restrict__ w, const float* __restrict__ scale,
                                 const float* __restrict__ fbar, float* __restrict__ mbar,
                                 float* __restrict__ wpart, float4* __restrict__ edge_grad) {
  int lane = threadIdx.x & 31;
  int wib = threadIdx.x >> 5;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // per-warp partial of w_bar for this chunk, lanes over channels
  float wacc[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) wacc[u] = 0.f;
  for (int64_t e = warp; e < ne; e += nwarps) {
    int64_t v = recv[e];
    float4 g = geo[e];
    float bx = fbar[3 * v], by = fbar[3 * v + 1], bz = fbar[3 * v + 2];
    float sbar = bx * g.x + by * g.y + bz * g.z;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      int c = c0 + u * 32 + lane;
      if (c < d) {
        mbar[e * d + c] += sbar * w[c];
        wacc[u] = fmaf(sbar, m[e * d + c], wacc[u]);
      }
    }
    if (lane == 0 && c0 == 0) {
      float s = scale[e];
      // units_bar = s * fbar; d(unit)/d(v) adjoint: (ub - (ub.u) u) / d
      float ux = s * bx, uy = s * by, uz = s * bz;
      float pr = ux * g.x + uy * g.y + uz * g.z;
      float inv = 1.f / g.w;
      float4 eg = edge_grad[e];
      eg.x += (ux - pr * g.x) * inv;
      eg.y += (uy - pr * g.y) * inv;
      eg.z += (uz - pr * g.z) * inv;
      edge_grad[e] = eg;
    }
  }
  int64_t slot = blockIdx.x * (int64_t)(blockDim.x >> 5) + wib;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    int c = c0 + u * 32 + lane;
    if (c < d) wpart[slot * d + c] = wacc[u];
  }
}


// ---------------------------------------------------------------- K <= 8 linears of the basis
// out[e, n] = sum_k rbf[e, k] W[n, k] (+ b[n]): edge_init (engine.py:109-111) and the
// per-block rbf gate (engine.py:138).  HBM-bound: one float4 store per 4 outputs.
__global__ void rbf_linear_kernel(const float* __restrict__ rbf, int64_t ne, int K, const float* __restrict__ W,
                                  const float* __restrict__ b, int N, float* __restrict__ out, int64_t ldo) {
  extern __shared__ float ws[];  // [K][N] then bias [N]
  for (int i = threadIdx.x; i < K * N; i += blockDim.x) ws[(i % K) * N + i / K] = W[i];
  for (int i = threadIdx.x; i < N; i += blockDim.x) ws[K * N + i] = b ? b[i] : 0.f;
  __syncthreads();
  const int n4 = N >> 2;
  // the column chunk is fixed per thread when the stride is a multiple of N / 4 (the usual
  // case): no 64-bit division per output
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool fixed = stride % n4 == 0;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int c_fixed = static_cast<int>(t0 % n4) * 4;
  const int64_t de = stride / n4;
  for (int64_t idx = t0, e = t0 / n4; idx < ne * n4; idx += stride, e += de) {
    int c = c_fixed;
    if (!fixed) {
      e = idx / n4;
      c = static_cast<int>(idx - e * n4) * 4;
    }
    float4 o = *reinterpret_cast<const float4*>(ws + K * N + c);
    for (int k = 0; k < K; ++k) {
      const float r = __ldg(rbf + e * K + k);
      const float4 w4 = *reinterpret_cast<const float4*>(ws + k * N + c);
      o.x = fmaf(r, w4.x, o.x);
      o.y = fmaf(r, w4.y, o.y);
      o.z = fmaf(r, w4.z, o.z);
      o.w = fmaf(r, w4.w, o.w);
    }
    *reinterpret_cast<float4*>(out + e * ldo + c) = o;
  }
}

// Adjoint of rbf_linear for N <= 128, tiles of 32 edges staged in shared memory:
//   rbf_bar[e, k] += sum_n g[e, n] W[n, k]        (thread per (edge, k) of the tile)
//   part[block]    = (sum_e g[e, n] rbf[e, k])[n, k] and (sum_e g[e, n])[n]
//                    (thread-owned accumulators over the block's tiles, fixed order)
constexpr int kRlTile = 32;
__global__ void __launch_bounds__(256) rbf_linear_bwd_kernel(const float* __restrict__ rbf, int64_t ne, int K,
                                                             const float* __restrict__ W, int N,
                                                             const float* __restrict__ g,
                                                             const float* __restrict__ g2, int64_t ldg,
                                                             float* __restrict__ rbf_bar, float* __restrict__ part) {
  __shared__ float ws[128 * 8];
  __shared__ float gs[kRlTile][129];
  __shared__ float rs[kRlTile][9];
  const int tid = threadIdx.x;
  for (int i = tid; i < N * K; i += 256) ws[i] = W[i];
  const int len = N * K + N;
  float acc[5];  // owned slots tid + 256 r of [N*K weights | N biases]
#pragma unroll
  for (int r = 0; r < 5; ++r) acc[r] = 0.f;
  const int64_t ntiles = (ne + kRlTile - 1) / kRlTile;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t e0 = t * kRlTile;
    const int te = ne - e0 < kRlTile ? static_cast<int>(ne - e0) : kRlTile;
    __syncthreads();
    for (int i = tid; i < kRlTile * N; i += 256) {
      const int e = i / N, n = i - (i / N) * N;
      gs[e][n] = e < te ? (g2 ? g[(e0 + e) * ldg + n] * g2[(e0 + e) * ldg + n] : g[(e0 + e) * ldg + n]) : 0.f;
    }
    for (int i = tid; i < kRlTile * K; i += 256) {
      const int e = i / K, k = i - (i / K) * K;
      rs[e][k] = e < te ? rbf[(e0 + e) * K + k] : 0.f;
    }
    __syncthreads();
    if (tid < kRlTile * K) {
      const int e = tid / K, k = tid - (tid / K) * K;
      if (e < te) {
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        int n = 0;
        for (; n + 4 <= N; n += 4) {
          s0 = fmaf(gs[e][n], ws[n * K + k], s0);
          s1 = fmaf(gs[e][n + 1], ws[(n + 1) * K + k], s1);
          s2 = fmaf(gs[e][n + 2], ws[(n + 2) * K + k], s2);
          s3 = fmaf(gs[e][n + 3], ws[(n + 3) * K + k], s3);
        }
        for (; n < N; ++n) s0 = fmaf(gs[e][n], ws[n * K + k], s0);
        rbf_bar[(e0 + e) * K + k] += (s0 + s1) + (s2 + s3);
      }
    }
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const int slot = tid + 256 * r;
      if (slot < N * K) {
        const int n = slot / K, k = slot - (slot / K) * K;
        float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
        for (int e = 0; e < kRlTile; e += 2) {
          a0 = fmaf(gs[e][n], rs[e][k], a0);
          a1 = fmaf(gs[e + 1][n], rs[e + 1][k], a1);
        }
        acc[r] += a0 + a1;
      } else if (slot < len) {
        const int n = slot - N * K;
        float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
        for (int e = 0; e < kRlTile; e += 2) {
          a0 += gs[e][n];
          a1 += gs[e + 1][n];
        }
        acc[r] += a0 + a1;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int slot = tid + 256 * r;
    if (slot < len) part[blockIdx.x * (int64_t)len + slot] = acc[r];
  }
}

// Lane group per edge: LPE = N / 4 lanes hold float4 slices of g's row (32 / LPE edges per
// warp instruction) and the matching W rows in registers.  rbf_bar[e, k] = sum_n g[e, n] W[n, k]
// is an 8-value transpose reduction inside the lane group; W_bar[n, k] += g[e, n] rbf[e, k] and
// b_bar[n] += g[e, n] accumulate in registers, then a fixed-order sum over the CTA's warps (and
// the lane groups) gives one partial row per CTA (reduced by reduce_parts_kernel).
template <int LPE, int KT, int U = 2>
__global__ void __launch_bounds__(256) rbf_linear_bwd_group_kernel(const float* __restrict__ rbf, int64_t ne,
                                                                   int K, const float* __restrict__ W, int N,
                                                                   const float* __restrict__ g,
                                                                   const float* __restrict__ g2, int64_t ldg,
                                                                   float* __restrict__ rbf_bar,
                                                                   float* __restrict__ part) {
  constexpr int EPW = 32 / LPE;  // edges per warp instruction
  static_assert(LPE >= 8 && LPE <= 32, "lane group of 8..32");
  __shared__ float red[8 * EPW][36 * LPE];  // per slot: N K weights + N biases, N = 4 LPE, K <= 8
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / LPE, gl = lane % LPE;  // lane group (edge slot) and lane inside it
  const int len = N * K + N;
  const int kk_n = KT == 8 ? K : KT;
  float wr[4][8], wacc[4][8], bacc[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    bacc[i] = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      wr[i][k] = k < kk_n ? W[(gl * 4 + i) * kk_n + k] : 0.f;
      wacc[i][k] = 0.f;
    }
  }
  // bits of the lane-group index that pick the reduced column (levels LPE/2, LPE/4, LPE/8)
  const int b4 = (gl / (LPE / 2)) & 1, b3 = (gl / (LPE / 4)) & 1, b2 = (gl / (LPE / 8)) & 1;
  const int kk = b4 * 4 + b3 * 2 + b2;
  const bool writer = (gl % (LPE / 8)) == 0 && kk < kk_n;
  const int64_t slots = static_cast<int64_t>(gridDim.x) * 8 * EPW;  // edge slots in flight
  const int64_t my = (static_cast<int64_t>(blockIdx.x) * 8 + warp) * EPW + grp;
  for (int64_t e0 = my; e0 - grp < ne; e0 += U * slots) {
    float gv[U][4], r[U][8], old[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * slots;
      ok[u] = e < ne;
      const int64_t ec = ok[u] ? e : 0;
      float4 v = ok[u] ? __ldg(reinterpret_cast<const float4*>(g + ec * ldg + gl * 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (g2 != nullptr && ok[u]) {  // g = g * g2 (fused elementwise product)
        const float4 v2 = __ldg(reinterpret_cast<const float4*>(g2 + ec * ldg + gl * 4));
        v.x *= v2.x; v.y *= v2.y; v.z *= v2.z; v.w *= v2.w;
      }
      gv[u][0] = v.x; gv[u][1] = v.y; gv[u][2] = v.z; gv[u][3] = v.w;
#pragma unroll
      for (int k = 0; k < 8; ++k) r[u][k] = (k < kk_n && ok[u]) ? __ldg(rbf + ec * kk_n + k) : 0.f;
      old[u] = (writer && ok[u]) ? rbf_bar[ec * kk_n + kk] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float sv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float t = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) t = fmaf(gv[u][i], wr[i][k], t);
        sv[k] = k < kk_n ? t : 0.f;
      }
      float w4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float mine = b4 ? sv[4 + j] : sv[j];
        const float other = b4 ? sv[j] : sv[4 + j];
        w4[j] = mine + __shfl_xor_sync(0xffffffffu, other, LPE / 2);
      }
      float w2[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float mine = b3 ? w4[2 + j] : w4[j];
        const float other = b3 ? w4[j] : w4[2 + j];
        w2[j] = mine + __shfl_xor_sync(0xffffffffu, other, LPE / 4);
      }
      float x = (b2 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? w2[0] : w2[1], LPE / 8);
#pragma unroll
      for (int o = LPE / 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (!ok[u]) continue;
      if (writer) rbf_bar[(e0 + u * slots) * kk_n + kk] = old[u] + x;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        bacc[i] += gv[u][i];
#pragma unroll
        for (int k = 0; k < 8; ++k) wacc[i][k] = fmaf(gv[u][i], r[u][k], wacc[i][k]);
      }
    }
  }
  // fixed-order reduction over the CTA's (warp, lane group) slots
  float* mine = red[warp * EPW + grp];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int n = gl * 4 + i;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < kk_n) mine[n * kk_n + k] = wacc[i][k];
    mine[N * kk_n + n] = bacc[i];
  }
  __syncthreads();
  for (int slot = threadIdx.x; slot < len; slot += 256) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8 * EPW; ++w) t += red[w][slot];
    part[blockIdx.x * static_cast<int64_t>(len) + slot] = t;
  }
}

// out1[i] = sum_p part[p][i] for i < split, out2[i - split] for i >= split (out2 may be
// null): 8 warps split the parts, fixed-order combine (32 outputs per block).
__global__ void reduce_parts_kernel(const float* __restrict__ part, int nparts, int len, int split,
                                    float* __restrict__ out1, float* __restrict__ out2) {
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if (i < len) {
    int p = w;
    for (; p + 24 < nparts; p += 32) {  // four independent loads in flight per thread
      s0 += part[static_cast<int64_t>(p) * len + i];
      s1 += part[static_cast<int64_t>(p + 8) * len + i];
      s2 += part[static_cast<int64_t>(p + 16) * len + i];
      s3 += part[static_cast<int64_t>(p + 24) * len + i];
    }
    for (; p < nparts; p += 8) s0 += part[static_cast<int64_t>(p) * len + i];
  }
  red[w][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (w == 0 && i < len) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][lane];
    if (i < split) out1[i] = t;
    else if (out2) out2[i - split] = t;
  }
}

// ---------------------------------------------------------------- geometry adjoints
__global__ void rbf_bwd_kernel(const float4* __restrict__ geo, const float* __restrict__ rbar,
                               int64_t ne, int K, RbfParams rp, float4* __restrict__ edge_grad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    float d = geo[e].w;
    float s = 0.f;
    for (int k = 0; k < K; ++k) {
      float dd = d - rp.step * k;
      float r = __expf(-rp.gamma * dd * dd);
      s = fmaf(rbar[e * K + k], -2.f * rp.gamma * dd * r, s);
    }
    edge_grad[e].w += s;
  }
}

// pos_bar[a] = sum_{e in out(a)} (g_{rev e} - g_e), g_e = grad_v(e) + dd_e * u_e: warp per
// atom, lanes over the out-edges, fp64 partials, fixed butterfly reduction
__global__ void positions_bwd_warp_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ rev,
                                          const float4* __restrict__ geo, int64_t nv, const float4* __restrict__ eg,
                                          double* __restrict__ pos_bar) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t a = warp; a < nv; a += nwarps) {
    double sx = 0.0, sy = 0.0, sz = 0.0;
    for (int64_t e = edge_ptr[a] + lane; e < edge_ptr[a + 1]; e += 32) {
      const int64_t ie = rev[e];
      const float4 gi = eg[ie], ui = geo[ie];
      const float4 go = eg[e], uo = geo[e];
      sx += (double)fmaf(gi.w, ui.x, gi.x) - (double)fmaf(go.w, uo.x, go.x);
      sy += (double)fmaf(gi.w, ui.y, gi.y) - (double)fmaf(go.w, uo.y, go.y);
      sz += (double)fmaf(gi.w, ui.z, gi.z) - (double)fmaf(go.w, uo.z, go.z);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sx += __shfl_xor_sync(0xffffffffu, sx, o);
      sy += __shfl_xor_sync(0xffffffffu, sy, o);
      sz += __shfl_xor_sync(0xffffffffu, sz, o);
    }
    if (lane == 0) {
      pos_bar[3 * a + 0] = sx;
      pos_bar[3 * a + 1] = sy;
      pos_bar[3 * a + 2] = sz;
    }
  }
}

// Column sums of a row-major [rows, d] matrix: stage 1 writes one partial row per
// 256-row chunk (threads over columns, coalesced), stage 2 sums the partials in
// chunk order (deterministic).
constexpr int kColChunk = 256;

__global__ void column_sum_partial_kernel(const float* __restrict__ x, int64_t rows, int d, int64_t ld,
                                          float* __restrict__ part) {
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kColChunk;
  const int64_t r1 = r0 + kColChunk < rows ? r0 + kColChunk : rows;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int64_t r = r0;
    for (; r + 3 < r1; r += 4) {
      s0 += x[r * ld + c];
      s1 += x[(r + 1) * ld + c];
      s2 += x[(r + 2) * ld + c];
      s3 += x[(r + 3) * ld + c];
    }
    for (; r < r1; ++r) s0 += x[r * ld + c];
    part[static_cast<int64_t>(blockIdx.x) * d + c] = (s0 + s1) + (s2 + s3);
  }
}

// AdamW (decoupled weight decay; torch.optim.AdamW's update order):
//   w *= 1 - lr wd;  m += (1 - b1)(g - m);  v = b2 v + (1 - b2) g^2;
//   w -= (lr / bc1) m / (sqrt(v) / sqrt(bc2) + eps),  bc = 1 - beta^t
__global__ void adamw_kernel(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m,
                             float* __restrict__ v, int64_t n, float lr, float b1, float b2, float eps, float wd,
                             float step_size, float bc2_sqrt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    float p = w[i] * (1.f - lr * wd);
    const float mi = m[i] + (1.f - b1) * (gi - m[i]);
    const float vi = v[i] * b2 + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p -= step_size * (mi / (sqrtf(vi) / bc2_sqrt + eps));
    w[i] = p;
  }
}

__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g, int64_t n, float lr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] -= lr * g[i];
}

}  // namespace egn

using namespace egn;

extern "C" {

int egn_rbf(const float* geo, int64_t num_edges, int k_rbf, double cutoff, float* rbf,
            egn_stream_t stream) {
  EGN_REQUIRE(k_rbf >= 1, "k_rbf must be >= 1");
  if (num_edges == 0) return 0;
  rbf_kernel<<<grid_for(num_edges * k_rbf, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(geo), num_edges, k_rbf, rbf_params(k_rbf, cutoff), rbf);
  return check_launch("rbf");
}

int egn_sbf(const float* geo, const int64_t* edge_ptr, const int64_t* tri_ptr, int64_t num_nodes,
            int k_rbf, int l_sbf, double cutoff, float* sbf, egn_stream_t stream) {
  EGN_REQUIRE(k_rbf >= 1 && l_sbf >= 1, "k_rbf and l_sbf must be >= 1");
  if (num_nodes == 0) return 0;
  int grid = static_cast<int>(num_nodes < 65535 ? num_nodes : 65535);
  sbf_kernel<<<grid, 128, 0, as_stream(stream)>>>(reinterpret_cast<const float4*>(geo), edge_ptr,
                                                  tri_ptr, num_nodes, k_rbf, l_sbf,
                                                  rbf_params(k_rbf, cutoff), sbf);
  return check_launch("sbf");
}

int egn_aggregate_in_edges(const int64_t* edge_ptr, const int32_t* rev, int64_t num_nodes,
                           const float* x, int64_t ld_x, int d, float* out, egn_stream_t stream) {
  if (num_nodes == 0) return 0;
  if (d % 4 == 0 && ld_x % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    aggregate_in_edges_v4_kernel<<<grid_for(num_nodes * 32, 256), 256, 0, as_stream(stream)>>>(
        edge_ptr, rev, num_nodes, x, ld_x, d, out);
  } else {
    aggregate_in_edges_kernel<<<grid_for(num_nodes * 32, 256), 256, 0, as_stream(stream)>>>(
        edge_ptr, rev, num_nodes, x, ld_x, d, out);
  }
  return check_launch("aggregate_in_edges");
}

int egn_gather_rows(const int32_t* idx, int64_t rows, const float* x, int64_t ld_x, int d,
                    float* out, int64_t ld_out, int accumulate, egn_stream_t stream) {
  if (rows == 0) return 0;
  gather_rows_kernel<<<grid_for(rows * 32, 256), 256, 0, as_stream(stream)>>>(
      idx, rows, x, ld_x, d, out, ld_out, accumulate);
  return check_launch("gather_rows");
}

int egn_scatter_rows(const int32_t* dst, const int32_t* src, int64_t rows, const float* x, int64_t ld_x, int d,
                     float* out, int64_t ld_out, int accumulate, egn_stream_t stream) {
  if (rows == 0) return 0;
  scatter_rows_kernel<<<grid_for(rows * 32, 256), 256, 0, as_stream(stream)>>>(dst, src, rows, x, ld_x, d, out,
                                                                               ld_out, accumulate);
  return check_launch("scatter_rows");
}

int egn_graph_sum(const int64_t* graph_ptr, int64_t num_graphs, const float* x, int d,
                  float* out, egn_stream_t stream) {
  if (num_graphs == 0) return 0;
  int64_t items = num_graphs * ((d + 31) / 32);
  graph_sum_kernel<<<static_cast<int>(std::min<int64_t>(items, 148 * 16)), 256, 0,
                     as_stream(stream)>>>(graph_ptr, num_graphs, x, d, out);
  return check_launch("graph_sum");
}

int egn_force_head_fwd(const int64_t* edge_ptr, const int32_t* rev, const float* geo,
                       int64_t num_nodes, int64_t num_edges, const float* m, int d,
                       const float* w, float* scale, float* forces, egn_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  if (num_edges > 0 && m != nullptr) {
    edge_dot_kernel<<<grid_for(num_edges * 32, 256), 256, 0, st>>>(m, num_edges, d, w, scale);
    if (check_launch("force_head_dot")) return 1;
  }
  if (num_nodes == 0 || forces == nullptr) return 0;
  force_gather_warp_kernel<<<grid_for(num_nodes * 32, 256), 256, 0, st>>>(
      edge_ptr, rev, reinterpret_cast<const float4*>(geo), num_nodes, scale, forces);
  return check_launch("force_head_gather");
}

int64_t egn_force_head_bwd_workspace_bytes(int64_t num_edges, int d) {
  int grid = grid_for(num_edges * 32, 256, 148 * 2);
  return static_cast<int64_t>(grid) * 8 * d * 4;
}

int egn_force_head_bwd(const int32_t* recv, const float* geo, int64_t num_edges, const float* m,
                       int d, const float* w, const float* scale, const float* f_bar,
                       float* m_bar, float* w_bar, float* edge_grad, void* workspace,
                       egn_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  if (num_edges == 0) {
    cudaMemsetAsync(w_bar, 0, sizeof(float) * d, st);
    return check_launch("force_head_bwd_empty");
  }
  int grid = grid_for(num_edges * 32, 256, 148 * 2);
  float* part = reinterpret_cast<float*>(workspace);
  const int lpe = d / 4;
  if (d % 4 == 0 && (lpe == 8 || lpe == 16 || lpe == 32) && (reinterpret_cast<uintptr_t>(m) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(m_bar) & 15) == 0) {
    // lane group per edge; one partial row per CTA (the workspace holds grid * 8 rows)
    const auto* g4 = reinterpret_cast<const float4*>(geo);
    auto* eg4 = reinterpret_cast<float4*>(edge_grad);
    if (lpe == 32) force_bwd_group_kernel<32><<<grid, 256, 0, st>>>(recv, g4, num_edges, m, d, w, scale, f_bar, m_bar, part, eg4);
    else if (lpe == 16) force_bwd_group_kernel<16><<<grid, 256, 0, st>>>(recv, g4, num_edges, m, d, w, scale, f_bar, m_bar, part, eg4);
    else force_bwd_group_kernel<8><<<grid, 256, 0, st>>>(recv, g4, num_edges, m, d, w, scale, f_bar, m_bar, part, eg4);
    if (check_launch("force_head_bwd")) return 1;
    reduce_parts_kernel<<<(d + 31) / 32, 256, 0, st>>>(part, grid, d, d, w_bar, nullptr);
    return check_launch("force_head_bwd_reduce");
  }
  for (int c0 = 0; c0 < d; c0 += 512) {
    force_bwd_kernel<<<grid, 256, 0, st>>>(recv, reinterpret_cast<const float4*>(geo), num_edges, m, d, c0, w,
                                           scale, f_bar, m_bar, part, reinterpret_cast<float4*>(edge_grad));
    if (check_launch("force_head_bwd")) return 1;
  }
  reduce_parts_kernel<<<(d + 31) / 32, 256, 0, st>>>(part, grid * 8, d, d, w_bar, nullptr);
  return check_launch("force_head_bwd_reduce");
}

int egn_rbf_linear(const float* rbf, int64_t num_edges, int k, const float* w, const float* b, int n, float* out,
                   int64_t ldo, egn_stream_t stream) {
  EGN_REQUIRE(k >= 1 && k <= 8 && n >= 4 && n % 4 == 0 && ldo % 4 == 0, "rbf_linear needs K <= 8, N % 4 == 0");
  if (num_edges == 0) return 0;
  const size_t smem = sizeof(float) * (k * n + n);
  EGN_REQUIRE(smem <= 200 * 1024, "rbf_linear: N too large");
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(rbf_linear_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  // grid: a multiple of N / 4 threads in total (fixed column chunk per thread)
  const int n4 = n / 4;
  int64_t blocks = grid_for(num_edges * n4, 256, 148 * 8);
  while ((blocks * 256) % n4 != 0) ++blocks;
  rbf_linear_kernel<<<static_cast<int>(blocks), 256, smem, as_stream(stream)>>>(rbf, num_edges, k, w, b, n, out, ldo);
  return check_launch("rbf_linear");
}

static int rbf_linear_bwd_grid(int64_t num_edges) {
  const int64_t tiles = (num_edges + kRlTile - 1) / kRlTile;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(tiles, kNumSMs * 4)));
}

int64_t egn_rbf_linear_bwd_workspace_bytes(int64_t num_edges, int k, int n) {
  return static_cast<int64_t>(rbf_linear_bwd_grid(num_edges)) * (n * k + n) * 4;
}

int egn_rbf_linear_bwd(const float* rbf, int64_t num_edges, int k, const float* w, int n, const float* g,
                       const float* g2, int64_t ldg, float* rbf_bar, float* w_bar, float* b_bar, void* workspace,
                       egn_stream_t stream) {
  EGN_REQUIRE(k >= 1 && k <= 8 && n >= 1 && n <= 128, "rbf_linear_bwd needs K <= 8, N <= 128");
  cudaStream_t st = as_stream(stream);
  if (num_edges == 0) {
    cudaMemsetAsync(w_bar, 0, sizeof(float) * n * k, st);
    if (b_bar) cudaMemsetAsync(b_bar, 0, sizeof(float) * n, st);
    return check_launch("rbf_linear_bwd_empty");
  }
  int grid = rbf_linear_bwd_grid(num_edges);
  float* part = reinterpret_cast<float*>(workspace);
  const int lpe = n / 4;
  const bool group_path = n % 4 == 0 && (lpe == 8 || lpe == 16 || lpe == 32) && ldg % 4 == 0 &&
                          (reinterpret_cast<uintptr_t>(g) & 15) == 0 && (reinterpret_cast<uintptr_t>(g2) & 15) == 0;
  if (group_path) {
    // lane group per edge; grid sized to one wave (the workspace holds rbf_linear_bwd_grid rows)
    grid = std::min(grid, k == 6 ? kNumSMs * 2 : kNumSMs);  // 98 / 136 registers per thread
    // K = 6: four edges in flight per lane group (128 registers; two: 75 -> 65 us at C2)
#define EGN_RLB(L)                                                                                      \
    (k == 6 ? rbf_linear_bwd_group_kernel<L, 6, 4><<<grid, 256, 0, st>>>(rbf, num_edges, k, w, n, g, g2, ldg, rbf_bar, part) \
            : rbf_linear_bwd_group_kernel<L, 8><<<grid, 256, 0, st>>>(rbf, num_edges, k, w, n, g, g2, ldg, rbf_bar, part))
    if (lpe == 32) EGN_RLB(32);
    else if (lpe == 16) EGN_RLB(16);
    else EGN_RLB(8);
#undef EGN_RLB
  } else {
    rbf_linear_bwd_kernel<<<grid, 256, 0, st>>>(rbf, num_edges, k, w, n, g, g2, ldg, rbf_bar, part);
  }
  if (check_launch("rbf_linear_bwd")) return 1;
  // part rows are [n*k weights | n biases]
  const int len = n * k + n;
  reduce_parts_kernel<<<(len + 31) / 32, 256, 0, st>>>(part, grid, len, n * k, w_bar, b_bar);
  return check_launch("rbf_linear_bwd_reduce");
}

// Radial Bessel basis with the DimeNet polynomial envelope (the edge basis of
// DimeNet++ / GemNet): e_n(d) = sqrt(2/c) u(d/c) sin(n pi d/c), n = 1..K, u(x) = 1/x - 28 x^5 +
// 48 x^6 - 21 x^7 (p = 6) on (0, 1).  Evaluated in fp64 per edge, stored fp32.
__device__ __forceinline__ void bessel_env(double x, double& u, double& du) {
  if (x >= 1.0) {
    u = du = 0.0;
    return;
  }
  const double x2 = x * x, x4 = x2 * x2, x5 = x4 * x, x6 = x5 * x;
  u = 1.0 / x - 28.0 * x5 + 48.0 * x6 - 21.0 * x6 * x;
  du = -1.0 / x2 - 140.0 * x4 + 288.0 * x5 - 147.0 * x6;
}

__global__ void rbf_bessel_kernel(const float4* __restrict__ geo, int64_t ne, int K, double cutoff,
                                  float* __restrict__ out) {
  const double nrm = sqrt(2.0 / cutoff);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const double x = geo[e].w / cutoff;
    double u, du;
    bessel_env(x, u, du);
    for (int k = 0; k < K; ++k) out[e * K + k] = static_cast<float>(nrm * u * sinpi((k + 1) * x));
  }
}

__global__ void rbf_bessel_bwd_kernel(const float4* __restrict__ geo, const float* __restrict__ rbar, int64_t ne,
                                      int K, double cutoff, float4* __restrict__ edge_grad) {
  const double nrm = sqrt(2.0 / cutoff);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const double x = geo[e].w / cutoff;
    double u, du;
    bessel_env(x, u, du);
    double s = 0.0;
    for (int k = 0; k < K; ++k) {
      double sn, cs;
      sincospi((k + 1) * x, &sn, &cs);
      s += rbar[e * K + k] * nrm * (du * sn + u * (k + 1) * 3.14159265358979323846 * cs) / cutoff;
    }
    edge_grad[e].w += static_cast<float>(s);
  }
}

int egn_rbf_bessel(const float* geo, int64_t num_edges, int k_rbf, double cutoff, float* rbf, egn_stream_t stream) {
  EGN_REQUIRE(k_rbf >= 1 && cutoff > 0.0, "bessel rbf needs k_rbf >= 1 and a positive cutoff");
  if (num_edges == 0) return 0;
  rbf_bessel_kernel<<<grid_for(num_edges, 256), 256, 0, as_stream(stream)>>>(reinterpret_cast<const float4*>(geo),
                                                                             num_edges, k_rbf, cutoff, rbf);
  return check_launch("rbf_bessel");
}

int egn_rbf_bessel_bwd(const float* geo, const float* rbf_bar, int64_t num_edges, int k_rbf, double cutoff,
                       float* edge_grad, egn_stream_t stream) {
  if (num_edges == 0) return 0;
  rbf_bessel_bwd_kernel<<<grid_for(num_edges, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(geo), rbf_bar, num_edges, k_rbf, cutoff, reinterpret_cast<float4*>(edge_grad));
  return check_launch("rbf_bessel_bwd");
}

int egn_rbf_bwd(const float* geo, const float* rbf_bar, int64_t num_edges, int k_rbf,
                double cutoff, float* edge_grad, egn_stream_t stream) {
  if (num_edges == 0) return 0;
  rbf_bwd_kernel<<<grid_for(num_edges, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(geo), rbf_bar, num_edges, k_rbf, rbf_params(k_rbf, cutoff),
      reinterpret_cast<float4*>(edge_grad));
  return check_launch("rbf_bwd");
}

int egn_positions_bwd(const int64_t* edge_ptr, const int32_t* rev, const float* geo,
                      int64_t num_nodes, const float* edge_grad, double* pos_bar,
                      egn_stream_t stream) {
  if (num_nodes == 0) return 0;
  positions_bwd_warp_kernel<<<grid_for(num_nodes * 32, 256), 256, 0, as_stream(stream)>>>(
      edge_ptr, rev, reinterpret_cast<const float4*>(geo), num_nodes,
      reinterpret_cast<const float4*>(edge_grad), pos_bar);
  return check_launch("positions_bwd");
}

int64_t egn_column_sum_workspace_bytes(int64_t rows, int d) {
  return ((rows + kColChunk - 1) / kColChunk + 1) * static_cast<int64_t>(d) * 4;
}

int egn_column_sum(const float* x, int64_t rows, int d, int64_t ld, float* out, void* workspace,
                   egn_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  if (rows == 0) {
    cudaMemsetAsync(out, 0, sizeof(float) * d, st);
    return check_launch("column_sum_empty");
  }
  const int chunks = static_cast<int>((rows + kColChunk - 1) / kColChunk);
  float* part = reinterpret_cast<float*>(workspace);
  const int threads = d >= 256 ? 256 : ((d + 31) / 32) * 32;
  column_sum_partial_kernel<<<chunks, threads, 0, st>>>(x, rows, d, ld, part);
  if (check_launch("column_sum_partial")) return 1;
  reduce_parts_kernel<<<(d + 31) / 32, 256, 0, st>>>(part, chunks, d, d, out, nullptr);
  return check_launch("column_sum_reduce");
}

// Loss and its seeds in one CTA (tasks.py:166-176 per sample; fp64 like the reference):
// res = E - E*, d_energy = 2 w_e res / n, delta = F - F*, d_forces = 2 w_f delta / (n count),
// loss = (sum w_e res^2 + w_f sum_v |delta_v|^2 / count_v) / n.  Seeds are cast to fp32 (the
// precision the backward consumes); the loss sums run in a fixed order.
__global__ void __launch_bounds__(1024) loss_seeds_kernel(const float* __restrict__ energy,
                                                          const double* __restrict__ e_target, int64_t G,
                                                          const float* __restrict__ forces,
                                                          const double* __restrict__ f_target,
                                                          const double* __restrict__ count, int64_t V, double w_e,
                                                          double w_f, double n, double* __restrict__ loss,
                                                          float* __restrict__ d_energy,
                                                          float* __restrict__ d_forces) {
  __shared__ double red[2][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double le = 0.0, lf = 0.0;
  for (int64_t g = tid; g < G; g += blockDim.x) {
    const double r = static_cast<double>(energy[g]) - e_target[g];
    d_energy[g] = static_cast<float>(2.0 * w_e * r / n);
    le += w_e * r * r;
  }
  if (forces != nullptr) {
    for (int64_t v = tid; v < V; v += blockDim.x) {
      const double cnt = count[v];
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double d = static_cast<double>(forces[3 * v + c]) - f_target[3 * v + c];
        d_forces[3 * v + c] = static_cast<float>(2.0 * w_f * d / (n * cnt));
        s += d * d;
      }
      lf += s / cnt;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    le += __shfl_xor_sync(0xffffffffu, le, o);
    lf += __shfl_xor_sync(0xffffffffu, lf, o);
  }
  if (lane == 0) {
    red[0][warp] = le;
    red[1][warp] = lf;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    loss[0] = a / n + w_f * b / n;
  }
}

int egn_loss_seeds(const float* energy, const double* e_target, int64_t num_graphs, const float* forces,
                   const double* f_target, const double* atom_count, int64_t num_nodes, double w_energy,
                   double w_forces, double n, double* loss, float* d_energy, float* d_forces, egn_stream_t stream) {
  EGN_REQUIRE(n > 0.0, "loss normaliser must be positive");
  EGN_REQUIRE(forces == nullptr || (f_target != nullptr && atom_count != nullptr && d_forces != nullptr),
              "force terms need targets, atom counts and a seed buffer");
  loss_seeds_kernel<<<1, 1024, 0, as_stream(stream)>>>(energy, e_target, num_graphs, forces, f_target, atom_count,
                                                        num_nodes, w_energy, w_forces, n, loss, d_energy, d_forces);
  return check_launch("loss_seeds");
}

int egn_adamw(float* w, const float* g, float* m, float* v, int64_t n, float lr, float beta1, float beta2,
              float eps, float weight_decay, int64_t step, egn_stream_t stream) {
  EGN_REQUIRE(step >= 1, "adamw step count starts at 1");
  if (n == 0) return 0;
  const double bc1 = 1.0 - std::pow(static_cast<double>(beta1), static_cast<double>(step));
  const double bc2 = 1.0 - std::pow(static_cast<double>(beta2), static_cast<double>(step));
  adamw_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(w, g, m, v, n, lr, beta1, beta2, eps, weight_decay,
                                                                static_cast<float>(lr / bc1),
                                                                static_cast<float>(std::sqrt(bc2)));
  return check_launch("adamw");
}

int egn_sgd(float* w, const float* g, int64_t n, float lr, egn_stream_t stream) {
  if (n == 0) return 0;
  sgd_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(w, g, n, lr);
  return check_launch("sgd");
}

}  // extern "C"

// ---------------------------------------------------------------- batched weight-sized products
// C = op(A) op(B) for up to kMaxSmall independent small problems in one launch (the weight
// folds A W_down, W1b W_up, B W_sbf and their adjoints): one 32 x 32 output tile per CTA,
// fp32 FFMA, shared-memory K tiles.
namespace egn {
constexpr int kMaxSmall = 32;
struct SmallBatch {
  egn_small_gemm_t g[kMaxSmall];
  int tile0[kMaxSmall + 1];
  int count;
};

__global__ void __launch_bounds__(256) small_gemm_kernel(const __grid_constant__ SmallBatch b) {
  __shared__ float As[32][33];
  __shared__ float Bs[32][33];
  int pi = 0;
  while (pi + 1 < b.count && static_cast<int>(blockIdx.x) >= b.tile0[pi + 1]) ++pi;
  const egn_small_gemm_t& g = b.g[pi];
  const int t = blockIdx.x - b.tile0[pi];
  const int tn = (g.n + 31) / 32;
  const int m0 = (t / tn) * 32, n0 = (t % tn) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 row groups x 32 columns
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k0 = 0; k0 < g.k; k0 += 32) {
    for (int i = threadIdx.x; i < 32 * 32; i += 256) {
      const int r = i >> 5, c = i & 31;
      const int m = m0 + r, k = k0 + c;
      As[r][c] = (m < g.m && k < g.k) ? (g.trans_a ? g.a[static_cast<int64_t>(k) * g.lda + m]
                                                    : g.a[static_cast<int64_t>(m) * g.lda + k])
                                       : 0.f;
      const int kk = k0 + r, n = n0 + c;
      Bs[r][c] = (kk < g.k && n < g.n) ? (g.trans_b ? g.b[static_cast<int64_t>(n) * g.ldb + kk]
                                                     : g.b[static_cast<int64_t>(kk) * g.ldb + n])
                                        : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      const float bv = Bs[kk][tx];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = fmaf(As[ty + 8 * i][kk], bv, acc[i]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 8 * i, n = n0 + tx;
    if (m < g.m && n < g.n) {
      if (g.trans_c) g.c[static_cast<int64_t>(n) * g.ldc + m] = acc[i];
      else g.c[static_cast<int64_t>(m) * g.ldc + n] = acc[i];
    }
  }
}

// The same products on 64 x 64 output tiles with a 4 x 4 register tile per thread (16-deep K
// slabs staged k-major in shared memory, one 16-byte load of A and of B per 16 FMAs): for
// batches with large problems (the XL weight folds, 2048 x 2048 x 256), ~3x the 32 x 32 kernel.
__global__ void __launch_bounds__(256) small_gemm64_kernel(const __grid_constant__ SmallBatch b) {
  __shared__ __align__(16) float As[16][68];  // [k][m]
  __shared__ __align__(16) float Bs[16][68];  // [k][n]
  int pi = 0;
  while (pi + 1 < b.count && static_cast<int>(blockIdx.x) >= b.tile0[pi + 1]) ++pi;
  const egn_small_gemm_t& g = b.g[pi];
  const int t = blockIdx.x - b.tile0[pi];
  const int tn = (g.n + 63) / 64;
  const int m0 = (t / tn) * 64, n0 = (t % tn) * 64;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;  // rows m0 + 4 ty + i, cols n0 + 4 tx + j
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < g.k; k0 += 16) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + 256 * u;  // 1024 elements of each 64 x 16 slab
      // k-contiguous source ([m][k] A / [n][k] B): lanes along k; else lanes along m / n
      const int kk_a = g.trans_a ? (e >> 6) : (e & 15), mm = g.trans_a ? (e & 63) : (e >> 4);
      const int m = m0 + mm, k = k0 + kk_a;
      As[kk_a][mm] = (m < g.m && k < g.k) ? (g.trans_a ? g.a[static_cast<int64_t>(k) * g.lda + m]
                                                        : g.a[static_cast<int64_t>(m) * g.lda + k])
                                           : 0.f;
      const int kk_b = g.trans_b ? (e & 15) : (e >> 6), nn = g.trans_b ? (e >> 4) : (e & 63);
      const int n = n0 + nn, kb = k0 + kk_b;
      Bs[kk_b][nn] = (kb < g.k && n < g.n) ? (g.trans_b ? g.b[static_cast<int64_t>(n) * g.ldb + kb]
                                                        : g.b[static_cast<int64_t>(kb) * g.ldb + n])
                                           : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const float4 av = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 bv = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float a4[4] = {av.x, av.y, av.z, av.w}, b4[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a4[i], b4[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < g.m && n < g.n) {
        if (g.trans_c) g.c[static_cast<int64_t>(n) * g.ldc + m] = acc[i][j];
        else g.c[static_cast<int64_t>(m) * g.ldc + n] = acc[i][j];
      }
    }
}
}  // namespace egn

extern "C" int egn_small_gemm_batched(const egn_small_gemm_t* problems, int count, egn_stream_t stream) {
  using namespace egn;
  cudaStream_t st = as_stream(stream);
  for (int base = 0; base < count; base += kMaxSmall) {
    SmallBatch b;
    b.count = std::min(kMaxSmall, count - base);
    int64_t work = 0;
    for (int i = 0; i < b.count; ++i) {
      const egn_small_gemm_t& g = problems[base + i];
      EGN_REQUIRE(g.m >= 0 && g.n >= 0 && g.k >= 0, "small_gemm: negative size");
      work = std::max<int64_t>(work, static_cast<int64_t>(g.m) * g.n * g.k);
    }
    // 64 x 64 tiles once the products are large enough to fill the GPU with them
    const int T = work >= (int64_t(1) << 25) ? 64 : 32;
    b.tile0[0] = 0;
    for (int i = 0; i < b.count; ++i) {
      const egn_small_gemm_t& g = problems[base + i];
      b.g[i] = g;
      b.tile0[i + 1] = b.tile0[i] + ((g.m + T - 1) / T) * ((g.n + T - 1) / T);
    }
    if (b.tile0[b.count] == 0) continue;
    if (T == 64) small_gemm64_kernel<<<b.tile0[b.count], 256, 0, st>>>(b);
    else small_gemm_kernel<<<b.tile0[b.count], 256, 0, st>>>(b);
    if (int rc = check_launch("small_gemm_batched")) return rc;
  }
  return 0;
}

// ---------------------------------------------------------------- small device utilities
// (so the training step launches no framework elementwise kernels: zero fills, the DimeNet
// gate product, the W_sbf gradient transpose, CSR offsets of a user-given sorted edge list)
namespace egn {
__global__ void hadamard_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out,
                                int64_t n) {
  const int64_t n4 = n / 4;
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  float4* o4 = reinterpret_cast<float4*>(out);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 x = a4[i], y = b4[i];
    o4[i] = make_float4(x.x * y.x, x.y * y.y, x.z * y.z, x.w * y.w);
  }
  for (int64_t i = 4 * n4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = a[i] * b[i];
}

// out[c][r] = in[r][c] through 32 x 33 shared tiles
__global__ void transpose_kernel(const float* __restrict__ in, int64_t rows, int64_t cols, int64_t ld_in,
                                 float* __restrict__ out, int64_t ld_out) {
  __shared__ float t[32][33];
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) t[i][threadIdx.x] = in[r * ld_in + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * ld_out + r] = t[threadIdx.x][i];
  }
}

// ptr[v] = first k with keys[k] >= v (keys sorted ascending), v in [0, nv]
__global__ void csr_ptr_kernel(const int64_t* __restrict__ keys, int64_t n, int64_t nv, int64_t* __restrict__ ptr) {
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v <= nv;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    ptr[v] = lo;
  }
}
}  // namespace egn

extern "C" {
int egn_zero(void* ptr, int64_t bytes, egn_stream_t stream) {
  EGN_REQUIRE(bytes >= 0, "negative size");
  if (bytes == 0) return 0;
  cudaMemsetAsync(ptr, 0, static_cast<size_t>(bytes), as_stream(stream));
  return check_launch("zero");
}

int egn_hadamard(const float* a, const float* b, float* out, int64_t n, egn_stream_t stream) {
  using namespace egn;
  EGN_REQUIRE(((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(out)) &
               15) == 0,
              "hadamard operands must be 16-byte aligned");
  if (n == 0) return 0;
  hadamard_kernel<<<static_cast<int>(std::min<int64_t>((n / 4 + 255) / 256 + 1, kNumSMs * 16)), 256, 0,
                    as_stream(stream)>>>(a, b, out, n);
  return check_launch("hadamard");
}

int egn_transpose(const float* in, int64_t rows, int64_t cols, int64_t ld_in, float* out, int64_t ld_out,
                  egn_stream_t stream) {
  using namespace egn;
  EGN_REQUIRE(rows >= 0 && cols >= 0 && ld_in >= cols && ld_out >= rows, "bad transpose shape / strides");
  if (rows == 0 || cols == 0) return 0;
  const dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(in, rows, cols, ld_in, out, ld_out);
  return check_launch("transpose");
}

int egn_csr_ptr(const int64_t* keys, int64_t n, int64_t nv, int64_t* ptr, egn_stream_t stream) {
  using namespace egn;
  EGN_REQUIRE(n >= 0 && nv >= 0, "negative size");
  csr_ptr_kernel<<<grid_for(nv + 1, 256), 256, 0, as_stream(stream)>>>(keys, n, nv, ptr);
  return check_launch("csr_ptr");
}
}  // extern "C"
