// Graph construction kernels: neighbour list, CSR scans, reverse edges,
// triplet index materialisation and per-edge geometry.
//
// Reference: egn/graph.py (build_graph :82-103, enumerate_triplets :106-139,
// reverse_edges :40-55, edge_distances/units :142-150, triplet_angles
// :162-170).  The neighbour test is evaluated in fp64 with explicit
// round-to-nearest intrinsics so that no FMA contraction changes a
// distance by one ulp: d = sqrt((dx*dx + dy*dy) + dz*dz) exactly as numpy
// evaluates (diff*diff).sum(axis=2); the edge set and its order are then
// bit-identical to the reference's row-major np.nonzero.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace egn {

static thread_local char g_err[512] = "no error";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

__device__ __forceinline__ double pair_dist(const double* __restrict__ pos, int64_t a, int64_t b) {
  // diff = pos[b] - pos[a]   (graph.py:88: pos[None,:,:] - pos[:,None,:])
  double dx = __dsub_rn(pos[3 * b + 0], pos[3 * a + 0]);
  double dy = __dsub_rn(pos[3 * b + 1], pos[3 * a + 1]);
  double dz = __dsub_rn(pos[3 * b + 2], pos[3 * a + 2]);
  double s = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return __dsqrt_rn(s);
}

// One warp per source atom a; lanes sweep the atoms of a's graph.
__global__ void neighbors_count_kernel(const double* __restrict__ pos,
                                       const int64_t* __restrict__ graph_ptr,
                                       const int32_t* __restrict__ node_graph, int64_t n,
                                       double cutoff, int32_t* __restrict__ deg) {
  int lane = threadIdx.x & 31;
  int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t a = warp; a < n; a += nwarps) {
    int g = node_graph[a];
    int64_t b0 = graph_ptr[g], b1 = graph_ptr[g + 1];
    int count = 0;
    for (int64_t b = b0 + lane; b < b1; b += 32) {
      double d = pair_dist(pos, a, b);
      count += (b != a) && (d > 0.0) && (d <= cutoff);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) count += __shfl_xor_sync(0xffffffffu, count, o);
    if (lane == 0) deg[a] = count;
  }
}

__global__ void neighbors_fill_kernel(const double* __restrict__ pos,
                                      const int64_t* __restrict__ graph_ptr,
                                      const int32_t* __restrict__ node_graph, int64_t n,
                                      double cutoff, const int64_t* __restrict__ edge_ptr,
                                      int32_t* __restrict__ src, int32_t* __restrict__ recv) {
  int lane = threadIdx.x & 31;
  int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t a = warp; a < n; a += nwarps) {
    int g = node_graph[a];
    int64_t b0 = graph_ptr[g], b1 = graph_ptr[g + 1];
    int64_t out = edge_ptr[a];
    for (int64_t base = b0; base < b1; base += 32) {
      int64_t b = base + lane;
      bool hit = false;
      if (b < b1) {
        double d = pair_dist(pos, a, b);
        hit = (b != a) && (d > 0.0) && (d <= cutoff);
      }
      unsigned mask = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        int64_t slot = out + __popc(mask & ((1u << lane) - 1u));
        src[slot] = static_cast<int32_t>(a);
        recv[slot] = static_cast<int32_t>(b);
      }
      out += __popc(mask);
    }
  }
}

// Single-CTA exclusive scan (n+1 outputs).  Graph-construction sizes
// (nodes <= ~10^6) make one 1024-thread CTA sufficient.
__global__ void scan_counts_kernel(const int32_t* __restrict__ in, int64_t n, int sq,
                                   int64_t* __restrict__ out) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t carry;
  int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += blockDim.x) {
    int64_t i = base + tid;
    int64_t v = 0;
    if (i < n) {
      int64_t x = in[i];
      v = sq ? x * (x - 1) : x;
    }
    int64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int64_t t = lane < (blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;  // inclusive prefix of warp totals
    }
    __syncthreads();
    int64_t before = carry + (wid > 0 ? warp_tot[wid - 1] : 0);
    if (i < n) out[i] = before + incl - v;
    __syncthreads();
    if (tid == blockDim.x - 1) carry = before + incl;
    __syncthreads();
  }
  if (tid == 0) out[n] = carry;
}

// rev[e]: binary search for src(e) among the receivers of recv(e)'s row.
__global__ void reverse_edges_kernel(const int64_t* __restrict__ edge_ptr,
                                     const int32_t* __restrict__ src,
                                     const int32_t* __restrict__ recv, int64_t ne,
                                     int32_t* __restrict__ rev, int32_t* __restrict__ missing) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    int32_t a = src[e], b = recv[e];
    int64_t lo = edge_ptr[b], hi = edge_ptr[b + 1];
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (recv[mid] < a) lo = mid + 1; else hi = mid;
    }
    if (lo < edge_ptr[b + 1] && recv[lo] == a) {
      rev[e] = static_cast<int32_t>(lo);
    } else {
      rev[e] = -1;
      atomicAdd(missing, 1);
    }
  }
}

// One CTA per centre j: triplet (p, q), q != p, lives at
// tri_ptr[j] + p*(n-1) + (q < p ? q : q-1); id3_ji = off+p, id3_kj = rev[off+q].
__global__ void triplets_fill_kernel(const int64_t* __restrict__ edge_ptr,
                                     const int32_t* __restrict__ rev,
                                     const int64_t* __restrict__ tri_ptr, int64_t nv,
                                     int64_t* __restrict__ id3_kj, int64_t* __restrict__ id3_ji) {
  for (int64_t j = blockIdx.x; j < nv; j += gridDim.x) {
    int64_t off = edge_ptr[j];
    int64_t n = edge_ptr[j + 1] - off;
    if (n < 2) continue;
    int64_t t0 = tri_ptr[j];
    int64_t cnt = n * (n - 1);
    for (int64_t k = threadIdx.x; k < cnt; k += blockDim.x) {
      int64_t p = k / (n - 1);
      int64_t r = k - p * (n - 1);
      int64_t q = r < p ? r : r + 1;
      id3_ji[t0 + k] = off + p;
      id3_kj[t0 + k] = rev[off + q];
    }
  }
}

__global__ void geometry_kernel(const double* __restrict__ pos, const int32_t* __restrict__ src,
                                const int32_t* __restrict__ recv, int64_t ne,
                                float4* __restrict__ geo, double* __restrict__ dist64,
                                double* __restrict__ unit64) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = src[e], b = recv[e];
    double dx = __dsub_rn(pos[3 * b + 0], pos[3 * a + 0]);
    double dy = __dsub_rn(pos[3 * b + 1], pos[3 * a + 1]);
    double dz = __dsub_rn(pos[3 * b + 2], pos[3 * a + 2]);
    double d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    double ux = __ddiv_rn(dx, d), uy = __ddiv_rn(dy, d), uz = __ddiv_rn(dz, d);
    geo[e] = make_float4(static_cast<float>(ux), static_cast<float>(uy), static_cast<float>(uz),
                         static_cast<float>(d));
    if (dist64) dist64[e] = d;
    if (unit64) {
      unit64[3 * e + 0] = ux;
      unit64[3 * e + 1] = uy;
      unit64[3 * e + 2] = uz;
    }
  }
}

// Angle of triplet (q -> p) at centre j: v1 = x_k - x_j (edge off+q),
// v2 = x_i - x_j (edge off+p); atan2(|v1 x v2|, v1 . v2) in fp64.
__global__ void triplet_angles_kernel(const double* __restrict__ pos,
                                      const int64_t* __restrict__ edge_ptr,
                                      const int32_t* __restrict__ recv,
                                      const int64_t* __restrict__ tri_ptr, int64_t nv,
                                      double* __restrict__ angles) {
  for (int64_t j = blockIdx.x; j < nv; j += gridDim.x) {
    int64_t off = edge_ptr[j];
    int64_t n = edge_ptr[j + 1] - off;
    if (n < 2) continue;
    int64_t t0 = tri_ptr[j];
    int64_t cnt = n * (n - 1);
    double xj = pos[3 * j], yj = pos[3 * j + 1], zj = pos[3 * j + 2];
    for (int64_t k = threadIdx.x; k < cnt; k += blockDim.x) {
      int64_t p = k / (n - 1);
      int64_t r = k - p * (n - 1);
      int64_t q = r < p ? r : r + 1;
      int64_t kk = recv[off + q], ii = recv[off + p];
      double v1x = pos[3 * kk] - xj, v1y = pos[3 * kk + 1] - yj, v1z = pos[3 * kk + 2] - zj;
      double v2x = pos[3 * ii] - xj, v2y = pos[3 * ii + 1] - yj, v2z = pos[3 * ii + 2] - zj;
      double cx = __dsub_rn(__dmul_rn(v1y, v2z), __dmul_rn(v1z, v2y));
      double cy = __dsub_rn(__dmul_rn(v1z, v2x), __dmul_rn(v1x, v2z));
      double cz = __dsub_rn(__dmul_rn(v1x, v2y), __dmul_rn(v1y, v2x));
      double s = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz)));
      double c = __dadd_rn(__dadd_rn(__dmul_rn(v1x, v2x), __dmul_rn(v1y, v2y)), __dmul_rn(v1z, v2z));
      angles[t0 + k] = atan2(s, c);
    }
  }
}

// ---------------------------------------------------------------------------
// Periodic cells.  Per graph: cell rows c0, c1, c2 (lattice vectors)
// and image ranges nimg = (na, nb, nc); image index img = ((i+na)(2nb+1) + (j+nb))(2nc+1)
// + (k+nc) for the shift s = (i c0 + j c1) + k c2 (per component, round-to-nearest, no FMA).
// An edge (a, b, img) is the vector (x_b - x_a) + s; candidates of a row are ordered by
// (b, img), so rows are sorted by (recv, img) and the mirrored image of img is
// n_img - 1 - img.
struct Img {
  int na, nb, nc, n;
};
__device__ __forceinline__ Img img_dims(const int32_t* __restrict__ nimg, int g) {
  Img m;
  m.na = nimg[3 * g];
  m.nb = nimg[3 * g + 1];
  m.nc = nimg[3 * g + 2];
  m.n = (2 * m.na + 1) * (2 * m.nb + 1) * (2 * m.nc + 1);
  return m;
}
__device__ __forceinline__ void img_shift(const double* __restrict__ cell, int g, const Img& m, int img,
                                          double& sx, double& sy, double& sz) {
  const int kc = img % (2 * m.nc + 1) - m.nc;
  const int r = img / (2 * m.nc + 1);
  const int jb = r % (2 * m.nb + 1) - m.nb;
  const int ia = r / (2 * m.nb + 1) - m.na;
  const double* c = cell + 9 * g;
  const double fi = ia, fj = jb, fk = kc;
  sx = __dadd_rn(__dadd_rn(__dmul_rn(fi, c[0]), __dmul_rn(fj, c[3])), __dmul_rn(fk, c[6]));
  sy = __dadd_rn(__dadd_rn(__dmul_rn(fi, c[1]), __dmul_rn(fj, c[4])), __dmul_rn(fk, c[7]));
  sz = __dadd_rn(__dadd_rn(__dmul_rn(fi, c[2]), __dmul_rn(fj, c[5])), __dmul_rn(fk, c[8]));
}
__device__ __forceinline__ double pair_dist_shift(const double* __restrict__ pos, int64_t a, int64_t b, double sx,
                                                  double sy, double sz) {
  // (x_b - x_a) + s: exactly antisymmetric under (a, b, s) -> (b, a, -s), so an edge and its
  // reverse always pass or fail the cutoff together (s = 0: the reference's x_b - x_a)
  const double dx = __dadd_rn(__dsub_rn(pos[3 * b + 0], pos[3 * a + 0]), sx);
  const double dy = __dadd_rn(__dsub_rn(pos[3 * b + 1], pos[3 * a + 1]), sy);
  const double dz = __dadd_rn(__dsub_rn(pos[3 * b + 2], pos[3 * a + 2]), sz);
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

// One warp per source atom; lanes sweep (b, img) candidates in (b, img) order.
template <bool FILL>
__global__ void neighbors_pbc_kernel(const double* __restrict__ pos, const int64_t* __restrict__ graph_ptr,
                                     const int32_t* __restrict__ node_graph, int64_t n,
                                     const double* __restrict__ cell, const int32_t* __restrict__ nimg,
                                     double cutoff, int32_t* __restrict__ deg, const int64_t* __restrict__ edge_ptr,
                                     int32_t* __restrict__ src, int32_t* __restrict__ recv,
                                     int32_t* __restrict__ eimg, double* __restrict__ shift) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t a = warp; a < n; a += nwarps) {
    const int g = node_graph[a];
    const int64_t b0 = graph_ptr[g], b1 = graph_ptr[g + 1];
    const Img m = img_dims(nimg, g);
    const int centre = m.n / 2;
    const int64_t ncand = (b1 - b0) * m.n;
    int count = 0;
    int64_t out = FILL ? edge_ptr[a] : 0;
    for (int64_t base = 0; base < ncand; base += 32) {
      const int64_t c = base + lane;
      bool hit = false;
      int64_t b = 0;
      int img = 0;
      double sx = 0.0, sy = 0.0, sz = 0.0;
      if (c < ncand) {
        b = b0 + c / m.n;
        img = static_cast<int>(c % m.n);
        img_shift(cell, g, m, img, sx, sy, sz);
        const double d = pair_dist_shift(pos, a, b, sx, sy, sz);
        hit = !(b == a && img == centre) && (d > 0.0) && (d <= cutoff);
      }
      if (!FILL) {
        count += hit;
      } else {
        const unsigned mask = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const int64_t slot = out + __popc(mask & ((1u << lane) - 1u));
          src[slot] = static_cast<int32_t>(a);
          recv[slot] = static_cast<int32_t>(b);
          eimg[slot] = img;
          shift[3 * slot + 0] = sx;
          shift[3 * slot + 1] = sy;
          shift[3 * slot + 2] = sz;
        }
        out += __popc(mask);
      }
    }
    if (!FILL) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) count += __shfl_xor_sync(0xffffffffu, count, o);
      if (lane == 0) deg[a] = count;
    }
  }
}

// rev[e]: the edge (recv_e, src_e, mirrored image): binary search on (recv, img) in recv_e's row.
__global__ void reverse_edges_pbc_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ src,
                                         const int32_t* __restrict__ recv, const int32_t* __restrict__ eimg,
                                         const int32_t* __restrict__ node_graph, const int32_t* __restrict__ nimg,
                                         int64_t ne, int32_t* __restrict__ rev, int32_t* __restrict__ missing) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = src[e], b = recv[e];
    const Img m = img_dims(nimg, node_graph[a]);
    const int64_t key = static_cast<int64_t>(a) * m.n + (m.n - 1 - eimg[e]);
    int64_t lo = edge_ptr[b], hi = edge_ptr[b + 1];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (static_cast<int64_t>(recv[mid]) * m.n + eimg[mid] < key) lo = mid + 1;
      else hi = mid;
    }
    if (lo < edge_ptr[b + 1] && static_cast<int64_t>(recv[lo]) * m.n + eimg[lo] == key) {
      rev[e] = static_cast<int32_t>(lo);
    } else {
      rev[e] = -1;
      atomicAdd(missing, 1);
    }
  }
}

// Edge geometry from (x_recv - x_src) + shift (shift NULL: the non-periodic form).
__global__ void geometry_shift_kernel(const double* __restrict__ pos, const int32_t* __restrict__ src,
                                      const int32_t* __restrict__ recv, const double* __restrict__ shift, int64_t ne,
                                      float4* __restrict__ geo, double* __restrict__ dist64,
                                      double* __restrict__ unit64) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = src[e], b = recv[e];
    const double dx = __dadd_rn(__dsub_rn(pos[3 * b + 0], pos[3 * a + 0]), shift[3 * e + 0]);
    const double dy = __dadd_rn(__dsub_rn(pos[3 * b + 1], pos[3 * a + 1]), shift[3 * e + 1]);
    const double dz = __dadd_rn(__dsub_rn(pos[3 * b + 2], pos[3 * a + 2]), shift[3 * e + 2]);
    const double d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    const double ux = __ddiv_rn(dx, d), uy = __ddiv_rn(dy, d), uz = __ddiv_rn(dz, d);
    geo[e] = make_float4(static_cast<float>(ux), static_cast<float>(uy), static_cast<float>(uz),
                         static_cast<float>(d));
    if (dist64) dist64[e] = d;
    if (unit64) {
      unit64[3 * e + 0] = ux;
      unit64[3 * e + 1] = uy;
      unit64[3 * e + 2] = uz;
    }
  }
}

// Triplet angles from edge vectors: v1 = -vec(rev-side in-edge) = vec(off+q), v2 = vec(off+p),
// vec(e) = (x_recv - x_src) + shift, all per the centre's out-edges.
__global__ void triplet_angles_shift_kernel(const double* __restrict__ pos, const int64_t* __restrict__ edge_ptr,
                                            const int32_t* __restrict__ recv, const double* __restrict__ shift,
                                            const int64_t* __restrict__ tri_ptr, int64_t nv,
                                            double* __restrict__ angles) {
  for (int64_t j = blockIdx.x; j < nv; j += gridDim.x) {
    const int64_t off = edge_ptr[j];
    const int64_t n = edge_ptr[j + 1] - off;
    if (n < 2) continue;
    const int64_t t0 = tri_ptr[j];
    const int64_t cnt = n * (n - 1);
    const double xj = pos[3 * j], yj = pos[3 * j + 1], zj = pos[3 * j + 2];
    for (int64_t k = threadIdx.x; k < cnt; k += blockDim.x) {
      const int64_t p = k / (n - 1);
      const int64_t r = k - p * (n - 1);
      const int64_t q = r < p ? r : r + 1;
      const int64_t eq = off + q, ep = off + p;
      const int64_t kk = recv[eq], ii = recv[ep];
      const double v1x = __dadd_rn(__dsub_rn(pos[3 * kk], xj), shift[3 * eq]);
      const double v1y = __dadd_rn(__dsub_rn(pos[3 * kk + 1], yj), shift[3 * eq + 1]);
      const double v1z = __dadd_rn(__dsub_rn(pos[3 * kk + 2], zj), shift[3 * eq + 2]);
      const double v2x = __dadd_rn(__dsub_rn(pos[3 * ii], xj), shift[3 * ep]);
      const double v2y = __dadd_rn(__dsub_rn(pos[3 * ii + 1], yj), shift[3 * ep + 1]);
      const double v2z = __dadd_rn(__dsub_rn(pos[3 * ii + 2], zj), shift[3 * ep + 2]);
      const double cx = __dsub_rn(__dmul_rn(v1y, v2z), __dmul_rn(v1z, v2y));
      const double cy = __dsub_rn(__dmul_rn(v1z, v2x), __dmul_rn(v1x, v2z));
      const double cz = __dsub_rn(__dmul_rn(v1x, v2y), __dmul_rn(v1y, v2x));
      const double s = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz)));
      const double c = __dadd_rn(__dadd_rn(__dmul_rn(v1x, v2x), __dmul_rn(v1y, v2y)), __dmul_rn(v1z, v2z));
      angles[t0 + k] = atan2(s, c);
    }
  }
}

// ---------------------------------------------------------------------------
// Neighbour cap (SURVEY.md 8(f) f1, OC20's max-neighbours): an out-edge survives when it is
// among the max_nb nearest of its source (distance, then edge index, in fp64) and its
// reverse survives the same test at the other end (mutual, so the graph stays symmetric
// for the reverse-edge algebra).  Then the kept edges are compacted in row order.
__global__ void cap_rank_kernel(const int64_t* __restrict__ edge_ptr, const double* __restrict__ dist, int64_t nv,
                                int max_nb, int32_t* __restrict__ keep) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < nv; v += nwarps) {
    const int64_t e0 = edge_ptr[v], e1 = edge_ptr[v + 1];
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const double d = dist[e];
      int64_t rank = 0;
      for (int64_t f = e0; f < e1; ++f) {
        const double df = dist[f];
        rank += (df < d) || (df == d && f < e);
      }
      keep[e] = rank < max_nb;
    }
  }
}

__global__ void cap_mutual_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ rev, int64_t nv,
                                  const int32_t* __restrict__ keep1, int32_t* __restrict__ keep,
                                  int32_t* __restrict__ deg) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < nv; v += nwarps) {
    int count = 0;
    for (int64_t e = edge_ptr[v] + lane; e < edge_ptr[v + 1]; e += 32) {
      const int32_t k = keep1[e] && keep1[rev[e]];
      keep[e] = k;
      count += k;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) count += __shfl_xor_sync(0xffffffffu, count, o);
    if (lane == 0) deg[v] = count;
  }
}

// kept edges of each row compacted in order: new_id[e] (or -1), and the per-edge payload
__global__ void cap_compact_kernel(const int64_t* __restrict__ edge_ptr, const int64_t* __restrict__ new_ptr,
                                   int64_t nv, const int32_t* __restrict__ keep, const int32_t* __restrict__ src,
                                   const int32_t* __restrict__ recv, const int32_t* __restrict__ img,
                                   const double* __restrict__ shift, int32_t* __restrict__ new_id,
                                   int32_t* __restrict__ nsrc, int32_t* __restrict__ nrecv, int32_t* __restrict__ nimg,
                                   double* __restrict__ nshift) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < nv; v += nwarps) {
    const int64_t e1 = edge_ptr[v + 1];
    int64_t out = new_ptr[v];
    for (int64_t base = edge_ptr[v]; base < e1; base += 32) {
      const int64_t e = base + lane;
      const bool k = e < e1 && keep[e];
      const unsigned mask = __ballot_sync(0xffffffffu, k);
      if (e < e1) {
        if (k) {
          const int64_t slot = out + __popc(mask & ((1u << lane) - 1u));
          new_id[e] = static_cast<int32_t>(slot);
          nsrc[slot] = src[e];
          nrecv[slot] = recv[e];
          if (img) nimg[slot] = img[e];
          if (shift) {
            nshift[3 * slot] = shift[3 * e];
            nshift[3 * slot + 1] = shift[3 * e + 1];
            nshift[3 * slot + 2] = shift[3 * e + 2];
          }
        } else {
          new_id[e] = -1;
        }
      }
      out += __popc(mask);
    }
  }
}

__global__ void cap_rev_kernel(int64_t ne, const int32_t* __restrict__ rev, const int32_t* __restrict__ new_id,
                               int32_t* __restrict__ nrev) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t n = new_id[e];
    if (n >= 0) nrev[n] = new_id[rev[e]];
  }
}

}  // namespace egn

using namespace egn;

extern "C" {

const char* egn_last_error(void) { return g_err; }
int egn_abi_version(void) { return 3; }

int egn_neighbors_count(const double* pos, const int64_t* graph_ptr, const int32_t* node_graph,
                        int64_t num_nodes, double cutoff, int32_t* deg, egn_stream_t stream) {
  EGN_REQUIRE(cutoff > 0, "cutoff must be positive");
  if (num_nodes == 0) return 0;
  int threads = 256;
  int grid = grid_for(num_nodes * 32, threads);
  neighbors_count_kernel<<<grid, threads, 0, as_stream(stream)>>>(pos, graph_ptr, node_graph,
                                                                  num_nodes, cutoff, deg);
  return check_launch("neighbors_count");
}

int egn_scan_counts(const int32_t* in, int64_t n, int square_minus_one, int64_t* out,
                    egn_stream_t stream) {
  scan_counts_kernel<<<1, 1024, 0, as_stream(stream)>>>(in, n, square_minus_one, out);
  return check_launch("scan_counts");
}

int egn_neighbors_fill(const double* pos, const int64_t* graph_ptr, const int32_t* node_graph,
                       int64_t num_nodes, double cutoff, const int64_t* edge_ptr, int32_t* src,
                       int32_t* recv, egn_stream_t stream) {
  if (num_nodes == 0) return 0;
  int threads = 256;
  int grid = grid_for(num_nodes * 32, threads);
  neighbors_fill_kernel<<<grid, threads, 0, as_stream(stream)>>>(
      pos, graph_ptr, node_graph, num_nodes, cutoff, edge_ptr, src, recv);
  return check_launch("neighbors_fill");
}

int egn_reverse_edges(const int64_t* edge_ptr, const int32_t* src, const int32_t* recv,
                      int64_t num_edges, int32_t* rev, int32_t* missing, egn_stream_t stream) {
  if (num_edges == 0) return 0;
  int threads = 256;
  reverse_edges_kernel<<<grid_for(num_edges, threads), threads, 0, as_stream(stream)>>>(
      edge_ptr, src, recv, num_edges, rev, missing);
  return check_launch("reverse_edges");
}

int egn_triplets_fill(const int64_t* edge_ptr, const int32_t* rev, const int64_t* tri_ptr,
                      int64_t num_nodes, int64_t* id3_kj, int64_t* id3_ji, egn_stream_t stream) {
  if (num_nodes == 0) return 0;
  int grid = static_cast<int>(num_nodes < 65535 ? num_nodes : 65535);
  triplets_fill_kernel<<<grid, 256, 0, as_stream(stream)>>>(edge_ptr, rev, tri_ptr, num_nodes,
                                                            id3_kj, id3_ji);
  return check_launch("triplets_fill");
}

int egn_geometry(const double* pos, const int32_t* src, const int32_t* recv, int64_t num_edges,
                 float* geo, double* dist64, double* unit64, egn_stream_t stream) {
  if (num_edges == 0) return 0;
  int threads = 256;
  geometry_kernel<<<grid_for(num_edges, threads), threads, 0, as_stream(stream)>>>(
      pos, src, recv, num_edges, reinterpret_cast<float4*>(geo), dist64, unit64);
  return check_launch("geometry");
}

int egn_triplet_angles(const double* pos, const int64_t* edge_ptr, const int32_t* recv,
                       const int64_t* tri_ptr, int64_t num_nodes, double* angles,
                       egn_stream_t stream) {
  if (num_nodes == 0) return 0;
  int grid = static_cast<int>(num_nodes < 65535 ? num_nodes : 65535);
  triplet_angles_kernel<<<grid, 256, 0, as_stream(stream)>>>(pos, edge_ptr, recv, tri_ptr,
                                                             num_nodes, angles);
  return check_launch("triplet_angles");
}

int egn_neighbors_count_pbc(const double* pos, const int64_t* graph_ptr, const int32_t* node_graph,
                            int64_t num_nodes, const double* cell, const int32_t* nimg, double cutoff, int32_t* deg,
                            egn_stream_t stream) {
  EGN_REQUIRE(cutoff > 0, "cutoff must be positive");
  if (num_nodes == 0) return 0;
  neighbors_pbc_kernel<false><<<grid_for(num_nodes * 32, 256), 256, 0, as_stream(stream)>>>(
      pos, graph_ptr, node_graph, num_nodes, cell, nimg, cutoff, deg, nullptr, nullptr, nullptr, nullptr, nullptr);
  return check_launch("neighbors_count_pbc");
}

int egn_neighbors_fill_pbc(const double* pos, const int64_t* graph_ptr, const int32_t* node_graph,
                           int64_t num_nodes, const double* cell, const int32_t* nimg, double cutoff,
                           const int64_t* edge_ptr, int32_t* src, int32_t* recv, int32_t* img, double* shift,
                           egn_stream_t stream) {
  if (num_nodes == 0) return 0;
  neighbors_pbc_kernel<true><<<grid_for(num_nodes * 32, 256), 256, 0, as_stream(stream)>>>(
      pos, graph_ptr, node_graph, num_nodes, cell, nimg, cutoff, nullptr, edge_ptr, src, recv, img, shift);
  return check_launch("neighbors_fill_pbc");
}

int egn_reverse_edges_pbc(const int64_t* edge_ptr, const int32_t* src, const int32_t* recv, const int32_t* img,
                          const int32_t* node_graph, const int32_t* nimg, int64_t num_edges, int32_t* rev,
                          int32_t* missing, egn_stream_t stream) {
  if (num_edges == 0) return 0;
  reverse_edges_pbc_kernel<<<grid_for(num_edges, 256), 256, 0, as_stream(stream)>>>(
      edge_ptr, src, recv, img, node_graph, nimg, num_edges, rev, missing);
  return check_launch("reverse_edges_pbc");
}

int egn_cap_keep(const int64_t* edge_ptr, const double* dist, const int32_t* rev, int64_t num_nodes, int max_neighbors,
                 int32_t* keep1, int32_t* keep, int32_t* deg, egn_stream_t stream) {
  EGN_REQUIRE(max_neighbors >= 0, "max_neighbors must be >= 0");
  if (num_nodes == 0) return 0;
  cudaStream_t st = as_stream(stream);
  cap_rank_kernel<<<grid_for(num_nodes * 32, 256), 256, 0, st>>>(edge_ptr, dist, num_nodes, max_neighbors, keep1);
  if (check_launch("cap_rank")) return 1;
  cap_mutual_kernel<<<grid_for(num_nodes * 32, 256), 256, 0, st>>>(edge_ptr, rev, num_nodes, keep1, keep, deg);
  return check_launch("cap_mutual");
}

int egn_cap_compact(const int64_t* edge_ptr, const int64_t* new_ptr, int64_t num_nodes, int64_t num_edges,
                    const int32_t* keep, const int32_t* src, const int32_t* recv, const int32_t* img,
                    const double* shift, const int32_t* rev, int32_t* new_id, int32_t* nsrc, int32_t* nrecv,
                    int32_t* nimg, double* nshift, int32_t* nrev, egn_stream_t stream) {
  if (num_nodes == 0 || num_edges == 0) return 0;
  cudaStream_t st = as_stream(stream);
  cap_compact_kernel<<<grid_for(num_nodes * 32, 256), 256, 0, st>>>(edge_ptr, new_ptr, num_nodes, keep, src, recv,
                                                                    img, shift, new_id, nsrc, nrecv, nimg, nshift);
  if (check_launch("cap_compact")) return 1;
  cap_rev_kernel<<<grid_for(num_edges, 256), 256, 0, st>>>(num_edges, rev, new_id, nrev);
  return check_launch("cap_rev");
}

int egn_geometry_shift(const double* pos, const int32_t* src, const int32_t* recv, const double* shift,
                       int64_t num_edges, float* geo, double* dist64, double* unit64, egn_stream_t stream) {
  if (num_edges == 0) return 0;
  if (shift == nullptr) return egn_geometry(pos, src, recv, num_edges, geo, dist64, unit64, stream);
  geometry_shift_kernel<<<grid_for(num_edges, 256), 256, 0, as_stream(stream)>>>(
      pos, src, recv, shift, num_edges, reinterpret_cast<float4*>(geo), dist64, unit64);
  return check_launch("geometry_shift");
}

int egn_triplet_angles_shift(const double* pos, const int64_t* edge_ptr, const int32_t* recv, const double* shift,
                             const int64_t* tri_ptr, int64_t num_nodes, double* angles, egn_stream_t stream) {
  if (num_nodes == 0) return 0;
  if (shift == nullptr) return egn_triplet_angles(pos, edge_ptr, recv, tri_ptr, num_nodes, angles, stream);
  const int grid = static_cast<int>(num_nodes < 65535 ? num_nodes : 65535);
  triplet_angles_shift_kernel<<<grid, 256, 0, as_stream(stream)>>>(pos, edge_ptr, recv, shift, tri_ptr, num_nodes,
                                                                   angles);
  return check_launch("triplet_angles_shift");
}

}  // extern "C"
