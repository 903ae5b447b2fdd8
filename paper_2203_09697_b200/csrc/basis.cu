// Basis features and closed-form geometry derivatives at the reference's public API (fp64).
//
// The training hot path never materialises these tables: the triplet kernels generate
// rbf_k(d) T_l(cos a) on the fly from the packed per-edge (u, d).  These entry points serve
// the drop-in surface of egn/basis.py (rbf_features :35-42, rbf_features_ddist :45-51,
// sbf_features :54-74, sbf_features_partials :77-95, compute_basis :98-103) and
// egn/gradients.py geometry_grads (:33-36 over egn/graph.py angle_gradients :173-197 and
// distance_gradients :200-203), element for element in fp64, one thread per row.
#include <cmath>

#include "common.cuh"

namespace egn {
namespace basis {

// numpy.linspace(0, cutoff, K): start + k * step, the last centre exactly `cutoff`.
__device__ __forceinline__ double centre(int k, int K, double cutoff) {
  if (K == 1) return 0.0;
  if (k == K - 1) return cutoff;
  return static_cast<double>(k) * (cutoff / static_cast<double>(K - 1));
}

__global__ void rbf_features_kernel(const double* __restrict__ d, int64_t n, int K, double cutoff, double gamma,
                                    double* __restrict__ out, double* __restrict__ dout,
                                    int32_t* __restrict__ invalid) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const double de = d[e];
    if (!(de > 0.0 && de <= cutoff) && invalid) atomicExch(invalid, 1);
    for (int k = 0; k < K; ++k) {
      const double delta = de - centre(k, K, cutoff);
      const double v = exp(-gamma * (delta * delta));
      if (out) out[e * K + k] = v;
      if (dout) dout[e * K + k] = -2.0 * gamma * delta * v;
    }
  }
}

// entry (t, k L + l) = rbf_k(d_t) cos(l a_t); partials w.r.t. d_t and a_t (optional).
__global__ void sbf_features_kernel(const double* __restrict__ d, const double* __restrict__ ang, int64_t n, int K,
                                    int L, double cutoff, double gamma, double* __restrict__ out,
                                    double* __restrict__ d_dist, double* __restrict__ d_ang,
                                    int32_t* __restrict__ invalid) {
  const double pi = 3.141592653589793;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const double dt = d[t], a = ang[t];
    if (invalid && (!(dt > 0.0 && dt <= cutoff) || !(a >= -1e-12 && a <= pi + 1e-12))) atomicExch(invalid, 1);
    for (int k = 0; k < K; ++k) {
      const double delta = dt - centre(k, K, cutoff);
      const double r = exp(-gamma * (delta * delta));
      const double dr = -2.0 * gamma * delta * r;
      for (int l = 0; l < L; ++l) {
        const double la = a * static_cast<double>(l);
        const double c = cos(la);
        const int64_t o = t * (K * L) + k * L + l;
        if (out) out[o] = r * c;
        if (d_dist) d_dist[o] = dr * c;
        if (d_ang) d_ang[o] = r * (-static_cast<double>(l) * sin(la));
      }
    }
  }
}

__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

__global__ void distance_grads_kernel(const double* __restrict__ pos, const int64_t* __restrict__ src,
                                      const int64_t* __restrict__ recv, int64_t ne, double* __restrict__ d_src,
                                      double* __restrict__ d_recv) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = src[e], b = recv[e];
    double v[3];
    for (int i = 0; i < 3; ++i) v[i] = pos[3 * b + i] - pos[3 * a + i];
    const double d = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    for (int i = 0; i < 3; ++i) {
      d_src[3 * e + i] = -(v[i] / d);
      d_recv[3 * e + i] = v[i] / d;
    }
  }
}

// v1 = x_k - x_j, v2 = x_i - x_j; g_k = (v1/|v1| x n) / |v1|, g_i = (n x v2/|v2|) / |v2|,
// n = v1 x v2 / |v1 x v2|; zero when |v1 x v2| <= 1e-14 (collinear); g_j = -(g_k + g_i).
__global__ void angle_grads_kernel(const double* __restrict__ pos, const int64_t* __restrict__ src,
                                   const int64_t* __restrict__ recv, const int64_t* __restrict__ trip_in,
                                   const int64_t* __restrict__ trip_out, int64_t nt, double* __restrict__ gk,
                                   double* __restrict__ gj, double* __restrict__ gi) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ek = trip_in[t], ei = trip_out[t];
    const int64_t k = src[ek], j = recv[ek], i = recv[ei];
    double v1[3], v2[3], c[3];
    for (int q = 0; q < 3; ++q) {
      v1[q] = pos[3 * k + q] - pos[3 * j + q];
      v2[q] = pos[3 * i + q] - pos[3 * j + q];
    }
    cross3(v1, v2, c);
    const double s = sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    double a[3] = {0.0, 0.0, 0.0}, b[3] = {0.0, 0.0, 0.0};
    if (s > 1e-14) {
      double nh[3] = {c[0] / s, c[1] / s, c[2] / s};
      const double n1 = sqrt(v1[0] * v1[0] + v1[1] * v1[1] + v1[2] * v1[2]);
      const double n2 = sqrt(v2[0] * v2[0] + v2[1] * v2[1] + v2[2] * v2[2]);
      double u1[3] = {v1[0] / n1, v1[1] / n1, v1[2] / n1}, u2[3] = {v2[0] / n2, v2[1] / n2, v2[2] / n2};
      cross3(u1, nh, a);
      cross3(nh, u2, b);
      for (int q = 0; q < 3; ++q) {
        a[q] /= n1;
        b[q] /= n2;
      }
    }
    for (int q = 0; q < 3; ++q) {
      gk[3 * t + q] = a[q];
      gi[3 * t + q] = b[q];
      gj[3 * t + q] = -(a[q] + b[q]);
    }
  }
}

}  // namespace basis
}  // namespace egn

using namespace egn;

extern "C" {

int egn_rbf_features(const double* distances, int64_t n, int k_rbf, double cutoff, double* out, double* d_out,
                     int32_t* invalid, egn_stream_t stream) {
  EGN_REQUIRE(k_rbf >= 1, "k_rbf must be >= 1");
  EGN_REQUIRE(cutoff > 0.0, "cutoff must be positive");
  if (n == 0) return 0;
  const double gamma = (static_cast<double>(k_rbf) / cutoff) * (static_cast<double>(k_rbf) / cutoff);
  basis::rbf_features_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(distances, n, k_rbf, cutoff, gamma,
                                                                               out, d_out, invalid);
  return check_launch("rbf_features");
}

int egn_sbf_features(const double* in_edge_distances, const double* angles, int64_t n, int k_rbf, int l_sbf,
                     double cutoff, double* out, double* d_dist, double* d_ang, int32_t* invalid,
                     egn_stream_t stream) {
  EGN_REQUIRE(k_rbf >= 1, "k_rbf must be >= 1");
  EGN_REQUIRE(l_sbf >= 1, "l_sbf must be >= 1");
  EGN_REQUIRE(cutoff > 0.0, "cutoff must be positive");
  if (n == 0) return 0;
  const double gamma = (static_cast<double>(k_rbf) / cutoff) * (static_cast<double>(k_rbf) / cutoff);
  basis::sbf_features_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(
      in_edge_distances, angles, n, k_rbf, l_sbf, cutoff, gamma, out, d_dist, d_ang, invalid);
  return check_launch("sbf_features");
}

int egn_geometry_grads(const double* pos, const int64_t* src, const int64_t* recv, int64_t num_edges,
                       const int64_t* trip_in, const int64_t* trip_out, int64_t num_triplets, double* dist_d_src,
                       double* dist_d_recv, double* angle_d_k, double* angle_d_j, double* angle_d_i,
                       egn_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  if (num_edges > 0) {
    basis::distance_grads_kernel<<<grid_for(num_edges, 256), 256, 0, st>>>(pos, src, recv, num_edges, dist_d_src,
                                                                           dist_d_recv);
    if (check_launch("distance_grads")) return 1;
  }
  if (num_triplets > 0) {
    basis::angle_grads_kernel<<<grid_for(num_triplets, 256), 256, 0, st>>>(pos, src, recv, trip_in, trip_out,
                                                                           num_triplets, angle_d_k, angle_d_j,
                                                                           angle_d_i);
    return check_launch("angle_grads");
  }
  return 0;
}

}  // extern "C"
