// Graph-level update block GU (egn/engine.py:207-217): per graph g
//   pre = s W1^T + b1,  act = silu(pre),  u += act W2^T + b2        (s = sum of v over g's nodes)
// and its adjoint.  G (graphs in the batch) is small, so these are SIMT kernels with one warp
// per output element and the activations / bias / residual fused (two launches forward,
// three backward) instead of library GEMM calls plus elementwise passes.  fp32 FMA in
// fixed order (deterministic).
#include <algorithm>

#include "common.cuh"

namespace egn {
namespace gmlp {

__device__ __forceinline__ float silu_f(float x) { return x / (1.f + __expf(-x)); }
__device__ __forceinline__ float dsilu_f(float x) {
  const float sg = 1.f / (1.f + __expf(-x));
  return sg * (1.f + x * (1.f - sg));
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Row-parallel layers: grid (graphs, ceil(out / 8)), warp = one output (r, j); the lanes split
// the dot product (4 independent loads in flight per lane), fixed butterfly reduction.
//   x_stride: distance between consecutive inputs of one weight row (1: W[j, :] rows,
//   out: W[:, j] columns), w_row: distance between consecutive outputs.
__device__ __forceinline__ float warp_dot(const float* __restrict__ x, const float* __restrict__ w, int n,
                                          int64_t w_step, int lane) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  int k = lane;
  for (; k + 96 < n; k += 128) {
    const float w0 = __ldg(w + k * w_step), w1 = __ldg(w + (k + 32) * w_step), w2 = __ldg(w + (k + 64) * w_step),
                w3 = __ldg(w + (k + 96) * w_step);
    a0 = fmaf(x[k], w0, a0);
    a1 = fmaf(x[k + 32], w1, a1);
    a2 = fmaf(x[k + 64], w2, a2);
    a3 = fmaf(x[k + 96], w3, a3);
  }
  for (; k < n; k += 32) a0 = fmaf(x[k], __ldg(w + k * w_step), a0);
  return warp_sum((a0 + a1) + (a2 + a3));
}

// layer 1 forward: pre = s W1^T + b1, act = silu(pre).  W1 NULL: s is already projected
// (pre = s + b1, dv == du; the graph-parallel reference schedule all-reduces z = s W1^T);
// b1 / act NULL: no bias / no activation output (the bare linear z = s W1^T).
__global__ void __launch_bounds__(256) fwd1_kernel(int dv, int du, const float* __restrict__ s,
                                                   const float* __restrict__ W1, const float* __restrict__ b1,
                                                   float* __restrict__ pre, float* __restrict__ act) {
  const int64_t r = blockIdx.x;
  const int j = blockIdx.y * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= du) return;
  float h = W1 ? warp_dot(s + r * dv, W1 + static_cast<int64_t>(j) * dv, dv, 1, lane) : s[r * dv + j];
  if (b1) h += b1[j];
  if (lane == 0) {
    pre[r * du + j] = h;
    if (act) act[r * du + j] = silu_f(h);
  }
}

// layer 2 forward: u += act W2^T + b2
__global__ void __launch_bounds__(256) fwd2_kernel(int du, const float* __restrict__ act,
                                                   const float* __restrict__ W2, const float* __restrict__ b2,
                                                   float* __restrict__ u) {
  const int64_t r = blockIdx.x;
  const int j = blockIdx.y * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= du) return;
  const float y = warp_dot(act + r * du, W2 + static_cast<int64_t>(j) * du, du, 1, lane);
  if (lane == 0) u[r * du + j] += y + b2[j];
}

// backward layer 2: pre_bar = silu'(pre) (u_bar W2)   (W2 columns)
__global__ void __launch_bounds__(256) bwd2_kernel(int du, const float* __restrict__ u_bar,
                                                   const float* __restrict__ pre, const float* __restrict__ W2,
                                                   float* __restrict__ pre_bar) {
  const int64_t r = blockIdx.x;
  const int j = blockIdx.y * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= du) return;
  const float y = warp_dot(u_bar + r * du, W2 + j, du, du, lane);
  if (lane == 0) pre_bar[r * du + j] = y * dsilu_f(pre[r * du + j]);
}

// backward layer 1: s_bar = pre_bar W1   (W1 columns; W1 NULL: s_bar = pre_bar)
__global__ void __launch_bounds__(256) bwd1_kernel(int dv, int du, const float* __restrict__ pre_bar,
                                                   const float* __restrict__ W1, float* __restrict__ s_bar) {
  const int64_t r = blockIdx.x;
  const int i = blockIdx.y * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= dv) return;
  const float y = W1 ? warp_dot(pre_bar + r * du, W1 + i, du, dv, lane) : pre_bar[r * du + i];
  if (lane == 0) s_bar[r * dv + i] = y;
}

// backward weights: CTA (j, layer): row j of W2_bar [du, du] (layer 0) or W1_bar [du, dv]
// (layer 1) and the bias entry j:
//   W2_bar[j, k] = sum_g u_bar[g, j] act[g, k],  W1_bar[j, i] = sum_g pre_bar[g, j] s[g, i],
//   b2_bar[j] = sum_g u_bar[g, j],  b1_bar[j] = sum_g pre_bar[g, j]   (graphs in order)
__global__ void __launch_bounds__(256) bwd_weights_kernel(int64_t G, int dv, int du, const float* __restrict__ u_bar,
                                                          const float* __restrict__ act,
                                                          const float* __restrict__ pre_bar,
                                                          const float* __restrict__ s, float* __restrict__ gW1,
                                                          float* __restrict__ gb1, float* __restrict__ gW2,
                                                          float* __restrict__ gb2) {
  const int j = blockIdx.x;
  const bool l2 = blockIdx.y == 0;
  // NULL outputs are skipped (the split head / tail of the graph-parallel reference schedule)
  if (l2 && gW2 == nullptr && gb2 == nullptr) return;
  const float* lhs = l2 ? u_bar : pre_bar;  // [G, du], column j
  const float* rhs = l2 ? act : s;          // [G, width]
  const int width = l2 ? du : dv;
  float* gw = l2 ? gW2 : gW1;
  // graphs in chunks of 8 with every load of a chunk issued before its FMAs (explicit ILP:
  // the sequential accumulation chain alone serialises the loads)
  for (int k = threadIdx.x; k < width; k += blockDim.x) {
    float a = 0.f, bsum = 0.f;
    int g = 0;
    for (; g + 8 <= G; g += 8) {
      float l[8], r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        l[u] = __ldg(lhs + static_cast<int64_t>(g + u) * du + j);
        r[u] = __ldg(rhs + static_cast<int64_t>(g + u) * width + k);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a = fmaf(l[u], r[u], a);
        bsum += l[u];
      }
    }
    for (; g < G; ++g) {
      const float l = __ldg(lhs + static_cast<int64_t>(g) * du + j);
      a = fmaf(l, __ldg(rhs + static_cast<int64_t>(g) * width + k), a);
      bsum += l;
    }
    if (gw) gw[static_cast<int64_t>(j) * width + k] = a;
    float* gb = l2 ? gb2 : gb1;
    if (k == 0 && gb) gb[j] = bsum;
  }
}

}  // namespace gmlp
}  // namespace egn

using namespace egn;

extern "C" int egn_graph_mlp_fwd(int64_t num_graphs, int dv, int du, const float* s, const float* w1,
                                 const float* b1, const float* w2, const float* b2, float* pre, float* act,
                                 float* u, egn_stream_t stream) {
  EGN_REQUIRE(dv >= 1 && du >= 1, "graph MLP dims must be positive");
  EGN_REQUIRE(num_graphs < 65536, "graph MLP: at most 65535 graphs per batch");
  EGN_REQUIRE(w1 != nullptr || dv == du, "graph MLP: identity first layer needs dv == du");
  if (num_graphs == 0) return 0;
  cudaStream_t st = as_stream(stream);
  const dim3 grid(static_cast<unsigned>(num_graphs), (du + 7) / 8);
  gmlp::fwd1_kernel<<<grid, 256, 0, st>>>(dv, du, s, w1, b1, pre, act);
  if (check_launch("graph_mlp_fwd1")) return 1;
  gmlp::fwd2_kernel<<<grid, 256, 0, st>>>(du, act, w2, b2, u);
  return check_launch("graph_mlp_fwd2");
}

extern "C" int egn_graph_mlp_bwd(int64_t num_graphs, int dv, int du, const float* u_bar, const float* s,
                                 const float* pre, const float* act, const float* w1, const float* w2,
                                 float* pre_bar, float* s_bar, float* w1_bar, float* b1_bar, float* w2_bar,
                                 float* b2_bar, egn_stream_t stream) {
  EGN_REQUIRE(dv >= 1 && du >= 1, "graph MLP dims must be positive");
  EGN_REQUIRE(num_graphs < 65536, "graph MLP: at most 65535 graphs per batch");
  cudaStream_t st = as_stream(stream);
  if (num_graphs > 0) {
    gmlp::bwd2_kernel<<<dim3(static_cast<unsigned>(num_graphs), (du + 7) / 8), 256, 0, st>>>(du, u_bar, pre, w2,
                                                                                              pre_bar);
    if (check_launch("graph_mlp_bwd2")) return 1;
    gmlp::bwd1_kernel<<<dim3(static_cast<unsigned>(num_graphs), (dv + 7) / 8), 256, 0, st>>>(dv, du, pre_bar, w1,
                                                                                              s_bar);
    if (check_launch("graph_mlp_bwd1")) return 1;
  }
  gmlp::bwd_weights_kernel<<<dim3(du, 2), 256, 0, st>>>(num_graphs, dv, du, u_bar, act, pre_bar, s, w1_bar, b1_bar,
                                                         w2_bar, b2_bar);
  return check_launch("graph_mlp_bwd_weights");
}

// z = x W^T (+ b) over G rows (the GU head of the graph-parallel reference schedule,
// egn/engine.py:207-211: z = (sum of own v) W1^T, all-reduced before the tail).
extern "C" int egn_graph_linear(int64_t num_graphs, int din, int dout, const float* x, const float* w,
                                const float* b, float* y, egn_stream_t stream) {
  EGN_REQUIRE(din >= 1 && dout >= 1, "graph linear dims must be positive");
  EGN_REQUIRE(num_graphs < 65536, "graph linear: at most 65535 graphs per batch");
  EGN_REQUIRE(w != nullptr || din == dout, "graph linear: identity needs din == dout");
  if (num_graphs == 0) return 0;
  const dim3 grid(static_cast<unsigned>(num_graphs), (dout + 7) / 8);
  gmlp::fwd1_kernel<<<grid, 256, 0, as_stream(stream)>>>(din, dout, x, w, b, y, nullptr);
  return check_launch("graph_linear");
}

// Adjoint of egn_graph_linear: x_bar = y_bar W, w_bar = y_bar^T x, b_bar = column sums of
// y_bar (each output optional, graphs summed in order).
extern "C" int egn_graph_linear_bwd(int64_t num_graphs, int din, int dout, const float* y_bar, const float* x,
                                    const float* w, float* x_bar, float* w_bar, float* b_bar, egn_stream_t stream) {
  EGN_REQUIRE(din >= 1 && dout >= 1, "graph linear dims must be positive");
  EGN_REQUIRE(num_graphs < 65536, "graph linear: at most 65535 graphs per batch");
  cudaStream_t st = as_stream(stream);
  if (x_bar && num_graphs > 0) {
    gmlp::bwd1_kernel<<<dim3(static_cast<unsigned>(num_graphs), (din + 7) / 8), 256, 0, st>>>(din, dout, y_bar, w,
                                                                                               x_bar);
    if (check_launch("graph_linear_bwd_x")) return 1;
  }
  if (w_bar || b_bar) {
    gmlp::bwd_weights_kernel<<<dim3(dout, 2), 256, 0, st>>>(num_graphs, din, dout, nullptr, nullptr, y_bar, x, w_bar,
                                                            b_bar, nullptr, nullptr);
    return check_launch("graph_linear_bwd_w");
  }
  return 0;
}
