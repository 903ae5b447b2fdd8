// Linear-in-degree triplet interaction: the angular sum factorised with the spherical-harmonic
// addition theorem (checked in fp64 by tools/sh_triplet_check.py).
//
// Per centre j with out-edges p, q (unit vectors u, distances d) the reference's triplet sum
// (egn/engine.py:136-148 with cos(l alpha) = T_l(u_p . u_q), the same algebra as triplet.cu)
//     S[p, c] = sum_{q != p} sum_l T_l(u_p . u_q) Q[q, l, c],   Q[q, l, c] = X[rq, c] sum_k rbf_k(d_q) W[k, l, c]
// costs O(n^2 L) per centre.  With T_l = sum_j a_lj P_j (Chebyshev in the Legendre basis, exact
// rationals below) and P_j(u_p . u_q) = 4 pi / (2j+1) sum_m Y_jm(u_p) Y_jm(u_q):
//     W'[k, j, c]  = sum_l W[k, l, c] A[l][j],          A[l][j] = a_lj 4 pi / (2j+1)
//     Q'[q, j, c]  = X[rq, c] sum_k rbf_k(d_q) W'[k, j, c]
//     M[jm, c]     = sum_q Y_jm(u_q) Q'[q, j, c]                       (L^2 = 49 moments)
//     S[p, c]      = sum_jm Y_jm(u_p) M[jm, c] - sum_j s_j Q'[p, j, c],  s_j = (2j+1) / (4 pi)
// (the last term removes q = p, where T_l(1) = 1): O(n L^2) per centre.  At deg 500 (C5) that is
// ~36x fewer FMAs than the pairwise form, and the kernels become bound by the X gather.
//
// Backward (S_bar given), per centre:
//     Mbar[jm, c]   = sum_p Y_jm(u_p) S_bar[p, c]
//     Q'bar[e, j, c] = sum_m Y_jm(u_e) Mbar[jm, c] - s_j S_bar[e, c]
//     X_bar[re, c]  = sum_j Q'bar R'_j,  R'bar = Q'bar X[re, c] -> W'_bar, dE/dd_e (rbf')
//     dE/du_e       = sum_jm grad Y_jm(u_e) P[e, jm],  P[e, jm] = sum_c (S_bar[e, c] M[jm, c] + Mbar[jm, c] Q'[e, j, c])
// and dE/dv_e = (I - u u^T) dE/du_e / d_e.  W_bar[k, l, c] = sum_j A[l][j] W'_bar[k, j, c].
//
// Mapping: one warp per (centre, 32-channel block), lane = channel; 4 independent warps per CTA
// (no block-level barriers).  Edges go in tiles of 32: lane t evaluates Y(u_t) (49 values)
// into the warp's shared tile, then every lane sweeps the tile (broadcast reads).  Sums over
// channels (P, dE/dd) are warp butterflies.  Everything is fixed-order: deterministic.
#include <algorithm>

#include "common.cuh"

namespace egn {
namespace sh {

constexpr int kW = 4;     // warps per CTA
constexpr int kTile = 32;  // edges per tile
constexpr float kPi = 3.14159265358979323846f;

// a_lj: T_l = sum_j a_lj P_j (l, j < 8), exact rationals
__host__ __device__ constexpr double cheb_leg(int l, int j) {
  constexpr double a[8][8] = {
      {1, 0, 0, 0, 0, 0, 0, 0},
      {0, 1, 0, 0, 0, 0, 0, 0},
      {-1.0 / 3, 0, 4.0 / 3, 0, 0, 0, 0, 0},
      {0, -3.0 / 5, 0, 8.0 / 5, 0, 0, 0, 0},
      {-1.0 / 15, 0, -16.0 / 21, 0, 64.0 / 35, 0, 0, 0},
      {0, -1.0 / 7, 0, -8.0 / 9, 0, 128.0 / 63, 0, 0},
      {-1.0 / 35, 0, -4.0 / 21, 0, -384.0 / 385, 0, 512.0 / 231, 0},
      {0, -1.0 / 15, 0, -112.0 / 495, 0, -128.0 / 117, 0, 1024.0 / 429}};
  return a[l][j];
}

__host__ __device__ constexpr double factd(int n) { return n <= 1 ? 1.0 : n * factd(n - 1); }
__host__ __device__ constexpr double dfact(int n) { return n <= 1 ? 1.0 : n * dfact(n - 2); }  // (2m-1)!!
__host__ __device__ constexpr double csqrt(double x) {
  double g = x > 1 ? x : 1.0;
  for (int i = 0; i < 60; ++i) g = 0.5 * (g + x / g);
  return x <= 0 ? 0.0 : g;
}

// Every constant the kernels need, evaluated by the compiler and placed in constant memory
// (indices are compile-time after unrolling, so they become constant-bank operands).
struct ShTables {
  float norm[8][8];  // orthonormal real-harmonic normalisation (sqrt 2 for m > 0)
  float qmm[8];      // Q_m^m = (2m-1)!!
  float A[8][8];     // A[l][j] = a_lj 4 pi / (2j+1): W' = W A (Chebyshev angular basis, MODE 0)
  float Ad[8];       // sqrt(4 pi / (2j+1)): W' = W diag(Ad) for the Y_l0 angular bases (MODE 1, 2)
  float s[8];        // (2j+1) / (4 pi): the q = p (self) term
};
constexpr ShTables make_tables() {
  ShTables t{};
  const double pi = 3.14159265358979323846;
  for (int j = 0; j < 8; ++j) {
    for (int m = 0; m < 8; ++m)
      t.norm[j][m] = m > j ? 0.f
                           : static_cast<float>(csqrt((2 * j + 1) / (4 * pi) * factd(j - m) / factd(j + m)) *
                                                (m > 0 ? 1.4142135623730950488 : 1.0));
    t.qmm[j] = static_cast<float>(dfact(2 * j - 1));
    t.s[j] = static_cast<float>((2 * j + 1) / (4 * pi));
    t.Ad[j] = static_cast<float>(csqrt(4 * pi / (2 * j + 1)));
    for (int l = 0; l < 8; ++l) t.A[l][j] = static_cast<float>(cheb_leg(l, j) * 4 * pi / (2 * j + 1));
  }
  return t;
}
__constant__ ShTables c_tab = make_tables();

// DimeNet SBF radial constants: z[l][n] = n-th positive zero of j_l, jinv = 1 / |j_{l+1}(z_ln)|
// (scipy brentq / spherical_jn; the oracle recomputes them independently)
struct SbfTables {
  double z[8][8];
  double jinv[8][8];
};
__constant__ SbfTables c_sbf = {
    {{3.141592653589793, 6.283185307179586, 9.42477796076938, 12.566370614359172, 15.707963267948966,
      18.849555921538762, 21.991148575128555, 25.132741228718345},
     {4.493409457909064, 7.725251836937707, 10.904121659428899, 14.066193912831473, 17.22075527193077,
      20.37130295928756, 23.519452498689006, 26.666054258812675},
     {5.76345919689455, 9.095011330476355, 12.322940970566583, 15.514603010886745, 18.689036355362823,
      21.853874222709766, 25.01280320228961, 28.167829707993622},
     {6.98793200050052, 10.417118547379365, 13.69802315324925, 16.92362128521384, 20.12180617445382,
      23.304246988939653, 26.476763664539124, 29.64260454031581},
     {8.182561452571242, 11.70490715457039, 15.03966470761652, 18.30125595954199, 21.525417733399944,
      24.727565547835034, 27.91557619942136, 31.093933214079307},
     {9.355812111042747, 12.966530172774345, 16.354709639350464, 19.653152101821185, 22.904550647903722,
      26.1277501372255, 29.332562578584827, 32.52466128857884},
     {10.512835408093999, 14.20739245884246, 17.647974870165896, 20.98346306894477, 24.26276804239701,
      27.507868364904258, 30.730380731646648, 33.9371083026413},
     {11.657032192516372, 15.431289210268378, 18.922999198546144, 22.29534801913077, 25.602855953810646,
      28.87037334704266, 32.1111962396826, 35.33319418271646}},
    {{3.141592653589793, 6.283185307179586, 9.42477796076938, 12.566370614359172, 15.707963267948966,
      18.849555921538762, 21.99114857512856, 25.132741228718345},
     {4.6033388487517, 7.789705767492723, 10.949879869826262, 14.10169533046921, 17.249765567558637,
      20.395832521843232, 23.540701897736362, 26.684798101802116},
     {6.040563197807522, 9.264342010446368, 12.446450951060557, 15.612184250673817, 18.76981212423012,
      21.92283428496274, 25.072987642052208, 28.221232674395463},
     {7.473091442496642, 10.721480766798642, 13.924153665362708, 17.10464317933209, 20.273125026195952,
      23.4344095314491, 26.591044813337703, 29.74450383351637},
     {8.908348935043326, 12.168747439919386, 15.388960028983778, 18.583685450027534, 21.763327322052017,
      24.933462345803836, 28.097246277145015, 31.256583482961755},
     {10.349655802515409, 13.610632122380693, 16.844809840109313, 20.05257889487107, 23.243116533114033,
      26.422236707117232, 29.593479081880883, 32.759076284270435},
     {11.798613629858298, 15.049969257269414, 18.294429523463386, 21.51371922159807, 24.714553484382066,
      27.902501464341643, 31.081267919249978, 34.25330499504689},
     {13.256000990958375, 16.488637691421197, 19.739775744045733, 22.968911668054954, 26.17924648704294,
      29.375674765038404, 32.5618617752044, 35.74037246851164}}};

// spherical Bessel j_l(x) (fp64): ascending series for x <= l + 1 (upward recurrence loses
// digits there), upward recurrence from j_0, j_1 above
__device__ __forceinline__ double sph_jl(int l, double x) {
  if (x <= l + 1.0) {
    double term = 1.0;
    for (int i = 1; i <= l; ++i) term *= x / (2 * i + 1);
    double sum = term;
    const double h = -0.5 * x * x;
    for (int k = 1; k < 40; ++k) {
      term *= h / (k * (2.0 * l + 2.0 * k + 1.0));
      sum += term;
      if (fabs(term) < 1e-17 * fabs(sum)) break;
    }
    return sum;
  }
  double sn, cs;
  sincos(x, &sn, &cs);
  const double j0 = sn / x;
  if (l == 0) return j0;
  double jm = j0, jc = sn / (x * x) - cs / x;
  for (int i = 1; i < l; ++i) {
    const double jn = (2 * i + 1) / x * jc - jm;
    jm = jc;
    jc = jn;
  }
  return jc;
}

// DimeNet / GemNet polynomial envelope u(x) = 1/x + a x^(p-1) + b x^p + c x^(p+1), p = 6, and u'
__device__ __forceinline__ void envelope6(double x, double& u, double& du) {
  constexpr double a = -28.0, b = 48.0, c = -21.0;  // -(p+1)(p+2)/2, p(p+2), -p(p+1)/2
  if (x >= 1.0) {
    u = du = 0.0;
    return;
  }
  const double x2 = x * x, x4 = x2 * x2, x5 = x4 * x, x6 = x5 * x;
  u = 1.0 / x + a * x5 + b * x6 + c * x6 * x;
  du = -1.0 / x2 + 5.0 * a * x4 + 6.0 * b * x5 + 7.0 * c * x6;
}

// Radial table of one edge (distance d) for the basis MODE, row layout radv<MODE> below:
//   MODE 0: Gaussian rbf_k(d) (the reference's surrogate, egn/basis.py:35-42); derivative on the fly
//   MODE 1: GemNet / DimeNet radial Bessel basis sqrt(2/c) u(d/c) sin(n pi d/c), n = k + 1, and d/dd
//   MODE 2: DimeNet SBF radial sqrt(2/c^3) / |j_{l+1}(z_ln)| u(d/c) j_l(z_ln d/c) [k][l], and d/dd
template <int K, int L, int MODE>
__device__ __forceinline__ void radial_row(float d, float cutoff, RbfParams rp, float* row, float* drow) {
  if constexpr (MODE == 0) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float dd = d - rp.step * k;
      row[k] = k < K ? __expf(-rp.gamma * dd * dd) : 0.f;
    }
  } else if constexpr (MODE == 1) {
    const double c = cutoff, x = d / c, nrm = sqrt(2.0 / c);
    double u, du;
    envelope6(x, u, du);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k < K) {
        double sn, cs;
        sincospi((k + 1) * x, &sn, &cs);
        row[k] = static_cast<float>(nrm * u * sn);
        if (drow) drow[k] = static_cast<float>(nrm * (du * sn + u * (k + 1) * 3.14159265358979323846 * cs) / c);
      } else {
        row[k] = 0.f;
        if (drow) drow[k] = 0.f;
      }
    }
  } else {
    const double c = cutoff, x = d / c, nrm = sqrt(2.0 / (c * c * c));
    double u, du;
    envelope6(x, u, du);
    for (int l = 0; l < L; ++l) {
      for (int k = 0; k < K; ++k) {
        const double z = c_sbf.z[l][k], zx = z * x;
        const double j = sph_jl(l, zx);
        // j_l'(t) = j_{l-1}(t) - (l + 1) j_l(t) / t ; j_0' = -j_1
        const double dj = l == 0 ? -sph_jl(1, zx) : sph_jl(l - 1, zx) - (l + 1) * j / zx;
        const double f = nrm * c_sbf.jinv[l][k];
        row[k * L + l] = static_cast<float>(f * u * j);
        if (drow) drow[k * L + l] = static_cast<float>(f * (du * j + u * dj * z) / c);
      }
    }
  }
}
template <int MODE>
constexpr int rad_stride() { return MODE == 2 ? 44 : 8; }
template <int K, int L, int MODE>
__device__ __forceinline__ float radv(const float* row, int k, int j) {
  if constexpr (MODE == 2) return row[k * L + j];
  return row[k];
}

// j_l(x) and j_l'(x) in fp32 (table entries only; the oracle's fp64 values are matched to
// ~1e-6 relative): ascending series for x <= l + 1 (where the upward recurrence loses digits),
// else the upward recurrence from j_0, j_1, which also gives j_{l-1} for the derivative
// j_l' = j_{l-1} - (l + 1) j_l / x  (j_0' = -j_1).
__device__ __forceinline__ float sph_series(int l, float x) {
  float term = 1.f;
  for (int i = 1; i <= l; ++i) term *= x / (2 * i + 1);
  float sum = term;
  const float h = -0.5f * x * x;
  // x <= l + 1 <= 8: 18 terms reach fp32 round-off for every l < 8
#pragma unroll
  for (int k = 1; k <= 18; ++k) {
    term *= __fdividef(h, k * (2.f * l + 2.f * k + 1.f));
    sum += term;
  }
  return sum;
}
__device__ __forceinline__ void sph_jl_pair(int l, float x, float& j, float& dj) {
  if (x <= l + 1.f) {
    j = sph_series(l, x);
    dj = l == 0 ? -sph_series(1, x) : sph_series(l - 1, x) - (l + 1) * j / x;
    return;
  }
  float sn, cs;
  sincosf(x, &sn, &cs);
  const float inv = 1.f / x;
  float jm = sn * inv, jc = (sn * inv - cs) * inv;  // j_0, j_1
  if (l == 0) {
    j = jm;
    dj = -jc;
    return;
  }
  for (int i = 1; i < l; ++i) {
    const float jn = (2 * i + 1) * inv * jc - jm;
    jm = jc;
    jc = jn;
  }
  j = jc;
  dj = jm - (l + 1) * jc * inv;
}

// Element i of an edge's radial row (MODE 1 / 2, layout of radial_row) and its d-derivative.
// The Bessel rows depend on the geometry only, so for MODE 1 / 2 they are tabulated once per
// call by radial_table_kernel (one thread per element) and the triplet kernels copy rows from
// the table instead of evaluating the Bessel functions per lane.
template <int K, int L, int MODE>
__device__ __forceinline__ void radial_elem(float d, float cutoff, int i, float& v, float& dv) {
  const float x = d / cutoff;
  double ud, dud;
  envelope6(x, ud, dud);
  const float u = static_cast<float>(ud), du = static_cast<float>(dud);
  v = dv = 0.f;
  if constexpr (MODE == 1) {
    if (i >= K) return;
    const float nrm = sqrtf(2.f / cutoff);
    float sn, cs;
    sincospif((i + 1) * x, &sn, &cs);
    v = nrm * u * sn;
    dv = nrm * (du * sn + u * (i + 1) * 3.14159265358979323846f * cs) / cutoff;
  } else {
    if (i >= K * L) return;
    const int k = i / L, l = i - k * L;
    const float z = static_cast<float>(c_sbf.z[l][k]);
    float j, dj;
    sph_jl_pair(l, z * x, j, dj);
    const float f = static_cast<float>(sqrt(2.0 / (static_cast<double>(cutoff) * cutoff * cutoff)) * c_sbf.jinv[l][k]);
    v = f * u * j;
    dv = f * (du * j + u * dj * z) / cutoff;
  }
}

template <int K, int L, int MODE>
__global__ void __launch_bounds__(256) radial_table_kernel(const float4* __restrict__ geo, int64_t ne, float cutoff,
                                                           float* __restrict__ tab, float* __restrict__ dtab) {
  constexpr int RS = rad_stride<MODE>();
  const int64_t n = ne * RS;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < n;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = idx / RS;
    const int i = static_cast<int>(idx - e * RS);
    float v, dv;
    radial_elem<K, L, MODE>(geo[e].w, cutoff, i, v, dv);
    tab[idx] = v;
    if (dtab) dtab[idx] = dv;
  }
}

// row i of a tabulated radial table into shared memory (RS floats, 16-byte aligned rows)
template <int MODE>
__device__ __forceinline__ void copy_row(const float* __restrict__ tab, int64_t e, float* row) {
  constexpr int RS = rad_stride<MODE>();
  const float4* src = reinterpret_cast<const float4*>(tab + e * RS);
#pragma unroll
  for (int i = 0; i < RS / 4; ++i) reinterpret_cast<float4*>(row)[i] = __ldg(src + i);
}

// Y_jm(u) for j < L at index j*j + j + m (m in [-j, j]), written with stride `st`.
// Recurrences: C_m + i S_m = (x + i y)^m; Q_j^m(z) = associated Legendre without (1-z^2)^(m/2).
template <int L>
__device__ __forceinline__ void sh_eval(float x, float y, float z, float* out, int st) {
  float C[L], S[L];
  C[0] = 1.f;
  S[0] = 0.f;
#pragma unroll
  for (int m = 1; m < L; ++m) {
    C[m] = x * C[m - 1] - y * S[m - 1];
    S[m] = x * S[m - 1] + y * C[m - 1];
  }
#pragma unroll
  for (int m = 0; m < L; ++m) {
    float q2 = 0.f, q1 = c_tab.qmm[m];
#pragma unroll
    for (int j = m; j < L; ++j) {
      float q;
      if (j == m) {
        q = q1;
      } else if (j == m + 1) {
        q = static_cast<float>(2 * m + 1) * z * q1;
        q2 = q1;
        q1 = q;
      } else {
        q = (static_cast<float>(2 * j - 1) * z * q1 - static_cast<float>(j + m - 1) * q2) *
            static_cast<float>(1.0 / (j - m));
        q2 = q1;
        q1 = q;
      }
      const float nq = c_tab.norm[j][m] * q;
      if (m == 0) {
        out[(j * j + j) * st] = nq;
      } else {
        out[(j * j + j + m) * st] = nq * C[m];
        out[(j * j + j - m) * st] = nq * S[m];
      }
    }
  }
}

// g = sum_jm P[jm] grad Y_jm(u) (Cartesian gradient of the recurrence polynomials; only its
// tangential part is used, where it equals the spherical gradient).
template <int L>
__device__ __forceinline__ float3 sh_grad(float x, float y, float z, const float* P, int st) {
  float C[L], S[L];
  C[0] = 1.f;
  S[0] = 0.f;
#pragma unroll
  for (int m = 1; m < L; ++m) {
    C[m] = x * C[m - 1] - y * S[m - 1];
    S[m] = x * S[m - 1] + y * C[m - 1];
  }
  float gx = 0.f, gy = 0.f, gz = 0.f;
#pragma unroll
  for (int m = 0; m < L; ++m) {
    float q2 = 0.f, q1 = c_tab.qmm[m], d2 = 0.f, d1 = 0.f;
#pragma unroll
    for (int j = m; j < L; ++j) {
      float q, dq;
      if (j == m) {
        q = q1;
        dq = 0.f;
      } else if (j == m + 1) {
        q = static_cast<float>(2 * m + 1) * z * q1;
        dq = static_cast<float>(2 * m + 1) * (q1 + z * d1);
        q2 = q1;
        q1 = q;
        d2 = d1;
        d1 = dq;
      } else {
        const float inv = static_cast<float>(1.0 / (j - m));
        q = (static_cast<float>(2 * j - 1) * z * q1 - static_cast<float>(j + m - 1) * q2) * inv;
        dq = (static_cast<float>(2 * j - 1) * (q1 + z * d1) - static_cast<float>(j + m - 1) * d2) * inv;
        q2 = q1;
        q1 = q;
        d2 = d1;
        d1 = dq;
      }
      const float nrm = c_tab.norm[j][m];
      if (m == 0) {
        gz = fmaf(P[(j * j + j) * st], nrm * dq, gz);
      } else {
        const float pc = P[(j * j + j + m) * st] * nrm, ps = P[(j * j + j - m) * st] * nrm;
        const float fm = static_cast<float>(m);
        // d/dx (x+iy)^m = m (x+iy)^(m-1), d/dy = i m (x+iy)^(m-1)
        gx = fmaf(pc, q * fm * C[m - 1], fmaf(ps, q * fm * S[m - 1], gx));
        gy = fmaf(pc, -q * fm * S[m - 1], fmaf(ps, q * fm * C[m - 1], gy));
        gz = fmaf(pc, dq * C[m], fmaf(ps, dq * S[m], gz));
      }
    }
  }
  return make_float3(gx, gy, gz);
}

// grad Y_jm(u) (Cartesian gradient of the recurrence polynomials) for j < L, written as
// out[3 (j*j + j + m) + d], d = x, y, z
template <int L>
__device__ __forceinline__ void sh_grad_table(float x, float y, float z, float* out) {
  float C[L], S[L];
  C[0] = 1.f;
  S[0] = 0.f;
#pragma unroll
  for (int m = 1; m < L; ++m) {
    C[m] = x * C[m - 1] - y * S[m - 1];
    S[m] = x * S[m - 1] + y * C[m - 1];
  }
#pragma unroll
  for (int m = 0; m < L; ++m) {
    float q2 = 0.f, q1 = c_tab.qmm[m], d2 = 0.f, d1 = 0.f;
#pragma unroll
    for (int j = m; j < L; ++j) {
      float q, dq;
      if (j == m) {
        q = q1;
        dq = 0.f;
      } else if (j == m + 1) {
        q = static_cast<float>(2 * m + 1) * z * q1;
        dq = static_cast<float>(2 * m + 1) * (q1 + z * d1);
        q2 = q1;
        q1 = q;
        d2 = d1;
        d1 = dq;
      } else {
        const float inv = static_cast<float>(1.0 / (j - m));
        q = (static_cast<float>(2 * j - 1) * z * q1 - static_cast<float>(j + m - 1) * q2) * inv;
        dq = (static_cast<float>(2 * j - 1) * (q1 + z * d1) - static_cast<float>(j + m - 1) * d2) * inv;
        q2 = q1;
        q1 = q;
        d2 = d1;
        d1 = dq;
      }
      const float nrm = c_tab.norm[j][m];
      if (m == 0) {
        float* o = out + 3 * (j * j + j);
        o[0] = 0.f;
        o[1] = 0.f;
        o[2] = nrm * dq;
      } else {
        const float fm = static_cast<float>(m), nq = nrm * q * fm;
        float* oc = out + 3 * (j * j + j + m);
        oc[0] = nq * C[m - 1];
        oc[1] = -nq * S[m - 1];
        oc[2] = nrm * dq * C[m];
        float* os = out + 3 * (j * j + j - m);
        os[0] = nq * S[m - 1];
        os[1] = nq * C[m - 1];
        os[2] = nrm * dq * S[m];
      }
    }
  }
}

__device__ __forceinline__ float rbf1(float d, int k, RbfParams rp) {
  const float dd = d - rp.step * k;
  return __expf(-rp.gamma * dd * dd);
}

// W'[k][j] = sum_l W[k, l, c] A[l][j] for this lane's channel (MODE 1/2: A = diag(Ad))
template <int K, int L, int MODE = 0>
__device__ __forceinline__ void load_wprime(float (&wp)[K][L], const float* __restrict__ W, int dg, int c, bool cok) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    float w[L];
#pragma unroll
    for (int l = 0; l < L; ++l) w[l] = cok ? __ldg(W + (k * L + l) * dg + c) : 0.f;
#pragma unroll
    for (int j = 0; j < L; ++j) {
      if constexpr (MODE == 0) {
        float s = 0.f;
#pragma unroll
        for (int l = j; l < L; l += 2) s = fmaf(w[l], c_tab.A[l][j], s);  // a_lj = 0 unless l >= j, l - j even
        wp[k][j] = s;
      } else {
        wp[k][j] = w[j] * c_tab.Ad[j];
      }
    }
  }
}

template <int L>
__device__ __forceinline__ constexpr int jof(int jm) {
  int j = 0;
  while ((j + 1) * (j + 1) <= jm) ++j;
  return j;
}

// warp shared-memory carve-up (floats).  The Y tile is edge-major with a 16-byte aligned row
// (52 floats), so a lane reads four harmonics of one edge with one broadcast LDS.128.
constexpr int kYS = 52;
template <int K, int L, int T = kTile, int MODE = 0>
struct WarpSmem {
  static constexpr int J = L * L;
  static_assert(J <= kYS, "L <= 7 for the 52-float Y rows");
  static constexpr int ys = 0;                        // Y tile [T][kYS]
  static constexpr int rs = ys + T * kYS;             // radial tile [T][rad_stride]
  static constexpr int us = rs + T * rad_stride<MODE>();  // float4 (u, d) [T]
  static constexpr int rq = us + 4 * T;               // int rq [T]
  static constexpr int xs = rq + T;                   // X[rq_t, c] of the tile [T t][32 lanes]
  static constexpr int sbs = xs + T * 32;             // S_bar[e_t, c] of the tile (backward)
  static constexpr int ms = sbs + T * 32;             // M [J][32] (backward, lane columns)
  static constexpr int pt = ms + J * 32;              // P tile [J + 1][T] (backward)
  static constexpr int fwd_total = ms;
  static constexpr int bwd_total = pt + (J + 1) * T;
};

// stage the tile [t0, t0 + 32) of the centre's out-edges: Y, rbf, (u, d), rev, and this lane's
// channel of the gathered X rows (and of S_bar for the backward): all 32 row loads of the tile
// are issued back to back, so the sweep over the tile never waits on a dependent global load.
template <int K, int L, int T = kTile, int MODE = 0>
__device__ __forceinline__ void stage_tile(float* wsm, const float4* __restrict__ geo, const int32_t* __restrict__ rev,
                                           int64_t off, int t0, int n, RbfParams rp, float cutoff, int lane,
                                           const float* __restrict__ X = nullptr, const float* __restrict__ Sbar = nullptr,
                                           int dg = 0, int c = 0, bool cok = false, bool radial = true,
                                           const float* __restrict__ rtab = nullptr) {
  using SM = WarpSmem<K, L, T, MODE>;
  const int e = t0 + lane;
  int32_t rq = 0;
  if (lane < T && e < n) {
    const float4 g = geo[off + e];
    rq = rev[off + e];
    reinterpret_cast<float4*>(wsm + SM::us)[lane] = g;
    reinterpret_cast<int32_t*>(wsm + SM::rq)[lane] = rq;
    sh_eval<L>(g.x, g.y, g.z, wsm + SM::ys + lane * kYS, 1);
    if (radial) {  // MODE 1 / 2: rows of the per-call radial table (host guarantees rtab)
      if constexpr (MODE != 0) copy_row<MODE>(rtab, off + e, wsm + SM::rs + lane * rad_stride<MODE>());
      else radial_row<K, L, MODE>(g.w, cutoff, rp, wsm + SM::rs + lane * rad_stride<MODE>(), nullptr);
    }
  }
  const int nt = min(T, n - t0);
  if (X) {
    float xv[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int64_t r = __shfl_sync(0xffffffffu, rq, t);
      xv[t] = (t < nt && cok) ? __ldg(X + r * dg + c) : 0.f;
    }
#pragma unroll
    for (int t = 0; t < T; ++t) wsm[SM::xs + t * 32 + lane] = xv[t];
  }
  if (Sbar) {
    float sv[T];
#pragma unroll
    for (int t = 0; t < T; ++t) sv[t] = (t < nt && cok) ? __ldg(Sbar + (off + t0 + t) * dg + c) : 0.f;
#pragma unroll
    for (int t = 0; t < T; ++t) wsm[SM::sbs + t * 32 + lane] = sv[t];
  }
  __syncwarp();
}

// the harmonics / radial values of tile edge t as registers (broadcast vector loads)
template <int J>
__device__ __forceinline__ void load_y(const float* ys_row, float (&y)[J]) {
#pragma unroll
  for (int i = 0; i < J; i += 4) {
    const float4 v = *reinterpret_cast<const float4*>(ys_row + i);
    y[i] = v.x;
    if (i + 1 < J) y[i + 1] = v.y;
    if (i + 2 < J) y[i + 2] = v.z;
    if (i + 3 < J) y[i + 3] = v.w;
  }
}
template <int K>
__device__ __forceinline__ void load_rb(const float* rs_row, float (&rb)[K]) {
  const float4 a = *reinterpret_cast<const float4*>(rs_row);
  const float4 b = *reinterpret_cast<const float4*>(rs_row + 4);
  const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int k = 0; k < K; ++k) rb[k] = v[k];
}

// R'_j = sum_k rbf_k W'[k, j]
template <int K, int L>
__device__ __forceinline__ void rprime(const float (&rb)[K], const float (&wp)[K][L], float (&r)[L]) {
#pragma unroll
  for (int jj = 0; jj < L; ++jj) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) s = fmaf(rb[k], wp[k][jj], s);
    r[jj] = s;
  }
}

// R'_j of one staged edge row (any MODE)
template <int K, int L, int MODE>
__device__ __forceinline__ void rprime_row(const float* row, const float (&wp)[K][L], float (&r)[L]) {
  if constexpr (MODE == 2) {
#pragma unroll
    for (int jj = 0; jj < L; ++jj) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < K; ++k) s = fmaf(row[k * L + jj], wp[k][jj], s);
      r[jj] = s;
    }
  } else {
    float rb[K];
    load_rb<K>(row, rb);
    rprime<K, L>(rb, wp, r);
  }
}

template <int L>
__device__ __forceinline__ float self_w(int j) {
  return c_tab.s[j];
}

// ---------------------------------------------------------------------------
// work items: (centre j, chunk of kChunk out-edges, 32-channel block).  A centre of degree n
// has ceil(n / kChunk) chunks; items run over nv x nch x ncb (nch from the max degree), so a
// deg-500 centre is spread over 4 warps per channel block instead of one.  The moments of a
// centre are the fixed-order sum of its chunks' partial moments (global, [nv][nch][J][dg]).
// ---------------------------------------------------------------------------
constexpr int kChunk = 4 * kTile;

struct Item {
  int64_t j, off;
  int n, ch, e0, e1, c;
  bool cok, live;
};
__device__ __forceinline__ Item decode(int64_t it, int nch, int ncb, const int64_t* __restrict__ edge_ptr, int dg,
                                       int min_n, int lane) {
  Item x;
  const int64_t jc = it / ncb;
  x.c = static_cast<int>(it - jc * ncb) * 32 + lane;
  x.j = jc / nch;
  x.ch = static_cast<int>(jc - x.j * nch);
  x.off = edge_ptr[x.j];
  x.n = static_cast<int>(edge_ptr[x.j + 1] - x.off);
  x.e0 = x.ch * kChunk;
  x.e1 = min(x.n, x.e0 + kChunk);
  x.cok = x.c < dg;
  x.live = x.n >= 2 && x.n > min_n && x.e0 < x.n;
  return x;
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
// K1: partial moments of the chunk, and S = -self for its edges
template <int K, int L, int MODE>
__global__ void __launch_bounds__(kW * 32, 3)
fwd_moments_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ rev,
                   const float4* __restrict__ geo, int64_t nv, int nch, const float* __restrict__ X,
                   const float* __restrict__ W, int dg, RbfParams rp, float cutoff, float* __restrict__ S,
                   float* __restrict__ Mpart, int min_n, const float* __restrict__ rtab) {
  using SM = WarpSmem<K, L, kTile, MODE>;
  constexpr int RS = rad_stride<MODE>();
  constexpr int J = L * L;
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* wsm = smem + warp * SM::fwd_total;
  const float* Ys = wsm + SM::ys;
  const float* Rs = wsm + SM::rs;
  const float* Xs = wsm + SM::xs;
  const int ncb = (dg + 31) / 32;
  const int64_t items = nv * nch * ncb;
  for (int64_t it = static_cast<int64_t>(blockIdx.x) * kW + warp; it < items;
       it += static_cast<int64_t>(gridDim.x) * kW) {
    const Item q = decode(it, nch, ncb, edge_ptr, dg, min_n, lane);
    if (!q.live) {
      if (q.n == 1 && q.ch == 0 && q.n > min_n && q.cok) S[q.off * dg + q.c] = 0.f;
      continue;
    }
    float wp[K][L];
    load_wprime<K, L, MODE>(wp, W, dg, q.c, q.cok);
    float M[J];
#pragma unroll
    for (int i = 0; i < J; ++i) M[i] = 0.f;
    for (int t0 = q.e0; t0 < q.e1; t0 += kTile) {
      __syncwarp();
      stage_tile<K, L, kTile, MODE>(wsm, geo, rev, q.off, t0, q.e1, rp, cutoff, lane, X, nullptr, dg, q.c, q.cok, true,
                                    rtab);
      const int nt = min(kTile, q.e1 - t0);
#pragma unroll 1
      for (int t = 0; t < nt; ++t) {
        const float x = Xs[t * 32 + lane];
        float r[L], y[J];
        rprime_row<K, L, MODE>(Rs + t * RS, wp, r);
        load_y<J>(Ys + t * kYS, y);
        float self = 0.f;
#pragma unroll
        for (int jj = 0; jj < L; ++jj) {
          r[jj] *= x;  // Q'_j
          self = fmaf(self_w<L>(jj), r[jj], self);
        }
#pragma unroll
        for (int i = 0; i < J; ++i) M[i] = fmaf(y[i], r[jof<L>(i)], M[i]);
        if (q.cok) S[(q.off + t0 + t) * dg + q.c] = -self;
      }
    }
    if (q.cok) {
      float* dst = Mpart + ((q.j * nch + q.ch) * J) * static_cast<int64_t>(dg) + q.c;
#pragma unroll
      for (int i = 0; i < J; ++i) dst[static_cast<int64_t>(i) * dg] = M[i];
    }
  }
}

// moments of centre j for this lane's channel: the fixed-order sum of its chunks' partials
template <int J>
__device__ __forceinline__ void gather_moments(const float* __restrict__ Mpart, int64_t j, int nch, int nchunks,
                                               int dg, int c, float (&M)[J]) {
#pragma unroll
  for (int i = 0; i < J; ++i) M[i] = 0.f;
  for (int ch = 0; ch < nchunks; ++ch) {
    const float* src = Mpart + ((j * nch + ch) * J) * static_cast<int64_t>(dg) + c;
#pragma unroll
    for (int i = 0; i < J; ++i) M[i] += __ldg(src + static_cast<int64_t>(i) * dg);
  }
}

// K2: S = -self + sum_jm Y_jm(u_p) M[jm] for the chunk's edges
template <int K, int L, int MODE>
__global__ void __launch_bounds__(kW * 32, 3)
fwd_apply_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ rev,
                 const float4* __restrict__ geo, int64_t nv, int nch, int dg, RbfParams rp, float* __restrict__ S,
                 const float* __restrict__ Mpart, int min_n) {
  using SM = WarpSmem<K, L, kTile, MODE>;
  constexpr int J = L * L;
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* wsm = smem + warp * SM::fwd_total;
  const float* Ys = wsm + SM::ys;
  const float* Ss = wsm + SM::sbs;
  const int ncb = (dg + 31) / 32;
  const int64_t items = nv * nch * ncb;
  for (int64_t it = static_cast<int64_t>(blockIdx.x) * kW + warp; it < items;
       it += static_cast<int64_t>(gridDim.x) * kW) {
    const Item q = decode(it, nch, ncb, edge_ptr, dg, min_n, lane);
    if (!q.live) continue;
    float M[J];
    gather_moments<J>(Mpart, q.j, nch, (q.n + kChunk - 1) / kChunk, dg, q.cok ? q.c : 0, M);
    for (int t0 = q.e0; t0 < q.e1; t0 += kTile) {
      __syncwarp();
      stage_tile<K, L, kTile, MODE>(wsm, geo, rev, q.off, t0, q.e1, rp, 0.f, lane, nullptr, S, dg, q.c, q.cok,
                                    false);
      const int nt = min(kTile, q.e1 - t0);
#pragma unroll 1
      for (int t = 0; t < nt; ++t) {
        float y[J];
        load_y<J>(Ys + t * kYS, y);
        float a = Ss[t * 32 + lane];
#pragma unroll
        for (int i = 0; i < J; ++i) a = fmaf(y[i], M[i], a);
        if (q.cok) S[(q.off + t0 + t) * dg + q.c] = a;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------
// Sum of v over the 32 lanes for 16 values at once (reduce-scatter butterfly, 16 shuffles):
// afterwards lane pairs (lane, lane ^ 1) hold the total of value index idx16(lane).
__device__ __forceinline__ float reduce16(float (&v)[16], int lane) {
  float a[8];
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float send = hi ? v[i] : v[i + 8];
      const float keep = hi ? v[i + 8] : v[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
  float b[4];
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float send = hi ? a[i] : a[i + 4];
      const float keep = hi ? a[i + 4] : a[i];
      b[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
  }
  float cc[2];
  {
    const bool hi = lane & 4;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float send = hi ? b[i] : b[i + 2];
      const float keep = hi ? b[i + 2] : b[i];
      cc[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
  }
  float d;
  {
    const bool hi = lane & 2;
    const float send = hi ? cc[0] : cc[1];
    const float keep = hi ? cc[1] : cc[0];
    d = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  return d + __shfl_xor_sync(0xffffffffu, d, 1);
}
__device__ __forceinline__ int idx16(int lane) {
  return ((lane & 16) ? 8 : 0) + ((lane & 8) ? 4 : 0) + ((lane & 4) ? 2 : 0) + ((lane & 2) ? 1 : 0);
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// K1: partial moments M (forward) and Mbar = sum_p Y(u_p) S_bar[p] of the chunk
template <int K, int L, int MODE>
__global__ void __launch_bounds__(kW * 32, 3)
bwd_moments_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ rev,
                   const float4* __restrict__ geo, int64_t nv, int nch, const float* __restrict__ X,
                   const float* __restrict__ W, int dg, RbfParams rp, float cutoff, const float* __restrict__ Sbar,
                   float* __restrict__ Mpart, float* __restrict__ Mbpart, int min_n, const float* __restrict__ rtab) {
  using SM = WarpSmem<K, L, kTile, MODE>;
  constexpr int RS = rad_stride<MODE>();
  constexpr int J = L * L;
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* wsm = smem + warp * SM::fwd_total;
  const float* Ys = wsm + SM::ys;
  const float* Rs = wsm + SM::rs;
  const float* Xs = wsm + SM::xs;
  const float* Sbs = wsm + SM::sbs;
  const int ncb = (dg + 31) / 32;
  const int64_t items = nv * nch * ncb;
  for (int64_t it = static_cast<int64_t>(blockIdx.x) * kW + warp; it < items;
       it += static_cast<int64_t>(gridDim.x) * kW) {
    const Item q = decode(it, nch, ncb, edge_ptr, dg, min_n, lane);
    if (!q.live) continue;
    const int64_t base = ((q.j * nch + q.ch) * J) * static_cast<int64_t>(dg) + q.c;
    {
      float wp[K][L];
      load_wprime<K, L, MODE>(wp, W, dg, q.c, q.cok);
      float M[J];
#pragma unroll
      for (int i = 0; i < J; ++i) M[i] = 0.f;
      for (int t0 = q.e0; t0 < q.e1; t0 += kTile) {
        __syncwarp();
        // a single-tile chunk stages S_bar too and keeps the tile for the Mbar sweep
        stage_tile<K, L, kTile, MODE>(wsm, geo, rev, q.off, t0, q.e1, rp, cutoff, lane, X,
                                      q.e1 - q.e0 > kTile ? nullptr : Sbar, dg, q.c, q.cok, true, rtab);
        const int nt = min(kTile, q.e1 - t0);
#pragma unroll 1
        for (int t = 0; t < nt; ++t) {
          const float x = Xs[t * 32 + lane];
          float r[L], y[J];
          rprime_row<K, L, MODE>(Rs + t * RS, wp, r);
          load_y<J>(Ys + t * kYS, y);
#pragma unroll
          for (int jj = 0; jj < L; ++jj) r[jj] *= x;
#pragma unroll
          for (int i = 0; i < J; ++i) M[i] = fmaf(y[i], r[jof<L>(i)], M[i]);
        }
      }
      if (q.cok) {
#pragma unroll
        for (int i = 0; i < J; ++i) Mpart[base + static_cast<int64_t>(i) * dg] = M[i];
      }
    }
    float Mb[J];
#pragma unroll
    for (int i = 0; i < J; ++i) Mb[i] = 0.f;
    for (int t0 = q.e0; t0 < q.e1; t0 += kTile) {
      if (q.e1 - q.e0 > kTile) {  // else the tile is still staged
        __syncwarp();
        stage_tile<K, L, kTile, MODE>(wsm, geo, rev, q.off, t0, q.e1, rp, cutoff, lane, nullptr, Sbar, dg, q.c, q.cok,
                                      false);
      }
      const int nt = min(kTile, q.e1 - t0);
#pragma unroll 1
      for (int t = 0; t < nt; ++t) {
        const float sb = Sbs[t * 32 + lane];
        float y[J];
        load_y<J>(Ys + t * kYS, y);
#pragma unroll
        for (int i = 0; i < J; ++i) Mb[i] = fmaf(y[i], sb, Mb[i]);
      }
    }
    if (q.cok) {
#pragma unroll
      for (int i = 0; i < J; ++i) Mbpart[base + static_cast<int64_t>(i) * dg] = Mb[i];
    }
  }
}

// K2 per chunk, one pass per tile: M -> shared (lane columns), Mbar -> registers; per edge
//   Q'bar -> X_bar, W'_bar (flushed per tile into this warp's partial), dE/dd,
//   g_c = sum_jm grad Y_jm(u_e) (S_bar[e, c] M[jm, c] + Mbar[jm, c] Q'[e, j, c])
// and (g, dE/dd) summed over the 32 channel lanes with one 4-value butterfly (6 shuffles).
// Persistent warps with a fixed channel block (W'_bar partial per warp).
constexpr int kBT = 8;  // backward tile: 8 edges (shared memory for 3 CTAs per SM)
constexpr int kGS = 148;  // grad-Y row: 147 floats, 16-byte aligned
template <int K, int L, int MODE = 0>
struct BwdSmem {
  static constexpr int J = L * L;
  static constexpr int RS = rad_stride<MODE>();
  static constexpr int ys = 0;                  // Y [kBT][kYS]
  static constexpr int gs = ys + kBT * kYS;     // grad Y [kBT][kGS]
  static constexpr int rs = gs + kBT * kGS;     // radial [kBT][RS]
  static constexpr int drs = rs + kBT * RS;     // its d-derivative [kBT][RS] (MODE 1, 2)
  static constexpr int us = drs + (MODE == 0 ? 0 : kBT * RS);  // (u, d) [kBT]
  static constexpr int rq = us + 4 * kBT;       // rev [kBT]
  static constexpr int xs = rq + kBT;           // X tile [kBT][32]
  static constexpr int sbs = xs + kBT * 32;     // S_bar tile [kBT][32]
  static constexpr int ms = sbs + kBT * 32;     // M [J][32]
  static constexpr int total = ms + J * 32;
};

template <int K, int L, int MODE>
__global__ void __launch_bounds__(kW * 32, 2)  // 2 CTAs / SM, 255 registers: no spills (3: 168, spilling, 25% slower at C5)
bwd_apply_kernel(const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ rev,
                 const float4* __restrict__ geo, int64_t nv, int64_t ne, int nch, const float* __restrict__ X,
                 const float* __restrict__ W, int dg, RbfParams rp, float cutoff, const float* __restrict__ Sbar,
                 const float* __restrict__ Mpart, const float* __restrict__ Mbpart, float* __restrict__ Xbar,
                 float* __restrict__ wbar_part, float4* __restrict__ eg_part, float4* __restrict__ edge_grad,
                 int min_n, const float* __restrict__ rtab, const float* __restrict__ drtab) {
  using SM = BwdSmem<K, L, MODE>;
  constexpr int J = L * L;
  constexpr int RS = SM::RS;
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* wsm = smem + warp * SM::total;
  const float* Ys = wsm + SM::ys;
  const float* Gs = wsm + SM::gs;
  const float* Rs = wsm + SM::rs;
  const float* DRs = wsm + SM::drs;
  const float4* Us = reinterpret_cast<const float4*>(wsm + SM::us);
  const int32_t* Rq = reinterpret_cast<const int32_t*>(wsm + SM::rq);
  const float* Xs = wsm + SM::xs;
  const float* Sbs = wsm + SM::sbs;
  float* Ms = wsm + SM::ms;
  const int ncb = (dg + 31) / 32;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kW + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kW;  // multiple of ncb (host)
  const int cb = static_cast<int>(gw % ncb);
  float* wpart = wbar_part + gw * (K * L * 32) + lane;
#pragma unroll
  for (int i = 0; i < K * L; ++i) wpart[i * 32] = 0.f;
  for (int64_t jc = gw / ncb; jc < nv * nch; jc += nw / ncb) {
    const Item q = decode(jc * ncb + cb, nch, ncb, edge_ptr, dg, min_n, lane);
    if (!q.live) {
      if (q.n == 1 && q.ch == 0 && q.n > min_n && q.cok) Xbar[static_cast<int64_t>(rev[q.off]) * dg + q.c] = 0.f;
      continue;
    }
    const int nchunks = (q.n + kChunk - 1) / kChunk;
    {
      float M[J];
      gather_moments<J>(Mpart, q.j, nch, nchunks, dg, q.cok ? q.c : 0, M);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < J; ++i) Ms[i * 32 + lane] = M[i];
    }
    float Mb[J];
    gather_moments<J>(Mbpart, q.j, nch, nchunks, dg, q.cok ? q.c : 0, Mb);
    float wp[K][L];
    load_wprime<K, L, MODE>(wp, W, dg, q.c, q.cok);
    for (int t0 = q.e0; t0 < q.e1; t0 += kBT) {
      __syncwarp();
      // stage: Y, grad Y, rbf, (u, d), rev; X and S_bar tiles
      {
        const int e = t0 + lane;
        int32_t rq = 0;
        if (lane < kBT && e < q.e1) {
          const float4 g = geo[q.off + e];
          rq = rev[q.off + e];
          reinterpret_cast<float4*>(wsm + SM::us)[lane] = g;
          reinterpret_cast<int32_t*>(wsm + SM::rq)[lane] = rq;
          sh_eval<L>(g.x, g.y, g.z, wsm + SM::ys + lane * kYS, 1);
          sh_grad_table<L>(g.x, g.y, g.z, wsm + SM::gs + lane * kGS);
          if constexpr (MODE != 0) {  // per-call radial table (values, d-derivatives)
            copy_row<MODE>(rtab, q.off + e, wsm + SM::rs + lane * RS);
            copy_row<MODE>(drtab, q.off + e, wsm + SM::drs + lane * RS);
          } else {
            radial_row<K, L, MODE>(g.w, cutoff, rp, wsm + SM::rs + lane * RS, nullptr);
          }
        }
        const int nt = min(kBT, q.e1 - t0);
        float xv[kBT], sv[kBT];
#pragma unroll
        for (int t = 0; t < kBT; ++t) {
          const int64_t r = __shfl_sync(0xffffffffu, rq, t);
          xv[t] = (t < nt && q.cok) ? __ldg(X + r * dg + q.c) : 0.f;
          sv[t] = (t < nt && q.cok) ? __ldg(Sbar + (q.off + t0 + t) * dg + q.c) : 0.f;
        }
#pragma unroll
        for (int t = 0; t < kBT; ++t) {
          wsm[SM::xs + t * 32 + lane] = xv[t];
          wsm[SM::sbs + t * 32 + lane] = sv[t];
        }
        __syncwarp();
      }
      const int nt = min(kBT, q.e1 - t0);
      float wpb[K][L];
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int jj = 0; jj < L; ++jj) wpb[k][jj] = 0.f;
#pragma unroll 1
      for (int t = 0; t < nt; ++t) {
        const int64_t rq = Rq[t];
        const float sb = Sbs[t * 32 + lane];
        const float x = Xs[t * 32 + lane];
        const float d = Us[t].w;
        float r[L], qb[L];
        const float* rrow = Rs + t * RS;
        const float* drow = DRs + t * RS;
        float rb[K], drb[K];  // MODE 0 / 1: radial values of the edge
        if constexpr (MODE != 2) {
          load_rb<K>(rrow, rb);
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if constexpr (MODE == 0) drb[k] = -2.f * rp.gamma * (d - rp.step * k) * rb[k];
            else drb[k] = drow[k];
          }
        }
        rprime_row<K, L, MODE>(rrow, wp, r);
#pragma unroll
        for (int jj = 0; jj < L; ++jj) qb[jj] = -self_w<L>(jj) * sb;
        const float* yrow = Ys + t * kYS;
#pragma unroll
        for (int i = 0; i < J; i += 4) {
          const float4 v = *reinterpret_cast<const float4*>(yrow + i);
          const float yy[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (i + u < J) qb[jof<L>(i + u)] = fmaf(yy[u], Mb[i + u], qb[jof<L>(i + u)]);
        }
        float xb = 0.f, dd = 0.f;
#pragma unroll
        for (int jj = 0; jj < L; ++jj) {
          xb = fmaf(qb[jj], r[jj], xb);
          const float rbar = qb[jj] * x;
          float sdr = 0.f;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const float rv = MODE == 2 ? rrow[k * L + jj] : rb[k];
            const float dv = MODE == 2 ? drow[k * L + jj] : drb[k];
            wpb[k][jj] = fmaf(rv, rbar, wpb[k][jj]);
            sdr = fmaf(dv, wp[k][jj], sdr);
          }
          dd = fmaf(rbar, sdr, dd);
          r[jj] *= x;  // Q'_j
        }
        if (q.cok) Xbar[rq * dg + q.c] = xb;
        // g_c = sum_jm grad Y_jm (sb M[jm] + Mbar[jm] Q'_j): two accumulator sets (harmonic
        // parity) halve the 49-long dependent FMA chains
        float gxa[2] = {0.f, 0.f}, gya[2] = {0.f, 0.f}, gza[2] = {0.f, 0.f};
        const float* grow = Gs + t * kGS;
#pragma unroll
        for (int i = 0; i < J; i += 4) {
          // 4 harmonics = 12 gradient components = 3 float4 loads
          const float4 a = *reinterpret_cast<const float4*>(grow + 3 * i);
          const float4 b = *reinterpret_cast<const float4*>(grow + 3 * i + 4);
          const float4 cc = *reinterpret_cast<const float4*>(grow + 3 * i + 8);
          const float gv[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, cc.x, cc.y, cc.z, cc.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int jm = i + u;
            if (jm < J) {
              const float pv = fmaf(sb, Ms[jm * 32 + lane], Mb[jm] * r[jof<L>(jm < J ? jm : 0)]);
              gxa[u & 1] = fmaf(gv[3 * u], pv, gxa[u & 1]);
              gya[u & 1] = fmaf(gv[3 * u + 1], pv, gya[u & 1]);
              gza[u & 1] = fmaf(gv[3 * u + 2], pv, gza[u & 1]);
            }
          }
        }
        const float gx = gxa[0] + gxa[1], gy = gya[0] + gya[1], gz = gza[0] + gza[1];
        // (gx, gy, gz, dd) summed over the lanes: halve twice, then a 3-step butterfly
        {
          const bool h16 = lane & 16;
          const float s0 = h16 ? gx : gz, s1 = h16 ? gy : dd;
          const float k0 = h16 ? gz : gx, k1 = h16 ? dd : gy;
          const float a0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 16);
          const float a1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 16);
          const bool h8 = lane & 8;
          float v = (h8 ? a1 : a0) + __shfl_xor_sync(0xffffffffu, h8 ? a0 : a1, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          // lane (h16, h8) holds component 2 h16 + h8 of (gx, gy, gz, dd)
          if ((lane & 7) == 0) wsm[SM::xs + t * 32 + ((lane >> 3) & 3)] = v;  // X tile row t is consumed
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int jj = 0; jj < L; ++jj) wpart[(k * L + jj) * 32] += wpb[k][jj];
      __syncwarp();
      if (lane < nt) {
        const float4 u = Us[lane];
        const float* gr = wsm + SM::xs + lane * 32;
        const float gxx = gr[0], gyy = gr[1], gzz = gr[2], ddd = gr[3];
        const float gu = gxx * u.x + gyy * u.y + gzz * u.z;
        const float inv = 1.f / u.w;
        const float4 add = make_float4((gxx - gu * u.x) * inv, (gyy - gu * u.y) * inv, (gzz - gu * u.z) * inv, ddd);
        const int64_t e = q.off + t0 + lane;
        if (eg_part) {
          eg_part[static_cast<int64_t>(cb) * ne + e] = add;
        } else {
          float4 gg = edge_grad[e];
          gg.x += add.x;
          gg.y += add.y;
          gg.z += add.z;
          gg.w += add.w;
          edge_grad[e] = gg;
        }
      }
    }
  }
}

// W_bar[k, l, c] = sum_j A[l][j] sum_{warps w of block cb} W'_bar_w[k, j, c]: one CTA per (k, cb),
// 32 warps split the warp partials (strided), then a fixed-order combine: deterministic.
template <int K, int L, int MODE>
__global__ void __launch_bounds__(1024) reduce_wbar_kernel(const float* __restrict__ part, int64_t nw, int ncb, int dg,
                                                            float* __restrict__ out, int accumulate) {
  __shared__ float red[32][L][33];
  const int k = blockIdx.x / ncb, cb = blockIdx.x - (blockIdx.x / ncb) * ncb;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float acc[L];
#pragma unroll
  for (int jj = 0; jj < L; ++jj) acc[jj] = 0.f;
  for (int64_t w = cb + static_cast<int64_t>(wid) * ncb; w < nw; w += static_cast<int64_t>(32) * ncb) {
    const float* src = part + w * (K * L * 32) + (k * L) * 32 + lane;
#pragma unroll
    for (int jj = 0; jj < L; ++jj) acc[jj] += __ldg(src + jj * 32);
  }
#pragma unroll
  for (int jj = 0; jj < L; ++jj) red[wid][jj][lane] = acc[jj];
  __syncthreads();
  if (wid == 0) {
    float wpb[L];
#pragma unroll
    for (int jj = 0; jj < L; ++jj) {
      float t = 0.f;
      for (int u = 0; u < 32; ++u) t += red[u][jj][lane];
      wpb[jj] = t;
    }
    const int c = cb * 32 + lane;
    if (c < dg) {
#pragma unroll
      for (int l = 0; l < L; ++l) {
        float s = 0.f;
        if constexpr (MODE == 0) {
#pragma unroll
          for (int jj = 0; jj <= l && jj < L; ++jj)
            if (((l - jj) & 1) == 0) s = fmaf(wpb[jj], c_tab.A[l][jj], s);
        } else {
          s = wpb[l] * c_tab.Ad[l];
        }
        float* o = out + (static_cast<int64_t>(k) * L + l) * dg + c;
        *o = accumulate ? *o + s : s;
      }
    }
  }
}

// edge_grad[e] += sum over channel blocks (fixed order) for the centres handled here; one warp
// per centre, lanes over its edges
__global__ void add_eg_kernel(const int64_t* __restrict__ edge_ptr, int64_t nv, const float4* __restrict__ part,
                              int ncb, int64_t ne, int min_n, float4* __restrict__ edge_grad) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t v = w0; v < nv; v += nw) {
    const int64_t e0 = edge_ptr[v], e1 = edge_ptr[v + 1];
    if (e1 - e0 < 2 || e1 - e0 <= min_n) continue;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      float4 g = edge_grad[e];
      for (int b = 0; b < ncb; ++b) {
        const float4 p = part[b * ne + e];
        g.x += p.x;
        g.y += p.y;
        g.z += p.z;
        g.w += p.w;
      }
      edge_grad[e] = g;
    }
  }
}

}  // namespace sh

// ---------------------------------------------------------------------------
// host side (called from triplet.cu's ABI functions)
// ---------------------------------------------------------------------------
bool sh_supported(int K, int L, int dg) { return K == 6 && L == 7 && dg >= 1; }

static int sh_nch(int max_degree) { return std::max(1, (std::max(max_degree, 1) + sh::kChunk - 1) / sh::kChunk); }

static int sh_grid(int64_t items) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((items + sh::kW - 1) / sh::kW, kNumSMs * 24)));
}

int64_t sh_fwd_workspace_bytes(int64_t nv, int max_degree, int K, int L, int dg) {
  return std::max<int64_t>(nv, 1) * sh_nch(max_degree) * L * L * static_cast<int64_t>(dg) * 4;
}

template <typename F>
static void set_smem(F kern, size_t smem, bool& configured) {
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured = true;
  }
}

template <int MODE>
static int sh_fwd_mode(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, int nch,
                       const float* X, const float* W, int dg, RbfParams rp, float cutoff, float* S, float* Mpart,
                       int min_n, const float* rtab, cudaStream_t st) {
  using SM = sh::WarpSmem<6, 7, sh::kTile, MODE>;
  const int ncb = (dg + 31) / 32;
  const size_t smem = sizeof(float) * SM::fwd_total * sh::kW;
  static bool c1 = false, c2 = false;
  auto k1 = sh::fwd_moments_kernel<6, 7, MODE>;
  auto k2 = sh::fwd_apply_kernel<6, 7, MODE>;
  set_smem(k1, smem, c1);
  set_smem(k2, smem, c2);
  const int grid = sh_grid(nv * nch * ncb);
  k1<<<grid, sh::kW * 32, smem, st>>>(edge_ptr, rev, geo, nv, nch, X, W, dg, rp, cutoff, S, Mpart, min_n, rtab);
  if (check_launch("triplet_fwd_sh_moments")) return 1;
  k2<<<grid, sh::kW * 32, smem, st>>>(edge_ptr, rev, geo, nv, nch, dg, rp, S, Mpart, min_n);
  return check_launch("triplet_fwd_sh_apply");
}

int sh_fwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, int max_degree, const float* X,
           const float* W, int K, int L, int dg, RbfParams rp, float cutoff, int mode, float* S, void* ws, int min_n,
           cudaStream_t st, const float* rtab) {
  const int nch = sh_nch(max_degree);
  float* Mpart = reinterpret_cast<float*>(ws);
  if (mode == 1) return sh_fwd_mode<1>(edge_ptr, rev, geo, nv, nch, X, W, dg, rp, cutoff, S, Mpart, min_n, rtab, st);
  if (mode == 2) return sh_fwd_mode<2>(edge_ptr, rev, geo, nv, nch, X, W, dg, rp, cutoff, S, Mpart, min_n, rtab, st);
  return sh_fwd_mode<0>(edge_ptr, rev, geo, nv, nch, X, W, dg, rp, cutoff, S, Mpart, min_n, nullptr, st);
}

// radial tables of the Bessel bases (MODE 1 / 2): [ne][rad_stride] values and (dtab != null)
// d-derivatives
int64_t sh_radial_table_floats(int64_t ne, int mode) {
  return mode == 0 ? 0 : std::max<int64_t>(ne, 1) * (mode == 2 ? sh::rad_stride<2>() : sh::rad_stride<1>());
}
int sh_radial_table(const float4* geo, int64_t ne, float cutoff, int mode, float* tab, float* dtab, cudaStream_t st) {
  if (mode == 0 || ne == 0) return 0;
  const int64_t n = sh_radial_table_floats(ne, mode);
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, static_cast<int64_t>(kNumSMs) * 32));
  if (mode == 1) sh::radial_table_kernel<6, 7, 1><<<grid, 256, 0, st>>>(geo, ne, cutoff, tab, dtab);
  else sh::radial_table_kernel<6, 7, 2><<<grid, 256, 0, st>>>(geo, ne, cutoff, tab, dtab);
  return check_launch("triplet_sh_radial_table");
}

static int64_t sh_bwd_warps(int64_t nv, int nch, int dg, int* grid_out) {
  const int ncb = (dg + 31) / 32;
  // persistent warps: up to 48 per SM (6 waves of the 2 resident CTAs: the items are uneven and
  // finer scheduling balances them; 12 / 24 / 48 / 96 per SM measured 1.34 / 1.24 / 1.22 / 1.23 ms
  // at C5 deg 500, d_g 64), a multiple of ncb and of the CTA width
  int64_t want = std::min<int64_t>(nv * nch * ncb, static_cast<int64_t>(kNumSMs) * 48);
  const int64_t unit = static_cast<int64_t>(ncb) * sh::kW / std::__gcd(ncb, sh::kW);
  want = std::max<int64_t>(unit, (want + unit - 1) / unit * unit);
  *grid_out = static_cast<int>(want / sh::kW);
  return want;
}

int64_t sh_bwd_workspace_bytes(int64_t nv, int64_t ne, int max_degree, int K, int L, int dg) {
  int grid;
  const int nch = sh_nch(max_degree);
  const int64_t nw = sh_bwd_warps(std::max<int64_t>(nv, 1), nch, dg, &grid);
  const int ncb = (dg + 31) / 32;
  return nw * K * L * 32 * 4 + 2 * sh_fwd_workspace_bytes(nv, max_degree, K, L, dg) +
         (ncb > 1 ? static_cast<int64_t>(ncb) * std::max<int64_t>(ne, 1) * 16 : 0) + 256;
}

template <int MODE>
static int sh_bwd_mode(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, int64_t ne,
                       int nch, int grid, int64_t nw, const float* X, const float* W, int K, int L, int dg,
                       RbfParams rp, float cutoff, const float* Sbar, float* Xbar, float* Wbar, float4* edge_grad,
                       float* wpart, float* Mpart, float* Mbpart, float4* egp, int min_n, int accumulate,
                       const float* rtab, const float* drtab, cudaStream_t st) {
  using SM = sh::WarpSmem<6, 7, sh::kTile, MODE>;
  const int ncb = (dg + 31) / 32;
  static bool c1 = false, c2 = false;
  auto k1 = sh::bwd_moments_kernel<6, 7, MODE>;
  auto k2 = sh::bwd_apply_kernel<6, 7, MODE>;
  const size_t smem1 = sizeof(float) * SM::fwd_total * sh::kW;
  const size_t smem2 = sizeof(float) * sh::BwdSmem<6, 7, MODE>::total * sh::kW;
  set_smem(k1, smem1, c1);
  set_smem(k2, smem2, c2);
  k1<<<sh_grid(nv * nch * ncb), sh::kW * 32, smem1, st>>>(edge_ptr, rev, geo, nv, nch, X, W, dg, rp, cutoff, Sbar,
                                                         Mpart, Mbpart, min_n, rtab);
  if (check_launch("triplet_bwd_sh_moments")) return 1;
  k2<<<grid, sh::kW * 32, smem2, st>>>(edge_ptr, rev, geo, nv, ne, nch, X, W, dg, rp, cutoff, Sbar, Mpart, Mbpart,
                                       Xbar, wpart, egp, edge_grad, min_n, rtab, drtab);
  if (check_launch("triplet_bwd_sh_apply")) return 1;
  sh::reduce_wbar_kernel<6, 7, MODE><<<K * ncb, 1024, 0, st>>>(wpart, nw, ncb, dg, Wbar, accumulate);
  if (check_launch("triplet_bwd_sh_reduce")) return 1;
  if (ncb == 1) return 0;
  const int eg_grid = static_cast<int>(std::min<int64_t>((nv + 7) / 8, static_cast<int64_t>(kNumSMs) * 16));
  sh::add_eg_kernel<<<std::max(eg_grid, 1), 256, 0, st>>>(edge_ptr, nv, egp, ncb, ne, min_n, edge_grad);
  return check_launch("triplet_bwd_sh_eg");
}

int sh_bwd(const int64_t* edge_ptr, const int32_t* rev, const float4* geo, int64_t nv, int64_t ne, int max_degree,
           const float* X, const float* W, int K, int L, int dg, RbfParams rp, float cutoff, int mode,
           const float* Sbar, float* Xbar, float* Wbar, float4* edge_grad, void* ws, int min_n, int accumulate,
           cudaStream_t st, const float* rtab, const float* drtab) {
  const int nch = sh_nch(max_degree);
  int grid;
  const int64_t nw = sh_bwd_warps(std::max<int64_t>(nv, 1), nch, dg, &grid);
  const int ncb = (dg + 31) / 32;
  float* wpart = reinterpret_cast<float*>(ws);
  float* Mpart = wpart + nw * K * L * 32;
  float* Mbpart = Mpart + sh_fwd_workspace_bytes(nv, max_degree, K, L, dg) / 4;
  float4* egp = nullptr;
  if (ncb > 1) {
    const uintptr_t p = reinterpret_cast<uintptr_t>(Mbpart + sh_fwd_workspace_bytes(nv, max_degree, K, L, dg) / 4);
    egp = reinterpret_cast<float4*>((p + 15) & ~static_cast<uintptr_t>(15));
  }
#define EGN_SHB(M)                                                                                               \
  return sh_bwd_mode<M>(edge_ptr, rev, geo, nv, ne, nch, grid, nw, X, W, K, L, dg, rp, cutoff, Sbar, Xbar, Wbar, \
                        edge_grad, wpart, Mpart, Mbpart, egp, min_n, accumulate, M == 0 ? nullptr : rtab,        \
                        M == 0 ? nullptr : drtab, st)
  if (mode == 1) EGN_SHB(1);
  if (mode == 2) EGN_SHB(2);
  EGN_SHB(0);
#undef EGN_SHB
}

}  // namespace egn
