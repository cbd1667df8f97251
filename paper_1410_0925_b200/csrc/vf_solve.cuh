// Controller math shared by the on-device trackers (ICP, Ren, colour):
// Eigen-compatible pivoted LDLT, the reference's SVD condition test (decided
// by a rigorous bound when conclusive), pose increments, warp reductions.
//
// Reference: detail::well_conditioned, icp_track's LDLT solve
// (proj/include/voxfuse/engine/depth_tracker.hpp:99-104, :209-214),
// pose_increment / pose_rotate_increment / orthonormalize (proj/src/pose.cpp:9-30).
#pragma once

#include "vf_device.cuh"

namespace vf {
namespace {


constexpr int kAcc = 29;  // 21 H (upper triangle) + 6 g + cost + count
constexpr int kAccStride = 32;

// Controller-only FP64 reciprocal / square root: hardware approximation plus
// Newton steps (relative error ~1 ulp).  The controller's results already
// differ from the reference's Eigen LDLT by rounding, so it does not need the
// IEEE-rounded (and ~10x longer-latency) division; the per-pixel terms, which
// decide association and rejection, keep IEEE arithmetic.
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  return fma(r, fma(-x, r, 1.0), r);
}
__device__ __forceinline__ double sqrt_fast(double x) {
  if (!(x > 0)) return sqrt(x);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-0.5 * x * y, y, 1.5);
  y = y * fma(-0.5 * x * y, y, 1.5);
  const double s0 = x * y;
  return fma(fma(-s0, s0, x), 0.5 * y, s0);  // one Newton step on the square root
}


// Pivoted LDL^T of a symmetric n x n (row-major input) and solve, restating
// Eigen's LDLT as the reference calls it (depth_tracker.hpp:209,214).  Also
// returns the factor so the inverse can be formed for the condition bound.
struct Ldlt {
  double m[36];  // column-major, lower used
  int trans[6];
  int n;
  bool zero;
  bool issue;  // Eigen's info() == NumericalIssue
  __device__ double& at(int r, int c) { return m[r + c * n]; }
  __device__ void compute(const double* a, int nn) {
    n = nn;
    zero = false;
    issue = false;
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < n; ++c) at(r, c) = a[r * n + c];
    for (int k = 0; k < n; ++k) trans[k] = k;
    double temp[6];
    for (int k = 0; k < n; ++k) {
      int big = k;
      double bigv = fabs(at(k, k));
      for (int i = k + 1; i < n; ++i)
        if (fabs(at(i, i)) > bigv) {
          bigv = fabs(at(i, i));
          big = i;
        }
      trans[k] = big;
      if (k != big) {
        for (int c = 0; c < n; ++c) {
          const double t = at(k, c);
          at(k, c) = at(big, c);
          at(big, c) = t;
        }
        for (int r = 0; r < n; ++r) {
          const double t = at(r, k);
          at(r, k) = at(r, big);
          at(r, big) = t;
        }
      }
      if (k > 0) {
        for (int i = 0; i < k; ++i) temp[i] = at(i, i) * at(k, i);
        double s = 0;
        for (int i = 0; i < k; ++i) s = (i == 0) ? at(k, 0) * temp[0] : s + at(k, i) * temp[i];
        at(k, k) -= s;
        for (int r = k + 1; r < n; ++r) {
          double t = 0;
          for (int i = 0; i < k; ++i) t = (i == 0) ? at(r, 0) * temp[0] : t + at(r, i) * temp[i];
          at(r, k) -= t;
        }
      }
      const double akk = at(k, k);
      const bool ok = fabs(akk) > 0;
      if (k == 0 && !ok) {
        for (int j = 0; j < n; ++j) trans[j] = j;
        zero = true;
        issue = true;
        break;
      }
      if (k + 1 < n && ok) {
        for (int r = k + 1; r < n; ++r) at(r, k) /= akk;
      } else if (k + 1 < n) {
        for (int r = k + 1; r < n; ++r)
          if (at(r, k) != 0) issue = true;
      }
    }
  }
  __device__ void solve(const double* b, double* x) {
    for (int i = 0; i < n; ++i) x[i] = b[i];
    for (int k = 0; k < n; ++k) {
      const double t = x[k];
      x[k] = x[trans[k]];
      x[trans[k]] = t;
    }
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < i; ++j) x[i] -= at(i, j) * x[j];
    const double tol = 2.2250738585072014e-308;
    for (int i = 0; i < n; ++i) {
      if (!zero && fabs(at(i, i)) > tol)
        x[i] /= at(i, i);
      else
        x[i] = 0;
    }
    for (int i = n - 1; i >= 0; --i)
      for (int j = i + 1; j < n; ++j) x[i] -= at(j, i) * x[j];
    for (int k = n - 1; k >= 0; --k) {
      const double t = x[k];
      x[k] = x[trans[k]];
      x[trans[k]] = t;
    }
  }
};

// Jacobi SVD singular values (the reference's JacobiSVD; fallback path only).
__device__ void jacobi_singular_values(const double* a_rowmajor, int n, double* sv) {
  double w[36];
  double scale = 0;
  for (int i = 0; i < n * n; ++i) scale = fmax(scale, fabs(a_rowmajor[i]));
  if (!(scale > 0) || !isfinite(scale)) scale = 1.0;
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) w[r + c * n] = a_rowmajor[r * n + c] / scale;
  const double precision = 2.0 * 2.220446049250313e-16;
  const double dmin = 2.2250738585072014e-308;
  double max_diag = 0;
  for (int i = 0; i < n; ++i) max_diag = fmax(max_diag, fabs(w[i + i * n]));
  bool finished = false;
  for (int sweep = 0; !finished && sweep < 64; ++sweep) {
    finished = true;
    for (int p = 1; p < n; ++p)
      for (int q = 0; q < p; ++q) {
        const double threshold = fmax(dmin, precision * max_diag);
        if (fabs(w[p + q * n]) > threshold || fabs(w[q + p * n]) > threshold) {
          finished = false;
          const double m00 = w[p + p * n], m01 = w[p + q * n], m10 = w[q + p * n], m11 = w[q + q * n];
          double c1 = 1, s1 = 0;
          const double t = m00 + m11, d = m10 - m01;
          if (!(fabs(d) < dmin)) {
            const double u = t / d;
            const double tmp = sqrt(1.0 + u * u);
            s1 = 1.0 / tmp;
            c1 = u / tmp;
          }
          const double n00 = c1 * m00 + s1 * m10, n01 = c1 * m01 + s1 * m11, n11 = -s1 * m01 + c1 * m11;
          double cr = 1, sr = 0;
          const double deno = 2.0 * fabs(n01);
          if (!(deno < dmin)) {
            const double tau = (n00 - n11) / deno;
            const double ww = sqrt(tau * tau + 1.0);
            const double tt = tau > 0 ? 1.0 / (tau + ww) : 1.0 / (tau - ww);
            const double sign_t = tt > 0 ? 1.0 : -1.0;
            const double nn = 1.0 / sqrt(tt * tt + 1.0);
            sr = -sign_t * (n01 / fabs(n01)) * fabs(tt) * nn;
            cr = nn;
          }
          // j_left = rot1 * j_right^T
          const double cl = c1 * cr - s1 * (-sr), sl = c1 * (-sr) + s1 * cr;
          if (!(cl == 1 && sl == 0))
            for (int i = 0; i < n; ++i) {
              const double xi = w[p + i * n], yi = w[q + i * n];
              w[p + i * n] = cl * xi + sl * yi;
              w[q + i * n] = -sl * xi + cl * yi;
            }
          // columns with j_right^T
          const double cc = cr, ss = -sr;
          if (!(cc == 1 && ss == 0))
            for (int i = 0; i < n; ++i) {
              const double xi = w[i + p * n], yi = w[i + q * n];
              w[i + p * n] = cc * xi + ss * yi;
              w[i + q * n] = -ss * xi + cc * yi;
            }
          max_diag = fmax(max_diag, fmax(fabs(w[p + p * n]), fabs(w[q + q * n])));
        }
      }
  }
  for (int i = 0; i < n; ++i) sv[i] = fabs(w[i + i * n]) * scale;
  for (int i = 0; i < n; ++i)
    for (int k = i + 1; k < n; ++k)
      if (sv[k] > sv[i]) {
        const double t = sv[i];
        sv[i] = sv[k];
        sv[k] = t;
      }
}

// detail::well_conditioned (depth_tracker.hpp:99-104), decided by the bound
// cond_2(H) <= |H|_F * |H^-1|_F whenever it is conclusive.
__device__ bool well_conditioned(const double* h, int n, Ldlt& f, double max_condition) {
  bool pd = !f.zero;
  for (int i = 0; i < n && pd; ++i) pd = f.at(i, i) > 0;
  if (pd) {
    double hf = 0;
    for (int i = 0; i < n * n; ++i) hf += h[i] * h[i];
    double inv_f = 0;
    for (int c = 0; c < n; ++c) {
      double e[6] = {0, 0, 0, 0, 0, 0}, col[6];
      e[c] = 1.0;
      f.solve(e, col);
      for (int r = 0; r < n; ++r) inv_f += col[r] * col[r];
    }
    const double bound = sqrt(hf) * sqrt(inv_f);
    if (isfinite(bound) && bound * (1.0 + 1e-6) < max_condition) return true;
  }
  double sv[6];
  jacobi_singular_values(h, n, sv);
  const double smin = sv[n - 1], smax = sv[0];
  return smin > 0 && smax / smin < max_condition;
}

// orthonormalize(I + [w]x) (pose.cpp:9-18) in closed form:
// R = I + K / s + K^2 / (s (s + 1)),  K = [w]x,  s = sqrt(1 + |w|^2).
__device__ void rot_from_omega(const double* w, double* r) {
  const double th2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
  const double s = sqrt_fast(1.0 + th2);
  const double a = rcp_fast(s), b = a * rcp_fast(s + 1.0);
  const double K[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
  double K2[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) K2[i * 3 + j] = K[i * 3 + 0] * K[0 * 3 + j] + K[i * 3 + 1] * K[1 * 3 + j] + K[i * 3 + 2] * K[2 * 3 + j];
  for (int i = 0; i < 9; ++i) r[i] = (i % 4 == 0 ? 1.0 : 0.0) + a * K[i] + b * K2[i];
}
// pose_increment / pose_rotate_increment (pose.cpp:20-30)
__device__ PoseD pose_increment(const PoseD& p, const double* tw, bool rotate_only) {
  double rd[9];
  rot_from_omega(tw, rd);
  PoseD o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      o.r[i * 3 + j] = rd[i * 3 + 0] * p.r[0 * 3 + j] + rd[i * 3 + 1] * p.r[1 * 3 + j] + rd[i * 3 + 2] * p.r[2 * 3 + j];
  if (rotate_only) {
    for (int i = 0; i < 3; ++i) o.t[i] = p.t[i];
  } else {
    for (int i = 0; i < 3; ++i) o.t[i] = rd[i * 3 + 0] * p.t[0] + rd[i * 3 + 1] * p.t[1] + rd[i * 3 + 2] * p.t[2] + tw[3 + i];
  }
  return o;
}

// detail::sample_map_bilinear (depth_tracker.hpp:37-55)
__device__ __forceinline__ bool sample_map(const float4* __restrict__ map, int w, int h, double x, double y,
                                           float max_spread, D3& out) {
  if (x < 0 || y < 0 || x > w - 1.001 || y > h - 1.001) return false;
  const int ix = (int)x, iy = (int)y;
  const double fx = x - ix, fy = y - iy;
  const float4 a = __ldg(map + (size_t)iy * w + ix), b = __ldg(map + (size_t)iy * w + ix + 1);
  const float4 c = __ldg(map + (size_t)(iy + 1) * w + ix), d = __ldg(map + (size_t)(iy + 1) * w + ix + 1);
  if (a.w == 0.0f || b.w == 0.0f || c.w == 0.0f || d.w == 0.0f) return false;
#define MINF(p, q) ((q) < (p) ? (q) : (p))
#define MAXF(p, q) ((p) < (q) ? (q) : (p))
  const float sx = MAXF(MAXF(MAXF(a.x, b.x), c.x), d.x) - MINF(MINF(MINF(a.x, b.x), c.x), d.x);
  const float sy = MAXF(MAXF(MAXF(a.y, b.y), c.y), d.y) - MINF(MINF(MINF(a.y, b.y), c.y), d.y);
  const float sz = MAXF(MAXF(MAXF(a.z, b.z), c.z), d.z) - MINF(MINF(MINF(a.z, b.z), c.z), d.z);
#undef MINF
#undef MAXF
  if (sqrtf(sx * sx + sy * sy + sz * sz) > max_spread) return false;
  const float w0 = (float)((1 - fx) * (1 - fy)), w1 = (float)(fx * (1 - fy));
  const float w2 = (float)((1 - fx) * fy), w3 = (float)(fx * fy);
  out.x = (double)(a.x * w0 + b.x * w1 + c.x * w2 + d.x * w3);
  out.y = (double)(a.y * w0 + b.y * w1 + c.y * w2 + d.y * w3);
  out.z = (double)(a.z * w0 + b.z * w1 + c.z * w2 + d.z * w3);
  return true;
}

// Fast controller path, fully unrolled so everything stays in registers:
// unpivoted LDL^T of the SPD system (backward stable for SPD; differs from
// Eigen's pivoted LDLT only by rounding), the solve, and the condition bound
//   cond_2(H) <= |H|_F * trace(H^-1),   trace(H^-1) = |D^-1/2 L^-1|_F^2,
// which decides the reference's SVD test exactly whenever it is below the
// threshold.  Returns false (-> exact fallback path) if H is not numerically
// SPD or the bound is inconclusive.
template <int N>
__device__ __forceinline__ bool spd_solve_fast(const double* __restrict__ tot, double max_condition, double* twist) {
  double H[N][N];
#pragma unroll
  for (int s = 0, k = 0; s < 6; ++s)
#pragma unroll
    for (int t = s; t < 6; ++t, ++k)
      if (s < N && t < N) {
        H[s][t] = tot[k];
        H[t][s] = tot[k];
      }
  double L[N][N], D[N], Dinv[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double d = H[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) d -= (L[j][k] * L[j][k]) * D[k];
    if (!(d > 0)) return false;
    D[j] = d;
    Dinv[j] = rcp_fast(d);
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      double sum = H[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) sum -= (L[i][k] * L[j][k]) * D[k];
      L[i][j] = sum * Dinv[j];
    }
  }
  // Linv = L^-1 (unit lower triangular)
  double Li[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < i; ++j) {
      double sum = L[i][j];
#pragma unroll
      for (int k = j + 1; k < i; ++k) sum += L[i][k] * Li[k][j];
      Li[i][j] = -sum;
    }
  }
  double hf = 0, tr = 0;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) hf += H[i][j] * H[i][j];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double row = 1.0;  // Li[k][k] = 1
#pragma unroll
    for (int i = 0; i < k; ++i) row += Li[k][i] * Li[k][i];
    tr += row * Dinv[k];
  }
  const double bound = sqrt_fast(hf) * tr;
  if (!(bound * (1.0 + 1e-6) < max_condition)) return false;
  // solve H x = -g
  double y[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double v = -tot[21 + i];
#pragma unroll
    for (int k = 0; k < i; ++k) v -= L[i][k] * y[k];
    y[i] = v;
  }
#pragma unroll
  for (int i = 0; i < N; ++i) y[i] *= Dinv[i];
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    double v = y[i];
#pragma unroll
    for (int k = i + 1; k < N; ++k) v -= L[k][i] * twist[k];
    twist[i] = v;
  }
  return true;
}

// Levenberg-Marquardt step of color_track (color_tracker.hpp:126-133): solve
// (H with its diagonal scaled by 1 + lambda) x = -g, fully unrolled in
// registers (unpivoted LDL^T; differs from Eigen's pivoted LDLT by rounding
// only).  Returns false when the damped system is not numerically SPD, so the
// caller takes the reference's pivoted path.
__device__ __forceinline__ bool spd_solve_damped6(const double* __restrict__ tot, double lambda, double* twist) {
  constexpr int N = 6;
  double H[N][N];
#pragma unroll
  for (int s = 0, k = 0; s < N; ++s)
#pragma unroll
    for (int t = s; t < N; ++t, ++k) {
      H[s][t] = tot[k];
      H[t][s] = tot[k];
    }
#pragma unroll
  for (int s = 0; s < N; ++s) H[s][s] *= (1.0 + lambda);
  double L[N][N], D[N], Dinv[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double d = H[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) d -= (L[j][k] * L[j][k]) * D[k];
    if (!(d > 0) || !isfinite(d)) return false;
    D[j] = d;
    Dinv[j] = rcp_fast(d);
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      double sum = H[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) sum -= (L[i][k] * L[j][k]) * D[k];
      L[i][j] = sum * Dinv[j];
    }
  }
  double y[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double v = -tot[21 + i];
#pragma unroll
    for (int k = 0; k < i; ++k) v -= L[i][k] * y[k];
    y[i] = v;
  }
#pragma unroll
  for (int i = 0; i < N; ++i) y[i] *= Dinv[i];
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    double v = y[i];
#pragma unroll
    for (int k = i + 1; k < N; ++k) v -= L[k][i] * twist[k];
    twist[i] = v;
  }
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (!isfinite(twist[i])) return false;
  return true;
}

// Reduce 32 per-lane values across the warp with a transpose butterfly:
// 31 shuffles instead of 5 per value.  On return lane l holds the warp sum
// of value index l.
__device__ __forceinline__ double warp_reduce32(double (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int step = 0; step < 5; ++step) {
    const int half = 16 >> step;  // values kept per lane after this step
    const bool upper = (lane & half) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      // keep v[i] (lower lanes) or v[i + half] (upper lanes); send the other
      const double send = upper ? v[i] : v[i + half];
      const double keep = upper ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  return v[0];
}

}  // namespace
}  // namespace vf
