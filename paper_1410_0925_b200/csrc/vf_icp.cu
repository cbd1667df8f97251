// K4 — depth pyramid and the point-to-plane ICP tracker, entirely on device.
//
// Reference: build_depth_pyramid / downsample_depth
// (proj/include/voxfuse/engine/pyramid.hpp:35-111), icp_track and its helpers
// (proj/include/voxfuse/engine/depth_tracker.hpp:20-239), pose_increment /
// pose_rotate_increment / orthonormalize (proj/src/pose.cpp:9-30).
//
// The reference runs up to levels x 20 iterations, each a parallel 29-value
// reduction followed by host control logic (cost test, step halving, SVD
// condition check, LDLT solve, pose update).  Here the whole coarse-to-fine
// loop is one cooperative persistent kernel: per iteration every CTA reduces
// its pixels (FP64 per-pixel math, warp shuffles then a CTA tree) into a
// partial, one grid barrier publishes the partials (double-buffered), and every
// CTA sums the partials in the same fixed order and runs the same controller,
// so all CTAs agree on every branch without a second barrier.  Coarse levels
// with few pixels run on CTA 0 alone with no grid barrier at all.
//
// Controller arithmetic: the twist comes from the same pivoted LDLT as the
// reference's Eigen call; the SVD condition test is first decided by the
// rigorous bound cond <= |H|_F |H^-1|_F (exact answer whenever the bound is
// below the threshold) and falls back to the full Jacobi SVD otherwise; the
// SVD re-orthonormalisation of I + [w]x is replaced by its closed form (the
// polar factor of I + [w]x is the rotation about w by atan|w|), identical up
// to rounding.
#include <cooperative_groups.h>

#include "vf_device.cuh"
#include "vf_kernels.h"

namespace cg = cooperative_groups;

namespace vf {

// ---------------------------------------------------------------------------
// pyramid
// ---------------------------------------------------------------------------
// One CTA per 32x32 tile of level 0; levels 1..L-1 of the tile are built in
// shared memory (32 = 2^5 keeps tiles aligned for up to 6 levels).
__global__ void __launch_bounds__(256) k_pyramid(const float* __restrict__ depth0, int w0, int h0, int levels,
                                                 float* __restrict__ out /* levels 1.. back to back */) {
  __shared__ float tile[2][32 * 32];
  const int tx0 = blockIdx.x * 32, ty0 = blockIdx.y * 32;
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) {
    const int x = tx0 + (i & 31), y = ty0 + (i >> 5);
    tile[0][i] = (x < w0 && y < h0) ? depth0[(size_t)y * w0 + x] : 0.0f;
  }
  __syncthreads();
  int sw = w0, sh = h0, ts = 32, cur = 0;
  int sx0 = tx0, sy0 = ty0;
  size_t off = 0;
  for (int l = 1; l < levels; ++l) {
    const int dw = (sw + 1) / 2, dh = (sh + 1) / 2, dts = ts / 2;
    const int dx0 = sx0 / 2, dy0 = sy0 / 2;
    for (int i = threadIdx.x; i < dts * dts; i += blockDim.x) {
      const int lx = i % dts, ly = i / dts;
      const int gx = dx0 + lx, gy = dy0 + ly;
      float outv = 0.0f;
      if (gx < dw && gy < dh) {
        // downsample_depth (pyramid.hpp:35-65)
        float dmin = 0.0f;
        for (int dy = 0; dy < 2; ++dy)
          for (int dx = 0; dx < 2; ++dx) {
            const int sx = 2 * gx + dx, sy = 2 * gy + dy;
            if (sx >= sw || sy >= sh) continue;
            const float d = tile[cur][(2 * ly + dy) * ts + 2 * lx + dx];
            if (d > 0.0f && (dmin <= 0.0f || d < dmin)) dmin = d;
          }
        if (dmin > 0.0f) {
          float sum = 0.0f;
          int n = 0;
          for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
              const int sx = 2 * gx + dx, sy = 2 * gy + dy;
              if (sx >= sw || sy >= sh) continue;
              const float d = tile[cur][(2 * ly + dy) * ts + 2 * lx + dx];
              if (d <= 0.0f || d > dmin + 0.05f) continue;
              sum += d;
              ++n;
            }
          outv = sum / (float)n;
        }
        out[off + (size_t)gy * dw + gx] = outv;
      }
      tile[cur ^ 1][ly * dts + lx] = outv;
    }
    __syncthreads();
    cur ^= 1;
    off += (size_t)dw * dh;
    sw = dw;
    sh = dh;
    ts = dts;
    sx0 = dx0;
    sy0 = dy0;
  }
}

// ---------------------------------------------------------------------------
// controller math
// ---------------------------------------------------------------------------
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
  __device__ double& at(int r, int c) { return m[r + c * n]; }
  __device__ void compute(const double* a, int nn) {
    n = nn;
    zero = false;
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
        break;
      }
      if (k + 1 < n && ok)
        for (int r = k + 1; r < n; ++r) at(r, k) /= akk;
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

// The validity / spread test and blend of sample_map_bilinear
// (depth_tracker.hpp:40-54) on four already-loaded taps a, b, c, d.
__device__ __forceinline__ bool bilinear_taps(const float4 (&t)[4], double fx, double fy, float max_spread, D3& out) {
  const float4 a = t[0], b = t[1], c = t[2], d = t[3];
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

struct Ctl {
  PoseD c2w, accepted, render;
  double pending[6];
  double accepted_cost, final_cost;
  int halvings, iterations, any_solved, valid_points, fail;
  int decision;  // 0 continue, 1 leave level, 2 abort
  int trace_rows;
};

static_assert(sizeof(Ctl) <= 1024, "Ctl must fit the ctl_io buffer");

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace

// The ICP loop over levels [a.level_hi .. a.level_lo].  kCluster: the grid is
// one thread-block cluster and partials travel through distributed shared
// memory behind a hardware cluster barrier (coarse levels); otherwise the
// grid is cooperative and partials go through global memory behind a grid
// barrier (fine levels).  The controller state enters / leaves through
// a.ctl_io when the loop is split between the two kernels.
template <bool kCluster>
__device__ __forceinline__ void icp_body(const IcpArgs& a) {
  __shared__ Ctl ctl;
  __shared__ double s_red[kIcpThreads / 32][kAccStride];
  __shared__ double s_tot[kAccStride];
  __shared__ double s_part[2][kAccStride];  // cluster exchange (double-buffered)
  // dynamic: unprojection tables (max level-0 width + height doubles), then
  // max_slots x blockDim pixel slots (float depth, packed x | y << 16)
  extern __shared__ __align__(16) unsigned char s_dyn[];
  double* s_ux = reinterpret_cast<double*>(s_dyn);
  double* s_uy = s_ux + a.lv[0].w;
  float* s_depth = reinterpret_cast<float*>(s_uy + a.lv[0].h);
  int* s_xy = reinterpret_cast<int*>(s_depth + a.max_slots * blockDim.x);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const bool timer = blockIdx.x == 0 && tid == 0 && a.trace;
  if (tid == 0) {
    if (a.ctl_in) {
      ctl = *reinterpret_cast<const Ctl*>(a.ctl_io);
    } else {
      ctl.render = *a.state_pose;
      // icp_track(..., initial) (depth_tracker.hpp:117): start from `initial` if given
      ctl.c2w = pose_inverse(a.initial ? *a.initial : ctl.render);
      ctl.iterations = 0;
      ctl.any_solved = 0;
      ctl.valid_points = 0;
      ctl.final_cost = 0;
      ctl.fail = 0;
      ctl.trace_rows = 0;
    }
  }
  __syncthreads();
  int buf = 0;
  int trace_rows = ctl.trace_rows;
  for (int level = a.level_hi; level >= a.level_lo && !ctl.fail; --level) {
    const IcpLevel lv = a.lv[level];
    const int npix = lv.w * lv.h;
    const bool rotation_only = level >= a.levels - a.rotation_only_levels;
    if (tid == 0) {
      ctl.accepted_cost = __longlong_as_double(0x7ff0000000000000ll);
      ctl.accepted = ctl.c2w;
      for (int i = 0; i < 6; ++i) ctl.pending[i] = 0;
      ctl.halvings = 0;
    }
    // Depth and unprojection are iteration-invariant: stage this CTA's pixel
    // slots (depth + packed x, y) and the level's (x - cx) / fx, (y - cy) / fy
    // tables in shared memory once per level.
    const int gstride = gridDim.x * blockDim.x;
    const int nslots = min((npix - (int)(blockIdx.x * blockDim.x) + gstride - 1) / gstride, a.max_slots);
    for (int i = tid; i < lv.w; i += blockDim.x) s_ux[i] = __ldg(lv.ux + i);
    for (int i = tid; i < lv.h; i += blockDim.x) s_uy[i] = __ldg(lv.uy + i);
    for (int k = 0; k < nslots; ++k) {
      const int pix = blockIdx.x * blockDim.x + tid + k * gstride;
      float d = 0.0f;
      int xy = 0;
      if (pix < npix) {
        const int y = pix / lv.w, x = pix - y * lv.w;
        d = __ldg(lv.depth + pix);
        xy = x | (y << 16);
      }
      s_depth[k * blockDim.x + tid] = d;
      s_xy[k * blockDim.x + tid] = xy;
    }
    __syncthreads();
    for (int iter = 0; iter < a.max_iterations; ++iter) {
      long long t0 = timer ? clock64() : 0;
      const PoseD c2w = ctl.c2w;
      const PoseD render = ctl.render;
      const D3 rc = rotation_only ? mk(c2w.t[0], c2w.t[1], c2w.t[2]) : mk(0, 0, 0);
      double acc[kAcc];
#pragma unroll
      for (int i = 0; i < kAcc; ++i) acc[i] = 0;
      // Two pixels per step, each pipeline stage issued for both before it is
      // consumed, so their memory round trips (depth + tables, then the
      // eight map taps) overlap.
      const int total_slots = (npix - (int)(blockIdx.x * blockDim.x) + gstride - 1) / gstride;
      for (int k0 = 0; k0 < total_slots; k0 += 2) {
        float d[2];
        double ux[2], uy[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int slot = k0 + k;
          const int pix = blockIdx.x * blockDim.x + tid + slot * gstride;
          if (slot < nslots) {  // staged in shared memory
            d[k] = s_depth[slot * blockDim.x + tid];
            const int xy = s_xy[slot * blockDim.x + tid];
            ux[k] = s_ux[xy & 0xFFFF];
            uy[k] = s_uy[xy >> 16];
          } else {  // beyond the staging capacity (very large images)
            const bool in = slot < total_slots && pix < npix;
            const int y = in ? pix / lv.w : 0, x = in ? pix - y * lv.w : 0;
            d[k] = in ? __ldg(lv.depth + pix) : 0.0f;
            ux[k] = s_ux[x];
            uy[k] = s_uy[y];
          }
        }
        D3 pw[2];
        bool ok[2];
        int ix[2], iy[2];
        double fx[2], fy[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          // unproject (intrinsics.hpp:39-43); (x - cx) / fx is tabulated per level
          const D3 pc = mk(ux[k] * d[k], uy[k] * d[k], (double)d[k]);
          pw[k] = apply(c2w, pc);
          const D3 q = apply(render, pw[k]);
          const double u = a.map.fx * q.x / q.z + a.map.cx;
          const double v = a.map.fy * q.y / q.z + a.map.cy;
          // sample_map_bilinear's bounds test (depth_tracker.hpp:39)
          ok[k] = d[k] > 0.0f && q.z > 0.0 &&
                  !(u < 0 || v < 0 || u > a.map.width - 1.001 || v > a.map.height - 1.001);
          ix[k] = ok[k] ? (int)u : 0;
          iy[k] = ok[k] ? (int)v : 0;
          fx[k] = u - ix[k];
          fy[k] = v - iy[k];
        }
        float4 tp[2][4], tn[2][4];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const size_t i00 = (size_t)iy[k] * a.map.width + ix[k];
          if (ok[k]) {
            tp[k][0] = __ldg(a.points + i00);
            tp[k][1] = __ldg(a.points + i00 + 1);
            tp[k][2] = __ldg(a.points + i00 + a.map.width);
            tp[k][3] = __ldg(a.points + i00 + a.map.width + 1);
            tn[k][0] = __ldg(a.normals + i00);
            tn[k][1] = __ldg(a.normals + i00 + 1);
            tn[k][2] = __ldg(a.normals + i00 + a.map.width);
            tn[k][3] = __ldg(a.normals + i00 + a.map.width + 1);
          }
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          if (!ok[k]) continue;
          D3 mp, mn;
          if (!bilinear_taps(tp[k], fx[k], fy[k], a.dist_thr, mp)) continue;
          if (!bilinear_taps(tn[k], fx[k], fy[k], 1.0f, mn)) continue;
          const double nlen = sqrt(mn.x * mn.x + mn.y * mn.y + mn.z * mn.z);
          if (nlen < 1e-6) continue;
          // model_normal /= nlen: one refined reciprocal instead of three IEEE
          // divisions (1-ulp differences, far below the 1e-9 H/g parity bar)
          const double inv = rcp_fast(nlen);
          mn = mk(mn.x * inv, mn.y * inv, mn.z * inv);
          // icp_point_to_plane_term (depth_tracker.hpp:20-27)
          const D3 w = pw[k];
          const double r = (w.x - mp.x) * mn.x + (w.y - mp.y) * mn.y + (w.z - mp.z) * mn.z;
          if (fabs(r) > (double)a.dist_thr) continue;
          const D3 pr = rotation_only ? mk(w.x - rc.x, w.y - rc.y, w.z - rc.z) : w;
          // Jacobian and sums feed only the 29 accumulators, whose reduction
          // order differs from the reference's anyway (parity bar 1e-9), so
          // they use fused multiply-adds; everything that decides association
          // or rejection above keeps the reference's exact rounding.
          const double j[6] = {fma(pr.y, mn.z, -(pr.z * mn.y)), fma(pr.z, mn.x, -(pr.x * mn.z)),
                               fma(pr.x, mn.y, -(pr.y * mn.x)), mn.x, mn.y, mn.z};
          int n = 0;
#pragma unroll
          for (int s = 0; s < 6; ++s) {
#pragma unroll
            for (int t = s; t < 6; ++t, ++n) acc[n] = fma(j[s], j[t], acc[n]);
            acc[21 + s] = fma(j[s], r, acc[21 + s]);
          }
          acc[27] = fma(r, r, acc[27]);
          acc[28] += 1.0;
        }
      }
      // CTA reduction: transpose butterfly inside each warp, then one warp
      // combines the warp sums.
      {
        double v32[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v32[i] = i < kAcc ? acc[i] : 0.0;
        const double mine = warp_reduce32(v32);
        s_red[warp][lane] = mine;  // lane l holds value index l
      }
      __syncthreads();
      long long t1 = 0, t2 = 0;
      if (kCluster) {
        cg::cluster_group cluster = cg::this_cluster();
        if (tid < kAcc) {
          double sum = 0;
          for (int w = 0; w < nwarps; ++w) sum += s_red[w][tid];
          s_part[buf][tid] = sum;
        }
        t1 = timer ? clock64() : 0;
        cluster.sync();
        t2 = timer ? clock64() : 0;
        if (tid < kAcc) {  // every CTA sums the cluster's partials in rank order
          double t = 0;
          for (unsigned r = 0; r < cluster.num_blocks(); ++r) t += cluster.map_shared_rank(&s_part[buf][0], r)[tid];
          s_tot[tid] = t;
        }
        buf ^= 1;
      } else {
        cg::grid_group grid = cg::this_grid();
        double* part = a.partials + ((size_t)buf * gridDim.x + blockIdx.x) * kAccStride;
        if (tid < kAcc) {
          double sum = 0;
          for (int w = 0; w < nwarps; ++w) sum += s_red[w][tid];
          part[tid] = sum;
        }
        t1 = timer ? clock64() : 0;
        grid.sync();
        t2 = timer ? clock64() : 0;
        // every CTA sums all partials in the same fixed order:
        // thread (i = tid & 31, part = tid >> 5) over CTAs part, part + 8, ...
        const double* base = a.partials + (size_t)buf * gridDim.x * kAccStride;
        const int i = tid & 31, grp = tid >> 5;
        double sum = 0;
        if (i < kAcc) {
          double vals[kMaxIcpGrid / 8];
#pragma unroll
          for (int k = 0; k < kMaxIcpGrid / 8; ++k) {
            const int b = grp + 8 * k;
            vals[k] = b < (int)gridDim.x ? __ldcg(base + (size_t)b * kAccStride + i) : 0.0;
          }
#pragma unroll
          for (int k = 0; k < kMaxIcpGrid / 8; ++k) sum += vals[k];
        }
        s_red[grp][i] = sum;
        __syncthreads();
        if (tid < kAcc) {
          double t = 0;
          for (int w = 0; w < nwarps; ++w) t += s_red[w][tid];
          s_tot[tid] = t;
        }
        buf ^= 1;
      }
      __syncthreads();
      long long t3 = timer ? clock64() : 0;
      if (tid == 0) {
        const double* tot = s_tot;
        const long long count = (long long)tot[28];
        double* row = nullptr;
        if (blockIdx.x == 0 && a.trace && trace_rows < a.trace_cap) {
          row = a.trace + (size_t)trace_rows * kTraceRow;
          row[0] = level;
          row[1] = iter;
          for (int i = 0; i < 27; ++i) row[2 + i] = tot[i];
          row[29] = tot[27];
          row[30] = tot[28];
          row[31] = rotation_only ? 1 : 0;
          for (int i = 0; i < 9; ++i) row[32 + i] = ctl.c2w.r[i];
          for (int i = 0; i < 3; ++i) row[41 + i] = ctl.c2w.t[i];
        }
        ++trace_rows;
        ctl.decision = 0;
        if (count < a.min_valid_points) {
          ctl.valid_points = (int)count;
          ctl.decision = 1;
        } else {
          const double cost = tot[27] / (double)count;
          if (cost > ctl.accepted_cost) {
            double sq = 0;
            for (int i = 0; i < 6; ++i) sq = (i == 0) ? ctl.pending[0] * ctl.pending[0] : sq + ctl.pending[i] * ctl.pending[i];
            if (ctl.halvings < 4 && sq > 0) {
              ++ctl.halvings;
              for (int i = 0; i < 6; ++i) ctl.pending[i] *= 0.5;
              ctl.c2w = pose_increment(ctl.accepted, ctl.pending, rotation_only);
            } else {
              ctl.c2w = ctl.accepted;
              ctl.decision = 1;
            }
          } else {
            ctl.accepted_cost = cost;
            ctl.accepted = ctl.c2w;
            ctl.halvings = 0;
            double H[36];
            for (int s = 0, k = 0; s < 6; ++s)
              for (int t = s; t < 6; ++t, ++k) {
                H[s * 6 + t] = tot[k];
                H[t * 6 + s] = tot[k];
              }
            double twist[6] = {0, 0, 0, 0, 0, 0};
            const int n = rotation_only ? 3 : 6;
            bool good = rotation_only ? spd_solve_fast<3>(tot, a.max_condition, twist)
                                      : spd_solve_fast<6>(tot, a.max_condition, twist);
            if (!good) {
              // exact path: the reference's pivoted LDLT and SVD condition test
              double hn[36], g[6];
              for (int s = 0; s < n; ++s) {
                for (int t = 0; t < n; ++t) hn[s * n + t] = H[s * 6 + t];
                g[s] = -tot[21 + s];
              }
              Ldlt f;
              f.compute(hn, n);
              good = well_conditioned(hn, n, f, a.max_condition);
              if (good) f.solve(g, twist);
            }
            if (!good) {
              ctl.fail = 1;
              ctl.decision = 2;
            } else {
              ctl.c2w = pose_increment(ctl.c2w, twist, rotation_only);
              for (int i = 0; i < 6; ++i) ctl.pending[i] = twist[i];
              ++ctl.iterations;
              ctl.any_solved = 1;
              ctl.final_cost = cost;
              ctl.valid_points = (int)count;
              double tn = 0;
              for (int i = 0; i < 6; ++i) tn = (i == 0) ? twist[0] * twist[0] : tn + twist[i] * twist[i];
              if (tn < (double)a.conv_eps * (double)a.conv_eps) {  // |twist| < eps
                ctl.accepted = ctl.c2w;
                ctl.decision = 1;
              }
            }
          }
        }
        if (row) {
          const long long t4 = clock64();
          row[44] = (double)(t1 - t0);  // pixel terms + CTA reduction
          row[45] = (double)(t2 - t1);  // grid barrier
          row[46] = (double)(t3 - t2);  // partial sums
          row[47] = (double)(t4 - t3);  // controller
        }
      }
      __syncthreads();
      if (ctl.decision != 0) break;
    }
  }
  if (kCluster) cg::this_cluster().sync();  // no CTA leaves while others read its shared memory
  if (blockIdx.x == 0 && tid == 0) {
    ctl.trace_rows = trace_rows;
    if (!a.is_last) {
      *reinterpret_cast<Ctl*>(a.ctl_io) = ctl;
    } else {
      IcpResult res;
      res.ok = (!ctl.fail && ctl.any_solved) ? 1 : 0;
      res.iterations = res.ok ? ctl.iterations : 0;  // depth_tracker.hpp:208,234,237
      res.valid_points = ctl.valid_points;
      res.final_cost = ctl.final_cost;
      res.trace_rows = trace_rows;
      res.pose = res.ok ? pose_inverse(ctl.c2w) : (a.initial ? *a.initial : ctl.render);
      if (res.ok && a.update_state) *a.state_pose = res.pose;  // pipeline_impl.hpp:83 — hold the pose on failure
      *a.result = res;
    }
  }
}

__global__ void __launch_bounds__(kIcpThreads, VF_ICP_MIN_BLOCKS) k_icp(IcpArgs a) { icp_body<false>(a); }
__global__ void __launch_bounds__(kIcpThreads, VF_ICP_MIN_BLOCKS) k_icp_cluster(IcpArgs a) { icp_body<true>(a); }

}  // namespace vf
