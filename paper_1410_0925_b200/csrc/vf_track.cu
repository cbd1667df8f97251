// The reference's other trackers, on the device: SDF-based Ren refinement
// (TrackerType::icp_ren) and the photometric colour tracker
// (TrackerType::color).
//
// Reference: ren_refine / ren_point_energy / ren_point_residual
// (proj/include/voxfuse/engine/ren_tracker.hpp:14-120), trilinear_sdf_gradient
// (engine/raycast.hpp:119-142), color_track / detail::evaluate_color
// (engine/color_tracker.hpp:14-154), build_color_pyramid / downsample_mean /
// image_gradients (engine/pyramid.hpp:66-132), sample_bilinear
// (core/image.hpp:57-75), and their place in Pipeline::track
// (engine/pipeline_impl.hpp:180-209).
//
// Ren: one Gauss-Newton iteration = k_ren_terms (every valid full-resolution
// pixel: back-projection, trilinear SDF + analytic gradient from the hash
// volume, FP64 Jacobian, 21 + 6 + 2 sums reduced per CTA) then k_ren_ctl (one
// warp sums the CTA partials in a fixed order and runs the reference's
// controller: minimum count, gradient-norm exit, SVD condition test, LDLT
// solve, pose increment, convergence).  max_iterations pairs are captured in
// the frame graph; once the controller finishes, the remaining launches
// return immediately.
//
// Colour: the surface list forward-projected by the previous frame is a few
// thousand points, so the whole coarse-to-fine Levenberg-Marquardt runs in
// one 1024-thread CTA: each evaluation is a block reduction of 29 FP64 sums,
// thread 0 runs the damping / accept / reject logic, and nothing leaves the
// SM until the pose is decided.
#include <cooperative_groups.h>

#include "vf_device.cuh"
#include "vf_kernels.h"
#include "vf_solve.cuh"

namespace vf {

namespace {

// HashSdfSampler::read (raycast.hpp:73-76): value, found && w_depth > 0
__device__ __forceinline__ bool sdf_read(const HashView& hv, const uint32_t* __restrict__ vox, int stride, int vx,
                                         int vy, int vz, float& value) {
  const int s = find_slot(hv, vx >> 3, vy >> 3, vz >> 3);
  if (s < 0) {
    value = 1.0f;
    return false;
  }
  const uint32_t r = __ldg(vox + ((size_t)s * kBlockVolume + ((vx & 7) + (vy & 7) * 8 + (vz & 7) * 64)) * stride);
  value = sdf_to_float((int16_t)(r & 0xFFFFu));
  return ((r >> 16) & 0xFFu) > 0;
}

// trilinear_sdf + trilinear_sdf_gradient (raycast.hpp:102-142) on one set of
// eight corner reads (both read the same corners of the same base).
__device__ bool trilinear_value_grad(const HashView& hv, const uint32_t* __restrict__ vox, int stride, F3 p,
                                     float& value, F3& g) {
  const float qx = p.x - 0.5f, qy = p.y - 0.5f, qz = p.z - 0.5f;
  const int x0 = __float2int_rz(floorf(qx)), y0 = __float2int_rz(floorf(qy)), z0 = __float2int_rz(floorf(qz));
  const float fx = qx - (float)x0, fy = qy - (float)y0, fz = qz - (float)z0;
  float v[8];
  for (int corner = 0; corner < 8; ++corner) {
    const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
    if (!sdf_read(hv, vox, stride, x0 + dx, y0 + dy, z0 + dz, v[corner])) return false;
  }
  float acc = 0.0f;
  for (int corner = 0; corner < 8; ++corner) {
    const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
    const float w = (dx ? fx : 1 - fx) * (dy ? fy : 1 - fy) * (dz ? fz : 1 - fz);
    acc += w * v[corner];
  }
  value = acc;
  // v[dx][dy][dz] = v[dx | dy << 1 | dz << 2]
#define V(a, b, c) v[(a) | ((b) << 1) | ((c) << 2)]
  auto lerp = [](float a, float b, float t) { return a + (b - a) * t; };
  g.x = lerp(lerp(V(1, 0, 0) - V(0, 0, 0), V(1, 1, 0) - V(0, 1, 0), fy),
             lerp(V(1, 0, 1) - V(0, 0, 1), V(1, 1, 1) - V(0, 1, 1), fy), fz);
  g.y = lerp(lerp(V(0, 1, 0) - V(0, 0, 0), V(1, 1, 0) - V(1, 0, 0), fx),
             lerp(V(0, 1, 1) - V(0, 0, 1), V(1, 1, 1) - V(1, 0, 1), fx), fz);
  g.z = lerp(lerp(V(0, 0, 1) - V(0, 0, 0), V(1, 0, 1) - V(1, 0, 0), fx),
             lerp(V(0, 1, 1) - V(0, 1, 0), V(1, 1, 1) - V(1, 1, 0), fx), fy);
#undef V
  return true;
}

__device__ __forceinline__ void acc_jacobian(double (&acc)[32], const double* j, double r) {
  int k = 0;
#pragma unroll
  for (int a = 0; a < 6; ++a) {
#pragma unroll
    for (int b = a; b < 6; ++b) acc[k++] += j[a] * j[b];
    acc[21 + a] += j[a] * r;
  }
}

// Block reduction of 32 per-thread values (blockDim.x a multiple of 32,
// <= 1024); the CTA total of value k lands in out[k] (thread 0's view after
// the barrier).
__device__ void block_reduce32(double (&acc)[32], double* s_red /* [32][32] */, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double v = warp_reduce32(acc);  // lane l: warp sum of value l
  s_red[wid * 32 + lane] = v;
  __syncthreads();
  if (wid == 0) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += s_red[w * 32 + lane];
    out[lane] = t;
  }
  __syncthreads();
}

}  // namespace

// ---------------------------------------------------------------------------
// Ren refinement
// ---------------------------------------------------------------------------
__global__ void k_ren_init(const IcpResult* __restrict__ icp, const PoseD* __restrict__ state, int use_icp,
                           const PoseD* __restrict__ explicit_init, RenCtl* __restrict__ ctl) {
  pdl_enter();
  if (threadIdx.x != 0) return;
  PoseD init = *state;
  if (explicit_init) init = *explicit_init;
  else if (use_icp && icp->ok) init = icp->pose;  // pipeline_impl.hpp:197
  ctl->init = init;
  ctl->c2w = pose_inverse(init);
  ctl->final_cost = 0.0;
  ctl->iterations = 0;
  ctl->valid_points = 0;
  ctl->done = 0;
  ctl->ok = 0;
}

// one iteration's per-pixel terms (ren_tracker.hpp:53-80)
__global__ void __launch_bounds__(256) k_ren_terms(const float* __restrict__ depth, IntrD in, HashView hv,
                                                   const uint32_t* __restrict__ vox, int vstride, float vs,
                                                   double sigma, const RenCtl* __restrict__ ctl,
                                                   double* __restrict__ partials) {
  pdl_enter();
  __shared__ double s_red[32 * 32];
  __shared__ double s_out[32];
  if (ctl->done) return;
  const PoseD c2w = ctl->c2w;
  double acc[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) acc[k] = 0.0;
  const int npix = in.width * in.height;
  const float fsigma = (float)sigma;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npix; i += gridDim.x * blockDim.x) {
    const float d = __ldg(depth + i);
    if (d <= 0.0f) continue;
    const int x = i % in.width, y = i / in.width;
    // unproject (intrinsics.hpp:41-43) then cam_to_world.apply
    const double dd = (double)d;
    const D3 pc = mk((x - in.cx) / in.fx * dd, (y - in.cy) / in.fy * dd, dd);
    const D3 pw = apply(c2w, pc);
    const F3 pv{(float)(pw.x / (double)vs), (float)(pw.y / (double)vs), (float)(pw.z / (double)vs)};
    float sdf;
    F3 g;
    if (!trilinear_value_grad(hv, vox, vstride, pv, sdf, g)) continue;
    const D3 gw = mk((double)g.x / (double)vs, (double)g.y / (double)vs, (double)g.z / (double)vs);
    const double r = (double)tanhf(0.5f * fsigma * sdf);  // ren_point_residual
    const double dr = (1.0 - r * r) * 0.5 * sigma;
    // p_world x grad_world
    const D3 cr = mk(pw.y * gw.z - pw.z * gw.y, pw.z * gw.x - pw.x * gw.z, pw.x * gw.y - pw.y * gw.x);
    const double j[6] = {dr * cr.x, dr * cr.y, dr * cr.z, dr * gw.x, dr * gw.y, dr * gw.z};
    acc_jacobian(acc, j, r);
    const float es = expf(fsigma * sdf);  // ren_point_energy
    acc[27] += (double)(-4.0f * es / ((es + 1.0f) * (es + 1.0f)));
    acc[28] += 1.0;
  }
  block_reduce32(acc, s_red, s_out);
  if (threadIdx.x < 29) partials[(size_t)blockIdx.x * 32 + threadIdx.x] = s_out[threadIdx.x];
}

// the reference's per-iteration control (ren_tracker.hpp:82-110)
__global__ void k_ren_ctl(const double* __restrict__ partials, int nparts, RenCtl* __restrict__ ctl,
                          int min_valid_points, double max_condition, float convergence_eps) {
  pdl_enter();
  __shared__ double s_tot[32];
  if (ctl->done) return;
  const int lane = threadIdx.x;
  double t = 0.0;
  if (lane < 29) {  // CTA order; eight loads in flight per step
    int b = 0;
    for (; b + 8 <= nparts; b += 8) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = partials[(size_t)(b + k) * 32 + lane];
#pragma unroll
      for (int k = 0; k < 8; ++k) t += v[k];
    }
    for (; b < nparts; ++b) t += partials[(size_t)b * 32 + lane];
  }
  s_tot[lane] = t;
  __syncwarp();
  if (lane != 0) return;
  const double* tot = s_tot;
  const long long count = (long long)tot[28];
  if (count < min_valid_points) {  // tracking fails, input pose kept
    ctl->done = 1;
    return;
  }
  ctl->valid_points = (int)count;
  ctl->final_cost = tot[27] / (double)count;
  double gn = 0.0;
  for (int a = 0; a < 6; ++a) gn += tot[21 + a] * tot[21 + a];
  if (sqrt(gn) < 1e-12) {  // already at the minimum
    ctl->done = 1;
    ctl->ok = 1;
    return;
  }
  double twist[6];
  // the register LDL^T with the condition bound (as K4's controller); the
  // reference's pivoted LDLT + SVD test only when the bound is inconclusive
  if (!spd_solve_fast<6>(tot, max_condition, twist)) {
    double h[36];
    for (int a = 0, k = 0; a < 6; ++a)
      for (int b = a; b < 6; ++b, ++k) h[a * 6 + b] = h[b * 6 + a] = tot[k];
    Ldlt f;
    f.compute(h, 6);
    if (!well_conditioned(h, 6, f, max_condition)) {
      ctl->done = 1;
      return;
    }
    double ng[6];
    for (int a = 0; a < 6; ++a) ng[a] = -tot[21 + a];
    f.solve(ng, twist);
  }
  ctl->c2w = pose_increment(ctl->c2w, twist, false);
  ++ctl->iterations;
  double tn = 0.0;
  for (int a = 0; a < 6; ++a) tn += twist[a] * twist[a];
  if (sqrt(tn) < (double)convergence_eps) {
    ctl->done = 1;
    ctl->ok = 1;
  }
}

// ren_refine's result (ren_tracker.hpp:112-116) and, for icp_ren, Pipeline::track's
// combination with the coarse ICP (pipeline_impl.hpp:189-201); writes the
// frame's TrackingResult and, when ok and update_state, the pose.
__global__ void k_ren_finish(RenCtl* __restrict__ ctl, int combine_icp, IcpResult* __restrict__ res,
                             PoseD* __restrict__ state, int update_state) {
  pdl_enter();
  if (threadIdx.x != 0) return;
  const bool ok = ctl->done ? ctl->ok != 0 : true;  // max_iterations reached: ok
  IcpResult out;
  if (ok) {
    out.pose = pose_inverse(ctl->c2w);
    out.ok = 1;
    out.iterations = ctl->iterations + (combine_icp ? res->iterations : 0);
    out.final_cost = ctl->final_cost;
    out.valid_points = ctl->valid_points;
  } else if (combine_icp) {
    out = *res;  // ren failed: the coarse ICP's result stands
  } else {
    out.pose = ctl->init;
    out.ok = 0;
    out.iterations = 0;
    out.final_cost = ctl->final_cost;
    out.valid_points = ctl->valid_points;
  }
  out.trace_rows = res->trace_rows;
  *res = out;
  ctl->done = 1;
  if (update_state && out.ok) *state = out.pose;
}

// ---------------------------------------------------------------------------
// Colour pyramid (pyramid.hpp:66-132); colours as float4 (w unused)
// ---------------------------------------------------------------------------
__global__ void k_cpyr_base(const uint8_t* __restrict__ rgb, int n, float4* __restrict__ out) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = make_float4((float)rgb[3 * i] / 255.0f, (float)rgb[3 * i + 1] / 255.0f, (float)rgb[3 * i + 2] / 255.0f,
                       0.0f);
}

// downsample_mean: sum of the in-bounds 2x2 samples times 1 / n
__global__ void k_cpyr_down(const float4* __restrict__ src, int sw, int sh, float4* __restrict__ dst) {
  pdl_enter();
  const int dw = (sw + 1) / 2, dh = (sh + 1) / 2;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dw * dh) return;
  const int x = i % dw, y = i / dw;
  float sx = 0.0f, sy = 0.0f, sz = 0.0f;
  int n = 0;
  for (int dy = 0; dy < 2; ++dy)
    for (int dx = 0; dx < 2; ++dx) {
      const int px = 2 * x + dx, py = 2 * y + dy;
      if (px >= sw || py >= sh) continue;
      const float4 v = src[(size_t)py * sw + px];
      sx += v.x;
      sy += v.y;
      sz += v.z;
      ++n;
    }
  const float r = 1.0f / (float)n;
  dst[i] = make_float4(sx * r, sy * r, sz * r, 0.0f);
}

// image_gradients: central differences, zero on the border
__global__ void k_cpyr_grad(const float4* __restrict__ src, int w, int h, float4* __restrict__ gx,
                            float4* __restrict__ gy) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= w * h) return;
  const int x = i % w, y = i / w;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
  if (x >= 1 && y >= 1 && x + 1 < w && y + 1 < h) {
    const float4 xp = src[i + 1], xm = src[i - 1], yp = src[i + w], ym = src[i - w];
    a = make_float4((xp.x - xm.x) * 0.5f, (xp.y - xm.y) * 0.5f, (xp.z - xm.z) * 0.5f, 0.0f);
    b = make_float4((yp.x - ym.x) * 0.5f, (yp.y - ym.y) * 0.5f, (yp.z - ym.z) * 0.5f, 0.0f);
  }
  gx[i] = a;
  gy[i] = b;
}

namespace {

// sample_bilinear (image.hpp:57-75) on a float4 (Vec3f) image
__device__ __forceinline__ bool sample_bilinear3(const float4* __restrict__ img, int w, int h, float x, float y,
                                                 F3& out) {
  if (x < 0.f || y < 0.f || x > (float)(w - 1) || y > (float)(h - 1)) return false;
  int ix = min((int)x, w - 2), iy = min((int)y, h - 2);
  if (w == 1) ix = 0;
  if (h == 1) iy = 0;
  const float fx = x - (float)ix, fy = y - (float)iy;
  const int x1 = min(ix + 1, w - 1), y1 = min(iy + 1, h - 1);
  const float4 A = img[(size_t)iy * w + ix], B = img[(size_t)iy * w + x1];
  const float4 Cc = img[(size_t)y1 * w + ix], D = img[(size_t)y1 * w + x1];
  const float wa = (1.f - fx) * (1.f - fy), wb = fx * (1.f - fy), wc = (1.f - fx) * fy, wd = fx * fy;
  out.x = A.x * wa + B.x * wb + Cc.x * wc + D.x * wd;
  out.y = A.y * wa + B.y * wb + Cc.y * wc + D.y * wd;
  out.z = A.z * wa + B.z * wb + Cc.z * wc + D.z * wd;
  return true;
}

// detail::evaluate_color (color_tracker.hpp:24-101): one CTA, every thread a
// share of the points; acc: 21 H, 6 g, cost, count.
__device__ void evaluate_color(const float* __restrict__ pts, const float* __restrict__ cols, int n, int stride,
                               const ColorLevel& lv, const PoseD& w2c, double* s_red, double* s_out) {
  double acc[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) acc[k] = 0.0;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) * stride; i < n; i += gridDim.x * blockDim.x * stride) {
    const D3 p = mk((double)pts[3 * i], (double)pts[3 * i + 1], (double)pts[3 * i + 2]);
    const D3 q = apply(w2c, p);
    if (q.z <= 0.0) continue;
    const double u = lv.fx * q.x / q.z + lv.cx, v = lv.fy * q.y / q.z + lv.cy;  // project
    F3 smp;
    if (!sample_bilinear3(lv.color, lv.w, lv.h, (float)u, (float)v, smp)) continue;
    const float rx = smp.x - cols[3 * i], ry = smp.y - cols[3 * i + 1], rz = smp.z - cols[3 * i + 2];
    acc[27] += (double)(rx * rx + ry * ry + rz * rz);
    acc[28] += 1.0;
    F3 gx, gy;
    if (!sample_bilinear3(lv.gx, lv.w, lv.h, (float)u, (float)v, gx) ||
        !sample_bilinear3(lv.gy, lv.w, lv.h, (float)u, (float)v, gy))
      continue;
    // dpi (2x3) * dq (3x6), dq = [-skew(q) | I], products summed left to right
    const double qz2 = q.z * q.z;
    const double a00 = lv.fx / q.z, a02 = -lv.fx * q.x / qz2;
    const double a11 = lv.fy / q.z, a12 = -lv.fy * q.y / qz2;
    const double dq[3][6] = {{-0.0, q.z, -q.y, 1.0, 0.0, 0.0},
                             {-q.z, -0.0, q.x, 0.0, 1.0, 0.0},
                             {q.y, -q.x, -0.0, 0.0, 0.0, 1.0}};
    double r0[6], r1[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      r0[c] = a00 * dq[0][c] + 0.0 * dq[1][c] + a02 * dq[2][c];
      r1[c] = 0.0 * dq[0][c] + a11 * dq[1][c] + a12 * dq[2][c];
    }
    const float gxs[3] = {gx.x, gx.y, gx.z}, gys[3] = {gy.x, gy.y, gy.z}, rs[3] = {rx, ry, rz};
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      double j[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) j[c] = (double)gxs[ch] * r0[c] + (double)gys[ch] * r1[c];
      acc_jacobian(acc, j, (double)rs[ch]);
    }
  }
  block_reduce32(acc, s_red, s_out);
}

// evaluate_color over a cooperative grid: every CTA reduces its share, the
// per-CTA sums meet behind one grid barrier (double-buffered), and every CTA
// adds them in CTA order, so all CTAs hold identical sums and take identical
// decisions.  One CTA: evaluate_color itself.
__device__ void evaluate_color_grid(const ColorTrackArgs& a, int n, const ColorLevel& lv, const PoseD& w2c,
                                    double* s_red, double* s_out, int& buf) {
  evaluate_color(a.points, a.colors, n, a.stride, lv, w2c, s_red, s_out);
  if (gridDim.x == 1) return;
  double* part = a.partials + (size_t)buf * gridDim.x * 32;
  if (threadIdx.x < 29) part[(size_t)blockIdx.x * 32 + threadIdx.x] = s_out[threadIdx.x];
  cooperative_groups::this_grid().sync();
  if (threadIdx.x < 29) {
    double t = 0.0;
    int b = 0;
    for (; b + 8 <= (int)gridDim.x; b += 8) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldcg(part + (size_t)(b + k) * 32 + threadIdx.x);
#pragma unroll
      for (int k = 0; k < 8; ++k) t += v[k];
    }
    for (; b < (int)gridDim.x; ++b) t += __ldcg(part + (size_t)b * 32 + threadIdx.x);
    s_out[threadIdx.x] = t;
  }
  __syncthreads();
  buf ^= 1;
}

}  // namespace

// color_track (color_tracker.hpp:107-154), in one CTA or over a cooperative
// grid (every CTA runs the same damping logic on the same sums).  Writes the
// frame's TrackingResult; the pose when ok and update_state.
__global__ void __launch_bounds__(kColorThreads) k_color_track(ColorTrackArgs a) {
  pdl_wait();
  __shared__ double s_red[32 * 32];
  __shared__ double s_eval[32], s_trial[32];
  __shared__ PoseD s_pose, s_cand;
  __shared__ int s_flag;  // 0 continue, 1 leave the level
  __shared__ double s_twist_norm;
  const int n = a.count ? *a.count : a.n;
  const PoseD init = a.explicit_init ? *a.explicit_init : *a.state;
  int iterations_total = 0;
  bool any_level_ok = false;
  double final_cost = 0.0;
  int valid_points = 0;
  if (threadIdx.x == 0) s_pose = init;
  __syncthreads();
  const bool have = n > 0;  // points.empty() -> not ok (color_tracker.hpp:111)
  int buf = 0;
  for (int level = a.levels - 1; have && level >= 0; --level) {
    const ColorLevel& lv = a.lv[level];
    double lambda = 0.01;
    evaluate_color_grid(a, n, lv, s_pose, s_red, s_eval, buf);
    if ((long long)s_eval[28] < a.min_valid_points) continue;
    any_level_ok = true;
    for (int iter = 0; iter < a.max_iterations; ++iter) {
      // default: the unrolled register LDLT, the pivoted path only when the
      // damped system is not numerically SPD; exact_solve: always pivoted
      // (the reference's LDLT, so accept / convergence ties resolve alike)
      if (!a.exact_solve && threadIdx.x == 0) {
        double tw[6];
        if (spd_solve_damped6(s_eval, lambda, tw)) {
          s_flag = 0;
          s_cand = pose_increment(s_pose, tw, false);
          double tn = 0.0;
          for (int p = 0; p < 6; ++p) tn += tw[p] * tw[p];
          s_twist_norm = sqrt(tn);
        } else {
          s_flag = 2;  // not numerically SPD: the reference's pivoted path below
        }
      }
      __syncthreads();
      if ((a.exact_solve || s_flag == 2) && threadIdx.x == 0) {
        s_flag = 0;
        double h[36];
        for (int p = 0, k = 0; p < 6; ++p)
          for (int q = p; q < 6; ++q, ++k) h[p * 6 + q] = h[q * 6 + p] = s_eval[k];
        for (int p = 0; p < 6; ++p) h[p * 6 + p] *= (1.0 + lambda);  // damped.diagonal() *= (1 + lambda)
        Ldlt f;
        f.compute(h, 6);
        if (f.issue) {
          s_flag = 1;
        } else {
          double ng[6], tw[6];
          for (int p = 0; p < 6; ++p) ng[p] = -s_eval[21 + p];
          f.solve(ng, tw);
          s_cand = pose_increment(s_pose, tw, false);
          double tn = 0.0;
          for (int p = 0; p < 6; ++p) tn += tw[p] * tw[p];
          s_twist_norm = sqrt(tn);
        }
      }
      __syncthreads();
      if (s_flag) break;
      evaluate_color_grid(a, n, lv, s_cand, s_red, s_trial, buf);
      ++iterations_total;
      const double ec = s_eval[28] > 0 ? s_eval[27] / s_eval[28] : 0.0;
      const double tc = s_trial[28] > 0 ? s_trial[27] / s_trial[28] : 0.0;
      bool leave = false;
      if ((long long)s_trial[28] >= a.min_valid_points && tc < ec) {
        __syncthreads();
        if (threadIdx.x == 0) s_pose = s_cand;
        if (threadIdx.x < 32) s_eval[threadIdx.x] = s_trial[threadIdx.x];
        lambda = fmax(lambda * 0.1, 1e-7);
        if (s_twist_norm < (double)a.convergence_eps) leave = true;
      } else {
        lambda *= 10.0;
        if (lambda > 1e7) leave = true;
      }
      __syncthreads();
      final_cost = s_eval[28] > 0 ? s_eval[27] / s_eval[28] : 0.0;
      if (leave) break;
    }
    final_cost = s_eval[28] > 0 ? s_eval[27] / s_eval[28] : 0.0;
    valid_points = (int)s_eval[28];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    IcpResult r;
    r.final_cost = final_cost;
    r.valid_points = valid_points;
    r.trace_rows = 0;
    if (!any_level_ok) {
      r.pose = init;
      r.ok = 0;
      r.iterations = 0;
    } else {
      r.pose = s_pose;
      r.ok = 1;
      r.iterations = iterations_total;
    }
    *a.result = r;
    if (a.update_state && r.ok) *a.state = r.pose;
  }
}

// Pipeline::track for the colour tracker without an RGB frame or surface list
// (pipeline_impl.hpp:183-185): {state.pose, false, 0, 0.0, 0}.
__global__ void k_track_fail(const PoseD* __restrict__ state, IcpResult* __restrict__ res) {
  if (threadIdx.x != 0) return;
  IcpResult r;
  r.pose = *state;
  r.ok = 0;
  r.iterations = 0;
  r.final_cost = 0.0;
  r.valid_points = 0;
  r.trace_rows = 0;
  *res = r;
}

}  // namespace vf
