// Support kernels: synthetic depth/RGB rendering for benchmark inputs, VBA
// initialisation, compact-list rebuild after a state import, range reset.
#include "vf_device.cuh"
#include "vf_kernels.h"

namespace vf {

// render_synthetic_depth / render_synthetic_rgb (reference proj/src/synthetic.cpp:19-108),
// one thread per pixel, FP64 like the reference.  Used to generate the bench
// inputs on the device (the CPU oracle restates the same renderer for tests).
__global__ void __launch_bounds__(256) k_synth(int n_spheres, const double* __restrict__ spheres, int n_planes,
                                               const double* __restrict__ planes, PoseD c2w, IntrD in,
                                               double near_clip, double far_clip, float* __restrict__ depth,
                                               uint8_t* __restrict__ rgb) {
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= in.width * in.height) return;
  const int y = pix / in.width, x = pix - y * in.width;
  const D3 origin = mk(c2w.t[0], c2w.t[1], c2w.t[2]);
  const D3 dir = mat_vec(c2w.r, mk((x - in.cx) / in.fx, (y - in.cy) / in.fy, 1.0));
  double best_t = __longlong_as_double(0x7ff0000000000000ll);
  D3 best_p = mk(0, 0, 0), best_n = mk(0, 0, 0);
  float alb[3] = {0.f, 0.f, 0.f};
  for (int i = 0; i < n_spheres; ++i) {
    const double* s = spheres + 7 * i;
    const D3 oc = mk(origin.x - s[0], origin.y - s[1], origin.z - s[2]);
    const double a = dir.x * dir.x + dir.y * dir.y + dir.z * dir.z;
    const double b = 2.0 * (oc.x * dir.x + oc.y * dir.y + oc.z * dir.z);
    const double c = (oc.x * oc.x + oc.y * oc.y + oc.z * oc.z) - s[3] * s[3];
    const double disc = b * b - 4 * a * c;
    if (disc < 0) continue;
    const double sq = sqrt(disc);
    const double ts[2] = {(-b - sq) / (2 * a), (-b + sq) / (2 * a)};
    for (int k = 0; k < 2; ++k) {
      const double t = ts[k];
      if (t > near_clip && t < far_clip && t < best_t) {
        best_t = t;
        best_p = mk(origin.x + t * dir.x, origin.y + t * dir.y, origin.z + t * dir.z);
        const D3 nn = mk(best_p.x - s[0], best_p.y - s[1], best_p.z - s[2]);
        const double len = sqrt(nn.x * nn.x + nn.y * nn.y + nn.z * nn.z);
        best_n = len > 0 ? mk(nn.x / len, nn.y / len, nn.z / len) : nn;
        alb[0] = (float)s[4];
        alb[1] = (float)s[5];
        alb[2] = (float)s[6];
      }
    }
  }
  for (int i = 0; i < n_planes; ++i) {
    const double* p = planes + 9 * i;
    const double denom = p[0] * dir.x + p[1] * dir.y + p[2] * dir.z;
    if (fabs(denom) < 1e-12) continue;
    const double t = (p[3] - (p[0] * origin.x + p[1] * origin.y + p[2] * origin.z)) / denom;
    if (t > near_clip && t < far_clip && t < best_t) {
      best_t = t;
      best_p = mk(origin.x + t * dir.x, origin.y + t * dir.y, origin.z + t * dir.z);
      best_n = denom < 0 ? mk(p[0], p[1], p[2]) : mk(-p[0], -p[1], -p[2]);
      float a3[3] = {(float)p[4], (float)p[5], (float)p[6]};
      if (p[7] != 0.0) {
        const double na[3] = {fabs(p[0]), fabs(p[1]), fabs(p[2])};
        int drop = 0;
        if (na[1] > na[drop]) drop = 1;
        if (na[2] > na[drop]) drop = 2;
        const double pt[3] = {best_p.x, best_p.y, best_p.z};
        double uv[2] = {0, 0};
        int k = 0;
        for (int axis = 0; axis < 3; ++axis) {
          if (axis == drop) continue;
          uv[k++] = pt[axis];
        }
        const long long pu = (long long)floor(uv[0] / p[8]);
        const long long pv = (long long)floor(uv[1] / p[8]);
        if (((pu + pv) & 1) != 0)
          for (int ch = 0; ch < 3; ++ch) a3[ch] *= 0.35f;
      }
      alb[0] = a3[0];
      alb[1] = a3[1];
      alb[2] = a3[2];
    }
  }
  const bool valid = best_t < __longlong_as_double(0x7ff0000000000000ll);
  if (depth) depth[pix] = valid ? (float)best_t : 0.0f;
  if (rgb) {
    uint8_t* o = rgb + 3 * (size_t)pix;
    if (!valid) {
      o[0] = o[1] = o[2] = 0;
      return;
    }
    // light = (0.3, -0.7, -0.5).normalized()
    const double l0 = 0.3, l1 = -0.7, l2 = -0.5;
    const double ll = sqrt(l0 * l0 + l1 * l1 + l2 * l2);
    const D3 light = mk(l0 / ll, l1 / ll, l2 / ll);
    const double dd = best_n.x * -light.x + best_n.y * -light.y + best_n.z * -light.z;
    const float shade = 0.3f + 0.7f * (float)(0.0 < dd ? dd : 0.0);
    for (int ch = 0; ch < 3; ++ch) {
      const float cv = alb[ch] * shade * 255.0f;
      o[ch] = (uint8_t)__float2int_rz(cv < 255.f ? cv : 255.f);
    }
  }
}

// VoxelS{} / VoxelSRgb{}: sdf 32767, weights 0 (voxel.hpp:29-46).
// disparity_image_to_depth / disparity_to_depth (engine/view.hpp:18-28,
// io/calibration.hpp:45-60); big_endian: the samples are the raw bytes of a
// 16-bit P5 raster (read_pgm16, src/pnm.cpp:63-73), byte-swapped here.
__global__ void k_disparity_to_depth(const uint16_t* __restrict__ disp, int n, int big_endian, float a, float b,
                                     float fx, float max_depth, float* __restrict__ depth) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t d = __ldg(disp + i);
  if (big_endian) d = ((d & 0xFFu) << 8) | (d >> 8);
  const float denom = a - (float)d;
  float z = 0.0f;
  if (!(denom <= 0.0f)) {
    const float v = 8.0f * b * fx / denom;
    z = (v > 0.0f && v <= max_depth) ? v : 0.0f;
  }
  depth[i] = z;
}

__global__ void k_fill_voxels(uint32_t* __restrict__ vox, size_t n_voxels, int words_per_voxel) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_voxels; i += (size_t)gridDim.x * blockDim.x) {
    vox[i * words_per_voxel] = 0x00007FFFu;
    if (words_per_voxel == 2) vox[i * 2 + 1] = 0u;
  }
}

// Compact list of allocated / swapped-out entries after vf_import_state.
__global__ void k_rebuild_alloc_list(const HashEntry* __restrict__ entries, int n, int* __restrict__ alloc_list,
                                     int cap, Counters* __restrict__ ctr) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const HashEntry e = load_entry(entries + i);
    if (e.block_state >= kEntrySwappedOut) {
      const int pos = warp_aggregated_add(&ctr->alloc_count);
      if (pos < cap) alloc_list[pos] = i;
    }
  }
}

__global__ void k_init_ranges(float2* ranges, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    ranges[i] = make_float2(3.402823466e+38f, 0.0f);
}

// Self-test of div_rr against the IEEE operator (tests/test_gpu_kernels.py).
// mode 0: every float a with amin <= |a| <= amax (both signs), and a = 0, for the divisor b.
__global__ void k_divtest_const(float b, uint32_t lo_bits, uint32_t n_bits, unsigned long long* __restrict__ mism) {
  const float rb = rcp_refined(b);
  unsigned long long bad = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) bad += (0.0f / b != div_rr(0.0f, b, rb));
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_bits; i += gridDim.x * blockDim.x) {
    const float a = __uint_as_float(lo_bits + i);
    bad += (a / b != div_rr(a, b, rb)) + (-a / b != div_rr(-a, b, rb));
  }
  if (bad) atomicAdd(mism, bad);
}
// mode 1: n pseudo-random pairs, a uniform in [-amax, amax], b log-uniform in [bmin, bmax].
__global__ void k_divtest_rand(float amax, float bmin, float bmax, unsigned long long n,
                               unsigned long long* __restrict__ mism) {
  unsigned long long bad = 0;
  const float lb0 = __logf(bmin), lb1 = __logf(bmax);
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    unsigned long long x = i * 0x9E3779B97F4A7C15ull + 0x14100925ull;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
    const float ua = (float)(x & 0xFFFFFF) * (1.0f / 16777216.0f), ub = (float)((x >> 24) & 0xFFFFFF) * (1.0f / 16777216.0f);
    const float a = (2.0f * ua - 1.0f) * amax;
    const float b = __expf(lb0 + (lb1 - lb0) * ub) * ((x >> 63) ? -1.0f : 1.0f);
    bad += a / b != div_rr(a, b, rcp_refined(b));
  }
  if (bad) atomicAdd(mism, bad);
}

// vf_set_pose: the pose travels as a kernel parameter, captured at launch, so
// the host may set the next frame's pose while earlier frames are in flight.
__global__ void k_set_pose(PoseD* dst, PoseD pose) {
  if (threadIdx.x < 12) {
    const double* src = threadIdx.x < 9 ? pose.r + threadIdx.x : pose.t + (threadIdx.x - 9);
    double* d = threadIdx.x < 9 ? dst->r + threadIdx.x : dst->t + (threadIdx.x - 9);
    *d = *src;
  }
}

__global__ void k_reset_visible(Counters* ctr) {
  if (threadIdx.x == 0 && blockIdx.x == 0) ctr->visible_count = 0;
}

}  // namespace vf
