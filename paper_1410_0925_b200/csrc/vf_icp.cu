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
// The per-iteration pixel pass is software-pipelined one pixel deep: the next
// pixel's transforms run and its map taps are fetched into shared memory with
// cp.async while the current pixel's terms are summed.
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
#include "vf_solve.cuh"

namespace cg = cooperative_groups;

namespace vf {

// ---------------------------------------------------------------------------
// pyramid
// ---------------------------------------------------------------------------
// One CTA per 32x32 tile of level 0; levels 1..L-1 of the tile are built in
// shared memory (32 = 2^5 keeps tiles aligned for up to 6 levels).
__global__ void __launch_bounds__(256) k_pyramid(const float* __restrict__ depth0, int w0, int h0, int levels,
                                                 float* __restrict__ out /* levels 1.. back to back */) {
  pdl_enter();
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

// 16-byte cp.async into shared memory (L1-allocating); n = 0 zero-fills
// without reading global memory.
__device__ __forceinline__ void cp_async16(float4* dst_smem, const float4* src, unsigned n) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n) : "memory");
}

// What the front half of a pipelined ICP step hands its back half.
struct IcpStage {
  D3 pw[kInflight];
  double fx[kInflight], fy[kInflight];
  bool ok[kInflight];
};

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
// Sharded ICP: the iteration's 29 sums, summed across the
// shards inside the persistent kernel over peer memory (NVLink P2P / CUDA IPC
// mappings) -- the allreduce fused into the ICP loop, no kernel boundary and
// no host round trip.  CTA 0 of each shard writes its total into every
// shard's exchange area and raises its flag there (release, system scope),
// waits for all shards' flags in its own area (acquire), sums the totals in
// shard order -- identical on every shard, so every controller takes the
// same decision -- and hands the sum to its own CTAs through a local flag.
// Exchanges alternate between two parities: a shard can only write parity p
// again after every shard published the exchange in between, i.e. after every
// shard finished reading p.  If a peer does not answer within ~0.5 s the sum
// is replaced by zeros (count 0: every level is left, tracking fails) and an
// error flag is raised, so a missing shard cannot hang the frame.
__device__ __forceinline__ void shard_exchange(const IcpArgs& a, unsigned long long seq, double* s_tot, int tid) {
  __shared__ int s_bad;
  const int par = (int)(seq & 1ull);
  unsigned long long* local = a.xstate;  // [0] counter, [1] local flag, [2 + 32 * par + i] summed totals
  if (blockIdx.x == 0) {
    if (tid < kAcc)
      for (int r = 0; r < a.xranks; ++r) a.xpeer[r][kXchgTotals + (par * 16 + a.xrank) * 32 + tid] = s_tot[tid];
    __syncthreads();
    if (tid == 0) {
      __threadfence_system();
      for (int r = 0; r < a.xranks; ++r) {
        unsigned long long* f = reinterpret_cast<unsigned long long*>(a.xpeer[r] + kXchgFlags) + par * 16 + a.xrank;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(seq) : "memory");
      }
      const unsigned long long* own = reinterpret_cast<const unsigned long long*>(a.xpeer[a.xrank] + kXchgFlags);
      int bad = 0;
      for (int r = 0; r < a.xranks && !bad; ++r) {
        unsigned long long v = 0;
        for (long spin = 0;; ++spin) {
          asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(own + par * 16 + r) : "memory");
          if (v >= seq) break;
          if (spin > (1l << 22)) {
            bad = 1;
            break;
          }
          __nanosleep(64);
        }
      }
      s_bad = bad;
      if (bad) atomicOr(&a.ctr->error_flags, kErrShardXchg);
    }
    __syncthreads();
    if (tid < kAcc) {
      double t = 0;
      const double* tot = a.xpeer[a.xrank] + kXchgTotals;
      for (int r = 0; r < a.xranks; ++r) t += *reinterpret_cast<const volatile double*>(tot + (par * 16 + r) * 32 + tid);
      reinterpret_cast<double*>(local + 2)[32 * par + tid] = s_bad ? 0.0 : t;
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(local + 1), "l"(seq) : "memory");
    }
  } else if (tid == 0) {
    unsigned long long v = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(local + 1) : "memory");
    } while (v < seq);
  }
  __syncthreads();
  if (tid < kAcc) s_tot[tid] = *reinterpret_cast<const volatile double*>(reinterpret_cast<double*>(local + 2) + 32 * par + tid);
  __syncthreads();
}

template <bool kCluster>
__device__ __forceinline__ void icp_body(const IcpArgs& a) {
  // the successor (k_icp after the cluster kernel, k_mark after k_icp) may be
  // scheduled now; its CTAs wait in their own pdl_wait until this grid is done.
  // Not with the shard exchange: shards' ICP loops sharing a device must all
  // become resident, and waiting successor CTAs could hold the SMs they need.
  pdl_wait();
  if (a.xranks <= 1) pdl_trigger();
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
  // map taps of the pixels in flight, two stages: [stage][pixel k][tap q][thread]
  float4* s_taps = reinterpret_cast<float4*>(
      (reinterpret_cast<uintptr_t>(s_xy + a.max_slots * blockDim.x) + 15) & ~static_cast<uintptr_t>(15));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const bool timer = blockIdx.x == 0 && tid == 0 && a.trace;
  // pixel chunks: this CTA is chunk column vblk of a virtual grid of all
  // shards' CTAs (one shard: the grid itself)
  const int vblk = blockIdx.x + a.xrank * gridDim.x, vgrid = gridDim.x * a.xranks;
  const bool xchg = a.xranks > 1;
  const unsigned long long xseq0 = xchg ? *reinterpret_cast<volatile unsigned long long*>(a.xstate) : 0ull;
  unsigned long long nx = 0;  // exchanges done by this launch
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
    const int gstride = vgrid * blockDim.x;
    const int nslots = min((npix - (int)(vblk * blockDim.x) + gstride - 1) / gstride, a.max_slots);
    for (int i = tid; i < lv.w; i += blockDim.x) s_ux[i] = __ldg(lv.ux + i);
    for (int i = tid; i < lv.h; i += blockDim.x) s_uy[i] = __ldg(lv.uy + i);
    for (int k = 0; k < nslots; ++k) {
      const int pix = vblk * blockDim.x + tid + k * gstride;
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
#ifdef VF_ICP_FINE_TIMERS
      long long tf[6] = {0, 0, 0, 0, 0, 0};  // staging, transforms, taps, terms, warp reduce, CTA sum
#define VF_TF(i) if (timer && k0 == 0) tf[i] = clock64()
#else
#define VF_TF(i)
#endif
      const PoseD c2w = ctl.c2w;
      const PoseD render = ctl.render;
      const D3 rc = rotation_only ? mk(c2w.t[0], c2w.t[1], c2w.t[2]) : mk(0, 0, 0);
      double acc[kAcc];
#pragma unroll
      for (int i = 0; i < kAcc; ++i) acc[i] = 0;
#ifndef VF_ICP_LEGACY_LOOP
      // Software-pipelined pixel pass: the front half of step n + 1 (depth
      // and tables from shared memory, the two FP64 transforms, projection,
      // association test) runs and its eight map taps per pixel are copied
      // into shared memory with cp.async before the back half of step n
      // (bilinear blends, point-to-plane term, sums) consumes its own taps, so
      // the tap round trip and the next transforms overlap the current terms.
      const int total_slots = (npix - (int)(vblk * blockDim.x) + gstride - 1) / gstride;
      IcpStage st0, st1;
      auto front = [&](int k0, int stage, IcpStage& S) {
        float d[kInflight];
        double ux[kInflight], uy[kInflight];
#pragma unroll
        for (int k = 0; k < kInflight; ++k) {
          const int slot = k0 + k;
          const int pix = vblk * blockDim.x + tid + slot * gstride;
          if (slot < nslots) {
            d[k] = s_depth[slot * blockDim.x + tid];
            const int xy = s_xy[slot * blockDim.x + tid];
            ux[k] = s_ux[xy & 0xFFFF];
            uy[k] = s_uy[xy >> 16];
          } else {
            const bool in = slot < total_slots && pix < npix;
            const int y = in ? pix / lv.w : 0, x = in ? pix - y * lv.w : 0;
            d[k] = in ? __ldg(lv.depth + pix) : 0.0f;
            ux[k] = s_ux[x];
            uy[k] = s_uy[y];
          }
        }
#pragma unroll
        for (int k = 0; k < kInflight; ++k) {
          // unproject (intrinsics.hpp:39-43); (x - cx) / fx is tabulated per level
          const D3 pc = mk(ux[k] * d[k], uy[k] * d[k], (double)d[k]);
          S.pw[k] = apply(c2w, pc);
          const D3 q = apply(render, S.pw[k]);
          const double u = a.map.fx * q.x / q.z + a.map.cx;
          const double v = a.map.fy * q.y / q.z + a.map.cy;
          // sample_map_bilinear's bounds test (depth_tracker.hpp:39)
          S.ok[k] = d[k] > 0.0f && q.z > 0.0 &&
                    !(u < 0 || v < 0 || u > a.map.width - 1.001 || v > a.map.height - 1.001);
          const int ix = S.ok[k] ? (int)u : 0, iy = S.ok[k] ? (int)v : 0;
          S.fx[k] = u - ix;
          S.fy[k] = v - iy;
          const size_t i00 = (size_t)iy * a.map.width + ix;
          const size_t off[4] = {i00, i00 + 1, i00 + a.map.width, i00 + a.map.width + 1};
          const unsigned n = S.ok[k] ? 16u : 0u;  // 0: zero-fill, no global read
          float4* dst = s_taps + (size_t)((stage * kInflight + k) * 8) * blockDim.x + tid;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            cp_async16(dst + t * blockDim.x, a.points + off[t], n);
            cp_async16(dst + (4 + t) * blockDim.x, a.normals + off[t], n);
          }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      };
      auto back = [&](int stage, const IcpStage& S) {
#pragma unroll
        for (int k = 0; k < kInflight; ++k) {
          if (!S.ok[k]) continue;
          const float4* src = s_taps + (size_t)((stage * kInflight + k) * 8) * blockDim.x + tid;
          float4 tp[4], tn[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            tp[t] = src[t * blockDim.x];
            tn[t] = src[(4 + t) * blockDim.x];
          }
          D3 mp, mn;
          if (!bilinear_taps(tp, S.fx[k], S.fy[k], a.dist_thr, mp)) continue;
          if (!bilinear_taps(tn, S.fx[k], S.fy[k], 1.0f, mn)) continue;
          const double nlen = sqrt(mn.x * mn.x + mn.y * mn.y + mn.z * mn.z);
          if (nlen < 1e-6) continue;
          // model_normal /= nlen: one refined reciprocal instead of three IEEE
          // divisions (1-ulp differences, far below the 1e-9 H/g parity bar)
          const double inv = rcp_fast(nlen);
          mn = mk(mn.x * inv, mn.y * inv, mn.z * inv);
          // icp_point_to_plane_term (depth_tracker.hpp:20-27)
          const D3 w = S.pw[k];
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
          for (int s2 = 0; s2 < 6; ++s2) {
#pragma unroll
            for (int t = s2; t < 6; ++t, ++n) acc[n] = fma(j[s2], j[t], acc[n]);
            acc[21 + s2] = fma(j[s2], r, acc[21 + s2]);
          }
          acc[27] = fma(r, r, acc[27]);
          acc[28] += 1.0;
        }
      };
      if (total_slots > 0) front(0, 0, st0);
      for (int k0 = 0; k0 < total_slots; k0 += 2 * kInflight) {
        const bool more1 = k0 + kInflight < total_slots;
        if (more1) {
          front(k0 + kInflight, 1, st1);
          asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        back(0, st0);
        if (!more1) break;
        const bool more2 = k0 + 2 * kInflight < total_slots;
        if (more2) {
          front(k0 + 2 * kInflight, 0, st0);
          asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        back(1, st1);
      }
#else
      // kInflight pixels per step, each pipeline stage issued for all before it is
      // consumed, so their memory round trips (depth + tables, then the
      // eight map taps) overlap.
      const int total_slots = (npix - (int)(vblk * blockDim.x) + gstride - 1) / gstride;
      for (int k0 = 0; k0 < total_slots; k0 += kInflight) {
        float d[kInflight];
        double ux[kInflight], uy[kInflight];
#pragma unroll
        for (int k = 0; k < kInflight; ++k) {
          const int slot = k0 + k;
          const int pix = vblk * blockDim.x + tid + slot * gstride;
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
        VF_TF(0);
        D3 pw[kInflight];
        bool ok[kInflight];
        int ix[kInflight], iy[kInflight];
        double fx[kInflight], fy[kInflight];
#pragma unroll
        for (int k = 0; k < kInflight; ++k) {
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
        VF_TF(1);
        float4 tp[kInflight][4], tn[kInflight][4];
#pragma unroll
        for (int k = 0; k < kInflight; ++k) {
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
        for (int k = 0; k < kInflight; ++k) {
          if (k == 0) VF_TF(2);
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
        VF_TF(3);
      }
#endif
      // CTA reduction: transpose butterfly inside each warp, then one warp
      // combines the warp sums.
      {
        double v32[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v32[i] = i < kAcc ? acc[i] : 0.0;
        const double mine = warp_reduce32(v32);
#ifdef VF_ICP_FINE_TIMERS
        if (timer) tf[4] = clock64();
#endif
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
          // all remote loads issued before the first add (<= 16 CTAs per cluster)
          const unsigned nb = cluster.num_blocks();
          double v[16];
#pragma unroll
          for (unsigned r = 0; r < 16; ++r) v[r] = r < nb ? cluster.map_shared_rank(&s_part[buf][0], r)[tid] : 0.0;
          double t = 0;
#pragma unroll
          for (unsigned r = 0; r < 16; ++r)
            if (r < nb) t += v[r];
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
      if (xchg) shard_exchange(a, ++nx + xseq0, s_tot, tid);
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
#ifdef VF_ICP_FINE_TIMERS
          // sub-phases of the pixel term pass (first pixel pair of thread 0)
          for (int i = 0; i < 5; ++i) row[32 + i] = (double)(tf[i] - (i == 0 ? t0 : tf[i - 1]));
          row[37] = (double)(t1 - tf[4]);
#endif
        }
      }
      __syncthreads();
      if (ctl.decision != 0) break;
    }
  }
  if (kCluster) cg::this_cluster().sync();  // no CTA leaves while others read its shared memory
  if (blockIdx.x == 0 && tid == 0) {
    if (xchg) *reinterpret_cast<volatile unsigned long long*>(a.xstate) = xseq0 + nx;
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
