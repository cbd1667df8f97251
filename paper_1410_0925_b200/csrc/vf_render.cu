// Raycast epilogues: the colour tracker's surface point list, and the images
// behind IPipeline::get_image.
//
// Reference: sample_voxel_color / render_image / forward_project_points
// (proj/include/voxfuse/engine/raycast.hpp:441-509) and
// Pipeline::colourize_depth (engine/pipeline_impl.hpp:225-239).
//
// K3c k_forward_project runs at the end of every colour-voxel frame, after
// the raycast (pipeline_impl.hpp:218-221): the maps are subsampled on a
// stride-4 lattice, every valid lattice point samples the voxel colours
// trilinearly, and the valid points are compacted in raster order — the
// order of the reference's push_back loop — with a single-pass decoupled
// look-back scan over 256-item tiles (dynamic tile tickets, so a tile only
// ever waits on tiles that are already running).
#include "vf_device.cuh"
#include "vf_kernels.h"

namespace vf {

namespace {

// sample_voxel_color (raycast.hpp:441-464) on VoxelSRgb words:
// word 0 = sdf | w << 16 | r << 24, word 1 = g | b << 8 | w_color << 16.
__device__ __noinline__ F3 sample_color(const HashView hv, const uint32_t* __restrict__ vox, F3 p) {
  const float qx = p.x - 0.5f, qy = p.y - 0.5f, qz = p.z - 0.5f;
  const int x0 = __float2int_rz(floorf(qx)), y0 = __float2int_rz(floorf(qy)), z0 = __float2int_rz(floorf(qz));
  const float fx = qx - (float)x0, fy = qy - (float)y0, fz = qz - (float)z0;
  // the eight corners' slots: one probe when the stencil sits inside one
  // block, else one per corner; all probes and loads are issued before use
  int slot[8];
  if ((x0 & 7) < 7 && (y0 & 7) < 7 && (z0 & 7) < 7) {
    const int s0 = find_slot(hv, x0 >> 3, y0 >> 3, z0 >> 3);
#pragma unroll
    for (int c = 0; c < 8; ++c) slot[c] = s0;
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      slot[c] = find_slot(hv, (x0 + (c & 1)) >> 3, (y0 + ((c >> 1) & 1)) >> 3, (z0 + ((c >> 2) & 1)) >> 3);
  }
  uint2 vv[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int vx = x0 + (c & 1), vy = y0 + ((c >> 1) & 1), vz = z0 + ((c >> 2) & 1);
    vv[c] = slot[c] < 0 ? make_uint2(0u, 0u)
                        : __ldg(reinterpret_cast<const uint2*>(vox) +
                                ((size_t)slot[c] * kBlockVolume + ((vx & 7) + (vy & 7) * kBlockSide + (vz & 7) * 64)));
  }
  float sx = 0.0f, sy = 0.0f, sz = 0.0f, wsum = 0.0f;
#pragma unroll
  for (int corner = 0; corner < 8; ++corner) {
    const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
    if (slot[corner] < 0) continue;
    const uint2 v = vv[corner];
    if (((v.y >> 16) & 0xFFu) == 0) continue;  // w_color == 0
    const float w = (dx ? fx : 1 - fx) * (dy ? fy : 1 - fy) * (dz ? fz : 1 - fz);
    sx += (float)(v.x >> 24) * w;
    sy += (float)(v.y & 0xFFu) * w;
    sz += (float)((v.y >> 8) & 0xFFu) * w;
    wsum += w;
  }
  if (wsum > 0.0f) return F3{sx / wsum, sy / wsum, sz / wsum};
  return F3{0.0f, 0.0f, 0.0f};
}

constexpr int kFpTile = kFpTileItems;
constexpr uint32_t kFlagAggregate = 1u, kFlagPrefix = 2u;

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

}  // namespace

// forward_project_points (raycast.hpp:495-509) with stride `stride`.
// scan[0] is the tile ticket, scan[1 + t] tile t's (status << 32 | value);
// the frame zeroes them before the launch.
__global__ void __launch_bounds__(kFpTile) k_forward_project(HashView hv, const uint32_t* __restrict__ vox,
                                                             const float4* __restrict__ points, IntrD in, int stride,
                                                             float vs, unsigned long long* scan,
                                                             float* __restrict__ out_points,
                                                             float* __restrict__ out_colors, Counters* ctr) {
  __shared__ int s_tile;
  __shared__ int s_warp[kFpTile / 32];
  __shared__ int s_prefix;
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(scan, 1ull);
  __syncthreads();
  const int tile = s_tile;
  const int cols = (in.width + stride - 1) / stride, rows = (in.height + stride - 1) / stride;
  const int n = cols * rows;
  const int i = tile * kFpTile + threadIdx.x;
  bool valid = false;
  F3 p{0.f, 0.f, 0.f}, c{0.f, 0.f, 0.f};
  if (i < n) {
    const int x = (i % cols) * stride, y = (i / cols) * stride;
    const float4 q = __ldg(points + (size_t)y * in.width + x);
    if (q.w != 0.0f) {
      valid = true;
      p = F3{q.x, q.y, q.z};
      if (vox) {  // nullptr: a voxel type without colour (sample_voxel_color returns zero)
        c = sample_color(hv, vox, F3{q.x / vs, q.y / vs, q.z / vs});
        c = F3{c.x / 255.0f, c.y / 255.0f, c.z / 255.0f};
      }
    }
  }
  // block-exclusive scan of the valid flags
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned ball = __ballot_sync(0xffffffffu, valid);
  const int rank_in_warp = __popc(ball & ((1u << lane) - 1u));
  if (lane == 0) s_warp[wid] = __popc(ball);
  __syncthreads();
  if (wid == 0) {
    int v = lane < kFpTile / 32 ? s_warp[lane] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int agg = __shfl_sync(0xffffffffu, incl, 31);
    if (lane < kFpTile / 32) s_warp[lane] = incl - v;
    // decoupled look-back (tile order = raster order)
    unsigned long long* flags = scan + 1;
    if (lane == 0) {
      const unsigned long long st = tile == 0 ? kFlagPrefix : kFlagAggregate;
      atomicExch(flags + tile, (st << 32) | (unsigned)agg);
    }
    int prefix = 0;
    int j = tile - 1;
    while (j >= 0) {
      const int k = j - lane;
      unsigned long long f = 0;
      if (k >= 0) {
        do {
          f = ld_volatile(flags + k);
        } while ((f >> 32) == 0);
      }
      const uint32_t st = k >= 0 ? (uint32_t)(f >> 32) : kFlagPrefix;
      const unsigned pmask = __ballot_sync(0xffffffffu, st == kFlagPrefix);
      const int stop = pmask ? __ffs(pmask) - 1 : 31;  // nearest predecessor holding an inclusive prefix
      int val = (k >= 0 && lane <= stop) ? (int)(uint32_t)f : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
      prefix += val;
      if (pmask) break;
      j -= 32;
    }
    if (lane == 0) {
      if (tile > 0) atomicExch(flags + tile, ((unsigned long long)kFlagPrefix << 32) | (unsigned)(prefix + agg));
      s_prefix = prefix;
      if (tile == (n + kFpTile - 1) / kFpTile - 1) ctr->surface_count = prefix + agg;
    }
  }
  __syncthreads();
  if (valid) {
    const int o = s_prefix + s_warp[wid] + rank_in_warp;
    out_points[3 * o + 0] = p.x;
    out_points[3 * o + 1] = p.y;
    out_points[3 * o + 2] = p.z;
    out_colors[3 * o + 0] = c.x;
    out_colors[3 * o + 1] = c.y;
    out_colors[3 * o + 2] = c.z;
  }
}

// render_image (raycast.hpp:466-490): mode 0 shaded grey, 1 colour.
__global__ void __launch_bounds__(256) k_render_image(HashView hv, const uint32_t* __restrict__ vox,
                                                      const float4* __restrict__ points,
                                                      const float4* __restrict__ normals, const PoseD* __restrict__ w2c,
                                                      IntrD in, float vs, int color, uint8_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= in.width * in.height) return;
  uint8_t r = 0, g = 0, b = 0;
  const float4 q = __ldg(points + i);
  if (q.w != 0.0f) {
    const float4 nn = __ldg(normals + i);
    const float ax = (float)w2c->r[6], ay = (float)w2c->r[7], az = (float)w2c->r[8];
    const float shade = fabsf(nn.x * ax + nn.y * ay + nn.z * az);
    if (!color) {
      const float s = shade < 0.0f ? 0.0f : (1.0f < shade ? 1.0f : shade);
      r = g = b = (uint8_t)__float2int_rz(s * 255.0f);
    } else {
      F3 c = sample_color(hv, vox, F3{q.x / vs, q.y / vs, q.z / vs});
      c = F3{c.x * shade, c.y * shade, c.z * shade};
      auto u8 = [](float v) { return (uint8_t)__float2int_rz(v < 0.0f ? 0.0f : (255.0f < v ? 255.0f : v)); };
      r = u8(c.x);
      g = u8(c.y);
      b = u8(c.z);
    }
  }
  out[3 * i + 0] = r;
  out[3 * i + 1] = g;
  out[3 * i + 2] = b;
}

// Pipeline::colourize_depth (pipeline_impl.hpp:225-239), pass 1: dmax over
// the positive samples (std::max skips NaN; positive float bits order like
// the floats).
__global__ void k_depth_max(const float* __restrict__ depth, int n, int* dmax_bits) {
  int m = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float d = __ldg(depth + i);
    if (d > 0.0f) m = max(m, __float_as_int(d));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(dmax_bits, m);
}

// pass 2
__global__ void k_colourize_depth(const float* __restrict__ depth, int n, const int* __restrict__ dmax_bits,
                                  uint8_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float dmax = __int_as_float(*dmax_bits);
  const float d = __ldg(depth + i);
  uint8_t r = 0, g = 0, b = 0;
  if (dmax > 0.0f && d > 0.0f) {
    const float t = d / dmax;
    r = (uint8_t)__float2int_rz(255.0f * (1.0f - t));
    g = (uint8_t)__float2int_rz(255.0f * (1.0f - fabsf(2.0f * t - 1.0f)));
    b = (uint8_t)__float2int_rz(255.0f * t);
  }
  out[3 * i + 0] = r;
  out[3 * i + 1] = g;
  out[3 * i + 2] = b;
}

}  // namespace vf
