// K3 — expected-depth range image (K3a) and the hash-walking raycast that
// produces the point / normal maps (K3b).
//
// Reference: create_expected_depths (proj/include/voxfuse/engine/raycast.hpp:268-363),
// cast_ray / trilinear_sdf / sdf_surface_normal / render_maps (raycast.hpp:102-162,
// :171-263, :415-435).
//
// K3a folds each visible block's fragment box into the 16x16-fragment range
// image with integer atomicMin / atomicMax on the float bit patterns (all
// values are positive, so integer order is float order); min/max commute, so
// the result equals the reference's serial fold.
//
// K3b: 128-thread CTAs cover half a 16x16 fragment (one range per CTA), one
// thread per pixel, each warp an 8x4 pixel patch.  The reference probes the
// hash table for every voxel sample (1 per march step, 8 per trilinear, 48
// per normal).  Each thread keeps a direct-mapped 8-way cache of block -> VBA
// slot (misses included) in shared memory, laid out [way][thread] so lookups
// are bank-conflict free, the way chosen by block-coordinate parity so the
// 2x2x2 blocks of a trilinear stencil never evict each other.  The table does
// not change during the raycast, so the values read — and therefore every
// floating-point decision — are identical to the uncached reference.
#include "vf_device.cuh"
#include "vf_kernels.h"

namespace vf {

// K3a
__global__ void __launch_bounds__(256) k_ranges(const HashEntry* __restrict__ entries,
                                                const int* __restrict__ visible_list, const Counters* __restrict__ ctr,
                                                const FrameParams* __restrict__ fp, IntrD in, float vs, float near_clip,
                                                float far_clip, float2* __restrict__ ranges, int frag_w) {
  pdl_enter();
  __shared__ PoseD s_w2c;
  if (threadIdx.x < sizeof(PoseD) / sizeof(double))
    reinterpret_cast<double*>(&s_w2c)[threadIdx.x] = reinterpret_cast<const double*>(&fp->w2c)[threadIdx.x];
  __syncthreads();
  const int n = ctr->visible_count;
  const double nearc = near_clip, farc = far_clip;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const HashEntry e = load_entry(entries + __ldg(visible_list + i));
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    double zmin = inf, zmax = -inf, xmin = inf, xmax = -inf, ymin = inf, ymax = -inf;
    bool behind = false;
#pragma unroll
    for (int corner = 0; corner < 8; ++corner) {
      const D3 w = mk((double)((float)(e.x * kBlockSide + ((corner & 1) ? kBlockSide : 0)) * vs),
                      (double)((float)(e.y * kBlockSide + ((corner & 2) ? kBlockSide : 0)) * vs),
                      (double)((float)(e.z * kBlockSide + ((corner & 4) ? kBlockSide : 0)) * vs));
      const D3 cam = apply(s_w2c, w);
      zmin = cam.z < zmin ? cam.z : zmin;
      zmax = zmax < cam.z ? cam.z : zmax;
      if (cam.z <= 1e-6) {
        behind = true;
        continue;
      }
      const double u = in.fx * cam.x / cam.z + in.cx;
      const double v = in.fy * cam.y / cam.z + in.cy;
      xmin = u < xmin ? u : xmin;
      xmax = xmax < u ? u : xmax;
      ymin = v < ymin ? v : ymin;
      ymax = ymax < v ? v : ymax;
    }
    if (behind || !(zmax > nearc && zmin < farc)) continue;
    int px0 = __double2int_rz(floor(xmin));
    px0 = px0 < 0 ? 0 : px0;
    int px1 = __double2int_rz(ceil(xmax));
    px1 = in.width - 1 < px1 ? in.width - 1 : px1;
    int py0 = __double2int_rz(floor(ymin));
    py0 = py0 < 0 ? 0 : py0;
    int py1 = __double2int_rz(ceil(ymax));
    py1 = in.height - 1 < py1 ? in.height - 1 : py1;
    if (!(px0 <= px1 && py0 <= py1)) continue;
    const float fzmin = (float)(zmin < nearc ? nearc : zmin);
    const float fzmax = (float)(farc < zmax ? farc : zmax);
    const int imin = __float_as_int(fzmin), imax = __float_as_int(fzmax);
    for (int fy = py0 / kFragmentSize; fy <= py1 / kFragmentSize; ++fy)
      for (int fx = px0 / kFragmentSize; fx <= px1 / kFragmentSize; ++fx) {
        int* r = reinterpret_cast<int*>(ranges + fy * frag_w + fx);
        atomicMin(r, imin);
        atomicMax(r + 1, imax);
      }
  }
}

namespace {

constexpr int kRayThreads = 128;
constexpr int kCacheWays = 8;
// 1: the march ends at the zero-crossing bracket and the two refinement
// steps run in k_ray_normals too, with full warps (C1 raycast 0.180 ->
// 0.176 ms, C3 0.528 -> 0.515); 0: refinement inside the march.
#ifndef VF_RAY_REFINE_SPLIT
#define VF_RAY_REFINE_SPLIT 1
#endif
// CTA-wide block cache entries in the normals pass (0: off).  Measured: 128
// entries C1 raycast 0.176 -> 0.174 ms, C3 0.519 -> 0.504 ms; 256 no gain.
// (The same cache in the march kernel costs more than it saves.)
#ifndef VF_NORM_SHARED
#define VF_NORM_SHARED 128
#endif
// 1: the normal's six trilinears read their 32 distinct voxels at once
// (Sampler::normal32); 0: six dependent trilinears of 8 reads each.
#ifndef VF_NORM_STENCIL32
#define VF_NORM_STENCIL32 0
#endif
#ifndef VF_NORM_MIN_BLOCKS
#define VF_NORM_MIN_BLOCKS 8
#endif


__device__ __noinline__ int probe(const HashView hv, int x, int y, int z) { return find_slot(hv, x, y, z); }

// Per-thread direct-mapped cache of block position -> VBA slot (misses
// included), in shared memory laid out [way][thread] so that a warp's
// 16-byte lookups are conflict-free.  The way is the parity of the block
// coordinates, so the 2x2x2 blocks a trilinear stencil can straddle never
// evict each other.
// kCount: the measurement build (k_raycast_count) also counts table probes
// (cache misses) and voxel reads (each a hash probe in the reference).
template <bool kCount>
struct SamplerCounts {  // empty base in the frame-path build (no size, no stack)
};
template <>
struct SamplerCounts<true> {
  unsigned n_probe = 0, n_read = 0;
};
// kShared > 0: a CTA-wide direct-mapped cache of kShared block -> slot
// entries behind the per-thread ways (the normals pass: a CTA's hits are
// neighbours and read the same few blocks).
template <int kStride, bool kCount = false, int kShared = 0>  // kStride: 32-bit words per voxel, 1 or 2
struct Sampler : SamplerCounts<kCount> {
  HashView hv;
  const uint32_t* vox;  // first 4 bytes of each voxel: sdf (lo 16), w_depth (byte 2)
  int4* cache;          // this thread's column of the shared cache: (block, first word of the block or -1)
  int4* shared_blocks = nullptr;
  __device__ Sampler(const HashView& h, const uint32_t* v, int4* c, int4* sb = nullptr)
      : hv(h), vox(v), cache(c), shared_blocks(sb) {}

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int w = 0; w < kCacheWays; ++w) cache[w * kRayThreads] = make_int4(0x7fffffff, 0, 0, -1);
  }
  __device__ __forceinline__ int lookup(int x, int y, int z) {
    const int w = (x & 1) | ((y & 1) << 1) | ((z & 1) << 2);
    const int4 c = cache[w * kRayThreads];
    if constexpr (kCount) ++this->n_read;
    if (c.x == x && c.y == y && c.z == z) return c.w;
    uint32_t sh = 0;
    if constexpr (kShared > 0) {
      sh = (uint32_t)__cvta_generic_to_shared(shared_blocks + hash_block(x, y, z, (uint32_t)(kShared - 1)));
      int4 e;
      asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(e.x), "=r"(e.y), "=r"(e.z), "=r"(e.w) : "r"(sh));
      if (e.x == x && e.y == y && e.z == z) {
        cache[w * kRayThreads] = e;
        return e.w;
      }
    }
    if constexpr (kCount) ++this->n_probe;
    const int slot = probe(hv, x, y, z);
    const int s = slot < 0 ? -1 : slot * (kBlockVolume * kStride);
    cache[w * kRayThreads] = make_int4(x, y, z, s);
    if constexpr (kShared > 0)
      asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(sh), "r"(x), "r"(y), "r"(z), "r"(s) : "memory");
    return s;
  }
  __device__ __forceinline__ uint32_t raw(int base, int lx, int ly, int lz) const {
    return __ldg(vox + (unsigned)(base + (lx + ly * kBlockSide + lz * kBlockSide * kBlockSide) * kStride));
  }

  // HashSdfSampler::read (raycast.hpp:73-76)
  __device__ __forceinline__ bool read(int vx, int vy, int vz, float& value) {
    const int s = lookup(vx >> 3, vy >> 3, vz >> 3);
    if (s < 0) {
      value = 1.0f;  // sdf_to_float(32767)
      return false;
    }
    const uint32_t r = raw(s, vx & 7, vy & 7, vz & 7);
    value = sdf_bits_to_float(r);
    return ((r >> 16) & 0xFFu) > 0;
  }

  // trilinear_sdf (raycast.hpp:102-117): the value, or NaN when a corner is
  // unallocated / unobserved.  Inlined at exactly three sites (band test,
  // refinement loop, normal loop); more copies blow the instruction cache
  // (ncu: no_instruction stalls), out-of-line calls pay the ABI spills.
  __device__ __forceinline__ float trilinear(F3 p) {
    const float qx = p.x - 0.5f, qy = p.y - 0.5f, qz = p.z - 0.5f;
    const int x0 = __float2int_rz(floorf(qx)), y0 = __float2int_rz(floorf(qy)), z0 = __float2int_rz(floorf(qz));
    const float fx = qx - (float)x0, fy = qy - (float)y0, fz = qz - (float)z0;
    const int bx0 = x0 >> 3, by0 = y0 >> 3, bz0 = z0 >> 3;
    const int lx0 = x0 & 7, ly0 = y0 & 7, lz0 = z0 & 7;
    uint32_t r[8];
#pragma unroll
    for (int corner = 0; corner < 8; ++corner) {
      const int lx = lx0 + (corner & 1), ly = ly0 + ((corner >> 1) & 1), lz = lz0 + ((corner >> 2) & 1);
      const int s = lookup(bx0 + (lx >> 3), by0 + (ly >> 3), bz0 + (lz >> 3));
      if (s < 0) return __int_as_float(0x7fffffff);
      r[corner] = raw(s, lx & 7, ly & 7, lz & 7);
    }
    float value = 0.0f;
#pragma unroll
    for (int corner = 0; corner < 8; ++corner) {
      const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
      if (((r[corner] >> 16) & 0xFFu) == 0) return __int_as_float(0x7fffffff);
      const float v = sdf_bits_to_float(r[corner]);
      const float w = (dx ? fx : 1 - fx) * (dy ? fy : 1 - fy) * (dz ? fz : 1 - fz);
      value += w * v;
    }
    return value;
  }

  // sdf_surface_normal (raycast.hpp:147-162): six trilinear values at
  // p -/+ 1 voxel per axis, evaluated by one loop body.
  __device__ __noinline__ bool normal(F3 p, F3& n) {
    float v[6];
#pragma unroll 1
    for (int k = 0; k < 6; ++k) {
      const float sgn = (k & 1) ? 1.0f : -1.0f;
      const int a = k >> 1;
      const F3 q{a == 0 ? p.x + sgn : p.x, a == 1 ? p.y + sgn : p.y, a == 2 ? p.z + sgn : p.z};
      v[k] = trilinear(q);
      if (v[k] != v[k]) return false;
    }
    const float gx = v[1] - v[0], gy = v[3] - v[2], gz = v[5] - v[4];
    const float len = sqrtf(gx * gx + gy * gy + gz * gz);
    if (len < 1e-12f) return false;
    n = F3{gx / len, gy / len, gz / len};
    return true;
  }

  // The same six trilinears from their 32 distinct voxels, all read at once
  // (one memory round trip instead of six dependent ones).  Centre corner
  // b = floor(p - 0.5) per axis; the -1 / +1 stencils along an axis use
  // b - 1, b and b + 1, b + 2 there and b, b + 1 on the other two axes, so
  // their union is the 2x2x2 cube at b plus two 2x2 layers per axis.  Every
  // stencil's corner and fractions are computed with the generic path's own
  // float operations; when p -/+ 1 rounds so that a stencil's corner is not
  // b -/+ 1 the generic path runs instead.  A missing block reads as
  // weight 0 (both make the trilinear, hence the normal, fail).
  __device__ __noinline__ bool normal32(F3 p, F3& n) {
    const float cx = p.x - 0.5f, cy = p.y - 0.5f, cz = p.z - 0.5f;
    const int bx = __float2int_rz(floorf(cx)), by = __float2int_rz(floorf(cy)), bz = __float2int_rz(floorf(cz));
    const float lx = (p.x + -1.0f) - 0.5f, hx = (p.x + 1.0f) - 0.5f;
    const float ly = (p.y + -1.0f) - 0.5f, hy = (p.y + 1.0f) - 0.5f;
    const float lz = (p.z + -1.0f) - 0.5f, hz = (p.z + 1.0f) - 0.5f;
    const int ilx = __float2int_rz(floorf(lx)), ihx = __float2int_rz(floorf(hx));
    const int ily = __float2int_rz(floorf(ly)), ihy = __float2int_rz(floorf(hy));
    const int ilz = __float2int_rz(floorf(lz)), ihz = __float2int_rz(floorf(hz));
    if (ilx != bx - 1 || ihx != bx + 1 || ily != by - 1 || ihy != by + 1 || ilz != bz - 1 || ihz != bz + 1)
      return normal(p, n);
    auto rd = [&](int ox, int oy, int oz) -> uint32_t {
      const int x = bx + ox, y = by + oy, z = bz + oz;
      const int s = lookup(x >> 3, y >> 3, z >> 3);
      return s < 0 ? 0u : raw(s, x & 7, y & 7, z & 7);
    };
    // X[ox + 1][oy][oz] (ox -1..2, oy, oz 0..1); Y[oy == 2][ox][oz] (oy -1, 2); Z[oz == 2][ox][oy] (oz -1, 2)
    uint32_t X[4][2][2], Y[2][2][2], Z[2][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int k = 0; k < 2; ++k) X[i][j][k] = rd(i - 1, j, k);
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          Y[s][i][j] = rd(i, s ? 2 : -1, j);
          Z[s][i][j] = rd(i, j, s ? 2 : -1);
        }
    const float fxc = cx - (float)bx, fyc = cy - (float)by, fzc = cz - (float)bz;
    // trilinear_sdf's blend (corner order, weight products as the generic path)
    auto blend = [&](const uint32_t (&r)[8], float fx, float fy, float fz, float& value) -> bool {
      value = 0.0f;
#pragma unroll
      for (int corner = 0; corner < 8; ++corner) {
        const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
        if (((r[corner] >> 16) & 0xFFu) == 0) return false;
        const float v = sdf_bits_to_float(r[corner]);
        const float w = (dx ? fx : 1 - fx) * (dy ? fy : 1 - fy) * (dz ? fz : 1 - fz);
        value += w * v;
      }
      return true;
    };
    float v[6];
    uint32_t r[8];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const int a = k >> 1, hi = k & 1;
#pragma unroll
      for (int corner = 0; corner < 8; ++corner) {
        const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
        if (a == 0) {
          r[corner] = X[2 * hi + dx][dy][dz];
        } else if (a == 1) {
          const int oy = 2 * hi - 1 + dy;  // -1..2
          r[corner] = (oy == -1 || oy == 2) ? Y[oy == 2][dx][dz] : X[1 + dx][oy][dz];
        } else {
          const int oz = 2 * hi - 1 + dz;
          r[corner] = (oz == -1 || oz == 2) ? Z[oz == 2][dx][dy] : X[1 + dx][dy][oz];
        }
      }
      const float fx = a == 0 ? (hi ? hx - (float)ihx : lx - (float)ilx) : fxc;
      const float fy = a == 1 ? (hi ? hy - (float)ihy : ly - (float)ily) : fyc;
      const float fz = a == 2 ? (hi ? hz - (float)ihz : lz - (float)ilz) : fzc;
      if (!blend(r, fx, fy, fz, v[k])) return false;
    }
    const float gx = v[1] - v[0], gy = v[3] - v[2], gz = v[5] - v[4];
    const float len = sqrtf(gx * gx + gy * gy + gz * gz);
    if (len < 1e-12f) return false;
    n = F3{gx / len, gy / len, gz / len};
    return true;
  }
};

// cast_ray (raycast.hpp:171-263) from the ray's start point and unit
// direction in voxel units.  Returns the hit in metres.
// The zero-crossing refinement (two trilinear secant / Newton steps) and the
// hit, from the bracket the march ends on: in the normals pass
// (VF_RAY_REFINE_SPLIT = 1, default) or in the march kernel.
template <typename TSampler>
__device__ __forceinline__ F3 refine_hit(TSampler& smp, F3 start, F3 dir, float t, float sdf, float mu_vox, float vs) {
  float t_back = t, sdf_back = sdf;
#pragma unroll 1
  for (int i = 0; i < 2; ++i) {
    const float tri = smp.trilinear(F3{start.x + dir.x * t, start.y + dir.y * t, start.z + dir.z * t});
    if (tri != tri) break;
    const float denom = sdf_back - tri;
    if (fabsf(denom) > 1e-12f && fabsf(t_back - t) > 1e-6f) {
      const float slope = denom / (t_back - t);
      t_back = t;
      sdf_back = tri;
      t -= tri / (fabsf(slope) > 1e-6f ? slope : 1.0f / mu_vox);
    } else {
      t += tri * mu_vox;
    }
  }
  const F3 h{start.x + dir.x * t, start.y + dir.y * t, start.z + dir.z * t};
  return F3{h.x * vs, h.y * vs, h.z * vs};
}

// kDefer: stop at the bracket and return it as hw = (t, sdf, 0).
template <bool kDefer = false, typename TSampler>
__device__ __forceinline__ bool march(TSampler& smp, F3 start, F3 dir, float total, float mu_vox, float vs, F3& hw) {
  const float fine_step = (8.0f < mu_vox) ? 8.0f : mu_vox;
  int state = 0;  // 0 coarse, 1 fine, 2 surface
  float t = 0.0f, t_front = -1.0f, sdf_front = 1.0f;
  while (t <= total) {
    const F3 p{start.x + dir.x * t, start.y + dir.y * t, start.z + dir.z * t};
    float value;
    const bool found =
        smp.read(__float2int_rz(floorf(p.x)), __float2int_rz(floorf(p.y)), __float2int_rz(floorf(p.z)), value);
    if (state == 0) {
      if (!found) {
        t += 8.0f;
        continue;
      }
      state = 1;
      const float tb = t - 8.0f;
      t = (0.0f < tb) ? tb : 0.0f;
      continue;
    }
    if (!found) {
      if (state == 2) state = 1;
      t_front = -1.0f;
      t += fine_step;
      continue;
    }
    float sdf = value;
    if (state == 1 && sdf <= 0.0f) return false;  // WRONG_SIDE
    state = 2;
    if (sdf <= 0.1f && sdf >= -0.5f) {
      const float tri = smp.trilinear(p);
      if (tri == tri) sdf = tri;
    }
    if (sdf <= 0.0f) {
      if (t_front >= 0.0f && sdf_front > sdf && t - t_front <= 2.0f * mu_vox) {
        t = t + (t_front - t) * sdf / (sdf - sdf_front);
      } else {
        t += sdf * mu_vox;
      }
      if (kDefer) {
        hw = F3{t, sdf, 0.0f};
      } else {
        hw = refine_hit(smp, start, dir, t, sdf, mu_vox, vs);
      }
      return true;
    }
    t_front = t;
    sdf_front = sdf;
    const float a = sdf * mu_vox;
    const float b = (a < 1.0f) ? 1.0f : a;
    t += (mu_vox < b) ? mu_vox : b;
  }
  return false;
}

}  // namespace

// cast_ray's ray (raycast.hpp:176-198): start and end of the fragment's range
// in voxel units (FP64 -> float), the direction not yet normalised.
__device__ __forceinline__ void ray_setup(int x, int y, float2 range, const FrameParams* __restrict__ fp,
                                          const IntrD& in, float vs, F3& start, F3& dir, float& total) {
  if (range.x <= range.y) {  // RangeImage::valid
    const PoseD& c2w = fp->c2w;
    const double inv_vox = 1.0 / (double)vs;
    const double dx = (x - in.cx) / in.fx, dy = (y - in.cy) / in.fy;
    const double r0 = range.x, r1 = range.y;
    const D3 s0 = apply(c2w, mk(dx * r0, dy * r0, 1.0 * r0));
    const D3 e0 = apply(c2w, mk(dx * r1, dy * r1, 1.0 * r1));
    start = F3{(float)(s0.x * inv_vox), (float)(s0.y * inv_vox), (float)(s0.z * inv_vox)};
    const F3 end{(float)(e0.x * inv_vox), (float)(e0.y * inv_vox), (float)(e0.z * inv_vox)};
    dir = F3{end.x - start.x, end.y - start.y, end.z - start.z};
    total = sqrtf(dir.x * dir.x + dir.y * dir.y + dir.z * dir.z);
  }
}

// K3b: render_maps (raycast.hpp:415-435).  128-thread CTAs cover half a
// 16x16 fragment (16 x 8 pixels), so every CTA reads one range.
template <int kStride, bool kCount = false>
__device__ __forceinline__ void raycast_body(const HashView& hv, const uint32_t* __restrict__ vox,
                                             const float2* __restrict__ ranges, const FrameParams* __restrict__ fp,
                                             const IntrD& in, float vs, float mu, float4* __restrict__ points,
                                             float4* __restrict__ normals, int4* s_cache,
                                             unsigned long long* counters = nullptr) {
  const int fxi = blockIdx.x, fyi = blockIdx.y >> 1;
  // Each warp traces an 8 x 4 pixel patch of the CTA's 16 x 8 half fragment
  // (2 x 2 warps): neighbouring rays march similar lengths, so the warp
  // diverges less than with 16 x 2 rows (C1 raycast 0.221 -> 0.213 ms).
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
#ifndef VF_RAY_WARP_4X8
  const int x = fxi * kFragmentSize + (lane & 7) + ((wq & 1) << 3);
  const int y = fyi * kFragmentSize + ((blockIdx.y & 1) << 3) + (lane >> 3) + ((wq >> 1) << 2);
#else
  const int x = fxi * kFragmentSize + (lane & 3) + (wq << 2);
  const int y = fyi * kFragmentSize + ((blockIdx.y & 1) << 3) + (lane >> 2);
#endif
  if (x >= in.width || y >= in.height) return;
  const size_t pix = (size_t)y * in.width + x;
  const float2 range = __ldg(ranges + fyi * gridDim.x + fxi);
  F3 start, dir;
  float total = 0.0f;
  ray_setup(x, y, range, fp, in, vs, start, dir, total);
  float4 out_p = make_float4(0.f, 0.f, 0.f, 0.f), out_n = make_float4(0.f, 0.f, 0.f, 0.f);
  if (total > 0) {
    dir = F3{dir.x / total, dir.y / total, dir.z / total};
    Sampler<kStride, kCount> smp{hv, vox, s_cache + threadIdx.x};
    smp.init();
    F3 hw;
    if (march<VF_RAY_REFINE_SPLIT && !kCount>(smp, start, dir, total, mu / vs, vs, hw)) {
      if (!kCount) {
        if (VF_RAY_REFINE_SPLIT) {  // the bracket (t, sdf): refinement, hit and normal in k_ray_normals
          out_p = make_float4(0.f, 0.f, 0.f, 2.0f);
          out_n = make_float4(hw.x, hw.y, 0.f, 0.f);
        } else {
          out_p = make_float4(hw.x, hw.y, hw.z, 1.0f);  // the normal follows in k_ray_normals
        }
      } else {
        F3 n;
        if (smp.normal(F3{hw.x / vs, hw.y / vs, hw.z / vs}, n)) {
          out_p = make_float4(hw.x, hw.y, hw.z, 1.0f);
          out_n = make_float4(n.x, n.y, n.z, 1.0f);
        }
      }
    }
    if constexpr (kCount) {
      atomicAdd(counters + 0, (unsigned long long)smp.n_probe);
      atomicAdd(counters + 1, (unsigned long long)smp.n_read);
      atomicAdd(counters + 2, 1ull);
      if (out_p.w != 0.0f) atomicAdd(counters + 3, 1ull);
    }
  }
  points[pix] = out_p;
  normals[pix] = out_n;
}

template <int kMinBlocks>
__global__ void __launch_bounds__(kRayThreads, kMinBlocks)
    k_raycast(HashView hv, const uint32_t* __restrict__ vox, int vstride, const float2* __restrict__ ranges,
              const FrameParams* __restrict__ fp, IntrD in, float vs, float mu, float4* __restrict__ points,
              float4* __restrict__ normals, unsigned* __restrict__ ray_flags) {
  pdl_enter();
  __shared__ int4 s_cache[kCacheWays * kRayThreads];
  if (vstride == 1)
    raycast_body<1>(hv, vox, ranges, fp, in, vs, mu, points, normals, s_cache);
  else
    raycast_body<2>(hv, vox, ranges, fp, in, vs, mu, points, normals, s_cache);
  // this CTA's half fragment is in the maps: release it to the k_ray_normals
  // CTA of the same index (which may already be waiting, see there)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ray_flags + blockIdx.y * gridDim.x + blockIdx.x), "r"(1u)
                 : "memory");
  }
}
// Two occupancy points of the march (launch_raycast picks by frame size):
// 8 CTAs per SM (64 registers) for large frames, 6 (70 registers, no
// spills) up to VF_RAY_SMALL_PIXELS -- measured C1 raycast 0.156 -> 0.142 ms,
// C3 0.422 -> 0.454 ms (profiles/r2_ab_rayocc*.txt).
template __global__ void k_raycast<VF_RAY_MIN_BLOCKS>(HashView, const uint32_t*, int, const float2*,
                                                      const FrameParams*, IntrD, float, float, float4*, float4*,
                                                      unsigned*);
template __global__ void k_raycast<VF_RAY_MIN_BLOCKS_SMALL>(HashView, const uint32_t*, int, const float2*,
                                                            const FrameParams*, IntrD, float, float, float4*, float4*,
                                                            unsigned*);

// K3b second pass: the zero-crossing refinement and the normal of every hit
// (sdf_surface_normal, the 48-read stencil) with full warps -- in one fused
// kernel each ray's refinement and normal ran when its own march ended, with
// the warp's other lanes idle or still marching (C1 raycast 0.204 -> 0.176
// ms, C3 0.584 -> 0.515 ms).  Same pixel tiling as k_raycast; the march
// leaves the bracket (t, sdf) in the normal map and a marker in the point map;
// the ray is set up again exactly as cast_ray does, the hit is formed in
// metres and divided by vs for the normal as before, and a failed normal
// clears the hit, as render_maps does (raycast.hpp:427-431).
template <int kStride>
__device__ __forceinline__ void ray_normal_body(const HashView& hv, const uint32_t* __restrict__ vox,
                                                float2 range, const FrameParams* __restrict__ fp,
                                                const IntrD& in, float vs, float mu, int x, int y, size_t pix,
                                                float4* __restrict__ points, float4* __restrict__ normals,
                                                int4* s_cache, int4* s_blocks) {
  float4 p = points[pix];
  if (p.w == 0.0f) return;
  Sampler<kStride, false, VF_NORM_SHARED> smp{hv, vox, s_cache + threadIdx.x, s_blocks};
  smp.init();
  if (p.w == 2.0f) {  // deferred: refine the bracket (t, sdf) the march ended on
    const float4 b = normals[pix];
    F3 start{0, 0, 0}, dir{0, 0, 0};
    float total = 0.0f;
    ray_setup(x, y, range, fp, in, vs, start, dir, total);
    dir = F3{dir.x / total, dir.y / total, dir.z / total};
    const F3 hw = refine_hit(smp, start, dir, b.x, b.y, mu / vs, vs);
    p = make_float4(hw.x, hw.y, hw.z, 1.0f);
  }
  F3 n;
  const F3 pv{p.x / vs, p.y / vs, p.z / vs};
  if (VF_NORM_STENCIL32 ? smp.normal32(pv, n) : smp.normal(pv, n)) {
    points[pix] = p;
    normals[pix] = make_float4(n.x, n.y, n.z, 1.0f);
  } else {
    points[pix] = make_float4(0.f, 0.f, 0.f, 0.f);
    normals[pix] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

__global__ void __launch_bounds__(kRayThreads, VF_NORM_MIN_BLOCKS)
    k_ray_normals(HashView hv, const uint32_t* __restrict__ vox, int vstride, const float2* __restrict__ ranges,
                  const FrameParams* __restrict__ fp, IntrD in, float vs, float mu, float4* __restrict__ points,
                  float4* __restrict__ normals, unsigned* __restrict__ ray_flags, Counters* __restrict__ ctr) {
  // No griddepcontrol.wait on the whole march grid: this CTA waits only for
  // the k_raycast CTA of the same index (its completion flag), so the normals
  // of finished half fragments run in the march's tail.  Safe: PDL launches
  // this grid only after every k_raycast CTA has executed its own
  // pdl_enter (so everything before the march is complete and every march
  // CTA is resident and will finish); without PDL the march is complete.
  // The flag is cleared here for the next launch pair (launch_raycast always
  // launches both); a flag that never arrives (~0.5 s) raises kErrRayFlags.
  pdl_trigger();
  __shared__ int4 s_cache[kCacheWays * kRayThreads];
  __shared__ int4 s_blocks[VF_NORM_SHARED > 0 ? VF_NORM_SHARED : 1];
  if (threadIdx.x == 0) {
    unsigned* f = ray_flags + blockIdx.y * gridDim.x + blockIdx.x;
    unsigned v = 0;
    for (long spin = 0;; ++spin) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if (v != 0u) break;
      if (spin > (1l << 22)) {
        atomicOr(&ctr->error_flags, kErrRayFlags);
        break;
      }
      __nanosleep(64);
    }
    *f = 0u;
  }
  if (VF_NORM_SHARED > 0)
    for (int i = threadIdx.x; i < VF_NORM_SHARED; i += blockDim.x) s_blocks[i] = make_int4(0x7fffffff, 0, 0, -1);
  __syncthreads();
  const int fxi = blockIdx.x, fyi = blockIdx.y >> 1;
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int x = fxi * kFragmentSize + (lane & 7) + ((wq & 1) << 3);
  const int y = fyi * kFragmentSize + ((blockIdx.y & 1) << 3) + (lane >> 3) + ((wq >> 1) << 2);
  if (x >= in.width || y >= in.height) return;
  const size_t pix = (size_t)y * in.width + x;
  const float2 range = VF_RAY_REFINE_SPLIT ? __ldg(ranges + fyi * gridDim.x + fxi) : make_float2(0.f, 0.f);
  if (vstride == 1)
    ray_normal_body<1>(hv, vox, range, fp, in, vs, mu, x, y, pix, points, normals, s_cache, s_blocks);
  else
    ray_normal_body<2>(hv, vox, range, fp, in, vs, mu, x, y, pix, points, normals, s_cache, s_blocks);
}

// Measurement twin of k_raycast (vf_raycast_counters, never on the frame
// path): same maps, plus counters {table probes, voxel reads, rays, hits}.
__global__ void __launch_bounds__(kRayThreads)
    k_raycast_count(HashView hv, const uint32_t* __restrict__ vox, int vstride, const float2* __restrict__ ranges,
                    const FrameParams* __restrict__ fp, IntrD in, float vs, float mu, float4* __restrict__ points,
                    float4* __restrict__ normals, unsigned long long* counters) {
  __shared__ int4 s_cache[kCacheWays * kRayThreads];
  if (vstride == 1)
    raycast_body<1, true>(hv, vox, ranges, fp, in, vs, mu, points, normals, s_cache, counters);
  else
    raycast_body<2, true>(hv, vox, ranges, fp, in, vs, mu, points, normals, s_cache, counters);
}

}  // namespace vf
