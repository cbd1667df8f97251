// K1 — voxel-block allocation: mark (K1a), commit (K1b scan + apply) and the
// visible list (K1c).
//
// Reference: proj/include/voxfuse/engine/allocation.hpp:56-248 and
// proj/include/voxfuse/volume/hash_volume.hpp:161-258.
//
// Determinism.  The reference's mark_blocks writes one request per bucket with
// plain stores from many threads (allocation.hpp:134-136,155-159); with one
// worker the surviving request is the last visit in (raster index, DDA step)
// order.  K1a reproduces exactly that winner with a 64-bit atomicMax of the key
// ((pixel+1) << 12 | step) per bucket — the key is all that is stored; K1b
// re-walks the winning pixel's DDA to recover the block position.  K1b then
// commits the requests in ascending bucket order with prefix sums over the
// free-stack tops, which reproduces the sequential perform_allocations slot
// numbering (allocation.hpp:179-206) bit-for-bit; only when a free list would
// run dry does it fall back to the reference's sequential loop on one thread.
#include "vf_device.cuh"
#include "vf_kernels.h"

namespace vf {

namespace {

constexpr int kStepBits = 12;
constexpr unsigned long long kStepMask = (1ull << kStepBits) - 1ull;

// detail::dda_cells (allocation.hpp:60-96) in FP64.  Visit(cell, step) returns
// false to stop the walk early.
template <typename Visit>
__device__ __forceinline__ void dda_cells(const D3 p0, const D3 p1, Visit&& visit) {
  // per-axis state in named registers (an array indexed by the step axis
  // would live in local memory)
  int cx = __double2int_rz(floor(p0.x)), cy = __double2int_rz(floor(p0.y)), cz = __double2int_rz(floor(p0.z));
  const int ex = __double2int_rz(floor(p1.x)), ey = __double2int_rz(floor(p1.y)), ez = __double2int_rz(floor(p1.z));
  if (!visit(cx, cy, cz, 0)) return;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  auto setup = [&](double a0, double a1, int cell, int& step, double& t_max, double& t_delta) {
    const double d = a1 - a0;
    if (d > 0) {
      step = 1;
      t_max = (cell + 1 - a0) / d;
      t_delta = 1.0 / d;
    } else if (d < 0) {
      step = -1;
      t_max = (cell - a0) / d;
      t_delta = -1.0 / d;
    } else {
      step = 0;
      t_max = inf;
      t_delta = inf;
    }
  };
  int sx, sy, sz;
  double tmx, tmy, tmz, tdx, tdy, tdz;
  setup(p0.x, p1.x, cx, sx, tmx, tdx);
  setup(p0.y, p1.y, cy, sy, tmy, tdy);
  setup(p0.z, p1.z, cz, sz, tmz, tdz);
  const int max_steps = abs(ex - cx) + abs(ey - cy) + abs(ez - cz) + 3;
  for (int i = 0; i < max_steps && (cx != ex || cy != ey || cz != ez); ++i) {
    // ties pick the lower axis (strict <, allocation.hpp:89-90)
    int axis = 0;
    double tm = tmx;
    if (tmy < tm) {
      axis = 1;
      tm = tmy;
    }
    if (tmz < tm) {
      axis = 2;
      tm = tmz;
    }
    if (tm > 1.0) break;
    if (axis == 0) {
      cx += sx;
      tmx += tdx;
    } else if (axis == 1) {
      cy += sy;
      tmy += tdy;
    } else {
      cz += sz;
      tmz += tdz;
    }
    if (!visit(cx, cy, cz, i + 1)) return;
  }
}

// The per-pixel segment of mark_blocks (allocation.hpp:140-148).
__device__ __forceinline__ void pixel_segment(int x, int y, float d, const IntrD& in, const PoseD& c2w, float voxel_size,
                                              float mu, D3& p0, D3& p1) {
  const double inv_block = 1.0 / (double)(voxel_size * (float)kBlockSide);
  const D3 dir = mk((x - in.cx) / in.fx, (y - in.cy) / in.fy, 1.0);
  const double v = (double)d - (double)mu;
  const double near_d = (0.001 < v) ? v : 0.001;  // std::max(0.001, v)
  const double far_d = (double)d + (double)mu;
  const D3 q0 = apply(c2w, mk(dir.x * near_d, dir.y * near_d, dir.z * near_d));
  const D3 q1 = apply(c2w, mk(dir.x * far_d, dir.y * far_d, dir.z * far_d));
  p0 = mk(q0.x * inv_block, q0.y * inv_block, q0.z * inv_block);
  p1 = mk(q1.x * inv_block, q1.y * inv_block, q1.z * inv_block);
}

}  // namespace

// One thread computes the frame's derived camera parameters from the device
// pose (CameraF, integration.hpp:18-33; rgb camera integration.hpp:128).
__global__ void k_prep(const PoseD* __restrict__ pose, IntrD depth_in, IntrD rgb_in, PoseD depth_to_rgb,
                       FrameParams* __restrict__ fp) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const PoseD w2c = *pose;
  fp->w2c = w2c;
  fp->c2w = pose_inverse(w2c);
  fp->depth_cam = make_camf(w2c, depth_in);
  fp->rgb_cam = make_camf(pose_compose(depth_to_rgb, w2c), rgb_in);
}

// K1a: mark_blocks (allocation.hpp:137-168).  One thread per pixel.  Every
// CTA derives cam_to_world from the device pose itself; CTA 0 also publishes
// the frame's camera parameters (k_prep's job) for the later kernels.
// kCount: the measurement twin (vf_alloc_counters, never on the frame path):
// no requests and no frame parameters written; counts {pixels with depth,
// DDA cells probed (one bucket sector each), cells missing from the table}.
template <bool kCount>
__device__ __forceinline__ void mark_body(const float* __restrict__ depth, IntrD in, const PoseD* __restrict__ pose,
                                          IntrD rgb_in, PoseD depth_to_rgb, FrameParams* __restrict__ fp,
                                          HashView hv, float voxel_size, float mu, ShardSpec shard,
                                          unsigned long long* __restrict__ req_key, uint32_t* __restrict__ req_bits,
                                          Counters* __restrict__ ctr, unsigned long long* __restrict__ counts) {
  __shared__ PoseD s_c2w;
  if (threadIdx.x == 0) {
    const PoseD w2c = *pose;
    s_c2w = pose_inverse(w2c);
    if (!kCount && blockIdx.x == 0) {
      fp->w2c = w2c;
      fp->c2w = s_c2w;
      fp->depth_cam = make_camf(w2c, in);
      fp->rgb_cam = make_camf(pose_compose(depth_to_rgb, w2c), rgb_in);
    }
  }
  __syncthreads();
  // CTA = 32 x 8 pixel tile, warp = 8 x 4 patch: neighbouring rays walk the
  // same blocks (probe locality) and similar numbers of cells (divergence)
  const int tiles_x = (in.width + 31) >> 5;
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int x = (int)(blockIdx.x % tiles_x) * 32 + ((wq & 3) << 3) + (lane & 7);
  const int y = (int)(blockIdx.x / tiles_x) * 8 + ((wq >> 2) << 2) + (lane >> 3);
  unsigned n_cells = 0, n_missing = 0;
  const int pixel = y * in.width + x;
  const float d = (x < in.width && y < in.height) ? __ldg(depth + pixel) : 0.0f;
  if (!(d <= 0.0f)) {  // (kCount: every lane reaches the reduction below)
  D3 p0, p1;
  pixel_segment(x, y, d, in, s_c2w, voxel_size, mu, p0, p1);
  if (shard.count > 1) {
    // A pixel belongs to the shard owning the block of its observed surface
    // point; that shard allocates the whole +-mu band of the pixel, so every
    // surface is fused and raycast with its full band in one shard (blocks of
    // bands that straddle a seam are allocated by both neighbours).
    const double inv_block = 1.0 / (double)(voxel_size * (float)kBlockSide);
    const D3 dir = mk((x - in.cx) / in.fx, (y - in.cy) / in.fy, 1.0);
    const D3 ps = apply(s_c2w, mk(dir.x * (double)d, dir.y * (double)d, dir.z * (double)d));
    const int sbx = __double2int_rz(floor(ps.x * inv_block)), sby = __double2int_rz(floor(ps.y * inv_block)),
              sbz = __double2int_rz(floor(ps.z * inv_block));
    // ... and, with the halo, every shard owning a block within one block of
    // it, so trilinear / normal stencils never straddle a seam.
    bool mine = shard_owner(sbx, sby, sbz, shard) == shard.index;
    for (int k = 0; k < 27 && !mine && shard.halo; ++k)
      mine = shard_owner(sbx + k % 3 - 1, sby + (k / 3) % 3 - 1, sbz + k / 9 - 1, shard) == shard.index;
    if (!mine) {
      if (!kCount) return;
      n_cells = 0xFFFFFFFFu;  // not this shard's pixel: counted as such below
    }
  }
  const unsigned long long key_base = (unsigned long long)(pixel + 1) << kStepBits;
  // a missing block: bid for its bucket (the winning key reproduces the
  // reference's single-worker last writer)
  auto request = [&](int cx, int cy, int cz, int step) {
    if ((unsigned long long)step > kStepMask) {
      atomicOr(&ctr->error_flags, kErrDdaSteps);
      return;
    }
    const uint32_t bucket = hash_block(cx, cy, cz, hv.mask);
    const unsigned long long old = atomicMax(req_key + bucket, key_base | (unsigned long long)step);
    if (old == 0ull) atomicOr(req_bits + (bucket >> 5), 1u << (bucket & 31u));
  };
  if (n_cells != 0xFFFFFFFFu)
    dda_cells(p0, p1, [&](int cx, int cy, int cz, int step) {
      const bool missing = find_entry(hv, cx, cy, cz, kEntrySwappedOut) < 0;
      if (kCount) {
        ++n_cells;
        n_missing += missing ? 1u : 0u;
      } else if (missing) {
        request(cx, cy, cz, step);
      }
      return true;
    });
  }
  if constexpr (kCount) {
    const unsigned px = (!(d <= 0.0f) && n_cells != 0xFFFFFFFFu) ? 1u : 0u;
    if (n_cells == 0xFFFFFFFFu) n_cells = 0;
    unsigned long long v[3] = {px, n_cells, n_missing};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
      if ((threadIdx.x & 31) == 0 && v[k]) atomicAdd(counts + k, v[k]);
    }
  }
}

__global__ void __launch_bounds__(256) k_mark(const float* __restrict__ depth, IntrD in, const PoseD* __restrict__ pose,
                                              IntrD rgb_in, PoseD depth_to_rgb, FrameParams* __restrict__ fp,
                                              HashView hv, float voxel_size, float mu, ShardSpec shard,
                                              unsigned long long* __restrict__ req_key, uint32_t* __restrict__ req_bits,
                                              Counters* __restrict__ ctr) {
  pdl_enter();
  mark_body<false>(depth, in, pose, rgb_in, depth_to_rgb, fp, hv, voxel_size, mu, shard, req_key, req_bits, ctr,
                   nullptr);
}

__global__ void __launch_bounds__(256) k_mark_count(const float* __restrict__ depth, IntrD in,
                                                    const PoseD* __restrict__ pose, HashView hv, float voxel_size,
                                                    float mu, ShardSpec shard, unsigned long long* __restrict__ counts) {
  mark_body<true>(depth, in, pose, in, PoseD{}, nullptr, hv, voxel_size, mu, shard, nullptr, nullptr, nullptr, counts);
}

// Recover the block position a request key points at by re-walking that
// pixel's DDA (bit-identical FP64 arithmetic).
__device__ __forceinline__ void decode_request(unsigned long long key, const float* __restrict__ depth, const IntrD& in,
                                               const PoseD& c2w, float voxel_size, float mu, int& bx, int& by, int& bz) {
  const int pixel = (int)(key >> kStepBits) - 1;
  const int target = (int)(key & kStepMask);
  const int y = pixel / in.width, x = pixel - y * in.width;
  D3 p0, p1;
  pixel_segment(x, y, depth[pixel], in, c2w, voxel_size, mu, p0, p1);
  bx = by = bz = 0;
  dda_cells(p0, p1, [&](int cx, int cy, int cz, int step) {
    if (step == target) {
      bx = cx;
      by = cy;
      bz = cz;
      return false;
    }
    return true;
  });
}

// K1b-compact: perform_allocations' ascending walk over the requests
// (allocation.hpp:179-206) as an ordered compaction of the request bitmap,
// plus insert_block's bucket-full test (hash_volume.hpp:225-236) deciding
// which requests take an excess entry, and the prefix sums that fix every
// request's free-stack pops (k_alloc_apply), over all CTAs: one thread per
// bitmap word (256-word
// tiles in ascending order, dynamic tile tickets), a block scan of the
// packed (requests, excess) counts, then a decoupled look-back over the tiles
// for both prefixes at once.  The last tile publishes the frame's counters.
// scan[0] is the ticket, scan[1 + t] tile t's (status | requests | excess);
// the frame zeroes them before the launch.
__device__ __forceinline__ unsigned long long compact_flag(unsigned long long st, unsigned req, unsigned ex) {
  return (st << 62) | ((unsigned long long)req << 31) | (unsigned long long)ex;
}
__global__ void __launch_bounds__(kCompactThreads) k_alloc_compact(uint32_t* __restrict__ req_bits, int n_words,
                                                                   HashView hv, int* __restrict__ req_list,
                                                                   int* __restrict__ req_excess_rank,
                                                                   unsigned long long* scan, AllocMeta* __restrict__ meta,
                                                                   Counters* __restrict__ ctr,
                                                                   float2* __restrict__ ranges, int n_frag) {
  pdl_enter();
  __shared__ int s_tile;
  __shared__ int s_warp[kCompactThreads / 32];
  __shared__ unsigned s_base_req, s_base_ex;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_tile = (int)atomicAdd(scan, 1ull);
  for (int f = blockIdx.x * blockDim.x + tid; f < n_frag; f += gridDim.x * blockDim.x)
    ranges[f] = make_float2(3.402823466e+38f, 0.0f);  // RangeImage: invalid = (FLT_MAX, 0)
  __syncthreads();
  const int tile = s_tile;
  const int n_tiles = (n_words + kCompactThreads - 1) / kCompactThreads;
  const int w = tile * kCompactThreads + tid;
  const uint32_t bits = w < n_words ? __ldcg(req_bits + w) : 0u;
  // insert_block's bucket-full test: does the request need an excess entry?
  uint32_t needs_ex = 0u;
  for (uint32_t m = bits; m; m &= m - 1u) {
    const int b = __ffs(m) - 1;
    const int h = (w * 32 + b) * hv.bucket_size;
    bool has_free = false;
    if (hv.bucket_size == 2) {  // both slots' loads in flight at once
      const int s0 = load_entry_cg(hv.entries + h).block_state, s1 = load_entry_cg(hv.entries + h + 1).block_state;
      has_free = s0 == kEntryUnallocated || s1 == kEntryUnallocated;
    } else {
      for (int j = 0; j < hv.bucket_size && !has_free; ++j)
        has_free = load_entry_cg(hv.entries + h + j).block_state == kEntryUnallocated;
    }
    if (!has_free) needs_ex |= 1u << b;
  }
  // block exclusive scan of (requests << 16 | excess): both stay below 2^16 per tile
  const int v = (__popc(bits) << 16) | __popc(needs_ex);
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int wv = lane < kCompactThreads / 32 ? s_warp[lane] : 0;
    int wi = wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < kCompactThreads / 32) s_warp[lane] = wi - wv;
    const int agg = __shfl_sync(0xffffffffu, wi, kCompactThreads / 32 - 1);
    const unsigned agg_req = (unsigned)agg >> 16, agg_ex = (unsigned)agg & 0xFFFFu;
    unsigned long long* flags = scan + 1;
    if (lane == 0) atomicExch(flags + tile, compact_flag(tile == 0 ? 2ull : 1ull, agg_req, agg_ex));
    // decoupled look-back (tile order = ascending bucket order)
    unsigned pre_req = 0, pre_ex = 0;
    int j = tile - 1;
    while (j >= 0) {
      const int k = j - lane;
      unsigned long long f = 0;
      if (k >= 0) {
        do {
          asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(f) : "l"(flags + k) : "memory");
        } while ((f >> 62) == 0);
      }
      const unsigned st = k >= 0 ? (unsigned)(f >> 62) : 2u;
      const unsigned pmask = __ballot_sync(0xffffffffu, st == 2u);
      const int stop = pmask ? __ffs(pmask) - 1 : 31;
      const bool take = k >= 0 && lane <= stop;
      unsigned r = take ? (unsigned)((f >> 31) & 0x7FFFFFFFull) : 0u, e = take ? (unsigned)(f & 0x7FFFFFFFull) : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        r += __shfl_xor_sync(0xffffffffu, r, o);
        e += __shfl_xor_sync(0xffffffffu, e, o);
      }
      pre_req += r;
      pre_ex += e;
      if (pmask) break;
      j -= 32;
    }
    if (lane == 0) {
      if (tile > 0) atomicExch(flags + tile, compact_flag(2ull, pre_req + agg_req, pre_ex + agg_ex));
      s_base_req = pre_req;
      s_base_ex = pre_ex;
      if (tile == n_tiles - 1) {  // the frame's totals: allocation meta and per-frame counter resets
        const int n = (int)(pre_req + agg_req), n_ex = (int)(pre_ex + agg_ex);
        const Counters c = *ctr;
        AllocMeta m;
        m.n = n;
        m.n_excess = n_ex;
        m.vba_base = c.vba_top;
        m.excess_base = c.excess_top;
        m.slow = (n > c.vba_top || n_ex > c.excess_top) ? 1 : 0;
        if (!m.slow) {
          ctr->vba_top = c.vba_top - n;
          ctr->excess_top = c.excess_top - n_ex;
          ctr->allocated = n;
          ctr->dropped_vba_full = 0;
          ctr->dropped_excess_full = 0;
        }
        ctr->requested = n;
        ctr->n_requests = n;
        ctr->visible_count = 0;
        ctr->modified_voxels = 0;
        *meta = m;
      }
    }
  }
  __syncthreads();
  if (bits) {
    const int excl = s_warp[wid] + incl - v;
    int r = (int)s_base_req + (excl >> 16), e = (int)s_base_ex + (excl & 0xFFFF);
    for (uint32_t m = bits; m; m &= m - 1u) {
      const int b = __ffs(m) - 1;
      req_list[r] = w * 32 + b;
      req_excess_rank[r] = (needs_ex >> b) & 1u ? e++ : -1;
      ++r;
    }
    req_bits[w] = 0u;
  }
}

// K1b-apply: insert_block for every request (hash_volume.hpp:215-258).
__global__ void __launch_bounds__(256) k_alloc_apply(const float* __restrict__ depth, IntrD in,
                                                     const FrameParams* __restrict__ fp, float voxel_size, float mu,
                                                     HashEntry* __restrict__ entries, uint32_t mask, int bucket_size,
                                                     int ordered, unsigned long long* __restrict__ req_key,
                                                     const int* __restrict__ req_list,
                                                     const int* __restrict__ req_excess_rank,
                                                     const AllocMeta* __restrict__ meta, int* __restrict__ vba_slots,
                                                     int* __restrict__ excess_slots, int* __restrict__ alloc_list,
                                                     int alloc_cap, Counters* __restrict__ ctr,
                                                     unsigned long long* __restrict__ scan_reset, int n_reset) {
  pdl_enter();
  // k_alloc_compact has finished with its ticket and look-back words: clear
  // them for the next frame here (no memset node between k_mark and the
  // compaction, so that edge stays a programmatic one)
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < n_reset; i += blockDim.x) scan_reset[i] = 0ull;
  const AllocMeta m = *meta;
  const PoseD c2w = fp->c2w;
  if (!m.slow) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m.n; k += gridDim.x * blockDim.x) {
      const int bucket = req_list[k];
      const unsigned long long key = req_key[bucket];
      const int h = bucket * bucket_size;
      // The bucket's slot states, loaded before the request is decoded (one
      // request per bucket per frame: nothing else writes this bucket now).
      int st[2] = {0, 0};
      if (bucket_size == 2) {
        st[0] = entries[h].block_state;
        st[1] = entries[h + 1].block_state;
      }
      req_key[bucket] = 0ull;
      int bx, by, bz;
      decode_request(key, depth, in, c2w, voxel_size, mu, bx, by, bz);
      const int slot = vba_slots[m.vba_base - 1 - k];
      int idx = -1;
      const int er = req_excess_rank[k];
      if (er < 0) {
        for (int j = 0; j < bucket_size; ++j) {
          HashEntry* e = entries + h + j;
          if ((bucket_size == 2 ? st[j & 1] : e->block_state) == kEntryUnallocated) {
            e->x = (int16_t)bx;
            e->y = (int16_t)by;
            e->z = (int16_t)bz;
            e->block_state = slot;
            idx = h + j;
            break;
          }
        }
      } else {
        const int ex = excess_slots[m.excess_base - 1 - er];
        int last = h + bucket_size - 1;
        while (entries[last].offset > 0) last = ordered + entries[last].offset - 1;
        idx = ordered + ex;
        HashEntry* e = entries + idx;
        e->x = (int16_t)bx;
        e->y = (int16_t)by;
        e->z = (int16_t)bz;
        e->offset = 0;
        e->block_state = slot;
        entries[last].offset = ex + 1;
      }
      if (idx >= 0) {
        const int pos = atomicAdd(&ctr->alloc_count, 1);
        if (pos < alloc_cap)
          alloc_list[pos] = idx;
        else
          atomicOr(&ctr->error_flags, kErrAllocList);
      }
    }
    return;
  }
  // Slow path: a free list runs dry this frame — the reference's sequential
  // perform_allocations loop, verbatim, on one thread.
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  HashView hv{entries, mask, bucket_size, ordered};
  int vtop = ctr->vba_top, etop = ctr->excess_top;
  int allocated = 0, dvba = 0, dex = 0;
  for (int k = 0; k < m.n; ++k) {
    const int bucket = req_list[k];
    const unsigned long long key = req_key[bucket];
    req_key[bucket] = 0ull;
    int bx, by, bz;
    decode_request(key, depth, in, c2w, voxel_size, mu, bx, by, bz);
    const int existing = find_entry<true>(hv, bx, by, bz, kEntrySwappedOut);
    if (existing >= 0) {
      HashEntry* e = entries + existing;
      if (e->block_state >= 0) continue;
      if (vtop <= 0) {
        ++dvba;
        continue;
      }
      e->block_state = vba_slots[--vtop];
      continue;
    }
    const int h = (int)hash_block(bx, by, bz, mask) * bucket_size;
    int idx = -1;
    bool handled = false;
    for (int j = 0; j < bucket_size; ++j) {
      HashEntry* e = entries + h + j;
      if (e->block_state == kEntryUnallocated) {
        handled = true;
        if (vtop <= 0) {
          ++dvba;
          break;
        }
        e->x = (int16_t)bx;
        e->y = (int16_t)by;
        e->z = (int16_t)bz;
        e->block_state = vba_slots[--vtop];
        idx = h + j;
        break;
      }
    }
    if (!handled) {
      int last = h + bucket_size - 1;
      while (entries[last].offset > 0) last = ordered + entries[last].offset - 1;
      if (etop <= 0) {
        ++dex;
      } else {
        const int ex = excess_slots[--etop];
        if (vtop <= 0) {
          excess_slots[etop++] = ex;  // FreeStack::push of the unused excess index
          ++dvba;
        } else {
          idx = ordered + ex;
          HashEntry* e = entries + idx;
          e->x = (int16_t)bx;
          e->y = (int16_t)by;
          e->z = (int16_t)bz;
          e->offset = 0;
          e->block_state = vba_slots[--vtop];
          entries[last].offset = ex + 1;
        }
      }
    }
    if (idx >= 0) {
      ++allocated;
      const int pos = ctr->alloc_count++;
      if (pos < alloc_cap)
        alloc_list[pos] = idx;
      else
        ctr->error_flags |= kErrAllocList;
    }
  }
  ctr->vba_top = vtop;
  ctr->excess_top = etop;
  ctr->allocated = allocated;
  ctr->dropped_vba_full = dvba;
  ctr->dropped_excess_full = dex;
}

// K1c: build_visible_list (allocation.hpp:216-248) over the compact list of
// allocated entries instead of all 2.2 M table slots.  The result is the same
// set in a different order (order is irrelevant downstream).
__global__ void __launch_bounds__(256) k_visible(const HashEntry* __restrict__ entries, const int* __restrict__ alloc_list,
                                                 const FrameParams* __restrict__ fp, IntrD in, float vs, float near_clip,
                                                 float far_clip, int margin, int* __restrict__ visible_list,
                                                 Counters* __restrict__ ctr) {
  pdl_enter();
  __shared__ PoseD s_w2c;
  if (threadIdx.x < sizeof(PoseD) / sizeof(double))
    reinterpret_cast<double*>(&s_w2c)[threadIdx.x] = reinterpret_cast<const double*>(&fp->w2c)[threadIdx.x];
  __syncthreads();
  const int n = min(*(volatile int*)&ctr->alloc_count, 0x7fffffff);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int idx = alloc_list[i];
    const HashEntry e = load_entry(entries + idx);
    if (e.block_state < 0) continue;  // swapped out: never on the visible list
    if (block_projects_into_view(e.x, e.y, e.z, s_w2c, in, vs, near_clip, far_clip, margin)) {
      const int pos = warp_aggregated_add(&ctr->visible_count);
      visible_list[pos] = idx;
    }
  }
}

}  // namespace vf
