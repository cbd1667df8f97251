// Swap engine: voxel blocks paged between HBM and a host block store.
//
// Reference: GlobalCache / fuse_voxels / request_swap_ins / execute_swap_in /
// request_swap_outs / execute_swap_out (proj/include/voxfuse/engine/swap.hpp:45-253),
// run after integration (engine/pipeline_impl.hpp:104-113).
//
// B200 form.  The host store is pinned host memory mapped into the device
// address space: one slot of 512 device-layout voxels per stored block, with
// a device-side entry -> host-slot table and a device free stack of host
// slots.  Every step runs on the GPU inside the frame graph — no host
// round trip, no per-frame synchronisation:
//
//   k_swap_request   per allocated entry: the two request passes' state
//                    transitions (swap_visibility recomputed from the frame
//                    pose with the swap margin) and candidate lists;
//   k_swap_select    one CTA: the first min(B, free VBA) swap-in candidates and
//                    the first B swap-out candidates in ascending entry order
//                    (the reference's sequential loops), slot pops / pushes in
//                    the reference's stack order, table and state updates;
//   k_swap_transfer  one warp per staged block: swap-in reads the host slot over
//                    the C2C/PCIe link and fuses it into the fresh device block
//                    (secondary integration); swap-out streams the block to its
//                    host slot and resets it to default voxels.
//
// Entries swapped in this frame end ACTIVE, exactly as request_swap_outs
// leaves them in the reference (they were requested because visible), so the
// in and out transitions of one frame are evaluated in one pass.
#include "vf_device.cuh"
#include "vf_kernels.h"

namespace vf {

namespace {

constexpr uint8_t kSwInactive = 0, kSwNeedsIn = 1, kSwActive = 3, kSwNeedsOut = 4;

// The k smallest values of list[0..m) (distinct non-negative ints < 2^24),
// ascending, into out[0..k) (k <= kSwapSortCap).  Small lists are sorted
// whole; large ones first find the k-th smallest value with a two-pass
// 12-bit radix select, then sort the survivors.
__device__ void smallest_k(const int* __restrict__ list, int m, int k, int* __restrict__ out, int* s_sort,
                           int* s_hist, int* s_misc) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (k <= 0) return;
  int thr = 0x7fffffff;  // keep values <= thr
  if (m > kSwapSortCap) {
    int prefix = 0;  // high 12 bits of the threshold
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = tid; i < 4096; i += nt) s_hist[i] = 0;
      __syncthreads();
      for (int i = tid; i < m; i += nt) {
        const int v = __ldcg(list + i);
        if (pass == 0)
          atomicAdd(&s_hist[v >> 12], 1);
        else if ((v >> 12) == prefix)
          atomicAdd(&s_hist[v & 4095], 1);
      }
      __syncthreads();
      if (tid == 0) {  // bin holding the k-th smallest (k counts below earlier bins in pass 1)
        int need = pass == 0 ? k : s_misc[1];
        int b = 0;
        while (b < 4095 && s_hist[b] < need) need -= s_hist[b++];
        s_misc[0] = b;
        s_misc[1] = need;
      }
      __syncthreads();
      if (pass == 0) prefix = s_misc[0];
      else thr = (prefix << 12) | s_misc[0];
      __syncthreads();
    }
  }
  // gather the survivors (at most kSwapSortCap) and sort them
  if (tid == 0) s_misc[2] = 0;
  __syncthreads();
  for (int i = tid; i < m; i += nt) {
    const int v = __ldcg(list + i);
    if (v <= thr) {
      const int p = atomicAdd(&s_misc[2], 1);
      if (p < kSwapSortCap) s_sort[p] = v;
    }
  }
  __syncthreads();
  const int n = min(s_misc[2], kSwapSortCap);
  int P = 2;
  while (P < n) P <<= 1;
  for (int i = n + tid; i < P; i += nt) s_sort[i] = 0x7fffffff;
  __syncthreads();
  for (int kk = 2; kk <= P; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < P; i += nt) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int x = s_sort[i], y = s_sort[ixj];
          if ((x > y) == ((i & kk) == 0)) {
            s_sort[i] = y;
            s_sort[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < k; i += nt) out[i] = s_sort[i];
  __syncthreads();
}

}  // namespace

// request_swap_ins + request_swap_outs (swap.hpp:136-149, :204-227) over the
// allocated entries; swap_visibility is build_visible_list's enlarged-margin
// test (allocation.hpp:226-233).
__global__ void __launch_bounds__(256) k_swap_request(const HashEntry* __restrict__ entries,
                                                      const int* __restrict__ alloc_list,
                                                      const FrameParams* __restrict__ fp, IntrD in, float vs,
                                                      float near_clip, float far_clip, int margin, int swap_margin,
                                                      SwapDev sw, Counters* __restrict__ ctr) {
  pdl_enter();
  __shared__ PoseD s_w2c;
  if (threadIdx.x < sizeof(PoseD) / sizeof(double))
    reinterpret_cast<double*>(&s_w2c)[threadIdx.x] = reinterpret_cast<const double*>(&fp->w2c)[threadIdx.x];
  __syncthreads();
  const int n = *(volatile int*)&ctr->alloc_count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int idx = alloc_list[i];
    const HashEntry e = load_entry_cg(entries + idx);
    if (e.block_state < kEntrySwappedOut) continue;
    const BlockBox box = block_box(e.x, e.y, e.z, s_w2c, in, vs, near_clip, far_clip);
    const bool vis = box_in_view(box, in, margin) || box_in_view(box, in, swap_margin);
    uint8_t st = sw.state[idx];
    const uint8_t st0 = st;
    if (e.block_state == kEntrySwappedOut) {
      if (st == kSwNeedsIn && !vis) st = kSwInactive;
      if (sw.host_slot[idx] >= 0 && vis) st = kSwNeedsIn;
      if (st == kSwNeedsIn) sw.in_cand[warp_aggregated_add(&sw.ctr->n_in_cand)] = idx;
    } else {
      if (st == kSwInactive) st = vis ? kSwActive : kSwNeedsOut;
      else if (st == kSwActive && !vis) st = kSwNeedsOut;
      else if (st == kSwNeedsOut && vis) st = kSwActive;
      if (st == kSwNeedsOut) sw.out_cand[warp_aggregated_add(&sw.ctr->n_out_cand)] = idx;
    }
    if (st != st0) sw.state[idx] = st;
  }
}

// execute_swap_in / execute_swap_out bookkeeping (swap.hpp:151-198, :233-251)
// in one CTA: which blocks move, their VBA / host slots, table and states.
__global__ void __launch_bounds__(1024) k_swap_select(HashEntry* __restrict__ entries, int* __restrict__ vba_slots,
                                                      SwapDev sw, int buffer_blocks, int payload_bytes,
                                                      Counters* __restrict__ ctr) {
  pdl_enter();
  __shared__ int s_sort[kSwapSortCap];
  __shared__ int s_hist[4096];
  __shared__ int s_misc[4];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int m_in = sw.ctr->n_in_cand, m_out = sw.ctr->n_out_cand;
  const int vba_top = ctr->vba_top;
  const int host_top = sw.ctr->host_top;
  // swap in: pops succeed while the VBA has free slots, then the loop breaks
  const int k_in = min(min(buffer_blocks, m_in), vba_top);
  smallest_k(sw.in_cand, m_in, k_in, sw.stage_entry, s_sort, s_hist, s_misc);
  for (int r = tid; r < k_in; r += nt) {
    const int idx = sw.stage_entry[r];
    const int slot = vba_slots[vba_top - 1 - r];
    entries[idx].block_state = slot;
    sw.stage_slot[r] = slot;
    sw.stage_host[r] = sw.host_slot[idx];
    sw.host_slot[idx] = -1;  // store.clear
    sw.state[idx] = kSwActive;
  }
  // swap out: the first B candidates; host slots are popped before the
  // swap-in slots are returned, so one frame never reuses a slot it reads
  int k_out = min(buffer_blocks, m_out);
  int err = 0;
  if (k_out > host_top) {
    k_out = host_top;
    err = kErrHostStore;
  }
  smallest_k(sw.out_cand, m_out, k_out, sw.stage_entry + k_in, s_sort, s_hist, s_misc);
  const int vtop = vba_top - k_in;
  for (int r = tid; r < k_out; r += nt) {
    const int idx = sw.stage_entry[k_in + r];
    const int slot = entries[idx].block_state;
    const int hs = sw.host_free[host_top - 1 - r];
    vba_slots[vtop + r] = slot;  // vba_free().push, ascending entry order
    entries[idx].block_state = kEntrySwappedOut;
    sw.stage_slot[k_in + r] = slot;
    sw.stage_host[k_in + r] = hs;
    sw.host_slot[idx] = hs;
    sw.state[idx] = kSwInactive;
  }
  // the swap-out journal: the order the reference's file store would write
  // its records in (swap.hpp:233-251, block_store.cpp:96-115)
  const int jc = sw.ctr->journal_count;
  for (int r = tid; r < k_out; r += nt) sw.journal[(jc + r) & (kSwapJournal - 1)] = sw.stage_entry[k_in + r];
  __syncthreads();
  for (int r = tid; r < k_in; r += nt) sw.host_free[host_top - k_out + r] = sw.stage_host[r];
  if (tid == 0) {
    ctr->vba_top = vtop + k_out;
    ctr->error_flags |= err;
    SwapCounters& c = *sw.ctr;
    c.host_top = host_top - k_out + k_in;
    c.n_in_cand = 0;
    c.n_out_cand = 0;
    c.staged_in = k_in;
    c.staged_out = k_out;
    c.journal_count = jc + k_out;
    c.swapped_in = k_in;
    c.swapped_out = k_out;
    c.bytes_in = (unsigned long long)k_in * (unsigned long long)(payload_bytes + 4);
    c.bytes_out = (unsigned long long)k_out * (unsigned long long)(payload_bytes + 4);
  }
}

namespace {

// fuse_voxels (swap.hpp:96-131) on device-layout words: w0 = sdf | w << 16 |
// r << 24, w1 = g | b << 8 | w_color << 16.
template <bool kColor>
__device__ __forceinline__ void fuse(uint32_t h0, uint32_t h1, uint32_t& a0, uint32_t& a1, int max_weight) {
  uint32_t o0 = a0, o1 = a1;
  const int wh = (int)((h0 >> 16) & 0xFFu), wa = (int)((a0 >> 16) & 0xFFu);
  if (wh + wa > 0) {
    if (wa == 0) {
      o0 = (o0 & 0xFF000000u) | (h0 & 0x00FFFFFFu);
    } else if (wh != 0) {
      const float f = (sdf_to_float((int16_t)(h0 & 0xFFFFu)) * (float)wh +
                       sdf_to_float((int16_t)(a0 & 0xFFFFu)) * (float)wa) /
                      (float)(wh + wa);
      const uint32_t w = (uint32_t)(wh + wa < max_weight ? wh + wa : max_weight);
      o0 = (o0 & 0xFF000000u) | (uint32_t)(uint16_t)sdf_from_float(f) | (w << 16);
    }
  }
  if (kColor) {
    const int ch = (int)((h1 >> 16) & 0xFFu), ca = (int)((a1 >> 16) & 0xFFu);
    if (ca == 0) {
      o0 = (o0 & 0x00FFFFFFu) | (h0 & 0xFF000000u);
      o1 = (o1 & 0xFF000000u) | (h1 & 0x00FFFFFFu);
    } else if (ch != 0) {
      const float fch = (float)ch, fca = (float)ca, den = (float)(ch + ca);
      const float r = ((float)(h0 >> 24) * fch + (float)(a0 >> 24) * fca) / den;
      const float g = ((float)(h1 & 0xFFu) * fch + (float)(a1 & 0xFFu) * fca) / den;
      const float b = ((float)((h1 >> 8) & 0xFFu) * fch + (float)((a1 >> 8) & 0xFFu) * fca) / den;
      const uint32_t wc = (uint32_t)(ch + ca < max_weight ? ch + ca : max_weight);
      o0 = (o0 & 0x00FFFFFFu) | ((uint32_t)__float2uint_rz(r) << 24);
      o1 = (o1 & 0xFF000000u) | ((uint32_t)__float2uint_rz(g) & 0xFFu) | (((uint32_t)__float2uint_rz(b) & 0xFFu) << 8) |
           (wc << 16);
    }
  }
  a0 = o0;
  a1 = o1;
}

}  // namespace

// Moves the staged blocks, one warp per block.  which = 0: the swap-ins
// (host slot read over the link, fused into the fresh device block); they
// run before the raycast, which may read them.  which = 1: the swap-outs
// (device block streamed to its host slot, then reset); their entries were
// unlinked by k_swap_select, so nothing else in the frame reads these blocks
// and the copy overlaps the raycast on a side stream.
template <int kWords>
__device__ __forceinline__ void transfer_block(uint4* dev, uint4* host, bool in, int max_weight) {
  constexpr int kPerLane = kBlockVolume * kWords / 4 / 32;  // uint4 per lane: 4 (VoxelS) or 8 (VoxelSRgb)
  const int lane = threadIdx.x & 31;
  uint4 v[kPerLane];
  if (in) {
    uint4 h[kPerLane];
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) {  // all loads in flight before any use
      h[k] = __ldcv(host + lane + 32 * k);
      v[k] = dev[lane + 32 * k];
    }
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) {
      uint4 a = v[k];
      if (kWords == 1) {
        uint32_t d0 = 0, d1 = 0, d2 = 0, d3 = 0;
        fuse<false>(h[k].x, 0, a.x, d0, max_weight);
        fuse<false>(h[k].y, 0, a.y, d1, max_weight);
        fuse<false>(h[k].z, 0, a.z, d2, max_weight);
        fuse<false>(h[k].w, 0, a.w, d3, max_weight);
      } else {
        fuse<true>(h[k].x, h[k].y, a.x, a.y, max_weight);
        fuse<true>(h[k].z, h[k].w, a.z, a.w, max_weight);
      }
      dev[lane + 32 * k] = a;
    }
  } else {
    // TVoxel{} (voxel.hpp:29-30, :44-47)
    const uint4 def = kWords == 1 ? make_uint4(0x7FFFu, 0x7FFFu, 0x7FFFu, 0x7FFFu) : make_uint4(0x7FFFu, 0u, 0x7FFFu, 0u);
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) v[k] = dev[lane + 32 * k];
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) {
      __stcs(host + lane + 32 * k, v[k]);
      dev[lane + 32 * k] = def;
    }
  }
}

__global__ void __launch_bounds__(256) k_swap_transfer(uint32_t* __restrict__ voxels, int words_per_voxel,
                                                       SwapDev sw, int max_weight, int which) {
  pdl_enter();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int k_in = sw.ctr->staged_in, k_out = sw.ctr->staged_out;
  const int block_words = kBlockVolume * words_per_voxel;
  const int r0 = which == 0 ? 0 : k_in, r1 = which == 0 ? k_in : k_in + k_out;
  for (int r = r0 + gw; r < r1; r += nw) {
    uint4* dev = reinterpret_cast<uint4*>(voxels + (size_t)sw.stage_slot[r] * block_words);
    uint4* host = reinterpret_cast<uint4*>(host_block(sw, sw.stage_host[r], block_words));
    if (words_per_voxel == 1)
      transfer_block<1>(dev, host, which == 0, max_weight);
    else
      transfer_block<2>(dev, host, which == 0, max_weight);
  }
}

// The host store grows in pinned chunks as blocks leave (the reference keeps
// one host slot per hash entry, so its store never fills, swap.hpp:42-56):
// the chunk's slots go on top of the free stack, popped in ascending order.
__global__ void k_host_store_grow(SwapDev sw, int chunk, uint32_t* chunk_dev_ptr) {
  const int top = sw.ctr->host_top;
  const int first = chunk << kHostChunkShift;
  for (int i = threadIdx.x; i < kHostChunk; i += blockDim.x) sw.host_free[top + i] = first + kHostChunk - 1 - i;
  if (threadIdx.x == 0) {
    sw.host_chunks[chunk] = chunk_dev_ptr;
    sw.ctr->host_top = top + kHostChunk;
  }
}

}  // namespace vf
