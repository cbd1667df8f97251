// Kernel declarations shared between the kernel translation units and the
// host runtime (vf_api.cu).
#pragma once

#include "vf_device.cuh"

namespace vf {

#ifndef VF_ICP_THREADS
#define VF_ICP_THREADS 256
#endif
#ifndef VF_ICP_MIN_BLOCKS
#define VF_ICP_MIN_BLOCKS 1
#endif
#ifndef VF_ICP_INFLIGHT
#define VF_ICP_INFLIGHT 1  // pixels per pipelined step (2 with VF_ICP_LEGACY_LOOP)
#endif
constexpr int kIcpThreads = VF_ICP_THREADS;
constexpr int kInflight = VF_ICP_INFLIGHT;  // ICP pixels in flight per thread
constexpr int kMaxIcpGrid = 512;  // partial-sum loop bound (grid <= 512 CTAs)
constexpr int kMaxLevels = 6;

struct AllocMeta {
  int n, n_excess, vba_base, excess_base, slow;
  int pad[3];
};

struct IcpLevel {
  const float* depth;
  const double* ux;  // (x - cx) / fx per column
  const double* uy;  // (y - cy) / fy per row
  int w, h;
  double fx, fy, cx, cy;
};

constexpr int kTraceRow = 48;  // level, iter, 21 H, 6 g, cost, count, rot_only, c2w (12), 4 timers

struct IcpResult {
  PoseD pose;
  double final_cost;
  int ok, iterations, valid_points, trace_rows;
};

struct IcpArgs {
  IcpLevel lv[kMaxLevels];
  int levels, rotation_only_levels, max_iterations, min_valid_points;
  float dist_thr, conv_eps;
  double max_condition;
  const float4* points;
  const float4* normals;
  IntrD map;
  PoseD* state_pose;
  const PoseD* initial;  // optional initial world->camera pose (nullptr: the render pose)
  int update_state;      // 1: write the tracked pose back (pipeline); 0: pure icp_track (stage call)
  IcpResult* result;
  double* partials;
  double* trace;
  int trace_cap;
  int max_slots;  // pixel slots per thread staged in shared memory
  int level_hi, level_lo;  // levels run by this launch (coarse to fine)
  void* ctl_io;            // controller state handed from the cluster to the grid kernel
  int ctl_in;              // 1: start from *ctl_io instead of the pose
  int is_last;             // 1: write the IcpResult (and the tracked pose)
  // Pixel-sharded ICP (vf_settings.shard_icp): this shard sums the terms of
  // every xranks-th CTA-sized pixel chunk (offset xrank) and the 29 per-shard
  // totals of each iteration are summed across the shards through peer
  // memory (IcpXchg).  xranks == 1: no exchange.
  int xrank, xranks;
  double* xpeer[16];               // every shard's IcpXchg (own included; P2P / IPC mapped)
  unsigned long long* xstate;      // own IcpXchg::local (local totals, flags, exchange counter)
  Counters* ctr;                   // error flag on an exchange timeout
};

// Per-shard exchange area of the sharded ICP, one cudaMalloc (IPC-shareable):
//   [0, 2*16*32)        doubles: totals written by shard r for exchange parity p at [(p*16 + r)*32]
//   [1024, 1024 + 32)   u64: flags, shard r's latest exchange number at [1024 + p*16 + r]
//   local (xstate): [0] exchange counter, [1] local flag, [2..] 2 x 32 doubles of the summed totals
constexpr int kXchgTotals = 0, kXchgFlags = 1024, kXchgLocal = 1024 + 32;
constexpr size_t kXchgBytes = sizeof(double) * (kXchgLocal + 2 + 64);

__global__ void k_prep(const PoseD* pose, IntrD depth_in, IntrD rgb_in, PoseD depth_to_rgb, FrameParams* fp);
struct ShardSpec {
  int count, index, shift;  // G shards, this shard, super-block shift s
  int halo;                 // also fuse bands whose surface block neighbours this shard's territory
};
// Owner of a block: hash of its super-block (2^s blocks per axis) mod G.
__host__ __device__ inline int shard_owner(int bx, int by, int bz, const ShardSpec& sp) {
  if (sp.count <= 1) return 0;
  const uint32_t h = ((uint32_t)(bx >> sp.shift) * 73856093u) ^ ((uint32_t)(by >> sp.shift) * 19349669u) ^
                     ((uint32_t)(bz >> sp.shift) * 83492791u);
  return (int)(h % (uint32_t)sp.count);
}

__global__ void k_mark_count(const float* depth, IntrD in, const PoseD* pose, HashView hv, float voxel_size, float mu,
                             ShardSpec shard, unsigned long long* counts);
__global__ void k_mark(const float* depth, IntrD in, const PoseD* pose, IntrD rgb_in, PoseD depth_to_rgb,
                       FrameParams* fp, HashView hv, float voxel_size, float mu, ShardSpec shard,
                       unsigned long long* req_key, uint32_t* req_bits, Counters* ctr);
constexpr int kCompactThreads = 256;  // k_alloc_compact: one bitmap word per thread
__global__ void k_alloc_compact(uint32_t* req_bits, int n_words, HashView hv, int* req_list, int* req_excess_rank,
                                unsigned long long* scan, AllocMeta* meta, Counters* ctr, float2* ranges, int n_frag);
__global__ void k_alloc_apply(const float* depth, IntrD in, const FrameParams* fp, float voxel_size, float mu,
                              HashEntry* entries, uint32_t mask, int bucket_size, int ordered,
                              unsigned long long* req_key, const int* req_list, const int* req_excess_rank,
                              const AllocMeta* meta, int* vba_slots, int* excess_slots, int* alloc_list,
                              int alloc_cap, Counters* ctr, unsigned long long* scan_reset, int n_reset);
__global__ void k_visible(const HashEntry* entries, const int* alloc_list, const FrameParams* fp, IntrD in, float vs,
                          float near_clip, float far_clip, int margin, int* visible_list, Counters* ctr);
__global__ void k_integrate_s(const HashEntry* entries, const int* visible_list, const Counters* ctr, void* voxels,
                              const float* depth, const FrameParams* fp, float vs, float mu, int max_weight,
                              int stop_at_max);
// Launches k_integrate_s / k_integrate_rgb with their dynamic shared memory (staging ring).
void launch_integrate(int grid, cudaStream_t st, bool color, bool fast, const HashEntry* entries, const int* visible_list,
                      const Counters* ctr, void* voxels, const float* depth, const uint8_t* rgb,
                      const FrameParams* fp, float vs, float mu, int max_weight, int stop_at_max);
__global__ void k_integrate_rgb(const HashEntry* entries, const int* visible_list, const Counters* ctr, void* voxels,
                                const float* depth, const uint8_t* rgb, const FrameParams* fp, float vs, float mu,
                                int max_weight, int stop_at_max);
__global__ void k_ranges(const HashEntry* entries, const int* visible_list, const Counters* ctr,
                         const FrameParams* fp, IntrD in, float vs, float near_clip, float far_clip, float2* ranges,
                         int frag_w);
// the march's occupancy points (CTAs per SM): large frames / frames up to VF_RAY_SMALL_PIXELS
#ifndef VF_RAY_MIN_BLOCKS
#define VF_RAY_MIN_BLOCKS 8
#endif
#ifndef VF_RAY_MIN_BLOCKS_SMALL
#define VF_RAY_MIN_BLOCKS_SMALL 6
#endif
#ifndef VF_RAY_SMALL_PIXELS
#define VF_RAY_SMALL_PIXELS (640 * 480)
#endif
template <int kMinBlocks>
__global__ void k_raycast(HashView hv, const uint32_t* vox, int vstride, const float2* ranges, const FrameParams* fp,
                          IntrD in, float vs, float mu, float4* points, float4* normals, unsigned* ray_flags);
__global__ void k_ray_normals(HashView hv, const uint32_t* vox, int vstride, const float2* ranges, const FrameParams* fp,
                              IntrD in, float vs, float mu, float4* points, float4* normals, unsigned* ray_flags,
                              Counters* ctr);
__global__ void k_raycast_count(HashView hv, const uint32_t* vox, int vstride, const float2* ranges,
                                const FrameParams* fp, IntrD in, float vs, float mu, float4* points, float4* normals,
                                unsigned long long* counters);
__global__ void k_pyramid(const float* depth0, int w0, int h0, int levels, float* out);
__global__ void k_icp(IcpArgs a);
__global__ void k_icp_cluster(IcpArgs a);
__global__ void k_synth(int n_spheres, const double* spheres, int n_planes, const double* planes, PoseD c2w,
                        IntrD in, double near_clip, double far_clip, float* depth, uint8_t* rgb);
__global__ void k_fill_voxels(uint32_t* vox, size_t n_voxels, int words_per_voxel);
__global__ void k_disparity_to_depth(const uint16_t* disp, int n, int big_endian, float a, float b, float fx,
                                     float max_depth, float* depth);
__global__ void k_rebuild_alloc_list(const HashEntry* entries, int n, int* alloc_list, int cap, Counters* ctr);
__global__ void k_init_ranges(float2* ranges, int n);
__global__ void k_reset_visible(Counters* ctr);
__global__ void k_set_pose(PoseD* dst, PoseD pose);
__global__ void k_divtest_const(float b, uint32_t lo_bits, uint32_t n_bits, unsigned long long* mism);
__global__ void k_divtest_rand(float amax, float bmin, float bmax, unsigned long long n, unsigned long long* mism);

// raycast epilogues (vf_render.cu)
__global__ void k_forward_project(HashView hv, const uint32_t* vox, const float4* points, IntrD in, int stride,
                                  float vs, unsigned long long* scan, float* out_points, float* out_colors,
                                  Counters* ctr);
__global__ void k_render_image(HashView hv, const uint32_t* vox, const float4* points, const float4* normals,
                               const PoseD* w2c, IntrD in, float vs, int color, uint8_t* out);
__global__ void k_depth_max(const float* depth, int n, int* dmax_bits);
__global__ void k_colourize_depth(const float* depth, int n, const int* dmax_bits, uint8_t* out);
constexpr int kSurfaceStride = 4;  // pipeline_impl.hpp:219
constexpr int kFpTileItems = 256;

// other trackers (vf_track.cu)
struct RenCtl {
  PoseD init;  // ren_refine's init_world_to_cam
  PoseD c2w;
  double final_cost;
  int iterations, valid_points, done, ok;
};
__global__ void k_ren_init(const IcpResult* icp, const PoseD* state, int use_icp, const PoseD* explicit_init,
                           RenCtl* ctl);
__global__ void k_ren_terms(const float* depth, IntrD in, HashView hv, const uint32_t* vox, int vstride, float vs,
                            double sigma, const RenCtl* ctl, double* partials);
__global__ void k_ren_ctl(const double* partials, int nparts, RenCtl* ctl, int min_valid_points, double max_condition,
                          float convergence_eps);
__global__ void k_ren_finish(RenCtl* ctl, int combine_icp, IcpResult* res, PoseD* state, int update_state);
struct ColorLevel {
  const float4* color;
  const float4* gx;
  const float4* gy;
  int w, h;
  double fx, fy, cx, cy;
};
struct ColorTrackArgs {
  ColorLevel lv[kMaxLevels];
  int levels, stride, max_iterations, min_valid_points;
  float convergence_eps;
  const float* points;  // float3 surface points / colours (forward_project_points)
  const float* colors;
  const int* count;     // device count (Counters::surface_count), or nullptr: n
  int n;
  PoseD* state;
  const PoseD* explicit_init;  // nullptr: *state
  IcpResult* result;
  int update_state;
  double* partials;  // grid launch: 2 x gridDim x 32 per-CTA sums (double-buffered)
  int exact_solve;   // 1: every damped step through the reference's pivoted LDLT (vf_settings.tracker_exact_solve)
};
__global__ void k_cpyr_base(const uint8_t* rgb, int n, float4* out);
__global__ void k_cpyr_down(const float4* src, int sw, int sh, float4* dst);
__global__ void k_cpyr_grad(const float4* src, int w, int h, float4* gx, float4* gy);
#ifndef VF_COLOR_THREADS
#define VF_COLOR_THREADS 256
#endif
constexpr int kColorThreads = VF_COLOR_THREADS;  // colour tracker CTA size (one point per thread per evaluation)
__global__ void k_color_track(ColorTrackArgs a);
__global__ void k_track_fail(const PoseD* state, IcpResult* res);

// swap engine (vf_swap.cu)
constexpr int kSwapSortCap = 4096;  // max swap_buffer_blocks
struct SwapCounters {
  int host_top;  // free host-store slots
  int n_in_cand, n_out_cand;
  int staged_in, staged_out;
  int swapped_in, swapped_out;  // SwapMetrics (swap.hpp:28-40) of the last frame
  int journal_count;  // swap-outs ever journalled (sw.journal, a ring of kSwapJournal entries)
  unsigned long long bytes_in, bytes_out;
};
struct SwapDev {
  uint8_t* state;     // SwapState per entry (swap.hpp:19-25)
  int* host_slot;     // entry -> host-store slot, -1: no stored data (BlockStore::has)
  int* host_free;     // free host slots (stack)
  int* in_cand;       // this frame's needs_swap_in / needs_swap_out entries
  int* out_cand;
  int* stage_entry;   // staged transfers: swap-ins first, then swap-outs
  int* stage_slot;
  int* stage_host;
  int* journal;       // ring of swapped-out entry indices, in swap-out order (vf_swap_drain)
  uint32_t** host_chunks;  // pinned, device-mapped chunks of kHostChunk slots of 512 device-layout voxels
  SwapCounters* ctr;
};
constexpr int kSwapJournal = 1 << 16;
constexpr int kHostChunkShift = 12;  // 4096 host-store slots per pinned chunk
constexpr int kHostChunk = 1 << kHostChunkShift;
__device__ __forceinline__ uint32_t* host_block(const SwapDev& sw, int slot, int block_words) {
  return sw.host_chunks[slot >> kHostChunkShift] + (size_t)(slot & (kHostChunk - 1)) * block_words;
}
// appends a new chunk's slots to the free stack (host-store growth between frames)
__global__ void k_host_store_grow(SwapDev sw, int chunk, uint32_t* chunk_dev_ptr);
__global__ void k_swap_request(const HashEntry* entries, const int* alloc_list, const FrameParams* fp, IntrD in,
                               float vs, float near_clip, float far_clip, int margin, int swap_margin, SwapDev sw,
                               Counters* ctr);
__global__ void k_swap_select(HashEntry* entries, int* vba_slots, SwapDev sw, int buffer_blocks, int payload_bytes,
                              Counters* ctr);
__global__ void k_swap_transfer(uint32_t* voxels, int words_per_voxel, SwapDev sw, int max_weight, int which);

constexpr int kMaxShards = 16;
struct ShardGroupArgs {
  int n;
  const unsigned long long* keys[kMaxShards];
  float4* points[kMaxShards];
  float4* normals[kMaxShards];
};
__global__ void k_shard_keys(const float4* points, const FrameParams* fp, int npix, int rank, unsigned long long* keys);
__global__ void k_shard_select(const unsigned long long* keys_min, int npix, int rank, float4* points, float4* normals);
__global__ void k_shard_group_composite(ShardGroupArgs g, int npix);
// The nearest-depth composite over peer memory (one process per GPU, CUDA IPC
// mappings over NVLink; or shards sharing a device).  Flags area per shard:
// [kP2PReady + r] / [kP2PDone + r] = the latest frame shard r published /
// finished reading; [kP2PSeq] this shard's frame counter.
constexpr int kP2PReady = 0, kP2PDone = 16, kP2PSeq = 32, kP2PMask = 33, kP2PFlagWords = 40;
struct P2PArgs {
  int n, rank;
  const unsigned long long* keys[kMaxShards];
  const float4* points[kMaxShards];
  const float4* normals[kMaxShards];
  unsigned long long* flags[kMaxShards];  // every shard's flags area (own included)
  Counters* ctr;
};
__global__ void k_p2p_wait_done(P2PArgs a);
__global__ void k_p2p_signal_ready(P2PArgs a);
__global__ void k_p2p_wait_ready(P2PArgs a);
__global__ void k_p2p_composite(P2PArgs a, float4* points, float4* normals, int npix);
__global__ void k_p2p_signal_done(P2PArgs a);
int nccl_unique_id(void* out);
int nccl_comm_init(void** comm, const void* id_bytes, int nranks, int rank);
void nccl_comm_destroy(void* comm);
int nccl_composite(void* comm, cudaStream_t st, const FrameParams* fp, float4* points, float4* normals,
                   unsigned long long* keys, int npix, int rank);

// VF_PDL=0 turns programmatic dependent launch off (vf_api.cu).
bool pdl_enabled();
// A kernel launch on a frame stream with the programmatic-serialization
// attribute (the kernel starts with pdl_enter / pdl_wait).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace vf
