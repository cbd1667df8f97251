// Host runtime behind the C ABI (include/voxfuse_b200.h): one context owns
// the device-resident volume (hash table, VBA, free stacks), the per-frame
// scratch, the tracking state (pose, point / normal maps) and one CUDA
// stream; a frame is one CUDA-graph replay (pyramid -> ICP -> prep -> mark ->
// commit -> visible -> integrate -> ranges -> raycast), and the only host
// synchronisation per frame is the optional stats readback.
//
// Reference orchestration this replaces: Pipeline<TVoxel, hash>
// (proj/include/voxfuse/engine/pipeline_impl.hpp:33-248).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/voxfuse_b200.h"
#include "vf_device.cuh"
#include "vf_kernels.h"

using namespace vf;

namespace {

constexpr int kNumEvents = 16;
constexpr int kTraceCap = 256;

// Everything the host reads back after a frame, contiguous for one D2H copy.
struct DevState {
  Counters ctr;
  IcpResult icp;
  PoseD pose;
  PoseD init_pose;  // optional ICP initial pose (vf_stage_icp)
  FrameParams fp;
  AllocMeta meta;
  SwapCounters swap;
  RenCtl ren;
};

PoseD pose_from(const double* p) {
  PoseD o;
  std::memcpy(o.r, p, 9 * sizeof(double));
  std::memcpy(o.t, p + 9, 3 * sizeof(double));
  return o;
}
void pose_to(const PoseD& p, double* o) {
  std::memcpy(o, p.r, 9 * sizeof(double));
  std::memcpy(o + 9, p.t, 3 * sizeof(double));
}
IntrD intr_of(const vf_intrinsics& i) { return IntrD{i.fx, i.fy, i.cx, i.cy, i.width, i.height}; }
// Intrinsics::half (core/intrinsics.hpp:22-31)
IntrD intr_half(const IntrD& in) {
  IntrD h;
  h.fx = in.fx * 0.5;
  h.fy = in.fy * 0.5;
  h.cx = (in.cx - 0.5) * 0.5;
  h.cy = (in.cy - 0.5) * 0.5;
  h.width = (in.width + 1) / 2;
  h.height = (in.height + 1) / 2;
  return h;
}

}  // namespace

constexpr int kMaxFramesInFlight = VF_MAX_FRAMES_IN_FLIGHT;

struct vf_ctx {
  vf_settings s;
  vf_calib calib;
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // parallel graph branch (k_ranges)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_join2 = nullptr;  // swap-out transfers beside the raycast
  std::string err;

  int vsize = 4;
  int ordered = 0, entry_count = 0;
  uint32_t mask = 0;
  IntrD din{}, rgbin{};
  PoseD depth_to_rgb{};
  int npix = 0, frag_w = 0, frag_h = 0;
  std::vector<IntrD> levels;
  size_t pyr_floats = 0;

  // device buffers
  HashEntry* entries = nullptr;
  void* voxels = nullptr;
  int* vba_slots = nullptr;
  int* excess_slots = nullptr;
  unsigned long long* req_key = nullptr;
  uint32_t* req_bits = nullptr;
  int* req_list = nullptr;
  int* req_excess_rank = nullptr;
  unsigned long long* compact_scan = nullptr;  // k_alloc_compact's ticket + look-back flags
  int* alloc_list = nullptr;
  int alloc_cap = 0;
  int* visible_list = nullptr;
  DevState* dstate = nullptr;
  float* depth = nullptr;
  uint16_t* disp = nullptr;  // raw disparity frame (process_raw_frame)
  float* image_depth_scratch = nullptr;
  uint8_t* rgb = nullptr;
  float* pyr = nullptr;
  float2* ranges = nullptr;
  unsigned* ray_flags = nullptr;  // k_raycast -> k_ray_normals per-CTA completion flags
  float4* points = nullptr;
  float4* normals = nullptr;
  double* partials = nullptr;
  double* utab = nullptr;  // per level: (x - cx) / fx then (y - cy) / fy
  std::vector<size_t> utab_off;
  double* trace = nullptr;
  int icp_slots = 0;
  size_t icp_smem = 0;
  int icp_cluster = 0;      // CTAs of the coarse-level cluster (0: no cluster path)
  int icp_coarse_levels = 0;  // levels run by the cluster kernel
  void* icp_ctl = nullptr;
  void* flush_buf = nullptr;
  size_t flush_bytes = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> flush_ev;  // per vf_flush_l2 call, until vf_flush_time
  // sharding
  ShardSpec shard{1, 0, 2, 1};
  void* nccl_comm = nullptr;
  unsigned long long* shard_keys = nullptr;
  int icp_grid = 0;
  // colour-tracker surface list (forward_project_points, raycast.hpp:495-509)
  float* surf_points = nullptr;
  float* surf_colors = nullptr;
  unsigned long long* surf_scan = nullptr;  // tile ticket + look-back flags
  int surf_cap = 0, surf_tiles = 0;
  uint8_t* image = nullptr;  // get_image output (w*h*3) + depth-max word
  int* image_dmax = nullptr;
  // other trackers (vf_track.cu)
  double* ren_partials = nullptr;
  int ren_grid = 0;
  std::vector<IntrD> rgb_levels;  // colour pyramid intrinsics (Intrinsics::half per level)
  float4* cpyr = nullptr;         // per level: colour, grad_x, grad_y
  std::vector<size_t> cpyr_off;
  // swap engine (vf_swap.cu): device arrays + the pinned, mapped host store
  bool swapping = false;
  SwapDev sw{};
  std::vector<uint32_t*> host_chunk_ptrs;  // host pointers of the pinned store chunks
  std::vector<uint32_t*> host_dev_ptrs;    // their device-mapped aliases (sw.host_chunks)
  int host_cap = 0;       // host-store slots allocated (whole chunks)
  int host_max = 0;       // slots it may grow to: one per hash entry (the reference's bound) or swap_host_blocks
  long host_top_lb = 0;   // lower bound on the device's free host slots (host_top) before the next frame
  int journal_read = 0;   // swap-out journal position vf_swap_drain has reached

  // host state
  DevState* hstate = nullptr;  // pinned
  PoseD* hpose = nullptr;      // pinned staging for vf_set_pose
  int frame = 0;
  bool maps_valid = false;
  bool rgb_valid = false;

  // graphs: [tracking][rgb]
  // frame graphs per [tracking][rgb][stage timing]
  cudaGraphExec_t graph[2][2][2] = {};
  bool graphs_ok = true;

  cudaEvent_t ev[kNumEvents] = {};
  cudaEvent_t ev_frame0 = nullptr, ev_frame1 = nullptr;
  bool profiling = false;
  bool stage_timing = false;
  // pixel-sharded ICP (vf_settings.shard_icp): the exchange area and every
  // shard's mapping of its own (vf_shard_icp_link / _link_local)
  double* icp_xchg = nullptr;
  double* icp_peers[kMaxShards] = {};
  int icp_linked = 0;
  std::vector<void*> ipc_opened;
  // nearest-depth composite over peer memory (vf_shard_p2p_link / _link_local)
  unsigned long long* p2p_flags = nullptr;
  P2PArgs p2p{};
  int p2p_linked = 0;
  long l2_persist_bytes = 0;  // hash-table bytes under the persisting access-policy window  // per-frame FrameStats::ms_* (event nodes in the frame graph)
  double stage_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long profiled_frames = 0;
  int launches_last = 0;

  // streaming submission (vf_submit_frame / vf_collect_frame): the upload of
  // frame n + 1 runs on `copy` into a staging slot while frame n computes
  cudaStream_t copy = nullptr;
  float* depth_stage[kMaxFramesInFlight] = {};
  uint8_t* rgb_stage[kMaxFramesInFlight] = {};
  DevState* hstate_q[kMaxFramesInFlight] = {};  // pinned, one per slot
  cudaEvent_t ev_up[kMaxFramesInFlight] = {}, ev_consumed[kMaxFramesInFlight] = {};
  cudaEvent_t ev_done[kMaxFramesInFlight] = {}, ev_q0[kMaxFramesInFlight] = {}, ev_q1[kMaxFramesInFlight] = {};
  int q_head = 0, q_count = 0;
  int q_frame[kMaxFramesInFlight] = {};
  bool q_track[kMaxFramesInFlight] = {};
};

#define VF_CUDA(ctx, call)                                                                  \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      if (ctx) (ctx)->err = std::string(#call) + ": " + cudaGetErrorString(e_);             \
      std::fprintf(stderr, "[voxfuse_b200] %s failed: %s\n", #call, cudaGetErrorString(e_)); \
      return VF_ERR_CUDA;                                                                   \
    }                                                                                       \
  } while (0)

// Programmatic dependent launch between the frame's consecutive main-stream
// kernels (launch_pdl, vf_kernels.h): each kernel's launch and prologue
// overlap its predecessor's tail.  VF_PDL=0 turns it off (A/B runs).
bool vf::pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VF_PDL");
    return e ? std::atoi(e) != 0 : true;
  }();
  return on;
}

namespace {

HashView hash_view(vf_ctx* c) { return HashView{c->entries, c->mask, c->s.bucket_size, c->ordered}; }

// first_level 1: icp_track on the pyramid without its full-resolution level
// (the icp_ren tracker, pipeline_impl.hpp:189-195).
bool frame_trace() {
  static const bool on = std::getenv("VF_ICP_TRACE") != nullptr;
  return on;
}

// trace: record the per-iteration sums and phase timers (vf_icp_trace) —
// always for stage calls, in frames only with VF_ICP_TRACE set (the extra
// stores sit on the critical path of CTA 0 between grid barriers).
int launch_icp(vf_ctx* c, cudaStream_t st, bool with_initial = false, bool update_state = true,
               int first_level = 0, bool trace = true, bool exchange = false) {
  IcpArgs a{};
  a.xrank = 0;
  a.xranks = 1;
  a.ctr = &c->dstate->ctr;
  if (exchange && c->icp_linked > 1) {  // pixel-sharded ICP, sums exchanged through peer memory
    a.xrank = c->shard.index;
    a.xranks = c->icp_linked;
    for (int r = 0; r < c->icp_linked; ++r) a.xpeer[r] = c->icp_peers[r];
    a.xstate = reinterpret_cast<unsigned long long*>(c->icp_xchg + kXchgLocal);
  }
  const int L = c->s.hierarchy_levels - first_level;
  size_t off = 0;
  for (int g = 0; g < c->s.hierarchy_levels; ++g) {
    const IntrD& in = c->levels[g];
    const int l = g - first_level;
    if (l >= 0) {
      a.lv[l].depth = g == 0 ? c->depth : c->pyr + off;
      a.lv[l].ux = c->utab + c->utab_off[g];
      a.lv[l].uy = c->utab + c->utab_off[g] + in.width;
      a.lv[l].w = in.width;
      a.lv[l].h = in.height;
      a.lv[l].fx = in.fx;
      a.lv[l].fy = in.fy;
      a.lv[l].cx = in.cx;
      a.lv[l].cy = in.cy;
    }
    if (g > 0) off += (size_t)in.width * in.height;
  }
  a.levels = L;
  a.rotation_only_levels = c->s.rotation_only_levels;
  a.max_iterations = c->s.max_iterations;
  a.min_valid_points = c->s.min_valid_points;
  a.dist_thr = c->s.icp_dist_threshold;
  a.conv_eps = c->s.convergence_eps;
  a.max_condition = c->s.max_condition;
  a.points = c->points;
  a.normals = c->normals;
  a.map = c->din;
  a.state_pose = &c->dstate->pose;
  a.initial = with_initial ? &c->dstate->init_pose : nullptr;
  a.update_state = update_state ? 1 : 0;
  a.result = &c->dstate->icp;
  a.partials = c->partials;
  a.trace = trace ? c->trace : nullptr;
  a.trace_cap = kTraceCap;
  a.max_slots = c->icp_slots;
  a.ctl_io = c->icp_ctl;
  const int coarse = c->icp_cluster ? std::min(c->icp_coarse_levels, L) : 0;
  if (coarse > 0) {
    // coarse levels in one thread-block cluster (cluster barrier + DSMEM)
    IcpArgs ac = a;
    ac.level_hi = L - 1;
    ac.level_lo = L - coarse;
    ac.ctl_in = 0;
    ac.is_last = ac.level_lo == 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(c->icp_cluster);
    cfg.blockDim = dim3(kIcpThreads);
    cfg.dynamicSmemBytes = c->icp_smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c->icp_cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    VF_CUDA(c, cudaLaunchKernelEx(&cfg, k_icp_cluster, ac));
    if (ac.is_last) return VF_OK;
  }
  a.level_hi = L - 1 - coarse;
  a.level_lo = 0;
  a.ctl_in = coarse > 0 ? 1 : 0;
  a.is_last = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c->icp_grid);
  cfg.blockDim = dim3(kIcpThreads);
  cfg.dynamicSmemBytes = c->icp_smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  VF_CUDA(c, cudaLaunchKernelEx(&cfg, k_icp, a));
  return VF_OK;
}

void stage_mark(vf_ctx* c, int slot) {
  if (!(c->profiling || c->stage_timing)) return;
  // Under stream capture a plain record only marks a dependency; External
  // makes it a real event-record node of the frame graph (outside a capture
  // the flag is refused, so the plain record is used there).
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->stream, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(c->ev[slot], c->stream, cudaEventRecordExternal);
  else
    cudaEventRecord(c->ev[slot], c->stream);
}

// VF_DEBUG_SYNC=1: synchronise and check after every launch (debugging only).
bool debug_sync() {
  static const bool on = std::getenv("VF_DEBUG_SYNC") != nullptr;
  return on;
}
#define VF_LAUNCHED(ctx, name)                                                                      \
  do {                                                                                              \
    if (debug_sync()) {                                                                             \
      cudaError_t e_ = cudaStreamSynchronize((ctx)->stream);                                        \
      if (e_ == cudaSuccess) e_ = cudaGetLastError();                                               \
      if (e_ != cudaSuccess) {                                                                      \
        std::fprintf(stderr, "[voxfuse_b200] kernel %s failed: %s\n", name, cudaGetErrorString(e_)); \
        (ctx)->err = std::string(name) + ": " + cudaGetErrorString(e_);                             \
        return VF_ERR_CUDA;                                                                         \
      }                                                                                             \
    }                                                                                               \
  } while (0)

// forward_project_points (raycast.hpp:495-509) over the current maps
int launch_forward_project(vf_ctx* c) {
  cudaStream_t st = c->stream;
  VF_CUDA(c, cudaMemsetAsync(c->surf_scan, 0, sizeof(unsigned long long) * (1 + (size_t)c->surf_tiles), st));
  k_forward_project<<<c->surf_tiles, kFpTileItems, 0, st>>>(
      hash_view(c), c->vsize == 8 ? reinterpret_cast<const uint32_t*>(c->voxels) : nullptr, c->points, c->din,
      kSurfaceStride, c->s.voxel_size, c->surf_scan, c->surf_points, c->surf_colors, &c->dstate->ctr);
  VF_CUDA(c, cudaGetLastError());
  return VF_OK;
}

// SDF refinement (ren_refine, ren_tracker.hpp:30-120): max_iterations
// (terms, control) pairs, then the result.  combine_icp: the frame's icp_ren
// tracker (start from the coarse ICP's pose when it succeeded).
int enqueue_ren(vf_ctx* c, cudaStream_t st, bool combine_icp, const PoseD* explicit_init, bool update_state,
                int* launches) {
  const vf_settings& s = c->s;
  VF_CUDA(c, launch_pdl(k_ren_init, dim3(1), dim3(32), 0, st, &c->dstate->icp, &c->dstate->pose, combine_icp ? 1 : 0,
                        explicit_init, &c->dstate->ren));
  for (int it = 0; it < s.max_iterations; ++it) {
    VF_CUDA(c, launch_pdl(k_ren_terms, dim3(c->ren_grid), dim3(256), 0, st, c->depth, c->din, hash_view(c),
                          reinterpret_cast<const uint32_t*>(c->voxels), c->vsize / 4, s.voxel_size,
                          (double)s.ren_sigma, &c->dstate->ren, c->ren_partials));
    VF_CUDA(c, launch_pdl(k_ren_ctl, dim3(1), dim3(32), 0, st, c->ren_partials, c->ren_grid, &c->dstate->ren,
                          s.min_valid_points, s.max_condition, s.convergence_eps));
  }
  VF_CUDA(c, launch_pdl(k_ren_finish, dim3(1), dim3(32), 0, st, &c->dstate->ren, combine_icp ? 1 : 0, &c->dstate->icp,
                        &c->dstate->pose, update_state ? 1 : 0));
  VF_CUDA(c, cudaGetLastError());
  *launches += 2 + 2 * s.max_iterations;
  return VF_OK;
}

// build_color_pyramid (pyramid.hpp:112-132) of c->rgb, then color_track
// (color_tracker.hpp:107-154) of the current surface list.
int enqueue_color(vf_ctx* c, cudaStream_t st, const PoseD* explicit_init, bool update_state, int* launches) {
  const vf_settings& s = c->s;
  const int L = s.hierarchy_levels;
  ColorTrackArgs a{};
  for (int l = 0; l < L; ++l) {
    const IntrD& in = c->rgb_levels[l];
    const int n = in.width * in.height;
    float4* col = c->cpyr + c->cpyr_off[l];
    if (l == 0) {
      VF_CUDA(c, launch_pdl(k_cpyr_base, dim3((n + 255) / 256), dim3(256), 0, st, c->rgb, n, col));
    } else {
      const IntrD& up = c->rgb_levels[l - 1];
      VF_CUDA(c, launch_pdl(k_cpyr_down, dim3((n + 255) / 256), dim3(256), 0, st, c->cpyr + c->cpyr_off[l - 1],
                            up.width, 
                            up.height, col));
    }
    VF_CUDA(c, launch_pdl(k_cpyr_grad, dim3((n + 255) / 256), dim3(256), 0, st, col, in.width, in.height, col + n,
                          col + 2 * (size_t)n));
    a.lv[l] = ColorLevel{col, col + n, col + 2 * (size_t)n, in.width, in.height, in.fx, in.fy, in.cx, in.cy};
  }
  a.levels = L;
  a.stride = s.skip_points ? 2 : 1;
  a.max_iterations = s.max_iterations;
  a.min_valid_points = s.min_valid_points;
  a.convergence_eps = s.convergence_eps;
  a.points = c->surf_points;
  a.colors = c->surf_colors;
  a.count = &c->dstate->ctr.surface_count;
  a.state = &c->dstate->pose;
  a.explicit_init = explicit_init;
  a.result = &c->dstate->icp;
  a.update_state = update_state ? 1 : 0;
  a.partials = c->partials;
  a.exact_solve = s.tracker_exact_solve;
  // one CTA per kColorThreads surface points (up to one per SM), over a
  // cooperative grid: an evaluation is then one point per thread deep
  int g = std::max(1, std::min({c->num_sms, c->icp_grid, (c->surf_cap + kColorThreads - 1) / kColorThreads}));
  if (const char* e = std::getenv("VF_COLOR_GRID")) g = std::max(1, std::min(g, std::atoi(e)));  // tuning override
  if (g == 1) {
    VF_CUDA(c, launch_pdl(k_color_track, dim3(1), dim3(kColorThreads), 0, st, a));
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(kColorThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    VF_CUDA(c, cudaLaunchKernelEx(&cfg, k_color_track, a));
  }
  VF_CUDA(c, cudaGetLastError());
  *launches += 2 * L + 1;
  return VF_OK;
}

// Pipeline::track (pipeline_impl.hpp:180-209) for the configured tracker;
// the result lands in DevState::icp and, when ok and update_state, the pose.
int enqueue_tracker(vf_ctx* c, cudaStream_t st, bool with_rgb, const PoseD* explicit_init, bool update_state,
                    int* launches) {
  const vf_settings& s = c->s;
  if (s.tracker_type == VF_TRACKER_COLOR) {
    if (!with_rgb) {  // no RGB frame: {state.pose, false}
      k_track_fail<<<1, 32, 0, st>>>(&c->dstate->pose, &c->dstate->icp);
      ++*launches;
      return VF_OK;
    }
    return enqueue_color(c, st, explicit_init, update_state, launches);
  }
  if (s.hierarchy_levels > 1) {
    VF_CUDA(c, launch_pdl(k_pyramid, dim3((c->din.width + 31) / 32, (c->din.height + 31) / 32), dim3(256), 0, st,
                          c->depth, c->din.width, c->din.height, s.hierarchy_levels, c->pyr));
    VF_LAUNCHED(c, "k_pyramid");
    ++*launches;
  }
  if (s.tracker_type == VF_TRACKER_ICP_REN) {
    if (s.hierarchy_levels > 1) {
      if (int rc = launch_icp(c, st, false, /*update_state=*/false, /*first_level=*/1, frame_trace())) return rc;
      ++*launches;
    } else {
      k_track_fail<<<1, 32, 0, st>>>(&c->dstate->pose, &c->dstate->icp);
      ++*launches;
    }
    return enqueue_ren(c, st, true, explicit_init, update_state, launches);
  }
  if (int rc = launch_icp(c, st, false, update_state, 0, frame_trace(), /*exchange=*/true)) return rc;
  VF_LAUNCHED(c, "k_icp");
  ++*launches;
  return VF_OK;
}

// render_maps (raycast.hpp:415-435) over the current range image.
int launch_raycast(vf_ctx* c, cudaStream_t st) {
  const vf_settings& s = c->s;
  const uint32_t* vox = reinterpret_cast<const uint32_t*>(c->voxels);
  auto* march = c->npix <= VF_RAY_SMALL_PIXELS ? k_raycast<VF_RAY_MIN_BLOCKS_SMALL> : k_raycast<VF_RAY_MIN_BLOCKS>;
  VF_CUDA(c, launch_pdl(march, dim3(c->frag_w, c->frag_h * 2), dim3(128), 0, st, hash_view(c), vox, c->vsize / 4,
                        c->ranges, &c->dstate->fp, c->din, s.voxel_size, s.mu, c->points, c->normals, c->ray_flags));
  VF_CUDA(c, launch_pdl(k_ray_normals, dim3(c->frag_w, c->frag_h * 2), dim3(128), 0, st, hash_view(c), vox,
                        c->vsize / 4, c->ranges, &c->dstate->fp, c->din, s.voxel_size, s.mu, c->points, c->normals,
                        c->ray_flags, &c->dstate->ctr));
  VF_CUDA(c, cudaGetLastError());
  return VF_OK;
}

// The hash table (34 MiB at the default 2^20 x 2 + 2^17 entries) is the
// object every stage probes (allocation's DDA cells, the raycast's block
// lookups, visibility, the swap scan).  VF_L2_PERSIST=1 puts an
// access-policy window on the context's streams that marks it persisting in
// L2.  Measured (B200, bench.py, L2 flushed between
// frames): C1 0.204 -> 0.199 ms raycast, 0.042 -> 0.040 ms allocation but
// 0.035 -> 0.037 ms integration (+0.5 % frames/s, within run-to-run noise);
// C3's 68 MiB table carves half the L2 away from the voxel stream and the
// fast integration kernel loses 17 %.  Off by default.
void persist_hash_table(vf_ctx* c) {
  static const bool on = [] {
    const char* e = std::getenv("VF_L2_PERSIST");
    return e && std::atoi(e) != 0;
  }();
  if (!on) return;
  int max_persist = 0, max_window = 0;
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c->device);
  cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, c->device);
  if (max_persist <= 0 || max_window <= 0) return;
  const size_t table = sizeof(HashEntry) * (size_t)c->entry_count;
  size_t carve = 0;
  cudaDeviceGetLimit(&carve, cudaLimitPersistingL2CacheSize);
  const size_t want = std::min(table, (size_t)max_persist);
  if (carve < want && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) carve = want;
  if (carve == 0) {
    cudaGetLastError();
    return;
  }
  cudaStreamAttrValue v{};
  v.accessPolicyWindow.base_ptr = c->entries;
  v.accessPolicyWindow.num_bytes = std::min(table, (size_t)max_window);
  v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)carve / (float)v.accessPolicyWindow.num_bytes);
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  for (cudaStream_t st : {c->stream, c->side}) cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
  cudaGetLastError();
  c->l2_persist_bytes = (long)std::min(carve, (size_t)v.accessPolicyWindow.num_bytes);
}

// k_mark's grid: one thread per pixel, 32 x 8 pixel tiles.
int mark_grid(const vf_ctx* c) { return ((c->din.width + 31) / 32) * ((c->din.height + 7) / 8); }

// k_alloc_compact's ticket + per-tile look-back words.
int scan_words(const vf_ctx* c) { return 1 + (c->s.bucket_count / 32 + kCompactThreads - 1) / kCompactThreads; }

// perform_allocations' ordered compaction of the request bitmap (k_alloc_compact).
int launch_alloc_scan(vf_ctx* c, cudaStream_t st) {
  const int n_words = c->s.bucket_count / 32;
  const int tiles = (n_words + kCompactThreads - 1) / kCompactThreads;
  // compact_scan is zero here: cleared at creation and by every k_alloc_apply after its compaction
  VF_CUDA(c, launch_pdl(k_alloc_compact, dim3(tiles), dim3(kCompactThreads), 0, st, c->req_bits, n_words,
                        hash_view(c), c->req_list, c->req_excess_rank, c->compact_scan, &c->dstate->meta,
                        &c->dstate->ctr, c->ranges, c->frag_w * c->frag_h));
  VF_CUDA(c, cudaGetLastError());
  return VF_OK;
}

// Integration CTAs per SM (VF_INT_GRID_MULT overrides, for tuning runs).
int int_grid_mult() {
  static const int m = [] {
    const char* e = std::getenv("VF_INT_GRID_MULT");
    return e ? std::max(1, std::atoi(e)) : 8;
  }();
  return m;
}

// The frame, as stream work.  With track=true the ICP runs first against the
// maps of the previous frame; the updated pose stays on the device.
int enqueue_frame(vf_ctx* c, bool track, bool with_rgb) {
  cudaStream_t st = c->stream;
  const vf_settings& s = c->s;
  int launches = 0;
  stage_mark(c, 0);
  if (track) {
    if (int rc = enqueue_tracker(c, st, with_rgb, nullptr, true, &launches)) return rc;
  }
  stage_mark(c, 1);
  VF_CUDA(c, launch_pdl(k_mark, dim3(mark_grid(c)), dim3(256), 0, st, c->depth, c->din, &c->dstate->pose, c->rgbin,
                        c->depth_to_rgb, &c->dstate->fp, hash_view(c), s.voxel_size, s.mu, c->shard, c->req_key,
                        c->req_bits, &c->dstate->ctr));
  VF_LAUNCHED(c, "k_mark");
  if (int rc = launch_alloc_scan(c, st)) return rc;
  VF_LAUNCHED(c, "k_alloc_compact");
  VF_CUDA(c, launch_pdl(k_alloc_apply, dim3(c->num_sms * 2), dim3(256), 0, st, c->depth, c->din, &c->dstate->fp,
                        s.voxel_size, s.mu, c->entries, c->mask, s.bucket_size, c->ordered, c->req_key, c->req_list,
                        c->req_excess_rank, &c->dstate->meta, c->vba_slots, c->excess_slots, c->alloc_list,
                        c->alloc_cap, &c->dstate->ctr, c->compact_scan, scan_words(c)));
  VF_LAUNCHED(c, "k_alloc_apply");
  VF_CUDA(c, launch_pdl(k_visible, dim3(c->num_sms * 4), dim3(256), 0, st, c->entries, c->alloc_list, &c->dstate->fp,
                        c->din, s.voxel_size, s.near_clip, s.far_clip, s.visibility_margin_px, c->visible_list,
                        &c->dstate->ctr));
  VF_LAUNCHED(c, "k_visible");
  launches += 5;
  stage_mark(c, 2);
  // The side stream (a parallel branch of the frame graph) takes the work
  // that does not touch the blocks being integrated: the range image (it
  // reads only entry positions) and the whole swap engine — swap-out
  // candidates are outside the enlarged frustum and swap-in candidates are
  // swapped out, so neither is on the visible list (visible ⊂ swap-visible,
  // allocation.hpp:226-233); the VBA stack and the voxels they move are
  // disjoint from integration's.  Swap-ins join before the raycast (it may
  // read them); swap-outs join at the end of the frame.
  const bool fork = !c->profiling;
  cudaStream_t branch = fork ? c->side : st;
  auto enqueue_swap = [&](cudaStream_t sst) -> int {
    // request_swap_ins/outs + execute_swap_in/out (pipeline_impl.hpp:104-113)
    VF_CUDA(c, launch_pdl(k_swap_request, dim3(c->num_sms * 4), dim3(256), 0, sst, c->entries, c->alloc_list,
                          &c->dstate->fp, c->din, s.voxel_size, s.near_clip, s.far_clip, s.visibility_margin_px,
                          s.swap_margin_px, c->sw, &c->dstate->ctr));
    VF_LAUNCHED(c, "k_swap_request");
    VF_CUDA(c, launch_pdl(k_swap_select, dim3(1), dim3(1024), 0, sst, c->entries, c->vba_slots, c->sw,
                          s.swap_buffer_blocks, (c->vsize == 8 ? 7 : 3) * kBlockVolume, &c->dstate->ctr));
    VF_LAUNCHED(c, "k_swap_select");
    VF_CUDA(c, launch_pdl(k_swap_transfer, dim3(c->num_sms * 2), dim3(256), 0, sst,
                          reinterpret_cast<uint32_t*>(c->voxels), c->vsize / 4, c->sw, s.max_weight, 0));
    VF_LAUNCHED(c, "k_swap_transfer");
    launches += 3;
    return VF_OK;
  };
  if (fork) {
    VF_CUDA(c, cudaEventRecord(c->ev_fork, st));
    VF_CUDA(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    VF_CUDA(c, launch_pdl(k_ranges, dim3(c->num_sms * 2), dim3(256), 0, c->side, c->entries, c->visible_list,
                          &c->dstate->ctr, &c->dstate->fp, c->din, s.voxel_size, s.near_clip, s.far_clip, c->ranges,
                          c->frag_w));
    if (c->swapping)
      if (int rc = enqueue_swap(c->side)) return rc;
    VF_CUDA(c, cudaEventRecord(c->ev_join, c->side));
  }
  const bool color = c->vsize == 8;
  launch_integrate(c->num_sms * int_grid_mult(), st, color, s.integration_mode == VF_INTEGRATION_FAST, c->entries, c->visible_list, &c->dstate->ctr, c->voxels, c->depth,
                   with_rgb ? c->rgb : nullptr, &c->dstate->fp, s.voxel_size, s.mu, s.max_weight,
                   s.stop_integrating_at_max);
  VF_LAUNCHED(c, "k_integrate");
  ++launches;
  stage_mark(c, 3);
  if (fork) {
    VF_CUDA(c, cudaStreamWaitEvent(st, c->ev_join, 0));
  } else if (c->swapping) {
    if (int rc = enqueue_swap(st)) return rc;
  }
  if (c->swapping) {
    // swap-outs: after the selection, beside the raycast
    VF_CUDA(c, launch_pdl(k_swap_transfer, dim3(c->num_sms * 2), dim3(256), 0, branch,
                          reinterpret_cast<uint32_t*>(c->voxels), c->vsize / 4, c->sw, s.max_weight, 1));
    VF_LAUNCHED(c, "k_swap_transfer");
    if (fork) VF_CUDA(c, cudaEventRecord(c->ev_join2, c->side));
    ++launches;
  }
  stage_mark(c, 4);
  if (!fork) {
    VF_CUDA(c, launch_pdl(k_ranges, dim3(c->num_sms * 2), dim3(256), 0, st, c->entries, c->visible_list,
                          &c->dstate->ctr, &c->dstate->fp, c->din, s.voxel_size, s.near_clip, s.far_clip, c->ranges,
                          c->frag_w));
  }
  VF_LAUNCHED(c, "k_ranges");
  if (c->p2p_linked > 1) {  // the previous frame's maps and keys are no longer read by any shard
    k_p2p_wait_done<<<1, 32, 0, st>>>(c->p2p);
    ++launches;
  }
  if (int rc = launch_raycast(c, st)) return rc;
  VF_LAUNCHED(c, "k_raycast");
  launches += 3;  // k_ranges, k_raycast, k_ray_normals
  if (c->p2p_linked > 1) {  // nearest-depth composite over peer memory (vf_shard.cu)
    const int blocks = (c->npix + 255) / 256;
    k_shard_keys<<<blocks, 256, 0, st>>>(c->points, &c->dstate->fp, c->npix, c->shard.index, c->shard_keys);
    k_p2p_signal_ready<<<1, 32, 0, st>>>(c->p2p);
    k_p2p_wait_ready<<<1, 32, 0, st>>>(c->p2p);
    k_p2p_composite<<<c->num_sms * 4, 256, 0, st>>>(c->p2p, c->points, c->normals, c->npix);
    k_p2p_signal_done<<<1, 32, 0, st>>>(c->p2p);
    VF_LAUNCHED(c, "k_p2p_composite");
    launches += 5;
  } else if (c->nccl_comm) {  // nearest-depth composite across the GPUs (vf_shard.cu)
    if (nccl_composite(c->nccl_comm, st, &c->dstate->fp, c->points, c->normals, c->shard_keys, c->npix,
                       c->shard.index) != 0) {
      c->err = "NCCL composite failed";
      return VF_ERR_CUDA;
    }
    launches += 2;
  }
  if (c->vsize == 8) {
    // forward_project_points for the colour tracker (pipeline_impl.hpp:218-221)
    if (int rc = launch_forward_project(c)) return rc;
    VF_LAUNCHED(c, "k_forward_project");
    ++launches;
  }
  if (c->swapping && fork) VF_CUDA(c, cudaStreamWaitEvent(st, c->ev_join2, 0));
  stage_mark(c, 5);
  c->launches_last = launches;
  VF_CUDA(c, cudaGetLastError());
  return VF_OK;
}

int run_frame(vf_ctx* c, bool track, bool with_rgb) {
  if (c->s.use_graphs && c->graphs_ok && !c->profiling && !debug_sync()) {
    cudaGraphExec_t& g = c->graph[track][with_rgb][c->stage_timing];
    if (!g) {
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
      int rc = VF_OK;
      if (e == cudaSuccess) {
        rc = enqueue_frame(c, track, with_rgb);
        e = cudaStreamEndCapture(c->stream, &graph);
      }
      if (e == cudaSuccess && rc == VF_OK) e = cudaGraphInstantiate(&g, graph, 0);
      if (graph) cudaGraphDestroy(graph);
      if (e != cudaSuccess || rc != VF_OK) {
        // Capture of the cooperative launch is unsupported on this driver:
        // keep running the identical kernels without the graph.
        cudaGetLastError();
        g = nullptr;
        c->graphs_ok = false;
        std::fprintf(stderr, "[voxfuse_b200] CUDA graph capture unavailable (%s); launching kernels directly\n",
                     cudaGetErrorString(e));
        return enqueue_frame(c, track, with_rgb);
      }
    }
    VF_CUDA(c, cudaGraphLaunch(g, c->stream));
    return VF_OK;
  }
  return enqueue_frame(c, track, with_rgb);
}

int read_state(vf_ctx* c) {
  VF_CUDA(c, cudaMemcpyAsync(c->hstate, c->dstate, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  return VF_OK;
}

void fill_stats(vf_ctx* c, bool tracked, int frame_index, vf_frame_stats* st, const DevState* hs = nullptr) {
  const DevState& h = hs ? *hs : *c->hstate;
  std::memset(st, 0, sizeof(*st));
  st->frame = frame_index;
  st->tracking_ok = tracked ? h.icp.ok : 1;
  st->tracking_iterations = tracked ? h.icp.iterations : 0;
  st->tracking_cost = tracked ? h.icp.final_cost : 0.0;
  st->tracking_valid_points = tracked ? h.icp.valid_points : 0;
  st->allocation_requested = h.ctr.requested;
  st->blocks_allocated = h.ctr.allocated;
  st->allocation_dropped = h.ctr.dropped_vba_full + h.ctr.dropped_excess_full;
  st->visible_blocks = h.ctr.visible_count;
  st->allocated_total = c->s.block_count - h.ctr.vba_top;
  st->error_flags = h.ctr.error_flags;
  st->swapped_in = h.swap.swapped_in;
  st->swapped_out = h.swap.swapped_out;
  st->swap_bytes_in = h.swap.bytes_in;
  st->swap_bytes_out = h.swap.bytes_out;
  pose_to(h.pose, st->pose);
}

int upload(vf_ctx* c, void* dst, const void* src, size_t n, bool src_device) {
  VF_CUDA(c, cudaMemcpyAsync(dst, src, n, src_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
  return VF_OK;
}

int ensure_host_store(vf_ctx* c);

int frame_common(vf_ctx* c, const float* depth, const uint8_t* rgb, bool device_inputs, vf_frame_stats* stats,
                 const uint16_t* disparity = nullptr, bool big_endian = false) {
  if (!c || (!depth && !disparity)) return VF_ERR_INVALID;
  if (disparity) {
    // process_raw_frame (pipeline_impl.hpp:59-62): 2 bytes per pixel cross the
    // link, the conversion runs on the device
    if (int rc = upload(c, c->disp, disparity, sizeof(uint16_t) * (size_t)c->npix, device_inputs)) return rc;
    k_disparity_to_depth<<<(c->npix + 255) / 256, 256, 0, c->stream>>>(
        c->disp, c->npix, big_endian ? 1 : 0, (float)c->calib.disparity_a, (float)c->calib.disparity_b,
        (float)c->calib.depth.fx, c->s.max_depth, c->depth);
    VF_CUDA(c, cudaGetLastError());
  } else if (int rc = upload(c, c->depth, depth, sizeof(float) * (size_t)c->npix, device_inputs)) {
    return rc;
  }
  const bool with_rgb = rgb != nullptr && c->vsize == 8;
  if (with_rgb) {
    if (int rc = upload(c, c->rgb, rgb, 3 * (size_t)c->rgbin.width * c->rgbin.height, device_inputs)) return rc;
  }
  c->rgb_valid = with_rgb;
  const bool track = c->s.tracking && c->frame > 0 && c->maps_valid;
  const int frame_index = c->frame;
  if (int rc = ensure_host_store(c)) return rc;
  if (stats) VF_CUDA(c, cudaEventRecord(c->ev_frame0, c->stream));
  if (int rc = run_frame(c, track, with_rgb)) return rc;
  c->host_top_lb -= c->s.swap_buffer_blocks;  // worst case: B swap-outs, no swap-ins
  c->maps_valid = true;
  ++c->frame;
  if (c->profiling) {
    VF_CUDA(c, cudaStreamSynchronize(c->stream));
    for (int i = 0; i < 5; ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]);
      c->stage_ms[i] += ms;
    }
    ++c->profiled_frames;
  }
  if (stats) {
    VF_CUDA(c, cudaEventRecord(c->ev_frame1, c->stream));
    if (int rc = read_state(c)) return rc;
    c->host_top_lb = c->hstate->swap.host_top;
    fill_stats(c, track, frame_index, stats);
    float ms = 0;
    cudaEventElapsedTime(&ms, c->ev_frame0, c->ev_frame1);
    stats->ms_total = ms;
    if (c->stage_timing || c->profiling) {
      // FrameStats::ms_tracking .. ms_raycast (pipeline.hpp:56-57) from the
      // stage marks of this frame: tracking, allocation, integration, the
      // wait for the side branch (range image + swap engine), raycast
      double* out[5] = {&stats->ms_tracking, &stats->ms_allocation, &stats->ms_integration, &stats->ms_swapping,
                        &stats->ms_raycast};
      for (int i = 0; i < 5; ++i) {
        float m = 0;
        if (cudaEventElapsedTime(&m, c->ev[i], c->ev[i + 1]) == cudaSuccess) *out[i] = m;
      }
    }
    if (c->hstate->ctr.error_flags) return VF_ERR_OVERFLOW;
  }
  return VF_OK;
}

// Lazily created on the first vf_submit_frame: staging slots, the copy
// stream and the per-slot events.
int ensure_queue(vf_ctx* c) {
  if (c->copy) return VF_OK;
  // Every resource is created only if still missing, and the copy stream --
  // the "queue is ready" flag -- last: a failure part way leaves c->copy null,
  // so the next submit retries the missing pieces instead of running with
  // null staging buffers or events.
  for (int k = 0; k < kMaxFramesInFlight; ++k) {
    if (!c->depth_stage[k])
      VF_CUDA(c, cudaMalloc(reinterpret_cast<void**>(&c->depth_stage[k]), sizeof(float) * (size_t)c->npix));
    if (c->vsize == 8 && !c->rgb_stage[k])
      VF_CUDA(c, cudaMalloc(reinterpret_cast<void**>(&c->rgb_stage[k]), 3 * (size_t)c->rgbin.width * c->rgbin.height));
    if (!c->hstate_q[k]) VF_CUDA(c, cudaMallocHost(reinterpret_cast<void**>(&c->hstate_q[k]), sizeof(DevState)));
    for (cudaEvent_t* e : {&c->ev_up[k], &c->ev_consumed[k], &c->ev_done[k]})
      if (!*e) VF_CUDA(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    if (!c->ev_q0[k]) VF_CUDA(c, cudaEventCreate(&c->ev_q0[k]));
    if (!c->ev_q1[k]) VF_CUDA(c, cudaEventCreate(&c->ev_q1[k]));
  }
  cudaStream_t copy = nullptr;
  VF_CUDA(c, cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
  c->copy = copy;
  return VF_OK;
}

// vf_submit_frame: enqueue one frame and return.  Copy stream: wait until the
// slot's previous contents were consumed, H2D into the slot.  Main stream:
// wait for the upload, D2D into the frame buffers, the frame's graph, D2H of
// the frame's DevState into the slot's pinned copy.
int submit_frame(vf_ctx* c, const float* depth, const uint8_t* rgb, const uint16_t* disparity = nullptr,
                 bool big_endian = false) {
  if (c->q_count >= kMaxFramesInFlight) {
    c->err = "vf_submit_frame: collect the oldest frame first";
    return VF_ERR_STATE;
  }
  if (c->profiling) {
    c->err = "vf_submit_frame: stage profiling needs vf_process_frame";
    return VF_ERR_STATE;
  }
  if (int rc = ensure_queue(c)) return rc;
  if (int rc = ensure_host_store(c)) return rc;
  const int k = (c->q_head + c->q_count) % kMaxFramesInFlight;
  const bool with_rgb = rgb != nullptr && c->vsize == 8;
  const size_t dbytes = sizeof(float) * (size_t)c->npix, cbytes = 3 * (size_t)c->rgbin.width * c->rgbin.height;
  VF_CUDA(c, cudaStreamWaitEvent(c->copy, c->ev_consumed[k], 0));
  // a raw disparity frame (2 bytes per pixel) shares the slot and is decoded
  // straight from it into the frame's depth buffer
  if (disparity)
    VF_CUDA(c, cudaMemcpyAsync(c->depth_stage[k], disparity, sizeof(uint16_t) * (size_t)c->npix,
                               cudaMemcpyHostToDevice, c->copy));
  else
    VF_CUDA(c, cudaMemcpyAsync(c->depth_stage[k], depth, dbytes, cudaMemcpyHostToDevice, c->copy));
  if (with_rgb) VF_CUDA(c, cudaMemcpyAsync(c->rgb_stage[k], rgb, cbytes, cudaMemcpyHostToDevice, c->copy));
  VF_CUDA(c, cudaEventRecord(c->ev_up[k], c->copy));
  VF_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_up[k], 0));
  if (disparity) {
    k_disparity_to_depth<<<(c->npix + 255) / 256, 256, 0, c->stream>>>(
        reinterpret_cast<const uint16_t*>(c->depth_stage[k]), c->npix, big_endian ? 1 : 0,
        (float)c->calib.disparity_a, (float)c->calib.disparity_b, (float)c->calib.depth.fx, c->s.max_depth, c->depth);
    VF_CUDA(c, cudaGetLastError());
  } else {
    VF_CUDA(c, cudaMemcpyAsync(c->depth, c->depth_stage[k], dbytes, cudaMemcpyDeviceToDevice, c->stream));
  }
  if (with_rgb) VF_CUDA(c, cudaMemcpyAsync(c->rgb, c->rgb_stage[k], cbytes, cudaMemcpyDeviceToDevice, c->stream));
  VF_CUDA(c, cudaEventRecord(c->ev_consumed[k], c->stream));
  c->rgb_valid = with_rgb;
  const bool track = c->s.tracking && c->frame > 0 && c->maps_valid;
  c->q_frame[k] = c->frame;
  c->q_track[k] = track;
  VF_CUDA(c, cudaEventRecord(c->ev_q0[k], c->stream));
  if (int rc = run_frame(c, track, with_rgb)) return rc;
  c->host_top_lb -= c->s.swap_buffer_blocks;
  c->maps_valid = true;
  ++c->frame;
  VF_CUDA(c, cudaEventRecord(c->ev_q1[k], c->stream));
  VF_CUDA(c, cudaMemcpyAsync(c->hstate_q[k], c->dstate, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
  VF_CUDA(c, cudaEventRecord(c->ev_done[k], c->stream));
  ++c->q_count;
  return VF_OK;
}

int collect_frame(vf_ctx* c, vf_frame_stats* stats) {
  if (c->q_count == 0) {
    c->err = "vf_collect_frame: no frame in flight";
    return VF_ERR_STATE;
  }
  const int k = c->q_head;
  VF_CUDA(c, cudaEventSynchronize(c->ev_done[k]));
  c->q_head = (k + 1) % kMaxFramesInFlight;
  --c->q_count;
  const DevState* h = c->hstate_q[k];
  if (stats) {
    fill_stats(c, c->q_track[k], c->q_frame[k], stats, h);
    float ms = 0;
    cudaEventElapsedTime(&ms, c->ev_q0[k], c->ev_q1[k]);
    stats->ms_total = ms;
  }
  return h->ctr.error_flags ? VF_ERR_OVERFLOW : VF_OK;
}

template <typename T>
int dalloc(vf_ctx* c, T** p, size_t bytes) {
  VF_CUDA(c, cudaMalloc(reinterpret_cast<void**>(p), bytes));
  return VF_OK;
}
int dzero(vf_ctx* c, void* p, size_t bytes) {
  VF_CUDA(c, cudaMemset(p, 0, bytes));
  return VF_OK;
}

void free_all(vf_ctx* c) {
  if (c->nccl_comm) nccl_comm_destroy(c->nccl_comm);
  for (auto& plane : c->graph)
    for (auto& row : plane)
      for (auto& g : row)
        if (g) cudaGraphExecDestroy(g);
  void* ptrs[] = {c->entries, c->voxels, c->vba_slots, c->excess_slots, c->req_key, c->req_bits, c->req_list,
                  c->req_excess_rank, c->alloc_list, c->visible_list, c->dstate, c->depth, c->rgb, c->pyr,
                  c->ranges, c->ray_flags, c->points, c->normals, c->partials, c->utab, c->trace, c->flush_buf,
                  c->shard_keys, c->icp_ctl,
                  c->surf_points, c->surf_colors, c->surf_scan, c->image, c->image_dmax,
                  c->sw.state, c->sw.host_slot, c->sw.host_free, c->sw.in_cand, c->sw.out_cand,
                  c->sw.stage_entry, c->sw.stage_slot, c->sw.stage_host, c->disp, c->image_depth_scratch,
                  c->ren_partials, c->cpyr, c->compact_scan, c->sw.host_chunks, c->sw.journal};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->hstate) cudaFreeHost(c->hstate);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  c->ipc_opened.clear();
  if (c->icp_xchg) cudaFree(c->icp_xchg);
  if (c->p2p_flags) cudaFree(c->p2p_flags);
  for (uint32_t* h : c->host_chunk_ptrs) cudaFreeHost(h);
  c->host_chunk_ptrs.clear();
  if (c->hpose) cudaFreeHost(c->hpose);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->ev_frame0) cudaEventDestroy(c->ev_frame0);
  if (c->ev_frame1) cudaEventDestroy(c->ev_frame1);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->ev_join2) cudaEventDestroy(c->ev_join2);
  for (int k = 0; k < kMaxFramesInFlight; ++k) {
    if (c->depth_stage[k]) cudaFree(c->depth_stage[k]);
    if (c->rgb_stage[k]) cudaFree(c->rgb_stage[k]);
    if (c->hstate_q[k]) cudaFreeHost(c->hstate_q[k]);
    for (cudaEvent_t e : {c->ev_up[k], c->ev_consumed[k], c->ev_done[k], c->ev_q0[k], c->ev_q1[k]})
      if (e) cudaEventDestroy(e);
  }
  for (auto& e : c->flush_ev) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  if (c->copy) cudaStreamDestroy(c->copy);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->stream) cudaStreamDestroy(c->stream);
}

int reset_swap(vf_ctx* c);

int reset_volume(vf_ctx* c) {
  // HashVolume(HashConfig) (hash_volume.hpp:133-140): all entries unallocated,
  // default voxels, iota free stacks.
  std::vector<HashEntry> he((size_t)c->entry_count);
  for (auto& e : he) {
    e.x = e.y = e.z = e.pad = 0;
    e.offset = 0;
    e.block_state = kEntryUnallocated;
  }
  VF_CUDA(c, cudaMemcpy(c->entries, he.data(), sizeof(HashEntry) * he.size(), cudaMemcpyHostToDevice));
  const size_t nvox = (size_t)c->s.block_count * kBlockVolume;
  k_fill_voxels<<<c->num_sms * 8, 256, 0, c->stream>>>(reinterpret_cast<uint32_t*>(c->voxels), nvox, c->vsize / 4);
  std::vector<int> iota((size_t)std::max(c->s.block_count, c->s.excess_count));
  for (size_t i = 0; i < iota.size(); ++i) iota[i] = (int)i;
  VF_CUDA(c, cudaMemcpy(c->vba_slots, iota.data(), sizeof(int) * c->s.block_count, cudaMemcpyHostToDevice));
  VF_CUDA(c, cudaMemcpy(c->excess_slots, iota.data(), sizeof(int) * c->s.excess_count, cudaMemcpyHostToDevice));
  VF_CUDA(c, cudaMemset(c->req_key, 0, sizeof(unsigned long long) * c->s.bucket_count));
  VF_CUDA(c, cudaMemset(c->req_bits, 0, sizeof(uint32_t) * (c->s.bucket_count / 32)));
  DevState ds;
  std::memset(&ds, 0, sizeof(ds));
  ds.ctr.vba_top = c->s.block_count;
  ds.ctr.excess_top = c->s.excess_count;
  for (int i = 0; i < 9; ++i) ds.pose.r[i] = (i % 4 == 0) ? 1.0 : 0.0;  // tracking_state.hpp:27: identity
  VF_CUDA(c, cudaMemcpy(c->dstate, &ds, sizeof(ds), cudaMemcpyHostToDevice));
  VF_CUDA(c, cudaMemset(c->points, 0, sizeof(float4) * c->npix));
  VF_CUDA(c, cudaMemset(c->normals, 0, sizeof(float4) * c->npix));
  if (int rc = reset_swap(c)) return rc;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  VF_CUDA(c, cudaGetLastError());
  if (c->copy) VF_CUDA(c, cudaStreamSynchronize(c->copy));
  c->q_head = c->q_count = 0;
  c->frame = 0;
  c->maps_valid = false;
  return VF_OK;
}

// One more pinned chunk of the host store (its slots are pushed by
// k_host_store_grow when the free stack is (re)built).
int add_host_chunk(vf_ctx* c) {
  if (c->host_cap + kHostChunk > c->host_max) return VF_ERR_OVERFLOW;
  const size_t bytes = (size_t)kHostChunk * kBlockVolume * (size_t)c->vsize;
  void* hp = nullptr;
  void* dp = nullptr;
  if (cudaHostAlloc(&hp, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
      cudaHostGetDevicePointer(&dp, hp, 0) != cudaSuccess) {
    if (hp) cudaFreeHost(hp);
    cudaGetLastError();
    std::fprintf(stderr, "[voxfuse_b200] cannot allocate a %zu-byte pinned host-store chunk\n", bytes);
    c->err = "pinned host-store chunk allocation failed";
    return VF_ERR_CUDA;
  }
  c->host_chunk_ptrs.push_back(reinterpret_cast<uint32_t*>(hp));
  c->host_dev_ptrs.push_back(reinterpret_cast<uint32_t*>(dp));
  c->host_cap += kHostChunk;
  return VF_OK;
}

// Grow the store by one chunk between frames: allocate, then push its slots
// on the device free stack (stream-ordered before the next frame).
int grow_host_store(vf_ctx* c) {
  if (int rc = add_host_chunk(c)) return rc;
  const int k = (int)c->host_chunk_ptrs.size() - 1;
  k_host_store_grow<<<1, 256, 0, c->stream>>>(c->sw, k, c->host_dev_ptrs[(size_t)k]);
  VF_CUDA(c, cudaGetLastError());
  c->host_top_lb += kHostChunk;
  return VF_OK;
}

// Before a frame is enqueued: a frame swaps out at most B blocks, so while
// the lower bound on free host slots covers two frames nothing is needed;
// otherwise read the device's count (waits for the frames in flight) and
// grow until it does, up to one slot per hash entry.
int ensure_host_store(vf_ctx* c) {
  if (!c->swapping) return VF_OK;
  const long need = 2L * c->s.swap_buffer_blocks;
  if (c->host_top_lb >= need || c->host_cap >= c->host_max) return VF_OK;
  if (int rc = read_state(c)) return rc;
  c->host_top_lb = c->hstate->swap.host_top;
  while (c->host_top_lb < need && c->host_cap < c->host_max)
    if (int rc = grow_host_store(c)) return rc;
  return VF_OK;
}

// Empty host store, every entry inactive (GlobalCache constructor, swap.hpp:48-52).
int reset_swap(vf_ctx* c) {
  if (!c->swapping) return VF_OK;
  VF_CUDA(c, cudaMemset(c->sw.state, 0, (size_t)c->entry_count));
  VF_CUDA(c, cudaMemset(c->sw.host_slot, 0xFF, sizeof(int) * (size_t)c->entry_count));
  SwapCounters sc;
  std::memset(&sc, 0, sizeof(sc));
  VF_CUDA(c, cudaMemcpy(&c->dstate->swap, &sc, sizeof(sc), cudaMemcpyHostToDevice));
  // every chunk's slots on the free stack, chunk 0 on top: pops hand out 0, 1, 2, ...
  for (int k = (int)c->host_dev_ptrs.size() - 1; k >= 0; --k)
    k_host_store_grow<<<1, 256, 0, c->stream>>>(c->sw, k, c->host_dev_ptrs[(size_t)k]);
  VF_CUDA(c, cudaGetLastError());
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  c->host_top_lb = c->host_cap;
  c->journal_read = 0;
  return VF_OK;
}

// Host address of a host-store slot (the VXBS save / load / read paths).
uint32_t* host_slot_ptr(const vf_ctx* c, int slot) {
  return c->host_chunk_ptrs[(size_t)(slot >> kHostChunkShift)] +
         (size_t)(slot & (kHostChunk - 1)) * kBlockVolume * (size_t)(c->vsize / 4);
}

int set_pose_dev(vf_ctx* c, const double* pose) {
  k_set_pose<<<1, 32, 0, c->stream>>>(&c->dstate->pose, pose_from(pose));
  VF_CUDA(c, cudaGetLastError());
  return VF_OK;
}

}  // namespace

extern "C" {

int vf_abi_version(void) { return VF_ABI_VERSION; }

long vf_struct_size(int which) {
  switch (which) {
    case 0: return (long)sizeof(vf_settings);
    case 1: return (long)sizeof(vf_calib);
    case 2: return (long)sizeof(vf_frame_stats);
    case 3: return (long)sizeof(vf_alloc_stats);
    case 4: return (long)sizeof(vf_intrinsics);
    default: return -1;
  }
}

void vf_default_settings(vf_settings* s) {
  std::memset(s, 0, sizeof(*s));
  s->voxel_type = VF_VOXEL_S;
  s->voxel_size = 0.004f;  // scene_params.hpp:7
  s->mu = 0.02f;
  s->max_weight = 100;
  s->stop_integrating_at_max = 0;
  s->bucket_count = 1 << 20;  // hash_volume.hpp:50-53
  s->bucket_size = 2;
  s->excess_count = 1 << 17;
  s->block_count = 1 << 18;
  s->near_clip = 0.1f;  // pipeline.hpp:32-35
  s->far_clip = 8.0f;
  s->visibility_margin_px = 8;
  s->swap_margin_px = 48;
  s->hierarchy_levels = 5;  // tracking_state.hpp:14-22
  s->rotation_only_levels = 2;
  s->max_iterations = 20;
  s->min_valid_points = 30;
  s->icp_dist_threshold = 0.1f;
  s->convergence_eps = 1e-5f;
  s->max_condition = 1e8;
  s->tracking = 1;
  s->use_graphs = 1;
  s->shard_count = 1;
  s->shard_index = 0;
  s->shard_shift = 3;
  s->shard_halo = 1;
  s->use_swapping = 0;  // pipeline.hpp:20-23
  s->swap_buffer_blocks = 100;
  s->swap_host_blocks = 0;
  s->max_depth = 8.0f;  // pipeline.hpp:37 (disparity conversion clamp)
  s->tracker_type = VF_TRACKER_ICP;  // tracking_state.hpp:12-22
  s->ren_sigma = 10.0f;
  s->skip_points = 0;
}

int vf_create(const vf_settings* s, const vf_calib* calib, int device, vf_ctx** out) {
  if (!s || !calib || !out) return VF_ERR_INVALID;
  *out = nullptr;
  if (s->bucket_count < 32 || (s->bucket_count & (s->bucket_count - 1)) != 0 || s->bucket_size < 1 ||
      s->block_count < 1 || s->excess_count < 1 || (s->voxel_type != VF_VOXEL_S && s->voxel_type != VF_VOXEL_S_RGB) ||
      s->hierarchy_levels < 1 || s->hierarchy_levels > kMaxLevels || calib->depth.width < 2 ||
      calib->depth.height < 2 || !(s->voxel_size > 0) || !(s->mu > 0))
    return VF_ERR_INVALID;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device) {
    cudaGetLastError();
    std::fprintf(stderr, "[voxfuse_b200] no CUDA device: the B200 path has no CPU fallback\n");
    return VF_ERR_NO_DEVICE;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major < 10) {
    std::fprintf(stderr, "[voxfuse_b200] device %d is not sm_100-class\n", device);
    return VF_ERR_NO_DEVICE;
  }
  vf_ctx* c = new vf_ctx();
  c->s = *s;
  c->calib = *calib;
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join2, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return VF_ERR_CUDA;
  }
  c->vsize = s->voxel_type == VF_VOXEL_S_RGB ? 8 : 4;
  if (s->integration_mode < VF_INTEGRATION_EXACT || s->integration_mode > VF_INTEGRATION_FAST ||
      s->tracker_type < VF_TRACKER_ICP || s->tracker_type > VF_TRACKER_ICP_REN ||
      (s->tracker_type == VF_TRACKER_COLOR && c->vsize != 8)) {
    // "colour tracker requires a voxel type with colour information" (pipeline_impl.hpp:55-57)
    free_all(c);
    delete c;
    return VF_ERR_INVALID;
  }
  if (s->use_swapping) {
    const long entries = (long)s->bucket_count * s->bucket_size + s->excess_count;
    if (s->swap_buffer_blocks < 1 || s->swap_buffer_blocks > kSwapSortCap || s->swap_host_blocks < 0 ||
        entries >= (1L << 24)) {
      free_all(c);
      delete c;
      return VF_ERR_INVALID;
    }
    c->swapping = true;
    // one host slot per hash entry, as the reference's GlobalCache (swap.hpp:42-56),
    // allocated in pinned chunks as the walk needs them; swap_host_blocks > 0 caps it
    const long want = s->swap_host_blocks > 0 ? s->swap_host_blocks : entries;
    c->host_max = (int)((want + kHostChunk - 1) / kHostChunk * kHostChunk);
  }
  if (s->shard_count > 1) {
    if (s->shard_count > kMaxShards || s->shard_index < 0 || s->shard_index >= s->shard_count || s->shard_shift < 0 ||
        s->shard_shift > 8 ||
        // Only ICP is shard-safe: it reads the composited maps, identical on
        // every rank.  The Ren and colour trackers read the shard's own voxels,
        // so each rank would compute a different pose (vf_shard.cu header).
        s->tracker_type != VF_TRACKER_ICP) {
      free_all(c);
      delete c;
      return VF_ERR_INVALID;
    }
    c->shard = ShardSpec{s->shard_count, s->shard_index, s->shard_shift, s->shard_halo};
  }
  c->ordered = s->bucket_count * s->bucket_size;
  c->entry_count = c->ordered + s->excess_count;
  c->mask = (uint32_t)(s->bucket_count - 1);
  c->din = intr_of(calib->depth);
  c->rgbin = intr_of(calib->rgb);
  if (c->rgbin.width <= 0) c->rgbin = c->din;
  {
    PoseD r2d = pose_from(calib->rgb_to_depth);
    c->depth_to_rgb = pose_inverse(r2d);  // Pose::inverse (pose.hpp:30-33)
  }
  c->npix = c->din.width * c->din.height;
  c->frag_w = (c->din.width + kFragmentSize - 1) / kFragmentSize;
  c->frag_h = (c->din.height + kFragmentSize - 1) / kFragmentSize;
  c->levels.push_back(c->din);
  c->pyr_floats = 0;
  for (int l = 1; l < s->hierarchy_levels; ++l) {
    c->levels.push_back(intr_half(c->levels.back()));
    c->pyr_floats += (size_t)c->levels.back().width * c->levels.back().height;
  }
  std::vector<double> utab_h;
  for (const IntrD& in : c->levels) {
    // unproject's (px - cx) / fx and (py - cy) / fy (intrinsics.hpp:39-43), IEEE double
    c->utab_off.push_back(utab_h.size());
    for (int x = 0; x < in.width; ++x) utab_h.push_back((x - in.cx) / in.fx);
    for (int y = 0; y < in.height; ++y) utab_h.push_back((y - in.cy) / in.fy);
  }
  c->alloc_cap = c->entry_count;
  c->ren_grid = c->num_sms * 4;
  c->rgb_levels.push_back(c->rgbin);
  for (int l = 1; l < s->hierarchy_levels; ++l) c->rgb_levels.push_back(intr_half(c->rgb_levels.back()));
  size_t cpyr_n = 0;
  for (const IntrD& in : c->rgb_levels) {
    c->cpyr_off.push_back(cpyr_n);
    cpyr_n += 3 * (size_t)in.width * in.height;
  }
  c->surf_cap = ((c->din.width + kSurfaceStride - 1) / kSurfaceStride) *
                ((c->din.height + kSurfaceStride - 1) / kSurfaceStride);
  c->surf_tiles = (c->surf_cap + kFpTileItems - 1) / kFpTileItems;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_icp, kIcpThreads, 0);
  if (occ < 1) occ = 1;
  c->icp_grid = std::min(c->num_sms * std::min(occ, 2), kMaxIcpGrid);
  // several sharded ICP loops on one device must be co-resident (each waits
  // for the others' sums): vf_settings.icp_max_ctas caps the grid
  if (s->icp_max_ctas > 0) c->icp_grid = std::min(c->icp_grid, s->icp_max_ctas);
  {
    // stage up to the whole level-0 share of each thread in shared memory,
    // within what the SM leaves each of its resident ICP CTAs
    const long threads = (long)c->icp_grid * kIcpThreads;
    const long need = (c->npix + threads - 1) / threads;
    const size_t tables = sizeof(double) * (size_t)(c->din.width + c->din.height);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_icp);
    int sm_smem = 0;
    cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, c->device);
    const long per_cta = std::min<long>(sm_smem / std::max(1, c->icp_grid / c->num_sms) - 1024, 200 * 1024) -
                         (long)fa.sharedSizeBytes;
    // the pipelined pixel pass's tap buffers: 2 stages x kInflight pixels x 8 taps
    const size_t taps = (size_t)2 * kInflight * 8 * kIcpThreads * sizeof(float4) + 16;
    const long cap = std::max(1L, (long)((per_cta - (long)tables - (long)taps) / (8 * kIcpThreads)));
    c->icp_slots = (int)std::max(1L, std::min(need, cap));
    c->icp_smem = tables + (size_t)c->icp_slots * kIcpThreads * 8 + taps;
    cudaFuncSetAttribute(k_icp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->icp_smem);
    cudaFuncSetAttribute(k_icp_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->icp_smem);
    // Coarse levels (<= kClusterPixels pixels) go to one cluster of 16 CTAs
    // (non-portable size) or 8 if the device cannot co-schedule 16.
    // (VF_ICP_CLUSTER_PIXELS / VF_ICP_CLUSTER_SIZE: tuning overrides)
    const int kClusterPixels = std::getenv("VF_ICP_CLUSTER_PIXELS") ? std::atoi(std::getenv("VF_ICP_CLUSTER_PIXELS")) : 8192;
    const int cs_want = std::getenv("VF_ICP_CLUSTER_SIZE") ? std::atoi(std::getenv("VF_ICP_CLUSTER_SIZE")) : 16;
    cudaFuncSetAttribute(k_icp_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {cs_want, 8}) {
      cudaLaunchConfig_t q{};
      q.gridDim = dim3(cs);
      q.blockDim = dim3(kIcpThreads);
      q.dynamicSmemBytes = c->icp_smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      q.attrs = at;
      q.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, k_icp_cluster, &q) == cudaSuccess && nclusters > 0) {
        c->icp_cluster = cs;
        break;
      }
      cudaGetLastError();
    }
    for (int l = (int)c->levels.size() - 1; l >= 0; --l) {
      if ((long)c->levels[l].width * c->levels[l].height > kClusterPixels) break;
      ++c->icp_coarse_levels;
    }
    if (std::getenv("VF_ICP_NO_CLUSTER")) c->icp_cluster = 0;
  }
  int rc = VF_OK;
  const size_t nvox = (size_t)s->block_count * kBlockVolume;
  if ((rc = dalloc(c, &c->entries, sizeof(HashEntry) * (size_t)c->entry_count)) ||
      (rc = dalloc(c, &c->voxels, nvox * (size_t)c->vsize)) ||
      (rc = dalloc(c, &c->vba_slots, sizeof(int) * (size_t)s->block_count)) ||
      (rc = dalloc(c, &c->excess_slots, sizeof(int) * (size_t)s->excess_count)) ||
      (rc = dalloc(c, &c->req_key, sizeof(unsigned long long) * (size_t)s->bucket_count)) ||
      (rc = dalloc(c, &c->req_bits, sizeof(uint32_t) * (size_t)(s->bucket_count / 32))) ||
      (rc = dalloc(c, &c->req_list, sizeof(int) * (size_t)s->bucket_count)) ||
      (rc = dalloc(c, &c->req_excess_rank, sizeof(int) * (size_t)s->bucket_count)) ||
      (rc = dalloc(c, &c->compact_scan,
                   sizeof(unsigned long long) * (2 + (size_t)s->bucket_count / 32 / kCompactThreads))) ||
      (rc = dzero(c, c->compact_scan,
                  sizeof(unsigned long long) * (2 + (size_t)s->bucket_count / 32 / kCompactThreads))) ||
      (rc = dalloc(c, &c->alloc_list, sizeof(int) * (size_t)c->alloc_cap)) ||
      (rc = dalloc(c, &c->visible_list, sizeof(int) * (size_t)c->alloc_cap)) ||
      (rc = dalloc(c, &c->dstate, sizeof(DevState))) ||
      (rc = dalloc(c, &c->depth, sizeof(float) * (size_t)c->npix)) ||
      (rc = dalloc(c, &c->disp, sizeof(uint16_t) * (size_t)c->npix)) ||
      (rc = dalloc(c, &c->image_depth_scratch, sizeof(float) * (size_t)c->npix)) ||
      (rc = dalloc(c, &c->rgb, 3 * (size_t)c->rgbin.width * c->rgbin.height)) ||
      (rc = dalloc(c, &c->pyr, sizeof(float) * std::max<size_t>(c->pyr_floats, 1))) ||
      (rc = dalloc(c, &c->ranges, sizeof(float2) * (size_t)c->frag_w * c->frag_h)) ||
      (rc = dalloc(c, &c->ray_flags, sizeof(unsigned) * 2 * (size_t)c->frag_w * c->frag_h)) ||
      (rc = dzero(c, c->ray_flags, sizeof(unsigned) * 2 * (size_t)c->frag_w * c->frag_h)) ||
      (rc = dalloc(c, &c->points, sizeof(float4) * (size_t)c->npix)) ||
      (rc = dalloc(c, &c->normals, sizeof(float4) * (size_t)c->npix)) ||
      (rc = dalloc(c, &c->partials, sizeof(double) * 2 * 32 * (size_t)c->icp_grid)) ||
      (rc = dalloc(c, &c->trace, sizeof(double) * kTraceRow * kTraceCap)) ||
      (rc = dalloc(c, &c->shard_keys, sizeof(unsigned long long) * (size_t)c->npix)) ||
      (rc = dalloc(c, &c->icp_ctl, 1024)) ||
      (rc = dalloc(c, &c->surf_points, sizeof(float) * 3 * (size_t)c->surf_cap)) ||
      (rc = dalloc(c, &c->surf_colors, sizeof(float) * 3 * (size_t)c->surf_cap)) ||
      (rc = dalloc(c, &c->surf_scan, sizeof(unsigned long long) * (1 + (size_t)c->surf_tiles))) ||
      (rc = dalloc(c, &c->image, 3 * (size_t)c->npix)) || (rc = dalloc(c, &c->image_dmax, sizeof(int))) ||
      (rc = dalloc(c, &c->ren_partials, sizeof(double) * 32 * (size_t)c->ren_grid)) ||
      (c->vsize == 8 && (rc = dalloc(c, &c->cpyr, sizeof(float4) * cpyr_n))) ||
      (c->swapping &&
       ((rc = dalloc(c, &c->sw.state, (size_t)c->entry_count)) ||
        (rc = dalloc(c, &c->sw.host_slot, sizeof(int) * (size_t)c->entry_count)) ||
        (rc = dalloc(c, &c->sw.host_free, sizeof(int) * (size_t)c->host_max)) ||
        (rc = dalloc(c, &c->sw.host_chunks, sizeof(uint32_t*) * (size_t)(c->host_max / kHostChunk))) ||
        (rc = dalloc(c, &c->sw.in_cand, sizeof(int) * (size_t)c->entry_count)) ||
        (rc = dalloc(c, &c->sw.out_cand, sizeof(int) * (size_t)c->entry_count)) ||
        (rc = dalloc(c, &c->sw.stage_entry, sizeof(int) * 2 * kSwapSortCap)) ||
        (rc = dalloc(c, &c->sw.stage_slot, sizeof(int) * 2 * kSwapSortCap)) ||
        (rc = dalloc(c, &c->sw.stage_host, sizeof(int) * 2 * kSwapSortCap)) ||
        (rc = dalloc(c, &c->sw.journal, sizeof(int) * kSwapJournal))))) {
    free_all(c);
    delete c;
    return rc;
  }
  if (dalloc(c, &c->utab, sizeof(double) * utab_h.size()) ||
      cudaMemcpy(c->utab, utab_h.data(), sizeof(double) * utab_h.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    free_all(c);
    delete c;
    return VF_ERR_CUDA;
  }
  if (c->swapping) {
    // host block store: pinned chunks mapped into the device address space
    // (UVA); the first ones cover one VBA's worth of blocks
    c->sw.ctr = &c->dstate->swap;
    const int first = std::min(c->host_max, (c->s.block_count + kHostChunk - 1) / kHostChunk * kHostChunk);
    for (int k = 0; k < first / kHostChunk; ++k)
      if (int rc2 = add_host_chunk(c)) {
        free_all(c);
        delete c;
        return rc2;
      }
  }
  if (cudaMallocHost(reinterpret_cast<void**>(&c->hstate), sizeof(DevState)) != cudaSuccess ||
      cudaMallocHost(reinterpret_cast<void**>(&c->hpose), sizeof(PoseD)) != cudaSuccess) {
    free_all(c);
    delete c;
    return VF_ERR_CUDA;
  }
  for (auto& e : c->ev) cudaEventCreate(&e);
  cudaEventCreate(&c->ev_frame0);
  cudaEventCreate(&c->ev_frame1);
  if (s->shard_count > 1 && (cudaMalloc(reinterpret_cast<void**>(&c->p2p_flags),
                                        sizeof(unsigned long long) * kP2PFlagWords) != cudaSuccess ||
                             cudaMemset(c->p2p_flags, 0, sizeof(unsigned long long) * kP2PFlagWords) != cudaSuccess)) {
    free_all(c);
    delete c;
    return VF_ERR_CUDA;
  }
  if (s->shard_icp && s->shard_count > 1 &&
      (cudaMalloc(reinterpret_cast<void**>(&c->icp_xchg), kXchgBytes) != cudaSuccess ||
       cudaMemset(c->icp_xchg, 0, kXchgBytes) != cudaSuccess)) {
    free_all(c);
    delete c;
    return VF_ERR_CUDA;
  }
  persist_hash_table(c);
  if ((rc = reset_volume(c))) {
    free_all(c);
    delete c;
    return rc;
  }
  *out = c;
  return VF_OK;
}

int vf_destroy(vf_ctx* c) {
  if (!c) return VF_ERR_INVALID;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  free_all(c);
  delete c;
  return VF_OK;
}

const char* vf_last_error(const vf_ctx* c) { return c ? c->err.c_str() : "null context"; }

int vf_process_frame(vf_ctx* c, const float* depth_m, const uint8_t* rgb, vf_frame_stats* stats) {
  vf_frame_stats local;
  return frame_common(c, depth_m, rgb, false, stats ? stats : &local);
}

int vf_process_frame_device(vf_ctx* c, const float* d_depth, const uint8_t* d_rgb, vf_frame_stats* stats) {
  return frame_common(c, d_depth, d_rgb, true, stats);
}

int vf_submit_frame(vf_ctx* c, const float* depth_m, const uint8_t* rgb) {
  if (!c || !depth_m) return VF_ERR_INVALID;
  return submit_frame(c, depth_m, rgb);
}

int vf_submit_raw_frame(vf_ctx* c, const uint16_t* disparity, const uint8_t* rgb, int big_endian) {
  if (!c || !disparity) return VF_ERR_INVALID;
  return submit_frame(c, nullptr, rgb, disparity, big_endian != 0);
}

int vf_collect_frame(vf_ctx* c, vf_frame_stats* stats) {
  if (!c) return VF_ERR_INVALID;
  return collect_frame(c, stats);
}

int vf_frames_in_flight(const vf_ctx* c) { return c ? c->q_count : VF_ERR_INVALID; }

int vf_process_raw_frame(vf_ctx* c, const uint16_t* disparity, const uint8_t* rgb, int big_endian,
                         vf_frame_stats* stats) {
  vf_frame_stats local;
  return frame_common(c, nullptr, rgb, false, stats ? stats : &local, disparity, big_endian != 0);
}

int vf_process_raw_frame_device(vf_ctx* c, const uint16_t* d_disparity, const uint8_t* d_rgb, int big_endian,
                                vf_frame_stats* stats) {
  return frame_common(c, nullptr, d_rgb, true, stats, d_disparity, big_endian != 0);
}

int vf_disparity_to_depth(vf_ctx* c, const uint16_t* disparity, int big_endian, float* depth_out) {
  if (!c || !disparity || !depth_out) return VF_ERR_INVALID;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  VF_CUDA(c, cudaMemcpy(c->disp, disparity, sizeof(uint16_t) * (size_t)c->npix, cudaMemcpyHostToDevice));
  k_disparity_to_depth<<<(c->npix + 255) / 256, 256, 0, c->stream>>>(
      c->disp, c->npix, big_endian ? 1 : 0, (float)c->calib.disparity_a, (float)c->calib.disparity_b,
      (float)c->calib.depth.fx, c->s.max_depth, c->image_depth_scratch);
  VF_CUDA(c, cudaGetLastError());
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  VF_CUDA(c, cudaMemcpy(depth_out, c->image_depth_scratch, sizeof(float) * (size_t)c->npix, cudaMemcpyDeviceToHost));
  return VF_OK;
}

int vf_synchronize(vf_ctx* c) {
  if (!c) return VF_ERR_INVALID;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  return VF_OK;
}

int vf_read_stats(vf_ctx* c, vf_frame_stats* st) {
  if (!c || !st) return VF_ERR_INVALID;
  if (int rc = read_state(c)) return rc;
  fill_stats(c, c->s.tracking && c->frame > 1, c->frame - 1, st);
  return VF_OK;
}

int vf_set_pose(vf_ctx* c, const double pose[12]) {
  if (!c || !pose) return VF_ERR_INVALID;
  return set_pose_dev(c, pose);
}

int vf_get_pose(vf_ctx* c, double pose[12]) {
  if (!c || !pose) return VF_ERR_INVALID;
  if (int rc = read_state(c)) return rc;
  pose_to(c->hstate->pose, pose);
  return VF_OK;
}

int vf_frame_count(const vf_ctx* c) { return c ? c->frame : -1; }

int vf_get_maps(vf_ctx* c, float* points, float* normals) {
  if (!c) return VF_ERR_INVALID;
  if (!c->maps_valid) return VF_ERR_STATE;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  if (points) VF_CUDA(c, cudaMemcpy(points, c->points, sizeof(float4) * c->npix, cudaMemcpyDeviceToHost));
  if (normals) VF_CUDA(c, cudaMemcpy(normals, c->normals, sizeof(float4) * c->npix, cudaMemcpyDeviceToHost));
  return VF_OK;
}

int vf_set_maps(vf_ctx* c, const float* points, const float* normals, const double render_pose[12]) {
  if (!c || !points || !normals || !render_pose) return VF_ERR_INVALID;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  VF_CUDA(c, cudaMemcpy(c->points, points, sizeof(float4) * c->npix, cudaMemcpyHostToDevice));
  VF_CUDA(c, cudaMemcpy(c->normals, normals, sizeof(float4) * c->npix, cudaMemcpyHostToDevice));
  if (int rc = set_pose_dev(c, render_pose)) return rc;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  c->maps_valid = true;
  return VF_OK;
}

int vf_stage_forward_project(vf_ctx* c) {
  if (!c) return VF_ERR_INVALID;
  if (!c->maps_valid) return VF_ERR_STATE;
  if (int rc = launch_forward_project(c)) return rc;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  return VF_OK;
}

long vf_get_surface_points(vf_ctx* c, float* points, float* colors, long cap) {
  if (!c) return VF_ERR_INVALID;
  if (int rc = read_state(c)) return rc;
  const long n = c->hstate->ctr.surface_count;
  if (n > 0 && (points || colors)) {
    if (cap < n) return VF_ERR_INVALID;
    if (points) VF_CUDA(c, cudaMemcpy(points, c->surf_points, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost));
    if (colors) VF_CUDA(c, cudaMemcpy(colors, c->surf_colors, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost));
  }
  return n;
}

int vf_render_image(vf_ctx* c, int mode, uint8_t* out) {
  if (!c || !out) return VF_ERR_INVALID;
  cudaStream_t st = c->stream;
  const size_t bytes = 3 * (size_t)c->npix;
  switch (mode) {
    case VF_DISPLAY_RGB_PASSTHROUGH:
      if (!c->rgb_valid) return VF_ERR_STATE;
      VF_CUDA(c, cudaStreamSynchronize(st));
      VF_CUDA(c, cudaMemcpy(out, c->rgb, 3 * (size_t)c->rgbin.width * c->rgbin.height, cudaMemcpyDeviceToHost));
      return VF_OK;
    case VF_DISPLAY_DEPTH_COLOURIZED:
      if (c->frame == 0) return VF_ERR_STATE;
      VF_CUDA(c, cudaMemsetAsync(c->image_dmax, 0, sizeof(int), st));
      k_depth_max<<<c->num_sms, 256, 0, st>>>(c->depth, c->npix, c->image_dmax);
      k_colourize_depth<<<(c->npix + 255) / 256, 256, 0, st>>>(c->depth, c->npix, c->image_dmax, c->image);
      break;
    case VF_DISPLAY_RAYCAST:
    case VF_DISPLAY_RAYCAST_GREY:
      if (!c->maps_valid) return VF_ERR_STATE;
      k_render_image<<<(c->npix + 255) / 256, 256, 0, st>>>(
          hash_view(c), reinterpret_cast<const uint32_t*>(c->voxels), c->points, c->normals, &c->dstate->pose, c->din,
          c->s.voxel_size, (mode == VF_DISPLAY_RAYCAST && c->vsize == 8) ? 1 : 0, c->image);
      break;
    default:
      return VF_ERR_INVALID;
  }
  VF_CUDA(c, cudaGetLastError());
  VF_CUDA(c, cudaMemcpyAsync(out, c->image, bytes, cudaMemcpyDeviceToHost, st));
  VF_CUDA(c, cudaStreamSynchronize(st));
  return VF_OK;
}

// --- swap engine: host store access (block_store.hpp / block_store.cpp) ---
namespace {
constexpr uint32_t kVxbsMagic = 0x53425856u;  // 'VXBS' (block_store.hpp:41)
constexpr uint16_t kVxbsVersion = 1;
int codec_bytes(const vf_ctx* c) { return c->vsize == 8 ? 7 : 3; }
// VoxelCodec::encode / decode (voxel.hpp:124-155) on device-layout words
void encode_block(const vf_ctx* c, const uint32_t* words, uint8_t* out) {
  const int cb = codec_bytes(c);
  for (int v = 0; v < kBlockVolume; ++v) {
    const uint32_t w0 = words[v * (c->vsize / 4)];
    uint8_t* p = out + (size_t)v * cb;
    p[0] = (uint8_t)(w0 & 0xFF);
    p[1] = (uint8_t)((w0 >> 8) & 0xFF);
    p[2] = (uint8_t)((w0 >> 16) & 0xFF);
    if (c->vsize == 8) {
      const uint32_t w1 = words[v * 2 + 1];
      p[3] = (uint8_t)(w0 >> 24);
      p[4] = (uint8_t)(w1 & 0xFF);
      p[5] = (uint8_t)((w1 >> 8) & 0xFF);
      p[6] = (uint8_t)((w1 >> 16) & 0xFF);
    }
  }
}
void decode_block(const vf_ctx* c, const uint8_t* in, uint32_t* words) {
  const int cb = codec_bytes(c);
  for (int v = 0; v < kBlockVolume; ++v) {
    const uint8_t* p = in + (size_t)v * cb;
    if (c->vsize == 8) {
      words[v * 2] = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
      words[v * 2 + 1] = (uint32_t)p[4] | ((uint32_t)p[5] << 8) | ((uint32_t)p[6] << 16);
    } else {
      words[v] = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16);
    }
  }
}
void put_u16(uint8_t* p, uint16_t v) {
  p[0] = (uint8_t)(v & 0xFF);
  p[1] = (uint8_t)(v >> 8);
}
void put_u32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (uint8_t)((v >> (8 * i)) & 0xFF);
}
uint32_t get_u32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
}  // namespace

int vf_swap_states(vf_ctx* c, uint8_t* out) {
  if (!c || !out) return VF_ERR_INVALID;
  if (!c->swapping) return VF_ERR_STATE;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  VF_CUDA(c, cudaMemcpy(out, c->sw.state, (size_t)c->entry_count, cudaMemcpyDeviceToHost));
  return VF_OK;
}

long vf_swap_stored_count(vf_ctx* c) {
  if (!c) return VF_ERR_INVALID;
  if (!c->swapping) return 0;
  if (int rc = read_state(c)) return rc;
  return (long)c->host_cap - c->hstate->swap.host_top;
}

int vf_swap_store_read(vf_ctx* c, int entry, uint8_t* payload) {
  if (!c || entry < 0 || entry >= c->entry_count) return VF_ERR_INVALID;
  if (!c->swapping) return 0;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  int hs = -1;
  VF_CUDA(c, cudaMemcpy(&hs, c->sw.host_slot + entry, sizeof(int), cudaMemcpyDeviceToHost));
  if (hs < 0) return 0;
  if (payload) encode_block(c, host_slot_ptr(c, hs), payload);
  return 1;
}

long vf_swap_drain(vf_ctx* c, int* entries, long cap, long* lost) {
  if (!c || (cap > 0 && !entries)) return VF_ERR_INVALID;
  if (lost) *lost = 0;
  if (!c->swapping) return 0;
  if (int rc = read_state(c)) return rc;
  const int count = c->hstate->swap.journal_count;
  long avail = (long)count - c->journal_read;
  if (avail > kSwapJournal) {  // the ring wrapped before this drain
    if (lost) *lost = avail - kSwapJournal;
    c->journal_read = count - kSwapJournal;
    avail = kSwapJournal;
  }
  const long n = std::min(avail, cap);
  for (long done = 0; done < n;) {
    const int pos = (c->journal_read + (int)done) & (kSwapJournal - 1);
    const long run = std::min(n - done, (long)(kSwapJournal - pos));
    VF_CUDA(c, cudaMemcpy(entries + done, c->sw.journal + pos, sizeof(int) * run, cudaMemcpyDeviceToHost));
    done += run;
  }
  c->journal_read += (int)n;
  return n;
}

int vf_swap_save_store(vf_ctx* c, const char* path) {
  if (!c || !path) return VF_ERR_INVALID;
  if (!c->swapping) return VF_ERR_STATE;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  std::vector<int> hs((size_t)c->entry_count);
  VF_CUDA(c, cudaMemcpy(hs.data(), c->sw.host_slot, sizeof(int) * hs.size(), cudaMemcpyDeviceToHost));
  std::FILE* f = std::fopen(path, "wb");
  if (!f) {
    c->err = std::string("cannot create block store file: ") + path;
    return VF_ERR_INVALID;
  }
  const int payload = codec_bytes(c) * kBlockVolume;
  uint8_t header[16] = {};
  put_u32(header, kVxbsMagic);
  put_u16(header + 4, kVxbsVersion);
  put_u16(header + 6, (uint16_t)(c->vsize == 8 ? VF_VOXEL_S_RGB : VF_VOXEL_S));  // VoxelType tag (voxel.hpp:90)
  put_u32(header + 8, (uint32_t)c->entry_count);
  put_u32(header + 12, (uint32_t)payload);
  bool ok = std::fwrite(header, 1, 16, f) == 16;
  std::vector<uint8_t> rec((size_t)payload + 4);
  for (int i = 0; ok && i < c->entry_count; ++i) {
    if (hs[(size_t)i] < 0) continue;
    put_u32(rec.data(), (uint32_t)i);
    encode_block(c, host_slot_ptr(c, hs[(size_t)i]), rec.data() + 4);
    ok = std::fwrite(rec.data(), 1, rec.size(), f) == rec.size();
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) {
    c->err = std::string("short write to block store file: ") + path;
    return VF_ERR_INVALID;
  }
  return VF_OK;
}

int vf_swap_load_store(vf_ctx* c, const char* path) {
  if (!c || !path) return VF_ERR_INVALID;
  if (!c->swapping) return VF_ERR_STATE;
  std::FILE* f = std::fopen(path, "rb");
  if (!f) {
    c->err = std::string("cannot open block store file: ") + path;
    return VF_ERR_INVALID;
  }
  uint8_t header[16];
  const int payload = codec_bytes(c) * kBlockVolume;
  const uint16_t tag = (uint16_t)(c->vsize == 8 ? VF_VOXEL_S_RGB : VF_VOXEL_S);
  if (std::fread(header, 1, 16, f) != 16 || get_u32(header) != kVxbsMagic ||
      (uint16_t)(header[4] | (header[5] << 8)) != kVxbsVersion || (uint16_t)(header[6] | (header[7] << 8)) != tag ||
      get_u32(header + 8) != (uint32_t)c->entry_count || get_u32(header + 12) != (uint32_t)payload) {
    std::fclose(f);
    c->err = std::string("not a compatible block store file: ") + path;
    return VF_ERR_INVALID;
  }
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  if (int rc = read_state(c)) {
    std::fclose(f);
    return rc;
  }
  std::vector<int> hs((size_t)c->entry_count), hfree((size_t)c->host_cap);
  std::vector<HashEntry> ents((size_t)c->entry_count);
  cudaMemcpy(hs.data(), c->sw.host_slot, sizeof(int) * hs.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(hfree.data(), c->sw.host_free, sizeof(int) * hfree.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(ents.data(), c->entries, sizeof(HashEntry) * ents.size(), cudaMemcpyDeviceToHost);
  int top = c->hstate->swap.host_top;
  std::vector<uint8_t> rec((size_t)payload + 4);
  int rc = VF_OK;
  for (;;) {
    const size_t got = std::fread(rec.data(), 1, rec.size(), f);
    if (got == 0) break;
    if (got != rec.size()) {
      rc = VF_ERR_INVALID;
      c->err = "truncated block store record";
      break;
    }
    const uint32_t idx = get_u32(rec.data());
    if (idx >= (uint32_t)c->entry_count) {
      rc = VF_ERR_INVALID;
      c->err = "block store record index out of range";
      break;
    }
    // only swapped-out entries can ever be paged back in (swap.hpp:145)
    if (ents[idx].block_state != kEntrySwappedOut) continue;
    int slot = hs[idx];
    if (slot < 0) {
      if (top == 0) {  // grow: publish the pops so far, push a chunk, re-read the stack
        VF_CUDA(c, cudaMemcpy(&c->dstate->swap.host_top, &top, sizeof(int), cudaMemcpyHostToDevice));
        if (grow_host_store(c) != VF_OK || cudaStreamSynchronize(c->stream) != cudaSuccess) {
          rc = VF_ERR_OVERFLOW;
          c->err = "host block store full";
          break;
        }
        hfree.resize((size_t)c->host_cap);
        cudaMemcpy(hfree.data(), c->sw.host_free, sizeof(int) * hfree.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(&top, &c->dstate->swap.host_top, sizeof(int), cudaMemcpyDeviceToHost);
      }
      slot = hfree[(size_t)--top];
      hs[idx] = slot;
    }
    decode_block(c, rec.data() + 4, host_slot_ptr(c, slot));
  }
  std::fclose(f);
  VF_CUDA(c, cudaMemcpy(c->sw.host_slot, hs.data(), sizeof(int) * hs.size(), cudaMemcpyHostToDevice));
  VF_CUDA(c, cudaMemcpy(&c->dstate->swap.host_top, &top, sizeof(int), cudaMemcpyHostToDevice));
  c->host_top_lb = top;
  return rc;
}

long vf_entry_count(const vf_ctx* c) { return c ? c->entry_count : -1; }
long vf_voxel_bytes(const vf_ctx* c) { return c ? (long)c->s.block_count * kBlockVolume * c->vsize : -1; }

int vf_export_entries(vf_ctx* c, void* out) {
  if (!c || !out) return VF_ERR_INVALID;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  VF_CUDA(c, cudaMemcpy(out, c->entries, sizeof(HashEntry) * c->entry_count, cudaMemcpyDeviceToHost));
  return VF_OK;
}

int vf_export_voxels(vf_ctx* c, void* out) {
  if (!c || !out) return VF_ERR_INVALID;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  VF_CUDA(c, cudaMemcpy(out, c->voxels, (size_t)vf_voxel_bytes(c), cudaMemcpyDeviceToHost));
  return VF_OK;
}

int vf_export_free_stacks(vf_ctx* c, int* vba_top, int* vba_slots, int* excess_top, int* excess_slots) {
  if (!c) return VF_ERR_INVALID;
  if (int rc = read_state(c)) return rc;
  if (vba_top) *vba_top = c->hstate->ctr.vba_top;
  if (excess_top) *excess_top = c->hstate->ctr.excess_top;
  if (vba_slots) VF_CUDA(c, cudaMemcpy(vba_slots, c->vba_slots, sizeof(int) * c->s.block_count, cudaMemcpyDeviceToHost));
  if (excess_slots)
    VF_CUDA(c, cudaMemcpy(excess_slots, c->excess_slots, sizeof(int) * c->s.excess_count, cudaMemcpyDeviceToHost));
  return VF_OK;
}

int vf_import_state(vf_ctx* c, const void* entries, const void* voxels, int vba_top, const int* vba_slots,
                    int excess_top, const int* excess_slots) {
  if (!c || !entries || !voxels || !vba_slots || !excess_slots) return VF_ERR_INVALID;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  VF_CUDA(c, cudaMemcpy(c->entries, entries, sizeof(HashEntry) * c->entry_count, cudaMemcpyHostToDevice));
  VF_CUDA(c, cudaMemcpy(c->voxels, voxels, (size_t)vf_voxel_bytes(c), cudaMemcpyHostToDevice));
  VF_CUDA(c, cudaMemcpy(c->vba_slots, vba_slots, sizeof(int) * c->s.block_count, cudaMemcpyHostToDevice));
  VF_CUDA(c, cudaMemcpy(c->excess_slots, excess_slots, sizeof(int) * c->s.excess_count, cudaMemcpyHostToDevice));
  if (int rc = read_state(c)) return rc;
  DevState ds = *c->hstate;
  std::memset(&ds.ctr, 0, sizeof(ds.ctr));
  ds.ctr.vba_top = vba_top;
  ds.ctr.excess_top = excess_top;
  VF_CUDA(c, cudaMemcpy(c->dstate, &ds, sizeof(ds), cudaMemcpyHostToDevice));
  k_rebuild_alloc_list<<<c->num_sms * 4, 256, 0, c->stream>>>(c->entries, c->entry_count, c->alloc_list, c->alloc_cap,
                                                              &c->dstate->ctr);
  VF_CUDA(c, cudaGetLastError());
  if (int rc = reset_swap(c)) return rc;  // imported tables come without host data
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  return VF_OK;
}

long vf_export_visible_list(vf_ctx* c, int* out, long cap) {
  if (!c) return VF_ERR_INVALID;
  if (int rc = read_state(c)) return rc;
  const long n = c->hstate->ctr.visible_count;
  if (out && cap > 0) {
    const long k = n < cap ? n : cap;
    if (k > 0 && cudaMemcpy(out, c->visible_list, sizeof(int) * k, cudaMemcpyDeviceToHost) != cudaSuccess)
      return VF_ERR_CUDA;
  }
  return n;
}

long vf_export_ranges(vf_ctx* c, float* out) {
  if (!c) return VF_ERR_INVALID;
  const long n = (long)c->frag_w * c->frag_h;
  if (out) {
    VF_CUDA(c, cudaStreamSynchronize(c->stream));
    VF_CUDA(c, cudaMemcpy(out, c->ranges, sizeof(float2) * n, cudaMemcpyDeviceToHost));
  }
  return n;
}

int vf_stage_allocate(vf_ctx* c, const float* depth_m, const double pose[12], vf_alloc_stats* out) {
  if (!c || !depth_m || !pose) return VF_ERR_INVALID;
  const vf_settings& s = c->s;
  cudaStream_t st = c->stream;
  if (int rc = upload(c, c->depth, depth_m, sizeof(float) * c->npix, false)) return rc;
  if (int rc = set_pose_dev(c, pose)) return rc;
  k_mark<<<mark_grid(c), 256, 0, st>>>(c->depth, c->din, &c->dstate->pose, c->rgbin, c->depth_to_rgb,
                                                &c->dstate->fp, hash_view(c), s.voxel_size, s.mu, c->shard, c->req_key,
                                                c->req_bits, &c->dstate->ctr);
  if (int rc = launch_alloc_scan(c, st)) return rc;
  k_alloc_apply<<<c->num_sms * 2, 256, 0, st>>>(c->depth, c->din, &c->dstate->fp, s.voxel_size, s.mu, c->entries,
                                                c->mask, s.bucket_size, c->ordered, c->req_key, c->req_list,
                                                c->req_excess_rank, &c->dstate->meta, c->vba_slots, c->excess_slots,
                                                c->alloc_list, c->alloc_cap, &c->dstate->ctr, c->compact_scan,
                                                scan_words(c));
  k_visible<<<c->num_sms * 4, 256, 0, st>>>(c->entries, c->alloc_list, &c->dstate->fp, c->din, s.voxel_size,
                                            s.near_clip, s.far_clip, s.visibility_margin_px, c->visible_list,
                                            &c->dstate->ctr);
  VF_CUDA(c, cudaGetLastError());
  if (int rc = read_state(c)) return rc;
  if (out) {
    out->requested = c->hstate->ctr.requested;
    out->allocated = c->hstate->ctr.allocated;
    out->dropped_vba_full = c->hstate->ctr.dropped_vba_full;
    out->dropped_excess_full = c->hstate->ctr.dropped_excess_full;
  }
  return c->hstate->ctr.error_flags ? VF_ERR_OVERFLOW : VF_OK;
}

int vf_stage_integrate(vf_ctx* c, const float* depth_m, const uint8_t* rgb, const double pose[12]) {
  if (!c || !depth_m || !pose) return VF_ERR_INVALID;
  const vf_settings& s = c->s;
  cudaStream_t st = c->stream;
  if (int rc = upload(c, c->depth, depth_m, sizeof(float) * c->npix, false)) return rc;
  const bool with_rgb = rgb && c->vsize == 8;
  if (with_rgb && upload(c, c->rgb, rgb, 3 * (size_t)c->rgbin.width * c->rgbin.height, false)) return VF_ERR_CUDA;
  if (int rc = set_pose_dev(c, pose)) return rc;
  k_prep<<<1, 32, 0, st>>>(&c->dstate->pose, c->din, c->rgbin, c->depth_to_rgb, &c->dstate->fp);
  launch_integrate(c->num_sms * int_grid_mult(), st, c->vsize == 8, s.integration_mode == VF_INTEGRATION_FAST, c->entries, c->visible_list, &c->dstate->ctr, c->voxels, c->depth,
                   with_rgb ? c->rgb : nullptr, &c->dstate->fp, s.voxel_size, s.mu, s.max_weight,
                   s.stop_integrating_at_max);
  VF_CUDA(c, cudaGetLastError());
  VF_CUDA(c, cudaStreamSynchronize(st));
  return VF_OK;
}

int vf_stage_raycast(vf_ctx* c, const double pose[12]) {
  if (!c || !pose) return VF_ERR_INVALID;
  const vf_settings& s = c->s;
  cudaStream_t st = c->stream;
  if (int rc = set_pose_dev(c, pose)) return rc;
  k_prep<<<1, 32, 0, st>>>(&c->dstate->pose, c->din, c->rgbin, c->depth_to_rgb, &c->dstate->fp);
  k_init_ranges<<<(c->frag_w * c->frag_h + 255) / 256, 256, 0, st>>>(c->ranges, c->frag_w * c->frag_h);
  VF_CUDA(c, launch_pdl(k_ranges, dim3(c->num_sms * 2), dim3(256), 0, st, c->entries, c->visible_list,
                        &c->dstate->ctr, &c->dstate->fp, c->din, s.voxel_size, s.near_clip, s.far_clip, c->ranges,
                        c->frag_w));
  if (int rc = launch_raycast(c, st)) return rc;
  VF_CUDA(c, cudaGetLastError());
  VF_CUDA(c, cudaStreamSynchronize(st));
  c->maps_valid = true;
  return VF_OK;
}

int vf_stage_icp(vf_ctx* c, const float* depth_m, const double initial_pose[12], double out_pose[12],
                 int* iterations, double* cost, int* valid_points, int* ok) {
  if (!c || !depth_m) return VF_ERR_INVALID;
  if (!c->maps_valid) return VF_ERR_STATE;
  cudaStream_t st = c->stream;
  if (int rc = upload(c, c->depth, depth_m, sizeof(float) * c->npix, false)) return rc;
  if (initial_pose) {
    *c->hpose = pose_from(initial_pose);
    VF_CUDA(c, cudaMemcpyAsync(&c->dstate->init_pose, c->hpose, sizeof(PoseD), cudaMemcpyHostToDevice, st));
  }
  if (c->s.hierarchy_levels > 1)
    k_pyramid<<<dim3((c->din.width + 31) / 32, (c->din.height + 31) / 32), 256, 0, st>>>(
        c->depth, c->din.width, c->din.height, c->s.hierarchy_levels, c->pyr);
  if (int rc = launch_icp(c, st, initial_pose != nullptr, /*update_state=*/false)) return rc;
  VF_CUDA(c, cudaGetLastError());
  if (int rc = read_state(c)) return rc;
  const IcpResult& r = c->hstate->icp;
  if (out_pose) pose_to(r.pose, out_pose);
  if (iterations) *iterations = r.iterations;
  if (cost) *cost = r.final_cost;
  if (valid_points) *valid_points = r.valid_points;
  if (ok) *ok = r.ok;
  return VF_OK;
}

namespace {
int stage_result(vf_ctx* c, double* out_pose, int* iterations, double* cost, int* valid_points, int* ok) {
  if (int rc = read_state(c)) return rc;
  const IcpResult& r = c->hstate->icp;
  if (out_pose) pose_to(r.pose, out_pose);
  if (iterations) *iterations = r.iterations;
  if (cost) *cost = r.final_cost;
  if (valid_points) *valid_points = r.valid_points;
  if (ok) *ok = r.ok;
  return VF_OK;
}
}  // namespace

int vf_stage_ren(vf_ctx* c, const float* depth_m, const double initial_pose[12], double out_pose[12],
                 int* iterations, double* cost, int* valid_points, int* ok) {
  if (!c || !depth_m || !initial_pose) return VF_ERR_INVALID;
  cudaStream_t st = c->stream;
  if (int rc = upload(c, c->depth, depth_m, sizeof(float) * c->npix, false)) return rc;
  *c->hpose = pose_from(initial_pose);
  VF_CUDA(c, cudaMemcpyAsync(&c->dstate->init_pose, c->hpose, sizeof(PoseD), cudaMemcpyHostToDevice, st));
  int launches = 0;
  if (int rc = enqueue_ren(c, st, false, &c->dstate->init_pose, false, &launches)) return rc;
  return stage_result(c, out_pose, iterations, cost, valid_points, ok);
}

int vf_stage_color(vf_ctx* c, const uint8_t* rgb, const double initial_pose[12], double out_pose[12],
                   int* iterations, double* cost, int* valid_points, int* ok) {
  if (!c || !rgb || !initial_pose) return VF_ERR_INVALID;
  if (c->vsize != 8) return VF_ERR_INVALID;
  cudaStream_t st = c->stream;
  if (int rc = upload(c, c->rgb, rgb, 3 * (size_t)c->rgbin.width * c->rgbin.height, false)) return rc;
  *c->hpose = pose_from(initial_pose);
  VF_CUDA(c, cudaMemcpyAsync(&c->dstate->init_pose, c->hpose, sizeof(PoseD), cudaMemcpyHostToDevice, st));
  int launches = 0;
  if (int rc = enqueue_color(c, st, &c->dstate->init_pose, false, &launches)) return rc;
  return stage_result(c, out_pose, iterations, cost, valid_points, ok);
}

long vf_icp_trace(vf_ctx* c, double* out, long max_rows) {
  if (!c) return VF_ERR_INVALID;
  if (int rc = read_state(c)) return rc;
  const long n = std::min<long>(c->hstate->icp.trace_rows, kTraceCap);
  if (out && max_rows > 0) {
    const long k = std::min(n, max_rows);
    if (cudaMemcpy(out, c->trace, sizeof(double) * kTraceRow * k, cudaMemcpyDeviceToHost) != cudaSuccess)
      return VF_ERR_CUDA;
  }
  return n;
}

int vf_depth_pyramid(vf_ctx* c, const float* depth_m, float* out) {
  if (!c || !depth_m || !out) return VF_ERR_INVALID;
  if (int rc = upload(c, c->depth, depth_m, sizeof(float) * c->npix, false)) return rc;
  if (c->s.hierarchy_levels > 1)
    k_pyramid<<<dim3((c->din.width + 31) / 32, (c->din.height + 31) / 32), 256, 0, c->stream>>>(
        c->depth, c->din.width, c->din.height, c->s.hierarchy_levels, c->pyr);
  VF_CUDA(c, cudaGetLastError());
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  VF_CUDA(c, cudaMemcpy(out, c->depth, sizeof(float) * c->npix, cudaMemcpyDeviceToHost));
  if (c->pyr_floats)
    VF_CUDA(c, cudaMemcpy(out + c->npix, c->pyr, sizeof(float) * c->pyr_floats, cudaMemcpyDeviceToHost));
  return VF_OK;
}

int vf_volume_digest(vf_ctx* c, uint64_t* out) {
  // FNV-1a over allocated entries ascending: pos bytes, then the LE
  // VoxelCodec bytes of each voxel (pipeline_impl.hpp:144-164, voxel.hpp:123-155).
  if (!c || !out) return VF_ERR_INVALID;
  std::vector<HashEntry> e((size_t)c->entry_count);
  std::vector<uint8_t> v((size_t)vf_voxel_bytes(c));
  if (int rc = vf_export_entries(c, e.data())) return rc;
  if (int rc = vf_export_voxels(c, v.data())) return rc;
  uint64_t h = 1469598103934665603ull;
  auto fnv = [&](uint8_t b) {
    h ^= b;
    h *= 1099511628211ull;
  };
  const int codec = c->vsize == 8 ? 7 : 3;
  for (const HashEntry& he : e) {
    if (he.block_state < 0) continue;
    const uint8_t* pb = reinterpret_cast<const uint8_t*>(&he);
    for (int k = 0; k < 6; ++k) fnv(pb[k]);
    for (int i = 0; i < kBlockVolume; ++i) {
      const uint8_t* vx = v.data() + ((size_t)he.block_state * kBlockVolume + i) * c->vsize;
      for (int k = 0; k < codec; ++k) fnv(vx[k]);
    }
  }
  *out = h;
  return VF_OK;
}

int vf_render_synthetic(int device, int n_spheres, const double* spheres, int n_planes, const double* planes,
                        const double world_to_cam[12], const vf_intrinsics* intr, double near_clip, double far_clip,
                        float* d_depth, uint8_t* d_rgb) {
  if (!world_to_cam || !intr || (n_spheres > 0 && !spheres) || (n_planes > 0 && !planes)) return VF_ERR_INVALID;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device) {
    cudaGetLastError();
    return VF_ERR_NO_DEVICE;
  }
  cudaSetDevice(device);
  double* dsp = nullptr;
  double* dpl = nullptr;
  const size_t bs = sizeof(double) * 7 * std::max(n_spheres, 1), bp = sizeof(double) * 9 * std::max(n_planes, 1);
  if (cudaMalloc(&dsp, bs) != cudaSuccess || cudaMalloc(&dpl, bp) != cudaSuccess) return VF_ERR_CUDA;
  if (n_spheres) cudaMemcpy(dsp, spheres, sizeof(double) * 7 * n_spheres, cudaMemcpyHostToDevice);
  if (n_planes) cudaMemcpy(dpl, planes, sizeof(double) * 9 * n_planes, cudaMemcpyHostToDevice);
  const PoseD c2w = pose_inverse(pose_from(world_to_cam));
  const IntrD in = intr_of(*intr);
  const int npix = in.width * in.height;
  k_synth<<<(npix + 255) / 256, 256>>>(n_spheres, dsp, n_planes, dpl, c2w, in, near_clip, far_clip, d_depth, d_rgb);
  cudaError_t e = cudaDeviceSynchronize();
  cudaFree(dsp);
  cudaFree(dpl);
  return e == cudaSuccess ? VF_OK : VF_ERR_CUDA;
}

void* vf_device_alloc(size_t bytes) {
  void* p = nullptr;
  return cudaMalloc(&p, bytes) == cudaSuccess ? p : nullptr;
}
int vf_device_free(void* p) { return cudaFree(p) == cudaSuccess ? VF_OK : VF_ERR_CUDA; }
int vf_memcpy_h2d(void* dst, const void* src, size_t bytes) {
  return cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess ? VF_OK : VF_ERR_CUDA;
}
int vf_memcpy_d2h(void* dst, const void* src, size_t bytes) {
  return cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost) == cudaSuccess ? VF_OK : VF_ERR_CUDA;
}
void* vf_host_alloc_pinned(size_t bytes) {
  void* p = nullptr;
  return cudaMallocHost(&p, bytes) == cudaSuccess ? p : nullptr;
}
int vf_host_free_pinned(void* p) { return cudaFreeHost(p) == cudaSuccess ? VF_OK : VF_ERR_CUDA; }

int vf_event_record(vf_ctx* c, int slot) {
  if (!c || slot < 8 || slot >= kNumEvents) return VF_ERR_INVALID;  // 0..7 reserved for stage profiling
  VF_CUDA(c, cudaEventRecord(c->ev[slot], c->stream));
  return VF_OK;
}
int vf_event_elapsed_ms(vf_ctx* c, int a, int b, float* ms) {
  if (!c || !ms || a < 0 || b < 0 || a >= kNumEvents || b >= kNumEvents) return VF_ERR_INVALID;
  VF_CUDA(c, cudaEventSynchronize(c->ev[b]));
  VF_CUDA(c, cudaEventElapsedTime(ms, c->ev[a], c->ev[b]));
  return VF_OK;
}
int vf_set_profiling(vf_ctx* c, int enabled) {
  if (!c) return VF_ERR_INVALID;
  c->profiling = enabled != 0;
  for (double& m : c->stage_ms) m = 0;
  c->profiled_frames = 0;
  return VF_OK;
}
int vf_alloc_counters(vf_ctx* c, unsigned long long* out) {
  if (!c || !out) return VF_ERR_INVALID;
  if (!c->maps_valid) {
    c->err = "vf_alloc_counters: no frame processed yet";
    return VF_ERR_STATE;
  }
  unsigned long long* d = nullptr;
  VF_CUDA(c, cudaMallocAsync(reinterpret_cast<void**>(&d), 3 * sizeof(unsigned long long), c->stream));
  VF_CUDA(c, cudaMemsetAsync(d, 0, 3 * sizeof(unsigned long long), c->stream));
  k_mark_count<<<mark_grid(c), 256, 0, c->stream>>>(c->depth, c->din, &c->dstate->pose, hash_view(c),
                                                    c->s.voxel_size, c->s.mu, c->shard, d);
  VF_CUDA(c, cudaGetLastError());
  VF_CUDA(c, cudaMemcpyAsync(out, d, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
  VF_CUDA(c, cudaFreeAsync(d, c->stream));
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  return VF_OK;
}
int vf_raycast_counters(vf_ctx* c, unsigned long long* out) {
  if (!c || !out) return VF_ERR_INVALID;
  if (!c->maps_valid) {
    c->err = "vf_raycast_counters: no frame processed yet";
    return VF_ERR_STATE;
  }
  unsigned long long* d = nullptr;
  VF_CUDA(c, cudaMallocAsync(reinterpret_cast<void**>(&d), 4 * sizeof(unsigned long long), c->stream));
  VF_CUDA(c, cudaMemsetAsync(d, 0, 4 * sizeof(unsigned long long), c->stream));
  k_raycast_count<<<dim3(c->frag_w, c->frag_h * 2), 128, 0, c->stream>>>(
      hash_view(c), reinterpret_cast<const uint32_t*>(c->voxels), c->vsize / 4, c->ranges, &c->dstate->fp, c->din,
      c->s.voxel_size, c->s.mu, c->points, c->normals, d);
  VF_CUDA(c, cudaGetLastError());
  VF_CUDA(c, cudaMemcpyAsync(out, d, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
  VF_CUDA(c, cudaFreeAsync(d, c->stream));
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  return VF_OK;
}
int vf_set_stage_timing(vf_ctx* c, int enabled) {
  if (!c) return VF_ERR_INVALID;
  c->stage_timing = enabled != 0;
  return VF_OK;
}
int vf_stage_times(vf_ctx* c, double* ms_out, long* frames) {
  if (!c || !ms_out) return VF_ERR_INVALID;
  for (int i = 0; i < 8; ++i) ms_out[i] = c->stage_ms[i];
  if (frames) *frames = c->profiled_frames;
  return VF_OK;
}
long vf_selftest_division(int device, int mode, float p0, float p1, float p2, long n) {
  if (cudaSetDevice(device) != cudaSuccess) return VF_ERR_NO_DEVICE;
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, sizeof(unsigned long long)) != cudaSuccess) return VF_ERR_CUDA;
  cudaMemset(d, 0, sizeof(unsigned long long));
  if (mode == 0) {  // divisor p0, amin p2 <= |a| <= amax p1
    const uint32_t lo = __builtin_bit_cast(uint32_t, p2), hi = __builtin_bit_cast(uint32_t, p1);
    k_divtest_const<<<4096, 256>>>(p0, lo, hi >= lo ? hi - lo + 1u : 0u, d);
  } else {
    k_divtest_rand<<<4096, 256>>>(p0, p1, p2, (unsigned long long)n, d);
  }
  unsigned long long h = 0;
  cudaError_t e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? (long)h : VF_ERR_CUDA;
}

// ---- pixel-sharded ICP: peer mappings of the exchange areas ----
namespace {
void drop_graphs(vf_ctx* c) {
  for (auto& plane : c->graph)
    for (auto& row : plane)
      for (auto& g : row)
        if (g) {
          cudaGraphExecDestroy(g);
          g = nullptr;
        }
}
}  // namespace

// ---- nearest-depth composite over peer memory ----
namespace {
void p2p_fill(vf_ctx* c, int r, const unsigned long long* keys, const float4* pts, const float4* nrm,
              unsigned long long* flags) {
  c->p2p.keys[r] = keys;
  c->p2p.points[r] = pts;
  c->p2p.normals[r] = nrm;
  c->p2p.flags[r] = flags;
}
}  // namespace

int vf_shard_p2p_link_local(vf_ctx** ctxs, int count) {
  if (!ctxs || count < 2 || count > kMaxShards) return VF_ERR_INVALID;
  for (int r = 0; r < count; ++r) {
    vf_ctx* c = ctxs[r];
    if (!c || !c->p2p_flags || c->shard.count != count || c->shard.index != r || c->device != ctxs[0]->device ||
        c->npix != ctxs[0]->npix || c->nccl_comm)
      return VF_ERR_INVALID;
  }
  for (int r = 0; r < count; ++r) {
    vf_ctx* c = ctxs[r];
    cudaSetDevice(c->device);
    VF_CUDA(c, cudaStreamSynchronize(c->stream));
    VF_CUDA(c, cudaMemset(c->p2p_flags, 0, sizeof(unsigned long long) * kP2PFlagWords));
    c->p2p.n = count;
    c->p2p.rank = r;
    c->p2p.ctr = &c->dstate->ctr;
    for (int k = 0; k < count; ++k)
      p2p_fill(c, k, ctxs[k]->shard_keys, ctxs[k]->points, ctxs[k]->normals, ctxs[k]->p2p_flags);
    c->p2p_linked = count;
    drop_graphs(c);
  }
  return VF_OK;
}

int vf_shard_p2p_handles(vf_ctx* c, void* out) {
  if (!c || !out) return VF_ERR_INVALID;
  if (!c->p2p_flags) return VF_ERR_STATE;
  cudaSetDevice(c->device);
  void* ptrs[4] = {c->shard_keys, c->points, c->normals, c->p2p_flags};
  for (int k = 0; k < 4; ++k) {
    cudaIpcMemHandle_t h;
    VF_CUDA(c, cudaIpcGetMemHandle(&h, ptrs[k]));
    std::memcpy(static_cast<uint8_t*>(out) + k * sizeof(h), &h, sizeof(h));
  }
  return VF_OK;
}

int vf_shard_p2p_link(vf_ctx* c, const void* handles, int count) {
  if (!c || !handles || count != c->shard.count || count < 2 || count > kMaxShards || c->nccl_comm)
    return VF_ERR_INVALID;
  if (!c->p2p_flags) return VF_ERR_STATE;
  cudaSetDevice(c->device);
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  VF_CUDA(c, cudaMemset(c->p2p_flags, 0, sizeof(unsigned long long) * kP2PFlagWords));
  c->p2p.n = count;
  c->p2p.rank = c->shard.index;
  c->p2p.ctr = &c->dstate->ctr;
  for (int r = 0; r < count; ++r) {
    if (r == c->shard.index) {
      p2p_fill(c, r, c->shard_keys, c->points, c->normals, c->p2p_flags);
      continue;
    }
    void* p[4];
    for (int k = 0; k < 4; ++k) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const uint8_t*>(handles) + ((size_t)r * 4 + k) * sizeof(h), sizeof(h));
      VF_CUDA(c, cudaIpcOpenMemHandle(&p[k], h, cudaIpcMemLazyEnablePeerAccess));
      c->ipc_opened.push_back(p[k]);
    }
    p2p_fill(c, r, static_cast<const unsigned long long*>(p[0]), static_cast<const float4*>(p[1]),
             static_cast<const float4*>(p[2]), static_cast<unsigned long long*>(p[3]));
  }
  c->p2p_linked = count;
  drop_graphs(c);
  return VF_OK;
}

int vf_shard_icp_link_local(vf_ctx** ctxs, int count) {
  if (!ctxs || count < 2 || count > kMaxShards) return VF_ERR_INVALID;
  for (int r = 0; r < count; ++r) {
    vf_ctx* c = ctxs[r];
    if (!c || !c->icp_xchg || c->shard.count != count || c->shard.index != r || c->device != ctxs[0]->device)
      return VF_ERR_INVALID;
  }
  for (int r = 0; r < count; ++r) {
    vf_ctx* c = ctxs[r];
    cudaSetDevice(c->device);
    VF_CUDA(c, cudaStreamSynchronize(c->stream));
    VF_CUDA(c, cudaMemset(c->icp_xchg, 0, kXchgBytes));
    for (int k = 0; k < count; ++k) c->icp_peers[k] = ctxs[k]->icp_xchg;
    c->icp_linked = count;
    drop_graphs(c);  // the frame graph now carries the exchange
  }
  return VF_OK;
}

int vf_shard_icp_handle(vf_ctx* c, void* handle_out) {
  if (!c || !handle_out) return VF_ERR_INVALID;
  if (!c->icp_xchg) {
    c->err = "vf_shard_icp_handle: create the context with shard_icp = 1 and shard_count > 1";
    return VF_ERR_STATE;
  }
  cudaSetDevice(c->device);
  cudaIpcMemHandle_t h;
  VF_CUDA(c, cudaIpcGetMemHandle(&h, c->icp_xchg));
  std::memcpy(handle_out, &h, sizeof(h));
  return VF_OK;
}

int vf_shard_icp_link(vf_ctx* c, const void* handles, int count) {
  if (!c || !handles || count != c->shard.count || count < 2 || count > kMaxShards) return VF_ERR_INVALID;
  if (!c->icp_xchg) return VF_ERR_STATE;
  cudaSetDevice(c->device);
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  VF_CUDA(c, cudaMemset(c->icp_xchg, 0, kXchgBytes));
  for (int r = 0; r < count; ++r) {
    if (r == c->shard.index) {
      c->icp_peers[r] = c->icp_xchg;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const uint8_t*>(handles) + (size_t)r * sizeof(h), sizeof(h));
    void* p = nullptr;
    VF_CUDA(c, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(p);
    c->icp_peers[r] = static_cast<double*>(p);
  }
  c->icp_linked = count;
  drop_graphs(c);
  return VF_OK;
}

int vf_shard_owner(int bx, int by, int bz, int shard_shift, int shard_count) {
  return shard_owner(bx, by, bz, ShardSpec{shard_count, 0, shard_shift, 0});
}

int vf_shard_nccl_unique_id(void* out128) {
  if (!out128) return VF_ERR_INVALID;
  return nccl_unique_id(out128) == 0 ? VF_OK : VF_ERR_NO_DEVICE;
}

int vf_shard_attach_nccl(vf_ctx* c, const void* id, int nranks, int rank) {
  if (!c || !id || nranks != c->shard.count || rank != c->shard.index) return VF_ERR_INVALID;
  cudaSetDevice(c->device);
  if (nccl_comm_init(&c->nccl_comm, id, nranks, rank) != 0) {
    c->err = "ncclCommInitRank failed";
    return VF_ERR_CUDA;
  }
  for (auto& plane : c->graph)  // the frame graph now ends with the composite
    for (auto& row : plane)
      for (auto& g : row)
        if (g) {
          cudaGraphExecDestroy(g);
          g = nullptr;
        }
  return VF_OK;
}

int vf_shard_composite_local(vf_ctx** ctxs, int n) {
  if (!ctxs || n < 1 || n > kMaxShards) return VF_ERR_INVALID;
  const int npix = ctxs[0]->npix;
  ShardGroupArgs g{};
  g.n = n;
  for (int i = 0; i < n; ++i) {
    vf_ctx* c = ctxs[i];
    if (!c || c->npix != npix || c->device != ctxs[0]->device || c->shard.index != i) return VF_ERR_INVALID;
    k_shard_keys<<<(npix + 255) / 256, 256, 0, c->stream>>>(c->points, &c->dstate->fp, npix, i, c->shard_keys);
    VF_CUDA(c, cudaGetLastError());
    VF_CUDA(c, cudaStreamSynchronize(c->stream));
    g.keys[i] = c->shard_keys;
    g.points[i] = c->points;
    g.normals[i] = c->normals;
  }
  k_shard_group_composite<<<(npix + 255) / 256, 256, 0, ctxs[0]->stream>>>(g, npix);
  VF_CUDA(ctxs[0], cudaGetLastError());
  VF_CUDA(ctxs[0], cudaStreamSynchronize(ctxs[0]->stream));
  return VF_OK;
}

long vf_readback_bytes(const vf_ctx* c) { return c ? (long)sizeof(DevState) : -1; }

int vf_flush_l2(vf_ctx* c, size_t bytes) {
  if (!c) return VF_ERR_INVALID;
  if (c->flush_bytes < bytes) {
    if (c->flush_buf) cudaFree(c->flush_buf);
    c->flush_buf = nullptr;
    c->flush_bytes = 0;
    VF_CUDA(c, cudaMalloc(&c->flush_buf, bytes));
    c->flush_bytes = bytes;
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  VF_CUDA(c, cudaEventCreate(&e0));
  VF_CUDA(c, cudaEventCreate(&e1));
  c->flush_ev.emplace_back(e0, e1);
  VF_CUDA(c, cudaEventRecord(e0, c->stream));
  VF_CUDA(c, cudaMemsetAsync(c->flush_buf, (int)(c->frame & 0xFF), bytes, c->stream));
  VF_CUDA(c, cudaEventRecord(e1, c->stream));
  return VF_OK;
}

int vf_flush_time(vf_ctx* c, double* ms) {
  if (!c || !ms) return VF_ERR_INVALID;
  VF_CUDA(c, cudaStreamSynchronize(c->stream));
  double total = 0;
  for (auto& e : c->flush_ev) {
    float t = 0;
    cudaEventElapsedTime(&t, e.first, e.second);
    total += t;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  c->flush_ev.clear();
  *ms = total;
  return VF_OK;
}

long vf_last_modified_voxels(vf_ctx* c) {
  if (!c) return VF_ERR_INVALID;
  if (int rc = read_state(c)) return rc;
  return c->hstate->ctr.modified_voxels;
}

int vf_kernel_launches_per_frame(vf_ctx* c, int tracking_frame) {
  if (!c) return VF_ERR_INVALID;
  int icp = 1 + ((c->icp_cluster && c->icp_coarse_levels > 0 && c->icp_coarse_levels < c->s.hierarchy_levels) ? 1 : 0);
  const int L = c->s.hierarchy_levels;
  int track = 0;
  if (tracking_frame) {
    switch (c->s.tracker_type) {
      case VF_TRACKER_COLOR:
        track = 2 * L + 1;  // colour pyramid + the one-CTA tracker (RGB frames)
        break;
      case VF_TRACKER_ICP_REN: {
        const int coarse = (c->icp_cluster && c->icp_coarse_levels > 0) ? std::min(c->icp_coarse_levels, L - 1) : 0;
        track = (L > 1 ? 1 : 0) + (L > 1 ? 1 + ((coarse > 0 && coarse < L - 1) ? 1 : 0) : 1) + 2 +
                2 * c->s.max_iterations;
        break;
      }
      default:
        track = (L > 1 ? 1 : 0) + icp;
    }
  }
  return 8 + track + (c->p2p_linked > 1 ? 6 : c->nccl_comm ? 2 : 0) + (c->vsize == 8 ? 1 : 0) + (c->swapping ? 4 : 0);
}

}  // extern "C"
