/*
 * voxfuse_b200 — C ABI of the B200 (sm_100a) dense-fusion hot path.
 *
 * Drop-in replacement for the reference's per-frame path
 * (/root/reference/proj, the CPU re-implementation of InfiniTAM, arXiv 1410.0925):
 * voxel-block-hash allocation, TSDF / colour integration, hash-walking raycast
 * and the point-to-plane ICP tracker.  The reference exposes that path as the
 * C++ interface IPipeline + make_pipeline (proj/include/voxfuse/engine/pipeline.hpp:66-86)
 * and as stage templates (allocation.hpp, integration.hpp, raycast.hpp,
 * pyramid.hpp, depth_tracker.hpp); every entry point below names the
 * reference interface it replaces.  Plain C types only: pointers, sizes, POD
 * structs.  INTEGRATION.md shows the C++ IPipeline adapter and ctypes binding.
 *
 * Conventions (reference SPEC.md:708, pipeline.hpp): one context = one volume
 * = one CUDA stream; a context is not thread-safe; the hot path never throws;
 * every function returns VF_OK or a negative status.  There is no CPU
 * fallback: without a usable sm_100 device vf_create fails with
 * VF_ERR_NO_DEVICE.
 *
 * Poses are world-to-camera rigid transforms stored as 12 doubles: the
 * row-major 3x3 rotation followed by the translation (reference Pose,
 * proj/include/voxfuse/core/pose.hpp:8-46).  Images are row-major; depth is
 * float metres with <= 0 marking missing samples; RGB is packed u8 x 3.
 */
#ifndef VOXFUSE_B200_H
#define VOXFUSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define VF_ABI_VERSION 3

enum vf_status {
  VF_OK = 0,
  VF_ERR_INVALID = -1,   /* bad argument / settings (reference: std::invalid_argument) */
  VF_ERR_CUDA = -2,      /* CUDA runtime error; see vf_last_error */
  VF_ERR_NO_DEVICE = -3, /* no sm_100 device: there is no CPU fallback */
  VF_ERR_STATE = -4,     /* call not valid in the current state (e.g. maps not rendered yet) */
  VF_ERR_OVERFLOW = -5   /* a device-side capacity was exceeded (see vf_frame_stats.error_flags) */
};

enum vf_voxel_type { VF_VOXEL_S = 1, VF_VOXEL_S_RGB = 2 }; /* voxel.hpp:90 (VoxelS, VoxelSRgb) */

/* EngineSettings + SceneParams + HashConfig + TrackerSettings
 * (pipeline.hpp:19-41, scene_params.hpp:6-13, hash_volume.hpp:49-58,
 * tracking_state.hpp:12-23).  vf_default_settings() fills the reference
 * defaults. */
typedef struct vf_settings {
  int voxel_type;
  float voxel_size; /* metres */
  float mu;         /* truncation band, metres */
  int max_weight;
  int stop_integrating_at_max;
  int bucket_count; /* power of two */
  int bucket_size;
  int excess_count;
  int block_count;
  float near_clip;
  float far_clip;
  int visibility_margin_px;
  int swap_margin_px;
  int hierarchy_levels; /* <= 6 */
  int rotation_only_levels;
  int max_iterations;
  int min_valid_points;
  float icp_dist_threshold;
  float convergence_eps;
  double max_condition;
  int tracking; /* 1: ICP tracker (reference behaviour); 0: known poses via vf_set_pose (config 2) */
  int use_graphs; /* 1: replay each frame as one CUDA graph */
  /* Spatial sharding (config 5): this context owns the blocks whose super-block
   * (2^shard_shift blocks per axis) hashes to shard_index mod shard_count. */
  int shard_count;
  int shard_index;
  int shard_shift;
  int shard_halo; /* 1: also fuse surfaces within one block of this shard's territory */
  /* Host swapping (EngineSettings::use_swapping / swap_buffer_blocks,
   * pipeline.hpp:20-23; swap.hpp).  The host block store is pinned host
   * memory mapped into the device, allocated in chunks of 4096 blocks as
   * blocks leave, up to swap_host_blocks slots (0 = one per hash entry, the
   * reference's bound, swap.hpp:42-56: it never fills);
   * swap_buffer_blocks <= 4096. */
  int use_swapping;
  int swap_buffer_blocks;
  int swap_host_blocks;
  float max_depth; /* disparity conversion clamp, metres (EngineSettings::max_depth, pipeline.hpp:37) */
  /* TrackerSettings::type / ren_sigma / skip_points (tracking_state.hpp:10-22) */
  int tracker_type; /* vf_tracker_type */
  float ren_sigma;
  int skip_points;
  /* TSDF integration arithmetic (no reference counterpart):
   *   VF_INTEGRATION_EXACT (0, default): the reference's FP32 operation
   *     sequence, bit-exact (integration.hpp:40-148);
   *   VF_INTEGRATION_FAST (1): the same voxels, pixels and update rule with
   *     FMA-contracted camera transform, approximate reciprocals and an FMA
   *     blend; parity bar: SDF within 1 LSB of int16 and weight exact on
   *     >= 99.9 % of voxels (SURVEY §8(c) TSDF tolerance); VoxelSRgb: colours
   *     within one count, colour weights exact. */
  int integration_mode;
  /* Pixel-sharded ICP (config 5): 1 = each shard sums the ICP
   * terms of 1/shard_count of the pixels and the per-iteration 29 sums are
   * added across shards inside the ICP kernel through peer memory (link the
   * shards with vf_shard_icp_link / vf_shard_icp_link_local); 0 = every shard
   * runs the whole ICP on the composited maps (replicated, no exchange). */
  int shard_icp;
  int icp_max_ctas; /* 0: one ICP CTA per SM (x occupancy); > 0 caps it (shards sharing a device) */
  int tracker_exact_solve; /* colour tracker: 1 = every damped LM step through the reference's pivoted
                              LDLT (color_tracker.hpp:126-128); 0 = register LDLT, pivoted fallback */
} vf_settings;

enum vf_integration_mode { VF_INTEGRATION_EXACT = 0, VF_INTEGRATION_FAST = 1 };

enum vf_tracker_type { /* TrackerType (tracking_state.hpp:10) */
  VF_TRACKER_ICP = 0,
  VF_TRACKER_COLOR = 1,  /* photometric, needs VoxelSRgb and RGB frames */
  VF_TRACKER_ICP_REN = 2 /* ICP on the coarse levels + SDF (Ren) refinement */
};

typedef struct vf_intrinsics { /* Intrinsics (core/intrinsics.hpp:10-32) */
  double fx, fy, cx, cy;
  int width, height;
} vf_intrinsics;

typedef struct vf_calib { /* Calibration (io/calibration.hpp:31-36) */
  vf_intrinsics rgb;
  vf_intrinsics depth;
  double rgb_to_depth[12];
  double disparity_a, disparity_b;
} vf_calib;

/* FrameStats (pipeline.hpp:45-58) plus device counters. */
typedef struct vf_frame_stats {
  int frame;
  int tracking_ok;
  int tracking_iterations;
  int blocks_allocated;
  int allocation_dropped;
  int visible_blocks;
  double tracking_cost;
  int tracking_valid_points;
  int allocation_requested;
  int allocated_total; /* HashVolume::allocated_block_count */
  int error_flags; /* 1 DDA steps, 2 allocated list, 4 request list, 8 host store full, 16 shard exchange
                      timeout, 32 raycast hand-off timeout */
  double pose[12];
  double ms_tracking, ms_allocation, ms_integration, ms_swapping, ms_raycast, ms_total;
  /* SwapMetrics (swap.hpp:28-40) */
  int swapped_in, swapped_out;
  uint64_t swap_bytes_in, swap_bytes_out;
} vf_frame_stats;

typedef struct vf_alloc_stats { /* AllocationStats (allocation.hpp:42-47) */
  int requested, allocated, dropped_vba_full, dropped_excess_full;
} vf_alloc_stats;

typedef struct vf_ctx vf_ctx;

/* --- lifecycle (make_pipeline, pipeline.hpp:86; src/pipeline_factory.cpp:18-30) --- */
int vf_abi_version(void);
/* sizeof of the ABI structs, for FFI layout checks: 0 vf_settings, 1 vf_calib,
 * 2 vf_frame_stats, 3 vf_alloc_stats, 4 vf_intrinsics; -1 otherwise. */
long vf_struct_size(int which);
void vf_default_settings(vf_settings* s);
int vf_create(const vf_settings* s, const vf_calib* calib, int device, vf_ctx** out);
int vf_destroy(vf_ctx* ctx);
const char* vf_last_error(const vf_ctx* ctx);

/* --- frame (IPipeline::process_frame, pipeline.hpp:70; pipeline_impl.hpp:65-123) ---
 * Host buffers; the H2D copy of depth (and rgb) and the D2H of the stats are
 * part of the call.  rgb may be NULL. */
int vf_process_frame(vf_ctx* ctx, const float* depth_m, const uint8_t* rgb, vf_frame_stats* stats);
/* Same with inputs already resident in device memory (d_depth / d_rgb are
 * device pointers).  stats may be NULL: then nothing is read back and the call
 * does not synchronise. */
int vf_process_frame_device(vf_ctx* ctx, const float* d_depth, const uint8_t* d_rgb, vf_frame_stats* stats);
/* Streaming submission (no reference counterpart; process_frame split in two):
 * vf_submit_frame enqueues the frame -- its H2D upload on a copy stream into
 * one of VF_MAX_FRAMES_IN_FLIGHT staging slots, then the frame itself -- and
 * returns without waiting, so the upload of frame n + 1 overlaps the
 * processing of frame n.  vf_collect_frame waits for the OLDEST frame in
 * flight and returns its stats (same values as vf_process_frame's).  The host
 * buffers must stay unchanged until that frame is collected.  Submitting with
 * VF_MAX_FRAMES_IN_FLIGHT frames outstanding, or collecting with none, is
 * VF_ERR_STATE.  Other calls may be interleaved; they run in submission
 * order. */
#define VF_MAX_FRAMES_IN_FLIGHT 2
int vf_submit_frame(vf_ctx* ctx, const float* depth_m, const uint8_t* rgb);
/* process_raw_frame's streaming form: the raw disparity frame (2 bytes per
 * pixel) is uploaded and decoded on the device, as in vf_process_raw_frame. */
int vf_submit_raw_frame(vf_ctx* ctx, const uint16_t* disparity, const uint8_t* rgb, int big_endian);
int vf_collect_frame(vf_ctx* ctx, vf_frame_stats* stats);
int vf_frames_in_flight(const vf_ctx* ctx);
/* IPipeline::process_raw_frame (pipeline.hpp:71, pipeline_impl.hpp:59-62):
 * a raw 16-bit disparity frame, converted on the device by
 * disparity_image_to_depth (view.hpp:18-28) with the calibration's a, b and
 * depth fx and settings.max_depth.  big_endian != 0: the buffer holds the raw
 * bytes of a 16-bit P5 raster (read_pgm16, src/pnm.cpp:63-73). */
int vf_process_raw_frame(vf_ctx* ctx, const uint16_t* disparity, const uint8_t* rgb, int big_endian,
                         vf_frame_stats* stats);
int vf_process_raw_frame_device(vf_ctx* ctx, const uint16_t* d_disparity, const uint8_t* d_rgb, int big_endian,
                                vf_frame_stats* stats);
/* disparity_image_to_depth alone (stage entry point): width*height floats out. */
int vf_disparity_to_depth(vf_ctx* ctx, const uint16_t* disparity, int big_endian, float* depth_out);
int vf_synchronize(vf_ctx* ctx);
int vf_read_stats(vf_ctx* ctx, vf_frame_stats* stats);

/* --- pose / state (IPipeline::pose, tracking_state; no reference setter: SURVEY §3(C)) --- */
int vf_set_pose(vf_ctx* ctx, const double pose[12]);
int vf_get_pose(vf_ctx* ctx, double pose[12]);
int vf_frame_count(const vf_ctx* ctx);
/* World-space point / normal maps (TrackingState::points/normals): width*height float4 each. */
int vf_get_maps(vf_ctx* ctx, float* points, float* normals);
int vf_set_maps(vf_ctx* ctx, const float* points, const float* normals, const double render_pose[12]);
/* Colour-tracker surface list (TrackingState::surface_points / surface_colors,
 * tracking_state.hpp:30-31), filled at the end of every VoxelSRgb frame by
 * forward_project_points (raycast.hpp:495-509, stride 4, pipeline_impl.hpp:218-221):
 * n x float3 world points and n x float3 colours in [0,1], raster order.
 * Returns n (points/colors may be NULL to query it); cap is in points. */
long vf_get_surface_points(vf_ctx* ctx, float* points, float* colors, long cap);
/* forward_project_points over the current maps and volume (stage entry point). */
int vf_stage_forward_project(vf_ctx* ctx);
/* IPipeline::get_image (pipeline.hpp:74, pipeline_impl.hpp:125-137) into a
 * width*height*3 u8 host buffer: DisplayMode (pipeline.hpp:60) raycast ->
 * render_image (raycast.hpp:466-490) in colour for VoxelSRgb, shaded grey
 * otherwise; VF_DISPLAY_RAYCAST_GREY forces RenderMode::shaded_grey. */
enum vf_display_mode {
  VF_DISPLAY_RAYCAST = 0,
  VF_DISPLAY_DEPTH_COLOURIZED = 1,
  VF_DISPLAY_RGB_PASSTHROUGH = 2,
  VF_DISPLAY_RAYCAST_GREY = 3
};
int vf_render_image(vf_ctx* ctx, int mode, uint8_t* out);
/* FNV-1a volume digest (IPipeline::volume_digest, pipeline_impl.hpp:144-164). */
int vf_volume_digest(vf_ctx* ctx, uint64_t* out);

/* --- state export / import (stage-isolated parity) --- */
long vf_entry_count(const vf_ctx* ctx);
long vf_voxel_bytes(const vf_ctx* ctx);
int vf_export_entries(vf_ctx* ctx, void* out /* entry_count * 16 B HashEntry */);
int vf_export_voxels(vf_ctx* ctx, void* out /* block_count * 512 * sizeof(voxel) */);
int vf_export_free_stacks(vf_ctx* ctx, int* vba_top, int* vba_slots, int* excess_top, int* excess_slots);
int vf_import_state(vf_ctx* ctx, const void* entries, const void* voxels, int vba_top, const int* vba_slots,
                    int excess_top, const int* excess_slots);
long vf_export_visible_list(vf_ctx* ctx, int* out, long cap);
long vf_export_ranges(vf_ctx* ctx, float* out /* frag_w * frag_h * 2 */);

/* --- stage entry points (the stage templates) --- */
/* mark_blocks + perform_allocations + build_visible_list (allocation.hpp:137-248) */
int vf_stage_allocate(vf_ctx* ctx, const float* depth_m, const double pose[12], vf_alloc_stats* out);
/* integrate_frame, hash overload (integration.hpp:123-148), over the current visible list */
int vf_stage_integrate(vf_ctx* ctx, const float* depth_m, const uint8_t* rgb, const double pose[12]);
/* create_expected_depths + render_maps (raycast.hpp:268-435) over the current visible list */
int vf_stage_raycast(vf_ctx* ctx, const double pose[12]);
/* build_depth_pyramid + icp_track (pyramid.hpp:101-111, depth_tracker.hpp:115-239)
 * against the current maps; the current pose is the render pose;
 * initial_pose (nullable) is icp_track's `initial` argument.  Like the
 * reference's icp_track it does not change the context's pose. */
int vf_stage_icp(vf_ctx* ctx, const float* depth_m, const double initial_pose[12], double out_pose[12],
                 int* iterations, double* cost, int* valid_points, int* ok);
/* ren_refine (ren_tracker.hpp:30-120) of depth_m against the current volume
 * from initial_pose; does not change the context's pose. */
int vf_stage_ren(vf_ctx* ctx, const float* depth_m, const double initial_pose[12], double out_pose[12],
                 int* iterations, double* cost, int* valid_points, int* ok);
/* build_color_pyramid + color_track (color_tracker.hpp:107-154) of the current
 * surface list (vf_get_surface_points) against an RGB frame (VoxelSRgb only). */
int vf_stage_color(vf_ctx* ctx, const uint8_t* rgb, const double initial_pose[12], double out_pose[12],
                   int* iterations, double* cost, int* valid_points, int* ok);
/* Per-iteration ICP sums of the last track: rows of 48 doubles
 * (level, iter, 21 H, 6 g, cost, count, rotation_only, evaluation camera-to-world
 * pose (12), 4 phase timers in SM cycles). Returns the row count. */
long vf_icp_trace(vf_ctx* ctx, double* out, long max_rows);
/* Depth pyramid levels 0..levels-1 back to back (pyramid.hpp:101-111). */
int vf_depth_pyramid(vf_ctx* ctx, const float* depth_m, float* out);

/* --- synthetic input (io/synthetic.hpp:14-51; bench inputs rendered on the GPU) --- */
/* spheres: n x {cx,cy,cz,r,ar,ag,ab}; planes: n x {nx,ny,nz,offset,ar,ag,ab,checker,checker_size}.
 * Outputs are device pointers (d_depth: w*h floats, d_rgb: w*h*3 bytes or NULL). */
int vf_render_synthetic(int device, int n_spheres, const double* spheres, int n_planes, const double* planes,
                        const double world_to_cam[12], const vf_intrinsics* intr, double near_clip,
                        double far_clip, float* d_depth, uint8_t* d_rgb);

/* --- swap engine / host block store (swap.hpp:45-253, block_store.hpp:14-53) --- */
/* Per-entry SwapState codes (swap.hpp:19-25: 0 inactive, 1 needs_swap_in,
 * 2 in_transfer, 3 active, 4 needs_swap_out) into out[entry_count]. */
int vf_swap_states(vf_ctx* ctx, uint8_t* out);
/* BlockStore::stored_count / has + read: the stored block of entry `entry` in
 * the VoxelCodec layout (voxel.hpp:93-189; 512 x 3 B VoxelS, 512 x 7 B
 * VoxelSRgb).  Returns 1 and fills payload (may be NULL) if stored, else 0. */
long vf_swap_stored_count(vf_ctx* ctx);
int vf_swap_store_read(vf_ctx* ctx, int entry, uint8_t* payload);
/* Write every stored block to a VXBS file (make_file_block_store /
 * load_block_store_file format, block_store.hpp:14-53): 16-byte header then
 * (u32 entry index, payload) records, ascending entry order. */
/* The entries swapped out since the last drain, in swap-out order (the order
 * the reference's file-backed BlockStore writes its records, block_store.cpp:
 * 96-115): up to cap of them into entries; returns the count.  Waits for the
 * frames in flight.  *lost (optional) counts entries that fell out of the
 * 65536-entry ring between drains.  The adapter drains after every frame
 * and writes the VXBS records of swap_store_path as blocks leave. */
long vf_swap_drain(vf_ctx* ctx, int* entries, long cap, long* lost);
int vf_swap_save_store(vf_ctx* ctx, const char* path);
/* Load a VXBS file into the host store (load_block_store_file): records for
 * entries that are swapped out in the current table become their host data. */
int vf_swap_load_store(vf_ctx* ctx, const char* path);

/* --- spatial sharding ---
 * Owner shard of a block position (the device rule, for hosts and tests). */
/* Pixel-sharded ICP links.  One process per GPU: every rank publishes
 * vf_shard_icp_handle (a 64-byte CUDA IPC handle of its exchange area), the
 * handles are gathered in rank order, and each rank calls vf_shard_icp_link
 * with all of them.  Shards sharing one device in one process:
 * vf_shard_icp_link_local with the contexts in shard order.  Either replaces
 * the frame graphs; afterwards the shards' frames must run concurrently
 * (each ICP iteration waits for every shard's sums; ~0.5 s without them
 * fails the frame's tracking instead of hanging). */
/* The per-frame nearest-depth composite over peer memory instead of NCCL
 * (one kernel reads the other shards' keys and winning map entries over
 * NVLink; flags instead of collectives).  One process per GPU: gather every
 * rank's vf_shard_p2p_handles (4 CUDA IPC handles, 256 bytes) in rank order
 * and call vf_shard_p2p_link with all of them; shards sharing a device in one
 * process: vf_shard_p2p_link_local.  Mutually exclusive with the NCCL
 * attach; the shards' frames must then run concurrently. */
int vf_shard_p2p_handles(vf_ctx* ctx, void* out /* 4 x 64 bytes */);
int vf_shard_p2p_link(vf_ctx* ctx, const void* handles /* count x 256 bytes */, int count);
int vf_shard_p2p_link_local(vf_ctx** ctxs, int count);
int vf_shard_icp_handle(vf_ctx* ctx, void* handle_out /* 64 bytes */);
int vf_shard_icp_link(vf_ctx* ctx, const void* handles /* count x 64 bytes */, int count);
int vf_shard_icp_link_local(vf_ctx** ctxs, int count);
int vf_shard_owner(int bx, int by, int bz, int shard_shift, int shard_count);
/* One process per GPU: rank 0 creates an NCCL unique id (128 bytes), every
 * rank attaches with it; each frame then ends with the nearest-depth map
 * composite (all-reduce MIN of depth keys, masked all-reduce SUM of the maps)
 * inside the frame graph, and the replicated ICP needs no collective. */
int vf_shard_nccl_unique_id(void* out128);
int vf_shard_attach_nccl(vf_ctx* ctx, const void* unique_id128, int nranks, int rank);
/* Several shards in one process on the same device (tests, single-GPU
 * boxes): composite the n contexts' maps after each frame. */
int vf_shard_composite_local(vf_ctx** ctxs, int n);

/* --- device memory helpers for callers without a CUDA runtime of their own --- */
void* vf_device_alloc(size_t bytes);
int vf_device_free(void* p);
int vf_memcpy_h2d(void* dst, const void* src, size_t bytes);
int vf_memcpy_d2h(void* dst, const void* src, size_t bytes);
void* vf_host_alloc_pinned(size_t bytes);
int vf_host_free_pinned(void* p);

/* --- timing: CUDA events on the context's stream --- */
int vf_event_record(vf_ctx* ctx, int slot);
int vf_event_elapsed_ms(vf_ctx* ctx, int slot_a, int slot_b, float* ms);
/* per-kernel profiling: when enabled, each stage is bracketed by events and
 * vf_stage_times returns accumulated milliseconds per stage. */
int vf_set_profiling(vf_ctx* ctx, int enabled);
int vf_stage_times(vf_ctx* ctx, double* ms_out /* 8 */, long* frames);
/* FrameStats::ms_* per frame (pipeline.hpp:56-57; the reference fills them on
 * every frame, pipeline_impl.hpp:66-120): when enabled, the blocking calls
 * (vf_process_frame / _device / vf_process_raw_frame) return the stage times
 * of that frame in vf_frame_stats.ms_tracking .. ms_raycast, from event
 * records inside the frame graph (no extra launches, no serialisation; the
 * side branch -- range image and swap engine -- overlaps integration, so
 * ms_swapping is the wait for it).  The streaming pair returns ms_total only.
 * Off by default in the C ABI; the IPipeline adapter turns it on. */
int vf_set_stage_timing(vf_ctx* ctx, int enabled);
/* Measurement only (not on the frame path): re-runs the last frame's raycast
 * (render_maps, raycast.hpp:415-435) with counters -- identical maps -- and
 * returns {hash-table probes (block-cache misses), voxel reads (each one
 * hash probe in the reference's HashSdfSampler::read, raycast.hpp:73-76),
 * rays marched, rays hit}. */
int vf_raycast_counters(vf_ctx* ctx, unsigned long long* out /* 4 */);
/* Measurement only: mark_blocks' walk (allocation.hpp:137-168) over the last
 * frame's depth and pose, without requests: {pixels with depth, DDA cells
 * probed (one hash-bucket read each), cells still missing from the table
 * (after the frame: blocks whose bucket already took this frame's one
 * request, allocation.hpp:155-159, and dropped requests)}. */
int vf_alloc_counters(vf_ctx* ctx, unsigned long long* out /* 3 */);
int vf_kernel_launches_per_frame(vf_ctx* ctx, int tracking_frame);
/* Bytes of the per-frame stats readback (the D2H of vf_process_frame). */
long vf_readback_bytes(const vf_ctx* ctx);
/* Evict the L2 by writing `bytes` of scratch on the context's stream (bench hygiene). */
int vf_flush_l2(vf_ctx* ctx, size_t bytes);
/* Sum of the device-timed durations of the vf_flush_l2 calls since the last
 * call (synchronises the stream), so a streaming measurement can flush L2
 * between frames in-stream and take the flushes out of its wall time. */
int vf_flush_time(vf_ctx* ctx, double* ms);
/* Self-test of the branch-free IEEE division used by integration against the
 * IEEE operator; returns the mismatch count.  mode 0: divisor p0, a = 0 and
 * every numerator with p2 <= |a| <= p1; mode 1: n random pairs, |a| <= p0,
 * p1 <= |b| <= p2. */
long vf_selftest_division(int device, int mode, float p0, float p1, float p2, long n);
/* Voxels whose state the last frame's integration changed (roofline accounting). */
long vf_last_modified_voxels(vf_ctx* ctx);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* VOXFUSE_B200_H */
