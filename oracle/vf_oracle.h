/* TEST INFRASTRUCTURE ONLY — the CPU parity oracle.
 *
 * A plain-C restatement of the reference's per-frame dense-fusion path
 * (/root/reference/proj, "voxfuse", the CPU re-implementation of InfiniTAM,
 * arXiv 1410.0925).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference legs may load it; the product library never does.
 *
 * Pinning: tests/test_oracle_vs_ref.py checks this restatement bit-for-bit
 * against the reference's own sources compiled unmodified (oracle/_ref, via
 * oracle/eigen_shim) and tests/golden/ holds fixtures generated from that
 * build.  Arithmetic contract: IEEE binary32/binary64, strict left-to-right
 * reductions, no FMA contraction (-ffp-contract=off).
 */
#ifndef VF_ORACLE_H
#define VF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same field layout as oracle/ref_driver.cpp's vfr_config (ctypes shares one
 * mirror for both). */
typedef struct vfo_config {
  int voxel_type; /* 1 = VoxelS, 2 = VoxelSRgb */
  float voxel_size, mu;
  int max_weight, stop_integrating_at_max;
  int bucket_count, bucket_size, excess_count, block_count;
  float near_clip, far_clip;
  int margin_px, swap_margin_px;
  int levels, rotation_only_levels, max_iterations, min_valid_points;
  float icp_dist_threshold, convergence_eps;
  double max_condition;
  double fx, fy, cx, cy;
  int width, height;
  double rgb_fx, rgb_fy, rgb_cx, rgb_cy;
  int rgb_width, rgb_height;
  double rgb_to_depth[12];
  /* EngineSettings::use_swapping / swap_buffer_blocks (pipeline.hpp:20-23) */
  int use_swapping, swap_buffer_blocks;
  /* TrackerSettings::type / ren_sigma / skip_points (the restatement covers the ICP tracker only) */
  int tracker_type;
  float ren_sigma;
  int skip_points;
} vfo_config;

typedef struct vfo_stats {
  int frame, tracking_ok, tracking_iterations, blocks_allocated, allocation_dropped, visible_blocks;
  double tracking_cost;
  double pose[12];
  double ms_tracking, ms_allocation, ms_integration, ms_raycast, ms_total;
  /* SwapMetrics (swap.hpp:28-40), accumulated over swap-in and swap-out */
  int swapped_in, swapped_out;
  uint64_t bytes_in, bytes_out;
  double ms_swapping;
} vfo_stats;

typedef struct vfo_alloc_stats {
  int requested, allocated, dropped_vba_full, dropped_excess_full;
} vfo_alloc_stats;

typedef struct vfo_ctx vfo_ctx;

vfo_ctx* vfo_create(const vfo_config* cfg, int tracking);
void vfo_destroy(vfo_ctx* c);
/* One frame.  tracking != 0: IPipeline::process_frame semantics
 * (pipeline_impl.hpp:65-123).  tracking == 0: `pose` (row-major R, t) is the
 * known world->camera pose and the stages run in pipeline order. */
int vfo_process(vfo_ctx* c, const float* depth, const uint8_t* rgb, const double* pose, vfo_stats* st);

/* Stage entry points (stage-isolated parity). */
int vfo_stage_allocate(vfo_ctx* c, const float* depth, const double* pose, vfo_alloc_stats* out);
int vfo_stage_integrate(vfo_ctx* c, const float* depth, const uint8_t* rgb, const double* pose);
int vfo_stage_raycast(vfo_ctx* c, const double* pose);
int vfo_stage_icp(vfo_ctx* c, const float* depth, double* out_pose, int* out_iters, double* out_cost,
                  int* out_valid);
/* icp_track(pyramid, state, settings, initial) with an explicit initial pose (depth_tracker.hpp:115-118) */
int vfo_stage_icp_init(vfo_ctx* c, const float* depth, const double* initial, double* out_pose, int* out_iters,
                       double* out_cost, int* out_valid);

void vfo_get_pose(const vfo_ctx* c, double* out);
void vfo_set_pose(vfo_ctx* c, const double* pose);
int vfo_get_maps(const vfo_ctx* c, float* points, float* normals);
int vfo_set_maps(vfo_ctx* c, const float* points, const float* normals, const double* render_pose);
long vfo_export_entries(const vfo_ctx* c, void* out);
long vfo_export_voxels(const vfo_ctx* c, void* out);
long vfo_visible_list(const vfo_ctx* c, int* out);
long vfo_export_ranges(const vfo_ctx* c, float* out);
long vfo_allocated_blocks(const vfo_ctx* c);
/* free-stack state: tops and slot arrays (hash_volume.hpp:62-110) */
void vfo_free_stacks(const vfo_ctx* c, int* vba_top, int* vba_slots, int* excess_top, int* excess_slots);
uint64_t vfo_digest(const vfo_ctx* c);
/* raycast counters of the last render: rays, samples, voxel reads, trilinear calls, coarse samples */
long vfo_raycast_counters(long* out);
/* last ICP solve trace: rows of 48 doubles (level, iter, 21 H, 6 g, cost, count,
 * rotation_only, evaluation camera-to-world pose (12), 4 unused) */
long vfo_icp_trace(const vfo_ctx* c, double* out, long max_rows);
/* raycast epilogues (raycast.hpp:441-509): surface list of the last render
 * (n x float3 points, n x float3 colours; returns n), forward_project_points
 * over the current maps, render_image (color 0: shaded grey, 1: colour). */
long vfo_surface_points(const vfo_ctx* c, float* points, float* colors);
int vfo_stage_forward_project(vfo_ctx* c);
int vfo_render_image(vfo_ctx* c, int color, uint8_t* out);
void vfo_colourize_depth(const float* depth, int w, int h, uint8_t* out);
/* disparity_image_to_depth (view.hpp:18-28, calibration.hpp:45-60) */
void vfo_disparity_to_depth(const uint16_t* disp, long n, double a, double b, double fx, float max_depth,
                            float* depth);
/* swap engine (swap.hpp:14-253): per-entry SwapState codes (inactive 0,
 * needs_swap_in 1, in_transfer 2, active 3, needs_swap_out 4); host store
 * contents in the VoxelCodec layout (voxel.hpp:93-189, 3 / 7 bytes per voxel):
 * vfo_store_read returns 1 and fills payload when entry idx holds data. */
long vfo_swap_states(const vfo_ctx* c, uint8_t* out);
int vfo_store_read(const vfo_ctx* c, int idx, uint8_t* payload);
long vfo_store_count(const vfo_ctx* c);

/* Free functions. */
uint32_t vfo_hash_block_pos(int x, int y, int z, uint32_t mask);
void vfo_depth_pyramid(const float* depth, int w, int h, int levels, float* out);
void vfo_render_depth(int n_spheres, const double* spheres, int n_planes, const double* planes,
                      const double* world_to_cam, double fx, double fy, double cx, double cy, int w,
                      int h, double near_clip, double far_clip, float* out);
void vfo_render_rgb(int n_spheres, const double* spheres, int n_planes, const double* planes,
                    const double* world_to_cam, double fx, double fy, double cx, double cy, int w,
                    int h, double near_clip, double far_clip, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
