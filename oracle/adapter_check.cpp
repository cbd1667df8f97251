// TEST INFRASTRUCTURE ONLY — the drop-in check.
//
// Compiled with the UNMODIFIED reference sources (via oracle/eigen_shim) and
// linked against the product library: runs the same frames through
//   voxfuse::make_pipeline(...)              (the reference CPU engine)
//   voxfuse_b200::make_b200_pipeline(...)    (paper_1410_0925_b200/cpp/b200_pipeline.hpp)
// both used only through the reference's IPipeline interface, and returns
// poses, stats, FNV volume digests and maps for tests/test_gpu_adapter.py.
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "b200_pipeline.hpp"
#include "voxfuse/core/parallel.hpp"
#include "voxfuse/engine/pipeline.hpp"

using namespace voxfuse;

extern "C" {

// FrameStats::ms_* of the last frame vfa_run processed through
// IPipeline::process_frame (tracking, allocation, integration, swapping,
// raycast, total; pipeline.hpp:56-57)
static double g_last_ms[6];
void vfa_last_stage_ms(double* out) { std::memcpy(out, g_last_ms, sizeof(g_last_ms)); }

// EngineSettings::swap_store_path for the next vfa_run (empty: in-memory store)
static std::string g_store_path;
void vfa_set_store_path(const char* path) { g_store_path = path ? path : ""; }

struct vfa_config {  // same layout as vfr_config (oracle/ref_driver.cpp)
  int voxel_type;
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
  int use_swapping, swap_buffer_blocks;
  int tracker_type;
  float ren_sigma;
  int skip_points;
};

// Runs n frames through IPipeline.  engine: 0 = reference make_pipeline,
// 1 = make_b200_pipeline, 2 = make_b200_pipeline driven through its streaming
// extension (submit_frame / collect_frame, two frames in flight).  Outputs per frame: pose (12), iterations, ok,
// visible blocks, allocated; final FNV digest and maps.
int vfa_run(const vfa_config* c, int engine, int n_frames, const float* depth, const std::uint8_t* rgb,
            double* poses, int* iters, int* ok, int* visible, std::uint64_t* digest, float* points,
            float* normals, std::uint8_t* image, std::uint8_t* image_depth) {
  try {
    EngineSettings s;
    s.backend = VolumeBackend::hash;
    s.voxel_type = c->voxel_type == 2 ? VoxelType::s_rgb : VoxelType::s;
    s.scene.voxel_size = c->voxel_size;
    s.scene.mu = c->mu;
    s.scene.max_weight = c->max_weight;
    s.hash.bucket_count = c->bucket_count;
    s.hash.bucket_size = c->bucket_size;
    s.hash.excess_count = c->excess_count;
    s.hash.block_count = c->block_count;
    s.near_clip = c->near_clip;
    s.far_clip = c->far_clip;
    s.visibility_margin_px = c->margin_px;
    s.swap_margin_px = c->swap_margin_px;
    s.tracker.hierarchy_levels = c->levels;
    s.tracker.rotation_only_levels = c->rotation_only_levels;
    s.tracker.max_iterations = c->max_iterations;
    s.tracker.min_valid_points = c->min_valid_points;
    s.tracker.icp_dist_threshold = c->icp_dist_threshold;
    s.tracker.convergence_eps = c->convergence_eps;
    s.tracker.max_condition = c->max_condition;
    s.tracker.type = c->tracker_type == 1 ? TrackerType::color : c->tracker_type == 2 ? TrackerType::icp_ren
                                                                                      : TrackerType::icp;
    s.tracker.ren_sigma = c->ren_sigma;
    s.use_swapping = c->use_swapping != 0;
    s.swap_buffer_blocks = c->swap_buffer_blocks;
    s.swap_store_path = g_store_path;
    Calibration k;
    k.depth.fx = c->fx;
    k.depth.fy = c->fy;
    k.depth.cx = c->cx;
    k.depth.cy = c->cy;
    k.depth.width = c->width;
    k.depth.height = c->height;
    k.rgb = k.depth;
    std::unique_ptr<IPipeline> p =
        engine >= 1 ? voxfuse_b200::make_b200_pipeline(s, k) : make_pipeline(s, k);
    const std::size_t npix = static_cast<std::size_t>(c->width) * c->height;
    if (engine == 2) {
      auto* b = dynamic_cast<voxfuse_b200::B200Pipeline*>(p.get());
      if (!b) return -1;
      std::vector<Image2D<float>> d(n_frames);
      int next = 0;
      auto collect = [&]() {
        const FrameStats st = b->collect_frame();
        const int f = st.frame;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) poses[f * 12 + i * 3 + j] = st.pose.rotation()(i, j);
        for (int i = 0; i < 3; ++i) poses[f * 12 + 9 + i] = st.pose.translation()(i);
        iters[f] = st.tracking_iterations;
        ok[f] = st.tracking_ok ? 1 : 0;
        visible[f] = st.visible_blocks;
      };
      for (; next < n_frames; ++next) {
        d[next] = Image2D<float>(c->width, c->height, 0.0f);
        std::memcpy(d[next].pixels().data(), depth + next * npix, sizeof(float) * npix);
        b->submit_frame(nullptr, d[next]);
        if (b->frames_in_flight() == VF_MAX_FRAMES_IN_FLIGHT) collect();
      }
      while (b->frames_in_flight() > 0) collect();
      n_frames = 0;  // frames done; fall through to the outputs
    }
    for (int f = 0; f < n_frames; ++f) {
      Image2D<float> d(c->width, c->height, 0.0f);
      std::memcpy(d.pixels().data(), depth + f * npix, sizeof(float) * npix);
      Image2D<Vec3u8> col;
      if (rgb) {
        col = Image2D<Vec3u8>(c->width, c->height, Vec3u8::Zero());
        std::memcpy(col.pixels().data(), rgb + f * npix * 3, npix * 3);
      }
      const FrameStats st = p->process_frame(rgb ? &col : nullptr, d);
      const double ms[6] = {st.ms_tracking, st.ms_allocation, st.ms_integration,
                            st.ms_swapping, st.ms_raycast, st.ms_total};
      std::memcpy(g_last_ms, ms, sizeof(ms));
      const Pose& pose = p->pose();
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) poses[f * 12 + i * 3 + j] = pose.rotation()(i, j);
      for (int i = 0; i < 3; ++i) poses[f * 12 + 9 + i] = pose.translation()(i);
      iters[f] = st.tracking_iterations;
      ok[f] = st.tracking_ok ? 1 : 0;
      visible[f] = st.visible_blocks;
    }
    *digest = p->volume_digest();
    const TrackingState& ts = p->tracking_state();
    std::memcpy(points, ts.points.pixels().data(), sizeof(float) * 4 * npix);
    std::memcpy(normals, ts.normals.pixels().data(), sizeof(float) * 4 * npix);
    // get_image (pipeline_impl.hpp:125-137): raycast render and colourised depth
    const Image2D<Vec3u8> img = p->get_image(DisplayMode::raycast);
    const Image2D<Vec3u8> dimg = p->get_image(DisplayMode::depth_colourized);
    for (std::size_t i = 0; i < npix; ++i)
      for (int ch = 0; ch < 3; ++ch) {
        if (image) image[3 * i + ch] = img.empty() ? 0 : img.pixels()[i](ch);
        if (image_depth) image_depth[3 * i + ch] = dimg.empty() ? 0 : dimg.pixels()[i](ch);
      }
    return p->frame_count();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "vfa_run: %s\n", e.what());
    return -1;
  }
}

void vfa_set_threads(int n) { set_worker_count(n); }

}  // extern "C"
