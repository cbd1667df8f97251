// TEST / BASELINE INFRASTRUCTURE ONLY — compiled together with the UNMODIFIED
// reference sources (/root/reference/proj) into oracle/_ref/libvoxfuse_ref.so
// by oracle/Makefile.  Never linked into the product.
//
// It exposes a small C ABI (vfr_*) over the reference's own public API so
// the parity tests and bench.py's reference arm can drive it through ctypes:
//   * tracking mode: make_pipeline() + IPipeline::process_frame
//     (proj/include/voxfuse/engine/pipeline.hpp:66-86, pipeline_impl.hpp:65-123)
//   * known-pose mode (config 2): the stage templates in pipeline order,
//     because IPipeline cannot set a pose:
//     mark_blocks → perform_allocations → build_visible_list → integrate_frame
//     → create_expected_depths → render_maps.
//   * stage entry points for stage-isolated parity: icp_track on given maps,
//     render_synthetic_depth / render_synthetic_rgb (proj/src/synthetic.cpp).
#include <cstdint>
#include <cstring>
#include <fstream>
#include <memory>
#include <optional>
#include <vector>

#include "voxfuse/core/parallel.hpp"
#include "voxfuse/engine/pipeline.hpp"
#include "voxfuse/engine/pipeline_impl.hpp"
#include "voxfuse/io/calibration.hpp"
#include "voxfuse/io/pnm.hpp"
#include "voxfuse/io/synthetic.hpp"

using namespace voxfuse;

extern "C" {

// Keep in sync with oracle/vf_ref.py (ctypes mirror).
struct vfr_config {
  int voxel_type;  // 1 = VoxelS, 2 = VoxelSRgb
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
  double rgb_to_depth[12];  // row-major R (9) then t (3)
  int use_swapping, swap_buffer_blocks;
  int tracker_type;  // TrackerType: 0 icp, 1 color, 2 icp_ren
  float ren_sigma;
  int skip_points;
};

struct vfr_stats {
  int frame, tracking_ok, tracking_iterations, blocks_allocated, allocation_dropped, visible_blocks;
  double tracking_cost;
  double pose[12];
  double ms_tracking, ms_allocation, ms_integration, ms_raycast, ms_total;
  int swapped_in, swapped_out;
  std::uint64_t bytes_in, bytes_out;
  double ms_swapping;
};

}  // extern "C"

namespace {

Pose pose_from(const double* p) {
  Mat3d r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = p[i * 3 + j];
  return Pose(r, Vec3d(p[9], p[10], p[11]));
}
void pose_to(const Pose& pose, double* p) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) p[i * 3 + j] = pose.rotation()(i, j);
  for (int i = 0; i < 3; ++i) p[9 + i] = pose.translation()(i);
}

EngineSettings settings_from(const vfr_config& c) {
  EngineSettings s;
  s.backend = VolumeBackend::hash;
  s.voxel_type = c.voxel_type == 2 ? VoxelType::s_rgb : VoxelType::s;
  s.scene.voxel_size = c.voxel_size;
  s.scene.mu = c.mu;
  s.scene.max_weight = c.max_weight;
  s.scene.stop_integrating_at_max = c.stop_integrating_at_max != 0;
  s.hash.bucket_count = c.bucket_count;
  s.hash.bucket_size = c.bucket_size;
  s.hash.excess_count = c.excess_count;
  s.hash.block_count = c.block_count;
  s.near_clip = c.near_clip;
  s.far_clip = c.far_clip;
  s.visibility_margin_px = c.margin_px;
  s.swap_margin_px = c.swap_margin_px;
  s.tracker.hierarchy_levels = c.levels;
  s.tracker.rotation_only_levels = c.rotation_only_levels;
  s.tracker.max_iterations = c.max_iterations;
  s.tracker.min_valid_points = c.min_valid_points;
  s.tracker.icp_dist_threshold = c.icp_dist_threshold;
  s.tracker.convergence_eps = c.convergence_eps;
  s.tracker.max_condition = c.max_condition;
  s.tracker.type = c.tracker_type == 1 ? TrackerType::color : c.tracker_type == 2 ? TrackerType::icp_ren
                                                                                  : TrackerType::icp;
  s.tracker.ren_sigma = c.ren_sigma;
  s.tracker.skip_points = c.skip_points != 0;
  s.use_swapping = c.use_swapping != 0;
  s.swap_buffer_blocks = c.swap_buffer_blocks;
  return s;
}

Calibration calib_from(const vfr_config& c) {
  Calibration k;
  k.depth.fx = c.fx;
  k.depth.fy = c.fy;
  k.depth.cx = c.cx;
  k.depth.cy = c.cy;
  k.depth.width = c.width;
  k.depth.height = c.height;
  k.rgb.fx = c.rgb_fx;
  k.rgb.fy = c.rgb_fy;
  k.rgb.cx = c.rgb_cx;
  k.rgb.cy = c.rgb_cy;
  k.rgb.width = c.rgb_width;
  k.rgb.height = c.rgb_height;
  k.rgb_to_depth = pose_from(c.rgb_to_depth);
  return k;
}

struct CtxBase {
  virtual ~CtxBase() = default;
  virtual int process(const float* depth, const std::uint8_t* rgb, const double* pose, vfr_stats* st) = 0;
  virtual Pose pose() const = 0;
  virtual const TrackingState& state() const = 0;
  virtual long export_entries(void* out) const = 0;
  virtual long export_voxels(void* out) const = 0;
  virtual long visible_list(int* out) const = 0;
  virtual std::uint64_t digest() const = 0;
  virtual long allocated_blocks() const = 0;
  virtual long export_ranges(float* out) const { (void)out; return -1; }
  // get_image (pipeline_impl.hpp:125-137) / render_image (raycast.hpp:466-490)
  virtual int image(int mode, std::uint8_t* out) const = 0;
  // swap engine state (swap.hpp:45-91); nullptr without swapping
  virtual const void* cache_ptr() const { return nullptr; }
  // ren_refine / color_track on this context's volume and surface list
  virtual TrackingResult stage_ren(const float*, const Pose&) const { return {}; }
  virtual TrackingResult stage_color(const std::uint8_t*, const Pose&) const { return {}; }
  virtual int voxel_type() const = 0;
};

void fill_swap(const SwapMetrics& m, vfr_stats* st) {
  st->swapped_in = m.swapped_in;
  st->swapped_out = m.swapped_out;
  st->bytes_in = m.bytes_in;
  st->bytes_out = m.bytes_out;
}

void copy_image(const Image2D<Vec3u8>& img, std::uint8_t* out) {
  for (std::size_t i = 0; i < img.size(); ++i)
    for (int c = 0; c < 3; ++c) out[3 * i + c] = img.pixels()[i](c);
}

Image2D<float> depth_image(const float* d, int w, int h) {
  Image2D<float> img(w, h, 0.0f);
  std::memcpy(img.pixels().data(), d, sizeof(float) * static_cast<std::size_t>(w) * h);
  return img;
}
Image2D<Vec3u8> rgb_image(const std::uint8_t* p, int w, int h) {
  Image2D<Vec3u8> img(w, h, Vec3u8::Zero());
  for (std::size_t i = 0; i < img.size(); ++i) img.pixels()[i] = Vec3u8(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
  return img;
}

template <typename TVoxel>
long export_volume_entries(const HashVolume<TVoxel>& v, void* out) {
  static_assert(sizeof(HashEntry) == 16, "HashEntry must be 16 B");
  if (out) std::memcpy(out, &v.entry(0), sizeof(HashEntry) * static_cast<std::size_t>(v.entry_count()));
  return v.entry_count();
}
template <typename TVoxel>
long export_volume_voxels(const HashVolume<TVoxel>& v, void* out) {
  const std::size_t n = static_cast<std::size_t>(v.config().block_count) * kBlockVolume;
  if (out) std::memcpy(out, v.block(0), sizeof(TVoxel) * n);
  return static_cast<long>(n * sizeof(TVoxel));
}

// Tracking mode: the reference's own IPipeline.
template <typename TVoxel>
struct PipelineCtx final : CtxBase {
  Pipeline<TVoxel, VolumeBackend::hash> p;
  vfr_config cfg;
  PipelineCtx(const vfr_config& c) : p(settings_from(c), calib_from(c)), cfg(c) {}
  int process(const float* depth, const std::uint8_t* rgb, const double*, vfr_stats* st) override {
    const Image2D<float> d = depth_image(depth, cfg.width, cfg.height);
    FrameStats fs;
    if (rgb) {
      const Image2D<Vec3u8> c = rgb_image(rgb, cfg.rgb_width, cfg.rgb_height);
      fs = p.process_frame(&c, d);
    } else {
      fs = p.process_frame(nullptr, d);
    }
    if (st) {
      st->frame = fs.frame;
      st->tracking_ok = fs.tracking_ok;
      st->tracking_iterations = fs.tracking_iterations;
      st->tracking_cost = fs.tracking_cost;
      st->blocks_allocated = fs.blocks_allocated;
      st->allocation_dropped = fs.allocation_dropped;
      st->visible_blocks = fs.visible_blocks;
      pose_to(fs.pose, st->pose);
      st->ms_tracking = fs.ms_tracking;
      st->ms_allocation = fs.ms_allocation;
      st->ms_integration = fs.ms_integration;
      st->ms_raycast = fs.ms_raycast;
      st->ms_total = fs.ms_total;
      st->ms_swapping = fs.ms_swapping;
      fill_swap(fs.swap, st);
    }
    return 0;
  }
  const void* cache_ptr() const override { return const_cast<Pipeline<TVoxel, VolumeBackend::hash>&>(p).cache(); }
  int voxel_type() const override { return TVoxel::has_color ? 2 : 1; }
  Pose pose() const override { return p.pose(); }
  const TrackingState& state() const override { return p.tracking_state(); }
  long export_entries(void* out) const override { return export_volume_entries(p.volume(), out); }
  long export_voxels(void* out) const override { return export_volume_voxels(p.volume(), out); }
  long visible_list(int* out) const override {
    const auto& vl = p.scratch().visible_list;
    if (out) std::memcpy(out, vl.data(), sizeof(int) * vl.size());
    return static_cast<long>(vl.size());
  }
  std::uint64_t digest() const override { return p.volume_digest(); }
  long allocated_blocks() const override { return p.volume().allocated_block_count(); }
  int image(int mode, std::uint8_t* out) const override {
    // mode: DisplayMode (pipeline.hpp:60); 3 = render_image in shaded grey
    Image2D<Vec3u8> img;
    if (mode == 3) {
      const TrackingState& s = p.tracking_state();
      if (!s.maps_valid) return -1;
      img = render_image(p.volume(), s.points, s.normals, s.pose, p.settings().scene, RenderMode::shaded_grey);
    } else {
      img = p.get_image(static_cast<DisplayMode>(mode));
    }
    if (img.empty()) return -1;
    copy_image(img, out);
    return 0;
  }
};

// Known-pose mode: stage templates in pipeline order (pipeline_impl.hpp:88-117).
template <typename TVoxel>
struct StagesCtx final : CtxBase {
  EngineSettings s;
  Calibration calib;
  HashVolume<TVoxel> volume;
  AllocationScratch scratch;
  TrackingState st;
  RangeImage range;
  vfr_config cfg;
  std::optional<GlobalCache<TVoxel>> cache;
  int frame = 0;
  StagesCtx(const vfr_config& c) : s(settings_from(c)), calib(calib_from(c)), volume(s.hash), cfg(c) {
    scratch.reset(volume.entry_count());
    if (s.use_swapping)  // pipeline_impl.hpp:42-51 (in-memory store)
      cache.emplace(GlobalCache<TVoxel>::in_memory(volume.entry_count(), s.swap_buffer_blocks));
  }
  const void* cache_ptr() const override { return cache ? &*cache : nullptr; }
  TrackingResult stage_ren(const float* depth, const Pose& init) const override {
    return ren_refine(depth_image(depth, cfg.width, cfg.height), calib.depth, volume, s.scene, init, s.tracker);
  }
  TrackingResult stage_color(const std::uint8_t* rgb, const Pose& init) const override {
    const ColorPyramid pyr =
        build_color_pyramid(rgb_image(rgb, cfg.rgb_width, cfg.rgb_height), calib.rgb, s.tracker.hierarchy_levels);
    return color_track(st.surface_points, st.surface_colors, pyr, init, s.tracker);
  }
  int voxel_type() const override { return TVoxel::has_color ? 2 : 1; }
  int process(const float* depth, const std::uint8_t* rgb, const double* pose, vfr_stats* out) override {
    if (!pose) return -1;
    using clk = std::chrono::steady_clock;
    const auto t_start = clk::now();
    View view;
    view.calib = calib;
    view.depth = depth_image(depth, cfg.width, cfg.height);
    if (rgb) view.rgb = rgb_image(rgb, cfg.rgb_width, cfg.rgb_height);
    st.pose = pose_from(pose);
    auto t0 = clk::now();
    mark_blocks(view.depth, st.pose, calib.depth, s.scene, volume, scratch);
    const AllocationStats alloc = perform_allocations(scratch, volume);
    build_visible_list(volume, st.pose, calib.depth, s.scene, s.frustum(), scratch);
    const double ms_alloc = detail::ms_since(t0);
    t0 = clk::now();
    integrate_frame(volume, scratch.visible_list, view, st.pose, s.scene);
    const double ms_int = detail::ms_since(t0);
    t0 = clk::now();
    SwapMetrics swap;
    if (cache) {  // pipeline_impl.hpp:104-113
      request_swap_ins(volume, scratch, *cache);
      swap.accumulate(execute_swap_in(volume, *cache, s.scene));
      request_swap_outs(volume, scratch, *cache);
      swap.accumulate(execute_swap_out(volume, *cache));
    }
    const double ms_swap = detail::ms_since(t0);
    t0 = clk::now();
    range = create_expected_depths(volume, scratch.visible_list, st.pose, calib.depth, s.scene,
                                   s.near_clip, s.far_clip);
    render_maps(volume, range, st.pose, calib.depth, s.scene, st.points, st.normals);
    st.maps_valid = true;
    if constexpr (TVoxel::has_color) {  // pipeline_impl.hpp:218-221
      forward_project_points(volume, st.points, s.scene, 4, st.surface_points, st.surface_colors);
    }
    const double ms_ray = detail::ms_since(t0);
    if (out) {
      out->frame = frame;
      out->tracking_ok = 1;
      out->tracking_iterations = 0;
      out->tracking_cost = 0;
      out->blocks_allocated = alloc.allocated;
      out->allocation_dropped = alloc.dropped_vba_full + alloc.dropped_excess_full;
      out->visible_blocks = static_cast<int>(scratch.visible_list.size());
      pose_to(st.pose, out->pose);
      out->ms_tracking = 0;
      out->ms_allocation = ms_alloc;
      out->ms_integration = ms_int;
      out->ms_raycast = ms_ray;
      out->ms_swapping = ms_swap;
      fill_swap(swap, out);
      out->ms_total = detail::ms_since(t_start);
    }
    ++frame;
    return 0;
  }
  Pose pose() const override { return st.pose; }
  const TrackingState& state() const override { return st; }
  long export_entries(void* out) const override { return export_volume_entries(volume, out); }
  long export_voxels(void* out) const override { return export_volume_voxels(volume, out); }
  long visible_list(int* out) const override {
    if (out) std::memcpy(out, scratch.visible_list.data(), sizeof(int) * scratch.visible_list.size());
    return static_cast<long>(scratch.visible_list.size());
  }
  std::uint64_t digest() const override { return 0; }
  long allocated_blocks() const override { return volume.allocated_block_count(); }
  int image(int mode, std::uint8_t* out) const override {
    if (!st.maps_valid || (mode != 0 && mode != 3)) return -1;
    const RenderMode rm = (mode == 0 && TVoxel::has_color) ? RenderMode::color : RenderMode::shaded_grey;
    copy_image(render_image(volume, st.points, st.normals, st.pose, s.scene, rm), out);
    return 0;
  }
  long export_ranges(float* out) const override {
    const long n = static_cast<long>(range.fragments_x()) * range.fragments_y();
    if (out) {
      for (int fy = 0; fy < range.fragments_y(); ++fy)
        for (int fx = 0; fx < range.fragments_x(); ++fx) {
          const Vec2f& r = range.fragment(fx, fy);
          out[2 * (fy * range.fragments_x() + fx)] = r.x();
          out[2 * (fy * range.fragments_x() + fx) + 1] = r.y();
        }
    }
    return n;
  }
};

SyntheticScene scene_from(int n_spheres, const double* spheres, int n_planes, const double* planes) {
  // sphere: cx cy cz r ar ag ab ; plane: nx ny nz offset ar ag ab checker checker_size
  SyntheticScene sc;
  for (int i = 0; i < n_spheres; ++i) {
    const double* s = spheres + 7 * i;
    sc.spheres.push_back({Vec3d(s[0], s[1], s[2]), s[3],
                          Vec3f(static_cast<float>(s[4]), static_cast<float>(s[5]), static_cast<float>(s[6]))});
  }
  for (int i = 0; i < n_planes; ++i) {
    const double* p = planes + 9 * i;
    ScenePlane pl;
    pl.normal = Vec3d(p[0], p[1], p[2]);
    pl.offset = p[3];
    pl.albedo = Vec3f(static_cast<float>(p[4]), static_cast<float>(p[5]), static_cast<float>(p[6]));
    pl.checker = p[7] != 0.0;
    pl.checker_size = p[8];
    sc.planes.push_back(pl);
  }
  return sc;
}

}  // namespace

namespace {
template <typename TVoxel, typename F>
long with_cache(const CtxBase* b, F&& f) {
  const auto* c = static_cast<const GlobalCache<TVoxel>*>(b->cache_ptr());
  if (!c) return -1;
  return f(*c);
}
}  // namespace

extern "C" {

void vfr_set_threads(int n) { set_worker_count(n); }
int vfr_get_threads(void) { return worker_count(); }
int vfr_sizeof_config(void) { return static_cast<int>(sizeof(vfr_config)); }
int vfr_sizeof_stats(void) { return static_cast<int>(sizeof(vfr_stats)); }

void* vfr_create(const vfr_config* c, int tracking) {
  try {
    if (tracking) {
      if (c->voxel_type == 2) return static_cast<CtxBase*>(new PipelineCtx<VoxelSRgb>(*c));
      return static_cast<CtxBase*>(new PipelineCtx<VoxelS>(*c));
    }
    if (c->voxel_type == 2) return static_cast<CtxBase*>(new StagesCtx<VoxelSRgb>(*c));
    return static_cast<CtxBase*>(new StagesCtx<VoxelS>(*c));
  } catch (...) {
    return nullptr;
  }
}
void vfr_destroy(void* ctx) { delete static_cast<CtxBase*>(ctx); }

int vfr_process(void* ctx, const float* depth, const std::uint8_t* rgb, const double* pose, vfr_stats* st) {
  return static_cast<CtxBase*>(ctx)->process(depth, rgb, pose, st);
}
void vfr_get_pose(void* ctx, double* out) { pose_to(static_cast<CtxBase*>(ctx)->pose(), out); }
int vfr_get_maps(void* ctx, float* points, float* normals) {
  const TrackingState& st = static_cast<CtxBase*>(ctx)->state();
  if (!st.maps_valid) return -1;
  std::memcpy(points, st.points.pixels().data(), sizeof(Vec4f) * st.points.size());
  std::memcpy(normals, st.normals.pixels().data(), sizeof(Vec4f) * st.normals.size());
  return 0;
}
long vfr_export_entries(void* ctx, void* out) { return static_cast<CtxBase*>(ctx)->export_entries(out); }
long vfr_export_voxels(void* ctx, void* out) { return static_cast<CtxBase*>(ctx)->export_voxels(out); }
long vfr_visible_list(void* ctx, int* out) { return static_cast<CtxBase*>(ctx)->visible_list(out); }
long vfr_export_ranges(void* ctx, float* out) { return static_cast<CtxBase*>(ctx)->export_ranges(out); }
long vfr_surface_points(void* ctx, float* points, float* colors) {
  const TrackingState& s = static_cast<CtxBase*>(ctx)->state();
  const long n = static_cast<long>(s.surface_points.size());
  for (long i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) {
      if (points) points[3 * i + c] = s.surface_points[static_cast<std::size_t>(i)](c);
      if (colors) colors[3 * i + c] = s.surface_colors[static_cast<std::size_t>(i)](c);
    }
  return n;
}
int vfr_image(void* ctx, int mode, std::uint8_t* out) { return static_cast<CtxBase*>(ctx)->image(mode, out); }

// Swap engine state: per-entry SwapState codes, host store contents (codec layout).
long vfr_swap_states(void* ctx, std::uint8_t* out) {
  const CtxBase* b = static_cast<CtxBase*>(ctx);
  auto f = [&](const auto& c) -> long {
    for (int i = 0; i < c.entry_count(); ++i) out[i] = static_cast<std::uint8_t>(c.state(i));
    return c.entry_count();
  };
  return b->voxel_type() == 2 ? with_cache<VoxelSRgb>(b, f) : with_cache<VoxelS>(b, f);
}
int vfr_store_read(void* ctx, int idx, std::uint8_t* payload) {
  const CtxBase* b = static_cast<CtxBase*>(ctx);
  auto f = [&](const auto& c) -> long {
    if (!c.has_stored_data(idx)) return 0;
    if (payload) c.store().read(idx, payload);
    return 1;
  };
  return static_cast<int>(b->voxel_type() == 2 ? with_cache<VoxelSRgb>(b, f) : with_cache<VoxelS>(b, f));
}
long vfr_store_count(void* ctx) {
  const CtxBase* b = static_cast<CtxBase*>(ctx);
  auto f = [&](const auto& c) -> long { return c.store().stored_count(); };
  return b->voxel_type() == 2 ? with_cache<VoxelSRgb>(b, f) : with_cache<VoxelS>(b, f);
}
// ren_refine / color_track through the reference (stage isolation)
int vfr_stage_track(void* ctx, int which, const void* frame, const double* init, double* out_pose, int* iters,
                    double* cost, int* valid, int* ok) {
  const CtxBase* b = static_cast<CtxBase*>(ctx);
  const Pose p0 = pose_from(init);
  const TrackingResult r = which == 1 ? b->stage_color(static_cast<const std::uint8_t*>(frame), p0)
                                      : b->stage_ren(static_cast<const float*>(frame), p0);
  pose_to(r.pose, out_pose);
  *iters = r.iterations;
  *cost = r.final_cost;
  *valid = r.valid_points;
  *ok = r.ok ? 1 : 0;
  return 0;
}
// Recorded-sequence I/O through the reference (pnm.cpp, calibration.cpp, sequence.cpp).
// out: rgb (w, h, fx, fy, cx, cy), depth (same), rgb_to_depth (R row-major, t), a, b.
int vfr_parse_calibration(const char* text, double* out, int* err_line) {
  try {
    const Calibration c = parse_calibration_text(text);
    const Intrinsics* cams[2] = {&c.rgb, &c.depth};
    for (int k = 0; k < 2; ++k) {
      const Intrinsics& i = *cams[k];
      double* o = out + 6 * k;
      o[0] = i.width, o[1] = i.height, o[2] = i.fx, o[3] = i.fy, o[4] = i.cx, o[5] = i.cy;
    }
    pose_to(c.rgb_to_depth, out + 12);
    out[24] = c.disparity.a;
    out[25] = c.disparity.b;
    return 0;
  } catch (const CalibrationError& e) {
    if (err_line) *err_line = e.line();
    return -1;
  }
}
int vfr_read_pgm16(const char* path, std::uint16_t* out, long cap, int* w, int* h) {
  try {
    std::ifstream in(path, std::ios::binary);
    const Image2D<std::uint16_t> img = read_pgm16(in);
    *w = img.width();
    *h = img.height();
    if ((long)img.size() > cap) return -2;
    std::memcpy(out, img.pixels().data(), sizeof(std::uint16_t) * img.size());
    return 0;
  } catch (const PnmError&) {
    return -1;
  }
}
int vfr_read_ppm(const char* path, std::uint8_t* out, long cap, int* w, int* h) {
  try {
    std::ifstream in(path, std::ios::binary);
    const Image2D<Vec3u8> img = read_ppm(in);
    *w = img.width();
    *h = img.height();
    if ((long)img.size() * 3 > cap) return -2;
    for (std::size_t i = 0; i < img.size(); ++i)
      for (int ch = 0; ch < 3; ++ch) out[3 * i + ch] = img.pixels()[i](ch);
    return 0;
  } catch (const PnmError&) {
    return -1;
  }
}
// disparity_image_to_depth through the reference's own Calibration (view.hpp:18-28)
void vfr_disparity_to_depth(const std::uint16_t* disp, int w, int h, double a, double b, double fx,
                            float max_depth, float* depth) {
  Image2D<std::uint16_t> img(w, h);
  std::memcpy(img.pixels().data(), disp, sizeof(std::uint16_t) * static_cast<std::size_t>(w) * h);
  Calibration k;
  k.depth.fx = fx;
  k.disparity.a = a;
  k.disparity.b = b;
  const Image2D<float> d = disparity_image_to_depth(img, k, max_depth);
  std::memcpy(depth, d.pixels().data(), sizeof(float) * static_cast<std::size_t>(w) * h);
}
std::uint64_t vfr_digest(void* ctx) { return static_cast<CtxBase*>(ctx)->digest(); }
long vfr_allocated_blocks(void* ctx) { return static_cast<CtxBase*>(ctx)->allocated_blocks(); }

void vfr_render_depth(int n_spheres, const double* spheres, int n_planes, const double* planes,
                      const double* world_to_cam, double fx, double fy, double cx, double cy, int w, int h,
                      double near_clip, double far_clip, float* out) {
  Intrinsics in;
  in.fx = fx;
  in.fy = fy;
  in.cx = cx;
  in.cy = cy;
  in.width = w;
  in.height = h;
  const Image2D<float> d = render_synthetic_depth(scene_from(n_spheres, spheres, n_planes, planes),
                                                  pose_from(world_to_cam), in, near_clip, far_clip);
  std::memcpy(out, d.pixels().data(), sizeof(float) * d.size());
}

void vfr_render_rgb(int n_spheres, const double* spheres, int n_planes, const double* planes,
                    const double* world_to_cam, double fx, double fy, double cx, double cy, int w, int h,
                    double near_clip, double far_clip, std::uint8_t* out) {
  Intrinsics in;
  in.fx = fx;
  in.fy = fy;
  in.cx = cx;
  in.cy = cy;
  in.width = w;
  in.height = h;
  const Image2D<Vec3u8> c = render_synthetic_rgb(scene_from(n_spheres, spheres, n_planes, planes),
                                                 pose_from(world_to_cam), in, near_clip, far_clip);
  for (std::size_t i = 0; i < c.size(); ++i) {
    out[3 * i] = c.pixels()[i].x();
    out[3 * i + 1] = c.pixels()[i].y();
    out[3 * i + 2] = c.pixels()[i].z();
  }
}

// Stage entry: the reference's icp_track on a caller-provided pyramid base
// depth and world-space maps rendered at `render_pose` (depth_tracker.hpp:115).
int vfr_icp_track(const vfr_config* c, const float* depth, const float* points, const float* normals,
                  const double* render_pose, double* out_pose, int* out_iters, double* out_cost,
                  int* out_valid) {
  const EngineSettings s = settings_from(*c);
  const Calibration k = calib_from(*c);
  TrackingState st;
  st.pose = pose_from(render_pose);
  st.points = Image2D<Vec4f>(c->width, c->height, Vec4f::Zero());
  st.normals = Image2D<Vec4f>(c->width, c->height, Vec4f::Zero());
  std::memcpy(st.points.pixels().data(), points, sizeof(Vec4f) * st.points.size());
  std::memcpy(st.normals.pixels().data(), normals, sizeof(Vec4f) * st.normals.size());
  st.maps_valid = true;
  const DepthPyramid pyr = build_depth_pyramid(depth_image(depth, c->width, c->height), k.depth,
                                               s.tracker.hierarchy_levels);
  const TrackingResult r = icp_track(pyr, st, s.tracker);
  pose_to(r.pose, out_pose);
  *out_iters = r.iterations;
  *out_cost = r.final_cost;
  *out_valid = r.valid_points;
  return r.ok ? 1 : 0;
}

// Stage entry: the reference's depth pyramid (pyramid.hpp:101-111); levels
// are written back to back.
void vfr_depth_pyramid(const float* depth, int w, int h, int levels, float* out) {
  Intrinsics in;
  in.fx = in.fy = 1;
  in.cx = w / 2.0;
  in.cy = h / 2.0;
  in.width = w;
  in.height = h;
  const DepthPyramid pyr = build_depth_pyramid(depth_image(depth, w, h), in, levels);
  std::size_t off = 0;
  for (int l = 0; l < pyr.levels(); ++l) {
    const auto& img = pyr.depth[static_cast<std::size_t>(l)];
    std::memcpy(out + off, img.pixels().data(), sizeof(float) * img.size());
    off += img.size();
  }
}

}  // extern "C"
