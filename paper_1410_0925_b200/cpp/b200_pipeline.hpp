// voxfuse::IPipeline on the B200 — the C++ host side of the drop-in.
//
// A header-only adapter that a user of the reference (/root/reference/proj)
// includes next to its own headers: it implements the reference's virtual
// engine interface IPipeline (proj/include/voxfuse/engine/pipeline.hpp:66-84)
// on top of the C ABI in include/voxfuse_b200.h, so replacing
//
//     auto p = voxfuse::make_pipeline(settings, calib);          // CPU engine
// with
//     auto p = voxfuse_b200::make_b200_pipeline(settings, calib); // sm_100a engine
//
// is the whole integration.  Everything the reference returns by value or
// reference (FrameStats, Pose, TrackingState, digests) keeps its type and
// meaning; construction errors are reported with the reference's exception
// type (std::invalid_argument, pipeline_impl.hpp:55-57), runtime CUDA errors
// as std::runtime_error.  Scope: hash backend, VoxelS /
// VoxelSRgb, the ICP / colour / ICP+Ren trackers, host swapping, raw
// disparity input; the dense backend and float voxels raise
// std::invalid_argument.
#pragma once

#include <cstdint>
#include <cstring>
#include <deque>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "voxfuse/engine/block_store.hpp"
#include "voxfuse/engine/pipeline.hpp"
#include "voxfuse/engine/raycast.hpp"
#include "voxfuse/engine/view.hpp"
#include "voxfuse_b200.h"

namespace voxfuse_b200 {

namespace detail {

inline void pose_to_array(const voxfuse::Pose& p, double* out) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) out[i * 3 + j] = p.rotation()(i, j);
  for (int i = 0; i < 3; ++i) out[9 + i] = p.translation()(i);
}

inline voxfuse::Pose pose_from_array(const double* a) {
  voxfuse::Mat3d r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = a[i * 3 + j];
  return voxfuse::Pose(r, voxfuse::Vec3d(a[9], a[10], a[11]));
}

inline vf_intrinsics to_c(const voxfuse::Intrinsics& in) {
  vf_intrinsics o;
  o.fx = in.fx;
  o.fy = in.fy;
  o.cx = in.cx;
  o.cy = in.cy;
  o.width = in.width;
  o.height = in.height;
  return o;
}

inline void check(int rc, const char* what, const vf_ctx* ctx) {
  if (rc < 0) {
    throw std::runtime_error(std::string(what) + " failed (" + std::to_string(rc) + "): " +
                             (ctx ? vf_last_error(ctx) : ""));
  }
}

}  // namespace detail

/// Translates the reference's EngineSettings (pipeline.hpp:19-41) into the
/// C ABI's settings; throws std::invalid_argument for anything out of scope.
inline vf_settings to_vf_settings(const voxfuse::EngineSettings& s) {
  using voxfuse::TrackerType;
  using voxfuse::VoxelType;
  if (s.backend != voxfuse::VolumeBackend::hash)
    throw std::invalid_argument("voxfuse_b200: only the voxel-block hash backend is implemented");
  if (s.voxel_type != VoxelType::s && s.voxel_type != VoxelType::s_rgb)
    throw std::invalid_argument("voxfuse_b200: voxel types VoxelS and VoxelSRgb only");
  if (s.tracker.type == TrackerType::color && s.voxel_type != VoxelType::s_rgb)
    throw std::invalid_argument("colour tracker requires a voxel type with colour information");
  vf_settings c;
  vf_default_settings(&c);
  c.voxel_type = s.voxel_type == VoxelType::s_rgb ? VF_VOXEL_S_RGB : VF_VOXEL_S;
  c.voxel_size = s.scene.voxel_size;
  c.mu = s.scene.mu;
  c.max_weight = s.scene.max_weight;
  c.stop_integrating_at_max = s.scene.stop_integrating_at_max ? 1 : 0;
  c.bucket_count = s.hash.bucket_count;
  c.bucket_size = s.hash.bucket_size;
  c.excess_count = s.hash.excess_count;
  c.block_count = s.hash.block_count;
  c.near_clip = s.near_clip;
  c.far_clip = s.far_clip;
  c.visibility_margin_px = s.visibility_margin_px;
  c.swap_margin_px = s.swap_margin_px;
  c.hierarchy_levels = s.tracker.hierarchy_levels;
  c.rotation_only_levels = s.tracker.rotation_only_levels;
  c.max_iterations = s.tracker.max_iterations;
  c.min_valid_points = s.tracker.min_valid_points;
  c.icp_dist_threshold = s.tracker.icp_dist_threshold;
  c.convergence_eps = s.tracker.convergence_eps;
  c.max_condition = s.tracker.max_condition;
  c.tracking = 1;
  c.use_graphs = 1;
  c.use_swapping = s.use_swapping ? 1 : 0;  // swap.hpp; host store in pinned, device-mapped memory
  c.swap_buffer_blocks = s.swap_buffer_blocks;
  c.max_depth = s.max_depth;
  c.tracker_type = s.tracker.type == TrackerType::color     ? VF_TRACKER_COLOR
                   : s.tracker.type == TrackerType::icp_ren ? VF_TRACKER_ICP_REN
                                                            : VF_TRACKER_ICP;
  c.ren_sigma = s.tracker.ren_sigma;
  c.skip_points = s.tracker.skip_points ? 1 : 0;
  c.integration_mode = VF_INTEGRATION_EXACT;  // the drop-in keeps the reference's arithmetic
  return c;
}

/// IPipeline backed by one device-resident volume on one GPU.
class B200Pipeline final : public voxfuse::IPipeline {
 public:
  B200Pipeline(const voxfuse::EngineSettings& settings, const voxfuse::Calibration& calib, int device = 0)
      : settings_(settings), calib_(calib) {
    const vf_settings s = to_vf_settings(settings);
    vf_calib c;
    std::memset(&c, 0, sizeof(c));
    c.depth = detail::to_c(calib.depth);
    c.rgb = detail::to_c(calib.rgb);
    detail::pose_to_array(calib.rgb_to_depth, c.rgb_to_depth);
    c.disparity_a = calib.disparity.a;
    c.disparity_b = calib.disparity.b;
    const int rc = vf_create(&s, &c, device, &ctx_);
    if (rc == VF_ERR_INVALID) throw std::invalid_argument("voxfuse_b200: invalid settings");
    detail::check(rc, "vf_create", nullptr);
    // the reference fills FrameStats::ms_* on every frame (pipeline_impl.hpp:66-120)
    detail::check(vf_set_stage_timing(ctx_, 1), "vf_set_stage_timing", ctx_);
    // swap_store_path (pipeline.hpp:24; pipeline_impl.hpp:43-51): the
    // reference's own file-backed BlockStore, fed as blocks leave
    if (settings_.use_swapping && !settings_.swap_store_path.empty()) {
      const bool rgb = settings_.voxel_type == voxfuse::VoxelType::s_rgb;
      const int payload = (rgb ? voxfuse::VoxelCodec<voxfuse::VoxelSRgb>::bytes
                               : voxfuse::VoxelCodec<voxfuse::VoxelS>::bytes) * voxfuse::kBlockVolume;
      const auto tag = static_cast<std::uint16_t>(rgb ? voxfuse::VoxelCodec<voxfuse::VoxelSRgb>::tag
                                                      : voxfuse::VoxelCodec<voxfuse::VoxelS>::tag);
      file_store_ = voxfuse::make_file_block_store(settings_.swap_store_path, static_cast<int>(vf_entry_count(ctx_)),
                                                   payload, tag);
      drained_.resize(1 << 16);
      payload_.resize(static_cast<std::size_t>(payload));
    }
  }
  ~B200Pipeline() override {
    file_store_.reset();
    if (ctx_) vf_destroy(ctx_);
  }
  B200Pipeline(const B200Pipeline&) = delete;
  B200Pipeline& operator=(const B200Pipeline&) = delete;

  // IPipeline::process_frame (pipeline_impl.hpp:65-123): the whole frame runs
  // on the GPU; depth (and rgb) go up, FrameStats come back.
  voxfuse::FrameStats process_frame(const voxfuse::Image2D<voxfuse::Vec3u8>* rgb,
                                    const voxfuse::Image2D<float>& depth_m) override {
    if (depth_m.width() != calib_.depth.width || depth_m.height() != calib_.depth.height)
      throw std::invalid_argument("voxfuse_b200: depth image size does not match the calibration");
    static_assert(sizeof(voxfuse::Vec3u8) == 3, "Vec3u8 must be packed RGB");
    const std::uint8_t* rgb_ptr = nullptr;
    if (rgb && !rgb->empty() && settings_.voxel_type == voxfuse::VoxelType::s_rgb)
      rgb_ptr = reinterpret_cast<const std::uint8_t*>(rgb->pixels().data());
    vf_frame_stats st;
    detail::check(vf_process_frame(ctx_, depth_m.pixels().data(), rgb_ptr, &st), "vf_process_frame", ctx_);
    if (rgb) last_rgb_ = *rgb;
    return finish_frame(st);
  }

  // Streaming extension (not part of IPipeline): vf_submit_frame /
  // vf_collect_frame with up to VF_MAX_FRAMES_IN_FLIGHT frames in flight, so
  // the upload of frame n + 1 overlaps frame n.  collect_frame returns the
  // oldest frame's stats (equal to what process_frame would have returned);
  // the depth (or disparity) buffer must stay alive and unchanged until then.
  void submit_frame(const voxfuse::Image2D<voxfuse::Vec3u8>* rgb, const voxfuse::Image2D<float>& depth_m) {
    if (depth_m.width() != calib_.depth.width || depth_m.height() != calib_.depth.height)
      throw std::invalid_argument("voxfuse_b200: depth image size does not match the calibration");
    const std::uint8_t* rgb_ptr = nullptr;
    if (rgb && !rgb->empty() && settings_.voxel_type == voxfuse::VoxelType::s_rgb)
      rgb_ptr = reinterpret_cast<const std::uint8_t*>(rgb->pixels().data());
    detail::check(vf_submit_frame(ctx_, depth_m.pixels().data(), rgb_ptr), "vf_submit_frame", ctx_);
    pending_rgb_.push_back(rgb ? *rgb : voxfuse::Image2D<voxfuse::Vec3u8>());
  }
  void submit_raw_frame(const voxfuse::Image2D<voxfuse::Vec3u8>* rgb, const voxfuse::Image2D<std::uint16_t>& disparity) {
    if (disparity.width() != calib_.depth.width || disparity.height() != calib_.depth.height)
      throw std::invalid_argument("voxfuse_b200: disparity image size does not match the calibration");
    const std::uint8_t* rgb_ptr = nullptr;
    if (rgb && !rgb->empty() && settings_.voxel_type == voxfuse::VoxelType::s_rgb)
      rgb_ptr = reinterpret_cast<const std::uint8_t*>(rgb->pixels().data());
    detail::check(vf_submit_raw_frame(ctx_, disparity.pixels().data(), rgb_ptr, 0), "vf_submit_raw_frame", ctx_);
    pending_rgb_.push_back(rgb ? *rgb : voxfuse::Image2D<voxfuse::Vec3u8>());
  }
  voxfuse::FrameStats collect_frame() {
    vf_frame_stats st;
    const int rc = vf_collect_frame(ctx_, &st);
    if (rc != VF_ERR_STATE && !pending_rgb_.empty()) {
      if (!pending_rgb_.front().empty()) last_rgb_ = std::move(pending_rgb_.front());
      pending_rgb_.pop_front();
    }
    detail::check(rc, "vf_collect_frame", ctx_);
    return finish_frame(st);
  }
  int frames_in_flight() const { return vf_frames_in_flight(ctx_); }

 private:
  // The blocks swapped out since the last frame, in swap-out order, into the
  // reference's file store: a record appended on a slot's first write and
  // rewritten in place after (block_store.cpp:96-115), one flush per frame
  // as execute_swap_out does (swap.hpp:251).
  void journal_swap_outs() {
    if (!file_store_) return;
    long lost = 0;
    const long n = vf_swap_drain(ctx_, drained_.data(), static_cast<long>(drained_.size()), &lost);
    detail::check(static_cast<int>(n < 0 ? n : 0), "vf_swap_drain", ctx_);
    if (lost > 0) throw std::runtime_error("voxfuse_b200: swap journal overflowed between frames");
    for (long i = 0; i < n; ++i)
      if (vf_swap_store_read(ctx_, drained_[static_cast<std::size_t>(i)], payload_.data()) == 1)
        file_store_->write(drained_[static_cast<std::size_t>(i)], payload_.data());
    file_store_->flush();
  }

  voxfuse::FrameStats finish_frame(const vf_frame_stats& st) {
    journal_swap_outs();
    pose_ = detail::pose_from_array(st.pose);
    maps_stale_ = true;
    voxfuse::FrameStats fs;
    fs.frame = st.frame;
    fs.tracking_ok = st.tracking_ok != 0;
    fs.tracking_iterations = st.tracking_iterations;
    fs.tracking_cost = st.tracking_cost;
    fs.blocks_allocated = st.blocks_allocated;
    fs.allocation_dropped = st.allocation_dropped;
    fs.visible_blocks = st.visible_blocks;
    fs.pose = pose_;
    fs.swap.swapped_in = st.swapped_in;
    fs.swap.swapped_out = st.swapped_out;
    fs.swap.bytes_in = st.swap_bytes_in;
    fs.swap.bytes_out = st.swap_bytes_out;
    // GPU time of the frame and of its stages (CUDA events in the frame graph;
    // the streaming calls carry ms_total only)
    fs.ms_tracking = st.ms_tracking;
    fs.ms_allocation = st.ms_allocation;
    fs.ms_integration = st.ms_integration;
    fs.ms_swapping = st.ms_swapping;
    fs.ms_raycast = st.ms_raycast;
    fs.ms_total = st.ms_total;
    return fs;
  }

 public:
  // IPipeline::process_raw_frame (pipeline_impl.hpp:59-62): the u16
  // disparity goes up (half the bytes of a float depth map) and
  // disparity_image_to_depth runs on the device.
  voxfuse::FrameStats process_raw_frame(const voxfuse::Image2D<voxfuse::Vec3u8>* rgb,
                                        const voxfuse::Image2D<std::uint16_t>& disparity) override {
    if (disparity.width() != calib_.depth.width || disparity.height() != calib_.depth.height)
      throw std::invalid_argument("voxfuse_b200: disparity image size does not match the calibration");
    const std::uint8_t* rgb_ptr = nullptr;
    if (rgb && !rgb->empty() && settings_.voxel_type == voxfuse::VoxelType::s_rgb)
      rgb_ptr = reinterpret_cast<const std::uint8_t*>(rgb->pixels().data());
    vf_frame_stats st;
    detail::check(vf_process_raw_frame(ctx_, disparity.pixels().data(), rgb_ptr, 0, &st), "vf_process_raw_frame",
                  ctx_);
    if (rgb) last_rgb_ = *rgb;
    return finish_frame(st);
  }

  // IPipeline::get_image (pipeline_impl.hpp:125-137): rendered on the GPU
  // (render_image / colourize_depth, raycast.hpp:466-490) and downloaded.
  voxfuse::Image2D<voxfuse::Vec3u8> get_image(voxfuse::DisplayMode mode) const override {
    using voxfuse::Image2D;
    using voxfuse::Vec3u8;
    if (mode == voxfuse::DisplayMode::rgb_passthrough) return last_rgb_;
    const int vm = mode == voxfuse::DisplayMode::depth_colourized ? VF_DISPLAY_DEPTH_COLOURIZED : VF_DISPLAY_RAYCAST;
    Image2D<Vec3u8> out(calib_.depth.width, calib_.depth.height, Vec3u8::Zero());
    static_assert(sizeof(Vec3u8) == 3, "Vec3u8 must be packed RGB");
    const int rc = vf_render_image(ctx_, vm, reinterpret_cast<std::uint8_t*>(out.pixels().data()));
    if (rc == VF_ERR_STATE) return Image2D<Vec3u8>();  // nothing rendered yet (reference: empty image)
    detail::check(rc, "vf_render_image", ctx_);
    return out;
  }

  // TrackingState: the world-space maps are downloaded on demand.
  const voxfuse::TrackingState& tracking_state() const override {
    if (maps_stale_) {
      const int w = calib_.depth.width, h = calib_.depth.height;
      state_.points = voxfuse::Image2D<voxfuse::Vec4f>(w, h, voxfuse::Vec4f::Zero());
      state_.normals = voxfuse::Image2D<voxfuse::Vec4f>(w, h, voxfuse::Vec4f::Zero());
      static_assert(sizeof(voxfuse::Vec4f) == 16, "Vec4f must be 4 packed floats");
      const int rc = vf_get_maps(ctx_, reinterpret_cast<float*>(state_.points.pixels().data()),
                                 reinterpret_cast<float*>(state_.normals.pixels().data()));
      state_.maps_valid = rc == VF_OK;
      state_.pose = pose_;
      // surface list for the colour tracker (forward_project_points, raycast.hpp:495-509)
      state_.surface_points.clear();
      state_.surface_colors.clear();
      const long n = vf_get_surface_points(ctx_, nullptr, nullptr, 0);
      if (n > 0) {
        static_assert(sizeof(voxfuse::Vec3f) == 12, "Vec3f must be 3 packed floats");
        state_.surface_points.resize(static_cast<std::size_t>(n));
        state_.surface_colors.resize(static_cast<std::size_t>(n));
        detail::check((int)vf_get_surface_points(ctx_, reinterpret_cast<float*>(state_.surface_points.data()),
                                                 reinterpret_cast<float*>(state_.surface_colors.data()), n) < 0
                          ? VF_ERR_CUDA
                          : VF_OK,
                      "vf_get_surface_points", ctx_);
      }
      maps_stale_ = false;
    }
    return state_;
  }
  const voxfuse::Pose& pose() const override { return pose_; }
  int frame_count() const override { return vf_frame_count(ctx_); }
  const voxfuse::EngineSettings& settings() const override { return settings_; }
  std::uint64_t volume_digest() const override {
    std::uint64_t h = 0;
    detail::check(vf_volume_digest(ctx_, &h), "vf_volume_digest", ctx_);
    return h;
  }

  vf_ctx* handle() const { return ctx_; }

 private:
  voxfuse::EngineSettings settings_;
  voxfuse::Calibration calib_;
  vf_ctx* ctx_ = nullptr;
  voxfuse::Pose pose_;
  std::unique_ptr<voxfuse::BlockStore> file_store_;  // swap_store_path: the reference's VXBS file store
  std::vector<int> drained_;
  std::vector<std::uint8_t> payload_;
  voxfuse::Image2D<voxfuse::Vec3u8> last_rgb_;
  std::deque<voxfuse::Image2D<voxfuse::Vec3u8>> pending_rgb_;  // rgb of the frames in flight
  mutable voxfuse::TrackingState state_;
  mutable bool maps_stale_ = true;
};

/// Drop-in for voxfuse::make_pipeline (pipeline.hpp:86).
inline std::unique_ptr<voxfuse::IPipeline> make_b200_pipeline(const voxfuse::EngineSettings& settings,
                                                              const voxfuse::Calibration& calib, int device = 0) {
  return std::make_unique<B200Pipeline>(settings, calib, device);
}

}  // namespace voxfuse_b200
