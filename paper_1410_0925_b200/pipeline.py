"""Host-side mirror of the reference's engine interface over the C ABI.

Names, argument order and meaning follow the reference:

* ``make_pipeline(settings, calib)`` -> ``Pipeline`` (IPipeline,
  proj/include/voxfuse/engine/pipeline.hpp:66-86);
* ``Pipeline.process_frame(rgb, depth_m)`` -> ``FrameStats`` (pipeline.hpp:70);
* ``pose()``, ``frame_count()``, ``settings()``, ``tracking_state()``,
  ``volume_digest()``;
* stage functions mirroring the stage templates (allocation.hpp,
  integration.hpp, raycast.hpp, pyramid.hpp, depth_tracker.hpp) for
  stage-isolated use.

All compute runs in the sm_100a library; this module only marshals buffers.
Construction fails with ``VoxfuseError(VF_ERR_NO_DEVICE)`` without a GPU.
"""
from __future__ import annotations

import collections
import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import VfAllocStats, VfCalib, VfFrameStats, VfIntrinsics, VfSettings, check

ENTRY_DTYPE = np.dtype(
    [("x", "<i2"), ("y", "<i2"), ("z", "<i2"), ("pad", "<i2"), ("offset", "<i4"), ("block_state", "<i4")]
)
TRACKER_TYPES = {"icp": 0, "color": 1, "icp_ren": 2}
VOXEL_TYPE_S = 1
VOXEL_TYPE_S_RGB = 2


@dataclass
class Intrinsics:
    """Intrinsics (proj/include/voxfuse/core/intrinsics.hpp:10-32)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def to_c(self) -> VfIntrinsics:
        return VfIntrinsics(self.fx, self.fy, self.cx, self.cy, self.width, self.height)


@dataclass
class Calibration:
    """Calibration (proj/include/voxfuse/io/calibration.hpp:31-36)."""

    depth: Intrinsics
    rgb: Intrinsics | None = None
    rgb_to_depth: np.ndarray = field(default_factory=lambda: np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0], float))
    disparity_a: float = 0.0
    disparity_b: float = 0.0

    def to_c(self) -> VfCalib:
        c = VfCalib()
        c.depth = self.depth.to_c()
        c.rgb = (self.rgb or self.depth).to_c()
        for i, v in enumerate(np.asarray(self.rgb_to_depth, float).reshape(-1)):
            c.rgb_to_depth[i] = float(v)
        c.disparity_a = self.disparity_a
        c.disparity_b = self.disparity_b
        return c


@dataclass
class EngineSettings:
    """EngineSettings + SceneParams + HashConfig + TrackerSettings with the
    reference defaults (pipeline.hpp:19-41, scene_params.hpp:6-13,
    hash_volume.hpp:49-58, tracking_state.hpp:12-23)."""

    voxel_type: int = VOXEL_TYPE_S
    voxel_size: float = 0.004
    mu: float = 0.02
    max_weight: int = 100
    stop_integrating_at_max: bool = False
    bucket_count: int = 1 << 20
    bucket_size: int = 2
    excess_count: int = 1 << 17
    block_count: int = 1 << 18
    near_clip: float = 0.1
    far_clip: float = 8.0
    visibility_margin_px: int = 8
    swap_margin_px: int = 48
    hierarchy_levels: int = 5
    rotation_only_levels: int = 2
    max_iterations: int = 20
    min_valid_points: int = 30
    icp_dist_threshold: float = 0.1
    convergence_eps: float = 1e-5
    max_condition: float = 1e8
    tracking: bool = True
    use_graphs: bool = True
    shard_count: int = 1   # spatial sharding (config 5): G shards ...
    shard_index: int = 0   # ... this context's shard ...
    shard_shift: int = 3   # ... owning super-blocks of 2^shift blocks per axis
    shard_halo: bool = True  # ... and fusing surfaces within one block of them
    use_swapping: bool = False  # host swapping (pipeline.hpp:20-23, swap.hpp)
    swap_buffer_blocks: int = 100
    swap_host_blocks: int = 0  # host store slot cap (0: one per hash entry, like the reference; grown in chunks)
    max_depth: float = 8.0  # disparity conversion clamp (pipeline.hpp:37)
    tracker_type: int = 0  # TrackerType: 0 icp, 1 color, 2 icp_ren (tracking_state.hpp:10)
    ren_sigma: float = 10.0
    skip_points: bool = False
    integration_mode: int = 0  # 0 exact (bit-exact), 1 fast (<= 1 LSB / 1 colour count tolerance)
    shard_icp: bool = False  # pixel-sharded ICP, per-iteration sums exchanged through peer memory
    icp_max_ctas: int = 0    # cap of the ICP grid (shards sharing one device)
    tracker_exact_solve: bool = False  # colour tracker: the reference's pivoted LDLT on every step

    def to_c(self) -> VfSettings:
        s = VfSettings()
        for name, _ in VfSettings._fields_:
            v = getattr(self, name)
            setattr(s, name, int(v) if isinstance(v, bool) else v)
        return s

    @property
    def entry_count(self) -> int:
        return self.bucket_count * self.bucket_size + self.excess_count


def settings_from_config(cfg) -> tuple[EngineSettings, Calibration]:
    """EngineSettings + Calibration for a paper_1410_0925_b200.scene.BenchConfig."""
    fx, fy, cx, cy, w, h = cfg.intrinsics
    s = EngineSettings(
        voxel_type=cfg.voxel_type, voxel_size=cfg.voxel_size, mu=cfg.mu, max_weight=cfg.max_weight,
        stop_integrating_at_max=getattr(cfg, "stop_integrating_at_max", False),
        bucket_count=cfg.hash.bucket_count, bucket_size=cfg.hash.bucket_size, excess_count=cfg.hash.excess_count,
        block_count=cfg.hash.block_count, near_clip=cfg.near_clip, far_clip=cfg.far_clip,
        visibility_margin_px=cfg.margin_px, swap_margin_px=cfg.swap_margin_px, hierarchy_levels=cfg.levels,
        rotation_only_levels=cfg.rotation_only_levels, max_iterations=cfg.max_iterations,
        min_valid_points=cfg.min_valid_points, icp_dist_threshold=cfg.icp_dist_threshold,
        convergence_eps=cfg.convergence_eps, max_condition=cfg.max_condition, tracking=cfg.tracking,
        use_swapping=getattr(cfg, "use_swapping", False), swap_buffer_blocks=getattr(cfg, "swap_buffer_blocks", 100),
        tracker_type=TRACKER_TYPES[getattr(cfg, "tracker", "icp")],
    )
    intr = Intrinsics(fx, fy, cx, cy, w, h)
    return s, Calibration(depth=intr, rgb=intr)


@dataclass
class FrameStats:
    """FrameStats (pipeline.hpp:45-58)."""

    frame: int
    tracking_ok: bool
    tracking_iterations: int
    tracking_cost: float
    blocks_allocated: int
    allocation_dropped: int
    visible_blocks: int
    pose: np.ndarray
    ms_total: float
    allocation_requested: int = 0
    allocated_total: int = 0
    tracking_valid_points: int = 0
    error_flags: int = 0
    swapped_in: int = 0  # SwapMetrics (swap.hpp:28-40)
    swapped_out: int = 0
    bytes_in: int = 0
    bytes_out: int = 0
    ms_tracking: float = 0.0  # per-stage ms (pipeline.hpp:56), with set_stage_timing(True)
    ms_allocation: float = 0.0
    ms_integration: float = 0.0
    ms_swapping: float = 0.0
    ms_raycast: float = 0.0

    @classmethod
    def from_c(cls, s: VfFrameStats) -> "FrameStats":
        return cls(s.frame, bool(s.tracking_ok), s.tracking_iterations, s.tracking_cost, s.blocks_allocated,
                   s.allocation_dropped, s.visible_blocks, np.array(s.pose[:]), s.ms_total, s.allocation_requested,
                   s.allocated_total, s.tracking_valid_points, s.error_flags, s.swapped_in, s.swapped_out,
                   s.swap_bytes_in, s.swap_bytes_out, s.ms_tracking, s.ms_allocation, s.ms_integration,
                   s.ms_swapping, s.ms_raycast)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f32(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    if shape is not None and a.size != int(np.prod(shape)):
        raise ValueError(f"expected {shape}, got {a.shape}")
    return a


def _pose(p):
    p = np.ascontiguousarray(p, dtype=np.float64).reshape(-1)
    if p.size != 12:
        raise ValueError("pose must be 12 doubles: row-major R then t")
    return p


class Pipeline:
    """IPipeline over one device-resident voxel-block hash volume."""

    def __init__(self, settings: EngineSettings, calib: Calibration, device: int = 0):
        if settings.shard_count > 1 and settings.tracker_type != TRACKER_TYPES["icp"]:
            # mirrors vf_create: only ICP reads the composited (rank-identical)
            # maps; Ren / colour read the shard's own voxels and would diverge
            raise ValueError("spatial sharding (shard_count > 1) requires the ICP tracker")
        self._L = _abi.load()
        self._settings = settings
        self._calib = calib
        self._c_settings = settings.to_c()
        self._c_calib = calib.to_c()
        h = C.c_void_p()
        check("vf_create", self._L.vf_create(C.byref(self._c_settings), C.byref(self._c_calib), device, C.byref(h)))
        self._h = h
        self._in_flight = collections.deque()
        self.width, self.height = calib.depth.width, calib.depth.height
        rgb = calib.rgb or calib.depth
        self.rgb_width, self.rgb_height = rgb.width, rgb.height

    # -- lifecycle --
    def close(self):
        if getattr(self, "_h", None):
            self._L.vf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def _chk(self, fn, rc):
        return check(fn, rc, self._h)

    # -- IPipeline --
    def process_frame(self, rgb, depth_m) -> FrameStats:
        """IPipeline::process_frame(rgb*, depth_m) with host arrays."""
        d = _f32(depth_m, (self.height, self.width))
        c = None if rgb is None else np.ascontiguousarray(rgb, dtype=np.uint8)
        st = VfFrameStats()
        self._chk("vf_process_frame", self._L.vf_process_frame(self._h, _ptr(d), _ptr(c), C.byref(st)))
        return FrameStats.from_c(st)

    def submit_frame(self, rgb, depth_m) -> None:
        """vf_submit_frame: enqueue a frame and return; its upload overlaps the
        previous frame's processing.  At most MAX_FRAMES_IN_FLIGHT (2) frames may be
        outstanding; collect_frame returns them oldest first."""
        d = _f32(depth_m, (self.height, self.width))
        c = None if rgb is None else np.ascontiguousarray(rgb, dtype=np.uint8)
        self._chk("vf_submit_frame", self._L.vf_submit_frame(self._h, _ptr(d), _ptr(c)))
        self._in_flight.append((d, c))  # the host buffers stay alive until collected

    def submit_raw_frame(self, rgb, disparity, big_endian: bool = False) -> None:
        """vf_submit_raw_frame: process_raw_frame's streaming form."""
        d = np.ascontiguousarray(disparity, dtype=np.uint16).reshape(self.height, self.width)
        c = None if rgb is None else np.ascontiguousarray(rgb, dtype=np.uint8)
        self._chk("vf_submit_raw_frame", self._L.vf_submit_raw_frame(self._h, _ptr(d), _ptr(c), 1 if big_endian else 0))
        self._in_flight.append((d, c))

    def collect_frame(self) -> FrameStats:
        """vf_collect_frame: wait for the oldest frame in flight, return its stats."""
        st = VfFrameStats()
        rc = self._L.vf_collect_frame(self._h, C.byref(st))
        if rc != _abi.VF_ERR_STATE and self._in_flight:
            self._in_flight.popleft()
        self._chk("vf_collect_frame", rc)
        return FrameStats.from_c(st)

    def frames_in_flight(self) -> int:
        return int(self._L.vf_frames_in_flight(self._h))

    def process_raw_frame(self, rgb, disparity, big_endian: bool = False) -> FrameStats:
        """IPipeline::process_raw_frame(rgb*, disparity) (pipeline_impl.hpp:59-62):
        u16 disparity (or, big_endian, the raw bytes of a 16-bit P5 raster)."""
        d = np.ascontiguousarray(disparity, dtype=np.uint16).reshape(self.height, self.width)
        c = None if rgb is None else np.ascontiguousarray(rgb, dtype=np.uint8)
        st = VfFrameStats()
        self._chk("vf_process_raw_frame",
                  self._L.vf_process_raw_frame(self._h, _ptr(d), _ptr(c), 1 if big_endian else 0, C.byref(st)))
        return FrameStats.from_c(st)

    def disparity_to_depth(self, disparity, big_endian: bool = False) -> np.ndarray:
        """disparity_image_to_depth (view.hpp:18-28) on the device."""
        d = np.ascontiguousarray(disparity, dtype=np.uint16).reshape(self.height, self.width)
        out = np.zeros((self.height, self.width), np.float32)
        self._chk("vf_disparity_to_depth",
                  self._L.vf_disparity_to_depth(self._h, _ptr(d), 1 if big_endian else 0, _ptr(out)))
        return out

    def process_frame_device(self, d_depth: int, d_rgb: int | None = None, read_stats: bool = False):
        """Inputs already in device memory (raw device pointers)."""
        st = VfFrameStats() if read_stats else None
        self._chk("vf_process_frame_device",
                  self._L.vf_process_frame_device(self._h, C.c_void_p(d_depth),
                                                  C.c_void_p(d_rgb) if d_rgb else None,
                                                  C.byref(st) if st is not None else None))
        return FrameStats.from_c(st) if st is not None else None

    def synchronize(self):
        self._chk("vf_synchronize", self._L.vf_synchronize(self._h))

    def pose(self) -> np.ndarray:
        out = np.zeros(12)
        self._chk("vf_get_pose", self._L.vf_get_pose(self._h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def set_pose(self, pose) -> None:
        p = _pose(pose)
        self._chk("vf_set_pose", self._L.vf_set_pose(self._h, p.ctypes.data_as(C.POINTER(C.c_double))))

    def frame_count(self) -> int:
        return int(self._L.vf_frame_count(self._h))

    def settings(self) -> EngineSettings:
        return self._settings

    def tracking_state(self):
        """(points, normals) world-space maps, each H x W x 4 float32 (w = validity)."""
        pts = np.zeros((self.height, self.width, 4), np.float32)
        nrm = np.zeros((self.height, self.width, 4), np.float32)
        self._chk("vf_get_maps", self._L.vf_get_maps(self._h, _ptr(pts), _ptr(nrm)))
        return pts, nrm

    def set_maps(self, points, normals, render_pose) -> None:
        p = _f32(points, (self.height, self.width, 4))
        n = _f32(normals, (self.height, self.width, 4))
        rp = _pose(render_pose)
        self._chk("vf_set_maps", self._L.vf_set_maps(self._h, _ptr(p), _ptr(n),
                                                     rp.ctypes.data_as(C.POINTER(C.c_double))))

    # -- swap engine (swap.hpp) --
    def swap_states(self) -> np.ndarray:
        """Per-entry SwapState codes (swap.hpp:19-25)."""
        out = np.zeros(self._settings.entry_count, np.uint8)
        self._chk("vf_swap_states", self._L.vf_swap_states(self._h, _ptr(out)))
        return out

    def store_count(self) -> int:
        """BlockStore::stored_count (block_store.hpp:34-38)."""
        return int(self._chk("vf_swap_stored_count", self._L.vf_swap_stored_count(self._h)))

    def store_read(self, entry: int):
        """BlockStore::read of one entry (VoxelCodec bytes), or None when not stored."""
        payload = np.zeros(512 * (7 if self._settings.voxel_type == VOXEL_TYPE_S_RGB else 3), np.uint8)
        rc = self._chk("vf_swap_store_read", self._L.vf_swap_store_read(self._h, int(entry), _ptr(payload)))
        return payload if rc == 1 else None

    def store(self) -> dict:
        """{entry index: payload} for every stored block."""
        e = self.entries()
        out = {}
        for i in np.nonzero(e["block_state"] == -1)[0]:
            p = self.store_read(int(i))
            if p is not None:
                out[int(i)] = p
        return out

    def swap_drain(self, cap: int = 1 << 16):
        """Entries swapped out since the last drain, in swap-out order, and
        how many fell out of the journal ring (vf_swap_drain)."""
        out = np.zeros(cap, np.int32)
        lost = C.c_long()
        n = self._L.vf_swap_drain(self._h, out.ctypes.data_as(C.POINTER(C.c_int)), cap, C.byref(lost))
        if n < 0:
            check("vf_swap_drain", n, self._h)
        return out[:n].copy(), lost.value

    def save_store(self, path: str) -> None:
        """Write the host store as a VXBS file (block_store.hpp:14-53)."""
        self._chk("vf_swap_save_store", self._L.vf_swap_save_store(self._h, str(path).encode()))

    def load_store(self, path: str) -> None:
        """load_block_store_file into the host store (block_store.cpp:143-181)."""
        self._chk("vf_swap_load_store", self._L.vf_swap_load_store(self._h, str(path).encode()))

    def surface_points(self):
        """TrackingState::surface_points / surface_colors (tracking_state.hpp:30-31):
        the stride-4 surface samples of the last render (colour voxels), n x 3 each."""
        n = int(self._chk("vf_get_surface_points", self._L.vf_get_surface_points(self._h, None, None, 0)))
        pts = np.zeros((n, 3), np.float32)
        cols = np.zeros((n, 3), np.float32)
        if n:
            self._chk("vf_get_surface_points", self._L.vf_get_surface_points(self._h, _ptr(pts), _ptr(cols), n))
        return pts, cols

    def forward_project_points(self) -> None:
        """forward_project_points (raycast.hpp:495-509) over the current maps."""
        self._chk("vf_stage_forward_project", self._L.vf_stage_forward_project(self._h))

    def get_image(self, mode: int = 0) -> np.ndarray:
        """IPipeline::get_image(DisplayMode) (pipeline.hpp:74): 0 raycast, 1 depth
        colourised, 2 RGB passthrough, 3 raycast in shaded grey; H x W x 3 u8."""
        out = np.zeros((self.height, self.width, 3), np.uint8)
        self._chk("vf_render_image", self._L.vf_render_image(self._h, int(mode), _ptr(out)))
        return out

    def volume_digest(self) -> int:
        out = C.c_uint64()
        self._chk("vf_volume_digest", self._L.vf_volume_digest(self._h, C.byref(out)))
        return int(out.value)

    # -- state export / import --
    def entries(self) -> np.ndarray:
        out = np.zeros(self._L.vf_entry_count(self._h), ENTRY_DTYPE)
        self._chk("vf_export_entries", self._L.vf_export_entries(self._h, _ptr(out)))
        return out

    def voxels(self) -> np.ndarray:
        out = np.zeros(self._L.vf_voxel_bytes(self._h), np.uint8)
        self._chk("vf_export_voxels", self._L.vf_export_voxels(self._h, _ptr(out)))
        return out

    def free_stacks(self):
        s = self._settings
        vs = np.zeros(s.block_count, np.int32)
        es = np.zeros(s.excess_count, np.int32)
        vt, et = C.c_int(), C.c_int()
        self._chk("vf_export_free_stacks",
                  self._L.vf_export_free_stacks(self._h, C.byref(vt), _ptr(vs), C.byref(et), _ptr(es)))
        return vt.value, vs, et.value, es

    def import_state(self, entries, voxels, vba_top, vba_slots, excess_top, excess_slots) -> None:
        e = np.ascontiguousarray(entries)
        v = np.ascontiguousarray(voxels)
        vs = np.ascontiguousarray(vba_slots, np.int32)
        es = np.ascontiguousarray(excess_slots, np.int32)
        self._chk("vf_import_state", self._L.vf_import_state(self._h, _ptr(e), _ptr(v), int(vba_top), _ptr(vs),
                                                             int(excess_top), _ptr(es)))

    def visible_list(self) -> np.ndarray:
        n = self._L.vf_export_visible_list(self._h, None, 0)
        self._chk("vf_export_visible_list", n)
        out = np.zeros(n, np.int32)
        if n:
            self._L.vf_export_visible_list(self._h, _ptr(out), n)
        return out

    def ranges(self) -> np.ndarray:
        n = self._L.vf_export_ranges(self._h, None)
        out = np.zeros((n, 2), np.float32)
        self._chk("vf_export_ranges", self._L.vf_export_ranges(self._h, _ptr(out)))
        return out

    # -- stage templates --
    def allocate(self, depth_m, pose) -> VfAllocStats:
        """mark_blocks + perform_allocations + build_visible_list."""
        d = _f32(depth_m, (self.height, self.width))
        p = _pose(pose)
        st = VfAllocStats()
        self._chk("vf_stage_allocate", self._L.vf_stage_allocate(self._h, _ptr(d), p.ctypes.data_as(
            C.POINTER(C.c_double)), C.byref(st)))
        return st

    def integrate(self, depth_m, rgb, pose) -> None:
        """integrate_frame over the current visible list."""
        d = _f32(depth_m, (self.height, self.width))
        c = None if rgb is None else np.ascontiguousarray(rgb, dtype=np.uint8)
        p = _pose(pose)
        self._chk("vf_stage_integrate", self._L.vf_stage_integrate(self._h, _ptr(d), _ptr(c),
                                                                   p.ctypes.data_as(C.POINTER(C.c_double))))

    def raycast(self, pose) -> None:
        """create_expected_depths + render_maps."""
        p = _pose(pose)
        self._chk("vf_stage_raycast", self._L.vf_stage_raycast(self._h, p.ctypes.data_as(C.POINTER(C.c_double))))

    def icp_track(self, depth_m, initial=None):
        """build_depth_pyramid + icp_track(pyramid, state, settings, initial) against the current maps."""
        d = _f32(depth_m, (self.height, self.width))
        pose = np.zeros(12)
        init = None if initial is None else _pose(initial)
        it, valid, ok = C.c_int(), C.c_int(), C.c_int()
        cost = C.c_double()
        self._chk("vf_stage_icp", self._L.vf_stage_icp(
            self._h, _ptr(d), None if init is None else init.ctypes.data_as(C.POINTER(C.c_double)),
            pose.ctypes.data_as(C.POINTER(C.c_double)), C.byref(it), C.byref(cost), C.byref(valid), C.byref(ok)))
        return dict(pose=pose, ok=bool(ok.value), iterations=it.value, cost=cost.value, valid_points=valid.value)

    def _track_stage(self, fn, first, initial):
        out = np.zeros(12)
        it, cost, valid, ok = C.c_int(), C.c_double(), C.c_int(), C.c_int()
        ini = _pose(initial)
        self._chk(fn, getattr(self._L, fn)(self._h, _ptr(first), ini.ctypes.data_as(C.POINTER(C.c_double)),
                                           out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(it), C.byref(cost),
                                           C.byref(valid), C.byref(ok)))
        return out, it.value, cost.value, valid.value, bool(ok.value)

    def ren_refine(self, depth_m, initial):
        """ren_refine (ren_tracker.hpp:30-120) against the current volume:
        (pose, iterations, cost, valid_points, ok)."""
        return self._track_stage("vf_stage_ren", _f32(depth_m, (self.height, self.width)), initial)

    def color_track(self, rgb, initial):
        """build_color_pyramid + color_track (color_tracker.hpp:107-154) of the
        current surface list: (pose, iterations, cost, valid_points, ok)."""
        c = np.ascontiguousarray(rgb, dtype=np.uint8)
        return self._track_stage("vf_stage_color", c, initial)

    def icp_trace(self) -> np.ndarray:
        """Rows of 48: level, iter, 21 H, 6 g, cost, count, rotation_only, eval cam->world pose (12), 4 timers."""
        n = self._L.vf_icp_trace(self._h, None, 0)
        out = np.zeros((max(n, 0), 48))
        if n > 0:
            self._L.vf_icp_trace(self._h, _ptr(out), n)
        return out

    def depth_pyramid(self, depth_m) -> list:
        d = _f32(depth_m, (self.height, self.width))
        sizes, w, h = [], self.width, self.height
        for _ in range(self._settings.hierarchy_levels):
            sizes.append((h, w))
            w, h = (w + 1) // 2, (h + 1) // 2
        out = np.zeros(sum(a * b for a, b in sizes), np.float32)
        self._chk("vf_depth_pyramid", self._L.vf_depth_pyramid(self._h, _ptr(d), _ptr(out)))
        res, off = [], 0
        for hh, ww in sizes:
            res.append(out[off:off + hh * ww].reshape(hh, ww))
            off += hh * ww
        return res

    # -- profiling --
    def set_profiling(self, enabled: bool) -> None:
        self._chk("vf_set_profiling", self._L.vf_set_profiling(self._h, int(enabled)))

    def raycast_counters(self) -> dict:
        """Re-run the last raycast with counters (measurement only, same maps)."""
        out = (C.c_ulonglong * 4)()
        self._chk("vf_raycast_counters", self._L.vf_raycast_counters(self._h, out))
        return {"table_probes": out[0], "voxel_reads": out[1], "rays": out[2], "hits": out[3]}

    def alloc_counters(self) -> dict:
        """mark_blocks' DDA walk over the last frame without requests (measurement only)."""
        out = (C.c_ulonglong * 3)()
        self._chk("vf_alloc_counters", self._L.vf_alloc_counters(self._h, out))
        return {"pixels": out[0], "cells_probed": out[1], "cells_missing": out[2]}

    def set_stage_timing(self, enabled: bool) -> None:
        """Fill FrameStats.ms_tracking .. ms_raycast on every blocking frame
        (pipeline.hpp:56-57) from event records inside the frame graph."""
        self._chk("vf_set_stage_timing", self._L.vf_set_stage_timing(self._h, int(enabled)))

    def stage_times(self):
        ms = np.zeros(8)
        n = C.c_long()
        self._chk("vf_stage_times", self._L.vf_stage_times(self._h, ms.ctypes.data_as(C.POINTER(C.c_double)),
                                                           C.byref(n)))
        return ms, n.value

    def kernel_launches_per_frame(self, tracking_frame: bool) -> int:
        return self._chk("vf_kernel_launches_per_frame",
                         self._L.vf_kernel_launches_per_frame(self._h, int(tracking_frame)))


def make_pipeline(settings: EngineSettings, calib: Calibration, device: int = 0) -> Pipeline:
    """make_pipeline (pipeline.hpp:86; src/pipeline_factory.cpp:18-30), hash backend."""
    return Pipeline(settings, calib, device)


# ---------------------------------------------------------------------------
# device buffers + synthetic input rendering (bench inputs, no torch needed)
# ---------------------------------------------------------------------------
class DeviceBuffer:
    def __init__(self, nbytes: int):
        L = _abi.load()
        self.nbytes = int(nbytes)
        self.ptr = L.vf_device_alloc(self.nbytes)
        if not self.ptr:
            raise _abi.VoxfuseError("vf_device_alloc", _abi.VF_ERR_CUDA)

    def free(self):
        if self.ptr:
            _abi.load().vf_device_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def to_host(self, dtype, shape) -> np.ndarray:
        out = np.zeros(shape, dtype)
        check("vf_memcpy_d2h", _abi.load().vf_memcpy_d2h(_ptr(out), C.c_void_p(self.ptr), out.nbytes))
        return out

    def from_host(self, arr: np.ndarray) -> None:
        a = np.ascontiguousarray(arr)
        check("vf_memcpy_h2d", _abi.load().vf_memcpy_h2d(C.c_void_p(self.ptr), _ptr(a), a.nbytes))


def render_synthetic(pose, intr: Intrinsics, spheres, planes, d_depth: int, d_rgb: int | None = None,
                     near: float = 0.05, far: float = 100.0, device: int = 0) -> None:
    """render_synthetic_depth / _rgb (proj/src/synthetic.cpp) on the GPU into device buffers."""
    sp = np.ascontiguousarray(spheres, np.float64)
    pl = np.ascontiguousarray(planes, np.float64)
    p = _pose(pose)
    ci = intr.to_c()
    check("vf_render_synthetic", _abi.load().vf_render_synthetic(
        device, len(sp), _ptr(sp), len(pl), _ptr(pl), p.ctypes.data_as(C.POINTER(C.c_double)), C.byref(ci),
        near, far, C.c_void_p(d_depth), C.c_void_p(d_rgb) if d_rgb else None))
