"""TEST / BASELINE INFRASTRUCTURE ONLY — ctypes bindings of the CPU oracle.

Two libraries share one binding because their C ABIs mirror each other:

* ``oracle/liboracle.so`` — the plain-C restatement (vf_oracle.c), the parity checker;
* ``oracle/_ref/libvoxfuse_ref.so`` — the reference's own sources compiled
  unmodified against oracle/eigen_shim (ref_driver.cpp), which pins the
  restatement and serves as the CPU baseline ("kind": "reference").

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libvoxfuse_ref.so"
# the same reference build with Eigen's halving reduction association
# (eigen_shim VF_SHIM_HALVING; `make -C oracle ref_halving`)
REF_HALVING_SO = HERE / "_ref_halving" / "libvoxfuse_ref.so"

ENTRY_DTYPE = np.dtype(
    [("x", "<i2"), ("y", "<i2"), ("z", "<i2"), ("pad", "<i2"), ("offset", "<i4"), ("block_state", "<i4")]
)


class Config(C.Structure):
    _fields_ = [
        ("voxel_type", C.c_int),
        ("voxel_size", C.c_float),
        ("mu", C.c_float),
        ("max_weight", C.c_int),
        ("stop_integrating_at_max", C.c_int),
        ("bucket_count", C.c_int),
        ("bucket_size", C.c_int),
        ("excess_count", C.c_int),
        ("block_count", C.c_int),
        ("near_clip", C.c_float),
        ("far_clip", C.c_float),
        ("margin_px", C.c_int),
        ("swap_margin_px", C.c_int),
        ("levels", C.c_int),
        ("rotation_only_levels", C.c_int),
        ("max_iterations", C.c_int),
        ("min_valid_points", C.c_int),
        ("icp_dist_threshold", C.c_float),
        ("convergence_eps", C.c_float),
        ("max_condition", C.c_double),
        ("fx", C.c_double),
        ("fy", C.c_double),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("width", C.c_int),
        ("height", C.c_int),
        ("rgb_fx", C.c_double),
        ("rgb_fy", C.c_double),
        ("rgb_cx", C.c_double),
        ("rgb_cy", C.c_double),
        ("rgb_width", C.c_int),
        ("rgb_height", C.c_int),
        ("rgb_to_depth", C.c_double * 12),
        ("use_swapping", C.c_int),
        ("swap_buffer_blocks", C.c_int),
        ("tracker_type", C.c_int),
        ("ren_sigma", C.c_float),
        ("skip_points", C.c_int),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("frame", C.c_int),
        ("tracking_ok", C.c_int),
        ("tracking_iterations", C.c_int),
        ("blocks_allocated", C.c_int),
        ("allocation_dropped", C.c_int),
        ("visible_blocks", C.c_int),
        ("tracking_cost", C.c_double),
        ("pose", C.c_double * 12),
        ("ms_tracking", C.c_double),
        ("ms_allocation", C.c_double),
        ("ms_integration", C.c_double),
        ("ms_raycast", C.c_double),
        ("ms_total", C.c_double),
        ("swapped_in", C.c_int),
        ("swapped_out", C.c_int),
        ("bytes_in", C.c_uint64),
        ("bytes_out", C.c_uint64),
        ("ms_swapping", C.c_double),
    ]


class AllocStats(C.Structure):
    _fields_ = [("requested", C.c_int), ("allocated", C.c_int), ("dropped_vba_full", C.c_int),
                ("dropped_excess_full", C.c_int)]


def make_config(cfg) -> Config:
    """Config from a paper_1410_0925_b200.scene.BenchConfig."""
    fx, fy, cx, cy, w, h = cfg.intrinsics
    c = Config()
    c.voxel_type = cfg.voxel_type
    c.voxel_size = cfg.voxel_size
    c.mu = cfg.mu
    c.max_weight = cfg.max_weight
    c.stop_integrating_at_max = 1 if getattr(cfg, "stop_integrating_at_max", False) else 0
    c.bucket_count = cfg.hash.bucket_count
    c.bucket_size = cfg.hash.bucket_size
    c.excess_count = cfg.hash.excess_count
    c.block_count = cfg.hash.block_count
    c.near_clip = cfg.near_clip
    c.far_clip = cfg.far_clip
    c.margin_px = cfg.margin_px
    c.swap_margin_px = cfg.swap_margin_px
    c.levels = cfg.levels
    c.rotation_only_levels = cfg.rotation_only_levels
    c.max_iterations = cfg.max_iterations
    c.min_valid_points = cfg.min_valid_points
    c.icp_dist_threshold = cfg.icp_dist_threshold
    c.convergence_eps = cfg.convergence_eps
    c.max_condition = cfg.max_condition
    c.fx, c.fy, c.cx, c.cy, c.width, c.height = fx, fy, cx, cy, w, h
    c.rgb_fx, c.rgb_fy, c.rgb_cx, c.rgb_cy, c.rgb_width, c.rgb_height = fx, fy, cx, cy, w, h
    ident = [1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0]
    for i, v in enumerate(ident):
        c.rgb_to_depth[i] = v
    c.use_swapping = 1 if getattr(cfg, "use_swapping", False) else 0
    c.swap_buffer_blocks = getattr(cfg, "swap_buffer_blocks", 100)
    c.tracker_type = {"icp": 0, "color": 1, "icp_ren": 2}[getattr(cfg, "tracker", "icp")]
    c.ren_sigma = 10.0
    c.skip_points = 0
    return c


def _p(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


class _Lib:
    prefix = ""

    def __init__(self, path: Path):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(str(path))
        p = self.prefix
        L = self.lib
        getattr(L, p + "create").restype = C.c_void_p
        getattr(L, p + "create").argtypes = [C.POINTER(Config), C.c_int]
        getattr(L, p + "destroy").argtypes = [C.c_void_p]
        getattr(L, p + "process").argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(Stats)]
        getattr(L, p + "process").restype = C.c_int
        getattr(L, p + "get_pose").argtypes = [C.c_void_p, C.c_void_p]
        getattr(L, p + "get_maps").argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        getattr(L, p + "get_maps").restype = C.c_int
        for fn in ("export_entries", "export_voxels", "visible_list", "export_ranges"):
            getattr(L, p + fn).argtypes = [C.c_void_p, C.c_void_p]
            getattr(L, p + fn).restype = C.c_long
        getattr(L, p + "digest").argtypes = [C.c_void_p]
        getattr(L, p + "digest").restype = C.c_uint64
        getattr(L, p + "allocated_blocks").argtypes = [C.c_void_p]
        getattr(L, p + "allocated_blocks").restype = C.c_long
        for fn in ("render_depth", "render_rgb"):
            getattr(L, p + fn).argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p] + [C.c_double] * 4 + [
                C.c_int, C.c_int, C.c_double, C.c_double, C.c_void_p]
        getattr(L, p + "depth_pyramid").argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        getattr(L, p + "surface_points").argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        getattr(L, p + "surface_points").restype = C.c_long
        getattr(L, p + "swap_states").argtypes = [C.c_void_p, C.c_void_p]
        getattr(L, p + "swap_states").restype = C.c_long
        getattr(L, p + "store_read").argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        getattr(L, p + "store_read").restype = C.c_int
        getattr(L, p + "store_count").argtypes = [C.c_void_p]
        getattr(L, p + "store_count").restype = C.c_long


class OracleLib(_Lib):
    prefix = "vfo_"

    def __init__(self, path: Path = ORACLE_SO):
        super().__init__(path)
        L = self.lib
        L.vfo_stage_allocate.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(AllocStats)]
        L.vfo_stage_integrate.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.vfo_stage_raycast.argtypes = [C.c_void_p, C.c_void_p]
        L.vfo_stage_icp.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int),
                                    C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.vfo_stage_icp.restype = C.c_int
        L.vfo_stage_icp_init.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int),
                                         C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.vfo_stage_icp_init.restype = C.c_int
        L.vfo_set_pose.argtypes = [C.c_void_p, C.c_void_p]
        L.vfo_set_maps.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.vfo_free_stacks.argtypes = [C.c_void_p] * 5
        L.vfo_icp_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_long]
        L.vfo_icp_trace.restype = C.c_long
        L.vfo_hash_block_pos.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint32]
        L.vfo_hash_block_pos.restype = C.c_uint32
        L.vfo_stage_forward_project.argtypes = [C.c_void_p]
        L.vfo_render_image.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.vfo_render_image.restype = C.c_int
        L.vfo_colourize_depth.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]


class RefLib(_Lib):
    prefix = "vfr_"

    def __init__(self, path: Path = REF_SO):
        super().__init__(path)
        L = self.lib
        L.vfr_set_threads.argtypes = [C.c_int]
        L.vfr_get_threads.restype = C.c_int
        L.vfr_icp_track.argtypes = [C.POINTER(Config)] + [C.c_void_p] * 5 + [
            C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.vfr_icp_track.restype = C.c_int
        L.vfr_image.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.vfr_image.restype = C.c_int
        assert L.vfr_sizeof_config() == C.sizeof(Config), "vfr_config layout mismatch"
        assert L.vfr_sizeof_stats() == C.sizeof(Stats), "vfr_stats layout mismatch"


_cache: dict = {}


def oracle_lib() -> OracleLib:
    if "o" not in _cache:
        _cache["o"] = OracleLib()
    return _cache["o"]


def ref_lib() -> RefLib:
    if "r" not in _cache:
        _cache["r"] = RefLib()
    return _cache["r"]


def ref_available() -> bool:
    return REF_SO.exists()


def ref_halving_lib() -> RefLib:
    if "rh" not in _cache:
        _cache["rh"] = RefLib(REF_HALVING_SO)
    return _cache["rh"]


def ref_halving_available() -> bool:
    return REF_HALVING_SO.exists()


class Volume:
    """One oracle / reference context (a HashVolume plus pipeline state)."""

    def __init__(self, lib: _Lib, cfg, tracking: bool):
        self.L = lib
        self.cfg = cfg
        self.c = make_config(cfg)
        self.p = lib.prefix
        self.h = getattr(lib.lib, self.p + "create")(C.byref(self.c), 1 if tracking else 0)
        if not self.h:
            raise RuntimeError("create failed")
        self.width, self.height = cfg.width, cfg.height

    def close(self):
        if self.h:
            getattr(self.L.lib, self.p + "destroy")(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _f(self, name):
        return getattr(self.L.lib, self.p + name)

    def process(self, depth: np.ndarray, rgb: np.ndarray | None = None, pose: np.ndarray | None = None) -> Stats:
        st = Stats()
        depth = np.ascontiguousarray(depth, dtype=np.float32)
        rgb = None if rgb is None else np.ascontiguousarray(rgb, dtype=np.uint8)
        pose = None if pose is None else np.ascontiguousarray(pose, dtype=np.float64)
        rc = self._f("process")(self.h, _p(depth, C.c_float), _p(rgb, C.c_uint8), _p(pose, C.c_double), C.byref(st))
        if rc != 0:
            raise RuntimeError(f"process failed: {rc}")
        return st

    def pose(self) -> np.ndarray:
        out = np.zeros(12)
        self._f("get_pose")(self.h, _p(out, C.c_double))
        return out

    def maps(self):
        n = self.width * self.height
        pts = np.zeros((n, 4), np.float32)
        nrm = np.zeros((n, 4), np.float32)
        if self._f("get_maps")(self.h, _p(pts, C.c_float), _p(nrm, C.c_float)) != 0:
            return None, None
        return pts.reshape(self.height, self.width, 4), nrm.reshape(self.height, self.width, 4)

    def entries(self) -> np.ndarray:
        n = self._f("export_entries")(self.h, None)
        out = np.zeros(n, ENTRY_DTYPE)
        self._f("export_entries")(self.h, out.ctypes.data_as(C.c_void_p))
        return out

    def voxels(self) -> np.ndarray:
        n = self._f("export_voxels")(self.h, None)
        out = np.zeros(n, np.uint8)
        self._f("export_voxels")(self.h, out.ctypes.data_as(C.c_void_p))
        return out

    def visible_list(self) -> np.ndarray:
        n = self._f("visible_list")(self.h, None)
        out = np.zeros(n, np.int32)
        if n:
            self._f("visible_list")(self.h, out.ctypes.data_as(C.c_void_p))
        return out

    def ranges(self) -> np.ndarray:
        n = self._f("export_ranges")(self.h, None)
        out = np.zeros((max(n, 0), 2), np.float32)
        if n > 0:
            self._f("export_ranges")(self.h, out.ctypes.data_as(C.c_void_p))
        return out

    def digest(self) -> int:
        return int(self._f("digest")(self.h))

    def swap_states(self) -> np.ndarray:
        """Per-entry SwapState codes (swap.hpp:19-25)."""
        out = np.zeros(self.cfg.hash.entry_count, np.uint8)
        if self._f("swap_states")(self.h, out.ctypes.data_as(C.c_void_p)) < 0:
            return None
        return out

    def store_count(self) -> int:
        return int(self._f("store_count")(self.h))

    def store_read(self, idx: int):
        """Host store payload of entry idx (VoxelCodec bytes), or None."""
        payload = np.zeros(512 * (7 if self.cfg.voxel_type == 2 else 3), np.uint8)
        if self._f("store_read")(self.h, int(idx), payload.ctypes.data_as(C.c_void_p)) != 1:
            return None
        return payload

    def store(self) -> dict:
        """{entry index: payload} for every stored block."""
        st = self.swap_states()
        out = {}
        e = self.entries()
        for i in np.nonzero(e["block_state"] == -1)[0]:
            p = self.store_read(int(i))
            if p is not None:
                out[int(i)] = p
        return out

    def stage_track(self, which: str, frame: np.ndarray, initial: np.ndarray):
        """Reference ren_refine ("ren", depth) / color_track ("color", rgb) on this
        (known-pose) context: (pose, iterations, cost, valid_points, ok)."""
        f = self.L.lib.vfr_stage_track
        f.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int),
                      C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        frame = np.ascontiguousarray(frame)
        ini = np.ascontiguousarray(initial, np.float64)
        out = np.zeros(12)
        it, cost, valid, ok = C.c_int(), C.c_double(), C.c_int(), C.c_int()
        f(self.h, 1 if which == "color" else 0, frame.ctypes.data_as(C.c_void_p), ini.ctypes.data_as(C.c_void_p),
          out.ctypes.data_as(C.c_void_p), C.byref(it), C.byref(cost), C.byref(valid), C.byref(ok))
        return out, it.value, cost.value, valid.value, bool(ok.value)

    def surface_points(self):
        """TrackingState::surface_points / surface_colors (n x 3 float32 each)."""
        n = self._f("surface_points")(self.h, None, None)
        pts = np.zeros((n, 3), np.float32)
        cols = np.zeros((n, 3), np.float32)
        if n:
            self._f("surface_points")(self.h, _p(pts, C.c_float), _p(cols, C.c_float))
        return pts, cols

    def image(self, mode: int = 0) -> np.ndarray | None:
        """render_image of the current maps: mode 0 raycast (colour for VoxelSRgb),
        3 shaded grey (vf_display_mode numbering)."""
        out = np.zeros((self.height, self.width, 3), np.uint8)
        if self.p == "vfo_":
            rc = self.L.lib.vfo_render_image(self.h, 1 if mode == 0 else 0, out.ctypes.data_as(C.c_void_p))
        else:
            rc = self.L.lib.vfr_image(self.h, mode, out.ctypes.data_as(C.c_void_p))
        return out if rc == 0 else None

    def allocated_blocks(self) -> int:
        return int(self._f("allocated_blocks")(self.h))


def render_depth(lib: _Lib, cfg, pose: np.ndarray, spheres, planes, near=0.05, far=100.0) -> np.ndarray:
    fx, fy, cx, cy, w, h = cfg.intrinsics
    out = np.zeros((h, w), np.float32)
    sp = np.ascontiguousarray(spheres, np.float64)
    pl = np.ascontiguousarray(planes, np.float64)
    pose = np.ascontiguousarray(pose, np.float64)
    getattr(lib.lib, lib.prefix + "render_depth")(len(sp), _p(sp, C.c_double), len(pl), _p(pl, C.c_double),
                                                   _p(pose, C.c_double), fx, fy, cx, cy, w, h, near, far,
                                                   _p(out, C.c_float))
    return out


def render_rgb(lib: _Lib, cfg, pose: np.ndarray, spheres, planes, near=0.05, far=100.0) -> np.ndarray:
    fx, fy, cx, cy, w, h = cfg.intrinsics
    out = np.zeros((h, w, 3), np.uint8)
    sp = np.ascontiguousarray(spheres, np.float64)
    pl = np.ascontiguousarray(planes, np.float64)
    pose = np.ascontiguousarray(pose, np.float64)
    getattr(lib.lib, lib.prefix + "render_rgb")(len(sp), _p(sp, C.c_double), len(pl), _p(pl, C.c_double),
                                                 _p(pose, C.c_double), fx, fy, cx, cy, w, h, near, far,
                                                 _p(out, C.c_uint8))
    return out


def colourize_depth(depth: np.ndarray) -> np.ndarray:
    """Pipeline::colourize_depth (pipeline_impl.hpp:225-239), oracle restatement."""
    depth = np.ascontiguousarray(depth, dtype=np.float32)
    h, w = depth.shape
    out = np.zeros((h, w, 3), np.uint8)
    oracle_lib().lib.vfo_colourize_depth(depth.ctypes.data_as(C.c_void_p), w, h, out.ctypes.data_as(C.c_void_p))
    return out


def disparity_to_depth(lib: _Lib, disp: np.ndarray, a: float, b: float, fx: float, max_depth: float = 8.0):
    """disparity_image_to_depth: oracle (vfo_) or reference (vfr_)."""
    disp = np.ascontiguousarray(disp, dtype=np.uint16)
    out = np.zeros(disp.shape, np.float32)
    vp = C.c_void_p
    if lib.prefix == "vfo_":
        f = lib.lib.vfo_disparity_to_depth
        f.argtypes = [vp, C.c_long, C.c_double, C.c_double, C.c_double, C.c_float, vp]
        f(disp.ctypes.data_as(vp), disp.size, a, b, fx, max_depth, out.ctypes.data_as(vp))
    else:
        f = lib.lib.vfr_disparity_to_depth
        f.argtypes = [vp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_float, vp]
        f(disp.ctypes.data_as(vp), disp.shape[1], disp.shape[0], a, b, fx, max_depth, out.ctypes.data_as(vp))
    return out


def depth_pyramid(lib: _Lib, depth: np.ndarray, levels: int) -> list:
    h, w = depth.shape
    sizes = []
    ww, hh = w, h
    for _ in range(levels):
        sizes.append((hh, ww))
        ww, hh = (ww + 1) // 2, (hh + 1) // 2
    out = np.zeros(sum(a * b for a, b in sizes), np.float32)
    d = np.ascontiguousarray(depth, np.float32)
    getattr(lib.lib, lib.prefix + "depth_pyramid")(_p(d, C.c_float), w, h, levels, _p(out, C.c_float))
    res, off = [], 0
    for hh, ww in sizes:
        res.append(out[off:off + hh * ww].reshape(hh, ww))
        off += hh * ww
    return res
