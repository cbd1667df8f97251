"""ctypes binding of the C ABI in include/voxfuse_b200.h.

Loads the in-tree ``lib/libvoxfuse_b200.so`` and fails loudly if it is missing:
the product path has no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("VOXFUSE_B200_LIB", Path(__file__).resolve().parent / "lib" / "libvoxfuse_b200.so"))

VF_OK = 0
VF_ERR_INVALID = -1
VF_ERR_CUDA = -2
VF_ERR_NO_DEVICE = -3
VF_ERR_STATE = -4
VF_ERR_OVERFLOW = -5

STATUS_NAMES = {
    VF_OK: "VF_OK",
    VF_ERR_INVALID: "VF_ERR_INVALID",
    VF_ERR_CUDA: "VF_ERR_CUDA",
    VF_ERR_NO_DEVICE: "VF_ERR_NO_DEVICE",
    VF_ERR_STATE: "VF_ERR_STATE",
    VF_ERR_OVERFLOW: "VF_ERR_OVERFLOW",
}

# Every symbol include/voxfuse_b200.h declares (checked by tests/test_abi.py).
ABI_VERSION = 3  # VF_ABI_VERSION in include/voxfuse_b200.h

EXPORTS = [
    "vf_abi_version", "vf_struct_size", "vf_default_settings", "vf_create", "vf_destroy", "vf_last_error",
    "vf_process_frame", "vf_process_frame_device", "vf_synchronize", "vf_read_stats",
    "vf_submit_frame", "vf_submit_raw_frame", "vf_collect_frame", "vf_frames_in_flight",
    "vf_process_raw_frame", "vf_process_raw_frame_device", "vf_disparity_to_depth",
    "vf_set_pose", "vf_get_pose", "vf_frame_count", "vf_get_maps", "vf_set_maps", "vf_volume_digest",
    "vf_get_surface_points", "vf_stage_forward_project", "vf_render_image",
    "vf_swap_states", "vf_swap_stored_count", "vf_swap_store_read", "vf_swap_drain", "vf_swap_save_store", "vf_swap_load_store",
    "vf_entry_count", "vf_voxel_bytes", "vf_export_entries", "vf_export_voxels", "vf_export_free_stacks",
    "vf_import_state", "vf_export_visible_list", "vf_export_ranges",
    "vf_stage_allocate", "vf_stage_integrate", "vf_stage_raycast", "vf_stage_icp", "vf_icp_trace",
    "vf_stage_ren", "vf_stage_color",
    "vf_depth_pyramid", "vf_render_synthetic",
    "vf_shard_owner", "vf_shard_p2p_handles", "vf_shard_p2p_link", "vf_shard_p2p_link_local", "vf_shard_icp_handle", "vf_shard_icp_link", "vf_shard_icp_link_local", "vf_shard_nccl_unique_id", "vf_shard_attach_nccl", "vf_shard_composite_local",
    "vf_device_alloc", "vf_device_free", "vf_memcpy_h2d", "vf_memcpy_d2h", "vf_host_alloc_pinned",
    "vf_host_free_pinned", "vf_event_record", "vf_event_elapsed_ms", "vf_set_profiling", "vf_set_stage_timing", "vf_raycast_counters", "vf_alloc_counters", "vf_stage_times",
    "vf_kernel_launches_per_frame", "vf_readback_bytes", "vf_flush_l2", "vf_flush_time", "vf_last_modified_voxels",
    "vf_selftest_division",
]


class VfSettings(C.Structure):
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
        ("visibility_margin_px", C.c_int),
        ("swap_margin_px", C.c_int),
        ("hierarchy_levels", C.c_int),
        ("rotation_only_levels", C.c_int),
        ("max_iterations", C.c_int),
        ("min_valid_points", C.c_int),
        ("icp_dist_threshold", C.c_float),
        ("convergence_eps", C.c_float),
        ("max_condition", C.c_double),
        ("tracking", C.c_int),
        ("use_graphs", C.c_int),
        ("shard_count", C.c_int),
        ("shard_index", C.c_int),
        ("shard_shift", C.c_int),
        ("shard_halo", C.c_int),
        ("use_swapping", C.c_int),
        ("swap_buffer_blocks", C.c_int),
        ("swap_host_blocks", C.c_int),
        ("max_depth", C.c_float),
        ("tracker_type", C.c_int),
        ("ren_sigma", C.c_float),
        ("skip_points", C.c_int),
        ("integration_mode", C.c_int),
        ("shard_icp", C.c_int),
        ("icp_max_ctas", C.c_int),
        ("tracker_exact_solve", C.c_int),
    ]


class VfIntrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int), ("height", C.c_int)]


class VfCalib(C.Structure):
    _fields_ = [("rgb", VfIntrinsics), ("depth", VfIntrinsics), ("rgb_to_depth", C.c_double * 12),
                ("disparity_a", C.c_double), ("disparity_b", C.c_double)]


class VfFrameStats(C.Structure):
    _fields_ = [
        ("frame", C.c_int),
        ("tracking_ok", C.c_int),
        ("tracking_iterations", C.c_int),
        ("blocks_allocated", C.c_int),
        ("allocation_dropped", C.c_int),
        ("visible_blocks", C.c_int),
        ("tracking_cost", C.c_double),
        ("tracking_valid_points", C.c_int),
        ("allocation_requested", C.c_int),
        ("allocated_total", C.c_int),
        ("error_flags", C.c_int),
        ("pose", C.c_double * 12),
        ("ms_tracking", C.c_double),
        ("ms_allocation", C.c_double),
        ("ms_integration", C.c_double),
        ("ms_swapping", C.c_double),
        ("ms_raycast", C.c_double),
        ("ms_total", C.c_double),
        ("swapped_in", C.c_int),
        ("swapped_out", C.c_int),
        ("swap_bytes_in", C.c_uint64),
        ("swap_bytes_out", C.c_uint64),
    ]


class VfAllocStats(C.Structure):
    _fields_ = [("requested", C.c_int), ("allocated", C.c_int), ("dropped_vba_full", C.c_int),
                ("dropped_excess_full", C.c_int)]


class VoxfuseError(RuntimeError):
    def __init__(self, fn: str, status: int, detail: str = ""):
        super().__init__(f"{fn} returned {STATUS_NAMES.get(status, status)}{': ' + detail if detail else ''}")
        self.status = status


_lib = None


def load() -> C.CDLL:
    """Load the sm_100a library (built by paper_1410_0925_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing — build it with `python -m paper_1410_0925_b200.build`; "
            "the dense-fusion path has no CPU fallback")
    L = C.CDLL(str(LIB_PATH))
    vp, ip, dp, fp = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_float)
    sig = {
        "vf_abi_version": (C.c_int, []),
        "vf_struct_size": (C.c_long, [C.c_int]),
        "vf_default_settings": (None, [C.POINTER(VfSettings)]),
        "vf_create": (C.c_int, [C.POINTER(VfSettings), C.POINTER(VfCalib), C.c_int, C.POINTER(C.c_void_p)]),
        "vf_destroy": (C.c_int, [vp]),
        "vf_last_error": (C.c_char_p, [vp]),
        "vf_process_frame": (C.c_int, [vp, vp, vp, C.POINTER(VfFrameStats)]),
        "vf_process_frame_device": (C.c_int, [vp, vp, vp, C.POINTER(VfFrameStats)]),
        "vf_submit_frame": (C.c_int, [vp, vp, vp]),
        "vf_submit_raw_frame": (C.c_int, [vp, vp, vp, C.c_int]),
        "vf_collect_frame": (C.c_int, [vp, C.POINTER(VfFrameStats)]),
        "vf_frames_in_flight": (C.c_int, [vp]),
        "vf_synchronize": (C.c_int, [vp]),
        "vf_process_raw_frame": (C.c_int, [vp, vp, vp, C.c_int, C.POINTER(VfFrameStats)]),
        "vf_process_raw_frame_device": (C.c_int, [vp, vp, vp, C.c_int, C.POINTER(VfFrameStats)]),
        "vf_disparity_to_depth": (C.c_int, [vp, vp, C.c_int, vp]),
        "vf_read_stats": (C.c_int, [vp, C.POINTER(VfFrameStats)]),
        "vf_set_pose": (C.c_int, [vp, dp]),
        "vf_get_pose": (C.c_int, [vp, dp]),
        "vf_frame_count": (C.c_int, [vp]),
        "vf_get_maps": (C.c_int, [vp, vp, vp]),
        "vf_set_maps": (C.c_int, [vp, vp, vp, dp]),
        "vf_volume_digest": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
        "vf_get_surface_points": (C.c_long, [vp, vp, vp, C.c_long]),
        "vf_swap_states": (C.c_int, [vp, vp]),
        "vf_swap_stored_count": (C.c_long, [vp]),
        "vf_swap_store_read": (C.c_int, [vp, C.c_int, vp]),
        "vf_swap_save_store": (C.c_int, [vp, C.c_char_p]),
        "vf_swap_drain": (C.c_long, [vp, ip, C.c_long, C.POINTER(C.c_long)]),
        "vf_swap_load_store": (C.c_int, [vp, C.c_char_p]),
        "vf_stage_forward_project": (C.c_int, [vp]),
        "vf_render_image": (C.c_int, [vp, C.c_int, vp]),
        "vf_entry_count": (C.c_long, [vp]),
        "vf_voxel_bytes": (C.c_long, [vp]),
        "vf_export_entries": (C.c_int, [vp, vp]),
        "vf_export_voxels": (C.c_int, [vp, vp]),
        "vf_export_free_stacks": (C.c_int, [vp, ip, vp, ip, vp]),
        "vf_import_state": (C.c_int, [vp, vp, vp, C.c_int, vp, C.c_int, vp]),
        "vf_export_visible_list": (C.c_long, [vp, vp, C.c_long]),
        "vf_export_ranges": (C.c_long, [vp, vp]),
        "vf_stage_allocate": (C.c_int, [vp, vp, dp, C.POINTER(VfAllocStats)]),
        "vf_stage_integrate": (C.c_int, [vp, vp, vp, dp]),
        "vf_stage_raycast": (C.c_int, [vp, dp]),
        "vf_stage_icp": (C.c_int, [vp, vp, dp, dp, ip, dp, ip, ip]),
        "vf_icp_trace": (C.c_long, [vp, vp, C.c_long]),
        "vf_stage_ren": (C.c_int, [vp, vp, dp, dp, ip, dp, ip, ip]),
        "vf_stage_color": (C.c_int, [vp, vp, dp, dp, ip, dp, ip, ip]),
        "vf_depth_pyramid": (C.c_int, [vp, vp, vp]),
        "vf_render_synthetic": (C.c_int, [C.c_int, C.c_int, vp, C.c_int, vp, dp, C.POINTER(VfIntrinsics),
                                          C.c_double, C.c_double, vp, vp]),
        "vf_shard_p2p_handles": (C.c_int, [vp, vp]),
        "vf_shard_p2p_link": (C.c_int, [vp, vp, C.c_int]),
        "vf_shard_p2p_link_local": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
        "vf_shard_icp_handle": (C.c_int, [vp, vp]),
        "vf_shard_icp_link": (C.c_int, [vp, vp, C.c_int]),
        "vf_shard_icp_link_local": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
        "vf_shard_owner": (C.c_int, [C.c_int] * 5),
        "vf_shard_nccl_unique_id": (C.c_int, [vp]),
        "vf_shard_attach_nccl": (C.c_int, [vp, vp, C.c_int, C.c_int]),
        "vf_shard_composite_local": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
        "vf_device_alloc": (C.c_void_p, [C.c_size_t]),
        "vf_device_free": (C.c_int, [vp]),
        "vf_memcpy_h2d": (C.c_int, [vp, vp, C.c_size_t]),
        "vf_memcpy_d2h": (C.c_int, [vp, vp, C.c_size_t]),
        "vf_host_alloc_pinned": (C.c_void_p, [C.c_size_t]),
        "vf_host_free_pinned": (C.c_int, [vp]),
        "vf_event_record": (C.c_int, [vp, C.c_int]),
        "vf_event_elapsed_ms": (C.c_int, [vp, C.c_int, C.c_int, fp]),
        "vf_set_profiling": (C.c_int, [vp, C.c_int]),
        "vf_set_stage_timing": (C.c_int, [vp, C.c_int]),
        "vf_raycast_counters": (C.c_int, [vp, C.POINTER(C.c_ulonglong)]),
        "vf_alloc_counters": (C.c_int, [vp, C.POINTER(C.c_ulonglong)]),
        "vf_stage_times": (C.c_int, [vp, dp, C.POINTER(C.c_long)]),
        "vf_kernel_launches_per_frame": (C.c_int, [vp, C.c_int]),
        "vf_readback_bytes": (C.c_long, [vp]),
        "vf_flush_l2": (C.c_int, [vp, C.c_size_t]),
        "vf_flush_time": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "vf_last_modified_voxels": (C.c_long, [vp]),
        "vf_selftest_division": (C.c_long, [C.c_int, C.c_int, C.c_float, C.c_float, C.c_float, C.c_long]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(fn: str, status: int, ctx=None) -> int:
    if status < 0:
        detail = ""
        if ctx:
            try:
                detail = (load().vf_last_error(ctx) or b"").decode()
            except Exception:
                pass
        raise VoxfuseError(fn, status, detail)
    return status
