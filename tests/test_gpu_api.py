"""C ABI contract on the GPU: status codes for invalid settings and calls in
the wrong state (the reference throws std::invalid_argument at construction,
pipeline_impl.hpp:55-57; the hot path never throws — here nothing crosses
the ABI but a status)."""
import ctypes as C

import numpy as np
import pytest

from paper_1410_0925_b200 import _abi, make_pipeline, settings_from_config
from paper_1410_0925_b200._abi import VoxfuseError
from paper_1410_0925_b200.scene import CONFIGS

pytestmark = pytest.mark.gpu

VF_ERR_INVALID, VF_ERR_STATE = -1, -4


def _create(**overrides):
    from dataclasses import replace
    s, c = settings_from_config(CONFIGS["T160"])
    return make_pipeline(replace(s, **overrides), c)


@pytest.mark.parametrize("overrides", [
    {"bucket_count": 1000},                      # not a power of two
    {"voxel_size": 0.0},
    {"hierarchy_levels": 7},
    {"tracker_type": 1},                         # colour tracker with VoxelS
    {"tracker_type": 5},
    {"use_swapping": True, "swap_buffer_blocks": 5000},
    {"shard_count": 2, "shard_index": 2},
])
def test_invalid_settings_rejected(overrides):
    with pytest.raises(VoxfuseError) as e:
        _create(**overrides)
    assert e.value.status == VF_ERR_INVALID


def test_sharding_requires_icp():
    """Only ICP reads the rank-identical composited maps; Ren / colour would
    track against the shard's own voxels, so vf_create refuses them (and the
    Python mirror raises before reaching it)."""
    from dataclasses import replace
    s, c = settings_from_config(CONFIGS["T160"])
    bad = replace(s, shard_count=2, shard_index=0, tracker_type=2)
    with pytest.raises(ValueError):
        make_pipeline(bad, c)
    L = _abi.load()
    h = C.c_void_p()
    cs, cc = bad.to_c(), c.to_c()
    assert L.vf_create(C.byref(cs), C.byref(cc), 0, C.byref(h)) == VF_ERR_INVALID
    ok = replace(s, shard_count=2, shard_index=0, tracker_type=0)
    make_pipeline(ok, c).close()


def test_stage_timing_fills_frame_stats():
    """vf_set_stage_timing: the blocking call returns this frame's stage times
    (FrameStats::ms_*, pipeline.hpp:56-57) from the replayed graph."""
    p = _create()
    from paper_1410_0925_b200.scene import trajectory
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
    import vf_py
    from paper_1410_0925_b200.scene import BOX_ROOM_PLANES, BOX_ROOM_SPHERES
    olib = vf_py.oracle_lib()
    cfg = CONFIGS["T160"]
    poses = trajectory(4)
    frames = [vf_py.render_depth(olib, cfg, poses[i], BOX_ROOM_SPHERES, BOX_ROOM_PLANES) for i in range(4)]
    st = p.process_frame(None, frames[0])
    assert st.ms_tracking == 0 and st.ms_raycast == 0  # off by default
    p.set_stage_timing(True)
    for i in range(1, 4):
        st = p.process_frame(None, frames[i])
        parts = [st.ms_tracking, st.ms_allocation, st.ms_integration, st.ms_swapping, st.ms_raycast]
        assert st.tracking_ok and all(x >= 0 for x in parts) and st.ms_tracking > 0 and st.ms_raycast > 0
        assert sum(parts) <= st.ms_total * 1.05 + 0.02, (parts, st.ms_total)
    p.close()


def test_calls_in_the_wrong_state():
    p = _create()
    L = _abi.load()
    out = np.zeros((p.height, p.width, 3), np.uint8)
    # nothing rendered yet
    assert L.vf_render_image(p.handle, 0, out.ctypes.data_as(C.c_void_p)) == VF_ERR_STATE
    assert L.vf_render_image(p.handle, 1, out.ctypes.data_as(C.c_void_p)) == VF_ERR_STATE
    pts = np.zeros((p.height, p.width, 4), np.float32)
    assert L.vf_get_maps(p.handle, pts.ctypes.data_as(C.c_void_p), None) == VF_ERR_STATE
    # swapping off: no store
    assert L.vf_swap_states(p.handle, out.ctypes.data_as(C.c_void_p)) == VF_ERR_STATE
    assert L.vf_swap_stored_count(p.handle) == 0
    # null inputs and unknown modes
    assert L.vf_process_frame(p.handle, None, None, None) == VF_ERR_INVALID
    assert L.vf_render_image(p.handle, 9, out.ctypes.data_as(C.c_void_p)) == VF_ERR_INVALID
    d = np.full((p.height, p.width), 1.5, np.float32)
    p.process_frame(None, d)
    # a too-small buffer for the surface list is refused, not overrun
    assert L.vf_get_surface_points(p.handle, None, None, 0) == 0  # VoxelS: no colour list
    p.close()


def test_surface_list_capacity_checked():
    s, c = settings_from_config(CONFIGS["C2"])
    p = make_pipeline(s, c)
    import vf_py
    from helpers import frames
    (pose, depth, col), = frames(vf_py.oracle_lib(), CONFIGS["C2"], 1, rgb=True)
    p.set_pose(pose)
    p.process_frame(col, depth)
    L = _abi.load()
    n = L.vf_get_surface_points(p.handle, None, None, 0)
    assert n > 1000
    buf = np.zeros((n - 1, 3), np.float32)
    assert L.vf_get_surface_points(p.handle, buf.ctypes.data_as(C.c_void_p), None, n - 1) == VF_ERR_INVALID
    p.close()


@pytest.mark.parametrize("cfg_name,known_poses", [("T160", False), ("T160", True)])
def test_streaming_submit_matches_process_frame(olib, cfg_name, known_poses):
    """vf_submit_frame / vf_collect_frame (two frames in flight) produce the
    same frames as blocking vf_process_frame: identical stats, poses, maps and
    volume digest (same kernels, same order; only the upload overlaps)."""
    from helpers import frames
    cfg = CONFIGS[cfg_name]
    seq = frames(olib, cfg, 8, rgb=False)
    a, b = _create(), _create()
    ref = []
    for pose, d, _ in seq:
        if known_poses:
            a.set_pose(pose)
        ref.append(a.process_frame(None, d))
    got = []
    for i, (pose, d, _) in enumerate(seq):
        if known_poses:
            b.set_pose(pose)
        b.submit_frame(None, d)
        if b.frames_in_flight() == 2:
            got.append(b.collect_frame())
    while b.frames_in_flight():
        got.append(b.collect_frame())
    assert [g.frame for g in got] == [r.frame for r in ref]
    for g, r in zip(got, ref):
        assert g.tracking_ok == r.tracking_ok and g.tracking_iterations == r.tracking_iterations
        assert g.visible_blocks == r.visible_blocks and g.blocks_allocated == r.blocks_allocated
        assert np.array_equal(np.asarray(g.pose), np.asarray(r.pose))
    assert a.volume_digest() == b.volume_digest()
    pa, na = a.tracking_state()
    pb, nb = b.tracking_state()
    assert np.array_equal(pa, pb) and np.array_equal(na, nb)
    # queue discipline
    L = _abi.load()
    assert L.vf_collect_frame(b.handle, None) == VF_ERR_STATE
    d = seq[0][1]
    b.submit_frame(None, d)
    b.submit_frame(None, d)
    assert L.vf_submit_frame(b.handle, d.ctypes.data_as(C.c_void_p), None) == VF_ERR_STATE
    b.collect_frame()
    b.collect_frame()
    a.close()
    b.close()


def test_streaming_rgb_swapping_matches_process_frame(olib):
    """Streaming with the per-frame inputs and side branches on: VoxelSRgb with
    RGB uploads, known poses set between submissions, host swapping over a pan
    away and back: identical stats, volume and host store to vf_process_frame."""
    import vf_py
    from helpers import swap_config
    from paper_1410_0925_b200 import make_pipeline, settings_from_config
    from paper_1410_0925_b200.scene import BOX_ROOM_PLANES, BOX_ROOM_SPHERES, pan_trajectory
    cfg = swap_config("T160_swap_roundtrip").with_(voxel_type=2)
    poses = pan_trajectory(24)
    seq = [(pose, vf_py.render_depth(olib, cfg, pose, BOX_ROOM_SPHERES, BOX_ROOM_PLANES, 0.05, 100.0),
            vf_py.render_rgb(olib, cfg, pose, BOX_ROOM_SPHERES, BOX_ROOM_PLANES)) for pose in poses]
    s, c = settings_from_config(cfg)
    a, b = make_pipeline(s, c), make_pipeline(s, c)
    ref = []
    for pose, d, col in seq:
        a.set_pose(pose)
        ref.append(a.process_frame(col, d))
    got = []
    for pose, d, col in seq:
        b.set_pose(pose)
        b.submit_frame(col, d)
        if b.frames_in_flight() == 2:
            got.append(b.collect_frame())
    while b.frames_in_flight():
        got.append(b.collect_frame())
    assert len(got) == len(ref)
    for g, r in zip(got, ref):
        assert (g.frame, g.visible_blocks, g.blocks_allocated, g.swapped_in, g.swapped_out) == \
            (r.frame, r.visible_blocks, r.blocks_allocated, r.swapped_in, r.swapped_out)
    assert sum(r.swapped_out for r in ref) > 0 and sum(r.swapped_in for r in ref) > 0
    assert a.volume_digest() == b.volume_digest()
    assert a.store_count() == b.store_count()
    sa, sb = a.store(), b.store()
    assert sa.keys() == sb.keys() and all(np.array_equal(sa[k], sb[k]) for k in sa)
    a.close()
    b.close()


def test_raycast_counters_rerun_is_identical():
    """vf_raycast_counters re-runs the last raycast with counters: the maps
    are unchanged and the counts are consistent (hits == valid map pixels,
    every table probe is a voxel read that missed the block cache)."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
    import vf_py
    from paper_1410_0925_b200.scene import BOX_ROOM_PLANES, BOX_ROOM_SPHERES, trajectory
    s, c = settings_from_config(CONFIGS["C1"])
    p = make_pipeline(s, c)
    olib = vf_py.oracle_lib()
    for pose in trajectory(3):
        p.process_frame(None, vf_py.render_depth(olib, CONFIGS["C1"], pose, BOX_ROOM_SPHERES, BOX_ROOM_PLANES))
    pts0, nrm0 = p.tracking_state()
    cnt = p.raycast_counters()
    pts1, nrm1 = p.tracking_state()
    assert np.array_equal(pts0.view(np.uint32), pts1.view(np.uint32))
    assert np.array_equal(nrm0.view(np.uint32), nrm1.view(np.uint32))
    assert cnt["hits"] == int((pts1[..., 3] > 0).sum())
    assert 0 < cnt["rays"] <= p.width * p.height
    assert 0 < cnt["table_probes"] < cnt["voxel_reads"]
    p.close()


def test_alloc_counters_do_not_touch_the_volume():
    """vf_alloc_counters walks mark_blocks' DDA without requests: the table
    is unchanged and every pixel with depth is counted.  Cells can still be
    missing after the frame: a bucket takes one request per frame
    (allocation.hpp:155-159), so colliding blocks wait for a later frame --
    and the same walk after a second identical frame finds fewer."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
    import vf_py
    from paper_1410_0925_b200.scene import BOX_ROOM_PLANES, BOX_ROOM_SPHERES, trajectory
    s, c = settings_from_config(CONFIGS["C1"])
    p = make_pipeline(s, c)
    olib = vf_py.oracle_lib()
    d = vf_py.render_depth(olib, CONFIGS["C1"], trajectory(1)[0], BOX_ROOM_SPHERES, BOX_ROOM_PLANES)
    st = p.process_frame(None, d)
    e0 = p.entries()
    cnt = p.alloc_counters()
    assert np.array_equal(p.entries(), e0)
    assert cnt["pixels"] == int((d > 0).sum())
    assert cnt["cells_probed"] >= cnt["pixels"] and 0 < cnt["cells_missing"] < cnt["cells_probed"]
    assert st.allocation_dropped == 0
    p.process_frame(None, d)
    assert p.alloc_counters()["cells_missing"] < cnt["cells_missing"]
    p.close()
