"""GPU swap engine (vf_swap.cu) against the oracle's restatement of
swap.hpp, itself pinned to the reference (tests/test_oracle.py
::test_oracle_golden_swap).

Bar: bit-exact, frame by frame — hash entries (block_state incl. the VBA
slots the swap engine pops and pushes), voxels, per-entry swap states, the
host store's contents, SwapMetrics, maps.  Plus the VXBS file format
(block_store.hpp:14-53) and config 4's corridor walk."""
import struct

import numpy as np
import pytest

import vf_py
from helpers import SWAP_CASES, entries_equal, swap_config, voxel_payload
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import (BOX_ROOM_PLANES, BOX_ROOM_SPHERES, CONFIGS, corridor_trajectory,
                                        pan_trajectory, scene_for)

pytestmark = pytest.mark.gpu


def _run_pair(olib, cfg, poses, check_every=1, spheres=BOX_ROOM_SPHERES, planes=BOX_ROOM_PLANES, far=100.0):
    s, c = settings_from_config(cfg)
    p = make_pipeline(s, c)
    o = vf_py.Volume(olib, cfg, False)
    vsize = 8 if cfg.voxel_type == 2 else 4
    for i, pose in enumerate(poses):
        d = vf_py.render_depth(olib, cfg, pose, spheres, planes, 0.05, far)
        p.set_pose(pose)
        st = p.process_frame(None, d)
        so = o.process(d, None, pose)
        assert (st.blocks_allocated, st.allocation_dropped, st.visible_blocks) == \
            (so.blocks_allocated, so.allocation_dropped, so.visible_blocks), f"frame {i}: allocation"
        assert (st.swapped_in, st.swapped_out, st.bytes_in, st.bytes_out) == \
            (so.swapped_in, so.swapped_out, so.bytes_in, so.bytes_out), f"frame {i}: SwapMetrics"
        if i % check_every and i != len(poses) - 1:
            continue
        assert entries_equal(p.entries(), o.entries()), f"frame {i}: hash entries"
        assert np.array_equal(voxel_payload(p.voxels(), vsize), voxel_payload(o.voxels(), vsize)), f"frame {i}: voxels"
        assert np.array_equal(p.swap_states(), o.swap_states()), f"frame {i}: swap states"
        assert p.store_count() == o.store_count(), f"frame {i}: stored blocks"
        sg, so_ = p.store(), o.store()
        assert sg.keys() == so_.keys(), f"frame {i}: stored entries"
        assert all(np.array_equal(sg[k], so_[k]) for k in sg), f"frame {i}: stored payloads"
        pg, ng = p.tracking_state()
        po, no = o.maps()
        assert np.array_equal(pg.view(np.uint32), po.view(np.uint32)), f"frame {i}: points"
        assert np.array_equal(ng.view(np.uint32), no.view(np.uint32)), f"frame {i}: normals"
    return p, o


@pytest.mark.parametrize("name", list(SWAP_CASES))
def test_swap_pan_bit_exact(olib, name):
    """Pan away and back: swap-outs at the budget cap, swap-ins (deferred
    while the VBA is full), host store and states identical to the oracle."""
    cfg = swap_config(name)
    p, o = _run_pair(olib, cfg, pan_trajectory(24))
    p.close()


def test_swap_rgb_roundtrip(olib):
    """VoxelSRgb blocks (7-byte codec) through the store and back."""
    cfg = swap_config("T160_swap_roundtrip").with_(voxel_type=2)
    s, c = settings_from_config(cfg)
    p = make_pipeline(s, c)
    o = vf_py.Volume(olib, cfg, False)
    for i, pose in enumerate(pan_trajectory(24)):
        d = vf_py.render_depth(olib, cfg, pose, BOX_ROOM_SPHERES, BOX_ROOM_PLANES)
        col = vf_py.render_rgb(olib, cfg, pose, BOX_ROOM_SPHERES, BOX_ROOM_PLANES)
        p.set_pose(pose)
        st = p.process_frame(col, d)
        so = o.process(d, col, pose)
        assert (st.swapped_in, st.swapped_out) == (so.swapped_in, so.swapped_out)
    assert entries_equal(p.entries(), o.entries())
    assert np.array_equal(voxel_payload(p.voxels(), 8), voxel_payload(o.voxels(), 8))
    sg, so_ = p.store(), o.store()
    assert sg.keys() == so_.keys() and all(np.array_equal(sg[k], so_[k]) for k in sg)
    p.close()


def test_vxbs_file_roundtrip(olib, tmp_path):
    """vf_swap_save_store writes the reference's VXBS layout (16-byte header,
    (u32 entry, payload) records); vf_swap_load_store reads it back into a
    fresh context holding the same table."""
    cfg = swap_config("T160_swap_roundtrip")
    p, o = _run_pair(olib, cfg, pan_trajectory(12), check_every=100)
    path = tmp_path / "store.vxbs"
    p.save_store(path)
    raw = path.read_bytes()
    magic, version, tag, n_entries, payload = struct.unpack_from("<IHHII", raw, 0)
    assert (magic, version, tag, n_entries, payload) == (0x53425856, 1, 1, cfg.hash.entry_count, 512 * 3)
    recs = {}
    off = 16
    while off < len(raw):
        (idx,) = struct.unpack_from("<I", raw, off)
        recs[idx] = np.frombuffer(raw, np.uint8, payload, off + 4)
        off += 4 + payload
    ref = o.store()
    assert recs.keys() == ref.keys() and all(np.array_equal(recs[k], ref[k]) for k in recs)
    # a second context: same table (imported), store loaded from the file
    s, c = settings_from_config(cfg)
    q = make_pipeline(s, c)
    import ctypes as C
    vt, et = C.c_int(), C.c_int()
    vs = np.zeros(cfg.hash.block_count, np.int32)
    es = np.zeros(cfg.hash.excess_count, np.int32)
    olib.lib.vfo_free_stacks(o.h, C.byref(vt), vs.ctypes.data_as(C.c_void_p), C.byref(et),
                             es.ctypes.data_as(C.c_void_p))
    q.import_state(o.entries(), o.voxels(), vt.value, vs, et.value, es)
    assert q.store_count() == 0
    q.load_store(path)
    got = q.store()
    assert got.keys() == ref.keys() and all(np.array_equal(got[k], ref[k]) for k in got)
    p.close()
    q.close()


def test_corridor_config4_first_frames_bit_exact(olib):
    """Config 4 (corridor walk, 5 mm, swapping with B = 512): the first
    frames at full size against the oracle, known poses."""
    cfg = CONFIGS["C4"].with_(tracking=False)
    spheres, planes, far = scene_for(cfg)
    p, o = _run_pair(olib, cfg, corridor_trajectory(8), check_every=4, spheres=spheres, planes=planes, far=far)
    p.close()


def test_corridor_tracked_walk(olib):
    """Config 4 tracked: 150 frames (7.5 m) down the corridor; the tracker
    holds the trajectory, swapping keeps the VBA from running dry."""
    from helpers import centre_dist, rot_angle
    cfg = CONFIGS["C4"]
    spheres, planes, far = scene_for(cfg)
    s, c = settings_from_config(cfg)
    p = make_pipeline(s, c)
    poses = corridor_trajectory(150)
    outs = 0
    for i, pose in enumerate(poses):
        d = vf_py.render_depth(olib, cfg, pose, spheres, planes, 0.05, far)
        st = p.process_frame(None, d)
        assert st.tracking_ok, f"frame {i}: tracking lost"
        assert st.allocation_dropped == 0, f"frame {i}: allocations dropped"
        assert st.swapped_out <= cfg.swap_buffer_blocks
        outs += st.swapped_out
    assert outs > 10000
    assert rot_angle(p.pose(), poses[-1]) < 0.01 and centre_dist(p.pose(), poses[-1]) < 0.05
    p.close()


def test_host_store_grows_past_its_first_chunks(olib):
    """The host store starts at one VBA's worth of pinned slots and grows in
    4096-block chunks as blocks leave, up to one slot per hash entry -- the
    reference's GlobalCache bound (swap.hpp:42-56): a corridor walk that
    parks several times the VBA on the host never defers a swap-out, and
    stays bit-exact with the oracle (entries, voxels, states, store)."""
    from paper_1410_0925_b200.scene import HashConfig
    cfg = CONFIGS["C4"].with_(tracking=False, width=320, height=240, voxel_size=0.01, mu=0.03, swap_buffer_blocks=512,
                              hash=HashConfig(bucket_count=1 << 15, excess_count=1 << 13, block_count=1536))
    spheres, planes, far = scene_for(cfg)
    walk = corridor_trajectory(48, step=0.3)  # 14 m at known poses: blocks leave the swap frustum fast
    p, o = _run_pair(olib, cfg, walk, check_every=12, spheres=spheres, planes=planes, far=far)
    stored = p.store_count()
    print("stored blocks", stored)
    assert stored > 4096, "the walk should park more blocks than the first chunk holds"
    p.close()


def test_swap_journal_lists_swap_outs_in_order(olib):
    """vf_swap_drain: every swapped-out entry once, in the frames' order, and
    nothing after a drain (what the adapter feeds the VXBS file store)."""
    cfg = swap_config("T160_swap_small_vba")
    s, c = settings_from_config(cfg)
    p = make_pipeline(s, c)
    total, seen = 0, []
    for pose in pan_trajectory(24):
        d = vf_py.render_depth(olib, cfg, pose, BOX_ROOM_SPHERES, BOX_ROOM_PLANES)
        p.set_pose(pose)
        st = p.process_frame(None, d)
        ent, lost = p.swap_drain()
        assert lost == 0 and len(ent) == st.swapped_out
        total += st.swapped_out
        seen.extend(ent.tolist())
    assert len(seen) == total and total > 0
    assert len(p.swap_drain()[0]) == 0
    p.close()


def test_corridor_look_around_swaps_in_bit_exact(olib):
    """C4R's walk (config 4 scene, B = 100 as BASELINE states) at known poses:
    blocks leave the enlarged frustum and come back, so swap-ins with
    fuse_voxels (swap.hpp:96-131, 136-198) run alongside swap-outs -- entries,
    voxels, states and the host store stay bit-exact with the oracle."""
    from paper_1410_0925_b200.scene import trajectory_for
    cfg = CONFIGS["C4R"].with_(tracking=False)
    spheres, planes, far = scene_for(cfg)
    p, o = _run_pair(olib, cfg, trajectory_for(cfg, 44), check_every=11, spheres=spheres, planes=planes, far=far)
    ins = o.store_count()
    p.close()
    assert ins > 0
