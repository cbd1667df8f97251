"""CPU suite: the oracle against the reference's golden vectors and against
the reference itself (oracle/_ref) where it is built; known-answer values.
No GPU needed."""
import ctypes as C
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import vf_py
from helpers import swap_config
from paper_1410_0925_b200.scene import BOX_ROOM_PLANES, BOX_ROOM_SPHERES, CONFIGS, pan_trajectory, trajectory

GOLD = json.loads((Path(__file__).parent / "golden" / "golden_ref.json").read_text())


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_hash_block_pos_known_answers(olib):
    ka = GOLD["known_answers"]["hash_block_pos_mask_0xFFFFF"]
    for key, want in ka.items():
        x, y, z = (int(v) for v in key.split(","))
        assert olib.lib.vfo_hash_block_pos(x, y, z, 0xFFFFF) == want
        # the same arithmetic restated in Python (hash_volume.hpp:32-37)
        h = (((x & 0xFFFFFFFF) * 73856093) ^ ((y & 0xFFFFFFFF) * 19349669) ^ ((z & 0xFFFFFFFF) * 83492791))
        assert (h & 0xFFFFFFFF) & 0xFFFFF == want
    assert olib.lib.vfo_hash_block_pos(1, 0, 0, 0xFFFFF) != 471389  # SPEC.md:171 is wrong


def test_sdf_quantisation_known_answers():
    # sdf_float_to_value (voxel.hpp:16-19): clamp, then truncate toward zero
    for f, want in GOLD["known_answers"]["sdf_float_to_value"].items():
        v = np.clip(np.float32(float(f)), np.float32(-1), np.float32(1)) * np.float32(32767.0)
        assert int(np.trunc(v)) == want


def test_sdf_to_float_identity():
    """The device evaluates (float)v / 32767.0f as one FP64 multiply rounded
    to FP32 (vf_device.cuh); exhaustive proof that the two agree bit for bit."""
    v = np.arange(-32768, 32768, dtype=np.int64)
    a = v.astype(np.float32) / np.float32(32767.0)
    b = (v.astype(np.float64) * (1.0 / 32767.0)).astype(np.float32)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def _check_run(lib, cfg, frames_gold, tracking, rgb=False):
    from paper_1410_0925_b200.scene import scene_for, trajectory_for
    spheres, planes, far = scene_for(cfg)
    poses = trajectory_for(cfg, len(frames_gold))
    vol = vf_py.Volume(lib, cfg, tracking)
    vsize = 8 if cfg.voxel_type == 2 else 4
    for i, g in enumerate(frames_gold):
        d = vf_py.render_depth(lib, cfg, poses[i], spheres, planes, 0.05, far)
        assert sha(d) == g["depth_sha"], f"frame {i}: synthetic depth differs"
        c = None
        if rgb:
            c = vf_py.render_rgb(lib, cfg, poses[i], spheres, planes, 0.05, far)
            assert sha(c) == g["rgb_sha"]
        st = vol.process(d, c, None if tracking else poses[i])
        assert int(st.tracking_ok) == g["tracking_ok"]
        assert int(st.tracking_iterations) == g["tracking_iterations"]
        assert int(st.blocks_allocated) == g["blocks_allocated"]
        assert int(st.visible_blocks) == g["visible_blocks"]
        assert vol.allocated_blocks() == g["allocated_total"]
        assert [float(x) for x in vol.pose()] == g["pose"], f"frame {i}: pose"
        e = vol.entries()
        e["pad"] = 0
        assert sha(e) == g["entries_sha"], f"frame {i}: hash entries"
        assert sha(vol.voxels().reshape(-1, vsize)[:, : vsize - 1]) == g["voxels_sha"], f"frame {i}: voxels"
        pts, nrm = vol.maps()
        assert sha(pts) == g["points_sha"] and sha(nrm) == g["normals_sha"], f"frame {i}: maps"
        assert sha(np.sort(vol.visible_list())) == g["visible_sha"]
        if g.get("volume_digest") is not None and hasattr(lib, "prefix") and lib.prefix == "vfo_":
            assert str(vol.digest()) == g["volume_digest"], f"frame {i}: FNV volume digest"
        if g.get("ranges_sha") is not None:
            assert sha(vol.ranges()) == g["ranges_sha"]
        if "swapped_in" in g:  # swap engine (swap.hpp)
            assert (int(st.swapped_in), int(st.swapped_out)) == (g["swapped_in"], g["swapped_out"]), f"frame {i}"
            assert sha(vol.swap_states()) == g["states_sha"] and vol.store_count() == g["store_count"]
        if "surface_points_sha" in g:  # raycast epilogues (raycast.hpp:441-509)
            sp, sc = vol.surface_points()
            assert len(sp) == g["surface_count"], f"frame {i}: surface point count"
            assert sha(sp) == g["surface_points_sha"] and sha(sc) == g["surface_colors_sha"], f"frame {i}: surface list"
            assert sha(vol.image(0)) == g["image_sha"], f"frame {i}: render_image"
            assert sha(vol.image(3)) == g["image_grey_sha"], f"frame {i}: render_image (grey)"
        if "image_depth_sha" in g:
            assert sha(vf_py.colourize_depth(d)) == g["image_depth_sha"], f"frame {i}: colourize_depth"
    vol.close()


def test_oracle_golden_tracking_T160(olib):
    """4 tracked frames: poses bit-identical to the reference's, entries,
    voxels, maps, visible set and the reference's volume_digest."""
    _check_run(olib, CONFIGS["T160"], GOLD["T160_tracking"], tracking=True)


def test_oracle_golden_tracking_C3(olib):
    """BASELINE configs[2] (1280x960, 2 mm, 2^20 blocks): frame 0 pinned to
    the reference: entries, voxels, maps, visible set."""
    _check_run(olib, CONFIGS["C3"], GOLD["C3_tracking"], tracking=True)


def test_oracle_golden_tracking_C4_corridor(olib):
    """BASELINE configs[3]: the first tracked corridor frames with host
    swapping on, pinned to the reference (poses, entries, voxels, maps, swap
    states and store)."""
    _check_run(olib, CONFIGS["C4"], GOLD["C4_corridor_tracking"], tracking=True)


def test_oracle_golden_known_pose_T320(olib):
    _check_run(olib, CONFIGS["T320"].with_(tracking=False), GOLD["T320_known_pose"], tracking=False)


def test_oracle_golden_known_pose_rgb_C2(olib):
    _check_run(olib, CONFIGS["C2"], GOLD["C2_known_pose_rgb"], tracking=False, rgb=True)


def test_oracle_golden_pyramid(olib):
    cfg = CONFIGS["C1"]
    d = vf_py.render_depth(olib, cfg, trajectory(5)[3], BOX_ROOM_SPHERES, BOX_ROOM_PLANES)
    d[100:140, 200:260] = 0.0
    assert sha(d) == GOLD["C1_pyramid"]["depth_sha"]
    assert [sha(l) for l in vf_py.depth_pyramid(olib, d, 5)] == GOLD["C1_pyramid"]["levels_sha"]


def test_oracle_matches_reference_live(olib, rlib):
    """Where oracle/_ref is built: the restatement and the reference agree bit
    for bit on 3 tracked C1 frames (entries, voxels, maps, pose, digest)."""
    cfg = CONFIGS["C1"]
    poses = trajectory(3)
    vo, vr = vf_py.Volume(olib, cfg, True), vf_py.Volume(rlib, cfg, True)
    for i in range(3):
        d = vf_py.render_depth(olib, cfg, poses[i], BOX_ROOM_SPHERES, BOX_ROOM_PLANES)
        so, sr = vo.process(d), vr.process(d)
        assert so.tracking_iterations == sr.tracking_iterations
        assert np.array_equal(vo.pose(), vr.pose())
        eo, er = vo.entries(), vr.entries()
        eo["pad"] = er["pad"] = 0
        assert np.array_equal(eo, er)
        assert np.array_equal(vo.voxels().reshape(-1, 4)[:, :3], vr.voxels().reshape(-1, 4)[:, :3])
        for a, b in zip(vo.maps(), vr.maps()):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert vo.digest() == vr.digest()


def test_icp_reference_vs_oracle_stage(olib, rlib):
    """icp_track on identical maps: oracle and the reference agree exactly."""
    cfg = CONFIGS["T320"]
    poses = trajectory(3)
    o = vf_py.Volume(olib, cfg, tracking=False)
    for i in range(2):
        o.process(vf_py.render_depth(olib, cfg, poses[i], BOX_ROOM_SPHERES, BOX_ROOM_PLANES), None, poses[i])
    pts, nrm = o.maps()
    rp = o.pose()
    d = vf_py.render_depth(olib, cfg, poses[2], BOX_ROOM_SPHERES, BOX_ROOM_PLANES)
    out_o, out_r = np.zeros(12), np.zeros(12)
    it, cost, valid = C.c_int(), C.c_double(), C.c_int()
    ok_o = olib.lib.vfo_stage_icp(o.h, d.ctypes.data_as(C.c_void_p), out_o.ctypes.data_as(C.c_void_p), C.byref(it),
                                  C.byref(cost), C.byref(valid))
    cfgc = vf_py.make_config(cfg)
    it2, cost2, valid2 = C.c_int(), C.c_double(), C.c_int()
    ok_r = rlib.lib.vfr_icp_track(C.byref(cfgc), d.ctypes.data_as(C.c_void_p), pts.ctypes.data_as(C.c_void_p),
                                  nrm.ctypes.data_as(C.c_void_p), rp.ctypes.data_as(C.c_void_p),
                                  out_r.ctypes.data_as(C.c_void_p), C.byref(it2), C.byref(cost2), C.byref(valid2))
    assert bool(ok_o) == bool(ok_r) and it.value == it2.value and valid.value == valid2.value
    assert np.array_equal(out_o, out_r)
    assert cost.value == cost2.value


def _store_digest(vol):
    h = hashlib.sha256()
    for k, v in sorted(vol.store().items()):
        h.update(np.int32(k).tobytes())
        h.update(v.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", ["T160_swap_small_vba", "T160_swap_roundtrip"])
def test_oracle_golden_swap(olib, name):
    """Swap engine (swap.hpp): the restatement reproduces the reference's
    entries, voxels, per-entry swap states, host store contents and
    SwapMetrics on a pan away and back (budget caps, deferred swap-ins)."""
    cfg = swap_config(name)
    poses = pan_trajectory(len(GOLD[name]))
    vol = vf_py.Volume(olib, cfg, False)
    for i, g in enumerate(GOLD[name]):
        d = vf_py.render_depth(olib, cfg, poses[i], BOX_ROOM_SPHERES, BOX_ROOM_PLANES)
        assert sha(d) == g["depth_sha"]
        st = vol.process(d, None, poses[i])
        got = (st.blocks_allocated, st.allocation_dropped, st.visible_blocks, st.swapped_in, st.swapped_out,
               st.bytes_in, st.bytes_out)
        want = tuple(g[k] for k in ("blocks_allocated", "allocation_dropped", "visible_blocks", "swapped_in",
                                    "swapped_out", "bytes_in", "bytes_out"))
        assert got == want, f"frame {i}: stats {got} vs {want}"
        e = vol.entries()
        e["pad"] = 0
        assert sha(e) == g["entries_sha"], f"frame {i}: entries"
        assert sha(vol.voxels().reshape(-1, 4)[:, :3]) == g["voxels_sha"], f"frame {i}: voxels"
        assert sha(vol.swap_states()) == g["states_sha"], f"frame {i}: swap states"
        assert vol.store_count() == g["store_count"] and _store_digest(vol) == g["store_sha"], f"frame {i}: store"
    vol.close()


def _disparity_cases(seed=0x14100925):
    rng = np.random.default_rng(seed)
    d = rng.integers(0, 65536, size=(120, 160), dtype=np.uint16)
    d[0, :8] = [0, 1, 1134, 1135, 1136, 65535, 400, 900]  # pole a - d <= 0, saturated, in range
    return d


def test_disparity_to_depth_matches_reference(olib, rlib):
    """disparity_image_to_depth (view.hpp:18-28): restatement vs the reference,
    Kinect-style a / b, including the pole and the max_depth clamp."""
    d = _disparity_cases()
    for a, b, fx, mx in [(1135.09, 0.0819141, 573.71, 8.0), (1135.09, 0.0819141, 573.71, 3.0), (900.0, 0.2, 525.0, 8.0)]:
        o = vf_py.disparity_to_depth(olib, d, a, b, fx, mx)
        r = vf_py.disparity_to_depth(rlib, d, a, b, fx, mx)
        assert np.array_equal(o.view(np.uint32), r.view(np.uint32))
        assert (o > 0).any() and (o == 0).any()


def test_eigen_association_bound_known_pose():
    """The shim-built reference in Eigen's halving association
    (oracle/_ref_halving) against the left-to-right build on 4 known-pose C1
    frames: the delta a stock-Eigen reference could show against the GPU
    path, which is bit-exact to the left-to-right build (test_gpu_parity.py).
    Stays inside the §8(c) tolerances (tests/test_gpu_eigen_assoc.py checks
    the GPU against the halving build directly)."""
    if not (vf_py.ref_available() and vf_py.ref_halving_available()):
        pytest.skip("oracle/_ref and oracle/_ref_halving need /root/reference at build time")
    from assoc_stats import compare
    from helpers import frames
    ra, rh = vf_py.ref_lib(), vf_py.ref_halving_lib()
    ra.lib.vfr_set_threads(1)
    rh.lib.vfr_set_threads(1)
    cfg = CONFIGS["C1"].with_(tracking=False)
    va, vh = vf_py.Volume(ra, cfg, False), vf_py.Volume(rh, cfg, False)
    for pose, d, _ in frames(ra, cfg, 4):
        va.process(d, None, pose)
        vh.process(d, None, pose)
    out = compare(va.entries(), va.voxels(), vh.entries(), vh.voxels(), va.maps(), vh.maps(), cfg.voxel_size)
    va.close()
    vh.close()
    print(out)
    assert out["blocks_common_frac"] == 1.0
    assert out["sdf_le1_frac"] >= 0.999 and out["weight_exact_frac"] >= 0.999
    assert out["hit_agreement"] >= 0.999 and out["point_within_half_voxel_frac"] >= 0.999
    assert out["sdf_exact_frac"] < 1.0 or out["maps_bit_exact_frac"] < 1.0  # the two builds do differ
