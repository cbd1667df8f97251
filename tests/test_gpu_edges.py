"""Edge cases of the frame path against the oracle (bit-exact where the
reference is defined): frames without valid depth, invalid / extreme depth
samples, image sizes that are not multiples of the 16-pixel fragment or of
the pyramid's 2x2 reduction, the largest configuration (C3, 1280x960,
2 mm, 2^20 blocks) at full size, and non-default SceneParams / HashConfig
(stop_integrating_at_max, one- and four-slot buckets).

Not covered on purpose: NaN / inf depth.  mark_blocks converts
floor(NaN or inf) to int (allocation.hpp:62-63), undefined behaviour in the
reference, so there is no reference answer to match."""
import numpy as np
import pytest

import vf_py
from helpers import centre_dist, entries_equal, far_pose, frames, rot_angle, voxel_payload
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import BOX_ROOM_PLANES, BOX_ROOM_SPHERES, CONFIGS, HashConfig, trajectory

pytestmark = pytest.mark.gpu


def _pair(olib, cfg, tracking):
    s, c = settings_from_config(cfg.with_(tracking=tracking))
    return make_pipeline(s, c), vf_py.Volume(olib, cfg, tracking)


def _same_state(p, o, vsize=4):
    assert entries_equal(p.entries(), o.entries()), "hash entries"
    assert np.array_equal(voxel_payload(p.voxels(), vsize), voxel_payload(o.voxels(), vsize)), "voxels"
    pg, ng = p.tracking_state()
    po, no = o.maps()
    assert np.array_equal(pg.view(np.uint32), po.view(np.uint32)), "points"
    assert np.array_equal(ng.view(np.uint32), no.view(np.uint32)), "normals"


def test_frames_without_valid_depth(olib):
    """An all-invalid frame allocates nothing and renders nothing; tracked,
    the next frame's ICP fails (too few points) and the pose is held."""
    cfg = CONFIGS["T320"]
    fr = frames(olib, cfg, 3)
    empty = np.zeros_like(fr[0][1])
    for tracking in (False, True):
        p, o = _pair(olib, cfg, tracking)
        seq = [(fr[0][0], fr[0][1]), (fr[1][0], empty), (fr[2][0], fr[2][1])] if tracking else \
              [(fr[0][0], empty), (fr[1][0], fr[1][1]), (fr[2][0], empty)]
        for pose, d in seq:
            if not tracking:
                p.set_pose(pose)
            st = p.process_frame(None, d)
            so = o.process(d, None, None if tracking else pose)
            assert (st.blocks_allocated, st.visible_blocks, bool(st.tracking_ok)) == \
                (so.blocks_allocated, so.visible_blocks, bool(so.tracking_ok))
            if tracking:
                assert rot_angle(p.pose(), o.pose()) <= 1e-6 and centre_dist(p.pose(), o.pose()) <= 1e-6
            else:
                _same_state(p, o)
        p.close()


def test_invalid_and_extreme_depth_samples(olib):
    """Negative and zero samples are skipped, tiny (near the 1 mm segment
    clamp) and far (20 m) samples allocate along their full band: known
    poses, bit-exact."""
    cfg = CONFIGS["T320"].with_(tracking=False)
    rng = np.random.default_rng(0x14100925)
    p, o = _pair(olib, cfg, False)
    for pose, d, _ in frames(olib, cfg, 3):
        d = d.copy()
        m = rng.random(d.shape)
        d[m < 0.03] = -1.0
        d[(m >= 0.03) & (m < 0.05)] = 0.0
        d[(m >= 0.05) & (m < 0.06)] = 0.0012
        d[(m >= 0.06) & (m < 0.07)] = 20.0
        p.set_pose(pose)
        st = p.process_frame(None, d)
        so = o.process(d, None, pose)
        assert (st.blocks_allocated, st.visible_blocks) == (so.blocks_allocated, so.visible_blocks)
        _same_state(p, o)
    p.close()


@pytest.mark.parametrize("w,h", [(250, 190), (161, 97)])
def test_ragged_image_sizes(olib, w, h):
    """Images that are not multiples of the 16-pixel fragment (partial range
    tiles, partial raycast CTAs) nor of 2^levels (odd pyramid levels):
    known poses bit-exact; tracked poses within the tracker bar."""
    cfg = CONFIGS["T320"].with_(name=f"R{w}", width=w, height=h)
    kp = cfg.with_(tracking=False)
    p, o = _pair(olib, kp, False)
    fr = frames(olib, kp, 3)
    for pose, d, _ in fr:
        p.set_pose(pose)
        p.process_frame(None, d)
        o.process(d, None, pose)
        _same_state(p, o)
        assert np.array_equal(p.ranges().view(np.uint32), o.ranges().view(np.uint32))
    p.close()
    p, o = _pair(olib, cfg, True)
    for pose, d, _ in frames(olib, cfg, 4):
        st = p.process_frame(None, d)
        so = o.process(d)
        assert bool(st.tracking_ok) == bool(so.tracking_ok)
        assert rot_angle(p.pose(), o.pose()) <= 1e-4 and centre_dist(p.pose(), o.pose()) <= 1e-4
    p.close()


def test_largest_configuration_frame0_bit_exact(olib):
    """C3 at full size (1280x960, 2 mm voxels, 2^21 buckets, 2^20 blocks):
    the first frame is bit-exact — hash entries incl. excess chains, voxels,
    maps."""
    cfg = CONFIGS["C3"].with_(tracking=False)
    p, o = _pair(olib, cfg, False)
    pose = trajectory(1)[0]
    d = vf_py.render_depth(olib, cfg, pose, BOX_ROOM_SPHERES, BOX_ROOM_PLANES)
    p.set_pose(pose)
    st = p.process_frame(None, d)
    so = o.process(d, None, pose)
    assert (st.blocks_allocated, st.visible_blocks) == (so.blocks_allocated, so.visible_blocks)
    assert st.blocks_allocated > 100_000
    _same_state(p, o)
    p.close()


@pytest.mark.parametrize("variant", ["stop_at_max", "bucket1", "bucket4", "rgb_stop_at_max"])
def test_scene_and_hash_parameters(olib, variant):
    """Non-default SceneParams / HashConfig: stop_integrating_at_max with a
    small max_weight (integrate_voxel's early out, integration.hpp:105-107),
    one- and four-slot buckets (hash_volume.hpp:49-58): known poses,
    bit-exact over a short sequence."""
    cfg = CONFIGS["T320"].with_(tracking=False)
    if variant in ("stop_at_max", "rgb_stop_at_max"):
        cfg = cfg.with_(max_weight=3, stop_integrating_at_max=True, voxel_type=2 if variant.startswith("rgb") else 1)
    elif variant == "bucket1":
        cfg = cfg.with_(hash=HashConfig(bucket_count=1 << 17, bucket_size=1, excess_count=1 << 15, block_count=1 << 15))
    else:
        cfg = cfg.with_(hash=HashConfig(bucket_count=1 << 15, bucket_size=4, excess_count=1 << 13, block_count=1 << 15))
    rgb = cfg.voxel_type == 2
    vsize = 8 if rgb else 4
    p, o = _pair(olib, cfg, False)
    for pose, d, col in frames(olib, cfg, 6, rgb=rgb):
        p.set_pose(pose)
        st = p.process_frame(col, d)
        so = o.process(d, col, pose)
        assert (st.blocks_allocated, st.visible_blocks) == (so.blocks_allocated, so.visible_blocks)
        _same_state(p, o, vsize)
    p.close()


def test_far_from_origin_bit_exact(olib):
    """Integration skips the per-voxel border compares on blocks whose worst
    corner clears every image bound by a margin that grows with the
    coordinates (block_interior, vf_integrate.cu).  ~300 m from the origin the
    float camera coordinates carry ~1e-5 m of rounding; the known-pose
    sequence must still be bit-exact against the oracle."""
    cfg = CONFIGS["T320"].with_(tracking=False)
    p, o = _pair(olib, cfg, False)
    for pose, depth, _ in frames(olib, cfg, 3):
        q = far_pose(pose)
        p.set_pose(q)
        st = p.process_frame(None, depth)
        so = o.process(depth, None, q)
        assert (st.blocks_allocated, st.visible_blocks) == (so.blocks_allocated, so.visible_blocks)
        assert st.visible_blocks > 100
        _same_state(p, o)
    p.close()
