"""Fast integration mode (vf_settings.integration_mode = 1, VoxelS and
VoxelSRgb) against the oracle: the reference's voxels / pixels / update rule with FMA-contracted,
approximate-reciprocal arithmetic (vf_integrate.cu, k_integrate_fast).

Bar (SURVEY.md §8(c) TSDF tolerance: <= 1 LSB of int16, <= 1 count of
weight): starting from the oracle's own volume, over every voxel that either
side changes in the frame, |delta sdf| <= 1 LSB and weight identical on
>= 99.9 %.  Allocation, visibility and everything else stay bit-exact.
"""
from dataclasses import replace

import numpy as np
import pytest

import vf_py
from helpers import entries_equal, far_pose, frames, voxel_payload
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import CONFIGS

pytestmark = pytest.mark.gpu


def _free_stacks(olib, o, cfg):
    import ctypes as C
    vt, et = C.c_int(), C.c_int()
    vs = np.zeros(cfg.hash.block_count, np.int32)
    es = np.zeros(cfg.hash.excess_count, np.int32)
    olib.lib.vfo_free_stacks(o.h, C.byref(vt), vs.ctypes.data_as(C.c_void_p), C.byref(et),
                             es.ctypes.data_as(C.c_void_p))
    return vt.value, vs, et.value, es


def _sdf_w(v):
    v = voxel_payload(v, 4).reshape(-1, 3)
    return v[:, :2].copy().view(np.int16)[:, 0].astype(np.int64), v[:, 2].astype(np.int64)


@pytest.mark.parametrize("name,checked,far", [("T320", (0, 2, 4), False), ("C1", (0, 6, 12), False),
                                              ("T320", (0, 2), True)])
def test_fast_integration_within_one_lsb(olib, name, checked, far):
    """far: the same frames ~300 m from the origin (helpers.far_pose),
    where block_interior's rounding allowance is largest."""
    cfg = CONFIGS[name].with_(tracking=False)
    fr = frames(olib, cfg, max(checked) + 1)
    if far:
        fr = [(far_pose(pose), d, c) for pose, d, c in fr]
    o = vf_py.Volume(olib, cfg, tracking=False)
    s, c = settings_from_config(cfg)
    p = make_pipeline(replace(s, integration_mode=1), c)
    worst = 1.0
    for i, (pose, depth, _) in enumerate(fr):
        if i in checked:
            p.import_state(o.entries(), o.voxels(), *_free_stacks(olib, o, cfg))
            sdf0, w0 = _sdf_w(o.voxels())
            st_g = p.allocate(depth, pose)
            st = vf_py.AllocStats()
            olib.lib.vfo_stage_allocate(o.h, depth.ctypes.data_as(vf_py.C.c_void_p),
                                        pose.ctypes.data_as(vf_py.C.c_void_p), vf_py.C.byref(st))
            assert entries_equal(p.entries(), o.entries()), f"frame {i}: allocation differs"
            assert st_g.allocated == st.allocated
            olib.lib.vfo_stage_integrate(o.h, depth.ctypes.data_as(vf_py.C.c_void_p), None,
                                         pose.ctypes.data_as(vf_py.C.c_void_p))
            p.integrate(depth, None, pose)
            sdf_o, w_o = _sdf_w(o.voxels())
            sdf_g, w_g = _sdf_w(p.voxels())
            changed = (sdf_o != sdf0) | (w_o != w0) | (sdf_g != sdf0) | (w_g != w0)
            n = int(changed.sum())
            d = np.abs(sdf_g[changed] - sdf_o[changed])
            ok_sdf = float(np.mean(d <= 1))
            ok_w = float(np.mean(w_g[changed] == w_o[changed]))
            exact = float(np.mean(d == 0))
            print(f"{name} frame {i}: {n} voxels updated, sdf exact {exact:.5f}, <=1 LSB {ok_sdf:.6f}, "
                  f"max {int(d.max()) if n else 0}, weight exact {ok_w:.6f}")
            assert n > 1000
            assert ok_sdf >= 0.999 and ok_w >= 0.999, (i, ok_sdf, ok_w)
            worst = min(worst, ok_sdf, ok_w)
            # the rest of the frame runs from here on the oracle's volume
            olib.lib.vfo_stage_raycast(o.h, pose.ctypes.data_as(vf_py.C.c_void_p))
        else:
            o.process(depth, None, pose)
    p.close()
    print(f"{name}: worst fraction within the bar {worst:.6f}")


def test_fast_mode_tracked_sequence_close_to_exact(olib):
    """Tracked C1 frames with fast integration: same tracking decisions as the
    exact pipeline, poses within the §8(c) pose bar."""
    from helpers import centre_dist, rot_angle
    cfg = CONFIGS["C1"]
    s, c = settings_from_config(cfg)
    pe, pf = make_pipeline(s, c), make_pipeline(replace(s, integration_mode=1), c)
    for i, (pose, depth, _) in enumerate(frames(olib, cfg, 12)):
        se, sf = pe.process_frame(None, depth), pf.process_frame(None, depth)
        assert se.tracking_ok and sf.tracking_ok
        assert rot_angle(pe.pose(), pf.pose()) <= 1e-4 and centre_dist(pe.pose(), pf.pose()) <= 1e-4, i
    pe.close()
    pf.close()


def test_fast_integration_colour_voxels(olib):
    """VoxelSRgb (config 2 frames, known poses) from the oracle's own volume:
    SDF within 1 LSB and weights exact as for VoxelS; colour channels within
    one count and colour weights exact on >= 99.9 % of the voxels either side
    changes (the colour blend's quotient is an approximate product, and the RGB
    camera's pixel may flip within a few ulp of a pixel edge)."""
    cfg = CONFIGS["C2"]
    fr = frames(olib, cfg, 7, rgb=True)
    o = vf_py.Volume(olib, cfg, tracking=False)
    s, c = settings_from_config(cfg)
    p = make_pipeline(replace(s, integration_mode=1), c)
    for i, (pose, depth, col) in enumerate(fr):
        if i not in (0, 6):
            o.process(depth, col, pose)
            continue
        p.import_state(o.entries(), o.voxels(), *_free_stacks(olib, o, cfg))
        before = voxel_payload(o.voxels(), 8).reshape(-1, 7).astype(np.int64)
        p.allocate(depth, pose)
        st = vf_py.AllocStats()
        olib.lib.vfo_stage_allocate(o.h, depth.ctypes.data_as(vf_py.C.c_void_p),
                                    pose.ctypes.data_as(vf_py.C.c_void_p), vf_py.C.byref(st))
        assert entries_equal(p.entries(), o.entries())
        olib.lib.vfo_stage_integrate(o.h, depth.ctypes.data_as(vf_py.C.c_void_p),
                                     col.ctypes.data_as(vf_py.C.c_void_p), pose.ctypes.data_as(vf_py.C.c_void_p))
        p.integrate(depth, col, pose)
        vo = voxel_payload(o.voxels(), 8).reshape(-1, 7).astype(np.int64)
        vg = voxel_payload(p.voxels(), 8).reshape(-1, 7).astype(np.int64)
        changed = (vo != before).any(1) | (vg != before).any(1)
        sdf = lambda v: (v[:, 0] | (v[:, 1] << 8)).astype(np.uint16).view(np.int16).astype(np.int64)
        d_sdf = np.abs(sdf(vg[changed]) - sdf(vo[changed]))
        d_w = vg[changed, 2] != vo[changed, 2]
        d_clr = np.abs(vg[changed, 3:6] - vo[changed, 3:6]).max(1)
        d_wc = vg[changed, 6] != vo[changed, 6]
        print(f"C2 frame {i}: {int(changed.sum())} voxels updated, sdf <=1 LSB {np.mean(d_sdf <= 1):.6f}, "
              f"weight exact {1 - np.mean(d_w):.6f}, colour <=1 {np.mean(d_clr <= 1):.6f} (exact "
              f"{np.mean(d_clr == 0):.5f}), colour weight exact {1 - np.mean(d_wc):.6f}")
        assert np.mean(d_sdf <= 1) >= 0.999 and np.mean(d_w) <= 0.001
        assert np.mean(d_clr <= 1) >= 0.999 and np.mean(d_wc) <= 0.001
        olib.lib.vfo_stage_raycast(o.h, pose.ctypes.data_as(vf_py.C.c_void_p))
    p.close()
