"""How far does Eigen's reduction order move the results?

The oracle, the shim-built reference (oracle/_ref) and the kernels share one
arithmetic contract: every 3-term sum left to right (oracle/eigen_shim).  A
stock Eigen build may associate fixed-size reductions differently -- its
unrolled redux splits them in halves, x0 + (x1 + x2) (Redux.h).  The
reference is therefore also built with every reduction in that association
(oracle/_ref_halving, `make -C oracle ref_halving`), and the GPU path is
compared against THAT build at the §8(c) tolerances:

* known poses (C1, 10 frames): block sets identical; SDF within 1 LSB and
  weights exact on >= 99.9 % of voxels; hit masks >= 99.9 % identical;
  points within half a voxel on >= 99.9 % and normals within 1 deg on >= 99 %
  of the pixels both hit;
* tracked (C1, 12 frames): poses within 1e-4 rad / 0.1 mm per frame, then the
  long-sequence bars of tests/test_gpu_parity_long.py.

Measured numbers go to VF_PARITY_OUT (JSON) when set.
"""
from __future__ import annotations

import json
import os

import pytest

import vf_py
from assoc_stats import compare
from helpers import centre_dist, frames, rot_angle
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import CONFIGS

pytestmark = pytest.mark.gpu
RESULTS = {}


@pytest.fixture(scope="module")
def hlib():
    if not vf_py.ref_halving_available():
        pytest.skip("oracle/_ref_halving not built (needs /root/reference at build time)")
    lib = vf_py.ref_halving_lib()
    lib.lib.vfr_set_threads(1)
    return lib


def _record(name, out):
    RESULTS[name] = out
    path = os.environ.get("VF_PARITY_OUT")
    if path:
        with open(path, "w") as f:
            json.dump(RESULTS, f, indent=1)
    print(name, json.dumps(out))


def test_known_pose_gpu_vs_halving_reference(hlib):
    cfg = CONFIGS["C1"].with_(tracking=False)
    s, c = settings_from_config(cfg)
    p = make_pipeline(s, c)
    r = vf_py.Volume(hlib, cfg, tracking=False)
    for pose, d, _ in frames(hlib, cfg, 10):
        p.set_pose(pose)
        p.process_frame(None, d)
        r.process(d, None, pose)
    out = compare(p.entries(), p.voxels(), r.entries(), r.voxels(), p.tracking_state(), r.maps(), cfg.voxel_size)
    p.close()
    r.close()
    _record("C1_known_pose_10", out)
    assert out["blocks_common_frac"] >= 0.999
    assert out["sdf_le1_frac"] >= 0.999 and out["weight_exact_frac"] >= 0.999
    assert out["hit_agreement"] >= 0.999 and out["point_within_half_voxel_frac"] >= 0.999
    assert out["normal_within_1deg_frac"] >= 0.99


def test_tracked_gpu_vs_halving_reference(hlib):
    cfg = CONFIGS["C1"]
    s, c = settings_from_config(cfg)
    p = make_pipeline(s, c)
    r = vf_py.Volume(hlib, cfg, tracking=True)
    worst = [0.0, 0.0]
    for pose, d, _ in frames(hlib, cfg, 12):
        sg, sr = p.process_frame(None, d), r.process(d)
        assert sg.tracking_ok == bool(sr.tracking_ok)
        worst = [max(worst[0], rot_angle(p.pose(), r.pose())), max(worst[1], centre_dist(p.pose(), r.pose()))]
    out = compare(p.entries(), p.voxels(), r.entries(), r.voxels(), p.tracking_state(), r.maps(), cfg.voxel_size)
    out.update({"max_rot_rad": worst[0], "max_centre_m": worst[1]})
    p.close()
    r.close()
    _record("C1_tracked_12", out)
    assert worst[0] <= 1e-4 and worst[1] <= 1e-4
    assert out["blocks_common_frac"] >= 0.999
    assert out["sdf_le64_frac"] >= 0.99 and out["hit_agreement"] >= 0.999
