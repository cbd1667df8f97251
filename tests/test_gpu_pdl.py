"""GPU: programmatic dependent launch (PDL) changes scheduling only.  The
frame's main-stream kernels (pyramid, ICP, allocation, integration, raycast,
the Ren loop) are launched with the programmatic-serialization attribute and
each waits on its predecessor grid first (vf_kernels.h launch_pdl,
vf_device.cuh pdl_enter).  A tracked C1 run and a C1R run (ICP + Ren) with
PDL on must end bit-identical -- volume digest, poses, maps -- to the same
runs in a process with VF_PDL=0 (the switch is read once per process)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

_RUN = r"""
import hashlib, json, sys
sys.path.insert(0, %(root)r); sys.path.insert(0, %(root)r + '/oracle'); sys.path.insert(0, %(root)r + '/tests')
import numpy as np
import vf_py
from helpers import frames
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import CONFIGS
olib = vf_py.oracle_lib()
out = {}
for name in ("C1", "C1R"):
    cfg = CONFIGS[name]
    s, c = settings_from_config(cfg)
    p = make_pipeline(s, c)
    poses, its = [], []
    for pose, d, _ in frames(olib, cfg, 6):
        st = p.process_frame(None, d)
        poses.append(p.pose().tolist())
        its.append(int(st.tracking_iterations))
    pts, nrm = p.tracking_state()
    out[name] = {"digest": int(p.volume_digest()), "poses": poses, "iters": its,
                 "maps": hashlib.sha256(pts.tobytes() + nrm.tobytes()).hexdigest()}
    p.close()
print(json.dumps(out))
"""


def _run(pdl: str):
    env = dict(os.environ, VF_PDL=pdl)
    r = subprocess.run([sys.executable, "-c", _RUN % {"root": str(ROOT)}], env=env, capture_output=True, text=True,
                       timeout=600, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_pdl_on_off_bit_identical():
    on, off = _run("1"), _run("0")
    for name in ("C1", "C1R"):
        assert on[name]["digest"] == off[name]["digest"], name
        assert on[name]["iters"] == off[name]["iters"], name
        assert np.array_equal(np.array(on[name]["poses"]), np.array(off[name]["poses"])), name
        assert on[name]["maps"] == off[name]["maps"], name
