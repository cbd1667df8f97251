"""A recorded sequence on disk (16-bit P5 disparity, P6 colour, calibration
text) through paper_1410_0925_b200.io.run_sequence — raw big-endian
payloads into IPipeline::process_raw_frame, byte swap and
disparity_image_to_depth on the GPU — against the same frames converted by
the oracle and fed as depth."""
import numpy as np
import pytest

import vf_py
from helpers import entries_equal, frames
from paper_1410_0925_b200 import io as vio
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import CONFIGS

pytestmark = pytest.mark.gpu


def test_recorded_sequence_through_raw_frames(olib, tmp_path):
    cfg = CONFIGS["T320"]
    fx, fy, cx, cy, w, h = cfg.intrinsics
    a, b = 1135.09, 0.0819141
    calib_text = (f"{w} {h}\n{fx} {fy}\n{cx} {cy}\n\n{w} {h}\n{fx} {fy}\n{cx} {cy}\n\n"
                  "1 0 0 0\n0 1 0 0\n0 0 1 0\n\n" f"{a} {b}\n")
    (tmp_path / "calib.txt").write_text(calib_text)
    fr = frames(olib, cfg, 4)
    for i, (_, d, _) in enumerate(fr):
        # depth_to_disparity (calibration.hpp:62-70)
        with np.errstate(divide="ignore"):
            dd = np.where(d > 0, np.float32(a) - np.float32(8.0) * np.float32(b) * np.float32(fx) / d, 65535)
        disp = np.where((dd < 0) | (dd > 65535), 65535, dd + 0.5).astype(np.uint16)
        vio.write_pgm16(str(tmp_path / f"{i:04d}.pgm"), disp)
    calib = vio.load_calibration(str(tmp_path / "calib.txt"))
    s, _ = settings_from_config(cfg)
    scan = vio.scan_sequence_dir(str(tmp_path))
    assert [f.index for f in scan.frames] == [0, 1, 2, 3] and scan.disparity_only == 4
    p = make_pipeline(s, calib)
    stats = vio.run_sequence(p, scan)  # streaming: vf_submit_raw_frame / vf_collect_frame
    r = make_pipeline(s, calib)
    stats_sync = vio.run_sequence(r, scan, streaming=False)  # vf_process_raw_frame
    for a_, b_ in zip(stats, stats_sync):
        assert a_.frame == b_.frame and np.array_equal(a_.pose, b_.pose)
    assert entries_equal(p.entries(), r.entries()) and np.array_equal(p.voxels(), r.voxels())
    r.close()
    q = make_pipeline(s, calib)
    for fp, st in zip(scan.frames, stats):
        depth = vf_py.disparity_to_depth(olib, vio.read_pgm16(fp.disparity_path), a, b, fx, s.max_depth)
        sq = q.process_frame(None, depth)
        assert bool(st.tracking_ok) == bool(sq.tracking_ok)
        assert np.array_equal(st.pose, sq.pose)
    assert entries_equal(p.entries(), q.entries())
    assert np.array_equal(p.voxels(), q.voxels())
    p.close()
    q.close()
