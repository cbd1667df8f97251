"""CPU suite: the Python recorded-sequence I/O (paper_1410_0925_b200/io.py)
against the reference's own readers (pnm.cpp, calibration.cpp,
sequence.cpp through oracle/_ref).  No GPU needed."""
import ctypes as C

import numpy as np
import pytest

from paper_1410_0925_b200 import io as vio

CALIB = """640 480
573.71 574.394
346.471 249.031

640 480
573.71 574.394
346.471 249.031

0.99999 0.0001 0 0.025
-0.0001 0.99999 0 0
0 0 1 0

1135.09 0.0819141
"""


def _ref_calib(rlib, text):
    f = rlib.lib.vfr_parse_calibration
    f.argtypes = [C.c_char_p, C.c_void_p, C.POINTER(C.c_int)]
    out = np.zeros(26)
    line = C.c_int(-1)
    rc = f(text.encode(), out.ctypes.data_as(C.c_void_p), C.byref(line))
    return rc, out, line.value


def test_calibration_matches_reference(rlib):
    c = vio.parse_calibration(CALIB)
    rc, out, _ = _ref_calib(rlib, CALIB)
    assert rc == 0
    for k, cam in enumerate((c.rgb, c.depth)):
        assert [cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy] == list(out[6 * k:6 * k + 6])
    # the re-orthonormalised extrinsic: LAPACK vs the reference's Jacobi SVD
    assert np.abs(np.asarray(c.rgb_to_depth) - out[12:24]).max() < 1e-12
    assert (c.disparity_a, c.disparity_b) == (out[24], out[25])


@pytest.mark.parametrize("bad", [
    CALIB.replace("573.71 574.394\n346.471", "573.71 x\n346.471", 1),   # non-numeric
    CALIB.rsplit("1135.09", 1)[0],                                        # truncated
    CALIB.replace("346.471 249.031", "700 249.031", 1),                   # cx outside the image
    CALIB.replace("0.99999 0.0001 0 0.025", "0.9 0.1 0 0.025"),           # not orthonormal
])
def test_calibration_errors_match_reference(rlib, bad):
    rc, _, _ = _ref_calib(rlib, bad)
    assert rc == -1
    with pytest.raises(vio.CalibrationError):
        vio.parse_calibration(bad)


def test_pnm_round_trip_matches_reference(rlib, tmp_path):
    rng = np.random.default_rng(7)
    d = rng.integers(0, 65536, size=(37, 53), dtype=np.uint16)
    c = rng.integers(0, 256, size=(37, 53, 3), dtype=np.uint8)
    pg, pp = tmp_path / "0007.pgm", tmp_path / "0007.ppm"
    vio.write_pgm16(str(pg), d)
    vio.write_ppm(str(pp), c)
    # a header comment, as the reference's reader allows
    raw = pg.read_bytes()
    pg.write_bytes(raw.replace(b"P5\n", b"P5\n# recorded\n", 1))
    assert np.array_equal(vio.read_pgm16(str(pg)), d)
    assert np.array_equal(vio.read_pgm16_raw(str(pg)).byteswap(), d)
    assert np.array_equal(vio.read_ppm(str(pp)), c)
    f = rlib.lib.vfr_read_pgm16
    f.argtypes = [C.c_char_p, C.c_void_p, C.c_long, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    out = np.zeros(d.size, np.uint16)
    w, h = C.c_int(), C.c_int()
    assert f(str(pg).encode(), out.ctypes.data_as(C.c_void_p), out.size, C.byref(w), C.byref(h)) == 0
    assert (w.value, h.value) == (53, 37) and np.array_equal(out.reshape(37, 53), d)
    g = rlib.lib.vfr_read_ppm
    g.argtypes = [C.c_char_p, C.c_void_p, C.c_long, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    outc = np.zeros(c.size, np.uint8)
    assert g(str(pp).encode(), outc.ctypes.data_as(C.c_void_p), outc.size, C.byref(w), C.byref(h)) == 0
    assert np.array_equal(outc.reshape(37, 53, 3), c)
    # malformed: wrong maxval
    bad = tmp_path / "bad.pgm"
    bad.write_bytes(b"P5\n2 2\n255\n" + bytes(8))
    with pytest.raises(vio.PnmError):
        vio.read_pgm16(str(bad))
    assert f(str(bad).encode(), out.ctypes.data_as(C.c_void_p), out.size, C.byref(w), C.byref(h)) == -1


def test_sequence_scan_matches_reference(rlib, tmp_path):
    z = np.zeros((2, 2), np.uint16)
    zc = np.zeros((2, 2, 3), np.uint8)
    for i in (0, 1, 2, 5):
        vio.write_pgm16(str(tmp_path / f"depth{i:04d}.pgm"), z)
    for i in (0, 2, 3):
        vio.write_ppm(str(tmp_path / f"rgb{i:04d}.PPM"), zc)
    (tmp_path / "notes.txt").write_text("x")
    scan = vio.scan_sequence_dir(str(tmp_path))
    import subprocess
    from pathlib import Path
    tool = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "ref_tools"
    if not tool.exists():
        pytest.skip("oracle/_ref/ref_tools not built")
    lines = subprocess.run([str(tool), "scan", str(tmp_path)], capture_output=True, text=True,
                           check=True).stdout.split("\n")
    head = lines[0].split()
    n, ro, do = int(head[1]), int(head[3]), int(head[5])
    ref = [tuple(map(int, ln.split())) for ln in lines[1:1 + n]]
    assert [(fp.index, 1 if fp.rgb_path else 0) for fp in scan.frames] == ref
    assert (scan.rgb_only, scan.disparity_only) == (ro, do)
