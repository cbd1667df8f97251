"""Recorded-sequence input for the Python mirror: the reference's file formats
and the disparity path into the GPU.

Host I/O, restated from the reference's behaviour (not its code):

* ``read_pgm16`` / ``read_ppm`` — binary P5 (maxval 65535, big-endian
  samples) and P6 (maxval 255) rasters, '#' comments in the header
  (proj/src/pnm.cpp:12-95);
* ``parse_calibration`` / ``load_calibration`` — the four-block text format:
  RGB intrinsics, depth intrinsics, the 3x4 RGB-to-depth extrinsic (rows of
  R | t, re-orthonormalised when within 1e-3 of orthonormal), the disparity
  scalars a, b (proj/src/calibration.cpp:12-88);
* ``scan_sequence_dir`` — numbered ``*.ppm`` / ``*.pgm`` pairs
  (proj/src/sequence.cpp:9-43).

``run_sequence`` feeds a scanned sequence to a ``Pipeline`` through
``process_raw_frame`` (or its streaming form, the default) with the P5
payload's raw big-endian bytes: the byte swap and disparity_image_to_depth
run on the GPU (vf_process_raw_frame / vf_submit_raw_frame), the host only
reads the files, overlapped with the GPU when streaming.
"""
from __future__ import annotations

import os
import re
from dataclasses import dataclass, field

import numpy as np

from .pipeline import Calibration, Intrinsics


class PnmError(ValueError):
    """pnm.cpp's PnmError."""


class CalibrationError(ValueError):
    """calibration.hpp's CalibrationError (with the 1-based line)."""

    def __init__(self, what: str, line: int):
        super().__init__(what)
        self.line = line


# ---------------------------------------------------------------------------
# PNM (pnm.cpp)
# ---------------------------------------------------------------------------
def _header(buf: bytes, magic: bytes, maxval_expected: int):
    if len(buf) < 2 or buf[:2] != magic:
        raise PnmError(f"bad magic, expected {magic.decode()}")
    pos = 2
    vals = []
    for what in ("width", "height", "maxval"):
        while True:
            if pos >= len(buf):
                raise PnmError(f"unexpected end of header before {what}")
            c = buf[pos:pos + 1]
            if c.isspace():
                pos += 1
            elif c == b"#":
                nl = buf.find(b"\n", pos)
                pos = len(buf) if nl < 0 else nl + 1
            else:
                break
        start = pos
        while pos < len(buf) and buf[pos:pos + 1].isdigit():
            pos += 1
        if pos == start:
            raise PnmError(f"malformed header field: {what}")
        vals.append(int(buf[start:pos]))
    w, h, maxval = vals
    if maxval != maxval_expected:
        raise PnmError(f"unsupported maxval {maxval}, expected {maxval_expected}")
    pos += 1  # single whitespace byte before the raster
    if w <= 0 or h <= 0:
        raise PnmError("non-positive image dimensions")
    return w, h, pos


def read_pgm16_raw(path: str) -> np.ndarray:
    """The P5 raster's raw bytes as big-endian u16 words, viewed as native
    ``uint16`` (H x W): ready for ``process_raw_frame(..., big_endian=True)``."""
    buf = open(path, "rb").read()
    w, h, pos = _header(buf, b"P5", 65535)
    if len(buf) - pos < w * h * 2:
        raise PnmError("truncated raster data")
    return np.frombuffer(buf, np.uint16, w * h, pos).reshape(h, w)


def read_pgm16(path: str) -> np.ndarray:
    """read_pgm16 (pnm.cpp:63-73): H x W uint16 samples."""
    return read_pgm16_raw(path).byteswap()


def read_ppm(path: str) -> np.ndarray:
    """read_ppm (pnm.cpp:85-95): H x W x 3 uint8."""
    buf = open(path, "rb").read()
    w, h, pos = _header(buf, b"P6", 255)
    if len(buf) - pos < w * h * 3:
        raise PnmError("truncated raster data")
    return np.frombuffer(buf, np.uint8, w * h * 3, pos).reshape(h, w, 3).copy()


def write_pgm16(path: str, img: np.ndarray) -> None:
    """write_pgm16 (pnm.cpp:75-83)."""
    h, w = img.shape
    with open(path, "wb") as f:
        f.write(f"P5\n{w} {h}\n65535\n".encode())
        f.write(np.ascontiguousarray(img, np.uint16).astype(">u2").tobytes())


def write_ppm(path: str, img: np.ndarray) -> None:
    """write_ppm (pnm.cpp:97-106)."""
    h, w, _ = img.shape
    with open(path, "wb") as f:
        f.write(f"P6\n{w} {h}\n255\n".encode())
        f.write(np.ascontiguousarray(img, np.uint8).tobytes())


# ---------------------------------------------------------------------------
# calibration (calibration.cpp)
# ---------------------------------------------------------------------------
def _orthonormalize(m: np.ndarray) -> np.ndarray:
    """orthonormalize (pose.cpp:9-18): U V^T of the SVD, reflection-fixed.
    (The reference's Jacobi SVD and LAPACK's agree to rounding.)"""
    u, _, vt = np.linalg.svd(m)
    r = u @ vt
    if np.linalg.det(r) < 0:
        r = u @ np.diag([1.0, 1.0, -1.0]) @ vt
    return r


def parse_calibration(text: str) -> Calibration:
    """parse_calibration (calibration.cpp:66-88)."""
    toks = []  # (token, line)
    line = 1
    for piece in re.split(r"(\s+)", text):
        if not piece:
            continue
        if piece.isspace():
            line += piece.count("\n")
        else:
            toks.append((piece, line))
    it = iter(toks)
    last_line = [line]

    def number(what):
        try:
            tok, ln = next(it)
        except StopIteration:
            raise CalibrationError(f"unexpected end of file while reading {what}", last_line[0]) from None
        last_line[0] = ln
        try:
            return float(tok)
        except ValueError:
            raise CalibrationError(f"non-numeric token '{tok}' while reading {what}", ln) from None

    def intrinsics(camera):
        w, h = int(number(camera)), int(number(camera))
        fx, fy, cx, cy = number(camera), number(camera), number(camera), number(camera)
        if not (fx > 0 and fy > 0 and 0 < cx < w and 0 < cy < h):  # Intrinsics::valid
            raise CalibrationError(f"invalid intrinsics for {camera}", last_line[0])
        return Intrinsics(fx, fy, cx, cy, w, h)

    rgb = intrinsics("rgb camera (block 1)")
    depth = intrinsics("depth camera (block 2)")
    r = np.zeros((3, 3))
    t = np.zeros(3)
    for row in range(3):
        for col in range(3):
            r[row, col] = number("extrinsic (block 3)")
        t[row] = number("extrinsic (block 3)")
    if np.linalg.norm(r.T @ r - np.eye(3)) > 1e-3:  # Pose::orthonormality_error
        raise CalibrationError("extrinsic rotation is not orthonormal", last_line[0])
    r = _orthonormalize(r)
    a = number("disparity scalars (block 4)")
    b = number("disparity scalars (block 4)")
    return Calibration(depth=depth, rgb=rgb, rgb_to_depth=np.concatenate([r.reshape(-1), t]), disparity_a=a,
                       disparity_b=b)


def load_calibration(path: str) -> Calibration:
    try:
        text = open(path).read()
    except OSError:
        raise CalibrationError(f"cannot open calibration file: {path}", 0) from None
    return parse_calibration(text)


# ---------------------------------------------------------------------------
# sequences (sequence.cpp)
# ---------------------------------------------------------------------------
@dataclass
class FramePair:
    index: int
    rgb_path: str  # "" without colour
    disparity_path: str


@dataclass
class SequenceScan:
    frames: list = field(default_factory=list)
    rgb_only: int = 0
    disparity_only: int = 0


_FRAME = re.compile(r"^(.*?)(\d+)\.(ppm|pgm)$", re.IGNORECASE)


def scan_sequence_dir(path: str) -> SequenceScan:
    """scan_sequence_dir (sequence.cpp:9-43)."""
    slots: dict = {}
    for name in os.listdir(path):
        full = os.path.join(path, name)
        if not os.path.isfile(full):
            continue
        m = _FRAME.match(name)
        if not m:
            continue
        idx = int(m.group(2))
        slot = slots.setdefault(idx, {"rgb": "", "disparity": ""})
        slot["rgb" if m.group(3).lower() == "ppm" else "disparity"] = full
    scan = SequenceScan()
    for idx in sorted(slots):
        s = slots[idx]
        if not s["disparity"]:
            scan.rgb_only += 1
            continue
        if not s["rgb"]:
            scan.disparity_only += 1
        scan.frames.append(FramePair(idx, s["rgb"], s["disparity"]))
    return scan


def run_sequence(pipeline, scan: SequenceScan, limit: int | None = None, streaming: bool = True):
    """Feed a scanned recorded sequence through IPipeline::process_raw_frame;
    returns the per-frame FrameStats.  streaming: the submit / collect form
    with two frames in flight, so reading frame n + 1 from disk and its upload
    overlap frame n on the GPU (same results)."""
    out = []
    for fp in scan.frames[:limit]:
        raw = read_pgm16_raw(fp.disparity_path)
        rgb = read_ppm(fp.rgb_path) if fp.rgb_path else None
        if not streaming:
            out.append(pipeline.process_raw_frame(rgb, raw, big_endian=True))
            continue
        pipeline.submit_raw_frame(rgb, raw, big_endian=True)
        if pipeline.frames_in_flight() >= 2:
            out.append(pipeline.collect_frame())
    while streaming and pipeline.frames_in_flight() > 0:
        out.append(pipeline.collect_frame())
    return out
