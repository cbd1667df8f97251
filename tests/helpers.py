"""Shared helpers for the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

import vf_py
from paper_1410_0925_b200.scene import BOX_ROOM_PLANES, BOX_ROOM_SPHERES, CONFIGS, trajectory

ENTRY_FIELDS = ("x", "y", "z", "offset", "block_state")


def frames(olib, cfg, n, rgb=False, amplitude=1.0):
    poses = trajectory(n, amplitude)
    out = []
    for i in range(n):
        d = vf_py.render_depth(olib, cfg, poses[i], BOX_ROOM_SPHERES, BOX_ROOM_PLANES)
        c = vf_py.render_rgb(olib, cfg, poses[i], BOX_ROOM_SPHERES, BOX_ROOM_PLANES) if rgb else None
        out.append((poses[i], d, c))
    return out


def far_pose(pose, offset=(150.3, -80.7, 230.1)):
    """The same view with the world shifted: camera centre c -> c + offset,
    so t -> t - R offset (world-to-camera, scene.trajectory)."""
    q = np.array(pose, dtype=np.float64).copy()
    q[9:] = q[9:] - q[:9].reshape(3, 3) @ np.asarray(offset)
    return q


def entries_equal(a, b):
    return all(np.array_equal(a[f], b[f]) for f in ENTRY_FIELDS)


def voxel_payload(v: np.ndarray, vsize: int) -> np.ndarray:
    """Voxel bytes without the padding byte (sizeof VoxelS = 4, VoxelSRgb = 8)."""
    v = v.reshape(-1, vsize)
    return v[:, : vsize - 1]


def allocated_blocks(entries, voxels, vsize):
    """{(x,y,z): voxel payload bytes} for all allocated entries — layout-independent."""
    pay = voxel_payload(voxels, vsize).reshape(-1, 512, vsize - 1)
    out = {}
    for e in entries[entries["block_state"] >= 0]:
        out[(int(e["x"]), int(e["y"]), int(e["z"]))] = pay[int(e["block_state"])]
    return out


def rot_angle(p, q):
    """Angle (rad) between the rotations of two 12-double poses."""
    ra, rb = np.asarray(p[:9]).reshape(3, 3), np.asarray(q[:9]).reshape(3, 3)
    return float(2.0 * np.arcsin(min(1.0, np.linalg.norm(ra - rb) / np.sqrt(8.0))))


def centre_dist(p, q):
    ra, rb = np.asarray(p[:9]).reshape(3, 3), np.asarray(q[:9]).reshape(3, 3)
    ca, cb = -ra.T @ np.asarray(p[9:]), -rb.T @ np.asarray(q[9:])
    return float(np.linalg.norm(ca - cb))


# Swap-engine parity cases (tests/golden/make_golden.py): (block_count,
# swap_buffer_blocks) on T160 with the pan trajectory — a VBA so small that
# swap-ins are deferred, and one large enough that blocks come back.
SWAP_CASES = {
    "T160_swap_small_vba": (1200, 16),
    "T160_swap_roundtrip": (6000, 64),
}


def swap_config(name):
    from paper_1410_0925_b200.scene import CONFIGS, HashConfig
    blocks, b = SWAP_CASES[name]
    return CONFIGS["T160"].with_(tracking=False, use_swapping=True, swap_buffer_blocks=b,
                                 hash=HashConfig(bucket_count=1 << 14, excess_count=1 << 12, block_count=blocks))
