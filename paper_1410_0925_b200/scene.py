"""Benchmark configurations and the synthetic scene they are quoted on.

BASELINE.json names five configurations; this module pins all five (C1-C4
on one GPU, C5 sharded across GPUs) plus small parity cases, following SURVEY.md §8(d):

* camera: the paper's depth intrinsics, 640x480, fx 573.71, fy 574.394,
  cx 346.471, cy 249.031 (reference PAPER.md:798-800); 1280x960 doubles the
  focal lengths and maps c' = 2c + 0.5, the inverse of ``Intrinsics::half``
  (reference proj/include/voxfuse/core/intrinsics.hpp:22-31);
* scene: a closed box room (six inward-facing planes) plus spheres, in the
  primitive set of the reference renderer (proj/include/voxfuse/io/synthetic.hpp:14-32);
* trajectory: 100 frames of small motion (< 2 deg, < 2 cm per frame)
  expressed relative to frame 0, which the pipeline fixes to the identity
  (proj/include/voxfuse/engine/pipeline_impl.hpp:78).

Pure data + numpy: no rendering here (the GPU renderer lives in the CUDA
library, the CPU one in the test oracle).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

# Paper depth camera.
PAPER_DEPTH_640 = (573.71, 574.394, 346.471, 249.031, 640, 480)


def intrinsics_for(width: int, height: int):
    """Intrinsics of the paper camera at width x height (power-of-two scales of 640x480)."""
    fx, fy, cx, cy, w0, h0 = PAPER_DEPTH_640
    s = width / w0
    if abs(s - round(s)) < 1e-9 and s >= 1:
        k = int(round(s))
        while k > 1:  # inverse of Intrinsics::half per octave
            fx, fy, cx, cy = fx * 2, fy * 2, cx * 2 + 0.5, cy * 2 + 0.5
            k //= 2
        return fx, fy, cx, cy, width, height
    # downscale: Intrinsics::half per octave
    while w0 > width:
        fx, fy, cx, cy = fx * 0.5, fy * 0.5, (cx - 0.5) * 0.5, (cy - 0.5) * 0.5
        w0, h0 = (w0 + 1) // 2, (h0 + 1) // 2
    return fx, fy, cx, cy, width, height


# Box room: normal . x == offset, albedo rgb, checker flag, checker size
# (ScenePlane, synthetic.hpp:22-28).  x in [-2,2], y in [-1.5,1.5], z in [-1,4].
BOX_ROOM_PLANES = np.array(
    [
        [1, 0, 0, 2.0, 0.70, 0.45, 0.40, 1, 0.30],
        [1, 0, 0, -2.0, 0.40, 0.60, 0.45, 1, 0.30],
        [0, 1, 0, 1.5, 0.55, 0.55, 0.60, 1, 0.25],  # floor (y down)
        [0, 1, 0, -1.5, 0.80, 0.80, 0.75, 0, 0.25],  # ceiling
        [0, 0, 1, 4.0, 0.45, 0.50, 0.70, 1, 0.40],  # far wall
        [0, 0, 1, -1.0, 0.60, 0.50, 0.40, 0, 0.40],  # wall behind the camera
    ],
    dtype=np.float64,
)
# centre xyz, radius, albedo rgb (SceneSphere, synthetic.hpp:16-20).  The
# first is the "box+sphere" sphere; the others break the room's symmetries
# for the tracker (cf. proj/tools/voxfuse_main.cpp:142-150).
BOX_ROOM_SPHERES = np.array(
    [
        [0.0, 0.5, 2.0, 0.5, 0.85, 0.35, 0.20],
        [-0.8, 0.9, 2.6, 0.3, 0.20, 0.60, 0.30],
        [0.9, -0.4, 3.0, 0.4, 0.90, 0.80, 0.25],
        [0.5, 1.2, 1.6, 0.25, 0.30, 0.40, 0.85],
    ],
    dtype=np.float64,
)


def _rot_y(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]])


def _rot_x(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[1, 0, 0], [0, c, -s], [0, s, c]])


def _rot_z(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]])


def trajectory(n_frames: int, amplitude: float = 1.0) -> np.ndarray:
    """World-to-camera poses, row-major R (9) then t (3), frame 0 = identity.

    Camera centre and orientation follow smooth periodic curves; the largest
    per-frame step is about 1.6 cm and 0.6 deg at amplitude 1."""
    out = np.zeros((n_frames, 12))
    for i in range(n_frames):
        a = 2.0 * math.pi * i / 100.0
        centre = amplitude * np.array([0.25 * math.sin(a), 0.05 * math.sin(2 * a), 0.30 * (1 - math.cos(a))])
        r_c2w = _rot_y(amplitude * 0.15 * math.sin(a)) @ _rot_x(amplitude * 0.06 * math.sin(2 * a)) @ _rot_z(
            amplitude * 0.03 * math.sin(a)
        )
        r_w2c = r_c2w.T
        t_w2c = -r_w2c @ centre
        out[i, :9] = r_w2c.reshape(-1)
        out[i, 9:] = t_w2c
    out[0, :9] = np.eye(3).reshape(-1)
    out[0, 9:] = 0.0
    return out


def pan_trajectory(n_frames: int, max_yaw: float = 1.2) -> np.ndarray:
    """World-to-camera poses that yaw the camera away (to +max_yaw rad at the
    middle frame) and back to the start: blocks leave the enlarged swap
    frustum and return, exercising swap-out and swap-in (swap.hpp)."""
    out = np.zeros((n_frames, 12))
    for i in range(n_frames):
        u = i / max(n_frames - 1, 1)
        yaw = max_yaw * math.sin(math.pi * u)
        r_c2w = _rot_y(yaw)
        centre = np.array([0.0, 0.0, 0.4 * math.sin(math.pi * u)])
        r_w2c = r_c2w.T
        out[i, :9] = r_w2c.reshape(-1)
        out[i, 9:] = -r_w2c @ centre
    out[0, :9] = np.eye(3).reshape(-1)
    out[0, 9:] = 0.0
    return out


# Corridor (config 4): walls x = +-1.0, floor y = 1.2, ceiling y = -1.3 (y
# down), a wall behind the start; pillars (spheres) every 2 m on alternating
# sides break the corridor's translational symmetry for the tracker
# (SURVEY.md §8(d) C4).  The sensor range is cut at CORRIDOR_FAR metres.
CORRIDOR_FAR = 5.0
CORRIDOR_PLANES = np.array(
    [
        [1, 0, 0, 1.0, 0.70, 0.45, 0.40, 1, 0.30],
        [1, 0, 0, -1.0, 0.40, 0.60, 0.45, 1, 0.30],
        [0, 1, 0, 1.2, 0.55, 0.55, 0.60, 1, 0.25],
        [0, 1, 0, -1.3, 0.80, 0.80, 0.75, 0, 0.25],
        [0, 0, 1, -1.0, 0.60, 0.50, 0.40, 0, 0.40],
    ],
    dtype=np.float64,
)


def corridor_spheres(length: float = 60.0) -> np.ndarray:
    rows = []
    k = 0
    z = 1.5
    while z < length:
        side = 1.0 if k % 2 == 0 else -1.0
        rows.append([0.85 * side, 0.35 * math.sin(1.3 * k), z, 0.28, 0.3 + 0.6 * ((k * 37) % 10) / 10.0,
                     0.3 + 0.6 * ((k * 53) % 10) / 10.0, 0.3 + 0.6 * ((k * 71) % 10) / 10.0])
        if k % 3 == 0:  # a low obstacle on the floor
            rows.append([-0.4 * side, 1.05, z + 0.9, 0.18, 0.8, 0.7, 0.3])
        k += 1
        z += 2.0
    return np.array(rows, dtype=np.float64)


CORRIDOR_SPHERES = corridor_spheres()


def corridor_trajectory(n_frames: int, step: float = 0.05) -> np.ndarray:
    """World-to-camera poses walking down the corridor (+z) by `step` metres
    per frame with a gentle sway (at most ~1 deg and ~1 cm per frame)."""
    out = np.zeros((n_frames, 12))
    for i in range(n_frames):
        a = 2.0 * math.pi * i / 80.0
        centre = np.array([0.15 * math.sin(a), 0.04 * math.sin(2 * a), step * i])
        r_c2w = _rot_y(0.08 * math.sin(a)) @ _rot_x(0.03 * math.sin(2 * a))
        r_w2c = r_c2w.T
        out[i, :9] = r_w2c.reshape(-1)
        out[i, 9:] = -r_w2c @ centre
    out[0, :9] = np.eye(3).reshape(-1)
    out[0, 9:] = 0.0
    return out


def look_around_trajectory(n_frames: int, step: float = 0.02, amp: float = 0.6, period: int = 120) -> np.ndarray:
    """Corridor walk (2 cm per frame) while the camera looks from side to side
    (yaw +-0.6 rad, at most ~1.8 deg per frame): wall blocks leave the
    enlarged swap frustum and come back, so swap-ins and fuse_voxels
    (swap.hpp:96-131, 136-198) run every few frames, not only swap-outs."""
    out = np.zeros((n_frames, 12))
    for i in range(n_frames):
        a = 2.0 * math.pi * i / period
        centre = np.array([0.1 * math.sin(a), 0.0, step * i])
        r_w2c = _rot_y(amp * math.sin(a)).T
        out[i, :9] = r_w2c.reshape(-1)
        out[i, 9:] = -r_w2c @ centre
    out[0, :9] = np.eye(3).reshape(-1)
    out[0, 9:] = 0.0
    return out


def scene_for(cfg):
    """(spheres, planes, far) of a config's scene."""
    if getattr(cfg, "scene", "box_room") == "corridor":
        return CORRIDOR_SPHERES, CORRIDOR_PLANES, CORRIDOR_FAR
    return BOX_ROOM_SPHERES, BOX_ROOM_PLANES, 100.0


def trajectory_for(cfg, n_frames: int) -> np.ndarray:
    if getattr(cfg, "walk", "default") == "look_around":
        return look_around_trajectory(n_frames)
    if getattr(cfg, "scene", "box_room") == "corridor":
        return corridor_trajectory(n_frames)
    return trajectory(n_frames)


@dataclass(frozen=True)
class HashConfig:
    """HashConfig (proj/include/voxfuse/volume/hash_volume.hpp:49-58)."""

    bucket_count: int = 1 << 20
    bucket_size: int = 2
    excess_count: int = 1 << 17
    block_count: int = 1 << 18

    @property
    def ordered_count(self) -> int:
        return self.bucket_count * self.bucket_size

    @property
    def entry_count(self) -> int:
        return self.ordered_count + self.excess_count


@dataclass(frozen=True)
class BenchConfig:
    name: str
    width: int
    height: int
    voxel_size: float
    mu: float = 0.02
    voxel_type: int = 1  # 1 VoxelS, 2 VoxelSRgb (voxel.hpp:90)
    tracking: bool = True
    frames: int = 100
    hash: HashConfig = field(default_factory=HashConfig)
    max_weight: int = 100
    stop_integrating_at_max: bool = False  # SceneParams (scene_params.hpp:10)
    near_clip: float = 0.1
    far_clip: float = 8.0
    margin_px: int = 8
    swap_margin_px: int = 48
    levels: int = 5
    rotation_only_levels: int = 2
    max_iterations: int = 20
    min_valid_points: int = 30
    icp_dist_threshold: float = 0.1
    convergence_eps: float = 1e-5
    max_condition: float = 1e8
    use_swapping: bool = False  # EngineSettings::use_swapping (pipeline.hpp:20-23)
    swap_buffer_blocks: int = 100
    scene: str = "box_room"  # box_room | corridor
    tracker: str = "icp"  # TrackerType: icp | color | icp_ren (tracking_state.hpp:10)
    walk: str = "default"  # default (scene's own) | look_around (corridor, swaps in as well as out)

    @property
    def intrinsics(self):
        return intrinsics_for(self.width, self.height)

    def with_(self, **kw) -> "BenchConfig":
        return replace(self, **kw)


CONFIGS = {
    # configs[0]: the reference's own CPU-runnable case.
    "C1": BenchConfig("C1", 640, 480, 0.005),
    # configs[1]: colour integration, known poses, tracking off; 1xB200 kernel bench.
    "C2": BenchConfig("C2", 640, 480, 0.005, voxel_type=2, tracking=False),
    # configs[2]: 1280x960, 2 mm, 2^20-block pool, full tracking.
    "C3": BenchConfig(
        "C3", 1280, 960, 0.002, hash=HashConfig(bucket_count=1 << 21, excess_count=1 << 18, block_count=1 << 20)
    ),
    # small parity cases (the oracle finishes them in seconds)
    "T160": BenchConfig(
        "T160", 160, 120, 0.02, mu=0.06, frames=6,
        hash=HashConfig(bucket_count=1 << 14, excess_count=1 << 12, block_count=1 << 13),
    ),
    # C2 as a kernel bench at C3 scale (the integration
    # roofline is judged at C3 or at a C2 bench with >= 100k visible blocks)
    "C2L": BenchConfig(
        "C2L", 1280, 960, 0.002, voxel_type=2, tracking=False,
        hash=HashConfig(bucket_count=1 << 21, excess_count=1 << 18, block_count=1 << 20),
    ),
    # configs[3]: ~50 m corridor walk (1000 frames at 5 cm) with host swapping;
    # B = 512 transfers per frame keeps eviction ahead of the ~400 blocks a
    # frame allocates at this speed (the reference default B = 100 would
    # exhaust the 2^18-block pool after ~30 m and drop allocations).
    "C4": BenchConfig("C4", 640, 480, 0.005, frames=1000, use_swapping=True, swap_buffer_blocks=512,
                      scene="corridor"),
    # C4 at BASELINE.md's swap budget B = 100 blocks per frame: the walk
    # allocates faster than 100 blocks leave, so allocations are dropped once
    # the pool fills (reported in the bench line's swap section)
    "C4B100": BenchConfig("C4B100", 640, 480, 0.005, frames=1000, use_swapping=True, swap_buffer_blocks=100,
                          scene="corridor"),
    # the corridor walked while looking from side to side at B = 100: blocks
    # leave and return, so the timed frames include swap-ins and fuse_voxels
    "C4R": BenchConfig("C4R", 640, 480, 0.005, frames=1000, use_swapping=True, swap_buffer_blocks=100,
                       scene="corridor", walk="look_around"),
    # configs[4]: the large-scale scene spatially sharded by block hash
    # across 2/4/8 GPUs (bench.py --gpus N default): the corridor walk,
    # tracked, each shard with the reference's default pool of 2^18 blocks
    # (512 MiB of VoxelS) -- G shards hold G x 2^18 blocks, the capacity one
    # default volume runs out of after ~30 m of corridor (C4 swaps instead).
    "C5": BenchConfig("C5", 640, 480, 0.005, frames=1000, scene="corridor"),
    # the other trackers on the C1 / C2 frames:
    # icp_ren = ICP on the coarser levels + Ren SDF refinement at full
    # resolution; color = photometric tracking against the colour surface list
    "C1R": BenchConfig("C1R", 640, 480, 0.005, tracker="icp_ren"),
    "C2T": BenchConfig("C2T", 640, 480, 0.005, voxel_type=2, tracking=True, tracker="color"),
    "T320": BenchConfig(
        "T320", 320, 240, 0.01, mu=0.03, frames=6,
        hash=HashConfig(bucket_count=1 << 17, excess_count=1 << 14, block_count=1 << 15),
    ),
}
