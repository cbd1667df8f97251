"""Generate tests/golden/golden_ref.json from the REFERENCE itself.

Runs the reference's own sources (compiled unmodified against the Eigen shim
into oracle/_ref/libvoxfuse_ref.so, one worker thread for the deterministic
allocation winner) on the synthetic scenes and records digests of everything
the oracle and the GPU path must reproduce.  Needs /root/reference at build
time (this container); the JSON it writes is committed.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))

import vf_py  # noqa: E402
from helpers import SWAP_CASES, swap_config  # noqa: E402
from paper_1410_0925_b200.scene import BOX_ROOM_PLANES, BOX_ROOM_SPHERES, CONFIGS, trajectory  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def entries_digest(e: np.ndarray) -> str:
    e = e.copy()
    e["pad"] = 0
    return sha(e)


def voxels_digest(v: np.ndarray, vsize: int) -> str:
    return sha(v.reshape(-1, vsize)[:, : vsize - 1])


def run(lib, cfg, n, tracking, rgb=False, epilogues=True):
    from paper_1410_0925_b200.scene import scene_for, trajectory_for
    spheres, planes, far = scene_for(cfg)
    poses = trajectory_for(cfg, n)
    vol = vf_py.Volume(lib, cfg, tracking)
    vsize = 8 if cfg.voxel_type == 2 else 4
    out = []
    for i in range(n):
        d = vf_py.render_depth(lib, cfg, poses[i], spheres, planes, 0.05, far)
        c = vf_py.render_rgb(lib, cfg, poses[i], spheres, planes, 0.05, far) if rgb else None
        st = vol.process(d, c, None if tracking else poses[i])
        pts, nrm = vol.maps()
        out.append({
            "frame": i,
            "depth_sha": sha(d),
            "rgb_sha": sha(c) if rgb else None,
            "tracking_ok": int(st.tracking_ok),
            "tracking_iterations": int(st.tracking_iterations),
            "blocks_allocated": int(st.blocks_allocated),
            "visible_blocks": int(st.visible_blocks),
            "allocated_total": int(vol.allocated_blocks()),
            "pose": [float(x) for x in vol.pose()],
            "entries_sha": entries_digest(vol.entries()),
            "voxels_sha": voxels_digest(vol.voxels(), vsize),
            "points_sha": sha(pts),
            "normals_sha": sha(nrm),
            "visible_sha": sha(np.sort(vol.visible_list())),
            "volume_digest": str(vol.digest()) if tracking else None,
            "ranges_sha": sha(vol.ranges()) if not tracking else None,
        })
        if cfg.use_swapping:
            out[-1].update({"swapped_in": int(st.swapped_in), "swapped_out": int(st.swapped_out),
                            "states_sha": sha(vol.swap_states()), "store_count": int(vol.store_count())})
        if not epilogues:
            continue
        # raycast epilogues (raycast.hpp:441-509, pipeline_impl.hpp:125-137, 218-221)
        sp, sc = vol.surface_points()
        out[-1]["surface_count"] = int(len(sp))
        out[-1]["surface_points_sha"] = sha(sp)
        out[-1]["surface_colors_sha"] = sha(sc)
        out[-1]["image_sha"] = sha(vol.image(0))
        out[-1]["image_grey_sha"] = sha(vol.image(3))
        if tracking:
            out[-1]["image_depth_sha"] = sha(vol.image(1))
    vol.close()
    return out


def store_digest(vol) -> str:
    """sha over (entry index, payload) of every stored block, ascending."""
    h = hashlib.sha256()
    for k, v in sorted(vol.store().items()):
        h.update(np.int32(k).tobytes())
        h.update(v.tobytes())
    return h.hexdigest()


def run_swap(lib, name, n=24):
    from paper_1410_0925_b200.scene import pan_trajectory
    cfg = swap_config(name)
    poses = pan_trajectory(n)
    vol = vf_py.Volume(lib, cfg, False)
    out = []
    for i in range(n):
        d = vf_py.render_depth(lib, cfg, poses[i], BOX_ROOM_SPHERES, BOX_ROOM_PLANES)
        st = vol.process(d, None, poses[i])
        pts, nrm = vol.maps()
        out.append({
            "frame": i, "depth_sha": sha(d),
            "blocks_allocated": int(st.blocks_allocated), "allocation_dropped": int(st.allocation_dropped),
            "visible_blocks": int(st.visible_blocks), "allocated_total": int(vol.allocated_blocks()),
            "swapped_in": int(st.swapped_in), "swapped_out": int(st.swapped_out),
            "bytes_in": int(st.bytes_in), "bytes_out": int(st.bytes_out),
            "entries_sha": entries_digest(vol.entries()), "voxels_sha": voxels_digest(vol.voxels(), 4),
            "states_sha": sha(vol.swap_states()), "store_count": int(vol.store_count()),
            "store_sha": store_digest(vol), "points_sha": sha(pts), "normals_sha": sha(nrm),
        })
    vol.close()
    return out


def main():
    lib = vf_py.ref_lib()
    lib.lib.vfr_set_threads(1)
    gold = {
        "generator": "tests/golden/make_golden.py (reference sources via oracle/_ref, 1 worker)",
        "known_answers": {
            # hash_volume.hpp:32-37 evaluated by hand (SPEC.md:171's 471389 is wrong)
            "hash_block_pos_mask_0xFFFFF": {"1,0,0": 455773, "1,1,1": 543567, "-1,0,0": 592803},
            # voxel.hpp:16-19 truncates toward zero
            "sdf_float_to_value": {"1.0": 32767, "0.5": 16383, "-1.0": -32767, "2.0": 32767},
        },
        "T160_tracking": run(lib, CONFIGS["T160"], 4, tracking=True),
        "T320_known_pose": run(lib, CONFIGS["T320"].with_(tracking=False), 3, tracking=False),
        "C2_known_pose_rgb": run(lib, CONFIGS["C2"], 2, tracking=False, rgb=True),
    }
    # the large configurations (BASELINE configs[2], configs[3]): C3 frame 0
    # (1280x960, 2 mm, 2^20 blocks) and the first tracked corridor frames of
    # C4 with host swapping
    gold["C3_tracking"] = run(lib, CONFIGS["C3"], 1, tracking=True, epilogues=False)
    gold["C4_corridor_tracking"] = run(lib, CONFIGS["C4"], 3, tracking=True, epilogues=False)
    for name in SWAP_CASES:
        gold[name] = run_swap(lib, name)
    cfg = CONFIGS["C1"]
    d = vf_py.render_depth(lib, cfg, trajectory(5)[3], BOX_ROOM_SPHERES, BOX_ROOM_PLANES)
    d[100:140, 200:260] = 0.0
    gold["C1_pyramid"] = {"depth_sha": sha(d), "levels_sha": [sha(l) for l in vf_py.depth_pyramid(lib, d, 5)]}
    out = ROOT / "tests" / "golden" / "golden_ref.json"
    out.write_text(json.dumps(gold, indent=1))
    print(f"wrote {out} ({out.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
