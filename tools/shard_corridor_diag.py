"""Diagnostic: sharded corridor vs the single volume, with / without swapping, known / tracked poses."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
from dataclasses import replace
import numpy as np
import vf_py
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import CONFIGS, corridor_trajectory, scene_for
from paper_1410_0925_b200.sharding import LocalShardGroup

olib = vf_py.oracle_lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for swap in (False, True):
    for track in (False, True):
        cfg = CONFIGS["C4"].with_(use_swapping=swap, tracking=track)
        spheres, planes, far = scene_for(cfg)
        s, c = settings_from_config(cfg)
        s = replace(s, swap_host_blocks=1 << 17)
        ref = make_pipeline(s, c)
        grp = LocalShardGroup(s, c, 4, shift=3)
        poses = corridor_trajectory(n)
        for i, pose in enumerate(poses):
            d = vf_py.render_depth(olib, cfg, pose, spheres, planes, 0.05, far)
            if not track:
                ref.set_pose(pose); grp.set_pose(pose)
            ref.process_frame(None, d)
            grp.process_frame(None, d)
            if i in (0, 1, 5, n - 1):
                pr, nr = ref.tracking_state(); pg, ng = grp.shards[0].tracking_state()
                hr, hg = pr[..., 3] > 0, pg[..., 3] > 0
                both = hr & hg
                dp = np.linalg.norm(pr[..., :3] - pg[..., :3], axis=-1)[both]
                ang = np.degrees(np.arccos(np.clip((nr[..., :3] * ng[..., :3]).sum(-1)[both], -1, 1)))
                print(f"swap={swap} track={track} frame {i}: hits ref {hr.mean():.3f} shard {hg.mean():.3f} agree {np.mean(hr == hg):.4f} pts {np.mean(dp <= 0.0025):.4f} nrm {np.mean(ang <= 1):.4f}")
        grp.close(); ref.close()
