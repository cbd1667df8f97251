"""Sharded (G virtual shards on one GPU) vs unsharded: allocation, voxels, maps, poses."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import numpy as np
import vf_py
from helpers import frames, allocated_blocks, rot_angle, centre_dist
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.sharding import LocalShardGroup
from paper_1410_0925_b200.scene import CONFIGS
name, G, shift, tracking, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4] == '1', int(sys.argv[5])
cfg = CONFIGS[name].with_(tracking=tracking)
olib = vf_py.oracle_lib()
s, c = settings_from_config(cfg)
ref = make_pipeline(s, c)
grp = LocalShardGroup(s, c, G, shift)
for i, (pose, d, _) in enumerate(frames(olib, cfg, n)):
    if not tracking:
        ref.set_pose(pose); grp.set_pose(pose)
    ref.process_frame(None, d); st = grp.process_frame(None, d)
    pr = ref.pose(); ps = [g.pose() for g in grp.shards]
    same = all(np.array_equal(ps[0], p) for p in ps)
    print(f"f{i} shards_pose_identical={same} rot={rot_angle(pr, ps[0]):.2e} dist={centre_dist(pr, ps[0]):.2e} vis={[x.visible_blocks for x in st]}")
br = allocated_blocks(ref.entries(), ref.voxels(), 4)
bs = {}
for g in grp.shards:
    bs.update(allocated_blocks(g.entries(), g.voxels(), 4))
common = set(br) & set(bs)
print("blocks ref", len(br), "union shards", len(bs), "common", len(common), "only_ref", len(set(br) - set(bs)), "only_shards", len(set(bs) - set(br)))
eq = np.mean([np.array_equal(br[k], bs[k]) for k in common])
print("common blocks with identical voxels:", eq)
pr_, nr_ = ref.tracking_state()
pg, ng = grp.shards[0].tracking_state()
for g in grp.shards[1:]:
    p2, n2 = g.tracking_state()
    assert np.array_equal(p2.view(np.uint32), pg.view(np.uint32))
hr, hg = pr_[..., 3] > 0, pg[..., 3] > 0
both = hr & hg
dp = np.linalg.norm(pr_[..., :3] - pg[..., :3], axis=-1)[both]
cosang = np.clip((nr_[..., :3] * ng[..., :3]).sum(-1)[both], -1, 1)
ang = np.degrees(np.arccos(cosang))
print(f"hit agreement {np.mean(hr == hg):.5f} (ref hits {hr.mean():.4f}, shard hits {hg.mean():.4f}); point dmm p50 {np.median(dp)*1000:.4f} p99 {np.quantile(dp,0.99)*1000:.3f} frac<=0.5vox {np.mean(dp <= 0.5*cfg.voxel_size):.5f}; normal deg p99 {np.quantile(ang,0.99):.3f} frac<=1deg {np.mean(ang<=1):.5f}; exact {np.mean(dp==0):.4f}")
