import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import numpy as np
import vf_py
from helpers import frames
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.sharding import shard_owner
from paper_1410_0925_b200.scene import CONFIGS
from dataclasses import replace
cfg = CONFIGS["C1"].with_(tracking=False)
olib = vf_py.oracle_lib()
s, c = settings_from_config(cfg)
ref = make_pipeline(s, c)
G, shift = 2, 2
sh = [make_pipeline(replace(s, shard_count=G, shard_index=i, shard_shift=shift), c) for i in range(G)]
(pose, d, _), = frames(olib, cfg, 1)
ref.set_pose(pose); ref.process_frame(None, d)
for p in sh: p.set_pose(pose); p.process_frame(None, d)
pr, _ = ref.tracking_state()
hit = pr[..., 3] > 0
vb = np.floor(pr[..., :3] / cfg.voxel_size).astype(np.int64) >> 3
own = shard_owner(vb[..., 0], vb[..., 1], vb[..., 2], shift, G)
for i, p in enumerate(sh):
    ps, _ = p.tracking_state()
    hs = ps[..., 3] > 0
    mine = hit & (own == i)
    print(f"shard {i}: ref-hits owned {mine.sum()}, of those shard hit {np.sum(hs & mine)}; shard hits total {hs.sum()}; ranges valid {np.mean(p.ranges()[:,0] <= p.ranges()[:,1]):.3f}")
    print("   visible", len(p.visible_list()), "ref visible", len(ref.visible_list()))
print("ref ranges valid", np.mean(ref.ranges()[:,0] <= ref.ranges()[:,1]))
# where do shard rays fail?
p = sh[0]
ps, _ = p.tracking_state()
hs = ps[..., 3] > 0
mine = hit & (own == 0)
miss = mine & ~hs
rs = p.ranges().reshape(30, 40, 2); rr = ref.ranges().reshape(30, 40, 2)
ys, xs = np.nonzero(miss)
w2c = pose
R = np.array(w2c[:9]).reshape(3, 3); t = np.array(w2c[9:])
zhit = (pr[ys, xs, :3] @ R.T + t)[:, 2]
fr_s = rs[ys // 16, xs // 16]; fr_r = rr[ys // 16, xs // 16]
print("missed", len(ys), "shard range start - hit depth: p5/p50/p95", np.percentile(fr_s[:, 0] - zhit, [5, 50, 95]))
print("ref   range start - hit depth: p5/p50/p95", np.percentile(fr_r[:, 0] - zhit, [5, 50, 95]))
print("shard range end - hit depth p5/p50", np.percentile(fr_s[:, 1] - zhit, [5, 50]))
ys2, xs2 = np.nonzero(mine & hs)
z2 = (pr[ys2, xs2, :3] @ R.T + t)[:, 2]
print("hit ok: shard range start - hit depth p5/p50/p95", np.percentile(rs[ys2 // 16, xs2 // 16][:, 0] - z2, [5, 50, 95]))
