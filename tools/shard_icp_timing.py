#!/usr/bin/env python
"""Virtual shards on ONE device (the only multi-shard setup this sandbox can
run): per-frame wall time and ICP iterations of a G-shard group with
replicated ICP vs pixel-sharded ICP (per-iteration sums through peer
memory).  Both groups run G full pipelines on the same GPU, so this measures
the exchange's overhead and correctness at speed, not multi-GPU scaling."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

import vf_py  # noqa: E402
from helpers import frames  # noqa: E402
from paper_1410_0925_b200 import settings_from_config  # noqa: E402
from paper_1410_0925_b200.scene import CONFIGS  # noqa: E402
from paper_1410_0925_b200.sharding import LocalShardGroup  # noqa: E402

olib = vf_py.oracle_lib()
cfg = CONFIGS["C1"]
fr = frames(olib, cfg, 40)
s, c = settings_from_config(cfg)
for G in (2, 4):
    for icp in (False, True):
        grp = LocalShardGroup(s, c, G, shift=3, shard_icp=icp)
        ms, its = [], []
        for i, (_, d, _) in enumerate(fr):
            for sh in grp.shards:
                sh.synchronize()
            t0 = time.perf_counter()
            st = grp.process_frame(None, d)
            ms.append((time.perf_counter() - t0) * 1e3)
            its.append(st[0].tracking_iterations)
        grp.close()
        print(f"G={G} {'pixel-sharded ICP' if icp else 'replicated ICP   '}: {np.median(ms[5:]):.3f} ms/frame "
              f"(median over frames 5..39, all shards + composite), ICP iterations {np.mean(its[1:]):.1f}")
