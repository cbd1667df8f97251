"""CPU suite, world_size 2 over gloo: the bench's one-process-per-GPU
plumbing (barrier, max-over-ranks timing, whole-job sums)."""
import os
import socket
import sys
from pathlib import Path

import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import bench

    d = bench.Dist(world)
    d.barrier()
    t = d.max(1.0 + rank)          # slowest rank's time
    frames = d.sum(10.0 * (rank + 1))  # frames processed by all ranks
    d.close()
    q.put((rank, t, frames))


def test_dist_max_and_sum_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == [2.0, 2.0]
    assert [r[2] for r in res] == [30.0, 30.0]
