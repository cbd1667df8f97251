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


def _composite_worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch.distributed as dist

    from paper_1410_0925_b200.sharding import composite

    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(100 + rank)
    h, w = 24, 32
    pts = np.zeros((h, w, 4), np.float32)
    nrm = np.zeros((h, w, 4), np.float32)
    hit = rng.random((h, w)) < 0.7
    z = rng.uniform(0.5, 4.0, (h, w)).astype(np.float32)
    pts[..., 0] = rng.normal(size=(h, w))
    pts[..., 1] = rng.normal(size=(h, w))
    pts[..., 2] = z            # identity pose: camera z == world z
    pts[..., 3] = hit
    nrm[..., :3] = rng.normal(size=(h, w, 3))
    nrm[..., 3] = hit
    pts[~hit] = 0
    nrm[~hit] = 0
    ident = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0], float)
    out_p, out_n = composite(pts, nrm, ident, rank, dist)
    dist.destroy_process_group()
    q.put((rank, pts, nrm, out_p, out_n))


def test_nearest_depth_composite_world2():
    """The per-frame exchange of the sharded pipeline over a real process
    group (gloo, 2 ranks): every rank ends with the map of the nearest hit."""
    import numpy as np

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_composite_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    (_, p0, n0, o0p, o0n), (_, p1, n1, o1p, o1n) = res
    assert np.array_equal(o0p, o1p) and np.array_equal(o0n, o1n)
    z0 = np.where(p0[..., 3] > 0, p0[..., 2], np.inf)
    z1 = np.where(p1[..., 3] > 0, p1[..., 2], np.inf)
    take1 = z1 < z0
    want_p = np.where(take1[..., None], p1, p0)
    want_n = np.where(take1[..., None], n1, n0)
    none = ~np.isfinite(np.minimum(z0, z1))
    want_p[none] = 0
    want_n[none] = 0
    assert np.array_equal(o0p, want_p) and np.array_equal(o0n, want_n)


def _nccl_id_worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from paper_1410_0925_b200.sharding import share_nccl_id

    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = share_nccl_id(rank, dist)
    dist.destroy_process_group()
    q.put((rank, uid))


def test_product_nccl_id_shared_world2():
    """The product's communicator bootstrap (sharding.attach_nccl up to the
    device attach): rank 0's ncclGetUniqueId, through the library, reaches
    every rank of a real 2-process group byte for byte."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    assert res[0][1] == res[1][1] and len(res[0][1]) == 128 and any(res[0][1])
