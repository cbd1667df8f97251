"""Spatial sharding of the volume across GPUs (BASELINE config 5).

Host-side mirror of the device rules in csrc/vf_shard.cu plus the drivers:

* ``shard_owner`` — block -> shard: hash of the super-block (2^s blocks per
  axis) mod G (same arithmetic as ``vf_shard_owner``);
* ``composite_keys`` / ``composite`` — the per-frame nearest-depth exchange,
  written against ``torch.distributed`` so the protocol is testable on CPU
  with gloo (tests/test_multi_rank.py); on GPUs the same exchange runs as
  NCCL collectives inside the frame graph (``vf_shard_attach_nccl``);
* ``LocalShardGroup`` — G shards in one process on one device (tests,
  single-GPU boxes), composited by ``vf_shard_composite_local``;
* ``attach_nccl`` — one process per GPU: NCCL unique id from rank 0 over the
  host process group, then every rank's context attaches.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from .pipeline import Pipeline, make_pipeline

NO_HIT = np.uint64(0xFFFFFFFFFFFFFFFF)


def shard_owner(bx, by, bz, shift: int, count: int):
    """Owner shard of block positions (numpy arrays or ints)."""
    if count <= 1:
        return np.zeros(np.broadcast(bx, by, bz).shape, np.int64) if np.ndim(bx) else 0
    sx = (np.asarray(bx, np.int64) >> shift).astype(np.uint32)
    sy = (np.asarray(by, np.int64) >> shift).astype(np.uint32)
    sz = (np.asarray(bz, np.int64) >> shift).astype(np.uint32)
    with np.errstate(over="ignore"):
        h = (sx * np.uint32(73856093)) ^ (sy * np.uint32(19349669)) ^ (sz * np.uint32(83492791))
    return (h % np.uint32(count)).astype(np.int64)


def composite_keys(points: np.ndarray, w2c: np.ndarray, rank: int) -> np.ndarray:
    """Per-pixel key float_bits(camera z of the hit) << 32 | rank, NO_HIT
    where the shard has no hit (k_shard_keys)."""
    p = points.reshape(-1, 4).astype(np.float64)
    r = np.asarray(w2c, np.float64)
    z = r[6] * p[:, 0] + r[7] * p[:, 1] + r[8] * p[:, 2] + r[11]
    zf = np.where(z > 0, z, 0).astype(np.float32)
    keys = (zf.view(np.uint32).astype(np.uint64) << np.uint64(32)) | np.uint64(rank)
    return np.where(points.reshape(-1, 4)[:, 3] != 0, keys, NO_HIT)


def composite(points: np.ndarray, normals: np.ndarray, w2c: np.ndarray, rank: int, dist) -> tuple:
    """The exchange over a torch.distributed process group: all_reduce(MIN)
    of the keys, mask to the winner, all_reduce(SUM) of the maps.  Exact:
    every pixel sums one non-zero contribution with zeros."""
    import torch

    keys = composite_keys(points, w2c, rank)
    kt = torch.from_numpy(keys.view(np.int64).copy())
    # uint64 keys compare like int64 once the sign bit is flipped
    kt ^= torch.tensor(np.int64(-(2 ** 63)))
    dist.all_reduce(kt, op=dist.ReduceOp.MIN)
    kt ^= torch.tensor(np.int64(-(2 ** 63)))
    kmin = kt.numpy().view(np.uint64)
    won = (kmin != NO_HIT) & ((kmin & np.uint64(0xFFFFFFFF)) == np.uint64(rank))
    p = np.where(won[:, None], points.reshape(-1, 4), 0).astype(np.float32)
    n = np.where(won[:, None], normals.reshape(-1, 4), 0).astype(np.float32)
    pt, nt = torch.from_numpy(p), torch.from_numpy(n)
    dist.all_reduce(pt, op=dist.ReduceOp.SUM)
    dist.all_reduce(nt, op=dist.ReduceOp.SUM)
    return pt.numpy().reshape(points.shape), nt.numpy().reshape(normals.shape)


class LocalShardGroup:
    """G shards of one volume in this process on one device.

    shard_icp=True: pixel-sharded ICP, the shards' per-iteration sums
    exchanged inside the ICP kernels (vf_shard_icp_link_local); the shards'
    frames are then submitted together so their ICP loops run concurrently,
    each capped to 128 / G CTAs so they are co-resident on the device."""

    def __init__(self, settings, calib, count: int, shift: int = 3, device: int = 0, halo: bool = True,
                 shard_icp: bool = False, transport: str = "local"):
        from dataclasses import replace

        if transport not in ("local", "p2p"):
            raise ValueError("transport: 'local' (one composite kernel over all shards) or 'p2p' (per-shard "
                             "composite over peer memory, inside each shard's frame)")
        extra = {"shard_icp": True, "icp_max_ctas": max(8, 128 // count)} if shard_icp else {}
        self.shards = [make_pipeline(replace(settings, shard_count=count, shard_index=i, shard_shift=shift,
                                             shard_halo=halo, **extra), calib, device) for i in range(count)]
        self._handles = (C.c_void_p * count)(*[s.handle.value for s in self.shards])
        self.shard_icp = shard_icp
        self.transport = transport
        L = _abi.load()
        if shard_icp:
            _abi.check("vf_shard_icp_link_local", L.vf_shard_icp_link_local(self._handles, count))
        if transport == "p2p":
            _abi.check("vf_shard_p2p_link_local", L.vf_shard_p2p_link_local(self._handles, count))

    def set_pose(self, pose):
        for s in self.shards:
            s.set_pose(pose)

    def process_frame(self, rgb, depth_m):
        if self.shard_icp or self.transport == "p2p":
            # all shards in flight at once: their exchanges wait for each other
            for s in self.shards:
                s.submit_frame(rgb, depth_m)
            stats = [s.collect_frame() for s in self.shards]
        else:
            stats = [s.process_frame(rgb, depth_m) for s in self.shards]
        if self.transport == "local":
            _abi.check("vf_shard_composite_local",
                       _abi.load().vf_shard_composite_local(self._handles, len(self.shards)))
        return stats

    def close(self):
        for s in self.shards:
            s.close()


def _load_torch_nccl() -> None:
    """The library dlopens libnccl.so.2 on first use and reuses one already
    loaded.  In a Python process that is PyTorch's (its own, newer build):
    import torch first, or the system library the C side would otherwise load
    shadows it and a later `import torch` fails on missing NCCL symbols."""
    import torch  # noqa: F401  (loads libtorch_cuda and its libnccl.so.2)


def share_nccl_id(rank: int, dist) -> bytes:
    """Rank 0 creates the NCCL unique id (vf_shard_nccl_unique_id, no GPU
    needed) and every rank receives it over the host process group."""
    _load_torch_nccl()
    L = _abi.load()
    buf = (C.c_uint8 * 128)()
    if rank == 0:
        _abi.check("vf_shard_nccl_unique_id", L.vf_shard_nccl_unique_id(buf))
    obj = [bytes(buf)]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def attach_nccl(pipe: Pipeline, rank: int, world: int, dist) -> None:
    """One process per GPU: share rank 0's NCCL id over `dist` and attach."""
    idb = (C.c_uint8 * 128).from_buffer_copy(share_nccl_id(rank, dist))
    _abi.check("vf_shard_attach_nccl", _abi.load().vf_shard_attach_nccl(pipe.handle, idb, world, rank))


def attach_icp_peers(pipe: Pipeline, rank: int, world: int, dist) -> None:
    """One process per GPU, pixel-sharded ICP: gather every rank's CUDA IPC
    handle of its exchange area in rank order and link (vf_shard_icp_link)."""
    L = _abi.load()
    own = (C.c_uint8 * 64)()
    _abi.check("vf_shard_icp_handle", L.vf_shard_icp_handle(pipe.handle, own))
    allh = [None] * world
    dist.all_gather_object(allh, bytes(own))
    buf = (C.c_uint8 * (64 * world)).from_buffer_copy(b"".join(allh))
    _abi.check("vf_shard_icp_link", L.vf_shard_icp_link(pipe.handle, buf, world))


def attach_p2p(pipe: Pipeline, rank: int, world: int, dist) -> None:
    """One process per GPU, the composite over peer memory: gather every
    rank's four CUDA IPC handles (keys, points, normals, flags) in rank order
    and link (vf_shard_p2p_link)."""
    L = _abi.load()
    own = (C.c_uint8 * 256)()
    _abi.check("vf_shard_p2p_handles", L.vf_shard_p2p_handles(pipe.handle, own))
    allh = [None] * world
    dist.all_gather_object(allh, bytes(own))
    buf = (C.c_uint8 * (256 * world)).from_buffer_copy(b"".join(allh))
    _abi.check("vf_shard_p2p_link", L.vf_shard_p2p_link(pipe.handle, buf, world))
