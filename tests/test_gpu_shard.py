"""GPU: spatial sharding (config 5) with G shards of one volume on one device
(vf_shard_composite_local), against the unsharded pipeline.  The cross-GPU
transport (NCCL) carries the identical exchange; its protocol is tested over
gloo in tests/test_multi_rank.py and its plumbing with one rank below."""
import ctypes as C

import numpy as np
import pytest

import vf_py
from helpers import allocated_blocks, centre_dist, frames, rot_angle
from paper_1410_0925_b200 import _abi, make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import CONFIGS
from paper_1410_0925_b200.sharding import LocalShardGroup, shard_owner

pytestmark = pytest.mark.gpu


def _maps_agreement(ref, shard, vs):
    pr, nr = ref.tracking_state()
    pg, ng = shard.tracking_state()
    hr, hg = pr[..., 3] > 0, pg[..., 3] > 0
    both = hr & hg
    dp = np.linalg.norm(pr[..., :3] - pg[..., :3], axis=-1)[both]
    ang = np.degrees(np.arccos(np.clip((nr[..., :3] * ng[..., :3]).sum(-1)[both], -1, 1)))
    return np.mean(hr == hg), np.mean(dp <= 0.5 * vs), np.mean(ang <= 1.0)


@pytest.mark.parametrize("G", [2, 4])
def test_sharded_known_pose_matches_unsharded(olib, G):
    cfg = CONFIGS["C1"].with_(tracking=False)
    s, c = settings_from_config(cfg)
    ref = make_pipeline(s, c)
    grp = LocalShardGroup(s, c, G, shift=3)
    for pose, d, _ in frames(olib, cfg, 3):
        ref.set_pose(pose)
        grp.set_pose(pose)
        ref.process_frame(None, d)
        grp.process_frame(None, d)
    # every shard holds the identical composited maps
    p0, n0 = grp.shards[0].tracking_state()
    for g in grp.shards[1:]:
        p1, n1 = g.tracking_state()
        assert np.array_equal(p0.view(np.uint32), p1.view(np.uint32))
        assert np.array_equal(n0.view(np.uint32), n1.view(np.uint32))
    # the shards together hold every block the single volume holds
    br = allocated_blocks(ref.entries(), ref.voxels(), 4)
    union = set()
    for g in grp.shards:
        union |= set(allocated_blocks(g.entries(), g.voxels(), 4))
    assert set(br) <= union
    # ownership: a shard's blocks are its own territory or within one block of it
    hit, pts, nrm = _maps_agreement(ref, grp.shards[0], cfg.voxel_size)
    assert hit >= 0.99 and pts >= 0.995 and nrm >= 0.98, (hit, pts, nrm)
    grp.close()
    ref.close()


def test_sharded_tracking_replicated_icp(olib):
    """Replicated ICP on the composited maps: every shard computes the same
    pose bit for bit; poses stay within tracking tolerance of the unsharded run."""
    cfg = CONFIGS["C1"]
    s, c = settings_from_config(cfg)
    ref = make_pipeline(s, c)
    grp = LocalShardGroup(s, c, 2, shift=3)
    for pose, d, _ in frames(olib, cfg, 6):
        sr = ref.process_frame(None, d)
        st = grp.process_frame(None, d)
        assert all(x.tracking_ok for x in st)
        ps = [g.pose() for g in grp.shards]
        assert all(np.array_equal(ps[0], p) for p in ps[1:])
        assert rot_angle(ref.pose(), ps[0]) < 1e-3 and centre_dist(ref.pose(), ps[0]) < 1e-3
    hit, pts, _ = _maps_agreement(ref, grp.shards[0], cfg.voxel_size)
    assert hit >= 0.99 and pts >= 0.99
    grp.close()
    ref.close()


@pytest.mark.parametrize("G", [2, 3])
def test_sharded_tracking_exchanged_icp(olib, G):
    """Pixel-sharded ICP: each shard sums the ICP terms of 1/G
    of the pixels and the 29 sums of every iteration are added across the
    shards inside the ICP kernels through peer memory.  Every shard ends each
    frame with the bit-identical pose; the poses agree with the replicated-ICP
    group (only the order of the FP64 sums differs) and the unsharded run
    within the tracking tolerance."""
    cfg = CONFIGS["C1"]
    s, c = settings_from_config(cfg)
    ref = make_pipeline(s, c)
    rep = LocalShardGroup(s, c, G, shift=3)
    grp = LocalShardGroup(s, c, G, shift=3, shard_icp=True)
    for pose, d, _ in frames(olib, cfg, 8):
        ref.process_frame(None, d)
        sr = rep.process_frame(None, d)
        st = grp.process_frame(None, d)
        assert all(x.tracking_ok for x in st) and all(x.error_flags == 0 for x in st)
        assert [x.tracking_iterations for x in st] == [st[0].tracking_iterations] * G
        ps = [g.pose() for g in grp.shards]
        assert all(np.array_equal(ps[0], p) for p in ps[1:]), "shards disagree on the pose"
        pr = rep.shards[0].pose()
        assert rot_angle(pr, ps[0]) < 1e-4 and centre_dist(pr, ps[0]) < 1e-4
        assert rot_angle(ref.pose(), ps[0]) < 1e-3 and centre_dist(ref.pose(), ps[0]) < 1e-3
    grp.close()
    rep.close()
    ref.close()


def test_owner_rule_matches_device():
    L = _abi.load()
    rng = np.random.default_rng(7)
    b = rng.integers(-500, 500, size=(2000, 3))
    for shift, g in [(0, 2), (3, 4), (3, 8), (2, 3)]:
        dev = [L.vf_shard_owner(int(x), int(y), int(z), shift, g) for x, y, z in b]
        assert np.array_equal(dev, shard_owner(b[:, 0], b[:, 1], b[:, 2], shift, g))


def test_nccl_composite_plumbing_single_rank(olib):
    """NCCL path with one rank: unique id, communicator, collectives captured
    in the frame graph; with one rank the composite must be the identity."""
    from paper_1410_0925_b200.sharding import _load_torch_nccl
    _load_torch_nccl()  # the NCCL the library finds loaded is then PyTorch's own
    L = _abi.load()
    cfg = CONFIGS["T320"].with_(tracking=False)
    s, c = settings_from_config(cfg)
    ref = make_pipeline(s, c)
    p = make_pipeline(s, c)
    buf = (C.c_uint8 * 128)()
    rc = L.vf_shard_nccl_unique_id(buf)
    if rc != 0:
        pytest.skip("libnccl not loadable")
    assert L.vf_shard_attach_nccl(p.handle, buf, 1, 0) == 0
    for pose, d, _ in frames(olib, cfg, 3):
        ref.set_pose(pose)
        p.set_pose(pose)
        ref.process_frame(None, d)
        p.process_frame(None, d)
    a, b = ref.tracking_state(), p.tracking_state()
    assert np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32))
    assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))


def test_sharded_corridor_with_swapping(olib):
    """Config 5 on the config-4 scene: the corridor walk sharded over 4 virtual
    shards, each with its own swap engine and host store.  Known poses: the
    composited maps match the unsharded swapping volume (swapping changes
    nothing in the agreement — tools/shard_corridor_diag.py).  Tracked: the
    replicated ICP follows the walk with every shard paging blocks out."""
    from dataclasses import replace
    from paper_1410_0925_b200.scene import corridor_trajectory, scene_for
    cfg = CONFIGS["C4"]
    spheres, planes, far = scene_for(cfg)
    poses = corridor_trajectory(40)
    depths = [vf_py.render_depth(olib, cfg, p, spheres, planes, 0.05, far) for p in poses]
    for track in (False, True):
        s, c = settings_from_config(cfg.with_(tracking=track))
        s = replace(s, swap_host_blocks=1 << 17)  # 256 MiB of pinned host store per context
        ref = make_pipeline(s, c) if not track else None
        grp = LocalShardGroup(s, c, 4, shift=3)
        outs = 0
        for i, (pose, d) in enumerate(zip(poses, depths)):
            if not track:
                ref.set_pose(pose)
                grp.set_pose(pose)
                ref.process_frame(None, d)
            sts = grp.process_frame(None, d)
            assert all(st.tracking_ok for st in sts) and all(st.allocation_dropped == 0 for st in sts), i
            outs += sum(st.swapped_out for st in sts)
        assert outs > 1000
        if track:
            p0 = grp.shards[0].pose()
            assert all(np.array_equal(g.pose(), p0) for g in grp.shards[1:])
            assert rot_angle(p0, poses[-1]) < 0.01 and centre_dist(p0, poses[-1]) < 0.02
        else:
            hit, pts, nrm = _maps_agreement(ref, grp.shards[0], cfg.voxel_size)
            assert hit >= 0.99 and pts >= 0.99 and nrm >= 0.97, (hit, pts, nrm)
            ref.close()
        grp.close()


@pytest.mark.parametrize("G", [2, 3])
def test_p2p_composite_matches_group_composite(olib, G):
    """The composite over peer memory (each shard reads the others' keys and
    winning map entries inside its own frame) gives the maps of the
    single-kernel group composite bit for bit, on every shard."""
    cfg = CONFIGS["T320"].with_(tracking=False)
    s, c = settings_from_config(cfg)
    loc = LocalShardGroup(s, c, G, shift=2)
    p2p = LocalShardGroup(s, c, G, shift=2, transport="p2p")
    for pose, d, _ in frames(olib, cfg, 4):
        loc.set_pose(pose)
        p2p.set_pose(pose)
        loc.process_frame(None, d)
        st = p2p.process_frame(None, d)
        assert all(x.error_flags == 0 for x in st)
        a = loc.shards[0].tracking_state()
        for sh in p2p.shards:
            b = sh.tracking_state()
            assert np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32))
            assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))
    loc.close()
    p2p.close()


def _mp_shard_worker(rank, world, port, frames_np, q):
    """One shard per process, both on device 0: IPC handles over gloo,
    composite and ICP sums over peer memory (the multi-GPU code path; on one
    device the two contexts time-slice, so only correctness is meaningful)."""
    import os
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import hashlib
    from dataclasses import replace

    import torch.distributed as dist

    from paper_1410_0925_b200 import make_pipeline, settings_from_config
    from paper_1410_0925_b200.scene import CONFIGS
    from paper_1410_0925_b200.sharding import attach_icp_peers, attach_p2p

    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, c = settings_from_config(CONFIGS["T320"])
    s = replace(s, shard_count=world, shard_index=rank, shard_shift=2, shard_icp=True, icp_max_ctas=64)
    p = make_pipeline(s, c, device=0)
    attach_p2p(p, rank, world, dist)
    attach_icp_peers(p, rank, world, dist)
    out = []
    for d in frames_np:
        st = p.process_frame(None, d)
        pts, nrm = p.tracking_state()
        out.append((bool(st.tracking_ok), int(st.error_flags), p.pose().tolist(),
                    hashlib.sha256(pts.tobytes() + nrm.tobytes()).hexdigest()))
    p.close()
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, out))


def test_two_processes_p2p_shards_match_in_process_group(olib):
    """The multi-process sharded pipeline -- one process per shard, CUDA IPC
    mappings exchanged over a real process group, the map composite and the
    per-iteration ICP sums over peer memory -- reproduces the in-process
    group bit for bit (poses and maps), on both ranks."""
    import hashlib
    import socket
    from dataclasses import replace

    import torch.multiprocessing as mp
    cfg = CONFIGS["T320"]
    fr = [d for _, d, _ in frames(olib, cfg, 4)]
    s, c = settings_from_config(cfg)
    grp = LocalShardGroup(s, c, 2, shift=2, shard_icp=True, transport="p2p")
    want = []
    for d in fr:
        st = grp.process_frame(None, d)
        pts, nrm = grp.shards[0].tracking_state()
        want.append((bool(st[0].tracking_ok), grp.shards[0].pose().tolist(),
                     hashlib.sha256(pts.tobytes() + nrm.tobytes()).hexdigest()))
    grp.close()
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_mp_shard_worker, args=(r, 2, port, fr, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        for i, ((ok, err, pose, digest), (wok, wpose, wdigest)) in enumerate(zip(res[r], want)):
            assert err == 0, f"rank {r} frame {i}: exchange error flags {err}"
            assert ok == wok and pose == wpose, f"rank {r} frame {i}: pose differs from the in-process group"
            assert digest == wdigest, f"rank {r} frame {i}: maps differ"
