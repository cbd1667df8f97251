#!/usr/bin/env python
"""Benchmark: frames/s of the dense-fusion hot path (ICP + allocation +
integration + raycast) at 640x480 on B200, plus voxel updates/s.

One step = one frame of the synthetic box-room sequence through the full
per-frame path (pipeline_impl.hpp:65-123).  Frames are rendered on the GPU
once, outside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1] [--impl ours|reference]

* value: device-resident inputs (vf_process_frame_device), CUDA events on the
  pipeline's stream around each frame, L2 flushed between frames (outside the
  per-frame intervals), summed over the K timed frames; max over ranks.
* e2e: pinned HOST buffers through the public API, depth (+rgb) H2D and the
  stats / pose D2H inside every timed step: streaming (vf_submit_frame /
  vf_collect_frame, two frames in flight) as `value`, and the blocking
  reference-shaped vf_process_frame as `sync_value`.
* roofline: per-stage CUDA events (profiling pass, same frames) for the
  dominant kernel and for integration.
* cpu_baseline: the reference's own code (oracle/_ref, shim-built) on the
  host cores, bounded sample, rank 0 at N=1 only.
* --impl reference: that CPU reference as the arm of record.
N>1 (`--gpus N` re-launches itself under torch.distributed.run, one rank
per GPU): by default config 5 — one volume (the C5 corridor) spatially
sharded by block hash across the GPUs, every rank on the same frames,
allocation / integration / raycast on its own shard, maps composited per
pixel with NCCL collectives inside the frame graph, ICP replicated on the
composited maps ("scaling": "strong": it adds capacity and shares the voxel
work, the frame is still one sequential step).  `--mode replica` runs an
independent copy of the sequence per GPU instead (no data-path collective,
"weak").  `--dry-run` launches the ranks and forms the process group only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frames/sec (alloc+integrate+raycast+ICP) at 640\u00d7480; voxel updates/sec"  # BASELINE.json metric, verbatim
UNIT = "frames/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=None,
                    help="default: C1 at N=1; C5 (the sharded corridor) at N>1 in shard mode")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="cpu_baseline sample inside our arm")
    ap.add_argument("--ref-seconds", type=float, default=240.0, help="--impl reference: time budget")
    ap.add_argument("--l2-flush-mib", type=int, default=256)
    ap.add_argument("--mode", default=None, choices=["shard", "replica"],
                    help="N>1: one volume spatially sharded by block hash across the GPUs (default; config 5, "
                         "NCCL nearest-depth map composite in the frame graph) or independent sequences per GPU")
    ap.add_argument("--no-roofline-large", action="store_true", help="skip the C3 integration roofline leg")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="shard mode: the per-frame map composite over peer memory in one kernel (default) or "
                         "as NCCL collectives in the frame graph")
    ap.add_argument("--shard-icp", action="store_true",
                    help="shard mode: pixel-sharded ICP with the per-iteration sums exchanged through peer memory "
                         "(default: every rank runs the whole ICP on the composited maps)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch the ranks and set up the process group, report them, run nothing on the GPU")
    return ap.parse_args()


def resolve(args, world: int):
    """Mode and config after the launch: N>1 defaults to config 5 sharded."""
    if world > 1:
        args.mode = args.mode or "shard"
        args.config = args.config or ("C5" if args.mode == "shard" else "C1")
    else:
        args.mode = "single"
        args.config = args.config or "C1"
    return args


def free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-run this command under
    torch.distributed.run with one rank per GPU (rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def config_dict(cfg, args, world: int) -> dict:
    """The `config` of the JSON line -- identical in both arms."""
    fx, fy, cx, cy, w, h = cfg.intrinsics
    rgb = cfg.voxel_type == 2
    sharded = world > 1 and args.mode == "shard"
    return {
        "workload": f"{cfg.name}: {w}x{h} depth, {cfg.voxel_size * 1000:.0f} mm voxels, mu {cfg.mu * 1000:.0f} mm, "
                    f"{'VoxelSRgb' if rgb else 'VoxelS'}, hash {cfg.hash.bucket_count}x{cfg.hash.bucket_size}"
                    f"+{cfg.hash.excess_count} / {cfg.hash.block_count} blocks"
                    f"{' per shard' if sharded else ''}, "
                    f"{'ICP tracking on' if cfg.tracking else 'known poses'}"
                    + (f", {cfg.scene} scene" if cfg.scene != "box_room" else "")
                    + (f", swapping B={cfg.swap_buffer_blocks}" if cfg.use_swapping else ""),
        "frames": f"{args.warmup} warm-up (incl. frame 0) then frames {args.warmup}..{args.warmup + args.steps - 1} timed",
        "parallelism": (f"volume sharded by block hash over {world} GPUs "
                        f"({'peer-memory' if getattr(args, 'transport', 'p2p') == 'p2p' else 'NCCL'} map composite, "
                        f"{'pixel-sharded ICP, peer-memory sums' if getattr(args, 'shard_icp', False) else 'replicated ICP'})"
                        if sharded
                        else f"one sequence per GPU x{world}" if world > 1 else "single GPU"),
        "l2": f"flushed between frames ({args.l2_flush_mib} MiB write, outside the timed intervals)",
        "graphs": True,
    }


# ---------------------------------------------------------------------------
# distributed plumbing (one process per GPU; torch.distributed for barrier/max)
# ---------------------------------------------------------------------------
class Dist:
    def __init__(self, n_expected: int):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.dev = None
        if self.world > 1:
            import torch
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            # the host-side plumbing (barriers, max over ranks, handle exchange)
            # over NCCL when every rank has its own GPU, else gloo (CPU tests,
            # VF_BENCH_ONE_DEVICE plumbing runs: NCCL refuses two ranks on one GPU)
            backend = "gloo"
            if (torch.cuda.is_available() and torch.cuda.device_count() >= self.world
                    and not os.environ.get("VF_BENCH_ONE_DEVICE")):
                backend = "nccl"
                torch.cuda.set_device(self.local_rank)
                self.dev = torch.device("cuda", self.local_rank)
            dist.init_process_group(backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, v: float) -> float:
        if not self.pg:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64, device=self.dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: float) -> float:
        if not self.pg:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64, device=self.dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference (CPU) arm
# ---------------------------------------------------------------------------
def cpu_reference_run(cfg, n_frames: int, budget_s: float, threads: int = 0):
    """Time the reference's own pipeline (oracle/_ref) on the host cores.
    Frames 1.. (tracked) are timed; frame 0 (no tracking) is untimed."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import vf_py
    from paper_1410_0925_b200.scene import scene_for, trajectory_for

    if not vf_py.ref_available():
        return None
    spheres, planes, far = scene_for(cfg)
    lib = vf_py.ref_lib()
    lib.lib.vfr_set_threads(threads if threads > 0 else (os.cpu_count() or 1))
    cores = int(lib.lib.vfr_get_threads())
    poses = trajectory_for(cfg, n_frames + 1)
    vol = vf_py.Volume(lib, cfg, tracking=cfg.tracking)
    rgb = cfg.voxel_type == 2
    depth0 = vf_py.render_depth(lib, cfg, poses[0], spheres, planes, 0.05, far)
    c0 = vf_py.render_rgb(lib, cfg, poses[0], spheres, planes, 0.05, far) if rgb else None
    vol.process(depth0, c0, None if cfg.tracking else poses[0])
    t_total, frames, voxels = 0.0, 0, 0
    stage = np.zeros(5)  # FrameStats::ms_* (pipeline.hpp:56-57)
    for i in range(1, n_frames + 1):
        d = vf_py.render_depth(lib, cfg, poses[i], spheres, planes, 0.05, far)
        c = vf_py.render_rgb(lib, cfg, poses[i], spheres, planes, 0.05, far) if rgb else None
        t0 = time.perf_counter()
        st = vol.process(d, c, None if cfg.tracking else poses[i])
        t_total += time.perf_counter() - t0
        frames += 1
        voxels += st.visible_blocks * 512
        stage += [st.ms_tracking, st.ms_allocation, st.ms_integration, st.ms_swapping, st.ms_raycast]
        if t_total >= budget_s:
            break
    vol.close()
    names = ("tracking", "allocation", "integration", "swapping", "raycast")
    return {"fps": frames / t_total, "frames": frames, "seconds": t_total, "cores": cores,
            "voxel_updates_per_s": voxels / t_total,
            "stage_ms": {k: float(v) / max(frames, 1) for k, v in zip(names, stage)}}


def run_reference_arm(args, dist: Dist):
    """The reference's own CPU pipeline (oracle/_ref: the unmodified reference
    sources, shim-built) on the SAME frames as our arm: frames 0..W-1 untimed
    (frame 0 fixes the pose), frames W..W+K-1 timed one step each, all host
    threads in the reference's pool (parallel.cpp:67-71).  Rank 0 only."""
    from paper_1410_0925_b200.scene import CONFIGS, scene_for, trajectory_for

    cfg = CONFIGS[args.config]
    if dist.rank != 0:
        return
    sys.path.insert(0, str(ROOT / "oracle"))
    import vf_py

    if not vf_py.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libvoxfuse_ref.so not built"}))
        return
    spheres, planes, far = scene_for(cfg)
    lib = vf_py.ref_lib()
    lib.lib.vfr_set_threads(os.cpu_count() or 1)
    cores = int(lib.lib.vfr_get_threads())
    n_frames = args.warmup + args.steps
    poses = trajectory_for(cfg, n_frames)
    vol = vf_py.Volume(lib, cfg, tracking=cfg.tracking)
    rgb = cfg.voxel_type == 2
    budget = max(60.0, args.ref_seconds)
    times, vox = [], 0
    stage = np.zeros(5)  # FrameStats::ms_* (pipeline.hpp:56-57)
    for i in range(n_frames):
        d = vf_py.render_depth(lib, cfg, poses[i], spheres, planes, 0.05, far)
        c = vf_py.render_rgb(lib, cfg, poses[i], spheres, planes, 0.05, far) if rgb else None
        t0 = time.perf_counter()
        st = vol.process(d, c, None if cfg.tracking else poses[i])
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            vox += st.visible_blocks * 512
            stage += [st.ms_tracking, st.ms_allocation, st.ms_integration, st.ms_swapping, st.ms_raycast]
            if sum(times) > budget:  # bounded: a slow config stops early and says so
                break
    vol.close()
    total = float(sum(times))
    fps = len(times) / total
    names = ("tracking", "allocation", "integration", "swapping", "raycast")
    sample = (f"{cfg.name}: frames {args.warmup}..{args.warmup + len(times) - 1} of the sequence timed one per step "
              f"after {args.warmup} untimed (frame 0 included), the reference pipeline via make_pipeline/process_frame")
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": 1000.0 * total / len(times),
        "higher_is_better": True, "scaling": "strong" if args.mode == "shard" else "weak", "vs_baseline": None,
        "dtype": "f32 (TSDF/raycast) + f64 (allocation DDA, ICP)", "data": data_desc(cfg, n_frames),
        "config": config_dict(cfg, args, dist.world),
        "voxel_updates_per_s": vox / total,
        "cpu_baseline": {"value": fps, "unit": UNIT, "cores": cores, "kind": "reference",
                         "build": "the reference's unmodified sources, -O3, against the scalar Eigen shim "
                                  "(oracle/eigen_shim: no SIMD Eigen on the box)",
                         "sample": sample},
        "stage_ms": {k: float(v) / max(len(times), 1) for k, v in zip(names, stage)},
        "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        **({"budget_stop": f"stopped after {total:.0f} s ({len(times)} of {args.steps} steps)"}
           if len(times) < args.steps else {}),
    }
    print(json.dumps(line))


def data_desc(cfg, n_frames: int) -> str:
    if cfg.scene == "corridor":
        return f"synthetic (corridor + pillars, {n_frames}-frame walk at 5 cm/frame)"
    return "synthetic (box room + spheres, 100-frame small-motion trajectory)"


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, dist: Dist):
    from paper_1410_0925_b200 import DeviceBuffer, Intrinsics, make_pipeline, render_synthetic, settings_from_config
    from paper_1410_0925_b200 import _abi
    from paper_1410_0925_b200.scene import CONFIGS, scene_for, trajectory_for

    L = _abi.load()
    cfg = CONFIGS[args.config]
    if dist.world > 1 and not os.environ.get("VF_BENCH_ONE_DEVICE"):
        import torch

        if torch.cuda.device_count() < dist.world:
            raise SystemExit(f"bench.py --gpus {dist.world}: only {torch.cuda.device_count()} GPU(s) visible "
                             "(VF_BENCH_ONE_DEVICE=1 runs every rank on GPU 0 for a plumbing test)")
    # VF_BENCH_ONE_DEVICE=1 puts every rank on GPU 0 (exercises the N>1 plumbing on a one-GPU box)
    device = 0 if os.environ.get("VF_BENCH_ONE_DEVICE") else dist.local_rank
    fx, fy, cx, cy, w, h = cfg.intrinsics
    intr = Intrinsics(fx, fy, cx, cy, w, h)
    rgb = cfg.voxel_type == 2
    n_frames = args.warmup + args.steps
    poses = trajectory_for(cfg, n_frames)
    spheres, planes, far = scene_for(cfg)
    # inputs rendered once on the GPU, resident in HBM
    d_frames = [DeviceBuffer(w * h * 4) for _ in range(n_frames)]
    c_frames = [DeviceBuffer(w * h * 3) for _ in range(n_frames)] if rgb else None
    for i in range(n_frames):
        render_synthetic(poses[i], intr, spheres, planes, d_frames[i].ptr, c_frames[i].ptr if rgb else None,
                         far=far, device=device)
    settings, calib = settings_from_config(cfg)
    flush = args.l2_flush_mib << 20
    sharded = dist.world > 1 and args.mode == "shard"
    if sharded:
        from dataclasses import replace

        settings = replace(settings, shard_count=dist.world, shard_index=dist.rank, shard_icp=args.shard_icp)

    def new_pipeline():
        p = make_pipeline(settings, calib, device=device)
        if sharded:  # NCCL nearest-depth composite inside the frame graph
            from paper_1410_0925_b200.sharding import attach_nccl

            if args.transport == "p2p":  # one composite kernel over peer memory (CUDA IPC over NVLink)
                from paper_1410_0925_b200.sharding import attach_p2p

                attach_p2p(p, dist.rank, dist.world, dist.pg)
            else:
                attach_nccl(p, dist.rank, dist.world, dist.pg)
            if args.shard_icp:  # pixel-sharded ICP: per-iteration sums over CUDA IPC peer memory
                from paper_1410_0925_b200.sharding import attach_icp_peers

                attach_icp_peers(p, dist.rank, dist.world, dist.pg)
        return p

    swaps = []

    def run_device(collect_stages=False):
        p = new_pipeline()
        hctx = p.handle
        ms_frames, vis_blocks, modified, iters = [], [], [], []
        swaps.clear()
        stage = np.zeros(8)
        for i in range(n_frames):
            timed = i >= args.warmup
            if collect_stages and i == args.warmup:
                p.set_profiling(True)  # resets the per-stage accumulators
            if not cfg.tracking:
                p.set_pose(poses[i])
            if timed:
                _abi.check("vf_flush_l2", L.vf_flush_l2(hctx, flush))
                if i == args.warmup:
                    p.synchronize()
                    dist.barrier()
                _abi.check("vf_event_record", L.vf_event_record(hctx, 8))
            p.process_frame_device(d_frames[i].ptr, c_frames[i].ptr if rgb else None)
            if timed:
                _abi.check("vf_event_record", L.vf_event_record(hctx, 9))
                ms = C.c_float()
                _abi.check("vf_event_elapsed_ms", L.vf_event_elapsed_ms(hctx, 8, 9, C.byref(ms)))
                ms_frames.append(ms.value)
                st = _abi.VfFrameStats()
                _abi.check("vf_read_stats", L.vf_read_stats(hctx, C.byref(st)))
                vis_blocks.append(st.visible_blocks)
                iters.append(st.tracking_iterations)
                swaps.append((st.swapped_in, st.swapped_out, st.swap_bytes_in + st.swap_bytes_out,
                              st.allocation_dropped))
                modified.append(L.vf_last_modified_voxels(hctx))
        counters = None
        if collect_stages:
            stage, nprof = p.stage_times()
            stage = stage / max(nprof, 1)
            counters = p.raycast_counters()  # last frame's raycast re-run with counters (untimed)
            run_device.alloc = p.alloc_counters()  # and mark_blocks' walk
            if cfg.tracking and cfg.tracker == "icp":
                run_device.icp = icp_rates(p, cfg, intr, poses, spheres, planes, far, device)
        launches = sum(p.kernel_launches_per_frame(cfg.tracking and i > 0) for i in range(args.warmup, n_frames))
        if not cfg.tracking:
            launches += n_frames - args.warmup  # k_set_pose per known-pose frame
        p.close()
        run_device.counters = counters
        run_device.iters = float(np.mean(iters)) if iters else 0.0
        return np.array(ms_frames), np.array(vis_blocks), np.array(modified), stage, launches

    # --- timed pass (graphs on) ---
    clocks = ClockSampler(device)
    clocks.start()
    ms_frames, vis, modified, _, launches = run_device()
    swaps_t = list(swaps)
    clk = clocks.stop()
    t_local = float(ms_frames.sum()) / 1000.0
    t_max = dist.max(t_local)
    # sharded: all ranks cooperate on the same frames; replicas: each rank its own
    frames_total = float(args.steps) if sharded else dist.sum(float(args.steps))
    value = frames_total / t_max
    vox_updates = dist.sum(float(vis.sum() * 512)) / t_max

    # --- e2e pass: host pinned buffers through vf_process_frame ---
    p = new_pipeline()
    hctx = p.handle
    npix = w * h
    host_depth = []
    for i in range(n_frames):
        ptr = L.vf_host_alloc_pinned(npix * 4)
        arr = np.ctypeslib.as_array((C.c_float * npix).from_address(ptr))
        arr[:] = d_frames[i].to_host(np.float32, (npix,))
        host_depth.append((ptr, arr))
    host_rgb = []
    if rgb:
        for i in range(n_frames):
            ptr = L.vf_host_alloc_pinned(npix * 3)
            arr = np.ctypeslib.as_array((C.c_uint8 * (npix * 3)).from_address(ptr))
            arr[:] = c_frames[i].to_host(np.uint8, (npix * 3,))
            host_rgb.append((ptr, arr))
    st = _abi.VfFrameStats()

    def pose_frame(i):
        if not cfg.tracking:
            p.set_pose(poses[i])

    def rgb_ptr(i):
        return C.c_void_p(host_rgb[i][0]) if rgb else None

    # (1) synchronous: one vf_process_frame per step (upload, frame, stats
    # readback, wait), L2 flushed before each step outside the interval
    e2e_sync_ms = 0.0
    for i in range(n_frames):
        timed = i >= args.warmup
        pose_frame(i)
        if timed:
            _abi.check("vf_flush_l2", L.vf_flush_l2(hctx, flush))
            p.synchronize()
            if i == args.warmup:
                dist.barrier()
            t0 = time.perf_counter()
        _abi.check("vf_process_frame", L.vf_process_frame(hctx, C.c_void_p(host_depth[i][0]), rgb_ptr(i),
                                                          C.byref(st)))
        if timed:
            e2e_sync_ms += (time.perf_counter() - t0) * 1000.0
    # (2) streaming: vf_submit_frame / vf_collect_frame with two frames in
    # flight, so frame n + 1's upload overlaps frame n; every step still
    # uploads its depth (+ rgb) from pinned host memory and reads its stats
    # back.  L2 is flushed in-stream before every frame; the flushes' own
    # event-timed durations are taken out of the wall time.
    p2 = new_pipeline()
    h2 = p2.handle
    for i in range(args.warmup):
        if not cfg.tracking:
            p2.set_pose(poses[i])
        _abi.check("vf_submit_frame", L.vf_submit_frame(h2, C.c_void_p(host_depth[i][0]), rgb_ptr(i)))
        _abi.check("vf_collect_frame", L.vf_collect_frame(h2, C.byref(st)))
    fl = C.c_double(0.0)
    _abi.check("vf_flush_l2", L.vf_flush_l2(h2, flush))  # allocates the flush buffer outside the timed loop
    _abi.check("vf_flush_time", L.vf_flush_time(h2, C.byref(fl)))
    dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.warmup, n_frames):
        if not cfg.tracking:
            p2.set_pose(poses[i])
        _abi.check("vf_flush_l2", L.vf_flush_l2(h2, flush))
        _abi.check("vf_submit_frame", L.vf_submit_frame(h2, C.c_void_p(host_depth[i][0]), rgb_ptr(i)))
        if L.vf_frames_in_flight(h2) >= 2:
            _abi.check("vf_collect_frame", L.vf_collect_frame(h2, C.byref(st)))
    while L.vf_frames_in_flight(h2) > 0:
        _abi.check("vf_collect_frame", L.vf_collect_frame(h2, C.byref(st)))
    wall = time.perf_counter() - t0
    _abi.check("vf_flush_time", L.vf_flush_time(h2, C.byref(fl)))
    e2e_ms = wall * 1000.0 - fl.value
    e2e_flush_ms = fl.value
    p2.close()
    readback = int(L.vf_readback_bytes(hctx))
    p.close()
    for ptr, _ in host_depth + host_rgb:
        L.vf_host_free_pinned(ptr)
    e2e_t = dist.max(e2e_ms / 1000.0)
    e2e_value = frames_total / e2e_t
    e2e_sync_value = frames_total / dist.max(e2e_sync_ms / 1000.0)

    # --- profiling pass: per-stage events (no graphs) ---
    _, vis_p, mod_p, stage_ms, _ = run_device(collect_stages=True)
    st_iters = run_device.iters
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"
    vsize = 8 if rgb else 4
    nvis = float(vis_p.mean())
    nmod = float(mod_p.mean())
    # B = N_vis (512 sizeof(V) + 4 + 16) + N_mod sizeof(V) + W H 4 (+ W H 3 rgb)
    integ_bytes = nvis * (512 * vsize + 4 + 16) + nmod * vsize + npix * 4 + (npix * 3 if rgb else 0)
    stages = {"tracking": stage_ms[0], "allocation": stage_ms[1], "integration": stage_ms[2],
              "raycast": stage_ms[4]}
    if cfg.use_swapping:
        stages["swapping"] = stage_ms[3]
    integ_ms = stage_ms[2]
    integ_gbs = integ_bytes / (integ_ms * 1e-3) / 1e9 if integ_ms > 0 else 0.0
    dominant = max(stages, key=stages.get)
    traffic = ncu_traffic(args.config)
    roofline = {
        "kernel": "k_integrate (TSDF integration)", "bound": "hbm", "achieved": integ_gbs, "peak": hbm_peak,
        "unit": "GB/s", "frac": integ_gbs / hbm_peak, "traffic": traffic["bytes"] if traffic else None,
        **({"traffic_source": traffic["source"]} if traffic else {}),
        "algorithmic_bytes_per_launch": integ_bytes, "ms_per_launch": integ_ms, "peak_source": peak_src,
        "note": f"dominant stage by time is {dominant}; integration is the HBM-graded kernel",
    }
    # The latency-bound stages against the same HBM peak, from the committed
    # capture's DRAM bytes per launch over this run's event-timed stage: shows
    # how far from memory-bound they are (C1 only; the capture is C1's).
    if args.config == "C1":
        stage_kernels = {"raycast": ("k_raycast", "k_ray_normals"), "tracking": ("k_pyramid", "k_icp_cluster", "k_icp")}
        rows = {}
        for stage, kernels in stage_kernels.items():
            b = sum((ncu_kernel_bytes("r2_ncu.json", "c1_full", k) or 0.0) for k in kernels)
            ms = stages.get(stage, 0.0)
            if b > 0 and ms > 0:
                gbs = b / (ms * 1e-3) / 1e9
                rows[stage] = {"kernels": list(kernels), "dram_bytes": b, "ms": ms, "achieved_gbs": gbs,
                               "frac_of_hbm": gbs / hbm_peak}
        if rows:
            roofline["latency_bound_stages"] = rows

    if dist.rank == 0 and not args.no_roofline_large:
        roofline["large"] = roofline_large(args, device, hbm_peak, peak_src)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * t_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None,
        "dtype": "f32 (TSDF/raycast) + f64 (allocation DDA, ICP)",
        "data": data_desc(cfg, n_frames),
        "config": config_dict(cfg, args, dist.world),
        "voxel_updates_per_s": vox_updates,
        "stage_ms": stages,
        # per-stage throughput in the units of SURVEY.md §8(d)
        "stage_throughput": {
            "raycast_rays_per_s": npix / (stages["raycast"] * 1e-3) if stages["raycast"] > 0 else None,
            **raycast_rates(run_device.counters, stages["raycast"]),
            **alloc_rates(getattr(run_device, "alloc", None), stages["allocation"]),
            **icp_throughput(getattr(run_device, "icp", None), stages["tracking"], st_iters),
            "integration_voxel_visits_per_s": nvis * 512 / (integ_ms * 1e-3) if integ_ms > 0 else None,
            "allocation_pixels_per_s": npix / (stages["allocation"] * 1e-3) if stages["allocation"] > 0 else None,
        },
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": npix * 4 + (npix * 3 if rgb else 0),
                "d2h_bytes_per_step": readback,
                "mode": "streaming: vf_submit_frame / vf_collect_frame, 2 frames in flight (upload of n+1 "
                        "overlaps frame n), pinned host buffers, L2 flushed in-stream before every frame and "
                        "the flushes' event-timed ms taken out of the wall time",
                "l2_flush_ms_removed": e2e_flush_ms,
                "sync_value": e2e_sync_value,
                "sync_mode": "one blocking vf_process_frame per step (upload, frame, stats readback), "
                             "L2 flushed before each step outside the interval"},
        "gpu_launches": launches,
        **({"swap": {"swapped_in_per_frame": float(np.mean([x[0] for x in swaps_t])),
                     "swapped_out_per_frame": float(np.mean([x[1] for x in swaps_t])),
                     "bytes_per_frame": float(np.mean([x[2] for x in swaps_t])),
                     "allocation_dropped_total": int(sum(x[3] for x in swaps_t)),
                     "buffer_blocks": cfg.swap_buffer_blocks,
                     "host_store": "pinned host memory mapped into the device; transfers by k_swap_transfer"}}
           if cfg.use_swapping else {}),
        "roofline": roofline,
        "clocks": clk,
    }
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        ref = cpu_reference_run(cfg, min(n_frames - 1, 30), args.cpu_seconds)
        if ref:
            line["cpu_baseline"] = {"value": ref["fps"], "unit": UNIT, "cores": ref["cores"], "kind": "reference",
                                    "build": "the reference's unmodified sources, -O3, against the scalar Eigen "
                                             "shim (oracle/eigen_shim: no SIMD Eigen on the box)",
                                    "stage_ms": ref["stage_ms"],
                                    "sample": f"{cfg.name} frames 1..{ref['frames']} ({ref['seconds']:.1f} s), "
                                              "reference pipeline (oracle/_ref) via process_frame"}
    if dist.rank == 0:
        print(json.dumps(line))


def icp_rates(p, cfg, intr, poses, spheres, planes, far, device) -> dict:
    """SURVEY.md §8(d) K4 units: one icp_track call (untimed, traced) of the
    next frame of the trajectory against the last frame's maps --
    iterations per level, pixel-iterations (pyramid pixels x iterations) and
    the per-iteration phase timers of the persistent kernels."""
    from paper_1410_0925_b200 import DeviceBuffer, render_synthetic
    from paper_1410_0925_b200.scene import trajectory_for

    nxt = trajectory_for(cfg, len(poses) + 1)[-1]
    buf = DeviceBuffer(intr.width * intr.height * 4)
    render_synthetic(nxt, intr, spheres, planes, buf.ptr, None, far=far, device=device)
    d = buf.to_host(np.float32, (intr.height, intr.width))
    buf.free()
    r = p.icp_track(d)
    tr = p.icp_trace()
    if not len(tr):
        return {}
    levels = {}
    w, h = intr.width, intr.height
    sizes = []
    for _ in range(cfg.levels):
        sizes.append(w * h)
        w, h = (w + 1) // 2, (h + 1) // 2
    pix_it = 0
    for row in tr:
        lv = int(row[0])
        levels[lv] = levels.get(lv, 0) + 1
        pix_it += sizes[lv]
    cyc = tr[:, 44:48].sum(0)
    return {"icp_iterations_per_level": {str(k): v for k, v in sorted(levels.items(), reverse=True)},
            "icp_pixel_iterations": int(pix_it), "icp_tracking_ok": bool(r["ok"]),
            "icp_note": "one traced icp_track call: the trajectory's next frame against the last timed frame's maps",
            "icp_phase_cycles": {"pixel_terms": float(cyc[0]), "barrier": float(cyc[1]), "partial_sums": float(cyc[2]),
                                 "controller": float(cyc[3])}}


def icp_throughput(icp, track_ms: float, iters: float) -> dict:
    """The traced icp_track call's K4 units, plus the timed frames' solved
    iterations.  The traced call counts every evaluation (accepted steps,
    halvings, rejected steps); its device time comes from its phase timers
    (SM cycles at the 1965 MHz the clocks report under load)."""
    if not icp or track_ms <= 0:
        return {}
    out = dict(icp)
    evals = sum(icp["icp_iterations_per_level"].values())
    t = sum(icp["icp_phase_cycles"].values()) / 1.965e9
    out["icp_evaluations"] = evals
    out["icp_us_per_evaluation"] = 1e6 * t / max(evals, 1)
    out["icp_pixel_evaluations_per_s"] = icp["icp_pixel_iterations"] / t if t > 0 else None
    out["icp_solved_iterations_per_frame"] = iters  # FrameStats::tracking_iterations, timed frames
    return out


def alloc_rates(cnt, alloc_ms: float) -> dict:
    """SURVEY.md §8(d) K1 units: mark_blocks' DDA cells (one hash-bucket probe
    each) of the last frame, over the allocation stage's time."""
    if not cnt or alloc_ms <= 0:
        return {}
    return {"allocation_cells_probed_per_frame": cnt["cells_probed"],
            "allocation_probes_per_s": cnt["cells_probed"] / (alloc_ms * 1e-3),
            "allocation_cells_per_depth_pixel": cnt["cells_probed"] / max(cnt["pixels"], 1)}


def raycast_rates(cnt, ray_ms: float) -> dict:
    """SURVEY.md §8(d) K3 units from the counting re-run of the last frame's
    raycast (vf_raycast_counters): hash-table probes (our block-cache misses),
    voxel reads (each a hash probe in the reference's sampler), rays, hits."""
    if not cnt or ray_ms <= 0:
        return {}
    t = ray_ms * 1e-3
    return {"raycast_table_probes_per_frame": cnt["table_probes"], "raycast_voxel_reads_per_frame": cnt["voxel_reads"],
            "raycast_rays_marched_per_frame": cnt["rays"], "raycast_hits_per_frame": cnt["hits"],
            "raycast_table_probes_per_s": cnt["table_probes"] / t, "raycast_voxel_reads_per_s": cnt["voxel_reads"] / t,
            "raycast_probe_cache_hit_rate": 1.0 - cnt["table_probes"] / max(cnt["voxel_reads"], 1)}


def roofline_large(args, device: int, hbm_peak: float, peak_src: str) -> dict:
    """the >= 60 % HBM target is judged at C3 or at a C2
    kernel bench with >= 100k visible blocks; C1's ~19k-block launch is
    latency-bound.  Same process, same GPU: the C3 frames (1280x960, 2 mm,
    2^20 blocks, VoxelS) and the C2L frames (the same at VoxelSRgb, with RGB)
    at their known poses, per-stage CUDA events around the integration
    kernel, L2 flushed between frames; both integration modes (exact:
    bit-exact vs the reference; fast: <= 1 LSB, tests/test_gpu_integration_fast.py)."""
    from dataclasses import replace

    from paper_1410_0925_b200 import DeviceBuffer, Intrinsics, make_pipeline, render_synthetic, settings_from_config
    from paper_1410_0925_b200 import _abi
    from paper_1410_0925_b200.scene import CONFIGS, scene_for, trajectory_for

    L = _abi.load()
    warm, timed = 3, 10
    out = {"config": f"C3 (VoxelS) and C2L (VoxelSRgb + RGB) frames {warm}..{warm + timed - 1} at known poses "
                     f"(integration kernel only timed), L2 flushed ({args.l2_flush_mib} MiB) before every frame",
           "bound": "hbm", "unit": "GB/s", "peak": hbm_peak, "peak_source": peak_src}
    for cname in ("C3", "C2L"):
        cfg = CONFIGS[cname].with_(tracking=False)
        rgb = cfg.voxel_type == 2
        vsize = 8 if rgb else 4
        fx, fy, cx, cy, w, h = cfg.intrinsics
        poses = trajectory_for(cfg, warm + timed)
        spheres, planes, far = scene_for(cfg)
        frames = [DeviceBuffer(w * h * 4) for _ in poses]
        colours = [DeviceBuffer(w * h * 3) for _ in poses] if rgb else None
        for i, pose in enumerate(poses):
            render_synthetic(pose, Intrinsics(fx, fy, cx, cy, w, h), spheres, planes, frames[i].ptr,
                             colours[i].ptr if rgb else None, far=far, device=device)
        settings, calib = settings_from_config(cfg)
        for mode, name in ((0, "exact"), (1, "fast")):
            p = make_pipeline(replace(settings, integration_mode=mode), calib, device=device)
            nvis, nmod = [], []
            for i, pose in enumerate(poses):
                if i == warm:
                    p.set_profiling(True)
                p.set_pose(pose)
                _abi.check("vf_flush_l2", L.vf_flush_l2(p.handle, args.l2_flush_mib << 20))
                st = p.process_frame_device(frames[i].ptr, colours[i].ptr if rgb else None, read_stats=True)
                if i >= warm:
                    nvis.append(st.visible_blocks)
                    nmod.append(L.vf_last_modified_voxels(p.handle))
            stage, nprof = p.stage_times()
            p.close()
            ms = stage[2] / max(nprof, 1)
            # B = N_vis (512 sizeof(V) + 4 + 16) + N_mod sizeof(V) + W H 4 (+ W H 3)
            b = (float(np.mean(nvis)) * (512 * vsize + 20) + float(np.mean(nmod)) * vsize + w * h * 4
                 + (w * h * 3 if rgb else 0))
            gbs = b / (ms * 1e-3) / 1e9
            kname = ("k_integrate_rgb" if rgb else "k_integrate_s") if mode == 0 else \
                ("k_integrate_fast_rgb" if rgb else "k_integrate_fast")
            key = name if cname == "C3" else f"{name}_rgb"
            entry = {"config": cname, "kernel": kname, "achieved": gbs, "frac": gbs / hbm_peak, "ms_per_launch": ms,
                     "algorithmic_bytes_per_launch": b, "visible_blocks": float(np.mean(nvis)),
                     "voxel_visits_per_s": float(np.mean(nvis)) * 512 / (ms * 1e-3)}
            if cname == "C3":
                tb = ncu_kernel_bytes("r2_ncu.json", "c3_integrate_exact" if mode == 0 else "c3_integrate_fast", kname)
                entry.update({"traffic": tb, "traffic_source": "profiles/r2_ncu.json (ncu --set full, same kernel "
                                                               "at C3): dram read + write"})
            out[key] = entry
        for f in frames + (colours or []):
            f.free()
    return out


# Committed `ncu --set full` captures of the roofline kernel per config
# (profiles/): dram__bytes_read.sum + dram__bytes_write.sum of one launch.
NCU_TRAFFIC = {
    "C1": ("r2_ncu.json", "c1_full", "k_integrate_s"),
    "C3": ("r2_ncu.json", "c3_integrate_exact", "k_integrate_s"),
    "C2": ("r1d_ncu_c2c4.json", "c2_rgb", "k_integrate_rgb"),
}


def ncu_kernel_bytes(fname, section, kernel):
    """dram read + write bytes of `kernel` in a committed capture, or None."""
    try:
        rows = json.loads((ROOT / "profiles" / fname).read_text())[section]
    except (OSError, KeyError, ValueError):
        return None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows:
        if r.get("kernel") == kernel:
            tot = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v, u = r[k].split()
                tot += float(v) * scale[u]
            return tot
    return None


def ncu_traffic(config):
    """DRAM bytes of one launch of the roofline kernel from the committed
    capture, or None.  ncu replays with caches flushed; L2 is write-back, so
    voxels written by the kernel drain to DRAM after it ends and the write
    side of a launch whose working set fits L2 reads near zero."""
    ent = NCU_TRAFFIC.get(config)
    if not ent:
        return None
    b = ncu_kernel_bytes(*ent)
    if b is None:
        return None
    return {"bytes": b, "source": f"profiles/{ent[0]} [{ent[1]}] {ent[2]}: dram read + write per launch"}


def dry_run(args, dist: Dist):
    """Ranks up, process group formed, config resolved; nothing on the GPU."""
    info = {"rank": dist.rank, "local_rank": dist.local_rank, "world": dist.world, "pid": os.getpid()}
    ranks = [info]
    if dist.pg:
        ranks = [None] * dist.world
        dist.pg.all_gather_object(ranks, info)
    if dist.rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": args.gpus, "world": dist.world, "mode": args.mode,
                          "config": args.config, "impl": args.impl, "ranks": ranks}))


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    dist = Dist(args.gpus)
    resolve(args, dist.world)
    if dist.world > 1 and args.mode == "shard":
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines in the log (rank check)
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    try:
        if args.dry_run:
            dry_run(args, dist)
            return
        if args.impl == "reference":
            run_reference_arm(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
