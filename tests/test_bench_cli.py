"""CPU suite: bench.py's launch contract.

* `--gpus N` outside torchrun re-launches itself with one rank per GPU
  (torch.distributed.run, rendezvous on 127.0.0.1) and N>1 defaults to
  config 5 sharded; `--dry-run` stops after the process group is formed.
* `--impl reference` times the reference's own pipeline on the same frames
  (W untimed, K timed) and prints the identical `config` as our arm.
"""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def _run(*args, timeout=240):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_gpus2_spawns_two_ranks():
    d = _run("--gpus", "2", "--dry-run")
    assert d["world"] == 2 and d["n_gpus"] == 2
    assert sorted(r["rank"] for r in d["ranks"]) == [0, 1]
    assert len({r["pid"] for r in d["ranks"]}) == 2
    assert d["mode"] == "shard" and d["config"] == "C5"


def test_gpus2_replica_mode_keeps_c1():
    d = _run("--gpus", "2", "--mode", "replica", "--dry-run")
    assert d["world"] == 2 and d["mode"] == "replica" and d["config"] == "C1"


def test_single_gpu_default_is_c1():
    d = _run("--dry-run")
    assert d["world"] == 1 and d["config"] == "C1"


def test_reference_arm_times_the_same_frames():
    import vf_py

    if not vf_py.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    import argparse

    import bench
    from paper_1410_0925_b200.scene import CONFIGS

    d = _run("--impl", "reference", "--config", "T160", "--steps", "3", "--warmup", "2")
    assert d["impl"] == "reference" and d["steps"] == 3 and d["warmup"] == 2
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    args = argparse.Namespace(warmup=2, steps=3, l2_flush_mib=256, mode="single")
    assert d["config"] == bench.config_dict(CONFIGS["T160"], args, 1)
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
