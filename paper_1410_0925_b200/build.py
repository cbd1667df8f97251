"""Build the in-tree sm_100a library ``paper_1410_0925_b200/lib/libvoxfuse_b200.so``.

nvcc cross-compiles for sm_100a without a GPU.  Flags that matter:

* ``-gencode arch=compute_100a,code=sm_100a``: B200 only, no other targets;
* ``--fmad=false`` (+ IEEE div/sqrt, the defaults): the kernels evaluate the
  reference's FP32/FP64 expressions with the reference's rounding, which is
  what makes block allocation, TSDF and the maps bit-exact;
* ``-lineinfo``: ncu source pages map to the .cu lines.

Usage: ``python -m paper_1410_0925_b200.build [--verbose]``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "lib"
LIB = OUT_DIR / "libvoxfuse_b200.so"
INCLUDE = PKG.parent / "include"

SOURCES = ["vf_alloc.cu", "vf_integrate.cu", "vf_raycast.cu", "vf_icp.cu", "vf_misc.cu", "vf_shard.cu", "vf_render.cu", "vf_swap.cu", "vf_track.cu", "vf_api.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-prec-div=true", "-prec-sqrt=true",
    "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-I", str(CSRC), "-I", str(INCLUDE),
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale(out: Path, deps) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, out_dir: Path | None = None, defines=()) -> Path:
    """Compile to out_dir (default: the in-tree lib/); `defines` are extra -D
    flags for tuning experiments (variants go to a separate directory)."""
    nvcc = nvcc_path()
    out = Path(out_dir) if out_dir else OUT_DIR
    lib = out / "libvoxfuse_b200.so"
    obj_dir = out / "obj"
    obj_dir.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [INCLUDE / "voxfuse_b200.h"]
    jobs = []
    for src in SOURCES:
        s = CSRC / src
        o = obj_dir / (src + ".o")
        if force or _stale(o, [s, *headers]):
            cmd = [nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-Xptxas", "-v", "-c", str(s), "-o", str(o)]
            jobs.append((src, cmd))
    log_lines = []

    def run(job):
        src, cmd = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, r

    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            for src, r in ex.map(run, jobs):
                log_lines.append(f"== {src}\n{r.stderr}")
                if r.returncode != 0:
                    sys.stderr.write(r.stderr)
                    raise RuntimeError(f"nvcc failed on {src}")
        (out / "ptxas.log").write_text("\n".join(log_lines))
    objs = [str(obj_dir / (s + ".o")) for s in SOURCES]
    if force or jobs or _stale(lib, objs):
        cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(lib), *objs,
               "-Xcompiler", "-fPIC", "-cudart", "static", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stderr)
            raise RuntimeError("link failed")
    if verbose and log_lines:
        print("\n".join(log_lines))
    return lib


if __name__ == "__main__":
    build(verbose="--verbose" in sys.argv, force="--force" in sys.argv)
    print(LIB)
