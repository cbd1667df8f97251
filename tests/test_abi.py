"""CPU suite: the C-ABI library loads, exports every symbol the header
declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_1410_0925_b200 import _abi
from paper_1410_0925_b200.pipeline import EngineSettings

HEADER = Path(__file__).resolve().parents[1] / "include" / "voxfuse_b200.h"


def declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(vf_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert sorted(_abi.EXPORTS) == declared()


def test_library_exports_every_declared_symbol():
    L = _abi.load()
    missing = [n for n in declared() if not hasattr(L, n)]
    assert not missing, f"not exported: {missing}"
    assert L.vf_abi_version() == _abi.ABI_VERSION


def test_struct_layouts_match_the_c_abi():
    L = _abi.load()
    assert L.vf_struct_size(0) == C.sizeof(_abi.VfSettings)
    assert L.vf_struct_size(1) == C.sizeof(_abi.VfCalib)
    assert L.vf_struct_size(2) == C.sizeof(_abi.VfFrameStats)
    assert L.vf_struct_size(3) == C.sizeof(_abi.VfAllocStats)
    assert L.vf_struct_size(4) == C.sizeof(_abi.VfIntrinsics)


def test_default_settings_are_the_reference_defaults():
    """vf_default_settings == EngineSettings() == the reference's defaults
    (scene_params.hpp:6-13, hash_volume.hpp:49-58, tracking_state.hpp:12-23,
    pipeline.hpp:32-35)."""
    L = _abi.load()
    s = _abi.VfSettings()
    L.vf_default_settings(C.byref(s))
    py = EngineSettings().to_c()
    for name, _ in _abi.VfSettings._fields_:
        assert getattr(s, name) == getattr(py, name), name
    assert (s.voxel_size, s.mu, s.max_weight) == (pytest.approx(0.004), pytest.approx(0.02), 100)
    assert (s.bucket_count, s.bucket_size, s.excess_count, s.block_count) == (1 << 20, 2, 1 << 17, 1 << 18)


def test_invalid_settings_rejected():
    L = _abi.load()
    s = EngineSettings(bucket_count=1000).to_c()  # not a power of two (hash_volume.hpp:138)
    cal = _abi.VfCalib()
    cal.depth.width, cal.depth.height = 64, 48
    h = C.c_void_p()
    assert L.vf_create(C.byref(s), C.byref(cal), 0, C.byref(h)) == _abi.VF_ERR_INVALID


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    from paper_1410_0925_b200 import VoxfuseError, make_pipeline, settings_from_config
    from paper_1410_0925_b200.scene import CONFIGS

    s, c = settings_from_config(CONFIGS["T160"])
    with pytest.raises(VoxfuseError) as ei:
        make_pipeline(s, c)
    assert ei.value.status == _abi.VF_ERR_NO_DEVICE


def test_no_fp32x2_contraction_in_sass():
    """ptxas (CUDA 12.9) contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2
    although .rn forbids it; the kernels keep such products scalar.  Guard:
    every object's SASS has exactly as many FFMA2 as its PTX has fma.*.f32x2."""
    import shutil
    import subprocess

    from paper_1410_0925_b200 import build as B

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    nvcc = B.nvcc_path()
    B.build()
    for src in B.SOURCES:
        ptx = subprocess.run([nvcc, *B.NVCC_FLAGS, "-ptx", str(B.CSRC / src), "-o", "-"], capture_output=True,
                             text=True, check=True).stdout
        sass = subprocess.run(["cuobjdump", "-sass", str(B.OUT_DIR / "obj" / (src + ".o"))], capture_output=True,
                              text=True, check=True).stdout
        n_ptx = len(re.findall(r"\bfma\.r[nzmp]\.f32x2\b", ptx))
        n_sass = len(re.findall(r"\bFFMA2\b", sass))
        assert n_ptx == n_sass, f"{src}: {n_sass} FFMA2 in SASS vs {n_ptx} fma.f32x2 in PTX"


def test_bench_metric_is_the_baseline_metric():
    """bench.py reports BASELINE.json's metric verbatim (both arms)."""
    import json
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    import bench
    assert bench.METRIC == json.loads((root / "BASELINE.json").read_text())["metric"]
