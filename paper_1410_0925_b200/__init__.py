"""paper_1410_0925_b200 — B200-native (sm_100a) dense-fusion hot path of InfiniTAM.

The product is the C-ABI library ``lib/libvoxfuse_b200.so`` (include/voxfuse_b200.h);
this package is its host-side mirror of the reference's engine interface
(``make_pipeline`` / ``IPipeline``) plus the benchmark scene definitions.
"""
from .pipeline import (  # noqa: F401
    Calibration,
    DeviceBuffer,
    EngineSettings,
    FrameStats,
    Intrinsics,
    Pipeline,
    make_pipeline,
    render_synthetic,
    settings_from_config,
)
from ._abi import LIB_PATH, VoxfuseError  # noqa: F401

__all__ = [
    "Calibration", "DeviceBuffer", "EngineSettings", "FrameStats", "Intrinsics", "Pipeline", "make_pipeline",
    "render_synthetic", "settings_from_config", "LIB_PATH", "VoxfuseError",
]
