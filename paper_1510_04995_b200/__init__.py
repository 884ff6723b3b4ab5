"""girih-b200: B200-native temporally-blocked fp64 3-D stencil sweep (arXiv 1510.04995 path).

The compute path is libgirih_gpu.so (sm_100a CUDA, C ABI in include/girih_gpu.h); this package
is its host-side mirror of the reference's stencil/run interface.
"""
from ._lib import GirihError, InvalidArgument, LIB_PATH, load
from .stencil import (CONST7PT, CONST25PT, KINDS, VAR7PT, VAR25PT, DeviceState, GpuConfig,
                      GridSpec, PerfReport, ProblemState, StencilTraits, device_info, fp64_peak,
                      init_state, interior_checksum, model, nccl_unique_id, pinned_empty, plan,
                      run, run_instrumented, trim,
                      slab_layout,
                      stencil_from_name,
                      traits, variants)

__all__ = [
    "CONST7PT", "VAR7PT", "CONST25PT", "VAR25PT", "KINDS", "DeviceState", "GpuConfig", "GridSpec",
    "PerfReport", "ProblemState", "StencilTraits", "GirihError", "InvalidArgument", "LIB_PATH",
    "device_info", "fp64_peak", "init_state", "interior_checksum", "load", "model", "nccl_unique_id", "pinned_empty", "plan",
    "run", "run_instrumented", "slab_layout", "stencil_from_name", "traits", "trim", "variants",
]
