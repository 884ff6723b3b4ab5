"""ctypes binding of libgirih_gpu.so (include/girih_gpu.h).

The CUDA library is the product: if it is missing or fails to load, importing this module
raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# GIRIH_LIB overrides the library path (A/B measurements of two builds in one process)
LIB_PATH = os.environ.get("GIRIH_LIB") or os.path.join(HERE, "libgirih_gpu.so")

GIRIH_OK = 0
GIRIH_EINVAL = -1
GIRIH_ECUDA = -2
GIRIH_ENCCL = -3
GIRIH_ENOMEM = -4
GIRIH_ESTATE = -5


GIRIH_GPU_IPC_BYTES = 512  # include/girih_gpu.h


class GirihStateView(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("pad_x", C.c_int),
        ("t_current", C.c_longlong),
        ("u", C.POINTER(C.c_double)),
        ("v", C.POINTER(C.c_double)),
        ("coeffs", C.POINTER(C.POINTER(C.c_double))),
        ("n_coeffs", C.c_int),
        ("cc", C.c_double * 5),
    ]


class GirihGpuConfig(C.Structure):
    _fields_ = [
        ("tb", C.c_int), ("variant", C.c_int), ("zchunks", C.c_int), ("ngpus", C.c_int),
        ("exact", C.c_int), ("device", C.c_int), ("graphs", C.c_int), ("reserved", C.c_int),
        ("chain", C.c_int), ("tile_order", C.c_int),
    ]


class GirihGpuReport(C.Structure):
    _fields_ = [
        ("wall_s", C.c_double), ("kernel_s", C.c_double),
        ("h2d_s", C.c_double), ("d2h_s", C.c_double),
        ("lups", C.c_longlong), ("mlups", C.c_double),
        ("model_bytes_per_lup", C.c_double), ("tb_used", C.c_int), ("n_launches", C.c_int),
        ("pass_s", C.c_double), ("computed_lups", C.c_longlong),
        ("h2d_bytes", C.c_longlong), ("d2h_bytes", C.c_longlong),
        ("variant_used", C.c_int), ("zchunks_used", C.c_int), ("grid_ctas", C.c_int),
        ("streamed", C.c_int), ("n_passes", C.c_int), ("units", C.c_longlong),
    ]


class GirihGpuVariant(C.Structure):
    _fields_ = [("kind", C.c_int), ("tb", C.c_int), ("lx", C.c_int), ("ly", C.c_int),
                ("threads", C.c_int), ("prefetch", C.c_int), ("smem_bytes", C.c_int),
                ("cluster_y", C.c_int), ("aux_prefetch", C.c_int), ("direct_out", C.c_int),
                ("paced", C.c_int), ("narrow", C.c_int)]


class GirihGpuTraceRecord(C.Structure):
    _fields_ = [("pass_", C.c_int), ("unit", C.c_int), ("cta", C.c_int), ("sm", C.c_int),
                ("start_ns", C.c_ulonglong), ("end_ns", C.c_ulonglong)]


GIRIH_TRACE_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(GirihGpuTraceRecord), C.c_longlong)


class GirihGpuRunOptions(C.Structure):
    _fields_ = [("trace_cb", GIRIH_TRACE_FN), ("trace_ctx", C.c_void_p),
                ("trace_capacity", C.c_longlong), ("trace_total", C.c_longlong),
                ("ledger", C.POINTER(C.c_uint))]


# every symbol include/girih_gpu.h declares, with (restype, argtypes)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
class GirihGpuModel(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("tb", "variant", "lx", "ly", "ox", "oy", "threads",
                                        "smem_bytes", "ctas_per_sm", "tiles_x", "tiles_y",
                                        "zchunks", "zc_len")] + \
               [(n, C.c_double) for n in ("redundancy", "code_balance", "code_balance_no_l2",
                                           "hbm_mlups", "fp64_mlups", "roofline_mlups")]


SIGNATURES = {
    "girih_gpu_last_error": (C.c_char_p, []),
    "girih_gpu_abi_version": (C.c_int, []),
    "girih_gpu_traits": (C.c_int, [C.c_int, _ip, _ip, _ip, _ip, _ip]),
    "girih_gpu_kind_from_name": (C.c_int, [C.c_char_p, _ip]),
    "girih_gpu_variant_count": (C.c_int, []),
    "girih_gpu_variant_info": (C.c_int, [C.c_int, C.POINTER(GirihGpuVariant)]),
    "girih_gpu_open": (C.c_int, [C.POINTER(GirihStateView), C.POINTER(GirihGpuConfig),
                                 C.POINTER(C.c_void_p)]),
    "girih_gpu_open_seeded": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_ulonglong, C.c_int, C.POINTER(GirihGpuConfig),
                                        C.POINTER(C.c_void_p)]),
    "girih_gpu_nccl_unique_id": (C.c_int, [C.c_char_p, C.c_int]),
    "girih_gpu_open_slab_seeded": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.c_ulonglong, C.c_int, C.c_int, C.c_int, C.c_char_p,
                                             C.POINTER(GirihGpuConfig), C.POINTER(C.c_void_p)]),
    "girih_gpu_ipc_export": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int]),
    "girih_gpu_ipc_connect": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p]),
    "girih_gpu_upload": (C.c_int, [C.c_void_p, C.POINTER(GirihStateView)]),
    "girih_gpu_step": (C.c_int, [C.c_void_p, C.c_longlong, C.POINTER(GirihGpuReport)]),
    "girih_gpu_download": (C.c_int, [C.c_void_p, C.POINTER(GirihStateView)]),
    "girih_gpu_download_coeffs": (C.c_int, [C.c_void_p, C.POINTER(_dp), C.c_int, _dp]),
    "girih_gpu_row_digest": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_ulonglong)]),
    "girih_gpu_run_ex": (C.c_int, [C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p]),
    "girih_gpu_update_units": (C.c_int, [C.c_void_p, C.c_longlong, C.c_longlong, C.c_longlong,
                                         C.POINTER(C.c_longlong)]),
    "girih_gpu_get_t": (C.c_int, [C.c_void_p, C.POINTER(C.c_longlong)]),
    "girih_gpu_set_config": (C.c_int, [C.c_void_p, C.POINTER(GirihGpuConfig)]),
    "girih_gpu_close": (C.c_int, [C.c_void_p]),
    "girih_gpu_run": (C.c_int, [C.POINTER(GirihStateView), C.c_longlong,
                                C.POINTER(GirihGpuConfig), C.POINTER(GirihGpuReport)]),
    "girih_gpu_plan": (C.c_int, [C.c_int, C.c_longlong, C.c_longlong, C.c_int, C.c_int,
                                 _ip, _ip, _ip, _ip, _ip, _ip]),
    "girih_gpu_slab_layout": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _ip, _ip, _ip]),
    "girih_gpu_compare": (C.c_int, [C.c_void_p, C.c_int, _dp, C.POINTER(C.c_longlong),
                                    C.POINTER(C.c_longlong)]),
    "girih_gpu_trim": (C.c_int, []),
    "girih_gpu_model": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.c_double, C.c_double, C.POINTER(GirihGpuModel)]),
    "girih_gpu_tune": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(GirihGpuConfig), _dp, _ip]),
    "girih_gpu_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "girih_gpu_host_free": (C.c_int, [C.c_void_p]),
    "girih_gpu_interior_checksum": (C.c_int, [C.POINTER(GirihStateView),
                                              C.POINTER(C.c_ulonglong)]),
    "girih_gpu_fp64_peak": (C.c_int, [C.c_int, _dp, _dp]),
    "girih_gpu_device_info": (C.c_int, [C.c_int, _ip, C.c_char_p, C.c_int]),
}

_LIB = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the CUDA library (fails loudly when it has not been built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


class GirihError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(GirihError, ValueError):
    """Maps the reference's std::invalid_argument (GIRIH_EINVAL)."""


def check(rc: int) -> None:
    if rc == GIRIH_OK:
        return
    msg = load().girih_gpu_last_error().decode(errors="replace")
    if rc == GIRIH_EINVAL:
        raise InvalidArgument(rc, msg)
    raise GirihError(rc, msg)
