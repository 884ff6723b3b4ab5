"""Host-side mirror of the reference's stencil / run interface over the CUDA C ABI.

Names and semantics follow the reference headers so code written against girih reads the same:

* ``traits`` / ``stencil_from_name``  -- proj/include/girih/stencil.hpp:15-27 (stencil.cpp:11-47)
* ``GridSpec``                         -- stencil.hpp:31-44
* ``ProblemState``                     -- stencil.hpp:83-98 (numpy arrays, [k][j][i] layout,
                                          level parity convention u = even, v = odd)
* ``init_state``                       -- stencil.cpp:58-85 (generated ON THE GPU, bit-identical)
* ``run``                              -- engine.hpp:111-115, the drop-in hot path; returns a
                                          ``PerfReport`` (engine.hpp:93-98) extended with GPU fields
* ``interior_checksum``                -- stencil.cpp:129-146
* ``DeviceState``                      -- a device-resident state (open / step / download / tune)

Errors: ``InvalidArgument`` (a ``ValueError``) wherever the reference throws
``std::invalid_argument``; ``GirihError`` for CUDA/NCCL/OOM failures.
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import (GIRIH_TRACE_FN, GirihGpuConfig, GirihGpuReport, GirihGpuRunOptions, GirihGpuVariant, GirihStateView, InvalidArgument,
                   check, load)

KINDS = ("const7pt", "var7pt", "const25pt", "var25pt")
CONST7PT, VAR7PT, CONST25PT, VAR25PT = range(4)


@dataclass(frozen=True)
class StencilTraits:
    name: str
    radius: int
    domain_streams: int
    flops_per_lup: int
    time_order: int
    coeff_arrays: int


def traits(kind: int) -> StencilTraits:
    r, nd, fl, to, nc = (C.c_int() for _ in range(5))
    check(load().girih_gpu_traits(int(kind), C.byref(r), C.byref(nd), C.byref(fl), C.byref(to),
                                  C.byref(nc)))
    return StencilTraits(KINDS[kind], r.value, nd.value, fl.value, to.value, nc.value)


def stencil_from_name(name: str) -> int:
    k = C.c_int()
    check(load().girih_gpu_kind_from_name(name.encode(), C.byref(k)))
    return k.value


@dataclass(frozen=True)
class GridSpec:
    nx: int
    ny: int
    nz: int
    pad_x: int = 0
    element_bytes: int = 8

    def x_alloc(self, radius: int) -> int:
        return self.nx + 2 * radius + self.pad_x

    def leading_dim_bytes(self, radius: int) -> int:
        return self.x_alloc(radius) * self.element_bytes


@dataclass
class ProblemState:
    kind: int
    grid: GridSpec
    u: np.ndarray
    v: np.ndarray
    coeffs: List[np.ndarray] = field(default_factory=list)
    cc: np.ndarray = field(default_factory=lambda: np.zeros(5))
    t_current: int = 0

    @property
    def radius(self) -> int:
        return traits(self.kind).radius

    def level(self, t: int) -> np.ndarray:
        return self.u if t % 2 == 0 else self.v

    def current(self) -> np.ndarray:
        return self.level(self.t_current)

    def shape(self):
        R = self.radius
        g = self.grid
        return (g.nz + 2 * R, g.ny + 2 * R, g.x_alloc(R))


@dataclass
class GpuConfig:
    """Execution parameters replacing the CPU engine's (dw, wf, shape, variant, n_groups)."""

    tb: int = 0          # time steps fused per HBM pass (0 = default for the kind)
    variant: int = -1    # compiled kernel variant (-1 = default for tb)
    zchunks: int = 0     # z chunks per tile column (0 = wave-quantisation model)
    ngpus: int = 1       # z-slab decomposition over devices
    device: int = 0
    graphs: int = 0
    emulate_slabs: int = 0  # >1: that many z-slabs on ONE device (decomposition tests)
    chain: int = 0       # 1: chain same-depth passes into one dependency-driven launch; -1: off;
                         # 0: auto (grids <= 256^3 cells, not var7pt)
    tile_order: int = 0  # W > 0: column strips of W tiles inside a z-chunk row; -1: row-major;
                         # 0: auto (strips of 8 for var7pt two-step passes, >= 17 tile columns)

    def to_c(self) -> GirihGpuConfig:
        return GirihGpuConfig(self.tb, self.variant, self.zchunks, self.ngpus, 1, self.device,
                              self.graphs, self.emulate_slabs, self.chain, self.tile_order)


@dataclass
class PerfReport:
    wall_seconds: float
    kernel_seconds: float
    lups: int
    glups: float
    mlups: float
    h2d_seconds: float = 0.0
    d2h_seconds: float = 0.0
    model_bytes_per_lup: float = 0.0
    tb_used: int = 0
    n_launches: int = 0
    pass_seconds: float = 0.0
    computed_lups: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    variant_used: int = -1
    zchunks_used: int = 0
    grid_ctas: int = 0
    streamed: int = 0  # girih_gpu_run pipelined the copies with the passes along z
    n_passes: int = 0  # stencil passes (a chained launch runs several)
    units: int = 0     # work units (tile column x z chunk per pass): PerfReport::tiles

    @staticmethod
    def from_c(r: GirihGpuReport) -> "PerfReport":
        return PerfReport(r.wall_s, r.kernel_s, r.lups, r.mlups / 1e3, r.mlups, r.h2d_s, r.d2h_s,
                          r.model_bytes_per_lup, r.tb_used, r.n_launches, r.pass_s,
                          r.computed_lups, r.h2d_bytes, r.d2h_bytes, r.variant_used,
                          r.zchunks_used, r.grid_ctas, r.streamed, r.n_passes, r.units)


def variants():
    lib = load()
    out = []
    for i in range(lib.girih_gpu_variant_count()):
        v = GirihGpuVariant()
        check(lib.girih_gpu_variant_info(i, C.byref(v)))
        out.append(dict(index=i, kind=v.kind, tb=v.tb, lx=v.lx, ly=v.ly, threads=v.threads,
                        prefetch=v.prefetch, smem_bytes=v.smem_bytes, cluster_y=v.cluster_y,
                        aux_prefetch=v.aux_prefetch, direct_out=v.direct_out,
                        paced=v.paced, narrow=v.narrow))
    return out


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _check_array(a: np.ndarray, shape, name: str) -> None:
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous:
        raise InvalidArgument(_lib.GIRIH_EINVAL, f"{name} must be a C-contiguous float64 array")
    if a.size != int(np.prod(shape)):
        raise InvalidArgument(_lib.GIRIH_EINVAL, f"{name} has the wrong size")


class _View:
    """Keeps a GirihStateView and the ctypes arrays it points into alive."""

    def __init__(self, s: ProblemState, need_coeffs: bool = True):
        shape = s.shape()
        _check_array(s.u, shape, "u")
        _check_array(s.v, shape, "v")
        nc = traits(s.kind).coeff_arrays
        if need_coeffs:
            if len(s.coeffs) != nc:
                raise InvalidArgument(_lib.GIRIH_EINVAL, "coefficient field count does not match kind")
            for i, c in enumerate(s.coeffs):
                _check_array(c, shape, f"coeffs[{i}]")
        self.cptrs = (C.POINTER(C.c_double) * max(nc, 1))(*[_dptr(c) for c in s.coeffs])
        g = s.grid
        self.view = GirihStateView(s.kind, g.nx, g.ny, g.nz, g.pad_x, int(s.t_current), _dptr(s.u),
                                   _dptr(s.v), C.cast(self.cptrs, C.POINTER(C.POINTER(C.c_double))),
                                   len(s.coeffs), (C.c_double * 5)(*[float(x) for x in s.cc]))


def run(state: ProblemState, steps: int, config: Optional[GpuConfig] = None) -> PerfReport:
    """Advance ``state`` by ``steps`` on the GPU: the drop-in for girih::run (engine.cpp:332-418).

    Host arrays are uploaded, advanced, and both solution fields downloaded (the timed wall
    includes the copies; ``kernel_seconds`` is the device-resident part)."""
    cfg = (config or GpuConfig()).to_c()
    v = _View(state)
    rep = GirihGpuReport()
    check(load().girih_gpu_run(C.byref(v.view), int(steps), C.byref(cfg), C.byref(rep)))
    state.t_current = v.view.t_current
    return PerfReport.from_c(rep)


def interior_checksum(state: ProblemState) -> int:
    v = _View(state, need_coeffs=False)
    out = C.c_ulonglong()
    check(load().girih_gpu_interior_checksum(C.byref(v.view), C.byref(out)))
    return out.value


def plan(kind: int, t0: int, steps: int, tb: int):
    """The host pass planner: list of (tb, src, src_prev, dst, dst_penult) buffer ids
    (0 = u, 1 = v, 2 = even scratch, 3 = odd scratch, -1 = none)."""
    lib = load()
    n = C.c_int()
    cap = int(steps) + 8
    arrs = [(C.c_int * cap)() for _ in range(5)]
    check(lib.girih_gpu_plan(int(kind), int(t0), int(steps), int(tb), cap, C.byref(n), *arrs))
    return [tuple(a[i] for a in arrs) for i in range(n.value)]


def run_instrumented(state: ProblemState, steps: int, config: Optional[GpuConfig] = None,
                     trace: bool = True, ledger: bool = True):
    """girih_gpu_run_ex: the drop-in call with the reference's RunOptions instrumentation
    (engine.hpp:100-103). Returns (report, trace, ledger): `trace` a structured array of
    per-unit records (pass, unit, cta, sm, start_ns, end_ns), sorted by (pass, unit); `ledger`
    the [steps][nz][ny][nx] counts of owned cell updates (all 1 when the run covered every cell
    update exactly once)."""
    config = config or GpuConfig()
    cfg = config.to_c()
    rep = GirihGpuReport()
    v = _View(state)
    opts = GirihGpuRunOptions()
    recs = []

    def collect(_ctx, ptr, n):
        for i in range(n):
            r = ptr[i]
            recs.append((r.pass_, r.unit, r.cta, r.sm, r.start_ns, r.end_ns))

    cb = GIRIH_TRACE_FN(collect)
    if trace:
        opts.trace_cb = cb
    led = None
    if ledger and steps > 0:
        led = np.zeros((steps, state.grid.nz, state.grid.ny, state.grid.nx), dtype=np.uint32)
        opts.ledger = led.ctypes.data_as(C.POINTER(C.c_uint))
    check(load().girih_gpu_run_ex(C.byref(v.view), int(steps), C.byref(cfg), C.byref(rep),
                                  C.byref(opts)))
    state.t_current = v.view.t_current
    dt = np.dtype([("pass", "i4"), ("unit", "i4"), ("cta", "i4"), ("sm", "i4"),
                   ("start_ns", "u8"), ("end_ns", "u8")])
    return PerfReport.from_c(rep), np.array(recs, dtype=dt), led


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for girih_gpu_open_slab_seeded (call on rank 0, broadcast)."""
    buf = C.create_string_buffer(128)
    check(load().girih_gpu_nccl_unique_id(buf, 128))
    return buf.raw


def slab_layout(kind: int, nz: int, nslabs: int, g: int):
    """(z0, z1, hz): interior planes [z0, z1) of slab g and its halo depth (multi-GPU z-slabs)."""
    z0, z1, hz = C.c_int(), C.c_int(), C.c_int()
    check(load().girih_gpu_slab_layout(int(kind), int(nz), int(nslabs), int(g), C.byref(z0),
                                       C.byref(z1), C.byref(hz)))
    return z0.value, z1.value, hz.value


def model(kind: int, grid: "GridSpec", tb: int = 0, variant: int = -1, hbm_gbs: float = 0.0,
          fp64_ops: float = 0.0) -> dict:
    """GPU analogue of the reference's analytic models (proj/src/models.cpp:12-84): tile geometry,
    shared memory per CTA, redundancy, code balance and roofline of one configuration (host-only;
    see girih_gpu_model in include/girih_gpu.h)."""
    from ._lib import GirihGpuModel
    out = GirihGpuModel()
    check(load().girih_gpu_model(int(kind), grid.nx, grid.ny, grid.nz, int(tb), int(variant),
                                 float(hbm_gbs), float(fp64_ops), C.byref(out)))
    return {name: getattr(out, name) for name, _ in GirihGpuModel._fields_}


def trim() -> None:
    """Release device memory cached between handles (girih_gpu_trim)."""
    check(load().girih_gpu_trim())


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """A numpy array in page-locked host memory (freed when the array is collected)."""
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    p = C.c_void_p()
    check(load().girih_gpu_host_alloc(max(nbytes, 8), C.byref(p)))
    buf = (C.c_byte * max(nbytes, 8)).from_address(p.value)
    arr = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)
    lib = load()
    addr = p.value
    weakref.finalize(buf, lambda: lib.girih_gpu_host_free(C.c_void_p(addr)))
    return arr  # arr.base -> buf keeps the page-locked allocation alive


class DeviceState:
    """A device-resident ProblemState (the handle of include/girih_gpu.h)."""

    def __init__(self, handle: C.c_void_p, kind: int, grid: GridSpec, config: GpuConfig):
        self._h = handle
        self.kind = kind
        self.grid = grid
        self.config = config

    @classmethod
    def from_state(cls, state: ProblemState, config: Optional[GpuConfig] = None) -> "DeviceState":
        config = config or GpuConfig()
        cfg = config.to_c()
        v = _View(state)
        h = C.c_void_p()
        check(load().girih_gpu_open(C.byref(v.view), C.byref(cfg), C.byref(h)))
        return cls(h, state.kind, state.grid, config)

    @classmethod
    def seeded(cls, kind: int, grid: GridSpec, seed: int, remap: bool = False,
               config: Optional[GpuConfig] = None) -> "DeviceState":
        config = config or GpuConfig()
        cfg = config.to_c()
        h = C.c_void_p()
        check(load().girih_gpu_open_seeded(int(kind), grid.nx, grid.ny, grid.nz, grid.pad_x,
                                           int(seed), int(bool(remap)), C.byref(cfg), C.byref(h)))
        return cls(h, kind, grid, config)

    @classmethod
    def slab_seeded(cls, kind: int, grid: GridSpec, seed: int, remap: bool, rank: int, nranks: int,
                    nccl_id: Optional[bytes], config: Optional[GpuConfig] = None) -> "DeviceState":
        """This process's z-slab `rank` of `nranks` of the global grid (one process per GPU).
        With `nccl_id` (from nccl_unique_id() on rank 0) halos move over NCCL after every pass;
        with None the passes push them into the neighbours' memory: call ipc_export(), hand the
        blobs to the z neighbours, ipc_connect() and barrier before the first step."""
        config = config or GpuConfig()
        cfg = config.to_c()
        h = C.c_void_p()
        idbuf = (C.create_string_buffer(bytes(nccl_id), max(len(nccl_id), 128))
                 if nccl_id is not None else None)
        check(load().girih_gpu_open_slab_seeded(int(kind), grid.nx, grid.ny, grid.nz, grid.pad_x,
                                                int(seed), int(bool(remap)), int(rank), int(nranks),
                                                idbuf, C.byref(cfg), C.byref(h)))
        return cls(h, kind, grid, config)

    def ipc_export(self) -> bytes:
        """This slab's IPC blob (buffers + pass flags) for its z neighbours."""
        buf = C.create_string_buffer(_lib.GIRIH_GPU_IPC_BYTES)
        check(load().girih_gpu_ipc_export(self._handle(), buf, _lib.GIRIH_GPU_IPC_BYTES))
        return buf.raw

    def ipc_connect(self, lower: Optional[bytes], upper: Optional[bytes]) -> None:
        """Map the z neighbours' blobs (None where there is no neighbour)."""
        check(load().girih_gpu_ipc_connect(self._handle(), lower, upper))

    def _handle(self):
        if self._h is None or not self._h.value:
            raise _lib.GirihError(_lib.GIRIH_ESTATE, "device state is closed")
        return self._h

    def step(self, steps: int) -> PerfReport:
        rep = GirihGpuReport()
        check(load().girih_gpu_step(self._handle(), int(steps), C.byref(rep)))
        return PerfReport.from_c(rep)

    @property
    def t_current(self) -> int:
        t = C.c_longlong()
        check(load().girih_gpu_get_t(self._handle(), C.byref(t)))
        return t.value

    def set_config(self, config: GpuConfig) -> None:
        cfg = config.to_c()
        check(load().girih_gpu_set_config(self._handle(), C.byref(cfg)))
        self.config = config

    def empty_state(self, pinned: bool = False) -> ProblemState:
        R = traits(self.kind).radius
        g = self.grid
        shape = (g.nz + 2 * R, g.ny + 2 * R, g.x_alloc(R))
        alloc = pinned_empty if pinned else (lambda s: np.empty(s, np.float64))
        nc = traits(self.kind).coeff_arrays
        return ProblemState(self.kind, g, alloc(shape), alloc(shape), [alloc(shape) for _ in range(nc)],
                            np.zeros(5), 0)

    def download(self, state: Optional[ProblemState] = None, coeffs: bool = True,
                 pinned: bool = False) -> ProblemState:
        if state is None:
            state = self.empty_state(pinned=pinned)
        v = _View(state, need_coeffs=False)
        check(load().girih_gpu_download(self._handle(), C.byref(v.view)))
        state.t_current = v.view.t_current
        state.cc = np.array(list(v.view.cc), dtype=np.float64)
        if coeffs and state.coeffs:
            ptrs = (C.POINTER(C.c_double) * len(state.coeffs))(*[_dptr(c) for c in state.coeffs])
            check(load().girih_gpu_download_coeffs(self._handle(), ptrs, len(state.coeffs), None))
        return state

    def compare(self, field, host: np.ndarray):
        """Bitwise compare of a device field ('u', 'v' or coefficient index c) with a host array
        of the full allocated grid, on the device (girih_gpu_compare). Returns (n_diff, first)
        with first = (i, j, k) of the lowest differing cell or None."""
        f = {"u": 0, "v": 1}[field] if isinstance(field, str) else 2 + int(field)
        arr = np.ascontiguousarray(host, dtype=np.float64)
        n, first = C.c_longlong(), C.c_longlong()
        check(load().girih_gpu_compare(self._handle(), f, _dptr(arr), C.byref(n), C.byref(first)))
        if n.value == 0:
            return 0, None
        k, rem = divmod(first.value, arr.shape[1] * arr.shape[2])
        j, i = divmod(rem, arr.shape[2])
        return n.value, (i, j, k)

    def update_units(self, steps: int, begin: int, end: int) -> int:
        """update_tile (engine.cpp:294-330): runs work units [begin, end) -- numbered pass-major
        over the plan that advances the state by `steps` -- (girih_gpu_update_units); the state
        advances once every unit has run. Returns the plan's unit count."""
        n = C.c_longlong()
        check(load().girih_gpu_update_units(self._handle(), int(steps), int(begin), int(end),
                                            C.byref(n)))
        return n.value

    def row_digest(self, field) -> int:
        """Device-side digest of a whole field ('u', 'v' or coefficient index c), ghosts and pad
        included: FNV-1a over the per-row FNV-1a hashes (girih_gpu_row_digest)."""
        f = {"u": 0, "v": 1}[field] if isinstance(field, str) else 2 + int(field)
        d = C.c_ulonglong()
        check(load().girih_gpu_row_digest(self._handle(), f, C.byref(d)))
        return d.value

    def upload(self, state: ProblemState) -> None:
        v = _View(state)
        check(load().girih_gpu_upload(self._handle(), C.byref(v.view)))

    def tune(self, max_tb: int = 0):
        best = GirihGpuConfig()
        mlups = C.c_double()
        n = C.c_int()
        check(load().girih_gpu_tune(self._handle(), int(max_tb), C.byref(best), C.byref(mlups),
                                    C.byref(n)))
        cfg = GpuConfig(best.tb, best.variant, best.zchunks, best.ngpus, best.device, best.graphs,
                        best.reserved, best.chain, best.tile_order)
        return cfg, mlups.value, n.value

    def close(self) -> None:
        if self._h is not None and self._h.value:
            check(load().girih_gpu_close(self._h))
        self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def init_state(kind: int, grid: GridSpec, seed: int, remap: bool = False,
               config: Optional[GpuConfig] = None) -> ProblemState:
    """init_state (stencil.cpp:58-85), generated on the device and downloaded."""
    with DeviceState.seeded(kind, grid, seed, remap, config) as ds:
        return ds.download()


def fp64_peak(device: int = 0):
    """Measured FP64 rates: (separate DADD/DMUL ops/s, DFMA flops/s)."""
    a, f = C.c_double(), C.c_double()
    check(load().girih_gpu_fp64_peak(int(device), C.byref(a), C.byref(f)))
    return a.value, f.value


def device_info(device: int = 0):
    n = C.c_int()
    name = C.create_string_buffer(256)
    check(load().girih_gpu_device_info(int(device), C.byref(n), name, 256))
    return n.value, name.value.decode()
