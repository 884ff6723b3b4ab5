"""ctypes bindings to the CHECKERS under oracle/ (test infrastructure only).

* ``Oracle``  -- oracle/liboracle.so, the plain-C restatement of the reference's
  naive sweep / init / checksum (oracle/girih_oracle.c).
* ``RefLib``  -- oracle/_ref/libgirih_ref.so, the unmodified reference core compiled
  from /root/reference sources (oracle/Makefile) behind oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libgirih_ref.so")

KINDS = ("const7pt", "var7pt", "const25pt", "var25pt")
# proj/src/stencil.cpp:11-17: (R, N_D, flops, time order, coefficient arrays)
TRAITS = {
    0: (1, 2, 7, 1, 0),
    1: (1, 9, 13, 1, 7),
    2: (4, 3, 33, 2, 1),
    3: (4, 15, 37, 1, 13),
}

_dp = C.POINTER(C.c_double)


def _ensure_built(path: str) -> None:
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


@dataclass
class HostState:
    """numpy mirror of girih::ProblemState (proj/include/girih/stencil.hpp:83-98)."""

    kind: int
    nx: int
    ny: int
    nz: int
    pad_x: int
    u: np.ndarray
    v: np.ndarray
    coeffs: list = field(default_factory=list)
    cc: np.ndarray = None
    t_current: int = 0

    @property
    def radius(self) -> int:
        return TRAITS[self.kind][0]

    @property
    def shape(self):
        R = self.radius
        return (self.nz + 2 * R, self.ny + 2 * R, self.nx + 2 * R + self.pad_x)

    def copy(self) -> "HostState":
        return HostState(self.kind, self.nx, self.ny, self.nz, self.pad_x, self.u.copy(),
                         self.v.copy(), [c.copy() for c in self.coeffs], self.cc.copy(),
                         self.t_current)

    def current(self) -> np.ndarray:
        return self.u if self.t_current % 2 == 0 else self.v


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        _ensure_built(path)
        L = C.CDLL(path)
        L.orc_init_value.restype = C.c_double
        L.orc_init_value.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int]
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_init_state.restype = C.c_int
        L.orc_init_state.argtypes = [C.c_int] * 5 + [C.c_uint64, _dp, _dp, C.POINTER(_dp), _dp]
        L.orc_apply_remap.restype = None
        L.orc_apply_remap.argtypes = [C.c_int] * 5 + [_dp, _dp, C.POINTER(_dp), _dp]
        L.orc_naive_sweep.restype = C.c_long
        L.orc_naive_sweep.argtypes = [C.c_int] * 5 + [_dp, _dp, C.POINTER(_dp), _dp, C.c_long,
                                                      C.c_long]
        L.orc_apply_point.restype = C.c_double
        L.orc_apply_point.argtypes = [C.c_int] * 5 + [_dp, _dp, C.POINTER(_dp), _dp, C.c_long,
                                                      C.c_int, C.c_int, C.c_int]
        L.orc_interior_checksum.restype = C.c_uint64
        L.orc_interior_checksum.argtypes = [_dp] + [C.c_int] * 5
        L.orc_fnv_all.restype = C.c_uint64
        L.orc_fnv_all.argtypes = [_dp, C.c_uint64]
        L.orc_row_digest.restype = C.c_uint64
        L.orc_row_digest.argtypes = [_dp, C.c_uint64, C.c_uint64]
        self.L = L

    def init_value(self, seed, field_id, k, j, i) -> float:
        return self.L.orc_init_value(seed, field_id, k, j, i)

    def init_state(self, kind: int, nx: int, ny: int, nz: int, pad_x: int, seed: int,
                   remap: bool = False) -> HostState:
        R, _, _, _, nc = TRAITS[kind]
        shape = (nz + 2 * R, ny + 2 * R, nx + 2 * R + pad_x)
        u = np.empty(shape, np.float64)
        v = np.empty(shape, np.float64)
        coeffs = [np.empty(shape, np.float64) for _ in range(nc)]
        cc = np.zeros(5, np.float64)
        cp = (_dp * max(nc, 1))(*[_ptr(c) for c in coeffs])
        rc = self.L.orc_init_state(kind, nx, ny, nz, pad_x, seed, _ptr(u), _ptr(v), cp, _ptr(cc))
        if rc != 0:
            raise ValueError("grid extent below 2R+1 for stencil radius")
        if remap:
            self.L.orc_apply_remap(kind, nx, ny, nz, pad_x, _ptr(u), _ptr(v), cp, _ptr(cc))
        return HostState(kind, nx, ny, nz, pad_x, u, v, coeffs, cc, 0)

    def naive_sweep(self, s: HostState, steps: int) -> None:
        nc = len(s.coeffs)
        cp = (_dp * max(nc, 1))(*[_ptr(c) for c in s.coeffs])
        t = self.L.orc_naive_sweep(s.kind, s.nx, s.ny, s.nz, s.pad_x, _ptr(s.u), _ptr(s.v), cp,
                                   _ptr(s.cc), s.t_current, steps)
        if t < 0:
            raise ValueError("negative step count")
        s.t_current = t

    def apply_point(self, s: HostState, i: int, j: int, k: int) -> float:
        nc = len(s.coeffs)
        cp = (_dp * max(nc, 1))(*[_ptr(c) for c in s.coeffs])
        return self.L.orc_apply_point(s.kind, s.nx, s.ny, s.nz, s.pad_x, _ptr(s.u), _ptr(s.v), cp,
                                      _ptr(s.cc), s.t_current, i, j, k)

    def interior_checksum(self, s: HostState) -> int:
        return self.L.orc_interior_checksum(_ptr(s.current()), s.nx, s.ny, s.nz, s.pad_x,
                                            s.radius)

    def row_digest(self, a: np.ndarray) -> int:
        """FNV-1a over the per-row FNV-1a hashes of a [Z][Y][X] field (girih_gpu_row_digest)."""
        assert a.dtype == np.float64 and a.flags.c_contiguous and a.ndim == 3
        return self.L.orc_row_digest(_ptr(a), a.shape[0] * a.shape[1], a.shape[2])

    def fnv_all(self, a: np.ndarray) -> int:
        a = np.ascontiguousarray(a)
        return self.L.orc_fnv_all(_ptr(a), a.size)


class RefLib:
    """The reference core itself (oracle/_ref). Raises FileNotFoundError if not built."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            _ensure_built(path)
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_hardware_concurrency.restype = C.c_uint
        L.ref_state_new.restype = C.c_void_p
        L.ref_state_new.argtypes = [C.c_int] * 5 + [C.c_ulonglong]
        L.ref_state_alloc.restype = C.c_void_p
        L.ref_state_alloc.argtypes = [C.c_int] * 5
        L.ref_state_free.argtypes = [C.c_void_p]
        L.ref_state_dims.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 5
        L.ref_state_field.restype = _dp
        L.ref_state_field.argtypes = [C.c_void_p, C.c_int]
        L.ref_state_cc.restype = _dp
        L.ref_state_cc.argtypes = [C.c_void_p]
        L.ref_state_t.restype = C.c_long
        L.ref_state_t.argtypes = [C.c_void_p]
        L.ref_state_set_t.argtypes = [C.c_void_p, C.c_long]
        L.ref_naive_sweep.restype = C.c_int
        L.ref_naive_sweep.argtypes = [C.c_void_p, C.c_long]
        L.ref_run.restype = C.c_int
        L.ref_run.argtypes = [C.c_void_p, C.c_long] + [C.c_int] * 7 + [_dp, _dp]
        L.ref_checksum.restype = C.c_ulonglong
        L.ref_checksum.argtypes = [C.c_void_p]
        L.ref_apply_point.restype = C.c_double
        L.ref_apply_point.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        self.L = L

    def error(self) -> str:
        return self.L.ref_last_error().decode()


class RefState:
    """Owns a reference girih::ProblemState; numpy views alias its std::vector storage."""

    def __init__(self, lib: RefLib, kind: int, nx: int, ny: int, nz: int, pad_x: int, seed: int,
                 oracle_fill: "Oracle" = None, remap: bool = False):
        """seed -> the reference's own init_state; with ``oracle_fill`` the reference allocates
        and the oracle's multi-threaded copy of the same generator fills (bench CPU legs)."""
        self.lib = lib
        if oracle_fill is None:
            self.h = lib.L.ref_state_new(kind, nx, ny, nz, pad_x, seed)
        else:
            self.h = lib.L.ref_state_alloc(kind, nx, ny, nz, pad_x)
        if not self.h:
            raise ValueError(lib.error())
        self.kind, self.nx, self.ny, self.nz, self.pad_x = kind, nx, ny, nz, pad_x
        X, Y, Z, R, nc = (C.c_int() for _ in range(5))
        lib.L.ref_state_dims(self.h, C.byref(X), C.byref(Y), C.byref(Z), C.byref(R), C.byref(nc))
        self.shape = (Z.value, Y.value, X.value)
        self.radius = R.value
        n = Z.value * Y.value * X.value

        def view(p, count, shape):
            return np.ctypeslib.as_array(p, shape=(count,)).reshape(shape)

        self.u = view(lib.L.ref_state_field(self.h, 0), n, self.shape)
        self.v = view(lib.L.ref_state_field(self.h, 1), n, self.shape)
        self.coeffs = [view(lib.L.ref_state_field(self.h, 2 + c), n, self.shape)
                       for c in range(nc.value)]
        self.cc = view(lib.L.ref_state_cc(self.h), 5, (5,))
        if oracle_fill is not None:
            cp = (_dp * max(nc.value, 1))(*[_ptr(c) for c in self.coeffs])
            rc = oracle_fill.L.orc_init_state(kind, nx, ny, nz, pad_x, seed, _ptr(self.u),
                                              _ptr(self.v), cp, _ptr(self.cc))
            if rc != 0:
                raise ValueError("grid extent below 2R+1 for stencil radius")
            if remap:
                self.apply_remap(oracle_fill)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.ref_state_free(self.h)
            self.h = None

    @property
    def t_current(self) -> int:
        return self.lib.L.ref_state_t(self.h)

    @t_current.setter
    def t_current(self, t: int) -> None:
        self.lib.L.ref_state_set_t(self.h, t)

    def naive_sweep(self, steps: int) -> None:
        if self.lib.L.ref_naive_sweep(self.h, steps) != 0:
            raise ValueError(self.lib.error())

    def run(self, steps: int, dw: int, nf: int, tgs=(1, 1, 1), variant: int = 0,
            groups: int = 1):
        wall, glups = C.c_double(), C.c_double()
        rc = self.lib.L.ref_run(self.h, steps, dw, nf, tgs[0], tgs[1], tgs[2], variant, groups,
                                C.byref(wall), C.byref(glups))
        if rc != 0:
            raise ValueError(self.lib.error())
        return wall.value, glups.value

    def checksum(self) -> int:
        return self.lib.L.ref_checksum(self.h)

    def apply_remap(self, oracle: "Oracle") -> None:
        nc = len(self.coeffs)
        cp = (_dp * max(nc, 1))(*[_ptr(c) for c in self.coeffs])
        oracle.L.orc_apply_remap(self.kind, self.nx, self.ny, self.nz, self.pad_x, _ptr(self.u),
                                 _ptr(self.v), cp, _ptr(self.cc))

    def to_host(self) -> HostState:
        return HostState(self.kind, self.nx, self.ny, self.nz, self.pad_x, self.u.copy(),
                         self.v.copy(), [c.copy() for c in self.coeffs], self.cc.copy(),
                         self.t_current)
