"""Thin ctypes binding of libspin (include/spin.h) — argument marshalling only.

Every step of the spin-image path runs inside libspin's sm_100a kernels; this module
converts tensors / arrays to pointers and statuses to exceptions.  There is no CPU
fallback: if libspin.so is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPIN_LIB_PATH") or os.path.join(_HERE, "libspin.so")  # override: A/B builds
if not os.path.exists(LIB_PATH):
    raise ImportError(f"libspin.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")
_lib = C.CDLL(LIB_PATH)

STATIC, SS, GSS, FAC, WF, AWF = 0, 1, 2, 3, 4, 5
NEAREST, BILINEAR = 0, 1
BRUTE, CELLS = 0, 1
F_LITERAL_HALF_WIDTH, F_FLOOR_BINS, F_NO_SORT, F_NO_FAST_CERT, F_SUPPORT_LAST = 0x1, 0x2, 0x4, 0x8, 0x10
F_SUPPORT_FIRST, F_CLUSTER_PAIR, F_NO_DENSE = 0x20, 0x40, 0x80
SCHEDULES = {"STATIC": STATIC, "SS": SS, "GSS": GSS, "FAC": FAC, "WF": WF, "AWF": AWF}
MODES = {"nearest": NEAREST, "bilinear": BILINEAR}
PRUNES = {"brute": BRUTE, "cells": CELLS}
STATUS = {0: "SPIN_OK", 1: "SPIN_E_INVAL", 2: "SPIN_E_RANGE", 3: "SPIN_E_INPUT",
          4: "SPIN_E_NOMEM", 5: "SPIN_E_CUDA", 6: "SPIN_E_OVERFLOW"}


class ChunkParams(C.Structure):
    _fields_ = [("P", C.c_int32), ("unit", C.c_int32), ("gss_min_chunk", C.c_int32),
                ("fac_divisor", C.c_int32), ("flags", C.c_uint32),
                ("slow_ctas", C.c_int32), ("slowdown", C.c_float), ("slow_first", C.c_int32),
                ("grid", C.c_int32), ("cta_offset", C.c_int32), ("d_counter", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("elapsed_ms", C.c_double), ("grid_build_ms", C.c_double),
                ("pairs_visited", C.c_int64), ("pairs_candidate", C.c_int64),
                ("pairs_accepted", C.c_int64), ("fp64_fallbacks", C.c_int64),
                ("exact_fallbacks", C.c_int64), ("P", C.c_int32), ("G", C.c_int32),
                ("n_units", C.c_int32), ("n_chunks", C.c_int32),
                ("h_cta_start_ns", C.POINTER(C.c_uint64)), ("h_cta_end_ns", C.POINTER(C.c_uint64)),
                ("h_cta_units", C.POINTER(C.c_int32)), ("cta_capacity", C.c_int32),
                ("tiles_support_hot", C.c_int64), ("filter_mma", C.c_int32),
                ("cta_per_worker", C.c_int32), ("tiles_dense", C.c_int64),
                ("dense_rows", C.c_int64)]


_vp = C.c_void_p
_lib.spin_create.argtypes = [_vp, _vp, C.c_int64, _vp, C.POINTER(_vp)]
_lib.spin_load_cloud.argtypes = [_vp, _vp, _vp, C.c_int64, _vp]
_lib.spin_generate.argtypes = [_vp, _vp, C.c_int64, C.c_int32, C.c_double, C.c_double, C.c_int,
                               C.POINTER(ChunkParams), C.c_int, C.c_int, _vp, C.POINTER(Stats), _vp]
_lib.spin_generate_host.argtypes = _lib.spin_generate.argtypes
_lib.spin_chunk_sequence.argtypes = [C.c_int, C.c_int64, C.c_int32, C.POINTER(ChunkParams),
                                     C.POINTER(C.c_int64), C.c_int64, C.POINTER(C.c_int64)]
_lib.spin_region_radius.argtypes = [C.c_int32, C.c_double, C.c_int, C.c_uint32]
_lib.spin_region_radius.restype = C.c_double
_lib.spin_cos_from_degrees.argtypes = [C.c_double]
_lib.spin_cos_from_degrees.restype = C.c_double
_lib.spin_default_P.argtypes = [C.c_int32, C.c_int, C.c_int]
_lib.spin_default_P.restype = C.c_int32
_lib.spin_destroy.argtypes = [_vp]
_lib.spin_last_error.restype = C.c_char_p
_lib.spin_abi_version.restype = C.c_int32
for _f in ("spin_create", "spin_load_cloud", "spin_generate", "spin_generate_host", "spin_chunk_sequence"):
    getattr(_lib, _f).restype = C.c_int

_lib.spin_read_xyzn.argtypes = [C.c_char_p, _vp, _vp, C.c_int64, C.POINTER(C.c_int64)]
_lib.spin_read_off.argtypes = [C.c_char_p, _vp, C.c_int64, _vp, C.c_int64,
                               C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
_lib.spin_vertex_normals.argtypes = [_vp, C.c_int64, _vp, C.c_int64, _vp]
for _f in ("spin_read_xyzn", "spin_read_off", "spin_vertex_normals"):
    getattr(_lib, _f).restype = C.c_int

_lib.spin_dealer_alloc.argtypes = [C.POINTER(_vp)]
_lib.spin_dealer_ipc_handle.argtypes = [_vp, C.c_char_p]
_lib.spin_dealer_ipc_open.argtypes = [C.c_char_p, C.POINTER(_vp)]
_lib.spin_dealer_reset.argtypes = [_vp, _vp]
_lib.spin_dealer_free.argtypes = [_vp, C.c_int32]
for _f in ("spin_dealer_alloc", "spin_dealer_ipc_handle", "spin_dealer_ipc_open",
           "spin_dealer_reset", "spin_dealer_free"):
    getattr(_lib, _f).restype = C.c_int


class Dealer:
    """A shared dealer counter (spin_dealer_*): `Dealer()` allocates one on the current
    device; `Dealer.open(handle)` maps another process's through CUDA IPC.  `.ptr` is the
    device address to pass as generate(shared_counter=...)."""

    def __init__(self, _ptr=None, _opened=False):
        if _ptr is None:
            p = _vp()
            _check(_lib.spin_dealer_alloc(C.byref(p)))
            _ptr = p.value
        self.ptr, self._opened = _ptr, _opened

    @classmethod
    def open(cls, handle: bytes):
        p = _vp()
        _check(_lib.spin_dealer_ipc_open(C.create_string_buffer(bytes(handle), 64), C.byref(p)))
        return cls(p.value, True)

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        _check(_lib.spin_dealer_ipc_handle(self.ptr, buf))
        return buf.raw

    def reset(self, stream=None):
        _check(_lib.spin_dealer_reset(self.ptr, _stream(stream)))

    def close(self):
        if self.ptr:
            _check(_lib.spin_dealer_free(self.ptr, int(self._opened)))
            self.ptr = None


_lib.spin_count_in_sphere.argtypes = [_vp, _vp, C.c_int64, C.c_double, C.POINTER(C.c_int64), _vp]
_lib.spin_count_in_sphere.restype = C.c_int
_lib.spin_pair_codes.argtypes = [_vp, _vp, C.c_int64, C.c_int32, C.c_double, C.c_double, C.c_int,
                                 C.c_uint32, _vp, _vp]
_lib.spin_pair_codes.restype = C.c_int

EXPORTS = ["spin_create", "spin_load_cloud", "spin_generate", "spin_generate_host",
           "spin_chunk_sequence", "spin_region_radius", "spin_cos_from_degrees", "spin_default_P",
           "spin_destroy", "spin_last_error", "spin_abi_version",
           "spin_read_xyzn", "spin_read_off", "spin_vertex_normals",
           "spin_dealer_alloc", "spin_dealer_ipc_handle", "spin_dealer_ipc_open",
           "spin_dealer_reset", "spin_dealer_free", "spin_count_in_sphere", "spin_pair_codes"]


def read_xyzn(path):
    """spin_read_xyzn: (points fp32 [N,3], unit normals fp32 [N,3]) in file order."""
    n = C.c_int64()
    _check(_lib.spin_read_xyzn(os.fsencode(path), None, None, 0, C.byref(n)))
    P = np.empty((n.value, 3), np.float32)
    Nn = np.empty((n.value, 3), np.float32)
    _check(_lib.spin_read_xyzn(os.fsencode(path), P.ctypes.data, Nn.ctypes.data, n.value, C.byref(n)))
    return P, Nn


def read_off(path):
    """spin_read_off: (vertices fp32 [nv,3], triangles int32 [nf,3])."""
    nv, nf = C.c_int64(), C.c_int64()
    _check(_lib.spin_read_off(os.fsencode(path), None, 0, None, 0, C.byref(nv), C.byref(nf)))
    V = np.empty((nv.value, 3), np.float32)
    F = np.empty((nf.value, 3), np.int32)
    _check(_lib.spin_read_off(os.fsencode(path), V.ctypes.data, nv.value, F.ctypes.data, nf.value,
                              C.byref(nv), C.byref(nf)))
    return V, F


def vertex_normals(V, F):
    """spin_vertex_normals: area-weighted unit vertex normals fp32 [nv,3]."""
    V = np.ascontiguousarray(V, np.float32)
    F = np.ascontiguousarray(F, np.int32)
    out = np.empty_like(V)
    _check(_lib.spin_vertex_normals(V.ctypes.data, len(V), F.ctypes.data if len(F) else None,
                                    len(F), out.ctypes.data))
    return out


def load_mesh_cloud(path):
    """An oriented point cloud from an OFF mesh: its vertices with area-weighted normals."""
    V, F = read_off(path)
    return V, vertex_normals(V, F)


class SpinError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(st: int):
    if st != 0:
        raise SpinError(st, (_lib.spin_last_error() or b"").decode())


def _enum(v, table):
    return table[v] if isinstance(v, str) else int(v)


def _ptr(t):
    """Device or host pointer of a torch tensor or numpy array (must be contiguous)."""
    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return t.ctypes.data
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


def _dtype_name(t):
    return str(t.dtype).replace("torch.", "")


def _check_array(t, what, dtype, shape, device=None):
    """Refuse (ValueError) anything but a contiguous `dtype` array of `shape` — no silent
    casts: a float64 cloud or a short output buffer would be reinterpreted or overrun."""
    if _dtype_name(t) != dtype:
        raise ValueError(f"{what} must be {dtype}, got {_dtype_name(t)}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{what} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if device is not None:
        on_dev = (not isinstance(t, np.ndarray)) and t.is_cuda
        if device == "host" and on_dev:
            raise ValueError(f"{what} must be host memory")
        if device != "host" and (not on_dev or t.device != device):
            raise ValueError(f"{what} must be on {device}")
    _ptr(t)


def _check_cloud(points, normals):
    n = int(points.shape[0]) if len(points.shape) == 2 else -1
    _check_array(points, "points", "float32", (n, 3))
    _check_array(normals, "normals", "float32", (n, 3))
    return n


def _stream(stream):
    if stream is None:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_stream().cuda_stream
        return None
    return getattr(stream, "cuda_stream", stream)


def abi_version() -> int:
    return _lib.spin_abi_version()


def cos_from_degrees(deg: float) -> float:
    return _lib.spin_cos_from_degrees(float(deg))


def region_radius(W: int, b: float, mode="nearest", flags: int = 0) -> float:
    return _lib.spin_region_radius(int(W), float(b), _enum(mode, MODES), int(flags))


def default_P(W: int, mode="nearest", prune="brute") -> int:
    return _lib.spin_default_P(int(W), _enum(mode, MODES), _enum(prune, PRUNES))


def chunk_sequence(schedule, n_units: int, P: int, gss_min_chunk: int = 0, fac_divisor: int = 0,
                   slow_ctas: int = 0, slowdown: float = 0.0):
    """Chunk boundaries [0, b1, ..., n_units] of a schedule (host-only; spin_chunk_sequence;
    WF with requests in round-robin worker order and the emulation's weights)."""
    cp = ChunkParams(0, 0, gss_min_chunk, fac_divisor, 0)
    cp.slow_ctas = slow_ctas
    cp.slowdown = slowdown
    n = C.c_int64(0)
    st = _lib.spin_chunk_sequence(_enum(schedule, SCHEDULES), n_units, P, C.byref(cp), None, 0, C.byref(n))
    if st not in (0, 2):
        _check(st)
    buf = (C.c_int64 * (n.value + 1))()
    _check(_lib.spin_chunk_sequence(_enum(schedule, SCHEDULES), n_units, P, C.byref(cp), buf,
                                    n.value + 1, C.byref(n)))
    return list(buf)


def _stats_dict(s: Stats, t0=None, t1=None, un=None):
    d = {f: getattr(s, f) for f, _ in Stats._fields_ if not f.startswith("h_cta") and f != "cta_capacity"}
    if t0 is not None:
        d["cta_start_ns"] = np.asarray(t0)
        d["cta_end_ns"] = np.asarray(t1)
        d["cta_units"] = np.asarray(un)
    return d


class SpinEngine:
    """A libspin handle: the oriented point cloud resident in HBM (spin_create)."""

    def __init__(self, points, normals, stream=None):
        n = _check_cloud(points, normals)
        h = _vp()
        _check(_lib.spin_create(_ptr(points), _ptr(normals), n, _stream(stream), C.byref(h)))
        self._h = h
        self.N = n

    def close(self):
        if getattr(self, "_h", None):
            _lib.spin_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_cloud(self, points, normals, stream=None):
        n = _check_cloud(points, normals)
        _check(_lib.spin_load_cloud(self._h, _ptr(points), _ptr(normals), n, _stream(stream)))
        self.N = n

    @staticmethod
    def _params(P, unit, gss_min_chunk, fac_divisor, flags, slow_ctas=0, slowdown=0.0,
                slow_first=False, grid=0, cta_offset=0, d_counter=None):
        return ChunkParams(int(P), int(unit), int(gss_min_chunk), int(fac_divisor), int(flags),
                           int(slow_ctas), float(slowdown), int(bool(slow_first)), int(grid),
                           int(cta_offset), d_counter)

    def generate(self, centre_idx, W, b, cos_As, schedule="STATIC", mode="nearest", prune="brute",
                 P=0, unit=0, gss_min_chunk=0, fac_divisor=0, flags=0, out=None, stats=False,
                 cta_capacity=0, stream=None, slow_ctas=0, slowdown=0.0, slow_first=False,
                 grid=0, cta_offset=0, shared_counter=None):
        """Images for device int32 centre_idx [M] into a device fp32 [M, W, W] tensor.
        schedule: STATIC / SS / GSS / FAC (the paper's), WF / AWF (weighted factoring; the
        WF weights come from the slow-worker emulation below).
        slow_ctas / slowdown / slow_first: heterogeneous-worker emulation (timing only).
        grid / cta_offset / shared_counter (device address of a zeroed u32): one schedule
        dealt across devices; only this device's chunks are written to `out`."""
        import torch
        M = int(centre_idx.shape[0])
        if isinstance(centre_idx, np.ndarray) or not centre_idx.is_cuda:
            raise ValueError("centre_idx must be a CUDA tensor (generate_host takes host arrays)")
        _check_array(centre_idx, "centre_idx", "int32", (M,))
        if out is None:
            out = torch.empty((M, W, W), dtype=torch.float32, device=centre_idx.device)
        _check_array(out, "out", "float32", (M, W, W), centre_idx.device)
        cp = self._params(P, unit, gss_min_chunk, fac_divisor, flags, slow_ctas, slowdown, slow_first,
                          grid, cta_offset, shared_counter)
        st = Stats()
        t0 = t1 = un = None
        if stats and cta_capacity:
            t0 = (C.c_uint64 * cta_capacity)()
            t1 = (C.c_uint64 * cta_capacity)()
            un = (C.c_int32 * cta_capacity)()
            st.h_cta_start_ns = C.cast(t0, C.POINTER(C.c_uint64))
            st.h_cta_end_ns = C.cast(t1, C.POINTER(C.c_uint64))
            st.h_cta_units = C.cast(un, C.POINTER(C.c_int32))
            st.cta_capacity = cta_capacity
        _check(_lib.spin_generate(self._h, _ptr(centre_idx) if M else None, M, int(W), float(b),
                                  float(cos_As), _enum(schedule, SCHEDULES), C.byref(cp),
                                  _enum(mode, MODES), _enum(prune, PRUNES),
                                  _ptr(out) if M else None, C.byref(st) if stats else None,
                                  _stream(stream)))
        if stats:
            return out, _stats_dict(st, t0, t1, un)
        return out

    def count_in_sphere(self, centre_idx, R, stream=None) -> int:
        """spin_count_in_sphere: sum over device int32 centres of #{x : |x - p| <= R}."""
        n = C.c_int64()
        M = int(centre_idx.shape[0])
        _check(_lib.spin_count_in_sphere(self._h, _ptr(centre_idx) if M else None, M, float(R),
                                         C.byref(n), _stream(stream)))
        return n.value

    def pair_codes(self, centre_idx, W, b, cos_As, mode="nearest", flags=0, out=None, stream=None):
        """spin_pair_codes (diagnostic): int32 [M, N] device codes of every (centre, point)
        pair — -1 or the pair's bin (NEAREST k*W+l, BILINEAR i0*W+j0) as the accept path
        decides it."""
        import torch
        M = int(centre_idx.shape[0])
        if isinstance(centre_idx, np.ndarray) or not centre_idx.is_cuda:
            raise ValueError("centre_idx must be a CUDA tensor")
        _check_array(centre_idx, "centre_idx", "int32", (M,))
        if out is None:
            out = torch.empty((M, self.N), dtype=torch.int32, device=centre_idx.device)
        _check_array(out, "out", "int32", (M, self.N), centre_idx.device)
        _check(_lib.spin_pair_codes(self._h, _ptr(centre_idx) if M else None, M, int(W), float(b),
                                    float(cos_As), _enum(mode, MODES), int(flags),
                                    _ptr(out) if M else None, _stream(stream)))
        return out

    def generate_host(self, centre_idx: np.ndarray, W, b, cos_As, schedule="STATIC",
                      mode="nearest", prune="brute", P=0, unit=0, gss_min_chunk=0,
                      fac_divisor=0, flags=0, out: np.ndarray | None = None, stats=False,
                      stream=None):
        """spin_generate_host: host int32 centres in, host fp32 [M, W, W] images out."""
        centre_idx = np.ascontiguousarray(centre_idx, dtype=np.int32)
        M = int(centre_idx.shape[0])
        if out is None:
            out = np.empty((M, W, W), np.float32)
        _check_array(out, "out", "float32", (M, W, W), "host")
        cp = self._params(P, unit, gss_min_chunk, fac_divisor, flags)
        st = Stats()
        _check(_lib.spin_generate_host(self._h, _ptr(centre_idx) if M else None, M, int(W),
                                       float(b), float(cos_As), _enum(schedule, SCHEDULES),
                                       C.byref(cp), _enum(mode, MODES), _enum(prune, PRUNES),
                                       _ptr(out) if M else None, C.byref(st) if stats else None,
                                       _stream(stream)))
        if stats:
            return out, _stats_dict(st)
        return out


def generate(points, normals, centre_idx, W, b, cos_As, **kw):
    """One-shot convenience: create a handle, generate, destroy."""
    eng = SpinEngine(points, normals)
    try:
        return eng.generate(centre_idx, W, b, cos_As, **kw)
    finally:
        eng.close()


NO_SUPPORT = -math.inf
