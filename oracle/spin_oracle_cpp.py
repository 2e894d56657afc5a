"""ctypes binding of the C++ oracle (oracle/spin_oracle.cpp) — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl
reference` legs may import this module; the product path never does, and this module
imports nothing from it.  Same contract as oracle/spin_oracle.py's `generate` /
`generate_cells` (Alg. 1, under DESIGN.md §3's readings): the C++
library decides every pair in double (certified bounds), then in threshold form with
measured rounding errors (double, then __float128); the few pairs it leaves undecided
(exact ties whose operations are not all exact) are decided here by the Python
oracle's exact rational arithmetic (`spin_oracle.exact_pair`).
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

from . import spin_oracle as PY

NEAREST, BILINEAR = PY.NEAREST, PY.BILINEAR
F_LITERAL_HALF_WIDTH, F_FLOOR_BINS = PY.F_LITERAL_HALF_WIDTH, PY.F_FLOOR_BINS
# test-only: send every pair to stage 2 / 3 / 4 (threshold double / __float128 / exact)
F_FORCE_STAGE2, F_FORCE_STAGE3, F_FORCE_STAGE4 = 1 << 8, 1 << 9, 1 << 10

_lib = None
_P = ctypes.c_void_p


def lib():
    global _lib
    if _lib is None:
        from . import build as B
        path = B.OUT
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(B.SRC):
            B.build()
        L = ctypes.CDLL(path)
        L.so_generate.restype = ctypes.c_int
        L.so_generate.argtypes = [_P, _P, ctypes.c_int64, _P, ctypes.c_int64, ctypes.c_int,
                                  ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, ctypes.c_int64,
                                  _P, _P]
        L.so_pair_bins.restype = ctypes.c_int
        L.so_pair_bins.argtypes = [_P, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                   ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, _P, _P, _P, _P, _P]
        L.so_region_radius.restype = ctypes.c_double
        L.so_region_radius.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _splat_exact(img, cnt, r, mode):
    if mode == NEAREST:
        img[r[0], r[1]] += 1.0
        return
    i0, j0, a, c = r
    for di, dj, wt in ((0, 0, (1 - a) * (1 - c)), (1, 0, a * (1 - c)),
                       (0, 1, (1 - a) * c), (1, 1, a * c)):
        img[i0 + di, j0 + dj] += wt
        if cnt is not None:
            cnt[i0 + di, j0 + dj] += int(wt > 0)


def _run(points, normals, centre_idx, W, b, cos_As, mode, flags, stats, cells, threads):
    X = np.ascontiguousarray(points, np.float32)
    Nr = np.ascontiguousarray(normals, np.float32)
    cen = np.ascontiguousarray(centre_idx, np.int32).reshape(-1)
    M, N = len(cen), len(X)
    out = np.zeros((M, W, W), np.float64)
    cnt = np.zeros((M, W, W), np.int32) if mode == BILINEAR else None
    inr = np.zeros(M, np.int64)
    st = np.zeros(4, np.int64)
    nun = ctypes.c_int64(0)
    cap = 1 << 16
    while True:
        uns = np.zeros((cap, 2), np.int64)
        rc = lib().so_generate(_ptr(X), _ptr(Nr), N, _ptr(cen), M, int(W), float(b), float(cos_As),
                               int(mode), int(flags), int(bool(cells)), int(threads), _ptr(out),
                               _ptr(cnt), _ptr(inr), _ptr(uns), cap, ctypes.byref(nun), _ptr(st))
        if rc == 1:
            cap = int(nun.value)
            continue
        if rc != 0:
            raise ValueError(f"so_generate: bad arguments (rc {rc})")
        break
    # stage 4: exact rational decisions of the pairs the floating stages left undecided
    for m, j in uns[:nun.value]:
        c = int(cen[m])
        r = PY.exact_pair(X[c], Nr[c], X[j], Nr[j], W, b, cos_As, mode, flags & 3)
        if r is None:
            continue
        inr[m] += 1
        _splat_exact(out[m], cnt[m] if cnt is not None else None, r, mode)
    if stats is not None:
        stats["exact_pairs"] = stats.get("exact_pairs", 0) + int(nun.value)
        stats["stage2_pairs"] = stats.get("stage2_pairs", 0) + int(st[0])
        stats["stage3_pairs"] = stats.get("stage3_pairs", 0) + int(st[1])
        stats["stage4_pairs"] = stats.get("stage4_pairs", 0) + int(st[2])
        stats["visited"] = stats.get("visited", 0) + int(st[3])
        stats.setdefault("in_region", []).extend(inr.tolist())
        if cnt is not None:
            # one (M, W, W) block (np.stack of it is itself); appended blocks concatenate
            prev = stats.get("contributors")
            stats["contributors"] = cnt if prev is None or len(prev) == 0 else \
                np.concatenate([np.asarray(prev), cnt])
    return out


def generate(points, normals, centre_idx, W: int, b: float, cos_As: float, mode: int,
             flags: int = 0, stats: dict | None = None, threads: int = 0) -> np.ndarray:
    """Oracle-BRUTE (every point visited, Alg. 1): (M, W, W) float64 images."""
    return _run(points, normals, centre_idx, W, b, cos_As, mode, flags, stats, False, threads)


def generate_cells(points, normals, centre_idx, W: int, b: float, cos_As: float, mode: int,
                   flags: int = 0, stats: dict | None = None, threads: int = 0) -> np.ndarray:
    """Oracle-CELLS: the same per-pair decision over the 27-cell neighbourhood of an
    independent grid (edge 1.0001 R); equals oracle-BRUTE."""
    return _run(points, normals, centre_idx, W, b, cos_As, mode, flags, stats, True, threads)


def region_radius(W: int, b: float, mode: int, flags: int = 0) -> float:
    return float(lib().so_region_radius(int(W), float(b), int(mode), int(flags)))


def pair_codes(points, normals, centres, W: int, b: float, cos_As: float, mode: int,
               flags: int = 0, threads: int = 0) -> np.ndarray:
    """int32 [len(centres), N]: -1 or the pair's bin code (NEAREST k*W + l, BILINEAR
    i0*W + j0) — the oracle side of the GPU's spin_pair_codes diagnostic."""
    X = np.ascontiguousarray(points, np.float32)
    out = np.empty((len(centres), len(X)), np.int32)
    for i, c in enumerate(np.asarray(centres).reshape(-1)):
        st, k, l, _, _ = pair_bins(X, normals, int(c), W, b, cos_As, mode, flags, threads)
        out[i] = np.where(st == 1, k * W + l, -1)
    return out


def pair_bins(points, normals, c: int, W: int, b: float, cos_As: float, mode: int,
              flags: int = 0, threads: int = 0):
    """Per-pair decisions of centre c against every point: (state, k, l, u, v) arrays.

    state 1 = contributes at (k, l) (NEAREST bin, BILINEAR (i0, j0)), 0 = does not;
    u and v = sqrt(max(w, 0)) in double.  Undecided pairs are decided exactly here."""
    X = np.ascontiguousarray(points, np.float32)
    Nr = np.ascontiguousarray(normals, np.float32)
    N = len(X)
    state = np.zeros(N, np.int32)
    kk = np.zeros(N, np.int32)
    ll = np.zeros(N, np.int32)
    uu = np.zeros(N, np.float64)
    vv = np.zeros(N, np.float64)
    rc = lib().so_pair_bins(_ptr(X), _ptr(Nr), N, int(c), int(W), float(b), float(cos_As),
                            int(mode), int(flags), int(threads), _ptr(state), _ptr(kk), _ptr(ll),
                            _ptr(uu), _ptr(vv))
    if rc != 0:
        raise ValueError(f"so_pair_bins: bad arguments (rc {rc})")
    for j in np.nonzero(state == 2)[0]:
        r = PY.exact_pair(X[c], Nr[c], X[j], Nr[j], W, b, cos_As, mode, flags & 3)
        state[j] = 0 if r is None else 1
        if r is not None:
            kk[j], ll[j] = r[0], r[1]
    return state, kk, ll, uu, vv


__all__ = ["generate", "generate_cells", "region_radius", "pair_bins", "pair_codes", "NEAREST", "BILINEAR",
           "F_LITERAL_HALF_WIDTH", "F_FLOOR_BINS", "math"]
