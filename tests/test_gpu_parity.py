"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

NEAREST must be bit-exact; BILINEAR within the north-star tolerance (per-image rel
L1 <= 1e-5, per-bin <= 1e-4 x contributing points).  Inputs are the seeded
generators of synth/clouds.py; expected values come only from oracle/.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import spin_oracle as O
from oracle import spin_oracle_cpp as OC
from synth import clouds
from parity_util import assert_bilinear_close, assert_nearest_exact

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def torch():
    import torch as t
    if not t.cuda.is_available():
        pytest.skip("no CUDA device")
    return t


@pytest.fixture(scope="module")
def spin(torch):
    from paper_1811_00901_b200 import spin as s
    return s


def _dev(torch, a, dtype=None):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def run_gpu(spin, torch, pts, Nn, cen, W, b, c, mode, prune="brute", stats=False, **kw):
    eng = spin.SpinEngine(_dev(torch, pts), _dev(torch, Nn))
    try:
        r = eng.generate(_dev(torch, np.asarray(cen, np.int32)), W, b, c, mode=mode, prune=prune,
                         stats=stats, **kw)
        torch.cuda.synchronize()
        if stats:
            return r[0].cpu().numpy(), r[1]
        return r.cpu().numpy()
    finally:
        eng.close()


def oracle(P, Nn, cen, W, b, c, mode, flags=0, cells=False):
    st = {}
    f = O.generate_cells if cells else O.generate
    img = f(P, Nn, cen, W, b, c, O.NEAREST if mode == "nearest" else O.BILINEAR, flags, stats=st)
    return img, st


def check(gpu, ora, st, mode, what):
    if mode == "nearest":
        assert_nearest_exact(gpu, ora, what)
    else:
        assert_bilinear_close(gpu, ora, np.stack(st["contributors"]), what)


# ------------------------------------------------------------------ hand-worked goldens

def _gold(name):
    g = json.load(open(os.path.join(GOLD, name)))
    return g, np.asarray(g["points"], np.float32), np.asarray(g["normals"], np.float32)


def test_x1_goldens(spin, torch):
    g, P, Nn = _gold("x1.json")
    for mode in ("nearest", "bilinear"):
        for flags in (0, spin.F_NO_FAST_CERT):
            img = run_gpu(spin, torch, P, Nn, [0], g["W"], g["b"], -math.inf, mode, flags=flags)[0]
            np.testing.assert_array_equal(img, np.asarray(g[mode], np.float32), err_msg=f"{mode} {flags}")


def test_x2_x3_x4_goldens(spin, torch):
    g, P, Nn = _gold("x2.json")
    img = run_gpu(spin, torch, P, Nn, [0], g["W"], g["b"], -math.inf, "nearest")[0]
    np.testing.assert_array_equal(img, g["nearest_scaled"])
    img = run_gpu(spin, torch, P, Nn, [0], g["W"], g["b"], -math.inf, "nearest",
                  flags=spin.F_LITERAL_HALF_WIDTH)[0]
    np.testing.assert_array_equal(img, g["nearest_literal"])
    g, P, Nn = _gold("x3.json")
    img = run_gpu(spin, torch, P, Nn, [0], g["W"], g["b"], -math.inf, "nearest")[0]
    np.testing.assert_array_equal(img, g["nearest"])
    g, P, Nn = _gold("x4.json")
    img = run_gpu(spin, torch, P, Nn, [0], g["W"], g["b"], 0.0, "nearest")[0]
    np.testing.assert_array_equal(img, g["cos_zero"])
    img = run_gpu(spin, torch, P, Nn, [0], g["W"], g["b"], math.cos(math.pi / 2), "nearest")[0]
    np.testing.assert_array_equal(img, g["cos_fl_half_pi"])


# ------------------------------------------------------------------ seeded clouds

@pytest.mark.parametrize("mode", ["nearest", "bilinear"])
def test_config1_full(spin, torch, mode):
    """Config 1 in full (N = M = 2000, W=8, b=0.05, 60 deg), STATIC, brute force."""
    cfg = clouds.CONFIGS[1]
    P, Nn = clouds.make_cloud(1)
    cen = clouds.make_centres(1, cfg["N"])
    gpu = run_gpu(spin, torch, P, Nn, cen, cfg["W"], cfg["b"], cfg["cos_As"], mode)
    ora, st = oracle(P, Nn, cen, cfg["W"], cfg["b"], cfg["cos_As"], mode)
    check(gpu, ora, st, mode, f"C1 {mode}")


@pytest.mark.parametrize("mode", ["nearest", "bilinear"])
@pytest.mark.parametrize("N,M", [(5000, 300), (1, 1), (1023, 37), (1025, 70)])
def test_bumpy_ragged(spin, torch, mode, N, M):
    """Several 1024-point tiles plus a ragged tail; partial groups; W=16, b=0.02, 60 deg."""
    P, Nn = clouds.bumpy_sphere(N, 2)
    cen = np.arange(M, dtype=np.int32) % N
    gpu = run_gpu(spin, torch, P, Nn, cen, 16, 0.02 if N > 100 else 0.5, 0.5, mode)
    ora, st = oracle(P, Nn, cen, 16, 0.02 if N > 100 else 0.5, 0.5, mode)
    check(gpu, ora, st, mode, f"bumpy N={N} M={M} {mode}")


@pytest.mark.parametrize("W", [1, 2, 5, 17, 24, 28, 32, 33, 41, 64])
def test_widths(spin, torch, W):
    """W = 1 .. 64 across every BRUTE launch shape the planner picks (768 threads with
    G = 64 / 32 / 24 / 16 / 8 / 4, 512 threads with G = 32 at W = 33), odd W (real W/2, #3)."""
    P, Nn = clouds.bumpy_sphere(3000, 7)
    cen = np.arange(0, 3000, 41, dtype=np.int32)
    b = 0.4 / W
    for mode in ("nearest", "bilinear"):
        if mode == "bilinear" and W < 2:
            continue
        gpu = run_gpu(spin, torch, P, Nn, cen, W, b, 0.0, mode)
        ora, st = oracle(P, Nn, cen, W, b, 0.0, mode)
        check(gpu, ora, st, mode, f"W={W} {mode}")


@pytest.mark.parametrize("flags", [1, 2, 8])   # LITERAL, FLOOR, NO_FAST_CERT
def test_flags(spin, torch, flags):
    P, Nn = clouds.bumpy_sphere(4000, 9)
    cen = np.arange(0, 4000, 29, dtype=np.int32)
    W, b = (4, 0.5) if flags == 1 else (16, 0.02)
    for mode in ("nearest", "bilinear"):
        if flags == 2 and mode == "bilinear":
            continue
        gpu = run_gpu(spin, torch, P, Nn, cen, W, b, 0.5, mode, flags=flags)
        ora, st = oracle(P, Nn, cen, W, b, 0.5, mode, flags & 3)
        check(gpu, ora, st, mode, f"flags={flags} {mode}")


def _dyadic_ties(n, seed):
    rng = np.random.default_rng(seed)
    P = (np.round(rng.uniform(-1, 1, (n, 3)) * 8) / 8).astype(np.float32)
    g = rng.normal(size=(n, 3))
    Nn = (g / np.linalg.norm(g, axis=1, keepdims=True)).astype(np.float32)
    Nn[::3] = [0, 0, 1]
    Nn[1::3] = [1, 0, 0]
    return P, Nn


@pytest.mark.parametrize("flags", [0, 1, 2])
def test_exact_ties_dyadic(spin, torch, flags):
    """Many pairs sit EXACTLY on bin edges: exercises the fp64 and exact stages."""
    P, Nn = _dyadic_ties(400, 3)
    cen = np.arange(400, dtype=np.int32)
    W, b = 6, (1.0 if flags == 1 else 0.25)
    for c in (-math.inf, 0.0):
        for mode in ("nearest", "bilinear"):
            if flags == 2 and mode == "bilinear":
                continue
            gpu, st_g = run_gpu(spin, torch, P, Nn, cen, W, b, c, mode, flags=flags, stats=True)
            ora, st = oracle(P, Nn, cen, W, b, c, mode, flags)
            check(gpu, ora, st, mode, f"ties flags={flags} c={c} {mode}")
            assert st_g["fp64_fallbacks"] > 0 and st_g["exact_fallbacks"] > 0


def test_region_corners(spin, torch):
    """Points on and 1-2 ulps around the corners and rims of the region cylinder (beta at
    both window edges, alpha at its bound) about an off-origin centre with an oblique
    normal: the pairs closest to the BRUTE hot loop's bounding sphere."""
    rng = np.random.default_rng(11)
    for W, b in ((16, 0.02), (5, 0.1), (32, 0.01)):
        for mode in ("nearest", "bilinear"):
            p0 = np.array([0.31, -0.22, 0.7])
            n0 = rng.normal(size=3)
            n0 /= np.linalg.norm(n0)
            t1 = np.cross(n0, [0.3, 0.5, 0.8])
            t1 /= np.linalg.norm(t1)
            t2 = np.cross(n0, t1)
            if mode == "nearest":
                ulo, uhi, vmax = -1.0, W - 1.0, W - 1.0
            else:
                ulo, uhi, vmax = 0.0, W - 1.0, W - 1.0
            xs = [p0]
            for u in (ulo, uhi, 0.5 * (ulo + uhi)):
                beta = (W / 2 - u) * b
                for ang in np.linspace(0, 2 * np.pi, 7, endpoint=False):
                    for a in (vmax * b, 0.5 * vmax * b):
                        x = p0 + beta * n0 + a * (np.cos(ang) * t1 + np.sin(ang) * t2)
                        x32 = x.astype(np.float32)
                        for d in (-2, -1, 0, 1, 2):
                            xs.append(x32 + d * np.spacing(x32) * np.sign(x32 - p0))
            X = np.asarray(xs, np.float32)
            Nn = np.tile(n0.astype(np.float32), (len(X), 1))
            for c in (-math.inf, 0.5):
                gpu = run_gpu(spin, torch, X, Nn, [0], W, b, c, mode)
                ora, st = oracle(X, Nn, [0], W, b, c, mode)
                check(gpu, ora, st, mode, f"corners W={W} {mode} c={c}")


@pytest.mark.parametrize("offset,scale", [((300.0, -200.0, 500.0), 1.0), ((0.0, 0.0, 0.0), 1e-3),
                                          ((1e4, 0.0, 0.0), 1.0)])
def test_far_from_origin_and_tiny_scale(spin, torch, offset, scale):
    """Clouds far from the origin (|x| up to 1e4: the fp32 hot-loop bounds grow with |x|,
    so the filter loosens and more decisions go to fp64 / exact) and at a tiny scale
    (1e-3): results stay oracle-exact (NEAREST) / within tolerance (BILINEAR)."""
    P0, Nn = clouds.bumpy_sphere(3000, 13)
    P = (P0.astype(np.float64) * scale + np.asarray(offset)).astype(np.float32)
    cen = np.arange(0, 3000, 97, dtype=np.int32)
    b = 0.02 * scale
    for mode in ("nearest", "bilinear"):
        for prune in ("brute", "cells"):
            gpu = run_gpu(spin, torch, P, Nn, cen, 16, b, 0.5, mode, prune=prune)
            ora, st = oracle(P, Nn, cen, 16, b, 0.5, mode)
            check(gpu, ora, st, mode, f"offset={offset} scale={scale} {mode} {prune}")


def test_near_threshold_ulps(spin, torch):
    """Points 1 fp32 ulp either side of every row / column edge."""
    W, b = 16, 0.02
    xs = [[0, 0, 0]]
    for k in range(0, W + 2):
        edge = np.float32((W / 2 - k) * b)
        for z in (np.nextafter(edge, np.float32(-1)), edge, np.nextafter(edge, np.float32(1))):
            xs.append([0.05, 0, z])
        r = np.float32(k * b)
        for xr in (np.nextafter(r, np.float32(0)), r, np.nextafter(r, np.float32(1))):
            xs.append([xr, 0, 0.01])
            xs.append([xr * np.float32(0.6), xr * np.float32(0.8), 0.01])
    X = np.asarray(xs, np.float32)
    Nn = np.tile(np.array([0, 0, 1], np.float32), (len(X), 1))
    for mode in ("nearest", "bilinear"):
        gpu = run_gpu(spin, torch, X, Nn, [0], W, b, -math.inf, mode)
        ora, st = oracle(X, Nn, [0], W, b, -math.inf, mode)
        check(gpu, ora, st, mode, f"ulps {mode}")


# ------------------------------------------------------------------ schedules

def test_schedule_invariance(spin, torch):
    """S:169 keystone: STATIC/SS/GSS/FAC x P x unit give bit-identical images."""
    P, Nn = clouds.bumpy_sphere(6000, 4)
    cen = np.arange(0, 6000, 3, dtype=np.int32)
    for mode in ("nearest", "bilinear"):
        ref = run_gpu(spin, torch, P, Nn, cen, 16, 0.02, 0.5, mode)
        for sched in ("STATIC", "SS", "GSS", "FAC", "WF", "AWF"):
            for Pn in (1, 7, 148, 0):
                for unit in (0, 1, 5):
                    got = run_gpu(spin, torch, P, Nn, cen, 16, 0.02, 0.5, mode, schedule=sched,
                                  P=Pn, unit=unit)
                    np.testing.assert_array_equal(got, ref, err_msg=f"{mode} {sched} P={Pn} u={unit}")
        ora, st = oracle(P, Nn, cen[:200], 16, 0.02, 0.5, mode)
        check(ref[:200], ora, st, mode, f"sched ref {mode}")


def test_dealer_stats_and_cta_times(spin, torch):
    P, Nn = clouds.bumpy_sphere(8000, 5)
    cen = np.arange(8000, dtype=np.int32)
    for sched in ("STATIC", "SS", "GSS", "FAC"):
        _, st = run_gpu(spin, torch, P, Nn, cen, 16, 0.02, 0.5, "nearest", stats=True,
                        schedule=sched, P=64, cta_capacity=64)
        assert st["P"] == 64 and st["pairs_visited"] == 8000 * 8000
        assert int(st["cta_units"].sum()) == st["n_units"] == -(-8000 // st["G"])
        assert np.all(st["cta_end_ns"] >= st["cta_start_ns"])
        exp = len(spin.chunk_sequence(sched, st["n_units"], 64)) - 1
        assert st["n_chunks"] == exp
    # WF / AWF claim their chunks by compare-and-swap: every unit exactly once, the claim
    # count between the FAC count (equal weights) and SS's
    fac = len(spin.chunk_sequence("FAC", -(-8000 // 64), 64)) - 1
    for sched in ("WF", "AWF"):
        img, st = run_gpu(spin, torch, P, Nn, cen, 16, 0.02, 0.5, "nearest", stats=True,
                          schedule=sched, P=64, cta_capacity=64, slow_ctas=8, slowdown=3.0)
        assert int(st["cta_units"].sum()) == st["n_units"]
        assert fac // 2 <= st["n_chunks"] <= st["n_units"], (sched, st["n_chunks"], fac)


# ------------------------------------------------------------------ cell list

@pytest.mark.parametrize("mode", ["nearest", "bilinear"])
def test_cells_vs_oracle_and_brute(spin, torch, mode):
    P, Nn = clouds.clustered(30000, 3)
    cen = clouds.sample_centres(30000, 600, 13)
    W, b, c = 16, 0.01, 0.5
    cells, st_c = run_gpu(spin, torch, P, Nn, cen, W, b, c, mode, prune="cells", stats=True)
    brute = run_gpu(spin, torch, P, Nn, cen, W, b, c, mode, prune="brute")
    np.testing.assert_array_equal(cells, brute)
    ora, st = oracle(P, Nn, cen[:150], W, b, c, mode, cells=True)
    check(cells[:150], ora, st, mode, f"cells {mode}")
    assert st_c["pairs_visited"] < 600 * 30000
    # unsorted control and every schedule give the same images
    for sched in ("SS", "GSS", "FAC"):
        got = run_gpu(spin, torch, P, Nn, cen, W, b, c, mode, prune="cells", schedule=sched)
        np.testing.assert_array_equal(got, cells)
    got = run_gpu(spin, torch, P, Nn, cen, W, b, c, mode, prune="cells", flags=spin.F_NO_SORT)
    np.testing.assert_array_equal(got, cells)


@pytest.mark.parametrize("W", [3, 24, 33, 64])
def test_cells_widths(spin, torch, W):
    """CELLS at widths that select G = 32 / 16 / 8 / 4: equal to BRUTE, and to the oracle."""
    P, Nn = clouds.clustered(12000, 21)
    cen = clouds.sample_centres(12000, 200, 22)
    b = 0.16 / W
    for mode in ("nearest", "bilinear"):
        cells = run_gpu(spin, torch, P, Nn, cen, W, b, 0.5, mode, prune="cells")
        brute = run_gpu(spin, torch, P, Nn, cen, W, b, 0.5, mode)
        np.testing.assert_array_equal(cells, brute, err_msg=f"W={W} {mode}")
        ora, st = oracle(P, Nn, cen[:25], W, b, 0.5, mode, cells=True)
        check(cells[:25], ora, st, mode, f"cells W={W} {mode}")


def test_cells_floor_and_literal(spin, torch):
    P, Nn = clouds.clustered(20000, 8)
    cen = clouds.sample_centres(20000, 300, 14)
    for flags, W, b in ((2, 8, 0.01), (1, 4, 0.3)):
        cells = run_gpu(spin, torch, P, Nn, cen, W, b, 0.5, "nearest", prune="cells", flags=flags)
        brute = run_gpu(spin, torch, P, Nn, cen, W, b, 0.5, "nearest", flags=flags)
        np.testing.assert_array_equal(cells, brute)
        ora, _ = oracle(P, Nn, cen[:60], W, b, 0.5, "nearest", flags)
        assert_nearest_exact(cells[:60], ora, f"cells flags={flags}")


# ------------------------------------------------------------------ edge cases and errors

def test_edge_cases(spin, torch):
    P, Nn = clouds.bumpy_sphere(2000, 6)
    eng = spin.SpinEngine(_dev(torch, P), _dev(torch, Nn))
    try:
        empty = torch.zeros(0, dtype=torch.int32, device="cuda")
        out = eng.generate(empty, 8, 0.05, 0.5)
        assert out.shape == (0, 8, 8)
        # duplicated centres give identical images
        cen = _dev(torch, np.array([5, 5, 17, 5], np.int32))
        out = eng.generate(cen, 8, 0.05, 0.5).cpu().numpy()
        np.testing.assert_array_equal(out[0], out[1])
        np.testing.assert_array_equal(out[0], out[3])
        # support disabled (S = 2 pi) and S = 0 (only parallel normals)
        for c in (-math.inf, 1.0):
            g = eng.generate(_dev(torch, np.arange(0, 2000, 97, dtype=np.int32)), 8, 0.05, c).cpu().numpy()
            o, _ = oracle(P, Nn, np.arange(0, 2000, 97), 8, 0.05, c, "nearest")
            assert_nearest_exact(g, o, f"c={c}")
        # out-of-range centre: zero image, SPIN_E_RANGE
        bad = _dev(torch, np.array([3, 2000, -1, 4], np.int32))
        out = torch.full((4, 8, 8), 7.0, device="cuda")
        with pytest.raises(spin.SpinError) as ei:
            eng.generate(bad, 8, 0.05, 0.5, out=out, stats=True)
        assert ei.value.status == 2
        o = out.cpu().numpy()
        assert np.all(o[1] == 0) and np.all(o[2] == 0) and o[0].sum() > 0
        # the next call is clean
        eng.generate(_dev(torch, np.array([1], np.int32)), 8, 0.05, 0.5, stats=True)
        # invalid arguments
        ok = _dev(torch, np.array([1], np.int32))
        for kw in (dict(W=0), dict(W=65), dict(b=0.0), dict(b=float("nan")), dict(cos_As=1.5),
                   dict(W=1, mode="bilinear")):
            args = dict(W=8, b=0.05, cos_As=0.5, mode="nearest")
            args.update(kw)
            with pytest.raises(spin.SpinError) as ei:
                eng.generate(ok, args["W"], args["b"], args["cos_As"], mode=args["mode"])
            assert ei.value.status == 1
    finally:
        eng.close()


def test_invalid_cloud(spin, torch):
    P, Nn = clouds.bumpy_sphere(100, 6)
    Nn2 = Nn.copy()
    Nn2[42] *= 1.01
    with pytest.raises(spin.SpinError) as ei:
        spin.SpinEngine(_dev(torch, P), _dev(torch, Nn2))
    assert ei.value.status == 3 and "42" in str(ei.value)
    P2 = P.copy()
    P2[7, 1] = np.inf
    with pytest.raises(spin.SpinError) as ei:
        spin.SpinEngine(_dev(torch, P2), _dev(torch, Nn))
    assert ei.value.status == 3 and "7" in str(ei.value)


def test_host_path_and_reload(spin, torch):
    """spin_generate_host (host buffers) equals the device path; spin_load_cloud swaps clouds."""
    P, Nn = clouds.bumpy_sphere(3000, 10)
    cen = np.arange(0, 3000, 7, dtype=np.int32)
    eng = spin.SpinEngine(P, Nn)      # host arrays: spin_create copies with cudaMemcpyDefault
    try:
        h = eng.generate_host(cen, 16, 0.02, 0.5, mode="bilinear")
        d = eng.generate(_dev(torch, cen), 16, 0.02, 0.5, mode="bilinear").cpu().numpy()
        np.testing.assert_array_equal(h, d)
        P2, N2 = clouds.bumpy_sphere(5000, 11)
        eng.load_cloud(P2, N2)
        h2 = eng.generate_host(cen, 16, 0.02, 0.5)
        o, _ = oracle(P2, N2, cen, 16, 0.02, 0.5, "nearest")
        assert_nearest_exact(h2, o, "reloaded cloud")
        h3 = eng.generate_host(cen, 16, 0.02, 0.5, prune="cells")
        np.testing.assert_array_equal(h3, h2)
    finally:
        eng.close()


# (full-size configs at the BASELINE sample sizes: tests/test_gpu_scale.py)


def test_bilinear_fixed_point_carries(spin, torch):
    """> 512 units of weight in one bin exercise the 2^-23 fixed-point carry words."""
    rng = np.random.default_rng(21)
    n = 4000
    P = (rng.normal(size=(n, 3)) * 1e-3).astype(np.float32)
    Nn = np.tile(np.array([0, 0, 1], np.float32), (n, 1))
    cen = np.arange(0, n, 400, dtype=np.int32)
    for W, b in ((4, 1.0), (6, 0.0013)):
        gpu = run_gpu(spin, torch, P, Nn, cen, W, b, 0.5, "bilinear")
        ora, st = oracle(P, Nn, cen, W, b, 0.5, "bilinear")
        assert ora.max() > 600
        check(gpu, ora, st, "bilinear", f"carries W={W}")
        again = run_gpu(spin, torch, P, Nn, cen, W, b, 0.5, "bilinear", schedule="SS", unit=1)
        np.testing.assert_array_equal(again, gpu)    # deterministic (integer accumulation)


def test_host_path_pipelined_d2h(spin, torch):
    """spin_generate_host delivers the device path's images bit for bit on each of its three
    routes: page-locked output written by the kernel directly (any processing order), pageable
    output through device scratch with the D2H after the kernel (Morton order), and with the
    D2H pipelined per output segment (caller order, SPIN_F_NO_SORT)."""
    P, Nn = clouds.bumpy_sphere(20000, 12)
    cen = np.arange(20000, dtype=np.int32)[::-1].copy()
    eng = spin.SpinEngine(P, Nn)
    pinned = torch.empty((len(cen), 16, 16), dtype=torch.float32).pin_memory()
    try:
        for mode in ("nearest", "bilinear"):
            for sched, unit in (("SS", 0), ("GSS", 1), ("STATIC", 0)):
                d = eng.generate(_dev(torch, cen), 16, 0.02, 0.5, mode=mode).cpu().numpy()
                for route, flags in (("pinned", 0), ("pageable", 0), ("pageable", spin.F_NO_SORT)):
                    out = pinned.numpy() if route == "pinned" else np.empty((len(cen), 16, 16), np.float32)
                    out.fill(-1.0)
                    h = eng.generate_host(cen, 16, 0.02, 0.5, mode=mode, schedule=sched, unit=unit,
                                          out=out, flags=flags)
                    np.testing.assert_array_equal(h, d, err_msg=f"{mode} {sched} unit={unit} {route} {flags}")
        pick = np.arange(0, 20000, 997)
        ora, _ = oracle(P, Nn, cen[pick], 16, 0.02, 0.5, "nearest")
        assert_nearest_exact(eng.generate_host(cen, 16, 0.02, 0.5, out=pinned.numpy())[pick], ora, "pinned host")
        assert_nearest_exact(eng.generate_host(cen, 16, 0.02, 0.5)[pick], ora, "pageable host")
    finally:
        eng.close()


@pytest.mark.gpu
def test_support_placement_same_images(spin, torch):
    """BRUTE support placement: adaptive (default), SPIN_F_SUPPORT_FIRST (every pair, P:166
    order) and SPIN_F_SUPPORT_LAST give identical images.  Random normals make the support
    test reject most sphere candidates, so the adaptive CTAs must move it into the hot loop
    (tiles_support_hot > 0); a smooth surface keeps it in the accept path."""
    P, Nn = clouds.clustered(20000, 23)
    rng = np.random.default_rng(5)
    Nr = rng.normal(size=Nn.shape)
    Nr = (Nr / np.linalg.norm(Nr, axis=1, keepdims=True)).astype(np.float32)
    cen = clouds.sample_centres(20000, 3000, 24)
    for mode in ("nearest", "bilinear"):
        a, sa = run_gpu(spin, torch, P, Nr, cen, 16, 0.01, 0.5, mode, stats=True)
        b, sb = run_gpu(spin, torch, P, Nr, cen, 16, 0.01, 0.5, mode, stats=True, flags=spin.F_SUPPORT_FIRST)
        a16 = run_gpu(spin, torch, P, Nr, cen, 16, 0.01, 0.5, mode, P=16)
        np.testing.assert_array_equal(a, a16, err_msg=mode)
        c = run_gpu(spin, torch, P, Nr, cen, 16, 0.01, 0.5, mode, flags=spin.F_SUPPORT_LAST)
        np.testing.assert_array_equal(a, b, err_msg=mode)
        np.testing.assert_array_equal(a, c, err_msg=mode)
        assert sa["tiles_support_hot"] > 0, sa
        assert sb["tiles_support_hot"] == 0          # the forced variant does not count
        ora, st = oracle(P, Nr, cen[:40], 16, 0.01, 0.5, mode)
        check(a[:40], ora, st, mode, f"adaptive support {mode}")
    Ps, Ns = clouds.sphere(20000, 25)
    cs = clouds.sample_centres(20000, 2000, 26)
    a, sa = run_gpu(spin, torch, Ps, Ns, cs, 16, 0.01, 0.5, "nearest", stats=True)
    b = run_gpu(spin, torch, Ps, Ns, cs, 16, 0.01, 0.5, "nearest", flags=spin.F_SUPPORT_FIRST)
    np.testing.assert_array_equal(a, b)
    assert sa["tiles_support_hot"] == 0, sa


@pytest.mark.parametrize("prune", ["brute", "cells"])
def test_support_last_same_images(spin, torch, prune):
    """SPIN_F_SUPPORT_LAST (support test decided after the region test) and the no-support
    case (cos_As = -inf, hot loop without the support test) leave the images unchanged."""
    P, Nn = clouds.clustered(20000, 17)
    cen = clouds.sample_centres(20000, 500, 18)
    for mode in ("nearest", "bilinear"):
        for c in (0.5, 0.0, -math.inf):
            a = run_gpu(spin, torch, P, Nn, cen, 16, 0.01, c, mode, prune=prune)
            b = run_gpu(spin, torch, P, Nn, cen, 16, 0.01, c, mode, prune=prune,
                        flags=spin.F_SUPPORT_LAST)
            np.testing.assert_array_equal(a, b, err_msg=f"{mode} c={c}")
        ora, st = oracle(P, Nn, cen[:40], 16, 0.01, 0.5, mode, cells=(prune == "cells"))
        check(b if c == 0.5 else run_gpu(spin, torch, P, Nn, cen[:40], 16, 0.01, 0.5, mode, prune=prune,
                                         flags=spin.F_SUPPORT_LAST), ora, st, mode, f"support-last {mode}")


def test_heterogeneous_workers_same_images_and_trend(spin, torch):
    """Heterogeneity emulation (the paper's Type1/Type2 runs):
    slow CTAs change timing only, never images (every slowed run equals the ORACLE's images
    of all 60,000 centres, ~940 units of 64); with a quarter of the CTAs 4x slower, a
    dynamic schedule beats STATIC (ideal ratio 4 * (111 + 37/4) / 148 = 3.25, SPEC
    acceptance #5 asks >= 1.5), and the slow CTAs process fewer units under SS."""
    P, Nn = clouds.bumpy_sphere(60000, 31)
    cen = np.arange(60000, dtype=np.int32)
    eng = spin.SpinEngine(_dev(torch, P), _dev(torch, Nn))
    try:
        d_cen = _dev(torch, cen)
        ora = OC.generate(P, Nn, cen, 16, 0.02, 0.5, OC.NEAREST)
        ref = torch.from_numpy(ora.astype(np.float32)).cuda()
        times = {}
        for sched in ("STATIC", "SS", "GSS", "FAC", "WF", "AWF"):
            for slow_first in (False, True):
                kw = dict(schedule=sched, P=148, slow_ctas=37, slowdown=4.0, slow_first=slow_first)
                out, st = eng.generate(d_cen, 16, 0.02, 0.5, stats=True, cta_capacity=148, **kw)
                torch.cuda.synchronize()
                assert torch.equal(out, ref), (sched, slow_first)
                ts = []
                for _ in range(3):
                    _, st = eng.generate(d_cen, 16, 0.02, 0.5, stats=True, cta_capacity=148, **kw)
                    ts.append(st["elapsed_ms"])
                times[(sched, slow_first)] = (float(np.median(ts)), st)
        t_static = times[("STATIC", False)][0]
        t_ss, st_ss = times[("SS", False)]
        assert t_static / t_ss >= 1.5, times
        u = st_ss["cta_units"]
        assert u[:37].mean() < 0.6 * u[37:].mean(), u
        # weighted factoring knows the slow workers a priori (WF): well ahead of FAC's equal
        # chunks, the slow CTAs get fewer units; AWF measures them, but only after its first
        # (equal-weight) batch, which already overloads the slow CTAs: it must still beat STATIC
        t_wf, st_w = times[("WF", False)]
        assert t_wf <= 0.9 * times[("FAC", False)][0], times
        uw = st_w["cta_units"]
        assert uw[:37].mean() < 0.6 * uw[37:].mean(), uw
        assert t_static / times[("AWF", False)][0] >= 1.5, times
    finally:
        eng.close()


def test_count_in_sphere_matches_numpy(spin, torch):
    """spin_count_in_sphere (CELLS work measure independent of the
    implementation) equals a float64 brute-force count, on a clustered cloud."""
    P, Nn = clouds.clustered(30000, 51)
    cen = clouds.sample_centres(30000, 700, 52)
    R = spin.region_radius(16, 0.01, "bilinear")
    eng = spin.SpinEngine(_dev(torch, P), _dev(torch, Nn))
    try:
        got = eng.count_in_sphere(_dev(torch, cen), R)
    finally:
        eng.close()
    X = P.astype(np.float64)
    want = 0
    for c in cen:
        d = X - X[c]
        want += int(np.count_nonzero((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2] <= R * R))
    assert got == want


def test_tensor_core_filter_selection_and_parity(spin, torch):
    """The BRUTE sphere filter runs on the tensor cores (tf32 mma.sync)
    for clouds near the origin and falls back to packed fp32 where the tf32 bound would
    loosen the sphere (far from the origin); both give oracle-exact NEAREST images, and
    the fp32 arm forced by SPIN_NO_MMA gives the identical images."""
    P, Nn = clouds.bumpy_sphere(4000, 21)
    cen = np.arange(0, 4000, 13, dtype=np.int32)
    gpu, st = run_gpu(spin, torch, P, Nn, cen, 16, 0.02, 0.5, "nearest", stats=True)
    assert st["filter_mma"] == 1
    ora, ost = oracle(P, Nn, cen, 16, 0.02, 0.5, "nearest")
    check(gpu, ora, ost, "nearest", "tensor-core filter")
    os.environ["SPIN_NO_MMA"] = "1"
    try:
        g2, st2 = run_gpu(spin, torch, P, Nn, cen, 16, 0.02, 0.5, "nearest", stats=True)
    finally:
        del os.environ["SPIN_NO_MMA"]
    assert st2["filter_mma"] == 0
    assert np.array_equal(gpu, g2)
    # candidates: the tf32 sphere may only be slightly looser than the fp32 one
    assert 0.99 * st2["pairs_candidate"] <= st["pairs_candidate"] <= 1.06 * st2["pairs_candidate"]
    Pf = (P.astype(np.float64) + np.asarray([1e4, 0.0, 0.0])).astype(np.float32)
    g3, st3 = run_gpu(spin, torch, Pf, Nn, cen[:40], 16, 0.02, 0.5, "nearest", stats=True)
    assert st3["filter_mma"] == 0
    ora3, ost3 = oracle(Pf, Nn, cen[:40], 16, 0.02, 0.5, "nearest")
    check(g3, ora3, ost3, "nearest", "far cloud, fp32 filter")


def _fuzz_cloud(rng, kind, n):
    """Small seeded clouds with the structures that stress the filters and the decisions:
    surfaces, volumes, exact duplicates, coplanar / collinear sets, dyadic grids (exact
    ties), far offsets and tiny scales."""
    if kind == "bumpy":
        P, Nn = clouds.bumpy_sphere(n, int(rng.integers(1 << 30)))
    elif kind == "clustered":
        P, Nn = clouds.clustered(n, int(rng.integers(1 << 30)))
    else:
        if kind == "dyadic":
            P = rng.integers(-16, 17, size=(n, 3)).astype(np.float64) / 16.0
        elif kind == "planar":
            P = np.c_[rng.uniform(-1, 1, (n, 2)), np.zeros(n)]
        else:  # collinear
            P = np.c_[rng.uniform(-1, 1, n), np.zeros(n), np.zeros(n)]
        g = rng.normal(size=(n, 3))
        Nn = g / np.linalg.norm(g, axis=1, keepdims=True)
        if kind != "collinear":
            Nn[: n // 2] = [0.0, 0.0, 1.0]
    P = np.asarray(P, np.float64)
    dup = rng.integers(0, n, size=max(1, n // 20))
    P[dup[: len(dup) // 2]] = P[dup[len(dup) // 2: 2 * (len(dup) // 2)]]   # exact duplicates
    scale = float(rng.choice([1.0, 1.0, 1e-2, 64.0]))
    off = rng.uniform(-1, 1, 3) * float(rng.choice([0.0, 0.0, 2.0, 50.0]))
    return (P * scale + off).astype(np.float32), np.asarray(Nn, np.float32), scale


def _split_launches(spin, torch, P, Nn, cen, W, b, c, mode, kw):
    """The shared-dealer contract in one process: two launches of ONE schedule (global P,
    grid = P/2 each, cta_offset 0 / P/2, one counter); each writes only the images of the
    chunks its CTAs took, so the two zero-initialised outputs sum to the full result."""
    Pg = max(2, kw["P"] or 2 * 148)
    half = Pg // 2
    eng = spin.SpinEngine(_dev(torch, P), _dev(torch, Nn))
    dealer = spin.Dealer()
    try:
        d_cen = _dev(torch, np.asarray(cen, np.int32))
        outs = []
        for off, g in ((0, half), (half, Pg - half)):
            out = torch.zeros((len(cen), W, W), dtype=torch.float32, device="cuda")
            k2 = dict(kw, P=Pg, grid=g, cta_offset=off, shared_counter=dealer.ptr)
            k2.pop("slow_first", None)
            eng.generate(d_cen, W, b, c, mode=mode, out=out, **k2)
            outs.append(out)
        torch.cuda.synchronize()
        return (outs[0] + outs[1]).cpu().numpy()
    finally:
        dealer.close()
        eng.close()


def test_fuzz_against_oracle(spin, torch):
    """Seeded random configurations (widths, bin sizes, support angles, modes, flags,
    pruning, every schedule incl. WF/AWF, P, unit, slow-worker emulation, schedules split
    over two launches sharing one dealer) on small structured clouds: NEAREST bit-exact and
    BILINEAR within tolerance against the oracle, CELLS = BRUTE."""
    # (SPIN_FUZZ_CASES / SPIN_FUZZ_SEED widen the campaign for one-off runs)
    rng = np.random.default_rng(int(os.environ.get("SPIN_FUZZ_SEED", "20261020")))
    kinds = ["bumpy", "clustered", "dyadic", "planar", "collinear"]
    scheds = ["STATIC", "SS", "GSS", "FAC", "WF", "AWF"]
    for case in range(int(os.environ.get("SPIN_FUZZ_CASES", "40"))):
        kind = kinds[case % len(kinds)]
        n = int(rng.integers(50, 1500))
        P, Nn, scale = _fuzz_cloud(rng, kind, n)
        M = int(rng.integers(1, 80))
        cen = rng.integers(0, n, size=M).astype(np.int32)
        W = int(rng.choice([2, 3, 4, 5, 8, 13, 16, 24, 32]))
        b = float(rng.choice([0.02, 0.05, 0.1, 0.25])) * scale
        c = float(rng.choice([0.5, 0.0, -0.5, -math.inf, math.cos(math.radians(37.0))]))
        mode = "nearest" if case % 2 == 0 else "bilinear"
        flags = int(rng.choice([0, 0, 0, 1, 2])) if mode == "nearest" else 0
        # knobs that must not change images: NO_SORT, NO_FAST_CERT, SUPPORT_LAST / FIRST,
        # CLUSTER_PAIR, NO_DENSE
        knobs = int(rng.choice([0, 0, 0x4, 0x8, 0x10, 0x20, 0x40, 0x80]))
        kw = dict(schedule=scheds[case % len(scheds)], P=int(rng.choice([0, 1, 5, 148])),
                  unit=int(rng.choice([0, 1, 3])), flags=flags | knobs)
        # heterogeneous-worker emulation (NEXT-1: timing only, never images)
        if rng.random() < 0.3:
            kw.update(slow_ctas=int(rng.integers(1, 40)), slowdown=float(rng.choice([2.0, 4.0])),
                      slow_first=bool(rng.random() < 0.5))
        split = kw["schedule"] not in ("WF", "AWF") and rng.random() < 0.25
        what = f"case {case} {kind} n={n} M={M} W={W} b={b:g} c={c:g} {mode} {kw} split={split}"
        if split:
            # one schedule dealt to two launches (the shared-dealer contract of NEXT-2):
            # global P, each launch its grid and cta_offset, one shared counter
            brute = _split_launches(spin, torch, P, Nn, cen, W, b, c, mode, kw)
        else:
            brute = run_gpu(spin, torch, P, Nn, cen, W, b, c, mode, **kw)
        ora, st = oracle(P, Nn, cen, W, b, c, mode, flags=flags)
        check(brute, ora, st, mode, what + " brute")
        cells = run_gpu(spin, torch, P, Nn, cen, W, b, c, mode, prune="cells", **kw)
        if mode == "nearest":
            np.testing.assert_array_equal(cells, brute, err_msg=what + " cells != brute")
        else:
            check(cells, ora, st, mode, what + " cells")


@pytest.mark.parametrize("mode", ["nearest", "bilinear"])
def test_dense_tiles_same_images(spin, torch, mode):
    """Dense lane-per-centre tiles (BRUTE on the Morton-ordered cloud): the
    default run takes them (tiles_dense > 0) and gives the images of the compaction-only
    control (SPIN_F_NO_DENSE) bit for bit, and the oracle's on a subsample; W = 32 runs the
    512-thread G = 32 launch, W = 16 / 8 the 768-thread G = 64 one (two centres per lane)."""
    P, Nn = clouds.bumpy_sphere(100000, 91)
    cen = np.arange(100000, dtype=np.int32)
    for W, b, c in ((32, 0.01, 0.0), (16, 0.02, 0.5), (8, 0.05, -math.inf)):
        got, st = run_gpu(spin, torch, P, Nn, cen, W, b, c, mode, stats=True)
        assert st["tiles_dense"] > 0 and st["dense_rows"] > 0, st
        assert st["G"] == (32 if W == 32 else 64), st
        ctl, st2 = run_gpu(spin, torch, P, Nn, cen, W, b, c, mode, stats=True, flags=spin.F_NO_DENSE)
        assert st2["tiles_dense"] == 0
        assert st["pairs_accepted"] == st2["pairs_accepted"]
        np.testing.assert_array_equal(got, ctl, err_msg=f"dense vs compaction W={W} {mode}")
        sub = cen[::997]
        ora, ost = oracle(P, Nn, sub, W, b, c, mode)
        check(got[sub], ora, ost, mode, f"dense W={W} {mode}")


def test_bilinear_near_normal_axis(spin, torch):
    """BILINEAR splat positions of points on or near a centre's normal axis (alpha << |d|):
    |d|^2 - beta^2 cancels there, so the GPU takes alpha^2 from Lagrange's identity
    (reading 25).  Oblique normals, off-origin centres, points at 0 to 1e-3
    rad off the axis across the whole beta window; both prunings."""
    rng = np.random.default_rng(5)
    for W, b in ((16, 0.02), (32, 0.01), (8, 0.05)):
        n0 = rng.normal(size=3)
        n0 /= np.linalg.norm(n0)
        t1 = np.cross(n0, [0.3, 0.5, 0.8])
        t1 /= np.linalg.norm(t1)
        P0 = np.array([0.4, -0.3, 0.6])
        xs = [P0]
        for u in np.linspace(0.05, W - 1.05, 23):
            beta = (W / 2 - u) * b
            for off in (0.0, 1e-6, 1e-5, 1e-4, 1e-3):
                xs.append(P0 + beta * n0 + off * abs(beta) * t1)
        X = np.asarray(xs, np.float32)
        Nn = np.tile(n0.astype(np.float32), (len(X), 1))
        cen = [0, 7, 40]
        ora, st = oracle(X, Nn, cen, W, b, 0.5, "bilinear")
        for prune in ("brute", "cells"):
            gpu = run_gpu(spin, torch, X, Nn, cen, W, b, 0.5, "bilinear", prune=prune)
            check(gpu, ora, st, "bilinear", f"near-axis W={W} {prune}")


@pytest.mark.filterwarnings("ignore:The CUDA Graph is empty")  # the refused stats capture
def test_cuda_graph_capture(spin, torch):
    """spin_generate can be captured in a CUDA graph after one uncaptured call (spin.h):
    replays reproduce the images (BRUTE and CELLS, whose centre-ordering kernels are part
    of the graph); stats inside a capture are refused."""
    P, Nn = clouds.bumpy_sphere(5000, 17)
    cen = _dev(torch, np.arange(0, 5000, 7, dtype=np.int32))
    eng = spin.SpinEngine(_dev(torch, P), _dev(torch, Nn))
    try:
        s = torch.cuda.Stream()
        for prune, mode in (("brute", "bilinear"), ("cells", "nearest")):
            out = torch.empty((cen.shape[0], 16, 16), dtype=torch.float32, device="cuda")
            with torch.cuda.stream(s):
                eng.generate(cen, 16, 0.02, 0.5, out=out, schedule="SS", prune=prune, mode=mode)
                torch.cuda.synchronize()
                ref = out.clone()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    eng.generate(cen, 16, 0.02, 0.5, out=out, schedule="SS", prune=prune, mode=mode)
                for _ in range(3):
                    out.zero_()
                    g.replay()
                    torch.cuda.synchronize()
                    assert torch.equal(out, ref), (prune, mode)
        with torch.cuda.stream(s):
            g2 = torch.cuda.CUDAGraph()
            with pytest.raises(spin.SpinError):
                with torch.cuda.graph(g2, stream=s):
                    eng.generate(cen, 16, 0.02, 0.5, schedule="SS", stats=True)
        torch.cuda.synchronize()
    finally:
        eng.close()


def test_failed_load_leaves_no_cloud(spin, torch):
    """A spin_load_cloud that fails validation on a live handle leaves NO cloud (never the
    old grid with new centres, stale bounds or NaN points): generate refuses with
    SPIN_E_INVAL until a good load, which then gives the oracle's images again."""
    P, Nn = clouds.bumpy_sphere(3000, 61)
    cen = _dev(torch, np.arange(0, 3000, 31, dtype=np.int32))
    eng = spin.SpinEngine(_dev(torch, P), _dev(torch, Nn))
    try:
        eng.generate(cen, 16, 0.02, 0.5, prune="cells")
        bad = P.copy()
        bad[100, 0] = np.nan
        with pytest.raises(spin.SpinError) as ei:
            eng.load_cloud(_dev(torch, bad), _dev(torch, Nn))
        assert ei.value.status == 3
        for prune in ("brute", "cells"):
            with pytest.raises(spin.SpinError) as ei:
                eng.generate(cen, 16, 0.02, 0.5, prune=prune)
            assert ei.value.status == 1 and "no valid cloud" in str(ei.value)
        eng.load_cloud(_dev(torch, P), _dev(torch, Nn))
        got = eng.generate(cen, 16, 0.02, 0.5, prune="cells").cpu().numpy()
        ora, _ = oracle(P, Nn, np.arange(0, 3000, 31), 16, 0.02, 0.5, "nearest")
        assert_nearest_exact(got, ora, "after a failed load")
    finally:
        eng.close()


def test_deferred_range_error_not_lost(spin, torch):
    """Back-to-back asynchronous calls: the first has an out-of-range centre index; the
    error must be reported by a later call (spin.h: "returned by the next call"), even
    though the second call's own readback is queued before anyone looks."""
    P, Nn = clouds.bumpy_sphere(2000, 62)
    eng = spin.SpinEngine(_dev(torch, P), _dev(torch, Nn))
    try:
        bad = _dev(torch, np.array([3, 5000, 4], np.int32))
        good = _dev(torch, np.array([1, 2], np.int32))
        eng.generate(bad, 8, 0.05, 0.5)          # asynchronous: no error yet
        # the second call reports it if the first call's readback has landed, else it is
        # queued behind it and the third call reports it (the device flag is sticky):
        # exactly once either way
        raised = []
        for _ in range(2):
            try:
                eng.generate(good, 8, 0.05, 0.5)
            except spin.SpinError as e:
                raised.append(e.status)
            torch.cuda.synchronize()
        assert raised == [2], raised
        eng.generate(good, 8, 0.05, 0.5, stats=True)   # reported once, then clean
    finally:
        eng.close()


def test_python_binding_refuses_bad_buffers(spin, torch):
    """spin.py validates dtype / shape / device of every buffer it passes (no silent
    reinterpretation of a float64 cloud, no overrun of a short output)."""
    P, Nn = clouds.bumpy_sphere(500, 63)
    with pytest.raises(ValueError):
        spin.SpinEngine(_dev(torch, P.astype(np.float64)), _dev(torch, Nn))
    eng = spin.SpinEngine(_dev(torch, P), _dev(torch, Nn))
    try:
        cen = _dev(torch, np.arange(10, dtype=np.int32))
        for out in (torch.empty((9, 8, 8), device="cuda"), torch.empty((10, 8, 8), dtype=torch.float64, device="cuda"),
                    torch.empty((10, 8, 8)), torch.empty((10, 8, 16), device="cuda")[:, :, :8]):
            with pytest.raises(ValueError):
                eng.generate(cen, 8, 0.05, 0.5, out=out)
        with pytest.raises(ValueError):
            eng.generate(cen.to(torch.int64), 8, 0.05, 0.5)
        with pytest.raises(ValueError):
            eng.generate_host(np.arange(10), 8, 0.05, 0.5, out=np.empty((10, 8, 7), np.float32))
    finally:
        eng.close()


@pytest.mark.parametrize("mode", ["nearest"])
def test_cluster_workers_w32(spin, torch, mode):
    """W = 28 / 32 BRUTE NEAREST on request (SPIN_F_CLUSTER_PAIR) runs on two-CTA clusters
    (one worker = a CTA pair sharing G = 48 images over DSMEM): every schedule x
    P x unit gives the oracle's images, units are dealt exactly once, and the one-CTA launches
    (the default: 512 threads, G = 32 with dense tiles; WF; slow-worker emulation) give the
    identical images."""
    P, Nn = clouds.bumpy_sphere(12000, 71)
    cen = np.arange(0, 12000, 23, dtype=np.int32)
    CL = spin.F_CLUSTER_PAIR
    for W, b in ((32, 0.01), (28, 0.012)):
        ora, st = oracle(P, Nn, cen, W, b, 0.0, mode)
        ref, s0 = run_gpu(spin, torch, P, Nn, cen, W, b, 0.0, mode, stats=True, schedule="SS",
                          cta_capacity=4096, flags=CL)
        assert s0["cta_per_worker"] == 2 and s0["G"] == 48, s0
        assert int(s0["cta_units"].sum()) == s0["n_units"]
        check(ref, ora, st, mode, f"cluster W={W} {mode}")
        for sched in ("STATIC", "SS", "GSS", "FAC"):
            for Pn in (1, 7, 0):
                for unit in (0, 1, 5):
                    got = run_gpu(spin, torch, P, Nn, cen, W, b, 0.0, mode, schedule=sched, P=Pn,
                                  unit=unit, flags=CL)
                    np.testing.assert_array_equal(got, ref, err_msg=f"W={W} {sched} P={Pn} u={unit}")
        for kw in (dict(schedule="SS"), dict(schedule="WF", flags=CL),
                   dict(schedule="SS", slow_ctas=20, slowdown=2.0, flags=CL)):
            got, s1 = run_gpu(spin, torch, P, Nn, cen, W, b, 0.0, mode, stats=True, **kw)
            assert s1["cta_per_worker"] == 1 and s1["G"] == 32, s1
            np.testing.assert_array_equal(got, ref, err_msg=str(kw))
