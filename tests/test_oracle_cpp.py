"""Pins of the C++ oracle (oracle/spin_oracle.cpp) against things other than itself
(CPU, `-m "not gpu"`).

The C++ oracle is what the at-scale GPU parity tests compare against (it is ~50x faster
than the numpy oracle).  It is pinned the same way the Python oracle is — hand-worked
goldens X1-X4 (Alg. 1 lines P:166-174), the config-1 closed form
(SURVEY Appendix A), total weight = in-region count, exact rigid-motion / scale invariance
on dyadic clouds, CELLS == BRUTE — and, because it shares no code with the Python oracle
(different language, different decision structure: threshold form with measured rounding
errors, double -> __float128 -> exact), by element-wise equality with it on seeded clouds
that include dyadic clouds full of exact ties.  Its three escalation stages are each
forced on every pair and must reproduce the same images.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import spin_oracle as PY
from oracle import spin_oracle_cpp as C
from synth import clouds
from test_oracle_pins import _closed_form_c1, _dyadic_cloud

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        g = json.load(f)
    g["points"] = np.asarray(g.get("points", []), np.float32)
    g["normals"] = np.asarray(g.get("normals", []), np.float32)
    return g


def _cos(g):
    v = g.get("cos_As", "-inf")
    return -math.inf if v == "-inf" else float(v)


FORCES = [0, C.F_FORCE_STAGE2, C.F_FORCE_STAGE3, C.F_FORCE_STAGE4]


# ---------------------------------------------------------------- hand-worked X1-X4

@pytest.mark.parametrize("force", FORCES)
def test_x1_goldens(force):
    g = _load("x1.json")
    for mode, key in ((C.NEAREST, "nearest"), (C.BILINEAR, "bilinear")):
        img = C.generate(g["points"], g["normals"], [g["centre"]], g["W"], g["b"], _cos(g), mode,
                         force)[0]
        np.testing.assert_array_equal(img, np.asarray(g[key], np.float64), err_msg=f"{key} {force}")


@pytest.mark.parametrize("force", FORCES)
def test_x2_x3_x4_goldens(force):
    g = _load("x2.json")
    s = C.generate(g["points"], g["normals"], [0], g["W"], g["b"], _cos(g), C.NEAREST, force)[0]
    lit = C.generate(g["points"], g["normals"], [0], g["W"], g["b"], _cos(g), C.NEAREST,
                     C.F_LITERAL_HALF_WIDTH | force)[0]
    np.testing.assert_array_equal(s, g["nearest_scaled"])
    np.testing.assert_array_equal(lit, g["nearest_literal"])
    g = _load("x3.json")
    img = C.generate(g["points"], g["normals"], [0], g["W"], g["b"], _cos(g), C.NEAREST, force)[0]
    np.testing.assert_array_equal(img, g["nearest"])
    g = _load("x4.json")
    a = C.generate(g["points"], g["normals"], [0], g["W"], g["b"], 0.0, C.NEAREST, force)[0]
    c = C.generate(g["points"], g["normals"], [0], g["W"], g["b"], math.cos(math.pi / 2),
                   C.NEAREST, force)[0]
    np.testing.assert_array_equal(a, g["cos_zero"])
    np.testing.assert_array_equal(c, g["cos_fl_half_pi"])


# ---------------------------------------------------------------- closed form and invariants

@pytest.mark.parametrize("mode", [C.NEAREST, C.BILINEAR])
def test_config1_closed_form(mode):
    """Config 1 in FULL (2,000 images) vs SURVEY Appendix A's closed form (Poisson bars)."""
    cfg = clouds.CONFIGS[1]
    P, Nn = clouds.make_cloud(1)
    imgs = C.generate(P, Nn, np.arange(cfg["M"]), cfg["W"], cfg["b"], cfg["cos_As"], mode)
    M = len(imgs)
    E = _closed_form_c1(mode=mode) * (cfg["N"] - 1)
    E[4, 0] += 1.0          # the self pair (reading #8)
    tol = 6 * np.sqrt(np.maximum(E, 0.05) / M) + 1e-9
    assert np.all(np.abs(imgs.mean(axis=0) - E) <= tol)
    if mode == C.NEAREST:
        allowed = np.zeros((8, 8), bool)
        allowed[4, 0] = True
        allowed[5, 1:8] = True
        allowed[6, 7] = True
        assert np.all(imgs[:, 4, 0] >= 1) and np.all(imgs[:, ~allowed] == 0)


@pytest.mark.parametrize("mode", [C.NEAREST, C.BILINEAR])
def test_total_weight_and_contributors(mode):
    """Each in-region pair contributes total weight exactly 1 (north star); BILINEAR
    contributor counts are at least the weight of every bin."""
    P, Nn = clouds.bumpy_sphere(5000, 3)
    st = {}
    imgs = C.generate(P, Nn, np.arange(0, 5000, 37), 16, 0.02, 0.5, mode, stats=st)
    tot = imgs.reshape(len(imgs), -1).sum(axis=1)
    np.testing.assert_allclose(tot, np.asarray(st["in_region"], np.float64), rtol=0, atol=1e-11)
    assert tot.sum() > 1000
    if mode == C.BILINEAR:
        cnt = np.stack(st["contributors"])
        assert np.all(imgs <= cnt + 1e-12) and np.all((cnt > 0) | (imgs == 0))


@pytest.mark.parametrize("mode", [C.NEAREST, C.BILINEAR])
def test_rigid_motion_and_scale_invariance_dyadic(mode):
    P, Nn = _dyadic_cloud(300, 1)
    W, b, c = 8, 0.0625, 0.25
    cen = np.arange(0, 300, 11)
    ref = C.generate(P, Nn, cen, W, b, c, mode)
    rng = np.random.default_rng(7)
    for _ in range(3):
        perm = rng.permutation(3)
        sgn = rng.choice([-1.0, 1.0], 3).astype(np.float32)
        P2 = (P[:, perm] * sgn).astype(np.float32)
        N2 = (Nn[:, perm] * sgn).astype(np.float32)
        P2 = (P2 + (rng.integers(-64, 64, 3) * 2.0 ** -12).astype(np.float32)).astype(np.float32)
        got = C.generate(P2, N2, cen, W, b, c, mode)
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 if mode else 0)
    for k in (-3, 2):
        got = C.generate((P * 2.0 ** k).astype(np.float32), Nn, cen, W, b * 2.0 ** k, c, mode)
        np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("mode,flags", [(C.NEAREST, 0), (C.NEAREST, C.F_FLOOR_BINS),
                                        (C.BILINEAR, 0), (C.NEAREST, C.F_LITERAL_HALF_WIDTH)])
def test_cells_equals_brute(mode, flags):
    P, Nn = clouds.clustered(8000, 11)
    cen = clouds.sample_centres(8000, 300, 12)
    W, b = (4, 0.1) if flags & C.F_LITERAL_HALF_WIDTH else (8, 0.02)
    sb, sc = {}, {}
    br = C.generate(P, Nn, cen, W, b, 0.5, mode, flags, stats=sb)
    ce = C.generate_cells(P, Nn, cen, W, b, 0.5, mode, flags, stats=sc)
    # (BILINEAR: the cell order changes only the order of the double sums)
    np.testing.assert_allclose(ce, br, rtol=0, atol=1e-12 if mode else 0)
    if not flags & C.F_LITERAL_HALF_WIDTH:      # (literal: R ~ W/2 covers the cloud)
        assert sc["visited"] < sb["visited"] / 3
    assert abs(C.region_radius(W, b, mode, flags) - PY.region_radius(W, b, mode, flags)) < 1e-8


# ---------------------------------------------------------------- against the Python oracle

def _cases():
    P1, N1 = clouds.bumpy_sphere(3000, 41)
    P2, N2 = clouds.clustered(4000, 42)
    P3, N3 = _dyadic_cloud(250, 43, grid=2.0 ** -3)
    N3[::3] = np.array([0, 0, 1], np.float32)          # exact axis normals: exact ties
    N3[1::3] = np.array([1, 0, 0], np.float32)
    P4 = (P1.astype(np.float64) + [300.0, -200.0, 500.0]).astype(np.float32)
    P5 = (P2.astype(np.float64) * 1e-3).astype(np.float32)
    return [("bumpy", P1, N1, 16, 0.02), ("clustered", P2, N2, 8, 0.02),
            ("dyadic-ties", P3, N3, 6, 0.25), ("far", P4, N1, 16, 0.02),
            ("tiny", P5, N2, 8, 2e-5)]


@pytest.mark.parametrize("case", range(5))
def test_equals_python_oracle(case):
    """Element-wise equality with the Python oracle (independently pinned), every mode and
    flag, several support angles: NEAREST bit-exact, BILINEAR to 1e-12, identical in-region
    counts and contributor counts."""
    name, P, Nn, W, b = _cases()[case]
    cen = np.arange(0, len(P), max(1, len(P) // 40))
    for mode, flags in ((C.NEAREST, 0), (C.NEAREST, C.F_FLOOR_BINS), (C.BILINEAR, 0),
                        (C.NEAREST, C.F_LITERAL_HALF_WIDTH)):
        bb = 1.0 if (flags & C.F_LITERAL_HALF_WIDTH and name == "dyadic-ties") else b
        for c in (0.5, -math.inf, 0.0):
            sp, sc = {}, {}
            a = PY.generate(P, Nn, cen, W, bb, c, mode, flags, stats=sp)
            g = C.generate(P, Nn, cen, W, bb, c, mode, flags, stats=sc)
            what = f"{name} mode={mode} flags={flags} c={c}"
            if mode == C.NEAREST:
                np.testing.assert_array_equal(g, a, err_msg=what)
            else:
                np.testing.assert_allclose(g, a, rtol=0, atol=1e-12, err_msg=what)
                np.testing.assert_array_equal(np.stack(sc["contributors"]), np.stack(sp["contributors"]))
            assert sc["in_region"] == sp["in_region"], what
            if name == "dyadic-ties":
                # exact ties: stage 2 (measured roundings) decides nearly all of them
                assert sc["stage2_pairs"] > 50 and sc["exact_pairs"] <= sc["stage2_pairs"] // 4, sc


@pytest.mark.parametrize("force", [C.F_FORCE_STAGE2, C.F_FORCE_STAGE3])
def test_threshold_stages_on_every_pair(force):
    """Stage 2 (threshold form, double with measured roundings) and stage 3 (__float128)
    forced on EVERY pair reproduce the stage-1 images (and the Python oracle's) on a
    surface, a volume and a tie-laden dyadic cloud."""
    for name, P, Nn, W, b in _cases()[:3]:
        cen = np.arange(0, len(P), max(1, len(P) // 12))
        for mode, flags in ((C.NEAREST, 0), (C.NEAREST, C.F_FLOOR_BINS), (C.BILINEAR, 0)):
            ref = C.generate(P, Nn, cen, W, b, 0.5, mode, flags)
            st = {}
            got = C.generate(P, Nn, cen, W, b, 0.5, mode, flags | force, stats=st)
            np.testing.assert_array_equal(got, ref, err_msg=f"{name} {mode} {flags} {force}")
            assert st["stage2_pairs" if force == C.F_FORCE_STAGE2 else "stage3_pairs"] == len(cen) * len(P)


def test_exact_stage_on_every_pair_tiny():
    """Stage 4 (the exact rational decision) on every pair of a tiny tie-laden cloud equals
    the floating stages."""
    P, Nn = _dyadic_cloud(40, 5, grid=2.0 ** -3)
    Nn[::3] = np.array([0, 0, 1], np.float32)
    for mode in (C.NEAREST, C.BILINEAR):
        ref = C.generate(P, Nn, np.arange(40), 6, 0.25, 0.0, mode)
        got = C.generate(P, Nn, np.arange(40), 6, 0.25, 0.0, mode, C.F_FORCE_STAGE4)
        # (BILINEAR weights from exact u, v rounded once vs double u, v: 1e-15 apart)
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 if mode else 0)


def test_near_threshold_ulps():
    """Points 1 fp32 ulp either side of every row / column edge decide exactly."""
    W, b = 16, 0.02
    p = np.zeros(3, np.float32)
    n = np.array([0, 0, 1], np.float32)
    xs = []
    for k in range(0, W + 2):
        edge = np.float32((W / 2 - k) * b)
        for z in (np.nextafter(edge, np.float32(-1)), edge, np.nextafter(edge, np.float32(1))):
            xs.append([np.float32(0.05), 0, z])
        r = np.float32(k * b)
        for xr in (np.nextafter(r, np.float32(0)), r, np.nextafter(r, np.float32(1))):
            xs.append([xr, 0, np.float32(0.01)])
    X = np.concatenate([p[None], np.asarray(xs, np.float32)])
    Nn = np.tile(n, (len(X), 1))
    for mode in (C.NEAREST, C.BILINEAR):
        got = C.generate(X, Nn, [0], W, b, -math.inf, mode)[0]
        ex = PY.exact_image(X, Nn, 0, W, b, -math.inf, mode)
        np.testing.assert_allclose(got, ex, rtol=0, atol=1e-12 if mode else 0)


def test_pair_bins_rebuild_the_image():
    """pair_bins (the per-pair decisions used for the BILINEAR flip count) rebuild exactly
    the images generate() returns."""
    P, Nn = clouds.bumpy_sphere(4000, 8)
    for mode in (C.NEAREST, C.BILINEAR):
        for c in (17, 2500):
            st, k, l, u, v = C.pair_bins(P, Nn, c, 16, 0.02, 0.5, mode)
            img = np.zeros((16, 16))
            sel = np.nonzero(st == 1)[0]
            if mode == C.NEAREST:
                np.add.at(img, (k[sel], l[sel]), 1.0)
            else:
                a = np.clip(u[sel] - k[sel], 0, 1)
                cc = np.clip(v[sel] - l[sel], 0, 1)
                for di, dj, wt in ((0, 0, (1 - a) * (1 - cc)), (1, 0, a * (1 - cc)),
                                   (0, 1, (1 - a) * cc), (1, 1, a * cc)):
                    np.add.at(img, (k[sel] + di, l[sel] + dj), wt)
            ref = C.generate(P, Nn, [c], 16, 0.02, 0.5, mode)[0]
            np.testing.assert_allclose(img, ref, rtol=0, atol=1e-12)
