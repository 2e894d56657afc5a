"""Pins of the oracle against things other than itself (CPU, `-m "not gpu"`).

Each test names the passage / closed form / invariant it pins.  A plausible slip
in the oracle (dropped term, wrong sign, transposed index, floor/ceil swap, an
un-scaled W/2, strict vs inclusive support test, a too-small error bound)
fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import spin_oracle as O
from synth import clouds

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


# ---------------------------------------------------------------- hand-worked X1-X4

@pytest.mark.parametrize("fn", ["generate", "exact"])
def test_x1_nearest_and_bilinear(fn):
    g = _load("x1.json")
    for mode, key in ((O.NEAREST, "nearest"), (O.BILINEAR, "bilinear")):
        if fn == "generate":
            img = O.generate(g["points"], g["normals"], [g["centre"]], g["W"], g["b"], _cos(g), mode)[0]
        else:
            img = O.exact_image(g["points"], g["normals"], g["centre"], g["W"], g["b"], _cos(g), mode)
        np.testing.assert_array_equal(img, np.asarray(g[key], np.float64), err_msg=key)


def test_x2_scaled_vs_literal():
    g = _load("x2.json")
    s = O.generate(g["points"], g["normals"], [0], g["W"], g["b"], _cos(g), O.NEAREST)[0]
    l = O.generate(g["points"], g["normals"], [0], g["W"], g["b"], _cos(g), O.NEAREST,
                   O.F_LITERAL_HALF_WIDTH)[0]
    np.testing.assert_array_equal(s, g["nearest_scaled"])
    np.testing.assert_array_equal(l, g["nearest_literal"])


def test_x3_odd_width_real_half():
    g = _load("x3.json")
    img = O.generate(g["points"], g["normals"], [0], g["W"], g["b"], _cos(g), O.NEAREST)[0]
    np.testing.assert_array_equal(img, g["nearest"])


def test_x4_inclusive_support_cosine_form():
    g = _load("x4.json")
    a = O.generate(g["points"], g["normals"], [0], g["W"], g["b"], 0.0, O.NEAREST)[0]
    c = O.generate(g["points"], g["normals"], [0], g["W"], g["b"], math.cos(math.pi / 2), O.NEAREST)[0]
    assert math.cos(math.pi / 2) > 0
    np.testing.assert_array_equal(a, g["cos_zero"])
    np.testing.assert_array_equal(c, g["cos_fl_half_pi"])


# ---------------------------------------------------------------- SPEC worked examples

def test_spec_project_and_bins():
    g = _load("spec_examples.json")
    p = np.zeros(3, np.float32)
    n = np.array([0, 0, 1], np.float32)
    for ex in g["project"]:
        # a point contributes at (k, l) = (ceil(W/2 - beta), ceil(alpha)) with W=8, b=1
        x = np.asarray(ex["x"], np.float32)
        kl = O.exact_pair(p, n, x, n, 8, 1.0, -math.inf, O.NEAREST)
        assert kl == (math.ceil(4 - ex["beta"]), math.ceil(ex["alpha"])), ex["cite"]
    for ex in g["bin_indices_W4_B1"]:
        x = np.array([ex["alpha"], 0, ex["beta"]], np.float32)
        for flags in (0, O.F_LITERAL_HALF_WIDTH):
            assert O.exact_pair(p, n, x, n, 4, 1.0, -math.inf, O.NEAREST, flags) == tuple(ex["kl"]), ex["cite"]
    s = g["self_W5_B0.1"]
    assert O.exact_pair(p, n, p, n, 5, 0.1, -math.inf, O.NEAREST, O.F_LITERAL_HALF_WIDTH) is None
    assert O.exact_pair(p, n, p, n, 5, 0.1, -math.inf, O.NEAREST) == tuple(s["scaled"])


def test_spec_support_examples():
    """identical normals pass; antipodal fails at pi/2; S = 2pi (cos -inf) passes."""
    p = np.zeros(3, np.float32)
    n = np.array([0, 0, 1], np.float32)
    x = np.array([0.5, 0, 0], np.float32)
    assert O.exact_pair(p, n, x, n, 4, 1.0, 0.0, O.NEAREST) is not None
    assert O.exact_pair(p, n, x, -n, 4, 1.0, math.cos(math.pi / 2), O.NEAREST) is None
    assert O.exact_pair(p, n, x, -n, 4, 1.0, -math.inf, O.NEAREST) is not None


# ---------------------------------------------------------------- config-1 closed form

def _closed_form_c1(W=8, b=0.05, cos_As=0.5, mode=O.NEAREST, n_t=4_000_000):
    """Expected non-self image for the unit sphere with radial normals.

    A point at angle theta from the centre has beta = cos(theta) - 1, alpha = sin(theta)
    and t = cos(theta) is uniform on [-1, 1] (density 1/2); integrate by the midpoint
    rule in t over [t0, 1], where t0 = 0.85 is below every contributing t
    (|X-P|^2 = 2 - 2t <= (2 * W * b)^2 = 0.64 needs t >= 0.68; the k-window needs
    beta >= (1 - W/2) b = -0.15, i.e. t >= 0.85).  Written from the geometry, not from
    the oracle's code.
    """
    t0 = max(cos_As, 0.85)
    t = t0 + (np.arange(n_t) + 0.5) * ((1.0 - t0) / n_t)
    wt = 0.5 * ((1.0 - t0) / n_t)
    beta = t - 1.0
    alpha = np.sqrt(np.maximum(1 - t * t, 0))
    u = W / 2.0 - beta / b
    v = alpha / b
    E = np.zeros((W, W))
    if mode == O.NEAREST:
        k = np.ceil(u).astype(int)
        l = np.ceil(v).astype(int)
        ok = (k >= 0) & (k < W) & (l >= 0) & (l < W)
        np.add.at(E, (k[ok], l[ok]), wt)
    else:
        i0 = np.floor(u).astype(int)
        j0 = np.floor(v).astype(int)
        ok = (i0 >= 0) & (i0 <= W - 2) & (j0 >= 0) & (j0 <= W - 2)
        a, c = u[ok] - i0[ok], v[ok] - j0[ok]
        i0, j0 = i0[ok], j0[ok]
        for di, dj, w in ((0, 0, (1 - a) * (1 - c)), (1, 0, a * (1 - c)), (0, 1, (1 - a) * c), (1, 1, a * c)):
            np.add.at(E, (i0 + di, j0 + dj), w * wt)
    return E


def test_closed_form_matches_appendix_a():
    """The integration itself reproduces SURVEY.md Appendix A's printed rows (x (N-1))."""
    E = _closed_form_c1() * 1999
    np.testing.assert_allclose(E[5], [0, 1.250, 3.760, 6.298, 8.886, 11.544, 14.300, 3.937], atol=2e-3)
    np.testing.assert_allclose(E[6], [0, 0, 0, 0, 0, 0, 0, 13.243], atol=2e-3)
    assert abs(E.sum() - 63.218) < 2e-2
    B = _closed_form_c1(mode=O.BILINEAR) * 1999
    np.testing.assert_allclose(B[4], [0.413, 2.409, 4.458, 5.772, 5.947, 4.534, 1.440, 0.013], atol=2e-3)
    np.testing.assert_allclose(B[5], [0.003, 0.094, 0.568, 1.815, 4.261, 8.379, 13.861, 7.497], atol=2e-3)


@pytest.mark.parametrize("mode", [O.NEAREST, O.BILINEAR])
def test_config1_closed_form_statistics(mode):
    """Oracle on config 1 (first 400 centres) vs the closed form, Poisson error bars."""
    cfg = clouds.CONFIGS[1]
    P, Nn = clouds.make_cloud(1)
    M = 400
    imgs = O.generate(P, Nn, np.arange(M), cfg["W"], cfg["b"], cfg["cos_As"], mode)
    mean = imgs.mean(axis=0)
    E = _closed_form_c1(mode=mode) * (cfg["N"] - 1)
    E[4, 0] += 1.0    # self pair: u = W/2 = 4 exactly, v = 0 (reading #8)
    tol = 6 * np.sqrt(np.maximum(E, 0.05) / M) + 1e-9
    assert np.all(np.abs(mean - E) <= tol), (mean - E)
    if mode == O.NEAREST:
        # exact structure: self at (4,0) in every image; support within {(4,0),(5,1..7),(6,7)}
        assert np.all(imgs[:, 4, 0] >= 1)
        allowed = np.zeros((8, 8), bool)
        allowed[4, 0] = True
        allowed[5, 1:8] = True
        allowed[6, 7] = True
        assert np.all(imgs[:, ~allowed] == 0)


# ---------------------------------------------------------------- invariants

def _dyadic_cloud(n, seed, grid=2.0 ** -12):
    """Coordinates on a 2^-12 grid in (-1, 1); normals are fp32 unit vectors."""
    rng = np.random.default_rng(seed)
    P = (np.round(rng.uniform(-1, 1, (n, 3)) / grid) * grid).astype(np.float32)
    g = rng.normal(size=(n, 3))
    Nn = (g / np.linalg.norm(g, axis=1, keepdims=True)).astype(np.float32)
    return P, Nn


@pytest.mark.parametrize("mode", [O.NEAREST, O.BILINEAR])
def test_total_weight_equals_in_region_count(mode):
    """north star: each in-support point contributes total weight exactly 1."""
    P, Nn = clouds.make_cloud(1, n=600)
    st = {}
    imgs = O.generate(P, Nn, np.arange(0, 600, 7), 8, 0.05, 0.5, mode, stats=st)
    tot = imgs.reshape(len(imgs), -1).sum(axis=1)
    np.testing.assert_allclose(tot, np.asarray(st["in_region"], np.float64), rtol=0, atol=1e-12)


@pytest.mark.parametrize("mode", [O.NEAREST, O.BILINEAR])
def test_rigid_motion_and_scale_invariance_dyadic(mode):
    """Signed permutations, dyadic translations and 2^k scaling (cloud and b) are exact."""
    P, Nn = _dyadic_cloud(300, 1)
    W, b, c = 8, 0.0625, 0.25
    cen = np.arange(0, 300, 11)
    ref = O.generate(P, Nn, cen, W, b, c, mode)
    rng = np.random.default_rng(7)
    for trial in range(3):
        perm = rng.permutation(3)
        sgn = rng.choice([-1.0, 1.0], 3).astype(np.float32)
        P2 = (P[:, perm] * sgn).astype(np.float32)
        N2 = (Nn[:, perm] * sgn).astype(np.float32)
        shift = (rng.integers(-64, 64, 3) * 2.0 ** -12).astype(np.float32)
        P2 = (P2 + shift).astype(np.float32)
        got = O.generate(P2, N2, cen, W, b, c, mode)
        if mode == O.NEAREST:
            np.testing.assert_array_equal(got, ref)
        else:
            np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)
    for k in (-3, 2):
        got = O.generate((P * 2.0 ** k).astype(np.float32), Nn, cen, W, b * 2.0 ** k, c, mode)
        np.testing.assert_array_equal(got, ref)


def test_duplicate_point_adds_its_increment():
    """duplicating point j adds exactly its own increment to each image."""
    P, Nn = clouds.make_cloud(2, n=3000)
    cen = np.arange(0, 3000, 97)
    W, b, c = 16, 0.02 * 8, 0.5
    ref = O.generate(P, Nn, cen, W, b, c, O.NEAREST)
    j = 5
    P2 = np.concatenate([P, P[j:j + 1]])
    N2 = np.concatenate([Nn, Nn[j:j + 1]])
    got = O.generate(P2, N2, cen, W, b, c, O.NEAREST)
    delta = got - ref
    for m, ci in enumerate(cen):
        r = O.exact_pair(P[ci], Nn[ci], P[j], Nn[j], W, b, c, O.NEAREST)
        exp = np.zeros((W, W))
        if r is not None:
            exp[r] = 1
        np.testing.assert_array_equal(delta[m], exp)


def test_order_invariance():
    P, Nn = clouds.make_cloud(3, n=4000)
    cen = clouds.sample_centres(4000, 40, 9)
    ref = O.generate(P, Nn, cen, 16, 0.02, 0.5, O.NEAREST)
    perm = np.random.default_rng(3).permutation(4000)
    inv = np.argsort(perm)
    got = O.generate(P[perm], Nn[perm], inv[cen], 16, 0.02, 0.5, O.NEAREST)
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("mode,flags", [(O.NEAREST, 0), (O.NEAREST, O.F_FLOOR_BINS),
                                        (O.BILINEAR, 0), (O.NEAREST, O.F_LITERAL_HALF_WIDTH)])
def test_cells_equals_brute(mode, flags):
    P, Nn = clouds.clustered(6000, 11)
    cen = clouds.sample_centres(6000, 60, 12)
    W, b = 8, 0.02
    if flags & O.F_LITERAL_HALF_WIDTH:
        W, b = 4, 0.1     # literal: beta window near W/2 = 2 (mostly empty but exercised)
    br = O.generate(P, Nn, cen, W, b, 0.5, mode, flags)
    ce = O.generate_cells(P, Nn, cen, W, b, 0.5, mode, flags)
    if mode == O.NEAREST:
        np.testing.assert_array_equal(ce, br)
    else:
        np.testing.assert_allclose(ce, br, rtol=0, atol=1e-12)


@pytest.mark.parametrize("mode,flags", [(O.NEAREST, 0), (O.NEAREST, O.F_FLOOR_BINS),
                                        (O.BILINEAR, 0), (O.NEAREST, O.F_LITERAL_HALF_WIDTH)])
def test_filtered_equals_exact_definition_with_ties(mode, flags):
    """Brute force on tiny inputs: the float64-filtered oracle equals the pure exact
    definition, on dyadic clouds where many pairs sit EXACTLY on bin edges (ties)."""
    P, Nn = _dyadic_cloud(70, 5, grid=2.0 ** -3)
    Nn[::3] = np.array([0, 0, 1], np.float32)          # exact axis normals -> exact ties
    Nn[1::3] = np.array([1, 0, 0], np.float32)
    W, b = 6, 0.25
    if flags & O.F_LITERAL_HALF_WIDTH:
        b = 1.0
    for c in (-math.inf, 0.0):
        st = {}
        got = O.generate(P, Nn, np.arange(70), W, b, c, mode, flags, stats=st)
        assert st["exact_pairs"] > 70                  # the tie path was exercised
        for ci in range(70):
            ex = O.exact_image(P, Nn, ci, W, b, c, mode, flags)
            if mode == O.NEAREST:
                np.testing.assert_array_equal(got[ci], ex)
            else:
                np.testing.assert_allclose(got[ci], ex, rtol=0, atol=1e-12)


def test_near_threshold_pairs_are_certified():
    """Points placed 1 ulp (fp32) on either side of a bin edge must land exactly per the
    exact definition; a filter bound that is too small would misplace some of them."""
    W, b = 16, 0.02
    p = np.zeros(3, np.float32)
    n = np.array([0, 0, 1], np.float32)
    xs = []
    for k in range(1, 15):
        edge = np.float32((W / 2 - k) * b)              # beta at a row edge
        for z in (np.nextafter(edge, np.float32(-1)), edge, np.nextafter(edge, np.float32(1))):
            xs.append([np.float32(0.05), 0, z])
        r = np.float32(k * b)                            # alpha at a column edge
        for xr in (np.nextafter(r, np.float32(0)), r, np.nextafter(r, np.float32(1))):
            xs.append([xr, 0, np.float32(0.01)])
    X = np.concatenate([p[None], np.asarray(xs, np.float32)])
    Nn = np.tile(n, (len(X), 1))
    got = O.generate(X, Nn, [0], W, b, -math.inf, O.NEAREST)[0]
    ex = O.exact_image(X, Nn, 0, W, b, -math.inf, O.NEAREST)
    np.testing.assert_array_equal(got, ex)


# ---------------------------------------------------------------- scheduling pins

def test_chunk_goldens():
    g = _load("chunks.json")
    assert O.chunk_sizes(O.GSS, 100, 4) == g["GSS_100_4"]
    assert O.chunk_sizes(O.FAC, 100, 4) == g["FAC_100_4"]
    assert O.chunk_sizes(O.SS, 100, 4) == [1] * g["SS_100_4_len"]
    assert O.chunk_sizes(O.STATIC, 10, 4) == g["STATIC_10_4"]
    assert O.chunk_sizes(O.STATIC, 7, 7) == g["STATIC_7_7"]
    for n, (gc, gf, fc, ff) in ((int(k), v) for k, v in g["appendix_c_P296"].items() if k != "cite"):
        gs = O.chunk_sizes(O.GSS, n, 296)
        fs = O.chunk_sizes(O.FAC, n, 296)
        assert (len(gs), gs[0], len(fs), fs[0]) == (gc, gf, fc, ff)


def test_chunk_properties_random():
    """coverage, positivity, GSS monotone head, FAC batch structure."""
    rng = np.random.default_rng(0)
    for _ in range(300):
        n = int(rng.integers(0, 100_000))
        P = int(rng.integers(1, 257))
        for kind in (O.STATIC, O.SS, O.GSS, O.FAC):
            if kind == O.SS and n > 20_000:
                continue
            s = O.chunk_sizes(kind, n, P)
            assert sum(s) == n and all(x >= 1 for x in s)
            if kind == O.STATIC:
                assert len(s) == min(P, n) and max(s, default=0) - min(s, default=0) <= 1
            if kind == O.GSS and n:
                assert s[0] == -(-n // P) and all(a >= b for a, b in zip(s, s[1:]))
            if kind == O.FAC:
                for i in range(0, len(s), P):
                    batch = s[i:i + P]
                    assert len(set(batch[:-1])) <= 1 and batch[-1] <= batch[0]


def test_metrics():
    assert O.parallel_cost(160, 25.0) == 4000.0          # SPEC S:366 (P:489-490 numbers)
    mx, cov = O.load_imbalance([1, 1, 1, 5])
    assert mx == 2.5 and abs(cov - math.sqrt(3) / 2) < 1e-12
    assert O.load_imbalance([5, 5, 5, 5]) == (1.0, 0.0)


def test_region_radius_bounds_contributors():
    """|X-P| <= R for every contributing pair (H5), and R is tight to within a bin."""
    P, Nn = clouds.clustered(5000, 4)
    for mode, flags in ((O.NEAREST, 0), (O.NEAREST, O.F_FLOOR_BINS), (O.BILINEAR, 0)):
        W, b = 8, 0.03
        R = O.region_radius(W, b, mode, flags)
        for ci in range(0, 5000, 250):
            d = np.linalg.norm(P.astype(np.float64) - P[ci], axis=1)
            for j in np.nonzero(d > R)[0][:200]:
                assert O.exact_pair(P[ci], Nn[ci], P[j], Nn[j], W, b, -math.inf, mode, flags) is None


def test_weighted_factoring_pins():
    """WF (beyond the paper, spin.h SPIN_WF): equal weights reproduce FAC2 (P:229-230,
    reading #15) exactly; a hand-derived heterogeneous golden; every batch of P chunks
    covers at least half of the units left at its start and the sizes tile n."""
    g = json.load(open(os.path.join(GOLD, "chunks.json")))
    assert O.chunk_sizes(O.WF, 100, 4, slow=1, slowdown=2.0) == g["WF_100_4_slow1_x2"]["sizes"]
    rng = np.random.default_rng(7)
    for _ in range(300):
        n = int(rng.integers(0, 20000))
        P = int(rng.integers(1, 300))
        f = int(rng.integers(1, 4))
        assert O.chunk_sizes(O.WF, n, P, fac_divisor=f) == O.chunk_sizes(O.FAC, n, P, fac_divisor=f)
        S = int(rng.integers(0, P + 1))
        sd = float(rng.uniform(1.0, 8.0))
        s = O.chunk_sizes(O.WF, n, P, fac_divisor=f, slow=S, slowdown=sd)
        assert sum(s) == n and all(c >= 1 for c in s)
        wq = O.wf_integer_weights(P, S, sd)
        R = n
        for b in range(0, len(s), P):
            batch = s[b:b + P]
            left = R - sum(batch)
            if left > 0:
                # a complete batch hands out at least R_batch * sum(wq) / (f P 1024) units
                assert len(batch) == P
                assert sum(batch) * f * P * 1024 >= R * sum(wq)
                # and a slow worker never gets more than a fast one
                if 0 < S < P:
                    assert max(batch[:S]) <= min(batch[S:])
            R = left


def test_bilinear_on_the_normal_axis():
    """Points on the centre's normal axis have alpha = 0 exactly: all their BILINEAR weight
    lies in column 0, split between rows i0 = floor(u) and i0 + 1 by a = u - i0 with
    u = W/2 - beta/b (reading 12; the GPU's near-axis splat, reading 25, is
    checked against this).  Dyadic inputs: every step is exact."""
    W, b = 8, 0.25
    zs = [-0.75, -0.5, -0.3125, 0.0625, 0.5, 0.8125]
    X = np.array([[0.0, 0.0, 0.0]] + [[0.0, 0.0, z] for z in zs], np.float32)
    Nn = np.tile(np.array([0.0, 0.0, 1.0], np.float32), (len(X), 1))
    img = O.generate(X, Nn, [0], W, b, -math.inf, O.BILINEAR)[0]
    exp = np.zeros((W, W))
    for z in [0.0] + zs:
        u = W / 2 - z / b
        i0 = math.floor(u)
        if 0 <= i0 <= W - 2:
            exp[i0, 0] += 1 - (u - i0)
            exp[i0 + 1, 0] += u - i0
    assert np.array_equal(img, exp)
    assert np.all(img[:, 1:] == 0)
