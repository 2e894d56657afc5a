"""ORACLE for the spin-image hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this module.  The product path
(`paper_1811_00901_b200`, `libspin.so`) never imports, links or executes it, and
this module imports nothing from the product path: the two share no code
(DESIGN.md "Oracle").

What it computes is the plain definition of the paper's Algorithm 1
(`calculateSpinImages`, `algo:spin`; per-chunk form Alg. 2
`adCalculateSpinImages`) under the readings of SURVEY.md §8(c)
(each listed in DESIGN.md "Readings"):

  for every centre P = OP[c] and every point X = OP[j] (j = c included, #8):
      support   acos(np_i . np_j) <= S   read as   n.nx >= cos_As   (#5, #6)
      beta  = n.(X - P)
      alpha = sqrt(|X - P|^2 - beta^2)
      u = W/2 - beta/b   (scaled reading #2; flag LITERAL: (W/2 - beta)/b)
      v = alpha / b
      NEAREST : k = ceil(u), l = ceil(v)  (flag FLOOR: floor)      (#4)
                if 0 <= k < W and 0 <= l < W: image[k, l] += 1
      BILINEAR: i0 = floor(u), j0 = floor(v); if 0 <= i0 <= W-2 and
                0 <= j0 <= W-2 split weight 1 over the 4 corners   (#12, not in the paper)

Precision reading (#14): the result is defined in EXACT real arithmetic on the
fp32 inputs, with b and cos_As taken as exact doubles.  The oracle evaluates
every pair in float64 with a certified forward error bound per decision; a pair
whose float64 margin does not exceed its bound is re-decided exactly with
`fractions.Fraction` (`exact_pair`).  So every integer decision equals the exact
one.  BILINEAR weights are then evaluated in float64 (they are continuous inside
the region, so the exactly-decided region plus float64 weights is the
definition to ~1e-15).

Pins (tests/test_oracle_pins.py, `-m "not gpu"`): hand-worked clouds X1-X4
(tests/golden/*.json), SPEC.md:118-138 examples, the config-1 closed form
(SURVEY.md Appendix A), total-weight and duplicate invariants, rigid-motion and
scale invariance on dyadic clouds, order invariance, CELLS == BRUTE, and the
chunk-sequence goldens.  The BILINEAR splat rule itself is
"parity unpinned" by the paper (it is not in the paper; #12): it is pinned only
by X1 and its own invariants.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

NEAREST, BILINEAR = 0, 1
F_LITERAL_HALF_WIDTH = 1   # u = (W/2 - beta)/b, the formula exactly as printed
F_FLOOR_BINS = 2           # NEAREST k, l with floor instead of the paper's ceil (Johnson)

_U = 2.0 ** -53            # float64 unit roundoff


# ============================================================================ exact

def _fr(v) -> Fraction:
    return Fraction(float(v))


def _ceil_sqrt_rational(w: Fraction) -> int:
    """Smallest integer m >= 0 with m^2 >= w (w >= 0), exactly."""
    if w <= 0:
        return 0
    m = math.isqrt(w.numerator // w.denominator)
    while m * m < w:
        m += 1
    while m > 0 and (m - 1) * (m - 1) >= w:
        m -= 1
    return m


def _floor_sqrt_rational(w: Fraction) -> int:
    """Largest integer m >= 0 with m^2 <= w (w >= 0), exactly."""
    if w <= 0:
        return 0
    m = math.isqrt(w.numerator // w.denominator)
    while (m + 1) * (m + 1) <= w:
        m += 1
    while m * m > w:
        m -= 1
    return m


def exact_pair(p, n, x, nx, W: int, b: float, cos_As: float, mode: int, flags: int = 0):
    """Alg. 1 lines 10-16 for ONE (centre, point) pair in exact arithmetic.

    Returns None when the point does not contribute.
      NEAREST : (k, l)
      BILINEAR: (i0, j0, a, c) with weights (1-a)(1-c), a(1-c), (1-a)c, ac on
                (i0,j0), (i0+1,j0), (i0,j0+1), (i0+1,j0+1)
    """
    P = [_fr(t) for t in p]
    Nn = [_fr(t) for t in n]
    X = [_fr(t) for t in x]
    NX = [_fr(t) for t in nx]
    B = _fr(b)
    # support test  acos(np_i . np_j) <= S  <=>  np_i . np_j >= cos S   (#5/#6)
    if cos_As != -math.inf:
        s = Nn[0] * NX[0] + Nn[1] * NX[1] + Nn[2] * NX[2]
        if s < _fr(cos_As):
            return None
    d = [X[i] - P[i] for i in range(3)]
    beta = Nn[0] * d[0] + Nn[1] * d[1] + Nn[2] * d[2]                    # np_i . (X - P)
    q = d[0] * d[0] + d[1] * d[1] + d[2] * d[2] - beta * beta           # ||X-P||^2 - beta^2
    if q < 0:
        q = Fraction(0)                                                # clamp
    half = Fraction(W, 2)                                              # W/2 real (#3)
    if flags & F_LITERAL_HALF_WIDTH:
        u = (half - beta) / B
    else:
        u = half - beta / B
    w = q / (B * B)                                                    # v^2 = alpha^2 / b^2
    if mode == NEAREST:
        if flags & F_FLOOR_BINS:
            k = math.floor(u)
            l = _floor_sqrt_rational(w)
        else:
            k = math.ceil(u)
            l = _ceil_sqrt_rational(w)
        if 0 <= k < W and 0 <= l < W:
            return (k, l)
        return None
    # BILINEAR
    i0 = math.floor(u)
    if not (0 <= i0 <= W - 2):
        return None
    if not (w < (W - 1) * (W - 1)):                                   # j0 = floor(v) <= W-2
        return None
    j0 = _floor_sqrt_rational(w)
    a = float(u - i0)
    v = math.sqrt(float(w))
    c = min(max(v - j0, 0.0), 1.0)
    return (i0, j0, a, c)


def exact_image(points, normals, c: int, W: int, b: float, cos_As: float, mode: int,
                flags: int = 0) -> np.ndarray:
    """The definition written out: one image by exact pair evaluation over ALL points.

    Pure-Python loop; for tiny clouds only (pins and filter cross-checks).
    """
    img = np.zeros((W, W), np.float64)
    for j in range(len(points)):
        r = exact_pair(points[c], normals[c], points[j], normals[j], W, b, cos_As, mode, flags)
        if r is None:
            continue
        if mode == NEAREST:
            img[r[0], r[1]] += 1.0
        else:
            i0, j0, a, cc = r
            img[i0, j0] += (1 - a) * (1 - cc)
            img[i0 + 1, j0] += a * (1 - cc)
            img[i0, j0 + 1] += (1 - a) * cc
            img[i0 + 1, j0 + 1] += a * cc
    return img


# ============================================================================ float64 + certification

def region_radius(W: int, b: float, mode: int, flags: int = 0) -> float:
    """Upper bound on |X - P| for any contributing pair.

    |X-P|^2 = alpha^2 + beta^2 exactly (alpha^2 := |X-P|^2 - beta^2), so the bound is
    sqrt(alpha_max^2 + beta_absmax^2) from the u- and v-ranges that contribute.
    """
    if mode == NEAREST and not (flags & F_FLOOR_BINS):
        u_lo, u_hi, v_max = -1.0, W - 1.0, W - 1.0          # ceil: k in [0,W) <=> u in (-1, W-1]
    elif mode == NEAREST:
        u_lo, u_hi, v_max = 0.0, float(W), float(W)          # floor: u in [0, W), v < W
    else:
        u_lo, u_hi, v_max = 0.0, W - 1.0, W - 1.0            # bilinear: u in [0, W-1), v < W-1
    if flags & F_LITERAL_HALF_WIDTH:
        betas = [W / 2.0 - u_lo * b, W / 2.0 - u_hi * b]      # beta = W/2 - u b
    else:
        betas = [(W / 2.0 - u_lo) * b, (W / 2.0 - u_hi) * b]  # beta = (W/2 - u) b
    bmax = max(abs(t) for t in betas)
    return math.sqrt((v_max * b) ** 2 + bmax ** 2) * (1.0 + 1e-12) + 1e-300


def _dist_to_int(x: np.ndarray) -> np.ndarray:
    return np.abs(x - np.rint(x))


def _dist_to_square(w: np.ndarray) -> np.ndarray:
    """Distance from w to the nearest perfect square m^2, m >= 0 (w may be < 0)."""
    r = np.floor(np.sqrt(np.maximum(w, 0.0)))
    best = np.abs(w)                                  # m = 0
    for dm in (-1.0, 0.0, 1.0, 2.0):
        m = np.maximum(r + dm, 0.0)
        best = np.minimum(best, np.abs(w - m * m))
    return best


def pair_decisions(p, n, X, Nx, W: int, b: float, cos_As: float, mode: int, flags: int = 0):
    """Vectorised float64 evaluation of Alg. 1's per-pair test for one centre.

    p, n: (3,) fp32 centre; X, Nx: (K, 3) fp32 points.  Every operation is a single
    IEEE float64 op (no fused multiply-add), so the bounds below hold:
      products of two fp32 values are exact in float64; each + - * / sqrt adds a
      relative error <= u = 2^-53.  Bounds are taken with generous constants.
    Returns dict with the contributions of CERTIFIED pairs and the indices of
    pairs that must be decided exactly.
    """
    p = p.astype(np.float64)
    n = n.astype(np.float64)
    X = X.astype(np.float64)
    Nx = Nx.astype(np.float64)
    K = X.shape[0]
    unsure = np.zeros(K, bool)
    # --- support: s = n . nx, three exact products, two additions
    if cos_As != -math.inf:
        t0, t1, t2 = n[0] * Nx[:, 0], n[1] * Nx[:, 1], n[2] * Nx[:, 2]
        s = (t0 + t1) + t2
        es = 4 * _U * (np.abs(t0) + np.abs(t1) + np.abs(t2))
        ok_s = s >= cos_As
        unsure |= np.abs(s - cos_As) <= es
    else:
        ok_s = np.ones(K, bool)
    # --- projection
    d0, d1, d2 = X[:, 0] - p[0], X[:, 1] - p[1], X[:, 2] - p[2]          # |err| <= u|d_i|
    b0, b1, b2 = n[0] * d0, n[1] * d1, n[2] * d2
    beta = (b0 + b1) + b2
    eb = 6 * _U * (np.abs(b0) + np.abs(b1) + np.abs(b2))
    dd = (d0 * d0 + d1 * d1) + d2 * d2
    edd = 6 * _U * dd
    bb = beta * beta
    q = dd - bb
    eq = edd + (2 * np.abs(beta) + eb) * eb + 2 * _U * (bb + np.abs(q))
    # --- u (row coordinate) and w = v^2 = q / b^2 (column coordinate squared)
    half = W / 2.0
    if flags & F_LITERAL_HALF_WIDTH:
        t = half - beta
        u = t / b
        eu = (eb + _U * np.abs(t)) / b * (1 + 4 * _U) + 2 * _U * np.abs(u)
    else:
        t = beta / b
        u = half - t
        eu = eb / b * (1 + 4 * _U) + 2 * _U * (np.abs(t) + np.abs(u))
    b2 = b * b
    w = q / b2
    ew = eq / b2 * (1 + 6 * _U) + 4 * _U * np.abs(w)
    # a tiny absolute floor so that exactly-representable ties always go exact
    eu = eu + 1e-300
    ew = ew + 1e-300
    if mode == NEAREST:
        unsure |= _dist_to_int(u) <= eu
        unsure |= _dist_to_square(w) <= ew
        if flags & F_FLOOR_BINS:
            k = np.floor(u)
            l = np.floor(np.sqrt(np.maximum(w, 0.0)))
        else:
            k = np.ceil(u)
            l = np.ceil(np.sqrt(np.maximum(w, 0.0)))
        # l from sqrt is exact when w is certified away from squares, but re-derive
        # it from the square thresholds to be independent of sqrt rounding:
        lf = l.copy()
        if not (flags & F_FLOOR_BINS):
            lf = np.where((lf > 0) & ((lf - 1) ** 2 >= w), lf - 1, lf)
            lf = np.where(lf * lf < w, lf + 1, lf)
        else:
            lf = np.where(lf * lf > w, lf - 1, lf)
            lf = np.where((lf + 1) ** 2 <= w, lf + 1, lf)
        inside = ok_s & (k >= 0) & (k < W) & (lf >= 0) & (lf < W)
        return dict(inside=inside & ~unsure, k=k.astype(np.int64), l=lf.astype(np.int64),
                    unsure=np.nonzero(unsure)[0])
    # BILINEAR region: 0 <= u < W-1  and  w < (W-1)^2
    unsure |= np.abs(u) <= eu
    unsure |= np.abs(u - (W - 1)) <= eu
    unsure |= np.abs(w - (W - 1) ** 2) <= ew
    inside = ok_s & (u >= 0) & (u < W - 1) & (w < (W - 1) ** 2)
    v = np.sqrt(np.maximum(w, 0.0))
    i0 = np.clip(np.floor(u), 0, W - 2)
    j0 = np.clip(np.floor(v), 0, W - 2)
    a = np.clip(u - i0, 0.0, 1.0)
    c = np.clip(v - j0, 0.0, 1.0)
    return dict(inside=inside & ~unsure, i0=i0.astype(np.int64), j0=j0.astype(np.int64),
                a=a, c=c, unsure=np.nonzero(unsure)[0])


def _splat(img, cnt, dec, idx, mode, W):
    if mode == NEAREST:
        np.add.at(img, (dec["k"][idx], dec["l"][idx]), 1.0)
        return
    i0, j0, a, c = dec["i0"][idx], dec["j0"][idx], dec["a"][idx], dec["c"][idx]
    for di, dj, wt in ((0, 0, (1 - a) * (1 - c)), (1, 0, a * (1 - c)),
                       (0, 1, (1 - a) * c), (1, 1, a * c)):
        np.add.at(img, (i0 + di, j0 + dj), wt)
        if cnt is not None:
            np.add.at(cnt, (i0 + di, j0 + dj), (wt > 0).astype(np.int64))


def _image_from_candidates(points, normals, ci, cand, W, b, cos_As, mode, flags, stats):
    img = np.zeros((W, W), np.float64)
    cnt = np.zeros((W, W), np.int64) if mode == BILINEAR else None
    X, Nx = points[cand], normals[cand]
    dec = pair_decisions(points[ci], normals[ci], X, Nx, W, b, cos_As, mode, flags)
    sel = np.nonzero(dec["inside"])[0]
    _splat(img, cnt, dec, sel, mode, W)
    n_in = len(sel)
    for t in dec["unsure"]:
        r = exact_pair(points[ci], normals[ci], X[t], Nx[t], W, b, cos_As, mode, flags)
        if r is None:
            continue
        n_in += 1
        if mode == NEAREST:
            img[r[0], r[1]] += 1.0
        else:
            i0, j0, a, c = r
            for di, dj, wt in ((0, 0, (1 - a) * (1 - c)), (1, 0, a * (1 - c)),
                               (0, 1, (1 - a) * c), (1, 1, a * c)):
                img[i0 + di, j0 + dj] += wt
                cnt[i0 + di, j0 + dj] += int(wt > 0)
    if stats is not None:
        stats["exact_pairs"] = stats.get("exact_pairs", 0) + len(dec["unsure"])
        stats.setdefault("in_region", []).append(n_in)
        if cnt is not None:
            stats.setdefault("contributors", []).append(cnt)
    return img


def generate(points, normals, centre_idx, W: int, b: float, cos_As: float, mode: int,
             flags: int = 0, stats: dict | None = None) -> np.ndarray:
    """Oracle-BRUTE: images[m] for centre_idx[m], every point visited (Alg. 1).

    points, normals: (N, 3) float32; centre_idx: (M,) int.  Returns (M, W, W) float64.
    Optional `stats` collects in-region counts, per-bin contributor counts (BILINEAR)
    and the number of pairs decided exactly.
    """
    points = np.asarray(points, np.float32)
    normals = np.asarray(normals, np.float32)
    allidx = np.arange(len(points))
    out = np.zeros((len(centre_idx), W, W), np.float64)
    for m, ci in enumerate(np.asarray(centre_idx)):
        out[m] = _image_from_candidates(points, normals, int(ci), allidx, W, b, cos_As,
                                        mode, flags, stats)
    return out


class CellGrid:
    """Oracle-CELLS grid: an independent uniform grid with edge h = 1.0001 * R.

    Any point within distance R of a centre lies in the 27 cells around the centre's
    cell, so visiting them and applying the same per-pair decision reproduces
    Oracle-BRUTE exactly (pinned by tests/test_oracle_pins.py::test_cells_equals_brute).
    """

    def __init__(self, points, R: float):
        self.h = 1.0001 * R
        P = np.asarray(points, np.float64)
        self.origin = P.min(axis=0)
        self.key3 = np.floor((P - self.origin) / self.h).astype(np.int64)
        self.dims = self.key3.max(axis=0) + 1
        key = self._lin(self.key3)
        self.order = np.argsort(key, kind="stable")
        self.sorted_keys = key[self.order]

    def _lin(self, k3):
        return (k3[..., 2] * self.dims[1] + k3[..., 1]) * self.dims[0] + k3[..., 0]

    def neighbours(self, p) -> np.ndarray:
        c = np.floor((np.asarray(p, np.float64) - self.origin) / self.h).astype(np.int64)
        out = []
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    k3 = c + np.array([dx, dy, dz])
                    if np.any(k3 < 0) or np.any(k3 >= self.dims):
                        continue
                    key = self._lin(k3)
                    lo = np.searchsorted(self.sorted_keys, key, "left")
                    hi = np.searchsorted(self.sorted_keys, key, "right")
                    out.append(self.order[lo:hi])
        return np.concatenate(out) if out else np.zeros(0, np.int64)


def generate_cells(points, normals, centre_idx, W: int, b: float, cos_As: float, mode: int,
                   flags: int = 0, stats: dict | None = None) -> np.ndarray:
    """Oracle-CELLS: same per-pair decision, candidates from the 27-cell neighbourhood."""
    points = np.asarray(points, np.float32)
    normals = np.asarray(normals, np.float32)
    grid = CellGrid(points, region_radius(W, b, mode, flags))
    out = np.zeros((len(centre_idx), W, W), np.float64)
    for m, ci in enumerate(np.asarray(centre_idx)):
        cand = np.sort(grid.neighbours(points[int(ci)]))
        out[m] = _image_from_candidates(points, normals, int(ci), cand, W, b, cos_As,
                                        mode, flags, stats)
    return out


# ============================================================================ scheduling

STATIC, SS, GSS, FAC, WF, AWF = 0, 1, 2, 3, 4, 5


def wf_integer_weights(P: int, slow: int, slowdown: float):
    """Weighted factoring's relative speeds for the heterogeneous-worker emulation
    (spin.h SPIN_WF): slow workers 1/slowdown, the rest 1, normalised to mean 1, as
    integers round(1024 w) (at least 1)."""
    S = min(max(slow, 0), P)
    ws = 1.0 / slowdown if slowdown > 1.0 else 1.0
    mean = (S * ws + (P - S)) / P
    return [max(1, math.floor(1024.0 * (ws if i < S else 1.0) / mean + 0.5)) for i in range(P)]


def chunk_sizes(kind: int, n: int, P: int, gss_min_chunk: int = 1, fac_divisor: int = 2,
                slow: int = 0, slowdown: float = 1.0):
    """Chunk sizes of the paper's loop schedules (§2.2).

    STATIC: P near-equal blocks, the first n mod P of size ceil(n/P) (#17)
    SS    : one iteration per request
    GSS   : ceil(remaining / P) per request, at least gss_min_chunk (#16)
    FAC   : batches of P equal chunks, ceil(R_batch / (fac_divisor * P)) (P:229-230,
            FAC2 reading #15)
    WF    : weighted factoring (beyond the paper, its future work P:238): batches of P
            chunks, worker i's chunk ceil(R_batch * wq_i / (fac_divisor * P * 1024)),
            requests in round-robin worker order; with equal weights it is FAC
    Every chunk is capped at the remaining count and is at least 1.
    """
    if P < 1 or n < 0:
        raise ValueError("need P >= 1 and n >= 0")
    sizes = []
    if kind == STATIC:
        q, r = divmod(n, P)
        for i in range(min(P, n) if n < P else P):
            sizes.append(q + 1 if i < r else q)
        return [s for s in sizes if s > 0]
    R = n
    if kind == SS:
        return [1] * n
    if kind == GSS:
        while R > 0:
            c = min(R, max(gss_min_chunk, -(-R // P)))
            sizes.append(c)
            R -= c
        return sizes
    if kind == FAC:
        while R > 0:
            c = max(1, -(-R // (fac_divisor * P)))
            for _ in range(P):
                if R == 0:
                    break
                t = min(c, R)
                sizes.append(t)
                R -= t
        return sizes
    if kind == WF:
        wq = wf_integer_weights(P, slow, slowdown)
        worker = 0
        while R > 0:
            R_batch = R
            for _ in range(P):
                if R == 0:
                    break
                want = -(-(R_batch * wq[worker]) // (fac_divisor * P * 1024))
                t = min(max(1, want), R)
                sizes.append(t)
                R -= t
                worker = (worker + 1) % P
        return sizes
    raise ValueError("unknown schedule")


def chunk_bounds(kind: int, n: int, P: int, **kw):
    """[0, b1, b2, ..., n] boundaries of the chunk sequence."""
    out = [0]
    for s in chunk_sizes(kind, n, P, **kw):
        out.append(out[-1] + s)
    return out


# ============================================================================ metrics

def parallel_cost(P: int, t_par: float) -> float:
    """Parallel cost = resources x parallel time."""
    return P * t_par


def load_imbalance(times):
    """(max/mean, population CoV) of finishing times (fig:loadim P:194-207)."""
    t = np.asarray(times, np.float64)
    if t.size == 0 or np.any(t <= 0):
        raise ValueError("need non-empty positive times")
    mean = t.mean()
    return float(t.max() / mean), float(t.std() / mean)
