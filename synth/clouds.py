"""Seeded synthetic oriented-point clouds shaped like the paper's workloads.

This module is the ONE piece shared by the oracle side (tests, bench's
cpu_baseline) and the CUDA side (tests, bench, smoke): it produces INPUTS only
and holds none of the spin-image arithmetic.  The paper's dataset (the 3-D mesh
watermarking set, Ramesses ~826K points, Table `tab:dataset`)
is not available, so these clouds stand in for it (SURVEY.md §8(d)
"Generators").

Randomness: a counter-based SplitMix64, u64 = mix(seed*PHI + (stream << 40) + i),
so every draw is a pure function of (seed, stream, index) and any sub-range can be
regenerated independently.  Uniforms are (u >> 11) * 2^-53 in [0, 1); Gaussians use
Box-Muller on two uniforms.  Geometry is computed in float64 and rounded to
float32 (round-to-nearest) once at the end: the fp32 arrays are THE inputs.

Streams: 0 positions/directions, 1 normals, 2 positional noise, 3 cluster/bump
parameters, 4 centre sampling.
"""
from __future__ import annotations

import numpy as np

_PHI = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def rand_u64(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * _PHI + (np.uint64(stream) << np.uint64(40))
        return _mix(base + idx)


def uniform(seed: int, stream: int, idx) -> np.ndarray:
    """U[0,1) float64, counter-based."""
    return (rand_u64(seed, stream, idx) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def gaussian(seed: int, stream: int, idx) -> np.ndarray:
    """N(0,1) float64 via Box-Muller on draws (2i, 2i+1)."""
    idx = np.asarray(idx, dtype=np.uint64)
    u1 = uniform(seed, stream, idx * np.uint64(2))
    u2 = uniform(seed, stream, idx * np.uint64(2) + np.uint64(1))
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


def gaussian3(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    i = np.arange(offset, offset + n, dtype=np.uint64)
    return np.stack([gaussian(seed, stream, 3 * i + np.uint64(k)) for k in range(3)], axis=1)


def unit3(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    g = gaussian3(seed, stream, n, offset)
    return g / np.linalg.norm(g, axis=1, keepdims=True)


def _f32(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _f32_unit(v: np.ndarray) -> np.ndarray:
    """Round a float64 unit vector to fp32 (|n| stays within ~1e-7 of 1)."""
    v = v / np.linalg.norm(v, axis=1, keepdims=True)
    return _f32(v)


# --------------------------------------------------------------------------- clouds

def sphere(n: int, seed: int):
    """Config 1: points uniform on the unit sphere, normals = the same radial vectors.

    The position and the normal are bit-identical fp32 vectors.
    """
    w = _f32_unit(unit3(seed, 0, n))
    return w.copy(), w.copy()


def _bumps(seed: int, nb: int = 32):
    c = unit3(seed, 3, nb)
    a = 0.2 * uniform(seed, 3, np.arange(1000, 1000 + nb))
    w = 0.1 + 0.3 * uniform(seed, 3, np.arange(2000, 2000 + nb))
    return c, a, w


def bumpy_sphere(n: int, seed: int, chunk: int = 1 << 18):
    """Configs 2 and 4: unit sphere radius perturbed by 32 Gaussian bumps.

    r(w) = 1 + sum_k a_k exp(-|w - c_k|^2 / (2 w_k^2)) (chordal distance),
    a_k ~ U[0, 0.2], w_k ~ U[0.1, 0.4], c_k uniform on S^2;
    x = r(w) w + N(0, 0.002^2 I);  n = normalize(r w - grad_S r), the analytic
    normal of the noise-free surface (BASELINE.json configs[1], configs[3]).
    """
    c, a, wd = _bumps(seed)
    P = np.empty((n, 3), np.float32)
    Nn = np.empty((n, 3), np.float32)
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        w = unit3(seed, 0, m, s)
        diff = w[:, None, :] - c[None, :, :]               # (m, 32, 3)
        d2 = np.einsum("mkj,mkj->mk", diff, diff)
        e = a[None, :] * np.exp(-d2 / (2.0 * wd[None, :] ** 2))
        r = 1.0 + e.sum(axis=1)
        g = np.einsum("mk,mkj->mj", -e / (wd[None, :] ** 2), diff)   # grad of r in R^3
        gs = g - np.einsum("mj,mj->m", g, w)[:, None] * w             # tangential part
        nrm = r[:, None] * w - gs
        x = r[:, None] * w + 0.002 * gaussian3(seed, 2, m, s)
        P[s:s + m] = x
        Nn[s:s + m] = _f32_unit(nrm)
    return P, Nn


def clustered(n: int, seed: int, n_clusters: int = 8, background_frac: float = 0.1,
              sigma: float = 0.03, density_span: float = 1.0, blend: float = 0.5):
    """Configs 3 and 5: Gaussian clusters plus a uniform background in [0,1]^3.

    Cluster means ~ U[0.15, 0.85]^3; cluster points mu_k + sigma N(0, I).
    Cluster point counts: equal (density_span=1) or weights 10^U[0, log10(span)]
    normalised with largest-remainder rounding (config 5 uses span 100).
    Normals: background random unit vectors; cluster points
    normalize(rhat + blend * ghat), rhat = (x - mu)/|x - mu|, ghat random unit.
    """
    n_bg = int(round(n * background_frac))
    n_cl = n - n_bg
    mu = 0.15 + 0.7 * uniform(seed, 3, np.arange(3 * n_clusters)).reshape(n_clusters, 3)
    if density_span > 1.0:
        wts = 10.0 ** (np.log10(density_span) * uniform(seed, 3, np.arange(500, 500 + n_clusters)))
    else:
        wts = np.ones(n_clusters)
    share = wts / wts.sum() * n_cl
    cnt = np.floor(share).astype(np.int64)
    rem = n_cl - int(cnt.sum())
    order = np.argsort(-(share - cnt), kind="stable")
    cnt[order[:rem]] += 1
    P = np.empty((n, 3), np.float64)
    Nn = np.empty((n, 3), np.float64)
    pos = 0
    for k in range(n_clusters):
        m = int(cnt[k])
        off = g_off = pos
        g = gaussian3(seed, 0, m, off)
        x = mu[k] + sigma * g
        rhat = g / np.maximum(np.linalg.norm(g, axis=1, keepdims=True), 1e-300)
        ghat = unit3(seed, 1, m, g_off)
        P[pos:pos + m] = x
        Nn[pos:pos + m] = rhat + blend * ghat
        pos += m
    i = np.arange(pos, n, dtype=np.uint64)
    P[pos:] = np.stack([uniform(seed, 0, 3 * i + np.uint64(k)) for k in range(3)], axis=1)
    Nn[pos:] = unit3(seed, 1, n - pos, pos)
    return _f32(P), _f32_unit(Nn)


def sample_centres(n_points: int, m: int, seed: int) -> np.ndarray:
    """M distinct indices in [0, N), in random (key) order, from stream 4."""
    if m > n_points:
        raise ValueError("cannot draw more distinct centres than points")
    keys = rand_u64(seed, 4, np.arange(n_points, dtype=np.uint64))
    return np.argsort(keys, kind="stable")[:m].astype(np.int32)


# --------------------------------------------------------------------------- configs

# BASELINE.json configs (N = points, M = images), with SURVEY.md §8(c) #25 readings
# where the config is silent (support 60 deg for C3/C5; C3 bilinear; C5 nearest).
CONFIGS = {
    1: dict(name="C1-sphere2k", kind="sphere", N=2000, M=2000, W=8, b=0.05, deg=60.0, cos_As=0.5,
            mode="bilinear", prune="brute", centres="iota"),
    2: dict(name="C2-bumpy100k", kind="bumpy", N=100_000, M=100_000, W=16, b=0.02, deg=60.0, cos_As=0.5,
            mode="bilinear", prune="brute", centres="iota"),
    3: dict(name="C3-clustered1M", kind="clustered", N=1_000_000, M=200_000, W=16, b=0.01,
            deg=60.0, cos_As=0.5, mode="bilinear", prune="cells", centres="random"),
    4: dict(name="C4-bumpy1M-W32", kind="bumpy", N=1_000_000, M=1_000_000, W=32, b=0.01,
            deg=90.0, cos_As=0.0, mode="bilinear", prune="brute", centres="iota"),
    5: dict(name="C5-clustered4M", kind="clustered", N=4_000_000, M=500_000, W=8, b=0.005,
            deg=60.0, cos_As=0.5, mode="nearest", prune="cells", centres="random", density_span=100.0),
    # the paper's own workload shape -- an ~826K-point closed surface
    # standing in for the Ramesses mesh (not available), W = 5, B = 0.1, S = 2 pi
    # (support test disabled), paper-N = 10% of the points; b taken as an
    # absolute length (reading #11), counts (Alg. 1 increments) with real W/2 (#3)
    6: dict(name="P6-paper826k", kind="bumpy", N=826_000, M=82_600, W=5, b=0.1, deg=360.0,
            cos_As=float("-inf"), mode="nearest", prune="brute", centres="iota"),
}


def make_cloud(cfg_id: int, n: int | None = None):
    """(points fp32 [N,3], normals fp32 [N,3]) for a config; seed = config number."""
    cfg = CONFIGS[cfg_id]
    n = cfg["N"] if n is None else n
    if cfg["kind"] == "sphere":
        return sphere(n, cfg_id)
    if cfg["kind"] == "bumpy":
        return bumpy_sphere(n, cfg_id)
    return clustered(n, cfg_id, density_span=cfg.get("density_span", 1.0))


def make_centres(cfg_id: int, n_points: int, m: int | None = None) -> np.ndarray:
    cfg = CONFIGS[cfg_id]
    m = cfg["M"] if m is None else m
    if cfg["centres"] == "iota":
        return np.arange(m, dtype=np.int32)
    return sample_centres(n_points, m, 100 + cfg_id)


def subsample(m_total: int, k: int, seed: int) -> np.ndarray:
    """k distinct positions in [0, m_total) for oracle subsamples (seed 200 + config)."""
    keys = rand_u64(seed, 5, np.arange(m_total, dtype=np.uint64))
    return np.sort(np.argsort(keys, kind="stable")[:k])
