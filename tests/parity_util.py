"""Comparison helpers for GPU-vs-oracle parity (the bars of BASELINE.json north_star)."""
import numpy as np

REL_L1 = 1e-5      # per-image relative L1 (bilinear fp32 mode)
PER_BIN = 1e-4     # per-bin |err| <= PER_BIN * contributing points (floored at 1)


def assert_nearest_exact(gpu, ora, what=""):
    gpu = np.asarray(gpu, np.float64)
    ora = np.asarray(ora, np.float64)
    bad = np.argwhere(gpu != ora)
    assert bad.size == 0, f"{what}: {len(bad)} NEAREST bins differ, first {bad[:5].tolist()}"


def assert_bilinear_close(gpu, ora, contributors, what=""):
    """north star: per-image rel L1 <= 1e-5, per-bin |err| <= 1e-4 x contributors."""
    gpu = np.asarray(gpu, np.float64)
    ora = np.asarray(ora, np.float64)
    M = gpu.shape[0]
    err = np.abs(gpu - ora).reshape(M, -1)
    den = np.abs(ora).reshape(M, -1).sum(axis=1)
    num = err.sum(axis=1)
    zero = den == 0
    assert np.all(num[zero] == 0), f"{what}: nonzero GPU image where the oracle image is empty"
    rel = num[~zero] / den[~zero]
    assert rel.size == 0 or rel.max() <= REL_L1, f"{what}: max per-image rel L1 {rel.max():.3e}"
    cnt = np.maximum(np.asarray(contributors).reshape(M, -1), 1)
    ratio = err / (PER_BIN * cnt)
    assert ratio.max() <= 1.0, f"{what}: per-bin error {ratio.max():.3f}x the bound"
    return float(rel.max()) if rel.size else 0.0


def flip_counts(gpu_codes, ora_codes):
    """Per-pair decisions (spin_pair_codes vs the oracle's pair codes, -1 = no contribution,
    else the pair's bin / BILINEAR base corner i0*W + j0): returns (region mismatches =
    pairs only one side lets contribute, flips = pairs both let contribute at different
    (i0, j0), pairs both let contribute).  Region decisions are certified exact on both
    sides, so mismatches must be 0; NEAREST bins are exact, so NEAREST flips must be 0;
    BILINEAR flips are pairs within fp32 rounding of an interior bin edge, where the splat
    is continuous (north star: "bin-edge rounding flips counted and reported")."""
    g = np.asarray(gpu_codes)
    o = np.asarray(ora_codes)
    both = (g >= 0) & (o >= 0)
    return (int(np.count_nonzero((g >= 0) != (o >= 0))), int(np.count_nonzero(both & (g != o))),
            int(np.count_nonzero(both)))


def log_parity(record: dict):
    """Print one parity record and append it (JSON) to $SPIN_PARITY_LOG when set (the
    committed campaign logs under profiles/ come from this)."""
    import json
    import os
    line = json.dumps(record)
    print("PARITY", line)
    path = os.environ.get("SPIN_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(line + "\n")
