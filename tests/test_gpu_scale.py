"""GPU parity AT THE BASELINE SCALES: the CUDA path (through the C ABI, in bench.py's launch
configuration: SS, unit G, default P and flags) against the C++ oracle
(oracle/spin_oracle.cpp, pinned in tests/test_oracle_cpp.py), element by element.

Sample sizes are BASELINE.json / BASELINE.md's:
  C2  all 100,000 images (1e10 pairs), BILINEAR and NEAREST;
  C4  the seeded 1,000-image subsample (1e9 pairs; clouds.subsample(M, 1000, 204));
  C3  a seeded 2,000-centre oracle-BRUTE sample (both modes) plus a FULL oracle-CELLS run
      (all 200,000 images, BILINEAR), and GPU-CELLS == GPU-BRUTE over all images (NEAREST);
  C5  a seeded 5,000-centre oracle-BRUTE sample at W = 8 and W = 24 (NEAREST, bit-exact),
      and GPU-CELLS == GPU-BRUTE over all 500,000 images.
NEAREST must be bit-exact; BILINEAR within the north-star tolerance (per-image rel L1
<= 1e-5, per-bin |err| <= 1e-4 x contributors).  Per-pair decisions (spin_pair_codes) of 64
seeded images per config are compared with the oracle's: region mismatches must be 0,
NEAREST bins identical, BILINEAR interior-edge flips counted and reported (log_parity).
Definition checked: Alg. 1, under DESIGN.md §3's readings.
"""
import os
import numpy as np
import pytest

from oracle import spin_oracle_cpp as OC
from synth import clouds
from parity_util import assert_bilinear_close, assert_nearest_exact, flip_counts, log_parity

pytestmark = pytest.mark.gpu

FLIP_IMAGES = 64
MAX_FLIP_FRAC = 1e-3       # BILINEAR flips per contributing pair (measured ~1e-5)


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


class Run:
    """One full-size GPU run of a config in bench.py's launch configuration."""

    def __init__(self, spin, torch, cfg_id, mode, prune=None, W=None, sched="SS"):
        self.cfg = dict(clouds.CONFIGS[cfg_id])
        self.id = cfg_id
        self.W = W or self.cfg["W"]
        self.mode = mode
        self.prune = prune or self.cfg["prune"]
        self.P, self.Nn = clouds.make_cloud(cfg_id)
        self.cen = clouds.make_centres(cfg_id, self.cfg["N"])
        self.torch = torch
        self.eng = spin.SpinEngine(torch.from_numpy(self.P).cuda(), torch.from_numpy(self.Nn).cuda())
        self.d_cen = torch.from_numpy(self.cen).cuda()
        self.out, self.st = self.eng.generate(self.d_cen, self.W, self.cfg["b"], self.cfg["cos_As"],
                                              mode=mode, prune=self.prune, schedule=sched, stats=True)
        torch.cuda.synchronize()

    def rows(self, idx):
        return self.out[self.torch.from_numpy(np.asarray(idx, np.int64)).cuda()].cpu().numpy()

    def oracle(self, idx, cells=False):
        st = {}
        f = OC.generate_cells if cells else OC.generate
        img = f(self.P, self.Nn, self.cen[idx], self.W, self.cfg["b"], self.cfg["cos_As"],
                OC.NEAREST if self.mode == "nearest" else OC.BILINEAR, stats=st)
        return img, st

    def check(self, idx, what, cells=False):
        gpu = self.rows(idx)
        ora, st = self.oracle(idx, cells)
        rec = {"config": self.cfg["name"], "W": self.W, "mode": self.mode, "prune": self.prune,
               "check": what, "images": int(len(idx)), "oracle": "cells" if cells else "brute",
               "pairs_oracle": int(st["visited"]), "oracle_stage4_pairs": int(st["exact_pairs"])}
        if self.mode == "nearest":
            assert_nearest_exact(gpu, ora, f"{self.cfg['name']} {what}")
            rec["nearest_bins_differing"] = 0
        else:
            rec["max_rel_l1"] = assert_bilinear_close(gpu, ora, np.stack(st["contributors"]),
                                                      f"{self.cfg['name']} {what}")
        log_parity(rec)
        return gpu, ora

    def flips(self, n_img=FLIP_IMAGES, seed=None):
        """Per-pair decisions of n_img seeded images: GPU spin_pair_codes vs the oracle."""
        pick = clouds.subsample(len(self.cen), n_img, seed or (300 + self.id))
        m = OC.NEAREST if self.mode == "nearest" else OC.BILINEAR
        g = self.eng.pair_codes(self.d_cen[self.torch.from_numpy(pick).cuda()].contiguous(), self.W,
                                self.cfg["b"], self.cfg["cos_As"], mode=self.mode).cpu().numpy()
        o = OC.pair_codes(self.P, self.Nn, self.cen[pick], self.W, self.cfg["b"], self.cfg["cos_As"], m)
        region, flips, both = flip_counts(g, o)
        rec = {"config": self.cfg["name"], "W": self.W, "mode": self.mode, "check": "per-pair decisions",
               "images": n_img, "pairs": int(g.size), "contributing_pairs": both,
               "region_mismatches": region, "bin_flips": flips,
               "flip_fraction": flips / max(both, 1)}
        log_parity(rec)
        assert region == 0, rec
        if self.mode == "nearest":
            assert flips == 0, rec
        else:
            assert flips <= MAX_FLIP_FRAC * both, rec
        # the images of those pairs: the codes must rebuild the GPU's NEAREST images
        if self.mode == "nearest":
            W = self.W
            img = np.zeros((n_img, W * W))
            for i in range(n_img):
                c = g[i][g[i] >= 0]
                np.add.at(img[i], c, 1.0)
            np.testing.assert_array_equal(img.reshape(n_img, W, W), self.rows(pick))
        return rec

    def close(self):
        self.eng.close()


@pytest.mark.parametrize("mode", ["bilinear", "nearest"])
def test_c2_full(spin, torch, mode):
    """C2 in FULL: all 100,000 images (1e10 pairs) against the oracle."""
    r = Run(spin, torch, 2, mode)
    try:
        r.check(np.arange(len(r.cen)), "all images")
        if mode == "nearest":
            assert float(r.out.sum(dtype=torch.float64).item()) == r.st["pairs_accepted"]
        r.flips()
    finally:
        r.close()


def test_c4_subsample_1000(spin, torch):
    """C4 (1M x 1M, W = 32, BILINEAR): the seeded 1,000-image subsample BASELINE names."""
    r = Run(spin, torch, 4, "bilinear")
    try:
        r.check(clouds.subsample(len(r.cen), 1000, 204), "seeded 1,000-image subsample")
        r.flips()
    finally:
        r.close()


@pytest.mark.parametrize("mode", ["bilinear", "nearest"])
def test_c3_cells(spin, torch, mode):
    """C3 cell lists: a seeded 2,000-centre oracle-BRUTE sample; BILINEAR also against a
    FULL oracle-CELLS run (all 200,000 images); NEAREST GPU-CELLS == GPU-BRUTE in full."""
    r = Run(spin, torch, 3, mode)
    try:
        r.check(clouds.subsample(len(r.cen), 2000, 203), "seeded 2,000-centre oracle-BRUTE")
        if mode == "bilinear":
            r.check(np.arange(len(r.cen)), "all images, oracle-CELLS", cells=True)
        else:
            brute = r.eng.generate(r.d_cen, r.W, r.cfg["b"], r.cfg["cos_As"], mode=mode,
                                   prune="brute", schedule="SS")
            assert torch.equal(brute, r.out), "C3 NEAREST: GPU-CELLS != GPU-BRUTE"
            log_parity({"config": r.cfg["name"], "check": "GPU-CELLS == GPU-BRUTE, all images",
                        "mode": mode, "images": len(r.cen), "equal": True})
        r.flips()
    finally:
        r.close()


@pytest.mark.parametrize("W", [8, 24])
def test_c5_cells(spin, torch, W):
    """C5 (4M clustered points, densities over 100x, NEAREST bit-exact): a seeded
    5,000-centre oracle-BRUTE sample, and GPU-CELLS == GPU-BRUTE over all 500,000 images."""
    r = Run(spin, torch, 5, "nearest", W=W)
    try:
        r.check(clouds.subsample(len(r.cen), 5000, 205), "seeded 5,000-centre oracle-BRUTE")
        brute = r.eng.generate(r.d_cen, W, r.cfg["b"], r.cfg["cos_As"], mode="nearest",
                               prune="brute", schedule="SS")
        assert torch.equal(brute, r.out), f"C5 W={W}: GPU-CELLS != GPU-BRUTE"
        log_parity({"config": r.cfg["name"], "W": W, "check": "GPU-CELLS == GPU-BRUTE, all images",
                    "mode": "nearest", "images": len(r.cen), "equal": True})
        assert float(r.out.sum(dtype=torch.float64).item()) == r.st["pairs_accepted"]
        r.flips()
    finally:
        r.close()


def test_p6_paper_shape(spin, torch):
    """NEXT-3, the paper's own workload shape (826K points, W = 5, no support test): a
    seeded 2,000-image oracle sample, bit-exact."""
    r = Run(spin, torch, 6, "nearest")
    try:
        r.check(clouds.subsample(len(r.cen), 2000, 206), "seeded 2,000-image subsample")
        r.flips()
    finally:
        r.close()


@pytest.mark.skipif(os.environ.get("SPIN_WIDE") != "1", reason="one-off wide campaign (SPIN_WIDE=1)")
def test_wide_campaign(spin, torch):
    """One-off wider oracle samples on a build (not part of the default suite: ~10 minutes of
    oracle time): 20,000 seeded images each of C4 (both modes), C3 (both prunings), C5 W = 8
    and P6 against oracle-BRUTE; logged through SPIN_PARITY_LOG like the default checks."""
    n = int(os.environ.get("SPIN_WIDE_IMAGES", "20000"))
    for cfg_id, mode, prune, seed in ((4, "bilinear", None, 404), (4, "nearest", None, 405),
                                      (3, "bilinear", "cells", 403), (3, "nearest", "brute", 406),
                                      (5, "nearest", "cells", 407), (6, "nearest", None, 408)):
        r = Run(spin, torch, cfg_id, mode, prune=prune)
        try:
            r.check(clouds.subsample(len(r.cen), n, seed), f"wide: seeded {n}-image subsample")
        finally:
            r.close()
