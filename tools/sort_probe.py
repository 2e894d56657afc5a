#!/usr/bin/env python
"""Probe: kernel time of a BRUTE config with the cloud in generator order vs Morton order
(the images are a permutation-invariant function of the cloud; centres = every point).

  python tools/sort_probe.py --config 4 [--mode nearest]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def morton_order(P, bits=10):
    lo, hi = P.min(0), P.max(0)
    q = ((P - lo) / np.maximum(hi - lo, 1e-30) * ((1 << bits) - 1)).astype(np.uint64)
    key = np.zeros(len(P), np.uint64)
    for b in range(bits):
        for a in range(3):
            key |= ((q[:, a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + a)
    return np.argsort(key, kind="stable")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--mode", default=None)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    from paper_1811_00901_b200 import spin
    from synth import clouds
    cfg = dict(clouds.CONFIGS[a.config])
    W, mode = cfg["W"], a.mode or cfg["mode"]
    P, Nn = clouds.make_cloud(a.config)
    perm = morton_order(P)
    for name, (PP, NN) in (("generator", (P, Nn)), ("morton", (P[perm], Nn[perm]))):
        cen = torch.arange(len(PP), dtype=torch.int32, device="cuda")
        eng = spin.SpinEngine(torch.from_numpy(np.ascontiguousarray(PP)).cuda(),
                              torch.from_numpy(np.ascontiguousarray(NN)).cuda())
        out = torch.empty((len(cen), W, W), dtype=torch.float32, device="cuda")
        ts = []
        for _ in range(a.reps + 1):
            _, st = eng.generate(cen, W, cfg["b"], cfg["cos_As"], mode=mode, prune=cfg["prune"],
                                 schedule="SS", out=out, stats=True)
            ts.append(st["elapsed_ms"])
        torch.cuda.synchronize()
        print(f"{cfg['name']} {mode} {name}: {min(ts[1:]):.3f} ms (all {['%.2f' % t for t in ts]}), "
              f"G={st['G']} cand={st['pairs_candidate']} acc={st['pairs_accepted']}", flush=True)
        eng.close()


if __name__ == "__main__":
    main()
