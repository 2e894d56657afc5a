#!/usr/bin/env python
"""One warm-up + one measured spin_generate call of a config (the command the ncu captures
in profiles/ run: `ncu -k regex:spin_persistent -s 1 -c 1 python tools/one_call.py ...`).

  python tools/one_call.py --config 4 [--mode nearest] [--W 24] [--schedule SS]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--mode", default=None)
    ap.add_argument("--W", type=int, default=None)
    ap.add_argument("--schedule", default="SS")
    ap.add_argument("--flags", type=lambda v: int(v, 0), default=0)
    a = ap.parse_args()
    import torch
    from paper_1811_00901_b200 import spin
    from synth import clouds
    cfg = dict(clouds.CONFIGS[a.config])
    W = a.W or cfg["W"]
    mode = a.mode or cfg["mode"]
    P, Nn = clouds.make_cloud(a.config)
    cen = torch.from_numpy(clouds.make_centres(a.config, cfg["N"])).cuda()
    eng = spin.SpinEngine(torch.from_numpy(P).cuda(), torch.from_numpy(Nn).cuda())
    out = torch.empty((len(cen), W, W), dtype=torch.float32, device="cuda")
    for _ in range(2):
        _, st = eng.generate(cen, W, cfg["b"], cfg["cos_As"], mode=mode, prune=cfg["prune"],
                             schedule=a.schedule, out=out, stats=True, flags=a.flags)
    torch.cuda.synchronize()
    print(f"{cfg['name']} W={W} {mode}: {st['elapsed_ms']:.3f} ms, G={st['G']}, "
          f"cta_per_worker={st['cta_per_worker']}, candidates={st['pairs_candidate']}, "
          f"accepted={st['pairs_accepted']}, tiles_dense={st['tiles_dense']}, dense_rows={st['dense_rows']}")
    eng.close()


if __name__ == "__main__":
    main()
