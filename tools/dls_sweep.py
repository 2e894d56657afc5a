#!/usr/bin/env python
"""DLS sweep: STATIC / SS / GSS / FAC x resident-CTA count x unit on one config.

The paper's experiment (§5: 15 repetitions, min/max/mean/median/Q1/Q3,
P:456; rank finishing times, fig:loadim P:194-207; parallel cost P x T) on
one B200: the "workers" are the persistent CTAs, the "master" is the device chunk
counter.  Prints one JSON line per (policy, P, unit) and a summary of which
policies beat STATIC (median below STATIC's median and Q3 below STATIC's Q1,
SURVEY.md §8(d)).

  python tools/dls_sweep.py --config 3 --reps 15 [--mode nearest] [--P 0,148,296]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def quartiles(x):
    x = np.sort(np.asarray(x, np.float64))
    q = np.quantile(x, [0.0, 0.25, 0.5, 0.75, 1.0])   # inclusive linear interpolation
    return dict(min=q[0], q1=q[1], median=q[2], q3=q[3], max=q[4], mean=float(x.mean()))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--mode", default=None)
    ap.add_argument("--W", type=int, default=None)
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--P", default="0")
    ap.add_argument("--units", default="0,1")
    ap.add_argument("--policies", default="STATIC,SS,GSS,FAC",
                    help="STATIC,SS,GSS,FAC,WF,AWF and HW (one CTA per unit, the hardware block "
                         "scheduler as the dealer: the non-persistent control of SURVEY 8(d))")
    ap.add_argument("--no-sort", action="store_true")
    # heterogeneous-worker emulation: CTAs 0..slow-1 run `slowdown` x slower
    ap.add_argument("--slow", type=int, default=0, help="number of slow CTAs")
    ap.add_argument("--slowdown", type=float, default=0.0)
    ap.add_argument("--slow-first", action="store_true", help="slow CTAs request first (P:449, P:564)")
    ap.add_argument("--steps-tag", default="")
    args = ap.parse_args(argv)

    import torch
    from paper_1811_00901_b200 import spin
    from synth import clouds
    from bench import ClockSampler          # clocks during every line's repetitions

    cfg = dict(clouds.CONFIGS[args.config])
    W = args.W or cfg["W"]
    mode = args.mode or cfg["mode"]
    P, Nn = clouds.make_cloud(args.config)
    cen = clouds.make_centres(args.config, cfg["N"])
    eng = spin.SpinEngine(torch.from_numpy(P).cuda(), torch.from_numpy(Nn).cuda())
    d_cen = torch.from_numpy(cen).cuda()
    out = torch.empty((len(cen), W, W), dtype=torch.float32, device="cuda")
    flags = spin.F_NO_SORT if args.no_sort else 0
    ref = None
    results = {}
    lastP = 0
    for Pn in [int(x) for x in args.P.split(",")]:
        for unit in [int(x) for x in args.units.split(",")]:
            for pol in args.policies.split(","):
                if pol == "SS" and unit == 1 and len(cen) > 20000:
                    continue   # one image per request: G-fold wasted slots, skip at scale
                sched, Pp = pol, Pn
                if pol == "HW":   # non-persistent control: STATIC with one unit per CTA
                    G0 = eng.generate(d_cen[:1], W, cfg["b"], cfg["cos_As"], mode=mode, prune=cfg["prune"],
                                      stats=True)[1]["G"]
                    sched, Pp = "STATIC", -(-len(cen) // (unit or G0))
                kw = dict(schedule=sched, mode=mode, prune=cfg["prune"], P=Pp, unit=unit,
                          flags=flags, out=out, slow_ctas=args.slow, slowdown=args.slowdown,
                          slow_first=args.slow_first)
                eng.generate(d_cen, W, cfg["b"], cfg["cos_As"], **kw)   # warm-up
                times, busy_max_over_mean, busy_cov, finish_cov = [], [], [], []
                st = None
                clock = ClockSampler(torch.cuda.current_device())
                clock.start()
                for _ in range(args.reps):
                    _, st = eng.generate(d_cen, W, cfg["b"], cfg["cos_As"], stats=True,
                                         cta_capacity=4096, **kw)
                    times.append(st["elapsed_ms"])
                    npc = min(st["P"], 4096)
                    t0 = st["cta_start_ns"][:npc].astype(np.float64)
                    t1 = st["cta_end_ns"][:npc].astype(np.float64)
                    fin = t1 - t0.min()
                    busy = t1 - t0
                    busy_max_over_mean.append(busy.max() / busy.mean())
                    busy_cov.append(busy.std() / busy.mean())
                    finish_cov.append(fin.std() / fin.mean())
                torch.cuda.synchronize()
                clocks = clock.stop()
                if ref is None:
                    ref = out.clone()
                elif mode == "nearest" or True:
                    assert torch.equal(out, ref), f"{pol} P={Pn} unit={unit} changed the images"
                q = quartiles(times)
                if pol != "HW":
                    lastP = st["P"]
                key = (pol, lastP if pol == "HW" else st["P"], unit or st["G"])
                results[key] = q
                print(json.dumps({"config": cfg["name"], "W": W, "mode": mode, "policy": pol,
                                  "slow_ctas": args.slow, "slowdown": args.slowdown,
                                  "slow_first": args.slow_first,
                                  "P": st["P"], "unit": unit or st["G"], "G": st["G"],
                                  "n_chunks": st["n_chunks"], "ms": q,
                                  "parallel_cost_cta_s": st["P"] * q["median"] * 1e-3,
                                  "cta_busy_max_over_mean": float(np.median(busy_max_over_mean)),
                                  "cta_busy_cov": float(np.median(busy_cov)),
                                  "cta_finish_cov": float(np.median(finish_cov)),
                                  "pairs_visited": st["pairs_visited"],
                                  "pairs_accepted": st["pairs_accepted"],
                                  "sorted": not args.no_sort, "clocks": clocks}), flush=True)
    summary = []
    for (pol, Pn, unit), q in results.items():
        s = results.get(("STATIC", Pn, unit))
        if pol == "STATIC" or s is None:
            continue
        summary.append({"policy": pol, "P": Pn, "unit": unit,
                        "speedup_vs_static": s["median"] / q["median"],
                        "beats_static": bool(q["median"] < s["median"] and q["q3"] < s["q1"])})
    print(json.dumps({"summary": summary}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
