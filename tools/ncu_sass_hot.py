#!/usr/bin/env python
"""Per-SASS-instruction hot spots of an ncu report (read here, on the CPU box).

  ncu -i rep --page source --csv --print-source sass > src.csv
  python tools/ncu_sass_hot.py src.csv [--top 40] [--ranges a0-a1,b0-b1]

Prints the instructions with the most stall samples, and per address range the share of
samples, executed warp instructions and excess shared-memory wavefronts.
"""
import argparse
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--ranges", default="")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    recs = []
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        try:
            addr = int(r[ix["Address"]], 16)
        except ValueError:
            continue
        num = lambda k: float(r[ix[k]] or 0) if k in ix else 0.0
        recs.append((addr, r[ix["Source"]].strip(), num("Warp Stall Sampling (All Samples)"),
                     num("Instructions Executed"), num("L1 Wavefronts Shared Excessive")))
    S = sum(x[2] for x in recs) or 1
    I = sum(x[3] for x in recs) or 1
    print(f"total samples {S:.0f}, warp instructions {I:.3e}")
    for x in sorted(recs, key=lambda x: -x[2])[: a.top]:
        print(f"{x[0]:#07x} {100 * x[2] / S:5.2f}% smp {x[3]:.2e} inst exc_wf {x[4]:.2e}  {x[1][:70]}")
    for rg in filter(None, a.ranges.split(",")):
        lo, hi = (int(v, 16) for v in rg.split("-"))
        sel = [x for x in recs if lo <= x[0] < hi]
        print(f"[{lo:#x},{hi:#x}): samples {100 * sum(x[2] for x in sel) / S:.1f}%  "
              f"inst {100 * sum(x[3] for x in sel) / I:.1f}%  exc_wf {sum(x[4] for x in sel):.2e}")


if __name__ == "__main__":
    main()
