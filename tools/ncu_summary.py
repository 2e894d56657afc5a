#!/usr/bin/env python
"""Summarise ncu outputs into profiles/ (read here, on the CPU box).

  python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
      --out profiles/round1/c2_bilinear.json

From a `--set full` report: duration, issue/pipe utilisation, DRAM/L2 bytes, stall
breakdown, registers/smem/occupancy, and the hot-loop instruction share.  From a
`gpu__time_duration` launch list: per-kernel launch count, total and share of time.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_active.avg",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__warps_eligible.avg.per_cycle_active",
    # the counters that justify the design: tensor pipe and its HMMA
    # sub-pipe, ALU pipe, L2 sectors (-> GB/s), shared-memory wavefronts by op, DSMEM atomics
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
    "sm__inst_executed_pipe_alu_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_sectors.sum", "lts__t_sectors.sum.per_second", "lts__t_sectors.sum.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_lookup_hit.sum",
    "lts__t_sectors_lookup_miss.sum", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
    "l1tex__t_requests_pipe_lsu_mem_dshared_op_atom.sum",
    "l1tex__m_l1tex2xbar_write_sectors_mem_dshared_op_atom.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra],
                         capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full_summary(rep):
    rows = ncu_csv(rep, "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    d, u = {}, {}
    for k, unit, v in zip(hdr, units, vals):
        short = k.split(".", 2)[2] if k.count(".") >= 3 and k.split(".")[1] == "TriageCompute" else k
        d.setdefault(short, v)
        u.setdefault(short, unit)
        d[k] = v
        u[k] = unit
    res = {"kernel": d.get("Kernel Name"), "metrics": {}}
    for k in KEYS:
        if k in d:
            try:
                res["metrics"][k] = {"value": float(d[k].replace(",", "")), "unit": u.get(k, "")}
            except ValueError:
                res["metrics"][k] = {"value": d[k], "unit": u.get(k, "")}
    m = res["metrics"]
    try:   # derived: L2 and DRAM bytes per second over the kernel's duration
        scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
                 "msecond": 1e-3, "s": 1.0, "second": 1.0}
        dur = m["gpu__time_duration.sum"]["value"] * scale[m["gpu__time_duration.sum"]["unit"]]
        res["derived"] = {
            "l2_GBps": m["lts__t_sectors.sum"]["value"] * 32 / dur / 1e9,
            "dram_GBps": sum(m[k]["value"] * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                                              "Tbyte": 1e12}.get(m[k]["unit"], 1)
                             for k in ("dram__bytes_read.sum", "dram__bytes_write.sum")) / dur / 1e9,
            "duration_s": dur}
    except (KeyError, TypeError, ZeroDivisionError):
        pass
    stalls = {}
    for k in hdr:
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                v = float(d[k].replace(",", ""))
            except ValueError:
                continue
            if v:
                stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = v
    tot = sum(stalls.values()) or 1.0
    res["stall_share"] = {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda x: -x[1])}
    # instruction-count hot spots (blocks with equal execution counts)
    src = ncu_csv(rep, "source", ["--print-source", "sass"])
    h = src[1]
    iE = h.index("Instructions Executed")
    data = []
    for r in src[2:]:
        try:
            data.append((int(r[0], 16), int(r[iE]), r[1].strip()))
        except (ValueError, IndexError):
            pass
    tot_i = sum(e for _, e, _ in data) or 1
    blocks, cur = [], None
    for a, e, s in data:
        if cur and cur["exec"] == e:
            cur["n"] += 1
        else:
            if cur:
                blocks.append(cur)
            cur = {"start": a - data[0][0], "exec": e, "n": 1, "first": s[:60]}
    if cur:
        blocks.append(cur)
    blocks.sort(key=lambda b: -b["exec"] * b["n"])
    res["top_blocks"] = [{"offset": hex(b["start"]), "instructions": b["n"], "executions": b["exec"],
                          "share": round(b["exec"] * b["n"] / tot_i, 4), "first": b["first"]}
                         for b in blocks[:8]]
    return res


def launches_summary(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    iN, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        try:
            agg[r[iN].split("(")[0]].append(float(r[iV].replace(",", "")))
        except (ValueError, IndexError):
            pass
    tot = sum(sum(v) for v in agg.values()) or 1.0
    return {k: {"launches": len(v), "total_ns": sum(v), "mean_ns": sum(v) / len(v),
                "share": round(sum(v) / tot, 4)} for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    res = {"note": a.note}
    if a.rep:
        res["full"] = full_summary(a.rep)
    if a.launches:
        res["launches"] = launches_summary(a.launches)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
