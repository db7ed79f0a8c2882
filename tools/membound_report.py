#!/usr/bin/env python
"""Memory-bound launch report (north_star piece 2): joins an ncu launch list
(gpu__time_duration + dram bytes per launch, one captured step of
tools/one_step.py) with the executor's per-launch algorithmic bytes / FLOPs
(tools/one_step.py --dump) and prints, for every launch, achieved GB/s =
algorithmic bytes / ncu duration and its fraction of the measured HBM copy
peak (MEASURED_PEAKS.json hbm_gbs), plus the convs' TFLOP/s.

  python tools/membound_report.py gpurun_out/r2_densenet201_ncu.csv \\
      gpurun_out/r2_densenet201_launches.json --title "DenseNet-201 b32" > profiles/x.md
"""

from __future__ import annotations

import argparse
import csv
import json
import os
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_ncu(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    out: "OrderedDict[int, dict]" = OrderedDict()
    for r in rows[start + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        e = out.setdefault(int(d["ID"]), {"kernel": d["Kernel Name"].split("(")[0]
                                          .replace("void ", "").replace("<unnamed>::", "")})
        val = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        if d["Metric Name"] == "gpu__time_duration.sum":
            e["us"] = val * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
                             "ms": 1e3, "msecond": 1e3}[unit]
        elif d["Metric Name"].startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
            e[d["Metric Name"].split(".")[0].replace("dram__bytes_", "")] = val * scale
    return list(out.values())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("ncu_csv")
    ap.add_argument("launches_json")
    ap.add_argument("--title", default="")
    ap.add_argument("--tensor-peak", type=float, default=None)
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks["hbm_gbs"])
    tpk = args.tensor_peak or float(peaks["bf16_tflops"])
    ncu = load_ncu(args.ncu_csv)
    launches = json.load(open(args.launches_json))
    assert len(ncu) == len(launches), (len(ncu), len(launches))
    mem, conv = [], []
    for k, l in zip(ncu, launches):
        us = k.get("us", 0.0)
        rec = dict(l, kernel=k["kernel"], us=us, dram=(k.get("read", 0) + k.get("write", 0)))
        (conv if l["flops"] and not l["name"].startswith("head") else mem).append(rec)
    tot = sum(r["us"] for r in mem + conv)
    mus = sum(r["us"] for r in mem)
    mb = sum(r["bytes"] for r in mem)
    print(f"# {args.title}: per-launch ncu times (cold cache, serialised) vs algorithmic bytes\n")
    print(f"HBM peak: {hbm:.0f} GB/s measured copy (MEASURED_PEAKS.json); tensor peak "
          f"{tpk:.0f} TFLOP/s.  {len(mem)} memory-bound launches, {mus:.1f} us = "
          f"{100 * mus / tot:.1f}% of {tot:.1f} us; aggregate {mb / mus / 1e3:.0f} GB/s = "
          f"{mb / mus / 1e3 / hbm:.2f} of HBM.\n")
    below = [r for r in mem if r["bytes"] / max(r["us"], 1e-3) / 1e3 / hbm < 0.6]
    print(f"Memory-bound launches below 0.6 of HBM: {len(below)} "
          f"({sum(r['us'] for r in below):.1f} us).\n")
    print("| # | launch | kernel | us | alg MB | GB/s | frac HBM | DRAM MB (ncu) |")
    print("|---|---|---|---|---|---|---|---|")
    for i, r in enumerate(mem):
        gbs = r["bytes"] / max(r["us"], 1e-3) / 1e3
        print(f"| {i} | {r['name']} | {r['kernel']} | {r['us']:.1f} | {r['bytes'] / 1e6:.1f} | "
              f"{gbs:.0f} | {gbs / hbm:.2f} | {r['dram'] / 1e6:.1f} |")
    cus = sum(r["us"] for r in conv)
    cfl = sum(r["flops"] for r in conv)
    print(f"\nConvs / dense: {len(conv)} launches, {cus:.1f} us, {cfl / cus / 1e6:.0f} TFLOP/s "
          f"= {cfl / cus / 1e6 / tpk:.2f} of the tensor peak (cold, serialised).\n")
    print("| # | launch | desc | us | TFLOP/s | frac tensor | GB/s (alg) |")
    print("|---|---|---|---|---|---|---|")
    for i, r in enumerate(conv):
        tf = r["flops"] / max(r["us"], 1e-3) / 1e6
        print(f"| {i} | {r['name']} | {r['desc']} | {r['us']:.1f} | {tf:.0f} | {tf / tpk:.2f} | "
              f"{r['bytes'] / max(r['us'], 1e-3) / 1e3:.0f} |")


if __name__ == "__main__":
    main()
