#!/usr/bin/env python
"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes per
launch, one captured step) into a markdown table and the per-step conv DRAM
traffic used by bench.py's roofline.traffic.

  python tools/summarize_launches.py gpurun_out/r1_launches.csv gpurun_out/one_step.log \
      profiles/r1_launches.md profiles/conv_traffic.json
"""

from __future__ import annotations

import csv
import json
import sys
from collections import OrderedDict


def main(csv_path, names_path, md_path, json_path):
    rows = list(csv.reader(open(csv_path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    launches: "OrderedDict[int, dict]" = OrderedDict()
    for r in rows[start + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        lid = int(d["ID"])
        e = launches.setdefault(lid, {"kernel": d["Kernel Name"], "grid": d["Grid Size"],
                                      "block": d["Block Size"]})
        val = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        if d["Metric Name"] == "gpu__time_duration.sum":
            e["us"] = val * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
                             "ms": 1e3, "msecond": 1e3}[unit]
        elif d["Metric Name"].startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
            e[d["Metric Name"].split(".")[0].replace("dram__bytes_", "")] = val * scale
    names = [ln.split(" ", 1)[1].strip() for ln in open(names_path) if ln[:1].isdigit()]
    total = sum(e.get("us", 0) for e in launches.values())
    conv_bytes = 0.0
    conv_us = 0.0
    lines = ["| # | launch | kernel | grid | us | share | DRAM read MB | DRAM write MB |",
             "|---|---|---|---|---|---|---|---|"]
    for i, (lid, e) in enumerate(launches.items()):
        name = names[i] if i < len(names) else "?"
        rd, wr = e.get("read", 0.0), e.get("write", 0.0)
        if "conv_tc_kernel" in e["kernel"] or "stem_conv_pool" in e["kernel"]:
            conv_bytes += rd + wr
            conv_us += e.get("us", 0)
        kern = e["kernel"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        lines.append(f"| {i} | {name} | {kern} | {e['grid']} | {e.get('us', 0):.1f} | "
                     f"{100 * e.get('us', 0) / total:.1f}% | {rd / 1e6:.1f} | {wr / 1e6:.1f} |")
    head = [f"# ncu launch list, one ResNet-50 b64 bf16 forward ({len(launches)} launches)",
            "",
            "Captured with `ncu --nvtx --nvtx-include step/ --metrics gpu__time_duration.sum,"
            "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none python tools/one_step.py`"
            " (cold-cache, serialised launches: compare shares, not absolutes).",
            "",
            f"* total kernel time {total:.1f} us; conv share (conv_tc_kernel + stem_conv_pool_kernel) "
            f"{100 * conv_us / total:.1f}% ({conv_us:.1f} us)",
            f"* conv DRAM traffic per step (conv_tc_kernel + stem_conv_pool_kernel): {conv_bytes / 1e6:.1f} MB",
            ""]
    open(md_path, "w").write("\n".join(head + lines) + "\n")
    json.dump({"bytes_per_step": conv_bytes, "conv_us_ncu": conv_us, "total_us_ncu": total,
               "source": md_path}, open(json_path, "w"), indent=1)
    print(f"{len(launches)} launches, total {total:.1f} us, conv {conv_us:.1f} us, "
          f"conv DRAM {conv_bytes / 1e6:.1f} MB")


if __name__ == "__main__":
    main(*sys.argv[1:5])
