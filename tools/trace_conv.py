#!/usr/bin/env python
"""Per-event timeline of CTA 0 of one conv launch (debug library built with
-DNEO_TRACE into tools/libneob200_trace.so).  Prints per-event average
intervals.  Usage: NEOB200_LIB=tools/libneob200_trace.so python tools/trace_conv.py ..."""

from __future__ import annotations

import ctypes
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

NAMES = {1: "prod:wait_empty>", 2: "prod:got_empty", 10: "mma:wait_tempty>", 11: "mma:got_tempty",
         12: "mma:got_full", 20: "epi0:start", 21: "epi1:start", 22: "epi0:res_issued",
         23: "epi1:res_issued", 24: "epi0:bar1", 25: "epi1:bar1", 26: "epi0:got_tfull",
         27: "epi1:got_tfull", 28: "epi0:got_res", 29: "epi1:got_res", 30: "epi0:computed",
         31: "epi1:computed", 32: "epi0:bar2", 33: "epi1:bar2", 13: "mma:committed", 14: "mma:wait_full>", 15: "mma:issued",
         40: "split:partial_stored", 41: "split:all_arrived", 42: "split:fixup_done",
         60: "kernel:entry", 61: "kernel:setup_done", 62: "kernel:final_sync", 64: "epi:bulk_done"}


def main():
    import numpy as np
    import torch
    argv = sys.argv[1:]
    sys.argv = [sys.argv[0]] + argv
    from paper_1809_02697_b200 import _lib as L
    lib = L.load()
    lib.neo_trace_dump.restype = ctypes.c_int
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import conv_bench
    conv_bench.main()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 65536)()
    lib.neo_trace_dump(buf, 0)          # drop the timed runs
    conv_bench_args = argv + ["--once"]
    sys.argv = [sys.argv[0]] + conv_bench_args
    conv_bench.main()
    torch.cuda.synchronize()
    n = lib.neo_trace_dump(buf, 65536)
    clk = [(buf[60000 + 2 * w], buf[60001 + 2 * w]) for w in range(16)]
    print("epilogue warp cycles (tmem-ld+params, math+smem):", clk)
    recs = [(int(v >> 56), int((v >> 40) & 0xFFFF), int(v & 0xFFFFFFFFFF)) for v in buf[:n]]
    t0 = min(r[2] for r in recs)
    by = defaultdict(list)
    for ev, tile, ns in recs:
        by[(ev, tile)].append(ns - t0)
    # print the first few tiles of the epilogue timelines
    tiles = sorted({t for (ev, t) in by if ev >= 20})[:8]
    for t in tiles:
        line = [f"tile {t:5d}:"]
        for ev in range(20, 34):
            if (ev, t) in by:
                line.append(f"{NAMES[ev]}={by[(ev, t)][-1] / 1000:.2f}us")
        print(" ".join(line))
    mma = sorted(v for (ev, t), vs in by.items() if ev == 12 for v in vs)
    if mma:
        print(f"mma full-waits: {len(mma)} first {mma[0] / 1000:.2f}us last {mma[-1] / 1000:.2f}us")
    prod = sorted(v for (ev, t), vs in by.items() if ev == 2 for v in vs)
    if prod:
        print(f"producer stages: {len(prod)} first {prod[0] / 1000:.2f}us last {prod[-1] / 1000:.2f}us")
    chunk = sorted((ns, ev) for ev, tile, ns in recs if 43 <= ev < 56)
    print("chunk events (first 24):", [(ev, round((ns - t0) / 1000, 2)) for ns, ev in chunk[:24]])
    print("all events in time order:")
    for ev, tile, ns in sorted(recs, key=lambda r: r[2])[:160]:
        print(f"  {(ns - t0) / 1000:8.3f} us  {NAMES.get(ev, ev)}  tile {tile}")
    total = max(r[2] for r in recs) - t0
    print(f"CTA0 span {total / 1000:.2f} us, records {n}")


if __name__ == "__main__":
    main()
