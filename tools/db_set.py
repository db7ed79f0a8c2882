#!/usr/bin/env python
"""Put one measured tile configuration at the head of a workload's entry in
the schedule DB (the executor takes the first scheme of the block pair):

  python tools/db_set.py --mode bf16 --batch 128 --workload 32,32,149,149,3,3,1,0 \\
      --us 309.4 --tile '{"tile_n":32,"slices_per_stage":3,"stages":5,"weight_stationary":2}'

The measurement itself comes from tools/conv_bench.py --sweep / geo_sweep.py
on the GPU; this script only records it (no GPU needed)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("--batch", type=int, required=True)
    ap.add_argument("--workload", required=True, help="C,K,H,W,R,S,stride,pad (the DB key)")
    ap.add_argument("--us", type=float, required=True)
    ap.add_argument("--tile", required=True)
    ap.add_argument("--db", default=None)
    args = ap.parse_args()
    from paper_1809_02697_b200 import tuning
    from paper_1809_02697_b200.tuning import MeasuredScheme
    db = tuning.ScheduleDb(args.db or tuning.DEFAULT_DB)
    vals = [int(v) for v in args.workload.split(",")]
    keys = [(cpu, k) for (cpu, k) in db._data
            if cpu.endswith(f"/{args.mode}/b{args.batch}") and json.loads(k)[:len(vals)] == vals]
    assert len(keys) == 1, keys
    schemes = db._data[keys[0]]
    base = schemes[0].schedule
    sched = type(base).from_dict({"ic_bn": base.ic_bn, "oc_bn": base.oc_bn, "reg_n": base.reg_n,
                                  "unroll_ker": base.unroll_ker, **json.loads(args.tile)})
    ns = args.us * 1e3
    # stale entries measured under another default geometry must not sort
    # ahead of the new one: keep them, but no faster than it
    kept = [MeasuredScheme(m.schedule, max(m.mean_ns, ns * 1.001), m.stderr_ns, m.repeats)
            for m in schemes if m.schedule.as_dict() != sched.as_dict()]
    wl = tuning._workload_from_key(keys[0][1])
    db.put(keys[0][0], wl, [MeasuredScheme(sched, ns, 0.0, 10)] + kept)
    print(keys[0], "->", db.get(keys[0][0], wl)[0].to_dict())


if __name__ == "__main__":
    main()
