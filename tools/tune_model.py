#!/usr/bin/env python
"""Per-layer tensor-core tile tuning of a model's convs on the local GPU
(north_star piece 3).  Results are appended to the schedule database that
bench.py and compile_graph(db=...) read:

  python tools/tune_model.py --model resnet50 --batch 64 --mode bf16
"""

from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("--db", default=None)
    ap.add_argument("--repeats", type=int, default=10)
    ap.add_argument("--refresh", action="store_true", help="re-measure existing entries")
    ap.add_argument("--pair", action="store_true", help="also time CTA-pair (cta_group::2) tiles")
    args = ap.parse_args()
    from paper_1809_02697_b200 import ScheduleDb, build_model
    from paper_1809_02697_b200.tuning import DEFAULT_DB, tune_tiles
    db = ScheduleDb(args.db or DEFAULT_DB)
    g = build_model(args.model, batch=args.batch)
    t0 = time.time()
    best = tune_tiles(g, db, args.mode, args.batch, repeats=args.repeats, refresh=args.refresh, pair=args.pair)
    print(f"tuned {len(best)} convs of {args.model} b{args.batch} {args.mode} in "
          f"{time.time() - t0:.1f}s -> {db.path}")


if __name__ == "__main__":
    main()
