#!/usr/bin/env python
"""Small targeted tile search for the workloads of one (mode, batch) DB key
whose output-channel count is not a multiple of 32 (detector heads: 16 / 24 /
84 / 126 channels): the generic variants only try N tiles of 64 / 128 / 256,
and 84 channels as two 64-wide tiles wastes a third of the MMA columns and
reads the activations twice.  Candidates: the kernel's own N tile (K rounded
up to 16) and 128, plain whole-row geometry vs the kernel's geometry, a few
(slices per stage, depth) pairs.  Faster candidates (>= --min-gain over the
current head entry) are recorded as the new head.

  python tools/minitune.py --model ssd_resnet50 --batch 32 [--mode bf16] [--db copy.npsd]
"""
import argparse
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="ssd_resnet50")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("--db", default=None)
    ap.add_argument("--min-gain", type=float, default=0.05)
    args = ap.parse_args()
    from paper_1809_02697_b200 import tuning
    from paper_1809_02697_b200.runtime import DevicePool
    from paper_1809_02697_b200.tuning import MeasuredScheme, tuning_key
    db = tuning.ScheduleDb(args.db or tuning.DEFAULT_DB)
    key = tuning_key(args.mode, args.batch)
    pool = DevicePool(0, args.mode)
    changed = 0
    for wl in db.workloads(key):
        if wl.out_channel % 32 == 0 or wl.kernel_h * wl.kernel_w == 1:
            continue
        schemes = db.get(key, wl)
        head = schemes[0]
        kpad = -(-wl.out_channel // 16) * 16
        ow, oh = wl.out_w, wl.out_h
        geos = [{}]
        if ow <= 128:
            bh = max(1, min(oh, 128 // ow))
            bni = max(1, min(args.batch, 128 // (ow * bh))) if bh == oh else 1
            geos.append({"tile_w": ow, "tile_h": bh, "tile_img": bni})
        cands = []
        for geo, tn, (g, st) in itertools.product(geos, sorted({min(kpad, 256), 128} if kpad <= 128
                                                              else {128, 256}),
                                                  [(1, 3), (2, 2), (2, 3), (1, 4)]):
            cands.append({**geo, "tile_n": tn, "slices_per_stage": g, "stages": st})
        try:
            best = tuning.measure(wl, head.schedule, repeats=8, pool=pool, batch=args.batch)
        except Exception as exc:  # noqa: BLE001
            print(f"{wl.key()}: head entry fails: {exc}")
            continue
        base_ns = best.mean_ns
        bench = None
        for tile in cands:
            sch = head.schedule.with_tile(**{f: 0 for f in tuning.ConvSchedule(1, 1, 1).tile()})
            sch = sch.with_tile(**tile)
            try:
                m = tuning.measure(wl, sch, repeats=8, pool=pool, batch=args.batch)
            except Exception:  # noqa: BLE001
                continue
            if m.mean_ns < best.mean_ns:
                best = m
        gain = 1 - best.mean_ns / base_ns
        take = gain >= args.min_gain
        print(f"{wl.key()}: head {base_ns / 1e3:.1f} us -> {best.mean_ns / 1e3:.1f} us "
              f"({gain * 100:+.1f}%) {best.schedule.tile() if take else ''}", flush=True)
        if take:
            kept = [MeasuredScheme(m.schedule, max(m.mean_ns, best.mean_ns * 1.001), m.stderr_ns,
                                   m.repeats) for m in schemes
                    if m.schedule.as_dict() != best.schedule.as_dict()]
            db.put(key, wl, [best] + kept)
            changed += 1
    print(f"{changed} entries updated")


if __name__ == "__main__":
    main()
