#!/usr/bin/env python
"""Re-measure the DB entries of the workloads that this round's additions
to the halo (band-reuse) mainloop apply to: stride-1 windowed convs over maps
wider than one 128-row tile (halo strips: VGG-16's 224-wide layers, SSD-512's
128-wide 3x3s, Inception-v3's 147-wide 3x3s), widths that fill little of a
full-width tile (strips), and 32-byte-row operands (SW32 shifted views:
Inception's 48 / 80-channel tensors).  Entries with explicit tile parameters
were tuned for the mainloops of their time and switch the automatic choice
off; for each one this times the head entry against the kernel's own choice
(no explicit tile parameters) and, when the latter is faster by
``--min-gain``, records it as the new head entry.

  python tools/retune_strips.py [--dry-run]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--db", default=None)
    ap.add_argument("--min-gain", type=float, default=0.03)
    ap.add_argument("--dry-run", action="store_true")
    ap.add_argument("--only", default="", help="substring of the machine key, e.g. bf16/b128")
    args = ap.parse_args()
    from paper_1809_02697_b200 import tuning
    from paper_1809_02697_b200.kernels import ConvSchedule
    from paper_1809_02697_b200.runtime import DevicePool
    from paper_1809_02697_b200.tuning import MeasuredScheme
    db = tuning.ScheduleDb(args.db or tuning.DEFAULT_DB)
    es = {"bf16": 2, "tf32": 4, "fp8": 1}
    changed = 0
    for (cpu, key), schemes in sorted(db._data.items()):
        mode, btag = cpu.split("/")[-2:]
        if mode not in es or not btag.startswith("b"):
            continue
        batch = int(btag[1:])
        wl = tuning._workload_from_key(key)
        sh, sw = wl.stride_hw
        head = schemes[0]
        rowb = head.schedule.ic_bn * es[mode]
        # candidates: stride-1 convs with a horizontal window (the halo
        # mainloop's domain: 128 / 64 / 32-byte rows, full-width tiles or strips)
        if not (sh == 1 and sw == 1 and wl.kernel_w > 1 and rowb in (32, 64, 128)):
            continue
        if args.only and args.only not in cpu:
            continue
        if not any(head.schedule.tile().values()):
            continue                               # already the kernel's own choice
        pool = DevicePool(0, mode)
        plain = ConvSchedule(head.schedule.ic_bn, head.schedule.oc_bn, head.schedule.reg_n,
                             head.schedule.unroll_ker)
        try:
            m_old = tuning.measure(wl, head.schedule, repeats=10, pool=pool, batch=batch)
            m_new = tuning.measure(wl, plain, repeats=10, pool=pool, batch=batch)
        except Exception as exc:  # noqa: BLE001
            print(f"{mode} b{batch} {key}: {type(exc).__name__}: {exc}")
            continue
        gain = 1.0 - m_new.mean_ns / m_old.mean_ns
        take = gain >= args.min_gain
        print(f"{mode} b{batch} {key}: DB head {m_old.mean_ns / 1e3:.1f} us -> strips "
              f"{m_new.mean_ns / 1e3:.1f} us ({gain * 100:+.1f}%) {'TAKEN' if take else 'kept'}",
              flush=True)
        if take and not args.dry_run:
            kept = [MeasuredScheme(m.schedule, max(m.mean_ns, m_new.mean_ns * 1.001), m.stderr_ns,
                                   m.repeats) for m in schemes]
            kept[0] = MeasuredScheme(head.schedule, max(m_old.mean_ns, m_new.mean_ns * 1.001),
                                     m_old.stderr_ns, m_old.repeats)
            db.put(cpu, wl, [m_new] + kept)
            changed += 1
    print(f"{changed} entries updated")


if __name__ == "__main__":
    main()
