import ctypes, os, sys, subprocess
sys.path.insert(0, '.')
sys.path.insert(0, 'tools')
os.environ['NEOB200_DBG'] = os.environ.get('NEOB200_DBG', '8')
sys.argv = ['conv_bench'] + sys.argv[1:]
import conv_bench
conv_bench.main()
from paper_1809_02697_b200 import _lib as L
lib = L.load()
buf = (ctypes.c_ulonglong * 8192)()
lib.neo_dbg_clk(buf, 8192)
cyc = [buf[2*i] for i in range(148)]; ns = [buf[2*i+1] for i in range(148)]
import statistics
if any(ns):
    print("cycles median", statistics.median(cyc), "ns median", statistics.median(ns), "GHz", statistics.median(c/n for c, n in zip(cyc, ns) if n))

if int(os.environ['NEOB200_DBG']) & 16:
    names = ["tempty wait", "full wait", "mma issue", "commit"]
    for j, nm in enumerate(names):
        print(nm, statistics.median(buf[2048 + 4 * i + j] for i in range(148)))

if int(os.environ['NEOB200_DBG']) & 32:
    names = ["pre (res issue, params, bar)", "tfull wait", "res wait", "compute", "store"]
    for j, nm in enumerate(names):
        vals = [buf[4096 + (i * 4 + g) * 5 + j] for i in range(148) for g in range(4)]
        vals = [v for v in vals if v]
        print(nm, statistics.median(vals) if vals else 0)

if int(os.environ['NEOB200_DBG']) & 64:
    ent = [buf[6144 + 3 * i] for i in range(148)]
    pdl = [buf[6144 + 3 * i + 1] for i in range(148)]
    ex = [buf[6144 + 3 * i + 2] for i in range(148)]
    t0 = min(ent)
    rel = lambda v: [(x - t0) / 1000 for x in v]
    import numpy as np
    for nm, v in (("entry", ent), ("pdl-wait done", pdl), ("exit", ex)):
        r = np.array(rel(v))
        print(f"{nm:14s} min {r.min():6.2f} med {np.median(r):6.2f} max {r.max():6.2f} us")
    if int(os.environ['NEOB200_DBG']) & 8:
        ms = np.array(rel([buf[7000 + 2 * i] for i in range(148)]))
        me = np.array(rel([buf[7000 + 2 * i + 1] for i in range(148)]))
        print(f"mma loop start min {ms.min():6.2f} med {np.median(ms):6.2f} max {ms.max():6.2f}")
        print(f"mma loop end   min {me.min():6.2f} med {np.median(me):6.2f} max {me.max():6.2f}")

if int(os.environ['NEOB200_DBG']) & 128:
    for w in range(2, 18):
        n = buf[7680 + w]
        if n:
            print(f"warp {w:2d}: {n} chunks, tmem ld+wait {buf[7600 + w] / n:6.0f} cyc, finish {buf[7640 + w] / n:6.0f} cyc")
