#!/usr/bin/env python
"""Time the fused image stem (neo_stem_conv_pool) at ResNet-50 b64 as CUDA-graph
replays; STEM_N sets the batch, NEOB200_STEM_DBG=32 prints per-role phase clocks."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1809_02697_b200 import device as D
dev = torch.device("cuda:0")
n = int(os.environ.get("STEM_N", 64)); c, h, w = 3, 224, 224
x = torch.randn((n, c, h, w), device=dev)
wimg = D.pack_stem_weights(torch.randn((64, c, 7, 7), device=dev) * 0.1)
bias = torch.randn(64, device=dev)
out = torch.zeros((n, 1, 56, 56, 64), dtype=torch.bfloat16, device=dev)
st = torch.cuda.Stream()
f = lambda: D.stem_conv_pool(x, wimg, out, n, c, h, w, 64, bias=bias, stream=st)
for _ in range(3): f()
torch.cuda.synchronize()
g = D.capture(lambda: [f() for _ in range(20)], st)
g.launch(st)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st); g.launch(st); b.record(st); b.synchronize()
print(os.environ.get("NEOB200_STEM_DBG", "0"), n, f"{a.elapsed_time(b) * 1e3 / 20:.1f} us")
if int(os.environ.get("NEOB200_STEM_DBG", "0")) & 32:
    import ctypes, statistics
    from paper_1809_02697_b200 import _lib as L
    lib = L.load()
    buf = (ctypes.c_ulonglong * (148 * 8))()
    lib.neo_stem_dbg_clk(buf, 148 * 8)
    names = ["mma: wait patch_full", "mma: wait tempty", "mma: issue+commit", "epi: wait tfull", "epi: math", "epi: barrier", "epi: pool"]
    for k, nm in enumerate(names):
        print(nm, statistics.median(buf[i * 8 + k] for i in range(148)))
