#!/usr/bin/env python
"""Time the fused classifier head (neo_classifier_head) at ResNet-50 b64 as
CUDA-graph replays; NEOB200_HEAD_DBG=1 prints the phase times of CTA 0."""
import sys, os, ctypes
sys.path.insert(0, os.getcwd())
import torch
from paper_1809_02697_b200 import device as D, _lib as L
dev = torch.device("cuda:0")
n, c, hw, y, units = 64, 2048, 49, 64, 1000
x = torch.randn((n, c // y, hw, y), device=dev).bfloat16()
w = (torch.randn((units, c), device=dev) * 0.02).bfloat16()
b = torch.randn(units, device=dev)
out = torch.empty((n, units), device=dev)
sc = D.HeadScratch(n, c, units, dev)
st = torch.cuda.Stream()
f = lambda: D.classifier_head(x, w, b, out, n, c, hw, y, units, True, sc, st)
for _ in range(3): f()
torch.cuda.synchronize()
g = D.capture(lambda: [f() for _ in range(20)], st)
g.launch(st)
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st); g.launch(st); e.record(st); e.synchronize()
print(f"head {a.elapsed_time(e) * 1e3 / 20:.1f} us")
if os.environ.get("NEOB200_HEAD_DBG"):
    f(); torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 8)()
    L.load().neo_head_dbg(buf)
    t = [buf[i] for i in range(7)]
    print("phases us:", [round((t[i + 1] - t[i]) / 1e3, 2) for i in range(6)])
