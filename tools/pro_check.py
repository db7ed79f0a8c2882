"""BN-ReLU prologue conv vs eltwise BN-ReLU + conv, bitwise (debug)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1809_02697_b200 import _lib as L, device as D
dev = torch.device("cuda:0")
rng = np.random.default_rng(0)
for x_bn, relu in ((32, True), (32, False), (64, True)):
    n, c, h, w, k = 2, 128, 14, 14, 128
    x = torch.from_numpy(rng.standard_normal((n, c // x_bn, h, w, x_bn)).astype(np.float32)).to(dev).bfloat16()
    sc = torch.from_numpy(rng.uniform(0.5, 1.5, c).astype(np.float32)).to(dev)
    sh = torch.from_numpy(rng.normal(0, 0.5, c).astype(np.float32)).to(dev)
    wt = torch.from_numpy((rng.standard_normal((k, c, 1, 1)) * 0.1).astype(np.float32)).to(dev)
    wd = D.pack_weights_umma(wt, x_bn, L.MODE_BF16)
    y = torch.empty_like(x)
    op = L.ELT_SCALE_SHIFT_RELU if relu else L.ELT_SCALE_SHIFT
    D.eltwise(op, x, None, y, n, c // x_bn, h * w, x_bn, sc, sh)
    o1 = torch.empty((n, k // 64, h, w, 64), dtype=torch.bfloat16, device=dev)
    o2 = torch.empty_like(o1)
    p1 = D.conv_params(L.MODE_BF16, y, wd, o1, n, c, h, w, k, 1, 1, ic_bn=x_bn, oc_bn=64)
    D.conv2d(p1)
    p2 = D.conv_params(L.MODE_BF16, x, wd, o2, n, c, h, w, k, 1, 1, ic_bn=x_bn, oc_bn=64,
                       prologue=(sc, sh, relu))
    D.conv2d(p2)
    torch.cuda.synchronize()
    a, b = o1.float().cpu().numpy(), o2.float().cpu().numpy()
    print(x_bn, relu, "equal", np.array_equal(a, b), "frac diff", np.mean(a != b), "max", np.abs(a - b).max())
