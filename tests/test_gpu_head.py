"""Fused classifier head (neo_classifier_head: global average pool ->
dense + bias -> softmax in one launch) against the oracle's _pool2d / dense /
softmax (reference executor.py:103-128, 197-203, 167-170).  bf16 operands
(the pooled mean rounded to bf16, bf16 weights) with fp32 accumulation:
tolerance 1e-2 relative on logits, 2e-2 on probabilities."""

import numpy as np
import pytest

import oracle
from oracle.ops import pack_nchw

pytestmark = pytest.mark.gpu


def bf16_round(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).bfloat16().float().numpy()


def run_head(x, w, bias, y, softmax):
    import torch
    from paper_1809_02697_b200 import device as D
    dev = torch.device("cuda:0")
    n, c, h, wd = x.shape
    units = w.shape[0]
    xt = torch.from_numpy(pack_nchw(x, y)).to(dev).bfloat16()
    wt = torch.from_numpy(w).to(dev).bfloat16()
    bt = torch.from_numpy(bias).to(dev) if bias is not None else None
    out = torch.full((n, units), 7.0, device=dev)
    scratch = D.HeadScratch(n, c, units, dev)
    for _ in range(3):      # the barriers must re-arm between launches
        D.classifier_head(xt, wt, bt, out, n, c, h * wd, y, units, softmax, scratch)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("n,c,hw,units,y,softmax", [
    (3, 256, 5, 37, 16, True), (64, 2048, 7, 1000, 64, True), (17, 256, 8, 130, 32, False),
    (1, 1024, 7, 10, 8, True), (40, 512, 7, 1000, 64, False)])
def test_head_matches_oracle(cuda, n, c, hw, units, y, softmax):
    rng = np.random.default_rng(n + c + units)
    x = np.abs(rng.standard_normal((n, c, hw, hw))).astype(np.float32)
    w = (rng.standard_normal((units, c)) * np.sqrt(2.0 / c)).astype(np.float32)
    bias = rng.normal(0, 0.1, units).astype(np.float32) if units != 10 else None
    got = run_head(bf16_round(x), w, bias, y, softmax)
    pooled = oracle.pool2d(bf16_round(x), hw, 1, 0, "avg").reshape(n, c)
    logits = oracle.dense(bf16_round(pooled), bf16_round(w), bias)
    ref = oracle.softmax(logits) if softmax else logits
    assert oracle.rel_err(got, ref) < (2e-2 if softmax else 1e-2)
    if softmax:
        assert np.allclose(got.sum(axis=1), 1.0, atol=1e-4)
        assert np.array_equal(got.argmax(axis=1), ref.argmax(axis=1))


def test_executor_uses_fused_head(cuda):
    import os
    from paper_1809_02697_b200 import (DevicePool, build_model, compile_graph, execute,
                                       model_input)
    from paper_1809_02697_b200.executor import DeviceProgram, ExecutablePlan
    # logits (no softmax): a random-init net's softmax is too peaked to compare
    # probabilities at bf16 precision
    g = build_model("resnet18", batch=3, image=64, num_classes=20, softmax=False)
    feeds = model_input(g)
    planned = compile_graph(g, mode="bf16")
    prog = DeviceProgram(ExecutablePlan.compile(planned), 0, "bf16")
    assert any(nm.startswith("head") for nm in prog.launch_names)
    assert not any(nm.startswith(("avgpool", "dense")) for nm in prog.launch_names)
    fused = execute(planned, feeds, DevicePool(0, "bf16"))[0]
    os.environ["NEOB200_NO_FUSED_HEAD"] = "1"
    try:
        unfused = execute(compile_graph(g, mode="bf16"), feeds, DevicePool(0, "bf16"))[0]
    finally:
        del os.environ["NEOB200_NO_FUSED_HEAD"]
    ref = oracle.execute_reference(g, feeds)[0]
    assert oracle.rel_err(fused, ref) < 2e-2 and oracle.rel_err(fused, unfused) < 2e-2
    assert np.array_equal(fused.argmax(axis=1), ref.argmax(axis=1))
