"""Fused image stem (neo_stem_conv_pool: conv 7x7/2 pad 3 + epilogue + max
pool 3x3/2 pad 1 in one launch) against the CPU oracle: the reference's
conv_blocked epilogue order (kernels.py:185-197) followed by _pool2d
(executor.py:103-128, -inf padding).  The kernel computes in bf16 with fp32
accumulation; the oracle sees the same bf16-rounded input and weights, so the
only differences are summation order and the final bf16 rounding of each
conv value (bound: 2^-8 relative, written as 8e-3 below)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def bf16_round(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).bfloat16().float().numpy()


def run_stem(x, w, y=64, scale=None, shift=None, bias=None, relu=True, out_cb=(0, 0)):
    import torch
    from paper_1809_02697_b200 import device as D
    dev = torch.device("cuda:0")
    n, c, h, wd = x.shape
    oh, ow = (h - 1) // 2 + 1, (wd - 1) // 2 + 1
    ph, pw = (oh - 1) // 2 + 1, (ow - 1) // 2 + 1
    total = out_cb[1] or 64 // y
    out = torch.full((n, total, ph, pw, y), 7.0, dtype=torch.bfloat16, device=dev)
    opt = lambda v: None if v is None else torch.from_numpy(np.asarray(v, np.float32)).to(dev)
    wimg = D.pack_stem_weights(torch.from_numpy(w).to(dev))
    D.stem_conv_pool(torch.from_numpy(x).to(dev), wimg, out, n, c, h, wd, y, opt(scale),
                     opt(shift), opt(bias), relu, out_cb)
    torch.cuda.synchronize()
    return out.float().cpu().numpy()


def reference(x, w, scale=None, shift=None, bias=None, relu=True):
    conv = oracle.conv2d(bf16_round(x), bf16_round(w), 2, 3, scale, shift, bias, relu=relu)
    return oracle.pool2d(conv, 3, 2, 1, "max")


def unblock(o):
    n, cb, ph, pw, y = o.shape
    return o.transpose(0, 1, 4, 2, 3).reshape(n, cb * y, ph, pw)


@pytest.mark.parametrize("shape", [(2, 3, 64, 64), (1, 3, 50, 60), (3, 3, 36, 20),
                                   (1, 3, 224, 224)])
def test_stem_matches_oracle(cuda, shape):
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape).astype(np.float32)
    w = (rng.standard_normal((64, shape[1], 7, 7)) * np.sqrt(2 / (shape[1] * 49))).astype(np.float32)
    bias = rng.normal(0, 0.1, 64).astype(np.float32)
    got = unblock(run_stem(x, w, bias=bias))
    ref = reference(x, w, bias=bias)
    assert got.shape == ref.shape
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 8e-3, err


@pytest.mark.parametrize("c,relu,y", [(1, True, 16), (2, False, 32), (4, True, 8), (3, False, 64)])
def test_stem_channels_epilogue_blocks(cuda, c, relu, y):
    rng = np.random.default_rng(c * 10 + y)
    x = rng.standard_normal((2, c, 40, 44)).astype(np.float32)
    w = (rng.standard_normal((64, c, 7, 7)) * 0.2).astype(np.float32)
    scale = rng.uniform(0.5, 1.5, 64).astype(np.float32)
    shift = rng.normal(0, 0.1, 64).astype(np.float32)
    bias = rng.normal(0, 0.1, 64).astype(np.float32)
    got = unblock(run_stem(x, w, y=y, scale=scale, shift=shift, bias=bias, relu=relu))
    ref = reference(x, w, scale, shift, bias, relu)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 8e-3, err


def test_stem_concat_window(cuda):
    """Output into channel blocks [2, 4) of a 5-block buffer; the rest untouched."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal((1, 3, 32, 32)).astype(np.float32)
    w = (rng.standard_normal((64, 3, 7, 7)) * 0.1).astype(np.float32)
    out = run_stem(x, w, y=32, out_cb=(2, 5))
    assert np.all(out[:, :2] == 7.0) and np.all(out[:, 4:] == 7.0)
    ref = reference(x, w)
    got = unblock(out[:, 2:4])
    assert np.abs(got - ref).max() / np.abs(ref).max() < 8e-3


def test_stem_rejects_unsupported(cuda):
    import torch
    from paper_1809_02697_b200 import device as D
    from paper_1809_02697_b200.errors import NeoplanError
    dev = torch.device("cuda:0")
    x = torch.zeros((1, 3, 30, 30), device=dev)      # width not a multiple of 4
    wimg = D.pack_stem_weights(torch.zeros((64, 3, 7, 7), device=dev))
    out = torch.zeros((1, 1, 8, 8, 64), dtype=torch.bfloat16, device=dev)
    with pytest.raises(NeoplanError):
        D.stem_conv_pool(x, wimg, out, 1, 3, 30, 30, 64)
    with pytest.raises(NeoplanError):
        D.pack_stem_weights(torch.zeros((32, 3, 7, 7), device=dev))


def test_resnet_executor_uses_fused_stem(cuda):
    """bf16 programs of the BASELINE stems launch the fused kernel, and the
    logits agree with the unfused path (NEOB200_NO_FUSED_STEM) and the oracle."""
    import os
    from paper_1809_02697_b200 import DevicePool, build_model, compile_graph, execute, model_input
    from paper_1809_02697_b200.executor import DeviceProgram, ExecutablePlan
    g = build_model("resnet18", batch=2, image=64, num_classes=10, softmax=False)
    feeds = model_input(g)
    planned = compile_graph(g, mode="bf16")
    prog = DeviceProgram(ExecutablePlan.compile(planned), 0, "bf16")
    assert any(nm.startswith("stem") and "_pool" in nm for nm in prog.launch_names)
    assert not any(nm.startswith("stemfold") or nm.startswith("maxpool")
                   for nm in prog.launch_names)
    fused = execute(planned, feeds, DevicePool(0, "bf16"))[0]
    os.environ["NEOB200_NO_FUSED_STEM"] = "1"
    try:
        unfused = execute(compile_graph(g, mode="bf16"), feeds, DevicePool(0, "bf16"))[0]
    finally:
        del os.environ["NEOB200_NO_FUSED_STEM"]
    ref = oracle.execute_reference(g, feeds)[0]
    assert oracle.rel_err(fused, ref) < 2e-2
    assert oracle.rel_err(fused, unfused) < 2e-2


@pytest.mark.parametrize("shape", [(2, 3, 64, 64), (3, 3, 40, 48), (1, 3, 224, 224)])
def test_stem_bf16_input_identical(cuda, shape):
    """A host-rounded bf16 image gives bit-identical results to the f32 image
    (the kernel rounds f32 input RN to bf16 itself); the executor stores a
    stem-only graph input as bf16 so uploads move half the bytes."""
    import torch
    from paper_1809_02697_b200 import device as D
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(9)
    x = rng.standard_normal(shape).astype(np.float32)
    w = (rng.standard_normal((64, 3, 7, 7)) * 0.1).astype(np.float32)
    n, c, h, wd = shape
    oh, ow = (h - 1) // 2 + 1, (wd - 1) // 2 + 1
    ph, pw = (oh - 1) // 2 + 1, (ow - 1) // 2 + 1
    wimg = D.pack_stem_weights(torch.from_numpy(w).to(dev))
    outs = []
    for xt in (torch.from_numpy(x).to(dev), torch.from_numpy(x).bfloat16().to(dev)):
        out = torch.empty((n, 1, ph, pw, 64), dtype=torch.bfloat16, device=dev)
        D.stem_conv_pool(xt, wimg, out, n, c, h, wd, 64)
        outs.append(out)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


def test_executor_bf16_stem_input(cuda):
    import torch
    from paper_1809_02697_b200 import build_model, compile_graph, model_input
    from paper_1809_02697_b200.executor import DeviceProgram, ExecutablePlan
    g = build_model("resnet18", batch=2, image=64, num_classes=10, softmax=False)
    prog = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode="bf16")), 0, "bf16")
    name = prog.input_names()[0]
    assert prog.input_tensor(name).dtype == torch.bfloat16
    assert prog.upload_bytes == 2 * 3 * 64 * 64 * 2
    feeds = model_input(g)
    a = prog.run(feeds)[0]
    # the serving loop (host rounding into pinned bf16, double-buffered uploads)
    pinned = torch.from_numpy(feeds[name]).pin_memory()
    outs = [torch.empty(a.shape, dtype=torch.float32).pin_memory() for _ in range(3)]
    prog.pipeline([pinned] * 3, outs)
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.numpy(), a)
