"""Checks at BASELINE.json's full sizes, where the CPU oracle would take too
long, through size-independent properties: bit-exact layout round trips of
the largest ResNet-50 b64 tensors, the tensor-core conv against cuDNN fp32
(the torch reference for a floating-point kernel) on the b64 layer shapes,
batch invariance of the b64 forward against per-image runs, and run-to-run
determinism of the whole b64 forward."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_fullsize_layout_round_trip(cuda):
    """(64, 256, 56, 56) bf16 -> NCHW[64]c -> NCHW and the (64, 3, 224, 224)
    f32 image -> NCHW[16]c (zero-padded lanes) match torch permutations bit
    for bit."""
    import torch
    from paper_1809_02697_b200 import device as D
    from paper_1809_02697_b200 import _lib as L
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((64, 256, 56, 56), device="cuda", generator=g).to(torch.bfloat16)
    packed = torch.empty((64, 4, 56, 56, 64), dtype=torch.bfloat16, device="cuda")
    D.layout_transform(x, packed, 64, 256, 56, 56, "NCHW", "NCHW64c")
    ref = x.view(64, 4, 64, 56, 56).permute(0, 1, 3, 4, 2).contiguous()
    assert torch.equal(packed.view(torch.int16), ref.view(torch.int16))
    back = torch.empty_like(x)
    D.layout_transform(packed, back, 64, 256, 56, 56, "NCHW64c", "NCHW")
    assert torch.equal(back.view(torch.int16), x.view(torch.int16))
    img = torch.randn((64, 3, 224, 224), device="cuda", generator=g)
    p16 = torch.full((64, 1, 224, 224, 16), float("nan"), device="cuda")
    D.layout_transform(img, p16, 64, 3, 224, 224, "NCHW", "NCHW16c", L.FLAG_PAD_CHANNELS)
    assert torch.equal(p16[..., :3], img.permute(0, 2, 3, 1).unsqueeze(1))
    assert not p16[..., 3:].any()


LAYERS = [
    # ResNet-50 b64 layer shapes: (c, k, hw, r, stride)
    (64, 64, 56, 3, 1),
    (64, 256, 56, 1, 1),
    (256, 128, 56, 1, 2),
    (128, 128, 28, 3, 1),
    (256, 256, 14, 3, 1),
    (1024, 256, 14, 1, 1),
    (512, 512, 7, 3, 1),
    (2048, 512, 7, 1, 1),
]


@pytest.mark.parametrize("layer", LAYERS)
def test_fullsize_conv_vs_cudnn(cuda, layer):
    """bf16 tensor-core conv (f32 output, residual + relu) vs cuDNN fp32 on
    the same bf16-rounded operands at batch 64: accumulation order only."""
    import torch
    import torch.nn.functional as F
    from paper_1809_02697_b200 import _lib as L
    from paper_1809_02697_b200 import device as D
    c, k, hw, r, st = layer
    pad = r // 2
    g = torch.Generator(device="cuda").manual_seed(c + k + r)
    x = torch.randn((64, c, hw, hw), device="cuda", generator=g).bfloat16().float()
    w = (torch.randn((k, c, r, r), device="cuda", generator=g) *
         (2.0 / (c * r * r)) ** 0.5).bfloat16().float()
    oh = (hw + 2 * pad - r) // st + 1
    res = torch.randn((64, k, oh, oh), device="cuda", generator=g)
    prev = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False
    try:
        ref = torch.relu(F.conv2d(x, w, stride=st, padding=pad) + res)
    finally:
        torch.backends.cudnn.allow_tf32 = prev
    xb = torch.empty((64, c // 64, hw, hw, 64), dtype=torch.bfloat16, device="cuda")
    D.layout_transform(x, xb, 64, c, hw, hw, "NCHW", "NCHW64c")
    wd = D.pack_weights_umma(w, 64, L.MODE_BF16)
    y = 32
    out = torch.empty((64, k // y, oh, oh, y), device="cuda")
    rb = torch.empty((64, k // y, oh, oh, y), device="cuda")
    D.layout_transform(res, rb, 64, k, oh, oh, "NCHW", f"NCHW{y}c")
    p = D.conv_params(L.MODE_BF16, xb, wd, out, 64, c, hw, hw, k, r, r, (st, st), (pad, pad),
                      64, y, residual=rb, relu=True)
    D.conv2d(p)
    got = torch.empty_like(ref)
    D.layout_transform(out, got, 64, k, oh, oh, f"NCHW{y}c", "NCHW")
    torch.cuda.synchronize()
    err = ((got - ref).abs().max() / ref.abs().max().clamp(min=1.0)).item()
    assert err < 1e-4, err


def _resnet50_program(batch):
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph)
    from paper_1809_02697_b200.tuning import DEFAULT_DB
    g = build_model("resnet50", batch=batch, softmax=False)
    prog = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode="bf16",
                                                              db=ScheduleDb(DEFAULT_DB))),
                         0, "bf16")
    return g, prog


def test_fullsize_resnet50_b64_invariance_and_determinism(cuda):
    """The b64 bench program (tuned tiles, CUDA graph): two runs are bitwise
    identical, and images 0 and 63 match separate batch-1 runs (different
    tile shapes) within the bf16 bound with the same top-1."""
    from paper_1809_02697_b200 import model_input
    g64, p64 = _resnet50_program(64)
    feeds = model_input(g64, seed=1)
    name = p64.input_names()[0]
    a = p64.run(feeds)[0]
    b = p64.run(feeds)[0]
    assert np.array_equal(a, b)
    g1, p1 = _resnet50_program(1)
    for i in (0, 63):
        one = p1.run({name: feeds[name][i:i + 1]})[0][0]
        err = np.abs(one - a[i]).max() / max(1.0, np.abs(a[i]).max())
        assert err < 2e-2, (i, err)
        assert one.argmax() == a[i].argmax()
