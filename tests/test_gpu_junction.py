"""The bottleneck-junction kernel (neo_conv_junction: a block's 1x1 expand
conv with its fused shortcut, chained in shared memory into the next block's
1x1 reduce conv) against the two stand-alone tensor-core convs it replaces --
bit for bit -- and against the CPU oracle; plus the executor's use of it."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

SHAPES = [  # (n, c1, hw, n1, n2): ResNet-50's junctions at 56^2, 28^2, 14^2
    (2, 64, 56, 256, 64),
    (3, 128, 28, 512, 128),
    (5, 256, 14, 1024, 256),
    (4, 64, 9, 128, 192),
]


def _run(n, c1, hw, n1, n2, residual=True, seed=0):
    import torch
    from paper_1809_02697_b200 import _lib as L
    from paper_1809_02697_b200 import device as D
    g = torch.Generator(device="cuda").manual_seed(seed)
    dev = "cuda"
    x = torch.randn((n, c1 // 64, hw, hw, 64), device=dev, generator=g).bfloat16()
    w1 = torch.randn((n1, c1, 1, 1), device=dev, generator=g) * (2.0 / c1) ** 0.5
    w2 = torch.randn((n2, n1, 1, 1), device=dev, generator=g) * (2.0 / n1) ** 0.5
    b1 = torch.randn(n1, device=dev, generator=g) * 0.1
    b2 = torch.randn(n2, device=dev, generator=g) * 0.1
    res = torch.randn((n, n1 // 64, hw, hw, 64), device=dev, generator=g).bfloat16() \
        if residual else None
    wd1 = D.pack_weights_umma(w1, 64, L.MODE_BF16)
    wd2 = D.pack_weights_umma(w2, 64, L.MODE_BF16)
    y1 = torch.full((n, n1 // 64, hw, hw, 64), float("nan"), device=dev).bfloat16()
    y2 = torch.full((n, n2 // 64, hw, hw, 64), float("nan"), device=dev).bfloat16()
    D.conv_junction(x, wd1, b1, res, y1, wd2, b2, y2, n, c1, hw, hw, n1, n2)
    # the two stand-alone convs
    z1 = torch.empty_like(y1)
    z2 = torch.empty_like(y2)
    p1 = D.conv_params(L.MODE_BF16, x, wd1, z1, n, c1, hw, hw, n1, 1, 1, (1, 1), (0, 0), 64, 64,
                       bias=b1, residual=res, relu=True)
    D.conv2d(p1)
    p2 = D.conv_params(L.MODE_BF16, z1, wd2, z2, n, n1, hw, hw, n2, 1, 1, (1, 1), (0, 0), 64, 64,
                       bias=b2, relu=True)
    D.conv2d(p2)
    torch.cuda.synchronize()
    return x, w1, w2, b1, b2, res, y1, y2, z1, z2


@pytest.mark.parametrize("shape", SHAPES)
def test_junction_bitwise_equals_two_convs(cuda, shape):
    _, _, _, _, _, _, y1, y2, z1, z2 = _run(*shape)
    assert not y1.float().isnan().any() and not y2.float().isnan().any()
    import torch
    assert y1.view(torch.int16).equal(z1.view(torch.int16))
    assert y2.view(torch.int16).equal(z2.view(torch.int16))


def test_junction_without_residual_vs_oracle(cuda):
    import torch
    n, c1, hw, n1, n2 = 2, 128, 12, 256, 64
    x, w1, w2, b1, b2, _, y1, y2, z1, z2 = _run(n, c1, hw, n1, n2, residual=False, seed=3)
    assert y2.view(torch.int16).equal(z2.view(torch.int16))
    xf = oracle.unpack_nchw(x.float().cpu().numpy())
    r1 = oracle.conv2d(xf, w1.bfloat16().float().cpu().numpy(), 1, 0,
                       bias=b1.cpu().numpy(), relu=True)
    got1 = oracle.unpack_nchw(y1.float().cpu().numpy())
    assert oracle.rel_err(got1, r1) < 2e-2
    r1b = torch.from_numpy(r1).bfloat16().float().numpy()
    r2 = oracle.conv2d(r1b, w2.bfloat16().float().cpu().numpy(), 1, 0,
                       bias=b2.cpu().numpy(), relu=True)
    got2 = oracle.unpack_nchw(y2.float().cpu().numpy())
    assert oracle.rel_err(got2, r2) < 2e-2


def test_resnet50_b64_uses_junctions_and_matches_unfused(cuda, monkeypatch):
    """The bench program with junctions equals the program without them bit
    for bit (same arithmetic, two launches fewer per junction)."""
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph, model_input)
    from paper_1809_02697_b200.tuning import DEFAULT_DB
    g = build_model("resnet50", batch=64, softmax=False)
    planned = compile_graph(g, mode="bf16", db=ScheduleDb(DEFAULT_DB))
    monkeypatch.setenv("NEOB200_JUNCTION", "1")       # opt-in (see executor._lower)
    fused = DeviceProgram(ExecutablePlan.compile(planned), 0, "bf16")
    names = fused.launch_names
    assert sum(">" in n for n in names) >= 8, names
    monkeypatch.delenv("NEOB200_JUNCTION")
    plain = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode="bf16",
                                                               db=ScheduleDb(DEFAULT_DB))),
                          0, "bf16")
    assert len(plain.launch_names) > len(names)
    feeds = model_input(g, seed=1)
    a, b = fused.run(feeds)[0], plain.run(feeds)[0]
    assert np.array_equal(a, b)
