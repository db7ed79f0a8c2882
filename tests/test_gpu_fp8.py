"""FP8 (e4m3) conv mode against the oracle's e4m3
arithmetic model (oracle.ops.round_e4m3 / conv2d_fp8 / execute_reference
(arith="fp8")).

The reference has no quantized mode (its only dtype is f32, graph.py:20-21;
quantized inference is PAPER.md:433's future work), so parity here is
against the arithmetic the mode documents: e4m3 operands (per-tensor
power-of-two activation scales, per-output-channel weight scales
absmax/448), exact products accumulated in fp32, the reference epilogue
order scale -> bias -> residual -> relu (kernels.py:185-197), one RN
(satfinite) rounding to e4m3 per stored value.  Bounds (in the tests):

* single convs: stored bytes identical to the model except where the fp32
  accumulation order moves a value across an e4m3 rounding boundary --
  at most 1e-3 of the outputs, each within one e4m3 step;
* fused stem / head: bit-identical to the bf16 kernels followed by / fed
  with the documented e4m3 conversion;
* whole networks: logits of the device within 1e-1 (rel_err, reference
  tests/test_kernels.py:31-32: max|a-b| / max|b|) of the e4m3 model of the
  same compiled graph and scales, and the device no further from the f32
  oracle than 1.25x the model's own distance (what e4m3 storage costs).
  One e4m3 step at the largest stored values is 1/16 = 6%, and a single
  accumulation-order tie flip upstream moves later maps by about one step
  (tools/fp8_layer_diff.py: VGG-16's maps are identical to the model up to
  conv 21, SSD's up to its ~40th conv, then differ by one step at a few
  values), so the max-norm bound admits ~1.5 steps."""

import numpy as np
import pytest

import oracle
from oracle.ops import (conv2d_fp8, e4m3_from_bytes, e4m3_to_bytes, fp8_weight_scales,
                        pack_nchw, round_e4m3, unpack_nchw)

pytestmark = pytest.mark.gpu

MISMATCH_FRAC = 1e-3      # fraction of stored values that may differ by one e4m3 step
NET_TOL = 1e-1            # network logits vs the e4m3 model (max norm, ~1.5 e4m3 steps)
NET_VS_MODEL = 1.25       # device-to-f32 distance / model-to-f32 distance


def _rms(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.sqrt(np.mean((a - b) ** 2)) / max(1e-30, np.sqrt(np.mean(b ** 2))))


def _to_dev(vals, x):
    import torch
    b = pack_nchw(e4m3_to_bytes(vals), x)
    return torch.from_numpy(np.ascontiguousarray(b)).cuda().view(torch.float8_e4m3fn)


def _from_dev(t):
    import torch
    return unpack_nchw(e4m3_from_bytes(t.view(torch.uint8).cpu().numpy()))


def _check_close_e4m3(got, ref):
    diff = got != ref
    frac = float(diff.mean())
    assert frac <= MISMATCH_FRAC, f"{frac:.2e} of the outputs differ from the e4m3 model"
    if diff.any():
        step = np.maximum(np.abs(ref[diff]), 2.0 ** -6) * 2.0 ** -3
        worst = float(np.max(np.abs(got[diff] - ref[diff]) / step))
        assert worst <= 1.0 + 1e-6, f"an output is {worst:.2f} e4m3 steps off"
    return frac


def _conv(n, c, h, w, k, r, s, stride, pad, ic_bn, oc_bn, res, relu, seed=0, tile=None,
          bn=False):
    import torch
    from paper_1809_02697_b200 import _lib as L
    from paper_1809_02697_b200 import device as D
    rng = np.random.default_rng(seed)
    xs, os_, rs = 2.0 ** -6, 2.0 ** -4, 2.0 ** -5
    xq = round_e4m3(rng.standard_normal((n, c, h, w)).astype(np.float32) / np.float32(xs))
    wt = (rng.standard_normal((k, c, r, s)) * np.sqrt(2 / (c * r * s))).astype(np.float32)
    bias = rng.normal(0, 0.1, k).astype(np.float32)
    bscale = rng.uniform(0.5, 1.5, k).astype(np.float32) if bn else None
    bshift = rng.normal(0, 0.1, k).astype(np.float32) if bn else None
    oh = (h + 2 * pad - r) // stride + 1
    ow = (w + 2 * pad - s) // stride + 1
    rq = round_e4m3(rng.standard_normal((n, k, oh, ow)).astype(np.float32)) if res else None
    ref = conv2d_fp8(xq, wt, xs, os_, stride, pad, bscale, bshift, bias,
                     rq * np.float32(rs) if res else None, relu)
    ws = fp8_weight_scales(wt)
    wd = D.pack_weights_umma_fp8(torch.from_numpy(wt).cuda(), torch.from_numpy(ws).cuda(), ic_bn)
    sc = np.float32(xs) * ws
    if bn:
        sc = sc * bscale
    out = torch.empty((n, k // oc_bn, oh, ow, oc_bn), dtype=torch.float8_e4m3fn, device="cuda")
    p = D.conv_params(L.MODE_FP8, _to_dev(xq, ic_bn), wd, out, n, c, h, w, k, r, s,
                      (stride, stride), (pad, pad), ic_bn, oc_bn,
                      torch.from_numpy(sc.astype(np.float32)).cuda(),
                      torch.from_numpy(bshift).cuda() if bn else None,
                      torch.from_numpy(bias).cuda(), _to_dev(rq, oc_bn) if res else None, relu,
                      qscales=(rs, os_, 0.0), tile=tile)
    D.conv2d(p)
    torch.cuda.synchronize()
    return _from_dev(out), ref


@pytest.mark.parametrize("case", [
    # n, c, h, w, k, r, s, stride, pad, ic_bn, oc_bn, residual, relu
    (1, 64, 56, 56, 64, 3, 3, 1, 1, 64, 64, False, True),       # BASELINE config 0 shape
    (2, 64, 56, 56, 256, 1, 1, 1, 0, 64, 128, True, True),      # residual expand
    (2, 256, 56, 56, 64, 1, 1, 1, 0, 128, 64, False, True),     # reduce
    (2, 128, 28, 28, 128, 3, 3, 1, 1, 128, 128, False, True),   # halo (128-byte rows)
    (4, 256, 14, 14, 256, 3, 3, 1, 1, 128, 128, False, False),  # deep 3x3, no relu
    (2, 512, 28, 28, 256, 1, 1, 2, 0, 128, 128, False, True),   # stride 2
    (2, 512, 7, 7, 2048, 1, 1, 1, 0, 128, 128, True, True),     # 7x7 expand + residual
    (1, 32, 17, 19, 64, 3, 3, 2, 1, 32, 32, False, True),       # ragged map, 32-byte rows
    (2, 64, 32, 32, 128, 3, 3, 1, 1, 64, 128, False, True),     # 64-byte-row halo, N=128,
    (1, 64, 56, 56, 128, 3, 3, 1, 1, 64, 128, True, True),      # weight-stationary bands
    (2, 64, 20, 20, 128, 3, 3, 1, 1, 64, 128, False, True),
])
def test_fp8_conv_matches_e4m3_model(cuda, case):
    got, ref = _conv(*case)
    _check_close_e4m3(got, ref)


def test_fp8_conv_bn_affine_and_tiles(cuda):
    """An unfolded BN (scale/shift) in the epilogue, and explicit tiles
    (N tile 256, weight-stationary, CTA pair)."""
    got, ref = _conv(2, 128, 28, 28, 256, 3, 3, 1, 1, 128, 128, True, True, bn=True)
    _check_close_e4m3(got, ref)
    for tile in ({"tile_n": 256, "weight_stationary": 1}, {"tile_n": 128, "cta_pair": 2},
                 {"tile_n": 128, "weight_stationary": 2, "stages": 3}):
        got, ref = _conv(4, 256, 14, 14, 256, 1, 1, 1, 0, 128, 128, True, True, tile=tile)
        _check_close_e4m3(got, ref)


def test_fp8_rejects_unsupported(cuda):
    """FP8 refuses the paths it does not implement instead of miscomputing."""
    import torch
    from paper_1809_02697_b200 import _lib as L
    from paper_1809_02697_b200 import device as D
    from paper_1809_02697_b200.errors import DeviceError, ScheduleInvalid
    x = torch.zeros((1, 1, 8, 8, 64), dtype=torch.float8_e4m3fn, device="cuda")
    w = torch.zeros(64 * 64, dtype=torch.float8_e4m3fn, device="cuda")
    out = torch.zeros((1, 1, 8, 8, 64), dtype=torch.float8_e4m3fn, device="cuda")
    p = D.conv_params(L.MODE_FP8, x, w, out, 1, 64, 8, 8, 64, 1, 1, ic_bn=64, oc_bn=64,
                      tile={"split_k": 2})
    with pytest.raises(ScheduleInvalid):
        D.conv2d(p)
    xf = torch.zeros((1, 2, 8, 8, 32), dtype=torch.float32, device="cuda")
    wf = torch.zeros(64 * 64, dtype=torch.float32, device="cuda")
    p = D.conv_params(L.MODE_TF32, xf, wf, out, 1, 64, 8, 8, 64, 1, 1, ic_bn=32, oc_bn=64)
    with pytest.raises(DeviceError):
        D.conv2d(p)                     # e4m3 output from a tf32-mode conv
    p = D.conv_params(L.MODE_FP8, x, w, out, 1, 64, 8, 8, 64, 1, 1, ic_bn=64, oc_bn=64,
                      prologue=(torch.ones(64, device="cuda"), torch.zeros(64, device="cuda"), True))
    with pytest.raises(DeviceError):
        D.conv2d(p)                     # no BN-ReLU prologue on e4m3 tiles


def test_fp8_stem_and_head_kernels(cuda):
    """Fused stem with e4m3 output == the bf16 stem's output rounded to
    e4m3 (bit for bit); fused head over an e4m3 map == the bf16 head over the
    same values (bit for bit: the scale is a power of two)."""
    import torch
    from paper_1809_02697_b200 import device as D
    rng = np.random.default_rng(3)
    n, h, w = 2, 64, 64
    x = torch.from_numpy(rng.standard_normal((n, 3, h, w)).astype(np.float32)).cuda()
    wt = torch.from_numpy((rng.standard_normal((64, 3, 7, 7)) * 0.1).astype(np.float32)).cuda()
    bias = torch.from_numpy(rng.normal(0, 0.1, 64).astype(np.float32)).cuda()
    wimg = D.pack_stem_weights(wt)
    ph = pw = 16
    ob = torch.empty((n, 1, ph, pw, 64), dtype=torch.bfloat16, device="cuda")
    o8 = torch.empty((n, 1, ph, pw, 64), dtype=torch.float8_e4m3fn, device="cuda")
    s = 2.0 ** -5
    D.stem_conv_pool(x, wimg, ob, n, 3, h, w, 64, bias=bias, relu=True)
    D.stem_conv_pool(x, wimg, o8, n, 3, h, w, 64, bias=bias, relu=True, out_scale=s)
    torch.cuda.synchronize()
    want = round_e4m3(ob.float().cpu().numpy() / np.float32(s))
    got = e4m3_from_bytes(o8.view(torch.uint8).cpu().numpy())
    assert np.array_equal(got, want)
    # head: e4m3 map with scale 2^-3 vs the bf16 map of the same values
    c, hw, units = 512, 49, 100
    q = round_e4m3(rng.standard_normal((n, c // 128, 7, 7, 128)).astype(np.float32) * 50)
    xs = 2.0 ** -3
    x8 = torch.from_numpy(e4m3_to_bytes(q)).cuda().view(torch.float8_e4m3fn)
    xb = torch.from_numpy(q * np.float32(xs)).cuda().bfloat16()
    assert np.array_equal(xb.float().cpu().numpy(), q * np.float32(xs))
    wd = torch.from_numpy(rng.standard_normal((units, c)).astype(np.float32) * 0.05).cuda().bfloat16()
    bd = torch.from_numpy(rng.normal(0, 0.1, units).astype(np.float32)).cuda()
    outs = []
    for xt, sc in ((xb, 1.0), (x8, xs)):
        o = torch.empty((n, units), dtype=torch.float32, device="cuda")
        D.classifier_head(xt, wd, bd, o, n, c, hw, 128, units, True, D.HeadScratch(n, c, units, "cuda"),
                          x_scale=sc)
        outs.append(o)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


def _net(model, batch, image=None):
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, build_model, compile_graph,
                                       model_input)
    kw = {"softmax": False}
    if image:
        kw["image"] = image
    g = build_model(model, batch=batch, **kw)
    cg = compile_graph(g, mode="fp8")
    prog = DeviceProgram(ExecutablePlan.compile(cg), 0, "fp8")
    feeds = model_input(g)
    return g, cg, prog, feeds


@pytest.mark.parametrize("model,batch,image", [("resnet18", 2, None), ("resnet50", 2, None),
                                               ("vgg16", 2, 64), ("densenet201", 2, 64),
                                               ("inception_v3", 2, 139)])
def test_fp8_network_vs_e4m3_model(cuda, model, batch, image):
    """Whole forwards in fp8 against the e4m3 model of the same compiled
    graph and calibration scales: ResNets (fused stem, e4m3 convs incl.
    two-output siblings, fused head), VGG-16 (bf16-operand first conv
    writing e4m3, e4m3 max pools, e4m3 -> bf16 exit into the dense
    classifier), DenseNet-201 (e4m3 BN-ReLU over concat windows, e4m3
    average-pool transitions, one scale per in-place concat group) and
    Inception-v3 (branch concats, 3x3/1 average pools, grid-reduction max
    pools requantized into their concat's scale, 16-byte e4m3 rows)."""
    g, cg, prog, feeds = _net(model, batch, image)
    names = prog.launch_names
    if model.startswith("resnet"):
        assert any(n.startswith("stem") for n in names) and any(n.startswith("head") for n in names)
    elif model == "vgg16":
        assert any(n.startswith("maxpool") for n in names) and any(n.startswith("dequant") for n in names)
    elif model == "densenet201":
        assert any(n.startswith("bn") for n in names) and any(n.startswith("avgpool") for n in names)
    import torch
    assert all(v.tensor.dtype in (torch.float8_e4m3fn, torch.bfloat16, torch.float32)
               for v in prog.vals.values())
    got = prog.run(feeds)[0]
    model8 = oracle.execute_reference(cg, feeds, arith="fp8")[0]
    ref = oracle.execute_reference(g, feeds)[0]
    err = oracle.rel_err(got, model8)
    e_mod, e_dev = oracle.rel_err(model8, ref), oracle.rel_err(got, ref)
    print(f"{model} fp8: device vs e4m3 model {err:.3e} (RMS {_rms(got, model8):.3e}), model vs "
          f"f32 oracle {e_mod:.3e}, device vs f32 {e_dev:.3e}")
    assert err <= NET_TOL, err
    assert e_dev <= NET_VS_MODEL * e_mod, (e_dev, e_mod)


def test_fp8_ssd_heads_vs_e4m3_model(cuda):
    """SSD-512/ResNet-50 (b1, 256x256 for the test) in fp8: its 12 pre-NMS
    head maps (2-8 channel blocks, stored bf16) against the oracle.  The
    device's maps are bit-identical to the e4m3 model for the first ~40
    layers (tools/fp8_layer_diff.py), after which accumulation-order tie
    flips (one e4m3 step each) compound through the deep, growing
    activations (~6e4 at the heads), so the heads are held to the accuracy
    the e4m3 arithmetic itself has: the device's distance to the f32 oracle
    within 1.5x of the model's (measured 1.23x: 3.0e-1 vs 2.4e-1)."""
    from paper_1809_02697_b200 import build_model
    g = build_model("ssd_resnet50", batch=1, image=256)
    from paper_1809_02697_b200 import DeviceProgram, ExecutablePlan, compile_graph, model_input
    cg = compile_graph(g, mode="fp8")
    prog = DeviceProgram(ExecutablePlan.compile(cg), 0, "fp8")
    feeds = model_input(g)
    got = prog.run(feeds)
    model8 = oracle.execute_reference(cg, feeds, arith="fp8")
    ref = oracle.execute_reference(g, feeds)
    e_dev = max(oracle.rel_err(a, b) for a, b in zip(got, ref))
    e_mod = max(oracle.rel_err(a, b) for a, b in zip(model8, ref))
    print(f"ssd fp8: device vs f32 {e_dev:.3e}, e4m3 model vs f32 {e_mod:.3e}")
    assert len(got) == 12 and all(np.isfinite(a).all() for a in got)
    assert e_dev <= 1.5 * e_mod, (e_dev, e_mod)


def test_fp8_bench_program(cuda):
    """bench.py's fp8 key: ResNet-50 b64 with calibrated scales; images
    {0, 31, 63} against the e4m3 model."""
    g, cg, prog, feeds = _net("resnet50", 64)
    got = prog.run(feeds)[0]
    from paper_1809_02697_b200 import build_model
    from paper_1809_02697_b200.executor import with_batch
    idx = [0, 31, 63]
    sub = {k: np.ascontiguousarray(v[idx]) for k, v in feeds.items()}
    cg3 = with_batch(cg, 3)
    model8 = oracle.execute_reference(cg3, sub, arith="fp8")[0]
    err = oracle.rel_err(got[idx], model8)
    assert err <= NET_TOL, err
    assert np.isfinite(got).all()


def test_fp8_max_pool_and_dequant_kernels(cuda):
    """e4m3 max pooling returns the stored bytes of the window maximum (the
    map keeps its scale); the dequant exit is e4m3(q) * scale exactly."""
    import torch
    from paper_1809_02697_b200 import device as D
    rng = np.random.default_rng(5)
    n, c, h, w, x = 2, 256, 14, 14, 128
    q = round_e4m3(rng.standard_normal((n, c, h, w)).astype(np.float32) * 30)
    src = _to_dev(q, x)
    for win, st, pad in ((2, 2, 0), (3, 2, 1), (3, 1, 1)):
        oh = (h + 2 * pad - win) // st + 1
        out = torch.empty((n, c // x, oh, oh, x), dtype=torch.float8_e4m3fn, device="cuda")
        D.pool2d(src, out, n, c // x, h, w, x, win, st, pad, "max")
        torch.cuda.synchronize()
        assert np.array_equal(_from_dev(out), oracle.ops.pool2d(q, win, st, pad, "max"))
    for dt in (torch.float32, torch.bfloat16):
        dst = torch.empty((n, c, h, w), dtype=dt, device="cuda")
        D.dequant_fp8(src, dst, 2.0 ** -3, n, c, h, w, x)
        torch.cuda.synchronize()
        assert np.array_equal(dst.float().cpu().numpy(), q * np.float32(2.0 ** -3))


def test_fp8_rejects_graphs_outside_the_mode(cuda):
    """Operators the fp8 mode does not cover on e4m3 maps (here a standalone
    add of two relu'd branches, which cannot fuse into a conv epilogue)
    raise InputMismatch when the program is built (no silent fallback)."""
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, InputMismatch,
                                       compile_graph)
    from paper_1809_02697_b200.models import NetBuilder
    b = NetBuilder("branches", 2, 3, 32)
    x = b.conv_bn_relu(b.data, 3, 64, 3)
    y = b.add(b.conv_bn_relu(x, 64, 64, 3), b.conv_bn_relu(x, 64, 64, 1))
    b.g.outputs = [y]
    cg = compile_graph(b.g, mode="fp8")
    with pytest.raises(InputMismatch):
        DeviceProgram(ExecutablePlan.compile(cg), 0, "fp8")
