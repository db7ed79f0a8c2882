"""Parity of the device conv (tcgen05 bf16 / tf32 and SIMT fp32) against the
CPU oracle, through the C-ABI.  Reference tests mirrored:
tests/test_kernels.py:71-125 (workload/schedule edge cases), :167-186
(epilogue order and residual)."""

import ctypes

import numpy as np
import pytest

import oracle
from oracle.ops import pack_nchw, unpack_nchw, pack_kcrs

pytestmark = pytest.mark.gpu


def bf16_round(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).bfloat16().float().numpy()


def tf32_round(a):
    """RN (ties away) to tf32, like cvt.rna.tf32.f32."""
    b = np.ascontiguousarray(a, np.float32).view(np.uint32).copy()
    finite = np.isfinite(a)
    b[finite] = (b[finite] + np.uint32(0x1000)) & np.uint32(0xFFFFE000)
    return b.view(np.float32)


def run_conv(mode, x_nchw, w_kcrs, stride, pad, ic_bn, oc_bn, scale=None, shift=None,
             bias=None, residual=None, relu=False, out_f32=True, tile=None, pad_channels=False,
             out_cb=None, workspace=False):
    import torch
    from paper_1809_02697_b200 import _lib as L
    from paper_1809_02697_b200 import device as D
    dev = torch.device("cuda:0")
    n, c, h, w = x_nchw.shape
    k, _, r, s = w_kcrs.shape
    sh, sw = stride
    ph, pw = pad
    oh = (h + 2 * ph - r) // sh + 1
    ow = (w + 2 * pw - s) // sw + 1
    if mode == L.MODE_BF16:
        act = torch.bfloat16
    else:
        act = torch.float32
    cb = -(-c // ic_bn)
    xpad = np.zeros((n, cb * ic_bn, h, w), np.float32)
    xpad[:, :c] = x_nchw
    xb = torch.from_numpy(pack_nchw(xpad, ic_bn)).to(dev).to(act)
    if mode == L.MODE_FP32:
        wdev = torch.from_numpy(pack_kcrs(w_kcrs, ic_bn, oc_bn)).to(dev)
    else:
        wdev = D.pack_weights_umma(torch.from_numpy(w_kcrs).to(dev), ic_bn, mode,
                                   pad_channels=pad_channels)
    out_dt = torch.float32 if (out_f32 or mode != L.MODE_BF16) else torch.bfloat16
    kb = k // oc_bn
    total_cb, off = (kb, 0) if out_cb is None else out_cb
    out = torch.full((n, total_cb, oh, ow, oc_bn), float("nan"), dtype=out_dt, device=dev)
    t = lambda v: None if v is None else torch.from_numpy(np.asarray(v, np.float32)).to(dev)
    res = None
    if residual is not None:
        res = torch.from_numpy(pack_nchw(residual, oc_bn)).to(dev).to(out_dt)
    # device vectors stay referenced until the launch finished (the params
    # hold raw pointers)
    vecs = (t(scale), t(shift), t(bias))
    p = D.conv_params(mode, xb, wdev, out, n, c, h, w, k, r, s, (sh, sw), (ph, pw), ic_bn,
                      oc_bn, *vecs, res, relu,
                      out_cb=(off, total_cb) if out_cb else (0, 0),
                      flags=(L.FLAG_PAD_CHANNELS if pad_channels else 0), tile=tile)
    ws = None
    if workspace:
        need = D.conv_workspace_bytes(p)
        ws = torch.zeros(max(need, 4) // 4, dtype=torch.float32, device=dev)
        D.set_workspace(p, ws)
    D.conv2d(p)
    torch.cuda.synchronize()
    o = out.float().cpu().numpy()
    if out_cb is not None:
        return o
    return unpack_nchw(o)


CASES = [
    # (n, c, h, w, k, r, s, stride, pad)
    (1, 64, 56, 56, 64, 3, 3, (1, 1), (1, 1)),      # BASELINE C0
    (2, 64, 14, 14, 128, 1, 1, (1, 1), (0, 0)),     # 1x1
    (2, 64, 28, 28, 128, 1, 1, (2, 2), (0, 0)),     # 1x1 stride 2 (downsample)
    (1, 64, 29, 29, 64, 3, 3, (2, 2), (1, 1)),      # 3x3 stride 2, odd size
    (3, 128, 7, 7, 256, 3, 3, (1, 1), (1, 1)),      # 7x7 maps, several images per tile
    (1, 64, 17, 17, 96, 1, 7, (1, 1), (0, 3)),      # Inception 1x7 asymmetric pad
    (1, 64, 17, 17, 80, 7, 1, (1, 1), (3, 0)),      # Inception 7x1, K=80
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("mode_name", ["bf16", "tf32"])
def test_tc_conv_accumulate(cuda, case, mode_name):
    """Operands pre-rounded to the tensor-core type, f32 output: any error is
    accumulation order only."""
    from paper_1809_02697_b200 import _lib as L
    n, c, h, w, k, r, s, st, pd = case
    rng = np.random.default_rng(hash(case) % 2**32)
    x = rng.standard_normal((n, c, h, w)).astype(np.float32)
    wt = (rng.standard_normal((k, c, r, s)) * np.sqrt(2.0 / (c * r * s))).astype(np.float32)
    rnd = bf16_round if mode_name == "bf16" else tf32_round
    mode = L.MODE_BF16 if mode_name == "bf16" else L.MODE_TF32
    x, wt = rnd(x), rnd(wt)
    ref = oracle.conv2d(x, wt, st, pd)
    x_bn = 64 if mode_name == "bf16" else 32
    x_bn = min(x_bn, c)
    got = run_conv(mode, x, wt, st, pd, x_bn, 16 if k % 16 == 0 else 8)
    assert got.shape == ref.shape
    assert oracle.rel_err(got, ref) < 1e-4


@pytest.mark.parametrize("x_bn", [8, 16, 32, 64])
def test_tc_conv_block_sizes(cuda, x_bn):
    """Every GPU-legal input block size (16..128-byte rows) in bf16."""
    from paper_1809_02697_b200 import _lib as L
    rng = np.random.default_rng(x_bn)
    x = bf16_round(rng.standard_normal((2, 64, 12, 12)).astype(np.float32))
    wt = bf16_round((rng.standard_normal((48, 64, 3, 3)) * 0.06).astype(np.float32))
    ref = oracle.conv2d(x, wt, 1, 1)
    for y in (16, 48):
        got = run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), x_bn, y)
        assert oracle.rel_err(got, ref) < 1e-4


def test_tc_conv_epilogue_order(cuda):
    """scale/shift -> bias -> residual -> relu (kernels.py:185-197)."""
    from paper_1809_02697_b200 import _lib as L
    rng = np.random.default_rng(7)
    x = tf32_round(rng.standard_normal((1, 32, 10, 10)).astype(np.float32))
    wt = tf32_round((rng.standard_normal((32, 32, 3, 3)) * 0.08).astype(np.float32))
    scale = rng.uniform(0.5, 1.5, 32).astype(np.float32)
    shift = rng.uniform(-1, 1, 32).astype(np.float32)
    bias = rng.uniform(-1, 1, 32).astype(np.float32)
    res = rng.standard_normal((1, 32, 10, 10)).astype(np.float32)
    ref = oracle.conv2d(x, wt, 1, 1, scale, shift, bias, res, True)
    got = run_conv(L.MODE_TF32, x, wt, (1, 1), (1, 1), 16, 16, scale, shift, bias, res, True)
    assert oracle.rel_err(got, ref) < 1e-4
    assert (got >= 0).all()


def test_tc_conv_stem_padded_channels(cuda):
    """ResNet stem: C=3 padded to one 8-lane block, 7x7 stride 2 pad 3."""
    from paper_1809_02697_b200 import _lib as L
    rng = np.random.default_rng(3)
    x = bf16_round(rng.standard_normal((2, 3, 64, 64)).astype(np.float32))
    wt = bf16_round((rng.standard_normal((64, 3, 7, 7)) * 0.1).astype(np.float32))
    ref = oracle.conv2d(x, wt, 2, 3)
    got = run_conv(L.MODE_BF16, x, wt, (2, 2), (3, 3), 8, 64, pad_channels=True)
    assert oracle.rel_err(got, ref) < 1e-4


def test_tc_conv_odd_out_channels(cuda):
    """SSD class head: K = 84 = 4 anchors x 21 classes, y = 84 (scalar epilogue)."""
    from paper_1809_02697_b200 import _lib as L
    rng = np.random.default_rng(5)
    x = bf16_round(rng.standard_normal((2, 64, 10, 10)).astype(np.float32))
    wt = bf16_round((rng.standard_normal((84, 64, 3, 3)) * 0.05).astype(np.float32))
    ref = oracle.conv2d(x, wt, 1, 1)
    got = run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), 64, 84)
    assert oracle.rel_err(got, ref) < 1e-4
    got = run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), 64, 12)
    assert oracle.rel_err(got, ref) < 1e-4


def test_tc_conv_concat_window(cuda):
    """Output written into a channel-block window of a wider buffer (concat in place)."""
    from paper_1809_02697_b200 import _lib as L
    rng = np.random.default_rng(11)
    x = bf16_round(rng.standard_normal((1, 32, 8, 8)).astype(np.float32))
    wt = bf16_round((rng.standard_normal((32, 32, 3, 3)) * 0.1).astype(np.float32))
    ref = oracle.conv2d(x, wt, 1, 1)
    o = run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), 32, 16, out_cb=(5, 2))
    got = unpack_nchw(o[:, 2:4])
    assert oracle.rel_err(got, ref) < 1e-4
    assert np.isnan(o[:, :2]).all() and np.isnan(o[:, 4:]).all()


@pytest.mark.parametrize("tile", [
    dict(tile_w=8, tile_h=8, tile_img=1, tile_n=32, slices_per_stage=1, stages=2),
    dict(tile_w=14, tile_h=9, tile_img=1, tile_n=64, slices_per_stage=3, stages=2),
    dict(tile_w=7, tile_h=7, tile_img=2, tile_n=128, slices_per_stage=2, stages=3),
    dict(tile_w=14, tile_h=9, tile_img=1, tile_n=256, slices_per_stage=1, stages=3),
    dict(tile_w=16, tile_h=8, tile_img=1, tile_n=128, slices_per_stage=1, stages=2),  # halo
])
def test_tc_conv_tile_configs(cuda, tile):
    """Explicit tile / pipeline configurations (the tuner's search space)."""
    from paper_1809_02697_b200 import _lib as L
    rng = np.random.default_rng(13)
    x = bf16_round(rng.standard_normal((2, 128, 14, 14)).astype(np.float32))
    wt = bf16_round((rng.standard_normal((256, 128, 3, 3)) * 0.03).astype(np.float32))
    ref = oracle.conv2d(x, wt, 1, 1)
    got = run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), 64, 64, tile=tile)
    assert oracle.rel_err(got, ref) < 1e-4


def test_bf16_end_to_end_c0(cuda):
    """BASELINE config 0 in bf16 storage: within the north_star 2e-2."""
    from paper_1809_02697_b200 import _lib as L
    rng = np.random.default_rng(0)
    x = rng.standard_normal((1, 64, 56, 56)).astype(np.float32)
    wt = (rng.standard_normal((64, 64, 3, 3)) * np.sqrt(2 / 576)).astype(np.float32)
    scale = rng.uniform(0.5, 1.5, 64).astype(np.float32)
    shift = rng.normal(0, 0.1, 64).astype(np.float32)
    ref = oracle.conv2d(x, wt, 1, 1, scale, shift, relu=True)
    got = run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), 64, 64, scale, shift, relu=True,
                   out_f32=False)
    assert oracle.rel_err(got, ref) < 2e-2


@pytest.mark.parametrize("case", CASES[:4])
def test_fp32_direct_matches_oracle(cuda, case):
    """SIMT fp32 path (NEO_MODE_FP32) within the reference's 1e-5 (Acceptance 1)."""
    from paper_1809_02697_b200 import _lib as L
    n, c, h, w, k, r, s, st, pd = case
    rng = np.random.default_rng(1)
    x = rng.standard_normal((n, c, h, w)).astype(np.float32)
    wt = rng.standard_normal((k, c, r, s)).astype(np.float32)
    ref = oracle.conv2d(x, wt, st, pd)
    got = run_conv(L.MODE_FP32, x, wt, st, pd, 16, 16)
    assert oracle.rel_err(got, ref) < 1e-5
    got1 = run_conv(L.MODE_FP32, x, wt, st, pd, 1, 1)
    assert oracle.rel_err(got1, ref) < 1e-5


def test_tc_conv_deterministic(cuda):
    from paper_1809_02697_b200 import _lib as L
    rng = np.random.default_rng(2)
    x = rng.standard_normal((2, 64, 20, 20)).astype(np.float32)
    wt = (rng.standard_normal((64, 64, 3, 3)) * 0.05).astype(np.float32)
    a = run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), 64, 64)
    b = run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), 64, 64)
    assert np.array_equal(a, b)


HALO_CASES = [
    # (n, c, h, w, k, stride, pad, r, s, tile_h)
    (2, 64, 56, 56, 64, 1, (1, 1), 3, 3, 2),      # ResNet stage 1: 58-wide rows
    (2, 128, 28, 28, 128, 1, (1, 1), 3, 3, 4),
    (2, 128, 14, 14, 256, 1, (1, 1), 3, 3, 8),    # exactly 128 rows
    (1, 64, 20, 20, 64, 1, (2, 2), 5, 5, 5),      # 5x5, 24-wide padded rows
    (1, 64, 17, 17, 64, 1, (0, 3), 1, 7, 5),      # 1x7 (Inception)
]


@pytest.mark.parametrize("case", HALO_CASES)
@pytest.mark.parametrize("mode_name", ["bf16", "tf32"])
def test_tc_conv_halo_mode(cuda, case, mode_name):
    """Stride-1 convs in halo mode (tiles span the padded width; horizontal
    taps read one loaded band through row-shifted UMMA descriptors)."""
    from paper_1809_02697_b200 import _lib as L
    n, c, h, w, k, st, pd, r, s, bh = case
    rng = np.random.default_rng(c + r + s)
    rnd = bf16_round if mode_name == "bf16" else tf32_round
    mode = L.MODE_BF16 if mode_name == "bf16" else L.MODE_TF32
    x = rnd(rng.standard_normal((n, c, h, w)).astype(np.float32))
    wt = rnd((rng.standard_normal((k, c, r, s)) * np.sqrt(2.0 / (c * r * s))).astype(np.float32))
    res = rng.standard_normal((n, k, h + 2 * pd[0] - r + 1, w + 2 * pd[1] - s + 1)).astype(np.float32)
    ref = oracle.conv2d(x, wt, st, pd, residual=res, relu=True)
    ow = w + 2 * pd[1] - s + 1
    x_bn = 64 if mode_name == "bf16" else 32
    tile = dict(tile_w=ow + s - 1, tile_h=bh, tile_img=1)
    got = run_conv(mode, x, wt, (st, st), pd, x_bn, 32, residual=res, relu=True, tile=tile)
    assert oracle.rel_err(got, ref) < 1e-4


@pytest.mark.parametrize("rs,pd", [((1, 7), (0, 3)), ((7, 1), (3, 0))])
def test_tc_conv_default_tiles_wide_kernels(cuda, rs, pd):
    """Kernel-picked tiles for Inception's 1x7 / 7x1 convs at 64-lane blocks
    (the halo stage of a 7-tap 1x7 must shrink its N tile to fit)."""
    from paper_1809_02697_b200 import _lib as L
    r, s = rs
    rng = np.random.default_rng(7)
    x = bf16_round(rng.standard_normal((4, 128, 17, 17)).astype(np.float32))
    wt = bf16_round((rng.standard_normal((192, 128, r, s)) * 0.05).astype(np.float32))
    ref = oracle.conv2d(x, wt, (1, 1), pd, relu=True)
    got = run_conv(L.MODE_BF16, x, wt, (1, 1), pd, 64, 64, relu=True)
    assert oracle.rel_err(got, ref) < 1e-4


@pytest.mark.parametrize("case", CASES + [(2, 256, 7, 7, 32, 3, 3, (1, 1), (1, 1))])
@pytest.mark.parametrize("mode_name", ["bf16", "tf32"])
@pytest.mark.parametrize("split", [0, 2, 3])
def test_tc_conv_split_k(cuda, case, mode_name, split):
    """Split-K (partials to the workspace, ordered fixup launch running the
    full epilogue: scale/shift, bias, residual, relu); split 0 = the kernel's
    automatic choice for under-filled grids."""
    from paper_1809_02697_b200 import _lib as L
    n, c, h, w, k, r, s, st, pd = case
    rng = np.random.default_rng(hash(case) % 2**32 + split)
    rnd = bf16_round if mode_name == "bf16" else tf32_round
    mode = L.MODE_BF16 if mode_name == "bf16" else L.MODE_TF32
    x = rnd(rng.standard_normal((n, c, h, w)).astype(np.float32))
    wt = rnd((rng.standard_normal((k, c, r, s)) * np.sqrt(2.0 / (c * r * s))).astype(np.float32))
    oh, ow = (h + 2 * pd[0] - r) // st[0] + 1, (w + 2 * pd[1] - s) // st[1] + 1
    scale = rng.uniform(0.5, 1.5, k).astype(np.float32)
    shift = rng.normal(0, 0.1, k).astype(np.float32)
    bias = rng.normal(0, 0.1, k).astype(np.float32)
    res = rng.standard_normal((n, k, oh, ow)).astype(np.float32)
    ref = oracle.conv2d(x, wt, st, pd, scale, shift, bias, residual=res, relu=True)
    x_bn = min(64 if mode_name == "bf16" else 32, c)
    y = 16 if k % 16 == 0 else 8
    got = run_conv(mode, x, wt, st, pd, x_bn, y, scale, shift, bias, residual=res, relu=True,
                   tile={"split_k": split} if split else None, workspace=True)
    assert oracle.rel_err(got, ref) < 1e-4


def test_tc_conv_split_k_window_and_halo(cuda):
    """Split-K writing into a concat window, and a halo-mode split."""
    from paper_1809_02697_b200 import _lib as L
    rng = np.random.default_rng(5)
    x = bf16_round(rng.standard_normal((1, 128, 14, 14)).astype(np.float32))
    wt = bf16_round((rng.standard_normal((64, 128, 3, 3)) * 0.03).astype(np.float32))
    ref = oracle.conv2d(x, wt, 1, 1, relu=True)
    o = run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), 64, 32, relu=True, out_cb=(5, 1),
                 tile={"split_k": 4}, workspace=True)
    assert oracle.rel_err(unpack_nchw(o[:, 1:3]), ref) < 1e-4
    assert np.isnan(o[:, :1]).all() and np.isnan(o[:, 3:]).all()
    halo = dict(tile_w=16, tile_h=8, tile_img=1, split_k=3)
    got = run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), 64, 32, relu=True, tile=halo,
                   workspace=True)
    assert oracle.rel_err(got, ref) < 1e-4


def test_tc_conv_split_k_needs_workspace(cuda):
    from paper_1809_02697_b200 import _lib as L
    from paper_1809_02697_b200.errors import NeoplanError as NeoError
    rng = np.random.default_rng(6)
    x = bf16_round(rng.standard_normal((1, 64, 8, 8)).astype(np.float32))
    wt = bf16_round((rng.standard_normal((64, 64, 3, 3)) * 0.05).astype(np.float32))
    with pytest.raises(NeoError):
        run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), 64, 64, tile={"split_k": 3})
    # automatic split without a workspace silently runs unsplit
    got = run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), 64, 64)
    assert oracle.rel_err(got, oracle.conv2d(x, wt, 1, 1)) < 1e-4


PAIR_CASES = [
    # (n, c, h, w, k, r, s, stride, pad), tile
    ((2, 64, 28, 28, 128, 1, 1, (1, 1), (0, 0)), {"cta_pair": 2}),
    ((2, 128, 28, 28, 256, 1, 1, (1, 1), (0, 0)), {"cta_pair": 2, "tile_n": 256}),
    ((3, 128, 14, 14, 256, 3, 3, (1, 1), (1, 1)), {"cta_pair": 2}),                     # halo
    ((3, 128, 14, 14, 256, 3, 3, (1, 1), (1, 1)), {"cta_pair": 2, "tile_w": 14, "tile_h": 9,
                                                    "tile_img": 1, "slices_per_stage": 2}),
    ((1, 64, 29, 29, 96, 3, 3, (2, 2), (1, 1)), {"cta_pair": 2, "tile_n": 96}),         # odd M tiles
    ((1, 3, 30, 30, 64, 3, 3, (1, 1), (1, 1)), {"cta_pair": 2}),                        # padded C
]


@pytest.mark.parametrize("case,tile", PAIR_CASES)
@pytest.mark.parametrize("mode_name", ["bf16", "tf32"])
def test_tc_conv_cta_pair(cuda, case, tile, mode_name):
    """cta_group::2 tiles: two CTAs hold the halves of a 256-row M tile and
    of the weight rows; full epilogue with residual, dummy odd M tiles."""
    from paper_1809_02697_b200 import _lib as L
    n, c, h, w, k, r, s, st, pd = case
    rng = np.random.default_rng(k + r + c)
    rnd = bf16_round if mode_name == "bf16" else tf32_round
    mode = L.MODE_BF16 if mode_name == "bf16" else L.MODE_TF32
    x = rnd(rng.standard_normal((n, c, h, w)).astype(np.float32))
    wt = rnd((rng.standard_normal((k, c, r, s)) * np.sqrt(2.0 / (c * r * s))).astype(np.float32))
    oh, ow = (h + 2 * pd[0] - r) // st[0] + 1, (w + 2 * pd[1] - s) // st[1] + 1
    bias = rng.normal(0, 0.1, k).astype(np.float32)
    res = rng.standard_normal((n, k, oh, ow)).astype(np.float32)
    ref = oracle.conv2d(x, wt, st, pd, bias=bias, residual=res, relu=True)
    lanes = 8 if mode_name == "bf16" else 4
    x_bn = min(64 if mode_name == "bf16" else 32, c) if c >= lanes else lanes
    got = run_conv(mode, x, wt, st, pd, x_bn, 32, bias=bias, residual=res, relu=True, tile=tile,
                   pad_channels=c < lanes)
    assert oracle.rel_err(got, ref) < 1e-4


@pytest.mark.parametrize("mode_name", ["bf16", "tf32"])
@pytest.mark.parametrize("shape", [(2, 128, 14, 14, 128, 32), (1, 256, 7, 7, 64, 64),
                                   (3, 64, 9, 11, 48, 16)])
def test_tc_conv_bn_relu_prologue(cuda, mode_name, shape):
    """BN-ReLU fused into a 1x1 conv's shared-memory tiles equals the
    unfused scale-shift-relu launch followed by the conv, bit for bit, and
    the oracle within accumulation error."""
    import torch
    from paper_1809_02697_b200 import _lib as L
    from paper_1809_02697_b200 import device as D
    n, c, h, w, k, x_bn = shape
    if mode_name == "tf32":
        x_bn = min(x_bn, 32)
    rng = np.random.default_rng(c + k)
    mode = L.MODE_BF16 if mode_name == "bf16" else L.MODE_TF32
    act = torch.bfloat16 if mode_name == "bf16" else torch.float32
    rnd = bf16_round if mode_name == "bf16" else tf32_round
    x = rnd(rng.standard_normal((n, c, h, w)).astype(np.float32))
    wt = rnd((rng.standard_normal((k, c, 1, 1)) * np.sqrt(2.0 / c)).astype(np.float32))
    scale = rng.uniform(0.5, 1.5, c).astype(np.float32)
    shift = rng.normal(0, 0.3, c).astype(np.float32)
    dev = torch.device("cuda")
    xb = torch.from_numpy(pack_nchw(x, x_bn)).to(dev).to(act)
    sc, sh = torch.from_numpy(scale).to(dev), torch.from_numpy(shift).to(dev)
    flags = L.FLAG_ROUND_TF32 if mode_name == "tf32" else 0
    tmp = torch.empty_like(xb)
    D.eltwise(L.ELT_SCALE_SHIFT_RELU, xb, None, tmp, n, c // x_bn, h * w, x_bn, sc, sh, flags)
    wd = D.pack_weights_umma(torch.from_numpy(wt).to(dev), x_bn, mode)
    y = 16
    out_a = torch.empty((n, k // y, h, w, y), device=dev)
    out_b = torch.empty_like(out_a)
    pa = D.conv_params(mode, tmp, wd, out_a, n, c, h, w, k, 1, 1, (1, 1), (0, 0), x_bn, y,
                       relu=True)
    pb = D.conv_params(mode, xb, wd, out_b, n, c, h, w, k, 1, 1, (1, 1), (0, 0), x_bn, y,
                       relu=True, prologue=(sc, sh, True))
    D.conv2d(pa)
    D.conv2d(pb)
    torch.cuda.synchronize()
    assert torch.equal(out_a, out_b)
    pre = np.maximum(x * scale[None, :, None, None] + shift[None, :, None, None], 0)
    ref = oracle.conv2d(rnd(pre.astype(np.float32)), wt, 1, 0, relu=True)
    assert oracle.rel_err(unpack_nchw(out_b.cpu().numpy()), ref) < 1e-4
    with pytest.raises(Exception):     # padded / wider kernels are rejected
        bad = D.conv_params(mode, xb, D.pack_weights_umma(
            torch.from_numpy(rnd(rng.standard_normal((k, c, 3, 3)).astype(np.float32))).to(dev),
            x_bn, mode), out_b, n, c, h, w, k, 3, 3, (1, 1), (1, 1), x_bn, y,
            prologue=(sc, sh, True))
        D.conv2d(bad)


@pytest.mark.parametrize("mode_name", ["bf16", "tf32"])
@pytest.mark.parametrize("ka,kb,tile_n,stride", [(128, 512, 128, 2), (256, 256, 256, 1),
                                                 (128, 192, 128, 1)])
def test_tc_conv_two_outputs(cuda, mode_name, ka, kb, tile_n, stride):
    """Sibling 1x1 convs as one launch: channels [0, ka) -> out (relu, bias),
    [ka, ka + kb) -> out2 (no relu, scale/shift) written into a channel window
    of a larger buffer; each part matches its own oracle conv."""
    import torch
    from paper_1809_02697_b200 import _lib as L
    from paper_1809_02697_b200 import device as D
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(ka + kb + stride)
    n, c, h, w = 4, 128, 14, 14
    rnd = bf16_round if mode_name == "bf16" else tf32_round
    mode = L.MODE_BF16 if mode_name == "bf16" else L.MODE_TF32
    act = torch.bfloat16 if mode_name == "bf16" else torch.float32
    x = rnd(rng.standard_normal((n, c, h, w)).astype(np.float32))
    wa = rnd((rng.standard_normal((ka, c, 1, 1)) * 0.1).astype(np.float32))
    wb = rnd((rng.standard_normal((kb, c, 1, 1)) * 0.1).astype(np.float32))
    ba = rng.normal(0, 0.1, ka).astype(np.float32)
    sb = rng.uniform(0.5, 1.5, kb).astype(np.float32)
    tb = rng.normal(0, 0.1, kb).astype(np.float32)
    oh = (h - 1) // stride + 1
    y = 8 if kb % 16 else 16
    xb = 64 if mode_name == "bf16" else 32
    xt = torch.from_numpy(pack_nchw(x, xb)).to(dev).to(act)
    wd = D.pack_weights_umma(torch.from_numpy(np.concatenate([wa, wb])).to(dev), xb, mode)
    oa = torch.empty((n, ka // y, oh, oh, y), dtype=act, device=dev)
    ob = torch.full((n, kb // y + 3, oh, oh, y), 5.0, dtype=act, device=dev)
    cat = lambda a, b: torch.from_numpy(np.concatenate([a, b]).astype(np.float32)).to(dev)
    p = D.conv_params(mode, xt, wd, oa, n, c, h, w, ka + kb, 1, 1, (stride, stride), (0, 0),
                      xb, y, cat(np.ones(ka), sb), cat(np.zeros(ka), tb), cat(ba, np.zeros(kb)),
                      None, True, tile={"tile_n": tile_n},
                      second=(ob, ka, False, (2, kb // y + 3)),
                      flags=L.FLAG_ROUND_TF32 if mode_name == "tf32" else 0)
    D.conv2d(p)
    torch.cuda.synchronize()
    ref_a = oracle.conv2d(x, wa, stride, 0, None, None, ba, relu=True)
    ref_b = oracle.conv2d(x, wb, stride, 0, sb, tb, None, relu=False)
    got_a = unpack_nchw(oa.float().cpu().numpy())
    obn = ob.float().cpu().numpy()
    got_b = unpack_nchw(obn[:, 2:2 + kb // y])
    tol = 2e-2 if mode_name == "bf16" else 1e-3
    assert oracle.rel_err(got_a, ref_a) < tol and oracle.rel_err(got_b, ref_b) < tol
    assert np.all(obn[:, :2] == 5.0) and np.all(obn[:, 2 + kb // y:] == 5.0)


@pytest.mark.gpu
def test_tc_conv_default_geometry_large_odd_maps(cuda):
    """Windowed conv over a large odd map with several images, too wide for
    halo tiles (Inception-v3's 147x147 3x3 layers at batch 128): the kernel's
    own geometry keeps an M tile inside ONE image (the unrestricted pick is a
    few pixels x many images, 22-29% slower there, tools/geo_sweep.py), and
    stays exact; a 1x1 conv over the same map keeps the image-spanning tile."""
    import torch
    from paper_1809_02697_b200 import _lib as L
    from paper_1809_02697_b200 import device as D
    rng = np.random.default_rng(11)
    n, c, k, hw = 16, 32, 32, 131
    x = bf16_round(rng.standard_normal((n, c, hw, hw)).astype(np.float32))
    wt = bf16_round((rng.standard_normal((k, c, 1, 3)) * 0.1).astype(np.float32))
    dev = torch.device("cuda:0")
    xb = torch.from_numpy(pack_nchw(x, 32)).to(dev).bfloat16()
    wd = D.pack_weights_umma(torch.from_numpy(wt).to(dev), 32, L.MODE_BF16)
    out = torch.empty((n, 1, hw, hw - 2, 32), dtype=torch.float32, device=dev)
    p = D.conv_params(L.MODE_BF16, xb, wd, out, n, c, hw, hw, k, 1, 3, (1, 1), (0, 0), 32, 32)
    cfg = D.default_tiles(p)
    assert cfg["tile_img"] == 1 and cfg["tile_w"] <= hw - 2, cfg
    assert cfg["tile_w"] * cfg["tile_h"] >= 0.85 * 128, cfg
    w1 = bf16_round((rng.standard_normal((k, c, 1, 1)) * 0.2).astype(np.float32))
    wd1 = D.pack_weights_umma(torch.from_numpy(w1).to(dev), 32, L.MODE_BF16)
    out1 = torch.empty((n, 1, hw, hw, 32), dtype=torch.float32, device=dev)
    p1 = D.conv_params(L.MODE_BF16, xb, wd1, out1, n, c, hw, hw, k, 1, 1, (1, 1), (0, 0), 32, 32)
    assert D.default_tiles(p1)["tile_img"] > 1
    ref = oracle.conv2d(x, wt, (1, 1), (0, 0), relu=True)
    got = run_conv(L.MODE_BF16, x, wt, (1, 1), (0, 0), 32, 32, relu=True)
    assert oracle.rel_err(got, ref) < 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("mode_name", ["bf16", "tf32"])
@pytest.mark.parametrize("shape,stride", [((3, 64, 29, 31), (2, 2)), ((2, 128, 28, 28), (2, 2)),
                                          ((2, 64, 17, 23), (3, 2)), ((5, 64, 8, 8), (2, 1))])
def test_tc_conv_strided_1x1(cuda, mode_name, shape, stride):
    """Strided unpadded 1x1 convs (the downsampling projections): odd sizes,
    unequal strides, residual + relu epilogue.  (A strided-VIEW tensor map --
    map strides = conv strides, dense boxes -- was measured against the
    element-stride boxes used here: identical times, not kept.)"""
    from paper_1809_02697_b200 import _lib as L
    n, c, h, w = shape
    k = 128
    rng = np.random.default_rng(h * 100 + w)
    rnd = bf16_round if mode_name == "bf16" else tf32_round
    mode = L.MODE_BF16 if mode_name == "bf16" else L.MODE_TF32
    x = rnd(rng.standard_normal(shape).astype(np.float32))
    wt = rnd((rng.standard_normal((k, c, 1, 1)) * np.sqrt(2.0 / c)).astype(np.float32))
    oh, ow = (h - 1) // stride[0] + 1, (w - 1) // stride[1] + 1
    res = rng.standard_normal((n, k, oh, ow)).astype(np.float32)
    bias = rng.standard_normal(k).astype(np.float32)
    ref = oracle.conv2d(x, wt, stride, (0, 0), bias=bias, residual=res, relu=True)
    got = run_conv(mode, x, wt, stride, (0, 0), 64 if mode_name == "bf16" else 32, 32, bias=bias,
                   residual=res, relu=True)
    assert got.shape == ref.shape
    assert oracle.rel_err(got, ref) < 1e-4


STRIP_CASES = [
    # (n, c, h, w, k, r, s, pad, ic_bn_bf16) -- maps wider than one 128-row halo tile
    (2, 64, 40, 150, 64, 3, 3, (1, 1), 64),      # 128-byte rows, 2 strips
    (1, 64, 33, 224, 128, 3, 3, (1, 1), 64),     # VGG width, several strips x rows
    (2, 32, 37, 147, 32, 3, 3, (0, 0), 32),      # Inception conv10: 64-byte rows, no pad
    (1, 64, 20, 140, 256, 1, 7, (0, 3), 64),     # 7 horizontal taps, two N tiles
    (3, 128, 9, 129, 64, 3, 3, (1, 1), 64),      # few rows, two channel blocks
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", STRIP_CASES)
@pytest.mark.parametrize("mode_name", ["bf16", "tf32"])
@pytest.mark.parametrize("wst", [0, 1])
def test_tc_conv_halo_strips(cuda, case, mode_name, wst):
    """Halo column strips (NEO_FLAG_HALO_STRIPS): stride-1 windowed convs over
    maps wider than one 128-row tile; the kernel picks the strips itself when
    only the geometry is left to it.  Residual + relu epilogue, exact
    accumulation check, and the picked geometry really is a strip."""
    import torch
    from paper_1809_02697_b200 import _lib as L
    from paper_1809_02697_b200 import device as D
    n, c, h, w, k, r, s, pd, xb16 = case
    rng = np.random.default_rng(h * 1000 + w)
    rnd = bf16_round if mode_name == "bf16" else tf32_round
    mode = L.MODE_BF16 if mode_name == "bf16" else L.MODE_TF32
    x_bn = xb16 if mode_name == "bf16" else min(32, xb16)
    x = rnd(rng.standard_normal((n, c, h, w)).astype(np.float32))
    wt = rnd((rng.standard_normal((k, c, r, s)) * np.sqrt(2.0 / (c * r * s))).astype(np.float32))
    oh, ow = h + 2 * pd[0] - r + 1, w + 2 * pd[1] - s + 1
    res = rng.standard_normal((n, k, oh, ow)).astype(np.float32)
    bias = rng.standard_normal(k).astype(np.float32)
    ref = oracle.conv2d(x, wt, (1, 1), pd, bias=bias, residual=res, relu=True)
    tile = {"weight_stationary": wst} if wst else None
    got = run_conv(mode, x, wt, (1, 1), pd, x_bn, 32, bias=bias, residual=res, relu=True,
                   tile=tile)
    assert got.shape == ref.shape
    assert oracle.rel_err(got, ref) < 1e-4
    # the kernel's own geometry for this shape: band narrower than the map,
    # at most 128 rows, one image
    dev = torch.device("cuda:0")
    act = torch.bfloat16 if mode_name == "bf16" else torch.float32
    xb = torch.empty((n, c // x_bn, h, w, x_bn), dtype=act, device=dev)
    wd = D.pack_weights_umma(torch.from_numpy(wt).to(dev), x_bn, mode)
    out = torch.empty((n, k // 32, oh, ow, 32), dtype=torch.float32, device=dev)
    p = D.conv_params(mode, xb, wd, out, n, c, h, w, k, r, s, (1, 1), pd, x_bn, 32)
    q = L.ConvParams.from_buffer_copy(p)
    L.check(L.load().neo_conv_default_tiles(ctypes.byref(q)), "neo_conv_default_tiles")
    assert q.flags & L.FLAG_HALO_STRIPS, "wide stride-1 windowed conv should run halo strips"
    assert q.tile_img == 1 and s <= q.tile_w < ow and q.tile_w * q.tile_h <= 128


@pytest.mark.gpu
def test_tc_conv_halo_strips_keep_explicit_tiles(cuda):
    """Explicit tile parameters (tuned for plain tiles) switch the automatic
    strips off; the result is the same conv either way."""
    from paper_1809_02697_b200 import _lib as L
    rng = np.random.default_rng(5)
    x = bf16_round(rng.standard_normal((1, 64, 24, 160)).astype(np.float32))
    wt = bf16_round((rng.standard_normal((64, 64, 3, 3)) * 0.06).astype(np.float32))
    ref = oracle.conv2d(x, wt, (1, 1), (1, 1), relu=True)
    a = run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), 64, 64, relu=True)
    b = run_conv(L.MODE_BF16, x, wt, (1, 1), (1, 1), 64, 64, relu=True,
                 tile={"tile_n": 64, "slices_per_stage": 1, "stages": 3})
    assert oracle.rel_err(a, ref) < 1e-4 and oracle.rel_err(b, ref) < 1e-4


HALO32_CASES = [
    # (n, c, h, w, k, r, s, pad, x_bn, mode): stride-1 windowed convs over 32-byte rows
    (2, 48, 35, 35, 64, 5, 5, (2, 2), 16, "bf16"),     # Inception 5x5 over 48 channels
    (2, 80, 37, 37, 192, 3, 3, (0, 0), 16, "bf16"),    # 80 channels = 5 x 16, two N tiles
    (1, 32, 17, 17, 96, 1, 7, (0, 3), 16, "bf16"),     # 7 horizontal taps
    (3, 16, 20, 50, 32, 3, 3, (1, 1), 16, "bf16"),     # one channel block
    (2, 32, 30, 140, 64, 3, 3, (1, 1), 16, "bf16"),    # wide map: strips over 32-byte rows
    (2, 80, 30, 73, 64, 3, 3, (0, 0), 16, "bf16"),     # 71 of 128 rows full-width -> strips
    (2, 24, 28, 28, 64, 3, 3, (1, 1), 8, "tf32"),      # tf32 blocks of 8 channels
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", HALO32_CASES)
@pytest.mark.parametrize("wst", [0, 1, 2])
def test_tc_conv_halo_32_byte_rows(cuda, case, wst):
    """Halo (band-reuse) mainloop over 32-byte rows (SWIZZLE_32B shifted
    views: kMmaHalo32 / kMmaHaloWst32), full-width tiles and strips, with the
    weight-stationary choice left to the kernel, forced off and forced on."""
    from paper_1809_02697_b200 import _lib as L
    n, c, h, w, k, r, s, pd, xb, mode = case
    rng = np.random.default_rng(c * 7 + h)
    rnd = bf16_round if mode == "bf16" else tf32_round
    x = rnd(rng.standard_normal((n, c, h, w)).astype(np.float32))
    wt = rnd((rng.standard_normal((k, c, r, s)) * np.sqrt(2.0 / (c * r * s))).astype(np.float32))
    bias = rng.standard_normal(k).astype(np.float32)
    ref = oracle.conv2d(x, wt, (1, 1), pd, bias=bias, relu=True)
    tile = {"weight_stationary": wst} if wst else None
    try:
        got = run_conv(L.MODE_BF16 if mode == "bf16" else L.MODE_TF32, x, wt, (1, 1), pd, xb, 32,
                       bias=bias, relu=True, tile=tile)
    except Exception as exc:       # forced weight-stationary tiles may not fit shared memory
        from paper_1809_02697_b200.errors import ScheduleInvalid
        if wst == 2 and isinstance(exc, ScheduleInvalid):
            pytest.skip(str(exc)[:80])
        raise
    assert oracle.rel_err(got, ref) < 1e-4
