"""The oracle's arithmetic model of the single-pass tensor-core modes
(oracle.ops.round_rn / conv2d_rounded): RN rounding to bf16 / tf32 must be
bit-identical to the hardware conversions (torch's f32 -> bf16 RN; tf32 =
RN to 10 explicit mantissa bits, what the kernels' producers store)."""

import numpy as np

import oracle
from oracle import ops


def test_round_rn_bf16_matches_torch(rng):
    import torch
    x = (rng.standard_normal(200_000) * rng.choice([1e-3, 1, 1e3], 200_000)).astype(np.float32)
    x[:4] = [0.0, -0.0, np.float32(1.00390625), np.float32(1.01171875)]   # ties
    want = torch.from_numpy(x).bfloat16().float().numpy()
    assert np.array_equal(ops.round_rn(x, "bf16").view(np.uint32), want.view(np.uint32))


def test_round_rn_tf32_is_rn_even_to_10_bits(rng):
    x = rng.standard_normal(100_000).astype(np.float32)
    r = ops.round_rn(x, "tf32")
    assert not (r.view(np.uint32) & 0x1FFF).any()
    # |error| <= half an ulp of the 10-bit mantissa, ties to even
    ulp = np.ldexp(np.float64(1.0), np.frexp(np.abs(x))[1] - 11)
    assert (np.abs(r.astype(np.float64) - x) <= ulp / 2 + 1e-30).all()
    tie = np.array([1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11], np.float32)
    assert np.array_equal(ops.round_rn(tie, "tf32"), np.array([1.0, 1.0 + 4 * 2.0 ** -11],
                                                               np.float32))


def test_conv2d_rounded_is_the_rounded_conv(rng):
    x = rng.standard_normal((1, 8, 6, 6)).astype(np.float32)
    w = rng.standard_normal((4, 8, 3, 3)).astype(np.float32)
    for kind in ("bf16", "tf32"):
        want = ops.round_rn(ops.conv2d(ops.round_rn(x, kind), ops.round_rn(w, kind), 1, 1), kind)
        assert np.array_equal(ops.conv2d_rounded(kind, x, w, 1, 1), want)
    assert oracle.rel_err(ops.conv2d_rounded("tf32", x, w, 1, 1), ops.conv2d(x, w, 1, 1)) < 3e-3


# --- e4m3 (FP8 mode) ------------------------------------------------------

def test_round_e4m3_matches_torch_float8(rng):
    """oracle.ops.round_e4m3 == torch's float8_e4m3fn conversion (RN-even)
    on 10^6 values over the whole normal / subnormal range, and the byte
    codecs round-trip every finite code."""
    import torch
    x = (rng.standard_normal(1_000_000) * np.exp(rng.uniform(-12, 7, 1_000_000))).astype(np.float32)
    x = np.clip(x, -448, 448)
    x[:6] = [0.0, -0.0, 2.0 ** -9, 2.0 ** -10, 1.0625, 1.1875]      # subnormal / ties
    want = torch.from_numpy(x).to(torch.float8_e4m3fn).float().numpy()
    got = ops.round_e4m3(x)
    assert np.array_equal(got, want)
    codes = np.arange(256, dtype=np.uint8)
    vals = ops.e4m3_from_bytes(codes)
    ref = torch.from_numpy(codes).view(torch.float8_e4m3fn).float().numpy()
    fin = ~np.isnan(ref)
    assert np.array_equal(vals[fin], ref[fin]) and np.isnan(vals[~fin]).all()
    assert np.array_equal(ops.e4m3_from_bytes(ops.e4m3_to_bytes(vals[fin])), vals[fin])


def test_round_e4m3_saturates():
    """satfinite: everything past 448 (in magnitude) stores as +-448."""
    x = np.array([448.0, 460.0, 464.0, 1e6, -1e6, -500.0], np.float32)
    assert np.array_equal(ops.round_e4m3(x), np.array([448, 448, 448, 448, -448, -448], np.float32))


def test_fp8_scales_rules():
    """Weight scales absmax/448 per output channel (1 for zero channels) in
    the product and the oracle are the same numbers; activation scales are
    powers of two covering the margin."""
    from paper_1809_02697_b200 import quant
    w = np.random.default_rng(3).standard_normal((8, 4, 3, 3)).astype(np.float32)
    w[5] = 0
    assert np.array_equal(quant.weight_scales(w), ops.fp8_weight_scales(w))
    assert quant.weight_scales(w)[5] == 1.0
    for a in (1e-3, 0.5, 7.0, 300.0, 448.0, 1e4):
        s = quant.act_scale(a)
        assert s == 2.0 ** round(np.log2(s)) and a * quant.CALIB_MARGIN / s <= 448.0
        assert a * quant.CALIB_MARGIN / s > 224.0
    assert quant.act_scale(0.0) == 1.0


def test_conv2d_fp8_model_is_exact_on_representable_data(rng):
    """With e4m3 inputs and weights already representable and scales 1, the
    model's only rounding is the final RN_e4m3 of the f32 epilogue."""
    x = ops.round_e4m3(rng.standard_normal((1, 8, 6, 6)).astype(np.float32))
    w = ops.round_e4m3(rng.standard_normal((4, 8, 3, 3)).astype(np.float32))
    ws = ops.fp8_weight_scales(w)
    got = ops.conv2d_fp8(x, w, 1.0, None, 1, 1)
    wq = ops.round_e4m3(w / ws.reshape(-1, 1, 1, 1))
    want = ops.conv2d(x, wq, 1, 1, ws, None, None, None, False)
    assert np.array_equal(got, want)
    assert np.array_equal(ops.conv2d_fp8(x, w, 1.0, 2.0, 1, 1), ops.round_e4m3(want / 2))
