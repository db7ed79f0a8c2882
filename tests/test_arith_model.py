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
