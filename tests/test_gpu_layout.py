"""Bit-exact device layout transforms vs the oracle (reference
tests/test_layout.py:74-117 index mappings and round trips,
tests/test_acceptance.py:114-142 exhaustive round trips for C <= 32)."""

import numpy as np
import pytest

from oracle import ops as O

pytestmark = pytest.mark.gpu


def _dev(a, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t if dtype is None else t.to(dtype)


def _empty(shape, dtype):
    import torch
    return torch.full(shape, float("nan"), dtype=dtype, device="cuda")


@pytest.mark.parametrize("shape,x", [((2, 12, 5, 7), 4), ((1, 64, 56, 56), 16),
                                     ((3, 48, 9, 9), 48), ((2, 8, 33, 31), 8),
                                     ((1, 256, 7, 7), 64), ((2, 6, 3, 3), 1)])
def test_pack_unpack_bitexact_f32(cuda, shape, x):
    import torch
    from paper_1809_02697_b200 import device as D
    rng = np.random.default_rng(0)
    a = rng.standard_normal(shape).astype(np.float32)
    n, c, h, w = shape
    src = _dev(a)
    dst = _empty((n, c // x, h, w, x), torch.float32)
    D.layout_transform(src, dst, n, c, h, w, "NCHW", f"NCHW{x}c")
    packed = dst.cpu().numpy()
    assert np.array_equal(packed.view(np.uint32), O.pack_nchw(a, x).view(np.uint32))
    back = _empty(shape, torch.float32)
    D.layout_transform(dst, back, n, c, h, w, f"NCHW{x}c", "NCHW")
    assert np.array_equal(back.cpu().numpy().view(np.uint32), a.view(np.uint32))


def test_exhaustive_round_trip_small(cuda):
    """every (C <= 32, x | C) pair, like Acceptance 2."""
    import torch
    from paper_1809_02697_b200 import device as D
    rng = np.random.default_rng(1)
    for c in range(1, 33):
        a = rng.standard_normal((2, c, 3, 5)).astype(np.float32)
        src = _dev(a)
        for x in [d for d in range(1, c + 1) if c % d == 0]:
            p = _empty((2, c // x, 3, 5, x), torch.float32)
            D.layout_transform(src, p, 2, c, 3, 5, "NCHW", f"NCHW{x}c")
            assert np.array_equal(p.cpu().numpy(), O.pack_nchw(a, x))
            b = _empty((2, c, 3, 5), torch.float32)
            D.layout_transform(p, b, 2, c, 3, 5, f"NCHW{x}c", "NCHW")
            assert np.array_equal(b.cpu().numpy(), a)


def test_retile_and_nhwc(cuda):
    import torch
    from paper_1809_02697_b200 import device as D
    rng = np.random.default_rng(2)
    a = rng.standard_normal((2, 48, 6, 6)).astype(np.float32)
    p16 = _dev(O.pack_nchw(a, 16))
    for b in (1, 3, 8, 16, 48):
        out = _empty((2, 48 // b, 6, 6, b), torch.float32)
        D.layout_transform(p16, out, 2, 48, 6, 6, "NCHW16c", f"NCHW{b}c")
        assert np.array_equal(out.cpu().numpy(), O.pack_nchw(a, b))
    nhwc = rng.standard_normal((2, 5, 7, 3)).astype(np.float32)
    out = _empty((2, 3, 5, 7), torch.float32)
    D.layout_transform(_dev(nhwc), out, 2, 3, 5, 7, "NHWC", "NCHW")
    assert np.array_equal(out.cpu().numpy(), O.nhwc_to_nchw(nhwc))


def test_pack_bf16_and_padding(cuda):
    import torch
    from paper_1809_02697_b200 import device as D
    from paper_1809_02697_b200 import _lib as L
    rng = np.random.default_rng(3)
    a = rng.standard_normal((2, 3, 10, 10)).astype(np.float32)
    out = _empty((2, 1, 10, 10, 8), torch.bfloat16)
    D.layout_transform(_dev(a), out, 2, 3, 10, 10, "NCHW", "NCHW8c", flags=L.FLAG_PAD_CHANNELS)
    got = out.float().cpu().numpy()
    ref = torch.from_numpy(a).bfloat16().float().numpy()
    assert np.array_equal(got[:, 0, :, :, :3], ref.transpose(0, 2, 3, 1))
    assert (got[:, 0, :, :, 3:] == 0).all()
    from paper_1809_02697_b200.errors import IndivisibleChannel
    with pytest.raises(IndivisibleChannel):
        D.layout_transform(_dev(a), out, 2, 3, 10, 10, "NCHW", "NCHW8c")


def test_weight_pack_bitexact(cuda):
    import torch
    from paper_1809_02697_b200 import device as D
    rng = np.random.default_rng(4)
    w = rng.standard_normal((8, 4, 3, 3)).astype(np.float32)
    for x, y in [(2, 4), (4, 8), (1, 1), (4, 2)]:
        dst = _empty((8 // y, 4 // x, 3, 3, x, y), torch.float32)
        D.pack_weights(_dev(w), dst, x, y)
        assert np.array_equal(dst.cpu().numpy(), O.pack_kcrs(w, x, y))
        back = _empty((8, 4, 3, 3), torch.float32)
        D.unpack_weights(dst, back)
        assert np.array_equal(back.cpu().numpy(), w)
