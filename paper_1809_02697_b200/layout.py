"""Layout descriptors, the Tensor container, and the public layout transforms.

API mirrors the reference layout.py (Layout :21-71, nchwc/kcrsck :79-84,
aligned_empty :87-92, Tensor :95-125, array transforms :131-235, Tensor-level
wrappers :189-216).  Differences, by design:

* a Tensor may live on the host (numpy) or on a B200 (torch CUDA tensor);
* every transform executes on the GPU through libneob200 (K-LAYOUT), also for
  host tensors (uploaded, transformed, downloaded) -- there is no CPU path.
  The results are bit-identical to the reference's numpy permutations
  (tests/test_gpu_layout.py, tests/test_oracle_golden.py);
* a blocked layout may carry zero-filled pad lanes when explicitly requested
  (``pad_channels=True``), which the tensor-core stem needs for C=3.
"""

from __future__ import annotations

import re
from dataclasses import dataclass

import numpy as np

from .errors import IndivisibleChannel, WrongLayout

ALIGNMENT = 64

_RANK = {"NCHW": 4, "NHWC": 4, "NCHWc": 5, "KCRS": 4, "KCRSck": 6, "VEC": 1, "MAT": 2}


@dataclass(frozen=True)
class Layout:
    """tag in NCHW | NHWC | NCHWc | KCRS | KCRSck | VEC | MAT; x / y are the
    channel / output-channel split factors of the blocked tags."""

    tag: str
    x: int = 0
    y: int = 0

    def __post_init__(self):
        if self.tag not in _RANK:
            raise WrongLayout(f"unknown layout tag {self.tag!r}")
        if self.tag == "NCHWc" and self.x < 1:
            raise WrongLayout("NCHW[x]c needs x >= 1")
        if self.tag == "KCRSck" and min(self.x, self.y) < 1:
            raise WrongLayout("KCRS[x]c[y]k needs x >= 1 and y >= 1")

    @property
    def rank(self) -> int:
        return _RANK[self.tag]

    @property
    def is_blocked(self) -> bool:
        return self.tag in ("NCHWc", "KCRSck")

    def __str__(self) -> str:
        if self.tag == "NCHWc":
            return f"NCHW{self.x}c"
        if self.tag == "KCRSck":
            return f"KCRS{self.x}c{self.y}k"
        return self.tag

    @classmethod
    def parse(cls, text: str) -> "Layout":
        if text in ("NCHW", "NHWC", "KCRS", "VEC", "MAT"):
            return cls(text)
        m = re.fullmatch(r"NCHW(\d+)c", text)
        if m:
            return cls("NCHWc", x=int(m.group(1)))
        m = re.fullmatch(r"KCRS(\d+)c(\d+)k", text)
        if m:
            return cls("KCRSck", x=int(m.group(1)), y=int(m.group(2)))
        raise WrongLayout(f"cannot parse layout {text!r}")


NCHW = Layout("NCHW")
NHWC = Layout("NHWC")
KCRS = Layout("KCRS")


def nchwc(x: int) -> Layout:
    return Layout("NCHWc", x=x)


def kcrsck(x: int, y: int) -> Layout:
    return Layout("KCRSck", x=x, y=y)


def aligned_empty(shape, align: int = ALIGNMENT) -> np.ndarray:
    """Host f32 buffer whose base address is a multiple of ``align`` bytes."""
    count = int(np.prod(shape, dtype=np.int64))
    raw = np.empty(count * 4 + align, dtype=np.uint8)
    start = (-raw.ctypes.data) % align
    return raw[start:start + count * 4].view(np.float32).reshape(shape)


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


class Tensor:
    """Array plus layout.  ``data`` is a C-contiguous float32 numpy array
    (host) or a contiguous torch CUDA tensor (device, f32 or bf16)."""

    def __init__(self, data, layout: Layout = NCHW):
        if _is_torch(data):
            data = data.contiguous()
        else:
            data = np.ascontiguousarray(data, dtype=np.float32)
        if data.ndim != layout.rank:
            raise WrongLayout(
                f"rank {data.ndim} does not match layout {layout} (rank {layout.rank})")
        if layout.tag == "NCHWc" and data.shape[4] != layout.x:
            raise WrongLayout("innermost dim must equal the channel split x")
        if layout.tag == "KCRSck" and tuple(data.shape[4:]) != (layout.x, layout.y):
            raise WrongLayout("innermost dims must equal (x, y)")
        self.data = data
        self.layout = layout

    @property
    def shape(self):
        return tuple(self.data.shape)

    @property
    def on_device(self) -> bool:
        return _is_torch(self.data)

    def logical_channels(self) -> int:
        tag = self.layout.tag
        if tag == "NCHW":
            return self.shape[1]
        if tag == "NHWC":
            return self.shape[3]
        if tag == "NCHWc":
            return self.shape[1] * self.layout.x
        raise WrongLayout(f"not a feature-map layout: {self.layout}")

    def numpy(self) -> np.ndarray:
        if self.on_device:
            return self.data.float().cpu().numpy()
        return self.data

    def __repr__(self) -> str:
        where = "cuda" if self.on_device else "host"
        return f"Tensor(shape={self.shape}, layout={self.layout}, {where})"


# ---------------------------------------------------------------------------
# device execution of the transforms (K-LAYOUT / K-WPACK)

def _to_device(a):
    import torch
    if _is_torch(a):
        return a.contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _like_input(result, original):
    """Device results stay on device; host inputs get host results."""
    if _is_torch(original):
        return result
    out = aligned_empty(tuple(result.shape))
    out[...] = result.float().cpu().numpy()
    return out


def _feature_dims(a, layout: Layout):
    sh = tuple(a.shape)
    if layout.tag == "NCHW":
        return sh
    if layout.tag == "NHWC":
        return sh[0], sh[3], sh[1], sh[2]
    if layout.tag == "NCHWc":
        return sh[0], sh[1] * sh[4], sh[2], sh[3]
    raise WrongLayout(f"not a feature-map layout: {layout}")


def _device_feature_transform(a, src: Layout, dst: Layout, pad_channels: bool = False):
    import torch
    from . import device as D
    from . import _lib as L
    n, c, h, w = _feature_dims(a, src)
    if dst.tag == "NCHWc" and c % dst.x and not pad_channels:
        raise IndivisibleChannel(f"C={c} not divisible by x={dst.x}")
    if dst.tag == "NCHW":
        shape = (n, c, h, w)
    else:
        shape = (n, -(-c // dst.x), h, w, dst.x)
    src_t = _to_device(a)
    out = torch.empty(shape, dtype=src_t.dtype, device=src_t.device)
    flags = L.FLAG_PAD_CHANNELS if pad_channels else 0
    D.layout_transform(src_t, out, n, c, h, w, src, dst, flags)
    return _like_input(out, a)


def pack_nchw_array(a, x: int):
    """(n,c,h,w) -> (n,c/x,h,w,x); bit-exact (reference layout.py:131-137)."""
    if a.shape[1] % x:
        raise IndivisibleChannel(f"C={a.shape[1]} not divisible by x={x}")
    return _device_feature_transform(a, NCHW, nchwc(x))


def unpack_nchw_array(a):
    """inverse of pack_nchw_array (reference layout.py:140-144)."""
    return _device_feature_transform(a, nchwc(a.shape[4]), NCHW)


def retile_nchw_array(a, b: int):
    """NCHW[a]c -> NCHW[b]c without an NCHW round trip (layout.py:163-177)."""
    c = a.shape[1] * a.shape[4]
    if c % b:
        raise IndivisibleChannel(f"C={c} not divisible by b={b}")
    return _device_feature_transform(a, nchwc(a.shape[4]), nchwc(b))


def nhwc_to_nchw_array(a):
    """NHWC ingest (layout.py:180-183)."""
    return _device_feature_transform(a, NHWC, NCHW)


def _weights_device(a, x: int, y: int, pack: bool):
    import torch
    from . import device as D
    src = _to_device(a)
    if pack:
        k, c, r, s = src.shape
        if c % x or k % y:
            raise IndivisibleChannel(f"(K={k}, C={c}) not divisible by (y={y}, x={x})")
        out = torch.empty((k // y, c // x, r, s, x, y), dtype=src.dtype, device=src.device)
        D.pack_weights(src, out, x, y)
    else:
        ko, co, r, s, xx, yy = src.shape
        out = torch.empty((ko * yy, co * xx, r, s), dtype=src.dtype, device=src.device)
        D.unpack_weights(src, out)
    return _like_input(out, a)


def pack_kcrs_array(a, x: int, y: int):
    """(k,c,r,s) -> (k/y,c/x,r,s,x,y); bit-exact (layout.py:147-153)."""
    return _weights_device(a, x, y, True)


def unpack_kcrs_array(a):
    """inverse of pack_kcrs_array (layout.py:156-160)."""
    return _weights_device(a, a.shape[4], a.shape[5], False)


# ---------------------------------------------------------------------------
# Tensor-level API (layout.py:189-216)

def pack_data(t: Tensor, x: int) -> Tensor:
    if t.layout.tag != "NCHW":
        raise WrongLayout(f"pack_data expects NCHW, got {t.layout}")
    return Tensor(pack_nchw_array(t.data, x), nchwc(x))


def unpack_data(t: Tensor) -> Tensor:
    if t.layout.tag != "NCHWc":
        raise WrongLayout(f"unpack_data expects NCHW[x]c, got {t.layout}")
    return Tensor(unpack_nchw_array(t.data), NCHW)


def pack_weights(t: Tensor, x: int, y: int) -> Tensor:
    if t.layout.tag != "KCRS":
        raise WrongLayout(f"pack_weights expects KCRS, got {t.layout}")
    return Tensor(pack_kcrs_array(t.data, x, y), kcrsck(x, y))


def unpack_weights(t: Tensor) -> Tensor:
    if t.layout.tag != "KCRSck":
        raise WrongLayout(f"unpack_weights expects KCRS[x]c[y]k, got {t.layout}")
    return Tensor(unpack_kcrs_array(t.data), KCRS)


def retile_data(t: Tensor, b: int) -> Tensor:
    if t.layout.tag != "NCHWc":
        raise WrongLayout(f"retile_data expects NCHW[x]c, got {t.layout}")
    return Tensor(retile_nchw_array(t.data, b), nchwc(b))


def transform_array(a, src: Layout, dst: Layout):
    """pack / unpack / retile / ingest dispatch (layout.py:219-235); the
    identity returns its argument unchanged."""
    if src == dst:
        return a
    route = {
        ("NHWC", "NCHW"): lambda: nhwc_to_nchw_array(a),
        ("NCHW", "NCHWc"): lambda: pack_nchw_array(a, dst.x),
        ("NCHWc", "NCHW"): lambda: unpack_nchw_array(a),
        ("NCHWc", "NCHWc"): lambda: retile_nchw_array(a, dst.x),
        ("KCRS", "KCRSck"): lambda: pack_kcrs_array(a, dst.x, dst.y),
        ("KCRSck", "KCRS"): lambda: unpack_kcrs_array(a),
    }.get((src.tag, dst.tag))
    if route is None:
        raise WrongLayout(f"no transform from {src} to {dst}")
    return route()


# ---------------------------------------------------------------------------
# compile-time host permutations used by graph passes (weights are constants
# of the graph, exactly as in the reference passes.py:258-286); runtime
# tensors never take this path.

def host_pack_kcrs(w: np.ndarray, x: int, y: int) -> np.ndarray:
    k, c, r, s = w.shape
    if c % x or k % y:
        raise IndivisibleChannel(f"(K={k}, C={c}) not divisible by (y={y}, x={x})")
    blocks = w.reshape(k // y, y, c // x, x, r, s)
    return np.ascontiguousarray(np.moveaxis(blocks, (1, 3), (5, 4)), dtype=np.float32)


def host_unpack_kcrs(w: np.ndarray) -> np.ndarray:
    ko, co, r, s, x, y = w.shape
    blocks = np.moveaxis(w, (5, 4), (1, 3))
    return np.ascontiguousarray(blocks.reshape(ko * y, co * x, r, s), dtype=np.float32)
