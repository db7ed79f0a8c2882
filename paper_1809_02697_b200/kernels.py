"""Convolution operators of the drop-in: workload / schedule / epilogue types
and the device conv entry points.

API mirrors the reference kernels.py (ConvWorkload :26-47, ConvSchedule
:50-71, Epilogue :74-87, UNROLL_LIMIT :90, vector_lane_width :93-114,
conv_reference :221-247, conv_blocked :250-303).  Both conv entry points run
on the GPU (libneob200):

* ``conv_reference`` -- the SIMT fp32 kernel with ic_bn = oc_bn = 1, i.e. the
  naive NCHW/KCRS convolution with the reference's c -> r -> s order and
  separately rounded multiply/add (bit-comparable to _naive_nchw :117-132);
* ``conv_blocked`` -- NCHW[x]c x KCRS[x]c[y]k with the fused epilogue.  mode
  "bf16" / "tf32" runs the tcgen05 implicit GEMM (csrc/conv_tc.cu); "fp32"
  runs the SIMT kernel.  Block sizes the tensor cores cannot take (x*sizeof
  not in {16,32,64,128} bytes) run the SIMT kernel on the GPU as well.

ConvSchedule keeps the reference's four fields (reg_n and unroll_ker are CPU
register-blocking knobs, carried for plan/DB compatibility and ignored by the
GPU kernels) and adds the tensor-core tile fields the GPU search tunes.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from .errors import ScheduleInvalid, ShapeMismatch, WrongLayout
from .graph import hw_pair
from .layout import NCHW, Tensor, kcrsck, nchwc

UNROLL_LIMIT = 25  # kept for API compatibility (CPU window-flattening limit)

TILE_FIELDS = ("tile_w", "tile_h", "tile_img", "tile_n", "slices_per_stage", "stages",
               "split_k", "cta_pair", "weight_stationary")


@dataclass(frozen=True)
class ConvWorkload:
    in_channel: int
    out_channel: int
    in_h: int
    in_w: int
    kernel_h: int
    kernel_w: int
    stride: object = 1   # int or (sh, sw)
    pad: object = 0      # int or (ph, pw)

    def __post_init__(self):
        for name in ("stride", "pad"):
            v = getattr(self, name)
            if isinstance(v, list):
                object.__setattr__(self, name, tuple(v))
        if self.out_h < 1 or self.out_w < 1:
            raise ShapeMismatch(f"workload {self} has empty output")

    @property
    def stride_hw(self) -> tuple[int, int]:
        return hw_pair(self.stride)

    @property
    def pad_hw(self) -> tuple[int, int]:
        return hw_pair(self.pad)

    @property
    def out_h(self) -> int:
        return (self.in_h + 2 * self.pad_hw[0] - self.kernel_h) // self.stride_hw[0] + 1

    @property
    def out_w(self) -> int:
        return (self.in_w + 2 * self.pad_hw[1] - self.kernel_w) // self.stride_hw[1] + 1

    def flops(self, batch: int = 1) -> int:
        """2 * N * K * C * R * S * OH * OW (one MAC = 2 FLOP)."""
        return (2 * batch * self.out_channel * self.in_channel * self.kernel_h * self.kernel_w
                * self.out_h * self.out_w)

    def key(self) -> list:
        """JSON-friendly identity (tuning.py:86-88 _workload_key order)."""
        enc = lambda v: list(v) if isinstance(v, tuple) else v
        return [self.in_channel, self.out_channel, self.in_h, self.in_w, self.kernel_h,
                self.kernel_w, enc(self.stride), enc(self.pad)]


@dataclass(frozen=True)
class ConvSchedule:
    ic_bn: int
    oc_bn: int
    reg_n: int
    unroll_ker: bool = False
    tile_w: int = 0
    tile_h: int = 0
    tile_img: int = 0
    tile_n: int = 0
    slices_per_stage: int = 0
    stages: int = 0
    split_k: int = 0
    cta_pair: int = 0
    weight_stationary: int = 0

    def check(self, wl: ConvWorkload) -> None:
        """Divisibility rules of the reference (kernels.py:56-63)."""
        if min(self.ic_bn, self.oc_bn, self.reg_n) < 1:
            raise ScheduleInvalid(f"non-positive factor in {self}")
        if wl.in_channel % self.ic_bn:
            raise ScheduleInvalid(f"ic_bn={self.ic_bn} does not divide C={wl.in_channel}")
        if wl.out_channel % self.oc_bn:
            raise ScheduleInvalid(f"oc_bn={self.oc_bn} does not divide K={wl.out_channel}")

    def tile(self) -> dict:
        return {f: getattr(self, f) for f in TILE_FIELDS}

    def with_tile(self, **tile) -> "ConvSchedule":
        d = self.as_dict()
        d.update({k: int(v) for k, v in tile.items() if k in TILE_FIELDS})
        return ConvSchedule.from_dict(d)

    def as_dict(self) -> dict:
        d = {"ic_bn": self.ic_bn, "oc_bn": self.oc_bn, "reg_n": self.reg_n,
             "unroll_ker": self.unroll_ker}
        d.update(self.tile())
        return d

    @classmethod
    def from_dict(cls, d: dict) -> "ConvSchedule":
        extra = {f: int(d.get(f, 0) or 0) for f in TILE_FIELDS}
        return cls(int(d["ic_bn"]), int(d["oc_bn"]), int(d["reg_n"]), bool(d["unroll_ker"]),
                   **extra)


@dataclass
class Epilogue:
    """Per-element post-processing in the order scale/shift -> bias ->
    residual_add -> relu (kernels.py:74-87)."""

    scale: object = None     # (K,) array or None
    shift: object = None
    bias: object = None
    relu: bool = False
    residual: object = None  # same shape/layout as the conv output

    def is_empty(self) -> bool:
        return (self.scale is None and self.shift is None and self.bias is None
                and not self.relu and self.residual is None)


def bytes_per_elem(mode: str) -> int:
    return {"bf16": 2, "fp8": 1}.get(mode, 4)


def vector_lane_width(mode: str = "bf16") -> int:
    """Channels per 128-byte tensor-core row: the GPU analogue of the CPU
    SIMD lane count the reference probes (kernels.py:93-114).  Overridable
    with NEOPLAN_LANE_WIDTH like the reference."""
    env = os.environ.get("NEOPLAN_LANE_WIDTH")
    if env:
        return int(env)
    return 128 // bytes_per_elem(mode)


def tc_legal_block(x: int, mode: str) -> bool:
    """Can the tensor-core conv consume NCHW[x]c input in ``mode``?"""
    return mode in ("bf16", "tf32", "fp8") and x * bytes_per_elem(mode) in (16, 32, 64, 128)


# ---------------------------------------------------------------------------
# device execution

def _mode_of(pool, mode) -> str:
    from .runtime import resolve_pool
    if mode is not None:
        return mode
    if pool is not None:
        return resolve_pool(pool).mode
    return os.environ.get("NEOB200_CONV_MODE", "fp32")


def _vec(v, dev):
    import torch
    if v is None:
        return None
    if isinstance(v, torch.Tensor):
        return v.to(dev, torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).to(dev)


def _dev(a, dev, dtype):
    import torch
    if isinstance(a, torch.Tensor):
        return a.to(dev).to(dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev).to(dtype)


def _run_device_conv(x_t, w_t, wl: ConvWorkload, ic_bn: int, oc_bn: int, epi, mode: str,
                     tile: dict | None, host_out: bool):
    """x_t: NCHW[ic_bn]c data, w_t: KCRS[ic_bn]c[oc_bn]k weights (host or device)."""
    import torch
    from . import _lib as L
    from . import device as D
    dev = torch.device("cuda", torch.cuda.current_device())
    use_tc = tc_legal_block(ic_bn, mode)
    act = torch.bfloat16 if (use_tc and mode == "bf16") else torch.float32
    xd = _dev(x_t, dev, act)
    n = xd.shape[0]
    if use_tc:
        wk = _dev(w_t, dev, torch.float32)
        if wk.dim() == 6:
            kcrs = torch.empty((wl.out_channel, wl.in_channel, wl.kernel_h, wl.kernel_w),
                               dtype=torch.float32, device=dev)
            D.unpack_weights(wk, kcrs)
        else:
            kcrs = wk
        lib_mode = L.MODE_BF16 if mode == "bf16" else L.MODE_TF32
        wd = D.pack_weights_umma(kcrs, ic_bn, lib_mode)
        x_in = xd if mode == "bf16" else _round_tf32_dev(xd)
    else:
        lib_mode = L.MODE_FP32
        wd = _dev(w_t, dev, torch.float32)
        x_in = xd
    out_dt = torch.bfloat16 if (use_tc and mode == "bf16") else torch.float32
    out = torch.empty((n, wl.out_channel // oc_bn, wl.out_h, wl.out_w, oc_bn), dtype=out_dt,
                      device=dev)
    e = epi or Epilogue()
    res = None
    if e.residual is not None:
        res_arr = e.residual.data if isinstance(e.residual, Tensor) else e.residual
        if tuple(res_arr.shape) != tuple(out.shape):
            raise ShapeMismatch("residual shape/layout mismatch")
        res = _dev(res_arr, dev, out_dt)
    scale, shift = e.scale, e.shift
    if scale is None and shift is not None:
        scale = np.ones(wl.out_channel, np.float32)
    if scale is not None and shift is None:
        shift = np.zeros(wl.out_channel, np.float32)
    p = D.conv_params(lib_mode, x_in, wd, out, n, wl.in_channel, wl.in_h, wl.in_w,
                      wl.out_channel, wl.kernel_h, wl.kernel_w, wl.stride_hw, wl.pad_hw, ic_bn,
                      oc_bn, _vec(scale, dev), _vec(shift, dev), _vec(e.bias, dev), res,
                      e.relu, tile=tile)
    D.conv2d(p)
    if host_out:
        from .layout import aligned_empty
        host = aligned_empty(tuple(out.shape))
        host[...] = out.float().cpu().numpy()
        return host
    return out


def _round_tf32_dev(t):
    """RN-to-tf32 copy of an f32 device tensor."""
    from . import device as D
    return D.round_tf32(t)


def conv_reference(ifmap: Tensor, weights: Tensor, wl: ConvWorkload,
                   epi: Epilogue | None = None) -> Tensor:
    """Naive NCHW x KCRS convolution on the GPU (fp32, reference order)."""
    if ifmap.layout.tag != "NCHW" or weights.layout.tag != "KCRS":
        raise ShapeMismatch("conv_reference expects NCHW data and KCRS weights")
    n, c, h, w = ifmap.shape
    if (c, h, w) != (wl.in_channel, wl.in_h, wl.in_w) or tuple(weights.shape) != (
            wl.out_channel, wl.in_channel, wl.kernel_h, wl.kernel_w):
        raise ShapeMismatch(f"tensors do not match workload {wl}")
    e = epi
    if e is not None and e.residual is not None:
        # NCHW residual == NCHW[1]c residual with a trailing unit axis
        r = e.residual.data if isinstance(e.residual, Tensor) else e.residual
        if tuple(r.shape) != (n, wl.out_channel, wl.out_h, wl.out_w):
            raise ShapeMismatch("residual shape mismatch")
        e = Epilogue(e.scale, e.shift, e.bias, e.relu, r.reshape(tuple(r.shape) + (1,)))
    x5 = ifmap.data.reshape(tuple(ifmap.shape) + (1,))
    w6 = weights.data.reshape(tuple(weights.shape) + (1, 1))
    out = _run_device_conv(x5, w6, wl, 1, 1, e, "fp32", None, not ifmap.on_device)
    return Tensor(out.reshape(out.shape[:4]), NCHW)


def conv_blocked(ifmap: Tensor, weights: Tensor, wl: ConvWorkload, sch: ConvSchedule,
                 epi: Epilogue | None = None, pool=None, mode: str | None = None) -> Tensor:
    """Blocked direct convolution with the fused epilogue, on the GPU.

    ``mode``: "fp32" (SIMT, equals the reference within 1e-5), "tf32" or
    "bf16" (tcgen05); default from ``pool`` (a DevicePool) or the
    NEOB200_CONV_MODE environment variable ("fp32")."""
    sch.check(wl)
    if ifmap.layout != nchwc(sch.ic_bn):
        raise ScheduleInvalid(f"ifmap layout {ifmap.layout} vs ic_bn={sch.ic_bn}")
    if weights.layout != kcrsck(sch.ic_bn, sch.oc_bn):
        raise ScheduleInvalid(f"weight layout {weights.layout} vs {sch}")
    m = _mode_of(pool, mode)
    tile = sch.tile() if any(sch.tile().values()) else None
    out = _run_device_conv(ifmap.data, weights.data, wl, sch.ic_bn, sch.oc_bn, epi, m, tile,
                           not ifmap.on_device)
    return Tensor(out, nchwc(sch.oc_bn))


__all__ = ["ConvWorkload", "ConvSchedule", "Epilogue", "UNROLL_LIMIT", "vector_lane_width",
           "conv_reference", "conv_blocked", "tc_legal_block", "TILE_FIELDS"]
