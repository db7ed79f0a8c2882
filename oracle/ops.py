"""Per-operator CPU restatements (numpy).  TEST INFRASTRUCTURE ONLY -- see
oracle/__init__.py.  Reference paths are relative to
/root/reference/pkg/src/neoplan unless noted."""

from __future__ import annotations

import numpy as np


def rel_err(a, b) -> float:
    """max|a-b| / max(1, max|b|)  (reference tests/test_kernels.py:31-32)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float(np.abs(a - b).max() / max(1.0, float(np.abs(b).max())))


# ---------------------------------------------------------------------------
# layouts: bit-exact index permutations (layout.py:131-183)

def pack_nchw(a: np.ndarray, x: int) -> np.ndarray:
    """(n,c,h,w) -> (n,c//x,h,w,c%x)   layout.py:131-137."""
    n, c, h, w = a.shape
    if c % x:
        raise ValueError(f"C={c} not divisible by x={x}")
    return np.ascontiguousarray(a.reshape(n, c // x, x, h, w).transpose(0, 1, 3, 4, 2))


def unpack_nchw(a: np.ndarray) -> np.ndarray:
    """inverse of pack_nchw   layout.py:140-144."""
    n, cb, h, w, x = a.shape
    return np.ascontiguousarray(a.transpose(0, 1, 4, 2, 3).reshape(n, cb * x, h, w))


def pack_kcrs(w: np.ndarray, x: int, y: int) -> np.ndarray:
    """(k,c,r,s) -> (k//y,c//x,r,s,c%x,k%y)   layout.py:147-153."""
    k, c, r, s = w.shape
    if c % x or k % y:
        raise ValueError("indivisible channel")
    return np.ascontiguousarray(
        w.reshape(k // y, y, c // x, x, r, s).transpose(0, 2, 4, 5, 3, 1))


def unpack_kcrs(w: np.ndarray) -> np.ndarray:
    """inverse of pack_kcrs   layout.py:156-160."""
    ko, co, r, s, x, y = w.shape
    return np.ascontiguousarray(w.transpose(0, 5, 1, 4, 2, 3).reshape(ko * y, co * x, r, s))


def retile_nchw(a: np.ndarray, b: int) -> np.ndarray:
    """NCHW[a]c -> NCHW[b]c == pack(unpack(a), b)   layout.py:163-177."""
    return pack_nchw(unpack_nchw(a), b)


def nhwc_to_nchw(a: np.ndarray) -> np.ndarray:
    """layout.py:180-183."""
    return np.ascontiguousarray(a.transpose(0, 3, 1, 2))


def transform(a: np.ndarray, src: str, dst: str) -> np.ndarray:
    """transform_array dispatch (layout.py:219-235) on layout strings such as
    'NCHW', 'NHWC', 'NCHW16c', 'KCRS', 'KCRS4c8k'."""
    import re
    if src == dst:
        return a
    ms = re.fullmatch(r"NCHW(\d+)c", src)
    md = re.fullmatch(r"NCHW(\d+)c", dst)
    if src == "NHWC" and dst == "NCHW":
        return nhwc_to_nchw(a)
    if src == "NCHW" and md:
        return pack_nchw(a, int(md.group(1)))
    if ms and dst == "NCHW":
        return unpack_nchw(a)
    if ms and md:
        return retile_nchw(a, int(md.group(1)))
    mk = re.fullmatch(r"KCRS(\d+)c(\d+)k", dst)
    if src == "KCRS" and mk:
        return pack_kcrs(a, int(mk.group(1)), int(mk.group(2)))
    if re.fullmatch(r"KCRS(\d+)c(\d+)k", src) and dst == "KCRS":
        return unpack_kcrs(a)
    raise ValueError(f"no transform from {src} to {dst}")


# ---------------------------------------------------------------------------
# convolution (kernels.py:221-247 conv_reference; oracle form of
# reference tests/test_kernels.py:11-28 im2col_conv, generalised to (ph, pw)
# and (sh, sw) for the Inception 1x7 / 7x1 layers the reference cannot express)

def _pair(v):
    return (v, v) if isinstance(v, (int, np.integer)) else (int(v[0]), int(v[1]))


def conv2d(x: np.ndarray, w: np.ndarray, stride=1, pad=0, scale=None,
           shift=None, bias=None, residual=None, relu=False) -> np.ndarray:
    """NCHW x KCRS -> NCHW f32; accumulation in float64 (im2col + BLAS), then
    the epilogue in reference order scale/shift -> bias -> residual -> relu
    (kernels.py:234-246), each step rounded to f32 like the numpy reference."""
    sh, sw = _pair(stride)
    ph, pw = _pair(pad)
    n, c, h, wd = x.shape
    k, c2, r, s = w.shape
    assert c2 == c, (c2, c)
    oh = (h + 2 * ph - r) // sh + 1
    ow = (wd + 2 * pw - s) // sw + 1
    xp = np.pad(x.astype(np.float64), ((0, 0), (0, 0), (ph, ph), (pw, pw)))
    cols = np.empty((n, oh * ow, c, r, s), dtype=np.float64)
    for ri in range(r):
        for si in range(s):
            patch = xp[:, :, ri:ri + (oh - 1) * sh + 1:sh, si:si + (ow - 1) * sw + 1:sw]
            cols[:, :, :, ri, si] = patch.reshape(n, c, oh * ow).transpose(0, 2, 1)
    wm = w.astype(np.float64).reshape(k, c * r * s)
    out = np.matmul(cols.reshape(n, oh * ow, c * r * s), wm.T)  # (n, ohw, k)
    out = out.transpose(0, 2, 1).reshape(n, k, oh, ow).astype(np.float32)
    if scale is not None or shift is not None:
        sc = np.ones(k, np.float32) if scale is None else np.asarray(scale, np.float32)
        sf = np.zeros(k, np.float32) if shift is None else np.asarray(shift, np.float32)
        out = out * sc.reshape(1, k, 1, 1)
        out = out + sf.reshape(1, k, 1, 1)
    if bias is not None:
        out = out + np.asarray(bias, np.float32).reshape(1, k, 1, 1)
    if residual is not None:
        out = out + residual.astype(np.float32)
    if relu:
        out = np.maximum(out, np.float32(0.0))
    return np.ascontiguousarray(out, dtype=np.float32)


# ---------------------------------------------------------------------------
# memory-bound ops (executor.py:96-203)

def pool2d(a: np.ndarray, win: int, stride: int, pad: int, mode: str) -> np.ndarray:
    """_pool2d executor.py:103-128 on NCHW or NCHW[x]c: max pads with -inf,
    avg pads with 0 and divides by win*win (count_include_pad)."""
    h, w = a.shape[2], a.shape[3]
    oh = (h + 2 * pad - win) // stride + 1
    ow = (w + 2 * pad - win) // stride + 1
    if pad:
        shape = list(a.shape)
        shape[2] += 2 * pad
        shape[3] += 2 * pad
        p = np.full(shape, -np.inf if mode == "max" else 0.0, dtype=np.float32)
        p[:, :, pad:pad + h, pad:pad + w] = a
        a = p
    out = None
    for r in range(win):
        for s in range(win):
            sl = a[:, :, r:r + oh * stride:stride, s:s + ow * stride:stride]
            if out is None:
                out = sl.astype(np.float32, copy=True)
            elif mode == "max":
                out = np.maximum(out, sl)
            else:
                out = out + sl
    if mode == "avg":
        out = out / np.float32(win * win)
    return np.ascontiguousarray(out, dtype=np.float32)


def channel_broadcast(vec: np.ndarray, a: np.ndarray) -> np.ndarray:
    """executor.py:96-100."""
    if a.ndim == 5:
        x = a.shape[4]
        return vec.reshape(a.shape[1], x).reshape(1, a.shape[1], 1, 1, x)
    return vec.reshape(1, -1, 1, 1)


def batchnorm(a, scale, shift):
    """standalone BN as a*scale + shift (executor.py:171-181)."""
    return (a * channel_broadcast(np.asarray(scale, np.float32), a)
            + channel_broadcast(np.asarray(shift, np.float32), a)).astype(np.float32)


def bn_scale_shift(gamma, beta, mean, var, eps=1e-5):
    """float64 folding constants (passes.py:92-96 / executor.py:176-178)."""
    g, b, m, v = (np.asarray(t, np.float64) for t in (gamma, beta, mean, var))
    scale = g / np.sqrt(v + eps)
    shift = b - m * scale
    return scale, shift


def relu(a):
    return np.maximum(a, np.float32(0.0))


def add(a, b):
    return (a + b).astype(np.float32)


def concat(arrays, axis=1):
    return np.concatenate(arrays, axis=axis)


def flatten(a):
    return np.ascontiguousarray(a).reshape(a.shape[0], -1)


def dense(a, w, b=None):
    """a @ w.T (+ b)  executor.py:197-203 (float64 accumulate)."""
    out = (a.astype(np.float64) @ w.astype(np.float64).T)
    if b is not None:
        out = out + np.asarray(b, np.float64)
    return out.astype(np.float32)


def softmax(a):
    """executor.py:167-170."""
    a = a.astype(np.float32)
    e = np.exp(a - a.max(axis=-1, keepdims=True))
    return (e / e.sum(axis=-1, keepdims=True)).astype(np.float32)


# ---------------------------------------------------------------------------
# arithmetic model of the single-pass tensor-core modes (TEST INFRASTRUCTURE:
# used to show what the bf16 / tf32 number formats alone cost on a graph, so
# a device error can be judged against the error of its own arithmetic).

def round_rn(a: np.ndarray, kind: str | None) -> np.ndarray:
    """Round f32 values to bf16 (8-bit significand) or tf32 (11-bit) with
    round-to-nearest-even, kept in f32 storage; ``None`` is the identity."""
    if kind is None:
        return a
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    drop = 16 if kind == "bf16" else 13
    u = (u + ((1 << (drop - 1)) - 1) + ((u >> drop) & 1)) & (0xFFFFFFFF ^ ((1 << drop) - 1))
    return u.astype(np.uint32).view(np.float32).reshape(np.shape(a))


def conv2d_rounded(kind, x, w, stride=1, pad=0, scale=None, shift=None, bias=None,
                   residual=None, relu=False):
    """conv2d with the operand and storage roundings of a single-pass
    ``kind`` tensor-core conv: activations and (folded) weights rounded RN
    to ``kind``, f32 accumulation and epilogue, output rounded RN."""
    out = conv2d(round_rn(x, kind), round_rn(w, kind), stride, pad, scale, shift, bias,
                 residual, relu)
    return round_rn(out, kind)


# ---------------------------------------------------------------------------
# e4m3 (OCP FP8 "e4m3fn": 4 exponent bits, bias 7, 3 mantissa bits, no
# infinities, max 448) -- TEST INFRASTRUCTURE for the FP8 conv mode, which the
# reference does not have (quantized inference is PAPER.md:433's future work).

E4M3_MAX = 448.0


def round_e4m3(a) -> np.ndarray:
    """Round to the nearest e4m3 value, ties to even, saturating to +-448
    (PTX cvt.rn.satfinite.e4m3x2.f32); f32 in, f32 out."""
    x = np.asarray(a, np.float64)
    mag = np.abs(x)
    _, ex = np.frexp(mag)                          # mag = m * 2^ex, m in [0.5, 1)
    e = np.maximum(ex - 1, -6)                     # normal exponent, subnormals below 2^-6
    q = np.ldexp(1.0, e - 3)                       # spacing: 3 mantissa bits
    r = np.minimum(np.rint(mag / q) * q, E4M3_MAX)  # rint: round half to even
    return (np.sign(x) * r).astype(np.float32)


def e4m3_to_bytes(v) -> np.ndarray:
    """Encode e4m3-representable values as their bytes (uint8)."""
    x = np.asarray(v, np.float64)
    sign = (np.signbit(x)).astype(np.uint8) << 7
    mag = np.abs(x)
    _, ex = np.frexp(mag)
    e = ex - 1
    normal = (mag >= 2.0 ** -6)
    exp_field = np.where(normal, e + 7, 0)
    man = np.where(normal, np.rint((mag / np.ldexp(1.0, np.where(normal, e, 0)) - 1.0) * 8),
                   np.rint(mag / 2.0 ** -9))
    out = sign | (exp_field.astype(np.uint8) << 3) | man.astype(np.uint8)
    return np.where(mag == 0, sign, out).astype(np.uint8)


def e4m3_from_bytes(b) -> np.ndarray:
    """Decode e4m3 bytes (uint8) to f32 (0x7f / 0xff, the NaN codes, -> nan)."""
    u = np.asarray(b, np.uint8).astype(np.int64)
    sign = np.where(u & 0x80, -1.0, 1.0)
    ef = (u >> 3) & 0xF
    man = u & 0x7
    val = np.where(ef == 0, man * 2.0 ** -9, (1.0 + man / 8.0) * np.ldexp(1.0, ef - 7))
    val = np.where((u & 0x7F) == 0x7F, np.nan, val)
    return (sign * val).astype(np.float32)


def fp8_weight_scales(w: np.ndarray) -> np.ndarray:
    """Per-output-channel e4m3 weight scales absmax_k / 448 in f32 (1 for an
    all-zero channel) -- the quantization rule the FP8 mode documents."""
    w = np.asarray(w, np.float32)
    ws = (np.abs(w.reshape(w.shape[0], -1)).max(axis=1).astype(np.float32)
          / np.float32(E4M3_MAX)).astype(np.float32)
    ws[ws == 0] = np.float32(1.0)
    return ws


def conv2d_fp8(x_q, w, x_scale, out_scale=None, stride=1, pad=0, scale=None, shift=None,
               bias=None, residual=None, relu=False):
    """Arithmetic model of an FP8 (e4m3) tensor-core conv: ``x_q`` holds the
    input's e4m3 values (stored value = x_q * x_scale), weights quantized per
    output channel (W_q = RN_e4m3(W / ws[k])), exact products accumulated
    (f64 here, f32 on the device), the epilogue scale x_scale * ws[k] (* BN
    scale) folded into the reference's scale slot, then bias -> residual ->
    relu (kernels.py:185-197) and one RN_e4m3 of value / out_scale (None:
    unquantized f32 output).  Returns the stored e4m3 values (or f32)."""
    ws = fp8_weight_scales(w)
    wq = round_e4m3(np.asarray(w, np.float32) / ws.reshape(-1, 1, 1, 1))
    sc = np.float32(x_scale) * ws
    if scale is not None:
        sc = (sc * np.asarray(scale, np.float32)).astype(np.float32)
    out = conv2d(x_q, wq, stride, pad, sc, shift, bias, residual, relu)
    if out_scale is None:
        return out
    return round_e4m3(out / np.float32(out_scale))
