"""Device-side operator calls: thin typed wrappers that pass torch CUDA
tensors (allocation only) to libneob200 through ctypes.  Every function is
stream-ordered on the current torch stream and raises the reference
exception types on failure.  No function here has a CPU path."""

from __future__ import annotations

import ctypes

import torch

from . import _lib as L
from . import errors as E

_DT = {torch.float32: L.F32, torch.bfloat16: L.BF16, torch.float8_e4m3fn: L.FP8}


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise E.InputMismatch(f"unsupported dtype {t.dtype}") from None


def torch_dtype(code: int) -> torch.dtype:
    return {L.BF16: torch.bfloat16, L.FP8: torch.float8_e4m3fn}.get(code, torch.float32)


def _ptr(t) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise E.InputMismatch("device operators take CUDA tensors")
    if not t.is_contiguous():
        raise E.InputMismatch("device operators take contiguous tensors")
    return t.data_ptr()


def stream_handle(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _tag(layout) -> tuple[int, int]:
    """(tag, x) of a Layout or layout string."""
    s = str(layout)
    if s == "NCHW":
        return L.NCHW_TAG, 1
    if s == "NHWC":
        return L.NHWC_TAG, 1
    if s.startswith("NCHW") and s.endswith("c"):
        return L.NCHWC_TAG, int(s[4:-1])
    raise E.WrongLayout(f"not a feature-map layout: {s}")


def layout_transform(src: torch.Tensor, dst: torch.Tensor, n: int, c: int, h: int, w: int,
                     src_layout, dst_layout, flags: int = 0, stream=None) -> None:
    st, sx = _tag(src_layout)
    dt, dx = _tag(dst_layout)
    L.call("neo_layout_transform", dtype_code(src), dtype_code(dst), _ptr(src), _ptr(dst),
           n, c, h, w, st, sx, dt, dx, flags, stream_handle(stream))


def pack_weights(src: torch.Tensor, dst: torch.Tensor, x: int, y: int, stream=None) -> None:
    k, c, r, s = src.shape
    L.call("neo_pack_weights", dtype_code(src), _ptr(src), _ptr(dst), k, c, r, s, x, y,
           stream_handle(stream))


def unpack_weights(src: torch.Tensor, dst: torch.Tensor, stream=None) -> None:
    ko, co, r, s, x, y = src.shape
    L.call("neo_unpack_weights", dtype_code(src), _ptr(src), _ptr(dst), ko * y, co * x, r, s,
           x, y, stream_handle(stream))


def umma_slices(mode: int, c: int, r: int, s: int, x: int) -> int:
    return int(L.load().neo_conv_umma_slices(mode, c, r, s, x, 1))


def pack_weights_umma(w_kcrs: torch.Tensor, x: int, mode: int, pad_channels: bool = False,
                      stream=None) -> torch.Tensor:
    """Device-private slice-major weight image for the tensor-core conv."""
    if w_kcrs.dtype != torch.float32:
        raise E.InputMismatch("umma weight packing takes f32 KCRS")
    k, c, r, s = w_kcrs.shape
    slices = umma_slices(mode, c, r, s, x)
    dt = L.BF16 if mode == L.MODE_BF16 else L.F32
    out = torch.empty(slices * k * x, dtype=torch_dtype(dt), device=w_kcrs.device)
    flags = (L.FLAG_ROUND_TF32 if mode == L.MODE_TF32 else 0) | \
        (L.FLAG_PAD_CHANNELS if pad_channels else 0)
    L.call("neo_pack_weights_umma", _ptr(w_kcrs), _ptr(out), dt, k, c, r, s, x, slices, flags,
           stream_handle(stream))
    return out


def pack_weights_umma_fp8(w_kcrs: torch.Tensor, wscale: torch.Tensor, x: int,
                          pad_channels: bool = False, stream=None) -> torch.Tensor:
    """e4m3 tensor-core weight image: RN_e4m3(w[k] / wscale[k]) in the
    slice-major layout (neo_pack_weights_umma_fp8)."""
    if w_kcrs.dtype != torch.float32 or wscale.dtype != torch.float32:
        raise E.InputMismatch("fp8 weight packing takes f32 KCRS and f32 scales")
    k, c, r, s = w_kcrs.shape
    slices = umma_slices(L.MODE_FP8, c, r, s, x)
    out = torch.empty(slices * k * x, dtype=torch.float8_e4m3fn, device=w_kcrs.device)
    flags = L.FLAG_PAD_CHANNELS if pad_channels else 0
    L.call("neo_pack_weights_umma_fp8", _ptr(w_kcrs), _ptr(out), _ptr(wscale), k, c, r, s, x,
           slices, flags, stream_handle(stream))
    return out


def dequant_fp8(src: torch.Tensor, dst: torch.Tensor, scale: float, n, c, h, w, x,
                cb=(0, 0), stream=None) -> None:
    """e4m3 NCHW[x]c -> NCHW f32 / bf16 times ``scale`` (neo_dequant_fp8)."""
    L.call("neo_dequant_fp8", _ptr(src), _ptr(dst), dtype_code(dst), float(scale), n, c, h, w, x,
           cb[0], cb[1], stream_handle(stream))


def absmax(t: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """max |t| into a one-element device f32 tensor (neo_absmax)."""
    if out is None:
        out = torch.empty(1, dtype=torch.float32, device=t.device)
    L.call("neo_absmax", dtype_code(t), _ptr(t), t.numel(), _ptr(out), stream_handle(stream))
    return out


def conv_params(mode, x, w, out, n, c, h, w_in, k, r, s, stride=(1, 1), pad=(0, 0), ic_bn=1,
                oc_bn=1, scale=None, shift=None, bias=None, residual=None, relu=False,
                x_cb=(0, 0), out_cb=(0, 0), res_cb=(0, 0), flags=0, tile=None,
                prologue=None, second=None, qscales=None) -> L.ConvParams:
    """``second`` = (out2, k_split, relu2, out2_cb): channels [k_split, k)
    are written to out2 (two sibling convs as one launch).  ``qscales`` =
    (res_scale, out_scale, out2_scale) of e4m3 residual / outputs."""
    p = L.ConvParams()
    p.mode = mode
    p.x, p.w, p.out = _ptr(x), _ptr(w), _ptr(out)
    p.scale, p.shift, p.bias, p.residual = _ptr(scale), _ptr(shift), _ptr(bias), _ptr(residual)
    p.relu = int(bool(relu))
    p.n, p.c, p.h, p.w_in, p.k, p.r, p.s = n, c, h, w_in, k, r, s
    p.stride_h, p.stride_w = stride
    p.pad_h, p.pad_w = pad
    p.ic_bn, p.oc_bn = ic_bn, oc_bn
    p.x_cb_offset, p.x_cb_total = x_cb
    p.out_cb_offset, p.out_cb_total = out_cb
    p.res_cb_offset, p.res_cb_total = res_cb
    p.out_dtype = dtype_code(out)
    p.flags = flags
    if prologue is not None:        # (scale, shift, relu): BN-ReLU on the input
        p.pro_scale, p.pro_shift = _ptr(prologue[0]), _ptr(prologue[1])
        p.pro_relu = int(bool(prologue[2]))
    if tile:
        for key in ("tile_w", "tile_h", "tile_img", "tile_n", "slices_per_stage", "stages",
                    "split_k", "cta_pair", "weight_stationary"):
            setattr(p, key, int(tile.get(key, 0) or 0))
    if second is not None:
        out2, k_split, relu2, out2_cb = second
        p.out2, p.k_split, p.relu2 = _ptr(out2), int(k_split), int(bool(relu2))
        p.out2_cb_offset, p.out2_cb_total = out2_cb
    if qscales is not None:
        p.res_scale, p.out_scale, p.out2_scale = (float(v or 0.0) for v in qscales)
    return p


def conv_junction(x, w1, b1, residual, y1, w2, b2, y2, n, c1, h, w, n1, n2, relu1=True,
                  relu2=True, stream=None) -> None:
    """y1 = relu1(x W1 + b1 + residual); y2 = relu2(y1 W2 + b2) in one launch
    (bf16 NCHW[64]c; w1 / w2 are pack_weights_umma images with x = 64)."""
    L.call("neo_conv_junction", _ptr(x), _ptr(w1), _ptr(b1), _ptr(residual), _ptr(y1), _ptr(w2),
           _ptr(b2), _ptr(y2), n, c1, h, w, n1, n2, int(bool(relu1)), int(bool(relu2)),
           stream_handle(stream))


def conv_workspace_bytes(p: L.ConvParams) -> int:
    """Split-K workspace the launch of ``p`` needs (0 = no split)."""
    out = ctypes.c_int64(0)
    L.call("neo_conv_workspace_bytes", ctypes.byref(p), ctypes.byref(out))
    return int(out.value)


def set_workspace(p: L.ConvParams, ws) -> None:
    p.workspace = _ptr(ws) if ws is not None else None
    p.workspace_bytes = ws.numel() * ws.element_size() if ws is not None else 0


def conv2d(p: L.ConvParams, stream=None) -> None:
    L.call("neo_conv2d_nchwc_fused", ctypes.byref(p), stream_handle(stream))


def default_tiles(p: L.ConvParams) -> dict:
    q = L.ConvParams.from_buffer_copy(p)
    L.check(L.load().neo_conv_default_tiles(ctypes.byref(q)), "neo_conv_default_tiles")
    return {k: getattr(q, k) for k in ("tile_w", "tile_h", "tile_img", "tile_n",
                                        "slices_per_stage", "stages", "split_k", "cta_pair",
                                        "weight_stationary")}


def pool2d(inp, out, n, cb, h, w, x, win, stride, pad, mode: str, flags=0, stream=None):
    L.call("neo_pool2d", dtype_code(inp), L.POOL_MAX if mode == "max" else L.POOL_AVG,
           _ptr(inp), _ptr(out), n, cb, h, w, x, win, stride, pad, flags, stream_handle(stream))


def pool2d_window(inp, out, n, cb, h, w, x, win, stride, pad, mode: str, in_win, out_win,
                  flags=0, stream=None):
    """Pooling between channel-block windows ((offset, total) pairs)."""
    L.call("neo_pool2d_window", dtype_code(inp), L.POOL_MAX if mode == "max" else L.POOL_AVG,
           _ptr(inp), _ptr(out), n, cb, h, w, x, win, stride, pad, in_win[0], in_win[1],
           out_win[0], out_win[1], flags, stream_handle(stream))


def pool2d_q(inp, out, n, cb, h, w, x, win, stride, pad, mode: str, in_win, out_win,
             in_scale: float, out_scale: float, stream=None):
    """e4m3 pooling with requantization (neo_pool2d_q)."""
    L.call("neo_pool2d_q", L.POOL_MAX if mode == "max" else L.POOL_AVG, _ptr(inp), _ptr(out), n,
           cb, h, w, x, win, stride, pad, in_win[0], in_win[1], out_win[0], out_win[1],
           float(in_scale), float(out_scale), stream_handle(stream))


def eltwise_q(op: int, a, out, n, cb, hw, x, a_win, out_win, a_scale: float, out_scale: float,
              scale=None, shift=None, stream=None):
    """e4m3 relu / scale-shift(-relu) with requantization (neo_eltwise_q)."""
    L.call("neo_eltwise_q", op, _ptr(a), _ptr(out), _ptr(scale), _ptr(shift), n, cb, hw, x,
           a_win[0], a_win[1], out_win[0], out_win[1], float(a_scale), float(out_scale),
           stream_handle(stream))


def eltwise_window(op: int, a, out, n, cb, hw, x, a_win, out_win, scale=None, shift=None,
                   flags=0, stream=None):
    L.call("neo_eltwise_window", dtype_code(a), op, _ptr(a), None, _ptr(out), _ptr(scale),
           _ptr(shift), n, cb, hw, x, a_win[0], a_win[1], out_win[0], out_win[1], flags,
           stream_handle(stream))


def eltwise(op: int, a, b, out, n, cb, hw, x, scale=None, shift=None, flags=0, stream=None):
    L.call("neo_eltwise", dtype_code(a), op, _ptr(a), _ptr(b), _ptr(out), _ptr(scale),
           _ptr(shift), n, cb, hw, x, flags, stream_handle(stream))


def concat_copy(src, dst, outer, chunk, dst_row, dst_off, stream=None):
    L.call("neo_concat_copy", dtype_code(src), _ptr(src), _ptr(dst), outer, chunk, dst_row,
           dst_off, stream_handle(stream))


def dense(a, w, bias, out, n, in_f, units, stream=None):
    L.call("neo_dense", dtype_code(a), _ptr(a), _ptr(w), _ptr(bias), _ptr(out), n, in_f, units,
           stream_handle(stream))


def softmax(inp, out, rows, cols, stream=None):
    L.call("neo_softmax", _ptr(inp), _ptr(out), rows, cols, stream_handle(stream))


class CapturedGraph:
    """A whole-forward CUDA graph captured from libneob200 launches."""

    def __init__(self, handle: int):
        self.handle = handle

    def launch(self, stream=None) -> None:
        L.call("neo_graph_launch", self.handle, stream_handle(stream))

    def __del__(self):
        try:
            if self.handle:
                L.load().neo_graph_destroy(self.handle)
        except Exception:
            pass


def capture(fn, stream=None) -> CapturedGraph:
    """Run ``fn`` under stream capture and return the instantiated graph.

    The garbage collector is paused for the capture: a collection inside it
    could free an unreachable program's pinned host buffers, and torch's
    pinned-memory allocator then queries CUDA events -- an operation a
    global-mode capture forbids, which would invalidate the graph."""
    import gc
    s = stream or torch.cuda.current_stream()
    gc_was = gc.isenabled()
    gc.disable()
    try:
        L.call("neo_capture_begin", stream_handle(s))
        try:
            fn()
        except BaseException:
            h = ctypes.c_void_p()
            L.load().neo_capture_end(stream_handle(s), ctypes.byref(h))
            if h.value:
                L.load().neo_graph_destroy(h)
            raise
        h = ctypes.c_void_p()
        L.call("neo_capture_end", stream_handle(s), ctypes.byref(h))
    finally:
        if gc_was:
            gc.enable()
    return CapturedGraph(h.value)


def round_tf32(t: torch.Tensor) -> torch.Tensor:
    """RN (ties away) rounding of an f32 device tensor to tf32 precision,
    as a same-layout transform with the rounding flag."""
    if t.dtype != torch.float32:
        raise E.InputMismatch("round_tf32 takes f32")
    out = torch.empty_like(t)
    L.call("neo_layout_transform", L.F32, L.F32, _ptr(t), _ptr(out), 1, t.numel(), 1, 1,
           L.NCHW_TAG, 1, L.NCHW_TAG, 1, L.FLAG_ROUND_TF32, stream_handle())
    return out


def stem_fold(src: torch.Tensor, dst: torch.Tensor, n, c, h, w, s, stride_w, pad_w, ow, xf,
              flags=0, stream=None) -> None:
    """NCHW f32 -> horizontally folded NCHW[xf]c (see neo_stem_fold)."""
    L.call("neo_stem_fold", _ptr(src), _ptr(dst), dtype_code(dst), n, c, h, w, s, stride_w,
           pad_w, ow, xf, flags, stream_handle(stream))


def pack_stem_weights(w_kcrs: torch.Tensor, stream=None) -> torch.Tensor:
    """KCRS f32 (64, C<=4, 7, 7) device weights -> the fused stem's bf16
    tensor-core image (neo_stem_pack_weights)."""
    w = w_kcrs.contiguous().float()
    k, c, r, s = w.shape
    img = torch.empty(L.load().neo_stem_weight_bytes() // 2, dtype=torch.bfloat16,
                      device=w.device)
    L.call("neo_stem_pack_weights", _ptr(w), _ptr(img), k, c, r, s, stream_handle(stream))
    return img


def stem_conv_pool(x: torch.Tensor, wimg: torch.Tensor, out: torch.Tensor, n, c, h, w, y,
                   scale=None, shift=None, bias=None, relu=True, out_cb=(0, 0),
                   stream=None, out_scale: float = 1.0) -> None:
    """Fused stem: maxpool3x3/2(relu(conv7x7/2(x) * scale + shift + bias))
    from NCHW f32 / bf16 straight into bf16 NCHW[y]c (neo_stem_conv_pool),
    or into e4m3 bytes of value / out_scale when ``out`` is float8_e4m3fn
    (neo_stem_conv_pool_q)."""
    if x.dtype not in (torch.float32, torch.bfloat16) or \
            out.dtype not in (torch.bfloat16, torch.float8_e4m3fn):
        raise E.InputMismatch("stem_conv_pool takes f32 or bf16 input and writes bf16 or e4m3")
    opt = lambda t: _ptr(t) if t is not None else None
    L.call("neo_stem_conv_pool_q", _ptr(x), dtype_code(x), _ptr(wimg), _ptr(out), dtype_code(out),
           float(out_scale), opt(scale), opt(shift), opt(bias), int(bool(relu)), n, c, h, w, y,
           out_cb[0], out_cb[1], stream_handle(stream))


class HeadScratch:
    """Device scratch of one fused classifier head (pooled features, logits,
    barrier counters)."""

    def __init__(self, n: int, c: int, units: int, device):
        self.pooled = torch.empty(n * c, dtype=torch.bfloat16, device=device)
        self.logits = torch.empty(2 * n * units, dtype=torch.float32, device=device)
        self.bar = torch.zeros(4, dtype=torch.int32, device=device)


def classifier_head(x: torch.Tensor, w_bf16: torch.Tensor, bias, out: torch.Tensor, n, c, hw, y,
                    units, softmax: bool, scratch: HeadScratch, stream=None,
                    x_scale: float = 1.0) -> None:
    """Global avg pool -> dense (+bias) -> optional softmax in one launch
    (neo_classifier_head; an e4m3 ``x`` is read with its scale ``x_scale``)."""
    if x.dtype not in (torch.bfloat16, torch.float8_e4m3fn) or w_bf16.dtype != torch.bfloat16 \
            or out.dtype != torch.float32:
        raise E.InputMismatch("classifier_head takes bf16 / e4m3 features, bf16 weights and "
                              "writes f32")
    L.call("neo_classifier_head_q", _ptr(x), dtype_code(x), float(x_scale), _ptr(w_bf16),
           _ptr(bias) if bias is not None else None, _ptr(scratch.pooled), _ptr(scratch.logits),
           _ptr(out), _ptr(scratch.bar), n, c, hw, y, units, int(bool(softmax)),
           stream_handle(stream))
