"""ctypes binding of libneob200.so (include/neob200.h).

The library is built in-tree by ``__graft_entry__.build()`` /
``python -m paper_1809_02697_b200.build``.  There is no fallback: if the
shared object is missing or fails to load, every device operation raises
NativeLibraryMissing.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors as E

LIB_NAME = "libneob200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

# status codes (neob200.h neo_status)
NEO_OK = 0
_STATUS_EXC = {
    1: E.ScheduleInvalid,
    2: E.ShapeMismatch,
    3: E.WrongLayout,
    4: E.IndivisibleChannel,
    5: E.DeviceError,
    6: E.DeviceError,
    7: E.InputMismatch,
}

# enums
F32, BF16, FP8 = 0, 1, 2
NCHW_TAG, NHWC_TAG, NCHWC_TAG = 0, 1, 2
MODE_FP32, MODE_TF32, MODE_BF16, MODE_FP8 = 0, 1, 2, 3
POOL_MAX, POOL_AVG = 0, 1
ELT_RELU, ELT_ADD, ELT_ADD_RELU, ELT_SCALE_SHIFT, ELT_SCALE_SHIFT_RELU = range(5)
FLAG_ROUND_TF32 = 0x1
FLAG_PAD_CHANNELS = 0x2
FLAG_STATIC_WEIGHTS = 0x4
FLAG_HALO_STRIPS = 0x8

_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_c_vp = ctypes.c_void_p


class ConvParams(ctypes.Structure):
    """Mirror of ``neo_conv_params`` (ABI v3: leading struct_size, filled in
    by the constructor and checked by the library; e4m3 storage scales at
    the end)."""

    def __init__(self, *args, **kw):
        super().__init__(*args, **kw)
        self.struct_size = ctypes.sizeof(ConvParams)

    _fields_ = [
        ("struct_size", _c_int),
        ("mode", _c_int),
        ("x", _c_vp), ("w", _c_vp), ("out", _c_vp),
        ("scale", _c_vp), ("shift", _c_vp), ("bias", _c_vp),
        ("residual", _c_vp),
        ("relu", _c_int),
        ("n", _c_i64), ("c", _c_i64), ("h", _c_i64), ("w_in", _c_i64),
        ("k", _c_i64), ("r", _c_i64), ("s", _c_i64),
        ("stride_h", _c_int), ("stride_w", _c_int), ("pad_h", _c_int), ("pad_w", _c_int),
        ("ic_bn", _c_int), ("oc_bn", _c_int),
        ("x_cb_offset", _c_int), ("x_cb_total", _c_int),
        ("out_cb_offset", _c_int), ("out_cb_total", _c_int),
        ("res_cb_offset", _c_int), ("res_cb_total", _c_int),
        ("out_dtype", _c_int),
        ("flags", _c_int),
        ("tile_w", _c_int), ("tile_h", _c_int), ("tile_img", _c_int), ("tile_n", _c_int),
        ("slices_per_stage", _c_int), ("stages", _c_int),
        ("split_k", _c_int), ("workspace", _c_vp), ("workspace_bytes", _c_i64),
        ("cta_pair", _c_int),
        ("pro_scale", _c_vp), ("pro_shift", _c_vp), ("pro_relu", _c_int),
        ("weight_stationary", _c_int),
        ("out2", _c_vp), ("k_split", _c_i64), ("relu2", _c_int),
        ("out2_cb_offset", _c_int), ("out2_cb_total", _c_int),
        ("res_scale", ctypes.c_float), ("out_scale", ctypes.c_float),
        ("out2_scale", ctypes.c_float),
    ]


# every exported symbol with its ctypes signature (restype, argtypes)
SIGNATURES = {
    "neo_last_error": (ctypes.c_char_p, []),
    "neo_abi_version": (_c_int, []),
    "neo_device_info": (_c_int, [_c_int, ctypes.c_char_p, _c_int]),
    "neo_layout_transform": (_c_int, [_c_int, _c_int, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64,
                                      _c_i64, _c_int, _c_int, _c_int, _c_int, _c_int, _c_vp]),
    "neo_pack_weights": (_c_int, [_c_int, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_i64,
                                  _c_int, _c_int, _c_vp]),
    "neo_unpack_weights": (_c_int, [_c_int, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_i64,
                                    _c_int, _c_int, _c_vp]),
    "neo_pack_weights_umma": (_c_int, [_c_vp, _c_vp, _c_int, _c_i64, _c_i64, _c_i64, _c_i64,
                                       _c_int, _c_i64, _c_int, _c_vp]),
    "neo_pack_weights_umma_fp8": (_c_int, [_c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_i64,
                                           _c_int, _c_i64, _c_int, _c_vp]),
    "neo_absmax": (_c_int, [_c_int, _c_vp, _c_i64, _c_vp, _c_vp]),
    "neo_dequant_fp8": (_c_int, [_c_vp, _c_vp, _c_int, ctypes.c_float, _c_i64, _c_i64, _c_i64,
                                 _c_i64, _c_int, _c_i64, _c_i64, _c_vp]),
    "neo_stem_fold": (_c_int, [_c_vp, _c_vp, _c_int, _c_i64, _c_i64, _c_i64, _c_i64, _c_int,
                               _c_int, _c_int, _c_i64, _c_int, _c_int, _c_vp]),
    "neo_stem_pack_weights": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_vp]),
    "neo_stem_weight_bytes": (_c_i64, []),
    "neo_stem_conv_pool": (_c_int, [_c_vp, _c_int, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_int, _c_i64,
                                    _c_i64, _c_i64, _c_i64, _c_int, _c_int, _c_int, _c_vp]),
    "neo_stem_conv_pool_q": (_c_int, [_c_vp, _c_int, _c_vp, _c_vp, _c_int, ctypes.c_float, _c_vp,
                                      _c_vp, _c_vp, _c_int, _c_i64, _c_i64, _c_i64, _c_i64, _c_int,
                                      _c_int, _c_int, _c_vp]),
    "neo_classifier_head_q": (_c_int, [_c_vp, _c_int, ctypes.c_float, _c_vp, _c_vp, _c_vp, _c_vp,
                                       _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_int, _c_i64, _c_int,
                                       _c_vp]),
    "neo_classifier_head": (_c_int, [_c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_i64,
                                     _c_i64, _c_i64, _c_int, _c_i64, _c_int, _c_vp]),
    "neo_conv_umma_slices": (_c_i64, [_c_int, _c_i64, _c_i64, _c_i64, _c_int, _c_int]),
    "neo_conv2d_nchwc_fused": (_c_int, [ctypes.POINTER(ConvParams), _c_vp]),
    "neo_conv_params_size": (_c_int, []),
    "neo_conv_junction": (_c_int, [_c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp,
                                   _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_int, _c_int,
                                   _c_vp]),
    "neo_conv_default_tiles": (_c_int, [ctypes.POINTER(ConvParams)]),
    "neo_conv_workspace_bytes": (_c_int, [ctypes.POINTER(ConvParams), ctypes.POINTER(_c_i64)]),
    "neo_pool2d": (_c_int, [_c_int, _c_int, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_i64,
                            _c_int, _c_int, _c_int, _c_int, _c_int, _c_vp]),
    "neo_pool2d_window": (_c_int, [_c_int, _c_int, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_i64,
                                   _c_int, _c_int, _c_int, _c_int, _c_i64, _c_i64, _c_i64, _c_i64,
                                   _c_int, _c_vp]),
    "neo_pool2d_q": (_c_int, [_c_int, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_int,
                              _c_int, _c_int, _c_int, _c_i64, _c_i64, _c_i64, _c_i64,
                              ctypes.c_float, ctypes.c_float, _c_vp]),
    "neo_eltwise_q": (_c_int, [_c_int, _c_vp, _c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64,
                               _c_int, _c_i64, _c_i64, _c_i64, _c_i64, ctypes.c_float,
                               ctypes.c_float, _c_vp]),
    "neo_eltwise_window": (_c_int, [_c_int, _c_int, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_i64,
                                    _c_i64, _c_i64, _c_int, _c_i64, _c_i64, _c_i64, _c_i64, _c_int,
                                    _c_vp]),
    "neo_eltwise": (_c_int, [_c_int, _c_int, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_i64,
                             _c_i64, _c_i64, _c_int, _c_int, _c_vp]),
    "neo_concat_copy": (_c_int, [_c_int, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_vp]),
    "neo_dense": (_c_int, [_c_int, _c_vp, _c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp]),
    "neo_softmax": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_vp]),
    "neo_capture_begin": (_c_int, [_c_vp]),
    "neo_capture_end": (_c_int, [_c_vp, ctypes.POINTER(_c_vp)]),
    "neo_graph_launch": (_c_int, [_c_vp, _c_vp]),
    "neo_graph_destroy": (_c_int, [_c_vp]),
}

_lock = threading.Lock()
_lib = None
_load_error = None


def load(path: str | None = None):
    """Load (once) and return the configured CDLL; raises NativeLibraryMissing."""
    global _lib, _load_error
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or os.environ.get("NEOB200_LIB", LIB_PATH)
        try:
            lib = ctypes.CDLL(p)
        except OSError as exc:
            _load_error = str(exc)
            raise E.NativeLibraryMissing(
                f"cannot load {p}: {exc}; build it with "
                f"`python -c 'import __graft_entry__ as g; g.build()'`") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def available() -> bool:
    try:
        load()
        return True
    except E.NativeLibraryMissing:
        return False


def check(status: int, what: str = "") -> None:
    if status == NEO_OK:
        return
    msg = load().neo_last_error().decode(errors="replace")
    exc = _STATUS_EXC.get(status, E.DeviceError)
    raise exc(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def device_info(device: int = 0) -> dict:
    buf = ctypes.create_string_buffer(512)
    check(load().neo_device_info(device, buf, 512), "neo_device_info")
    name, sms, cc, mem = buf.value.decode().split("|")
    return {"name": name, "sm_count": int(sms), "cc": cc, "hbm_bytes": int(mem)}
