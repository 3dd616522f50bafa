"""ctypes binding to libssd200.so (include/ssd200.h).

The library is built in-tree (``__graft_entry__.build()`` or ``make -C
paper_2603_09555_b200/csrc``).  There is no fallback: if the shared object is
missing or a call fails, this module raises.
"""

from __future__ import annotations

import contextlib
import contextvars
import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SSD200_LIBRARY: another build of the same library (A/B of compile-time variants)
LIB_PATH = os.environ.get("SSD200_LIBRARY") or os.path.join(_HERE, "libssd200.so")

F32, F64, BF16 = 0, 1, 2
DTYPE_CODE = {"f32": F32, "f64": F64, "bf16": BF16}

EINVAL, ELAUNCH, EUNSUPPORTED, EWORKSPACE = -1, -2, -3, -4

c_void_p = ctypes.c_void_p
c_int = ctypes.c_int
c_int64 = ctypes.c_int64
c_size_t = ctypes.c_size_t
c_double = ctypes.c_double


class Tuning(ctypes.Structure):
    """ssd200_tuning_t: implementation choices passed per call (NULL = defaults)."""

    _fields_ = [(n, c_int) for n in (
        "size", "prefill_pdl", "gemm_pair", "pair_min_tiles", "scan_variant",
        "chunkscan_multicast", "out_waves", "dec_pdl", "dec_swap", "dec_small_ring",
        "dec_small_max", "dec_split_in", "dec_split_out", "stream_stages", "stream_cps",
        "stream_cw", "out_interleave", "gemm_group_m", "gemm_stream", "stream_chunk", "stream_reg_state")]


class Dims(ctypes.Structure):
    _fields_ = [
        ("dtype", c_int),
        ("d_model", c_int),
        ("d_inner", c_int),
        ("n_heads", c_int),
        ("head_dim", c_int),
        ("d_state", c_int),
        ("n_groups", c_int),
        ("conv_kernel", c_int),
        ("chunk_size", c_int),
        ("norm_eps", c_double),
        ("dt_min", c_double),
        ("dt_max", c_double),
        ("tuning", ctypes.POINTER(Tuning)),
    ]


class Layer(ctypes.Structure):
    _fields_ = [
        (n, c_void_p)
        for n in ("W_in", "conv_w", "conv_b", "dt_bias", "a", "D", "norm_w", "W_out", "pre_norm_w")
    ]


# (name, restype, argtypes) — exactly the symbols declared in include/ssd200.h
SIGNATURES = [
    ("ssd200_abi_version", c_int, []),
    ("ssd200_last_error", ctypes.c_char_p, []),
    ("ssd200_chunk_scan_workspace", c_size_t, [c_int] * 7),
    (
        "ssd200_chunk_scan",
        c_int,
        [c_int] + [c_void_p] * 9 + [c_int] * 7 + [c_void_p, c_size_t, c_void_p],
    ),
    ("ssd200_tuning_defaults", None, [ctypes.POINTER(Tuning)]),
    ("ssd200_embed", c_int, [ctypes.POINTER(Dims), c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("ssd200_prefill_layer_workspace", c_size_t, [ctypes.POINTER(Dims), c_int, c_int]),
    (
        "ssd200_prefill_layer",
        c_int,
        [ctypes.POINTER(Dims), ctypes.POINTER(Layer)] + [c_void_p] * 4 + [c_int, c_int, c_void_p, c_size_t, c_void_p],
    ),
    (
        "ssd200_prefill_layer_partial",
        c_int,
        [ctypes.POINTER(Dims), ctypes.POINTER(Layer), c_void_p, c_void_p, ctypes.c_long, c_void_p,
         c_void_p, c_int, c_int, c_void_p, c_size_t, c_void_p],
    ),
    (
        "ssd200_decode_layer_partial",
        c_int,
        [ctypes.POINTER(Dims), ctypes.POINTER(Layer), c_void_p, c_void_p, ctypes.c_long, c_void_p,
         c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_size_t, c_void_p],
    ),
    (
        "ssd200_resid_norm_finish",
        c_int,
        [c_int, c_int, c_double, c_void_p, c_void_p, c_void_p, ctypes.c_long, ctypes.c_long, c_void_p],
    ),
    ("ssd200_decode_layer_workspace", c_size_t, [ctypes.POINTER(Dims), c_int]),
    (
        "ssd200_decode_layer",
        c_int,
        [ctypes.POINTER(Dims), ctypes.POINTER(Layer)] + [c_void_p] * 6 + [c_int, c_void_p, c_size_t, c_void_p],
    ),
    ("ssd200_decode_layers_workspace", c_size_t, [ctypes.POINTER(Dims), c_int]),
    (
        "ssd200_decode_layers",
        c_int,
        [ctypes.POINTER(Dims), ctypes.POINTER(Layer), c_int] + [c_void_p] * 6 + [c_int, c_void_p, c_size_t, c_void_p],
    ),
    ("ssd200_head_workspace", c_size_t, [ctypes.POINTER(Dims), c_int, c_int]),
    (
        "ssd200_head",
        c_int,
        [ctypes.POINTER(Dims), c_int, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_size_t, c_void_p],
    ),
    ("ssd200_gemm_bf16", c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p]),
    ("ssd200_launch_count", ctypes.c_uint64, []),
    ("ssd200_set_phase_events", c_int, [c_void_p, c_int]),
]

_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load libssd200.so once; raise (never fall back) if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                    " or `make -C paper_2603_09555_b200/csrc` (there is no CPU fallback)"
                )
            handle = ctypes.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().ssd200_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = f"{what}: {last_error()}"
    if rc == EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"{msg} (status {rc})")


def ptr(t) -> int | None:
    """Device pointer of a tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda(*tensors) -> None:
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise ValueError("ssd200 kernels take CUDA tensors")


# ------------------------------------------------------------------ tuning
# Implementation choices travel with each call inside ssd200_dims_t (the
# library keeps no option state).  ``tuning(**fields)`` scopes overrides to a
# with-block (tests and A/B measurements); outside one, calls pass NULL and
# the library uses its measured defaults.
_TUNING: contextvars.ContextVar = contextvars.ContextVar("ssd200_tuning", default=None)


def default_tuning() -> Tuning:
    t = Tuning()
    lib().ssd200_tuning_defaults(ctypes.byref(t))
    return t


@contextlib.contextmanager
def tuning(**fields):
    base = _TUNING.get()
    t = Tuning()
    src = base if base is not None else default_tuning()
    ctypes.memmove(ctypes.addressof(t), ctypes.addressof(src), ctypes.sizeof(Tuning))
    for k, v in fields.items():
        if k not in dict(Tuning._fields_) or k == "size":
            raise ValueError(f"unknown tuning field {k!r}")
        setattr(t, k, int(v))
    tok = _TUNING.set(t)
    try:
        yield t
    finally:
        _TUNING.reset(tok)


def current_tuning():
    """The Tuning in scope (or None: library defaults)."""
    return _TUNING.get()
