"""ctypes binding of libdfb200.so (include/df_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (make in
``csrc/``).  There is no fallback: if the shared object is missing or a call
fails, the error surfaces as the reference's exception type (or KernelError).
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DF_LIB_PATH") or os.path.join(_HERE, "libdfb200.so")  # env: dev A/B builds only

DF_OK = 0
DF_E_SHAPE = 1
DF_E_PACKING = 2
DF_E_ORDER = 3
DF_E_CONFIG = 4
DF_E_ASSIGN = 5
DF_E_CUDA = 6
DF_E_ARG = 7

DF_MAX_HEADS = 64
DF_MAX_ARENAS = 4
DF_TMAP_BYTES = 128
DF_MAPS_PER_ARENA = 3
DF_MAX_APPEND_SEGS = 128
DF_MAX_PEERS = 7
DF_ATTN_PROBE = 1
DF_ATTN_PAIR = 2
DF_ATTN_SINGLE_CTA = 4

_CODE_TO_EXC = {
    DF_E_SHAPE: errors.ShapeError,
    DF_E_PACKING: errors.PackingError,
    DF_E_ORDER: errors.OrderingError,
    DF_E_CONFIG: errors.ConfigError,
    DF_E_ASSIGN: errors.AssignmentError,
    DF_E_CUDA: errors.KernelError,
    DF_E_ARG: ValueError,
}


class HeadDesc(ctypes.Structure):
    _fields_ = [
        ("base_row", ctypes.c_int64),
        ("n_tok", ctypes.c_int32),
        ("q_head", ctypes.c_int32),
        ("o_head", ctypes.c_int32),
        ("arena", ctypes.c_int32),
    ]


class AttnArgs(ctypes.Structure):
    _fields_ = [
        ("q", ctypes.c_void_p),
        ("q_rows", ctypes.c_int64),
        ("out", ctypes.c_void_p),
        ("out_ld", ctypes.c_int64),
        ("hw", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("d_out", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("num_heads", ctypes.c_int32),
        ("num_arenas", ctypes.c_int32),
        ("heads", ctypes.POINTER(HeadDesc)),
        ("kv_maps", ctypes.c_void_p),
        ("flags", ctypes.c_uint32),
        ("max_slots", ctypes.c_int32),
        ("region_of_slot", ctypes.c_void_p),
        ("row_sampled", ctypes.c_void_p),
        ("probe_rows", ctypes.c_void_p),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_int64),
        ("peer_out", ctypes.POINTER(ctypes.c_void_p)),
        ("n_peers", ctypes.c_int32),
    ]


class CopySeg(ctypes.Structure):
    _fields_ = [
        ("src", ctypes.c_void_p),
        ("dst", ctypes.c_void_p),
        ("rows", ctypes.c_int64),
        ("src_ld", ctypes.c_int64),
        ("dst_ld", ctypes.c_int64),
        ("row_bytes", ctypes.c_int64),
    ]


class QkvArgs(ctypes.Structure):
    _fields_ = [
        ("x", ctypes.c_void_p),
        ("w_qkv", ctypes.c_void_p),
        ("hw", ctypes.c_int32),
        ("num_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("in_dim", ctypes.c_int32),
        ("q_out", ctypes.c_void_p),
        ("k_dst", ctypes.c_void_p * DF_MAX_HEADS),
        ("v_dst", ctypes.c_void_p * DF_MAX_HEADS),
        ("kv_ld", ctypes.c_int64),
    ]


class OprojArgs(ctypes.Structure):
    _fields_ = [
        ("o", ctypes.c_void_p),
        ("w_o", ctypes.c_void_p),
        ("hw", ctypes.c_int32),
        ("num_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("out_dim", ctypes.c_int32),
        ("x", ctypes.c_void_p),
        ("x_bf16", ctypes.c_void_p),
    ]


# Every symbol include/df_b200.h declares, with its ctypes signature.
_SIGNATURES = {
    "df_attn_fwd": (ctypes.c_int, [ctypes.POINTER(AttnArgs), ctypes.c_void_p]),
    "df_attn_workspace_bytes": (ctypes.c_int, [ctypes.POINTER(AttnArgs), ctypes.POINTER(ctypes.c_int64)]),
    "df_kv_arena_maps": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p],
    ),
    "df_kv_append": (ctypes.c_int, [ctypes.POINTER(CopySeg), ctypes.c_int32, ctypes.c_void_p]),
    "df_kv_append_overlapped": (ctypes.c_int, [ctypes.POINTER(CopySeg), ctypes.c_int32, ctypes.c_void_p]),
    "df_kv_pack": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p],
    ),
    "df_kv_pack_plan": (
        ctypes.c_int,
        [ctypes.POINTER(CopySeg), ctypes.c_int32, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)],
    ),
    "df_scores_finalize": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p],
    ),
    "df_greedy_classify": (
        ctypes.c_int,
        [
            ctypes.POINTER(ctypes.c_double),
            ctypes.c_int64,
            ctypes.c_int64,
            ctypes.POINTER(ctypes.c_int8),
            ctypes.POINTER(ctypes.c_double),
        ],
    ),
    "df_qkv_project": (ctypes.c_int, [ctypes.POINTER(QkvArgs), ctypes.c_void_p]),
    "df_out_project": (ctypes.c_int, [ctypes.POINTER(OprojArgs), ctypes.c_void_p]),
    "df_last_error": (ctypes.c_char_p, []),
    "df_version": (ctypes.c_int, []),
    "df_device_check": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int32)]),
}

_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load libdfb200.so once; raise KernelError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise errors.KernelError(
                    f"{LIB_PATH} not built; run __graft_entry__.build() (make -C csrc)"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def last_error() -> str:
    msg = load().df_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def raise_for(rc: int, what: str) -> None:
    if rc == DF_OK:
        return
    exc = _CODE_TO_EXC.get(rc, errors.KernelError)
    raise exc(f"{what}: {last_error()} (status {rc})")


def call(name: str, *args) -> None:
    rc = getattr(load(), name)(*args)
    raise_for(rc, name)


_device_checked: set[int] = set()


def require_device(device_index: int) -> int:
    """Fail loudly unless a sm_100 device is current; returns its SM count."""
    import torch

    if not torch.cuda.is_available():
        raise errors.KernelError("no CUDA device: the B200 path has no CPU fallback")
    n = ctypes.c_int32(0)
    with torch.cuda.device(device_index):
        call("df_device_check", ctypes.byref(n))
    _device_checked.add(device_index)
    return int(n.value)
