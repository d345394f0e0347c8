"""ctypes binding of liblss.so (the C ABI declared in include/lss.h).

The library is built in-tree (``paper_2311_02382_b200/liblss.so``, see
``build.py``).  There is no fallback: if the library is missing or fails to
load, every entry point raises :class:`NativeError`.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import (DegenerateRowError, NativeError, NumericsError, PartitionError, ShapeError,
                     UnsupportedError)

LIB_PATH = Path(__file__).resolve().parent / "liblss.so"

LSS_BF16 = 0
LSS_F32 = 1

_STATUS = {
    1: ShapeError,
    2: PartitionError,
    3: DegenerateRowError,
    4: NumericsError,
    5: NativeError,
    6: UnsupportedError,
    7: ValueError,
}

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_long
_F = ctypes.c_float


class GemmEpilogue(ctypes.Structure):
    _fields_ = [
        ("out", _P * 3),
        ("ldo", _L * 3),
        ("seg_width", _I),
        ("out_dtype", _I),
        ("alpha", _F),
        ("bias", _P),
        ("residual", _P),
        ("ld_res", _L),
        ("act", _I),
        ("pre", _P),
        ("ld_pre", _L),
        ("aux", _P),
        ("ld_aux", _L),
        ("aux_dtype", _I),
    ]


class DropoutDesc(ctypes.Structure):
    """lss_dropout (include/lss.h)."""

    _fields_ = [("site_key", ctypes.c_ulonglong), ("thresh", ctypes.c_ulonglong), ("scale", _F), ("active", _I)]


class BwdSource(ctypes.Structure):
    """lss_bwd_source (include/lss.h)."""

    _fields_ = [
        ("q", _P), ("grad_o", _P), ("grad_q", _P), ("m_src", _I), ("row0", _I), ("rows", _I),
        ("pos0", _L), ("g_begin", _I), ("g_end", _I), ("lse2", _P), ("delta", _P), ("pitch", _I),
        ("ready", _P), ("ready_seq", ctypes.c_uint), ("grad_q_fixed", _P),
    ]


# name -> argtypes (all return int status, except noted)
SIGNATURES = {
    "lss_layernorm_fwd": [_P, _P, _P, _P, _I, _P, _P, _L, _I, _F, _P],
    "lss_layernorm_bwd": [_P, _P, _P, _P, _P, _P, _P, _P, _P, _F, _L, _I, _P],
    "lss_gemm": [_I, _P, _L, _I, _P, _L, _I, _I, _I, _I, ctypes.POINTER(GemmEpilogue), _P],
    "lss_stage_weights": [_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P],
    "lss_cat_cast_colsum": [_I, ctypes.POINTER(_P), ctypes.POINTER(_L), ctypes.POINTER(_I), _I, _P, _L,
                            _P, _F, _L, _P],
    "lss_attn_fwd": [_I, _P, _P, _P, _L, _P, _P, _I, _I, _I, _I, _I, _I, _L, _I, _P],
    "lss_attn_bwd": [_I, _P, _P, _P, _L, _P, _P, _P, _P, _P, _P, _P, _L, _I, _I, _I, _I, _I, _I, _L, _I,
                     _P],
    "lss_attn_fwd_ex": [_I, _P, _I, _L, _P, _P, _L, _P, _L, _P, _I, _I, _I, _I, _I, _I, _L, _I, _I, _I,
                        ctypes.POINTER(DropoutDesc), _P],
    "lss_attn_fwd_split": [_I, _P, _I, _L, _P, _P, _L, _P, _L, _P, _I, _I, _I, _I, _I, _I, _L, _I, _I, _I,
                           ctypes.POINTER(DropoutDesc), _I, _P, _L, _P, _L, _P, ctypes.c_uint, _I, _P],
    "lss_attn_merge": [_P, _P, _P, _P, _P, _P, _I, _I, _I, _L, _I, _P],
    "lss_attn_delta": [_I, _P, _P, _P, _I, _I, _I, _I, _I, _P],
    "lss_attn_bwd_ex": [_I, _P, _P, _L, ctypes.POINTER(BwdSource), _I, _P, _P, _L, _I, _I, _I, _I, _I, _I,
                        ctypes.POINTER(DropoutDesc), _P],
    "lss_add_f32": [_P, _P, _L, _P],
    "lss_timestamp": [_P, _P],
    "lss_sum_slots_mask": [_P, _P, _I, ctypes.c_uint, _L, _L, _P],
    "lss_cat_cast_colsum_ex": [_I, ctypes.POINTER(_P), ctypes.POINTER(_L), ctypes.POINTER(_I), ctypes.POINTER(_I),
                               ctypes.POINTER(ctypes.c_uint), ctypes.POINTER(_L), _I, _P, _L, _P, _F, _L, _P],
    "lss_stream_signal": [_P, ctypes.c_uint, _P],
    "lss_stream_wait": [_P, ctypes.c_uint, _P],
    "lss_attn_bwd_p2p": [_I, _P, _P, _L, ctypes.POINTER(BwdSource), _I, ctypes.POINTER(_P), _I, _L, _I, _I, _I,
                         _I, _I, _I, ctypes.POINTER(DropoutDesc), _P],
    "lss_dropout_rows": [_I, _P, _L, _P, _L, _P, _L, _L, _I, _I, _L, ctypes.c_ulonglong, ctypes.c_ulonglong, _F, _P],
    "lss_sum_slots": [_P, _P, _I, _L, _L, _P],
    "lss_sgd_update": [_P, _P, _L, _F, _P],
    "lss_embed_fwd": [_P, _P, _P, _P, _I, _I, _I, _P],
    "lss_embed_bwd": [_P, _P, _P, _P, _I, _I, _I, _F, _F, _P],
    "lss_cross_entropy": [_P, _L, _P, _L, _I, _F, _P, _P, _L, _P],
    "lss_adam_update": [_P, _P, _P, _P, _L, _F, _F, _F, _F, _I, _P],
    "lss_ipc_export": [_P, ctypes.c_char_p, ctypes.POINTER(_L)],
    "lss_ipc_import": [ctypes.c_char_p, _L, ctypes.POINTER(_P)],
    "lss_ipc_close": [_P, _L],
    "lss_copy_d2d": [_P, _P, _L, _P],
    "lss_runtime_config": [ctypes.c_ulonglong, _I],
    "lss_status": [ctypes.POINTER(ctypes.c_uint), _I],
    "lss_check_finite": [_P, _L, _I, _P],
    "lss_flag_release": [_P, _L, ctypes.c_uint],
    "lss_fixed_to_f32": [_P, _P, _L, _I, _P],
    "lss_stream_wait_bounded": [_P, _I, _I, ctypes.c_uint, _P],
    "lss_abort_waits": [_I],
    "lss_stream_wait_guarded": [_P, _I, _I, ctypes.c_uint, _P],
}
ACT_NONE, ACT_GELU, ACT_GELU_BWD = 0, 1, 2
EXTRA = {
    "lss_abi_version": ([], _I),
    "lss_last_error": ([], ctypes.c_char_p),
    "lss_rows_pad": ([_L], _L),
    "lss_peer_access": ([_I, _I], _I),
}
ABI_VERSION = 10

_lib = None


def load():
    """Load liblss.so once; raise NativeError if it is absent or incompatible."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("LSS_LIB", LIB_PATH))
    if not path.exists():
        raise NativeError(f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    try:
        lib = ctypes.CDLL(str(path))
    except OSError as exc:  # pragma: no cover - depends on the box
        raise NativeError(f"failed to load {path}: {exc}") from exc
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _I
    for name, (argtypes, res) in EXTRA.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = res
    if lib.lss_abi_version() != ABI_VERSION:
        raise NativeError(f"liblss.so ABI {lib.lss_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


# kernels each entry point launches (bf16 path; attn_bwd = delta + main kernel)
KERNELS_PER_CALL = {"lss_layernorm_fwd": 1, "lss_layernorm_bwd": 1, "lss_gemm": 1, "lss_stage_weights": 1,
                    "lss_cat_cast_colsum": 1, "lss_attn_fwd": 1, "lss_attn_bwd": 2, "lss_attn_fwd_ex": 1,
                    "lss_attn_merge": 1, "lss_attn_delta": 1, "lss_attn_bwd_ex": 1, "lss_add_f32": 1,
                    "lss_attn_bwd_p2p": 1, "lss_sum_slots": 1, "lss_sgd_update": 1, "lss_adam_update": 1,
                    "lss_embed_fwd": 1, "lss_embed_bwd": 1, "lss_cross_entropy": 1,
                    "lss_dropout_rows": 1, "lss_attn_fwd_split": 1, "lss_sum_slots_mask": 1, "lss_cat_cast_colsum_ex": 1,
                    "lss_check_finite": 1, "lss_fixed_to_f32": 1, "lss_stream_wait_bounded": 1, "lss_stream_wait_guarded": 1}
launch_count = 0


def call(name: str, *args):
    """Invoke an entry point and map a non-zero status onto the reference's exceptions."""
    global launch_count
    lib = load()
    rc = getattr(lib, name)(*args)
    launch_count += KERNELS_PER_CALL.get(name, 0)
    if name == "lss_attn_fwd_split" and args[21] > 1:
        launch_count += 1  # + the N-way merge
    if rc != 0:
        msg = lib.lss_last_error().decode(errors="replace")
        raise _STATUS.get(rc, NativeError)(f"{name}: {msg}")


def rows_pad(rows: int) -> int:
    return int(load().lss_rows_pad(rows))
