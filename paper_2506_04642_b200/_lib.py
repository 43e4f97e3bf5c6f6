"""ctypes binding of libtadakv_b200.so (the C ABI in include/tadakv_b200.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, every compute entry point raises :class:`BackendUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, DataError, FormatError, ShapeError, StateError, TadaError

LIB_NAME = "libtadakv_b200.so"
LIB_PATH = os.environ.get("TADA_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

TADA_F32 = 0
TADA_BF16 = 1

TADA_ERR_CONFIG = 2
_ERRORS = {1: ShapeError, 2: ConfigError, 3: DataError, 4: FormatError, 5: StateError}


class BackendUnavailable(TadaError, RuntimeError):
    """libtadakv_b200.so (or a CUDA device) is unavailable; there is no CPU fallback."""


class PageLayout(C.Structure):
    """Mirror of ``tada_page_layout`` (include/tadakv_b200.h)."""

    _fields_ = [
        ("page_tokens", C.c_int32),
        ("heads", C.c_int32),
        ("head_dim", C.c_int32),
        ("bits", C.c_int32),
        ("group_bytes", C.c_int32),
        ("reserved", C.c_int32),
        ("page_bytes", C.c_int64),
        ("off_mean", C.c_int64 * 2),
        ("off_codes", C.c_int64 * 2),
        ("off_meta", C.c_int64 * 2),
    ]


P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
F = C.c_float

# name -> (restype, argtypes); every symbol declared in include/tadakv_b200.h
SIGNATURES = {
    "tada_abi_version": (I32, []),
    "tada_launch_count": (I64, []),
    "tada_last_error": (C.c_char_p, []),
    "tada_bytes_per_group": (I64, [I32, I32]),
    "tada_page_layout_init": (I32, [I32, I32, I32, I32, C.POINTER(PageLayout)]),
    "tada_quantize_groups": (I32, [P, I32, I64, I32, I32, P, P, P, P, P]),
    "tada_dequantize_groups": (I32, [P, P, P, I64, I32, I32, P, I64, P, P]),
    "tada_pack_codes": (I32, [P, I64, I32, I32, P, P]),
    "tada_unpack_codes": (I32, [P, I64, I32, I32, P, I64, P, P]),
    "tada_mean_center": (I32, [P, I32, I64, I32, I32, P, P, P, P]),
    "tada_quant_append": (I32, [C.POINTER(PageLayout), P, P, P, I32, I32, I64, I64, P, I32, P, I64, P, P]),
    "tada_apply_rope": (I32, [P, I32, I64, I32, I32, P, P, I32, P, P, P]),
    "tada_gather_compressed": (I32, [C.POINTER(PageLayout), P, P, I64, I32, P, P, P, P, P]),
    "tada_scatter_compressed": (I32, [C.POINTER(PageLayout), P, P, I64, I32, P, P, P, P, P]),
    "tada_decode_attn_workspace_bytes": (I64, [I32, I32, I32, I32]),
    "tada_decode_attn": (I32, [C.POINTER(PageLayout), P, P, I32, I32, I32, P, I32, P, P, P, P, I64, F, I32, P, P,
                               I32, I32, P, P]),
    "tada_decode_attn_lse": (I32, [C.POINTER(PageLayout), P, P, I32, I32, I32, P, I32, P, P, P, P, I64, F, I32, P,
                                   P, I32, I32, P, P, P]),
    "tada_combine_lse": (I32, [P, P, I32, I64, I32, P, I32, P, P]),
    "tada_quant_append_plan": (I32, [C.POINTER(PageLayout), P, P, P, I32, I32, I64, I64, P, I32, P, P, I32, I32, P,
                                     I32, P, I64, P, I32, P, P, P]),
    "tada_append_commit": (I32, [P, P, I64, I32, I32, P, P, I32, I32, I64, I32, P, I32, P, P, P, I64, P, I32, P, P]),
    "tada_decode_step": (I32, [C.POINTER(PageLayout), P, P, I32, I32, I32, P, I32, P, P, P, P, I64, I32, P, P, I32,
                               I32, P, F, I32, P, P, I32, I32, P, P, P]),
    "tada_decode_attn_suggest_splits": (I32, [I32, I64, I32]),
    "tada_decode_attn_plan_splits": (I32, [C.POINTER(PageLayout), I32, I32, I64]),
    "tada_decode_attn_plan_splits_mode": (I32, [C.POINTER(PageLayout), I32, I32, I64, I32]),
}

_lib = None
_load_error = None


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes library; raise BackendUnavailable if absent."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        _load_error = f"{path} not built (run `make` or __graft_entry__.build())"
        raise BackendUnavailable(_load_error)
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.tada_abi_version() != 1:
        raise BackendUnavailable("libtadakv_b200 ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = (_lib.tada_last_error() or b"").decode(errors="replace")
        raise _ERRORS.get(rc, TadaError)(msg or f"libtadakv_b200 error {rc}")


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point and raise the mapped reference error type."""
    check(getattr(load(), name)(*args))


def page_layout(page_tokens: int, heads: int, head_dim: int, bits: int) -> PageLayout:
    lay = PageLayout()
    call("tada_page_layout_init", page_tokens, heads, head_dim, bits, C.byref(lay))
    return lay


def launch_count() -> int:
    """Kernels launched by libtadakv_b200.so so far in this process."""
    return int(load().tada_launch_count())
