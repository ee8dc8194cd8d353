"""ctypes binding of libneob200.so (include/neo_tbe.h).

This is the only module that touches the C ABI.  It loads the in-tree
library and fails loudly when it is missing: there is no CPU fallback for
any operator of this package.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libneob200.so"

# status codes / enums (neo_tbe.h)
NEO_OK, NEO_E_INDEX_RANGE, NEO_E_LAYOUT, NEO_E_ARG, NEO_E_CUDA = 0, 1, 2, 3, 4
NEO_F32, NEO_F16, NEO_F64, NEO_BF16 = 0, 1, 2, 3
NEO_I32, NEO_I64 = 0, 1
NEO_POOL_SUM, NEO_POOL_MEAN = 0, 1
NEO_OPT_SGD, NEO_OPT_ROWWISE_ADAGRAD, NEO_OPT_ADAGRAD, NEO_OPT_NONE = 0, 1, 2, 3
NEO_BWD_UPDATE, NEO_BWD_AGGREGATE, NEO_BWD_DENSE = 0, 1, 2
NEO_BWD_FLAG_ALIGNED, NEO_BWD_FLAG_FULL_ROWS = 0x100, 0x200
NEO_BWD_FLAG_PREPARE, NEO_BWD_FLAG_APPLY = 0x400, 0x800
NEO_BWD_FLAG_DIM8 = 0x1000
NEO_CACHE_LRU, NEO_CACHE_LFU = 0, 1

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
F64 = C.c_double
SZ = C.c_size_t


class NeoPiece(C.Structure):
    """neo_piece (neo_tbe.h)."""

    _fields_ = [
        ("src", C.c_uint64),
        ("dst", C.c_uint64),
        ("src_stride", C.c_int64),
        ("dst_stride", C.c_int64),
        ("src_col", C.c_int32),
        ("dst_col", C.c_int32),
        ("width", C.c_int32),
        ("accumulate", C.c_int32),
    ]


# symbol -> (restype, argtypes); every symbol neo_tbe.h declares
SIGNATURES = {
    "neo_version": (C.c_int, []),
    "neo_last_error": (C.c_char_p, []),
    "neo_device_sm_count": (C.c_int, []),
    "neo_error_reset": (C.c_int, [P, P]),
    "neo_tbe_forward": (
        C.c_int,
        [I32, I64, P, P, I32, P, I32, P, I32, P, I32, P, I32, I64, P, P],
    ),
    "neo_set_forward_residency": (C.c_int, [I32]),
    "neo_cache_workspace_bytes": (SZ, [I64]),
    "neo_cache_simulate": (C.c_int, [I64, I32, I32, P, I64, P, P, P, P, SZ, P, P]),
    "neo_tier_workspace_bytes": (SZ, [I64]),
    "neo_tier_prepare": (C.c_int, [I64, I64, I32, P, I32, I64, P, P, C.c_uint32, P, P, P, P, I64, I64, P, P, P, SZ,
                                   P, P]),
    "neo_tier_flush": (C.c_int, [I64, P, P, P, P, P, I64, I64, P]),
    "neo_tier_prepare_spill": (C.c_int, [I64, I64, I32, P, I32, I64, P, P, C.c_uint32, P, P, P, P, I64, I64, P, P,
                                         I64, P, P, SZ, P, P]),
    "neo_tier_spill_writeback": (C.c_int, [P, P, I64, P, P, P, P, I64, I64, P]),
    "neo_tbe_forward_scatter": (
        C.c_int,
        [I32, I64, P, P, I32, P, I32, P, I32, P, I32, P, I64, I32, I64, P, P],
    ),
    "neo_tbe_backward_workspace_bytes": (SZ, [I64, I64, I32]),
    "neo_tbe_bucket_workspace_bytes": (SZ, [I32, I64, I64, I64, I32]),
    "neo_tbe_backward": (
        C.c_int,
        [I32, I64, P, I64, P, I32, P, I32, P, P, I32, P, I64, I32, P, I32, I64,
         I32, I32, F64, F64, P, P, P, P, P, SZ, P, P],
    ),
    "neo_apply_row_updates": (C.c_int, [I64, P, P, I32, P, I32, P, I32, F64, F64, P]),
    "neo_fp16_roundtrip": (C.c_int, [I64, P, P, P, P]),
    "neo_cast": (C.c_int, [I64, P, I32, P, I32, P]),
    "neo_lengths_to_offsets": (C.c_int, [I64, P, P, P, SZ, P]),
    "neo_scan_workspace_bytes": (SZ, [I64]),
    "neo_bucketize_workspace_bytes": (SZ, [I64, I32]),
    "neo_bucketize_rowwise": (
        C.c_int,
        [I64, P, P, I32, I32, C.POINTER(C.c_int64), P, P, P, I32, P, P, SZ, P],
    ),
    "neo_bucketize_rowwise_multi": (C.c_int, [I32, I64, P, P, P, I32, I32, P, P, P, P, P, P, SZ, P]),
    "neo_permute_workspace_bytes": (SZ, [I32, I32]),
    "neo_permute_blocks": (C.c_int, [I32, I32, I64, P, P, I32, P, P, P, SZ, P]),
    "neo_copy_pieces": (C.c_int, [I64, P, I32, I32, I32, P]),
    "neo_copy_chunks": (C.c_int, [I64, P, I32, I32, I32, P]),
    "neo_gather_blocks": (C.c_int, [I32, P, P, P, P, I32, P]),
    "neo_check_indices": (C.c_int, [I32, I64, P, P, P, I32, P, P]),
}


class NeoLibraryMissing(ImportError):
    pass


_lib = None


def lib() -> C.CDLL:
    """The loaded library (loaded once; raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("NEO_B200_LIB", LIB_PATH))
    if not path.exists():
        raise NeoLibraryMissing(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    handle = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    _lib = handle
    return handle


def last_error() -> str:
    msg = lib().neo_last_error()
    return msg.decode() if msg else ""


class NeoStatusError(RuntimeError):
    def __init__(self, code: int, what: str, msg: str):
        self.code = code
        super().__init__(f"{what} failed with status {code}: {msg}")


def check(code: int, what: str) -> None:
    """Raise for a non-OK status; argument errors map to the reference's
    InvalidValue / LayoutMismatch types (errors.py)."""
    if code == NEO_OK:
        return
    from . import errors

    msg = last_error()
    if code == NEO_E_ARG:
        path, _, reason = msg.partition(": ")
        raise errors.InvalidValue(path or what, reason or msg)
    if code == NEO_E_LAYOUT:
        raise errors.LayoutMismatch(msg)
    raise NeoStatusError(code, what, msg)
