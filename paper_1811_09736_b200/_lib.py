"""ctypes binding of the C-ABI library ``_tc_collectives.so``.

The library is the product: there is no Python or CPU fallback.  Importing
this module fails loudly (``ImportError``) when the shared object is missing
or does not export every symbol ``include/tc_collectives.h`` declares.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_NAME = "_tc_collectives.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

# status codes (include/tc_collectives.h)
TC_OK = 0
TC_BAD_LENGTH = 1
TC_BAD_CONFIG = 2
TC_BAD_ALIGNMENT = 3
TC_WORKSPACE_TOO_SMALL = 4
TC_CUDA_ERROR = 5
TC_NO_DEVICE = 6

TC_F16 = 0
TC_F32 = 1
TC_F64 = 2
TC_BF16 = 3

TC_OP_REDUCE = 0
TC_OP_SCAN = 1
TC_OP_BN_STATS = 2

_c_void_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_size = ctypes.c_size_t

#: name -> (restype, argtypes); mirrors include/tc_collectives.h exactly.
SIGNATURES = {
    "tc_workspace_bytes": (_size, [ctypes.c_int, _i64, _i64]),
    "tc_seg_reduce": (ctypes.c_int, [_c_void_p, _i64, _i64, _c_void_p, ctypes.c_int,
                                     _c_void_p, _size, _c_void_p]),
    "tc_seg_reduce_ex": (ctypes.c_int, [_c_void_p, ctypes.c_int, _i64, _i64, _c_void_p,
                                        ctypes.c_int, _c_void_p, _size, _c_void_p]),
    "tc_seg_scan_ex": (ctypes.c_int, [_c_void_p, ctypes.c_int, _i64, _i64, _c_void_p, ctypes.c_int,
                                      ctypes.c_int, _c_void_p, _c_void_p, _c_void_p, _size,
                                      _c_void_p]),
    "tc_full_reduce": (ctypes.c_int, [_c_void_p, _i64, _c_void_p, ctypes.c_int,
                                      _c_void_p, _size, _c_void_p]),
    "tc_seg_scan": (ctypes.c_int, [_c_void_p, _i64, _i64, _c_void_p, ctypes.c_int, ctypes.c_int,
                                   _c_void_p, _c_void_p, _c_void_p, _size, _c_void_p]),
    "tc_full_scan": (ctypes.c_int, [_c_void_p, _i64, _c_void_p, ctypes.c_int, ctypes.c_int,
                                    _c_void_p, _c_void_p, _c_void_p, _size, _c_void_p]),
    "tc_irreg_reduce": (ctypes.c_int, [_c_void_p, ctypes.c_int, _i64, _c_void_p, _i64, _c_void_p,
                                       ctypes.c_int, _c_void_p, _size, _c_void_p]),
    "tc_irreg_scan": (ctypes.c_int, [_c_void_p, ctypes.c_int, _i64, _c_void_p, _i64, _c_void_p,
                                     ctypes.c_int, ctypes.c_int, _c_void_p, _size, _c_void_p]),
    "tc_bn_stats": (ctypes.c_int, [_c_void_p, ctypes.c_int, _i64, _i64, _i64, _c_void_p, _c_void_p,
                                   ctypes.c_int, _c_void_p, _size, _c_void_p]),
    "tc_plan_info": (ctypes.c_int, [ctypes.c_int, _i64, _i64, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, _c_void_p, _c_void_p]),
    "tc_h2d_pageable": (ctypes.c_int, [_c_void_p, _c_void_p, _size, _c_void_p]),
    "tc_d2h_pageable": (ctypes.c_int, [_c_void_p, _c_void_p, _size, _c_void_p]),
    "tc_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "tc_last_error": (ctypes.c_char_p, []),
    "tc_launch_count": (ctypes.c_uint64, []),
    "tc_reset_launch_count": (None, []),
    "tc_abi_version": (ctypes.c_int, []),
}


def _load() -> ctypes.CDLL:
    path = os.environ.get("TC_COLLECTIVES_LIB", str(LIB_PATH))
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')"
        )
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError -> missing export: fail loudly
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.tc_last_error()
    return msg.decode() if msg else ""


def status_string(code: int) -> str:
    return lib.tc_status_string(code).decode()
