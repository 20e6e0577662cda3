"""ctypes binding of the C-ABI in include/spcv_cu.h (lib/libspcv_cu.so).

The shared library is built in-tree by ``paper_1911_09723_b200.build`` (or
``__graft_entry__.build()``). There is no fallback: if the library is missing
or cannot be loaded, importing this module raises ImportError.
"""
from __future__ import annotations

import ctypes
import os

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
LIB_PATH = os.environ.get("SPCV_CU_LIB") or os.path.join(LIB_DIR, "libspcv_cu.so")

from ._abi import *  # noqa: F401,F403  (status codes, layouts, modes)

# Every symbol include/spcv_cu.h declares, with (restype, argtypes).
_p, _i, _f, _z, _u64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_size_t, ctypes.c_uint64
_SPMM_ARGS = [_p, _p, _i, _i, _i, _i, _i, _p, _z, _i, _f, _f, _p, _i, _i, _i, _i, _i, _i, _i]
SIGNATURES = {
    "spcv_cu_pack": (_i, [_i, _i, _i, _p, _z, _p, _z, _p, _z, ctypes.POINTER(_p)]),
    "spcv_cu_unpack": (_i, [_p, _p, _p, _p]),
    "spcv_cu_weights_info": (_i, [_p, _p, _p, _p, _p, _p, _p]),
    "spcv_cu_free": (None, [_p]),
    "spcv_cu_weights_kernel": (_i, [_p, _i, _p]),
    "spcv_cu_weights_kernel_for": (_i, [_p, _i, _i, _i, _i, _p]),
    "spcv_cu_spmm_into": (_i, _SPMM_ARGS + [_p]),
    "spcv_cu_spmm_into_host": (_i, list(_SPMM_ARGS)),
    "spcv_cu_spmm_bcsr_into_host": (_i, [_i, _i, _i, _p, _z, _p, _z, _p, _z] + _SPMM_ARGS[1:]),
    "spcv_cu_weight_cache_clear": (None, []),
    "spcv_cu_cache_stats": (_i, [_p, _p, _p, _p, _p]),
    "spcv_cu_spmm_layer": (_i, [_p, _p, _i, _i, _i, _i, _p, _z, _i, _f, _f, _p, _p, _i, _i, _p]),
    "spcv_cu_dense_gemm_into": (_i, [_p, _i, _i] + _SPMM_ARGS[1:17] + [_i, _p]),
    "spcv_cu_model_parse": (_i, [_p, _z, _p]),
    "spcv_cu_model_load": (_i, [_p, _z, ctypes.POINTER(_p)]),
    "spcv_cu_model_layer": (_i, [_p, _i, _p]),
    "spcv_cu_model_weights": (_i, [_p, _i, ctypes.POINTER(_p)]),
    "spcv_cu_model_run": (_i, [_p, _i, _p, _i, _p, _p, _i, _p]),
    "spcv_cu_model_forward": (_i, [_p, _p, _i, _i, _i, _i, _p, _i, _p]),
    "spcv_cu_model_free": (None, [_p]),
    "spcv_cu_launch_count": (_u64, []),
    "spcv_cu_last_error": (ctypes.c_char_p, []),
    "spcv_cu_version": (ctypes.c_char_p, []),
}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    variant = bool(os.environ.get("SPCV_CU_LIB"))  # an A/B build may predate newer entry points
    for name, (res, args) in SIGNATURES.items():
        if variant and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.spcv_cu_last_error()
    return msg.decode() if msg else ""


def launch_count() -> int:
    return int(lib.spcv_cu_launch_count())


def cache_stats() -> dict:
    """spcv_cu_cache_stats: packed-weight cache and JIT compile counters."""
    n = ctypes.c_size_t()
    h, m, jc, jd = (ctypes.c_uint64() for _ in range(4))
    lib.spcv_cu_cache_stats(ctypes.byref(n), ctypes.byref(h), ctypes.byref(m), ctypes.byref(jc), ctypes.byref(jd))
    return {"entries": n.value, "hits": h.value, "misses": m.value, "jit_compiles": jc.value,
            "jit_disk_hits": jd.value}
