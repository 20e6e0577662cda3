"""paper_1911_09723_b200 — B200-native sparse 1x1-convolution SpMM.

A drop-in for the reference ``spcv::spmm_into`` hot path
(/root/reference/proj/src/kernels.cpp:304-334) built on hand-written sm_100a
kernels behind the C-ABI in ``include/spcv_cu.h``. See DESIGN.md.

Host-side types (``BcsrMatrix``, ``encode_bcsr``, ``Activation`` ...) come from
the pure-numpy ``bcsr`` module. Every device symbol (``DeviceBcsr``,
``spmm_into`` ...) is resolved on first access through ``spmm``, which loads
``lib/libspcv_cu.so`` and raises ImportError when it is missing — there is no
CPU fallback. Importing the package alone (e.g. ``workloads`` from the
reference arm of bench.py) maps no CUDA library.
"""
from __future__ import annotations

import importlib

from .bcsr import (
    Activation,
    BadMagicError,
    BcsrMatrix,
    BlockConfig,
    ChecksumError,
    DeviceError,
    FormatError,
    Layout,
    LayoutError,
    MicrokernelConfig,
    ModelFormatError,
    ModelIoError,
    ShapeError,
    Tensor,
    Tier,
    TruncatedError,
    UnsupportedVersionError,
    apply_mask,
    decode_bcsr,
    default_strip_width,
    encode_bcsr,
    generate_mask,
    parse_tier,
    parse_variant,
    resolve_tier,
    variant_name,
)

# device symbols -> defining module (loaded lazily; both load libspcv_cu.so)
_DEVICE = {
    "DeviceBcsr": "spmm", "DeviceModel": "spmm", "parse_model_status": "spmm",
    "dense_gemm_batched_into": "spmm", "spconv_1x1": "spmm", "spmm": "spmm",
    "spmm_batched_into": "spmm", "bind_batched": "spmm", "spmm_host_batched": "spmm", "spmm_into": "spmm",
    "spmm_layer": "spmm", "LIB_PATH": "_capi", "launch_count": "_capi", "cache_stats": "_capi",
}


def _bind() -> None:
    # importing the submodule ``spmm`` sets the package attribute ``spmm`` to
    # the module; rebind every device name (the function ``spmm`` included)
    for name, mod in _DEVICE.items():
        globals()[name] = getattr(importlib.import_module(f".{mod}", __name__), name)


def __getattr__(name: str):
    if name not in _DEVICE:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    _bind()
    return globals()[name]


def load() -> None:
    """Load the CUDA library now (ImportError if it is missing)."""
    _bind()


__all__ = [
    "BadMagicError", "ChecksumError", "ModelFormatError", "ModelIoError", "TruncatedError",
    "UnsupportedVersionError", "Activation", "BcsrMatrix", "BlockConfig", "apply_mask", "generate_mask",
    "DeviceError", "FormatError", "Layout", "LayoutError", "MicrokernelConfig", "ShapeError", "Tensor",
    "Tier", "decode_bcsr", "default_strip_width", "encode_bcsr", "parse_tier", "parse_variant",
    "resolve_tier", "variant_name", "load", *sorted(_DEVICE),
]
