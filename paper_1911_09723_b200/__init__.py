"""paper_1911_09723_b200 — B200-native sparse 1x1-convolution SpMM.

A drop-in for the reference ``spcv::spmm_into`` hot path
(/root/reference/proj/src/kernels.cpp:304-334) built on hand-written sm_100a
kernels behind the C-ABI in ``include/spcv_cu.h``. See DESIGN.md.
"""
from ._capi import LIB_PATH, launch_count
from .spmm import (
    BadMagicError,
    ChecksumError,
    DeviceModel,
    ModelFormatError,
    ModelIoError,
    TruncatedError,
    UnsupportedVersionError,
    parse_model_status,
    Activation,
    BcsrMatrix,
    BlockConfig,
    DeviceBcsr,
    DeviceError,
    FormatError,
    Layout,
    LayoutError,
    MicrokernelConfig,
    ShapeError,
    Tensor,
    Tier,
    decode_bcsr,
    default_strip_width,
    dense_gemm_batched_into,
    apply_mask,
    encode_bcsr,
    generate_mask,
    parse_tier,
    parse_variant,
    resolve_tier,
    spconv_1x1,
    spmm,
    spmm_batched_into,
    spmm_host_batched,
    spmm_into,
    spmm_layer,
    variant_name,
)

__all__ = [
    "BadMagicError", "ChecksumError", "DeviceModel", "ModelFormatError", "ModelIoError",
    "TruncatedError", "UnsupportedVersionError", "parse_model_status",
    "Activation", "BcsrMatrix", "BlockConfig", "apply_mask", "generate_mask", "dense_gemm_batched_into", "DeviceBcsr", "DeviceError", "FormatError", "Layout",
    "LayoutError", "MicrokernelConfig", "ShapeError", "Tensor", "Tier", "decode_bcsr",
    "default_strip_width", "encode_bcsr", "parse_tier", "parse_variant", "resolve_tier",
    "spconv_1x1", "spmm", "spmm_batched_into", "spmm_host_batched", "spmm_into", "spmm_layer",
    "variant_name", "launch_count", "LIB_PATH",
]
