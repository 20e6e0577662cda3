"""Python mirror of the reference SpMM operator surface, over the C-ABI.

Reference (``/root/reference/proj``):
  * ``Tensor``, ``Activation``, ``ShapeError``/``LayoutError`` — include/spcv/tensor.hpp:11-97
  * ``BcsrMatrix``, ``FormatError``, ``encode_bcsr``/``decode_bcsr`` — include/spcv/sparse.hpp:12-103,
    src/sparse.cpp:16-51,108-148
  * ``MicrokernelConfig``, ``Tier``, ``spmm_into``/``spmm``/``spconv_1x1`` — include/spcv/kernels.hpp:18-55,
    src/kernels.cpp:238-341

Names, argument meaning, validation order and error classes follow the
reference so parity tests read like ``proj/tests/test_kernels.cpp``. All
arithmetic runs in the sm_100a kernel (``csrc/spmm_kernel.cuh``); there is no
CPU path. Host (numpy) tensors go through ``spcv_cu_spmm_into_host`` (copy in,
kernel, copy out); torch CUDA tensors go through ``spcv_cu_spmm_into`` on the
current stream.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _capi
from ._capi import lib
from .bcsr import (  # host-side types (pure numpy), re-exported
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


def _raise(status: int) -> None:
    if status == _capi.OK:
        return
    msg = _capi.last_error()
    if status == _capi.ERR_LAYOUT:
        raise LayoutError(msg)
    if status == _capi.ERR_SHAPE:
        raise ShapeError(msg)
    if status == _capi.ERR_FORMAT:
        raise FormatError(msg)
    if status == _capi.ERR_INVALID:
        raise ValueError(msg)
    model_errors = {_capi.ERR_MODEL_IO: ModelIoError, _capi.ERR_BAD_MAGIC: BadMagicError,
                    _capi.ERR_VERSION: UnsupportedVersionError, _capi.ERR_TRUNCATED: TruncatedError,
                    _capi.ERR_CHECKSUM: ChecksumError, _capi.ERR_MODEL_FORMAT: ModelFormatError}
    if status in model_errors:
        raise model_errors[status](msg)
    raise DeviceError(msg or f"spcv_cu status {status}")


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


class DeviceBcsr:
    """BCSR weights packed once onto the current CUDA device (spcv_cu_pack)."""

    def __init__(self, m: BcsrMatrix):
        rp = np.ascontiguousarray(m.row_ptr, dtype=np.uint32)
        ci = np.ascontiguousarray(m.col_idx, dtype=np.uint32)
        va = np.ascontiguousarray(m.values, dtype=np.float32)
        h = ctypes.c_void_p()
        _raise(lib.spcv_cu_pack(int(m.rows), int(m.cols), int(m.block_h), _ptr(rp), rp.size,
                                _ptr(ci), ci.size, _ptr(va), va.size, ctypes.byref(h)))
        self._h = h
        self.rows, self.cols, self.block_h = int(m.rows), int(m.cols), int(m.block_h)
        self.nnz_blocks = int(ci.size)
        slots = ctypes.c_int()
        dev = ctypes.c_int()
        _raise(lib.spcv_cu_weights_info(self._h, None, None, None, None, ctypes.byref(slots),
                                        ctypes.byref(dev)))
        self.row_slots, self.device = slots.value, dev.value

    @property
    def handle(self):
        return self._h

    def kernel(self, strict: bool = True) -> str:
        """Which CUDA kernel runs these weights: "tile" or "jit" (spcv_cu_weights_kernel;
        compiles the weight-specialised kernel if it is due)."""
        k = ctypes.c_int()
        _raise(lib.spcv_cu_weights_kernel(self._h, _capi.MODE_STRICT if strict else _capi.MODE_FAST,
                                          ctypes.byref(k)))
        return "jit" if k.value == _capi.KERNEL_JIT else "tile"

    def kernel_for(self, images: int, h: int, w: int, strict: bool = True) -> str:
        """The kernel a call over `images` h x w images runs: "jit", "small"
        or "tile" (spcv_cu_weights_kernel_for)."""
        k = ctypes.c_int()
        _raise(lib.spcv_cu_weights_kernel_for(self._h, _capi.MODE_STRICT if strict else _capi.MODE_FAST,
                                              images, h, w, ctypes.byref(k)))
        return _capi.KERNEL_NAMES[k.value]

    def unpack(self) -> BcsrMatrix:
        """Bit-exact device decode of the counts/deltas/values streams."""
        rp = np.zeros(self.rows // self.block_h + 1, dtype=np.uint32)
        ci = np.zeros(self.nnz_blocks, dtype=np.uint32)
        va = np.zeros(self.nnz_blocks * self.block_h, dtype=np.float32)
        _raise(lib.spcv_cu_unpack(self._h, _ptr(rp), _ptr(ci) or None, _ptr(va) or None))
        return BcsrMatrix(self.rows, self.cols, self.block_h, rp, ci, va)

    def close(self) -> None:
        if getattr(self, "_h", None) and not getattr(self, "_borrowed", False):
            lib.spcv_cu_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------- spmm
def _mode(cfg: MicrokernelConfig) -> int:
    return _capi.MODE_STRICT if cfg.strict else _capi.MODE_FAST


def spmm_into(w, act: Tensor, bias, fused: Activation, out: Tensor,
              cfg: MicrokernelConfig | None = None) -> None:
    """kernels.hpp:45-46 with host tensors. ``w`` is a BcsrMatrix (packed per
    call, like the reference which takes it by const&) or a DeviceBcsr."""
    cfg = cfg or MicrokernelConfig()
    b = np.zeros(0, np.float32) if bias is None else np.ascontiguousarray(bias, np.float32).reshape(-1)
    # The reference checks arguments before it ever reads the matrix
    # (kernels.cpp:306-322); do the same so error precedence matches even for
    # a malformed BcsrMatrix, which the packer rejects afterwards.
    rows = w.rows
    if act.layout != Layout.CHW:
        raise LayoutError("spmm: activation must be CHW")
    if w.cols != act.channels:
        raise ShapeError(f"spmm: weight cols {w.cols} != activation channels {act.channels}")
    if cfg.n != w.block_h:
        raise FormatError(f"spmm: cfg out_block {cfg.n} != matrix block height {w.block_h}")
    if b.size and b.size != rows:
        raise ShapeError("spmm: bias length != rows")
    if (out.layout != Layout.CHW or out.channels != rows or out.height != act.height
            or out.width != act.width):
        raise ShapeError("spmm: output tensor shape/layout mismatch")
    m = cfg.m if cfg.m != 0 else default_strip_width(cfg.tier)
    if m not in (4, 8, 16):
        raise ValueError("spmm: strip width must be 4, 8 or 16")
    a = np.ascontiguousarray(act.data, np.float32)
    if out.data.dtype != np.float32 or not out.data.flags.c_contiguous:
        out.data = np.ascontiguousarray(out.data, np.float32)
    tail = (_ptr(a), int(act.layout), 1, act.channels, act.height, act.width,
            _ptr(b) or None, b.size, fused.kind, fused.lo, fused.hi, _ptr(out.data), int(out.layout),
            out.channels, out.height, out.width, cfg.m, cfg.n, _mode(cfg))
    if isinstance(w, DeviceBcsr):
        _raise(lib.spcv_cu_spmm_into_host(w.handle, *tail))
        return
    # a host BcsrMatrix: packed once per distinct content (spcv_cu_spmm_bcsr_into_host's cache)
    rp = np.ascontiguousarray(w.row_ptr, dtype=np.uint32)
    ci = np.ascontiguousarray(w.col_idx, dtype=np.uint32)
    va = np.ascontiguousarray(w.values, dtype=np.float32)
    _raise(lib.spcv_cu_spmm_bcsr_into_host(int(w.rows), int(w.cols), int(w.block_h), _ptr(rp), rp.size,
                                           _ptr(ci), ci.size, _ptr(va), va.size, *tail))


def spmm(w, act: Tensor, bias, fused: Activation | None = None,
         cfg: MicrokernelConfig | None = None) -> Tensor:
    """kernels.cpp:336-341."""
    out = Tensor(w.rows, act.height, act.width, Layout.CHW)
    spmm_into(w, act, bias, fused or Activation.none(), out, cfg)
    return out


spconv_1x1 = spmm


def spmm_host_batched(w: DeviceBcsr, act: np.ndarray, bias, fused: Activation, out: np.ndarray,
                      cfg: MicrokernelConfig | None = None) -> None:
    """Batched host path: act [B][K][H][W] -> out [B][M][H][W] (numpy, ideally pinned)
    through spcv_cu_spmm_into_host (H2D, kernel, D2H inside the call)."""
    cfg = cfg or MicrokernelConfig(n=w.block_h)
    if not isinstance(act, np.ndarray) or act.ndim != 4:
        raise ShapeError("spmm_host_batched: act must be a [B][K][H][W] numpy array")
    if act.dtype != np.float32 or not act.flags.c_contiguous:
        act = np.ascontiguousarray(act, dtype=np.float32)  # a copy (a pinned act should be float32 C-order)
    B, K, H, W = act.shape
    if (not isinstance(out, np.ndarray) or out.dtype != np.float32 or not out.flags.c_contiguous
            or not out.flags.writeable):
        raise ShapeError("spmm_host_batched: out must be a writeable C-contiguous float32 numpy array")
    if out.shape != (B, w.rows, H, W):
        raise ShapeError(f"spmm_host_batched: out shape {out.shape} != {(B, w.rows, H, W)}")
    b = None if bias is None else np.ascontiguousarray(bias, np.float32).reshape(-1)
    _raise(lib.spcv_cu_spmm_into_host(
        w.handle, act.ctypes.data, _capi.LAYOUT_CHW, B, K, H, W,
        None if b is None else b.ctypes.data, 0 if b is None else b.size, fused.kind, fused.lo,
        fused.hi, out.ctypes.data, _capi.LAYOUT_CHW, out.shape[1], out.shape[2], out.shape[3],
        cfg.m, cfg.n, _mode(cfg)))


def spmm_batched_into(w: DeviceBcsr, act, bias, fused: Activation, out,
                      cfg: MicrokernelConfig | None = None, stream=None) -> None:
    """Device path: torch CUDA float32 tensors, act [B][K][H][W] (or [K][H][W]),
    out [B][M][H][W]; asynchronous on ``stream`` (default: torch's current stream)."""
    import torch

    cfg = cfg or MicrokernelConfig(n=w.block_h)
    if act.dim() == 3:
        act = act.unsqueeze(0)
        out = out.unsqueeze(0)
    if act.device.type != "cuda" or out.device.type != "cuda":
        raise DeviceError("spmm_batched_into: tensors must be on a CUDA device")
    if act.dtype != torch.float32 or out.dtype != torch.float32:
        raise ShapeError("spmm_batched_into: float32 tensors required")
    if not (act.is_contiguous() and out.is_contiguous()):
        raise LayoutError("spmm_batched_into: contiguous NCHW tensors required")
    B, K, H, W = act.shape
    if out.shape[0] != B:
        raise ShapeError("spmm_batched_into: batch mismatch")
    bptr, blen = None, 0
    if bias is not None:
        if bias.device.type != "cuda" or bias.dtype != torch.float32:
            raise ShapeError("spmm_batched_into: bias must be a CUDA float32 tensor")
        bptr, blen = bias.data_ptr(), bias.numel()
    if stream is None:
        stream = torch.cuda.current_stream(act.device)
    sptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
    _raise(lib.spcv_cu_spmm_into(
        w.handle, act.data_ptr(), _capi.LAYOUT_CHW, B, K, H, W, bptr, blen, fused.kind, fused.lo,
        fused.hi, out.data_ptr(), _capi.LAYOUT_CHW, out.shape[1], out.shape[2], out.shape[3],
        cfg.m, cfg.n, _mode(cfg), sptr))


def bind_batched(w: DeviceBcsr, act, bias, fused: Activation, out,
                 cfg: MicrokernelConfig | None = None, stream=None):
    """spmm_batched_into with its arguments checked and converted once: returns
    a zero-argument callable that launches the same call again (serving loops
    over fixed buffers; the tensors must stay alive and keep their addresses).
    Each invocation is one C-ABI call (spcv_cu_spmm_into, its checks included)
    without the per-call torch attribute reads, ~2 us instead of ~10 us of host
    time — what bounds a batch-1 layer chain launched from Python."""
    import torch

    cfg = cfg or MicrokernelConfig(n=w.block_h)
    if act.dim() == 3:
        act = act.unsqueeze(0)
        out = out.unsqueeze(0)
    if act.device.type != "cuda" or out.device.type != "cuda":
        raise DeviceError("bind_batched: tensors must be on a CUDA device")
    if act.dtype != torch.float32 or out.dtype != torch.float32:
        raise ShapeError("bind_batched: float32 tensors required")
    if not (act.is_contiguous() and out.is_contiguous()):
        raise LayoutError("bind_batched: contiguous NCHW tensors required")
    B, K, H, W = act.shape
    if out.shape[0] != B:
        raise ShapeError("bind_batched: batch mismatch")
    bptr, blen = None, 0
    if bias is not None:
        if bias.device.type != "cuda" or bias.dtype != torch.float32:
            raise ShapeError("bind_batched: bias must be a CUDA float32 tensor")
        bptr, blen = bias.data_ptr(), bias.numel()
    if stream is None:
        stream = torch.cuda.current_stream(act.device)
    sptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
    fn = lib.spcv_cu_spmm_into
    args = [w.handle, act.data_ptr(), _capi.LAYOUT_CHW, B, K, H, W, bptr, blen, fused.kind, fused.lo,
            fused.hi, out.data_ptr(), _capi.LAYOUT_CHW, out.shape[1], out.shape[2], out.shape[3],
            cfg.m, cfg.n, _mode(cfg), sptr]
    cargs = tuple(a if a is None or isinstance(a, ctypes._SimpleCData) else t(a) for t, a in zip(fn.argtypes, args))
    keep = (w, act, bias, out, stream)  # the bound buffers live as long as the callable

    def call(_fn=fn, _a=cargs, _keep=keep):
        rc = _fn(*_a)
        if rc:
            _raise(rc)

    return call


def dense_gemm_batched_into(w, act, bias, fused: Activation, out, cfg: MicrokernelConfig | None = None,
                            stream=None) -> None:
    """Dense fp32 baseline (reference dense_gemm_into, kernels.cpp:345-373) on
    torch CUDA tensors: w [M][K] row-major, act [B][K][H][W], out [B][M][H][W].
    cuBLAS SGEMM (pedantic fp32) + fused bias/clamp epilogue; not bit-exact."""
    import torch

    cfg = cfg or MicrokernelConfig()
    if act.dim() == 3:
        act = act.unsqueeze(0)
        out = out.unsqueeze(0)
    for t in (w, act, out):
        if t.device.type != "cuda" or t.dtype != torch.float32 or not t.is_contiguous():
            raise DeviceError("dense_gemm_batched_into: contiguous CUDA float32 tensors required")
    M, K = w.shape
    B, C, H, W = act.shape
    bptr, blen = (None, 0) if bias is None else (bias.data_ptr(), bias.numel())
    if stream is None:
        stream = torch.cuda.current_stream(act.device)
    sptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
    _raise(lib.spcv_cu_dense_gemm_into(
        w.data_ptr(), M, K, act.data_ptr(), _capi.LAYOUT_CHW, B, C, H, W, bptr, blen, fused.kind,
        fused.lo, fused.hi, out.data_ptr(), _capi.LAYOUT_CHW, out.shape[1], out.shape[2],
        out.shape[3], cfg.m, sptr))


def spmm_layer(w: DeviceBcsr, act, bias, fused: Activation, out, residual=None,
               strict: bool = True, stream=None) -> None:
    """The executor's pointwise step on device (run_network, netdef.cpp:494-512):
    `w` may carry padded rows (rows padded to the block height); only the
    first out.shape[1] rows are stored. `residual` (optional, out's shape) is
    added after the activation (add_residual, netdef.cpp:448-452)."""
    import torch

    if act.dim() == 3:
        act = act.unsqueeze(0)
        out = out.unsqueeze(0)
        residual = None if residual is None else residual.unsqueeze(0)
    for t in (act, out) + (() if residual is None else (residual,)):
        if t.device.type != "cuda" or t.dtype != torch.float32 or not t.is_contiguous():
            raise DeviceError("spmm_layer: contiguous CUDA float32 tensors required")
    if residual is not None and tuple(residual.shape) != tuple(out.shape):
        raise ShapeError("spmm_layer: residual shape != output shape")
    B, K, H, W = act.shape
    if tuple(out.shape) != (B, out.shape[1], H, W):
        raise ShapeError("spmm_layer: output shape mismatch")
    bptr, blen = (None, 0) if bias is None else (bias.data_ptr(), bias.numel())
    if stream is None:
        stream = torch.cuda.current_stream(act.device)
    sptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
    _raise(lib.spcv_cu_spmm_layer(
        w.handle, act.data_ptr(), B, K, H, W, bptr, blen, fused.kind, fused.lo, fused.hi,
        None if residual is None else residual.data_ptr(), out.data_ptr(), out.shape[1],
        _capi.MODE_STRICT if strict else _capi.MODE_FAST, sptr))


# ------------------------------------------------------------ model files
LAYER_KINDS = ("entry_conv", "pointwise", "depthwise", "global_pool", "fully_connected")


def parse_model_status(data: bytes) -> int:
    """spcv_cu_model_parse: 0 or the typed-error status (no device work)."""
    buf = np.frombuffer(data, np.uint8)
    n = ctypes.c_int()
    return int(lib.spcv_cu_model_parse(buf.ctypes.data if buf.size else None, buf.size, ctypes.byref(n)))


class DeviceModel:
    """An SPCV model file (model_io.cpp) parsed with the reference's checks and
    uploaded once: sparse 1x1 / classifier layers packed on the device."""

    def __init__(self, data: bytes):
        buf = np.frombuffer(data, np.uint8)
        h = ctypes.c_void_p()
        _raise(lib.spcv_cu_model_load(buf.ctypes.data if buf.size else None, buf.size, ctypes.byref(h)))
        self._h = h
        n = ctypes.c_int()
        _raise(lib.spcv_cu_model_parse(buf.ctypes.data, buf.size, ctypes.byref(n)))
        self.layers = []
        info = np.zeros(12, np.int32)
        for i in range(n.value):
            _raise(lib.spcv_cu_model_layer(self._h, i, info.ctypes.data))
            k = info.tolist()
            self.layers.append(dict(kind=LAYER_KINDS[k[0]], cin=k[1], cout=k[2], in_h=k[3], in_w=k[4],
                                    out_h=k[5], out_w=k[6], sparse=bool(k[7]), block_h=k[8],
                                    act_kind=k[9], residual_src=k[10], stride=k[11]))

    def weights(self, i: int) -> "DeviceBcsr":
        """Borrowed packed weights of sparse layer i (valid while the model lives)."""
        p = ctypes.c_void_p()
        _raise(lib.spcv_cu_model_weights(self._h, i, ctypes.byref(p)))
        L = self.layers[i]
        w = DeviceBcsr.__new__(DeviceBcsr)
        w._h, w._borrowed = p, True
        w.cols, w.block_h = L["cin"], L["block_h"]
        rows = ctypes.c_int()
        nb = ctypes.c_size_t()
        _raise(lib.spcv_cu_weights_info(p, ctypes.byref(rows), None, None, ctypes.byref(nb), None, None))
        w.rows, w.nnz_blocks, w.row_slots, w.device = rows.value, nb.value, 0, 0
        return w

    def run(self, i: int, act, out, residual=None, strict: bool = True, stream=None) -> None:
        """Layer i on torch CUDA tensors: a 1x1 / classifier layer as run_network's
        pointwise step; an entry conv (HWC input), depthwise or pool layer as
        in forward()."""
        import torch

        L = self.layers[i]
        B = act.shape[0]
        for name, t, per in (("act", act, L["cin"] * L["in_h"] * L["in_w"]),
                             ("out", out, L["cout"] * L["out_h"] * L["out_w"]),
                             ("residual", residual, L["cout"] * L["out_h"] * L["out_w"])):
            if t is None:
                continue
            if (t.device.type != "cuda" or t.device != act.device or t.dtype != torch.float32
                    or not t.is_contiguous() or t.numel() != B * per):
                raise ShapeError(f"run: {name} must be a contiguous float32 CUDA tensor of {B}x{per} elements")
        if stream is None:
            stream = torch.cuda.current_stream(act.device)
        sptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        _raise(lib.spcv_cu_model_run(self._h, i, act.data_ptr(), B,
                                     None if residual is None else residual.data_ptr(), out.data_ptr(),
                                     _capi.MODE_STRICT if strict else _capi.MODE_FAST, sptr))

    def forward(self, images_hwc, strict: bool = True, stream=None, out=None):
        """run_network on the device: torch CUDA [B][H][W][C] fp32 -> logits [B][classes]
        (spcv_cu_model_forward; bit-exact with the reference executor in strict mode).
        `out`: optional preallocated logits (a forward repeated with the same
        input/output tensors on a non-default stream replays a CUDA graph)."""
        import torch

        if images_hwc.device.type != "cuda" or images_hwc.dtype != torch.float32 or images_hwc.dim() != 4:
            raise DeviceError("forward: images must be a [B][H][W][C] float32 CUDA tensor")
        x = images_hwc.contiguous()
        B, H, W, C = x.shape
        classes = self.layers[-1]["cout"]
        if out is None:
            out = torch.empty((B, classes), dtype=torch.float32, device=x.device)
        elif (out.device != x.device or out.dtype != torch.float32 or not out.is_contiguous()
              or tuple(out.shape) != (B, classes)):
            raise ShapeError(f"forward: out must be a contiguous float32 tensor of shape {(B, classes)} "
                             f"on {x.device}")
        if stream is None:
            stream = torch.cuda.current_stream(x.device)
        sptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        _raise(lib.spcv_cu_model_forward(self._h, x.data_ptr(), B, H, W, C, out.data_ptr(),
                                         _capi.MODE_STRICT if strict else _capi.MODE_FAST, sptr))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib.spcv_cu_model_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
