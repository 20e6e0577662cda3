"""Host-side types of the reference SpMM operator surface (pure numpy, no device).

Reference (``/root/reference/proj``):
  * ``Tensor``, ``Activation``, ``ShapeError``/``LayoutError`` — include/spcv/tensor.hpp:11-97
  * ``BcsrMatrix``, ``FormatError``, ``encode_bcsr``/``decode_bcsr`` — include/spcv/sparse.hpp:12-103,
    src/sparse.cpp:16-51,108-148
  * ``generate_mask``/``apply_mask``/``BlockConfig`` — src/sparse.cpp:63-106, sparse.hpp:20-57
  * ``MicrokernelConfig``, ``Tier`` and the tier/variant plumbing — include/spcv/kernels.hpp:18-37,
    src/kernels.cpp:238-300

This module never loads ``libspcv_cu.so``: the workload generators and the
reference arm of ``bench.py`` import it without touching the CUDA library.
The device entry points live in ``spmm.py``.
"""
from __future__ import annotations

import enum
import os
from dataclasses import dataclass, field

import numpy as np

from . import _abi

# ------------------------------------------------------------------ errors
class ShapeError(ValueError):
    """tensor.hpp:12-15 (derives from std::invalid_argument there)."""


class LayoutError(ValueError):
    """tensor.hpp:18-21."""


class FormatError(ValueError):
    """sparse.hpp:12-15."""


class DeviceError(RuntimeError):
    """CUDA failure or a shape beyond the device limits (no reference counterpart)."""


class ModelIoError(RuntimeError):
    """model_io.hpp:13-16 and its subclasses below (model_io.hpp:18-46)."""


class BadMagicError(ModelIoError):
    pass


class UnsupportedVersionError(ModelIoError):
    pass


class TruncatedError(ModelIoError):
    pass


class ChecksumError(ModelIoError):
    pass


class ModelFormatError(ModelIoError):
    pass


# ----------------------------------------------------------------- tensors
class Layout(enum.IntEnum):
    CHW = _abi.LAYOUT_CHW
    HWC = _abi.LAYOUT_HWC


class Tensor:
    """Single-image host tensor (tensor.hpp:30-54); ``data`` is a flat float32 array."""

    def __init__(self, c: int, h: int, w: int, layout: Layout = Layout.CHW, data=None):
        if c < 1 or h < 1 or w < 1:
            raise ShapeError("tensor dims must be >= 1")
        self.channels, self.height, self.width, self.layout = int(c), int(h), int(w), Layout(layout)
        n = self.channels * self.height * self.width
        if data is None:
            self.data = np.zeros(n, dtype=np.float32)
        else:
            self.data = np.ascontiguousarray(np.asarray(data, dtype=np.float32).reshape(-1))
            if self.data.size != n:
                raise ShapeError("tensor data size mismatch")

    def spatial(self) -> int:
        return self.height * self.width

    def size(self) -> int:
        return self.data.size


@dataclass
class Activation:
    """tensor.hpp:74-97. ``clamp`` enforces lo < hi; apply() is the ternary compare."""

    kind: int = _abi.ACT_NONE
    lo: float = 0.0
    hi: float = 0.0

    @staticmethod
    def none() -> "Activation":
        return Activation()

    @staticmethod
    def clamp(lo: float, hi: float) -> "Activation":
        if not (lo < hi):
            raise ValueError("clamp requires lo < hi")
        return Activation(_abi.ACT_CLAMP, float(lo), float(hi))

    @staticmethod
    def relu6() -> "Activation":
        return Activation.clamp(0.0, 6.0)

    @staticmethod
    def relu() -> "Activation":
        return Activation.clamp(0.0, float("inf"))


class Tier(enum.IntEnum):
    Scalar = 0
    Vector = 1
    Auto = 2


@dataclass
class MicrokernelConfig:
    """kernels.hpp:28-33 plus ``strict`` (bit-exact arithmetic, default) vs FFMA."""

    m: int = 0
    n: int = 1
    prefetch: bool = True
    tier: Tier = Tier.Auto
    strict: bool = True


def resolve_tier(requested: Tier) -> Tier:
    """kernels.cpp:248-256 (one CUDA path: 'vector' is always available)."""
    env = os.environ.get("SPCV_FORCE_SCALAR")
    if env and env != "0":
        return Tier.Scalar
    return Tier.Vector if requested == Tier.Auto else Tier(requested)


def default_strip_width(t: Tier) -> int:
    return 16 if resolve_tier(t) == Tier.Vector else 8


def variant_name(m: int, n: int) -> str:
    return f"{m}x{n}"


def parse_variant(s: str) -> tuple[int, int]:
    """kernels.cpp:281-300."""
    bad = ValueError(f"bad variant '{s}' (expected MxN, e.g. 16x2)")
    x = s.find("x")
    if x <= 0 or x + 1 >= len(s):
        raise bad
    a, b = s[:x], s[x + 1:]
    if not (a.isdigit() and b.isdigit()):
        raise bad
    m, n = int(a), int(b)
    if m not in (4, 8, 16):
        raise ValueError(f"variant strip width must be 4, 8 or 16 (got {s})")
    if n not in (1, 2, 4):
        raise ValueError(f"variant out_block must be 1, 2 or 4 (got {s})")
    return m, n


def parse_tier(s: str) -> Tier:
    try:
        return {"scalar": Tier.Scalar, "vector": Tier.Vector, "auto": Tier.Auto}[s]
    except KeyError:
        raise ValueError(f"unknown tier '{s}' (expected scalar|vector|auto)") from None


# --------------------------------------------------------------------- BCSR
@dataclass
class BcsrMatrix:
    """sparse.hpp:65-79: Nx1 block CSR; values block-contiguous, output-channel-minor."""

    rows: int = 0
    cols: int = 0
    block_h: int = 1
    row_ptr: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint32))
    col_idx: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    def block_rows(self) -> int:
        return self.rows // self.block_h

    def nnz_blocks(self) -> int:
        return int(self.col_idx.size)

    def nnz_values(self) -> int:
        return int(self.values.size)

    def validate(self) -> None:
        """sparse.cpp:16-51, same checks in the same order (FormatError)."""
        if self.rows < 1 or self.cols < 1:
            raise FormatError("bcsr: dims must be >= 1")
        if self.block_h not in (1, 2, 4):
            raise FormatError("bcsr: block height must be 1, 2 or 4")
        if self.rows % self.block_h:
            raise FormatError("bcsr: rows not divisible by block height")
        rp = np.asarray(self.row_ptr, dtype=np.int64)
        if rp.size != self.block_rows() + 1:
            raise FormatError("bcsr: row_ptr length != block rows + 1")
        if rp[0] != 0:
            raise FormatError("bcsr: row_ptr[0] != 0")
        if np.any(np.diff(rp) < 0):
            raise FormatError("bcsr: row_ptr not non-decreasing")
        if rp[-1] != self.col_idx.size:
            raise FormatError("bcsr: row_ptr[-1] != block count")
        if self.values.size != self.col_idx.size * self.block_h:
            raise FormatError("bcsr: values length != block count * block height")
        ci = np.asarray(self.col_idx, dtype=np.int64)
        if ci.size:
            if np.any(ci >= self.cols):
                raise FormatError("bcsr: column index out of range")
            d = np.diff(ci)
            first = np.zeros(ci.size, dtype=bool)
            first[rp[:-1][rp[:-1] < ci.size]] = True
            if np.any((d <= 0) & ~first[1:]):
                raise FormatError("bcsr: column indices not strictly increasing")


@dataclass
class BlockConfig:
    """sparse.hpp:20-28: tile shape of the mask (out_block x in_block, each 1, 2 or 4)."""

    out_block: int = 1
    in_block: int = 1

    def __post_init__(self):
        if self.out_block not in (1, 2, 4) or self.in_block not in (1, 2, 4):
            raise FormatError("block sizes must be 1, 2 or 4")


class _Mt19937:
    """std::mt19937 seeded with a 32-bit value (numpy's legacy MT19937 seeding
    is the same init_genrand), raw 32-bit draws."""

    def __init__(self, seed: int):
        self._rs = np.random.RandomState(int(seed) & 0xFFFFFFFF)

    def __call__(self) -> int:
        return int(self._rs.randint(0, 2**32, dtype=np.uint64))


def _uniform_size_t(draw, a: int, b: int) -> int:
    """std::uniform_int_distribution<size_t>(a, b) over a 32-bit engine as
    libstdc++ 13 implements it: Lemire's nearly divisionless downscaling with
    a 64-bit product when the range fits the engine's 32 bits."""
    urange = b - a
    if urange >= 0xFFFFFFFF:
        raise ValueError("range beyond 32 bits is not needed for masks")
    r = urange + 1
    prod = draw() * r
    low = prod & 0xFFFFFFFF
    if low < r:
        threshold = ((-r) & 0xFFFFFFFF) % r
        while low < threshold:
            prod = draw() * r
            low = prod & 0xFFFFFFFF
    return a + (prod >> 32)


def generate_mask(rows: int, cols: int, sparsity: float, block: BlockConfig = BlockConfig(),
                  seed: int = 0) -> np.ndarray:
    """sparse.cpp:63-98: keep-mask [rows][cols] (True = kept) with exactly
    llround(tiles * sparsity) whole out_block x in_block tiles zeroed, chosen
    by a partial Fisher-Yates shuffle driven by std::mt19937(seed). Same
    checks and order: sparsity in [0, 1) (ValueError), divisibility (FormatError)."""
    if not (0.0 <= sparsity < 1.0):
        raise ValueError("sparsity must be in [0, 1)")
    if rows % block.out_block:
        raise FormatError("generate_mask: rows not divisible by out_block")
    if cols % block.in_block:
        raise FormatError("generate_mask: cols not divisible by in_block")
    if rows < 1 or cols < 1:
        raise ShapeError("mask dims must be >= 1")
    trows, tcols = rows // block.out_block, cols // block.in_block
    tiles = trows * tcols
    zeroed = int(np.floor(tiles * sparsity + 0.5))  # llround of a non-negative value
    pos = list(range(tiles))
    draw = _Mt19937(seed)
    for i in range(min(zeroed, tiles - 1)):
        j = _uniform_size_t(draw, i, tiles - 1)
        pos[i], pos[j] = pos[j], pos[i]
    keep_t = np.ones(tiles, dtype=bool)
    keep_t[np.asarray(pos[:zeroed], dtype=np.int64)] = False
    keep = keep_t.reshape(trows, tcols)
    return np.repeat(np.repeat(keep, block.out_block, axis=0), block.in_block, axis=1)


def apply_mask(w: np.ndarray, keep: np.ndarray) -> np.ndarray:
    """sparse.cpp:100-106: zero the pruned positions (ShapeError on mismatch)."""
    if w.shape != keep.shape:
        raise ShapeError("apply_mask: matrix/mask shape mismatch")
    out = np.array(w, dtype=np.float32, copy=True)
    out[~keep] = 0.0
    return out


def encode_bcsr(w: np.ndarray, block_h: int) -> BcsrMatrix:
    """sparse.cpp:108-134: keep a block iff any member != 0 (so -0.0 is zero)."""
    if block_h not in (1, 2, 4):
        raise FormatError("encode_bcsr: block height must be 1, 2 or 4")
    w = np.ascontiguousarray(w, dtype=np.float32)
    rows, cols = w.shape
    if rows % block_h:
        raise ShapeError("encode_bcsr: rows not divisible by block height")
    blocks = w.reshape(rows // block_h, block_h, cols)           # [br][n][c]
    keep = np.any(blocks != 0.0, axis=1)                          # [br][c]
    counts = keep.sum(axis=1)
    row_ptr = np.zeros(rows // block_h + 1, dtype=np.uint32)
    np.cumsum(counts, out=row_ptr[1:])
    br, c = np.nonzero(keep)                                      # row-major: br then c ascending
    values = blocks.transpose(0, 2, 1)[br, c, :].reshape(-1)      # [blk][n]
    return BcsrMatrix(rows, cols, block_h, row_ptr, c.astype(np.uint32),
                      np.ascontiguousarray(values, dtype=np.float32))


def decode_bcsr(m: BcsrMatrix) -> np.ndarray:
    """sparse.cpp:136-148: validate, then scatter blocks into a dense matrix."""
    m.validate()
    w = np.zeros((m.rows, m.cols), dtype=np.float32)
    counts = np.diff(m.row_ptr.astype(np.int64))
    br = np.repeat(np.arange(m.block_rows()), counts)
    vals = m.values.reshape(-1, m.block_h)
    for n in range(m.block_h):
        w[br * m.block_h + n, m.col_idx.astype(np.int64)] = vals[:, n]
    return w

