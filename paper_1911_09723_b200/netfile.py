"""SPCV model files written from Python: the MobileNet-v1 builder and the
serializer of the reference, restated so a full network can be produced on
the GPU box without the reference library.

* ``build_mbv1`` follows ``build_mbv1`` / ``Chain`` (netdef.cpp:70-218) and
  ``default_plan("mbv1")`` (netdef.cpp:242-259): entry 3x3/2 conv, 13
  depthwise + pointwise pairs (strided at 2, 4, 6, 12), global pool, dense
  classifier; ReLU6 everywhere except the classifier; pointwise layers sparse,
  4x1 blocks from the 12th on.
* ``serialize`` writes the container of ``serialize_model``
  (model_io.cpp:146-227): little-endian fields, u32-length strings and arrays,
  CRC-32 (zlib) trailer over everything before it.

Weights are seeded synthetic values of the reference's shapes (not its
``instantiate_weights`` stream): entry / depthwise / classifier uniform
He-style, pointwise masks from ``workloads`` (uniform, block-aware), biases
N(0, 0.1).
"""
from __future__ import annotations

import math
import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

from .bcsr import BcsrMatrix, encode_bcsr
from .workloads import Layer as WLayer
from .workloads import make_layer_data

ENTRY, POINTWISE, DEPTHWISE, POOL, FC = 0, 1, 2, 3, 4
NONE_STORAGE, CONV, DW, DENSE, BCSR = 0, 1, 2, 3, 4


@dataclass
class NetLayer:
    kind: int
    name: str
    cin: int
    cout: int
    stride: int
    in_h: int
    in_w: int
    out_h: int
    out_w: int
    sparse: bool = False
    sparsity: float = 0.0
    block_h: int = 1
    act: tuple = ("none", 0.0, 0.0)
    residual_src: int = -1
    bias: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    weights: object = None  # np.ndarray (conv / depthwise / dense) or BcsrMatrix


@dataclass
class Network:
    name: str
    width: float
    input_h: int
    input_w: int
    input_c: int
    num_classes: int
    plan_sparsity: float
    block_start: int
    block_h_after: int
    layers: list


def same_pad_out(n: int, stride: int) -> int:
    """same_pad(...).out (tensor.cpp:7-16)."""
    return (n + stride - 1) // stride


def round_channels(base: int, width: float) -> int:
    """netdef.cpp:22-25 (llround: halves away from zero)."""
    c = int(math.floor(base * width / 8.0 + 0.5)) * 8
    return max(c, 8)


def build_mbv1(width: float = 1.0, sparsity: float = 0.9, seed: int = 1, input_hw: int = 224,
               num_classes: int = 1000, block_start: int = 12, block_h_after: int = 4) -> Network:
    rng = np.random.default_rng(seed)
    relu6 = ("clamp", 0.0, 6.0)
    layers = []
    c, h, w = 3, input_hw, input_hw

    def bias(n):
        return (rng.standard_normal(n) * 0.1).astype(np.float32)

    def uniform(shape, fan_in):
        lim = math.sqrt(6.0 / fan_in)
        return rng.uniform(-lim, lim, shape).astype(np.float32)

    co = round_channels(32, width)
    oh, ow = same_pad_out(h, 2), same_pad_out(w, 2)
    layers.append(NetLayer(ENTRY, "entry", c, co, 2, h, w, oh, ow, act=relu6, bias=bias(co),
                           weights=uniform((co, c, 3, 3), 9 * c)))
    c, h, w = co, oh, ow
    base = [64, 128, 128, 256, 256, 512, 512, 512, 512, 512, 512, 1024, 1024]
    for i in range(1, 14):
        s = 2 if i in (2, 4, 6, 12) else 1
        oh, ow = same_pad_out(h, s), same_pad_out(w, s)
        layers.append(NetLayer(DEPTHWISE, f"dw{i}", c, c, s, h, w, oh, ow, act=relu6, bias=bias(c),
                               weights=uniform((c, 3, 3), 9)))
        h, w = oh, ow
        co = round_channels(base[i - 1], width)
        bh = block_h_after if i >= block_start else 1
        L = NetLayer(POINTWISE, f"pw{i}", c, co, 1, h, w, h, w, act=relu6)
        if sparsity > 0.0:
            rows_p = (co + bh - 1) // bh * bh
            d = make_layer_data(WLayer(f"pw{i}", c, rows_p, h, w, relu6, 0.0, 6.0, sparsity, bh), 1,
                                int(rng.integers(1 << 31)), act=False)
            L.sparse, L.sparsity, L.block_h = True, float(sparsity), bh
            L.weights = d.weights
            L.bias = d.bias[:co].copy()
        else:
            L.weights = uniform((co, c), c)
            L.bias = bias(co)
        layers.append(L)
        c = co
    layers.append(NetLayer(POOL, "pool", c, c, 1, h, w, 1, 1))
    layers.append(NetLayer(FC, "fc", c, num_classes, 1, 1, 1, 1, 1, bias=bias(num_classes),
                           weights=uniform((num_classes, c), c)))
    return Network("mbv1", width, input_hw, input_hw, 3, num_classes, float(sparsity), block_start,
                   block_h_after, layers)


def serialize(net: Network) -> bytes:
    """serialize_model (model_io.cpp:146-227)."""
    out = bytearray(b"SPCV")

    def u8(v):
        out.extend(struct.pack("<B", v))

    def u32(v):
        out.extend(struct.pack("<I", v & 0xFFFFFFFF))

    def f32(v):
        out.extend(struct.pack("<f", v))

    def f64(v):
        out.extend(struct.pack("<d", v))

    def s(v):
        b = v.encode()
        u32(len(b))
        out.extend(b)

    def f32s(a):
        a = np.ascontiguousarray(a, dtype="<f4").reshape(-1)
        u32(a.size)
        out.extend(a.tobytes())

    def u32s(a):
        a = np.ascontiguousarray(a, dtype="<u4").reshape(-1)
        u32(a.size)
        out.extend(a.tobytes())

    out.extend(struct.pack("<H", 1))
    s(net.name)
    u32(int(math.floor(net.width * 1000.0 + 0.5)))
    for v in (net.input_h, net.input_w, net.input_c, net.num_classes):
        u32(v)
    f64(net.plan_sparsity)
    u32(net.block_start)
    u32(net.block_h_after)
    u32(len(net.layers))
    for L in net.layers:
        u8(L.kind)
        s(L.name)
        for v in (L.cin, L.cout, L.stride, L.in_h, L.in_w, L.out_h, L.out_w):
            u32(v)
        u8(1 if L.sparse else 0)
        f64(L.sparsity)
        u32(L.block_h)
        clamp = L.act[0] == "clamp"
        u8(1 if clamp else 0)
        f32(L.act[1] if clamp else 0.0)
        f32(L.act[2] if clamp else 0.0)
        u32(L.residual_src)
        f32s(L.bias)
        if L.kind == POOL:
            u8(NONE_STORAGE)
        elif L.kind == ENTRY:
            u8(CONV)
            for v in L.weights.shape:
                u32(v)
            f32s(L.weights)
        elif L.kind == DEPTHWISE:
            u8(DW)
            u32(L.weights.shape[0])
            f32s(L.weights)
        elif isinstance(L.weights, BcsrMatrix):
            m = L.weights
            u8(BCSR)
            u32(m.rows)
            u32(m.cols)
            u32(m.block_h)
            u32s(m.row_ptr)
            u32s(m.col_idx)
            f32s(m.values)
        else:
            u8(DENSE)
            u32(L.weights.shape[0])
            u32(L.weights.shape[1])
            f32s(L.weights)
    u32(zlib.crc32(bytes(out)) & 0xFFFFFFFF)
    return bytes(out)


def densify(net: Network) -> Network:
    """densify (netdef.cpp:417-431): every sparse 1x1 layer stored dense (the
    logical rows of the decoded matrix), for the effective-vs-dense comparison."""
    from .bcsr import decode_bcsr

    layers = []
    for L in net.layers:
        if isinstance(L.weights, BcsrMatrix):
            d = decode_bcsr(L.weights)[: L.cout]
            L = NetLayer(**{**L.__dict__, "weights": np.ascontiguousarray(d), "sparse": False,
                            "sparsity": 0.0, "block_h": 1})
        layers.append(L)
    return Network(**{**net.__dict__, "layers": layers})


__all__ = ["Network", "NetLayer", "build_mbv1", "serialize", "densify", "round_channels", "encode_bcsr"]
