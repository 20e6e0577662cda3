"""Seeded synthetic workloads for the five BASELINE.json configs.

The reference measures no public dataset on this path; these
generators produce inputs with the configs' shapes and value distributions.
They are input preparation only (host-side, untimed), shared by the GPU path,
the CPU checkers and the bench, so every side sees identical bytes.

Layer shapes follow the reference network builders:
  MobileNet-v1 pointwise stack   /root/reference/proj/src/netdef.cpp:202-218
  MobileNet-v2 1x1 convs         /root/reference/proj/src/netdef.cpp:168-198,220-225
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .bcsr import Activation, BcsrMatrix, encode_bcsr  # pure numpy: no CUDA library load

RELU = ("clamp", 0.0, float("inf"))
RELU6 = ("clamp", 0.0, 6.0)
NONE = ("none", 0.0, 0.0)


def activation_of(spec) -> Activation:
    return Activation.none() if spec[0] == "none" else Activation.clamp(spec[1], spec[2])


@dataclass(frozen=True)
class Layer:
    name: str
    cin: int     # K
    cout: int    # M
    h: int
    w: int
    act: tuple = RELU6
    in_lo: float = 0.0   # activation input distribution U[in_lo, in_hi]
    in_hi: float = 6.0
    sparsity: float = 0.9
    block_h: int = 1
    skew: bool = False   # per-row Beta(2,8) densities (config 5)
    net_index: int = -1  # index in the reference network's layer list (netdef.cpp)

    @property
    def spatial(self) -> int:
        return self.h * self.w


def mbv1_pointwise(sparsity: float = 0.9) -> list[Layer]:
    """MBv1-1.0 @224: the 13 pointwise layers (netdef.cpp:205-211)."""
    shapes = [(32, 64, 112), (64, 128, 56), (128, 128, 56), (128, 256, 28), (256, 256, 28),
              (256, 512, 14)] + [(512, 512, 14)] * 5 + [(512, 1024, 7), (1024, 1024, 7)]
    # layer list: entry conv (0), then dw_i (2i-1), pw_i (2i) for i = 1..13
    return [Layer(f"pw{i + 1}", k, m, hw, hw, RELU6, 0.0, 6.0, sparsity, net_index=2 * (i + 1))
            for i, (k, m, hw) in enumerate(shapes)]


def mbv2_pointwise(sparsity: float = 0.85) -> list[Layer]:
    """MBv2-1.0 @224 1x1 convs in network order (netdef.cpp:168-198,220-225).
    Expand (ReLU6) inputs follow linear projects/residual sums -> U[-1,1];
    project (no clamp) inputs follow the ReLU6 depthwise -> U[0,6]."""
    stages = [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1),
              (6, 160, 3, 2), (6, 320, 1, 1)]
    layers: list[Layer] = []
    c, hw, blk, idx = 32, 112, 0, 1  # layer 0 is the entry conv (netdef.cpp:176)
    for t, cout, n, s in stages:
        for i in range(n):
            blk += 1
            stride = s if i == 0 else 1
            if t != 1:
                layers.append(Layer(f"b{blk}_expand", c, c * t, hw, hw, RELU6, -1.0, 1.0, sparsity,
                                    net_index=idx))
                idx += 1
            hidden = c * t
            hw = (hw + stride - 1) // stride
            idx += 1  # depthwise
            layers.append(Layer(f"b{blk}_project", hidden, cout, hw, hw, NONE, 0.0, 6.0, sparsity,
                                net_index=idx))
            idx += 1
            c = cout
    layers.append(Layer("head", c, 1280, hw, hw, RELU6, -1.0, 1.0, sparsity, net_index=idx))
    return layers


def c1_layer() -> Layer:
    return Layer("c1", 128, 128, 28, 28, RELU, -1.0, 1.0, 0.8)


def c3_layer(sparsity: float = 0.9, block_h: int = 4) -> Layer:
    return Layer(f"c3_s{int(sparsity * 100)}_b{block_h}", 512, 512, 14, 14, RELU, -1.0, 1.0,
                 sparsity, block_h)


def c5_layer(sparsity: float = 0.9) -> Layer:
    return Layer(f"c5_s{int(round(sparsity * 100))}", 1024, 1024, 7, 7, RELU, -1.0, 1.0,
                 sparsity, 1, skew=True)


CONFIGS = {
    "c1": dict(layers=lambda: [c1_layer()], images=1),
    "c2-b1": dict(layers=lambda: mbv1_pointwise(0.9), images=1),
    "c2-b256": dict(layers=lambda: mbv1_pointwise(0.9), images=256),
    "c3": dict(layers=lambda: [c3_layer(s, b) for b in (4, 2, 1) for s in (0.7, 0.8, 0.9, 0.95)],
               images=64),
    "c4": dict(layers=lambda: mbv2_pointwise(0.85), images=128),
    "c5": dict(layers=lambda: [c5_layer(s) for s in (0.7, 0.8, 0.9, 0.95, 0.98)], images=1024),
}


# ------------------------------------------------------------- generators
def uniform_mask(rng: np.random.Generator, rows: int, cols: int, sparsity: float,
                 block_h: int) -> np.ndarray:
    """Zero round(tiles*sparsity) whole block_h x 1 tiles chosen uniformly
    (the reference's generate_mask contract, sparse.cpp:63-98)."""
    trows = rows // block_h
    tiles = trows * cols
    zeroed = int(np.floor(tiles * sparsity + 0.5))
    keep_t = np.ones(tiles, dtype=bool)
    keep_t[rng.permutation(tiles)[:zeroed]] = False
    return np.repeat(keep_t.reshape(trows, cols), block_h, axis=0)


def skewed_mask(rng: np.random.Generator, rows: int, cols: int, sparsity: float) -> np.ndarray:
    """Config 5: per-row density Beta(2,8) rescaled to mean (1-sparsity),
    clipped to [0,1]; nnz_r = round(d_r*cols) distinct columns per row."""
    target = 1.0 - sparsity
    d = np.clip(rng.beta(2.0, 8.0, size=rows) * (target / 0.2), 0.0, 1.0)
    nnz = np.rint(d * cols).astype(np.int64)
    keep = np.zeros((rows, cols), dtype=bool)
    for r in range(rows):
        keep[r, rng.choice(cols, size=nnz[r], replace=False)] = True
    return keep


@dataclass
class LayerData:
    layer: Layer
    images: int
    weights: BcsrMatrix
    dense: np.ndarray         # masked dense weights (rows x cols)
    bias: np.ndarray          # [M]
    act: np.ndarray           # [images][K][H][W]

    @property
    def nnz(self) -> int:
        return self.weights.nnz_values()

    def flops(self) -> float:
        """2*nnz*N with N = images*H*W (reference 'achieved', bench.cpp:211)."""
        return 2.0 * self.nnz * self.images * self.layer.spatial

    def alg_bytes(self) -> float:
        """act in + out + values + col_idx + row_ptr + bias (reference widths)."""
        L = self.layer
        N = self.images * L.spatial
        nb = self.weights.nnz_blocks()
        return 4.0 * (L.cin * N + L.cout * N + self.nnz + nb + (L.cout // L.block_h + 1) + L.cout)


def make_layer_data(layer: Layer, images: int, seed: int, act: bool = True) -> LayerData:
    rng = np.random.default_rng(seed)
    if layer.skew:
        keep = skewed_mask(rng, layer.cout, layer.cin, layer.sparsity)
    else:
        keep = uniform_mask(rng, layer.cout, layer.cin, layer.sparsity, layer.block_h)
    w = (rng.standard_normal((layer.cout, layer.cin), dtype=np.float32) * np.float32(0.1))
    w[~keep] = 0.0
    bias = rng.standard_normal(layer.cout, dtype=np.float32) * np.float32(0.1)
    a = None
    if act:
        a = rng.random((images, layer.cin, layer.h, layer.w), dtype=np.float32)
        a *= np.float32(layer.in_hi - layer.in_lo)
        a += np.float32(layer.in_lo)
    return LayerData(layer, images, encode_bcsr(w, layer.block_h), w, bias, a)
