"""Generate tests/golden/*.npz from the UNMODIFIED reference library.

Run in the dev container (where /root/reference exists and oracle/_ref was
built by `make -C oracle`):

    python tests/golden/make_golden.py

The fixtures hold inputs and the reference's own outputs (spcv::spmm_into via
oracle/_ref/libspcv_ref.so, and spcv::matmul_reference on the decoded
weights), so the oracle and the CUDA path can be pinned on machines where the
reference is absent (the GPU box). Inputs use the reference tests' own recipes
(tests/refcases.py) plus small BASELINE-shaped cases.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

from oracle import Oracle, Ref  # noqa: E402
from refcases import Mt, masked_case, random_bias, random_chw, random_matrix  # noqa: E402

from paper_1911_09723_b200 import encode_bcsr  # noqa: E402
from paper_1911_09723_b200.workloads import Layer, make_layer_data  # noqa: E402

import hashlib  # noqa: E402
import json  # noqa: E402
from dataclasses import asdict  # noqa: E402

RELU6 = ("clamp", 0.0, 6.0)
RELU = ("clamp", 0.0, float("inf"))
NONE = ("none", 0.0, 0.0)


DIGEST_CASES = [
    ("c2_pw13_b2", Layer("pw13", 1024, 1024, 7, 7, ("clamp", 0.0, 6.0), 0.0, 6.0, 0.9), 2, 2),
    ("c2_pw1_b1", Layer("pw1", 32, 64, 112, 112, ("clamp", 0.0, 6.0), 0.0, 6.0, 0.9), 1, 6),
    ("c3_bh4_s90_b2", Layer("c3", 512, 512, 14, 14, ("clamp", 0.0, float("inf")), -1.0, 1.0, 0.9, 4), 2, 3),
    ("c3_bh2_s70_b1", Layer("c3", 512, 512, 14, 14, ("clamp", 0.0, float("inf")), -1.0, 1.0, 0.7, 2), 1, 7),
    ("c4_project_b2", Layer("p", 960, 160, 7, 7, ("none", 0.0, 0.0), 0.0, 6.0, 0.85), 2, 4),
    ("c4_expand_b1", Layer("e", 24, 144, 56, 56, ("clamp", 0.0, 6.0), -1.0, 1.0, 0.85), 1, 8),
    ("c5_s90_b2", Layer("c5", 1024, 1024, 7, 7, ("clamp", 0.0, float("inf")), -1.0, 1.0, 0.9, 1, True), 2, 5),
]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def layer_to_dict(layer) -> dict:
    d = asdict(layer)
    d["act"] = list(d["act"])
    return d


def act_code(a):
    return {"none": 0, "clamp": 1}[a[0]], a[1], a[2]


def main():
    orc, ref = Oracle(), Ref()
    cases = {}

    def add(name, m, act, bias, fused, dense):
        B, K, H, W = act.shape
        rc, out = ref.spmm(m, act, bias, fused, H, W)
        assert rc == 0, (name, rc)
        dref = np.stack([ref.matmul_reference(dense, act[i].reshape(K, -1), bias, fused, H, W)
                         for i in range(B)])
        # The reference kernel is bit-exact against its own dense oracle on
        # finite inputs; keep one copy of the expected bytes.
        assert np.array_equal(out.reshape(-1).view(np.uint32), dref.reshape(-1).view(np.uint32)), name
        k, lo, hi = act_code(fused)
        cases[name] = dict(rows=m.rows, cols=m.cols, block_h=m.block_h, row_ptr=m.row_ptr,
                           col_idx=m.col_idx, values=m.values, act=act,
                           bias=np.zeros(0, np.float32) if bias is None else bias,
                           fused=np.array([k, lo, hi], np.float64),
                           expected=out.reshape(B, m.rows, H, W))

    # test_kernels.cpp:55-68 identity, bh 1/2/4
    rng = Mt(3)
    act = random_chw(8, 5, 7, rng)[None]
    eye = np.eye(8, dtype=np.float32)
    for bh in (1, 2, 4):
        add(f"identity_bh{bh}", encode_bcsr(eye, bh), act, np.zeros(8, np.float32), NONE, eye)

    # test_kernels.cpp:70-89 hand case -> {3, 6, 0, 0}
    w = np.zeros((2, 3), np.float32)
    w[0, 1], w[1, 1] = 2.0, -3.0
    act = np.array([9, 9, 1, 4, 9, 9], np.float32).reshape(1, 3, 1, 2)
    add("hand_case", encode_bcsr(w, 2), act, np.array([1.0, -1.0], np.float32), RELU6, w)

    # test_kernels.cpp:91-109 every variant: 64x64 @14x14, 90%, bh 1/2/4 (first m_width pass)
    rng = Mt(17)
    for bh in (1, 2, 4):
        dense, m = masked_case(64, 64, 0.9, bh, rng, orc)
        act = random_chw(64, 14, 14, rng)[None]
        bias = random_bias(64, rng)
        add(f"variant_64x64_bh{bh}", m, act, bias, RELU6, dense)

    # test_kernels.cpp:111-126 strip remainders S in {1,3,5,7,13,197}, 16x12, 70%, 2x1
    rng = Mt(19)
    for S in (1, 3, 5, 7, 13, 197):
        dense, m = masked_case(16, 12, 0.7, 2, rng, orc)
        act = random_chw(12, 1, S, rng)[None]
        bias = random_bias(16, rng)
        add(f"remainder_S{S}", m, act, bias, NONE, dense)

    # test_kernels.cpp:128-149 variants agree: 32x24, 80%, 4x1, 3x13
    rng = Mt(23)
    dense, m = masked_case(32, 24, 0.8, 4, rng, orc)
    act = random_chw(24, 3, 13, rng)[None]
    bias = random_bias(32, rng)
    add("agree_32x24_bh4", m, act, bias, RELU6, dense)

    # test_kernels.cpp:232-239 fully dense matrix through spmm
    rng = Mt(43)
    dense = random_matrix(16, 16, rng)
    act = random_chw(16, 6, 6, rng)[None]
    bias = random_bias(16, rng)
    add("fully_dense_16", encode_bcsr(dense, 1), act, bias, NONE, dense)

    # empty block rows + null bias
    rng = Mt(7)
    dense = random_matrix(12, 10, rng)
    dense[4:8, :] = 0.0
    act = random_chw(10, 3, 3, rng)[None]
    add("empty_rows_nobias", encode_bcsr(dense, 2), act, None, RELU6, dense)

    # Config 1 in full (it is small): BASELINE.json configs[0].
    d = make_layer_data(Layer("c1", 128, 128, 28, 28, RELU, -1.0, 1.0, 0.8), 1, 1)
    add("c1", d.weights, d.act, d.bias, RELU, d.dense)

    flat = {}
    for name, c in cases.items():
        for k, v in c.items():
            flat[f"{name}/{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(HERE, "spmm_cases.npz"), **flat)

    # generate_mask known answers (test_sparse.cpp:73-104) and a few seeds
    masks = {}
    for (r, c, s, ob, ib, seed) in [(8, 8, 0.5, 2, 1, 1234), (8, 8, 0.5, 2, 1, 1235),
                                    (10, 1, 0.25, 1, 1, 5), (4, 4, 0.0, 1, 1, 5),
                                    (4, 4, 0.999, 1, 1, 5), (16, 12, 0.7, 4, 2, 77),
                                    (64, 64, 0.9, 1, 1, 42), (64, 32, 0.8, 4, 1, 9)]:
        rc, keep = ref.generate_mask(r, c, s, ob, ib, seed)
        assert rc == 0
        masks[f"{r}x{c}_s{s}_b{ob}x{ib}_seed{seed}"] = np.packbits(keep.reshape(-1))
    np.savez_compressed(os.path.join(HERE, "masks.npz"), **masks)

    # BASELINE-shaped cases too large to commit as arrays: regeneration
    # parameters (workloads.make_layer_data, seeded) + SHA-256 digests of the
    # generated inputs and of the reference's output bytes.
    digests = {}
    for name, layer, images, seed in DIGEST_CASES:
        d = make_layer_data(layer, images, seed)
        B, K, H, W = d.act.shape
        rc, out = ref.spmm(d.weights, d.act, d.bias, layer.act, H, W)
        assert rc == 0, name
        digests[name] = dict(layer=layer_to_dict(layer), images=images, seed=seed,
                             sha_row_ptr=sha(d.weights.row_ptr), sha_col_idx=sha(d.weights.col_idx),
                             sha_values=sha(d.weights.values), sha_act=sha(d.act), sha_bias=sha(d.bias),
                             sha_expected=sha(out))
    with open(os.path.join(HERE, "digests.json"), "w") as f:
        json.dump(digests, f, indent=1, sort_keys=True)
    print(f"wrote {len(cases)} spmm cases, {len(masks)} masks, {len(digests)} digest cases")


if __name__ == "__main__":
    main()
