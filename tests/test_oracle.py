"""Pin the CPU oracle (oracle/spcv_oracle.c) before trusting it.

1. Against the committed golden fixtures (reference outputs) — runs anywhere.
2. Against the compiled reference itself (oracle/_ref) on the reference tests'
   own inputs — runs where the reference library was built.
Bit-exact throughout (the reference path is exact on finite
inputs when built without FMA contraction).
"""
import json
import os

import numpy as np
import pytest

from refcases import Mt, masked_case, random_bias, random_chw, random_matrix

from paper_1911_09723_b200 import BcsrMatrix, decode_bcsr, encode_bcsr
from paper_1911_09723_b200.workloads import Layer, make_layer_data

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).reshape(-1).view(np.uint32)


def load_cases():
    z = np.load(os.path.join(GOLD, "spmm_cases.npz"))
    cases = {}
    for k in z.files:
        name, field = k.split("/")
        cases.setdefault(name, {})[field] = z[k]
    return cases


CASES = load_cases()


def case_matrix(c):
    return BcsrMatrix(int(c["rows"]), int(c["cols"]), int(c["block_h"]), c["row_ptr"], c["col_idx"],
                      c["values"])


def fused_of(c):
    k, lo, hi = c["fused"]
    return ("none", 0.0, 0.0) if k == 0 else ("clamp", float(lo), float(hi))


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_spmm_matches_golden(oracle, name):
    c = CASES[name]
    m = case_matrix(c)
    bias = c["bias"] if c["bias"].size else None
    got = oracle.spmm(m, c["act"], bias, fused_of(c))
    assert np.array_equal(bits(got), bits(c["expected"]))


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matmul_reference_matches_golden(oracle, name):
    c = CASES[name]
    m = case_matrix(c)
    dense = decode_bcsr(m)
    bias = c["bias"] if c["bias"].size else None
    B, K = c["act"].shape[:2]
    for i in range(B):
        got = oracle.matmul_reference(dense, c["act"][i].reshape(K, -1), bias, fused_of(c))
        assert np.array_equal(bits(got), bits(c["expected"][i]))


def test_hand_case_known_answer():
    # test_kernels.cpp:70-89: {3, 6, 0, 0}
    assert CASES["hand_case"]["expected"].reshape(-1).tolist() == [3.0, 6.0, 0.0, 0.0]


def test_identity_known_answer():
    # test_kernels.cpp:55-68: identity weights return the input exactly
    for bh in (1, 2, 4):
        c = CASES[f"identity_bh{bh}"]
        assert np.array_equal(bits(c["expected"]), bits(c["act"]))


def test_golden_masks(oracle):
    z = np.load(os.path.join(GOLD, "masks.npz"))
    pops = {"8x8_s0.5_b2x1_seed1234": 32, "10x1_s0.25_b1x1_seed5": 7, "4x4_s0.0_b1x1_seed5": 16,
            "4x4_s0.999_b1x1_seed5": 0}
    for key in z.files:
        dims, s, b, seed = key.split("_")
        r, cc = map(int, dims.split("x"))
        ob, ib = map(int, b[1:].split("x"))
        rc, keep = oracle.generate_mask(r, cc, float(s[1:]), ob, ib, int(seed[4:]))
        assert rc == 0
        assert np.array_equal(np.packbits(keep.reshape(-1)), z[key]), key
        if key in pops:  # test_sparse.cpp:73-104 popcounts
            assert int(keep.sum()) == pops[key]


def sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


DIGESTS = json.load(open(os.path.join(GOLD, "digests.json")))


def digest_case(name):
    d = DIGESTS[name]
    L = dict(d["layer"])
    L["act"] = tuple(L["act"])
    layer = Layer(**L)
    data = make_layer_data(layer, d["images"], d["seed"])
    # the seeded generator must reproduce the exact bytes the reference saw
    assert sha(data.weights.row_ptr) == d["sha_row_ptr"]
    assert sha(data.weights.col_idx) == d["sha_col_idx"]
    assert sha(data.weights.values) == d["sha_values"]
    assert sha(data.act) == d["sha_act"]
    assert sha(data.bias) == d["sha_bias"]
    return layer, data, d["sha_expected"]


@pytest.mark.parametrize("name", sorted(DIGESTS))
def test_oracle_matches_golden_digests(oracle, name):
    layer, data, want = digest_case(name)
    got = oracle.spmm(data.weights, data.act, data.bias, layer.act, nthreads=4)
    assert sha(got) == want


# ----------------------------------------------------- against oracle/_ref
def test_oracle_equals_reference_on_reference_test_inputs(oracle, ref):
    """test_kernels.cpp:91-126 inputs, reference spmm vs oracle, every bh/S."""
    rng = Mt(17)
    for bh in (1, 2, 4):
        dense, m = masked_case(64, 64, 0.9, bh, rng, oracle)
        act = random_chw(64, 14, 14, rng)[None]
        bias = random_bias(64, rng)
        for cfg_m in (4, 8, 16):
            for tier in (0, 2):
                rc, r = ref.spmm(m, act, bias, ("clamp", 0.0, 6.0), cfg_m=cfg_m, tier=tier)
                assert rc == 0
                o = oracle.spmm(m, act, bias, ("clamp", 0.0, 6.0))
                assert np.array_equal(bits(r), bits(o))
    rng = Mt(19)
    for S in (1, 3, 5, 7, 13, 197):
        dense, m = masked_case(16, 12, 0.7, 2, rng, oracle)
        act = random_chw(12, 1, S, rng)[None]
        bias = random_bias(16, rng)
        rc, r = ref.spmm(m, act, bias, ("none", 0, 0))
        assert rc == 0
        assert np.array_equal(bits(r), bits(oracle.spmm(m, act, bias, ("none", 0, 0))))


def test_oracle_equals_reference_acceptance_sample(oracle, ref):
    """A slice of acceptance C1 (acceptance.cpp:89-139): MBv1/MBv2 shapes x
    sparsity x block height, reference spmm == oracle bit-for-bit."""
    rng = np.random.default_rng(101)
    shapes = [(64, 32, 14, 14), (128, 128, 7, 7), (144, 24, 14, 14), (160, 960, 7, 7),
              (1024, 512, 7, 7), (96, 16, 10, 10)]
    for (cout, cin, h, w) in shapes:
        act = rng.uniform(-1, 1, (1, cin, h, w)).astype(np.float32)
        bias = rng.uniform(-1, 1, cout).astype(np.float32)
        for s in (0.7, 0.9, 0.95):
            for bh in (1, 2, 4):
                dense = rng.uniform(-1, 1, (cout, cin)).astype(np.float32)
                rc, keep = oracle.generate_mask(cout, cin, s, bh, 1, int(rng.integers(1 << 31)))
                dense[~keep] = 0
                m = encode_bcsr(dense, bh)
                rc, r = ref.spmm(m, act, bias, ("clamp", 0.0, 6.0))
                assert rc == 0
                o = oracle.spmm(m, act, bias, ("clamp", 0.0, 6.0))
                assert np.array_equal(bits(r), bits(o))
                dref = ref.matmul_reference(dense, act[0].reshape(cin, -1), bias, ("clamp", 0.0, 6.0), h, w)
                assert np.array_equal(bits(dref), bits(o))


def test_oracle_masks_equal_reference(oracle, ref):
    for args in [(8, 8, 0.5, 2, 1, 1234), (37, 29, 0.63, 1, 1, 99), (64, 64, 0.9, 4, 1, 7),
                 (16, 12, 0.7, 2, 2, 77), (128, 128, 0.8, 1, 1, 2024)]:
        rc1, a = oracle.generate_mask(*args)
        rc2, b = ref.generate_mask(*args)
        assert rc1 == rc2 == 0
        assert np.array_equal(a, b)
    for bad in [(6, 4, 0.5, 4, 1, 1), (8, 3, 0.5, 1, 2, 1), (8, 4, 1.5, 1, 1, 1)]:
        assert oracle.generate_mask(*bad)[0] == ref.generate_mask(*bad)[0] != 0


def test_oracle_encode_validate_equal_reference(oracle, ref):
    rng = Mt(99)
    for bh in (1, 2, 4):
        for _ in range(15):
            rows = bh * (1 + int(rng() % 12))
            cols = 1 + int(rng() % 40)
            s = (rng() % 100) / 100.0
            w = random_matrix(rows, cols, rng)
            rc, keep = oracle.generate_mask(rows, cols, s, bh, 1, rng())
            w[~keep] = 0
            rc1, a = oracle.encode_bcsr(w, bh)
            rc2, b = ref.encode_bcsr(w, bh)
            assert rc1 == rc2 == 0
            for x, y in zip(a, b):
                assert np.array_equal(x, y)
            assert oracle.validate(rows, cols, bh, *a) == 0
    # validate rejections (test_sparse.cpp:137-187) agree in code
    w = np.zeros((4, 4), np.float32)
    w[0, 1], w[2, 3] = 1, 2
    _, (rp, ci, va) = oracle.encode_bcsr(w, 2)
    bad = [
        (5, 4, 2, rp, ci, va),
        (4, 4, 2, np.r_[1, rp[1:]], ci, va),
        (4, 4, 2, np.r_[rp[0], 3, rp[2:]], ci, va),
        (4, 4, 2, np.r_[rp[:-1], 1], ci, va),
        (4, 4, 2, rp, np.r_[99, ci[1:]], va),
        (4, 4, 2, rp, ci, np.r_[va, 0]),
        (4, 4, 3, rp, ci, va),
        (2, 4, 1, np.array([0, 2, 2]), np.array([2, 1]), np.array([1.0, 2.0])),
    ]
    for args in bad:
        assert oracle.validate(*args) == ref.validate(*args) == 3, args
