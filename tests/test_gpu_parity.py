"""Parity of the CUDA path (through the C-ABI) against the oracle and the
reference's golden outputs. Needs a B200 (marked gpu).

Bar (BASELINE.json north_star):
  * strict mode (default): bit-exact against the reference / oracle;
  * fast (FFMA) mode: |gpu - ref| <= 1e-5 * max(1, nnz_r/64) * A_ij with
    A_ij = |bias_r| + sum_k |w_rk x_kj| computed in fp64;
  * pack/unpack of the weight format: exact, byte for byte.
"""
import json
import os

import numpy as np
import pytest

from refcases import Mt, masked_case, random_bias, random_chw, random_matrix

import paper_1911_09723_b200 as sp
from paper_1911_09723_b200.workloads import (CONFIGS, Layer, c5_layer, make_layer_data,
                                             mbv1_pointwise, mbv2_pointwise)

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RELU6 = sp.Activation.relu6()
NONE = sp.Activation.none()


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).reshape(-1).view(np.uint32)


def act_of(spec):
    if isinstance(spec, sp.Activation):
        return spec
    return sp.Activation.none() if spec[0] == "none" else sp.Activation.clamp(spec[1], spec[2])


def run_device(m, act, bias, fused, strict=True, dw=None, stream=None):
    """act [B][K][H][W] numpy -> out numpy via spcv_cu_spmm_into on device."""
    import torch

    act = np.ascontiguousarray(act, np.float32)
    if act.ndim == 3:
        act = act[None]
    B, K, H, W = act.shape
    dw = dw or sp.DeviceBcsr(m)
    a = torch.from_numpy(act).cuda()
    o = torch.full((B, dw.rows, H, W), float("nan"), device="cuda")
    b = None if bias is None or len(bias) == 0 else torch.from_numpy(np.asarray(bias, np.float32)).cuda()
    sp.spmm_batched_into(dw, a, b, act_of(fused), o,
                         sp.MicrokernelConfig(n=dw.block_h, strict=strict), stream=stream)
    torch.cuda.synchronize()
    return o.cpu().numpy()


def use_kernel(monkeypatch, kernel):
    """Pack-time knobs that pick one kernel: "jit" (weight-specialised, where it
    serves the matrix), "tile" (the shared-memory tile kernel) or "small" (the
    few-column kernel)."""
    monkeypatch.setenv("SPCV_JIT", "1" if kernel == "jit" else "0")
    monkeypatch.setenv("SPCV_SMALL", "2" if kernel == "small" else "0")


KERNELS = ["jit", "tile", "small"]


def load_cases():
    z = np.load(os.path.join(GOLD, "spmm_cases.npz"))
    cases = {}
    for k in z.files:
        name, field = k.split("/")
        cases.setdefault(name, {})[field] = z[k]
    return cases


CASES = load_cases()


def case_matrix(c):
    return sp.BcsrMatrix(int(c["rows"]), int(c["cols"]), int(c["block_h"]), c["row_ptr"],
                         c["col_idx"], c["values"])


def case_fused(c):
    k, lo, hi = c["fused"]
    return NONE if k == 0 else sp.Activation.clamp(float(lo), float(hi))


# ------------------------------------------------------------ golden vectors
@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_device_path_bit_exact(name):
    c = CASES[name]
    got = run_device(case_matrix(c), c["act"], c["bias"] if c["bias"].size else None, case_fused(c))
    assert np.array_equal(bits(got), bits(c["expected"]))


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_host_path_bit_exact(name):
    """The reference-facing call shape: spmm with host tensors (per image)."""
    c = CASES[name]
    m = case_matrix(c)
    B, K, H, W = c["act"].shape
    for i in range(B):
        act = sp.Tensor(K, H, W, data=c["act"][i])
        out = sp.spmm(m, act, c["bias"] if c["bias"].size else None, case_fused(c),
                      sp.MicrokernelConfig(n=m.block_h))
        assert np.array_equal(bits(out.data), bits(c["expected"][i]))


def sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


DIGESTS = json.load(open(os.path.join(GOLD, "digests.json")))


@pytest.mark.parametrize("name", sorted(DIGESTS))
def test_golden_digest_cases_bit_exact(name):
    d = DIGESTS[name]
    L = dict(d["layer"])
    L["act"] = tuple(L["act"])
    layer = Layer(**L)
    data = make_layer_data(layer, d["images"], d["seed"])
    assert sha(data.act) == d["sha_act"] and sha(data.weights.values) == d["sha_values"]
    got = run_device(data.weights, data.act, data.bias, layer.act)
    assert sha(got.reshape(d["images"], layer.cout, -1)) == d["sha_expected"]


# ------------------------------------- reference hot-path tests, re-expressed
def test_identity_returns_input():
    # test_kernels.cpp:55-68
    rng = Mt(3)
    act = random_chw(8, 5, 7, rng)
    for bh in (1, 2, 4):
        m = sp.encode_bcsr(np.eye(8, dtype=np.float32), bh)
        out = sp.spmm(m, sp.Tensor(8, 5, 7, data=act), np.zeros(8, np.float32), NONE,
                      sp.MicrokernelConfig(n=bh))
        assert np.array_equal(bits(out.data), bits(act))


def test_hand_case():
    # test_kernels.cpp:70-89
    w = np.zeros((2, 3), np.float32)
    w[0, 1], w[1, 1] = 2.0, -3.0
    m = sp.encode_bcsr(w, 2)
    assert m.nnz_blocks() == 1
    act = sp.Tensor(3, 1, 2, data=[9, 9, 1, 4, 9, 9])
    out = sp.spmm(m, act, np.array([1.0, -1.0], np.float32), RELU6, sp.MicrokernelConfig(n=2))
    assert out.data.tolist() == [3.0, 6.0, 0.0, 0.0]


def test_every_variant_matches_oracle(oracle):
    # test_kernels.cpp:91-109 (tolerance 1e-5 there; bit-exact here)
    rng = Mt(17)
    for m_width in (4, 8, 16):
        for bh in (1, 2, 4):
            dense, m = masked_case(64, 64, 0.9, bh, rng, oracle)
            act = random_chw(64, 14, 14, rng)
            bias = random_bias(64, rng)
            want = oracle.matmul_reference(dense, act.reshape(64, -1), bias, RELU6)
            for tier in (sp.Tier.Scalar, sp.Tier.Auto):
                cfg = sp.MicrokernelConfig(m=m_width, n=bh, tier=tier)
                got = sp.spmm(m, sp.Tensor(64, 14, 14, data=act), bias, RELU6, cfg)
                assert np.array_equal(bits(got.data), bits(want))


def test_strip_remainders(oracle):
    # test_kernels.cpp:111-126: spatial extents not multiple of any strip width
    rng = Mt(19)
    for S in (1, 3, 5, 7, 13, 197):
        dense, m = masked_case(16, 12, 0.7, 2, rng, oracle)
        act = random_chw(12, 1, S, rng)
        bias = random_bias(16, rng)
        want = oracle.matmul_reference(dense, act.reshape(12, -1), bias, None)
        for m_width in (4, 8, 16):
            got = sp.spmm(m, sp.Tensor(12, 1, S, data=act), bias, NONE,
                          sp.MicrokernelConfig(m=m_width, n=2))
            assert np.array_equal(bits(got.data), bits(want))


def test_variants_tiers_prefetch_agree():
    # test_kernels.cpp:128-163
    rng = Mt(23)
    from oracle import Oracle

    dense, m = masked_case(32, 24, 0.8, 4, rng, Oracle())
    act = sp.Tensor(24, 3, 13, data=random_chw(24, 3, 13, rng))
    bias = random_bias(32, rng)
    first = None
    for tier in (sp.Tier.Scalar, sp.Tier.Vector, sp.Tier.Auto):
        for m_width in (4, 8, 16):
            for pf in (True, False):
                cfg = sp.MicrokernelConfig(m=m_width, n=4, tier=tier, prefetch=pf)
                out = sp.spmm(m, act, bias, RELU6, cfg).data
                if first is None:
                    first = out
                assert np.array_equal(bits(out), bits(first))


def test_fused_clamp_equals_unfused_then_clamped(oracle):
    # test_kernels.cpp:165-175
    rng = Mt(31)
    dense, m = masked_case(16, 16, 0.6, 1, rng, oracle)
    act = sp.Tensor(16, 4, 5, data=random_chw(16, 4, 5, rng))
    bias = random_bias(16, rng)
    fused = sp.spmm(m, act, bias, RELU6).data
    plain = sp.spmm(m, act, bias, NONE).data
    clamped = np.where(plain < 0, 0, np.where(plain > 6, 6, plain)).astype(np.float32)
    assert np.array_equal(bits(fused), bits(clamped))


def test_spmm_validates_inputs():
    # test_kernels.cpp:177-214
    from oracle import Oracle

    rng = Mt(37)
    dense, m = masked_case(8, 8, 0.5, 2, rng, Oracle())
    act = sp.Tensor(8, 2, 2, data=random_chw(8, 2, 2, rng))
    bias = np.zeros(8, np.float32)
    with pytest.raises(sp.FormatError):
        sp.spmm(m, act, bias, NONE, sp.MicrokernelConfig(n=4))
    with pytest.raises(sp.ShapeError):
        sp.spmm(m, sp.Tensor(9, 2, 2), bias, NONE, sp.MicrokernelConfig(n=2))
    with pytest.raises(sp.LayoutError):
        sp.spmm(m, sp.Tensor(8, 2, 2, sp.Layout.HWC), bias, NONE, sp.MicrokernelConfig(n=2))
    with pytest.raises(ValueError):
        sp.spmm(m, act, bias, NONE, sp.MicrokernelConfig(m=5, n=2))
    with pytest.raises(sp.ShapeError):
        sp.spmm(m, act, np.zeros(3, np.float32), NONE, sp.MicrokernelConfig(n=2))


def test_cabi_validation_order_on_device_pointers():
    """The same checks through spcv_cu_spmm_into itself (C-ABI codes)."""
    import ctypes

    import torch
    from paper_1911_09723_b200 import _capi

    m = sp.encode_bcsr(np.eye(8, dtype=np.float32), 2)
    dw = sp.DeviceBcsr(m)
    a = torch.zeros(1, 8, 2, 2, device="cuda")
    o = torch.zeros(1, 8, 2, 2, device="cuda")
    L = _capi.lib

    def call(act_layout=0, act_c=8, bias_len=0, out_layout=0, out_c=8, out_w=2, m_=0, n=2, kind=0,
             lo=0.0, hi=0.0):
        return L.spcv_cu_spmm_into(dw.handle, a.data_ptr(), act_layout, 1, act_c, 2, 2,
                                   a.data_ptr() if bias_len else None, bias_len, kind, lo, hi,
                                   o.data_ptr(), out_layout, out_c, 2, out_w, m_, n, 0, None)

    assert call() == _capi.OK
    assert call(act_layout=1, act_c=9) == _capi.ERR_LAYOUT      # layout checked first
    assert call(act_c=9, n=4) == _capi.ERR_SHAPE                 # then channels
    assert call(n=4, bias_len=3) == _capi.ERR_FORMAT             # then block height
    assert call(bias_len=3, out_c=9) == _capi.ERR_SHAPE          # then bias length
    assert call(out_w=3, m_=5) == _capi.ERR_SHAPE                # then out shape
    assert call(m_=5) == _capi.ERR_INVALID                       # then strip width
    assert call(kind=1, lo=1.0, hi=1.0) == _capi.ERR_INVALID     # clamp lo < hi
    torch.cuda.synchronize()


def test_fully_dense_matrix_equals_dense_oracle(oracle):
    # test_kernels.cpp:232-239
    rng = Mt(43)
    w = random_matrix(16, 16, rng)
    act = random_chw(16, 6, 6, rng)
    bias = random_bias(16, rng)
    got = sp.spmm(sp.encode_bcsr(w, 1), sp.Tensor(16, 6, 6, data=act), bias, NONE).data
    want = oracle.matmul_reference(w, act.reshape(16, -1), bias, None)
    assert np.array_equal(bits(got), bits(want))


# ------------------------------------------------------------ format round trip
def test_pack_unpack_bit_exact(oracle):
    rng = Mt(99)
    for bh in (1, 2, 4):
        for _ in range(15):
            rows = bh * (1 + int(rng() % 40))
            cols = 1 + int(rng() % 300)
            s = (rng() % 100) / 100.0
            w = random_matrix(rows, cols, rng)
            rc, keep = oracle.generate_mask(rows, cols, s, bh, 1, rng())
            w[~keep] = 0
            m = sp.encode_bcsr(w, bh)
            back = sp.DeviceBcsr(m).unpack()
            assert back.row_ptr.tobytes() == m.row_ptr.tobytes()
            assert back.col_idx.tobytes() == m.col_idx.tobytes()
            assert back.values.tobytes() == m.values.tobytes()


def test_pack_unpack_large_and_degenerate():
    for layer in (c5_layer(0.9), mbv1_pointwise()[-1], Layer("e", 4, 8, 1, 1, sparsity=0.0)):
        d = make_layer_data(layer, 1, 11, act=False)
        back = sp.DeviceBcsr(d.weights).unpack()
        assert back.row_ptr.tobytes() == d.weights.row_ptr.tobytes()
        assert back.col_idx.tobytes() == d.weights.col_idx.tobytes()
        assert back.values.tobytes() == d.weights.values.tobytes()
    empty = sp.encode_bcsr(np.zeros((8, 5), np.float32), 4)
    back = sp.DeviceBcsr(empty).unpack()
    assert back.row_ptr.tolist() == [0, 0, 0] and back.nnz_blocks() == 0


# ------------------------------------------------------- BASELINE configs
def check_layer(oracle, layer, images, seed, strict=True):
    d = make_layer_data(layer, images, seed)
    got = run_device(d.weights, d.act, d.bias, layer.act, strict=strict)
    want = oracle.spmm(d.weights, d.act, d.bias, layer.act, nthreads=8).reshape(got.shape)
    if strict:
        assert np.array_equal(bits(got), bits(want)), layer.name
    else:
        check_tolerance(d, got, want)
    return d, got


def check_tolerance(d, got, want):
    """|gpu - ref| <= 1e-5 * max(1, nnz_r/64) * A_ij (fp64 A_ij = |b| + sum|w x|)."""
    L = d.layer
    W = np.abs(d.dense.astype(np.float64))
    X = np.abs(d.act.astype(np.float64)).reshape(d.images, L.cin, -1)
    A = np.abs(d.bias.astype(np.float64))[None, :, None] + np.einsum("mk,bks->bms", W, X)
    nnz_r = (d.dense != 0).sum(axis=1).astype(np.float64)
    tol = 1e-5 * np.maximum(1.0, nnz_r / 64.0)[None, :, None] * A
    err = np.abs(got.reshape(A.shape).astype(np.float64) - want.reshape(A.shape).astype(np.float64))
    assert np.all(err <= tol), float((err - tol).max())


def test_config1_bit_exact(oracle):
    check_layer(oracle, CONFIGS["c1"]["layers"]()[0], 1, 1)


@pytest.mark.parametrize("li", range(13))
def test_config2_mbv1_layers_bit_exact(oracle, li):
    layer = mbv1_pointwise(0.9)[li]
    check_layer(oracle, layer, 2 if layer.spatial <= 784 else 1, 100 + li)


@pytest.mark.parametrize("bh", [4, 2, 1])
@pytest.mark.parametrize("s", [0.7, 0.8, 0.9, 0.95])
def test_config3_block_sweep_bit_exact(oracle, bh, s):
    from paper_1911_09723_b200.workloads import c3_layer

    check_layer(oracle, c3_layer(s, bh), 4, 7 + bh)


def test_config4_mbv2_layers_bit_exact(oracle):
    for i, layer in enumerate(mbv2_pointwise(0.85)):
        check_layer(oracle, layer, 1, 200 + i)


@pytest.mark.parametrize("s", [0.7, 0.8, 0.9, 0.95, 0.98])
def test_config5_skewed_bit_exact(oracle, s):
    check_layer(oracle, c5_layer(s), 8, 300)


@pytest.mark.parametrize("layer", [CONFIGS["c1"]["layers"]()[0], mbv1_pointwise()[0],
                                   mbv1_pointwise()[-1], c5_layer(0.9)],
                         ids=["c1", "pw1", "pw13", "c5"])
def test_fast_mode_within_tolerance(oracle, layer):
    check_layer(oracle, layer, 2, 400, strict=False)


# ----------------------------------- full-size, size-independent properties
def test_config5_full_batch_images_independent_of_position(oracle):
    """c5 at its full 1024 images: every sampled image equals the oracle run
    on that image alone (batch position cannot matter), and a rerun is
    bit-identical (determinism)."""
    d = make_layer_data(c5_layer(0.9), 1024, 5)
    got = run_device(d.weights, d.act, d.bias, d.layer.act)
    for i in (0, 1, 377, 511, 1023):
        want = oracle.spmm(d.weights, d.act[i:i + 1], d.bias, d.layer.act)
        assert np.array_equal(bits(got[i]), bits(want))
    again = run_device(d.weights, d.act, d.bias, d.layer.act)
    assert np.array_equal(bits(got), bits(again))


def test_config2_b256_sampled_images(oracle):
    layers = mbv1_pointwise(0.9)
    for li in (0, 6, 12):
        d = make_layer_data(layers[li], 256, 500 + li)
        got = run_device(d.weights, d.act, d.bias, d.layer.act)
        for i in (0, 128, 255):
            want = oracle.spmm(d.weights, d.act[i:i + 1], d.bias, d.layer.act)
            assert np.array_equal(bits(got[i]), bits(want))


# ----------------------------------------------------------------- edge cases
def test_empty_matrix_and_empty_rows_give_clamped_bias(oracle):
    m = sp.encode_bcsr(np.zeros((8, 5), np.float32), 2)
    bias = np.array([-1, 2, 7, 0.5, -0.0, 0.0, 3, -3], np.float32)
    act = np.ones((3, 5, 4, 4), np.float32)
    got = run_device(m, act, bias, RELU6)
    want = np.where(bias < 0, 0, np.where(bias > 6, 6, bias)).astype(np.float32)
    assert np.array_equal(bits(got), bits(np.broadcast_to(want[None, :, None, None], got.shape)))
    # -0.0 bias survives the ternary clamp (tensor.hpp:90-96)
    assert np.signbit(got[0, 4]).all()


def test_null_bias_is_plus_zero(oracle):
    rng = Mt(5)
    dense, m = masked_case(16, 16, 0.8, 1, rng, oracle)
    act = random_chw(16, 3, 7, rng)[None]
    got = run_device(m, act, None, NONE)
    want = oracle.spmm(m, act, None, None)
    assert np.array_equal(bits(got), bits(want))


def test_nan_propagates_like_reference(oracle):
    rng = Mt(6)
    dense, m = masked_case(16, 16, 0.5, 1, rng, oracle)
    act = random_chw(16, 2, 8, rng)[None]
    act[0, 3, 1, 2] = np.nan
    bias = random_bias(16, rng)
    got = run_device(m, act, bias, RELU6)
    want = oracle.spmm(m, act, bias, RELU6)  # NaN payloads may differ; positions must not
    assert np.array_equal(np.isnan(got).reshape(-1), np.isnan(want).reshape(-1))


def test_unaligned_and_odd_spatial_paths(oracle):
    """S % 4 != 0 and misaligned base pointers take the scalar-staging kernel."""
    import torch

    layer = Layer("odd", 40, 24, 5, 7, sparsity=0.6)
    d = make_layer_data(layer, 3, 9)
    want = oracle.spmm(d.weights, d.act, d.bias, layer.act).reshape(3, 24, 5, 7)
    assert np.array_equal(bits(run_device(d.weights, d.act, d.bias, layer.act)), bits(want))
    # S % 4 == 0 but buffers offset by one float
    layer = Layer("mis", 40, 24, 4, 8, sparsity=0.6)
    d = make_layer_data(layer, 3, 10)
    want = oracle.spmm(d.weights, d.act, d.bias, layer.act).reshape(3, 24, 4, 8)
    dw = sp.DeviceBcsr(d.weights)
    base_a = torch.zeros(d.act.size + 1, device="cuda")
    base_o = torch.zeros(want.size + 1, device="cuda")
    a = base_a[1:].view(d.act.shape)
    a.copy_(torch.from_numpy(d.act))
    o = base_o[1:].view(want.shape)
    sp.spmm_batched_into(dw, a, torch.from_numpy(d.bias).cuda(), act_of(layer.act), o,
                         sp.MicrokernelConfig(n=1))
    torch.cuda.synchronize()
    assert np.array_equal(bits(o.cpu().numpy()), bits(want))


def test_zero_images_is_a_noop():
    import torch

    dw = sp.DeviceBcsr(sp.encode_bcsr(np.eye(4, dtype=np.float32), 1))
    a = torch.zeros(0, 4, 2, 2, device="cuda")
    o = torch.zeros(0, 4, 2, 2, device="cuda")
    n0 = sp.launch_count()
    sp.spmm_batched_into(dw, a, None, NONE, o)
    assert sp.launch_count() == n0


@pytest.mark.parametrize("case", [
    ("k2000_id", 4, 2000, 1, 0.0, ("none", 0.0, 0.0), (3, 2), 2),
    ("k1100", 64, 1100, 1, 0.9, ("clamp", 0.0, 6.0), (7, 7), 6),
    ("k2048_bh4", 128, 2048, 4, 0.8, ("clamp", 0.0, float("inf")), (4, 4), 5),
    ("k2500_bh2", 40, 2500, 2, 0.95, ("none", 0.0, 0.0), (3, 5), 4),
    ("k3100_dense", 8, 3100, 1, 0.0, ("clamp", -1.0, 1.0), (2, 2), 3),
], ids=lambda c: c[0])
def test_wide_matrices_run_as_channel_passes_bit_exact(oracle, case):
    """Input channels beyond one shared-memory tile (K > 1024 per pass) run as
    channel passes that continue each other's sums (spcv_cu.cu: pack_passes):
    strict results equal the oracle bit for bit (the reference order of terms
    is kept across passes), fast ones stay within tolerance, and the packed
    matrix still unpacks to the original BCSR."""
    name, M, K, bh, sparsity, act, hw, images = case
    rng = np.random.default_rng(K)
    dense = (rng.standard_normal((M, K)) * 0.1).astype(np.float32)
    if name == "k2000_id":
        dense[:] = 0
        dense[np.arange(M), np.arange(M) * 499] = 1.0  # picks channels 0, 499, 998, 1497
    elif sparsity > 0:
        keep = rng.random((M // bh, K)) >= sparsity
        dense *= np.repeat(keep, bh, axis=0)
    m = sp.encode_bcsr(dense, bh)
    act_ = rng.uniform(-1, 1, (images, K) + hw).astype(np.float32)
    bias = (rng.standard_normal(M) * 0.1).astype(np.float32)
    got = run_device(m, act_, bias, act)
    want = oracle.spmm(m, act_, bias, act, nthreads=8).reshape(got.shape)
    assert np.array_equal(bits(got), bits(want))
    if name == "k2000_id":
        x = act_.reshape(images, K, -1)
        ident = np.stack([x[:, 0], x[:, 499], x[:, 998], x[:, 1497]], 1) + bias[None, :, None]
        assert np.array_equal(got.reshape(images, M, -1), ident.astype(np.float32))
    fast = run_device(m, act_, bias, act, strict=False)
    assert np.allclose(fast, want, rtol=1e-4, atol=1e-5)
    host_out = np.full_like(got, np.nan)  # the host-buffer entry point (chunked H2D|kernel|D2H)
    sp.spmm_host_batched(sp.DeviceBcsr(m), act_, bias, act_of(act), host_out, sp.MicrokernelConfig(n=bh))
    assert np.array_equal(bits(host_out), bits(want))
    u = sp.DeviceBcsr(m).unpack()
    assert np.array_equal(np.asarray(u.row_ptr), np.asarray(m.row_ptr))
    assert np.array_equal(np.asarray(u.col_idx), np.asarray(m.col_idx))
    assert np.array_equal(np.asarray(u.values, np.float32).view(np.uint32),
                          np.asarray(m.values, np.float32).view(np.uint32))


@pytest.mark.parametrize("images", [1, 4, 5, 9])
def test_host_path_large_images_chunking(oracle, images):
    """Host-buffer entry point with one image larger than half the 48 MiB chunk
    budget (chunk = 1 image): the chunk schedule must cover exactly `images`
    images (the ramp used to overrun the buffers at 4-5 images)."""
    rng = np.random.default_rng(100 + images)
    K = M = 64
    H = W = 224  # (64+64)*224*224*4 B = 25.7 MB per image
    dense = (rng.standard_normal((M, K)) * 0.1).astype(np.float32)
    dense *= rng.random((M, K)) >= 0.9
    m = sp.encode_bcsr(dense, 1)
    act_ = rng.uniform(-1, 1, (images, K, H, W)).astype(np.float32)
    bias = (rng.standard_normal(M) * 0.1).astype(np.float32)
    want = oracle.spmm(m, act_, bias, RELU6, nthreads=8).reshape(images, M, H, W)
    guard = 8
    buf = np.full((images + guard, M, H, W), np.nan, np.float32)  # images past `images` must stay untouched
    host_out = buf[:images]
    sp.spmm_host_batched(sp.DeviceBcsr(m), act_, bias, RELU6, host_out, sp.MicrokernelConfig(n=1))
    assert np.array_equal(bits(host_out), bits(want))
    assert np.isnan(buf[images:]).all()


def test_host_path_rejects_bad_outputs():
    m = sp.encode_bcsr(np.eye(8, dtype=np.float32), 1)
    w = sp.DeviceBcsr(m)
    act_ = np.ones((2, 8, 3, 3), np.float32)
    with pytest.raises(sp.ShapeError):
        sp.spmm_host_batched(w, act_, None, NONE, np.zeros((1, 8, 3, 3), np.float32))
    with pytest.raises(sp.ShapeError):
        sp.spmm_host_batched(w, act_, None, NONE, np.zeros((2, 8, 3, 3), np.float64))
    with pytest.raises(sp.ShapeError):
        sp.spmm_host_batched(w, act_, None, NONE, np.zeros((2, 8, 3, 3), np.float32)[:, :, :, ::-1])
    out = np.zeros((2, 8, 3, 3), np.float32)
    sp.spmm_host_batched(w, act_.astype(np.float64), None, NONE, out)  # act converted
    assert np.array_equal(out, np.ones_like(out))


def test_reference_call_shape_packs_and_compiles_once(oracle, tmp_path, monkeypatch):
    """spmm_into(BcsrMatrix, host tensors) in a loop (the reference's callers,
    run_network / bench_layers): the matrix is packed once per content, the
    weight-specialised kernel compiled at most once, every result bit-exact;
    a different matrix of the same shape is a different cache entry."""
    d = make_layer_data(Layer("loop", 48, 96, 6, 6, sparsity=0.85), 3, 321)  # K <= 64: JIT direct
    s0 = sp.cache_stats()
    for i in range(3):
        out = sp.spmm(d.weights, sp.Tensor(48, 6, 6, data=d.act[i]), d.bias, RELU6)
        want = oracle.spmm(d.weights, d.act[i:i + 1], d.bias, RELU6).reshape(-1)
        assert np.array_equal(bits(out.data), bits(want))
    s1 = sp.cache_stats()
    assert s1["misses"] - s0["misses"] == 1 and s1["hits"] - s0["hits"] == 2
    assert s1["jit_compiles"] + s1["jit_disk_hits"] - s0["jit_compiles"] - s0["jit_disk_hits"] <= 1
    other = sp.BcsrMatrix(d.weights.rows, d.weights.cols, 1, d.weights.row_ptr, d.weights.col_idx,
                          d.weights.values * np.float32(2.0))
    sp.spmm(other, sp.Tensor(48, 6, 6, data=d.act[0]), d.bias, RELU6)
    assert sp.cache_stats()["misses"] - s1["misses"] == 1


def test_tile_kernel_matrix_never_compiles_jit(monkeypatch):
    """A call the k-major JIT variant would not serve (too few columns) must not
    compile it (the plan decides before NVRTC runs)."""
    import torch

    monkeypatch.delenv("SPCV_JIT_KMAJOR_MIN_COLS", raising=False)  # production threshold
    d = make_layer_data(Layer("c1like", 128, 128, 28, 28, sparsity=0.8), 1, 5)
    w = sp.DeviceBcsr(d.weights)
    c0 = sp.cache_stats()["jit_compiles"]
    run_device(d.weights, d.act, d.bias, RELU6, dw=w)
    assert sp.cache_stats()["jit_compiles"] == c0


def test_concurrent_streams_agree(oracle):
    import torch

    d = make_layer_data(mbv1_pointwise()[6], 8, 77)
    dw = sp.DeviceBcsr(d.weights)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    r1 = run_device(d.weights, d.act, d.bias, d.layer.act, dw=dw, stream=s1)
    r2 = run_device(d.weights, d.act, d.bias, d.layer.act, dw=dw, stream=s2)
    assert np.array_equal(bits(r1), bits(r2))


def test_kernel_launches_are_counted():
    n0 = sp.launch_count()
    run_device(sp.encode_bcsr(np.eye(4, dtype=np.float32), 1), np.ones((1, 4, 2, 2), np.float32),
               None, NONE)
    assert sp.launch_count() == n0 + 1


# ------------------------------------------- both kernels on the same inputs
@pytest.mark.parametrize("layout", ["default", "steps2", "steps4", "nf2", "nf4_steps2"])
@pytest.mark.parametrize("case", [
    ("pw3_b8", Layer("pw3", 128, 128, 56, 56, sparsity=0.9), 8),
    ("c3_bh4", Layer("c3", 512, 512, 14, 14, ("clamp", 0.0, float("inf")), -1.0, 1.0, 0.8, 4), 12),
    ("c3_bh2", Layer("c3", 512, 512, 14, 14, ("clamp", 0.0, float("inf")), -1.0, 1.0, 0.9, 2), 12),
    ("tail", Layer("tail", 64, 96, 6, 10, sparsity=0.7), 37),       # N % T != 0
    ("k1024", Layer("k", 1024, 256, 4, 4, sparsity=0.95), 300),     # 1-stage tile -> fallback
], ids=lambda c: c[0] if isinstance(c, tuple) else c)
def test_tile_kernel_layouts_bit_exact(oracle, monkeypatch, case, layout):
    """SPCV_STEPS / SPCV_NF force the chunk length and lane width the packer
    would otherwise pick. Every combination must equal the oracle bit-for-bit."""
    use_kernel(monkeypatch, "tile")  # small K would otherwise take the JIT kernel
    env = {"steps2": {"SPCV_STEPS": "2"}, "steps4": {"SPCV_STEPS": "4"}, "nf2": {"SPCV_NF": "2"},
           "nf4_steps2": {"SPCV_NF": "4", "SPCV_STEPS": "2"}}.get(layout, {})
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _, layer, images = case
    d = make_layer_data(layer, images, 4242)
    got = run_device(d.weights, d.act, d.bias, layer.act)
    want = oracle.spmm(d.weights, d.act, d.bias, layer.act, nthreads=8).reshape(got.shape)
    assert np.array_equal(bits(got), bits(want))
    fast = run_device(d.weights, d.act, d.bias, layer.act, strict=False)
    check_tolerance(d, fast, want)


# ------------------------------------ weight-specialised small-K kernel (jit.cu)
JIT_CASES = [
    ("pw1", mbv1_pointwise()[0], 2),
    ("pw2", mbv1_pointwise()[1], 1),
    ("pw3", mbv1_pointwise()[2], 1),
    ("pw4", mbv1_pointwise()[3], 2),
    ("bh2_tail", Layer("b2", 96, 64, 8, 9, ("clamp", 0.0, 6.0), -1.0, 1.0, 0.8, 2), 5),
    ("bh4_none", Layer("b4", 128, 128, 4, 6, ("none", 0.0, 0.0), -1.0, 1.0, 0.9, 4), 4),
    ("k1", Layer("k1", 1, 8, 4, 4, ("none", 0.0, 0.0), -1.0, 1.0, 0.0), 2),
    ("k33_partial_chunk", Layer("k33", 33, 40, 4, 5, sparsity=0.5), 3),
    ("k72_partial_chunk", Layer("k72", 72, 40, 4, 5, sparsity=0.5), 3),
    ("direct_odd_spatial", Layer("odd", 48, 40, 7, 7, sparsity=0.8), 3),
    ("dense", Layer("d", 16, 32, 4, 4, sparsity=0.0), 2),
    ("empty_rows", Layer("e", 32, 40, 4, 5, ("clamp", -0.5, 0.5), -1.0, 1.0, 0.97), 3),
]


@pytest.mark.parametrize("kernel", ["jit", "tile"])
@pytest.mark.parametrize("case", JIT_CASES, ids=lambda c: c[0])
def test_jit_and_tile_small_k_bit_exact(oracle, monkeypatch, kernel, case):
    """The weight-specialised kernel (SPCV_JIT default) and the tile kernel
    (SPCV_JIT=0) both equal the oracle bit-for-bit in strict mode, with and
    without bias, and stay within the fast-mode bound (S % 4 == 0 cases: the
    JIT kernel's 16 B staging; column tails, partial channel chunks, empty
    rows and one-channel matrices included)."""
    monkeypatch.setenv("SPCV_JIT", "1" if kernel == "jit" else "0")
    monkeypatch.setenv("SPCV_JIT_MAX_SEGS", "48")  # exercise multi-segment plans too
    # (SPCV_JIT_KMAJOR_MIN_COLS=0 for this process: conftest.py)
    _, layer, images = case
    d = make_layer_data(layer, images, 99)
    dw = sp.DeviceBcsr(d.weights)
    assert dw.kernel(strict=True) == kernel and dw.kernel(strict=False) == kernel
    got = run_device(d.weights, d.act, d.bias, layer.act, dw=dw)
    want = oracle.spmm(d.weights, d.act, d.bias, layer.act, nthreads=8).reshape(got.shape)
    assert np.array_equal(bits(got), bits(want))
    got0 = run_device(d.weights, d.act, None, layer.act, dw=dw)
    want0 = oracle.spmm(d.weights, d.act, None, layer.act, nthreads=8).reshape(got.shape)
    assert np.array_equal(bits(got0), bits(want0))
    check_tolerance(d, run_device(d.weights, d.act, d.bias, layer.act, strict=False, dw=dw), want)


def test_jit_not_used_beyond_its_limits(monkeypatch):
    monkeypatch.delenv("SPCV_JIT", raising=False)
    monkeypatch.delenv("SPCV_JIT_MAX_SEGS", raising=False)
    monkeypatch.delenv("SPCV_JIT_SEG_INSTR", raising=False)
    small = make_layer_data(Layer("s", 300, 8, 2, 2, sparsity=0.5), 1, 1)
    assert sp.DeviceBcsr(small.weights).kernel() == "jit"
    # half-dense 1024 x 1024: far more row segments than the cap -> tile kernel
    big = make_layer_data(Layer("b", 1024, 1024, 2, 2, sparsity=0.5), 1, 1)
    assert sp.DeviceBcsr(big.weights).kernel() == "tile"


def test_jit_odd_spatial_falls_back_to_tile_bit_exact(oracle):
    """S % 4 != 0 (or unaligned buffers) cannot use the k-major variant's 16 B
    staging (K > 64): the call runs the tile kernel and stays bit-exact."""
    layer = Layer("odd", 96, 48, 7, 7, sparsity=0.8)
    d = make_layer_data(layer, 3, 5)
    got = run_device(d.weights, d.act, d.bias, layer.act)
    want = oracle.spmm(d.weights, d.act, d.bias, layer.act).reshape(got.shape)
    assert np.array_equal(bits(got), bits(want))


# ------------------------------------------------- dense fp32 baseline (§8f-1)
@pytest.mark.parametrize("layer", [mbv1_pointwise()[0], mbv1_pointwise()[6], mbv1_pointwise()[12],
                                   Layer("odd", 40, 24, 5, 7, sparsity=0.0),
                                   Layer("fc", 1024, 1000, 1, 1, ("none", 0.0, 0.0), -1.0, 1.0, 0.0)],
                         ids=["pw1", "pw7", "pw13", "odd", "classifier_s1"])
def test_dense_baseline_within_fp32_rounding(oracle, layer):
    """dense_gemm_into (kernels.cpp:345-373) through cuBLAS SGEMM (pedantic
    fp32): within the fp32 reordering bound of the dense oracle (the reference's
    own dense kernel is bit-exact with matmul_reference; cuBLAS sums in its own
    order, so the bound of check_tolerance applies with nnz_r = K)."""
    import torch

    d = make_layer_data(layer, 2, 31)
    w = torch.from_numpy(d.dense).cuda()
    a = torch.from_numpy(d.act).cuda()
    o = torch.empty(2, layer.cout, layer.h, layer.w, device="cuda")
    sp.dense_gemm_batched_into(w, a, torch.from_numpy(d.bias).cuda(), act_of(layer.act), o)
    torch.cuda.synchronize()
    want = np.stack([oracle.matmul_reference(d.dense, d.act[i].reshape(layer.cin, -1), d.bias, layer.act)
                     for i in range(2)])
    L = d.layer
    W = np.abs(d.dense.astype(np.float64))
    X = np.abs(d.act.astype(np.float64)).reshape(2, L.cin, -1)
    A = np.abs(d.bias.astype(np.float64))[None, :, None] + np.einsum("mk,bks->bms", W, X)
    tol = 1e-5 * max(1.0, L.cin / 64.0) * A
    err = np.abs(o.cpu().numpy().reshape(A.shape).astype(np.float64) - want.reshape(A.shape))
    assert np.all(err <= tol)


def test_dense_baseline_validation_order():
    import torch

    w = torch.zeros(8, 8, device="cuda")
    with pytest.raises(sp.ShapeError):
        sp.dense_gemm_batched_into(w, torch.zeros(1, 9, 2, 2, device="cuda"), None, NONE,
                                   torch.zeros(1, 8, 2, 2, device="cuda"))
    with pytest.raises(sp.ShapeError):
        sp.dense_gemm_batched_into(w, torch.zeros(1, 8, 2, 2, device="cuda"),
                                   torch.zeros(3, device="cuda"), NONE, torch.zeros(1, 8, 2, 2, device="cuda"))
    with pytest.raises(ValueError):
        sp.dense_gemm_batched_into(w, torch.zeros(1, 8, 2, 2, device="cuda"), None, NONE,
                                   torch.zeros(1, 8, 2, 2, device="cuda"), sp.MicrokernelConfig(m=5))


# ------------------------------- executor pointwise step on device (§8f-2)
@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("hw", [(7, 9), (8, 8)], ids=["odd_spatial", "vec"])
@pytest.mark.parametrize("bh", [2, 4])
def test_spmm_layer_padded_rows_and_residual(oracle, monkeypatch, hw, bh, kernel):
    """run_network's pointwise branch (netdef.cpp:494-512): weights padded to
    the block height are run wide (pad rows bias 0) and truncated to the
    logical rows; the residual is added after the activation. Bit-exact
    against the oracle doing the same steps on the host."""
    import torch

    H, W = hw
    rows, K, B = 10, 24, 3
    rng = np.random.default_rng(5)
    dense = (rng.standard_normal((rows, K)) * 0.3).astype(np.float32)
    dense[rng.random((rows, K)) < 0.6] = 0
    pad = (-rows) % bh
    wide = np.vstack([dense, np.zeros((pad, K), np.float32)])
    m = sp.encode_bcsr(wide, bh)
    act = rng.uniform(-1, 1, (B, K, H, W)).astype(np.float32)
    bias = rng.uniform(-1, 1, rows).astype(np.float32)
    res = rng.uniform(-1, 1, (B, rows, H, W)).astype(np.float32)
    want = oracle.spmm(m, act, np.r_[bias, np.zeros(pad, np.float32)], RELU6)[:, :rows].reshape(B, rows, H, W)
    want_res = (want + res).astype(np.float32)
    use_kernel(monkeypatch, kernel)
    dw = sp.DeviceBcsr(m)
    assert dw.kernel_for(B, H, W) == kernel
    a = torch.from_numpy(act).cuda()
    o = torch.full((B, rows, H, W), float("nan"), device="cuda")
    sp.spmm_layer(dw, a, torch.from_numpy(bias).cuda(), RELU6, o)
    torch.cuda.synchronize()
    assert np.array_equal(bits(o.cpu().numpy()), bits(want))
    sp.spmm_layer(dw, a, torch.from_numpy(bias).cuda(), RELU6, o, residual=torch.from_numpy(res).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(bits(o.cpu().numpy()), bits(want_res))


def test_spmm_layer_checks():
    import torch

    m = sp.encode_bcsr(np.ones((12, 8), np.float32), 4)
    dw = sp.DeviceBcsr(m)
    a = torch.zeros(1, 8, 2, 2, device="cuda")
    with pytest.raises(sp.ShapeError):  # more logical rows than stored
        sp.spmm_layer(dw, a, None, NONE, torch.zeros(1, 13, 2, 2, device="cuda"))
    with pytest.raises(sp.ShapeError):  # padding larger than one block
        sp.spmm_layer(dw, a, None, NONE, torch.zeros(1, 8, 2, 2, device="cuda"))
    with pytest.raises(sp.ShapeError):  # bias must match the logical rows
        sp.spmm_layer(dw, a, torch.zeros(12, device="cuda"), NONE, torch.zeros(1, 10, 2, 2, device="cuda"))
    with pytest.raises(sp.ShapeError):
        sp.spmm_layer(dw, torch.zeros(1, 9, 2, 2, device="cuda"), None, NONE,
                      torch.zeros(1, 10, 2, 2, device="cuda"))


def test_jit_variants_compile_concurrently(oracle):
    """Several host threads hit one packed matrix with different call shapes
    (strict/fast x bias/no bias x clamp/none) at once: every variant compiles
    once under the weights' lock, launches stay valid, strict results exact."""
    import threading

    import torch

    layer = Layer("cc", 48, 64, 8, 8, sparsity=0.8)
    d = make_layer_data(layer, 3, 21)
    dw = sp.DeviceBcsr(d.weights)
    a = torch.from_numpy(d.act).cuda()
    b = torch.from_numpy(d.bias).cuda()
    shapes = [(strict, bias, fused) for strict in (True, False) for bias in (True, False)
              for fused in (RELU6, NONE)]
    want = {(True, bias, fused.kind): oracle.spmm(d.weights, d.act, d.bias if bias else None, fused)
            for _, bias, fused in shapes}
    errors = []

    def work(tid):
        try:
            st = torch.cuda.Stream()
            for it in range(6):
                strict, bias, fused = shapes[(tid + it) % len(shapes)]
                o = torch.empty(3, 64, 8, 8, device="cuda")
                sp.spmm_batched_into(dw, a, b if bias else None, fused, o,
                                     sp.MicrokernelConfig(n=1, strict=strict), stream=st)
                st.synchronize()
                if strict:
                    ref = want[(True, bias, fused.kind)].reshape(o.shape)
                    if not np.array_equal(bits(o.cpu().numpy()), bits(ref)):
                        errors.append((tid, it))
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ts = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("kernel", KERNELS)
def test_signed_zeros_and_padding_are_bit_exact(oracle, monkeypatch, kernel):
    """-0.0 biases, -0.0 stored weights, zero activations of both signs and a
    clamp at lo = -0.0: the order of additions decides the sign of zero
    results, and every kernel must reproduce the reference bit for bit."""
    import torch

    use_kernel(monkeypatch, kernel)
    rng = np.random.default_rng(17)
    K, M, H, W = 24, 16, 4, 4
    dense = np.zeros((M, K), np.float32)
    for r in range(M):
        cols = rng.choice(K, size=1 + r % 5, replace=False)
        dense[r, cols] = rng.choice([-1.0, 1.0, -0.5, 2.0, -0.0], size=cols.size).astype(np.float32)
    m = sp.encode_bcsr(dense, 1)
    act = rng.choice([0.0, -0.0, 1.0, -1.0], size=(2, K, H, W)).astype(np.float32)
    bias = rng.choice([0.0, -0.0, 0.5], size=M).astype(np.float32)
    dw = sp.DeviceBcsr(m)
    for fused in (NONE, sp.Activation.clamp(-0.0, 6.0), RELU6):
        got = run_device(m, act, bias, fused, dw=dw)
        want = oracle.spmm(m, act, bias, fused).reshape(got.shape)
        assert np.array_equal(bits(got), bits(want)), fused


@pytest.mark.parametrize("kernel", KERNELS)
def test_randomized_shapes_bit_exact(oracle, monkeypatch, kernel):
    """Seeded random layers (K 1..200, M 1..96, block heights 1/2/4, odd and
    even spatial sizes, 1-3 images, 0-99 % sparsity, bias or none, clamp or
    none) through spcv_cu_spmm_into: bit-exact against the oracle for both the
    weight-specialised and the tile kernel."""
    use_kernel(monkeypatch, kernel)
    monkeypatch.setenv("SPCV_JIT_MAX_SEGS", "48")
    rng = np.random.default_rng(2024)
    for case in range(14):
        bh = int(rng.choice([1, 2, 4]))
        K = int(rng.integers(1, 201))
        M = int(rng.integers(1, 25)) * bh
        H, W = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        B = int(rng.integers(1, 4))
        sparsity = float(rng.choice([0.0, 0.5, 0.9, 0.99]))
        dense = (rng.standard_normal((M, K)) * 0.3).astype(np.float32)
        dense[rng.random((M // bh, K)).repeat(bh, axis=0) < sparsity] = 0
        m = sp.encode_bcsr(dense, bh)
        act = rng.uniform(-1, 1, (B, K, H, W)).astype(np.float32)
        bias = rng.uniform(-1, 1, M).astype(np.float32) if case % 3 else None
        fused = RELU6 if case % 2 else NONE
        dw = sp.DeviceBcsr(m)
        got = run_device(m, act, bias, fused, dw=dw)
        want = oracle.spmm(m, act, bias, fused).reshape(got.shape)
        assert np.array_equal(bits(got), bits(want)), (case, K, M, bh, H, W, B, sparsity)


def test_bound_call_equals_direct_call(oracle):
    """bind_batched: arguments checked and converted once, every invocation one
    C-ABI call — same bits as spmm_batched_into, one counted launch each, and
    the C-ABI's own argument checks still run at call time."""
    import torch

    layer = CONFIGS["c1"]["layers"]()[0]
    d = make_layer_data(layer, 2, 77)
    dw = sp.DeviceBcsr(d.weights)
    a = torch.from_numpy(d.act).cuda()
    b = torch.from_numpy(d.bias).cuda()
    o = torch.full((2, layer.cout, layer.h, layer.w), float("nan"), device="cuda")
    call = sp.bind_batched(dw, a, b, act_of(layer.act), o)
    want = oracle.spmm(d.weights, d.act, d.bias, layer.act).reshape(o.shape)
    for _ in range(3):
        o.fill_(float("nan"))
        n0 = sp.launch_count()
        call()
        torch.cuda.synchronize()
        assert sp.launch_count() == n0 + 1
        assert np.array_equal(bits(o.cpu().numpy()), bits(want))
    bad = sp.bind_batched(dw, a, b[:-1].contiguous(), act_of(layer.act), o)  # bias one short
    with pytest.raises(sp.ShapeError):
        bad()
    with pytest.raises(sp.DeviceError):
        sp.bind_batched(dw, a.cpu(), b, act_of(layer.act), o)


# ------------------------ unaligned layouts: coalesced epilogue (SPCV_COAL)
@pytest.mark.parametrize("coal", ["0", "2", "1"], ids=["scattered", "coalesced", "autotuned"])
@pytest.mark.parametrize("case", [
    ("pw13", mbv1_pointwise()[12], 10),                                   # K = 1024: one 16-warp CTA per SM
    ("c5_s98", Layer("c5", 1024, 1024, 7, 7, ("clamp", 0.0, float("inf")), -1.0, 1.0, 0.98, 1, True), 12),
    ("mbv2_7x7", Layer("b15e", 160, 960, 7, 7, sparsity=0.85), 16),        # 64-column tiles
    ("bh4_odd", Layer("bh4_odd", 96, 40, 5, 7, sparsity=0.7, block_h=4), 9),  # 4x1 blocks, 128-column tiles
    ("bh2_pad", Layer("bh2_pad", 200, 22, 3, 3, sparsity=0.5, block_h=2), 5),
], ids=lambda c: c[0])
def test_unaligned_epilogues_bit_exact(oracle, monkeypatch, coal, case):
    """H*W % 4 != 0: the scattered 4 B epilogue, the coalesced one (row group
    through a per-warp shared-memory scratch, stored row by row) and the
    autotuner's pick between them are bit-identical to the oracle, with and
    without a residual and with padded rows truncated."""
    import torch

    use_kernel(monkeypatch, "tile")
    monkeypatch.setenv("SPCV_COAL", coal)
    if coal != "1":
        monkeypatch.setenv("SPCV_AUTOTUNE", "0")
    _, layer, images = case
    d = make_layer_data(layer, images, 13)
    dw = sp.DeviceBcsr(d.weights)
    want = oracle.spmm(d.weights, d.act, d.bias, layer.act, nthreads=8)
    for _ in range(2):
        got = run_device(d.weights, d.act, d.bias, layer.act, dw=dw)
        assert np.array_equal(bits(got), bits(want.reshape(got.shape)))
    # executor step: logical rows < stored rows, residual added after the clamp
    rows = layer.cout - (1 if layer.block_h > 1 else 0)
    a = torch.from_numpy(d.act).cuda()
    res = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, (images, rows, layer.h, layer.w)).astype(np.float32)).cuda()
    o = torch.full((images, rows, layer.h, layer.w), float("nan"), device="cuda")
    sp.spmm_layer(dw, a, torch.from_numpy(d.bias[:rows].copy()).cuda(), act_of(layer.act), o, residual=res)
    torch.cuda.synchronize()
    w4 = want.reshape(images, layer.cout, layer.h, layer.w)[:, :rows]
    assert np.array_equal(bits(o.cpu().numpy()), bits((w4 + res.cpu().numpy()).astype(np.float32)))


# ------------------------------------ launch geometry: tail and row splits
@pytest.mark.parametrize("env", [{"SPCV_TAIL": "0"}, {"SPCV_TAIL": "2"}, {"SPCV_TAIL": "4"}, {"SPCV_TAIL": "8"},
                                 {"SPCV_SPLIT": "2", "SPCV_TAIL": "4"}, {"SPCV_NWARPS": "8", "SPCV_TAIL": "8"},
                                 {"SPCV_SPLIT": "4"}], ids=lambda e: ",".join(f"{k[5:]}={v}" for k, v in e.items()))
@pytest.mark.parametrize("case", [
    ("k1024", Layer("k1024", 1024, 256, 7, 7, sparsity=0.9), 120),          # one CTA per SM, 184 tiles
    ("skew", Layer("skew", 512, 512, 7, 7, ("clamp", 0.0, float("inf")), -1.0, 1.0, 0.9, 1, True), 200),
], ids=lambda c: c[0])
def test_tail_and_row_splits_bit_exact(oracle, monkeypatch, env, case):
    """The partial last round of tiles split 2/4/8 ways by rows (tail split),
    every tile split across CTAs (SPCV_SPLIT), other CTA sizes: the LPT bins
    each CTA takes change, the per-row arithmetic does not (bit-exact)."""
    use_kernel(monkeypatch, "tile")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _, layer, images = case
    d = make_layer_data(layer, images, 99)
    got = run_device(d.weights, d.act, d.bias, layer.act)
    want = oracle.spmm(d.weights, d.act, d.bias, layer.act, nthreads=8).reshape(got.shape)
    assert np.array_equal(bits(got), bits(want))


@pytest.mark.parametrize("case", [
    ("c3_bh4", Layer("c3", 512, 512, 14, 14, ("clamp", 0.0, float("inf")), -1.0, 1.0, 0.9, 4), 64),
    ("pw12", Layer("pw12", 512, 1024, 7, 7, sparsity=0.9), 256),
], ids=lambda c: c[0])
def test_autotuned_tail_split_bit_exact_and_uncounted(oracle, monkeypatch, case):
    """The first call of a shape times the tail-split candidates (spcv_cu.cu:
    tuned_tail): its result, the cached choice on later calls and the untuned
    heuristic (SPCV_AUTOTUNE=0) are bit-identical to the oracle, and each call
    counts as one launch (the tuning launches are internal)."""
    use_kernel(monkeypatch, "tile")
    _, layer, images = case
    d = make_layer_data(layer, images, 7)
    want = oracle.spmm(d.weights, d.act, d.bias, layer.act, nthreads=8)
    for tune in ("1", "0"):
        monkeypatch.setenv("SPCV_AUTOTUNE", tune)
        dw = sp.DeviceBcsr(d.weights)  # fresh weights: no cached choice
        for _ in range(2):
            n0 = sp.launch_count()
            got = run_device(d.weights, d.act, d.bias, layer.act, dw=dw)
            assert sp.launch_count() == n0 + 1
            assert np.array_equal(bits(got), bits(want.reshape(got.shape)))


@pytest.mark.parametrize("hw", [(7, 9), (8, 8)], ids=["odd_spatial", "vec"])
def test_wide_spmm_layer_padded_rows_and_residual(oracle, hw):
    """The executor's pointwise step on a wide matrix (channel passes): padded
    rows truncated, the clamp then the residual applied once, by the last pass."""
    import torch

    H, W = hw
    rows, K, B, bh = 10, 1700, 2, 4
    rng = np.random.default_rng(9)
    dense = (rng.standard_normal((rows, K)) * 0.1).astype(np.float32)
    dense[rng.random((rows, K)) < 0.9] = 0
    pad = (-rows) % bh
    m = sp.encode_bcsr(np.vstack([dense, np.zeros((pad, K), np.float32)]), bh)
    act = rng.uniform(-1, 1, (B, K, H, W)).astype(np.float32)
    bias = rng.uniform(-1, 1, rows).astype(np.float32)
    res = rng.uniform(-1, 1, (B, rows, H, W)).astype(np.float32)
    want = oracle.spmm(m, act, np.r_[bias, np.zeros(pad, np.float32)], RELU6)[:, :rows].reshape(B, rows, H, W)
    dw = sp.DeviceBcsr(m)
    o = torch.full((B, rows, H, W), float("nan"), device="cuda")
    sp.spmm_layer(dw, torch.from_numpy(act).cuda(), torch.from_numpy(bias).cuda(), RELU6, o,
                  residual=torch.from_numpy(res).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(bits(o.cpu().numpy()), bits((want + res).astype(np.float32)))


# ------------------------- every kernel on BASELINE-shaped layers (round 2)
@pytest.mark.parametrize("kernel", ["tile", "small"])
@pytest.mark.parametrize("case", [
    ("c1", CONFIGS["c1"]["layers"]()[0], 1),
    ("c3_b4", Layer("c3_b4", 512, 512, 14, 14, ("clamp", 0.0, float("inf")), -1.0, 1.0, 0.9, 4), 6),
    ("c3_b2", Layer("c3_b2", 512, 512, 14, 14, ("clamp", 0.0, float("inf")), -1.0, 1.0, 0.8, 2), 6),
    ("pw7", mbv1_pointwise()[6], 12),
    ("pw13", mbv1_pointwise()[12], 12),
    ("c5_s98", Layer("c5", 1024, 1024, 7, 7, ("clamp", 0.0, float("inf")), -1.0, 1.0, 0.98, 1, True), 8),
], ids=lambda c: c[0])
def test_kernels_on_config_layers_bit_exact(oracle, monkeypatch, kernel, case):
    """The tile kernel and the few-column kernel on the BASELINE layer shapes
    (either forced by the pack-time knobs, whatever the column count) equal
    the oracle bit for bit, and kernel_for names the kernel that ran."""
    use_kernel(monkeypatch, kernel)
    _, layer, images = case
    d = make_layer_data(layer, images, 31)
    dw = sp.DeviceBcsr(d.weights)
    assert dw.kernel_for(images, layer.h, layer.w) == kernel
    got = run_device(d.weights, d.act, d.bias, layer.act, dw=dw)
    want = oracle.spmm(d.weights, d.act, d.bias, layer.act, nthreads=8).reshape(got.shape)
    assert np.array_equal(bits(got), bits(want))


def test_default_kernel_choice_by_column_count(monkeypatch):
    """Production choice (no knobs): a single c1 image or one MBv1 batch-1
    layer has fewer column tiles than SMs and runs the few-column kernel; c3 at
    64 images and MBv1 pw13 at 256 images run the tile kernel."""
    monkeypatch.delenv("SPCV_JIT_KMAJOR_MIN_COLS", raising=False)  # production threshold (conftest sets 0)
    c1 = CONFIGS["c1"]["layers"]()[0]
    d = make_layer_data(c1, 1, 3)
    assert sp.DeviceBcsr(d.weights).kernel_for(1, 28, 28) == "small"
    p7 = mbv1_pointwise()[6]
    assert sp.DeviceBcsr(make_layer_data(p7, 1, 3).weights).kernel_for(1, 14, 14) == "small"
    c3 = Layer("c3", 512, 512, 14, 14, ("clamp", 0.0, float("inf")), -1.0, 1.0, 0.9, 4)
    d3 = make_layer_data(c3, 1, 3)
    assert sp.DeviceBcsr(d3.weights).kernel_for(64, 14, 14) == "tile"
    p13 = mbv1_pointwise()[12]
    d13 = make_layer_data(p13, 1, 3)
    assert sp.DeviceBcsr(d13.weights).kernel_for(256, 7, 7) == "tile"


def test_chained_layers_on_one_stream_bit_exact(oracle):
    """Layers launched back to back on one stream, each consuming the previous
    layer's output and overwriting a buffer an earlier layer read, across the
    three kernels (weight-specialised, tile, few-column): stream order alone
    makes every kernel see its predecessor's output, so the chain equals the
    oracle applied layer by layer, bit for bit."""
    import torch

    rng = np.random.default_rng(77)
    chans = [48, 64, 96, 96, 128, 64, 32]  # K=48 (JIT direct), larger K (tile / few-column)
    H = W = 14
    B = 8
    mats, biases = [], []
    for k, m in zip(chans[:-1], chans[1:]):
        d = (rng.standard_normal((m, k)) * 0.2).astype(np.float32)
        d[rng.random((m, k)) < 0.8] = 0
        mats.append(sp.encode_bcsr(d, 1))
        biases.append(rng.uniform(-0.5, 0.5, m).astype(np.float32))
    x = rng.uniform(-1, 1, (B, chans[0], H, W)).astype(np.float32)
    want = x
    for m, b in zip(mats, biases):
        want = oracle.spmm(m, want, b, RELU6).reshape(B, -1, H, W)
    dws = [sp.DeviceBcsr(m) for m in mats]
    # ping-pong buffers: layer i writes the buffer layer i-1 read from
    bufs = [torch.empty(B * max(chans) * H * W, device="cuda") for _ in range(2)]
    cur = bufs[0][: x.size].view(x.shape)
    cur.copy_(torch.from_numpy(x))
    s = torch.cuda.Stream()
    kinds = set()
    with torch.cuda.stream(s):
        for i, (dw, b) in enumerate(zip(dws, biases)):
            kinds.add(dw.kernel_for(B, H, W))
            out = bufs[(i + 1) % 2][: B * chans[i + 1] * H * W].view(B, chans[i + 1], H, W)
            sp.spmm_batched_into(dw, cur, torch.from_numpy(b).cuda(), RELU6, out, stream=s)
            cur = out
        s.synchronize()
    assert np.array_equal(bits(cur.cpu().numpy()), bits(want))
