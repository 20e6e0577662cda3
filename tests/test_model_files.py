"""SPCV model files -> device.

The parser (csrc/model.cu) restates parse_model (model_io.cpp:238-381): the
same checks in the same order with the same typed errors. CPU tests pin it
against the compiled reference on reference-written files and on thousands
of mutated / truncated ones (the reference's own fuzz contract,
test_model_io.cpp:166-188 and acceptance C10: only typed errors, never a
crash). GPU tests load the file, compare every uploaded sparse layer with the
reference's parsed arrays byte for byte, and run each 1x1 layer as
run_network's pointwise step against the oracle.
"""
import numpy as np
import pytest

import paper_1911_09723_b200 as sp

MODELS = [("mbv1", 0.25, 0.9), ("mbv2", 0.35, 0.8), ("ca-mbv2", 1.0, 0.85)]


@pytest.fixture(scope="module")
def files(ref):
    from paper_1911_09723_b200 import netfile

    out = {f"{a}-{w}": ref.model_bytes(a, w, s, 7) for a, w, s in MODELS}
    net = netfile.build_mbv1(0.25, 0.9, seed=3)
    out["ours-mbv1-0.25"] = netfile.serialize(net)          # python-written file
    out["ours-mbv1-0.25-dense"] = netfile.serialize(netfile.densify(net))
    return out


def test_python_written_files_parse_like_reference_files(ref, files):
    """netfile.py (the MBv1 builder + serialize_model restated) writes files the
    reference's parse_model accepts, with the layer list of build_mbv1."""
    for name in ("ours-mbv1-0.25", "ours-mbv1-0.25-dense"):
        rc, n = ref.model_parse(files[name])
        assert rc == 0 and n == 29, name
        assert sp.parse_model_status(files[name]) == 0
        ref_meta = [ref.model_layer(files["mbv1-0.25"], i)[0] for i in range(29)]
        our_meta = [ref.model_layer(files[name], i)[0] for i in range(29)]
        for a, b in zip(ref_meta, our_meta):
            assert (a["kind"], a["cin"], a["cout"], a["residual_src"]) == (b["kind"], b["cin"], b["cout"],
                                                                           b["residual_src"])


def test_reference_files_parse(ref, files):
    for name, data in files.items():
        rc_ref, n_ref = ref.model_parse(data)
        assert rc_ref == 0
        assert sp.parse_model_status(data) == 0, name


def test_canonical_errors_match_reference(ref, files):
    data = files["mbv1-0.25"]
    cases = {
        "bad_magic": b"SPCX" + data[4:],
        "version": data[:4] + bytes([2, 0]) + data[6:],
        "empty": b"",
        "short_magic": data[:3],
        "truncated": data[:len(data) // 2],
        "trailing": data + b"\x00",
        "checksum": data[:-1] + bytes([data[-1] ^ 0xFF]),
    }
    want = {"bad_magic": 8, "version": 9, "empty": 10, "short_magic": 10, "truncated": 10,
            "trailing": 12, "checksum": 11}
    for k, blob in cases.items():
        assert ref.model_parse(blob)[0] == want[k], k
        assert sp.parse_model_status(blob) == want[k], k


@pytest.mark.parametrize("name", [f"{a}-{w}" for a, w, _ in MODELS])
def test_fuzz_typed_errors_match_reference(ref, files, name):
    """Single-byte mutations (re-checksummed half the time so the structural
    checks are reached) and truncations: our status == the reference's."""
    import zlib

    data = bytearray(files[name])
    rng = np.random.default_rng(1234)
    for trial in range(600):
        blob = bytearray(data)
        if trial % 5 == 4:
            blob = blob[: int(rng.integers(0, len(blob)))]
        else:
            pos = int(rng.integers(0, len(blob) - 4))
            blob[pos] = int(rng.integers(0, 256))
            if trial % 2 == 0:  # fix the CRC so the mutation meets the semantic checks
                blob[-4:] = zlib.crc32(bytes(blob[:-4])).to_bytes(4, "little")
        blob = bytes(blob)
        assert sp.parse_model_status(blob) == ref.model_parse(blob)[0], (trial, len(blob))


@pytest.mark.gpu
@pytest.mark.parametrize("name", [f"{a}-{w}" for a, w, _ in MODELS])
def test_device_model_matches_reference_layers(ref, oracle, files, name):
    import torch

    data = files[name]
    m = sp.DeviceModel(data)
    rng = np.random.default_rng(3)
    checked = 0
    for i, L in enumerate(m.layers):
        if L["kind"] not in ("pointwise", "fully_connected"):
            continue
        meta, (rp, ci, va, bias) = ref.model_layer(data, i)
        assert (meta["cin"], meta["cout"]) == (L["cin"], L["cout"])
        if not L["sparse"]:
            continue
        w = m.weights(i)
        back = w.unpack()
        assert back.row_ptr.tobytes() == rp.tobytes()
        assert back.col_idx.tobytes() == ci.tobytes()
        assert back.values.tobytes() == va.tobytes()
        # run_network's pointwise step: padded rows, zero pad bias, truncation, residual
        B, H, W = 2, L["in_h"], L["in_w"]
        act = rng.uniform(-1, 1, (B, L["cin"], H, W)).astype(np.float32)
        mat = sp.BcsrMatrix(meta["rows"], meta["cols"], meta["block_h"], rp, ci, va)
        pad = meta["rows"] - L["cout"]
        fused = ("none", 0, 0) if L["act_kind"] == 0 else ("clamp", 0.0, 6.0)
        want = oracle.spmm(mat, act, np.r_[bias, np.zeros(pad, np.float32)], fused)[:, :L["cout"]]
        want = want.reshape(B, L["cout"], L["out_h"], L["out_w"])
        res = None
        if L["residual_src"] >= 0:
            res = rng.uniform(-1, 1, want.shape).astype(np.float32)
            want = (want + res).astype(np.float32)
        out = torch.empty(want.shape, device="cuda")
        m.run(i, torch.from_numpy(act).cuda(), out,
              None if res is None else torch.from_numpy(res).cuda())
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32)), L
        checked += 1
    assert checked > 5


# ----------------------------------------- the whole executor on the device
@pytest.mark.gpu
@pytest.mark.parametrize("name", [f"{a}-{w}" for a, w, _ in MODELS] + ["ours-mbv1-0.25", "ours-mbv1-0.25-dense"])
def test_device_forward_bit_exact_with_run_network(ref, files, name):
    """spcv_cu_model_forward (entry conv, depthwise, pooling, residuals and the
    sparse / dense 1x1 layers, all on the device) returns the reference
    run_network's logits bit for bit in strict mode; fast mode stays close."""
    import torch

    data = files[name]
    m = sp.DeviceModel(data)
    L0 = m.layers[0]
    B = 3
    x = np.random.default_rng(11).uniform(-1, 1, (B, L0["in_h"], L0["in_w"], L0["cin"])).astype(np.float32)
    want = ref.run_model(data, x)
    got = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    assert got.shape == want.shape
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), float(np.abs(got - want).max())
    fast = m.forward(torch.from_numpy(x).cuda(), strict=False).cpu().numpy()
    assert np.allclose(fast, want, rtol=1e-3, atol=1e-3 * float(np.abs(want).max()))
    # images are independent: a batch of one reproduces its row
    one = m.forward(torch.from_numpy(x[1:2]).cuda()).cpu().numpy()
    assert np.array_equal(one.view(np.uint32), want[1:2].view(np.uint32))


@pytest.mark.gpu
def test_device_forward_checks_input_shape(files):
    import torch

    m = sp.DeviceModel(files["mbv1-0.25"])
    L0 = m.layers[0]
    with pytest.raises(sp.ShapeError):
        m.forward(torch.zeros(1, L0["in_h"] + 1, L0["in_w"], L0["cin"], device="cuda"))
    assert m.forward(torch.zeros(0, L0["in_h"], L0["in_w"], L0["cin"], device="cuda")).shape[0] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mbv1-0.25", "mbv2-0.35", "ours-mbv1-0.25"])
def test_fused_depthwise_pointwise_matches_unfused(ref, files, monkeypatch, name):
    """Depthwise layers fused into the next sparse 1x1 layer's weight-specialised
    kernel (opt-in, SPCV_FUSE_DW=1) give the same bits as running them
    separately (the default) and as the reference run_network, with fewer
    launches."""
    import torch

    data = files[name]
    L0 = sp.DeviceModel(data).layers[0]
    x = np.random.default_rng(5).uniform(-1, 1, (2, L0["in_h"], L0["in_w"], L0["cin"])).astype(np.float32)
    want = ref.run_model(data, x)
    outs, launches = {}, {}
    for fuse in ("1", "0"):
        monkeypatch.setenv("SPCV_FUSE_DW", fuse)
        m = sp.DeviceModel(data)
        xt = torch.from_numpy(x).cuda()
        m.forward(xt)  # compile every variant first
        torch.cuda.synchronize()
        n0 = sp.launch_count()
        outs[fuse] = m.forward(xt).cpu().numpy()
        launches[fuse] = sp.launch_count() - n0
    assert np.array_equal(outs["1"].view(np.uint32), want.view(np.uint32))
    assert np.array_equal(outs["0"].view(np.uint32), want.view(np.uint32))
    assert launches["1"] < launches["0"], launches


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [21, 22, 23])
def test_random_mbv1_files_forward_bit_exact(ref, seed):
    """Python-written MBv1 files with seeded random width / sparsity / input size
    / block plan: spcv_cu_model_forward equals the reference run_network."""
    import torch

    from paper_1911_09723_b200 import netfile

    rng = np.random.default_rng(seed)
    width = float(rng.choice([0.25, 0.5]))
    sparsity = float(rng.choice([0.5, 0.8, 0.95]))
    hw = int(rng.choice([32, 64, 96]))
    net = netfile.build_mbv1(width, sparsity, seed=seed, input_hw=hw, num_classes=int(rng.integers(10, 100)),
                             block_start=int(rng.integers(1, 14)), block_h_after=int(rng.choice([1, 2, 4])))
    data = netfile.serialize(net)
    assert ref.model_parse(data)[0] == 0
    x = rng.uniform(-1, 1, (2, hw, hw, 3)).astype(np.float32)
    want = ref.run_model(data, x)
    m = sp.DeviceModel(data)
    got = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


# --------------------------- entry conv and depthwise layers vs the reference
def _spatial_case(seed, input_hw, width=0.25):
    from paper_1911_09723_b200 import netfile

    net = netfile.build_mbv1(width, 0.9, seed=seed, input_hw=input_hw, num_classes=10)
    return net


def _run_layer(net, i, x, strict=True):
    import torch

    from paper_1911_09723_b200 import netfile

    m = sp.DeviceModel(netfile.serialize(net))
    L = m.layers[i]
    out = torch.empty((x.shape[0], L["cout"], L["out_h"], L["out_w"]), device="cuda")
    m.run(i, torch.from_numpy(np.ascontiguousarray(x)).cuda(), out, strict=strict)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _ref_layer(ref, net, i, x):
    L = net.layers[i]
    kind = 1 if L.act[0] == "clamp" else 0
    b = L.bias if L.bias.size else None
    if i == 0:
        return ref.entry_conv(x, L.weights, b, L.stride, kind, L.act[1], L.act[2])
    return ref.depthwise(x, L.weights, b, L.stride, kind, L.act[1], L.act[2])


def _same_bits(got, want):
    nan = np.isnan(want)
    return np.array_equal(np.isnan(got), nan) and np.array_equal(got[~nan].view(np.uint32),
                                                                 want[~nan].view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("input_hw", [64, 33, 18])
def test_entry_and_depthwise_layers_bit_exact(ref, input_hw):
    """The executor's entry convolution and every depthwise layer (stride 1
    and 2, even and odd planes down to 1x1) through spcv_cu_model_run equal
    the reference's entry_conv_hwc_to_chw / depthwise_conv_chw bit for bit;
    the inputs include exact +0.0 / -0.0 values. Fast mode stays close."""
    net = _spatial_case(7, input_hw)
    rng = np.random.default_rng(input_hw)
    L0 = net.layers[0]
    x = rng.uniform(-1, 1, (3, L0.in_h, L0.in_w, L0.cin)).astype(np.float32)
    x[0, :4] = 0.0
    x[1, :2] = -0.0
    for i, L in enumerate(net.layers):
        if L.kind not in (0, 2):
            continue
        if i > 0:  # depthwise input: a CHW activation with zeros of both signs
            x = rng.uniform(-1, 6, (3, L.cin, L.in_h, L.in_w)).astype(np.float32)
            x[0] = np.where(x[0] < 1.0, 0.0, x[0])
            x[1] = np.where(x[1] < 1.0, -0.0, x[1])
        want = _ref_layer(ref, net, i, x)
        got = _run_layer(net, i, x)
        assert _same_bits(got, want), (L.name, float(np.nanmax(np.abs(got - want))))
        fast = _run_layer(net, i, x, strict=False)
        assert np.allclose(fast, want, rtol=1e-5, atol=1e-5), L.name


@pytest.mark.gpu
def test_spatial_layers_signed_zero_and_nonfinite_weights(ref):
    """Adversarial layers for the zero-padded kernels: a -0.0 bias with +0.0
    inputs and weights whose out-of-image taps are positive (a padded tap
    would turn the -0.0 result into +0.0), and an infinite weight (0 * inf =
    NaN at padded taps). Both make the executor fall back to the per-tap
    kernels, which skip out-of-image taps like the reference: bit-exact (NaN
    where the reference has NaN)."""
    net = _spatial_case(9, 16)
    i_dw = next(i for i, L in enumerate(net.layers) if L.kind == 2 and L.stride == 1)
    L = net.layers[i_dw]
    w = -np.abs(L.weights)
    w[:, 0, :] = 0.5   # top row taps (padded at oy = 0)
    w[:, :, 0] = 0.5   # left column taps (padded at ox = 0)
    L.weights = w.astype(np.float32)
    L.bias = np.full(L.cout, -0.0, np.float32)
    x = np.zeros((2, L.cin, L.in_h, L.in_w), np.float32)
    want = _ref_layer(ref, net, i_dw, x)
    assert np.signbit(want[0, 0, 0, 0]) and want[0, 0, 0, 0] == 0.0  # the reference keeps -0.0
    assert _same_bits(_run_layer(net, i_dw, x), want)
    # the same weights with a +0.0 bias take the zero-padded kernel: still exact
    L.bias = np.zeros(L.cout, np.float32)
    want = _ref_layer(ref, net, i_dw, x)
    assert _same_bits(_run_layer(net, i_dw, x), want)
    # an infinite weight: NaN wherever the reference multiplies it by 0
    L.weights = w.astype(np.float32)
    L.weights[0, 2, 2] = np.inf
    L.bias = (np.random.default_rng(1).standard_normal(L.cout) * 0.1).astype(np.float32)
    x = np.random.default_rng(2).uniform(0, 6, (2, L.cin, L.in_h, L.in_w)).astype(np.float32)
    x[:, 0, 3:5, 3:5] = 0.0
    want = _ref_layer(ref, net, i_dw, x)
    assert np.isnan(want).any()
    assert _same_bits(_run_layer(net, i_dw, x), want)
    # entry conv with a -0.0 bias entry: the per-tap entry kernel, exact
    E = net.layers[0]
    E.bias = E.bias.copy()
    E.bias[0] = -0.0
    E.weights = np.abs(E.weights).astype(np.float32)
    xe = np.zeros((2, E.in_h, E.in_w, E.cin), np.float32)
    want = _ref_layer(ref, net, 0, xe)
    assert _same_bits(_run_layer(net, 0, xe), want)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_forward_graph_replay_matches_run_network(ref, files, mode):
    """A forward repeated with the same tensors on a non-default stream is
    captured once and replayed as a CUDA graph: every replay reads the input's
    current contents and stays bit-identical to the reference run_network
    (strict) / matches the plain launches (fast), and counts the same launches."""
    import torch

    data = files["ours-mbv1-0.25"]
    m = sp.DeviceModel(data)
    L0 = m.layers[0]
    rng = np.random.default_rng(17)
    x = torch.empty((2, L0["in_h"], L0["in_w"], L0["cin"]), device="cuda")
    out = torch.empty((2, m.layers[-1]["cout"]), device="cuda")
    s = torch.cuda.Stream()
    strict = mode == "strict"
    counts = []
    for it in range(5):
        xh = rng.uniform(-1, 1, tuple(x.shape)).astype(np.float32)
        x.copy_(torch.from_numpy(xh))
        torch.cuda.synchronize()
        n0 = sp.launch_count()
        with torch.cuda.stream(s):
            m.forward(x, strict, s, out=out)
        s.synchronize()
        counts.append(sp.launch_count() - n0)
        got = out.cpu().numpy()
        if strict:
            want = ref.run_model(data, xh)
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), it
        else:
            plain = m.forward(torch.from_numpy(xh).cuda(), False).cpu().numpy()  # default stream: no graph
            assert np.allclose(got, plain, rtol=1e-5, atol=1e-6), it
    assert len(set(counts)) == 1 and counts[0] > 10, counts


@pytest.mark.gpu
def test_forward_graph_cache_eviction(ref, files):
    """More distinct (input, logits) pairs than the graph cache holds: entries
    are evicted and re-captured, every forward stays bit-exact."""
    import torch

    data = files["ours-mbv1-0.25"]
    m = sp.DeviceModel(data)
    L0 = m.layers[0]
    rng = np.random.default_rng(23)
    s = torch.cuda.Stream()
    xs = [rng.uniform(-1, 1, (1, L0["in_h"], L0["in_w"], L0["cin"])).astype(np.float32) for _ in range(6)]
    want = [ref.run_model(data, x) for x in xs]
    dev_x = [torch.from_numpy(x).cuda() for x in xs]
    outs = [torch.empty((1, m.layers[-1]["cout"]), device="cuda") for _ in xs]
    for rnd in range(3):
        for x, o, w in zip(dev_x, outs, want):
            with torch.cuda.stream(s):
                m.forward(x, True, s, out=o)
            s.synchronize()
            assert np.array_equal(o.cpu().numpy().view(np.uint32), w.view(np.uint32)), rnd
