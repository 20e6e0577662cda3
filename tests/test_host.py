"""CPU-only checks of the host side: the C-ABI libraries load and export every
declared symbol, host-side format helpers match the oracle, and the Python
mirror of the reference plumbing behaves like kernels.cpp:238-300.
No compute is launched here (no GPU in this container)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from refcases import Mt, random_matrix

import paper_1911_09723_b200 as sp
from paper_1911_09723_b200 import _capi
from paper_1911_09723_b200.workloads import CONFIGS, make_layer_data, mbv1_pointwise, mbv2_pointwise

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spcv_cu.h")
LIBDIR = os.path.join(ROOT, "paper_1911_09723_b200", "lib")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(spcv_cu_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("spcv_cu_pack", "spcv_cu_unpack", "spcv_cu_spmm_into", "spcv_cu_spmm_into_host",
              "spcv_cu_free", "spcv_cu_last_error"):
        assert s in syms


def test_cabi_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(os.path.join(LIBDIR, "libspcv_cu.so"))
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(_capi.SIGNATURES)


def test_cabi_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(LIBDIR, "libspcv_cu.so")],
                         capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


CAP = 1 << 20


def _jit_compile(m, mode, act_kind=1, has_bias=1, has_res=0, m_out=None):
    lib = ctypes.CDLL(os.path.join(LIBDIR, "libspcv_cu.so"))
    fn = lib.spcvx_jit_compile
    P, Z, I = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    fn.argtypes = [I, I, I, P, P, Z, P, I, I, I, I, I, I, ctypes.POINTER(I), ctypes.POINTER(Z),
                   ctypes.POINTER(Z), ctypes.c_char_p, Z]
    rp = np.ascontiguousarray(m.row_ptr, np.uint32)
    ci = np.ascontiguousarray(m.col_idx, np.uint32)
    va = np.ascontiguousarray(m.values, np.float32)
    sb, cb, nseg = Z(), Z(), I()
    buf = ctypes.create_string_buffer(CAP)
    rc = fn(m.rows, m.cols, m.block_h, rp.ctypes.data, ci.ctypes.data if ci.size else None, ci.size,
            va.ctypes.data if va.size else None, mode, act_kind, has_bias, has_res,
            m.rows if m_out is None else m_out, 148, ctypes.byref(nseg), ctypes.byref(sb),
            ctypes.byref(cb), buf, CAP)
    return rc, buf.value.decode(), cb.value, nseg.value


def _jit_terms(src):
    """(segment, accumulator) -> [(channel, weight bits, op)] in program order,
    parsed from the generated k-major source (chunk = one issue() per 32 channels)."""
    terms, seg, kc = {}, -1, -1
    for line in src.splitlines():
        m = re.match(r"__device__ __forceinline__ void seg(\d+)\(", line)
        if m:
            seg, kc = int(m.group(1)), -1
            continue
        if line.strip() == "issue();":
            kc += 1
        m = re.search(r"LDS(64|32)\(x, xs, (\d+)\)", line)
        if m:  # offset = channel-in-chunk x columns per group (64 or 32) x 4 B
            k = kc * 32 + int(m.group(2)) // (256 if m.group(1) == "64" else 128)
        m = re.search(r"a(\d+) = fma2\(a\d+, one, mul2\(0x([0-9a-f]{8})[0-9a-f]{8}ULL, x\)\)", line)
        if m:
            terms.setdefault((seg, int(m.group(1))), []).append((k, int(m.group(2), 16), "strict"))
        m = re.search(r"a(\d+) = fma2\(0x([0-9a-f]{8})[0-9a-f]{8}ULL, x, a\d+\)", line)
        if m:
            terms.setdefault((seg, int(m.group(1))), []).append((k, int(m.group(2), 16), "fast"))
        m = re.search(r"a(\d+) = __fadd_rn\(a\d+, __fmul_rn\(__uint_as_float\(0x([0-9a-f]{8})u\), x\)\)", line)
        if m:  # one column per lane (scalar) k-major variant
            terms.setdefault((seg, int(m.group(1))), []).append((k, int(m.group(2), 16), "strict"))
    return terms


def test_jit_kernel_source_and_nvrtc_compile_without_gpu(monkeypatch):
    """The weight-specialised kernel (jit.cu) is planned, generated and compiled
    by NVRTC for sm_100a without a device. Every stored weight of every row
    (zeros inside stored blocks included) appears exactly once as an immediate,
    in ascending channel order, split over row segments that cover the rows."""
    monkeypatch.setenv("SPCV_JIT_SEG_INSTR", "200")  # force several segments
    monkeypatch.setenv("SPCV_JIT_MAX_SEGS", "48")
    rng = np.random.default_rng(3)
    dense = rng.standard_normal((12, 70)).astype(np.float32)
    dense[rng.random((12, 70)) < 0.7] = 0
    m = sp.encode_bcsr(dense, 2)
    rp, ci, va = np.asarray(m.row_ptr), np.asarray(m.col_idx), np.asarray(m.values)
    for mode, m_out in ((_capi.MODE_STRICT, 12), (_capi.MODE_FAST, 11)):
        rc, src, cubin, nseg = _jit_compile(m, mode, m_out=m_out)
        assert rc == 0 and cubin > 0 and nseg > 1
        terms = _jit_terms(src)
        rows = []
        for seg in range(nseg):
            body = src.split("void seg%d(" % seg)[1].split("__device__")[0]
            rows += [int(r) for r in re.findall(r"// row (\d+)", body)]
        assert rows == list(range(m_out))  # segments partition the stored rows, in order
        r = 0
        for seg in range(nseg):
            q = 0
            while (seg, q) in terms or (r < m_out and rp[r // 2] == rp[r // 2 + 1]):
                blks = range(rp[r // 2], rp[r // 2 + 1])
                want = [(int(ci[b]), int(va[2 * b + r % 2].view(np.uint32)),
                         "strict" if mode == _capi.MODE_STRICT else "fast") for b in blks]
                assert terms.get((seg, q), []) == want, (seg, q, r)
                q += 1
                r += 1
        assert r == m_out


def test_jit_single_segment_one_column_per_lane(monkeypatch):
    """A 128-row matrix that needs two 2-column segments fits one segment at one
    column per lane: the planner picks it (activations read once), and every
    row's terms are still its stored weights in ascending channel order."""
    monkeypatch.delenv("SPCV_JIT_SEG_INSTR", raising=False)
    monkeypatch.delenv("SPCV_JIT_MAX_SEGS", raising=False)
    rng = np.random.default_rng(9)
    dense = rng.standard_normal((128, 128)).astype(np.float32)
    dense[rng.random((128, 128)) < 0.9] = 0
    m = sp.encode_bcsr(dense, 1)
    rc, src, cubin, nseg = _jit_compile(m, _capi.MODE_STRICT)
    assert rc == 0 and nseg == 1 and "LDS32(" in src and "LDS64(" not in src.split("void seg0")[1]
    rp, ci, va = np.asarray(m.row_ptr), np.asarray(m.col_idx), np.asarray(m.values)
    terms = _jit_terms(src)
    for r in range(128):
        want = [(int(ci[b]), int(va[b].view(np.uint32)), "strict") for b in range(rp[r], rp[r + 1])]
        assert terms.get((0, r), []) == want, r


def test_jit_direct_variant_source(monkeypatch):
    """Small K (<= 64): the direct variant (one thread per column). Each row's
    terms appear in ascending channel order with the exact stored weights."""
    monkeypatch.delenv("SPCV_JIT_SEG_INSTR", raising=False)
    rng = np.random.default_rng(4)
    dense = rng.standard_normal((10, 20)).astype(np.float32)
    dense[rng.random((10, 20)) < 0.6] = 0
    m = sp.encode_bcsr(dense, 1)
    rp, ci, va = np.asarray(m.row_ptr), np.asarray(m.col_idx), np.asarray(m.values)
    rc, src, cubin, nseg = _jit_compile(m, _capi.MODE_STRICT)
    assert rc == 0 and cubin > 0 and nseg == 0
    block, rows_seen = {}, []
    for line in src.splitlines():
        if line.strip() == "{":
            block = {}
        t = re.search(r"a(\d+) = __fadd_rn\(a\d+, __fmul_rn\(__uint_as_float\(0x([0-9a-f]{8})u\), x(\d+)\)\)", line)
        if t:
            block.setdefault(int(t.group(1)), []).append((int(t.group(3)), int(t.group(2), 16)))
        st = re.search(r"__stcs\(o \+ (\d+)LL \* S, a(\d+)\);", line)
        if st:
            r = int(st.group(1))
            rows_seen.append(r)
            want = [(int(ci[b]), int(va[b].view(np.uint32))) for b in range(rp[r], rp[r + 1])]
            assert block.get(int(st.group(2)), []) == want, r
    assert rows_seen == list(range(10))


MASK_CASES = [(8, 8, 0.5, 2, 1, 1234), (10, 1, 0.25, 1, 1, 5), (4, 4, 0.0, 1, 1, 5), (4, 4, 0.999, 1, 1, 5),
              (16, 12, 0.7, 4, 2, 77), (64, 64, 0.9, 1, 1, 42), (64, 32, 0.8, 4, 1, 9),
              (128, 128, 0.8, 1, 1, 3), (512, 512, 0.9, 4, 1, 11), (30, 30, 0.5, 4, 1, 1), (8, 8, 1.0, 1, 1, 1)]


def test_generate_mask_mirrors_match_reference(ref):
    """generate_mask (sparse.cpp:63-98) in the Python and C++ mirrors: the same
    keep bits as the compiled reference (std::mt19937 + libstdc++'s
    uniform_int_distribution), the same errors, test_sparse.cpp popcounts."""
    exe = os.path.join(ROOT, "tests", "cpp", "test_mask")
    r = subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include",
                        os.path.join(ROOT, "tests", "cpp", "test_mask.cpp"), "-o", exe,
                        f"-L{LIBDIR}", "-lspcv_b200", "-lspcv_cu", f"-Wl,-rpath,{LIBDIR}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    args = [str(v) for case in MASK_CASES for v in case]
    out = subprocess.run([exe] + args, capture_output=True, text=True).stdout.split("\n")
    os.remove(exe)
    for (rows, cols, s, ob, ib, seed), line in zip(MASK_CASES, out):
        rc, want = ref.generate_mask(rows, cols, s, ob, ib, seed)
        if rc != 0:  # reference rejected: both mirrors reject with the mapped error
            assert line in ("FormatError", "invalid_argument")
            with pytest.raises((sp.FormatError, ValueError)):
                sp.generate_mask(rows, cols, s, sp.BlockConfig(ob, ib), seed)
            continue
        got_py = sp.generate_mask(rows, cols, s, sp.BlockConfig(ob, ib), seed)
        assert np.array_equal(got_py, want), (rows, cols, s, ob, ib, seed)
        pop, bits_ = line.split()
        got_cpp = np.frombuffer(bits_.encode(), dtype=np.uint8).reshape(rows, cols) == ord("1")
        assert np.array_equal(got_cpp, want) and int(pop) == int(want.sum())
    assert [int(l.split()[0]) for l in out[:4]] == [32, 7, 16, 0]  # test_sparse.cpp:73-104
    w = np.ones((4, 4), np.float32)
    keep = sp.generate_mask(4, 4, 0.5, sp.BlockConfig(), 1)
    assert np.array_equal(sp.apply_mask(w, keep) != 0, keep)
    with pytest.raises(sp.ShapeError):
        sp.apply_mask(np.ones((3, 4), np.float32), keep)


def test_cpp_dropin_library_exports_reference_api():
    so = os.path.join(LIBDIR, "libspcv_b200.so")
    out = subprocess.run(["nm", "-DC", so], capture_output=True, text=True).stdout
    for sym in ("spcv::spmm_into(", "spcv::spmm(", "spcv::encode_bcsr(", "spcv::decode_bcsr(",
                "spcv::BcsrMatrix::validate() const", "spcv::DeviceBcsr::DeviceBcsr(",
                "spcv::spmm_batched_into(", "spcv::parse_variant("):
        assert sym in out, sym


def test_version_and_launch_counter_without_gpu():
    assert b"sm_100a" in _capi.lib.spcv_cu_version()
    assert sp.launch_count() == 0 or sp.launch_count() > 0


def test_pack_reports_cuda_error_without_gpu_or_format_error_first():
    # A malformed matrix is rejected before any device work (FormatError).
    bad = sp.BcsrMatrix(4, 4, 3, np.array([0, 0], np.uint32), np.zeros(0, np.uint32),
                        np.zeros(0, np.float32))
    with pytest.raises(sp.FormatError):
        sp.DeviceBcsr(bad)


def test_encode_decode_match_oracle(oracle):
    rng = Mt(99)
    for bh in (1, 2, 4):
        for _ in range(20):
            rows = bh * (1 + int(rng() % 12))
            cols = 1 + int(rng() % 40)
            s = (rng() % 100) / 100.0
            w = random_matrix(rows, cols, rng)
            rc, keep = oracle.generate_mask(rows, cols, s, bh, 1, rng())
            w[~keep] = 0
            m = sp.encode_bcsr(w, bh)
            rc, (rp, ci, va) = oracle.encode_bcsr(w, bh)
            assert np.array_equal(m.row_ptr, rp) and np.array_equal(m.col_idx, ci)
            assert np.array_equal(m.values.view(np.uint32), va.view(np.uint32))
            m.validate()
            assert np.array_equal(sp.decode_bcsr(m), w)


def test_encode_known_answers():
    # test_sparse.cpp:9-41
    m = sp.encode_bcsr(np.zeros((2, 2), np.float32), 1)
    assert m.row_ptr.tolist() == [0, 0, 0] and m.nnz_blocks() == 0
    m = sp.encode_bcsr(np.eye(2, dtype=np.float32), 2)
    assert m.row_ptr.tolist() == [0, 2] and m.col_idx.tolist() == [0, 1]
    assert m.values.tolist() == [1.0, 0.0, 0.0, 1.0] and m.nnz_values() == 4
    w = np.zeros((4, 3), np.float32)
    w[1, 2] = 5
    m = sp.encode_bcsr(w, 2)
    assert m.row_ptr.tolist() == [0, 1, 1] and m.col_idx.tolist() == [2]
    assert m.values.tolist() == [0.0, 5.0]
    with pytest.raises(sp.ShapeError):
        sp.encode_bcsr(np.zeros((3, 4), np.float32), 2)
    # -0.0 is zero for the keep test (sparse.cpp:124)
    m = sp.encode_bcsr(np.array([[-0.0, 1.0]], np.float32), 1)
    assert m.col_idx.tolist() == [1]


def test_validate_rejections_match_oracle(oracle):
    w = np.zeros((4, 4), np.float32)
    w[0, 1], w[2, 3] = 1, 2
    g = sp.encode_bcsr(w, 2)
    rp, ci, va = g.row_ptr, g.col_idx, g.values
    bad = [
        (5, 4, 2, rp, ci, va),
        (4, 4, 2, np.r_[1, rp[1:]].astype(np.uint32), ci, va),
        (4, 4, 2, np.r_[rp[0], 3, rp[2:]].astype(np.uint32), ci, va),
        (4, 4, 2, np.r_[rp[:-1], 1].astype(np.uint32), ci, va),
        (4, 4, 2, rp, np.r_[99, ci[1:]].astype(np.uint32), va),
        (4, 4, 2, rp, ci, np.r_[va, 0].astype(np.float32)),
        (4, 4, 3, rp, ci, va),
        (2, 4, 1, np.array([0, 2, 2], np.uint32), np.array([2, 1], np.uint32),
         np.array([1.0, 2.0], np.float32)),
    ]
    for args in bad:
        assert oracle.validate(*args) == 3
        with pytest.raises(sp.FormatError):
            sp.BcsrMatrix(*args).validate()
        with pytest.raises(sp.FormatError):  # the C-ABI packer rejects it the same way
            sp.DeviceBcsr(sp.BcsrMatrix(*args))


def test_variant_and_tier_parsing():
    # test_kernels.cpp:355-366
    assert sp.parse_variant("16x2") == (16, 2)
    assert sp.parse_variant("4x1") == (4, 1)
    assert sp.variant_name(8, 4) == "8x4"
    for bad in ["", "16", "x2", "16x", "16x3", "5x2", "16x2x1", "a.b"]:
        with pytest.raises(ValueError):
            sp.parse_variant(bad)
    assert sp.parse_tier("scalar") == sp.Tier.Scalar
    with pytest.raises(ValueError):
        sp.parse_tier("turbo")


def test_tier_env_override(monkeypatch):
    # test_kernels.cpp:368-381
    assert sp.resolve_tier(sp.Tier.Auto) == sp.Tier.Vector
    monkeypatch.setenv("SPCV_FORCE_SCALAR", "1")
    assert sp.resolve_tier(sp.Tier.Auto) == sp.Tier.Scalar
    monkeypatch.setenv("SPCV_FORCE_SCALAR", "0")
    assert sp.resolve_tier(sp.Tier.Auto) == sp.Tier.Vector
    assert sp.default_strip_width(sp.Tier.Scalar) == 8
    assert sp.default_strip_width(sp.Tier.Vector) == 16


def test_activation_contract():
    with pytest.raises(ValueError):
        sp.Activation.clamp(1.0, 1.0)
    r6 = sp.Activation.relu6()
    assert (r6.kind, r6.lo, r6.hi) == (1, 0.0, 6.0)


def test_host_argument_checks_precede_device_work():
    """spmm_into validation order (kernels.cpp:306-322) with host tensors; all
    of these fail before any CUDA call, so they run without a GPU."""
    w = sp.encode_bcsr(np.eye(8, dtype=np.float32), 2)
    act = sp.Tensor(8, 2, 2)
    out = sp.Tensor(8, 2, 2)
    cfg = sp.MicrokernelConfig(n=4)
    with pytest.raises(sp.FormatError):
        sp.spmm_into(w, act, None, sp.Activation.none(), out, cfg)
    with pytest.raises(sp.ShapeError):
        sp.spmm_into(w, sp.Tensor(9, 2, 2), None, sp.Activation.none(), out, sp.MicrokernelConfig(n=2))
    with pytest.raises(sp.LayoutError):
        sp.spmm_into(w, sp.Tensor(8, 2, 2, sp.Layout.HWC), None, sp.Activation.none(), out,
                     sp.MicrokernelConfig(n=2))
    with pytest.raises(ValueError):
        sp.spmm_into(w, act, None, sp.Activation.none(), out, sp.MicrokernelConfig(m=5, n=2))
    with pytest.raises(sp.ShapeError):
        sp.spmm_into(w, act, np.zeros(3, np.float32), sp.Activation.none(), out, sp.MicrokernelConfig(n=2))
    with pytest.raises(sp.ShapeError):
        sp.spmm_into(w, act, None, sp.Activation.none(), sp.Tensor(8, 2, 3), sp.MicrokernelConfig(n=2))


def test_workload_shapes():
    v1 = mbv1_pointwise()
    assert [(l.cin, l.cout, l.h) for l in v1][:3] == [(32, 64, 112), (64, 128, 56), (128, 128, 56)]
    assert len(v1) == 13 and v1[-1].cin == 1024 and v1[-1].h == 7
    v2 = mbv2_pointwise()
    names = [(l.cin, l.cout, l.h) for l in v2]
    for want in [(24, 144, 56), (32, 192, 28), (64, 384, 14), (160, 960, 7), (144, 24, 56),
                 (192, 32, 28), (384, 64, 14), (960, 160, 7), (32, 16, 112), (16, 96, 112),
                 (96, 24, 56), (960, 320, 7), (320, 1280, 7)]:
        assert want in names
    assert set(CONFIGS) == {"c1", "c2-b1", "c2-b256", "c3", "c4", "c5"}


def test_skewed_rows_mean_density():
    from paper_1911_09723_b200.workloads import c5_layer

    d = make_layer_data(c5_layer(0.9), 1, 5, act=False)
    counts = np.diff(d.weights.row_ptr.astype(np.int64))
    assert abs(counts.mean() / 1024 - 0.10) < 0.01
    assert counts.max() / counts.mean() > 2.0  # heavy-tailed rows


def test_uniform_mask_exact_count():
    d = make_layer_data(mbv1_pointwise()[0], 1, 1, act=False)
    assert d.weights.nnz_values() == 2048 - int(np.floor(2048 * 0.9 + 0.5))


def test_bench_layers_csv_schema_matches_reference():
    """tools/bench_layers.py emits the reference's 11-column schema
    (bench.cpp:428-445) with %.17g doubles."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "bench_layers", os.path.join(ROOT, "tools", "bench_layers.py"))
    bl = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bl)
    assert bl.CSV_HEADER == ("layer_index,kind,cout,cin,spatial,sparsity,block_h,variant,median_ns,"
                             "achieved_gflops,effective_gflops")
    text = bl.rows_to_csv([dict(layer_index=2, kind="pointwise", cout=64, cin=32, spatial=12544,
                                sparsity=0.9, block_h=1, variant="b200-strict", median_ns=1234.5,
                                achieved_gflops=0.1, effective_gflops=1.0 / 3.0)])
    lines = text.strip().split("\n")
    assert lines[0] == bl.CSV_HEADER
    assert lines[1] == "2,pointwise,64,32,12544,0.90000000000000002,1,b200-strict,1234.5,0.10000000000000001,0.33333333333333331"


def test_network_layer_indices():
    v1 = mbv1_pointwise()
    assert [l.net_index for l in v1] == [2 * i for i in range(1, 14)]
    v2 = mbv2_pointwise()
    assert v2[0].name == "b1_project" and v2[0].net_index == 2  # entry, dw, project
    assert v2[1].name == "b2_expand" and v2[1].net_index == 3
    assert v2[-1].name == "head" and v2[-1].net_index == 51  # 16 expands + 17 (dw, project) + entry
