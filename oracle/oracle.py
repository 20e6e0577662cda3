"""ctypes access to the CPU checkers. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the reported CPU baseline — never as the thing measured or shipped.

  Oracle  — liboracle.so: the in-repo C restatement (spcv_oracle.c, spcv_mask.cpp)
  Ref     — _ref/libspcv_ref.so: the unmodified reference library, compiled in
            place from /root/reference by oracle/Makefile (absent if the
            reference was never available to build it)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspcv_ref.so")

_p, _i, _f, _z, _d = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_size_t, ctypes.c_double


def _ptr(a):
    return None if a is None or a.size == 0 else a.ctypes.data


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _act(fused):
    """(kind, lo, hi) from an Activation-like object or tuple."""
    if fused is None:
        return 0, 0.0, 0.0
    if isinstance(fused, tuple):
        return (0, 0.0, 0.0) if fused[0] == "none" else (1, float(fused[1]), float(fused[2]))
    return int(fused.kind), float(fused.lo), float(fused.hi)


class Oracle:
    """The C restatement (oracle/spcv_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle`")
        lib = ctypes.CDLL(path)
        lib.oracle_matmul_reference.argtypes = [_i, _i, _i, _p, _p, _p, _i, _f, _f, _p]
        lib.oracle_spmm_bcsr.argtypes = [_i, _i, _i, _p, _p, _p, _i, _p, _p, _i, _f, _f, _p]
        lib.oracle_spmm_bcsr_batched.argtypes = [_i, _i, _i, _p, _p, _p, _i, _i, _p, _p, _i, _f,
                                                 _f, _p, _i]
        lib.oracle_encode_bcsr.argtypes = [_i, _i, _i, _p, _p, _p, _p, ctypes.POINTER(_z)]
        lib.oracle_validate_bcsr.argtypes = [_i, _i, _i, _p, _z, _p, _z, _z]
        lib.oracle_decode_bcsr.argtypes = [_i, _i, _i, _p, _z, _p, _z, _p, _z, _p]
        lib.oracle_generate_mask.argtypes = [_i, _i, _d, _i, _i, ctypes.c_uint32, _p]
        self.lib = lib

    def matmul_reference(self, w, act, bias, fused):
        """tensor.cpp:38-62 on one image: w [M][K], act [K][S] -> [M][S]."""
        w, act = _f32(w), _f32(act)
        M, K = w.shape
        S = act.size // K
        out = np.empty((M, S), np.float32)
        b = None if bias is None or len(bias) == 0 else _f32(bias)
        k, lo, hi = _act(fused)
        rc = self.lib.oracle_matmul_reference(M, K, S, _ptr(w), _ptr(act), _ptr(b), k, lo, hi,
                                              _ptr(out))
        assert rc == 0, rc
        return out

    def spmm(self, m, act, bias, fused, nthreads: int = 1):
        """kernels.cpp:14-43/101-130 semantics; act [B][K][S...] -> [B][M][S]."""
        act = _f32(act)
        B = act.shape[0]
        S = act[0].size // m.cols
        out = np.empty((B, m.rows, S), np.float32)
        b = None if bias is None or len(bias) == 0 else _f32(bias)
        k, lo, hi = _act(fused)
        rp, ci, va = _u32(m.row_ptr), _u32(m.col_idx), _f32(m.values)
        rc = self.lib.oracle_spmm_bcsr_batched(m.rows, m.cols, m.block_h, _ptr(rp), _ptr(ci),
                                               _ptr(va), B, S, _ptr(act), _ptr(b), k, lo, hi,
                                               _ptr(out), nthreads)
        assert rc == 0, rc
        return out

    def encode_bcsr(self, w, block_h):
        w = _f32(w)
        M, K = w.shape
        rp = np.zeros(M // block_h + 1 if block_h in (1, 2, 4) else 1, np.uint32)
        ci = np.zeros(max(M // max(block_h, 1) * K, 1), np.uint32)
        va = np.zeros(max(M * K, 1), np.float32)
        nb = _z(0)
        rc = self.lib.oracle_encode_bcsr(M, K, block_h, _ptr(w), _ptr(rp), _ptr(ci), _ptr(va),
                                         ctypes.byref(nb))
        if rc:
            return rc, None
        n = nb.value
        return 0, (rp, ci[:n].copy(), va[: n * block_h].copy())

    def validate(self, rows, cols, block_h, row_ptr, col_idx, values) -> int:
        rp, ci = _u32(row_ptr), _u32(col_idx)
        return self.lib.oracle_validate_bcsr(rows, cols, block_h, _ptr(rp), rp.size, _ptr(ci),
                                             ci.size, int(np.asarray(values).size))

    def generate_mask(self, rows, cols, sparsity, out_block, in_block, seed):
        keep = np.zeros(rows * cols, np.uint8)
        rc = self.lib.oracle_generate_mask(rows, cols, sparsity, out_block, in_block, seed,
                                           _ptr(keep))
        return rc, keep.reshape(rows, cols).astype(bool)


class RefLayer(ctypes.Structure):
    _fields_ = [("rows", _i), ("cols", _i), ("block_h", _i), ("row_ptr", _p), ("nrp", _z),
                ("col_idx", _p), ("nblk", _z), ("values", _p), ("nval", _z), ("images", _i),
                ("H", _i), ("W", _i), ("act", _p), ("bias", _p), ("act_kind", _i), ("lo", _f),
                ("hi", _f)]


class Ref:
    """The unmodified reference (oracle/_ref/libspcv_ref.so via oracle/ref_shim.cpp)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle ref` where /root/reference exists")
        lib = ctypes.CDLL(path)
        lib.ref_spmm.argtypes = [_i, _i, _i, _p, _z, _p, _z, _p, _z, _i, _i, _i, _i, _i, _p, _p, _z,
                                 _i, _f, _f, _i, _p, _i, _i, _i, _i]
        lib.ref_matmul_reference.argtypes = [_i, _i, _i, _i, _p, _p, _p, _i, _f, _f, _p]
        lib.ref_encode_bcsr.argtypes = [_i, _i, _i, _p, _p, _p, _p, ctypes.POINTER(_z)]
        lib.ref_validate_bcsr.argtypes = [_i, _i, _i, _p, _z, _p, _z, _p, _z]
        lib.ref_generate_mask.argtypes = [_i, _i, _d, _i, _i, ctypes.c_uint32, _p]
        lib.ref_model_bytes.argtypes = [ctypes.c_char_p, _d, _d, ctypes.c_uint32, _p, _z,
                                        ctypes.POINTER(_z)]
        lib.ref_model_parse.argtypes = [_p, _z, ctypes.POINTER(_i)]
        lib.ref_run_model.argtypes = [_p, _z, _p, _i, _i, _p, ctypes.POINTER(_i)]
        lib.ref_model_layer.argtypes = [_p, _z, _i, _p, _p, _p, _p, _p]
        lib.ref_bench_layers.argtypes = [ctypes.POINTER(RefLayer), _i, _i, _i, _i, ctypes.POINTER(_d)]
        lib.ref_depthwise.argtypes = [_i, _i, _i, _i, _i, _p, _p, _i, _f, _f, _p, _p, ctypes.POINTER(_i),
                                      ctypes.POINTER(_i)]
        lib.ref_entry_conv.argtypes = [_i, _i, _i, _i, _i, _i, _p, _p, _i, _f, _f, _p, _p, ctypes.POINTER(_i),
                                       ctypes.POINTER(_i)]
        lib.ref_bench_spmm.argtypes = [_i, _i, _i, _p, _z, _p, _z, _p, _z, _i, _i, _i, _p, _p, _i,
                                       _f, _f, _p, _i, _i, _i, ctypes.POINTER(_d)]
        self.lib = lib

    def spmm(self, m, act, bias, fused, H=None, W=None, cfg_m=0, cfg_n=None, prefetch=1, tier=2,
             act_layout=0, out_channels=None, act_channels=None):
        """spcv::spmm_into per image. act [B][K][H][W] (or [B][K][S] with H=1)."""
        act = _f32(act)
        B = act.shape[0]
        K = act_channels if act_channels is not None else m.cols
        if H is None:
            if act.ndim == 4:
                H, W = act.shape[2], act.shape[3]
            else:
                H, W = 1, act[0].size // K
        oc = m.rows if out_channels is None else out_channels
        out = np.zeros((B, oc, H * W), np.float32)
        b = None if bias is None or len(bias) == 0 else _f32(bias)
        k, lo, hi = _act(fused)
        rp, ci, va = _u32(m.row_ptr), _u32(m.col_idx), _f32(m.values)
        rc = self.lib.ref_spmm(m.rows, m.cols, m.block_h, _ptr(rp), rp.size, _ptr(ci), ci.size,
                               _ptr(va), va.size, B, K, H, W, act_layout, _ptr(act), _ptr(b),
                               0 if b is None else b.size, k, lo, hi, oc, _ptr(out), cfg_m,
                               m.block_h if cfg_n is None else cfg_n, prefetch, tier)
        return rc, out

    def matmul_reference(self, w, act, bias, fused, H, W):
        w, act = _f32(w), _f32(act)
        M, K = w.shape
        out = np.empty((M, H * W), np.float32)
        b = None if bias is None or len(bias) == 0 else _f32(bias)
        k, lo, hi = _act(fused)
        rc = self.lib.ref_matmul_reference(M, K, H, W, _ptr(w), _ptr(act), _ptr(b), k, lo, hi,
                                           _ptr(out))
        assert rc == 0, rc
        return out

    def encode_bcsr(self, w, block_h):
        w = _f32(w)
        M, K = w.shape
        rp = np.zeros(M // block_h + 1 if block_h in (1, 2, 4) and M % block_h == 0 else 1, np.uint32)
        ci = np.zeros(max(M * K, 1), np.uint32)
        va = np.zeros(max(M * K, 1), np.float32)
        nb = _z(0)
        rc = self.lib.ref_encode_bcsr(M, K, block_h, _ptr(w), _ptr(rp), _ptr(ci), _ptr(va),
                                      ctypes.byref(nb))
        if rc:
            return rc, None
        n = nb.value
        return 0, (rp, ci[:n].copy(), va[: n * block_h].copy())

    def validate(self, rows, cols, block_h, row_ptr, col_idx, values) -> int:
        rp, ci, va = _u32(row_ptr), _u32(col_idx), _f32(values)
        return self.lib.ref_validate_bcsr(rows, cols, block_h, _ptr(rp), rp.size, _ptr(ci), ci.size,
                                          _ptr(va), va.size)

    def generate_mask(self, rows, cols, sparsity, out_block, in_block, seed):
        keep = np.zeros(rows * cols, np.uint8)
        rc = self.lib.ref_generate_mask(rows, cols, sparsity, out_block, in_block, seed, _ptr(keep))
        return rc, keep.reshape(rows, cols).astype(bool)

    def bench_spmm(self, m, act, bias, fused, nthreads, warmups=1, reps=1, out=None):
        """Timed reference spmm_into over act [B][K][H][W]; returns per-rep seconds."""
        act = _f32(act)
        B, K, H, W = act.shape
        b = None if bias is None or len(bias) == 0 else _f32(bias)
        k, lo, hi = _act(fused)
        rp, ci, va = _u32(m.row_ptr), _u32(m.col_idx), _f32(m.values)
        secs = (_d * reps)()
        rc = self.lib.ref_bench_spmm(m.rows, m.cols, m.block_h, _ptr(rp), rp.size, _ptr(ci),
                                     ci.size, _ptr(va), va.size, B, H, W, _ptr(act), _ptr(b), k,
                                     lo, hi, None if out is None else _ptr(out), nthreads, warmups,
                                     reps, secs)
        assert rc == 0, rc
        return [secs[i] for i in range(reps)]


    def model_bytes(self, arch: str, width: float, sparsity: float, seed: int) -> bytes:
        """serialize_model(build_network(arch, width, default_plan(arch, sparsity)),
        instantiate_weights(seed)) — a reference model file."""
        n = _z(0)
        rc = self.lib.ref_model_bytes(arch.encode(), width, sparsity, seed, None, 0, ctypes.byref(n))
        assert rc == 0, rc
        buf = np.zeros(n.value, np.uint8)
        rc = self.lib.ref_model_bytes(arch.encode(), width, sparsity, seed, buf.ctypes.data, buf.size,
                                      ctypes.byref(n))
        assert rc == 0, rc
        return buf.tobytes()

    def run_model(self, data: bytes, images_hwc: np.ndarray, reference_executor: bool = False) -> np.ndarray:
        """run_network (or run_network_reference) per image: [B][H][W][C] -> logits [B][classes]."""
        buf = np.frombuffer(data, dtype=np.uint8)
        x = np.ascontiguousarray(images_hwc, dtype=np.float32)
        classes = _i()
        rc = self.lib.ref_run_model(buf.ctypes.data, buf.size, None, 0, 0, None, ctypes.byref(classes))
        if rc:
            raise RuntimeError(f"ref_run_model: code {rc}")
        out = np.zeros((x.shape[0], classes.value), np.float32)
        rc = self.lib.ref_run_model(buf.ctypes.data, buf.size, x.ctypes.data, x.shape[0],
                                    1 if reference_executor else 0, out.ctypes.data, ctypes.byref(classes))
        if rc:
            raise RuntimeError(f"ref_run_model: code {rc}")
        return out

    def depthwise(self, x, w, bias, stride, act_kind=0, lo=0.0, hi=0.0):
        """spcv::depthwise_conv_chw per image: x [B][C][H][W], w [C][3][3] -> [B][C][OH][OW]."""
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        b = None if bias is None else np.ascontiguousarray(bias, np.float32)
        B, C, H, W = x.shape
        oh, ow = (H + stride - 1) // stride, (W + stride - 1) // stride  # same_pad out
        out = np.zeros((B, C, oh, ow), np.float32)
        r_oh, r_ow = _i(), _i()
        rc = self.lib.ref_depthwise(B, C, H, W, stride, w.ctypes.data, None if b is None else b.ctypes.data,
                                    act_kind, lo, hi, x.ctypes.data, out.ctypes.data, ctypes.byref(r_oh),
                                    ctypes.byref(r_ow))
        assert rc == 0 and (B == 0 or (r_oh.value, r_ow.value) == (oh, ow)), rc
        return out

    def entry_conv(self, x_hwc, w, bias, stride, act_kind=0, lo=0.0, hi=0.0):
        """spcv::entry_conv_hwc_to_chw per image: x [B][H][W][C], w [CO][C][3][3] -> [B][CO][OH][OW]."""
        x = np.ascontiguousarray(x_hwc, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        b = None if bias is None else np.ascontiguousarray(bias, np.float32)
        B, H, W, C = x.shape
        CO = w.shape[0]
        oh, ow = (H + stride - 1) // stride, (W + stride - 1) // stride  # same_pad out
        out = np.zeros((B, CO, oh, ow), np.float32)
        r_oh, r_ow = _i(), _i()
        rc = self.lib.ref_entry_conv(B, C, H, W, CO, stride, w.ctypes.data, None if b is None else b.ctypes.data,
                                     act_kind, lo, hi, x.ctypes.data, out.ctypes.data, ctypes.byref(r_oh),
                                     ctypes.byref(r_ow))
        assert rc == 0 and (B == 0 or (r_oh.value, r_ow.value) == (oh, ow)), rc
        return out

    def model_parse(self, data: bytes):
        """parse_model: (status code, layer count)."""
        buf = np.frombuffer(data, np.uint8)
        layers = _i(0)
        rc = self.lib.ref_model_parse(buf.ctypes.data if buf.size else None, buf.size, ctypes.byref(layers))
        return rc, layers.value

    def model_layer(self, data: bytes, i: int):
        """Layer i of parse_model: meta dict and (row_ptr, col_idx, values, bias)."""
        buf = np.frombuffer(data, np.uint8)
        meta = np.zeros(12, np.int32)
        rc = self.lib.ref_model_layer(buf.ctypes.data, buf.size, i, meta.ctypes.data, None, None, None, None)
        assert rc == 0, rc
        names = ["kind", "cin", "cout", "is_sparse", "rows", "cols", "block_h", "nrp", "nblk", "nval",
                 "nbias", "residual_src"]
        m = dict(zip(names, meta.tolist()))
        rp = np.zeros(max(m["nrp"], 1), np.uint32)
        ci = np.zeros(max(m["nblk"], 1), np.uint32)
        va = np.zeros(max(m["nval"], 1), np.float32)
        bi = np.zeros(max(m["nbias"], 1), np.float32)
        rc = self.lib.ref_model_layer(buf.ctypes.data, buf.size, i, meta.ctypes.data, rp.ctypes.data,
                                      ci.ctypes.data, va.ctypes.data, bi.ctypes.data)
        assert rc == 0, rc
        return m, (rp[:m["nrp"]], ci[:m["nblk"]], va[:m["nval"]], bi[:m["nbias"]])

    def bench_layers(self, layers, nthreads, warmups=0, reps=1):
        """Timed reference spmm_into over several layers' (weights, act [B][K][H][W],
        bias, fused) tuples; (layer, image) units over nthreads threads.
        Returns per-rep seconds."""
        keep, arr = [], (RefLayer * len(layers))()
        for j, (m, act, bias, fused) in enumerate(layers):
            act = _f32(act)
            B, K, H, W = act.shape
            rp, ci, va = _u32(m.row_ptr), _u32(m.col_idx), _f32(m.values)
            b = None if bias is None or len(bias) == 0 else _f32(bias)
            k, lo, hi = _act(fused)
            keep += [act, rp, ci, va, b]
            arr[j] = RefLayer(m.rows, m.cols, m.block_h, _ptr(rp), rp.size, _ptr(ci), ci.size,
                              _ptr(va), va.size, B, H, W, _ptr(act), _ptr(b), k, lo, hi)
        secs = (_d * reps)()
        rc = self.lib.ref_bench_layers(arr, len(layers), nthreads, warmups, reps, secs)
        assert rc == 0, rc
        return [secs[i] for i in range(reps)]


def have_ref() -> bool:
    return os.path.exists(REF_SO)
