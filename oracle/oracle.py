"""ctypes view of the CPU checkers. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module. It loads:
  * oracle/_build/libsforacle.so — the plain-C restatement of the reference hot path;
  * oracle/_ref/libsfref.so     — the unmodified reference headers compiled in place
                                   (present where it was built; travels as a prebuilt .so).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libsforacle.so"
REF_SO = HERE / "_ref" / "libsfref.so"

PATTERNS = {
    "sliding": 0, "dilated": 1, "global": 2, "random": 3, "longformer": 4, "bigbird": 5,
    "causal": 6, "causal_local": 7, "strided": 8,
}


class MaskDesc(C.Structure):
    _fields_ = [("pattern", C.c_int32), ("seq_len", C.c_int32), ("band_width", C.c_int32),
                ("global_width", C.c_int32), ("dilation_rate", C.c_int32), ("block", C.c_int32),
                ("filling_rate", C.c_double), ("seed", C.c_uint64)]


class HwSpec(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("sm_num", C.c_int32), ("smem_size", C.c_int64),
                ("max_warp", C.c_int32), ("element_bytes", C.c_int32)]


class Plan(C.Structure):
    _fields_ = [("kind", C.c_int32), ("block_m", C.c_int32), ("block_n", C.c_int32),
                ("num_warps", C.c_int32), ("score", C.c_double), ("threshold", C.c_double),
                ("fallback", C.c_int32)]


class _Bsr(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("seq_len", "block_m", "block_n", "n_rows", "n_cols",
                                         "n_full", "n_part", "n_load", "n_pool")] + \
               [(n, C.POINTER(C.c_int32)) for n in ("full_row_ptr", "full_col_idx", "part_row_ptr",
                                                    "part_col_idx", "part_tile_ids", "load_row_ptr",
                                                    "load_col_idx")] + [("pool", C.POINTER(C.c_uint8))]


def make_desc(pattern: str, seq_len: int, band_width: int = 0, global_width: int = 0,
              dilation_rate: int = 0, filling_rate: float = 0.0, block: int = 16,
              seed: int = 0) -> MaskDesc:
    return MaskDesc(PATTERNS[pattern], seq_len, band_width, global_width, dilation_rate, block,
                    filling_rate, seed)


def terms_array(terms):
    arr = (MaskDesc * len(terms))()
    for i, t in enumerate(terms):
        arr[i] = t if isinstance(t, MaskDesc) else make_desc(**t)
    return arr


def build():
    """Build the checkers (the reference shim only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class Oracle:
    """The plain-C restatement (always available once built)."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            build()
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.sfo_mask_generate.argtypes = [C.POINTER(MaskDesc), C.c_int32, C.POINTER(C.c_uint8)]
        L.sfo_build_bsr.argtypes = [C.POINTER(C.c_uint8), C.c_int32, C.c_int32, C.c_int32, C.POINTER(_Bsr)]
        L.sfo_bsr_free.argtypes = [C.POINTER(_Bsr)]
        L.sfo_bsr_serialize.argtypes = [C.POINTER(_Bsr), C.POINTER(C.c_uint8)]
        L.sfo_bsr_serialize.restype = C.c_int64
        L.sfo_build_rowwise.argtypes = [C.POINTER(C.c_uint8), C.c_int32, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int32), C.c_int64, C.POINTER(C.c_int64)]
        L.sfo_block_sparse_sdpa.argtypes = [C.POINTER(C.c_float)] * 3 + [C.c_int32] * 4 + [
            C.POINTER(_Bsr), C.POINTER(C.c_float), C.POINTER(C.c_int64), C.c_int32]
        L.sfo_rowwise_sdpa.argtypes = [C.POINTER(C.c_double)] * 3 + [C.c_int32] * 4 + [
            C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_double)]
        L.sfo_dense_sdpa.argtypes = [C.POINTER(C.c_double)] * 3 + [C.c_int32] * 4 + [
            C.POINTER(C.c_uint8), C.POINTER(C.c_double)]
        L.sfo_random_attention_input.argtypes = [C.c_int32] * 4 + [C.c_uint64] + [C.POINTER(C.c_float)] * 3
        L.sfo_hw_preset.argtypes = [C.c_char_p, C.POINTER(HwSpec)]
        L.sfo_threshold.argtypes = [C.POINTER(C.c_uint8), C.c_int32, C.c_double, C.POINTER(C.c_double)]
        L.sfo_threshold_from_loads.argtypes = [C.c_int32, C.c_int64, C.c_double]
        L.sfo_threshold_from_loads.restype = C.c_double
        L.sfo_select_plan_from_loads.argtypes = [C.c_int64, C.POINTER(HwSpec), C.c_int64, C.c_int32,
                                                 C.c_int64, C.c_int32, C.c_int32, C.POINTER(Plan)]
        L.sfo_plan_score.argtypes = [C.c_int32] * 3 + [C.POINTER(HwSpec), C.c_int64, C.c_int32, C.c_int64, C.c_int32]
        L.sfo_plan_score.restype = C.c_double
        L.sfo_random_matrix.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_float, C.c_float, C.POINTER(C.c_float)]
        L.sfo_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.sfo_mix_seed.restype = C.c_uint64
        L.sfo_fnv1a.argtypes = [C.POINTER(C.c_uint8), C.c_size_t, C.c_uint64]
        L.sfo_fnv1a.restype = C.c_uint64
        L.sfo_gemm.argtypes = [C.POINTER(C.c_float)] * 2 + [C.c_int64] * 3 + [C.POINTER(C.c_float), C.c_int32]
        for f in ("sfo_bias", "sfo_add"):
            getattr(L, f).argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int64, C.POINTER(C.c_float)]
        for f in ("sfo_gelu", "sfo_relu"):
            getattr(L, f).argtypes = [C.POINTER(C.c_float), C.c_int64]
        L.sfo_layernorm.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int64, C.POINTER(C.c_float), C.POINTER(C.c_float)]
        L.sfo_softmax_rows.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int64]

    # ---- masks ----
    def mask(self, terms) -> np.ndarray:
        arr = terms_array(terms)
        n = arr[0].seq_len
        out = np.zeros((n, n), np.uint8)
        st = self.lib.sfo_mask_generate(arr, len(terms), _ptr(out, C.c_uint8))
        if st:
            raise ValueError(f"sfo_mask_generate status {st}")
        return out

    # ---- formats ----
    def bsr(self, mask: np.ndarray, bm: int, bn: int) -> dict:
        mask = np.ascontiguousarray(mask, np.uint8)
        n = mask.shape[0]
        b = _Bsr()
        st = self.lib.sfo_build_bsr(_ptr(mask, C.c_uint8), n, bm, bn, C.byref(b))
        if st:
            raise ValueError(f"sfo_build_bsr status {st}")
        def arr(p, cnt):
            return np.ctypeslib.as_array(p, shape=(cnt,)).copy() if cnt else np.zeros(0, np.int32)
        out = dict(seq_len=n, block_m=bm, block_n=bn, n_rows=b.n_rows, n_cols=b.n_cols,
                   full_row_ptr=arr(b.full_row_ptr, b.n_rows + 1), full_col_idx=arr(b.full_col_idx, b.n_full),
                   part_row_ptr=arr(b.part_row_ptr, b.n_rows + 1), part_col_idx=arr(b.part_col_idx, b.n_part),
                   part_tile_ids=arr(b.part_tile_ids, b.n_part), load_row_ptr=arr(b.load_row_ptr, b.n_rows + 1),
                   load_col_idx=arr(b.load_col_idx, b.n_load),
                   pool=(np.ctypeslib.as_array(b.pool, shape=(b.n_pool * bm * bn,)).copy().reshape(b.n_pool, bm * bn)
                         if b.n_pool else np.zeros((0, bm * bn), np.uint8)))
        size = self.lib.sfo_bsr_serialize(C.byref(b), None)
        buf = np.zeros(size, np.uint8)
        self.lib.sfo_bsr_serialize(C.byref(b), _ptr(buf, C.c_uint8))
        out["sfbr"] = buf.tobytes()
        self.lib.sfo_bsr_free(C.byref(b))
        return out

    def rowwise(self, mask: np.ndarray):
        mask = np.ascontiguousarray(mask, np.uint8)
        n = mask.shape[0]
        rp = np.zeros(n + 1, np.int32)
        nnz = C.c_int64()
        self.lib.sfo_build_rowwise(_ptr(mask, C.c_uint8), n, _ptr(rp, C.c_int32), None, 0, C.byref(nnz))
        ci = np.zeros(max(nnz.value, 1), np.int32)
        self.lib.sfo_build_rowwise(_ptr(mask, C.c_uint8), n, _ptr(rp, C.c_int32), _ptr(ci, C.c_int32),
                                   nnz.value, C.byref(nnz))
        return rp, ci[: nnz.value]

    def fnv1a(self, data: bytes, h: int = 0xcbf29ce484222325) -> int:
        a = np.frombuffer(data, np.uint8).copy()
        return self.lib.sfo_fnv1a(_ptr(a, C.c_uint8), len(a), h)

    # ---- attention ----
    def random_attention_input(self, bs, h, n, d, seed):
        q = np.zeros((bs, h, n, d), np.float32); k = np.zeros_like(q); v = np.zeros_like(q)
        self.lib.sfo_random_attention_input(bs, h, n, d, seed, _ptr(q, C.c_float), _ptr(k, C.c_float), _ptr(v, C.c_float))
        return q, k, v

    def block_sparse_sdpa(self, q, k, v, mask, bm, bn, threads=1):
        q, k, v = (np.ascontiguousarray(x, np.float32) for x in (q, k, v))
        bs, h, n, d = q.shape
        mask = np.ascontiguousarray(mask, np.uint8)
        b = _Bsr()
        self.lib.sfo_build_bsr(_ptr(mask, C.c_uint8), n, bm, bn, C.byref(b))
        out = np.zeros_like(q)
        stats = np.zeros(3, np.int64)
        st = self.lib.sfo_block_sparse_sdpa(_ptr(q, C.c_float), _ptr(k, C.c_float), _ptr(v, C.c_float),
                                            bs, h, n, d, C.byref(b), _ptr(out, C.c_float),
                                            _ptr(stats, C.c_int64), threads)
        self.lib.sfo_bsr_free(C.byref(b))
        if st:
            raise ValueError(f"sfo_block_sparse_sdpa status {st}")
        return out, stats

    def rowwise_sdpa(self, q, k, v, mask):
        q, k, v = (np.ascontiguousarray(x, np.float64) for x in (q, k, v))
        bs, h, n, d = q.shape
        rp, ci = self.rowwise(mask)
        ci = np.ascontiguousarray(ci if len(ci) else np.zeros(1, np.int32))
        out = np.zeros_like(q)
        self.lib.sfo_rowwise_sdpa(_ptr(q, C.c_double), _ptr(k, C.c_double), _ptr(v, C.c_double), bs, h, n, d,
                                  _ptr(rp, C.c_int32), _ptr(ci, C.c_int32), _ptr(out, C.c_double))
        return out

    def dense_sdpa(self, q, k, v, mask):
        q, k, v = (np.ascontiguousarray(x, np.float64) for x in (q, k, v))
        bs, h, n, d = q.shape
        mask = np.ascontiguousarray(mask, np.uint8)
        out = np.zeros_like(q)
        self.lib.sfo_dense_sdpa(_ptr(q, C.c_double), _ptr(k, C.c_double), _ptr(v, C.c_double), bs, h, n, d,
                                _ptr(mask, C.c_uint8), _ptr(out, C.c_double))
        return out

    # ---- planner ----
    def hw_preset(self, name: str) -> HwSpec:
        hw = HwSpec()
        if self.lib.sfo_hw_preset(name.encode(), C.byref(hw)):
            raise ValueError(name)
        return hw

    def select_plan_from_loads(self, loads16, hw, seq, h, bs, head, mode=0) -> Plan:
        p = Plan()
        st = self.lib.sfo_select_plan_from_loads(loads16, C.byref(hw), seq, h, bs, head, mode, C.byref(p))
        if st:
            raise ValueError(f"select_plan status {st}")
        return p

    # ---- fused-template semantics ----
    def mix_seed(self, seed, tag):
        return self.lib.sfo_mix_seed(seed, tag)

    def random_matrix(self, rows, cols, seed, lo=-1.0, hi=1.0):
        out = np.zeros((rows, cols), np.float32)
        self.lib.sfo_random_matrix(rows, cols, seed, lo, hi, _ptr(out, C.c_float))
        return out

    def gemm(self, x, w, threads=1):
        x = np.ascontiguousarray(x, np.float32); w = np.ascontiguousarray(w, np.float32)
        out = np.zeros((x.shape[0], w.shape[1]), np.float32)
        self.lib.sfo_gemm(_ptr(x, C.c_float), _ptr(w, C.c_float), x.shape[0], w.shape[1], x.shape[1],
                          _ptr(out, C.c_float), threads)
        return out

    def bias(self, x, b):
        x = np.ascontiguousarray(x, np.float32).copy(); b = np.ascontiguousarray(b, np.float32)
        self.lib.sfo_bias(_ptr(x, C.c_float), x.shape[0], x.shape[1], _ptr(b, C.c_float)); return x

    def add(self, x, a):
        x = np.ascontiguousarray(x, np.float32).copy(); a = np.ascontiguousarray(a, np.float32)
        self.lib.sfo_add(_ptr(x, C.c_float), x.shape[0], x.shape[1], _ptr(a, C.c_float)); return x

    def gelu(self, x):
        x = np.ascontiguousarray(x, np.float32).copy(); self.lib.sfo_gelu(_ptr(x, C.c_float), x.size); return x

    def relu(self, x):
        x = np.ascontiguousarray(x, np.float32).copy(); self.lib.sfo_relu(_ptr(x, C.c_float), x.size); return x

    def softmax(self, x):  # apply_row_op Softmax, backend.hpp:155-167
        x = np.ascontiguousarray(x, np.float32).copy()
        self.lib.sfo_softmax_rows(_ptr(x, C.c_float), x.shape[0], x.shape[1])
        return x

    def layernorm(self, x, g, b):
        x = np.ascontiguousarray(x, np.float32).copy()
        g = np.ascontiguousarray(g, np.float32); b = np.ascontiguousarray(b, np.float32)
        self.lib.sfo_layernorm(_ptr(x, C.c_float), x.shape[0], x.shape[1], _ptr(g, C.c_float), _ptr(b, C.c_float))
        return x


class Reference:
    """The reference headers compiled in place (oracle/_ref). Absent => .available False."""

    def __init__(self, path: Path = REF_SO):
        self.available = path.exists()
        if not self.available:
            return
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.ref_mask_generate.argtypes = [C.POINTER(MaskDesc), C.c_int, C.POINTER(C.c_uint8)]
        L.ref_build_bsr_sfbr.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint8),
                                         C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.ref_build_rowwise.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                        C.c_int64, C.POINTER(C.c_int64)]
        L.ref_block_sparse_sdpa.argtypes = [C.POINTER(C.c_float)] * 3 + [C.c_int] * 4 + [
            C.POINTER(C.c_uint8), C.c_int, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_int64), C.c_int]
        L.ref_rowwise_sdpa.argtypes = [C.POINTER(C.c_double)] * 3 + [C.c_int] * 4 + [C.POINTER(C.c_uint8), C.POINTER(C.c_double)]
        L.ref_dense_sdpa.argtypes = L.ref_rowwise_sdpa.argtypes
        L.ref_random_attention_input.argtypes = [C.c_int] * 4 + [C.c_uint64] + [C.POINTER(C.c_float)] * 3
        L.ref_threshold.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.c_double, C.POINTER(C.c_double)]
        L.ref_select_plan.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.POINTER(HwSpec), C.c_int64, C.c_int,
                                      C.c_int64, C.c_int, C.POINTER(Plan)]
        L.ref_hw_preset.argtypes = [C.c_char_p, C.POINTER(HwSpec)]
        L.ref_graph_param.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_uint64,
                                      C.c_int, C.c_int, C.POINTER(C.c_float), C.c_int64, C.POINTER(C.c_int64)]
        L.ref_run_chain.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_uint64,
                                    C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_char_p, C.POINTER(C.c_float), C.c_int,
                                    C.POINTER(C.c_double)]
        L.ref_exec_segment.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_uint64,
                                       C.c_int, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_float),
                                       C.POINTER(C.c_uint8), C.c_int, C.c_int]

    def exec_segment(self, model, bs, seq, hidden, heads, head_size, seed, seg, x, out_cols, mask=None, tile=(16, 16)):
        """exec_segment (backend.hpp:360-385) of nodes [seg[0], seg[1]) of a preset or "spec:" graph on
        GraphData(seed) (fp32, the reference's CPU executors); `mask` builds the MHA context."""
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros((x.shape[0], out_cols), np.float32)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        st = self.lib.ref_exec_segment(model.encode(), bs, seq, hidden, heads, head_size, seed, seg[0], seg[1],
                                       _ptr(x, C.c_float), _ptr(out, C.c_float),
                                       None if m is None else _ptr(m, C.c_uint8), tile[0], tile[1])
        if st:
            raise ValueError(f"ref_exec_segment status {st}")
        return out

    def validate_bsr(self, seq_len, bm, bn, a: dict):
        """validate_bsr of host arrays (keys as BsrMask.to_host(), `part_mask_pool` unpacked 0/1 tiles):
        (status, message)."""
        i32 = lambda k: np.ascontiguousarray(a[k], np.int32)
        arrs = [i32(k) for k in ("full_row_ptr", "full_col_idx", "part_row_ptr", "part_col_idx", "part_tile_ids",
                                 "load_row_ptr", "load_col_idx")]
        pool = np.ascontiguousarray(a["part_mask_pool"], np.uint8).reshape(-1)
        args = []
        for x in arrs:
            args += [_ptr(x, C.c_int32), x.size]
        msg = C.create_string_buffer(256)
        self.lib.ref_validate_bsr.argtypes = [C.c_int] * 3 + [C.POINTER(C.c_int32), C.c_int64] * 7 + [
            C.POINTER(C.c_uint8), C.c_int64, C.c_char_p, C.c_int64]
        st = self.lib.ref_validate_bsr(seq_len, bm, bn, *args, _ptr(pool, C.c_uint8), len(a["part_mask_pool"]), msg, 256)
        return st, msg.value.decode()

    def mask(self, terms) -> np.ndarray:
        arr = terms_array(terms)
        n = arr[0].seq_len
        out = np.zeros((n, n), np.uint8)
        st = self.lib.ref_mask_generate(arr, len(terms), _ptr(out, C.c_uint8))
        if st:
            raise ValueError(f"ref_mask_generate status {st}")
        return out

    def sfbr(self, mask, bm, bn):
        mask = np.ascontiguousarray(mask, np.uint8)
        n = mask.shape[0]
        nb = C.c_int64()
        counts = np.zeros(4, np.int64)
        st = self.lib.ref_build_bsr_sfbr(_ptr(mask, C.c_uint8), n, bm, bn, None, 0, C.byref(nb), _ptr(counts, C.c_int64))
        if st:
            raise ValueError(f"ref_build_bsr status {st}")
        buf = np.zeros(nb.value, np.uint8)
        self.lib.ref_build_bsr_sfbr(_ptr(mask, C.c_uint8), n, bm, bn, _ptr(buf, C.c_uint8), nb.value, C.byref(nb), None)
        return buf.tobytes(), counts

    def sfmk(self, mask) -> bytes:
        """the reference's write_dense_mask bytes (io.hpp:66-76)."""
        mask = np.ascontiguousarray(mask, np.uint8)
        n = mask.shape[0]
        nb = C.c_int64()
        self.lib.ref_mask_sfmk.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.POINTER(C.c_uint8), C.c_int64,
                                           C.POINTER(C.c_int64)]
        self.lib.ref_mask_sfmk(_ptr(mask, C.c_uint8), n, None, 0, C.byref(nb))
        buf = np.zeros(nb.value, np.uint8)
        if self.lib.ref_mask_sfmk(_ptr(mask, C.c_uint8), n, _ptr(buf, C.c_uint8), nb.value, C.byref(nb)):
            raise ValueError("ref_mask_sfmk failed")
        return buf.tobytes()

    def rowwise(self, mask):
        mask = np.ascontiguousarray(mask, np.uint8)
        n = mask.shape[0]
        rp = np.zeros(n + 1, np.int32)
        nnz = C.c_int64()
        self.lib.ref_build_rowwise(_ptr(mask, C.c_uint8), n, _ptr(rp, C.c_int32), None, 0, C.byref(nnz))
        ci = np.zeros(max(1, nnz.value), np.int32)
        self.lib.ref_build_rowwise(_ptr(mask, C.c_uint8), n, _ptr(rp, C.c_int32), _ptr(ci, C.c_int32), nnz.value, C.byref(nnz))
        return rp, ci[: nnz.value]

    def random_attention_input(self, bs, h, n, d, seed):
        q = np.zeros((bs, h, n, d), np.float32); k = np.zeros_like(q); v = np.zeros_like(q)
        self.lib.ref_random_attention_input(bs, h, n, d, seed, _ptr(q, C.c_float), _ptr(k, C.c_float), _ptr(v, C.c_float))
        return q, k, v

    def block_sparse_sdpa(self, q, k, v, mask, bm, bn, threads=1):
        q, k, v = (np.ascontiguousarray(x, np.float32) for x in (q, k, v))
        bs, h, n, d = q.shape
        mask = np.ascontiguousarray(mask, np.uint8)
        out = np.zeros_like(q)
        stats = np.zeros(3, np.int64)
        st = self.lib.ref_block_sparse_sdpa(_ptr(q, C.c_float), _ptr(k, C.c_float), _ptr(v, C.c_float), bs, h, n, d,
                                            _ptr(mask, C.c_uint8), bm, bn, _ptr(out, C.c_float), _ptr(stats, C.c_int64), threads)
        if st:
            raise ValueError(f"ref_block_sparse_sdpa status {st}")
        return out, stats

    def select_plan(self, mask, hw, seq, h, bs, head) -> Plan:
        mask = np.ascontiguousarray(mask, np.uint8)
        p = Plan()
        st = self.lib.ref_select_plan(_ptr(mask, C.c_uint8), mask.shape[0], C.byref(hw), seq, h, bs, head, C.byref(p))
        if st:
            raise ValueError(f"ref_select_plan status {st}")
        return p

    def graph_param(self, model, bs, seq, hidden, heads, head_size, seed, node, which):
        cnt = C.c_int64()
        self.lib.ref_graph_param(model.encode(), bs, seq, hidden, heads, head_size, seed, node, which, None, 0, C.byref(cnt))
        out = np.zeros(cnt.value, np.float32)
        self.lib.ref_graph_param(model.encode(), bs, seq, hidden, heads, head_size, seed, node, which,
                                 _ptr(out, C.c_float), cnt.value, C.byref(cnt))
        return out

    def run_pipeline_synthetic(self, model, bs, seq, model_seed, cfg_seed, planted=False) -> str:
        f = self.lib.ref_run_pipeline_synthetic
        f.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, C.c_int, C.c_char_p, C.c_int64]
        buf = C.create_string_buffer(1 << 16)
        st = f(model.encode(), bs, seq, model_seed, cfg_seed, int(planted), buf, len(buf))
        if st:
            raise ValueError(f"ref_run_pipeline_synthetic status {st}")
        return buf.value.decode()

    def cache_session(self, model, bs, seq, model_seed, cfg_seed, path_in="", path_out="") -> str:
        f = self.lib.ref_cache_session
        f.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, C.c_char_p, C.c_char_p,
                      C.c_char_p, C.c_int64]
        buf = C.create_string_buffer(1 << 16)
        st = f(model.encode(), bs, seq, model_seed, cfg_seed, path_in.encode(), path_out.encode(), buf, len(buf))
        if st:
            raise ValueError(f"ref_cache_session status {st}")
        return buf.value.decode()

    def run_chain(self, model, bs, seq, hidden, heads, head_size, seed, mask, bm, bn, code="", threads=1,
                  timing=False):
        """CpuBackend::run_chain output of copy 0; with timing=True also the wall seconds of the
        concurrent run_chain calls alone (backend construction excluded)."""
        mask = np.ascontiguousarray(mask, np.uint8)
        out = np.zeros((bs * seq, hidden), np.float32)
        sec = C.c_double(0.0)
        st = self.lib.ref_run_chain(model.encode(), bs, seq, hidden, heads, head_size, seed, _ptr(mask, C.c_uint8),
                                    bm, bn, code.encode(), _ptr(out, C.c_float), threads, C.byref(sec))
        if st:
            raise ValueError(f"ref_run_chain status {st}")
        return (out, sec.value) if timing else out


CONFIG_MASKS = {
    # SURVEY §8(d) config masks, w = floor(sqrt(n)).
    "cfg1": [dict(pattern="sliding", seq_len=512, band_width=22)],
    "cfg2": [dict(pattern="bigbird", seq_len=1024, global_width=32, band_width=32, filling_rate=0.10, seed=0, block=16)],
    "cfg3": [dict(pattern="strided", seq_len=2048, band_width=45)],
    "cfg4": [dict(pattern="dilated", seq_len=4096, band_width=64, dilation_rate=1),
             dict(pattern="global", seq_len=4096, global_width=64)],
}
