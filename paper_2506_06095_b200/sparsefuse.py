"""Host-side mirror of the reference operator API for the hot path, over the C ABI.

Names, argument meaning and error classes follow /root/reference/proj/include/sparsefuse/:
  generate_mask / gen_*            io.hpp:192-204, mask.hpp:74-179
  build_bsr / build_rowwise        bsr.hpp:47-101, 198-209
  block_stats                      bsr.hpp:186-196
  threshold / select_plan          planner.hpp:67-161 (+ a B200 mode)
  block_sparse_sdpa / rowwise_sdpa attention.hpp:71-213, planner.hpp:165-172
  mha                              the unified MHA entry (new: the reference's exec_mha always
                                   runs the block executor, backend.hpp:347)
Every computation runs in libsf_b200.so on the GPU; tensors are torch CUDA tensors used as
device memory only.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence, Union

import numpy as np
import torch

from . import _lib
from ._lib import (AttnArgs, AttnStats, BsrDev, CsrDev, HwSpec, MaskDesc, Plan, check, lib, SF_BF16, SF_F16,
                   SF_BLOCK_WISE, SF_ROW_WISE, SF_PATTERN, SF_PLAN_B200, SF_PLAN_REFERENCE)


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# ---------------------------------------------------------------------------------------------
# Mask descriptors (io.hpp:158-190 MaskDescriptor; mask.hpp:64-71 PatternParams)
@dataclass
class MaskDescriptor:
    pattern: str
    seq_len: int
    band_width: int = 0
    global_width: int = 0
    dilation_rate: int = 0
    filling_rate: float = 0.0
    block: int = 16
    seed: int = 0

    def to_c(self) -> MaskDesc:
        if self.pattern not in SF_PATTERN:
            raise _lib.InvalidParameter(f"unknown mask pattern: {self.pattern}")
        return MaskDesc(SF_PATTERN[self.pattern], self.seq_len, self.band_width, self.global_width,
                        self.dilation_rate, self.block, self.filling_rate, self.seed)

    @staticmethod
    def from_json(j: dict) -> "MaskDescriptor":
        # io.hpp:179-190 defaults
        return MaskDescriptor(j["pattern"], int(j["seq_len"]), int(j.get("band_width", 0)),
                              int(j.get("global_width", 0)), int(j.get("dilation_rate", 0)),
                              float(j.get("filling_rate", 0.0)), int(j.get("block", 16)), int(j.get("seed", 0)))

    def to_json(self) -> dict:
        # io.hpp:164-177: only the fields the pattern uses
        j = {"pattern": self.pattern, "seq_len": self.seq_len, "seed": self.seed}
        if self.pattern in ("sliding", "dilated", "longformer", "bigbird", "causal_local", "strided"):
            j["band_width"] = self.band_width
        if self.pattern == "dilated":
            j["dilation_rate"] = self.dilation_rate
        if self.pattern in ("global", "longformer", "bigbird"):
            j["global_width"] = self.global_width
        if self.pattern in ("random", "bigbird"):
            j["filling_rate"] = self.filling_rate
            j["block"] = self.block
        return j


class DenseMask:
    """A seq_len x seq_len validity mask resident on the GPU, bit-packed (sf_capi.h layout).

    Mirrors DenseMask (mask.hpp:18-54); the host uint8 form is available via to_numpy().
    """

    def __init__(self, seq_len: int, bits: torch.Tensor):
        self.seq_len = int(seq_len)
        self.bits = bits  # int32 [seq_len, words]

    @property
    def words(self) -> int:
        return int(lib().sf_mask_words(self.seq_len))

    @staticmethod
    def empty(seq_len: int, device="cuda") -> "DenseMask":
        if seq_len <= 0:
            raise _lib.InvalidParameter("seq_len must be positive")
        w = int(lib().sf_mask_words(seq_len))
        return DenseMask(seq_len, torch.zeros((seq_len, w), dtype=torch.int32, device=device))

    @staticmethod
    def from_numpy(m: np.ndarray, device="cuda", stream=None) -> "DenseMask":
        m = np.ascontiguousarray(m, dtype=np.uint8)
        n = m.shape[0]
        dm = DenseMask.empty(n, device)
        u8 = torch.from_numpy(m).to(device)
        st = _stream(stream)
        check(lib().sf_mask_pack_u8(u8.data_ptr(), n, dm.bits.data_ptr(), st))
        # the temporary u8 copy must outlive the pack kernel on the stream it ran on
        (stream if stream is not None else torch.cuda.current_stream()).synchronize()
        return dm

    def to_numpy(self) -> np.ndarray:
        w = self.bits.cpu().numpy().view(np.uint32)
        bits = np.unpackbits(w.view(np.uint8), axis=1, bitorder="little")
        return bits[:, : self.seq_len].astype(np.uint8)

    def sfmk(self, stream=None) -> bytes:
        """write_dense_mask bytes (io.hpp:61-76), packed on device."""
        nb = C.c_int64()
        check(lib().sf_mask_serialize(self.bits.data_ptr(), self.seq_len, None, 0, C.byref(nb), _stream(stream)))
        buf = (C.c_uint8 * nb.value)()
        check(lib().sf_mask_serialize(self.bits.data_ptr(), self.seq_len, buf, nb.value, C.byref(nb), _stream(stream)))
        return bytes(buf)

    @staticmethod
    def from_sfmk(data: bytes, device="cuda", stream=None) -> "DenseMask":
        """read_dense_mask (io.hpp:78-95): IoError on bad magic / version / truncation."""
        buf = (C.c_uint8 * len(data)).from_buffer_copy(data)
        n = C.c_int32()
        check(lib().sf_mask_deserialize(buf, len(data), C.byref(n), None, _stream(stream)))
        dm = DenseMask.empty(n.value, device)
        check(lib().sf_mask_deserialize(buf, len(data), C.byref(n), dm.bits.data_ptr(), _stream(stream)))
        return dm

    def true_count(self, stream=None) -> int:
        c = C.c_int64()
        check(lib().sf_mask_count(self.bits.data_ptr(), self.seq_len, C.byref(c), _stream(stream)))
        return c.value


def _descs(terms) -> tuple:
    if isinstance(terms, (MaskDescriptor, dict)):
        terms = [terms]
    ds = [t if isinstance(t, MaskDescriptor) else MaskDescriptor(**t) for t in terms]
    arr = (MaskDesc * len(ds))()
    for i, d in enumerate(ds):
        arr[i] = d.to_c()
    return arr, len(ds)


def generate_mask(terms: Union[MaskDescriptor, dict, Sequence], stream=None) -> DenseMask:
    """generate_mask (io.hpp:192) of one descriptor, or compose (mask.hpp:146) of several."""
    arr, cnt = _descs(terms)
    check(lib().sf_mask_validate(arr, cnt))
    dm = DenseMask.empty(arr[0].seq_len)
    check(lib().sf_mask_generate(arr, cnt, dm.bits.data_ptr(), _stream(stream)))
    return dm


def gen_sliding_window(seq_len, band_width):
    return generate_mask(MaskDescriptor("sliding", seq_len, band_width=band_width))


def gen_dilated(seq_len, band_width, dilation_rate):
    return generate_mask(MaskDescriptor("dilated", seq_len, band_width=band_width, dilation_rate=dilation_rate))


def gen_global(seq_len, global_width):
    return generate_mask(MaskDescriptor("global", seq_len, global_width=global_width))


def gen_random_blocks(seq_len, block, filling_rate, seed):
    return generate_mask(MaskDescriptor("random", seq_len, filling_rate=filling_rate, block=block, seed=seed))


def gen_longformer(seq_len, global_width, band_width):
    return generate_mask(MaskDescriptor("longformer", seq_len, band_width=band_width, global_width=global_width))


def gen_bigbird(seq_len, global_width, band_width, filling_rate, seed, block=16):
    return generate_mask(MaskDescriptor("bigbird", seq_len, band_width=band_width, global_width=global_width,
                                        filling_rate=filling_rate, block=block, seed=seed))


# ---------------------------------------------------------------------------------------------
# Storage formats
class BsrMask:
    """Device dual-BSR (bsr.hpp:21-37) built by sf_bsr_build; freed with the object."""

    def __init__(self, dev: BsrDev):
        self.dev = dev

    def __del__(self):
        try:
            if self.dev._alloc:
                lib().sf_bsr_free(C.byref(self.dev), None)
        except Exception:
            pass

    def __getattr__(self, name):
        if name in ("seq_len", "block_m", "block_n", "n_rows", "n_cols", "n_full", "n_part", "n_load", "n_pool",
                    "tile_bytes"):
            return getattr(self.dev, name)
        raise AttributeError(name)

    def to_host(self, stream=None) -> dict:
        d = self.dev
        rp = d.n_rows + 1
        out = {k: np.zeros(n, np.int32) for k, n in (("full_row_ptr", rp), ("full_col_idx", d.n_full),
                                                    ("part_row_ptr", rp), ("part_col_idx", d.n_part),
                                                    ("part_tile_ids", d.n_part), ("load_row_ptr", rp),
                                                    ("load_col_idx", d.n_load))}
        pool = np.zeros(d.n_pool * d.tile_bytes, np.uint8)
        ptr = lambda a: a.ctypes.data if a.size else None
        check(lib().sf_bsr_to_host(C.byref(d), ptr(out["full_row_ptr"]), ptr(out["full_col_idx"]),
                                   ptr(out["part_row_ptr"]), ptr(out["part_col_idx"]), ptr(out["part_tile_ids"]),
                                   ptr(out["load_row_ptr"]), ptr(out["load_col_idx"]), ptr(pool), _stream(stream)))
        out["pool_packed"] = pool.reshape(d.n_pool, d.tile_bytes) if d.n_pool else np.zeros((0, d.tile_bytes), np.uint8)
        nbits = d.block_m * d.block_n
        out["part_mask_pool"] = (np.unpackbits(out["pool_packed"], axis=1, bitorder="little")[:, :nbits]
                                 if d.n_pool else np.zeros((0, nbits), np.uint8))
        return out

    def sfbr(self, stream=None) -> bytes:
        """write_bsr bytes (io.hpp:103-122)."""
        nb = C.c_int64()
        check(lib().sf_bsr_serialize(C.byref(self.dev), None, 0, C.byref(nb), _stream(stream)))
        buf = (C.c_uint8 * nb.value)()
        check(lib().sf_bsr_serialize(C.byref(self.dev), buf, nb.value, C.byref(nb), _stream(stream)))
        return bytes(buf)


def bsr_from_host(arrays: dict, seq_len: int, block_m: int, block_n: int, stream=None) -> BsrMask:
    """Device copy of host BSR arrays (the reference's BsrMask fields; `part_mask_pool` as unpacked
    0/1 tiles of block_m*block_n, or `pool_packed` as pack_bits bytes)."""
    a = {k: np.ascontiguousarray(v, np.int32) for k, v in arrays.items()
         if k not in ("part_mask_pool", "pool_packed")}
    if "pool_packed" in arrays:
        pool = np.ascontiguousarray(arrays["pool_packed"], np.uint8)
    else:
        tiles = np.asarray(arrays.get("part_mask_pool", np.zeros((0, block_m * block_n))), np.uint8)
        pool = (np.packbits(tiles.reshape(len(tiles), -1), axis=1, bitorder="little")
                if len(tiles) else np.zeros((0, (block_m * block_n + 7) // 8), np.uint8))
    n_pool = pool.shape[0] if pool.ndim == 2 else 0
    ptr = lambda x: x.ctypes.data if x.size else None
    dev = BsrDev()
    check(lib().sf_bsr_from_host(seq_len, block_m, block_n, a["full_col_idx"].size, a["part_col_idx"].size,
                                 a["load_col_idx"].size, n_pool, ptr(a["full_row_ptr"]), ptr(a["full_col_idx"]),
                                 ptr(a["part_row_ptr"]), ptr(a["part_col_idx"]), ptr(a["part_tile_ids"]),
                                 ptr(a["load_row_ptr"]), ptr(a["load_col_idx"]), ptr(pool), C.byref(dev),
                                 _stream(stream)))
    return BsrMask(dev)


def validate_bsr(b: BsrMask, stream=None) -> None:
    """validate_bsr (bsr.hpp:104-153) on the device; raises InternalInconsistency with the
    reference's message."""
    check(lib().sf_bsr_validate(C.byref(b.dev), _stream(stream)))


def to_dense(b: BsrMask, stream=None) -> DenseMask:
    """to_dense (bsr.hpp:155-177): the exact inverse of build_bsr, on the device."""
    m = DenseMask.empty(b.seq_len)
    check(lib().sf_bsr_to_dense(C.byref(b.dev), m.bits.data_ptr(), _stream(stream)))
    return m


class BsrWorkspace(BsrMask):
    """A worst-case-sized BSR (sf_bsr_workspace) rebuilt in place by build_async() with no host
    synchronisation — capturable in a CUDA graph next to the attention that reads it. The device
    counts land in `counts` (int32 [4]: n_full, n_part, n_load, n_pool)."""

    def __init__(self, seq_len: int, block_m: int, block_n: int, stream=None):
        dev = BsrDev()
        check(lib().sf_bsr_workspace(seq_len, block_m, block_n, C.byref(dev), _stream(stream)))
        super().__init__(dev)
        self.counts = torch.zeros(4, dtype=torch.int32, device="cuda")

    def build_async(self, mask: DenseMask, stream=None) -> "BsrWorkspace":
        if mask.seq_len != self.dev.seq_len:
            raise _lib.ShapeError("mask seq_len differs from the workspace")
        check(lib().sf_bsr_build_async(mask.bits.data_ptr(), C.byref(self.dev), self.counts.data_ptr(), _stream(stream)))
        return self

    def snapshot(self) -> BsrMask:
        """A non-owning view with the built counts (reads `counts`: synchronises) for to_host / sfbr."""
        n = self.counts.cpu().tolist()
        d = BsrDev.from_buffer_copy(self.dev)
        d.n_full, d.n_part, d.n_load, d.n_pool = n
        d._alloc = None  # the workspace owns the memory
        v = BsrMask(d)
        v._owner = self
        return v


def build_bsr(mask: DenseMask, block_m: int, block_n: int, stream=None) -> BsrMask:
    dev = BsrDev()
    check(lib().sf_bsr_build(mask.bits.data_ptr(), mask.seq_len, block_m, block_n, C.byref(dev), _stream(stream)))
    return BsrMask(dev)


@dataclass
class BlockStats:
    full_count: int
    part_count: int
    empty_count: int
    valid_block_ratio: float


def block_stats(b: BsrMask) -> BlockStats:
    """bsr.hpp:186-196 (host arithmetic on the device builder's counts)."""
    total = b.n_rows * b.n_cols
    return BlockStats(b.n_full, b.n_part, total - b.n_full - b.n_part,
                      (b.n_full + b.n_part) / total if total > 0 else 0.0)


class RowwiseMask:
    """Device CSR (bsr.hpp:41-45)."""

    def __init__(self, dev: CsrDev):
        self.dev = dev

    def __del__(self):
        try:
            if self.dev._alloc:
                lib().sf_csr_free(C.byref(self.dev), None)
        except Exception:
            pass

    @property
    def seq_len(self):
        return self.dev.seq_len

    @property
    def nnz(self):
        return self.dev.nnz

    def to_host(self, stream=None):
        n, nnz = self.dev.seq_len, self.dev.nnz
        rp = np.zeros(n + 1, np.int32)
        ci = np.zeros(max(nnz, 1), np.int32)
        check(lib().sf_csr_to_host(C.byref(self.dev), rp.ctypes.data, ci.ctypes.data, _stream(stream)))
        return rp, ci[:nnz]


def build_rowwise(mask: DenseMask, stream=None) -> RowwiseMask:
    dev = CsrDev()
    check(lib().sf_rowwise_build(mask.bits.data_ptr(), mask.seq_len, C.byref(dev), _stream(stream)))
    return RowwiseMask(dev)


# ---------------------------------------------------------------------------------------------
# Analytical selector
@dataclass
class HardwareSpec:
    name: str
    sm_num: int
    smem_size: int
    max_warp: int
    element_bytes: int = 2

    def to_c(self) -> HwSpec:
        return HwSpec(self.name.encode()[:31], self.sm_num, self.smem_size, self.max_warp, self.element_bytes)


def hw_preset(name: str) -> HardwareSpec:
    hw = HwSpec()
    check(lib().sf_hw_preset(name.encode(), C.byref(hw)))
    return HardwareSpec(hw.name.decode(), hw.sm_num, hw.smem_size, hw.max_warp, hw.element_bytes)


@dataclass
class KernelPlan:
    kind: str = "row_wise"
    block_m: int = 0
    block_n: int = 0
    num_warps: int = 0
    score: float = 0.0
    threshold: float = float("nan")
    fallback: bool = False

    def to_c(self) -> Plan:
        return Plan(SF_BLOCK_WISE if self.kind == "block_wise" else SF_ROW_WISE, self.block_m, self.block_n,
                    self.num_warps, self.score, self.threshold, int(self.fallback))

    @staticmethod
    def from_c(p: Plan) -> "KernelPlan":
        return KernelPlan("block_wise" if p.kind == SF_BLOCK_WISE else "row_wise", p.block_m, p.block_n,
                          p.num_warps, p.score, p.threshold, bool(p.fallback))


def threshold(mask: DenseMask, tau: float = 1.2, stream=None) -> float:
    out = C.c_double()
    check(lib().sf_threshold(mask.bits.data_ptr(), mask.seq_len, tau, C.byref(out), _stream(stream)))
    return out.value


def select_plan(mask: DenseMask, hw: HardwareSpec, seq_len: int, h: int, bs: int, head_size: int,
                mode: str = "reference", stream=None) -> KernelPlan:
    if mask.seq_len != seq_len:
        raise _lib.ShapeError("mask seq_len differs from requested")  # planner.hpp:133
    p = Plan()
    hwc = hw.to_c()
    check(lib().sf_select_plan(mask.bits.data_ptr(), C.byref(hwc), seq_len, h, bs, head_size,
                               SF_PLAN_B200 if mode == "b200" else SF_PLAN_REFERENCE, C.byref(p), _stream(stream)))
    return KernelPlan.from_c(p)


# ---------------------------------------------------------------------------------------------
# Attention
def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float16:
        return SF_F16
    if t.dtype == torch.bfloat16:
        return SF_BF16
    raise _lib.InvalidParameter("attention tensors must be float16 or bfloat16")


def attn_args(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor, scale: float = 0.0) -> AttnArgs:
    """(bs, h, n, d) views with a unit last stride; q, k, v share strides."""
    for t in (q, k, v, o):
        if t.dim() != 4 or t.stride(3) != 1 or not t.is_cuda:
            raise _lib.ShapeError("attention tensors must be CUDA (bs, h, n, d) views with unit last stride")
    if not (q.shape == k.shape == v.shape == o.shape):
        raise _lib.ShapeError("Q, K, V shapes differ")  # tensor.hpp:46
    if not (q.stride() == k.stride() == v.stride()):
        raise _lib.ShapeError("q, k, v must share strides")
    if not (q.dtype == k.dtype == v.dtype == o.dtype):
        raise _lib.InvalidParameter("dtype mismatch")
    bs, h, n, d = q.shape
    return AttnArgs(bs, h, n, d, _dtype_code(q), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                    q.stride(0), q.stride(1), q.stride(2), o.stride(0), o.stride(1), o.stride(2), scale)


def block_sparse_sdpa(q, k, v, bsr: BsrMask, plan: Optional[KernelPlan] = None, out=None, stats: bool = False,
                      stream=None):
    """attention.hpp:71 (plan=None) / planner.hpp:165 (plan given: must match the BSR)."""
    o = out if out is not None else torch.empty_like(q)
    a = attn_args(q, k, v, o)
    st = AttnStats()
    pc = plan.to_c() if plan is not None else None
    check(lib().sf_mha_blockwise(C.byref(a), C.byref(bsr.dev), C.byref(pc) if pc is not None else None,
                                 C.byref(st), _stream(stream)))
    if stats:
        return o, {"tiles_loaded": st.tiles_loaded, "full_tiles": st.full_tiles, "part_tiles": st.part_tiles}
    return o


def rowwise_sdpa(q, k, v, rw: RowwiseMask, out=None, stream=None):
    """attention.hpp:177."""
    o = out if out is not None else torch.empty_like(q)
    a = attn_args(q, k, v, o)
    check(lib().sf_mha_rowwise(C.byref(a), C.byref(rw.dev), _stream(stream)))
    return o


def dense_sdpa_oracle(q, k, v, mask: "DenseMask", stream=None) -> torch.Tensor:
    """attention.hpp:15-56 on the device: dense masked SDPA from the DENSE mask, fp64 accumulation
    and output (bs, h, n, d). Independent of the storage formats; `attn verify` checks the sparse
    executors against it."""
    o64 = torch.empty(q.shape, dtype=torch.float64, device=q.device)
    a = attn_args(q, k, v, q)  # o (unused) must be non-null
    check(lib().sf_mha_dense_oracle(C.byref(a), mask.bits.data_ptr(), o64.data_ptr(), _stream(stream)))
    return o64


# below this length the block executor over the whole dilated mask is as fast (bs16 x 12 heads,
# dilated(sqrt n, 1): n 2048 66 vs 68 us, n 4096 144 vs 120 us, n 8192 363 vs 265 us; tools/dilated_time.py)
DILATED_MIN_SEQ = 4096


def strided_sdpa(q, k, v, band_width: int, band_bsr: BsrMask, out=None, stream=None):
    """Masked MHA over the strided(w) mask by decomposition (sf_mha_strided): the causal-local(w)
    band on the tcgen05 block kernel (band_bsr: its block_m 128 BSR) plus the i - j = k w diagonals
    as dense causal attention inside each residue class, merged by log-sum-exp. Same semantics as
    block_sparse_sdpa over the strided mask (attention.hpp:71-172)."""
    o = out if out is not None else torch.empty_like(q)
    a = attn_args(q, k, v, o)
    check(lib().sf_mha_strided(C.byref(a), int(band_width), C.byref(band_bsr.dev), _stream(stream)))
    return o


def strided_band(terms) -> Optional[int]:
    """The band w when the mask descriptor is exactly one strided(w) term with n >= 2048 that the
    decomposed executor covers (ceil(n / w) <= 128), else None."""
    ts = terms if isinstance(terms, (list, tuple)) else [terms]
    if len(ts) != 1:
        return None
    t = ts[0] if isinstance(ts[0], MaskDescriptor) else MaskDescriptor(**ts[0])
    # below n = 2048 the block-wise executor over the whole strided mask is as fast or faster
    # (bs16 x 12 heads, n 1024, w 32: 59 vs 67 us; n 2048, w 45: 196 vs 137 us; tools/strided_time.py)
    if t.pattern != "strided" or t.band_width < 1 or -(-t.seq_len // t.band_width) > 128 or t.seq_len < 2048:
        return None
    return int(t.band_width)


def mask_andnot(mask: DenseMask, minus: DenseMask, stream=None) -> DenseMask:
    """The cells of `mask` not in `minus` (sf_mask_andnot), as a new device mask."""
    if mask.seq_len != minus.seq_len:
        raise _lib.ShapeError("mask_andnot: seq_len differs")
    out = DenseMask(mask.seq_len, mask.bits.clone())
    check(lib().sf_mask_andnot(minus.bits.data_ptr(), out.bits.data_ptr(), mask.seq_len, _stream(stream)))
    return out


def dilated_sdpa(q, k, v, stride: int, class_bsr: BsrMask, rest_bsr: Optional[BsrMask] = None, out=None,
                 stream=None):
    """Masked MHA over a mask holding dilated(w, r) by decomposition (sf_mha_dilated): each residue
    class mod stride = r + 1 is a sliding(w) band over n / stride rows (class_bsr: its block_m 128
    BSR, shared by the classes) on the tcgen05 block kernel; rest_bsr (the mask minus the dilated
    cells, or None) runs over the full rows and the parts merge per row by log-sum-exp. Same
    semantics as block_sparse_sdpa over the whole mask (attention.hpp:71-172)."""
    o = out if out is not None else torch.empty_like(q)
    a = attn_args(q, k, v, o)
    rest = C.byref(rest_bsr.dev) if rest_bsr is not None else None
    check(lib().sf_mha_dilated(C.byref(a), int(stride), C.byref(class_bsr.dev), rest, _stream(stream)))
    return o


def dilated_split(terms, min_seq_len: int = DILATED_MIN_SEQ, allow_rest: bool = False) -> Optional[tuple]:
    """(stride, band_width) when the descriptor holds one dilated(w, r >= 1) term, seq_len % (r + 1)
    == 0 and seq_len >= min_seq_len; else None. Other terms (the decomposition's rest) only with
    allow_rest: a rest with global rows is slower than the block executor over the whole mask (its
    global row blocks are single 64-step items; T5 cfg4: 170 vs 115 us, tools/dilated_time.py)."""
    ts = terms if isinstance(terms, (list, tuple)) else [terms]
    ds = [t if isinstance(t, MaskDescriptor) else MaskDescriptor(**t) for t in ts]
    dil = [t for t in ds if t.pattern == "dilated"]
    if len(dil) != 1 or (len(ds) > 1 and not allow_rest):
        return None
    t = dil[0]
    s = int(t.dilation_rate) + 1
    if s < 2 or t.band_width < 1 or t.seq_len % s or t.seq_len < min_seq_len:
        return None
    return s, int(t.band_width)


def executor_label(ctx) -> list:
    """The executor a context runs, as reported by the bench: [kind, block_m, block_n],
    ["strided_decomposed", band_width, 0] or ["dilated_decomposed", stride, band_width]."""
    if getattr(ctx, "strided_band", None):
        return ["strided_decomposed", int(ctx.strided_band), 0]
    if getattr(ctx, "dilated", None):
        return ["dilated_decomposed", int(ctx.dilated[0]), int(ctx.dilated[1])]
    return [ctx.plan.kind, ctx.plan.block_m, ctx.plan.block_n]


class MhaContext:
    """Formats + plan for one session mask (backend.hpp:309-321 MhaContext), built on device.
    strided_band=w (a mask that is one strided(w) descriptor, see strided_band()): the unified MHA
    runs the decomposed strided executor (band BSR built here) instead of the plan's executor."""

    def __init__(self, mask: DenseMask, plan: KernelPlan, stream=None, strided_band: Optional[int] = None,
                 dilated: Optional[tuple] = None):
        self.mask = mask
        self.plan = plan
        self.strided_band = strided_band
        self.dilated = tuple(dilated) if dilated else None
        self.band_bsr = None
        self.class_bsr = self.rest_bsr = None
        if strided_band:
            band = generate_mask([dict(pattern="causal_local", seq_len=mask.seq_len, band_width=strided_band)], stream)
            # the band part on head pairs (block_m 64): bs16 x 12 x n2048, w45: band part 47.0 vs
            # 51.7 us, decomposed 130.5 vs 135.8 us (tools/strided_time.py)
            # (head pairs hold <= 128 row blocks of 64: n <= 8192; longer sequences keep block_m 128)
            self.band_bsr = build_bsr(band, 64 if mask.seq_len <= 8192 else 128, 16, stream)
        elif self.dilated:  # (stride, w) from dilated_split(): class band + the rest of the mask
            s, w = self.dilated
            n = mask.seq_len
            band = generate_mask([dict(pattern="sliding", seq_len=n // s, band_width=min(w, n // s))], stream)
            # block_m 128: on head pairs the class bands measured 119.5 / 282.6 us at n 4096 / 8192
            # vs 120 / 265 (tools/dilated_time.py)
            self.class_bsr = build_bsr(band, 128, 16, stream)
            dil = generate_mask([dict(pattern="dilated", seq_len=n, band_width=w, dilation_rate=s - 1)], stream)
            rest = build_bsr(mask_andnot(mask, dil, stream), 128, 16, stream)
            self.rest_bsr = rest if rest.dev.n_load > 0 else None
        if plan.kind == "block_wise":
            self.bsr = build_bsr(mask, plan.block_m, plan.block_n, stream)
            self.csr = None
        else:
            self.bsr = None
            self.csr = build_rowwise(mask, stream)


def context_for(terms, mask: DenseMask, plan: KernelPlan, stream=None) -> MhaContext:
    """The MhaContext the unified MHA should run for a session mask given by its descriptor terms:
    the decomposed strided executor for one strided(w) term, the class decomposition for one
    dilated(w, r) term, else the plan's executor (strided_band(), dilated_split())."""
    sb = strided_band(terms)
    if sb:
        return MhaContext(mask, plan, stream, strided_band=sb)
    return MhaContext(mask, plan, stream, dilated=dilated_split(terms))


def mha(q, k, v, ctx: MhaContext, out=None, stream=None):
    """Unified MHA entry: dispatches the row-wise or block-wise executor from the plan (or the
    decomposed strided executor when the context carries a strided band)."""
    if ctx.strided_band:
        return strided_sdpa(q, k, v, ctx.strided_band, ctx.band_bsr, out=out, stream=stream)
    if ctx.dilated:
        return dilated_sdpa(q, k, v, ctx.dilated[0], ctx.class_bsr, ctx.rest_bsr, out=out, stream=stream)
    if ctx.plan.kind == "block_wise":
        return block_sparse_sdpa(q, k, v, ctx.bsr, ctx.plan, out=out, stream=stream)
    return rowwise_sdpa(q, k, v, ctx.csr, out=out, stream=stream)


def set_attn_impl(impl: str) -> None:
    """'auto' | 'generic' | 'tcgen05' kernel selection for block_sparse_sdpa."""
    check(lib().sf_set_attn_impl({"auto": 0, "generic": 1, "tcgen05": 2}[impl]))
