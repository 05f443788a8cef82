"""ctypes binding of the C ABI (include/sf_capi.h) -> paper_2506_06095_b200/_lib/libsf_b200.so.

This is the Python side of the drop-in boundary. Nothing here computes: every call goes to the
sm_100a library. If the library is missing the import fails loudly — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libsf_b200.so"
if os.environ.get("SF_B200_LIB"):  # alternative build of the same sources (e.g. trace-instrumented)
    LIB_PATH = Path(os.environ["SF_B200_LIB"]).resolve()


class SfError(RuntimeError):
    """Base of the error taxonomy (reference common.hpp:14-36)."""


class InvalidParameter(SfError, ValueError): ...
class ShapeError(SfError, ValueError): ...
class PlanError(SfError): ...
class DegenerateInput(SfError, ValueError): ...
class IllegalSegment(SfError, ValueError): ...
class InternalInconsistency(SfError): ...
class BackendError(SfError): ...
class IoError(SfError): ...
class CudaError(SfError): ...


_STATUS = {1: InvalidParameter, 2: ShapeError, 3: PlanError, 4: DegenerateInput, 5: IllegalSegment,
           6: InternalInconsistency, 7: BackendError, 8: IoError, 9: CudaError}

SF_PATTERN = {"sliding": 0, "dilated": 1, "global": 2, "random": 3, "longformer": 4, "bigbird": 5,
              "causal": 6, "causal_local": 7, "strided": 8}
SF_F16, SF_BF16 = 0, 1
SF_ROW_WISE, SF_BLOCK_WISE = 0, 1
SF_PLAN_REFERENCE, SF_PLAN_B200 = 0, 1
SF_ACT = {"none": 0, "gelu": 1, "relu": 2}


class MaskDesc(C.Structure):
    _fields_ = [("pattern", C.c_int32), ("seq_len", C.c_int32), ("band_width", C.c_int32),
                ("global_width", C.c_int32), ("dilation_rate", C.c_int32), ("block", C.c_int32),
                ("filling_rate", C.c_double), ("seed", C.c_uint64)]


class BsrDev(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("seq_len", "block_m", "block_n", "n_rows", "n_cols", "n_full",
                                         "n_part", "n_load", "n_pool", "tile_bytes")] + \
               [(n, C.c_void_p) for n in ("full_row_ptr", "full_col_idx", "part_row_ptr", "part_col_idx",
                                          "part_tile_ids", "load_row_ptr", "load_col_idx", "load_tile",
                                          "pool", "_alloc")]


class CsrDev(C.Structure):
    _fields_ = [("seq_len", C.c_int32), ("nnz", C.c_int64), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
                ("_alloc", C.c_void_p)]


class HwSpec(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("sm_num", C.c_int32), ("smem_size", C.c_int64),
                ("max_warp", C.c_int32), ("element_bytes", C.c_int32)]


class Plan(C.Structure):
    _fields_ = [("kind", C.c_int32), ("block_m", C.c_int32), ("block_n", C.c_int32), ("num_warps", C.c_int32),
                ("score", C.c_double), ("threshold", C.c_double), ("fallback", C.c_int32)]


class AttnArgs(C.Structure):
    _fields_ = [("bs", C.c_int32), ("h", C.c_int32), ("seq_len", C.c_int32), ("head_size", C.c_int32),
                ("dtype", C.c_int32), ("q", C.c_void_p), ("k", C.c_void_p), ("v", C.c_void_p), ("o", C.c_void_p),
                ("q_sb", C.c_int64), ("q_sh", C.c_int64), ("q_sn", C.c_int64),
                ("o_sb", C.c_int64), ("o_sh", C.c_int64), ("o_sn", C.c_int64), ("scale", C.c_float)]


class AttnStats(C.Structure):
    _fields_ = [("tiles_loaded", C.c_int64), ("full_tiles", C.c_int64), ("part_tiles", C.c_int64)]


class GemmEpilogue(C.Structure):
    _fields_ = [("bias", C.c_void_p), ("act", C.c_int32), ("aux", C.c_void_p), ("ldaux", C.c_int64),
                ("ln_gamma", C.c_void_p), ("ln_beta", C.c_void_p), ("out_pre_ln", C.c_void_p),
                ("softmax", C.c_int32)]


class GemmArgs(C.Structure):
    _fields_ = [("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32), ("dtype", C.c_int32),
                ("x", C.c_void_p), ("ldx", C.c_int64), ("w", C.c_void_p), ("ldw", C.c_int64),
                ("out", C.c_void_p), ("ldout", C.c_int64), ("epi", GemmEpilogue), ("tile_n", C.c_int32)]


class GemmChainArgs(C.Structure):
    _fields_ = [("M", C.c_int32), ("K1", C.c_int32), ("N1", C.c_int32), ("N2", C.c_int32), ("dtype", C.c_int32),
                ("x", C.c_void_p), ("ldx", C.c_int64), ("w1", C.c_void_p), ("ldw1", C.c_int64),
                ("w2", C.c_void_p), ("ldw2", C.c_int64), ("out", C.c_void_p), ("ldout", C.c_int64),
                ("mid", GemmEpilogue), ("post", GemmEpilogue)]


LAUNCH_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)

# Every symbol include/sf_capi.h declares, with its ctypes signature.
_P, _I32, _I64, _D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
SIGNATURES = {
    "sf_last_error": (C.c_char_p, []),
    "sf_version": (C.c_char_p, []),
    "sf_mask_words": (_I32, [_I32]),
    "sf_mask_validate": (C.c_int, [C.POINTER(MaskDesc), _I32]),
    "sf_mask_generate": (C.c_int, [C.POINTER(MaskDesc), _I32, _P, _P]),
    "sf_mask_pack_u8": (C.c_int, [_P, _I32, _P, _P]),
    "sf_mask_count": (C.c_int, [_P, _I32, C.POINTER(_I64), _P]),
    "sf_mask_or": (C.c_int, [_P, _P, _I32, _P]),
    "sf_mask_andnot": (C.c_int, [_P, _P, _I32, _P]),
    "sf_bsr_build": (C.c_int, [_P, _I32, _I32, _I32, C.POINTER(BsrDev), _P]),
    "sf_bsr_free": (C.c_int, [C.POINTER(BsrDev), _P]),
    "sf_bsr_to_host": (C.c_int, [C.POINTER(BsrDev)] + [_P] * 8 + [_P]),
    "sf_bsr_serialize": (C.c_int, [C.POINTER(BsrDev), _P, _I64, C.POINTER(_I64), _P]),
    "sf_bsr_validate": (C.c_int, [C.POINTER(BsrDev), _P]),
    "sf_bsr_workspace": (C.c_int, [_I32, _I32, _I32, C.POINTER(BsrDev), _P]),
    "sf_bsr_build_async": (C.c_int, [_P, C.POINTER(BsrDev), _P, _P]),
    "sf_bsr_to_dense": (C.c_int, [C.POINTER(BsrDev), _P, _P]),
    "sf_bsr_from_host": (C.c_int, [_I32] * 7 + [_P] * 8 + [C.POINTER(BsrDev), _P]),
    "sf_mask_serialize": (C.c_int, [_P, _I32, _P, _I64, C.POINTER(_I64), _P]),
    "sf_mask_deserialize": (C.c_int, [_P, _I64, C.POINTER(_I32), _P, _P]),
    "sf_rowwise_build": (C.c_int, [_P, _I32, C.POINTER(CsrDev), _P]),
    "sf_csr_free": (C.c_int, [C.POINTER(CsrDev), _P]),
    "sf_csr_to_host": (C.c_int, [C.POINTER(CsrDev), _P, _P, _P]),
    "sf_hw_preset": (C.c_int, [C.c_char_p, C.POINTER(HwSpec)]),
    "sf_threshold": (C.c_int, [_P, _I32, _D, C.POINTER(_D), _P]),
    "sf_threshold_from_loads": (_D, [_I32, _I64, _D]),
    "sf_select_plan": (C.c_int, [_P, C.POINTER(HwSpec), _I64, _I32, _I64, _I32, _I32, C.POINTER(Plan), _P]),
    "sf_select_plan_from_loads": (C.c_int, [_I64, C.POINTER(HwSpec), _I64, _I32, _I64, _I32, _I32, C.POINTER(Plan)]),
    "sf_mha_blockwise": (C.c_int, [C.POINTER(AttnArgs), C.POINTER(BsrDev), C.POINTER(Plan), C.POINTER(AttnStats), _P]),
    "sf_mha_rowwise": (C.c_int, [C.POINTER(AttnArgs), C.POINTER(CsrDev), _P]),
    "sf_mha_strided": (C.c_int, [C.POINTER(AttnArgs), _I32, C.POINTER(BsrDev), _P]),
    "sf_mha_dilated": (C.c_int, [C.POINTER(AttnArgs), _I32, C.POINTER(BsrDev), C.POINTER(BsrDev), _P]),
    "sf_mha_dense_oracle": (C.c_int, [C.POINTER(AttnArgs), _P, _P, _P]),
    "sf_set_attn_impl": (C.c_int, [_I32]),
    "sf_set_pdl": (C.c_int, [_I32]),
    "sf_get_attn_impl": (_I32, []),
    "sf_gemm_fused": (C.c_int, [C.POINTER(GemmArgs), _P]),
    "sf_gemm_chain": (C.c_int, [C.POINTER(GemmChainArgs), _P]),
    "sf_mi_chain": (C.c_int, [_I32, _I32, _I32, _P, _I64, C.POINTER(GemmEpilogue), _P, _I64, _P]),
    "sf_time_best": (C.c_int, [LAUNCH_FN, _P, _I32, _I32, C.POINTER(C.c_float), _P]),
    "sf_launch_count": (_I64, []),
}

_lib = None


def lib():
    """Load the sm_100a library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status:
        msg = lib().sf_last_error().decode(errors="replace")
        raise _STATUS.get(status, SfError)(msg)


def version() -> str:
    return lib().sf_version().decode()


def launch_count() -> int:
    return int(lib().sf_launch_count())
