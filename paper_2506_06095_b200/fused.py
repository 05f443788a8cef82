"""Fused segment templates over the C ABI (backend.hpp:228-306 exec_mi_chain / exec_ci_mi).

Weights are kept in the kernel-native layout: a reference Gemm weight (inner x cols, row-major,
backend.hpp:54,81) is stored transposed as (cols x inner) = (N x K) row-major, the K-major
operand TMA stages for tcgen05. Bias / LayerNorm parameters stay fp32.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import _lib
from ._lib import GemmArgs, GemmChainArgs, GemmEpilogue, SF_ACT, check, lib
from .sparsefuse import _dtype_code, _stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def epilogue(bias=None, act: str = "none", aux=None, ln_gamma=None, ln_beta=None, out_pre_ln=None,
             softmax: bool = False) -> GemmEpilogue:
    for t in (bias, ln_gamma, ln_beta):
        if t is not None and t.dtype != torch.float32:
            raise _lib.InvalidParameter("bias / LayerNorm parameters must be float32")
    return GemmEpilogue(_ptr(bias), SF_ACT[act], _ptr(aux), aux.stride(0) if aux is not None else 0,
                        _ptr(ln_gamma), _ptr(ln_beta), _ptr(out_pre_ln), 1 if softmax else 0)


TILE_AUTO, TILE_PAIR = 0, 1  # sf_gemm_args.tile_n: SF_TILE_AUTO / SF_TILE_PAIR (or 128 / 256)


def gemm_fused(x: torch.Tensor, w_nk: torch.Tensor, out: Optional[torch.Tensor] = None, *, bias=None,
               act: str = "none", aux=None, ln_gamma=None, ln_beta=None, out_pre_ln=None, tile_n: int = 0,
               softmax: bool = False, stream=None) -> torch.Tensor:
    """out = LN(act(x @ w_nk.T + bias) + aux) — the CiMi template: one tcgen05 kernel (LayerNorm in
    the cluster epilogue), or with tile_n auto on small grids / unclusterable rows, the GEMM followed
    by a MiChain LayerNorm pass."""
    M, K = x.shape
    N, K2 = w_nk.shape
    if K != K2:
        raise _lib.ShapeError("gemm input width mismatch")  # backend.hpp:245
    if out is None:
        out = torch.empty((M, N), dtype=x.dtype, device=x.device)
    for t in (x, w_nk, out):
        if t.stride(1) != 1:
            raise _lib.ShapeError("GEMM operands must be row-major")
    a = GemmArgs(M, N, K, _dtype_code(x), x.data_ptr(), x.stride(0), w_nk.data_ptr(), w_nk.stride(0),
                 out.data_ptr(), out.stride(0), epilogue(bias, act, aux, ln_gamma, ln_beta, out_pre_ln, softmax), tile_n)
    check(lib().sf_gemm_fused(C.byref(a), _stream(stream)))
    return out


def mi_chain(x: torch.Tensor, out: Optional[torch.Tensor] = None, *, bias=None, act: str = "none", aux=None,
             ln_gamma=None, ln_beta=None, out_pre_ln=None, softmax: bool = False, stream=None) -> torch.Tensor:
    """The MiChain template: bias -> act -> +aux -> LayerNorm or Softmax (row ops, backend.hpp:140-167)
    in one pass."""
    M, N = x.shape
    if out is None:
        out = torch.empty_like(x)
    e = epilogue(bias, act, aux, ln_gamma, ln_beta, out_pre_ln, softmax)
    check(lib().sf_mi_chain(M, N, _dtype_code(x), x.data_ptr(), x.stride(0), C.byref(e), out.data_ptr(),
                            out.stride(0), _stream(stream)))
    return out


def gemm_chain(x: torch.Tensor, w1_nk: torch.Tensor, w2_nk: torch.Tensor, out: Optional[torch.Tensor] = None, *,
               bias1=None, act: str = "none", bias2=None, aux=None, ln_gamma=None, ln_beta=None, out_pre_ln=None,
               stream=None) -> torch.Tensor:
    """The CiCi template chained on chip (backend.hpp:270-306): out = LN(act(x @ w1.T + bias1) @ w2.T
    + bias2 + aux); the intermediate stays in shared memory (sf_gemm_chain)."""
    M, K1 = x.shape
    N1, K1b = w1_nk.shape
    N2, N1b = w2_nk.shape
    if K1 != K1b or N1 != N1b:
        raise _lib.ShapeError("gemm chain width mismatch")  # backend.hpp:278
    if out is None:
        out = torch.empty((M, N2), dtype=x.dtype, device=x.device)
    for t in (x, w1_nk, w2_nk, out):
        if t.stride(1) != 1:
            raise _lib.ShapeError("GEMM operands must be row-major")
    a = GemmChainArgs(M, K1, N1, N2, _dtype_code(x), x.data_ptr(), x.stride(0), w1_nk.data_ptr(), w1_nk.stride(0),
                      w2_nk.data_ptr(), w2_nk.stride(0), out.data_ptr(), out.stride(0), epilogue(bias1, act),
                      epilogue(bias2, "none", aux, ln_gamma, ln_beta, out_pre_ln))
    check(lib().sf_gemm_chain(C.byref(a), _stream(stream)))
    return out
