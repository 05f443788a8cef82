"""Fused templates (tcgen05 GEMM + epilogues, MI chain) vs the per-op oracle semantics
(backend.hpp:111-306; oracles.hpp:114-194 naive_apply_op), on fp16-rounded operands.
Tolerance: the north-star bar, max-abs 2e-2 and mean-rel 1e-3 against fp32 results."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
MAX_ABS, MEAN_REL = 2e-2, 1e-3


def parity(out, ref, max_abs=MAX_ABS, mean_rel=MEAN_REL):
    out = out.float().cpu().numpy().astype(np.float64)
    ref = np.asarray(ref, np.float64)
    d = np.abs(out - ref)
    ma, mr = float(d.max()), float(d.sum() / np.abs(ref).sum())
    assert ma <= max_abs and mr <= mean_rel, f"max_abs {ma:.3e} mean_rel {mr:.3e}"


def r16(x):
    return x.astype(np.float16).astype(np.float32)


def dev(x, dt=None):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt or torch.float16)


@pytest.fixture(scope="module")
def fz():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_06095_b200 import fused
    return fused


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 768, 768), (300, 512, 192), (1024, 2304, 768),
                                   (512, 768, 3072), (128, 96, 64)])
def test_gemm_plain(fz, oracle, M, N, K):
    x = r16(oracle.random_matrix(M, K, 1))
    w = r16(oracle.random_matrix(K, N, 2, -1 / np.sqrt(K), 1 / np.sqrt(K)))  # GraphData Gemm init (backend.hpp:80-81)
    out = fz.gemm_fused(dev(x), dev(w.T))
    parity(out, oracle.gemm(x, w, threads=8))


@pytest.mark.parametrize("act", ["gelu", "relu"])
def test_gemm_bias_act(fz, oracle, act):
    import torch
    M, N, K = 512, 3072, 768
    x = r16(oracle.random_matrix(M, K, 3))
    w = r16(oracle.random_matrix(K, N, 4, -1 / np.sqrt(K), 1 / np.sqrt(K)))
    b = oracle.random_matrix(1, N, 5, -0.5, 0.5)[0]
    ref = oracle.gelu(oracle.bias(oracle.gemm(x, w, 8), b)) if act == "gelu" else oracle.relu(oracle.bias(oracle.gemm(x, w, 8), b))
    out = fz.gemm_fused(dev(x), dev(w.T), bias=dev(b, torch.float32), act=act)
    parity(out, ref)


@pytest.mark.parametrize("N,K", [(768, 768), (768, 3072), (512, 256), (256, 128)])
def test_gemm_bias_add_layernorm(fz, oracle, N, K):
    import torch
    M = 384
    x = r16(oracle.random_matrix(M, K, 6))
    w = r16(oracle.random_matrix(K, N, 7, -1 / np.sqrt(K), 1 / np.sqrt(K)))
    b = oracle.random_matrix(1, N, 8, -0.5, 0.5)[0]
    aux = r16(oracle.random_matrix(M, N, 9))
    g = 0.5 + oracle.random_matrix(1, N, 10, 0, 1)[0]
    be = oracle.random_matrix(1, N, 11, -0.5, 0.5)[0]
    pre = oracle.add(oracle.bias(oracle.gemm(x, w, 8), b), aux)
    ref = oracle.layernorm(pre, g, be)
    pre_dev = torch.empty((M, N), dtype=torch.float16, device="cuda")
    out = fz.gemm_fused(dev(x), dev(w.T), bias=dev(b, torch.float32), aux=dev(aux), ln_gamma=dev(g, torch.float32),
                        ln_beta=dev(be, torch.float32), out_pre_ln=pre_dev)
    parity(out, ref)
    parity(pre_dev, pre)


def test_mi_chain(fz, oracle):
    import torch
    M, N = 1000, 768
    x = r16(oracle.random_matrix(M, N, 12))
    b = oracle.random_matrix(1, N, 13, -0.5, 0.5)[0]
    aux = r16(oracle.random_matrix(M, N, 14))
    g = 0.5 + oracle.random_matrix(1, N, 15, 0, 1)[0]
    be = oracle.random_matrix(1, N, 16, -0.5, 0.5)[0]
    ref = oracle.layernorm(oracle.add(oracle.gelu(oracle.bias(x, b)), aux), g, be)
    out = fz.mi_chain(dev(x), bias=dev(b, torch.float32), act="gelu", aux=dev(aux), ln_gamma=dev(g, torch.float32),
                      ln_beta=dev(be, torch.float32))
    parity(out, ref)


def test_gemm_shape_errors(fz):
    import torch
    from paper_2506_06095_b200 import _lib
    x = torch.zeros(128, 64, dtype=torch.float16, device="cuda")
    with pytest.raises(_lib.ShapeError):
        fz.gemm_fused(x, torch.zeros(128, 32, dtype=torch.float16, device="cuda"))
    with pytest.raises(_lib.ShapeError):  # LN over a row that cannot be split into <= 8 CTAs of 128/256
        fz.gemm_fused(x, torch.zeros(96, 64, dtype=torch.float16, device="cuda"),
                      ln_gamma=torch.ones(96, device="cuda"), ln_beta=torch.zeros(96, device="cuda"))
