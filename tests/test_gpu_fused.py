"""Fused templates (tcgen05 GEMM + epilogues, MI chain) vs the per-op oracle semantics
(backend.hpp:111-306; oracles.hpp:114-194 naive_apply_op), on fp16-rounded operands.
Tolerance: the north-star bar, max-abs 2e-2 and mean-rel 1e-3 against fp32 results."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
MAX_ABS, MEAN_REL = 2e-2, 1e-3
PAIR = 1  # SF_TILE_PAIR: two-SM CTA-pair tiles (tcgen05 cta_group::2)


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
@pytest.mark.parametrize("tile", [0, PAIR])
def test_gemm_plain(fz, oracle, M, N, K, tile):
    if tile == PAIR and M <= 128:
        pytest.skip("CTA pairs need M > 128")
    x = r16(oracle.random_matrix(M, K, 1))
    w = r16(oracle.random_matrix(K, N, 2, -1 / np.sqrt(K), 1 / np.sqrt(K)))  # GraphData Gemm init (backend.hpp:80-81)
    out = fz.gemm_fused(dev(x), dev(w.T), tile_n=tile)
    parity(out, oracle.gemm(x, w, threads=8))


@pytest.mark.parametrize("act", ["gelu", "relu"])
@pytest.mark.parametrize("tile", [0, 128, PAIR])
def test_gemm_bias_act(fz, oracle, act, tile):
    import torch
    M, N, K = 512, 3072, 768
    x = r16(oracle.random_matrix(M, K, 3))
    w = r16(oracle.random_matrix(K, N, 4, -1 / np.sqrt(K), 1 / np.sqrt(K)))
    b = oracle.random_matrix(1, N, 5, -0.5, 0.5)[0]
    ref = oracle.gelu(oracle.bias(oracle.gemm(x, w, 8), b)) if act == "gelu" else oracle.relu(oracle.bias(oracle.gemm(x, w, 8), b))
    out = fz.gemm_fused(dev(x), dev(w.T), bias=dev(b, torch.float32), act=act, tile_n=tile)
    parity(out, ref)


@pytest.mark.parametrize("N,K", [(768, 768), (768, 3072), (512, 256), (256, 128), (1024, 256)])
@pytest.mark.parametrize("tile", [0, 128, 256, PAIR, "panel"])
def test_gemm_bias_add_layernorm(fz, oracle, N, K, tile, monkeypatch):
    """tile "panel": the row-panel LayerNorm GEMM (gemm2_ln.cu) forced at this short M (it is the
    automatic choice only when the panels fill most of the pairs, e.g. 16384 rows)."""
    if tile == "panel":
        monkeypatch.setenv("SF_GEMM_LN_PANEL", "1")
        tile = PAIR
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
                        ln_beta=dev(be, torch.float32), out_pre_ln=pre_dev, tile_n=tile)
    parity(out, ref)
    parity(pre_dev, pre)


@pytest.mark.parametrize("ln", [False, True])
@pytest.mark.parametrize("tile", [0, 256, PAIR])
def test_gemm_large_multi_tile(fz, ln, tile):
    """cfg2-sized GEMM (several tiles per persistent CTA / pair, accumulator double buffering and
    barrier phase wrap-around) against a torch fp32 reference of the same op."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(7)
    M, N, K = 16384, 768, 768
    x = torch.randn(M, K, device="cuda", generator=g).half()
    w = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).half()
    b = torch.randn(N, device="cuda", generator=g) * 0.5
    aux = torch.randn(M, N, device="cuda", generator=g).half()
    pre = x.float() @ w.float().T + b + aux.float()
    kw = dict(bias=b, aux=aux, tile_n=tile)
    if ln:
        gam = 0.5 + torch.rand(N, device="cuda", generator=g)
        bet = torch.rand(N, device="cuda", generator=g) - 0.5
        ref = torch.nn.functional.layer_norm(pre, (N,), gam, bet, eps=1e-5)
        kw.update(ln_gamma=gam, ln_beta=bet)
    else:
        ref = pre
    out = fz.gemm_fused(x, w, **kw)
    parity(out, ref.cpu().numpy())


@pytest.mark.parametrize("M,N", [(1000, 768), (37, 100), (9, 4096), (64, 7), (300, 1024), (50, 3072)])
@pytest.mark.parametrize("ln", [True, False])
def test_mi_chain(fz, oracle, M, N, ln):
    import torch
    x = r16(oracle.random_matrix(M, N, 12))
    b = oracle.random_matrix(1, N, 13, -0.5, 0.5)[0]
    aux = r16(oracle.random_matrix(M, N, 14))
    g = 0.5 + oracle.random_matrix(1, N, 15, 0, 1)[0]
    be = oracle.random_matrix(1, N, 16, -0.5, 0.5)[0]
    ref = oracle.add(oracle.gelu(oracle.bias(x, b)), aux)
    kw = dict(bias=dev(b, torch.float32), act="gelu", aux=dev(aux))
    if ln:
        ref = oracle.layernorm(ref, g, be)
        kw.update(ln_gamma=dev(g, torch.float32), ln_beta=dev(be, torch.float32))
    parity(fz.mi_chain(dev(x), **kw), ref)


@pytest.mark.parametrize("M,N", [(1000, 768), (37, 100), (9, 4096), (300, 1024), (50, 3072)])
def test_mi_chain_softmax(fz, oracle, M, N):
    """Softmax MI op (backend.hpp:113,155-167) after bias -> GELU -> residual, one MiChain pass."""
    import torch
    x = r16(oracle.random_matrix(M, N, 22))
    b = oracle.random_matrix(1, N, 23, -0.5, 0.5)[0]
    aux = r16(oracle.random_matrix(M, N, 24))
    ref = oracle.softmax(oracle.add(oracle.gelu(oracle.bias(x, b)), aux))
    out = fz.mi_chain(dev(x), bias=dev(b, torch.float32), act="gelu", aux=dev(aux), softmax=True)
    # probabilities ~1/N: the north-star max-abs bar holds trivially, mean-rel carries the check
    parity(out, ref)
    assert abs(out.float().sum(1).mean().item() - 1.0) < 1e-2


@pytest.mark.parametrize("tile", [0, PAIR])
def test_gemm_softmax(fz, oracle, tile):
    """CiMi with a trailing Softmax: GEMM + bias, then the row softmax pass."""
    import torch
    M, N, K = 512, 768, 256
    x = r16(oracle.random_matrix(M, K, 31))
    w = r16(oracle.random_matrix(K, N, 32, -0.1, 0.1))
    b = oracle.random_matrix(1, N, 33, -0.5, 0.5)[0]
    ref = oracle.softmax(oracle.bias(x.astype(np.float64) @ w.astype(np.float64), b))
    out = fz.gemm_fused(dev(x), dev(np.ascontiguousarray(w.T)), bias=dev(b, torch.float32), softmax=True, tile_n=tile)
    parity(out, ref)


def test_gemm_shape_errors(fz):
    import torch
    from paper_2506_06095_b200 import _lib
    x = torch.zeros(128, 64, dtype=torch.float16, device="cuda")
    with pytest.raises(_lib.ShapeError):
        fz.gemm_fused(x, torch.zeros(128, 32, dtype=torch.float16, device="cuda"))
    with pytest.raises(_lib.ShapeError):  # LN over a row that cannot be split into <= 8 CTAs of 128
        fz.gemm_fused(x, torch.zeros(96, 64, dtype=torch.float16, device="cuda"), tile_n=128,
                      ln_gamma=torch.ones(96, device="cuda"), ln_beta=torch.zeros(96, device="cuda"))


@pytest.mark.parametrize("M,N,K,pre", [(96, 96, 64, False), (512, 768, 768, True), (300, 800, 128, False)])
def test_gemm_ln_split_auto(fz, M, N, K, pre):
    """tile_n auto with a LayerNorm that the cluster epilogue cannot (or should not) take: GEMM +
    bias + residual, then a MiChain LayerNorm pass (in place, or from out_pre_ln)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(M + N)
    r = lambda *s: (torch.rand(*s, generator=g) * 2 - 1)
    x, w, aux = r(M, K).half(), (r(N, K) / K ** 0.5).half(), r(M, N).half()
    bias, gam, bet = r(N), r(N) + 1.5, r(N)
    s = x.float() @ w.float().t() + bias + aux.float()
    mu, var = s.mean(1, keepdim=True), s.var(1, unbiased=False, keepdim=True)
    ref = (s - mu) / torch.sqrt(var + 1e-5) * gam + bet
    dev = lambda t: t.cuda()
    pre_t = torch.empty(M, N, dtype=torch.float16, device="cuda") if pre else None
    out = fz.gemm_fused(dev(x), dev(w), bias=dev(bias), aux=dev(aux), ln_gamma=dev(gam), ln_beta=dev(bet),
                        out_pre_ln=pre_t)
    torch.cuda.synchronize()
    err = (out.float().cpu() - ref).abs()
    assert err.max().item() <= 2e-2 and err.sum().item() / ref.abs().sum().item() <= 1e-3
    if pre:
        assert (pre_t.float().cpu() - s).abs().max().item() <= 2e-2


@pytest.mark.parametrize("M,K1,N1,N2", [(512, 768, 3072, 768), (300, 256, 384, 384), (128, 128, 128, 192),
                                        (4096, 768, 3072, 768), (512, 256, 1024, 256), (200, 128, 256, 64)])
@pytest.mark.parametrize("post", ["ln", "bias_aux", "none"])
def test_gemm_chain(fz, oracle, M, K1, N1, N2, post):
    """The CiCi template chained on chip (sf_gemm_chain, backend.hpp:270-306): X -> GEMM1 -> bias ->
    GELU -> GEMM2 -> bias -> +aux -> LayerNorm, vs the per-op oracle with the intermediate rounded
    to fp16 (the activation dtype both the chained and the two-launch forms carry it in)."""
    import torch
    x = r16(oracle.random_matrix(M, K1, 21))
    w1 = r16(oracle.random_matrix(K1, N1, 22, -1 / np.sqrt(K1), 1 / np.sqrt(K1)))
    w2 = r16(oracle.random_matrix(N1, N2, 23, -1 / np.sqrt(N1), 1 / np.sqrt(N1)))
    b1 = oracle.random_matrix(1, N1, 24, -0.5, 0.5)[0]
    b2 = oracle.random_matrix(1, N2, 25, -0.5, 0.5)[0]
    aux = r16(oracle.random_matrix(M, N2, 26))
    g = 0.5 + oracle.random_matrix(1, N2, 27, 0, 1)[0]
    be = oracle.random_matrix(1, N2, 28, -0.5, 0.5)[0]
    h = r16(oracle.gelu(oracle.bias(oracle.gemm(x, w1, 8), b1)))
    y = oracle.gemm(h, w2, 8)
    kw = {}
    if post != "none":
        y = oracle.add(oracle.bias(y, b2), aux)
        kw = dict(bias2=dev(b2, torch.float32), aux=dev(aux))
    if post == "ln":
        y = oracle.layernorm(y, g, be)
        kw.update(ln_gamma=dev(g, torch.float32), ln_beta=dev(be, torch.float32))
    out = fz.gemm_chain(dev(x), dev(w1.T), dev(w2.T), bias1=dev(b1, torch.float32), act="gelu", **kw)
    parity(out, y)


def test_gemm_chain_shape_errors(fz):
    import torch
    from paper_2506_06095_b200 import _lib
    x = torch.zeros(256, 768, dtype=torch.float16, device="cuda")
    with pytest.raises(_lib.BackendError):  # N2 % 64 != 0
        fz.gemm_chain(x, torch.zeros(3072, 768, dtype=torch.float16, device="cuda"),
                      torch.zeros(96, 3072, dtype=torch.float16, device="cuda"))
    with pytest.raises(_lib.ShapeError):
        fz.gemm_chain(x, torch.zeros(3072, 512, dtype=torch.float16, device="cuda"),
                      torch.zeros(768, 3072, dtype=torch.float16, device="cuda"))
