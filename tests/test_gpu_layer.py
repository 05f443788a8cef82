"""Fused encoder layers on the GPU vs the composed chain oracle (pinned to the reference's
CpuBackend::run_chain in test_oracle_vs_ref). Weights/inputs are the GraphData seeds rounded to
fp16; the oracle runs fp32 on those values. Bar: max-abs 2e-2, mean-rel 1e-3."""
import numpy as np
import pytest

from tests.chain_oracle import graph_data, run_chain

pytestmark = pytest.mark.gpu


def r16(x):
    return x.astype(np.float16).astype(np.float32)


def parity(out, ref, max_abs=2e-2, mean_rel=1e-3):
    out = out.float().cpu().numpy().astype(np.float64)
    d = np.abs(out - ref)
    ma, mr = float(d.max()), float(d.sum() / np.abs(ref).sum())
    assert ma <= max_abs and mr <= mean_rel, f"max_abs {ma:.3e} mean_rel {mr:.3e}"
    return ma, mr


def build(sf, layer, o, model, bs, seq, hid, heads, terms, compat, ln_split=False):
    import torch
    hs = hid // heads
    gd = graph_data(o, model, bs, seq, hid, 4 * hid, 1)
    ops = {"bert-layer": (1, 2, 4, 5, 6, 8, 9, 11, None), "gpt-layer": (2, 3, 5, 6, 7, 9, 10, 5, 0),
           "t5-layer": (2, 3, 5, 6, 7, 9, 10, 5, 0)}[model]
    g_wo, g_bo, g_ln_a, g_w1, g_b1, g_w2, g_b2, g_ln_b, g_ln0 = ops
    P = gd["params"]
    for p in P:
        for k in ("w", "aux"):
            if k in p:
                p[k] = r16(p[k])
    dev = lambda a, dt=torch.float16: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)
    f32 = torch.float32
    if model == "bert-layer":
        W = {"wo": dev(P[g_wo]["w"].T), "bo": dev(P[g_bo]["b"], f32), "w1": dev(P[g_w1]["w"].T),
             "b1": dev(P[g_b1]["b"], f32), "w2": dev(P[g_w2]["w"].T), "b2": dev(P[g_b2]["b"], f32),
             "ln1_g": dev(P[g_ln_a]["g"], f32), "ln1_b": dev(P[g_ln_a]["beta"], f32),
             "ln2_g": dev(P[11]["g"], f32), "ln2_b": dev(P[11]["beta"], f32)}
        aux = {"add1": dev(P[3]["aux"]), "add2": dev(P[10]["aux"])} if compat else None
    else:
        W = {"wo": dev(P[2]["w"].T), "bo": dev(P[3]["b"], f32), "w1": dev(P[6]["w"].T), "b1": dev(P[7]["b"], f32),
             "w2": dev(P[9]["w"].T), "b2": dev(P[10]["b"], f32), "ln1_g": dev(P[0]["g"], f32),
             "ln1_b": dev(P[0]["beta"], f32), "ln2_g": dev(P[5]["g"], f32), "ln2_b": dev(P[5]["beta"], f32)}
        aux = {"add1": dev(P[4]["aux"]), "add2": dev(P[11]["aux"])} if compat else None
    qkv = None
    if not compat:
        rng = np.random.default_rng(5)
        a = 1 / np.sqrt(hid)
        wq = r16(rng.uniform(-a, a, (hid, 3 * hid)).astype(np.float32))
        bq = rng.uniform(-0.5, 0.5, 3 * hid).astype(np.float32)
        W["wqkv"] = dev(wq.T)
        W["bqkv"] = dev(bq, f32)
        qkv = (wq, bq)
    x = r16(gd["input"])
    dm = sf.generate_mask(terms)
    plan = sf.select_plan(dm, sf.hw_preset("b200"), seq, heads, bs, hs, mode="b200")
    ctx = sf.MhaContext(dm, plan)
    shape = layer.LayerShape(bs, seq, hid, heads, hs)
    L = layer.EncoderLayer(model, shape, W, ctx, compat=compat, aux=aux, ln_split=ln_split)
    ref = run_chain(o, model, gd, x, o.mask(terms), bs, seq, heads, hs, 16, 16, threads=8, qkv=qkv)
    return L, dev(x), ref


@pytest.mark.parametrize("model", ["bert-layer", "gpt-layer", "t5-layer"])
@pytest.mark.parametrize("compat", [True, False])
@pytest.mark.parametrize("ln_split", [False, True])
def test_layer_matches_chain_oracle(sf, oracle, model, compat, ln_split):
    from paper_2506_06095_b200 import layer
    bs, seq, hid, heads = 2, 256, 256, 4
    terms = [dict(pattern="bigbird", seq_len=seq, global_width=16, band_width=16, filling_rate=0.1, seed=0)]
    L, x, ref = build(sf, layer, oracle, model, bs, seq, hid, heads, terms, compat, ln_split)
    parity(L.forward(x), ref)


@pytest.mark.parametrize("model", ["bert-layer", "gpt-layer"])
def test_layer_cluster_layernorm_path(sf, oracle, model):
    """M = 4096 rows: the out-projection / FFN2 LayerNorms run in the GEMM's cluster epilogue
    (the small layers above take the GEMM + MiChain path)."""
    from paper_2506_06095_b200 import layer
    bs, seq, hid, heads = 4, 1024, 256, 4
    terms = [dict(pattern="bigbird", seq_len=seq, global_width=32, band_width=32, filling_rate=0.1, seed=0)]
    L, x, ref = build(sf, layer, oracle, model, bs, seq, hid, heads, terms, False)
    parity(L.forward(x), ref)


def test_layer_cuda_graph_replay(sf, oracle):
    import torch
    from paper_2506_06095_b200 import layer
    terms = [dict(pattern="sliding", seq_len=512, band_width=22)]
    L, x, ref = build(sf, layer, oracle, "bert-layer", 1, 512, 768, 12, terms, False)
    L.capture(x)
    L.out.zero_()
    out = L.replay()
    torch.cuda.synchronize()
    parity(out, ref)


@pytest.mark.parametrize("cross", ["dense", "bigbird"])
def test_t5_decoder_layer_cross_attention(sf, oracle, cross):
    """T5 decoder layer (F3): causal self-attention, encoder-decoder cross-attention (dense or a
    sparse cross mask), ReLU FFN, three pre-norm LayerNorms; vs the same chain composed from the
    pinned per-op oracle functions in fp32 on the fp16-rounded weights and inputs."""
    import torch
    from paper_2506_06095_b200 import layer
    bs, seq, hid, heads = 2, 256, 256, 4
    hs, ff = hid // heads, 4 * hid
    o = oracle
    rng = np.random.default_rng(7)
    a = lambda k: 1 / np.sqrt(k)
    mat = lambda k, n: r16(rng.uniform(-a(k), a(k), (k, n)).astype(np.float32))  # reference layout inner x cols
    vec = lambda n, lo, hi: rng.uniform(lo, hi, n).astype(np.float32)
    P = {"wqkv": mat(hid, 3 * hid), "bqkv": vec(3 * hid, -.5, .5), "wo": mat(hid, hid), "bo": vec(hid, -.5, .5),
         "wqc": mat(hid, hid), "bqc": vec(hid, -.5, .5), "wkvc": mat(hid, 2 * hid), "bkvc": vec(2 * hid, -.5, .5),
         "woc": mat(hid, hid), "boc": vec(hid, -.5, .5), "w1": mat(hid, ff), "b1": vec(ff, -.5, .5),
         "w2": mat(ff, hid), "b2": vec(hid, -.5, .5)}
    for i in (1, 2, 3):
        P[f"ln{i}_g"], P[f"ln{i}_b"] = vec(hid, .5, 1.5), vec(hid, -.5, .5)
    x = r16(rng.uniform(-1, 1, (bs * seq, hid)).astype(np.float32))
    enc = r16(rng.uniform(-1, 1, (bs * seq, hid)).astype(np.float32))
    self_terms = [dict(pattern="causal", seq_len=seq)]
    cross_terms = ([dict(pattern="sliding", seq_len=seq, band_width=seq)] if cross == "dense" else
                   [dict(pattern="bigbird", seq_len=seq, global_width=16, band_width=16, filling_rate=0.1, seed=4)])

    # oracle composition (fp32)
    def split(t, c0):
        return np.ascontiguousarray(t[:, c0:c0 + hid].reshape(bs, seq, heads, hs).transpose(0, 2, 1, 3))

    def attn(q, k, v, terms):
        out, _ = o.block_sparse_sdpa(q, k, v, o.mask(terms), 16, 16, 8)
        return out.transpose(0, 2, 1, 3).reshape(bs * seq, hid)

    h = o.layernorm(x, P["ln1_g"], P["ln1_b"])
    qkv = o.bias(o.gemm(h, P["wqkv"], 8), P["bqkv"])
    x1 = o.add(o.bias(o.gemm(attn(split(qkv, 0), split(qkv, hid), split(qkv, 2 * hid), self_terms), P["wo"], 8),
                      P["bo"]), x)
    h2 = o.layernorm(x1, P["ln2_g"], P["ln2_b"])
    qc = o.bias(o.gemm(h2, P["wqc"], 8), P["bqc"])
    kvc = o.bias(o.gemm(enc, P["wkvc"], 8), P["bkvc"])
    x2 = o.add(o.bias(o.gemm(attn(split(qc, 0), split(kvc, 0), split(kvc, hid), cross_terms), P["woc"], 8), P["boc"]),
               x1)
    h3 = o.layernorm(x2, P["ln3_g"], P["ln3_b"])
    ref = o.add(o.bias(o.gemm(o.relu(o.bias(o.gemm(h3, P["w1"], 8), P["b1"])), P["w2"], 8), P["b2"]), x2)

    dev = lambda t, dt=torch.float16: torch.from_numpy(np.ascontiguousarray(t)).to("cuda", dt)
    W = {k: (dev(v.T) if v.ndim == 2 else dev(v, torch.float32)) for k, v in P.items()}
    ctx = lambda terms: sf.MhaContext(sf.generate_mask(terms), sf.select_plan(
        sf.generate_mask(terms), sf.hw_preset("b200"), seq, heads, bs, hs, mode="b200"))
    L = layer.DecoderLayer(layer.LayerShape(bs, seq, hid, heads, hs), W, ctx(self_terms), ctx(cross_terms))
    xd, ed = dev(x), dev(enc)
    parity(L.forward(xd, ed), ref)
    # the same step replayed as one CUDA graph
    L.capture(xd, ed)
    L.out.zero_()
    out = L.replay()
    torch.cuda.synchronize()
    parity(out, ref)
