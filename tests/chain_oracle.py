"""CPU oracle of a preset layer chain (fusion.hpp:350-397) composed from the pinned per-op oracle
functions (oracle/sf_oracle.c: gemm/bias/add/gelu/relu/layernorm + block_sparse_sdpa).
TEST INFRASTRUCTURE ONLY.

GraphData seeds (backend.hpp:65-106): input = random_matrix(rows, in_cols, mix_seed(seed, 0xa11));
node p: s = mix_seed(seed, id); Gemm W ~ U(+-1/sqrt(inner)) shape inner x cols; Bias U[-.5,.5);
LN gamma U[.5,1.5) then beta U[-.5,.5) from one stream; Add aux U[-1,1) rows x cols.
"""
import numpy as np

from oracle.oracle import make_desc  # noqa: F401

BERT = ["mha", "gemm", "bias", "add", "ln", "gemm", "bias", "gelu", "gemm", "bias", "add", "ln"]
GPT = ["ln", "mha", "gemm", "bias", "add", "ln", "gemm", "bias", "gelu", "gemm", "bias", "add"]
T5 = ["ln", "mha", "gemm", "bias", "add", "ln", "gemm", "bias", "relu", "gemm", "bias", "add"]
CHAINS = {"bert-layer": BERT, "gpt-layer": GPT, "t5-layer": T5}


def graph_data(o, model, bs, seq, hidden, ff, seed):
    """Per-node parameters exactly as GraphData::make (pinned by test_graph_params_restated)."""
    rows = bs * seq
    ops = CHAINS[model]
    cols = []
    inner = []
    for op_i, op in enumerate(ops):
        # shapes of build_preset_graph: the FFN-1 gemm/bias/act nodes are ff wide
        c = hidden
        if model == "bert-layer" and op_i in (5, 6, 7):
            c = ff
        if model != "bert-layer" and op_i in (6, 7, 8):
            c = ff
        cols.append(c)
    for op_i, op in enumerate(ops):
        inner.append((ff if (model == "bert-layer" and op_i == 8) or (model != "bert-layer" and op_i == 9) else hidden)
                     if op == "gemm" else 0)
    gd = {"input": o.random_matrix(rows, hidden, o.mix_seed(seed, 0xa11)), "params": []}
    for i, op in enumerate(ops):
        s = o.mix_seed(seed, i)
        p = {}
        if op == "gemm":
            a = np.float32(1.0) / np.sqrt(np.float32(inner[i]))
            p["w"] = o.random_matrix(inner[i], cols[i], s, -a, a)
        elif op == "bias":
            p["b"] = o.random_matrix(1, cols[i], s, 0.0, 1.0)[0] - np.float32(0.5)
        elif op == "ln":
            gb = o.random_matrix(1, 2 * cols[i], s, 0.0, 1.0)[0]
            p["g"] = np.float32(0.5) + gb[: cols[i]]
            p["beta"] = gb[cols[i]:] - np.float32(0.5)
        elif op == "add":
            p["aux"] = o.random_matrix(rows, cols[i], s)
        gd["params"].append(p)
    return gd


def run_chain(o, model, gd, x, mask, bs, seq, heads, head_size, bm=16, bn=16, threads=8, qkv=None):
    """Unfused chain on fp32 numpy (the values every fusion scheme must reproduce).
    qkv: optional (wqkv K x 3H, bqkv) to add the projection the reference abstracts away; then
    residual Adds use the skip activations instead of aux (the real-model variant)."""
    ops = CHAINS[model]
    cur = x.astype(np.float32)
    skip = cur
    adds = 0
    for i, op in enumerate(ops):
        p = gd["params"][i]
        if op == "mha":
            src = cur
            if qkv is None:
                q = k = v = src.reshape(bs, seq, heads, head_size).transpose(0, 2, 1, 3)
            else:
                t = o.bias(o.gemm(src, qkv[0], threads), qkv[1])
                H = heads * head_size
                q, k, v = (t[:, j * H:(j + 1) * H].reshape(bs, seq, heads, head_size).transpose(0, 2, 1, 3)
                           for j in range(3))
            out, _ = o.block_sparse_sdpa(np.ascontiguousarray(q), np.ascontiguousarray(k), np.ascontiguousarray(v),
                                         mask, bm, bn, threads)
            cur = out.transpose(0, 2, 1, 3).reshape(bs * seq, heads * head_size)
        elif op == "gemm":
            cur = o.gemm(cur, p["w"], threads)
        elif op == "bias":
            cur = o.bias(cur, p["b"])
        elif op == "add":
            if qkv is None:
                cur = o.add(cur, p["aux"])
            else:
                cur = o.add(cur, skip)
            adds += 1
        elif op == "ln":
            cur = o.layernorm(cur, p["g"], p["beta"])
        elif op == "gelu":
            cur = o.gelu(cur)
        elif op == "relu":
            cur = o.relu(cur)
        # residual stream bookkeeping for the real-model variant
        if qkv is not None:
            if model == "bert-layer" and i == 4:
                skip = cur            # X1 feeds the second residual
            if model != "bert-layer" and i == 4:
                skip = cur            # X1 (pre-LN2) feeds the second residual
    return cur
