"""The C restatement reproduces the reference-generated golden fixtures (CPU only)."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import CONFIG_MASKS

G = Path(__file__).resolve().parent / "golden"
FP = json.loads((G / "fingerprints.json").read_text())
PLANS = json.loads((G / "plans.json").read_text())

# SURVEY §8(c) published fingerprints (FNV-1a of the SFBR bytes), frozen here independently.
SURVEY_FNV = {
    ("cfg1", "16x16"): "c85e9687d60cee9c", ("cfg1", "64x16"): "b40769b9aeed53c6", ("cfg1", "128x64"): "2b5b9e7374822529",
    ("cfg2", "16x16"): "23d58a3f0e2c0415", ("cfg2", "64x16"): "2aeab4721d3094f5", ("cfg2", "128x64"): "2e353365a82b9c4e",
    ("cfg3", "16x16"): "d38d6458a38b7650", ("cfg3", "64x16"): "29bbb12a6a0f0ba5", ("cfg3", "128x64"): "f88519af0bb842c2",
    ("cfg4", "16x16"): "4ba6b7c0652f3b29", ("cfg4", "64x16"): "74183fbbc673448f", ("cfg4", "128x64"): "87e976bfc2dfa03d",
}


def test_fixtures_agree_with_survey():
    for (cfg, tile), h in SURVEY_FNV.items():
        assert FP[cfg]["tiles"][tile]["fnv"] == h


@pytest.mark.parametrize("cfg", list(CONFIG_MASKS))
def test_oracle_reproduces_fingerprints(oracle, cfg):
    m = oracle.mask(CONFIG_MASKS[cfg])
    ent = FP[cfg]
    assert int(m.sum()) == ent["true_count"]
    rp, ci = oracle.rowwise(m)
    assert "%016x" % oracle.fnv1a(rp.tobytes() + ci.tobytes()) == ent["rowwise_fnv"]
    for tile, t in ent["tiles"].items():
        bm, bn = map(int, tile.split("x"))
        b = oracle.bsr(m, bm, bn)["sfbr"]
        assert "%016x" % oracle.fnv1a(b) == t["fnv"], tile


def test_oracle_reproduces_small_bsr_dumps(oracle):
    z = np.load(G / "bsr_small.npz")
    for i in range(24):
        n, bm, bn = z[f"{i}/shape"]
        m = np.unpackbits(z[f"{i}/mask"], bitorder="little")[: n * n].reshape(n, n)
        assert oracle.bsr(m, int(bm), int(bn))["sfbr"] == z[f"{i}/sfbr"].tobytes()


def test_oracle_reproduces_attention_fixtures(oracle):
    from tests.golden.make_golden import ATTN_CASES, fp16_round
    z = np.load(G / "attn_small.npz")
    for name, (terms, bm, bn, bs, h, d, seed) in ATTN_CASES.items():
        m = oracle.mask(terms)
        q, k, v = (fp16_round(x) for x in oracle.random_attention_input(bs, h, m.shape[0], d, seed))
        out, stats = oracle.block_sparse_sdpa(q, k, v, m, bm, bn)
        assert np.array_equal(out, z[name + "/out"]), name
        assert np.array_equal(stats, z[name + "/stats"]), name


@pytest.mark.parametrize("key", sorted(PLANS))
def test_oracle_reproduces_plans(oracle, key):
    cfg, preset = key.split("/")
    m = oracle.mask(CONFIG_MASKS[cfg])
    loads = int(oracle.bsr(m, 16, 16)["load_row_ptr"][-1])
    p = oracle.select_plan_from_loads(loads, oracle.hw_preset(preset), m.shape[0], 12, PLANS[key]["bs"], 64)
    e = PLANS[key]
    assert (p.kind, p.block_m, p.block_n, p.num_warps, p.fallback) == \
           (e["kind"], e["block_m"], e["block_n"], e["num_warps"], e["fallback"])
    assert p.score == e["score"] and p.threshold == e["threshold"]
