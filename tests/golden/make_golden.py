"""Generate tests/golden/ fixtures from the REFERENCE itself (oracle/_ref/libsfref.so: the unmodified
/root/reference headers compiled in place). Run here, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

Outputs (committed):
  fingerprints.json — per config mask: true_count, row-wise nnz + FNV-1a of row_ptr||col_idx bytes,
                      per tile shape: FNV-1a of write_bsr bytes (io.hpp:103) and block counts.
                      cfg3 (causal+strided) has no reference generator; its mask comes from the
                      predicate in sf_capi.h, and its BSR from the reference build_bsr.
  plans.json        — select_plan (planner.hpp:130) per config mask and preset.
  attn_small.npz    — block_sparse_sdpa (attention.hpp:71) outputs on fp16-rounded
                      random_attention_input (tensor.hpp:62) for the test_attention.cpp shapes.
  bsr_small.npz     — full write_bsr dumps for small masks (test_bsr.cpp cases).
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
from oracle.oracle import CONFIG_MASKS, Oracle, Reference  # noqa: E402

TILES = [(16, 16), (64, 16), (128, 16), (128, 32), (128, 64), (128, 128)]

ATTN_CASES = {
    # name: (terms, bm, bn, bs, h, d, seed)
    "sliding64_16x16": ([dict(pattern="sliding", seq_len=64, band_width=8)], 16, 16, 2, 2, 16, 11),
    "dilated64_16x32": ([dict(pattern="dilated", seq_len=64, band_width=8, dilation_rate=1)], 16, 32, 2, 2, 16, 11),
    "bigbird100_16x16": ([dict(pattern="bigbird", seq_len=100, global_width=10, band_width=10, filling_rate=0.2,
                               seed=7)], 16, 16, 2, 2, 16, 11),
    "longformer96_32x16": ([dict(pattern="longformer", seq_len=96, global_width=8, band_width=8)], 32, 16, 2, 2, 16, 11),
    "cfg1_h2_128x16": (CONFIG_MASKS["cfg1"], 128, 16, 1, 2, 64, 1),
    "bigbird300_128x16": ([dict(pattern="bigbird", seq_len=300, global_width=17, band_width=17, filling_rate=0.1,
                                seed=0)], 128, 16, 1, 2, 64, 1),
}


def fp16_round(x):
    return x.astype(np.float16).astype(np.float32)


def main():
    o, r = Oracle(), Reference()
    assert r.available, "build oracle/_ref first (make -C oracle)"
    fp = {}
    plans = {}
    for cfg, terms in CONFIG_MASKS.items():
        m = o.mask(terms) if cfg == "cfg3" else r.mask(terms)
        rp, ci = r.rowwise(m)
        ent = {"terms": terms, "true_count": int(m.sum()), "rowwise_nnz": int(len(ci)),
               "rowwise_fnv": "%016x" % o.fnv1a(rp.tobytes() + ci.tobytes()), "tiles": {}}
        for bm, bn in TILES:
            b, c = r.sfbr(m, bm, bn)
            ent["tiles"][f"{bm}x{bn}"] = {"fnv": "%016x" % o.fnv1a(b), "nbytes": len(b), "full": int(c[0]),
                                          "part": int(c[1]), "empty": int(c[2]), "pool": int(c[3])}
        fp[cfg] = ent
        bs = {"cfg1": 1, "cfg2": 16, "cfg3": 8, "cfg4": 8}[cfg]
        for preset in ("a100", "rtx4090"):
            hw = o.hw_preset(preset)
            p = r.select_plan(m, hw, m.shape[0], 12, bs, 64)
            plans[f"{cfg}/{preset}"] = {"kind": p.kind, "block_m": p.block_m, "block_n": p.block_n,
                                        "num_warps": p.num_warps, "score": p.score, "threshold": p.threshold,
                                        "fallback": p.fallback, "bs": bs}
    (HERE / "fingerprints.json").write_text(json.dumps(fp, indent=1))
    (HERE / "plans.json").write_text(json.dumps(plans, indent=1))

    arrays = {}
    for name, (terms, bm, bn, bs, h, d, seed) in ATTN_CASES.items():
        m = r.mask(terms)
        q, k, v = (fp16_round(x) for x in r.random_attention_input(bs, h, m.shape[0], d, seed))
        out, stats = r.block_sparse_sdpa(q, k, v, m, bm, bn)
        arrays[name + "/out"] = out
        arrays[name + "/stats"] = stats
    np.savez_compressed(HERE / "attn_small.npz", **arrays)

    small = {}
    rng = np.random.default_rng(99)
    for i in range(24):
        n = int(rng.integers(1, 97)); bm = int(rng.integers(1, 25)); bn = int(rng.integers(1, 25))
        m = (rng.random((n, n)) < rng.random()).astype(np.uint8)
        b, _ = r.sfbr(m, bm, bn)
        small[f"{i}/mask"] = np.packbits(m, axis=None, bitorder="little")
        small[f"{i}/shape"] = np.array([n, bm, bn], np.int32)
        small[f"{i}/sfbr"] = np.frombuffer(b, np.uint8)
    np.savez_compressed(HERE / "bsr_small.npz", **small)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
