"""Debug aid: per-case max error of the tcgen05 attention on the golden cases."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2506_06095_b200.sparsefuse as sf
from oracle.oracle import Oracle
from tests.golden.make_golden import ATTN_CASES
o = Oracle()
z = np.load(Path(__file__).resolve().parents[1] / "tests/golden/attn_small.npz")
for name, (terms, bm, bn, bs, h, d, seed) in ATTN_CASES.items():
    dm = sf.generate_mask(terms)
    q, k, v = [x.astype(np.float16).astype(np.float32) for x in o.random_attention_input(bs, h, dm.seq_len, d, seed)]
    b = sf.build_bsr(dm, bm, bn)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.float16)
    out = sf.block_sparse_sdpa(dev(q), dev(k), dev(v), b).float().cpu().numpy()
    ref = z[name + "/out"]
    dd = np.abs(out - ref)
    bad = np.argwhere(dd > 2e-2)
    print(name, bm, bn, bs, h, dm.seq_len, "max", dd.max(), "nbad", len(bad), "rows", sorted(set(bad[:, 2].tolist()))[:20] if len(bad) else "")
