"""block_m 128 vs 64 (head pairs) on the cfg5 sweep masks (bs16 x 12 heads) and the bench configs:
device time (graph of 5, best of 20) and executed cells per slice — the data behind the B200
selector's block_m choice. usage: python tools/bm_sweep.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch
import paper_2506_06095_b200.sparsefuse as sf
from attn_cfg import best_us, SHAPES, TERMS
import bench

sf.set_attn_impl("tcgen05")
cases = [(f"{p} n{n}", 16, n, bench.sweep_terms(p, n)) for n in (1024, 4096) for p in ("sliding", "dilated", "longformer", "bigbird", "causal")]
cases += [(c, SHAPES[c][0], SHAPES[c][1], TERMS[c]) for c in ("cfg2", "cfg3", "cfg4")]
cases += [(f"{p}({w}) n2048", 8, 2048, [dict(pattern=p, seq_len=2048, band_width=w)])
          for p in ("sliding", "causal_local") for w in (1, 4, 16, 32)]
if len(sys.argv) > 1 and sys.argv[1] == "bands":
    cases = cases[-8:]
for name, bs, n, terms in cases:
    dm = sf.generate_mask(terms)
    q, k, v = (torch.randn(bs, 12, n, 64, device="cuda").half() for _ in range(3))
    res = []
    for bm in (128, 64):
        b = sf.build_bsr(dm, bm, 16)
        t = best_us(lambda: sf.block_sparse_sdpa(q, k, v, b))
        res.append((t, b.n_load * bm * 16))
    print(f"{name:16s} bm128 {res[0][0]:8.1f} us {res[0][1] / 1e6:7.2f} Mc | bm64 {res[1][0]:8.1f} us {res[1][1] / 1e6:7.2f} Mc"
          f" | cells64/128 {res[1][1] / res[0][1]:.2f} time64/128 {res[1][0] / res[0][0]:.2f}", flush=True)
