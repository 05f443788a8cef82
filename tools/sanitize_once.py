"""Small multi-item launches of the tcgen05 attention (both schedules) and the CTA-pair GEMM
for compute-sanitizer (racecheck / synccheck / memcheck). The attention grid is capped at 8
CTAs (SF_ATTN_MAX_CTAS) so every CTA walks ~24 items: Q double-buffering, the item ring, the
O-barrier phases across items and the counter reset all run. Checks the results too.
usage: compute-sanitizer --tool racecheck python tools/sanitize_once.py"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2506_06095_b200.sparsefuse as sf
from paper_2506_06095_b200 import fused
from oracle.oracle import Oracle

os.environ["SF_ATTN_MAX_CTAS"] = "8"
o = Oracle()
bs, h, n, d = 4, 12, 512, 64
terms = [dict(pattern="bigbird", seq_len=n, global_width=22, band_width=22, filling_rate=0.1, seed=0)]
m = o.mask(terms)
q, k, v = (x.astype(np.float16).astype(np.float32) for x in o.random_attention_input(bs, h, n, d, 1))
ref, _ = o.block_sparse_sdpa(q, k, v, m, 128, 16, threads=8)
Q, K, V = (torch.from_numpy(x).cuda().half() for x in (q, k, v))
b = sf.build_bsr(sf.generate_mask(terms), 128, 16)
sf.set_attn_impl("tcgen05")
for static in ("0", "1"):
    os.environ["SF_ATTN_STATIC"] = static
    for _ in range(2):
        out = sf.block_sparse_sdpa(Q, K, V, b)
        torch.cuda.synchronize()
        err = np.abs(out.float().cpu().numpy() - ref).max()
        assert err < 2e-2, err
        print(f"attn static={static} max_abs {err:.2e}")
x = torch.randn(512, 768, device="cuda").half()
w = torch.randn(768, 768, device="cuda").half() * 0.03
y = fused.gemm_fused(x, w, tile_n=1)
err = (y.float() - x.float() @ w.float().t()).abs().max().item()
print(f"gemm pair max_abs {err:.2e}")
assert err < 2e-2
print("sanitize_once ok")
