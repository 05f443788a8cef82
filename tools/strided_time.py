"""Strided masks: the decomposed executor (sf_mha_strided: causal-local band on tcgen05 + per-class
causal attention) vs the block-wise BSR executor on the whole strided mask, bs x 12 heads x 64,
graph of 5 launches, best of 20. usage: python tools/strided_time.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import math
import torch
import paper_2506_06095_b200.sparsefuse as sf
from attn_cfg import best_us

for bs, n, w in ((8, 2048, 45), (16, 1024, 32), (16, 2048, 45), (16, 4096, 64), (16, 8192, 90)):
    h, d = 12, 64
    q, k, v = (torch.randn(bs, h, n, d, device="cuda").half() for _ in range(3))
    o = torch.empty_like(q)
    dm = sf.generate_mask([dict(pattern="strided", seq_len=n, band_width=w)])
    b = sf.build_bsr(dm, 128, 16)
    band = sf.generate_mask([dict(pattern="causal_local", seq_len=n, band_width=w)])
    bb = sf.build_bsr(band, 128, 16)
    bb64 = sf.build_bsr(band, 64, 16)  # the band part on head pairs
    t_bw = best_us(lambda: sf.block_sparse_sdpa(q, k, v, b, out=o))
    t_dec = best_us(lambda: sf.strided_sdpa(q, k, v, w, bb, out=o))
    t_dec64 = best_us(lambda: sf.strided_sdpa(q, k, v, w, bb64, out=o))
    t_band = best_us(lambda: sf.block_sparse_sdpa(q, k, v, bb, out=o))
    t_band64 = best_us(lambda: sf.block_sparse_sdpa(q, k, v, bb64, out=o))
    print(f"bs{bs} n{n} w{w}: block-wise {t_bw:8.1f} us  decomposed {t_dec:8.1f} us / band on head pairs {t_dec64:8.1f} us"
          f" (band part alone {t_band:6.1f} / {t_band64:6.1f} us)  x{t_bw / t_dec:.2f}", flush=True)
