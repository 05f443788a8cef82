"""BigBird(sqrt n, sqrt n, 0.1) at bs16 x 12 heads: the tcgen05 executor at block_m 128 vs 64 (head
pairs), device time (graph of 5, best of 20) and executed cells. usage: python tools/bigbird_bm.py"""
import math
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_06095_b200.sparsefuse as sf
sys.path.insert(0, str(Path(__file__).resolve().parent))
from attn_cfg import best_us

sf.set_attn_impl("tcgen05")
for n in (1024, 2048, 4096, 8192):
    w = int(math.isqrt(n))
    dm = sf.gen_bigbird(n, w, w, 0.1, 0)
    q, k, v = (torch.randn(16, 12, n, 64, device="cuda").half() for _ in range(3))
    res = []
    for bm in (128, 64):
        b = sf.build_bsr(dm, bm, 16)
        t = best_us(lambda: sf.block_sparse_sdpa(q, k, v, b))
        res.append(f"bm{bm}: {t:7.1f} us, {b.n_load * bm * 16 / 1e6:6.2f} M cells/slice")
    print(f"n {n:5d}  " + "  ".join(res), flush=True)
