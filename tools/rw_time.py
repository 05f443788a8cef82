"""Row-wise vs block-wise masked-MHA device time on narrow sliding bands at the cfg3 shapes
(bs8 x 12 heads x n2048 x 64), graph of 5 launches, best of 20. usage: python tools/rw_time.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_06095_b200.sparsefuse as sf
sys.path.insert(0, str(Path(__file__).resolve().parent))
from attn_cfg import best_us

bs, h, n, d = 8, 12, 2048, 64
q, k, v = (torch.randn(bs, h, n, d, device="cuda").half() for _ in range(3))
o = torch.empty_like(q)
hbm = 4 * bs * h * n * d * 2 / 6.5e12 * 1e6
for w in (1, 2, 4, 8, 16, 32, 64):
    dm = sf.gen_sliding_window(n, w)
    rw = sf.build_rowwise(dm)
    b = sf.build_bsr(dm, 128, 16)
    t_rw = best_us(lambda: sf.rowwise_sdpa(q, k, v, rw, out=o))
    t_bw = best_us(lambda: sf.block_sparse_sdpa(q, k, v, b, out=o))
    print(f"band {w:3d}: row-wise {t_rw:7.1f} us  block-wise {t_bw:7.1f} us  (Q,K,V,O at HBM peak {hbm:.1f} us)")

# unstructured masks (gen_random_blocks with block 1: every cell drawn independently) — the case the
# row-wise executor exists for: (128,16) tiles are nearly all loaded but nearly empty
print("random cells (block 1), density p; B200 selector pick in brackets")
for n_ in (2048, 4096):
    qq, kk, vv = (torch.randn(bs, h, n_, d, device="cuda").half() for _ in range(3))
    oo = torch.empty_like(qq)
    for p in (0.002, 0.005, 0.01, 0.02, 0.05):
        dm = sf.gen_random_blocks(n_, 1, p, 7)
        plan = sf.select_plan(dm, sf.hw_preset("b200"), n_, h, bs, d, mode="b200")
        rw = sf.build_rowwise(dm)
        b = sf.build_bsr(dm, 128, 16)
        t_rw = best_us(lambda: sf.rowwise_sdpa(qq, kk, vv, rw, out=oo))
        t_bw = best_us(lambda: sf.block_sparse_sdpa(qq, kk, vv, b, out=oo))
        print(f"n {n_} p {p:.3f}: row-wise {t_rw:7.1f} us  block-wise {t_bw:7.1f} us  [{plan.kind} {plan.block_m}x{plan.block_n}]")
