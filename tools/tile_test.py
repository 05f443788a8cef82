import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd() + "/tools")
import torch
import paper_2506_06095_b200.sparsefuse as sf
from attn_cfg import best_us, SHAPES, TERMS
sf.set_attn_impl("tcgen05")
for cfg in ("cfg2", "cfg4"):
    bs, n = SHAPES[cfg]
    dm = sf.generate_mask(TERMS[cfg])
    q, k, v = (torch.randn(bs, 12, n, 64, device="cuda").half() for _ in range(3))
    for bm, bn in ((64, 16), (64, 32), (64, 64), (128, 16), (128, 32)):
        b = sf.build_bsr(dm, bm, bn)
        t = best_us(lambda: sf.block_sparse_sdpa(q, k, v, b))
        print(f"{cfg} ({bm},{bn}): {t:.1f} us  cells {b.n_load * bm * bn / 1e6:.2f} M/slice", flush=True)
