"""Dilated masks: block executor over the whole mask vs the class decomposition (sf_mha_dilated),
parity of both against the dense torch reference, and device time (graph of 5, best of 20).
Shapes: the cfg5 sweep's dilated(sqrt n, 1) at bs16 x 12 heads, and T5 cfg4's dilated(64,1) + global(64)
at bs8 x 12 x 4096. usage: python tools/dilated_time.py"""
import math
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_06095_b200.sparsefuse as sf
from attn_cfg import best_us

torch.manual_seed(0)
sf.set_attn_impl("tcgen05")
cases = [(f"sweep dilated n{n}", 16, n, [dict(pattern="dilated", seq_len=n, band_width=int(math.isqrt(n)), dilation_rate=1)])
         for n in (512, 1024, 2048, 4096, 8192)]
cases.append(("cfg4 dilated(64,1)+global(64)", 8, 4096,
              [dict(pattern="dilated", seq_len=4096, band_width=64, dilation_rate=1),
               dict(pattern="global", seq_len=4096, global_width=64)]))
for name, bs, n, terms in cases:
    h = 12
    q, k, v = (torch.randn(bs, h, n, 64, device="cuda").half() for _ in range(3))
    dm = sf.generate_mask(terms)
    bsr = sf.build_bsr(dm, 128, 16)
    split = sf.dilated_split(terms, min_seq_len=0, allow_rest=True)
    ctx = sf.MhaContext(dm, sf.KernelPlan("block_wise", 128, 16), dilated=split)
    o_bw = sf.block_sparse_sdpa(q, k, v, bsr)
    o_dec = sf.mha(q, k, v, ctx)
    # parity on two slices against a dense fp32 reference
    mask = torch.from_numpy(dm.to_numpy()).cuda().bool()
    err = 0.0
    for b, hh in ((0, 0), (bs - 1, h - 1)):
        s = (q[b, hh].float() @ k[b, hh].float().t()) / 8.0
        s = s.masked_fill(~mask, float("-inf"))
        ref = torch.nan_to_num(torch.softmax(s, -1), nan=0.0) @ v[b, hh].float()
        err = max(err, (o_dec[b, hh].float() - ref).abs().max().item(), (o_bw[b, hh].float() - ref).abs().max().item())
    t_bw = best_us(lambda: sf.block_sparse_sdpa(q, k, v, bsr))
    t_dec = best_us(lambda: sf.mha(q, k, v, ctx))
    print(f"{name:32s} block-wise {t_bw:7.1f} us  decomposed {t_dec:7.1f} us  max_abs {err:.2e}", flush=True)
