"""tcgen05 masked MHA at block_m 128 vs 64 (head pairs) at cfg2 shapes: parity against a dense
torch reference on the same fp16 inputs, and device time. usage: python tools/attn_bm.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_06095_b200.sparsefuse as sf
from attn_bn import best_us

torch.manual_seed(0)
for bs, h, n in ((16, 12, 1024), (2, 3, 1000), (1, 1, 300)):
    q, k, v = (torch.randn(bs, h, n, 64, device="cuda").half() for _ in range(3))
    for name, dm in (("dense", sf.gen_sliding_window(n, n)), ("bigbird", sf.gen_bigbird(n, 32, 32, 0.1, 0)),
                     ("sliding32", sf.gen_sliding_window(n, 32))):
        mask = torch.from_numpy(dm.to_numpy()).cuda().bool()
        s = (q.float() @ k.float().transpose(-1, -2)) / 8.0
        s = s.masked_fill(~mask, float("-inf"))
        ref = torch.nan_to_num(torch.softmax(s, -1), nan=0.0) @ v.float()
        for bm in (128, 64):
            b = sf.build_bsr(dm, bm, 16)
            o = sf.block_sparse_sdpa(q, k, v, b)
            err = (o.float() - ref).abs()
            rel = err.sum().item() / ref.abs().sum().item()
            t = best_us(lambda: sf.block_sparse_sdpa(q, k, v, b, out=o)) if bs == 16 else 0.0
            print(f"bs{bs} h{h} n{n} {name:9s} bm {bm:3d}: loads {b.n_load:5d} max_abs {err.max().item():.2e} "
                  f"mean_rel {rel:.2e}  {t:7.1f} us")
