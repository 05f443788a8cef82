"""One decomposed strided launch (cfg3 shapes: bs8 x 12 heads x n2048, w 45) for ncu."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_06095_b200.sparsefuse as sf
bs, h, n, d, w = 8, 12, 2048, 64, 45
q, k, v = (torch.randn(bs, h, n, d, device="cuda").half() for _ in range(3))
band = sf.generate_mask([dict(pattern="causal_local", seq_len=n, band_width=w)])
bb = sf.build_bsr(band, 128, 16)
for _ in range(3):
    sf.strided_sdpa(q, k, v, w, bb)
torch.cuda.synchronize()
print("ok")
