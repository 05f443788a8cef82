"""One row-wise masked-MHA launch (bs16 h12 d64) for ncu: sliding band (default 16) at n = 2048 — the
cfg3-sweep case Eq. 1 routes row-wise. usage: python tools/rw_once.py [band] [n]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_06095_b200.sparsefuse as sf

w = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
bs, h, d = 16, 12, 64
q, k, v = (torch.randn(bs, h, n, d, device="cuda").half() for _ in range(3))
rw = sf.build_rowwise(sf.gen_sliding_window(n, w))
for _ in range(2):
    sf.rowwise_sdpa(q, k, v, rw)
torch.cuda.synchronize()
print("ok", w, n, rw.nnz)
