"""One row-wise masked-MHA launch on an unstructured mask (independent cells, density p) at the cfg3
shapes (bs8 x 12 heads x n2048 x 64) for ncu. usage: python tools/rw_once_random.py [p]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_06095_b200.sparsefuse as sf

p = float(sys.argv[1]) if len(sys.argv) > 1 else 0.005
bs, h, n, d = 8, 12, 2048, 64
q, k, v = (torch.randn(bs, h, n, d, device="cuda").half() for _ in range(3))
rw = sf.build_rowwise(sf.gen_random_blocks(n, 1, p, 7))
for _ in range(2):
    sf.rowwise_sdpa(q, k, v, rw)
torch.cuda.synchronize()
print("ok", p, rw.nnz)
