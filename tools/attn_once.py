"""One masked-MHA launch per mask at cfg2 shapes (bs16 h12 n1024 d64) for ncu.
usage: python tools/attn_once.py [bigbird|dense|causal] [block_n] [block_m]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_06095_b200.sparsefuse as sf

name = sys.argv[1] if len(sys.argv) > 1 else "bigbird"
bn = int(sys.argv[2]) if len(sys.argv) > 2 else 16
bm = int(sys.argv[3]) if len(sys.argv) > 3 else 128
bs, h, n, d = 16, 12, 1024, 64
q, k, v = (torch.randn(bs, h, n, d, device="cuda").half() for _ in range(3))
dm = {"bigbird": lambda: sf.gen_bigbird(n, 32, 32, 0.1, 0), "dense": lambda: sf.gen_sliding_window(n, n),
      "causal": lambda: sf.generate_mask([dict(pattern="causal", seq_len=n)])}[name]()
b = sf.build_bsr(dm, bm, bn)
for _ in range(2):
    sf.block_sparse_sdpa(q, k, v, b)
torch.cuda.synchronize()
print("ok", name, bn, bm)
