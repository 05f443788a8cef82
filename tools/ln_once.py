import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2506_06095_b200 import fused
M, N, K = 16384, 768, 768
x = torch.randn(M, K, device="cuda").half(); w = (torch.randn(N, K, device="cuda") * 0.02).half()
b = torch.randn(N, device="cuda")
kw = {"ln_gamma": torch.rand(N, device="cuda") + 0.5, "ln_beta": torch.rand(N, device="cuda") - 0.5, "aux": torch.randn(M, N, device="cuda").half()}
out = torch.empty(M, N, device="cuda").half()
for _ in range(8):
    fused.gemm_fused(x, w, out, bias=b, tile_n=fused.TILE_PAIR, **kw)
torch.cuda.synchronize()
