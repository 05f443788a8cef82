import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd() + "/tools")
import torch
from paper_2506_06095_b200 import fused
from gemm_sweep import best_us
M = 16384
for name, N, K in (("qkv", 2304, 768), ("ffn1", 3072, 768), ("ffn2", 768, 3072)):
    x = torch.randn(M, K, device="cuda").half(); w = (torch.randn(N, K, device="cuda") * 0.02).half()
    b = torch.randn(N, device="cuda"); out = torch.empty(M, N, device="cuda").half()
    t = best_us(lambda: fused.gemm_fused(x, w, out, bias=b, tile_n=fused.TILE_PAIR))
    print(f"{name}: {t:.1f} us  ({2*M*N*K/t/1e6:.0f} TFLOP/s)", flush=True)
