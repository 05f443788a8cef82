"""One chained CiCi launch (the BERT FFN at cfg1's 512 rows: 768 -> 3072 -> 768, GELU, residual +
LayerNorm) for ncu."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2506_06095_b200 import fused
M, K1, N1, N2 = 512, 768, 3072, 768
x = (torch.rand(M, K1, device="cuda") * 2 - 1).half()
w1 = (torch.randn(N1, K1, device="cuda") * 0.02).half()
w2 = (torch.randn(N2, N1, device="cuda") * 0.02).half()
b1, b2 = torch.randn(N1, device="cuda"), torch.randn(N2, device="cuda")
aux = torch.randn(M, N2, device="cuda").half()
g, be = torch.rand(N2, device="cuda") + 0.5, torch.rand(N2, device="cuda") - 0.5
for _ in range(3):
    fused.gemm_chain(x, w1, w2, bias1=b1, act="gelu", bias2=b2, aux=aux, ln_gamma=g, ln_beta=be)
torch.cuda.synchronize()
print("ok")
