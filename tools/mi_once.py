"""One MiChain launch at the cfg2/cfg3 shapes for ncu: x (16384 x 768 fp16) -> LayerNorm (the GPT /
T5 pre-norm LN1), and bias + residual + LayerNorm (the ln_split out-projection tail).
usage: python tools/mi_once.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2506_06095_b200 import fused

M, N = 16384, 768
x = torch.randn(M, N, device="cuda").half()
aux = torch.randn(M, N, device="cuda").half()
out = torch.empty_like(x)
g, b, bias = torch.rand(N, device="cuda") + 0.5, torch.rand(N, device="cuda") - 0.5, torch.rand(N, device="cuda")
for _ in range(2):
    fused.mi_chain(x, out, ln_gamma=g, ln_beta=b)
    fused.mi_chain(x, out, bias=bias, aux=aux, ln_gamma=g, ln_beta=b)
torch.cuda.synchronize()
print("ok")
