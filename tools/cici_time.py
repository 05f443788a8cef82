"""The BERT FFN (768 -> 3072 -> 768, bias + GELU, then bias + residual + LayerNorm) as the on-chip
CiCi chain (sf_gemm_chain) vs two CiMi launches (sf_gemm_fused x 2, intermediate through memory),
for the short activations the reference forms CiCi segments at (bs*seq <= 4096, search.hpp:228).
Graph of 5 launches, best of 20 (warm L2)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch
from paper_2506_06095_b200 import fused
from attn_cfg import best_us

K1, N1, N2 = 768, 3072, 768
for M in (512, 1024, 2048, 4096, 8192):
    x = (torch.rand(M, K1, device="cuda") * 2 - 1).half()
    w1 = (torch.randn(N1, K1, device="cuda") * 0.02).half()
    w2 = (torch.randn(N2, N1, device="cuda") * 0.02).half()
    b1, b2 = torch.randn(N1, device="cuda"), torch.randn(N2, device="cuda")
    aux = torch.randn(M, N2, device="cuda").half()
    g, be = torch.rand(N2, device="cuda") + 0.5, torch.rand(N2, device="cuda") - 0.5
    h = torch.empty(M, N1, device="cuda").half()
    out = torch.empty(M, N2, device="cuda").half()

    def two():
        fused.gemm_fused(x, w1, h, bias=b1, act="gelu")
        fused.gemm_fused(h, w2, out, bias=b2, aux=aux, ln_gamma=g, ln_beta=be)

    chain = lambda: fused.gemm_chain(x, w1, w2, out, bias1=b1, act="gelu", bias2=b2, aux=aux, ln_gamma=g, ln_beta=be)
    t2, tc = best_us(two), best_us(chain)
    fl = 2 * M * K1 * N1 * 2
    print(f"M {M:5d}: two launches {t2:7.1f} us  chained {tc:7.1f} us  ({fl / tc / 1e6:.0f} TFLOP/s chained)")
