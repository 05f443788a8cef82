"""MiChain (sf_mi_chain) device time at the layer shapes, graph-timed (no host launch gaps)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2506_06095_b200 import fused
from gemm_sweep import best_us

for M in (16384, 32768):
    for N, kind in ((768, "ln"), (768, "bias_aux_ln"), (3072, "bias_gelu")):
        x = torch.randn(M, N, device="cuda").half()
        o = torch.empty_like(x)
        kw = {}
        nbytes = 2 * x.numel() * 2
        if "bias" in kind: kw["bias"] = torch.randn(N, device="cuda")
        if "gelu" in kind: kw["act"] = "gelu"
        if "aux" in kind: kw["aux"] = torch.randn(M, N, device="cuda").half(); nbytes += x.numel() * 2
        if "ln" in kind: kw["ln_gamma"] = torch.ones(N, device="cuda"); kw["ln_beta"] = torch.zeros(N, device="cuda")
        t = best_us(lambda: fused.mi_chain(x, o, **kw))
        print(f"M={M:6d} N={N:5d} {kind:12s}: {t:7.1f} us  {nbytes / t / 1e3:7.1f} GB/s")
