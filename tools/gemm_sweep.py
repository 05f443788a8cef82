"""GEMM tile sweep at the cfg2 layer shapes (device-timed, each launch alone, best of 20)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2506_06095_b200 import fused

M = 16384
shapes = {"qkv": (2304, 768, {}), "out_ln": (768, 768, {"ln": True, "aux": True}), "ffn1": (3072, 768, {"act": "gelu"}),
          "ffn2_ln": (768, 3072, {"ln": True, "aux": True}), "ffn1_noact": (3072, 768, {})}
x = torch.randn(M, 3072, device="cuda").half()
for name, (N, K, o) in shapes.items():
    w = torch.randn(N, K, device="cuda").half() * 0.02
    xin = x[:, :K].contiguous()
    out = torch.empty(M, N, device="cuda").half()
    kw = dict(bias=torch.randn(N, device="cuda"))
    if o.get("act"): kw["act"] = o["act"]
    if o.get("aux"): kw["aux"] = torch.randn(M, N, device="cuda").half()
    if o.get("ln"): kw["ln_gamma"] = torch.ones(N, device="cuda"); kw["ln_beta"] = torch.zeros(N, device="cuda")
    for tn in (128, 256):
        try:
            for _ in range(3): fused.gemm_fused(xin, w, out, tile_n=tn, **kw)
            best = 1e9
            for _ in range(20):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); fused.gemm_fused(xin, w, out, tile_n=tn, **kw); b.record(); torch.cuda.synchronize()
                best = min(best, a.elapsed_time(b))
            print(f"{name:10s} N={N} K={K} tile_n={tn}: {best*1e3:7.1f} us  {2*M*N*K/best/1e9:7.1f} TFLOP/s")
        except Exception as e:
            print(name, tn, "ERR", e)
