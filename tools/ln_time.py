"""Device time of the LayerNorm GEMMs at cfg2 shapes (M 16384, N 768, K 768 / 3072, bias + residual
+ LN), row-panel (gemm2_ln.cu) vs cluster (gemm2_tc.cu, SF_GEMM_LN_CLUSTER=1) form: warm (graph of
5 back-to-back launches) and cold (256 MB L2 flush, then one launch between events)."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2506_06095_b200 import fused

M = 16384
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, N, K in (("out_ln_aux", 768, 768), ("ffn2_ln_aux", 768, 3072)):
    x = torch.randn(M, K, device="cuda").half()
    w = (torch.randn(N, K, device="cuda") * 0.02).half()
    b = torch.randn(N, device="cuda")
    kw = {"ln_gamma": torch.rand(N, device="cuda") + 0.5, "ln_beta": torch.rand(N, device="cuda") - 0.5,
          "aux": torch.randn(M, N, device="cuda").half()}
    out = torch.empty(M, N, device="cuda").half()
    for form in ("panel", "cluster"):
        os.environ["SF_GEMM_LN_CLUSTER"] = "1" if form == "cluster" else "0"
        fn = lambda: fused.gemm_fused(x, w, out, bias=b, tile_n=fused.TILE_PAIR, **kw)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(5):
                fn()
        warm = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            warm = min(warm, e0.elapsed_time(e1) / 5 * 1e3)
        cold = []
        for _ in range(10):
            flush.fill_(1); flush.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            cold.append(e0.elapsed_time(e1) * 1e3)
        cold.sort()
        print(f"{name:12s} {form:8s} warm {warm:7.1f} us  cold median {cold[5]:7.1f} us")
