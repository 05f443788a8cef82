"""GEMM / MiChain sweep at the BASELINE layer shapes (device-timed, each launch alone, best of 20).

usage: python tools/gemm_sweep.py [M ...]      (default M = 16384, the cfg2 token count)
Epilogue variants isolate what each fused piece costs: plain, +bias/aux, +LN, +LN with out_pre_ln.
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2506_06095_b200 import fused


def best_us(fn, reps=10, inner=10):
    """Per-launch device time: `inner` launches captured in a CUDA graph (no host launch gaps),
    best replay of `reps`."""
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(inner): fn()
    g.replay(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / inner)
    return best * 1e3


def sweep(M):
    shapes = {
        "qkv": (2304, 768, {}),
        "out_plain": (768, 768, {}),
        "out_aux": (768, 768, {"aux": True}),
        "out_ln": (768, 768, {"ln": True}),
        "out_ln_aux": (768, 768, {"ln": True, "aux": True}),
        "out_ln_aux_pre": (768, 768, {"ln": True, "aux": True, "pre": True}),
        "ffn1_gelu": (3072, 768, {"act": "gelu"}),
        "ffn1_noact": (3072, 768, {}),
        "ffn2_aux": (768, 3072, {"aux": True}),
        "ffn2_ln_aux": (768, 3072, {"ln": True, "aux": True}),
    }
    x = torch.randn(M, 3072, device="cuda").half()
    print(f"--- M={M}")
    for name, (N, K, o) in shapes.items():
        w = torch.randn(N, K, device="cuda").half() * 0.02
        xin = x[:, :K].contiguous()
        out = torch.empty(M, N, device="cuda").half()
        kw = dict(bias=torch.randn(N, device="cuda"))
        if o.get("act"): kw["act"] = o["act"]
        if o.get("aux"): kw["aux"] = torch.randn(M, N, device="cuda").half()
        if o.get("ln"): kw["ln_gamma"] = torch.ones(N, device="cuda"); kw["ln_beta"] = torch.zeros(N, device="cuda")
        if o.get("pre"): kw["out_pre_ln"] = torch.empty(M, N, device="cuda").half()
        for tn in (128, 256, fused.TILE_PAIR):
            try:
                t = best_us(lambda: fused.gemm_fused(xin, w, out, tile_n=tn, **kw))
                print(f"{name:15s} N={N:5d} K={K:5d} tile_n={tn}: {t:7.1f} us  {2*M*N*K/t/1e6:7.1f} TFLOP/s")
            except Exception as e:  # noqa: BLE001 — report and continue the sweep
                print(name, tn, "ERR", e)
    h = torch.randn(M, 768, device="cuda").half()
    o = torch.empty_like(h)
    g, b = torch.ones(768, device="cuda"), torch.zeros(768, device="cuda")
    t = best_us(lambda: fused.mi_chain(h, o, ln_gamma=g, ln_beta=b))
    print(f"mi_chain_ln     N=  768: {t:7.1f} us  {2*h.numel()*2/t/1e3:7.1f} GB/s")


if __name__ == "__main__":
    for m in (sys.argv[1:] or ["16384"]):
        sweep(int(m))
