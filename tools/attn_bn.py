"""Masked-MHA time for one mask at BSR (128, 16/32/64): separates TMA gather granularity (G boxes
per 64-key step) from the softmax/MMA cost. usage: python tools/attn_bn.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_06095_b200.sparsefuse as sf

def best_us(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for _ in range(5): fn()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 5)
    return best * 1e3



if __name__ == "__main__":
    bs, h, n, d = 16, 12, 1024, 64
    q, k, v = (torch.randn(bs, h, n, d, device="cuda").half() for _ in range(3))
    o = torch.empty_like(q)


    for name, dm in (("dense", sf.gen_sliding_window(n, n)), ("bigbird", sf.gen_bigbird(n, 32, 32, 0.1, 0, 16)),
                     ("sliding32", sf.gen_sliding_window(n, 32))):
        for bn in (16, 32, 64):
            b = sf.build_bsr(dm, 128, bn)
            lrp = b.to_host()["load_row_ptr"]
            steps = sum((lrp[i + 1] - lrp[i] + 64 // bn - 1) // (64 // bn) for i in range(b.n_rows))
            us = best_us(lambda: sf.block_sparse_sdpa(q, k, v, b, out=o))
            print(f"{name:10s} bn {bn:2d}: loads {b.n_load:4d} steps/slice {steps:4d} -> {us:7.1f} us; "
                  f"{us * 1e3 / (steps * bs * h / 148):7.0f} ns per step per SM")
