"""Masked-MHA device time at a BASELINE config's shapes and mask, at the B200 plan's tile
(graph of 5 launches, best of 20). usage: python tools/attn_cfg.py [cfg2|cfg3|cfg4 ...]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_06095_b200.sparsefuse as sf


def best_us(fn, reps=20):
    """Graph of 5 launches on a side stream, best replay of `reps` (the stream runs the launch once
    before capture, so a dynamic-schedule work counter exists for it)."""
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
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 5)
    return best * 1e3

SHAPES = {"cfg2": (16, 1024), "cfg3": (8, 2048), "cfg4": (8, 4096), "dense": (16, 1024)}
TERMS = {"cfg2": [dict(pattern="bigbird", seq_len=1024, global_width=32, band_width=32, filling_rate=0.10, seed=0, block=16)],
         "cfg3": [dict(pattern="strided", seq_len=2048, band_width=45)],
         "cfg4": [dict(pattern="dilated", seq_len=4096, band_width=64, dilation_rate=1),
                  dict(pattern="global", seq_len=4096, global_width=64)],
         "dense": [dict(pattern="sliding", seq_len=1024, band_width=1024)]}
if __name__ == "__main__":
    for cfg in sys.argv[1:] or ["cfg2", "cfg3", "cfg4"]:
        bs, n = SHAPES[cfg]
        h, d = 12, 64
        dm = sf.generate_mask(TERMS[cfg])
        plan = sf.select_plan(dm, sf.hw_preset("b200"), n, h, bs, d, mode="b200")
        b = sf.build_bsr(dm, plan.block_m, plan.block_n)
        q, k, v = (torch.randn(bs, h, n, d, device="cuda").half() for _ in range(3))
        o = torch.empty_like(q)
        us = best_us(lambda: sf.block_sparse_sdpa(q, k, v, b, out=o))
        print(f"{cfg}: plan ({plan.block_m},{plan.block_n}) loads {b.n_load} -> {us:.1f} us")
