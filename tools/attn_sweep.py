"""Masked-MHA time vs load-list length at bs16 h12 n1024 d64, BSR (128,16): separates the fixed
per-CTA cost (intercept) from the per-step cost (slope)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_06095_b200.sparsefuse as sf

bs, h, n, d = 16, 12, 1024, 64
q, k, v = (torch.randn(bs, h, n, d, device="cuda").half() for _ in range(3))
o = torch.empty_like(q)
for w in (1, 16, 48, 112, 240, 496, 1024):
    dm = sf.gen_sliding_window(n, w)
    b = sf.build_bsr(dm, 128, 16)
    steps = sum(((b.to_host()["load_row_ptr"][i + 1] - b.to_host()["load_row_ptr"][i]) + 3) // 4 for i in range(b.n_rows))
    for _ in range(3): sf.block_sparse_sdpa(q, k, v, b, out=o)
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sf.block_sparse_sdpa(q, k, v, b, out=o); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    ctas = b.n_rows * bs * h
    print(f"band {w:5d}: loads {b.n_load:4d} steps/slice {steps:4d} -> {best*1e3:7.1f} us; per CTA-step {best*1e3*148*2/(steps*bs*h):6.2f} us (2 CTA/SM)")
