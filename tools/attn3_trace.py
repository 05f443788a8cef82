"""Trace of the head-group attention kernel (attn_tc3.cu) at cfg2 shapes: per-CTA spans (max /
mean / min, the schedule's imbalance) and CTA 0's per-step timeline (clock64).
Needs the trace build: make -C paper_2506_06095_b200/csrc OUT=$PWD/paper_2506_06095_b200/_lib_trace
EXTRA_NVFLAGS=-DSF_ATTN_TRACE, then SF_B200_LIB=paper_2506_06095_b200/_lib_trace/libsf_b200.so."""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2506_06095_b200.sparsefuse as sf
from paper_2506_06095_b200 import _lib
L = _lib.lib()
L.sf_debug_attn_trace.argtypes = [C.c_void_p]
bs, h, n, d = 16, 12, 1024, 64
q, k, v = (torch.randn(bs, h, n, d, device="cuda").half() for _ in range(3))
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 24
for name, dm in (("bigbird", sf.gen_bigbird(n, 32, 32, 0.1, 0)), ("dense", sf.gen_sliding_window(n, n))):
    b = sf.build_bsr(dm, 128, 16)
    buf = torch.zeros(4096 + 2 * 4096, dtype=torch.int64, device="cuda")
    sf.block_sparse_sdpa(q, k, v, b)
    L.sf_debug_attn_trace(buf.data_ptr())
    sf.block_sparse_sdpa(q, k, v, b)
    torch.cuda.synchronize()
    L.sf_debug_attn_trace(None)
    t = buf.cpu().numpy().astype(np.int64)
    spans = t[4096:4096 + 2 * 148].reshape(-1, 2)
    spans = spans[spans[:, 0] > 0]
    t0 = spans[:, 0].min()
    dur = (spans[:, 1] - spans[:, 0]) / 1e3
    ends = (spans[:, 1] - t0) / 1e3
    print(f"{name}: CTAs {len(spans)}  kernel span {ends.max():.1f} us  CTA busy max {dur.max():.1f} mean {dur.mean():.1f} "
          f"min {dur.min():.1f} us  end times p10 {np.percentile(ends, 10):.1f} p50 {np.percentile(ends, 50):.1f}")
    ev = t[:4096].reshape(-1, 32)
    base = ev[0, 2]
    print("g | MMA S(g) issued, PV(g) issued | K(g) issued, V(g) issued | head0: top Sseen max Parr | head1 ... | head2 ...")
    for g in range(min(steps, 64)):
        r = ev[g] - base
        if ev[g, 4] == 0:
            break
        print(f"{g:2d} | {r[0]:7d} {r[1]:7d} | {r[2]:7d} {r[3]:7d} | " +
              " | ".join(" ".join(f"{r[4 + 4 * hh + e]:7d}" for e in range(4)) for hh in range(3)))
