"""Masked-MHA time at cfg2 shapes for contiguous (b,h,n,d) Q/K/V vs the layer's in-place views of the
fused (bs*n, 3*H) QKV activation. usage: python tools/attn_layout.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_06095_b200.sparsefuse as sf
from attn_bn import best_us

bs, h, n, d = 16, 12, 1024, 64
H = h * d
dm = sf.gen_bigbird(n, 32, 32, 0.1, 0)
b = sf.build_bsr(dm, 128, 16)
qkv = torch.randn(bs * n, 3 * H, device="cuda").half()
heads = lambda t, c0: t[:, c0:c0 + H].view(bs, n, h, d).permute(0, 2, 1, 3)
qs, ks, vs = heads(qkv, 0), heads(qkv, H), heads(qkv, 2 * H)
attn = torch.empty(bs * n, H, device="cuda").half()
os_ = heads(attn, 0)
qc, kc, vc = (x.contiguous() for x in (qs, ks, vs))
oc = torch.empty_like(qc)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, args in (("contiguous", (qc, kc, vc, oc)), ("fused-qkv views", (qs, ks, vs, os_))):
    q, k, v, o = args
    t = best_us(lambda: sf.block_sparse_sdpa(q, k, v, b, out=o))
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sf.block_sparse_sdpa(q, k, v, b, out=o); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{name:16s}: {t:6.1f} us (graph, warm L2)   {sorted(ts)[len(ts)//2]:6.1f} us (single launch, L2 flushed)")

# the layer's order: L2 flushed, then the QKV GEMM writes qkv, then the attention reads it
from paper_2506_06095_b200 import fused
x = torch.randn(bs * n, H, device="cuda").half()
wqkv = (torch.randn(3 * H, H, device="cuda") * 0.02).half()
bqkv = torch.randn(3 * H, device="cuda")
ts = []
for _ in range(20):
    flush.zero_()
    fused.gemm_fused(x, wqkv, qkv, bias=bqkv)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sf.block_sparse_sdpa(qs, ks, vs, b, out=os_); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"{'after QKV GEMM':16s}: {sorted(ts)[len(ts)//2]:6.1f} us (single launch, L2 flushed before the GEMM)")
