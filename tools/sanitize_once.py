"""Small multi-item launches of the tcgen05 attention (both schedules, and the head-group kernel),
the CTA-pair GEMM, the row-panel LayerNorm GEMM and the chained CiCi kernel for compute-sanitizer
(racecheck / synccheck / memcheck). The attention grid is capped at 8
CTAs (SF_ATTN_MAX_CTAS) so every CTA walks ~24 items: Q double-buffering, the item ring, the
O-barrier phases across items and the counter reset all run. Checks the results too.
usage: compute-sanitizer --tool racecheck python tools/sanitize_once.py"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2506_06095_b200.sparsefuse as sf
from paper_2506_06095_b200 import fused
from oracle.oracle import Oracle

os.environ["SF_ATTN_MAX_CTAS"] = "8"
o = Oracle()
bs, h, n, d = 4, 12, 512, 64
terms = [dict(pattern="bigbird", seq_len=n, global_width=22, band_width=22, filling_rate=0.1, seed=0)]
m = o.mask(terms)
q, k, v = (x.astype(np.float16).astype(np.float32) for x in o.random_attention_input(bs, h, n, d, 1))
ref, _ = o.block_sparse_sdpa(q, k, v, m, 128, 16, threads=8)
Q, K, V = (torch.from_numpy(x).cuda().half() for x in (q, k, v))
b = sf.build_bsr(sf.generate_mask(terms), 128, 16)
sf.set_attn_impl("tcgen05")
for static in ("0", "1"):
    os.environ["SF_ATTN_STATIC"] = static
    for _ in range(2):
        out = sf.block_sparse_sdpa(Q, K, V, b)
        torch.cuda.synchronize()
        err = np.abs(out.float().cpu().numpy() - ref).max()
        assert err < 2e-2, err
        print(f"attn static={static} max_abs {err:.2e}")
os.environ["SF_ATTN_STATIC"] = "0"
os.environ["SF_ATTN_HEADGROUP"] = "1"  # attn_tc3.cu: three heads per item, ~16 items per CTA here
for _ in range(2):
    out = sf.block_sparse_sdpa(Q, K, V, b)
    torch.cuda.synchronize()
    err = np.abs(out.float().cpu().numpy() - ref).max()
    assert err < 2e-2, err
    print(f"attn head groups max_abs {err:.2e}")
os.environ["SF_ATTN_HEADGROUP"] = "0"
# head pairs (block_m 64) with the two-head 5-D K/V boxes: ~24 items per CTA here too
ref64, _ = o.block_sparse_sdpa(q, k, v, m, 64, 16, threads=8)
b64 = sf.build_bsr(sf.generate_mask(terms), 64, 16)
for _ in range(2):
    out = sf.block_sparse_sdpa(Q, K, V, b64)
    torch.cuda.synchronize()
    err = np.abs(out.float().cpu().numpy() - ref64).max()
    assert err < 2e-2, err
    print(f"attn head pairs max_abs {err:.2e}")
x = torch.randn(512, 768, device="cuda").half()
w = torch.randn(768, 768, device="cuda").half() * 0.03
y = fused.gemm_fused(x, w, tile_n=1)
err = (y.float() - x.float() @ w.float().t()).abs().max().item()
print(f"gemm pair max_abs {err:.2e}")
assert err < 2e-2
# row-panel LayerNorm GEMM (gemm2_ln.cu): 512 rows = two panels, N 768 = three sub-tiles
os.environ["SF_GEMM_LN_PANEL"] = "1"
g, be = torch.rand(768, device="cuda") + 0.5, torch.rand(768, device="cuda") - 0.5
aux = torch.randn(512, 768, device="cuda").half()
pre = torch.empty(512, 768, device="cuda").half()
y = fused.gemm_fused(x, w, aux=aux, ln_gamma=g, ln_beta=be, out_pre_ln=pre, tile_n=1)
r = x.float() @ w.float().t() + aux.float()
r = (r - r.mean(1, keepdim=True)) / torch.sqrt(r.var(1, unbiased=False, keepdim=True) + 1e-5) * g + be
err = (y.float() - r).abs().max().item()
print(f"gemm row-panel LN max_abs {err:.2e}")
assert err < 5e-2
# chained CiCi (cici.cu): 256 rows, 768 -> 1024 -> 768, GELU, LayerNorm
w1 = torch.randn(1024, 768, device="cuda").half() * 0.03
w2 = torch.randn(768, 1024, device="cuda").half() * 0.03
xc = x[:256].contiguous()
y = fused.gemm_chain(xc, w1, w2, act="gelu", aux=aux[:256].contiguous(), ln_gamma=g, ln_beta=be)
hmid = torch.nn.functional.gelu(xc.float() @ w1.float().t()).half().float()
r = hmid @ w2.float().t() + aux[:256].float()
r = (r - r.mean(1, keepdim=True)) / torch.sqrt(r.var(1, unbiased=False, keepdim=True) + 1e-5) * g + be
err = (y.float() - r).abs().max().item()
print(f"gemm chain max_abs {err:.2e}")
assert err < 5e-2
# decomposed strided executor (strided.cu): band part on tcgen05 with LSE, class part on mma.sync, merge
ts = [dict(pattern="strided", seq_len=2048, band_width=32)]
ms = o.mask(ts)
qs, ks, vs = (x.astype(np.float16).astype(np.float32) for x in o.random_attention_input(1, 2, 2048, d, 2))
refs, _ = o.block_sparse_sdpa(qs, ks, vs, ms, 128, 16, threads=8)
Qs, Ks, Vs = (torch.from_numpy(x).cuda().half() for x in (qs, ks, vs))
w_band = sf.strided_band(ts)
assert w_band == 32, w_band
bb = sf.build_bsr(sf.generate_mask([dict(pattern="causal_local", seq_len=2048, band_width=32)]), 128, 16)
out = sf.strided_sdpa(Qs, Ks, Vs, 32, bb)
torch.cuda.synchronize()
err = np.abs(out.float().cpu().numpy() - refs).max()
print(f"strided max_abs {err:.2e}")
assert err < 2e-2
# dilated class decomposition with a rest (dilated(16,1) + global(16), n 1024): classes, rest, merge
td = [dict(pattern="dilated", seq_len=1024, band_width=16, dilation_rate=1), dict(pattern="global", seq_len=1024, global_width=16)]
qd, kd, vd = (x.astype(np.float16).astype(np.float32) for x in o.random_attention_input(1, 2, 1024, d, 4))
refd, _ = o.block_sparse_sdpa(qd, kd, vd, o.mask(td), 128, 16, threads=8)
ctxd = sf.MhaContext(sf.generate_mask(td), sf.KernelPlan("block_wise", 128, 16), dilated=sf.dilated_split(td, 0, True))
out = sf.mha(*(torch.from_numpy(x).cuda().half() for x in (qd, kd, vd)), ctxd)
torch.cuda.synchronize()
err = np.abs(out.float().cpu().numpy() - refd).max()
print(f"dilated max_abs {err:.2e}")
assert err < 2e-2
print("sanitize_once ok")
