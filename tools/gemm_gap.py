"""Gap between two back-to-back CTA-pair GEMM launches inside one CUDA graph (trace build, see
tools/gemm_trace.py): per-CTA globaltimer spans of launch A and launch B, so the idle time between
A's last CTA and B's first CTA is measured on the device."""
import ctypes as C
import os
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
os.environ.setdefault("SF_B200_LIB", str(ROOT / "paper_2506_06095_b200" / "_lib_trace" / "libsf_b200.so"))
sys.path.insert(0, str(ROOT))
import torch
from paper_2506_06095_b200 import _lib, fused

L = _lib.lib()
L.sf_debug_gemm_trace.argtypes = [C.c_void_p]
M = 16384
ln = lambda N: {"ln_gamma": torch.rand(N, device="cuda") + 0.5, "ln_beta": torch.rand(N, device="cuda") - 0.5}
for name, N, K, kw in (("qkv", 2304, 768, {}), ("out_ln_aux", 768, 768, {**ln(768), "aux": torch.randn(M, 768, device="cuda").half()}),
                       ("ffn2_ln", 768, 3072, ln(768))):
    x = torch.randn(M, K, device="cuda").half()
    w = (torch.randn(N, K, device="cuda") * 0.02).half()
    b = torch.randn(N, device="cuda")
    out = torch.empty(M, N, device="cuda").half()
    bufs = [torch.zeros(512 + 8192, dtype=torch.int64, device="cuda") for _ in range(3)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fused.gemm_fused(x, w, out, bias=b, tile_n=fused.TILE_PAIR, stream=s, **kw)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for bf in bufs:
            L.sf_debug_gemm_trace(bf.data_ptr())
            fused.gemm_fused(x, w, out, bias=b, tile_n=fused.TILE_PAIR, stream=s, **kw)
    L.sf_debug_gemm_trace(None)
    for _ in range(3):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    spans = []
    for bf in bufs:
        sp = bf.cpu().numpy().astype("int64")[512:].reshape(-1, 8)
        spans.append(sp[sp[:, 0] > 0])
    t0 = spans[0][:, 0].min()
    desc = []
    for i, sp in enumerate(spans):
        r = lambda a: (a - t0) / 1e3
        desc.append(f"L{i}: entry {r(sp[:, 0].min()):6.1f}..{r(sp[:, 0].max()):6.1f} pdl {r(sp[:, 1].max()):6.1f} "
                    f"teardown {r(sp[:, 2].min()):6.1f}..{r(sp[:, 2].max()):6.1f} arrived {r(sp[:, 3].max()):6.1f} "
                    f"waited {r(sp[:, 4].min()):6.1f}..{r(sp[:, 4].max()):6.1f}")
    sp = spans[0]
    d = (sp[:, 3] - sp[:, 2]) / 1e3
    order = sorted(range(len(d)), key=lambda i: -d[i])[:12]
    print("   CTA lifetime by clock64 (us at 1.92 GHz) min/median/max:", sp[:, 7].min() / 1920, sorted(sp[:, 7])[len(sp) // 2] / 1920, sp[:, 7].max() / 1920,
          " by globaltimer:", ((sp[:, 4] - sp[:, 0]) / 1e3).min(), ((sp[:, 4] - sp[:, 0]) / 1e3).max())
    print("   arrive cycles thread0 / thread128 (median, max):", sorted(sp[:, 5])[len(sp) // 2], sp[:, 5].max(),
          sorted(sp[:, 6])[len(sp) // 2], sp[:, 6].max())
    print("   slowest arrive - teardown (us) [cta: delta, teardown]:",
          ", ".join(f"{i}: {d[i]:.1f}@{(sp[i, 2] - t0) / 1e3:.1f}" for i in order))
    print(f"{name:10s} graph of 3: {e0.elapsed_time(e1) * 1e3 / 3:.1f} us/launch\n   " + "\n   ".join(desc))
