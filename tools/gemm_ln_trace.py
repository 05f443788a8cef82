"""clock64 timeline of the row-panel LayerNorm GEMM (gemm2_ln.cu), leader CTA of pair 0, first row
block, plus per-CTA spans. Needs the trace build:
make -C paper_2506_06095_b200/csrc OUT=$PWD/paper_2506_06095_b200/_lib_trace EXTRA_NVFLAGS=-DSF_GEMM_TRACE
Events: per sub-tile s: MMA start, MMA committed, epilogue saw tfull, epilogue pass done;
then exchange done, normalise pass done (cycles from kernel entry)."""
import ctypes as C
import os
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
os.environ.setdefault("SF_B200_LIB", str(ROOT / "paper_2506_06095_b200" / "_lib_trace" / "libsf_b200.so"))
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
from paper_2506_06095_b200 import _lib, fused

L = _lib.lib()
L.sf_debug_gemm_trace.argtypes = [C.c_void_p]
M = 16384
for name, N, K in (("out_ln_aux", 768, 768), ("ffn2_ln_aux", 768, 3072)):
    x = torch.randn(M, K, device="cuda").half()
    w = (torch.randn(N, K, device="cuda") * 0.02).half()
    b = torch.randn(N, device="cuda")
    kw = {"ln_gamma": torch.rand(N, device="cuda") + 0.5, "ln_beta": torch.rand(N, device="cuda") - 0.5,
          "aux": torch.randn(M, N, device="cuda").half()}
    out = torch.empty(M, N, device="cuda").half()
    for _ in range(3):
        fused.gemm_fused(x, w, out, bias=b, tile_n=fused.TILE_PAIR, **kw)
    buf = torch.zeros(512 + 8 * 1024, dtype=torch.int64, device="cuda")
    L.sf_debug_gemm_trace(buf.data_ptr())
    fused.gemm_fused(x, w, out, bias=b, tile_n=fused.TILE_PAIR, **kw)
    torch.cuda.synchronize()
    L.sf_debug_gemm_trace(None)
    t = buf.cpu().numpy().astype(np.int64)
    sp = t[512:].reshape(-1, 8)[:, 1:3]
    sp = sp[sp[:, 0] > 0]
    t0s, dur = sp[:, 0].min(), (sp[:, 1] - sp[:, 0]) / 1e3
    print(f"{name}: {len(sp)} CTAs, start spread {(sp[:, 0].max() - t0s) / 1e3:.1f} us, span min/median/max "
          f"{dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us, last end {(sp[:, 1].max() - t0s) / 1e3:.1f} us")
    e0 = t[26]
    for s in range(3):
        print(f"  sub {s}: MMA start {t[8*s]-e0:8d}  committed {t[8*s+1]-e0:8d}  epi saw {t[8*s+2]-e0:8d}  epi done {t[8*s+3]-e0:8d}")
    print(f"  exchange done {t[24]-e0:8d}  normalise done {t[25]-e0:8d}")
