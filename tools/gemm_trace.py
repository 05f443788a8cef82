"""clock64 timeline of CTA pair 0 of the CTA-pair GEMM (needs the trace build:
make -C paper_2506_06095_b200/csrc OUT=$PWD/paper_2506_06095_b200/_lib_trace EXTRA_NVFLAGS=-DSF_GEMM_TRACE).
Events per tile: 0 producer first k-block, 1 MMA got accumulator, 2 MMA first stage full,
3 MMA committed tile, 4 epilogue saw tfull, 5 epilogue released TMEM, 6 epilogue stores issued
(LN: 6 = row-statistics exchange complete, 7 = own partials sent)."""
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
for name, N, K, kw in (("qkv", 2304, 768, {}), ("ffn1_gelu", 3072, 768, {"act": "gelu"}),
                       ("ffn2", 768, 3072, {}), ("out_ln", 768, 768, ln(768)), ("out_ln_aux", 768, 768, {**ln(768), "aux": torch.randn(M, 768, device="cuda").half()}), ("ffn2_ln", 768, 3072, ln(768))):
    x = torch.randn(M, K, device="cuda").half()
    w = (torch.randn(N, K, device="cuda") * 0.02).half()
    b = torch.randn(N, device="cuda")
    out = torch.empty(M, N, device="cuda").half()
    for _ in range(3):
        fused.gemm_fused(x, w, out, bias=b, tile_n=fused.TILE_PAIR, **kw)
    buf = torch.zeros(64 * 8 + 8 * 1024, dtype=torch.int64, device="cuda")
    L.sf_debug_gemm_trace(buf.data_ptr())
    fused.gemm_fused(x, w, out, bias=b, tile_n=fused.TILE_PAIR, **kw)
    torch.cuda.synchronize()
    L.sf_debug_gemm_trace(None)
    allb = buf.cpu().numpy().astype("int64")
    sp = allb[512:].reshape(-1, 8)[:, 1:3]
    sp = sp[sp[:, 0] > 0]
    if len(sp):
        t0s, dur = sp[:, 0].min(), (sp[:, 1] - sp[:, 0]) / 1e3
        print(f"{name}: {len(sp)} CTAs, start spread {(sp[:, 0].max() - t0s) / 1e3:.1f} us, "
              f"span min/median/max {dur.min():.1f}/{sorted(dur)[len(dur) // 2]:.1f}/{dur.max():.1f} us, "
              f"last end {(sp[:, 1].max() - t0s) / 1e3:.1f} us")
    t = allb[:512].reshape(64, 8)
    t0 = t[0, 0]
    print(f"{name}: M={M} N={N} K={K}  (cycles from tile 0 producer start)")
    prev = None
    for i in range(64):
        if t[i, 1] == 0:
            break
        r = t[i] - t0
        mma = r[3] - r[2]
        epi = r[6] - r[4]
        print(f"tile {i:2d}: prod {r[0]:7d} mma_acc {r[1]:7d} first_full {r[2]:7d} commit {r[3]:7d} | "
              f"epi_in {r[4]:7d} rel {r[5]:7d} done {r[6]:7d} ln_part {r[7]:7d} | mma {mma:6d} epi {epi:6d}"
              + (f" gap {r[2] - prev:6d}" if prev is not None else ""))
        prev = r[3]
