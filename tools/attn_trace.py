"""clock64 trace of CTA 0's first work item of the tcgen05 attention (cfg2 shapes).
Needs the trace build: make -C paper_2506_06095_b200/csrc OUT=$PWD/paper_2506_06095_b200/_lib_trace
EXTRA_NVFLAGS=-DSF_ATTN_TRACE, then SF_B200_LIB=paper_2506_06095_b200/_lib_trace/libsf_b200.so."""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2506_06095_b200.sparsefuse as sf
from paper_2506_06095_b200 import _lib
L = _lib.lib()
L.sf_debug_attn_trace.argtypes = [C.c_void_p]
bs, h, n, d = 16, 12, 1024, 64
q, k, v = (torch.randn(bs, h, n, d, device="cuda").half() for _ in range(3))
for name, dm, bn in (("dense", sf.gen_sliding_window(n, n), 16), ("dense", sf.gen_sliding_window(n, n), 64),
                     ("bigbird", sf.gen_bigbird(n, 32, 32, 0.1, 0), 16)):
    b = sf.build_bsr(dm, 128, bn)
    buf = torch.zeros(64 * 32, dtype=torch.int64, device="cuda")
    sf.block_sparse_sdpa(q, k, v, b)
    L.sf_debug_attn_trace(buf.data_ptr())
    sf.block_sparse_sdpa(q, k, v, b)
    torch.cuda.synchronize()
    L.sf_debug_attn_trace(None)
    t = buf.view(64, 32).cpu().numpy().astype('int64')
    t0 = t[0, 0]
    print(name, bn, "softmax: 0 top,1 kv_full,2 s_full,3 max,6 P arrived | MMA: 8 P seen,9 PV issued,13 S(j) kv wait, 14 kv ready, 10 S(j+2) issued | producer: 4 K wait, 5 K slot free, 7 V wait, 11 V slot free")
    for j in range(16):
        if t[j, 0] == 0: break
        r = t[j] - t0
        print(f"j={j:2d} " + " ".join(f"{e}:{r[e]:7d}" for e in (4, 5, 7, 11, 0, 1, 2, 3, 6, 8, 9, 13, 14, 10)))
    print("per softmax warp (lane 0), by CTA step g (across items): top / S seen / max done / P arrived, warps 2..5 (SMSP 2,3,0,1) | MMA P seen, PV issued, S(g+2) issued")
    for j in range(64):
        if t[j, 16] == 0: break
        r = t[j] - t0
        print(f"g={j:2d} " + " | ".join(" ".join(f"{r[16 + 4 * w + e]:7d}" for e in range(4)) for w in range(4))
              + f" | {r[8]:7d} {r[9]:7d} {r[10]:7d}")
