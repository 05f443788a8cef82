"""Run the bench layer eagerly a few times (for ncu: every launch is a separate kernel, no graph).
usage: python tools/layer_once.py [cfg2] [iters]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2506_06095_b200 import layer, sparsefuse as sf

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
s = layer.LayerShape(cfg["bs"], cfg["seq"], cfg["hidden"], cfg["heads"], cfg["hidden"] // cfg["heads"])
dm = sf.generate_mask(cfg["mask"])
plan = sf.select_plan(dm, sf.hw_preset("b200"), s.seq_len, s.heads, s.bs, s.head_size, mode="b200")
L = layer.EncoderLayer(cfg["model"], s, layer.init_weights(cfg["model"], s, seed=1), sf.context_for(cfg["mask"], dm, plan))
x = (torch.rand(s.rows, s.hidden, device="cuda") * 2 - 1).half()
for _ in range(iters):
    L.forward(x)
torch.cuda.synchronize()
print("ok", plan)
