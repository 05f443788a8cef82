#!/usr/bin/env python
"""Benchmark of the STOF hot path on B200.

Default workload = BASELINE.json configs[1]: one BERT-base encoder layer (masked MHA + fused
FFN/LayerNorm), batch 16, seq 1024, 12 heads x 64, BigBird(global 32, band 32, random 10% of
16x16 tiles, seed 0) mask. A step = one layer forward over the batch; metric = tokens/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU: the configured batch is sharded over the ranks
(dist.shard_range over its sequences; every rank holds the full weights and rebuilds the formats
from the mask descriptor), so the total work is fixed (strong scaling) and the attention path has
no exchange; timing is the max over ranks of device (CUDA-event) time. The e2e leg gathers the
layer outputs to every rank with one NCCL all-gather per step (rank 0 reads the full output
back), the only collective on the data path (north_star).
`--impl reference` times the reference's own CPU implementation (oracle/_ref: the unmodified
reference headers compiled in place; CpuBackend::run_chain of the same chain) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "cfg1": dict(model="bert-layer", bs=1, seq=512, hidden=768, heads=12,
                 mask=[dict(pattern="sliding", seq_len=512, band_width=22)],
                 desc="BERT-base MHA layer, bs1 seq512, sliding(22)"),
    "cfg2": dict(model="bert-layer", bs=16, seq=1024, hidden=768, heads=12,
                 mask=[dict(pattern="bigbird", seq_len=1024, global_width=32, band_width=32, filling_rate=0.10,
                            seed=0, block=16)],
                 desc="BERT-base encoder layer, bs16 seq1024, BigBird(32,32,0.10)"),
    "cfg3": dict(model="gpt-layer", bs=8, seq=2048, hidden=768, heads=12,
                 mask=[dict(pattern="strided", seq_len=2048, band_width=45)],
                 desc="GPT-2 decoder layer, bs8 seq2048, causal+strided(45)"),
    "cfg4": dict(model="t5-layer", bs=8, seq=4096, hidden=768, heads=12,
                 mask=[dict(pattern="dilated", seq_len=4096, band_width=64, dilation_rate=1),
                       dict(pattern="global", seq_len=4096, global_width=64)],
                 desc="T5-base layer, bs8 seq4096, dilated(64,1)+global(64)"),
}
METRIC = "BERT/GPT/T5 layer tokens/s (masked MHA + fused FFN/LayerNorm)"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return {"hbm_gbs": j["hbm_gbs"], "tflops": j["bf16_tflops"], "tflops_sustained": j.get("bf16_tflops_sustained"),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "tflops": 1590.0, "tflops_sustained": 1400.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, idx: int):
        self.idx, self.proc, self.lines = idx, None, []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ----------------------------------------------------------------------------------------------
# reference arm / CPU baseline
def cpu_reference(cfg, threads, reps):
    """Time the reference's CpuBackend::run_chain of the config chain (oracle/_ref), one sequence
    (bs = 1) per host thread; returns (tokens/s, kind, sample description)."""
    from oracle.oracle import Oracle, Reference
    o, r = Oracle(), Reference()
    m = o.mask(cfg["mask"])
    seq, hid, heads = cfg["seq"], cfg["hidden"], cfg["heads"]
    if r.available:
        kind = "reference"
        # seconds of the run_chain calls alone (each thread's CpuBackend is built before the clock)
        run = lambda n: r.run_chain(cfg["model"], 1, seq, hid, heads, hid // heads, 1, m, 16, 16, threads=n,
                                    timing=True)[1]
    else:  # the C restatement (oracle port), same chain semantics
        from tests.chain_oracle import graph_data, run_chain
        kind = "port"
        gd = graph_data(o, cfg["model"], 1, seq, hid, 4 * hid, 1)

        def run(n):
            t0 = time.perf_counter()
            run_chain(o, cfg["model"], gd, gd["input"], m, 1, seq, heads, hid // heads, 16, 16, threads=1)
            return time.perf_counter() - t0
        threads = 1
    best = min(run(threads) for _ in range(reps))
    tokens = threads * seq
    one = min(run(1) for _ in range(reps)) if threads > 1 else best  # the 1-core time too
    sample = (f"{threads} independent sequences x {seq} tokens (one per host thread; the batch holds {cfg['bs']}), "
              f"1 layer {cfg['model']} unfused chain, BSR 16x16 (the reference's own a100/rtx4090 plan); "
              f"CpuBackend construction outside the clock; best of {reps}")
    return tokens / best, kind, sample, threads, seq / one


def run_reference_arm(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import Oracle, Reference
    o, r = Oracle(), Reference()
    m = o.mask(cfg["mask"])
    seq, hid, heads = cfg["seq"], cfg["hidden"], cfg["heads"]
    # all host threads this process may use (std::threads in the reference shim, so torchrun's
    # OMP_NUM_THREADS=1 does not apply)
    threads = max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    kind = "reference" if r.available else "port"

    def run(n):  # n independent sequences through the chain, concurrently on n host threads; the
        # seconds of the run_chain calls (backend construction, i.e. GraphData::make, off the clock)
        if r.available:
            return r.run_chain(cfg["model"], 1, seq, hid, heads, hid // heads, 1, m, 16, 16, threads=n, timing=True)[1]
        from tests.chain_oracle import graph_data, run_chain
        gd = graph_data(o, cfg["model"], 1, seq, hid, 4 * hid, 1)
        t0 = time.perf_counter()
        for _ in range(n):
            run_chain(o, cfg["model"], gd, gd["input"], m, 1, seq, heads, hid // heads, 16, 16, threads=1)
        return time.perf_counter() - t0

    # a step = one sequence (seq tokens) through the reference's unfused chain; sequences run in
    # waves of one per host thread (every core busy; K rounded up to whole waves, all of them
    # timed), one warm-up wave first
    if args.warmup:
        run(threads)
    waves = max(1, -(-args.steps // threads))
    wall = sum(run(threads) for _ in range(waves))
    n_seq = waves * threads
    value = n_seq * seq / wall
    one_core = seq / run(1)  # BASELINE.md §3 also quotes the single-core time
    sample = (f"{n_seq} sequences x {seq} tokens ({waves} wave(s) of {threads} concurrent sequences >= the "
              f"{args.steps} steps asked; {cfg['model']}, unfused CpuBackend::run_chain, BSR 16x16 = the "
              f"reference's own a100/rtx4090 plan) on {threads} host threads; each thread's CpuBackend is "
              f"constructed before the clock starts")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * wall / n_seq,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (GraphData seeds)",
            "config": {"workload": cfg["desc"], "model": cfg["model"], "global_batch": cfg["bs"], "seq_len": cfg["seq"]},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": kind, "sample": sample,
                             "value_1core": one_core},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------------
def work_model(cfg, nnz):
    """Algorithmic work per launch: flops for GEMMs, compulsory bytes
    and useful flops for the masked MHA."""
    M, H, F = cfg["bs"] * cfg["seq"], cfg["hidden"], 4 * cfg["hidden"]
    d = H // cfg["heads"]
    w = {"qkv_gemm": ("tensor", 2.0 * M * 3 * H * H), "out_proj_gemm_ln": ("tensor", 2.0 * M * H * H),
         "ffn1_gemm_gelu": ("tensor", 2.0 * M * F * H), "ffn1_gemm_act": ("tensor", 2.0 * M * F * H),
         "ffn2_gemm_ln": ("tensor", 2.0 * M * H * F), "ffn2_gemm": ("tensor", 2.0 * M * H * F),
         "ln1_mi_chain": ("hbm", 2.0 * M * H * 2),
         "out_proj_gemm": ("tensor", 2.0 * M * H * H),          "out_proj_ln": ("hbm", 2.0 * M * H * 2), "ffn2_ln": ("hbm", 2.0 * M * H * 2),
         "masked_mha": ("hbm", 4.0 * cfg["bs"] * cfg["heads"] * cfg["seq"] * d * 2)}
    mha_flops = 4.0 * d * cfg["bs"] * cfg["heads"] * nnz
    return w, mha_flops


# ----------------------------------------------------------------------------------------------
# cfg5: masking-pattern x sequence-length sweep of the masked MHA (BASELINE configs[4])
SWEEP_PATTERNS = ("sliding", "dilated", "longformer", "bigbird", "causal", "strided")
SWEEP_SEQ = (128, 256, 512, 1024, 2048, 4096, 8192)
MUFU_PER_CLK_SM = 16  # ex2 throughput per SM per clock on sm_100 (B300's doubled SFU is sm_103 only)


def sweep_terms(pattern, n):
    w = int(np.floor(np.sqrt(n)))  # band and global width = sqrt(seq_len)
    return {"sliding": [dict(pattern="sliding", seq_len=n, band_width=w)],
            "dilated": [dict(pattern="dilated", seq_len=n, band_width=w, dilation_rate=1)],
            "longformer": [dict(pattern="longformer", seq_len=n, global_width=w, band_width=w)],
            "bigbird": [dict(pattern="bigbird", seq_len=n, global_width=w, band_width=w, filling_rate=0.10, seed=0,
                             block=16)],
            "causal": [dict(pattern="causal", seq_len=n)],
            "strided": [dict(pattern="strided", seq_len=n, band_width=w)]}[pattern]


def run_sweep(args):
    """Masked-MHA latency and % of roofline for every (pattern, n), bs 16 x 12 heads x 64 on one
    GPU (the sweep shards (b, h) units over ranks with no exchange, so per-GPU work is this at any
    N). Roofline per SURVEY §8(d): bound = max(useful flops / tensor peak, exps / MUFU rate,
    compulsory bytes / HBM peak). One JSON line per point; the reference's own block_sparse_sdpa
    (16x16 BSR, oracle/_ref) is timed on one (b, h) slice where that takes < ~2 s and scaled."""
    import torch
    from paper_2506_06095_b200 import dist as sfdist, sparsefuse as sf
    rank, world, local = dist_env()
    shared = os.environ.get("SF_BENCH_SHARED_GPU") == "1"
    torch.cuda.set_device(0 if shared else local)
    if world > 1:
        import torch.distributed as tdist
        if shared:
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pk = peaks()
    clk_hz = 1.965e9
    bs, h, d = 16, 12, 64
    # N > 1: the bs x h (b, h) slices are sharded contiguously over the ranks (no exchange: every
    # rank builds the formats from the descriptor); latency = max over ranks
    s0, s1 = sfdist.shard_range(bs * h, world, rank)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ref = None
    if not args.no_cpu_baseline and rank == 0:
        from oracle.oracle import Reference
        ref = Reference()
        if not ref.available:
            ref = None
    pats = args.patterns.split(",") if args.patterns else SWEEP_PATTERNS
    seqs = [int(x) for x in args.seqs.split(",")] if args.seqs else SWEEP_SEQ
    for n in seqs:
        g = torch.Generator(device="cuda").manual_seed(1)
        q, k, v = ((torch.rand(bs, h, n, d, device="cuda", generator=g) * 2 - 1).half()[:, :].reshape(bs * h, n, d)
                   [s0:s1].unsqueeze(0).contiguous() for _ in range(3))  # this rank's slices as (1, cnt, n, d)
        o = torch.empty_like(q)
        for pat in pats:
            dm = sf.generate_mask(sweep_terms(pat, n))
            nnz = dm.true_count()
            plan = sf.select_plan(dm, sf.hw_preset("b200"), n, h, bs, d, mode="b200")  # the job's plan
            ctx = sf.context_for(sweep_terms(pat, n), dm, plan)
            run = lambda: sf.mha(q, k, v, ctx, out=o)
            for _ in range(3):
                run()
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=st):
                sf.mha(q, k, v, ctx, out=o, stream=st)
            ts = []
            for _ in range(args.steps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); gr.replay(); b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            us = statistics.median(ts)
            if world > 1:
                us = sfdist.max_over_ranks(us, device="cpu" if shared else "cuda")
            flops = 4.0 * d * bs * h * nnz  # the whole job (all ranks); bounds are per GPU
            exps = float(bs * h * nnz)
            comp = 4.0 * bs * h * n * d * 2
            t_tc = flops / (pk["tflops"] * 1e12) * 1e6 / world
            t_exp = exps / (MUFU_PER_CLK_SM * 148 * clk_hz) * 1e6 / world
            t_hbm = comp / (pk["hbm_gbs"] * 1e9) * 1e6 / world
            bound_us = max(t_tc, t_exp, t_hbm)
            binds = ("tensor", "mufu", "hbm")[[t_tc, t_exp, t_hbm].index(bound_us)]
            line = {"sweep": "masked_mha", "pattern": pat, "seq_len": n, "bs": bs, "heads": h, "head_size": d,
                    "n_gpus": world, "slices_per_rank": s1 - s0, "scaling": "strong",
                    "nnz_per_slice": nnz, "density": nnz / float(n * n),
                    "plan": sf.executor_label(ctx), "latency_us": us,
                    "useful_tflops": flops / us / 1e6, "compulsory_gbs": comp / us / 1e3,  # whole job
                    "roofline": {"bound": binds, "bound_us": bound_us, "t_tensor_us": t_tc, "t_mufu_us": t_exp,
                                 "t_hbm_us": t_hbm, "frac": bound_us / us},
                    "l2": "flushed before each timed launch", "timing": f"median of {args.steps} single launches"}
            if plan.kind == "block_wise":
                line["executed_cells_per_slice"] = int(ctx.bsr.n_load) * plan.block_m * plan.block_n

            def time_launch(fn):
                st2 = torch.cuda.Stream()
                st2.wait_stream(torch.cuda.current_stream())
                for _ in range(2):
                    fn(None)
                g2 = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g2, stream=st2):
                    fn(st2)
                tt = []
                for _ in range(max(5, args.steps // 2)):
                    flush.zero_()
                    a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a2.record(); g2.replay(); b2.record()
                    torch.cuda.synchronize()
                    tt.append(a2.elapsed_time(b2) * 1e3)
                return statistics.median(tt)

            # both executors where the other one is affordable: the data behind the selector
            if args.both and world == 1 and bs * h * nnz <= 4e8:
                if plan.kind == "block_wise":
                    rw = sf.build_rowwise(dm)
                    line["rowwise_us"] = time_launch(lambda s_: sf.rowwise_sdpa(q, k, v, rw, out=o, stream=s_))
                    del rw
                else:
                    line["rowwise_us"] = us
            if args.both and world == 1 and plan.kind != "block_wise":
                bsr = sf.build_bsr(dm, 128, 16)
                line["blockwise_us"] = time_launch(lambda s_: sf.block_sparse_sdpa(q, k, v, bsr, out=o, stream=s_))
                line["executed_cells_per_slice"] = int(bsr.n_load) * 128 * 16
                del bsr
            elif args.both and world == 1:
                line["blockwise_us"] = us
            if ref is not None and nnz <= 6_000_000:
                from oracle.oracle import Oracle
                o_ = Oracle()
                m = o_.mask(sweep_terms(pat, n))
                q1, k1, v1 = (x[:1, :1].float().cpu().numpy() for x in (q, k, v))
                t0 = time.perf_counter()
                ref.block_sparse_sdpa(q1, k1, v1, m, 16, 16, threads=1)
                sl = time.perf_counter() - t0
                line["cpu_baseline"] = {"kind": "reference", "cores": 1, "slice_ms": sl * 1e3,
                                        "latency_us_scaled": sl * 1e6 * bs * h,
                                        "sample": "one (b,h) slice of the reference block_sparse_sdpa (16x16 BSR), "
                                                  "scaled by bs*h (the per-slice work is identical, attention.hpp:58-59)"}
            if rank == 0:
                print(json.dumps(line), flush=True)
            del ctx
        del q, k, v, o
        torch.cuda.empty_cache()
    if world > 1:
        torch.distributed.destroy_process_group()


# ----------------------------------------------------------------------------------------------
# cfg3 selector sweep: band width across the Eq. 1 boundary, both executors timed
def run_band_sweep(args):
    """BASELINE configs[2] (GPT-2 shapes, bs 8 x 12 heads x 64, n = 2048): sliding and causal-local
    bands of width {1,2,4,8,16,24,32,48,64} (Eq. 1 turns row-wise at w <= 16 sliding /
    w <= 48 causal-local). For each: Eq. 1's threshold, the reference-mode and B200-mode plans, and
    the measured time of BOTH executors, so the selector's choice can be checked against the
    faster one (regret = chosen / best)."""
    import torch
    from paper_2506_06095_b200 import sparsefuse as sf
    torch.cuda.set_device(0)
    bs, h, n, d = 8, 12, 2048, 64
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(1)
    q, k, v = ((torch.rand(bs, h, n, d, device="cuda", generator=g) * 2 - 1).half() for _ in range(3))
    o = torch.empty_like(q)

    def timed(fn):
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        for _ in range(2):
            fn(None)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            fn(st)
        ts = []
        for _ in range(max(5, args.steps)):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); gr.replay(); b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        return statistics.median(ts)

    # bands (Eq. 1's row-wise region), then unstructured cells (random blocks of 1 x 1 at density p:
    # every (128,16) tile loaded, nearly empty — the masks the row-wise executor is for)
    cases = [(pat, w, [dict(pattern=pat, seq_len=n, band_width=w)]) for pat in ("sliding", "causal_local")
             for w in (1, 2, 4, 8, 16, 24, 32, 48, 64)]
    cases += [("random_cells", p, [dict(pattern="random", seq_len=n, block=1, filling_rate=p, seed=7)])
              for p in (0.002, 0.005, 0.01, 0.02, 0.05)]
    for pat, w, terms in cases:
        dm = sf.generate_mask(terms)
        ref_plan = sf.select_plan(dm, sf.hw_preset("b200"), n, h, bs, d, mode="reference")
        b200_plan = sf.select_plan(dm, sf.hw_preset("b200"), n, h, bs, d, mode="b200")
        bsr = sf.build_bsr(dm, 128, 16)
        rw = sf.build_rowwise(dm)
        t_bw = timed(lambda s_: sf.block_sparse_sdpa(q, k, v, bsr, out=o, stream=s_))
        t_rw = timed(lambda s_: sf.rowwise_sdpa(q, k, v, rw, out=o, stream=s_))
        # the block executor also at the other tile height (block_m 64: head pairs), so the B200
        # plan's tile choice is checked too
        bsr64 = sf.build_bsr(dm, 64, 16)
        t_bw64 = timed(lambda s_: sf.block_sparse_sdpa(q, k, v, bsr64, out=o, stream=s_))
        best = min(t_bw, t_bw64, t_rw)
        chosen = lambda pl: (t_bw64 if pl.block_m == 64 else t_bw) if pl.kind == "block_wise" else t_rw
        print(json.dumps({"band_sweep": pat, "seq_len": n, ("density" if pat == "random_cells" else "band"): w, "bs": bs, "heads": h, "nnz": dm.true_count(),
                          "eq1_threshold": ref_plan.threshold, "reference_plan": ref_plan.kind,
                          "b200_plan": [b200_plan.kind, b200_plan.block_m, b200_plan.block_n],
                          "blockwise_us": t_bw, "blockwise_bm64_us": t_bw64, "rowwise_us": t_rw,
                          "regret_reference_mode": (t_bw if ref_plan.kind == "block_wise" else t_rw) / best,
                          "regret_b200_mode": chosen(b200_plan) / best}), flush=True)


# ----------------------------------------------------------------------------------------------
# format builders (A1-A4, A9): device latency vs the reference's own builders on the host
def run_formats(args):
    """Device latency (CUDA events around the C-ABI call, warm, median of --steps) of mask
    generation, build_bsr at the reference's 16x16 and the B200 plan's (128,16), build_rowwise
    and select_plan, for every BASELINE mask and n = 8192 masks; the reference's generate_mask /
    build_bsr / build_rowwise (oracle/_ref) timed on one host core beside them. These builders
    are latency-bound: the metric is microseconds, the roofline is not the point."""
    import torch
    from paper_2506_06095_b200 import sparsefuse as sf
    torch.cuda.set_device(0)
    ref = None
    if not args.no_cpu_baseline:
        from oracle.oracle import Reference
        ref = Reference()
        if not ref.available:
            ref = None
    masks = [(name, cfg["mask"]) for name, cfg in sorted(CONFIGS.items())]
    masks += [(f"{pat}-8192", sweep_terms(pat, 8192)) for pat in ("sliding", "bigbird", "causal")]

    def dev_us(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        return statistics.median(ts)

    def graph_of(fn):  # the call captured once into a CUDA graph; returns its replay
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            fn(st)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            fn(st)
        return gr.replay

    def host_ms(fn, reps=3):
        best = 1e30
        for _ in range(reps):
            t0 = time.perf_counter(); fn(); best = min(best, time.perf_counter() - t0)
        return best * 1e3

    for name, terms in masks:
        dm = sf.generate_mask(terms)
        n = dm.seq_len
        ws = sf.BsrWorkspace(n, 128, 16)
        line = {"formats": name, "seq_len": n, "nnz": dm.true_count(),
                "device_us": {"generate_mask": dev_us(lambda: sf.generate_mask(terms)),
                              "build_bsr_16x16": dev_us(lambda: sf.build_bsr(dm, 16, 16)),
                              "build_bsr_128x16": dev_us(lambda: sf.build_bsr(dm, 128, 16)),
                              "build_bsr_async_128x16": dev_us(lambda: ws.build_async(dm)),
                              "build_bsr_async_128x16_graph": dev_us(graph_of(lambda st: ws.build_async(dm, stream=st))),
                              "build_rowwise": dev_us(lambda: sf.build_rowwise(dm)),
                              "select_plan_b200": dev_us(lambda: sf.select_plan(dm, sf.hw_preset("b200"), n, 12, 16,
                                                                                 64, mode="b200"))},
                "timing": f"CUDA events around the call incl. its host sync (sizes), warm, median of {args.steps}"}
        if ref is not None:
            m = dm.to_numpy()  # the same mask bytes (strided/causal are generators the reference lacks)
            r = {"build_bsr_16x16": host_ms(lambda: ref.sfbr(m, 16, 16)),
                 "build_rowwise": host_ms(lambda: ref.rowwise(m))}
            try:
                r["generate_mask"] = host_ms(lambda: ref.mask(terms))
            except ValueError:
                pass
            line["reference_ms_1core"] = r
            line["reference_note"] = "build_bsr timed through write_bsr serialisation (SFBR bytes), one host core"
        print(json.dumps(line), flush=True)


def gather_check(L, x, x_global, W, ctx, cfg, s_global, args, shared):
    """The sharded run's gathered layer output against the same layer run on the whole batch on one
    GPU (rank 0): bit-exact when both shard sizes take the same kernel variants, else within the
    fp16 tolerance. The gather goes through dist.gather_rows (NCCL; gloo on CPU tensors in the
    shared-GPU test mode)."""
    import torch
    from paper_2506_06095_b200 import dist as sfdist, layer
    y = L.forward(x).clone()
    torch.cuda.synchronize()
    full = sfdist.gather_rows(y.cpu() if shared else y)
    out = {"world": int(torch.distributed.get_world_size()) if torch.distributed.is_initialized() else 1}
    full_ref = layer.EncoderLayer(cfg["model"], s_global, W, ctx, ln_split=args.ln_split).forward(x_global)
    torch.cuda.synchronize()
    a, b = full.float().cpu(), full_ref.float().cpu()
    out["bit_exact"] = bool(torch.equal(full.cpu(), full_ref.cpu()))
    out["max_abs"] = float((a - b).abs().max())
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ln-split", action="store_true", help="residual+LN as a MiChain pass after the GEMM")
    ap.add_argument("--sweep", action="store_true", help="cfg5: masked-MHA pattern x seq_len sweep (JSON lines)")
    ap.add_argument("--patterns", default="", help="--sweep: comma list (default: all six)")
    ap.add_argument("--seqs", default="", help="--sweep: comma list (default: 128..8192)")
    ap.add_argument("--both", action="store_true", help="--sweep: also time the executor the plan did not pick")
    ap.add_argument("--formats", action="store_true", help="format-builder latency (A1-A4, A9) vs the reference")
    ap.add_argument("--band-sweep", action="store_true", help="cfg3 selector sweep: both executors across Eq. 1")
    ap.add_argument("--check-gather", action="store_true",
                    help="N > 1: gathered sharded output vs the whole batch on one GPU (gather_check in the line)")
    args = ap.parse_args()
    if args.band_sweep:
        return run_band_sweep(args)
    if args.sweep:
        return run_sweep(args)
    if args.formats:
        return run_formats(args)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, cfg)

    import torch
    rank, world, local = dist_env()
    # SF_BENCH_SHARED_GPU=1 (test aid): every rank on cuda:0 with gloo — exercises the N > 1 code
    # path on a one-GPU box (NCCL refuses two ranks on one device). Real runs: one GPU per rank, NCCL.
    shared = os.environ.get("SF_BENCH_SHARED_GPU") == "1"
    torch.cuda.set_device(0 if shared else local)
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2506_06095_b200 import _lib, dist as sfdist, layer, sparsefuse as sf

    gbs = cfg["bs"]
    if world > gbs:
        raise SystemExit(f"{args.config}: batch {gbs} cannot be sharded over {world} ranks by sequence "
                         "(use --sweep, which shards (b, h) slices)")
    b0, b1 = sfdist.shard_range(gbs, world, rank)  # this rank's sequences of the global batch
    s = layer.LayerShape(b1 - b0, cfg["seq"], cfg["hidden"], cfg["heads"], cfg["hidden"] // cfg["heads"])
    s_global = layer.LayerShape(gbs, cfg["seq"], cfg["hidden"], cfg["heads"], cfg["hidden"] // cfg["heads"])
    dm = sf.generate_mask(cfg["mask"])
    nnz = dm.true_count()
    plan = sf.select_plan(dm, sf.hw_preset("b200"), s.seq_len, s.heads, s.bs, s.head_size, mode="b200")
    ctx = sf.context_for(cfg["mask"], dm, plan)
    W = layer.init_weights(cfg["model"], s, seed=1)  # one model: the same weights on every rank
    L = layer.EncoderLayer(cfg["model"], s, W, ctx, ln_split=args.ln_split)
    g = torch.Generator(device="cuda").manual_seed(7)
    x_global = (torch.rand(s_global.rows, s_global.hidden, device="cuda", generator=g) * 2 - 1).half()
    x = x_global[b0 * s.seq_len:b1 * s.seq_len].clone()
    if not args.check_gather:
        del x_global
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    clean = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")

    def l2_flush():
        # write a buffer larger than L2 (evicts everything the previous step left), then read
        # another one, so the flush's own dirty lines are written back here, outside the step
        # events, instead of inside the next step: the step starts from a cold, clean L2
        flush.zero_()
        clean.max()

    for _ in range(args.warmup):
        L.forward(x)
    torch.cuda.synchronize()
    # one step = one CUDA-graph replay of the layer's launches (no per-launch host overhead)
    launches0 = _lib.launch_count()
    L.capture(x)
    L.capture(x, timed=True)  # + event-record nodes between launches: per-kernel device time
    per_step_launches = _lib.launch_count() - launches0 - L.kernels_per_step()  # capture warms once
    for _ in range(3):
        L.replay()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed between steps (outside the per-step events) ----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    parts_sum = {}
    with ClockSampler(0 if shared else local) as clk:
        time.sleep(0.3)  # the sampler's first reading lands inside the timed region
        for a, b in evs:
            l2_flush()
            a.record()
            L.replay()
            b.record()
        torch.cuda.synchronize()
        # per-kernel device times: the same K steps again through the instrumented graph (event
        # nodes between the launches cost ~1 us each, so the headline above runs without them)
        for _ in range(args.steps):
            l2_flush()
            L.replay(timed=True)
            torch.cuda.synchronize()
            for k, v in L.kernel_ms().items():
                parts_sum[k] = parts_sum.get(k, 0.0) + v
    launches = per_step_launches * args.steps
    if world > 1:
        torch.distributed.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device="cpu" if shared else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    tokens = s_global.rows  # the whole job: the configured batch, sharded over the ranks
    value = tokens / (ms_per_step / 1e3)

    # ---- e2e through the public API with host buffers: every step copies its input from pinned
    # host memory and reads its output back. Copies run on their own streams (copy engines, both
    # PCIe directions at once) and overlap neighbouring steps' compute; NB layer instances (shared
    # weights and formats) rotate the activations so no buffer is overwritten while a copy still
    # reads it, and the copy streams never wait on the compute of the step just before.
    NB = int(os.environ.get("SF_E2E_BUFFERS", "8"))
    hx = torch.empty(s.rows, s.hidden, dtype=torch.float16, pin_memory=True)
    hx.copy_(x.cpu())
    # N > 1 (NCCL): each step's outputs are all-gathered into a full-batch buffer on every rank
    # (NVLink), and rank 0 reads the whole layer output back; N = 1 reads its own output back
    nccl_gather = world > 1 and not shared
    gath = [torch.empty(s_global.rows, s.hidden, dtype=torch.float16, device="cuda") for _ in range(NB)] \
        if nccl_gather else None
    read_back = rank == 0 or not nccl_gather
    hy = [torch.empty(gath[0].shape if nccl_gather else hx.shape, dtype=torch.float16, pin_memory=True)
          for _ in range(NB)]
    Ls = [L] + [layer.EncoderLayer(cfg["model"], s, W, ctx, ln_split=args.ln_split) for _ in range(NB - 1)]
    xs = [x] + [torch.empty_like(x) for _ in range(NB - 1)]
    for b in range(1, NB):
        Ls[b].capture(xs[b])
    s_in, s_comp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event(enable_timing=False)
    in_ready, comp_done, out_done = [ev() for _ in range(NB)], [ev() for _ in range(NB)], [ev() for _ in range(NB)]

    def e2e_run(n):
        for i in range(n):
            b = i % NB
            if i >= NB:
                s_in.wait_event(comp_done[b])       # x[b] no longer read by step i-NB
            with torch.cuda.stream(s_in):
                xs[b].copy_(hx, non_blocking=True)
                in_ready[b].record(s_in)
            s_comp.wait_event(in_ready[b])
            if i >= NB:
                s_comp.wait_event(out_done[b])      # out of layer b read back by step i-NB
            with torch.cuda.stream(s_comp):
                Ls[b].replay()                      # the layer's launches as one CUDA graph
            comp_done[b].record(s_comp)
            s_out.wait_event(comp_done[b])
            with torch.cuda.stream(s_out):
                src = Ls[b].out
                if nccl_gather:  # NCCL all-gather ordered on s_out (torch syncs its comm stream)
                    torch.distributed.all_gather_into_tensor(gath[b], src)
                    src = gath[b]
                if read_back:
                    hy[b].copy_(src, non_blocking=True)
                out_done[b].record(s_out)

    e2e_steps = max(4, min(args.steps, 100))
    e2e_run(e2e_steps)  # one untimed window first: the first windows of pinned-memory copies run slow
    torch.cuda.synchronize()
    if os.environ.get("SF_E2E_PROBE"):  # diagnosis: repeated e2e windows in one process
        for _ in range(6):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(s_in)
            t_host = time.perf_counter()
            e2e_run(e2e_steps)
            t_enq = time.perf_counter() - t_host
            s_out.wait_event(out_done[(e2e_steps - 1) % NB])
            a1.record(s_out)
            torch.cuda.synchronize()
            print(f"e2e probe: {a0.elapsed_time(a1) / e2e_steps:.3f} ms/step (host enqueue {t_enq * 1e3 / e2e_steps:.3f} ms/step)",
                  file=sys.stderr)
    # E2E_WINDOWS windows of e2e_steps steps each (max over ranks per window); the reported value
    # is the median window, with every window's figure beside it (host-side PCIe / pinned-copy
    # behaviour varies between windows and between boxes, so one window is not a measurement)
    windows = []
    for _ in range(int(os.environ.get("SF_E2E_WINDOWS", "5"))):
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_in)
        e2e_run(e2e_steps)
        s_out.wait_event(out_done[(e2e_steps - 1) % NB])
        e1.record(s_out)
        torch.cuda.synchronize()
        w_ms = e0.elapsed_time(e1) / e2e_steps
        if world > 1:
            t = torch.tensor([w_ms], device="cpu" if shared else "cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            w_ms = float(t.item())
        windows.append(w_ms)
    e2e_ms = statistics.median(windows)

    # the box's own PCIe ceiling for this e2e: the same per-step copies (H2D of the input, D2H of the
    # output, both directions concurrently on the two copy streams) with no compute, same step count
    cur = torch.cuda.current_stream()
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(cur)
    s_in.wait_stream(cur)
    s_out.wait_stream(cur)
    for i in range(e2e_steps):
        b = i % NB
        with torch.cuda.stream(s_in):
            xs[b].copy_(hx, non_blocking=True)
        if read_back:
            with torch.cuda.stream(s_out):
                hy[b].copy_(gath[b] if nccl_gather else Ls[b].out, non_blocking=True)
    cur.wait_stream(s_in)
    cur.wait_stream(s_out)
    c1.record(cur)
    torch.cuda.synchronize()
    copy_ms = c0.elapsed_time(c1) / e2e_steps
    pcie = {"copy_only_ms_per_step": copy_ms,
            "h2d_gbs": hx.numel() * 2 / (copy_ms / 1e3) / 1e9,
            "copy_only_tokens_per_s": tokens / (copy_ms / 1e3),
            "e2e_frac_of_copy_only": copy_ms / e2e_ms,
            "how": "the e2e's H2D and D2H copies alone, both directions concurrently, measured live on this box"}

    # ---- per-kernel breakdown (mean over the timed steps) and roofline of the dominant kernel ----
    parts = {k: v / args.steps for k, v in parts_sum.items()}
    wm, mha_flops = work_model(cfg, nnz)
    pk = peaks()
    dom = max(parts, key=parts.get)
    bound, work = wm[dom]
    if bound == "tensor":
        achieved = work / (parts[dom] / 1e3) / 1e12
        roof = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": pk["tflops"], "unit": "TFLOP/s",
                "frac": achieved / pk["tflops"], "peak_kind": "burst, " + pk["source"]}
    else:
        achieved = work / (parts[dom] / 1e3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "peak_kind": pk["source"]}
    traffic_file = ROOT / "profiles" / "traffic.json"
    roof["traffic"] = None
    if traffic_file.exists():
        roof["traffic"] = json.loads(traffic_file.read_text()).get(args.config, {}).get(dom)
    mha_ms = parts["masked_mha"]
    mha = {"latency_us": mha_ms * 1e3, "plan": sf.executor_label(ctx),
           "nnz_per_slice": nnz, "useful_tflops": mha_flops / (mha_ms / 1e3) / 1e12,
           "compulsory_gbs": wm["masked_mha"][1] / (mha_ms / 1e3) / 1e9,
           "hbm_frac": wm["masked_mha"][1] / (mha_ms / 1e3) / 1e9 / pk["hbm_gbs"]}

    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f16",
            "data": "synthetic (uniform[-1,1) activations, random-init weights of the architecture)",
            "config": {"workload": cfg["desc"], "model": cfg["model"], "global_batch": gbs,
                       "seq_len": cfg["seq"], "hidden": cfg["hidden"], "heads": cfg["heads"],
                       "parallelism": f"dp{world}: the batch's sequences sharded over ranks ({s.bs} per rank), full "
                                      "weights per rank, no collective in the timed layer step",
                       "l2": "flushed between timed steps, outside the step events: 256 MB write, then a 256 MB read so the flush's dirty lines are written back before the step (cold, clean L2)",
                       "kernel_timing": "event-record nodes between the launches of an instrumented copy of the step's CUDA graph, K extra steps, mean"},
            "e2e": {"value": tokens / (e2e_ms / 1e3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(hx.numel() * 2) * world,
                    "d2h_bytes_per_step": int(hy[0].numel() * 2) * (1 if nccl_gather else world),
                    "copies": "pinned host buffers, H2D/D2H on copy streams overlapping adjacent steps' compute"
                              + ("; each rank copies its shard in, an NCCL all-gather assembles the full output "
                                 "on every rank, rank 0 reads it back" if nccl_gather else ""),
                    "pcie_bound": pcie,
                    "windows_tokens_per_s": [tokens / (w / 1e3) for w in windows],
                    "window_steps": e2e_steps, "statistic": "median of the windows"},
            "gpu_launches": int(launches), "roofline": roof, "kernels_ms": parts, "mha": mha,
            "clocks": clk.summary()}
    if args.check_gather:
        line["gather_check"] = gather_check(L, x, x_global, W, ctx, cfg, s_global, args, shared)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        host = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
        v, kind, sample, thr, v1 = cpu_reference(cfg, max(1, host), 1)
        line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": thr, "kind": kind, "sample": sample,
                                "value_1core": v1}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
