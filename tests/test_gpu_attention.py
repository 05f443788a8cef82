"""Masked MHA on the GPU vs the reference executors (north-star bar: fp16 outputs within
max-abs 2e-2 and mean-rel (sum|d| / sum|ref|) 1e-3 of the reference's fp32 results on the same
fp16-rounded inputs). Cases follow test_attention.cpp."""
import os
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import CONFIG_MASKS

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"
MAX_ABS, MEAN_REL = 2e-2, 1e-3


def parity(out, ref, max_abs=MAX_ABS, mean_rel=MEAN_REL):
    out = out.float().cpu().numpy().astype(np.float64) if hasattr(out, "cpu") else out
    ref = np.asarray(ref, np.float64)
    d = np.abs(out - ref)
    ma = float(d.max()) if d.size else 0.0
    mr = float(d.sum() / max(np.abs(ref).sum(), 1e-30))
    assert ma <= max_abs and mr <= mean_rel, f"max_abs {ma:.3e} mean_rel {mr:.3e}"
    return ma, mr


def to_dev(x, dtype):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def fp16_inputs(oracle, bs, h, n, d, seed):
    return [x.astype(np.float16).astype(np.float32) for x in oracle.random_attention_input(bs, h, n, d, seed)]


@pytest.mark.parametrize("impl", ["generic", "auto"])
def test_golden_attention_cases(sf, oracle, impl):
    import torch
    from tests.golden.make_golden import ATTN_CASES
    z = np.load(G / "attn_small.npz")
    sf.set_attn_impl(impl)
    try:
        for name, (terms, bm, bn, bs, h, d, seed) in ATTN_CASES.items():
            dm = sf.generate_mask(terms)
            q, k, v = fp16_inputs(oracle, bs, h, dm.seq_len, d, seed)
            b = sf.build_bsr(dm, bm, bn)
            out, st = sf.block_sparse_sdpa(to_dev(q, torch.float16), to_dev(k, torch.float16),
                                           to_dev(v, torch.float16), b, stats=True)
            try:
                parity(out, z[name + "/out"])
            except AssertionError as e:
                raise AssertionError(f"{name} ({impl}): {e}")
            ref_stats = z[name + "/stats"]
            assert (st["tiles_loaded"], st["full_tiles"], st["part_tiles"]) == tuple(int(x) for x in ref_stats)
    finally:
        sf.set_attn_impl("auto")


@pytest.mark.parametrize("cfg,tile,bs,h", [("cfg1", (128, 16), 1, 12), ("cfg2", (128, 16), 2, 12),
                                           ("cfg3", (128, 16), 1, 4), ("cfg4", (128, 64), 1, 2),
                                           ("cfg2", (16, 16), 1, 4), ("cfg1", (64, 32), 1, 4),
                                           ("cfg2", (64, 16), 1, 3), ("cfg3", (64, 16), 1, 2), ("cfg4", (64, 64), 1, 1)])
def test_config_attention_matches_oracle(sf, oracle, cfg, tile, bs, h):
    import torch
    terms = CONFIG_MASKS[cfg]
    m = oracle.mask(terms)
    n = m.shape[0]
    q, k, v = fp16_inputs(oracle, bs, h, n, 64, 1)
    ref, _ = oracle.block_sparse_sdpa(q, k, v, m, *tile, threads=8)
    dm = sf.generate_mask(terms)
    b = sf.build_bsr(dm, *tile)
    # block_m 64 runs the tcgen05 head-pair kernel (two heads per TMEM tile; odd head counts
    # leave the last pair's second head empty)
    impls = ("generic", "tcgen05") if tile[0] in (64, 128) and tile[1] in (16, 32, 64) else ("generic", "auto")
    for impl in impls:
        sf.set_attn_impl(impl)
        out = sf.block_sparse_sdpa(to_dev(q, torch.float16), to_dev(k, torch.float16), to_dev(v, torch.float16), b)
        parity(out, ref)
    sf.set_attn_impl("auto")
    # row-wise executor over the same mask
    rw = sf.build_rowwise(dm)
    out = sf.rowwise_sdpa(to_dev(q, torch.float16), to_dev(k, torch.float16), to_dev(v, torch.float16), rw)
    parity(out, ref)


def test_fully_masked_rows_are_exact_zero(sf, oracle):
    import torch
    # test_attention.cpp:41-50
    q, k, v = fp16_inputs(oracle, 2, 2, 16, 8, 1)
    dm = sf.DenseMask.from_numpy(np.zeros((16, 16), np.uint8))
    o = sf.block_sparse_sdpa(to_dev(q, torch.float16), to_dev(k, torch.float16), to_dev(v, torch.float16),
                             sf.build_bsr(dm, 4, 4))
    assert torch.count_nonzero(o).item() == 0
    o = sf.rowwise_sdpa(to_dev(q, torch.float16), to_dev(k, torch.float16), to_dev(v, torch.float16),
                        sf.build_rowwise(dm))
    assert torch.count_nonzero(o).item() == 0
    # partially masked: rows 0..3 empty in a causal-shifted pattern
    m = np.tril(np.ones((200, 200), np.uint8), -4)
    q, k, v = fp16_inputs(oracle, 1, 2, 200, 64, 3)
    ref, _ = oracle.block_sparse_sdpa(q, k, v, m, 128, 16)
    o = sf.block_sparse_sdpa(to_dev(q, torch.float16), to_dev(k, torch.float16), to_dev(v, torch.float16),
                             sf.build_bsr(sf.DenseMask.from_numpy(m), 128, 16))
    parity(o, ref)
    assert torch.count_nonzero(o[:, :, :4]).item() == 0


def test_single_valid_position_copies_v(sf, oracle):
    import torch
    # test_attention.cpp:52-60 (diagonal) through both executors
    n, d = 40, 64
    q, k, v = fp16_inputs(oracle, 1, 1, n, d, 3)
    dm = sf.gen_sliding_window(n, 1)
    Q, K, V = (to_dev(x, torch.float16) for x in (q, k, v))
    for o in (sf.block_sparse_sdpa(Q, K, V, sf.build_bsr(dm, 128, 16)), sf.rowwise_sdpa(Q, K, V, sf.build_rowwise(dm))):
        assert np.abs(o.float().cpu().numpy() - v).max() <= 1e-3


def test_all_ones_v_normalisation(sf, oracle):
    import torch
    # test_attention.cpp:122-139: probabilities sum to one
    n = 48
    terms = [dict(pattern="bigbird", seq_len=n, global_width=4, band_width=6, filling_rate=0.2, seed=41)]
    m = oracle.mask(terms)
    q, k, _ = fp16_inputs(oracle, 1, 2, n, 64, 43)
    v = np.ones_like(q)
    dm = sf.generate_mask(terms)
    Q, K, V = (to_dev(x, torch.float16) for x in (q, k, v))
    expect = np.broadcast_to((m.sum(1) > 0).astype(np.float32)[None, None, :, None], q.shape)
    for o in (sf.block_sparse_sdpa(Q, K, V, sf.build_bsr(dm, 128, 16)), sf.rowwise_sdpa(Q, K, V, sf.build_rowwise(dm))):
        assert np.abs(o.float().cpu().numpy() - expect).max() <= 2e-3


def test_strided_activation_layout(sf, oracle):
    """(bs*seq, 3*heads*d) fused-QKV layout read in place; output in (bs*seq, heads*d)."""
    import torch
    bs, h, n, d = 2, 3, 256, 64
    terms = [dict(pattern="longformer", seq_len=n, global_width=16, band_width=16)]
    m = oracle.mask(terms)
    q, k, v = fp16_inputs(oracle, bs, h, n, d, 9)
    ref, _ = oracle.block_sparse_sdpa(q, k, v, m, 128, 16)
    qkv = torch.empty(bs * n, 3 * h * d, dtype=torch.float16, device="cuda")
    for t, x in enumerate((q, k, v)):
        qkv[:, t * h * d:(t + 1) * h * d] = to_dev(x.transpose(0, 2, 1, 3).reshape(bs * n, h * d), torch.float16)
    view = lambda t: qkv[:, t * h * d:(t + 1) * h * d].view(bs, n, h, d).permute(0, 2, 1, 3)
    out = torch.zeros(bs * n, h * d, dtype=torch.float16, device="cuda")
    ov = out.view(bs, n, h, d).permute(0, 2, 1, 3)
    dm = sf.generate_mask(terms)
    sf.block_sparse_sdpa(view(0), view(1), view(2), sf.build_bsr(dm, 128, 16), out=ov)
    parity(ov, ref)
    out.zero_()
    sf.rowwise_sdpa(view(0), view(1), view(2), sf.build_rowwise(dm), out=ov)
    parity(ov, ref)


def test_plan_errors(sf, oracle):
    import torch
    # test_attention.cpp:158-170
    q, k, v = (to_dev(x, torch.float16) for x in fp16_inputs(oracle, 1, 1, 64, 16, 3))
    b = sf.build_bsr(sf.DenseMask.from_numpy(np.ones((64, 64), np.uint8)), 16, 16)
    with pytest.raises(sf._lib.PlanError):
        sf.block_sparse_sdpa(q, k, v, b, sf.KernelPlan("block_wise", 32, 16, 4))
    sf.block_sparse_sdpa(q, k, v, b, sf.KernelPlan("block_wise", 16, 16, 4))
    with pytest.raises(sf._lib.PlanError):
        sf.block_sparse_sdpa(q, k, v, b, sf.KernelPlan("row_wise"))
    with pytest.raises(sf._lib.ShapeError):
        sf.block_sparse_sdpa(q, k, v, sf.build_bsr(sf.gen_sliding_window(32, 2), 16, 16))


def test_unified_mha_dispatch(sf, oracle):
    import torch
    n = 2048
    terms = [dict(pattern="sliding", seq_len=n, band_width=4)]  # narrow band: Eq. 1 routes row-wise
    dm = sf.generate_mask(terms)
    plan = sf.select_plan(dm, sf.hw_preset("b200"), n, 2, 1, 64, mode="b200")
    assert plan.kind == "row_wise" and plan.threshold < 0
    ctx = sf.MhaContext(dm, plan)
    q, k, v = fp16_inputs(oracle, 1, 2, n, 64, 5)
    ref, _ = oracle.block_sparse_sdpa(q, k, v, oracle.mask(terms), 16, 16, threads=8)
    parity(sf.mha(*(to_dev(x, torch.float16) for x in (q, k, v)), ctx), ref)
    wide = sf.generate_mask([dict(pattern="bigbird", seq_len=1024, global_width=32, band_width=32,
                                  filling_rate=0.1, seed=0)])
    plan = sf.select_plan(wide, sf.hw_preset("b200"), 1024, 12, 16, 64, mode="b200")
    # BigBird's 16-row random blocks: 64-row blocks (head pairs) execute 0.67x the cells
    assert plan.kind == "block_wise" and (plan.block_m, plan.block_n) == (64, 16), plan
    causal = sf.generate_mask([dict(pattern="causal", seq_len=1024)])
    cp = sf.select_plan(causal, sf.hw_preset("b200"), 1024, 12, 16, 64, mode="b200")
    assert cp.kind == "block_wise" and cp.block_m == 128, cp  # causal: 0.94x the cells, slower as pairs


def test_b200_selector_calibration(sf):
    """Eq. 1 routes a 16-wide band at n = 2048 row-wise; the B200 mode keeps
    that verdict when the work is tiny but moves the full bs16 x 12-head problem block-wise, where
    the tcgen05 executor is predicted (and measured, profiles/r01) several times faster."""
    dm = sf.gen_sliding_window(2048, 16)
    ref = sf.select_plan(dm, sf.hw_preset("b200"), 2048, 12, 16, 64, mode="reference")
    assert ref.kind == "row_wise" and ref.threshold < 0
    b200 = sf.select_plan(dm, sf.hw_preset("b200"), 2048, 12, 16, 64, mode="b200")
    # block_m 64 (head pairs): a 16-wide band executes 0.60x the cells of 128-row blocks
    assert b200.kind == "block_wise" and (b200.block_m, b200.block_n) == (64, 16)
    assert b200.threshold == ref.threshold
    small = sf.select_plan(sf.gen_sliding_window(2048, 4), sf.hw_preset("b200"), 2048, 2, 1, 64, mode="b200")
    assert small.kind == "row_wise"
    # the other direction: an unstructured low-density mask loads nearly every (128,16) tile but
    # leaves it nearly empty; Eq. 1 says block-wise, the B200 model keeps the row-wise gather
    # (measured 60 vs 178 us at this shape, profiles/r02/band_sweep_v3.jsonl)
    rnd = sf.gen_random_blocks(2048, 1, 0.002, 7)
    assert sf.select_plan(rnd, sf.hw_preset("b200"), 2048, 12, 8, 64, mode="reference").kind == "block_wise"
    assert sf.select_plan(rnd, sf.hw_preset("b200"), 2048, 12, 8, 64, mode="b200").kind == "row_wise"


def test_dynamic_schedule_graph_replay_and_streams(sf, oracle):
    """The tcgen05 kernel's work counter (per stream, reset by the last CTA): a skewed mask
    (global rows ~ all columns, the rest a narrow dilated band, like cfg4) replayed many times from
    one captured graph, eager launches on two streams, and empty row blocks at the end of the
    longest-first order must all give the oracle's result."""
    import torch
    bs, h, n, d = 2, 5, 1024, 64
    terms = [dict(pattern="dilated", seq_len=n, band_width=16, dilation_rate=1),
             dict(pattern="global", seq_len=n, global_width=32)]
    m = oracle.mask(terms)
    q, k, v = fp16_inputs(oracle, bs, h, n, d, 21)
    ref, _ = oracle.block_sparse_sdpa(q, k, v, m, 128, 16)
    qd, kd, vd = (to_dev(x, torch.float16) for x in (q, k, v))
    b = sf.build_bsr(sf.generate_mask(terms), 128, 16)
    for s in (torch.cuda.Stream(), torch.cuda.Stream()):  # eager, two streams
        with torch.cuda.stream(s):
            for _ in range(3):
                out = sf.block_sparse_sdpa(qd, kd, vd, b, stream=s)
        s.synchronize()
        parity(out, ref)
    s = torch.cuda.Stream()  # first seen inside the capture: its counter comes from the pool
    out = torch.zeros_like(qd)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sf.block_sparse_sdpa(qd, kd, vd, b, out=out, stream=s)
    for _ in range(10):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        parity(out, ref)
    # rows beyond a short mask's last valid row block: empty row blocks come last in the order
    mask_e = np.zeros((n, n), np.uint8)
    mask_e[: n // 4, : n // 2] = 1
    ref_e, _ = oracle.block_sparse_sdpa(q, k, v, mask_e, 128, 16)
    be = sf.build_bsr(sf.DenseMask.from_numpy(mask_e), 128, 16)
    for _ in range(3):
        parity(sf.block_sparse_sdpa(qd, kd, vd, be), ref_e)


@pytest.mark.parametrize("terms,n", [([dict(pattern="bigbird", seq_len=512, global_width=22, band_width=22,
                                            filling_rate=0.1, seed=3)], 512),
                                     ([dict(pattern="strided", seq_len=384, band_width=19)], 384),
                                     ([dict(pattern="random", seq_len=256, block=16, filling_rate=0.05, seed=2)], 256)])
def test_device_dense_oracle_matches_reference(sf, oracle, terms, n):
    """sf_mha_dense_oracle (attention.hpp:15-56 on the device, fp64) equals the reference's
    dense_sdpa_oracle restated in oracle/ on the same fp16-rounded inputs to fp64 rounding, and
    keeps fully masked rows exactly zero."""
    import torch
    m = oracle.mask(terms)
    q, k, v = fp16_inputs(oracle, 2, 3, n, 64, 11)
    ref = oracle.dense_sdpa(q, k, v, m)
    dm = sf.generate_mask(terms)
    got = sf.dense_sdpa_oracle(to_dev(q, torch.float16), to_dev(k, torch.float16), to_dev(v, torch.float16), dm)
    got = got.cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-9
    empty = ~m.any(axis=1)
    assert np.all(got[:, :, empty, :] == 0.0)


@pytest.mark.parametrize("n,w,bs,h", [(2048, 45, 8, 12), (2048, 45, 2, 12), (512, 22, 2, 3), (1000, 31, 1, 4),
                                     (8192, 90, 1, 2)])
def test_strided_decomposition_matches_oracle(sf, oracle, n, w, bs, h):
    """sf_mha_strided (causal-local band on the tcgen05 kernel + per-residue-class dense causal
    attention, merged by log-sum-exp) against the oracle's block_sparse_sdpa over the strided mask
    (attention.hpp:71-172): the decomposition changes the executor, not the result."""
    import torch
    terms = [dict(pattern="strided", seq_len=n, band_width=w)]
    m = oracle.mask(terms)
    q, k, v = (x.astype(np.float16).astype(np.float32) for x in oracle.random_attention_input(bs, h, n, 64, 3))
    ref, _ = oracle.block_sparse_sdpa(q, k, v, m, 128, 16, threads=os.cpu_count() or 8)
    assert sf.strided_band(terms) == (w if n >= 2048 else None)
    band = sf.generate_mask([dict(pattern="causal_local", seq_len=n, band_width=w)])
    bb = sf.build_bsr(band, 128, 16)
    dev = lambda x: torch.from_numpy(x).to("cuda", torch.float16)
    out = sf.strided_sdpa(dev(q), dev(k), dev(v), w, bb).float().cpu().numpy()
    d = np.abs(out - ref)
    assert d.max() <= 2e-2 and d.sum() / np.abs(ref).sum() <= 1e-3, (d.max(), d.sum() / np.abs(ref).sum())
    # through the unified MHA entry with a context that carries the band
    dm = sf.generate_mask(terms)
    plan = sf.select_plan(dm, sf.hw_preset("b200"), n, h, bs, 64, mode="b200")
    ctx = sf.MhaContext(dm, plan, strided_band=w)
    out2 = sf.mha(dev(q), dev(k), dev(v), ctx).float().cpu().numpy()
    # the context runs the band part on head pairs (block_m 64 band BSR)
    out3 = sf.strided_sdpa(dev(q), dev(k), dev(v), w, sf.build_bsr(band, 64, 16)).float().cpu().numpy()
    assert np.abs(out2 - out3).max() == 0.0
    d3 = np.abs(out3 - ref)
    assert d3.max() <= 2e-2 and d3.sum() / np.abs(ref).sum() <= 1e-3, (d3.max(), d3.sum() / np.abs(ref).sum())


@pytest.mark.parametrize("n,bs,h,dtype", [(1000, 3, 4, "f16"), (1000, 1, 6, "bf16"), (776, 2, 2, "f16")])
def test_head_pair_boxes_ragged(sf, oracle, monkeypatch, n, bs, h, dtype):
    """Head pairs (block_m 64) with the two-head 5-D K/V boxes (even head count, n % 8 == 0) at row
    counts that are not a multiple of the 64-row block, f16 and bf16, against the oracle; the
    one-box-per-head path (SF_ATTN_PAIR5=0) gives the same bits."""
    import torch
    terms = [dict(pattern="bigbird", seq_len=n, global_width=20, band_width=20, filling_rate=0.1, seed=3)]
    m = oracle.mask(terms)
    q, k, v = fp16_inputs(oracle, bs, h, n, 64, 9)
    ref, _ = oracle.block_sparse_sdpa(q, k, v, m, 64, 16, threads=8)
    b = sf.build_bsr(sf.generate_mask(terms), 64, 16)
    dt = torch.float16 if dtype == "f16" else torch.bfloat16
    sf.set_attn_impl("tcgen05")
    try:
        out = sf.block_sparse_sdpa(to_dev(q, dt), to_dev(k, dt), to_dev(v, dt), b)
        if dtype == "f16":
            parity(out, ref)
        else:
            parity(out, ref, max_abs=6e-2, mean_rel=6e-3)
        monkeypatch.setenv("SF_ATTN_PAIR5", "0")
        out1 = sf.block_sparse_sdpa(to_dev(q, dt), to_dev(k, dt), to_dev(v, dt), b)
        assert torch.equal(out, out1)
    finally:
        sf.set_attn_impl("auto")


def test_long_sequences_keep_block_m_128(sf):
    """Past n = 8192 the head-pair tile would exceed the tcgen05 kernel's 128 row blocks: the
    selector keeps block_m 128 there and the strided context keeps a block_m 128 band; the
    decomposed strided executor at n = 16384 agrees with the block executor over the whole mask."""
    import torch
    n, w = 16384, 128
    bb = sf.gen_bigbird(n, 128, 128, 0.1, 0)
    plan = sf.select_plan(bb, sf.hw_preset("b200"), n, 12, 1, 64, mode="b200")
    assert plan.kind == "block_wise" and plan.block_m == 128, plan
    terms = [dict(pattern="strided", seq_len=n, band_width=w)]
    dm = sf.generate_mask(terms)
    ctx = sf.context_for(terms, dm, sf.KernelPlan("block_wise", 128, 16))
    assert ctx.strided_band == w and ctx.band_bsr.dev.block_m == 128
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = ((torch.rand(1, 2, n, 64, device="cuda", generator=g) * 2 - 1).half() for _ in range(3))
    out = sf.mha(q, k, v, ctx)
    sf.set_attn_impl("tcgen05")
    try:
        ref = sf.block_sparse_sdpa(q, k, v, sf.build_bsr(dm, 128, 16))
    finally:
        sf.set_attn_impl("auto")
    d = (out.float() - ref.float()).abs()
    assert d.max().item() <= 2e-2 and (d.sum() / ref.float().abs().sum()).item() <= 1e-3
