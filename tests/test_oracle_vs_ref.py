"""Pin the C restatement (oracle/sf_oracle.c) against the reference itself (oracle/_ref, the
unmodified headers compiled in place). CPU only. Mirrors the reference's own test strategy:
test_mask.cpp predicates/sparsities, test_bsr.cpp 1000-case round trip (seed 2024),
test_planner.cpp 50 random argmax cases (seed 2025), test_attention.cpp executor cases."""
import math

import numpy as np
import pytest

from oracle.oracle import CONFIG_MASKS, HwSpec, make_desc


def _rng_masks(seed, count, nmax=96):
    rng = np.random.default_rng(seed)
    for _ in range(count):
        n = int(rng.integers(1, nmax + 1))
        bm = int(rng.integers(1, 25))
        bn = int(rng.integers(1, 25))
        dens = float(rng.random())
        yield n, bm, bn, (rng.random((n, n)) < dens).astype(np.uint8)


REF_PATTERNS = [
    [dict(pattern="sliding", seq_len=37, band_width=5)],
    [dict(pattern="dilated", seq_len=41, band_width=4, dilation_rate=2)],
    [dict(pattern="dilated", seq_len=8, band_width=2, dilation_rate=1)],
    [dict(pattern="global", seq_len=50, global_width=7)],
    [dict(pattern="random", seq_len=100, block=16, filling_rate=0.3, seed=11)],
    [dict(pattern="random", seq_len=97, block=5, filling_rate=0.5, seed=3)],
    [dict(pattern="longformer", seq_len=96, global_width=8, band_width=8)],
    [dict(pattern="bigbird", seq_len=100, global_width=10, band_width=10, filling_rate=0.2, seed=7)],
    [dict(pattern="bigbird", seq_len=1024, global_width=32, band_width=32, filling_rate=0.1, seed=3)],
    [dict(pattern="sliding", seq_len=64, band_width=8), dict(pattern="global", seq_len=64, global_width=3)],
]


@pytest.mark.parametrize("terms", REF_PATTERNS)
def test_masks_equal_reference(oracle, reference, terms):
    assert (oracle.mask(terms) == reference.mask(terms)).all()


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg4"])
def test_config_masks_equal_reference(oracle, reference, cfg):
    assert (oracle.mask(CONFIG_MASKS[cfg]) == reference.mask(CONFIG_MASKS[cfg])).all()


def test_published_sparsities(oracle):
    # test_mask.cpp:20-23,60-62,122-125,131-136 (Table 2 of the paper)
    def sp(terms):
        m = oracle.mask(terms)
        return 1.0 - m.sum() / m.size
    assert abs(sp([dict(pattern="sliding", seq_len=1024, band_width=32)]) - 0.938) <= 0.005
    assert abs(sp([dict(pattern="dilated", seq_len=1024, band_width=32, dilation_rate=1)]) - 0.938) <= 0.015
    assert abs(sp([dict(pattern="longformer", seq_len=1024, global_width=32, band_width=32)]) - 0.888) <= 0.015


def test_bsr_random_round_trip_bytes_equal_reference(oracle, reference):
    # test_bsr.cpp:65-84 shape distribution; SFBR bytes must be identical (pool order included)
    for n, bm, bn, m in _rng_masks(2024, 300):
        ob = oracle.bsr(m, bm, bn)
        rb, _ = reference.sfbr(m, bm, bn)
        assert ob["sfbr"] == rb, (n, bm, bn)


@pytest.mark.parametrize("cfg", list(CONFIG_MASKS))
@pytest.mark.parametrize("tile", [(16, 16), (64, 16), (128, 16), (128, 64)])
def test_config_bsr_bytes_equal_reference(oracle, reference, cfg, tile):
    m = oracle.mask(CONFIG_MASKS[cfg])
    assert oracle.bsr(m, *tile)["sfbr"] == reference.sfbr(m, *tile)[0]


def test_rowwise_equal_reference(oracle, reference):
    for n, _, _, m in _rng_masks(7, 50, 80):
        rp, ci = oracle.rowwise(m)
        rr, rc = reference.rowwise(m)
        assert (rp == rr).all() and (ci == rc).all()


def test_random_attention_input_equal_reference(oracle, reference):
    a = oracle.random_attention_input(2, 3, 17, 8, 5)
    b = reference.random_attention_input(2, 3, 17, 8, 5)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("terms,bm,bn,d", [
    ([dict(pattern="sliding", seq_len=64, band_width=8)], 16, 16, 16),
    ([dict(pattern="dilated", seq_len=64, band_width=8, dilation_rate=1)], 16, 32, 16),
    ([dict(pattern="bigbird", seq_len=100, global_width=10, band_width=10, filling_rate=0.2, seed=7)], 16, 16, 16),
    ([dict(pattern="longformer", seq_len=96, global_width=8, band_width=8)], 32, 16, 16),
    ([dict(pattern="sliding", seq_len=512, band_width=22)], 128, 16, 64),
])
def test_block_sparse_sdpa_bitwise_equal_reference(oracle, reference, terms, bm, bn, d):
    m = oracle.mask(terms)
    n = m.shape[0]
    q, k, v = oracle.random_attention_input(2, 2, n, d, 11)
    o1, s1 = oracle.block_sparse_sdpa(q, k, v, m, bm, bn)
    o2, s2 = reference.block_sparse_sdpa(q, k, v, m, bm, bn)
    assert np.array_equal(o1, o2)
    assert np.array_equal(s1, s2)


def test_rowwise_and_dense_match_reference(oracle, reference):
    m = oracle.mask([dict(pattern="bigbird", seq_len=64, global_width=8, band_width=8, filling_rate=0.15, seed=23)])
    q, k, v = (x.astype(np.float64) for x in oracle.random_attention_input(2, 2, 64, 16, 29))
    ro = oracle.rowwise_sdpa(q, k, v, m)
    do = oracle.dense_sdpa(q, k, v, m)
    import ctypes as C
    out = np.zeros_like(q)
    P = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    reference.lib.ref_rowwise_sdpa(P(q), P(k), P(v), 2, 2, 64, 16, m.ctypes.data_as(C.POINTER(C.c_uint8)), P(out))
    assert np.max(np.abs(ro - out)) <= 1e-12
    reference.lib.ref_dense_sdpa(P(q), P(k), P(v), 2, 2, 64, 16, m.ctypes.data_as(C.POINTER(C.c_uint8)), P(out))
    assert np.max(np.abs(do - out)) <= 1e-12
    assert np.max(np.abs(ro - do)) <= 1e-6  # test_attention.cpp:89-97


def test_select_plan_equals_reference_random_cases(oracle, reference):
    # test_planner.cpp:134-160 distribution (numpy RNG here; the argmax must agree exactly)
    rng = np.random.default_rng(2025)
    for _ in range(50):
        hw = HwSpec(b"rand", int(20 + rng.integers(120)), int((32 + rng.integers(224)) * 1024),
                    int([32, 48, 64][rng.integers(3)]), int(2 if rng.integers(2) else 4))
        seq = int([64, 128, 256, 512][rng.integers(4)])
        h = int(1 + rng.integers(16)); bs = int(1 + rng.integers(16)); head = int([16, 32, 64, 128][rng.integers(4)])
        m = oracle.mask([dict(pattern="random", seq_len=seq, block=16, filling_rate=0.3 + 0.7 * rng.random(),
                              seed=int(rng.integers(1 << 62)))])
        loads = oracle.bsr(m, 16, 16)["load_row_ptr"][-1]
        p1 = oracle.select_plan_from_loads(int(loads), hw, seq, h, bs, head)
        p2 = reference.select_plan(m, hw, seq, h, bs, head)
        assert (p1.kind, p1.block_m, p1.block_n, p1.num_warps, p1.fallback) == \
               (p2.kind, p2.block_m, p2.block_n, p2.num_warps, p2.fallback)
        assert p1.score == p2.score
        assert (math.isnan(p1.threshold) and math.isnan(p2.threshold)) or p1.threshold == p2.threshold


@pytest.mark.parametrize("cfg", list(CONFIG_MASKS))
@pytest.mark.parametrize("preset", ["a100", "rtx4090"])
def test_config_plans_equal_reference(oracle, reference, cfg, preset):
    m = oracle.mask(CONFIG_MASKS[cfg])
    n = m.shape[0]
    hw = oracle.hw_preset(preset)
    bs = {"cfg1": 1, "cfg2": 16, "cfg3": 8, "cfg4": 8}[cfg]
    loads = int(oracle.bsr(m, 16, 16)["load_row_ptr"][-1])
    p1 = oracle.select_plan_from_loads(loads, hw, n, 12, bs, 64)
    p2 = reference.select_plan(m, hw, n, 12, bs, 64)
    assert (p1.kind, p1.block_m, p1.block_n, p1.num_warps) == (p2.kind, p2.block_m, p2.block_n, p2.num_warps)
    assert p1.threshold == p2.threshold and p1.score == p2.score


def test_graph_params_restated(oracle, reference):
    # GraphData::make seeds (backend.hpp:65-106): input, Gemm W, Bias, LN gamma/beta, Add aux
    args = ("bert-layer", 1, 16, 64, 2, 32, 1)
    rows, hid, ff = 16, 64, 256
    inp = reference.graph_param(*args, 0, 0)
    assert np.array_equal(inp, oracle.random_matrix(rows, hid, oracle.mix_seed(1, 0xa11)).ravel())
    w = reference.graph_param(*args, 1, 1)
    a = 1.0 / np.sqrt(np.float32(hid))
    assert np.array_equal(w, oracle.random_matrix(hid, hid, oracle.mix_seed(1, 1), -a, a).ravel())
    aux = reference.graph_param(*args, 3, 5)
    assert np.array_equal(aux, oracle.random_matrix(rows, hid, oracle.mix_seed(1, 3)).ravel())


@pytest.mark.parametrize("model", ["bert-layer", "gpt-layer", "t5-layer"])
def test_chain_oracle_equals_reference_run_chain(oracle, reference, model):
    """The composed per-op oracle chain reproduces CpuBackend::run_chain (backend.hpp:430-441)."""
    from tests.chain_oracle import graph_data, run_chain
    bs, seq, hid, heads, hs = 1, 64, 64, 2, 32
    m = oracle.mask([dict(pattern="bigbird", seq_len=seq, global_width=8, band_width=8, filling_rate=0.2, seed=3)])
    gd = graph_data(oracle, model, bs, seq, hid, 4 * hid, 1)
    ours = run_chain(oracle, model, gd, gd["input"], m, bs, seq, heads, hs, 16, 16, threads=1)
    ref = reference.run_chain(model, bs, seq, hid, heads, hs, 1, m, 16, 16)
    assert np.max(np.abs(ours - ref)) <= 1e-5, np.max(np.abs(ours - ref))


def test_sfmk_format_restatement_matches_reference(reference):
    """The SFMK dump the GPU tests check against (header + LSB-first n*n bits, io.hpp:61-76) is
    byte-identical to the reference's write_dense_mask, ragged sizes included."""
    import numpy as np
    for n in (1, 7, 33, 300, 1024):
        m = (np.random.default_rng(n).random((n, n)) < 0.3).astype(np.uint8)
        restated = b"SFMK" + np.array([1, n, 0], np.uint32).tobytes() + np.packbits(m.flatten(), bitorder="little").tobytes()
        assert reference.sfmk(m) == restated
