"""Device mask generation and format builders are bit-exact with the reference (via the pinned
C oracle and the reference-generated golden fixtures)."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import CONFIG_MASKS

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"
FP = json.loads((G / "fingerprints.json").read_text())

PATTERN_CASES = [
    [dict(pattern="sliding", seq_len=37, band_width=5)],
    [dict(pattern="sliding", seq_len=4, band_width=4)],
    [dict(pattern="sliding", seq_len=8, band_width=1)],
    [dict(pattern="dilated", seq_len=41, band_width=4, dilation_rate=2)],
    [dict(pattern="dilated", seq_len=8, band_width=2, dilation_rate=1)],
    [dict(pattern="dilated", seq_len=300, band_width=17, dilation_rate=0)],
    [dict(pattern="global", seq_len=50, global_width=7)],
    [dict(pattern="global", seq_len=33, global_width=0)],
    [dict(pattern="random", seq_len=100, block=16, filling_rate=0.3, seed=11)],
    [dict(pattern="random", seq_len=97, block=5, filling_rate=0.5, seed=3)],
    [dict(pattern="random", seq_len=1000, block=1, filling_rate=0.25, seed=9)],  # > 312 draws per twist, many twists
    [dict(pattern="longformer", seq_len=96, global_width=8, band_width=8)],
    [dict(pattern="bigbird", seq_len=100, global_width=10, band_width=10, filling_rate=0.2, seed=7)],
    [dict(pattern="causal", seq_len=70)],
    [dict(pattern="causal_local", seq_len=70, band_width=9)],
    [dict(pattern="strided", seq_len=130, band_width=11)],
    [dict(pattern="sliding", seq_len=64, band_width=8), dict(pattern="global", seq_len=64, global_width=3)],
]


@pytest.mark.parametrize("terms", PATTERN_CASES)
def test_device_mask_equals_oracle(sf, oracle, terms):
    dm = sf.generate_mask(terms)
    assert np.array_equal(dm.to_numpy(), oracle.mask(terms))
    assert dm.true_count() == int(oracle.mask(terms).sum())


@pytest.mark.parametrize("cfg", list(CONFIG_MASKS))
def test_config_masks_and_formats_match_golden(sf, oracle, cfg):
    dm = sf.generate_mask(CONFIG_MASKS[cfg])
    ent = FP[cfg]
    assert dm.true_count() == ent["true_count"]
    rw = sf.build_rowwise(dm)
    rp, ci = rw.to_host()
    assert len(ci) == ent["rowwise_nnz"]
    assert "%016x" % oracle.fnv1a(rp.tobytes() + ci.tobytes()) == ent["rowwise_fnv"]
    for tile, t in ent["tiles"].items():
        bm, bn = map(int, tile.split("x"))
        b = sf.build_bsr(dm, bm, bn)
        s = sf.block_stats(b)
        assert (s.full_count, s.part_count, s.empty_count, b.n_pool) == (t["full"], t["part"], t["empty"], t["pool"])
        assert "%016x" % oracle.fnv1a(b.sfbr()) == t["fnv"], (cfg, tile)


def test_small_bsr_dumps_match_golden(sf):
    z = np.load(G / "bsr_small.npz")
    for i in range(24):
        n, bm, bn = (int(x) for x in z[f"{i}/shape"])
        m = np.unpackbits(z[f"{i}/mask"], bitorder="little")[: n * n].reshape(n, n)
        b = sf.build_bsr(sf.DenseMask.from_numpy(m), bm, bn)
        assert b.sfbr() == z[f"{i}/sfbr"].tobytes(), (i, n, bm, bn)


def test_randomized_round_trip_1000(sf, oracle):
    # test_bsr.cpp:65-84: 1000 random masks, n <= 96, bm, bn <= 24 — device bytes == oracle bytes,
    # validate_bsr passes and to_dense(build_bsr(m)) == m, all on the device
    rng = np.random.default_rng(2024)
    for it in range(1000):
        n = int(rng.integers(1, 97)); bm = int(rng.integers(1, 25)); bn = int(rng.integers(1, 25))
        m = (rng.random((n, n)) < rng.random()).astype(np.uint8)
        b = sf.build_bsr(sf.DenseMask.from_numpy(m), bm, bn)
        assert b.sfbr() == oracle.bsr(m, bm, bn)["sfbr"], (it, n, bm, bn)
        sf.validate_bsr(b)
        assert np.array_equal(sf.to_dense(b).to_numpy(), m), (it, n, bm, bn)
        if it % 50 == 0:  # host arrays -> device copy -> to_dense (read_bsr-style masks)
            h = sf.bsr_from_host(b.to_host(), n, bm, bn)
            assert h.sfbr() == b.sfbr()
            assert np.array_equal(sf.to_dense(h).to_numpy(), m)


def _corruptions(a, n_cols, n_pool):
    """(name, corrupted copy) pairs over a built BSR's host arrays; each breaks one invariant."""
    def cp():
        return {k: np.array(v, copy=True) for k, v in a.items()}
    out = []
    if len(a["full_col_idx"]):
        c = cp(); c["full_col_idx"][0] = n_cols; out.append(("full col out of range", c))
        c = cp(); fr = c["full_row_ptr"]; r = int(np.argmax(np.diff(fr) >= 1)); fr[r + 1] = fr[r] - 1
        out.append(("full row_ptr decreasing", c))
    if (np.diff(a["part_row_ptr"]) >= 2).any():
        c = cp(); r = int(np.argmax(np.diff(c["part_row_ptr"]) >= 2)); k = int(c["part_row_ptr"][r])
        c["part_col_idx"][[k, k + 1]] = c["part_col_idx"][[k + 1, k]]; out.append(("part cols unordered", c))
    if len(a["part_tile_ids"]):
        c = cp(); c["part_tile_ids"][0] = n_pool; out.append(("tile id past pool", c))
        c = cp(); c["part_mask_pool"] = c["part_mask_pool"].copy(); c["part_mask_pool"][0][:] = 1
        out.append(("pool tile all ones", c))
    c = cp(); lc = c["load_col_idx"]; lr = c["load_row_ptr"]
    for r in range(len(lr) - 1):  # shift one load column to a free neighbour, keeping order
        row = lc[lr[r]:lr[r + 1]]
        if len(row) and row[-1] + 1 < n_cols:
            row[-1] += 1
            break
    out.append(("load not the union", c))
    c = cp(); c["load_row_ptr"][-1] += 1; out.append(("load_row_ptr.back() + 1 (test_bsr.cpp:94-98)", c))
    return out


@pytest.mark.parametrize("terms,tile", [([dict(pattern="bigbird", seq_len=256, global_width=16, band_width=16,
                                               filling_rate=0.2, seed=3)], (16, 16)),
                                        ([dict(pattern="sliding", seq_len=64, band_width=8)], (16, 16)),
                                        ([dict(pattern="dilated", seq_len=200, band_width=24, dilation_rate=2)], (32, 8))])
def test_validate_bsr_rejects_corruptions_like_the_reference(sf, oracle, reference, terms, tile):
    """validate_bsr / to_dense on corrupted structures (test_bsr.cpp:94-98): the device check raises
    InternalInconsistency with the same message the reference's validate_bsr throws."""
    from paper_2506_06095_b200 import _lib
    dm = sf.generate_mask(terms)
    n = dm.seq_len
    b = sf.build_bsr(dm, *tile)
    a = b.to_host()
    a.pop("pool_packed")
    assert reference.validate_bsr(n, *tile, a) == (0, "")
    for name, c in _corruptions(a, b.n_cols, b.n_pool):
        st, msg = reference.validate_bsr(n, *tile, c)
        assert st == 6, name  # SF_INTERNAL_INCONSISTENCY
        h = sf.bsr_from_host(c, n, *tile)
        with pytest.raises(_lib.InternalInconsistency) as e:
            sf.validate_bsr(h)
        with pytest.raises(_lib.InternalInconsistency):
            sf.to_dense(h)
        if "back() + 1" not in name:  # that one reads past the column array in the reference (UB)
            assert str(e.value) == msg, (name, str(e.value), msg)


def test_extremes_and_dedup(sf, oracle):
    # test_bsr.cpp:14-34, 86-92
    b = sf.build_bsr(sf.DenseMask.from_numpy(np.zeros((64, 64), np.uint8)), 16, 16)
    assert (b.n_full, b.n_part, b.n_load, b.n_pool) == (0, 0, 0, 0)
    b = sf.build_bsr(sf.DenseMask.from_numpy(np.ones((64, 64), np.uint8)), 16, 16)
    assert (b.n_full, b.n_part, b.n_pool) == (16, 0, 0)
    i, j = np.indices((64, 64))
    b = sf.build_bsr(sf.DenseMask.from_numpy((i % 8 == j % 8).astype(np.uint8)), 8, 8)
    assert b.n_part == 64 and b.n_pool == 1


@pytest.mark.parametrize("n,tile", [(8192, (16, 16)), (8192, (128, 16)), (4096, (128, 64))])
def test_large_masks_match_oracle(sf, oracle, n, tile):
    w = int(np.sqrt(n))
    terms = [dict(pattern="bigbird", seq_len=n, global_width=w, band_width=w, filling_rate=0.1, seed=5)]
    m = oracle.mask(terms)
    dm = sf.generate_mask(terms)
    assert np.array_equal(dm.to_numpy(), m)
    assert sf.build_bsr(dm, *tile).sfbr() == oracle.bsr(m, *tile)["sfbr"]


def test_parameter_errors(sf):
    with pytest.raises(sf._lib.InvalidParameter):
        sf.gen_sliding_window(16, 0)
    with pytest.raises(sf._lib.InvalidParameter):
        sf.gen_sliding_window(16, 17)
    with pytest.raises(sf._lib.InvalidParameter):
        sf.gen_dilated(16, 2, -1)
    with pytest.raises(sf._lib.InvalidParameter):
        sf.gen_random_blocks(16, 0, 0.5, 1)
    with pytest.raises(sf._lib.ShapeError):
        sf.generate_mask([dict(pattern="sliding", seq_len=16, band_width=2), dict(pattern="sliding", seq_len=8, band_width=2)])
    with pytest.raises(sf._lib.InvalidParameter):
        sf.build_bsr(sf.gen_sliding_window(16, 2), 0, 4)


def test_planner_matches_golden(sf):
    plans = json.loads((G / "plans.json").read_text())
    for key, e in plans.items():
        cfg, preset = key.split("/")
        dm = sf.generate_mask(CONFIG_MASKS[cfg])
        p = sf.select_plan(dm, sf.hw_preset(preset), dm.seq_len, 12, e["bs"], 64)
        assert (p.kind == "block_wise") == (e["kind"] == 1)
        assert (p.block_m, p.block_n, p.num_warps) == (e["block_m"], e["block_n"], e["num_warps"])
        assert p.score == e["score"] and p.threshold == e["threshold"]
    with pytest.raises(sf._lib.DegenerateInput):
        sf.threshold(sf.generate_mask(dict(pattern="sliding", seq_len=16, band_width=2)))


def _sfmk_restated(m):
    """write_dense_mask (io.hpp:66-76) restated: header + the n*n bits, row-major, LSB-first."""
    n = m.shape[0]
    return b"SFMK" + np.array([1, n, 0], np.uint32).tobytes() + np.packbits(m.flatten(), bitorder="little").tobytes()


@pytest.mark.parametrize("cfg", list(CONFIG_MASKS))
def test_sfmk_dump_matches_reference_bytes(sf, oracle, cfg):
    terms = CONFIG_MASKS[cfg]
    dm = sf.generate_mask(terms)
    got = dm.sfmk()
    assert got == _sfmk_restated(oracle.mask(terms))
    from oracle.oracle import Reference
    r = Reference()
    if r.available:  # the reference's own writer on the same mask bytes
        assert got == r.sfmk(dm.to_numpy())
    back = sf.DenseMask.from_sfmk(got)  # read_dense_mask round trip
    assert back.seq_len == dm.seq_len and np.array_equal(back.to_numpy(), dm.to_numpy())


@pytest.mark.parametrize("n", [1, 7, 33, 300, 1000, 2049])
def test_sfmk_round_trip_ragged(sf, n):
    m = (np.random.default_rng(n).random((n, n)) < 0.3).astype(np.uint8)
    dm = sf.DenseMask.from_numpy(m)
    data = dm.sfmk()
    assert data == _sfmk_restated(m)
    assert np.array_equal(sf.DenseMask.from_sfmk(data).to_numpy(), m)


def test_sfmk_errors(sf):
    data = sf.gen_sliding_window(64, 4).sfmk()
    with pytest.raises(sf._lib.IoError):
        sf.DenseMask.from_sfmk(b"SFBR" + data[4:])  # io.hpp:80 bad magic
    with pytest.raises(sf._lib.IoError):
        sf.DenseMask.from_sfmk(data[:4] + np.array([2], np.uint32).tobytes() + data[8:])  # :82 version
    with pytest.raises(sf._lib.IoError):
        sf.DenseMask.from_sfmk(data[:-1])  # :88 truncated


def test_async_build_equals_build_bsr(sf, oracle):
    """sf_bsr_build_async on a worst-case workspace (no host sync) yields the same SFBR bytes as
    sf_bsr_build, on random masks (test_bsr.cpp:65-84 shapes) and the BASELINE masks."""
    rng = np.random.default_rng(77)
    cases = []
    for _ in range(100):
        n = int(rng.integers(1, 97)); bm = int(rng.integers(1, 25)); bn = int(rng.integers(1, 25))
        cases.append(((rng.random((n, n)) < rng.random()).astype(np.uint8), bm, bn))
    for cfg in ("cfg2", "cfg3", "cfg4"):
        m = oracle.mask(CONFIG_MASKS[cfg])
        cases += [(m, 128, 16), (m, 16, 16)]
    for m, bm, bn in cases:
        dm = sf.DenseMask.from_numpy(m)
        ws = sf.BsrWorkspace(dm.seq_len, bm, bn).build_async(dm)
        assert ws.snapshot().sfbr() == sf.build_bsr(dm, bm, bn).sfbr(), (m.shape, bm, bn)


def test_async_build_inside_a_cuda_graph(sf):
    """Mask -> BSR -> attention captured as ONE graph; new mask bits written into the captured mask
    buffer take effect at the next replay (per-request masks without host round trips)."""
    import torch
    n, bs, h, d = 1024, 2, 4, 64
    masks = [sf.generate_mask([dict(pattern="bigbird", seq_len=n, global_width=32, band_width=32,
                                    filling_rate=0.1, seed=s)]) for s in (1, 2)]
    mbuf = sf.DenseMask(n, masks[0].bits.clone())
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = ((torch.rand(bs, h, n, d, device="cuda", generator=g) * 2 - 1).half() for _ in range(3))
    ws = sf.BsrWorkspace(n, 128, 16)
    out = torch.empty_like(q)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):  # warm on the capture stream (attention work counter)
        ws.build_async(mbuf, stream=st)
        sf.block_sparse_sdpa(q, k, v, ws, out=out, stream=st)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        ws.build_async(mbuf, stream=st)
        sf.block_sparse_sdpa(q, k, v, ws, out=out, stream=st)
    for m in masks + masks[:1]:
        mbuf.bits.copy_(m.bits)
        out.zero_()
        gr.replay()
        torch.cuda.synchronize()
        ref = sf.block_sparse_sdpa(q, k, v, sf.build_bsr(m, 128, 16))
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
        assert ws.counts.cpu().tolist()[2] == sf.build_bsr(m, 128, 16).n_load
