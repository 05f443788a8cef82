"""The C++ host API (include/sparsefuse_b200/) driven through tests/cpp/host_api_test.

* search parity (CPU): the two-stage search over the SyntheticBackend must take exactly the
  reference's decisions (oracle/_ref: the reference's own run_pipeline) — scheme code, per-segment
  settings and durations, end-to-end time and every search counter.
* gpu-basics / gpu-backend (GPU): the reference test-suite cases through the drop-in C++ API, and
  the B200 MeasurementBackend (device-executed segments, CUDA-event timing) driving the search.
"""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "tests" / "cpp" / "_bin" / "host_api_test"


def _bin():
    if not BIN.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "tests" / "cpp")], check=True)
    return str(BIN)


CASES = [("bert-layer", 1, 128, 11, 0, 0), ("bert-layer", 16, 1024, 3, 7, 0), ("gpt-layer", 8, 2048, 5, 1, 0),
         ("t5-layer", 8, 4096, 9, 2, 0), ("bert-layer", 2, 512, 13, 4, 1), ("gpt-layer", 1, 256, 21, 3, 1),
         ("t5-layer", 4, 1024, 1, 9, 0)]


@pytest.mark.parametrize("case", CASES)
def test_search_decisions_match_reference(reference, case):
    model, bs, seq, mseed, cseed, planted = case
    ours = subprocess.run([_bin(), "search", model, str(bs), str(seq), str(mseed), str(cseed), str(planted)],
                          capture_output=True, text=True, check=True).stdout.strip()
    ref = reference.run_pipeline_synthetic(model, bs, seq, mseed, cseed, bool(planted))
    assert ours == ref


@pytest.mark.parametrize("case", [("bert-layer", 16, 1024, 3, 7), ("t5-layer", 8, 4096, 9, 2)])
def test_tuning_cache_files_are_interchangeable(reference, tmp_path, case):
    """io.hpp:407-458: a cache file written by either implementation warms the other exactly like
    its own (same decisions, durations and cache-hit counters), and a cold session's report is the
    same in both."""
    model, bs, seq, ms, cs = case
    ours_f, ref_f = str(tmp_path / "ours.jsonl"), str(tmp_path / "ref.jsonl")

    def ours(pin, pout):
        return subprocess.run([_bin(), "cache", model, str(bs), str(seq), str(ms), str(cs), pin or "-", pout or "-"],
                              capture_output=True, text=True, check=True).stdout.strip()

    cold_ours, cold_ref = ours("", ours_f), reference.cache_session(model, bs, seq, ms, cs, "", ref_f)
    assert cold_ours == cold_ref
    warm_ref_own = reference.cache_session(model, bs, seq, ms, cs, ref_f, "")
    assert reference.cache_session(model, bs, seq, ms, cs, ours_f, "") == warm_ref_own
    assert ours(ref_f, "") == ours(ours_f, "") == warm_ref_own
    assert warm_ref_own != cold_ref  # the warm session really was served from the file


@pytest.mark.gpu
def test_cpp_api_reference_cases_on_gpu():
    r = subprocess.run([_bin(), "gpu-basics"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "gpu-basics ok" in r.stdout


@pytest.mark.gpu
def test_gpu_measurement_backend_drives_the_search():
    r = subprocess.run([_bin(), "gpu-backend"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "gpu-backend ok" in r.stdout


SEGMENT_CASES = [  # (graph, segment, template) at bs 2, seq 256, hidden 256, 4 heads x 64
    ("bert-layer", (1, 2), "CiMi: out-projection GEMM"),
    ("bert-layer", (1, 5), "CiMi: GEMM + bias + residual + LayerNorm"),
    ("bert-layer", (5, 12), "CiCi: FFN1 + GELU -> FFN2 + bias + residual + LayerNorm"),
    ("gpt-layer", (0, 1), "MiChain: LayerNorm"),
    ("t5-layer", (6, 12), "CiCi: FFN with ReLU"),
    ("spec:g512,b,s", (0, 3), "CiMi + Softmax row op"),
    ("spec:b,e,a,s", (0, 4), "MiChain ending in Softmax"),
    ("spec:l,g256,b,r", (0, 4), "CiMi with a LayerNorm prologue"),
    ("bert-layer", (0, 1), "MhaFused unit (exec_mha), BigBird mask, BSR 128x16"),
    ("bert-layer", (0, 1), "MhaFused unit (exec_mha), strided(16) mask, decomposed executor"),
    ("t5-layer", (1, 2), "MhaFused unit (exec_mha), dilated(16,1)+global(16) mask, class decomposition"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("model,seg,what", SEGMENT_CASES)
def test_exec_segment_matches_reference(reference, tmp_path, model, seg, what):
    """exec_segment / exec_mha through the C++ host API (include/sparsefuse_b200/gpu_backend.hpp,
    reference signatures, host Matrix in / out, executed by the sm_100a templates) against the
    reference's own exec_segment (backend.hpp:360-385) on the same GraphData seeds and input.
    Bar: the north-star fp16 tolerance (max-abs 2e-2, mean-rel 1e-3) vs the fp32 reference."""
    import numpy as np
    bs, seq, hid, heads, hs, seed = 2, 256, 256, 4, 64, 5
    rng = np.random.default_rng(11)
    in_cols, out_cols = _seg_widths(model, seg, hid)
    x = (rng.random((bs * seq, in_cols), np.float32) * 2 - 1).astype(np.float16).astype(np.float32)
    mask = None
    extra = []
    if "Mha" in what:
        from oracle.oracle import Oracle
        if "strided" in what:
            terms, tail = [dict(pattern="strided", seq_len=seq, band_width=16)], ["16"]
        elif "dilated" in what:
            terms = [dict(pattern="dilated", seq_len=seq, band_width=16, dilation_rate=1),
                     dict(pattern="global", seq_len=seq, global_width=16)]
            tail = ["dil:16:1"]
        else:
            terms = [dict(pattern="bigbird", seq_len=seq, global_width=16, band_width=16, filling_rate=0.1, seed=2)]
            tail = []
        mask = Oracle().mask(terms)
        (tmp_path / "m.u8").write_bytes(mask.astype(np.uint8).tobytes())
        extra = [str(tmp_path / "m.u8"), "128", "16"] + tail
    (tmp_path / "x.f32").write_bytes(x.tobytes())
    r = subprocess.run([_bin(), "exec-segment", model, str(bs), str(seq), str(hid), str(heads), str(hs), str(seed),
                        str(seg[0]), str(seg[1]), str(tmp_path / "x.f32"), str(tmp_path / "y.f32")] + extra,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    ours = np.frombuffer((tmp_path / "y.f32").read_bytes(), np.float32).reshape(bs * seq, out_cols)
    ref = reference.exec_segment(model, bs, seq, hid, heads, hs, seed, seg, x, out_cols, mask=mask, tile=(128, 16))
    d = np.abs(ours.astype(np.float64) - ref)
    ma, mr = float(d.max()), float(d.sum() / np.abs(ref).sum())
    assert ma <= 2e-2 and mr <= 1e-3, (what, ma, mr)


def _seg_widths(model, seg, hid):
    """(input width of node seg[0], output width of node seg[1]-1) for presets / spec graphs."""
    if model.startswith("spec:"):
        w, ws = hid, []
        for tok in model[5:].split(","):
            wi = w
            if tok[0] == "g":
                w = int(tok[1:])
            ws.append((wi, w))
    else:
        ff = 4 * hid
        kinds = {"bert-layer": ["m", "g", "b", "a", "l", "g4", "b4", "e4", "g", "b", "a", "l"],
                 "gpt-layer": ["l", "m", "g", "b", "a", "l", "g4", "b4", "e4", "g", "b", "a"]}
        kinds["t5-layer"] = kinds["gpt-layer"]
        ws = []
        w = hid
        for k in kinds[model]:
            wi = w
            if k == "g4":
                w = ff
            elif k == "g":
                w = hid
            ws.append((wi, w))
    return ws[seg[0]][0], ws[seg[1] - 1][1]
