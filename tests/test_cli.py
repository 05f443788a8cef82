"""The `sparsefuse` CLI (SPEC.md cli module): JSON on stdout, exit codes 0 / 1 / 2. The codec
commands run anywhere; mask / plan / attention commands need the GPU."""
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_2506_06095_b200" / "_lib" / "sparsefuse"


def run(*args):
    if not CLI.exists():
        pytest.fail("sparsefuse CLI not built — run __graft_entry__.build()")
    r = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=300)
    return r.returncode, json.loads(r.stdout)


def test_fuse_codec_commands():
    rc, j = run("fuse", "decode", "0110")  # SPEC.md: segments [0],[1,2],[3]
    assert rc == 0 and j["segments"] == [[0, 1], [1, 3], [3, 4]]
    rc, j = run("fuse", "encode", "0-1,1-3,3-4")
    assert rc == 0 and j["code"] == "0110"


def test_usage_errors_exit_2():
    rc, j = run("mask", "nope")
    assert rc == 2 and j["error"] == "usage"


@pytest.mark.gpu
def test_mask_and_plan_commands(oracle, tmp_path):
    rc, j = run("mask", "gen", "--pattern", "sliding", "--seq-len", 1024, "--band", 32, "--dump", tmp_path / "m.sfmk")
    assert rc == 0 and abs(j["sparsity"] - 0.938) <= 0.005  # Table 2
    m = oracle.mask([dict(pattern="sliding", seq_len=1024, band_width=32)])
    rc, s = run("mask", "stats", "--sfmk", tmp_path / "m.sfmk", "--block", "16x16")
    b = oracle.bsr(m, 16, 16)
    assert rc == 0 and (s["full_count"], s["part_count"]) == (len(b["full_col_idx"]), len(b["part_col_idx"]))
    rc, p = run("plan", "select", "--sfmk", tmp_path / "m.sfmk", "--hw", "a100", "--heads", 12, "--bs", 8)
    assert rc == 0 and p["kind"] == "block_wise"


@pytest.mark.gpu
@pytest.mark.parametrize("pattern", [["--pattern", "sliding", "--band", 24], ["--pattern", "bigbird", "--band", 16,
                                                                               "--global", 16, "--fill", 0.1]])
def test_attn_verify_passes(pattern):
    """oracle vs block-wise vs row-wise on seeded inputs, errors and tile counts."""
    rc, j = run("attn", "verify", *pattern, "--seq-len", 512, "--bs", 1, "--heads", 2)
    assert rc == 0 and j["pass"] and j["tiles_loaded"] == j["valid_tiles"]
    assert j["oracle"].startswith("dense_sdpa_oracle") and j["fault_injected"] is None
    assert 0 < j["max_abs_blockwise"] <= 2e-2 and 0 < j["max_abs_rowwise"] <= 2e-2
    assert j["mean_rel_blockwise"] <= 1e-3 and j["mean_rel_rowwise"] <= 1e-3


@pytest.mark.gpu
def test_attn_verify_all_false_mask_is_zero_and_passes():
    """an all-false mask gives all-zero outputs (every executor and the oracle)."""
    rc, j = run("attn", "verify", "--pattern", "none", "--seq-len", 256, "--bs", 1, "--heads", 2)
    assert rc == 0 and j["pass"] and j["valid_tiles"] == 0
    assert j["max_abs_blockwise"] == 0 and j["max_abs_rowwise"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("pattern", [["--pattern", "sliding", "--band", 24],
                                     ["--pattern", "bigbird", "--band", 16, "--global", 16, "--fill", 0.1],
                                     ["--pattern", "none"]])
def test_attn_verify_injected_fault_fails(pattern):
    """injected-fault mode (one tile flipped) exits 1 with a diff report."""
    rc, j = run("attn", "verify", *pattern, "--seq-len", 512, "--bs", 1, "--heads", 2, "--inject-fault", "tile")
    assert rc == 1 and not j["pass"] and j["fault_injected"]
    assert j["diff"]["executor"] == "block_wise" and j["max_abs_blockwise"] > 2e-2
    assert abs(j["diff"]["got"] - j["diff"]["want"]) == pytest.approx(j["max_abs_blockwise"], rel=1e-9, abs=1e-12)


def test_report_show_renders_a_tuning_report():
    """`report show` (SPEC.md cli: a human-readable summary of a `tune run` report); the fixture
    is sf_tune's report for cfg2 measured on the B200 (profiles/r01/tune_configs_v2.jsonl)."""
    rep = ROOT / "tests" / "golden" / "tune_report_cfg2.jsonl"
    r = subprocess.run([str(CLI), "report", "show", str(rep)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0
    text = r.stdout
    j = json.loads(rep.read_text().splitlines()[0])
    assert j["graph"] in text and j["code"] in text and f"hex {j['code_hex']}" in text
    assert text.count("\n  [") == len(j["segments"])
    assert "(untuned)" in text and "cache hits" in text
    rc, back = run("report", "show", rep, "--output", "json")
    assert rc == 0 and back == j
    rc, err = run("report", "show", ROOT / "tests" / "golden" / "missing.jsonl")
    assert rc == 2 and err["error"] == "usage"
