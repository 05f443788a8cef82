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
