"""The C-ABI library loads and exports every symbol include/sf_capi.h declares (CPU, no compute)."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "sf_capi.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(sf_[a-z0-9_]+)\s*\(", text))
    types = set(re.findall(r"\}\s*(sf_[a-z0-9_]+)\s*;", text)) | {"sf_launch_fn"}
    return sorted(n for n in names if n not in types)


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for need in ("sf_mask_generate", "sf_bsr_build", "sf_rowwise_build", "sf_select_plan", "sf_mha_blockwise",
                 "sf_mha_rowwise", "sf_gemm_fused", "sf_time_best"):
        assert need in syms


def test_library_exports_every_declared_symbol():
    from paper_2506_06095_b200 import _lib
    if not _lib.LIB_PATH.exists():
        pytest.fail("libsf_b200.so not built — run __graft_entry__.build()")
    L = C.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    # the ctypes binding covers the same set
    assert set(declared_symbols()) <= set(_lib.SIGNATURES), set(declared_symbols()) - set(_lib.SIGNATURES)


def test_host_only_entry_points_without_gpu():
    """Pure host functions of the boundary work without a device (selector arithmetic)."""
    from paper_2506_06095_b200 import _lib
    L = _lib.lib()
    hw = _lib.HwSpec()
    _lib.check(L.sf_hw_preset(b"a100", C.byref(hw)))
    assert (hw.sm_num, hw.smem_size, hw.max_warp) == (108, 192 * 1024, 64)
    with pytest.raises(_lib.InvalidParameter):
        _lib.check(L.sf_hw_preset(b"h100", C.byref(hw)))
    # planner.hpp:67-76 hand value at n = 1024 (test_planner.cpp:48-53)
    assert abs(L.sf_threshold_from_loads(1024, 64 * 64, 1.2) - (1 - 1.2 / 36)) < 1e-12
    p = _lib.Plan()
    _lib.check(L.sf_select_plan_from_loads(64 * 64, C.byref(hw), 1024, 12, 8, 64, 0, C.byref(p)))
    assert p.kind == _lib.SF_BLOCK_WISE
    assert "sm_100a" in _lib.version()


def test_decomposition_routing_host_logic():
    """Which session masks the unified MHA decomposes (host logic, no device): one strided(w) term
    at n >= 2048 with ceil(n / w) <= 128; one dilated(w, r >= 1) term with n % (r + 1) == 0 at
    n >= DILATED_MIN_SEQ (others only as an explicit rest); everything else runs the plan's executor."""
    import paper_2506_06095_b200.sparsefuse as sf
    st = lambda n, w: [dict(pattern="strided", seq_len=n, band_width=w)]
    assert sf.strided_band(st(2048, 45)) == 45
    assert sf.strided_band(st(1024, 32)) is None          # below n = 2048
    assert sf.strided_band(st(8192, 32)) is None          # 256 classes > 128 rows per class kernel
    assert sf.strided_band(st(2048, 45) + [dict(pattern="global", seq_len=2048, global_width=8)]) is None
    dil = lambda n, w, r: dict(pattern="dilated", seq_len=n, band_width=w, dilation_rate=r)
    assert sf.dilated_split([dil(4096, 64, 1)]) == (2, 64)
    assert sf.dilated_split([dil(4096, 64, 2)]) is None   # 4096 % 3 != 0
    assert sf.dilated_split([dil(6144, 20, 2)]) == (3, 20)
    assert sf.dilated_split([dil(2048, 45, 1)]) is None   # below DILATED_MIN_SEQ
    assert sf.dilated_split([dil(2048, 45, 1)], min_seq_len=0) == (2, 45)
    assert sf.dilated_split([dil(4096, 64, 0)]) is None   # rate 0 is a plain band
    t5 = [dil(4096, 64, 1), dict(pattern="global", seq_len=4096, global_width=64)]
    assert sf.dilated_split(t5) is None and sf.dilated_split(t5, allow_rest=True) == (2, 64)
    assert sf.dilated_split([dict(pattern="sliding", seq_len=4096, band_width=64)]) is None
