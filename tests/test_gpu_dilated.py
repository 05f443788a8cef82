"""Dilated masks by class decomposition (sf_mha_dilated, csrc/dilated.cu) against the oracle's
block_sparse_sdpa over the whole mask (attention.hpp:71-172): pure dilated(w, r) (classes only),
dilated + global (T5, a rest part merged by log-sum-exp), rates 1 and 2, the cfg4 bench shape, and
the argument checks."""
import numpy as np
import pytest
import torch

import paper_2506_06095_b200.sparsefuse as sf
from paper_2506_06095_b200 import _lib
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def o():
    return Oracle()


CASES = [
    # (bs, h, terms, tolerance)
    (2, 3, [dict(pattern="dilated", seq_len=1024, band_width=32, dilation_rate=1)]),
    (1, 2, [dict(pattern="dilated", seq_len=768, band_width=20, dilation_rate=2)]),
    (2, 2, [dict(pattern="dilated", seq_len=1024, band_width=64, dilation_rate=1),
            dict(pattern="global", seq_len=1024, global_width=64)]),
    (1, 2, [dict(pattern="dilated", seq_len=1200, band_width=16, dilation_rate=3),
            dict(pattern="sliding", seq_len=1200, band_width=5)]),
    (8, 12, [dict(pattern="dilated", seq_len=4096, band_width=64, dilation_rate=1),  # cfg4 bench shape
             dict(pattern="global", seq_len=4096, global_width=64)]),
]


@pytest.mark.parametrize("bs,h,terms", CASES)
def test_dilated_decomposition_matches_oracle(o, bs, h, terms):
    n = terms[0]["seq_len"]
    m = o.mask(terms)
    q, k, v = (x.astype(np.float16).astype(np.float32) for x in o.random_attention_input(bs, h, n, 64, 7))
    ref, _ = o.block_sparse_sdpa(q, k, v, m, 16, 16, threads=16)
    dm = sf.generate_mask(terms)
    split = sf.dilated_split(terms, min_seq_len=0, allow_rest=True)
    assert split is not None
    ctx = sf.MhaContext(dm, sf.KernelPlan("block_wise", 128, 16), dilated=split)
    assert (ctx.rest_bsr is None) == (len(terms) == 1)
    Q, K, V = (torch.from_numpy(x).cuda().half() for x in (q, k, v))
    out = sf.mha(Q, K, V, ctx)
    torch.cuda.synchronize()
    err = np.abs(out.float().cpu().numpy() - ref).max()
    assert err < 2e-2, err
    assert sf.executor_label(ctx) == ["dilated_decomposed", split[0], split[1]]


def test_dilated_argument_checks():
    n = 1024
    q = torch.randn(1, 2, n, 64, device="cuda").half()
    band = sf.build_bsr(sf.gen_sliding_window(n // 2, 16), 128, 16)
    with pytest.raises(_lib.InvalidParameter):
        sf.dilated_sdpa(q, q, q, 1, band)  # stride must be >= 2
    with pytest.raises(_lib.ShapeError):
        sf.dilated_sdpa(q, q, q, 4, band)  # class BSR must have n / stride rows
    q2 = torch.randn(1, 2, n + 1, 64, device="cuda").half()
    with pytest.raises(_lib.PlanError):
        sf.dilated_sdpa(q2, q2, q2, 2, band)  # n % stride != 0
    assert sf.dilated_split([dict(pattern="dilated", seq_len=1001, band_width=8, dilation_rate=1)], 0) is None
    assert sf.dilated_split([dict(pattern="sliding", seq_len=1024, band_width=8)], 0) is None
    t5 = [dict(pattern="dilated", seq_len=4096, band_width=64, dilation_rate=1),
          dict(pattern="global", seq_len=4096, global_width=64)]
    assert sf.dilated_split(t5) is None and sf.dilated_split(t5, allow_rest=True) == (2, 64)
    assert sf.dilated_split([t5[0]]) == (2, 64)
    assert sf.dilated_split([dict(t5[0], seq_len=2048)]) is None  # below DILATED_MIN_SEQ
