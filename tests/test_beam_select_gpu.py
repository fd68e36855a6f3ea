"""Fused log-softmax + beam selection (launch_beam_select, beam.cu) from the
head GEMM's chunk statistics, against the unfused path (row_topk + beam_merge
over materialised logits, ORX_NO_FUSED_SELECT=1) and on degenerate ties."""
import math
import os

import numpy as np
import pytest

from parity_util import beams_match

pytestmark = pytest.mark.gpu

import paper_2506_13695_b200 as P  # noqa: E402


def _pair(cfg, weights=None, max_users=4, max_width=128):
    fused = P.PolicyModel(cfg, weights=weights, precision="bf16", max_users=max_users, max_width=max_width)
    os.environ["ORX_NO_FUSED_SELECT"] = "1"
    try:
        plain = P.PolicyModel(cfg, weights=weights, precision="bf16", max_users=max_users, max_width=max_width)
    finally:
        del os.environ["ORX_NO_FUSED_SELECT"]
    return fused, plain


@pytest.mark.parametrize("preset,users,width,lens", [("0.015B", 4, 128, (20, 64, 300)),
                                                      ("0.015B", 3, 64, (20, 256, 2000)),
                                                      ("0.015B", 2, 512, (20, 64, 300)),
                                                      ("0.121B", 2, 128, (20, 256, 2000))])
def test_fused_select_matches_unfused(preset, users, width, lens):
    cfg = P.PolicyConfig.preset(preset)
    fused, plain = _pair(cfg, max_users=users, max_width=width)
    b = P.SynthBatch(3, 0, users, *lens)
    cf, lf, nf = fused.beam_search_arrays(b, width)
    cp, lp, np_ = plain.beam_search_arrays(b, width)
    assert np.array_equal(nf, np_)
    exact_total = 0
    for u in range(users):
        # the two paths' fp32 log-sum-exp differ in the last bits (chunk-combined
        # vs streamed), so only near-ties (1e-5 relative) may reorder
        ok, exact, msg = beams_match(cf[u], lf[u], cp[u], lp[u], rtol=1e-5)
        assert ok, f"user {u}: {msg}"
        exact_total += exact
        np.testing.assert_allclose(lf[u], lp[u], rtol=1e-5, atol=1e-5)
    print(f"{preset} W={width}: exact-rank {exact_total}/{users * width}")
    assert exact_total >= 0.98 * users * width


def test_fused_select_degenerate_ties():
    """All-zero head weights: every logit is 0, every chunk ties, and the exact
    fallback must return the lexicographically first codes with log-prob
    -3 log V (generation.cpp:74-77 tie order)."""
    cfg = P.PolicyConfig.preset("0.015B")
    w = P.Weights.random(cfg)
    for j in range(cfg.n_code_layers):
        w.set(f"dec.head{j}.w", np.zeros_like(w.get(f"dec.head{j}.w")))
    fused, plain = _pair(cfg, weights=w, max_users=8, max_width=32)
    b = P.SynthBatch(1, 0, 8, 20, 64, 300)  # 8 x 32 rows > 128: the fused path runs
    V = cfg.codebook_size
    want = np.array([[0, 0, c] for c in range(32)], dtype=np.int32)
    for m in (fused, plain):
        codes, logp, _ = m.beam_search_arrays(b, 32)
        for u in range(8):
            assert np.array_equal(codes[u], want)
            np.testing.assert_allclose(logp[u], -3 * math.log(V), rtol=1e-6)
