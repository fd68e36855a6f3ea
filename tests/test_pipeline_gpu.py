"""Pipelined serving API (orx_beam_search_submit / _collect): two requests in
flight over two staging slots and a copy stream must return exactly what the
synchronous orx_beam_search returns for each request, in submission order."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_2506_13695_b200 as P  # noqa: E402


@pytest.fixture(scope="module")
def model():
    return P.PolicyModel(P.PolicyConfig.preset("0.015B"), precision="bf16", max_users=6, max_width=16)


def _batch(seed, n):
    return P.SynthBatch(seed, 0, n, 20, 64, 300)


def test_pipelined_equals_synchronous(model):
    batches = [_batch(s, n) for s, n in ((1, 6), (2, 5), (3, 6), (4, 3))]
    want = [model.beam_search_arrays(b, 16) for b in batches]
    got = []
    model.beam_search_submit(batches[0], 16)
    for i in range(1, len(batches)):
        model.beam_search_submit(batches[i], 16)
        got.append(model.beam_search_collect())
    got.append(model.beam_search_collect())
    for (wc, wl, wn), (gc, gl, gn) in zip(want, got):
        assert np.array_equal(wc, gc) and np.array_equal(wl, gl) and np.array_equal(wn, gn)


def test_in_flight_limit_and_empty_collect(model):
    b = _batch(5, 4)
    model.beam_search_submit(b, 8)
    model.beam_search_submit(b, 8)
    with pytest.raises(ValueError, match="in flight"):
        model.beam_search_submit(b, 8)
    c0 = model.beam_search_collect()
    c1 = model.beam_search_collect()
    assert np.array_equal(c0[0], c1[0]) and np.array_equal(c0[1], c1[1])
    with pytest.raises(ValueError):
        model.beam_search_collect()
    # a synchronous call after the pipeline still works
    codes, _, _ = model.beam_search_arrays(b, 8)
    assert np.array_equal(codes, c0[0])
