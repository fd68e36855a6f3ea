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


def test_synchronous_calls_refused_while_in_flight(model):
    """A synchronous entry point would reuse a submitted request's staging slot
    (and drain its result): it must refuse until the request is collected."""
    a, b = _batch(6, 4), _batch(7, 5)
    want_a = model.beam_search_arrays(a, 16)
    model.beam_search_submit(a, 16)
    with pytest.raises(ValueError, match="in flight"):
        model.score_prefixes(b, [0], [[1]])
    with pytest.raises(ValueError, match="in flight"):
        model.beam_search_arrays(b, 16)
    model.beam_search_submit(b, 16)
    got_a = model.beam_search_collect()
    got_b = model.beam_search_collect()
    assert np.array_equal(got_a[0], want_a[0]) and np.array_equal(got_a[1], want_a[1])
    want_b = model.beam_search_arrays(b, 16)
    assert np.array_equal(got_b[0], want_b[0]) and np.array_equal(got_b[1], want_b[1])
    # submit after a synchronous call: A then B in flight, both collected intact
    model.score_prefixes(a, [0], [[1]])
    model.beam_search_submit(a, 16)
    model.beam_search_submit(b, 16)
    ga, gb = model.beam_search_collect(), model.beam_search_collect()
    assert np.array_equal(ga[0], want_a[0]) and np.array_equal(gb[0], want_b[0])


def _rand_trie(seed, n_items, fanout=16):
    rng = np.random.default_rng(seed)
    t = P.SemanticTrie(3)
    for i in range(n_items):
        t.insert([int(x) for x in rng.integers(0, fanout, 3)], i)
    return t


def test_trie_switch_and_insert_reupload(model):
    """Constrained searches are replayed from captured CUDA graphs: switching
    the trie (same request shapes) or inserting into it must take effect."""
    b = _batch(8, 3)
    req = P.GenerationRequest(width=16, constrain_to_trie=True)
    t1, t2 = _rand_trie(1, 200), _rand_trie(2, 200)
    for t in (t1, t2, t1, t2):
        out = model.generate_batch(b, req, t)
        fresh = P.PolicyModel(P.PolicyConfig.preset("0.015B"), precision="bf16", max_users=6, max_width=16)
        want = fresh.generate_batch(b, req, t)
        for u in range(3):
            assert all(it.legal for it in out[u])
            assert [it.codes for it in out[u]] == [it.codes for it in want[u]]
    # items inserted after the first upload are seen by the device search
    extra = _rand_trie(3, 300, fanout=64)
    for k in extra._leaves:
        t2.insert(list(k), 10_000)
    out = model.generate_batch(b, req, t2)
    fresh = P.PolicyModel(P.PolicyConfig.preset("0.015B"), precision="bf16", max_users=6, max_width=16)
    want = fresh.generate_batch(b, req, t2)
    for u in range(3):
        assert all(it.legal for it in out[u])
        assert [it.codes for it in out[u]] == [it.codes for it in want[u]]
