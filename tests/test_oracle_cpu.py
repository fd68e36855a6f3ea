"""Pins the numpy restatement oracle (oracle/numpy_oracle.py) against golden
fixtures produced by the reference itself (tests/golden/make_golden.py runs the
compiled reference core). CPU only."""
import os

import numpy as np
import pytest

from oracle import numpy_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["tiny", "tiny_ragged", "tiny_wide", "tiny_moe", "tiny_moe_encdec"]


def _load(case):
    cfg, params = O.read_grcp(os.path.join(GOLDEN, case + ".grcp"))
    g = np.load(os.path.join(GOLDEN, case + ".npz"))
    n_users, width = int(g["meta"][0]), int(g["meta"][1])
    lens = tuple(int(x) for x in g["meta"][2:5])
    if lens[0] < 0:
        lens = (cfg["short_len"], cfg["positive_len"], cfg["lifelong_len"])
    return cfg, params, g, n_users, width, lens


@pytest.mark.parametrize("case", CASES)
def test_numpy_oracle_matches_reference_golden(case):
    cfg, params, g, n_users, width, lens = _load(case)
    m = O.Model(cfg, params)
    for u in range(n_users):
        ctx = O.synth_user(1, u, lens)
        z = m.encode(ctx)
        np.testing.assert_allclose(z, g[f"z_u{u}"], rtol=0, atol=1e-10)
        for pre, ref in zip(g[f"prefixes_u{u}"], g[f"logits_u{u}"]):
            p = [int(c) for c in pre if c >= 0]
            np.testing.assert_allclose(m.next_logits(g[f"z_u{u}"], p)[0], ref, rtol=0, atol=1e-10)
        beams = O.beam_search(lambda p: m.next_logits(g[f"z_u{u}"], p), cfg["n_code_layers"],
                              cfg["codebook_size"], width)
        assert [b[0] for b in beams] == [list(map(int, c)) for c in g[f"beam_codes_u{u}"]]
        np.testing.assert_allclose([b[1] for b in beams], g[f"beam_logp_u{u}"], rtol=0, atol=1e-10)


def test_beam_worked_example():
    """test_generation.cpp:86-106: top (0,0) with log-prob ln 0.54."""
    dist = {(): [0.6, 0.4], (0,): [0.9, 0.1], (1,): [0.5, 0.5]}
    beams = O.beam_search(lambda p: np.log(dist[tuple(p)]), 2, 2, 4)
    assert beams[0][0] == [0, 0]
    assert abs(beams[0][1] - np.log(0.54)) < 1e-12


def test_rng_stream_matches_reference_rng():
    """The Python Rng restatement reproduces the synthetic users the reference
    driver consumed (z_enc equality above depends on it); spot-check split()."""
    a = O.Rng(7).split(3)
    b = O.Rng(7).split(3)
    assert [a.next_u64() for _ in range(5)] == [b.next_u64() for _ in range(5)]
    assert O.hashed(-5, 4) == 3 and O.hashed(9, 4) == 1
