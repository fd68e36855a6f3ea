"""GPU parity against the reference oracle (oracle/_ref/ref_driver).

fp32 mode: logits within 1e-3 relative (||.||_inf per (user, prefix) row) and
identical beams up to near-ties; z_enc checked the same way.
bf16 mode: deviation reported and bounded loosely.
"""
import numpy as np
import pytest

from parity_util import beams_match, prefixes_of, ref_dump, rel_inf

pytestmark = pytest.mark.gpu

LOGIT_RTOL = 1e-3  # north_star: fp32 logits within 1e-3 relative error


def _model(preset, precision, max_users=4, max_width=128, **over):
    import paper_2506_13695_b200 as P
    cfg = P.PolicyConfig.preset(preset, **over)
    return P, P.PolicyModel(cfg, precision=precision, max_users=max_users, max_width=max_width)


def _check_user(P, model, batch, refs, width, rtol_z, rtol_logits, check_beams=True):
    z = model.encode_batch(batch)
    report = []
    for u, ref in enumerate(refs):
        ez = rel_inf(z[u], ref["z"])
        assert ez <= rtol_z, f"user {u}: z_enc rel err {ez}"
        pres = prefixes_of(ref["prefixes"])
        lg = model.score_prefixes(batch, [u] * len(pres), pres)
        errs = [rel_inf(lg[i], ref["logits"][i]) for i in range(len(pres))]
        assert max(errs) <= rtol_logits, f"user {u}: logits rel err {max(errs)} (per prefix {errs})"
        # decode on the reference's own z as well (next_logits_eval boundary)
        lg2 = model.next_logits_batch(ref["z"].astype(np.float32), [0] * len(pres), pres)
        errs2 = [rel_inf(lg2[i], ref["logits"][i]) for i in range(len(pres))]
        assert max(errs2) <= rtol_logits, f"user {u}: next_logits rel err {max(errs2)}"
        report.append((ez, max(errs), max(errs2)))
    if check_beams:
        codes, logp, n_items = model.beam_search_arrays(batch, width)
        for u, ref in enumerate(refs):
            W = len(ref["beam_codes"])
            assert n_items[u] == W
            ok, exact, msg = beams_match(codes[u, :W], logp[u, :W], ref["beam_codes"], ref["beam_logp"])
            assert ok, f"user {u}: {msg} (exact-rank {exact}/{W})"
            assert np.allclose(logp[u, :W], ref["beam_logp"], rtol=1e-3, atol=1e-3) or exact < W
    return report


@pytest.mark.parametrize("width", [16, 512])
def test_tiny_fp32_exhaustive(width):
    """tiny config (test_policy.cpp:14-32); W=512 >= 8^3 reproduces the full
    enumeration (test_generation.cpp:108-126)."""
    P, model = _model("tiny", "fp32", max_users=3, max_width=512)
    _, refs = ref_dump("tiny", 3, width)
    batch = P.SynthBatch(1, 0, 3, 4, 4, 8)
    _check_user(P, model, batch, refs, width, 1e-5, 1e-5)


def test_tiny_ragged_fp32():
    """Ragged / empty pathways: left padding and the empty-lifelong pad key."""
    P, model = _model("tiny", "fp32", max_users=2, max_width=16)
    for lens in [(0, 0, 0), (2, 1, 3), (4, 0, 1)]:
        _, refs = ref_dump("tiny", 2, 16, lens=lens)
        batch = P.SynthBatch(1, 0, 2, *lens)
        _check_user(P, model, batch, refs, 16, 1e-5, 1e-5)


@pytest.mark.parametrize("width", [8, 128])
def test_0015b_fp32(width):
    P, model = _model("0.015B", "fp32", max_users=2, max_width=128)
    _, refs = ref_dump("0.015B", 2, width)
    batch = P.SynthBatch(1, 0, 2)
    rep = _check_user(P, model, batch, refs, width, 1e-4, LOGIT_RTOL)
    print("0.015B fp32 W=%d (z, logits, next_logits) rel err:" % width, rep)


MOE_SETS = {
    # 0.935B-style: MoE in the decoder only, 24 experts top-2 (d=128 -> h_e=384)
    "dec": (dict(moe_enabled=True, n_experts=24, experts_active=2),
            ["moe_enabled=1", "n_experts=24", "experts_active=2"]),
    # 2.633B-style: MoE in every encoder and decoder layer, top-4
    "enc_and_dec": (dict(moe_enabled=True, n_experts=24, experts_active=4, moe_location="enc_and_dec"),
                    ["moe_enabled=1", "n_experts=24", "experts_active=4", "moe_location=enc_and_dec"]),
}


@pytest.mark.parametrize("kind", ["dec", "enc_and_dec"])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_moe_small(kind, precision):
    """MoE routing (stable top-k, ascending combine, nn.cpp:117-172) at d=128."""
    over, sets = MOE_SETS[kind]
    P, model = _model("0.015B", precision, max_users=2, max_width=32, **over)
    lens = (20, 64, 300)
    _, refs = ref_dump("0.015B", 2, 32, lens=lens, sets=sets)
    batch = P.SynthBatch(1, 0, 2, *lens)
    if precision == "fp32":
        rep = _check_user(P, model, batch, refs, 32, 1e-4, LOGIT_RTOL)
        print(f"MoE {kind} fp32:", rep)
    else:
        # bf16 is reported, not bit-matched: with 24 experts the k-th and
        # (k+1)-th gate scores are often within the bf16 activation error, so
        # a few percent of tokens per MoE layer route differently from the
        # f64 reference and their rows differ by O(1) (then mix through
        # attention). Bound the median row tightly and the worst row loosely.
        z = model.encode_batch(batch)
        codes, logp, _ = model.beam_search_arrays(batch, 32)
        for u, ref in enumerate(refs):
            pres = prefixes_of(ref["prefixes"])
            lg = model.score_prefixes(batch, [u] * len(pres), pres)
            el = max(rel_inf(lg[i], ref["logits"][i]) for i in range(len(pres)))
            zr = np.abs(z[u] - ref["z"]).max(axis=1) / np.abs(ref["z"]).max()
            overlap = len({tuple(c) for c in codes[u]} & {tuple(c) for c in ref["beam_codes"]})
            print(f"MoE {kind} bf16 user {u}: z max {zr.max():.3e} median {np.median(zr):.3e} "
                  f"p95 {np.percentile(zr, 95):.3e} logits {el:.3e} overlap {overlap}/32")
            # measured (round 2): dec logits ~6e-3, overlap 31-32/32; enc_and_dec (MoE in every
            # layer, more routing flips) logits 0.07-0.10, overlap 27-29/32, median z row 8e-3
            assert np.median(zr) < 2e-2 and zr.max() < 0.6
            if kind == "dec":
                assert el < 2e-2 and overlap >= 28
            else:
                assert el < 0.2 and overlap >= 24


def test_0015b_bf16_deviation():
    P, model = _model("0.015B", "bf16", max_users=2, max_width=128)
    _, refs = ref_dump("0.015B", 2, 128)
    batch = P.SynthBatch(1, 0, 2)
    z = model.encode_batch(batch)
    codes, logp, _ = model.beam_search_arrays(batch, 128)
    for u, ref in enumerate(refs):
        ez = rel_inf(z[u], ref["z"])
        pres = prefixes_of(ref["prefixes"])
        lg = model.score_prefixes(batch, [u] * len(pres), pres)
        el = max(rel_inf(lg[i], ref["logits"][i]) for i in range(len(pres)))
        overlap = len({tuple(c) for c in codes[u]} & {tuple(c) for c in ref["beam_codes"]})
        print(f"0.015B bf16 user {u}: z rel {ez:.3e} logits rel {el:.3e} beam overlap {overlap}/128")
        assert ez < 2e-2 and el < 2e-2 and overlap >= 120  # measured: 6e-3, 6e-3, 126-127


def test_cpp_dropin_shim_matches_reference():
    """The C++ adapter over the reference's own types (include/orx_genrec.hpp)
    reproduces PolicyModel::encode_eval / next_logits_eval / beam_search."""
    import os
    import subprocess
    demo = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "shim_demo")
    r = subprocess.run([demo, "16"], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("moe", [False, True])
def test_bf16_tcgen05_attention_dh128(moe):
    """bf16 engine with head dim 128 (the paper configs' dh): attention runs on
    the tcgen05 flash kernel with V written transposed by the producing GEMMs
    (encoder self-attention, QFormer over ragged lifelong keys, decoder cross
    attention over the cached encoder K/V). Checked against the f64
    reference and against the same engine on the mma.sync attention kernel."""
    import os
    over = dict(d_model=256, n_heads=2, ffn_hidden=512)
    sets = ["d_model=256", "n_heads=2", "ffn_hidden=512"]
    if moe:
        over.update(moe_enabled=True, n_experts=8, experts_active=2)
        sets += ["moe_enabled=1", "n_experts=8", "experts_active=2"]
    lens = (20, 64, 300)
    P, model = _model("0.015B", "bf16", max_users=2, max_width=32, **over)
    _, refs = ref_dump("0.015B", 2, 32, lens=lens, sets=sets)
    batch = P.SynthBatch(1, 0, 2, *lens)
    z = model.encode_batch(batch)
    codes, logp, _ = model.beam_search_arrays(batch, 32)
    os.environ["ORX_ATTN_MMA_SYNC"] = "1"
    try:
        _, ref_model = _model("0.015B", "bf16", max_users=2, max_width=32, **over)
    finally:
        del os.environ["ORX_ATTN_MMA_SYNC"]
    z_mma = ref_model.encode_batch(batch)
    for u, ref in enumerate(refs):
        pres = prefixes_of(ref["prefixes"])
        lg = model.score_prefixes(batch, [u] * len(pres), pres)
        lg_mma = ref_model.score_prefixes(batch, [u] * len(pres), pres)
        el = max(rel_inf(lg[i], ref["logits"][i]) for i in range(len(pres)))
        el_mma = max(rel_inf(lg_mma[i], ref["logits"][i]) for i in range(len(pres)))
        ez = rel_inf(z[u], ref["z"])
        overlap = len({tuple(c) for c in codes[u]} & {tuple(c) for c in ref["beam_codes"]})
        print(f"dh=128 bf16 moe={moe} user {u}: z {ez:.3e} (mma.sync {rel_inf(z_mma[u], ref['z']):.3e}) "
              f"logits {el:.3e} (mma.sync {el_mma:.3e}) overlap {overlap}/32")
        assert el < 2e-2 and overlap >= 28  # measured: 7e-3 .. 9e-3, 30-32/32
        assert el < 2 * el_mma + 1e-2  # no worse than the mma.sync attention path


def _trie_from(P, codes, depth):
    t = P.SemanticTrie(depth)
    for i, c in enumerate(codes):
        t.insert([int(x) for x in c], i)
    return t


@pytest.mark.parametrize("preset,width,items,fanout", [("tiny", 16, 40, 4), ("tiny", 16, 9, 4), ("0.015B", 32, 3000, 0),
                                                       ("0.015B", 64, 400, 12)])
def test_constrained_beam_fp32(preset, width, items, fanout):
    """Trie-constrained beam search (GenerationRequest::constrain_to_trie,
    generation.cpp:58-64): only trie children are expanded, fewer than W items
    when the trie is small; parity with the reference on the same seeded trie."""
    lens = (4, 4, 8) if preset == "tiny" else (20, 64, 300)
    P, model = _model(preset, "fp32", max_users=2, max_width=max(width, 16))
    _, refs = ref_dump(preset, 2, width, lens=lens, trie_items=items, trie_fanout=fanout)
    trie = _trie_from(P, refs[0]["trie_codes"], model.cfg.n_code_layers)
    batch = P.SynthBatch(1, 0, 2, *lens)
    req = P.GenerationRequest(width=width, constrain_to_trie=True)
    out = model.generate_batch(batch, req, trie)
    for u, ref in enumerate(refs):
        W = len(ref["beam_codes"])
        got = out[u]
        assert len(got) == W, (len(got), W)
        assert all(it.legal for it in got)  # every constrained output is a trie leaf
        codes = np.array([it.codes for it in got], dtype=np.int32).reshape(W, -1)
        logp = np.array([it.log_prob for it in got])
        ok, exact, msg = beams_match(codes, logp, ref["beam_codes"], ref["beam_logp"])
        print(f"{preset} trie({items}) W={width} user {u}: {W} items, exact-rank {exact}/{W}")
        assert ok, msg


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_sequence_log_prob(precision):
    """PolicyModel::sequence_log_prob (policy.cpp:297-310) on the reference's
    beam items: teacher-forced decode of [BOS, c1, c2], summed picked log-softmax."""
    P, model = _model("0.015B", precision, max_users=2, max_width=32)
    lens = (20, 64, 300)
    _, refs = ref_dump("0.015B", 2, 16, lens=lens)
    batch = P.SynthBatch(1, 0, 2, *lens)
    users, codes, want = [], [], []
    for u, ref in enumerate(refs):
        for c, lp in zip(ref["beam_codes"], ref["seq_logp"]):
            users.append(u)
            codes.append(c)
            want.append(lp)
    got = model.sequence_log_prob_batch(batch, users, codes)
    want = np.array(want)
    err = np.abs(got - want).max() / np.abs(want).max()
    print(f"sequence_log_prob {precision}: max rel err {err:.3e}")
    assert err < (1e-4 if precision == "fp32" else 3e-2)
    np.testing.assert_allclose(want, np.concatenate([r["beam_logp"] for r in refs]), rtol=1e-9)


SAMPLE_CASES = [("tiny", dict(temperature=1.0, top_k=0, top_p=1.0, seed=5)),
                ("tiny", dict(temperature=0.7, top_k=3, top_p=0.9, seed=9)),
                ("0.015B", dict(temperature=1.3, top_k=50, top_p=0.95, seed=11)),
                ("0.015B", dict(temperature=1.0, top_k=0, top_p=0.8, seed=3))]


@pytest.mark.parametrize("preset,sample", SAMPLE_CASES)
def test_topk_topp_sampling_fp32(preset, sample):
    """sample_topk_topp (generation.cpp:90-148): tempered, top-k / top-p cut,
    stable ordering, the reference Rng's uniforms per (sample, step). fp32
    logits can flip a pick only when a uniform lands within ~1e-6 of a bucket
    edge, so nearly every sampled sequence must match the reference exactly."""
    lens = (4, 4, 8) if preset == "tiny" else (20, 64, 300)
    W = 24
    P, model = _model(preset, "fp32", max_users=2, max_width=W)
    _, refs = ref_dump(preset, 2, W, lens=lens, sample=sample)
    batch = P.SynthBatch(1, 0, 2, *lens)
    req = P.GenerationRequest(strategy="topk_topp", width=W, temperature=sample["temperature"],
                              top_k=sample["top_k"], top_p=sample["top_p"])
    out = model.generate_batch(batch, req, seed=sample["seed"], streams=[0, 1])
    same = total = 0
    for u, ref in enumerate(refs):
        for s, it in enumerate(out[u]):
            total += 1
            if list(it.codes) == [int(x) for x in ref["sample_codes"][s]]:
                same += 1
                assert abs(it.log_prob - ref["sample_logp"][s]) <= 1e-4 * max(1.0, abs(ref["sample_logp"][s]))
    print(f"sampling {preset} {sample}: {same}/{total} sequences identical to the reference")
    assert same >= 0.9 * total


@pytest.mark.parametrize("users,hist_len,dim,threshold,max_out", [(3, 300, 32, 8, 320), (4, 2300, 256, 8, 2000),
                                                                   (2, 5, 16, 8, 4)])
def test_compress_lifelong_gpu(users, hist_len, dim, threshold, max_out):
    """compress_lifelong (policy.cpp:447-510) with hierarchical K-means
    (kmeans.cpp:22-183) on the GPU is bit-identical to the reference on seeded
    raw histories (clustered content rows, build_user_context's Rng seeds)."""
    import os
    import subprocess
    import tempfile

    import paper_2506_13695_b200 as P
    from parity_util import REF_DRIVER
    d = tempfile.mkdtemp(prefix="orx_cmp_")
    subprocess.run([REF_DRIVER, "compress", "--n-users", str(users), "--hist-len", str(hist_len), "--content-dim",
                    str(dim), "--threshold", str(threshold), "--max-out", str(max_out), "--out", d],
                   check=True, capture_output=True, timeout=1200)
    ld = lambda n: np.load(os.path.join(d, n + ".npy"))  # noqa: E731
    got = P.compress_lifelong_batch(ld("in_offsets"), ld("in_vid"), ld("in_aid"), ld("in_tag"), ld("in_ts"),
                                    ld("in_playtime"), ld("in_duration"), ld("in_labels"), ld("in_content"),
                                    ld("seeds"), threshold=threshold, max_out=max_out)
    assert np.array_equal(got["offsets"], ld("out_offsets"))
    for f in ("vid", "aid", "labels", "tag", "ts", "playtime", "duration"):
        want = ld("out_" + f)
        assert np.array_equal(got[f].astype(want.dtype), want), f
    n_rep = len(set(got["vid"].tolist()))
    print(f"compress {users} users x ~{hist_len} records (D={dim}): {len(got['vid'])} records, {n_rep} representatives")


@pytest.mark.parametrize("d", [128, 1024])
def test_bf16_feature_fold(d):
    """bf16 engine: the pathway fc1 folded through the feature tables
    (launch_fold_features) against the same engine with the explicit feature
    rows + fc1 GEMM (ORX_NO_FEATURE_FOLD=1) and against the f64 reference."""
    import os
    over, sets = {}, []
    if d != 128:
        over = dict(d_model=d, n_heads=d // 128, ffn_hidden=2 * d)
        sets = [f"d_model={d}", f"n_heads={d // 128}", f"ffn_hidden={2 * d}"]
    lens = (20, 64, 300)
    P, model = _model("0.015B", "bf16", max_users=2, max_width=32, **over)
    _, refs = ref_dump("0.015B", 2, 32, lens=lens, sets=sets, beam=False, n_prefix=1)
    batch = P.SynthBatch(1, 0, 2, *lens)
    z = model.encode_batch(batch)
    os.environ["ORX_NO_FEATURE_FOLD"] = "1"
    try:
        _, unf = _model("0.015B", "bf16", max_users=2, max_width=32, **over)
    finally:
        del os.environ["ORX_NO_FEATURE_FOLD"]
    z_unf = unf.encode_batch(batch)
    for u, ref in enumerate(refs):
        ez, ez_unf, e_pair = rel_inf(z[u], ref["z"]), rel_inf(z_unf[u], ref["z"]), rel_inf(z[u], z_unf[u])
        print(f"fold d={d} user {u}: z {ez:.3e} (unfolded {ez_unf:.3e}, fold vs unfolded {e_pair:.3e})")
        assert ez < 5e-2 and ez <= 1.5 * ez_unf + 2e-3


def _with_sids(P, batch, L, V):
    """The ref_driver's --sid-codes rule: sid[l] = (vid >> 8l) % V."""
    users = batch.to_contexts()
    for u in users:
        for seq in (u.short_seq, u.positive_seq, u.lifelong_seq):
            for f in seq:
                f.sid = [int((f.vid >> (8 * l)) % V) for l in range(L)]
    return P.UserBatch(users, L)


@pytest.mark.parametrize("flag", ["use_sid_history", "vid_only_features", "both"])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_feature_branches(flag, precision):
    """PolicyConfig::use_sid_history (record vid row = sum of the SID code
    embeddings, policy.cpp:146-160) and vid_only_features (feature row = the
    vid row alone, policy.cpp:166) against the reference."""
    flags = ["use_sid_history", "vid_only_features"] if flag == "both" else [flag]
    over = {f: True for f in flags}
    sets = [f"{f}=1" for f in flags]
    lens = (20, 64, 300)
    P, model = _model("0.015B", precision, max_users=2, max_width=16, **over)
    sid = "use_sid_history" in flags
    _, refs = ref_dump("0.015B", 2, 16, lens=lens, sets=sets, sid_codes=sid)
    batch = P.SynthBatch(1, 0, 2, *lens)
    if sid:
        batch = _with_sids(P, batch, model.cfg.n_code_layers, model.cfg.codebook_size)
    if precision == "fp32":
        rep = _check_user(P, model, batch, refs, 16, 1e-4, LOGIT_RTOL)
        print(f"{flag} fp32 (z, logits, next_logits):", rep)
    else:
        z = model.encode_batch(batch)
        codes, _, _ = model.beam_search_arrays(batch, 16)
        for u, ref in enumerate(refs):
            pres = prefixes_of(ref["prefixes"])
            lg = model.score_prefixes(batch, [u] * len(pres), pres)
            el = max(rel_inf(lg[i], ref["logits"][i]) for i in range(len(pres)))
            overlap = len({tuple(c) for c in codes[u]} & {tuple(c) for c in ref["beam_codes"]})
            print(f"{flag} bf16 user {u}: z {rel_inf(z[u], ref['z']):.3e} logits {el:.3e} overlap {overlap}/16")
            assert rel_inf(z[u], ref["z"]) < 3e-2 and el < 3e-2 and overlap >= 12


@pytest.mark.parametrize("lens", [(20, 64, 300), (5, 3, 0), (0, 0, 0)])
def test_bf16_lifelong_kv_fold(lens):
    """bf16 + tcgen05 attention: the lifelong pathway's fc2 folded into the
    QFormer K|V weights (EngineT::build_kv_fold) against the unfolded engine
    (ORX_NO_KV_FOLD=1: fc2 GEMM, key rows, K|V GEMM) and the f64 reference,
    including users without lifelong history (pad key written by
    launch_fill_kv_pad)."""
    import os
    over = dict(d_model=256, n_heads=2, ffn_hidden=512)
    sets = ["d_model=256", "n_heads=2", "ffn_hidden=512"]
    P, model = _model("0.015B", "bf16", max_users=2, max_width=16, **over)
    _, refs = ref_dump("0.015B", 2, 16, lens=lens, sets=sets, beam=False, n_prefix=2)
    batch = P.SynthBatch(1, 0, 2, *lens)
    z = model.encode_batch(batch)
    os.environ["ORX_NO_KV_FOLD"] = "1"
    try:
        _, unf = _model("0.015B", "bf16", max_users=2, max_width=16, **over)
    finally:
        del os.environ["ORX_NO_KV_FOLD"]
    z_unf = unf.encode_batch(batch)
    for u, ref in enumerate(refs):
        ez, ez_unf, pair = rel_inf(z[u], ref["z"]), rel_inf(z_unf[u], ref["z"]), rel_inf(z[u], z_unf[u])
        print(f"kv fold lens={lens} user {u}: z {ez:.3e} (unfolded {ez_unf:.3e}, fold vs unfolded {pair:.3e})")
        assert ez < 3e-2 and ez <= 1.5 * ez_unf + 2e-3
