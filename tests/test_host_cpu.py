"""Host-side logic on CPU (no GPU needed): the C-ABI library loads and exports
every symbol include/orx.h declares; seeded weight init and GRCP I/O are
bit-identical to the reference; input validation mirrors validate_context;
the engine refuses to run without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2506_13695_b200 as P
from paper_2506_13695_b200 import _lib
from parity_util import REF_DRIVER

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "orx.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(orx_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    names = _declared()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), f"liborx.so lacks {n}"
    bound = {s[0] for s in _lib.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_presets_and_expert_hidden():
    c = P.PolicyConfig.preset("0.935B")
    assert (c.d_model, c.n_heads, c.n_experts, c.experts_active, c.codebook_size) == (1024, 8, 24, 2, 8192)
    assert c.expert_hidden() == 2816  # test_moe.cpp:261-265
    assert c.enc_seq_len() == 405
    assert P.PolicyConfig.preset("2.633B").moe_location == "enc_and_dec"
    # MoE layers in engine order (the expert-placement table's rows)
    assert P.moe_layers(c) == 4  # decoder-only MoE: 4 decoder layers
    assert P.moe_layers(P.PolicyConfig.preset("2.633B")) == 24  # 12 encoder + 12 decoder
    assert P.moe_layers(P.PolicyConfig.preset("0.121B")) == 0
    with pytest.raises(ValueError):
        P.PolicyConfig.preset("nope")


@pytest.mark.parametrize("preset,sets", [("tiny", []), ("0.015B", []),
                                         ("tiny", ["moe_enabled=1", "n_experts=6", "experts_active=3",
                                                   "moe_location=enc_and_dec"])])
def test_seeded_init_bit_identical_to_reference(tmp_path, preset, sets):
    """PolicyModel(cfg) init order + Rng stream (policy.cpp:59-137, rng.cpp)."""
    if not os.path.exists(REF_DRIVER):
        pytest.skip("oracle/_ref not built")
    path = str(tmp_path / "ref.grcp")
    cmd = [REF_DRIVER, "save-grcp", "--preset", preset, "--out", path]
    for s in sets:
        cmd += ["--set", s]
    subprocess.run(cmd, check=True)
    ref = P.Weights.load(path)
    over = {}
    for s in sets:
        k, v = s.split("=")
        over[k] = (v if k == "moe_location" else (bool(int(v)) if k == "moe_enabled" else int(v)))
    ours = P.Weights.random(P.PolicyConfig.preset(preset, **over))
    assert ours.names() == ref.names()
    for n in ours.names():
        assert np.array_equal(ours.get(n), ref.get(n)), n
    # GRCP written by us carries the same header/config JSON as the reference's
    mine = str(tmp_path / "mine.grcp")
    ours.save(mine)
    a, b = open(path, "rb").read(), open(mine, "rb").read()
    n_hdr = 16 + int.from_bytes(a[8:16], "little")
    assert a[:n_hdr] == b[:n_hdr]
    back = P.Weights.load(mine)
    for n in ours.names()[:10]:
        assert np.array_equal(back.get(n), ours.get(n))


def test_grcp_errors():
    with pytest.raises(RuntimeError):
        P.Weights.load("/nonexistent/file.grcp")


def _ctx(n_short=2, n_pos=1, n_life=3):
    users = P.SynthBatch(5, 0, 1, n_short, n_pos, n_life).to_contexts()
    return users[0]


def test_synthetic_users_match_oracle_generator():
    from oracle import numpy_oracle as O
    ctx = _ctx(3, 2, 4)
    ref = O.synth_user(5, 0, (3, 2, 4))
    assert (ctx.uid, ctx.gender, ctx.age_bucket) == (ref["uid"], ref["gender"], ref["age"])
    for mine, theirs in ((ctx.short_seq, ref["short"]), (ctx.positive_seq, ref["positive"]),
                         (ctx.lifelong_seq, ref["lifelong"])):
        assert len(mine) == len(theirs)
        for a, b in zip(mine, theirs):
            assert (a.vid, a.aid, a.labels) == (b["vid"], b["aid"], b["labels"])
            assert (a.tag, a.ts, a.playtime, a.duration) == (b["tag"], b["ts"], b["playtime"], b["duration"])


def _validate(cfg, ctxs):
    b = P.UserBatch(ctxs, cfg.n_code_layers)
    _lib.check(_lib.lib().orx_validate_batch(C.byref(cfg.to_c()), C.byref(b.c)))


def test_validate_context_rules():
    """validate_context, policy.cpp:23-38: same rules, same messages, ValueError."""
    cfg = P.PolicyConfig.preset("tiny")
    _validate(cfg, [_ctx()])
    bad = _ctx()
    bad.short_seq[1].ts = bad.short_seq[0].ts - 1
    with pytest.raises(ValueError, match="not time-ordered"):
        _validate(cfg, [bad])
    bad = _ctx()
    bad.lifelong_seq[0].playtime = bad.lifelong_seq[0].duration + 0.1
    with pytest.raises(ValueError, match="playtime exceeds duration"):
        _validate(cfg, [bad])
    bad = _ctx()
    bad.positive_seq[0].labels = 1 << 5
    with pytest.raises(ValueError, match="label bits"):
        _validate(cfg, [bad])
    with pytest.raises(ValueError, match="exceeds its configured cap"):
        _validate(cfg, [_ctx(n_short=cfg.short_len + 1)])


def test_engine_refuses_without_gpu():
    """No CPU fallback: creating an engine without a CUDA device fails loudly."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(RuntimeError, match="CUDA"):
        P.PolicyModel(P.PolicyConfig.preset("tiny"), precision="fp32", max_users=1, max_width=4)


def test_request_validation():
    P.validate_request(P.GenerationRequest(width=4))
    for bad in (dict(width=0), dict(top_p=0.0), dict(top_k=-1), dict(temperature=0.0)):
        with pytest.raises(ValueError):
            P.validate_request(P.GenerationRequest(**bad))


def test_trie_lookup():
    t = P.SemanticTrie(3)
    t.insert([1, 2, 3], 7)
    t.insert([1, 2, 3], 8)
    assert t.lookup([1, 2, 3]) == [7, 8]
    assert t.lookup([1, 2]) is None
    assert t.item_count() == 2


def test_flops_model_matches_survey():
    import bench
    table = {"0.015B": (1.45, 2.06, 4.49), "0.121B": (80.7, 101.3, 183.7), "0.935B": (87.5, 128.3, 291.4),
             "2.633B": (509, 705, 1487)}
    for name, want in table.items():
        cfg = P.PolicyConfig.preset(name)
        got = [bench.flops_per_user(cfg, w, (20, 256, 2000))[0] / 1e9 for w in (32, 128, 512)]
        for g, w in zip(got, want):
            assert abs(g - w) / w < 0.01, (name, got, want)
    # folded pathway fc1 (bf16 engine): the per-record fc1 GEMM leaves the count
    cfg = P.PolicyConfig.preset("0.935B")
    d, n = cfg.d_model, 20 + 256 + 2000
    F = d + d // 2 + 5 * (d // 8)
    full, _ = bench.flops_per_user(cfg, 128, (20, 256, 2000))
    fold, _ = bench.flops_per_user(cfg, 128, (20, 256, 2000), fold_fc1=True)
    assert abs((full - fold) - 2.0 * n * (F * d - 10 * d)) < 1.0


def test_cpp_dropin_shim_builds_and_fails_loudly_without_gpu():
    """include/orx_genrec.hpp compiled against the reference's own headers
    (oracle/shim_demo.cpp); without a GPU the engine raises, never falls back."""
    demo = os.path.join(ROOT, "oracle", "_ref", "shim_demo")
    if not os.path.exists(demo):
        pytest.skip("oracle/_ref/shim_demo not built")
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present (covered by the gpu test)")
    except ImportError:
        pass
    r = subprocess.run([demo], capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "no CPU fallback" in r.stdout


def test_trie_csr_matches_children_of():
    """SemanticTrie.to_csr (the device trie layout) walks to the same children
    as children_of (trie.cpp:53-59), codes ascending, every leaf reachable."""
    import numpy as np

    import paper_2506_13695_b200 as P
    rng = np.random.default_rng(5)
    t = P.SemanticTrie(3)
    leaves = {tuple(int(x) for x in rng.integers(0, 6, 3)) for _ in range(60)}
    for i, c in enumerate(sorted(leaves)):
        t.insert(list(c), i)
    off, code, node = t.to_csr()
    assert off[0] == 0 and off[-1] == len(code) == len(node)

    def walk(prefix):
        n = 0
        for c in prefix:
            kids = code[off[n]:off[n + 1]]
            assert list(kids) == sorted(kids)
            n = int(node[off[n] + list(kids).index(c)])
        return n

    for leaf in leaves:
        for depth in range(3):
            n = walk(leaf[:depth])
            assert list(code[off[n]:off[n + 1]]) == t.children_of(list(leaf[:depth]))


def test_weights_set_roundtrip():
    """orx_weights_set overwrites a named parameter (host only)."""
    import numpy as np
    import pytest

    import paper_2506_13695_b200 as P
    w = P.Weights.random(P.PolicyConfig.preset("tiny"))
    x = w.get("dec.head0.w")
    y = np.arange(x.size, dtype=np.float32).reshape(x.shape)
    w.set("dec.head0.w", y)
    assert np.array_equal(w.get("dec.head0.w"), y)
    with pytest.raises(ValueError):
        w.set("dec.head0.w", y[:-1])
    with pytest.raises(ValueError):
        w.set("no.such.param", y)


def test_bench_static_presets_match_library():
    """bench.py's reference arm never loads liborx.so: its static preset table
    must equal the library's presets (include/orx.h / PolicyConfig)."""
    import bench

    import paper_2506_13695_b200 as P
    for name in bench.BenchConfig.PRESETS:
        b, p = bench.BenchConfig(name), P.PolicyConfig.preset(name)
        for f in bench.BenchConfig.BASE:
            assert getattr(b, f) == getattr(p, f), (name, f)
        assert b.expert_hidden() == p.expert_hidden()
        assert b.enc_seq_len() == p.enc_seq_len()
        assert bench.flops_per_user(b, 128, (20, 256, 2000)) == bench.flops_per_user(p, 128, (20, 256, 2000))


def test_bench_reference_arm_does_not_import_package():
    """--impl reference must not map liborx.so (the driver checks the loaded .so files)."""
    import subprocess
    import sys
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--config','0.015B','--steps','1',"
            "'--width','8','--users','1']\n"
            "import bench\n"
            "bench.run_reference_sample = lambda *a, **k: {'users_per_s': 1.0, 'procs': 1, 't_encode_s': 0.1, "
            "'beam_measured': True, 't_beam_s': 0.1, 'init_s': 0.0}\n"
            "bench.main()\n"
            "assert not any('paper_2506_13695_b200' in m for m in sys.modules), 'package imported'\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'liborx' not in maps, 'liborx.so mapped'\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=120)
    assert r.returncode == 0, r.stderr
    import json
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["config"]["model"] == "OneRec-0.015B"
