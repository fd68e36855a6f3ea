"""ORACLE / TEST INFRASTRUCTURE ONLY — never imported by the product path.

A float64 numpy restatement of the reference hot path (/root/reference/proj/core),
used by tests/ to cross-check the golden fixtures produced by the compiled
reference (oracle/_ref/ref_driver, see tests/golden/make_golden.py). Parity is
pinned: tests/test_oracle_cpu.py checks this module against those fixtures.

Each function cites the reference file:line it restates. Small configs only.
"""
from __future__ import annotations

import json
import struct
from typing import Dict, List, Sequence, Tuple

import numpy as np

MASK64 = (1 << 64) - 1


# ---- Rng: xoshiro256** + splitmix64 (rng.cpp:11-77) ------------------------------------------
def _splitmix64(x: int) -> Tuple[int, int]:
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return x, z ^ (z >> 31)


def _rotl(x: int, k: int) -> int:
    return ((x << k) | (x >> (64 - k))) & MASK64


class Rng:
    def __init__(self, seed: int):
        x = seed & MASK64
        self.s = []
        for _ in range(4):
            x, v = _splitmix64(x)
            self.s.append(v)

    def next_u64(self) -> int:  # rng.cpp:29-39
        s = self.s
        result = (_rotl((s[1] * 5) & MASK64, 7) * 9) & MASK64
        t = (s[1] << 17) & MASK64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = _rotl(s[3], 45)
        return result

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:  # rng.cpp:41-45
        u = float(self.next_u64() >> 11) * 2.0 ** -53
        return u if (lo, hi) == (0.0, 1.0) else lo + (hi - lo) * u

    def randint(self, n: int) -> int:  # rng.cpp:62-70
        limit = MASK64 - MASK64 % n
        v = self.next_u64()
        while v >= limit:
            v = self.next_u64()
        return v % n

    def split(self, id_: int) -> "Rng":  # rng.cpp:72-77
        x = self.s[0] ^ ((self.s[3] + 0x632BE59BD9B4E019) & MASK64)
        _, h = _splitmix64(x)
        h ^= (id_ * 0xFF51AFD7ED558CCD + 1) & MASK64
        return Rng(h)


def synth_user(seed: int, index: int, lens=(20, 256, 2000)):
    """Same generator as paper_2506_13695_b200/csrc/synth_users.hpp."""
    n_short, n_pos, n_life = lens
    rng = Rng(seed).split(index)
    ctx = {"uid": rng.randint(1 << 20), "gender": rng.randint(3), "age": rng.randint(8),
           "short": [], "positive": [], "lifelong": []}
    ts = -0.01 * (n_short + n_pos + n_life)
    for name, n in (("lifelong", n_life), ("positive", n_pos), ("short", n_short)):
        for _ in range(n):
            vid = rng.randint(1 << 20)
            aid = rng.randint(100000)
            tag = rng.uniform()
            dur = rng.uniform(0.05, 1.0)
            play = dur * rng.uniform()
            labels = rng.randint(32)
            ts += 0.01
            ctx[name].append(dict(vid=vid, aid=aid, tag=tag, ts=ts, playtime=play, duration=dur, labels=labels))
    return ctx


# ---- GRCP (policy.cpp:411-443, io.cpp:22-95) ------------------------------------------------
def read_grcp(path: str) -> Tuple[dict, Dict[str, np.ndarray]]:
    with open(path, "rb") as f:
        buf = f.read()
    if buf[:4] != b"GRCP":
        raise RuntimeError("bad magic bytes")
    off = 4
    (ver,) = struct.unpack_from("<I", buf, off)
    off += 4
    if ver != 1:
        raise ValueError("unsupported checkpoint version")
    (n,) = struct.unpack_from("<Q", buf, off)
    off += 8
    cfg = json.loads(buf[off:off + n].decode())
    off += n
    (count,) = struct.unpack_from("<Q", buf, off)
    off += 8
    params = {}
    for _ in range(count):
        (ln,) = struct.unpack_from("<Q", buf, off)
        off += 8
        name = buf[off:off + ln].decode()
        off += ln
        (nd,) = struct.unpack_from("<I", buf, off)
        off += 4
        dims = struct.unpack_from("<" + "I" * nd, buf, off)
        off += 4 * nd
        cnt = int(np.prod(dims))
        params[name] = np.frombuffer(buf, dtype="<f8", count=cnt, offset=off).reshape(dims).copy()
        off += 8 * cnt
    return cfg, params


# ---- model (policy.cpp, nn.cpp, tape.cpp) -------------------------------------------------------
def hashed(i: int, vocab: int) -> int:  # policy.cpp:14-17
    m = abs(int(i)) % vocab  # C++ % truncates toward zero
    m = -m if i < 0 else m
    return m + vocab if m < 0 else m


def rms_norm(x, gain, eps=1e-6):  # tape.cpp:462-503
    ms = (x * x).sum(axis=1, keepdims=True) / x.shape[1] + eps
    return x * (1.0 / np.sqrt(ms)) * gain.reshape(1, -1)


def silu(x):  # tape.cpp:531-537
    return x / (1.0 + np.exp(-x))


def leaky_relu(x, slope=0.01):  # tape.cpp:524-529
    return np.where(x > 0, x, slope * x)


class Model:
    def __init__(self, cfg: dict, params: Dict[str, np.ndarray]):
        self.c = cfg
        self.p = params
        self.d = cfg["d_model"]

    def lin(self, name, x, bias=True):  # linear, nn.cpp:18-22
        y = x @ self.p[name + ".w"]
        if bias and (name + ".b") in self.p:
            y = y + self.p[name + ".b"]
        return y

    def mlp(self, name, x):  # mlp_leaky, nn.cpp:32-34
        return self.lin(name + ".fc2", leaky_relu(self.lin(name + ".fc1", x)))

    def ffn(self, name, x):  # ffn, nn.cpp:71-73
        return self.lin(name + ".fc2", silu(self.lin(name + ".fc1", x)))

    def mha(self, q, k, v, causal=None):  # mha_core, tape.cpp:822-905
        H = self.c["n_heads"]
        dh = self.d // H
        out = np.zeros((q.shape[0], self.d))
        for h in range(H):
            sl = slice(h * dh, (h + 1) * dh)
            s = (q[:, sl] @ k[:, sl].T) * (1.0 / np.sqrt(dh))
            if causal is not None:
                for i, m in enumerate(causal):
                    s[i, m:] = -np.inf
            s = s - s.max(axis=1, keepdims=True)
            e = np.exp(s)
            out[:, sl] = (e / e.sum(axis=1, keepdims=True)) @ v[:, sl]
        return out

    def attention(self, name, q_in, kv_in, causal=None):  # attention, nn.cpp:56-62
        q = q_in @ self.p[name + ".wq.w"]
        k = kv_in @ self.p[name + ".wk.w"]
        v = kv_in @ self.p[name + ".wv.w"]
        return self.mha(q, k, v, causal) @ self.p[name + ".wo.w"]

    def moe(self, name, x):  # moe_forward, nn.cpp:117-172
        E, k = self.c["n_experts"], self.c["experts_active"]
        scores = x @ self.p[name + ".gate.w"]
        bias = self.p[name + ".routing_bias"].reshape(-1)
        out = np.zeros_like(x)
        sel = []
        for t in range(x.shape[0]):
            order = sorted(range(E), key=lambda e: (-(scores[t, e] + bias[e]), e))[:k]  # stable, ties -> lower id
            sel.append(sorted(order))
        for t in range(x.shape[0]):
            s = np.array([scores[t, e] for e in sel[t]])
            w = np.exp(s - s.max())
            w /= w.sum()
            for j, e in enumerate(sel[t]):
                en = f"{name}.expert{e}"
                xe = x[t:t + 1]
                he = (silu(xe @ self.p[en + ".w1.w"]) * (xe @ self.p[en + ".w3.w"])) @ self.p[en + ".w2.w"]
                out[t] += w[j] * he[0]
        return out

    def ffn_or_moe(self, prefix, x):  # policy.cpp:240-252
        return self.moe(prefix + ".moe", x) if (prefix + ".moe.gate.w") in self.p else self.ffn(prefix + ".ffn", x)

    def feature_rows(self, recs):  # policy.cpp:139-198
        c, p = self.c, self.p
        vid = p["emb.vid"][[hashed(r["vid"], c["vid_vocab"]) for r in recs]]
        if c.get("vid_only_features"):
            return vid
        aid = p["emb.aid"][[hashed(r["aid"], c["aid_vocab"]) for r in recs]]
        cols = [vid, aid]
        for key, pname in (("tag", "emb.tag"), ("ts", "emb.ts"), ("playtime", "emb.playtime"),
                           ("duration", "emb.duration")):
            x = np.array([[r[key]] for r in recs])
            cols.append(x @ p[pname][0:1] + p[pname][1:2])
        hot = np.array([[(r["labels"] >> f) & 1 for f in range(c["n_label_flags"])] for r in recs], dtype=np.float64)
        cols.append(hot @ p["emb.label"])
        return np.concatenate(cols, axis=1)

    def embed_records(self, recs, mlp, pad, target):  # policy.cpp:200-216
        content = self.mlp(mlp, self.feature_rows(recs)) if recs else None
        if target < 0:
            return content if recs else self.p[pad]
        parts = [self.p[pad]] * (target - len(recs)) + ([content] if recs else [])
        return np.concatenate(parts, axis=0)

    def encode(self, ctx):  # policy.cpp:254-265
        c, p = self.c, self.p
        st = np.concatenate([p["emb.uid"][hashed(ctx["uid"], c["uid_vocab"])],
                             p["emb.gender"][hashed(ctx["gender"], c["gender_vocab"])],
                             p["emb.age"][hashed(ctx["age"], c["age_vocab"])]])[None]
        static = self.mlp("pathway.static", st)
        short = self.embed_records(ctx["short"], "pathway.short", "pad.short", c["short_len"])
        pos = self.embed_records(ctx["positive"], "pathway.positive", "pad.positive", c["positive_len"])
        keys = self.embed_records(ctx["lifelong"], "pathway.lifelong", "pad.lifelong", -1)
        q = p["lifelong.queries"]
        for b in range(c["lifelong_blocks"]):  # qformer_block, nn.cpp:97-100 (no residual)
            n = f"lifelong.block{b}"
            q = self.attention(n + ".attn", q, keys)
            q = self.ffn(n + ".ffn", rms_norm(q, p[n + ".norm.gain"]))
        z = np.concatenate([static, short, pos, q], axis=0) + p["emb.pos"]
        for l in range(c["n_layers"] // 2):
            n = f"enc{l}"
            nz = rms_norm(z, p[n + ".n1.gain"])
            z = z + self.attention(n + ".attn", nz, nz)
            z = z + self.ffn_or_moe(n, rms_norm(z, p[n + ".n2.gain"]))
        return z

    def next_logits(self, z, prefix: Sequence[int]):  # decode + position_logits, policy.cpp:267-295,323-329
        p = self.p
        rows = [p["dec.bos"]] + [p[f"dec.tokens{j}"][t:t + 1] for j, t in enumerate(prefix)]
        d = np.concatenate(rows, axis=0)
        causal = list(range(1, d.shape[0] + 1))
        for l in range(self.c["n_layers"] - self.c["n_layers"] // 2):
            n = f"dec{l}"
            nd = rms_norm(d, p[n + ".n1.gain"])
            d = d + self.attention(n + ".self", nd, nd, causal)
            d = d + self.attention(n + ".cross", rms_norm(d, p[n + ".n2.gain"]), z)
            d = d + self.ffn_or_moe(n, rms_norm(d, p[n + ".n3.gain"]))
        pos = len(prefix)
        return d[pos:pos + 1] @ p[f"dec.head{pos}.w"]


def log_softmax(logits):  # generation.cpp:10-20
    mx = logits.max()
    return logits - (mx + np.log(np.exp(logits - mx).sum()))


def beam_search(scorer, depth: int, vocab: int, width: int) -> List[Tuple[List[int], float]]:
    """Unconstrained beam search (generation.cpp:41-88)."""
    beams = [([], 0.0)]
    for _ in range(depth):
        cand = []
        for codes, lp in beams:
            lsm = log_softmax(np.asarray(scorer(codes)).reshape(-1))
            for code in range(vocab):
                cand.append((codes + [code], lp + float(lsm[code])))
        cand.sort(key=lambda b: (-b[1], b[0]))
        beams = cand[:width]
    return beams
