"""Parity helpers shared by the GPU tests, smoke() and bench.py's checks.

The oracle is the reference C++ core itself (oracle/_ref/ref_driver, built
from /root/reference/proj/core by oracle/Makefile); it writes .npy dumps of
z_enc, teacher-forced logits and beams for seeded synthetic users.
"""
from __future__ import annotations

import os
import subprocess
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")


def ref_dump(preset: str, n_users: int, width: int, lens=None, user_seed: int = 1, user_begin: int = 0,
             n_prefix: int = 4, beam: bool = True, sets=(), out_dir=None, timeout=3600, trie_items: int = 0,
             trie_fanout: int = 0, trie_seed: int = 77, sample=None, sid_codes: bool = False):
    """Run the reference on synthetic users; returns (dir, per-user dict)."""
    if not os.path.exists(REF_DRIVER):
        raise FileNotFoundError(f"{REF_DRIVER} missing: run `make -C oracle`")
    out_dir = out_dir or tempfile.mkdtemp(prefix="orx_ref_")
    cmd = [REF_DRIVER, "dump", "--preset", preset, "--n-users", str(n_users), "--width", str(width),
           "--user-seed", str(user_seed), "--user-begin", str(user_begin), "--n-prefix", str(n_prefix),
           "--out", out_dir]
    for s in sets:
        cmd += ["--set", s]
    if lens is not None:
        cmd += ["--lens", ",".join(str(x) for x in lens)]
    if not beam:
        cmd += ["--no-beam"]
    if sid_codes:
        cmd += ["--sid-codes"]
    if trie_items:
        cmd += ["--trie-items", str(trie_items), "--trie-seed", str(trie_seed)]
        if trie_fanout:
            cmd += ["--trie-fanout", str(trie_fanout)]
    if sample is not None:  # dict(temperature, top_k, top_p, seed)
        cmd += ["--sample", "--temperature", str(sample.get("temperature", 1.0)), "--top-k",
                str(sample.get("top_k", 0)), "--top-p", str(sample.get("top_p", 1.0)), "--sample-seed",
                str(sample.get("seed", 5))]
    subprocess.run(cmd, check=True, timeout=timeout, capture_output=True)
    users = []
    for u in range(user_begin, user_begin + n_users):
        d = {k: np.load(os.path.join(out_dir, f"{k}_u{u}.npy")) for k in ("z", "prefixes", "logits")}
        if beam:
            d["beam_codes"] = np.load(os.path.join(out_dir, f"beam_codes_u{u}.npy"))
            d["beam_logp"] = np.load(os.path.join(out_dir, f"beam_logp_u{u}.npy"))
            d["seq_logp"] = np.load(os.path.join(out_dir, f"seq_logp_u{u}.npy"))
        if trie_items:
            d["trie_codes"] = np.load(os.path.join(out_dir, "trie_codes.npy"))
        if sample is not None:
            d["sample_codes"] = np.load(os.path.join(out_dir, f"sample_codes_u{u}.npy"))
            d["sample_logp"] = np.load(os.path.join(out_dir, f"sample_logp_u{u}.npy"))
        users.append(d)
    return out_dir, users


def prefixes_of(pre: np.ndarray):
    return [[int(c) for c in row if c >= 0] for row in pre]


def rel_inf(a, b) -> float:
    """||a - b||_inf / ||b||_inf."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def beams_match(codes_gpu, logp_gpu, codes_ref, logp_ref, rtol=1e-3):
    """Tie-aware beam equality: lists must be equal after
    allowing swaps of adjacent items whose reference scores differ by less than
    rtol*|score|; the last (boundary) member may differ under the same rule.
    Returns (ok, n_exact_rank, message)."""
    W = len(codes_ref)
    if len(codes_gpu) != W:
        return False, 0, f"length {len(codes_gpu)} != {W}"
    ref = [tuple(int(x) for x in c) for c in codes_ref]
    got = [tuple(int(x) for x in c) for c in codes_gpu]
    exact = sum(1 for a, b in zip(ref, got) if a == b)
    score = {c: float(s) for c, s in zip(ref, logp_ref)}
    # every GPU item must be a reference item, or tie with the boundary
    tol = lambda s: rtol * max(abs(s), 1e-12)  # noqa: E731
    boundary = float(logp_ref[-1])
    for i, c in enumerate(got):
        if c in score:
            # position may differ only within a near-tie band
            s = score[c]
            j = ref.index(c)
            if i != j:
                lo, hi = sorted((i, j))
                band = [float(x) for x in logp_ref[lo:hi + 1]]
                if max(band) - min(band) > tol(s) * 2 + 1e-12:
                    return False, exact, f"item {c} at rank {i}, reference rank {j}, scores {band[0]}..{band[-1]}"
        else:
            s = float(logp_gpu[i])
            if abs(s - boundary) > tol(boundary) * 2 + 1e-9:
                return False, exact, f"item {c} (score {s}) not in reference list (boundary {boundary})"
    return True, exact, "ok"
