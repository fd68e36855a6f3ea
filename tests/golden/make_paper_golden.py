#!/usr/bin/env python3
"""Regenerates the PAPER-CONFIG golden fixtures (tests/golden/paper_*.npz) from
the REFERENCE itself: oracle/_ref/ref_driver (the unmodified reference core,
oracle/Makefile) with the seeded random init (PolicyModel(cfg), policy.cpp:59-137)
at the benchmarked presets 0.121B and 0.935B, full-length
synthetic users (user seed 1; the generator in csrc/synth_users.hpp).

The reference needs ~20 s per encode and ~1.7 s per next_logits_eval at d=1024
(SURVEY.md §8(c) "Oracle cost"), far too slow for a test run, so the outputs
are generated once here and committed (the GPU box has no /root/reference).

Per fixture (one preset, one user, one beam width):
  z_rows      int32  which rows of z_enc are stored (every 8th + the last)
  z           f32    those rows of encode_eval (policy.cpp:317-321)
  prefixes    int32  [P][3] teacher-forced prefixes (-1 padded): [] and the
                     first n_prefix beam items' 1- and 2-code prefixes
  logits      f32    next_logits_eval(z, prefix) (policy.cpp:323-329), [P][V]
  beam_codes  int32  beam_search(width) via policy_scorer (generation.cpp:41-88)
  beam_logp   f64    their log-probs
  seq_logp    f64    sequence_log_prob of each beam item (policy.cpp:297-310),
                     only for the W=8 fixtures
f32 storage is exact enough for the 1e-3 relative logit bar (2^-24 rounding).
Usage: python tests/golden/make_paper_golden.py [-j PROCS]   (~15 min on 8 cores)
"""
import argparse
import os
import shutil
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")

# name -> (preset, user, width, with sequence_log_prob)
JOBS = {
    "paper_0935B_u0_w8": ("0.935B", 0, 8, True),
    "paper_0935B_u1_w8": ("0.935B", 1, 8, True),
    "paper_0121B_u0_w8": ("0.121B", 0, 8, True),
    "paper_0121B_u1_w8": ("0.121B", 1, 8, True),
    "paper_0935B_u0_w128": ("0.935B", 0, 128, False),
    "paper_0121B_u0_w128": ("0.121B", 0, 128, False),
}


def make(name):
    preset, u, width, seq = JOBS[name]
    tmp = tempfile.mkdtemp(prefix="orx_paper_")
    cmd = [DRIVER, "dump", "--preset", preset, "--n-users", "1", "--user-begin", str(u), "--width", str(width),
           "--n-prefix", "4", "--out", tmp]
    if not seq:
        cmd.append("--no-seq")
    r = subprocess.run(cmd, check=True, capture_output=True, text=True)
    ld = lambda k: np.load(os.path.join(tmp, f"{k}_u{u}.npy"))  # noqa: E731
    z = ld("z")
    rows = np.unique(np.r_[np.arange(0, z.shape[0], 8), z.shape[0] - 1]).astype(np.int32)
    out = dict(preset=np.array(preset), user=np.int32(u), width=np.int32(width), z_rows=rows,
               z=z[rows].astype(np.float32), prefixes=ld("prefixes"), logits=ld("logits").astype(np.float32),
               beam_codes=ld("beam_codes"), beam_logp=ld("beam_logp"))
    if seq:
        out["seq_logp"] = ld("seq_logp")
    np.savez(os.path.join(HERE, name + ".npz"), **out)
    shutil.rmtree(tmp)
    return name, r.stderr.strip()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=6)
    ap.add_argument("names", nargs="*")
    a = ap.parse_args()
    if not os.path.exists(DRIVER):
        sys.exit("build the oracle first: make -C oracle")
    with ThreadPoolExecutor(a.j) as ex:
        for name, log in ex.map(make, a.names or list(JOBS)):
            print(name, log, flush=True)
