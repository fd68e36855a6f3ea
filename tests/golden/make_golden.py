#!/usr/bin/env python3
"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs oracle/_ref/ref_driver (the unmodified reference core compiled by
oracle/Makefile) on small configs and seeded synthetic users, and stores:
  <case>.grcp  the reference's own GRCP checkpoint (PolicyModel(cfg).save)
  <case>.npz   per user: z_enc, teacher-forced prefixes/logits, beam codes/log-probs
Usage: python tests/golden/make_golden.py   (needs oracle/_ref built)
"""
import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")

# case -> (preset, --set overrides, lens or None, n_users, width)
CASES = {
    "tiny": ("tiny", [], None, 2, 16),
    "tiny_ragged": ("tiny", [], (2, 1, 0), 2, 16),
    "tiny_wide": ("tiny", [], None, 1, 512),
    "tiny_moe": ("tiny", ["moe_enabled=1", "n_experts=4", "experts_active=2", "expert_round_multiple=8"], None, 2,
                 16),
    "tiny_moe_encdec": ("tiny", ["moe_enabled=1", "n_experts=6", "experts_active=3", "moe_location=enc_and_dec",
                                 "expert_round_multiple=8"], None, 2, 16),
}


def make(case):
    preset, sets, lens, n_users, width = CASES[case]
    tmp = tempfile.mkdtemp()
    base = [DRIVER, "--preset", preset]
    for s in sets:
        base += ["--set", s]
    grcp = os.path.join(HERE, case + ".grcp")
    subprocess.run([DRIVER, "save-grcp", "--preset", preset] + sum((["--set", s] for s in sets), []) +
                   ["--out", grcp], check=True)
    cmd = [DRIVER, "dump", "--preset", preset] + sum((["--set", s] for s in sets), []) + [
        "--n-users", str(n_users), "--width", str(width), "--out", tmp]
    if lens:
        cmd += ["--lens", ",".join(map(str, lens))]
    subprocess.run(cmd, check=True, capture_output=True)
    arrays = {}
    for u in range(n_users):
        for k in ("z", "prefixes", "logits", "beam_codes", "beam_logp"):
            arrays[f"{k}_u{u}"] = np.load(os.path.join(tmp, f"{k}_u{u}.npy"))
    arrays["meta"] = np.array([n_users, width] + list(lens or (-1, -1, -1)))
    np.savez_compressed(os.path.join(HERE, case + ".npz"), **arrays)
    shutil.rmtree(tmp)


if __name__ == "__main__":
    if not os.path.exists(DRIVER):
        sys.exit("build the oracle first: make -C oracle")
    for c in CASES:
        make(c)
        print("wrote", c)
