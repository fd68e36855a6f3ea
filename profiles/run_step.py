#!/usr/bin/env python3
"""Minimal driver for ncu captures: build the engine, stage one batch, run
`--warmup` steps then `--steps` steps of encode + beam search (no host I/O)."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_13695_b200 as P  # noqa: E402
from paper_2506_13695_b200._lib import check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="0.935B")
ap.add_argument("--users", type=int, default=128)
ap.add_argument("--width", type=int, default=128)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--precision", default="bf16")
a = ap.parse_args()
m = P.PolicyModel(P.PolicyConfig.preset(a.config), precision=a.precision, max_users=a.users, max_width=a.width)
b = P.SynthBatch(1, 0, a.users)
check(lib().orx_engine_stage_batch(m._e, C.byref(b.c)))
for _ in range(a.warmup + a.steps):
    check(lib().orx_beam_search_staged(m._e, a.width, None))
print("launches", m.stats()["launches"])
print("topk fallback rows", lib().orx_debug_topk_fallback_rows())
