#!/usr/bin/env python3
"""Host-side breakdown of one end-to-end request (0.935B, 128 users, W=128):
stage_batch (validate + pack + H2D issue), the staged beam search alone, and
the full orx_beam_search call, wall-clock with the device synchronised."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_13695_b200 as P  # noqa: E402
from paper_2506_13695_b200._lib import check, lib, orx_beam_out  # noqa: E402

m = P.PolicyModel(P.PolicyConfig.preset("0.935B"), precision="bf16", max_users=128, max_width=128)
b = P.SynthBatch(1, 0, 128)
e = m._e
L = 3
codes = (C.c_int32 * (128 * 128 * L))()
logp = (C.c_double * (128 * 128))()
nitems = (C.c_int32 * 128)()
out = orx_beam_out(C.cast(codes, C.POINTER(C.c_int32)), C.cast(logp, C.POINTER(C.c_double)),
                   C.cast(nitems, C.POINTER(C.c_int32)))


def t(fn, n=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return sorted(ts)[len(ts) // 2]


print("stage_batch ms", t(lambda: check(lib().orx_engine_stage_batch(e, C.byref(b.c)))))
print("staged beam ms", t(lambda: check(lib().orx_beam_search_staged(e, 128, None))))
print("staged beam + out ms", t(lambda: check(lib().orx_beam_search_staged(e, 128, C.byref(out)))))
print("full call ms", t(lambda: check(lib().orx_beam_search(e, C.byref(b.c), 128, C.byref(out)))))
print("host cores", os.cpu_count())


def pipelined(n=20):
    check(lib().orx_beam_search_submit(e, C.byref(b.c), 128))
    check(lib().orx_beam_search_collect(e, C.byref(out)))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    check(lib().orx_beam_search_submit(e, C.byref(b.c), 128))
    for i in range(n):
        if i + 1 < n:
            check(lib().orx_beam_search_submit(e, C.byref(b.c), 128))
        check(lib().orx_beam_search_collect(e, C.byref(out)))
    return (time.perf_counter() - t0) * 1e3 / n


def sync(n=20):
    check(lib().orx_beam_search(e, C.byref(b.c), 128, C.byref(out)))
    t0 = time.perf_counter()
    for _ in range(n):
        check(lib().orx_beam_search(e, C.byref(b.c), 128, C.byref(out)))
    return (time.perf_counter() - t0) * 1e3 / n


def staged(n=20):
    check(lib().orx_beam_search_staged(e, 128, None))
    t0 = time.perf_counter()
    for _ in range(n):
        check(lib().orx_beam_search_staged(e, 128, None))
    return (time.perf_counter() - t0) * 1e3 / n


for _ in range(2):
    print(f"per request ms: staged only {staged():.3f}, synchronous {sync():.3f}, pipelined {pipelined():.3f}")
