#!/usr/bin/env python3
"""Times the tcgen05 GEMM on the hot path's dominant shapes (CUDA events,
L2-flushed between launches) through the orx_debug_gemm hook; used for the
ncu captures behind roofline.traffic. Prints one line per shape."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_kernels_gpu import run_gemm  # noqa: E402

SHAPES = {  # name: (M, N, K, act, bias, out_bf16, resid)
    "enc_fc1_silu": (51840, 2048, 1024, 2, True, True, False),
    "enc_wo_resid": (51840, 1024, 1024, 0, False, False, True),
    "enc_fc2_resid": (51840, 1024, 2048, 0, True, False, True),
    "enc_qk": (51840, 2048, 1024, 0, False, True, False),
    "life_fc1_leaky": (256000, 1024, 2176, 1, True, True, False),
    "dec_head": (16384, 8192, 1024, 0, False, False, False),
    "dec_so_resid": (16384, 1024, 1024, 0, False, False, True),
    "dec_cq": (16384, 1024, 1024, 0, False, True, False),
    "dec_sqkv": (16384, 3072, 1024, 0, False, True, False),
    "dec0_so_resid": (128, 1024, 1024, 0, False, False, True),  # decoder step 0 (one row per user)
    "dec0_cq": (128, 1024, 1024, 0, False, True, False),
}


def main():
    names = sys.argv[1:] or list(SHAPES)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in names:
        M, N, K, act, bias, obf, res = SHAPES[name]
        A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
        B = ((torch.rand(N, K, device="cuda") - 0.5) / K ** 0.5).to(torch.bfloat16)
        b = torch.zeros(N, device="cuda") if bias else None
        R = torch.zeros(M, N, device="cuda") if res else None
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16 if obf else torch.float32)
        ts = []
        reps = 5  # back-to-back launches per timing (hides the per-launch gap), L2 flushed before each group
        for it in range(6):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                run_gemm(A, B, out=out, bias=b, resid=R, act=act, sync=False)
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(e0.elapsed_time(e1) / reps)
        ms = sorted(ts)[len(ts) // 2]
        print(f"{name}: M={M} N={N} K={K} {ms * 1e3:.1f} us {2.0 * M * N * K / ms / 1e9:.0f} TFLOP/s", flush=True)
        del A, B, b, R, out


if __name__ == "__main__":
    main()
