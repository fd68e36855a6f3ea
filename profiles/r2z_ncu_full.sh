#!/bin/bash
# `--set full` captures at head (one 0.935B step, run_step.py --warmup 0 --steps 1):
# the SwiGLU grouped GEMM with the folded-norm row scales (46th tc2 launch),
# the grouped W2 GEMM (47th), and the split-K tensor-pipe router (first big launch).
set -u
out=gpurun_out/r2zf
mkdir -p $out
timeout 300 python profiles/run_step.py --warmup 0 --steps 1 > $out/plain.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc2_gemm_kernel -s 46 -c 2 \
  -o $out/gemm_swiglu_w2 python profiles/run_step.py --warmup 0 --steps 1 > $out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:moe_route_tc -c 1 \
  -o $out/route_tc python profiles/run_step.py --warmup 0 --steps 1 > $out/ncu_route.log 2>&1
echo done
