#!/bin/bash
# routing time per launch (instrumented bench step) and one `--set full` capture
# of a decoder cross-attention launch (fmha_tc_kernel, step 1, layer 0)
set -u
out=gpurun_out/r2c
mkdir -p $out
ORX_PROF_DUMP=1 timeout 600 python bench.py --no-cpu-baseline --steps 5 2> $out/dump.err > $out/bench.json
grep -E "route" $out/dump.err | head -20
timeout 400 ncu --set full --import-source on --clock-control none -k regex:fmha_tc_kernel -s 10 -c 1 -o $out/fmha_xattn \
  python profiles/run_step.py --warmup 0 --steps 1 > $out/ncu_fmha.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:dec_self_attn -s 4 -c 1 -o $out/dec_self \
  python profiles/run_step.py --warmup 0 --steps 1 > $out/ncu_dself.log 2>&1
echo done
