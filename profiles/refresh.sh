#!/bin/bash
# One-GPU evidence refresh (run under gpurun from the repo root):
#   bench line, BASELINE config sweep, ncu launch list of one 0.935B step,
#   per-GEMM DRAM traffic over that step, and one `--set full` capture of the
#   dominant GEMM shape. Outputs land in gpurun_out/refresh/.
set -u
out=gpurun_out/refresh
mkdir -p $out
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
bash profiles/sweep.sh > $out/sweep.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python profiles/run_step.py --warmup 1 --steps 1 > $out/ncu_launches.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k 'regex:tc.?_gemm' \
  --clock-control none --csv --log-file $out/gemm_dram.csv \
  python profiles/run_step.py --warmup 1 --steps 1 > $out/ncu_dram.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc2_gemm --launch-skip 3 --launch-count 1 \
  -o $out/life_fc1 python profiles/gemm_probe.py life_fc1_leaky > $out/ncu_full.log 2>&1
echo done
