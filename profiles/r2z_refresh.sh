#!/bin/bash
# Final round-2 evidence refresh on one GPU: smoke, bench line, ncu launch list
# of one 0.935B step (cold and warm cache), per-GEMM DRAM traffic, and `--set
# full` captures of the dominant GEMM and the decoder cross attention.
set -u
out=gpurun_out/r2z
mkdir -p $out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 300 python profiles/run_step.py --warmup 1 --steps 1 > $out/plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python profiles/run_step.py --warmup 1 --steps 1 > $out/ncu_launches.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file $out/launches_warm.csv python profiles/run_step.py --warmup 1 --steps 1 > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k 'regex:tc.?_gemm' \
  --clock-control none --csv --log-file $out/gemm_dram.csv \
  python profiles/run_step.py --warmup 1 --steps 1 > $out/ncu_dram.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:tc2_gemm_kernel<256, 5, 96>' -s 4 -c 1 \
  -o $out/gemm_swiglu python profiles/run_step.py --warmup 0 --steps 1 > $out/ncu_swiglu.log 2>&1
echo done
