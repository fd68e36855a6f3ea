#!/bin/bash
# One-GPU evidence pass after the RMSNorm fold / bf16 expert outputs: bench
# line, ncu launch list of one 0.935B step, `--set full` of routing and the
# folded pathway gather. Outputs in gpurun_out/r2b/.
set -u
out=gpurun_out/r2b
mkdir -p $out
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 300 python profiles/run_step.py --warmup 1 --steps 1 > $out/plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python profiles/run_step.py --warmup 1 --steps 1 > $out/ncu_launches.log 2>&1
for k in ${KERNELS:-moe_route_tc_kernel fold_features_kernel}; do
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:$k -s ${SKIP:-2} -c 1 -o $out/$k \
    python profiles/run_step.py --warmup 0 --steps 1 > $out/ncu_$k.log 2>&1
done
echo done
