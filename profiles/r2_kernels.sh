#!/bin/bash
# Round-2 evidence pass (run under gpurun from the repo root): A/B bench of the
# fused beam selection, the ncu launch list of one 0.935B step, and one
# `--set full` capture per HBM-bound kernel. Outputs in gpurun_out/r2k/.
set -u
out=gpurun_out/r2k
mkdir -p $out
ORX_NO_FUSED_SELECT=1 timeout 600 python bench.py --no-cpu-baseline > $out/bench_nofused.json 2> $out/bench_nofused.err
timeout 600 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err
timeout 300 python profiles/run_step.py --warmup 1 --steps 1 > $out/plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python profiles/run_step.py --warmup 1 --steps 1 > $out/ncu_launches.log 2>&1
for k in ${KERNELS:-moe_route2_kernel fold_features_kernel rmsnorm4_kernel moe_combine_norm_kernel moe_scatter32_kernel dec_self_attn_row_kernel beam_select_kernel}; do
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:$k -s ${SKIP:-2} -c 1 -o $out/$k \
    python profiles/run_step.py --warmup 0 --steps 1 > $out/ncu_$k.log 2>&1
done
echo done
