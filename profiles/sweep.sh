#!/bin/bash
# BASELINE.json configs 1, 2 and 5 on one B200 (config 3 is bench.py's default,
# config 4 is `--config 2.633B --ep` on N GPUs). One JSON line per run.
set -u
mkdir -p gpurun_out
run() { timeout 600 python bench.py --no-cpu-baseline "$@" 2>/dev/null | grep '^{' | tail -1; }
echo "# config 1: 0.015B, 1 user, W=128"
run --config 0.015B --users 1 --width 128 --steps 20 --warmup 5
echo "# config 2: 0.121B dense, 256 users, W=128"
run --config 0.121B --users 256 --width 128 --steps 5 --warmup 3
for W in 32 64 256 512; do
  echo "# config 5: 0.121B, 256 users, W=$W"
  run --config 0.121B --users 256 --width $W --steps 5 --warmup 3
done
echo "# config 3 at the paper's production beam: 0.935B, 128 users/GPU, W=512"
run --config 0.935B --users 128 --width 512 --steps 3 --warmup 3
