#!/bin/bash
# Interleaved A/B of bench.py over library builds: ab_bench.sh ROUNDS LIB1 LIB2 ...
# (a LIB of "cur" is the in-tree liborx.so). Prints users/s, step ms and class ms per run.
rounds=$1; shift
for r in $(seq "$rounds"); do
  for lib in "$@"; do
    if [ "$lib" = cur ]; then unset ORX_LIB_PATH; else export ORX_LIB_PATH=$lib; fi
    timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['kernel_classes_ms_per_step']
print('$(basename $lib)', round(d['value']), round(d['ms_per_step'],3), ' '.join(f'{k}={v[\"ms\"]:.3f}' for k,v in c.items()), flush=True)"
  done
done
