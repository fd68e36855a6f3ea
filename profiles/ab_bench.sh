#!/bin/bash
# Interleaved A/B of bench.py over library builds / settings:
#   ab_bench.sh ROUNDS ARM1 ARM2 ...
# ARM = LIB[:VAR=VAL[,VAR=VAL]] where LIB is a .so path or "cur" (the in-tree
# liborx.so). Prints users/s, step ms and per-class ms for every run.
rounds=$1; shift
for r in $(seq "$rounds"); do
  for arm in "$@"; do
    lib=${arm%%:*}; envs=""
    [ "$arm" != "$lib" ] && envs=${arm#*:}
    (
      if [ "$lib" = cur ]; then unset ORX_LIB_PATH; else export ORX_LIB_PATH=$lib; fi
      IFS=',' read -ra kv <<< "$envs"; for e in "${kv[@]}"; do [ -n "$e" ] && export "$e"; done
      timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['kernel_classes_ms_per_step']
print('$(basename $lib):$envs', round(d['value']), round(d['ms_per_step'],3), ' '.join(f'{k}={v[\"ms\"]:.3f}' for k,v in c.items()), flush=True)"
    )
  done
done
