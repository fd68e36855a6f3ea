#!/bin/bash
# Kernel time vs step time: sum of warm-cache kernel durations of one 0.935B
# step (ncu --cache-control none) against bench.py's graph-replayed step.
set -u
out=gpurun_out/gap
mkdir -p $out
timeout 600 python bench.py --no-cpu-baseline > $out/bench.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file $out/warm.csv python profiles/run_step.py --warmup 1 --steps 1 > /dev/null 2>&1
python3 - <<'P'
import csv, json
rows = list(csv.reader(open("gpurun_out/gap/warm.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]; iv = h.index("Metric Value")
v = [float(r[iv].replace(",", "")) / 1e3 for r in rows[hi + 1:] if len(r) > iv]
n = len(v) // 2
d = json.loads([l for l in open("gpurun_out/gap/bench.json") if l.startswith("{")][-1])
print("launches/step", n, "warm kernel sum ms", round(sum(v[n:]) / 1e3, 3), "bench ms/step", round(d["ms_per_step"], 3),
      "sm_mhz", d["clocks"]["sm_mhz"])
P
