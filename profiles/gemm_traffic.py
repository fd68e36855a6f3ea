#!/usr/bin/env python3
"""Turns an ncu CSV of dram__bytes_read/write + gpu__time_duration over the
tcgen05 GEMM launches of two 0.935B steps (profiles/run_step.py --warmup 1
--steps 1) into profiles/gemm_traffic.json: average DRAM bytes per GEMM launch
of the second step, the basis of bench.py's roofline.traffic."""
import csv
import json
import sys

src, dst = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
hdr = None
recs = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        recs.setdefault(int(d["ID"]), {})[d["Metric Name"]] = (float(d["Metric Value"]), d["Metric Unit"])
ids = sorted(recs)
second = ids[len(ids) // 2:]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
tot_b = tot_t = 0.0
for i in second:
    m = recs[i]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v, u = m[k]
        tot_b += v * scale.get(u, 1)
    v, u = m["gpu__time_duration.sum"]
    tot_t += v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1}.get(u, 1e-6)
out = {"bytes_per_launch": tot_b / len(second), "launches": len(second), "dram_bytes_step": tot_b,
       "ms_step_ncu": tot_t,
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:tc.?_gemm "
                 "over two 0.935B steps (profiles/run_step.py, W=128, 128 users); per-launch average over every "
                 "tcgen05 GEMM launch of the second step, matching roofline.flops_per_launch"}
json.dump(out, open(dst, "w"), indent=1)
print(out)
