#!/bin/bash
# End-of-round-2 evidence on one 4-GPU box: the GPU test suite (EP at 2 and 4
# ranks included), smoke, the 1-GPU bench line (with cpu_baseline), the
# reference arm, DP at 2 / 4 GPUs, 2.633B DP4 vs EP4 (balanced placement),
# and the BASELINE config sweep. Outputs in gpurun_out/final/.
set -u
out=gpurun_out/final
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s > $out/pytest_gpu.log 2>&1; tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
timeout 900 python bench.py > $out/bench1.json 2> $out/bench1.err
timeout 900 python bench.py --impl reference > $out/ref.json 2> $out/ref.err
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n \
    bench.py --gpus $n --no-cpu-baseline > $out/bench$n.json 2> $out/bench$n.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --gpus 4 --config 2.633B --no-cpu-baseline --steps 10 > $out/dp4_2633.json 2> $out/dp4_2633.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 \
  bench.py --gpus 4 --config 2.633B --ep --no-cpu-baseline --steps 10 > $out/ep4_2633.json 2> $out/ep4_2633.err
bash profiles/sweep.sh > $out/sweep.jsonl 2>&1
python - <<'P'
import json, glob
for f in sorted(glob.glob("gpurun_out/final/*.json")):
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
        print(f, d.get("value"), d.get("ms_per_step"), (d.get("e2e") or {}).get("value"), (d.get("clocks") or {}).get("sm_mhz"))
    except Exception as e:
        print(f, "fail", e)
P
echo done
