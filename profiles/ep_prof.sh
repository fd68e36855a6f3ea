# 4-GPU box: 2.633B EP4 bench, then one instrumented EP4 run with per-launch dumps per rank
set -x
tag=${1:-ep}
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --config 2.633B --ep --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_${tag}_ep4.json 2>gpurun_out/r2_${tag}_ep4.err
python - "$tag" <<'P'
import json, sys
d = json.loads([l for l in open(f"gpurun_out/r2_{sys.argv[1]}_ep4.json") if l.startswith("{")][-1])
print(round(d["value"]), round(d["ms_per_step"], 2), round(d["e2e"]["value"]), d["clocks"]["sm_mhz"], d.get("expert_parallel"))
P
rm -rf gpurun_out/eplogs_${tag}
ORX_PROF_DUMP=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 --redirects 3 --log-dir gpurun_out/eplogs_${tag} bench.py --gpus 4 --config 2.633B --ep --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/eplogs_${tag}/*/attempt_0/
