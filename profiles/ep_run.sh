# 4-GPU box: EP bitwise tests, bf16 parity, 2.633B EP4 (balanced placement) / DP4, 0.935B 1-GPU bench
set -x
tag=${1:-ep}
python -m pytest tests/test_ep_gpu.py tests/test_paper_parity_gpu.py tests/test_parity_gpu.py -q -p no:cacheprovider -s > gpurun_out/r2_${tag}_pytest.log 2>&1; tail -3 gpurun_out/r2_${tag}_pytest.log
grep -E "bf16: logits|rank 0" gpurun_out/r2_${tag}_pytest.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --config 2.633B --ep --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_${tag}_ep4.json 2>gpurun_out/r2_${tag}_ep4.err; tail -c 300 gpurun_out/r2_${tag}_ep4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --config 2.633B --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_${tag}_dp4.json 2>/dev/null
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_${tag}_b1.json 2>/dev/null
python - "$tag" <<'P'
import json, sys
tag = sys.argv[1]
for f in [f"r2_{tag}_ep4", f"r2_{tag}_dp4", f"r2_{tag}_b1"]:
    try:
        d = json.loads([l for l in open(f"gpurun_out/{f}.json") if l.startswith("{")][-1])
        print(f, round(d["value"]), round(d["ms_per_step"], 2), round(d["e2e"]["value"]), d["clocks"]["sm_mhz"],
              d.get("expert_parallel"))
    except Exception as e:
        print(f, "fail", e)
P
