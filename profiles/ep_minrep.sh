# 2.633B EP4 with at least m replicated experts per MoE layer (m = 0 2 4), DP4 for reference
for m in 0 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2962$m bench.py \
    --gpus 4 --config 2.633B --ep --ep-min-replicas $m --steps 10 --no-cpu-baseline > gpurun_out/r2_ep_min$m.json 2>/dev/null
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29629 bench.py \
  --gpus 4 --config 2.633B --steps 10 --no-cpu-baseline > gpurun_out/r2_ep_dp4.json 2>/dev/null
python - <<'P'
import json
for f in ["r2_ep_min0", "r2_ep_min2", "r2_ep_min4", "r2_ep_dp4"]:
    try:
        d = json.loads([l for l in open(f"gpurun_out/{f}.json") if l.startswith("{")][-1])
        print(f, round(d["value"]), round(d["ms_per_step"], 2), d["clocks"]["sm_mhz"], (d.get("expert_parallel") or {}).get("replicated_per_layer"))
    except Exception as e:
        print(f, "fail", e)
P
