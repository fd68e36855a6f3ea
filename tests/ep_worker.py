"""Worker for tests/test_ep_gpu.py (one process per GPU, launched by torchrun).

Each rank owns its own users; an expert-parallel engine (n_experts / world
experts per MoE layer, peer-memory dispatch / return) must reproduce a
replica engine (all experts) bitwise: encoder output, teacher-forced logits
and beams -- with contiguous expert blocks and with a load-balanced placement
(replicated hot experts, permuted owners) made from the first engine's
measured expert loads. Exits non-zero on any mismatch.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_13695_b200 as P  # noqa: E402
from paper_2506_13695_b200.dist import ep_unique_id  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    users, width = 3, 16
    ok = True
    for precision in ("fp32", "bf16"):
        # 2.633B-style: MoE in every encoder and decoder layer, top-4 of 24
        cfg = P.PolicyConfig.preset("0.015B", moe_enabled=True, n_experts=24, experts_active=4,
                                    moe_location="enc_and_dec")
        w = P.Weights.random(cfg)
        rep = P.PolicyModel(weights=w, precision=precision, device=local, max_users=users, max_width=width)
        # different users per rank (and a different ragged shape on odd ranks)
        lens = (20, 64, 300) if rank % 2 == 0 else (7, 31, 129)
        batch = P.SynthBatch(1, rank * users, users, *lens)
        pres = [[], [5], [5, 77], [1000]]
        who = [0, 1, 2, 2]
        z_rep = rep.encode_batch(batch)
        l_rep = rep.score_prefixes(batch, who, pres)
        c_rep, p_rep, _ = rep.beam_search_arrays(batch, width)
        # contiguous expert blocks, then a load-balanced placement from the first
        # engine's measured loads (replicated hot experts, permuted owners)
        owner = None
        for placement in ("contiguous", "balanced"):
            uid = ep_unique_id(device=torch.device("cuda", local))  # one id per communicator
            w_ep = P.Weights.random_ep(cfg, rank, world, owner=owner)  # only the experts this rank computes
            ep = P.PolicyModel(weights=w_ep, precision=precision, device=local, max_users=users, max_width=width,
                               ep=(rank, world, uid), ep_owner=owner)
            z_ep = ep.encode_batch(batch)
            l_ep = ep.score_prefixes(batch, who, pres)
            c_ep, p_ep, _ = ep.beam_search_arrays(batch, width)
            checks = {"z": np.array_equal(z_rep, z_ep), "logits": np.array_equal(l_rep, l_ep),
                      "beam codes": np.array_equal(c_rep, c_ep), "beam logp": np.array_equal(p_rep, p_ep)}
            if placement == "contiguous":
                load = ep.expert_load()
                lt = torch.from_numpy(load).to(torch.device("cuda", local))
                every = [torch.zeros_like(lt) for _ in range(world)]
                dist.all_gather(every, lt)  # the loads come from all-gathered histograms: equal on every rank
                checks["load"] = bool(load.sum() > 0 and all(torch.equal(t, lt) for t in every))
                owner, pred = P.ep_place(load, world, 4)
                # force at least one replicated expert per layer so the test covers that path
                for li in range(owner.shape[0]):
                    if (owner[li] < 0).sum() == 0:
                        owner[li, int(np.argmax(load[li]))] = -1
            else:
                checks["replicated"] = bool((owner < 0).any())
            print(f"rank {rank} {precision} {placement}: "
                  + ", ".join(f"{k} {'==' if v else '!='}" for k, v in checks.items()), flush=True)
            ok = ok and all(checks.values())
            del ep
        del rep
    flag = torch.tensor([1 if ok else 0], device=torch.device("cuda", local))
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    if rank == 0:
        print("EP bitwise OK" if flag.item() == 1 else "EP MISMATCH", flush=True)
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
