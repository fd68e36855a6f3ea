#!/usr/bin/env python3
"""Benchmark of the OneRec inference hot path on B200 (one rank per GPU).

A step = encode + depth-3 beam search (width W) for one batch of synthetic
users per GPU (BASELINE.json config 3: OneRec-0.935B MoE, 1024 users over 8
GPUs -> 128 users per GPU; weak scaling). Default N=1 runs the same 128-user
per-GPU batch.

  value    users/s over all ranks, inputs already resident in HBM
           (orx_engine_stage_batch once, then orx_beam_search_staged per step),
           CUDA events on the engine stream, max over ranks.
  e2e      same metric through the public C-ABI call orx_beam_search with
           host buffers: H2D of the step's packed user records and D2H of the
           beams inside the timed region.
  roofline the tcgen05 GEMM kernel class (dense + grouped MoE), algorithmic
           FLOPs / CUDA-event time per launch, from one instrumented step.
  cpu_baseline  the reference C++ core (oracle/_ref/ref_driver) on this
           host's cores, bounded sample (rank 0, N=1 only).

--impl reference times the reference's own CPU implementation instead.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "users/sec (beam-searched rec lists) per box at 1/2/4/8 B200; inference MFU"

BASELINE_CONFIG = {"0.015B": 1, "0.121B": 2, "0.935B": 3, "2.633B": 4}
PROF_NAMES = ["gemm_dense", "gemm_moe", "attention", "dec_self_attn", "moe_route", "beam_select", "other",
              "xattn_decode", "features", "rmsnorm"]


_JSON_OUT = None


def quiet_stdout():
    """Route fd 1 to stderr so native libraries' banners (NCCL's version line
    under NCCL_DEBUG=VERSION) never precede the one JSON line on stdout."""
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line):
    out = _JSON_OUT or sys.stdout
    print(json.dumps(line), file=out, flush=True)


class BenchConfig:
    """Static copy of the preset dims bench.py needs (include/orx.h presets =
    the reference PolicyConfig at PAPER.md:398-413), so the reference arm never
    imports the package or loads liborx.so. tests/test_host_cpu.py checks it
    against PolicyConfig.preset."""

    BASE = dict(n_layers=4, d_model=128, ffn_hidden=256, n_heads=4, moe_enabled=False, n_experts=0,
                experts_active=0, moe_location="decoder", expert_round_multiple=128, n_code_layers=3,
                codebook_size=64, short_len=20, positive_len=256, lifelong_len=2000, n_queries=128,
                lifelong_blocks=2, seed=123)
    PRESETS = {
        "0.015B": dict(n_layers=4, d_model=128, ffn_hidden=256, n_heads=4, codebook_size=8192),
        "0.121B": dict(n_layers=8, d_model=1024, ffn_hidden=2048, n_heads=8, codebook_size=8192),
        "0.935B": dict(n_layers=8, d_model=1024, ffn_hidden=2048, n_heads=8, codebook_size=8192, moe_enabled=True,
                       n_experts=24, experts_active=2),
        "2.633B": dict(n_layers=24, d_model=1024, ffn_hidden=2048, n_heads=8, codebook_size=8192, moe_enabled=True,
                       n_experts=24, experts_active=4, moe_location="enc_and_dec"),
    }

    def __init__(self, name):
        if name not in self.PRESETS:
            raise ValueError(f"unknown preset {name}")
        self.__dict__.update(self.BASE)
        self.__dict__.update(self.PRESETS[name])

    def enc_layers(self):
        return self.n_layers // 2

    def dec_layers(self):
        return self.n_layers - self.n_layers // 2

    def enc_seq_len(self):
        return 1 + self.short_len + self.positive_len + self.n_queries

    def expert_hidden(self):  # policy.cpp expert sizing: round_up((8 d + 2) / 3, multiple)
        raw = (2 * 4 * self.d_model + 2) // 3
        m = self.expert_round_multiple
        return (raw + m - 1) // m * m


def bench_config(args, cfg, lens, world):
    """The `config` object, identical for both arms (the driver compares them)."""
    return {"workload": f"OneRec-{args.config} (BASELINE config {BASELINE_CONFIG.get(args.config, '?')}): encoder + "
                        f"{'MoE ' if cfg.moe_enabled else ''}decoder + depth-{cfg.n_code_layers} beam search, "
                        f"W={args.width}, V={cfg.codebook_size}, {args.users} users/GPU "
                        f"(short,positive,lifelong)={tuple(lens)}, random-init weights (seed {cfg.seed})",
            "model": f"OneRec-{args.config}", "users_per_gpu": args.users, "global_batch": args.users * world,
            "width": args.width, "lens": list(lens), "parallelism": f"dp{world}" + (f"xep{world}" if args.ep else ""),
            "l2": "working set (weights ~2 GB + activations) exceeds the 126 MB L2; no flush"}


def flops_per_user(cfg, width, lens, fold_fc1=False, fold_kv=False):
    """Algorithmic FLOPs per user, KV-cached minimum.
    fold_fc1: the pathway fc1 folded through the feature tables (bf16 engine),
    so only fc2 is a per-record GEMM; fold_kv: the lifelong pathway's fc2 folded
    into the QFormer K|V weights (bf16 engine), so the lifelong records go
    through one GEMM (K|V) after the fold (what the engine executes)."""
    d, V, T = cfg.d_model, cfg.codebook_size, cfg.enc_seq_len()
    ns, npos, nl = lens
    nl_keys = max(nl, 1)
    ffn = lambda r: 4.0 * r * d * cfg.ffn_hidden  # noqa: E731
    moe = lambda r: 2.0 * r * d * cfg.n_experts + cfg.experts_active * 6.0 * r * d * cfg.expert_hidden()  # noqa: E731
    enc = 2.0 * (3 * (d // 16)) * d + 2.0 * d * d  # static MLP
    F = d + d // 2 + 5 * (d // 8)
    fc1 = 10 * d if fold_fc1 else F * d  # folded: a gather-add of ~10 d-vectors per record
    enc += 2.0 * (ns + npos + nl) * (fc1 + d * d)  # pathway MLPs
    if fold_kv and cfg.lifelong_blocks > 0:
        enc -= 2.0 * nl * d * d  # lifelong fc2 absorbed by the K|V projection
    Nq = cfg.n_queries
    enc += cfg.lifelong_blocks * (2.0 * Nq * d * d * 2 + 4.0 * nl_keys * d * d + 4.0 * Nq * nl_keys * d + ffn(Nq))
    enc_moe = cfg.moe_enabled and cfg.moe_location == "enc_and_dec"
    enc += cfg.enc_layers() * (8.0 * T * d * d + 4.0 * T * T * d + (moe(T) if enc_moe else ffn(T)))
    Ld = cfg.dec_layers()
    dec = Ld * 4.0 * T * d * d
    rows, live = [], 1
    for p in range(cfg.n_code_layers):
        rows.append((p, live))
        live = min(width, live * V)
    for p, r in rows:
        per = Ld * (8.0 * d * d + 4.0 * (p + 1) * d + 4.0 * d * d + 4.0 * T * d +
                    (moe(1) if cfg.moe_enabled else ffn(1))) + 2.0 * d * V
        dec += r * per
    return enc + dec, enc


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """SM clock, power and throttle reasons sampled every ~10 ms through NVML
    (the fields of the profiling recipe's nvidia-smi clocks line) on a side
    thread while the timed region runs; start() returns once the first sample
    is in, so a short timed region is still covered."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.rows, self.stop_flag, self.t = [], threading.Event(), None
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[gpu_index]) if vis and vis.split(",")[gpu_index].isdigit() else gpu_index
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_sm = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
        except Exception:
            self.nv = None
            return
        first = threading.Event()

        def run():
            nv = self.nv
            while not self.stop_flag.is_set():
                try:
                    self.rows.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)),
                                      nv.nvmlDeviceGetPowerUsage(self.h) / 1e3,
                                      int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))))
                except Exception:
                    pass
                first.set()
                self.stop_flag.wait(0.01)

        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()
        first.wait(5)
        self.rows.clear()  # keep only samples taken inside the timed region

    def stop(self):
        if self.t is None:
            return None
        self.stop_flag.set()
        self.t.join(5)
        rows = list(self.rows)
        if not rows:
            return None
        reasons = sorted(n for n, bit in self.REASONS.items() if any(r[2] & bit for r in rows))
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(rows), "power_w_max": round(max(r[1] for r in rows), 1), "source": "nvml 10 ms"}


def safe_procs(cfg_preset: str) -> int:
    """Worker processes for the reference CPU path, bounded by cores and RAM."""
    cores = os.cpu_count() or 1
    try:
        with open("/proc/meminfo") as f:
            avail_kb = next(int(l.split()[1]) for l in f if l.startswith("MemAvailable"))
    except Exception:
        avail_kb = 16 << 20
    model_gb = {"0.015B": 0.1, "0.121B": 1.4, "0.935B": 7.9, "2.633B": 42.0}.get(cfg_preset, 8.0)
    per_worker_gb = {"0.015B": 0.2, "0.121B": 1.0, "0.935B": 1.2, "2.633B": 3.0}.get(cfg_preset, 1.5)
    budget = 0.5 * avail_kb / (1 << 20) - model_gb
    by_mem = max(1, int(budget / per_worker_gb))
    return max(1, min(cores, by_mem, 64))


def run_reference_sample(preset: str, width: int, lens, procs: int, calls: int, user_begin: int = 0):
    """Reference core on `procs` worker processes: one user each (encode +
    `calls` decoder calls, extrapolated to the 1 + 2W scorer calls of a beam;
    calls < 0 runs the whole beam_search)."""
    cmd = [REF_DRIVER, "bench", "--preset", preset, "--n-users", str(procs), "--procs", str(procs),
           "--width", str(width), "--calls", str(calls), "--user-begin", str(user_begin),
           "--lens", ",".join(str(x) for x in lens)]
    out = subprocess.run(cmd, check=True, capture_output=True, text=True, timeout=1800)
    return json.loads(out.stdout.strip().splitlines()[-1])


def cpu_baseline_block(r, preset, width, kind="reference"):
    sample = (f"{r['procs']} worker processes x 1 user of {preset}: encode_eval measured "
              f"({r['t_encode_s']:.3g} s/user); " +
              (f"full beam_search W={width} measured ({r['t_beam_s']:.3g} s)" if r["beam_measured"] else
               f"{r['calls']} next_logits_eval calls measured ({r['t_call_s']:.3g} s each), beam of "
               f"1+2W={1 + 2 * width} calls extrapolated"))
    return {"value": r["users_per_s"], "unit": "users/s", "cores": r["procs"], "kind": kind, "sample": sample}


def reference_arm(args, cfg, lens):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    procs = safe_procs(args.config)
    calls = -1 if args.config in ("tiny", "0.015B") and args.width <= 32 else max(1, min(args.steps, 3))
    t0 = time.time()
    r = run_reference_sample(args.config, args.width, lens, procs, calls)
    wall = time.time() - t0
    flops_u, _ = flops_per_user(cfg, args.width, lens, fold_fc1=False)
    value = r["users_per_s"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "users/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, cfg, lens, args.gpus),
        "parallelism_detail": f"reference C++ core, {r['procs']} single-threaded worker processes on host cores",
        "cpu_baseline": cpu_baseline_block(r, args.config, args.width),
        "e2e": {"value": value, "unit": "users/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gflop_per_user": flops_u / 1e9, "wall_s": wall, "init_s": r["init_s"],
    }
    emit(line)


def parity_block(P, model, preset, width):
    """bf16 deviation of the benchmarked engine from the reference itself
    (tests/golden/paper_*.npz: the reference core's own encode / next_logits /
    beam_search outputs for users 0 and 1 at this preset; tests/golden/
    make_paper_golden.py). None when no fixture exists for the preset."""
    import glob

    import numpy as np
    tag = preset.replace(".", "")
    gold = os.path.join(ROOT, "tests", "golden")
    fx = {w: [dict(np.load(p)) for p in sorted(glob.glob(os.path.join(gold, f"paper_{tag}_u*_w{w}.npz")))]
          for w in (8, 128)}
    if not fx[8]:
        return None
    batch = P.SynthBatch(1, 0, 2)
    errs = []
    for f in fx[8]:
        u = int(f["user"])
        pres = [[int(c) for c in row if c >= 0] for row in f["prefixes"]]
        lg = model.score_prefixes(batch, [u] * len(pres), pres)
        for i in range(len(pres)):
            ref = f["logits"][i].astype(np.float64)
            errs.append(float(np.abs(lg[i] - ref).max() / np.abs(ref).max()))
    out = {"reference": "reference core (f64), tests/golden/paper_%s_*.npz" % tag, "users": 2,
           "logits_rel_err_max": max(errs), "logits_rel_err_median": float(np.median(errs)), "rows": len(errs)}
    for w in (8, 128):
        if fx[w] and w <= width:
            codes, _, _ = model.beam_search_arrays(batch, w)
            out[f"beam_overlap_at_{w}"] = [len({tuple(c) for c in codes[int(f["user"])]} &
                                               {tuple(c) for c in f["beam_codes"]}) for f in fx[w]]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="orx", choices=["orx", "reference"])
    ap.add_argument("--config", default="0.935B")
    ap.add_argument("--users", type=int, default=128, help="users per GPU per step")
    ap.add_argument("--width", type=int, default=128)
    ap.add_argument("--lens", default="20,256,2000", help="short,positive,lifelong records per user")
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--ep", action="store_true",
                    help="expert-parallel MoE over the N GPUs (peer-memory exchange, BASELINE config 4); "
                         "each rank computes n_experts / N experts (+ replicated hot ones, --ep-replicas)")
    ap.add_argument("--ep-replicas", type=int, default=None,
                    help="load-balanced expert placement: at most this many replicated experts per MoE layer, "
                         "from the expert loads of one calibration request on other users "
                         "(default n_experts / N; -1 = contiguous expert blocks, no calibration)")
    ap.add_argument("--ep-min-replicas", type=int, default=2,
                    help="replicate at least this many of each MoE layer's hottest experts (less NVLink traffic, "
                         "more expert memory per GPU; the line reports expert_slots_per_gpu)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    lens = tuple(int(x) for x in args.lens.split(","))

    cfg = BenchConfig(args.config)
    if args.impl == "reference":  # never imports the package (no liborx.so in this process)
        reference_arm(args, cfg, lens)
        return

    import paper_2506_13695_b200 as P
    from paper_2506_13695_b200._lib import check, lib, orx_beam_out
    pcfg = P.PolicyConfig.preset(args.config)

    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        quiet_stdout()
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    t_init = time.time()
    ep = args.ep and world > 1 and cfg.moe_enabled
    ep_info = None
    if ep:
        from paper_2506_13695_b200.dist import ep_unique_id, shard_users as _shard

        def ep_model(owner):
            uid = ep_unique_id(device=torch.device("cuda", local))
            return P.PolicyModel(weights=P.Weights.random_ep(pcfg, rank, world, owner=owner), precision=args.precision,
                                 device=local, max_users=args.users, max_width=args.width, ep=(rank, world, uid),
                                 ep_owner=owner)
        model = ep_model(None)
        reps = args.ep_replicas if args.ep_replicas is not None else pcfg.n_experts // world
        if reps >= 0:
            # expert placement from one calibration request on OTHER users (the loads
            # are all-gathered, so every rank computes the same placement)
            cb, cn = _shard(rank, world, args.users)
            calib = P.SynthBatch(7, 1_000_000 + cb, cn, *lens)
            model.beam_search_arrays(calib, args.width)
            owner, pred = P.ep_place(model.expert_load(), world, reps, min(args.ep_min_replicas, reps))
            del model
            model = ep_model(owner)
            ep_info = {"placement": "load-balanced (calibration: 1 request, other users, seed 7)",
                       "max_replicas": reps, "min_replicas": min(args.ep_min_replicas, reps),
                       "replicated_per_layer": float((owner < 0).sum(axis=1).mean()),
                       "expert_slots_per_gpu": int(max(((owner == q) | (owner < 0)).sum(axis=1).max()
                                                       for q in range(world))),
                       "experts_per_layer": int(pcfg.n_experts),
                       "predicted_busiest_over_mean": [round(float(x), 3) for x in pred]}
        else:
            ep_info = {"placement": "contiguous expert blocks"}
    else:
        model = P.PolicyModel(pcfg, precision=args.precision, device=local, max_users=args.users,
                              max_width=args.width)
    t_init = time.time() - t_init
    from paper_2506_13695_b200.dist import shard_users
    user_begin, n_users = shard_users(rank, world, args.users)
    batch = P.SynthBatch(1, user_begin, n_users, *lens)
    e = model._e
    L = cfg.n_code_layers
    stream = torch.cuda.ExternalStream(lib().orx_engine_stream(e), device=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    from paper_2506_13695_b200.dist import max_over_ranks as _mor

    def max_over_ranks(x):
        return _mor(x, device=torch.device("cuda", local))

    # ---- device-resident timing -------------------------------------------------------
    check(lib().orx_engine_stage_batch(e, C.byref(batch.c)))
    for _ in range(args.warmup):
        check(lib().orx_beam_search_staged(e, args.width, None))
    st0 = model.stats()
    barrier()
    sampler = ClockSampler(local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        check(lib().orx_beam_search_staged(e, args.width, None))
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    clocks = sampler.stop()
    st1 = model.stats()
    ms = ev0.elapsed_time(ev1)
    ms_max = max_over_ranks(ms)
    launches = st1["launches"] - st0["launches"]
    value = world * args.users * args.steps / (ms_max / 1e3)

    # ---- end-to-end through the public API (host buffers) -----------------------------------
    e2e_steps = args.e2e_steps or max(3, args.steps)
    codes = (C.c_int32 * (args.users * args.width * L))()
    logp = (C.c_double * (args.users * args.width))()
    nitems = (C.c_int32 * args.users)()
    out = orx_beam_out(C.cast(codes, C.POINTER(C.c_int32)), C.cast(logp, C.POINTER(C.c_double)),
                       C.cast(nitems, C.POINTER(C.c_int32)))
    check(lib().orx_beam_search(e, C.byref(batch.c), args.width, C.byref(out)))  # warm the pinned buffers
    s0 = model.stats()
    barrier()
    w0 = time.perf_counter()
    ev0.record(stream)
    for _ in range(e2e_steps):
        check(lib().orx_beam_search(e, C.byref(batch.c), args.width, C.byref(out)))
    ev1.record(stream)
    ev1.synchronize()
    w1 = time.perf_counter()
    barrier()
    s1 = model.stats()
    e2e_ms = max(ev0.elapsed_time(ev1), (w1 - w0) * 1e3)
    e2e_ms_max = max_over_ranks(e2e_ms)
    e2e_sync_value = world * args.users * e2e_steps / (e2e_ms_max / 1e3)

    # pipelined serving through orx_beam_search_submit / _collect: request i+1
    # is validated, packed and copied (copy stream) while request i runs; every
    # request still carries its own H2D and D2H inside the timed region
    check(lib().orx_beam_search_submit(e, C.byref(batch.c), args.width))
    check(lib().orx_beam_search_collect(e, C.byref(out)))  # warm both staging slots
    p0 = model.stats()
    barrier()
    w0 = time.perf_counter()
    ev0.record(stream)
    check(lib().orx_beam_search_submit(e, C.byref(batch.c), args.width))
    for i in range(e2e_steps):
        if i + 1 < e2e_steps:
            check(lib().orx_beam_search_submit(e, C.byref(batch.c), args.width))
        check(lib().orx_beam_search_collect(e, C.byref(out)))
    ev1.record(stream)
    ev1.synchronize()
    w1 = time.perf_counter()
    barrier()
    p1 = model.stats()
    pipe_ms = max(ev0.elapsed_time(ev1), (w1 - w0) * 1e3)
    pipe_ms_max = max_over_ranks(pipe_ms)
    e2e_value = world * args.users * e2e_steps / (pipe_ms_max / 1e3)
    assert p1["h2d_bytes"] - p0["h2d_bytes"] == s1["h2d_bytes"] - s0["h2d_bytes"]  # same copies per request
    h2d = (s1["h2d_bytes"] - s0["h2d_bytes"]) // e2e_steps
    d2h = (s1["d2h_bytes"] - s0["d2h_bytes"]) // e2e_steps

    # ---- per-kernel-class timing (one instrumented step) -------------------------------------
    check(lib().orx_profile_enable(1))
    check(lib().orx_beam_search_staged(e, args.width, None))
    torch.cuda.synchronize()
    n = len(PROF_NAMES)
    pl, pms, pfl, pby = (C.c_int64 * n)(), (C.c_double * n)(), (C.c_double * n)(), (C.c_double * n)()
    check(lib().orx_profile_read(n, pl, pms, pfl, pby))
    check(lib().orx_profile_enable(0))
    peaks, peak_src = load_peaks()
    hbm_peak = peaks.get("hbm_gbs")
    classes = {}
    for i in range(n):
        c = {"launches": pl[i], "ms": round(pms[i], 4),
             "tflops": (pfl[i] / (pms[i] * 1e-3) / 1e12) if pms[i] > 0 and pfl[i] > 0 else None}
        if pby[i] > 0 and pms[i] > 0:  # HBM-bound classes: algorithmic bytes / time vs the measured copy bandwidth
            c["gbs"] = pby[i] / (pms[i] * 1e-3) / 1e9
            c["frac_hbm"] = c["gbs"] / hbm_peak if hbm_peak else None
            c["bytes_per_step"] = pby[i]
        classes[PROF_NAMES[i]] = c
    prof_total = sum(pms[i] for i in range(n))
    gemm_ms = pms[0] + pms[1]
    gemm_launch = pl[0] + pl[1]
    gemm_flops = pfl[0] + pfl[1]
    achieved = gemm_flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    roofline = {"bound": "tensor", "kernel": "tc_gemm_kernel (tcgen05 dense + grouped MoE GEMMs)",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None, "traffic": None,
                "peak_kind": f"bf16_tflops_sustained ({peak_src}); kernel timed inside a long step",
                "flops_per_launch": gemm_flops / max(gemm_launch, 1),
                "ms_per_launch": gemm_ms / max(gemm_launch, 1),
                "share_of_step": gemm_ms / prof_total if prof_total else None}
    traffic_path = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(traffic_path):
        try:
            with open(traffic_path) as f:
                roofline["traffic"] = json.load(f).get("bytes_per_launch")
        except Exception:
            pass

    bf16 = args.precision == "bf16"
    flops_u, enc_flops_u = flops_per_user(cfg, args.width, lens, fold_fc1=bf16, fold_kv=bf16)
    mfu = value / world * flops_u / (peaks["bf16_tflops"] * 1e12)

    # ---- measured deviation from the reference (rank 0) ------------------------------------
    parity = None
    if rank == 0 and args.precision == "bf16":
        try:
            parity = parity_block(P, model, args.config, args.width)
        except Exception as ex:  # reported, not fatal
            parity = {"error": str(ex)}

    # ---- CPU baseline (rank 0, N=1 only) --------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and os.path.exists(REF_DRIVER):
        try:
            procs = safe_procs(args.config)
            r = run_reference_sample(args.config, args.width, lens, procs, 3)
            cpu = cpu_baseline_block(r, args.config, args.width)
        except Exception as ex:  # reported, not fatal
            cpu = {"value": None, "unit": "users/s", "cores": None, "kind": "reference", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "users/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16" if args.precision == "bf16" else "fp32", "data": "synthetic",
            "config": bench_config(args, cfg, lens, world),
            "parallelism_detail": (f"dp{world} x ep{world} (users sharded; MoE experts sharded, NCCL all-to-all "
                                   f"dispatch/combine over NVLink)") if ep else
                                  f"dp{world} (users sharded, no inter-GPU traffic)",
            "mfu": mfu, "mfu_peak": "bf16_tflops (burst) of MEASURED_PEAKS.json",
            "gflop_per_user": flops_u / 1e9, "gflop_per_user_encoder": enc_flops_u / 1e9,
            "e2e": {"value": e2e_value, "unit": "users/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps,
                    "api": "orx_beam_search_submit / orx_beam_search_collect: the serving loop, two requests in "
                           "flight; every request's host batch is validated, packed and copied H2D and its beams "
                           "copied D2H inside the timed region",
                    "sync_value": e2e_sync_value,
                    "sync_api": "orx_beam_search (one request at a time, host batch in, host beams out)"},
            "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
            "roofline": roofline, "kernel_classes_ms_per_step": classes,
            "cpu_baseline": cpu, "clocks": clocks, "init_s": t_init, "parity": parity,
        }
        if ep_info:
            line["expert_parallel"] = ep_info
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
