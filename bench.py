#!/usr/bin/env python
"""Benchmark of the SeeD draft-then-verify round (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config gsm8k] [--impl ours|reference]

One step = one whole round of the hot path: FCFS admission, gamma
batched draft steps, the batched target verify forward, the fused vocabulary kernel, KV
rollback and (N > 1) the all-gather of emitted tokens.  Workload (N = 1): BASELINE configs[1],
the GSM8K shape -- 3 streams, 68M-shape draft, Llama-2-7B-shape target, gamma = 4, random-init
weights, synthetic prompts (seedgen).  With N GPUs each rank runs a full replica with its own
streams (weak scaling; the rank's streams have global ids rank, rank + N, ...).

Prints one JSON line (rank 0).  --impl reference times the CPU oracle (oracle/) on the same
config as a bounded sample per step.
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import seedgen  # noqa: E402

METRIC = "accepted tokens/sec per round (device-timed)"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="gsm8k", choices=["gsm8k", "cw", "bw", "sweep", "toy"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--temperature", type=float, default=1.0)
    ap.add_argument("--streams", type=int, default=0, help="streams per GPU (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None

    def start(self):
        """Start sampling and return once the first sample arrived (so NVML start-up is not timed)."""
        self.first = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", "20"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.first = self.proc.stdout.readline()
        except OSError:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        out = (self.first or "") + out
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def traffic_from_profiles(kernel="k2_gemm"):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(kernel)
    return None


# ------------------------------------------------------------------ CPU oracle timing
def oracle_round_sample(cfg_name, temperature, n_streams, target_layers=2, rank_seed=0):
    """Time one oracle round on a bounded sample: the full draft, the target forward on
    `target_layers` of its layers (scaled to full depth), the full verification.
    Returns (estimated seconds per round, emitted tokens, description)."""
    import torch

    from oracle import llama as ll
    from oracle.seed_round import SeedOracle
    cfg = seedgen.CONFIGS[cfg_name]
    ds, ts = seedgen.SHAPES[cfg["draft"]], seedgen.SHAPES[cfg["target"]]
    tl = min(target_layers, ts["n_layers"])
    ts_s = dict(ts, n_layers=tl)
    dW = seedgen.model_weights(ds, seedgen.DRAFT_SEED)
    tW = seedgen.model_weights(ts_s, seedgen.TARGET_SEED)
    orc = SeedOracle(ll.LlamaShape(**ts_s), tW, ll.LlamaShape(**ds), dW, gamma=cfg["gamma"],
                     temperature=temperature, seed=seedgen.PHILOX_SEED, max_new=10 ** 6)
    prompts = seedgen.prompts(cfg_name, n_streams=n_streams)
    for i, p in enumerate(prompts):
        orc.add_stream(i, p)
    batch = list(range(n_streams))
    t0 = time.perf_counter()
    xs, zds, gaps = orc.draft(batch)
    t1 = time.perf_counter()
    zts = orc.verify(batch, xs)
    t2 = time.perf_counter()
    from oracle import sampling as sp
    emitted = 0
    for s in batch:
        st = orc.streams[s]
        r = sp.verify_stream(zts[s], np.stack(zds[s]), xs[s], temperature, seedgen.PHILOX_SEED, s, st.r)
        emitted += len(r.emitted)
    t3 = time.perf_counter()
    scale = ts["n_layers"] / tl
    est = (t1 - t0) + (t2 - t1) * scale + (t3 - t2)
    desc = (f"one {cfg_name} round, {n_streams} streams: full draft, target forward on {tl} of "
            f"{ts['n_layers']} layers scaled x{scale:g}, full verification; prefill excluded")
    return est, emitted, desc, torch.get_num_threads()


def config_of(args, cfg, n_local, world):
    """The workload description shared by both arms' JSON lines."""
    return {"workload": args.config, "streams_per_gpu": n_local, "gamma": cfg["gamma"], "draft": cfg["draft"],
            "target": cfg["target"], "temperature": args.temperature, "parallelism": f"replicas x{world}",
            "l2": "inputs larger than L2: all target weights (13.2 GB at 7B) streamed every round"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = seedgen.CONFIGS[args.config]
    n = args.streams or cfg["n_streams"]
    for _ in range(args.warmup):
        oracle_round_sample(args.config, args.temperature, n, target_layers=1)
    tot_t, tot_e = 0.0, 0
    desc, cores = "", os.cpu_count()
    for _ in range(args.steps):
        t, e, desc, cores = oracle_round_sample(args.config, args.temperature, n, target_layers=1)
        tot_t += t
        tot_e += e
    v = tot_e / tot_t
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(args, cfg, n, int(os.environ.get("WORLD_SIZE", "1"))),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2406_18200_b200 as pkg

    cfg = seedgen.CONFIGS[args.config]
    g = cfg["gamma"]
    n_local = args.streams or cfg["n_streams"]
    ds, ts = seedgen.SHAPES[cfg["draft"]], seedgen.SHAPES[cfg["target"]]
    steps, warm = args.steps, args.warmup
    prompts = seedgen.prompts(args.config, n_streams=n_local * world)
    max_prompt = max(len(p) for p in prompts)
    # e2e pass adds another warm + steps rounds; a stream must not finish inside any timed region
    prof_rounds = max(3, min(steps, 10))   # profiled rounds for the roofline, after the timed ones
    max_new = (2 * (steps + warm) + prof_rounds + 6) * (g + 1)
    max_ctx = max_prompt + max_new + g + 8

    # random-init weights drawn on the device (same recipe as seedgen on CPU)
    dW = seedgen.model_weights(ds, seedgen.DRAFT_SEED, device="cuda")
    tW = seedgen.model_weights(ts, seedgen.TARGET_SEED, device="cuda")
    nccl_id = None
    if world > 1:
        obj = [pkg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    eng = pkg.SeedEngine(ds, dW, ts, tW, gamma=g, temperature=args.temperature, seed=seedgen.PHILOX_SEED,
                         max_new=max_new, max_streams=n_local, max_batch=n_local, max_ctx=max_ctx, rank=rank,
                         world=world, nccl_id=nccl_id, profile=True)
    del dW, tW
    torch.cuda.empty_cache()
    eng.set_profile(False)   # the timed rounds run without the device timing records
    my_ids = [i for i in range(n_local * world) if i % world == rank]
    for gid in my_ids:
        eng.add_stream(gid, prompts[gid])
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def one_round():
        b = eng.schedule()
        eng.draft(b)
        eng.verify(b)
        return len(b)

    for _ in range(warm):
        one_round()
    eng.schedule(0)  # complete the last warm-up round on the host
    t_before = {gid: eng.stream_info(gid)["L"] for gid in my_ids}
    eng.reset_profile()
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        one_round()
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    launches = eng.profile()["kernel_launches"]
    ms = e0.elapsed_time(e1)
    emitted = sum(eng.stream_info(gid)["L"] - t_before[gid] for gid in my_ids)
    alpha_rounds = emitted / (steps * len(my_ids))

    # e2e: the same rounds through seed_round_host (host in, host out)
    for _ in range(warm):
        eng.round_host(eng.schedule())
    eng.schedule(0)
    t2 = {gid: eng.stream_info(gid)["L"] for gid in my_ids}
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    h2d = d2h = 0
    for _ in range(steps):
        b = eng.schedule()
        eng.round_host(b)
        h2d += 4 * len(b)
        d2h += 4 * len(b) * (g + 2)
    f1.record(stream)
    barrier()
    ms_e2e = f0.elapsed_time(f1)
    emitted_e2e = sum(eng.stream_info(gid)["L"] - t2[gid] for gid in my_ids)

    # roofline of K2 from separate, profiled rounds (device %globaltimer records per launch)
    eng.schedule(0)
    eng.set_profile(True)
    one_round()
    eng.schedule(0)
    eng.reset_profile()
    for _ in range(prof_rounds):
        one_round()
    eng.schedule(0)
    torch.cuda.synchronize()
    prof = eng.profile()

    # max over ranks of the device time, sum of the work
    vals = torch.tensor([ms, ms_e2e, float(emitted), float(emitted_e2e)], dtype=torch.float64, device="cuda")
    if world > 1:
        mx = vals[:2].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals[2:].clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        vals = torch.cat([mx, sm])
    ms, ms_e2e, emitted, emitted_e2e = vals.tolist()
    hbm, tf, peak_src = measured_peaks()
    gemm_avg_ms = prof["gemm_ms"] / max(prof["gemm_launches"], 1)
    gemm_bytes = prof["gemm_bytes"] / max(prof["gemm_launches"], 1)
    achieved = gemm_bytes / (gemm_avg_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": emitted / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": ms / steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init weights, seedgen prompts)",
        "config": config_of(args, cfg, n_local, world),
        "emitted_per_stream_round": alpha_rounds,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": "gemm_splitk_kernel (K2)", "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "peak_source": peak_src,
                     "traffic": traffic_from_profiles(), "launches": prof["gemm_launches"],
                     "gemm_share_of_step": (prof["gemm_ms"] / prof_rounds) / (ms / steps) if world == 1 else None,
                     "bytes_per_launch": gemm_bytes, "avg_launch_us": gemm_avg_ms * 1e3,
                     "timing": "device %globaltimer per launch: dependency release -> last CTA end "
                               "(the weight prefetch overlapped with the predecessor under PDL is not counted), "
                               f"over {prof_rounds} profiled rounds run after the timed ones",
                     "avg_span_us": prof["gemm_span_ms"] / max(prof["gemm_launches"], 1) * 1e3},
        "e2e": {"value": emitted_e2e / (ms_e2e * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d // steps,
                "d2h_bytes_per_step": d2h // steps},
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        t, e, desc, cores = oracle_round_sample(args.config, args.temperature, n_local)
        line["cpu_baseline"] = {"value": e / t, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
