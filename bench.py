#!/usr/bin/env python
"""Benchmark of the SeeD draft-then-verify round (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config sweep] [--impl ours|reference]

One step = one whole round of the hot path: FCFS admission, gamma
batched draft steps, the batched target verify forward, the fused vocabulary kernel, KV
rollback and (N > 1) the all-gather of the exchange blocks.  Workload (default): BASELINE
configs[4], the scaling sweep the metric is quoted on -- 24 streams per GPU, 68M-shape draft,
Llama-2-7B-shape target, gamma = 4, prompts of 300-500 tokens, random-init weights, synthetic
prompts (seedgen).  With N GPUs each rank runs a full replica with its own 24 streams (weak
scaling; the rank's streams have global ids rank, rank + N, ...).  --config gsm8k / cw / bw
select the other BASELINE shapes.

Prints one JSON line (rank 0).  --impl reference times the CPU oracle (oracle/) on the same
config as a bounded sample per step.
"""
import argparse
import json
import os
import statistics
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
    ap.add_argument("--config", default="sweep", choices=["gsm8k", "cw", "bw", "sweep", "toy"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--temperature", type=float, default=1.0)
    ap.add_argument("--streams", type=int, default=0, help="streams per GPU (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tree", default="", help="k_config tree rounds, e.g. 2,2,1 (default: the chain)")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 6650.0, 1590.0, "fallback"


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return "unknown"


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


def traffic_from_profiles(config):
    """DRAM bytes per K2 launch from the committed ncu capture of this config (profiles/)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        v = d.get(config, {})
        return v.get("k2_gemm") if isinstance(v, dict) else None
    return None


# ------------------------------------------------------------------ CPU oracle timing
def _synthetic_cache(shape, n, rng):
    """An oracle KV cache holding n positions of bf16-valued synthetic keys / values (timing only:
    the bounded CPU sample skips the prefill, which is not part of a round)."""
    import torch

    from oracle import llama as ll
    c = ll.KVCache(shape)
    for layer in range(shape.n_layers):
        for lst in (c.k, c.v):
            t = torch.from_numpy(rng.standard_normal((n, shape.kv_heads, shape.head_dim)).astype(np.float32))
            lst[layer] = t.to(torch.bfloat16).to(torch.float64).numpy()
    return c


class OracleSampler:
    """Times oracle rounds of a config's batch on a bounded sample: the full draft (every layer of
    the draft model, gamma steps), the target verify forward on `target_layers` of its layers
    (scaled to full depth: the per-layer time only), the final norm + LM head once, and the full
    verification (oracle.sampling.verify_stream).  The prefill is replaced by synthetic caches of
    the prompts' lengths (built once, rolled back after every sample)."""

    def __init__(self, cfg_name, temperature, n_streams, target_layers=1):
        from oracle import llama as ll
        from oracle.seed_round import SeedOracle, StreamState
        self.cfg = seedgen.CONFIGS[cfg_name]
        self.name, self.T, self.n = cfg_name, temperature, n_streams
        ds, ts = seedgen.SHAPES[self.cfg["draft"]], seedgen.SHAPES[self.cfg["target"]]
        self.L_full = ts["n_layers"]
        self.tl = min(target_layers, ts["n_layers"])
        self.dW = seedgen.model_weights(ds, seedgen.DRAFT_SEED)
        self.tW = seedgen.model_weights(dict(ts, n_layers=self.tl), seedgen.TARGET_SEED)
        self.dsh, self.tsh = ll.LlamaShape(**ds), ll.LlamaShape(**dict(ts, n_layers=self.tl))
        self.orc = SeedOracle(self.tsh, self.tW, self.dsh, self.dW, gamma=self.cfg["gamma"], temperature=temperature,
                              seed=seedgen.PHILOX_SEED, max_new=10 ** 6)
        rng = np.random.default_rng(0)
        for i, p in enumerate(seedgen.prompts(cfg_name, n_streams=n_streams)):
            self.orc.streams[i] = StreamState(sid=i, T=list(p), prompt_len=len(p),
                                              tcache=_synthetic_cache(self.tsh, len(p) - 1, rng),
                                              dcache=_synthetic_cache(self.dsh, len(p) - 1, rng))

    def sample(self, r=0):
        """One round (stream-local round r); returns (estimated s per full round, measured s, emitted)."""
        from oracle import llama as ll
        from oracle import sampling as sp
        orc, g = self.orc, self.cfg["gamma"]
        batch = list(range(self.n))
        for s in batch:
            orc.streams[s].r = r
        t0 = time.perf_counter()
        xs, zds, _ = orc.draft(batch)
        t1 = time.perf_counter()
        # the target layers (the LM head is timed once below, not scaled)
        seqs = [([orc.streams[s].T[-1]] + xs[s], orc.streams[s].tcache) for s in batch]
        ll.forward_batch(self.tsh, self.tW, seqs, mode="bf16", logits_rows=[[]] * len(seqs))
        t2 = time.perf_counter()
        xh = np.zeros((self.n * (g + 1), self.tsh.d_model))
        zt_all = ll.f32_round(ll.norm_matmul(xh, ll._w(self.tW["final_norm"]), [ll._w(self.tW["lm_head"])],
                                             self.tsh.rms_eps, True)[0])
        t3 = time.perf_counter()
        emitted = 0
        for k, s in enumerate(batch):
            zt = zt_all[k * (g + 1):(k + 1) * (g + 1)] + 0.1 * np.stack(zds[s] + [zds[s][-1]])   # synthetic rows
            res = sp.verify_stream(zt, np.stack(zds[s]), xs[s], self.T, seedgen.PHILOX_SEED, s, r)
            emitted += len(res.emitted)
        t4 = time.perf_counter()
        for s in batch:                      # roll the caches back to the prompt
            st = orc.streams[s]
            st.tcache.truncate(st.prompt_len - 1)
            st.dcache.truncate(st.prompt_len - 1)
        est = (t1 - t0) + (t2 - t1) * (self.L_full / self.tl) + (t3 - t2) + (t4 - t3)
        return est, t4 - t0, emitted

    def describe(self):
        return (f"one {self.name} round, {self.n} streams (prefill replaced by synthetic caches of the prompts' "
                f"lengths): full draft, target forward on {self.tl} of {self.L_full} layers (layer time "
                f"x{self.L_full / self.tl:g}), final norm + LM head once, full verification on the draft rows + "
                f"the head output")


def config_of(args, cfg, n_local, world):
    """The workload description shared by both arms' JSON lines."""
    tree = [int(c) for c in args.tree.split(",")] if getattr(args, "tree", "") else None
    extra = {"k_config": tree} if tree else {}
    return {"workload": args.config, "streams_per_gpu": n_local, "gamma": len(tree) if tree else cfg["gamma"],
            **extra, "draft": cfg["draft"],
            "target": cfg["target"], "prompt_len": list(cfg["prompt_len"]), "temperature": args.temperature,
            "parallelism": f"replicas x{world}",
            "l2": "inputs larger than L2: all target weights (13.2 GB at 7B) streamed every round"}


def run_reference(args):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = seedgen.CONFIGS[args.config]
    n = args.streams or cfg["n_streams"]
    smp = OracleSampler(args.config, args.temperature, n)
    for w in range(args.warmup):
        smp.sample(r=w)
    est, meas, emitted = [], [], 0
    for k in range(args.steps):
        t, m, e = smp.sample(r=args.warmup + k)
        est.append(t)
        meas.append(m)
        emitted += e
    v = emitted / sum(est)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(meas) / args.steps,
            "ms_per_round_estimate": 1e3 * sum(est) / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(args, cfg, n, int(os.environ.get("WORLD_SIZE", "1"))),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "oracle",
                             "cpu": cpu_model(),
                             "sample": smp.describe() + "; ms_per_step is the measured time of one sample, value = "
                                                        "emitted tokens / estimated full-round time"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def exposed_by_kind(tr):
    """Critical-path time per launch kind from one round's device trace: launch i owns
    [max(release_i, end_{i-1}), end_i] -- a partition of the round's traced timeline (PDL overlaps
    each kernel's prologue and prefetch with its predecessor; that time is the predecessor's)."""
    out = {1: 0.0, 2: 0.0}
    prev = None
    for s, r, e, k in tr:
        beg = max(r, prev) if prev is not None else r
        out[int(k)] = out.get(int(k), 0.0) + max(0, e - beg)
        prev = e if prev is None else max(prev, e)
    return out


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
    tree = [int(c) for c in args.tree.split(",")] if args.tree else None
    g = len(tree) if tree else cfg["gamma"]
    rows = 1 + sum(int(np.prod(tree[:d + 1])) for d in range(len(tree))) if tree else g + 1
    n_local = args.streams or cfg["n_streams"]
    ds, ts = seedgen.SHAPES[cfg["draft"]], seedgen.SHAPES[cfg["target"]]
    steps, warm = args.steps, args.warmup
    prompts = seedgen.prompts(args.config, n_streams=n_local * world)
    max_prompt = max(len(p) for p in prompts)
    # e2e pass adds another warm + steps rounds; a stream must not finish inside any timed region
    prof_rounds = max(3, min(steps, 10))   # profiled rounds for the roofline, after the timed ones
    max_new = (2 * (steps + warm) + prof_rounds + 6) * (g + 1)
    max_ctx = max_prompt + max_new + max(g, rows) + 8

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
                         world=world, nccl_id=nccl_id, profile=True, tree=tree)
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
        b = eng.schedule()     # every rank runs every round (an empty batch still joins the exchange)
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
    per_stream_round = emitted / (steps * len(my_ids))
    # mean target context over the timed rounds (prompt + tokens before + half of those emitted during)
    ctx_mean = statistics.mean(len(prompts[gid]) + t_before[gid] + 0.5 * (eng.stream_info(gid)["L"] - t_before[gid])
                               for gid in my_ids)

    # e2e: the same rounds through the public host-buffer call seed_round_host (batch ids in,
    # emitted tokens + counts out, every round), wall clock around the K rounds
    for _ in range(warm):
        eng.round_host(eng.schedule())
    eng.schedule(0)
    t2 = {gid: eng.stream_info(gid)["L"] for gid in my_ids}
    barrier()
    h2d = d2h = 0
    w0 = time.perf_counter()
    for _ in range(steps):
        b = eng.schedule()
        eng.round_host(b)
        h2d += 4 * len(b)
        d2h += 4 * len(b) * (g + 2)
    eng.schedule(0)
    w1 = time.perf_counter()
    barrier()
    ms_e2e = (w1 - w0) * 1e3
    emitted_e2e = sum(eng.stream_info(gid)["L"] - t2[gid] for gid in my_ids)

    # roofline of K2 from separate, profiled rounds: device %globaltimer records of every GEMM and
    # attention launch; each launch owns its critical-path interval (exposed_by_kind)
    eng.set_profile(True)
    one_round()
    eng.schedule(0)
    eng.reset_profile()
    k2_ns, k3_ns, round_ns = [], [], []
    for _ in range(prof_rounds):
        one_round()
        eng.schedule(0)
        tr = eng.launch_trace()
        ex = exposed_by_kind(tr)
        k2_ns.append(ex.get(1, 0.0))
        k3_ns.append(ex.get(2, 0.0))
        round_ns.append(float(tr[:, 2].max() - tr[:, 0].min()))
    torch.cuda.synchronize()
    prof = eng.profile()
    eng.set_profile(False)

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
    n_gemm = max(prof["gemm_launches"], 1)
    bytes_per_launch = prof["gemm_bytes"] / n_gemm
    launches_per_round = n_gemm / prof_rounds
    k2_us = statistics.median(k2_ns) * 1e-3 / launches_per_round        # exposed time per K2 launch
    achieved = bytes_per_launch / (k2_us * 1e-6) / 1e9
    rel_us = prof["gemm_ms"] / n_gemm * 1e3                              # release -> end per launch
    step_ms = ms / steps
    line = {
        "metric": METRIC, "value": emitted / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init weights, seedgen prompts)",
        "config": config_of(args, cfg, n_local, world),
        "emitted_per_stream_round": per_stream_round,
        "verified_positions_per_s": world * n_local * rows / (step_ms * 1e-3),
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": "gemm_splitk_kernel (K2)", "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "peak_source": peak_src,
                     "traffic": traffic_from_profiles(args.config), "bytes_per_launch": bytes_per_launch,
                     "launches_per_round": launches_per_round, "exposed_us_per_launch": k2_us,
                     "timing": ("device %globaltimer over " + str(prof_rounds) + " profiled rounds after the timed "
                                "ones: each GEMM launch is charged its critical-path interval [max(its release, "
                                "the previous launch's end), its end], so the weight prefetch it overlaps with its "
                                "predecessor is the predecessor's time; share = K2 time / traced round span"),
                     "k2_share_of_round": statistics.median(k2_ns) / statistics.median(round_ns),
                     "k3_share_of_round": statistics.median(k3_ns) / statistics.median(round_ns),
                     "frac_release_to_end": bytes_per_launch / (rel_us * 1e-6) / 1e9 / hbm,
                     "frac_round_level": (launches_per_round * bytes_per_launch) / (step_ms * 1e-3) / 1e9 / hbm},
        "e2e": {"value": emitted_e2e / (ms_e2e * 1e-3), "unit": UNIT, "ms_per_step": ms_e2e / steps,
                "h2d_bytes_per_step": h2d // steps, "d2h_bytes_per_step": d2h // steps,
                "timing": "wall clock (perf_counter) around the K seed_round_host rounds, host-synchronised"},
        "clocks": clk,
    }
    # the north-star number: T_roof / T per round (sum over phases of max(bytes / HBM,
    # flops / sustained bf16), at this run's mean context; scripts/troof.py)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "scripts"))
    from troof import troof
    tr = troof(args.config, n_local, ctx_mean, rows=rows, draft_steps=g)
    line["round_roofline"] = {"t_roof_ms": tr["t_roof_ms"], "t_round_ms": step_ms, "frac": tr["t_roof_ms"] / step_ms,
                              "ctx_mean": ctx_mean, "phases_ms": tr["phases_ms"],
                              "definition": "SURVEY 8(d): T_roof = sum_phase max(B/BW_hbm, F/F_bf16_sustained), "
                                            "phases GEMM / attention / draft / vocab; north_star bar 0.60"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import torch as _t
        smp = OracleSampler(args.config, args.temperature, n_local)
        runs = [smp.sample(r=k) for k in range(3)]
        est = statistics.median(x[0] for x in runs)
        line["cpu_baseline"] = {"value": runs[0][2] / est, "unit": UNIT, "cores": _t.get_num_threads(),
                                "kind": "oracle", "cpu": cpu_model(), "sample": smp.describe() + "; median of 3"}
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
