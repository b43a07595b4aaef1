#!/usr/bin/env python
"""Benchmark of the hot path: packed tokens/s of tri-model log-prob + GRPO loss
(+ policy backward, + gradient allreduce at N>1) on shared-prompt packed groups.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

A step = one global batch of prompt groups (C2 N=64 groups), split
over the ranks (pack -> tri-model forward -> GRPO loss -> policy backward ->
accumulate per group), then the gradient and the loss scalars are allreduced over
NCCL (N>1).  Strong scaling: the global batch is fixed as N grows.  The SGD update
(set N*G, snapshot, apply_update) is timed separately, outside the metric.

Prints ONE JSON line (rank 0).  `value` = device-resident inputs, CUDA-event
timed; `e2e` = the same through the public C-ABI from pinned host buffers with
H2D/D2H inside the timed region, measured right after `value`'s leg; `roofline` =
the dominant kernel class, every launch timed with CUDA events on its launch
stream over min(K, 4) further identical steps (a profiling leg kept out of
`value` and `e2e`); `cpu_baseline` = the
reference (oracle/_ref, built from the reference's own sources) on a bounded
sample it really executes, measured tokens/s (a FLOP-model extrapolation to this
workload is reported separately).  C2 packs 4 prompt groups per sequence (--pack).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[0]: tiny decoder, fp32 (CPU-runnable oracle case)
    "c1": dict(vocab=4096, d=256, L=2, H=4, F=1024, max_seq=576, P=64, G=4, R=128, prec="fp32", groups=8, pack=4),
    # BASELINE.json configs[1]: Qwen2.5-0.5B-shaped random-init tri-model, G=8, 512+1k, bf16, single B200
    # 4 prompt groups per packed sequence (each group shared-prompt packed as pack_group does)
    "c2": dict(vocab=151936, d=896, L=24, H=14, F=4864, max_seq=16384, P=512, G=8, R=1024, prec="bf16", groups=64,
               pack=4),
    # configs[2]: Qwen2.5-7B-shaped tri-model, G=16, 1k prompt + 4k responses (T=66,560 per group),
    # one group per rank (prompt groups sharded over the GPUs); runs with activation recomputation
    "c3": dict(vocab=152064, d=3584, L=28, H=28, F=18944, max_seq=66560, P=1024, G=16, R=4096, prec="bf16",
               groups=16),
    # configs[3]: long-CoT ragged batch, Qwen2.5-1.5B shape, 2k prompt + 8 responses of 1k-16k tokens
    # (SURVEY.md 8d seed: random.Random(20251118).randint(1024, 16384), group 0; T=87,893)
    "c4": dict(vocab=151936, d=1536, L=28, H=12, F=8960, max_seq=90112, P=2048, G=8, R=None, prec="bf16", groups=16,
               lens=[15781, 14233, 10574, 3139, 3977, 14992, 13452, 9697]),
}


def group_lens(c):
    return list(c["lens"]) if c.get("lens") else [c["R"]] * c["G"]
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")


def flops_per_group(c, P, lens, reference_head=False):
    """Algorithmic FLOPs of one micro-step:
    fwd = 2 T L (4d^2 + 2dF) + 4 pairs d L + 2 rows d V; tri-model = 3 fwd;
    policy bwd = 2x GEMM terms + 2.5x attention term + 2x head term."""
    d, L, F, V = c["d"], c["L"], c["F"], c["vocab"]
    T = P + sum(lens)
    pairs = P * (P + 1) / 2 + sum(r * P + r * (r + 1) / 2 for r in lens)
    rows = T if reference_head else 1 + sum(r - 1 for r in lens)
    gemm = 2.0 * T * L * (4 * d * d + 2 * d * F)
    attn = 4.0 * pairs * d * L
    head = 2.0 * rows * d * V
    return 3 * (gemm + attn + head) + 2 * gemm + 2.5 * attn + 2 * head


def measured_traffic(cls):
    """DRAM bytes per launch of a kernel class from the newest committed ncu traffic
    summary (profiles/rNN_traffic.json, scripts/traffic.py), or None."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    if not files:
        return None, None
    try:
        with open(files[-1]) as f:
            d = json.load(f)
        return d["classes"][cls]["dram_bytes_per_launch"], os.path.relpath(files[-1], ROOT)
    except Exception:
        return None, None


def sm_max_mhz():
    try:
        with open(MEASURED) as f:
            return float(json.load(f)["sm_max_mhz"])
    except Exception:
        return None


def peaks():
    try:
        with open(MEASURED) as f:
            m = json.load(f)
        return m["hbm_gbs"], m["bf16_tflops"], m.get("bf16_tflops_sustained", m["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region.

    nvidia-smi takes a few hundred ms to produce its first line, longer than a short timed
    region, so the sampler is started before the warm-up steps (same load) and `mark()` /
    `stop()` bracket the timed region; only samples stamped inside it are summarised. If the
    region was shorter than the 100 ms sampling period, the last warm-up sample stands in
    and the summary says so (`"window": "warmup"`)."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (monotonic time, fields)
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 7:
                self.samples.append((time.monotonic(), p))

    def mark(self):
        self.t0 = time.monotonic()

    def stop(self):
        self.t1 = time.monotonic()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        t0 = self.t0 if self.t0 is not None else -1e30
        t1 = self.t1 if self.t1 is not None else 1e30
        inside = [p for t, p in self.samples if t0 <= t <= t1]
        window = "timed"
        if not inside:
            before = [p for t, p in self.samples if t < t0]
            inside, window = before[-1:], "warmup"
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[1]) for s in inside if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in inside if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in inside for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside), "window": window}


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
        pg = dist
    return world, rank, local, pg


def allmax(pg, v: float) -> float:
    if pg is None:
        return v
    import torch

    t = torch.tensor([v], dtype=torch.float64)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        pg.barrier()


def host_mem_available() -> int:
    try:
        with open("/proc/meminfo") as f:
            return next(int(l.split()[1]) * 1024 for l in f if l.startswith("MemAvailable"))
    except Exception:
        return 16 << 30


def cpu_threads(per_thread_bytes: float) -> int:
    cores = os.cpu_count() or 1
    return max(1, min(cores, int(0.6 * host_mem_available() / per_thread_bytes)))


def _sample_cfg(c):
    from oracle import Cfg

    # C1 runs as is; at the large configs' model dims the reference holds fp64 T x V logits and
    # H x T x T probabilities per layer (C2: ~256 GB), so each worker runs
    # a tiny packed group of the same model: P=2, G=2, R=1 (T=4)
    sP, sG, sR = (2, 2, 1) if c["vocab"] > 10000 else (c["P"], c["G"], c["R"])
    return Cfg(c["vocab"], c["d"], c["L"], c["H"], c["F"], max(sP + sG * sR, 8)), sP, sG, sR


class RefBaseline:
    """The reference's own implementation (oracle/_ref, built from its sources) on the host
    cores: one TriModel per worker thread, built once outside any timing; each step runs one
    shared-prompt train_microbatch (pipeline.cpp:97-141) per worker, all workers concurrently."""

    def __init__(self, c, threads=None):
        from oracle import Oracle

        self.ref = Oracle("ref")  # FileNotFoundError when not built
        self.cfg, self.P, self.G, self.R = _sample_cfg(c)
        n_params = self.ref.param_count(self.cfg)
        per_thread = 6.0 * 8 * n_params  # fp64 params x3 + grads + forward caches
        if per_thread > 0.6 * host_mem_available():
            raise MemoryError("the reference's fp64 model does not fit host memory")
        self.threads = threads or cpu_threads(per_thread)
        self.T = self.P + self.G * self.R
        self.h = self.ref.bench_open(self.cfg, 7, self.threads)

    def step(self) -> float:
        return self.ref.bench_run(self.h, self.P, self.G, self.R, 1)

    def close(self):
        self.ref.bench_close(self.h)

    def describe(self, c, secs):
        T_w = c["P"] + sum(group_lens(c))
        tok_s = self.threads * self.T * len(secs) / sum(secs)
        same = self.T == T_w
        info = {"cores": self.threads, "value": tok_s, "same_config": same,
                "sample": f"reference Pipeline::train_microbatch (shared-prompt branch) at {c['name']} model dims, "
                          f"P={self.P} G={self.G} R={self.R} (T={self.T}) per worker, {self.threads} workers "
                          f"concurrently, {len(secs)} step(s), {np.mean(secs):.2f} s per step (measured, unscaled)"}
        if not same:  # context only: the FLOP model's per-token cost at the workload's T
            fl_s = flops_per_group(c, self.P, [self.R] * self.G, reference_head=True)
            fl_w = flops_per_group(c, c["P"], group_lens(c), reference_head=True)
            info["extrapolated_to_workload"] = {
                "value": tok_s * (fl_s / self.T) / (fl_w / T_w), "unit": "packed tokens/s",
                "method": f"FLOP model per packed token (SURVEY.md 8d, reference head over all rows), T={T_w}; "
                          f"not executed: needs ~256 GB host memory and hours per micro-step"}
        return info


def run_reference(args, c):
    world, rank, local, pg = dist_setup(args.gpus)
    if rank != 0:
        return
    c["name"] = args.config
    try:
        rb = RefBaseline(c)
    except FileNotFoundError:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libparl_ref.so not built"}))
        return
    except MemoryError:
        print(json.dumps({"impl": "reference", "unavailable": f"the reference's fp64 model at {args.config} dims does "
                                                              f"not fit this host's memory"}))
        return
    for _ in range(args.warmup):
        rb.step()
    secs = [rb.step() for _ in range(args.steps)]
    rb.close()
    info = rb.describe(c, secs)
    value = info["value"]
    out = {"metric": "packed tokens/s, tri-model logprob+GRPO loss at 1/2/4/8 B200 vs CPU ref", "value": value,
           "unit": "packed tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1000.0 * float(np.mean(secs)), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": f"{args.config} model dims: d={c['d']} H={c['H']} L={c['L']} F={c['F']} "
                                  f"V={c['vocab']}; executed sample: P={rb.P} G={rb.G} R={rb.R} (T={rb.T}) x "
                                  f"{rb.threads} workers per step",
                      "same_config": info["same_config"]},
           "cpu_baseline": {"value": value, "unit": "packed tokens/s", "cores": rb.threads, "kind": "reference",
                            "sample": info["sample"]},
           "e2e": {"value": value, "unit": "packed tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if "extrapolated_to_workload" in info:
        out["extrapolated_to_workload"] = info["extrapolated_to_workload"]
    print(json.dumps(out))


def run_ours(args, c):
    world, rank, local, pg = dist_setup(args.gpus)
    from paper_2511_18871_b200 import parl as P

    prec = P.PREC_BF16 if c["prec"] == "bf16" else P.PREC_FP32
    ctx = P.Context(local, prec)
    if world > 1:
        from paper_2511_18871_b200.dp import bootstrap_comm

        bootstrap_comm(ctx, rank, world)

    cfg = P.ModelConfig(c["vocab"], c["d"], c["L"], c["H"], c["F"], c["max_seq"])
    pol = P.ModelParams.init_device(cfg, 7, ctx)
    old = pol.clone(seed=11, noise=0.01)
    ref = pol.clone()
    tm = P.TriModel(pol, old, ref)
    grads = P.GradBuffer(pol)
    hyper = P.HyperParams(0.2, 0.04, "token")

    Pn, G = c["P"], c["G"]
    n_global = args.groups or c["groups"]  # global batch of prompt groups (strong scaling)
    mine = list(range(rank, n_global, world))  # this rank's groups (identical global batch at every N)
    ng = len(mine)
    lens = np.array(group_lens(c), np.int32)
    offs = np.concatenate([[0], np.cumsum(lens)])
    T = Pn + int(lens.sum())
    prompts, resps, rewards = [], [], []
    for gi in mine:  # per-group seeds: the same synthetic batch however it is split
        rng = np.random.default_rng([123, gi])
        prompts.append(rng.integers(4, c["vocab"], Pn).astype(np.int32))
        resps.append(rng.integers(4, c["vocab"], T - Pn).astype(np.int32))
        rewards.append(rng.random(G))
    K = max(1, args.pack or c.get("pack", 1))  # prompt groups packed into one sequence per micro-step (f4)
    chunks = [list(range(i, min(i + K, ng))) for i in range(0, ng, K)]
    group = P.Group(T * K, G * K, ctx)

    import torch

    torch.cuda.set_device(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{local}")
    d_prompts = [torch.from_numpy(np.concatenate([prompts[i] for i in ch])).cuda(local) for ch in chunks]
    d_resps = [torch.from_numpy(np.concatenate([resps[i] for i in ch])).cuda(local) for ch in chunks]
    rew_ch = [np.concatenate([rewards[i] for i in ch]) for ch in chunks]
    torch.cuda.synchronize(local)

    def pack_chunk(q):
        n = len(chunks[q])
        if n == 1:
            group.pack_device(d_prompts[q].data_ptr(), Pn, d_resps[q].data_ptr(), lens, c["max_seq"])
        else:
            group.pack_multi_device(d_prompts[q].data_ptr(), [Pn] * n, d_resps[q].data_ptr(), np.tile(lens, n),
                                    [G] * n, c["max_seq"])

    def step_device():
        grads.reset()
        for q in range(len(chunks)):
            pack_chunk(q)
            if world > 1 and q == len(chunks) - 1:
                grads.allreduce_overlap()  # the last backward streams its gradient slices to NCCL
            P.train_microbatch(tm, group, grads, hyper, rewards=rew_ch[q], want_stats=False)
        if world > 1:
            grads.allreduce()
            ctx.stats_allreduce()

    # pinned host inputs for the end-to-end leg
    h_prompts = [torch.from_numpy(p).pin_memory().numpy() for p in prompts]
    h_resps = [torch.from_numpy(r).pin_memory().numpy() for r in resps]

    def step_e2e():
        # host inputs in, the step's loss statistics out (one device -> host read per step,
        # after the last micro-batch; the statistics accumulate on the device)
        grads.reset()
        ctx.stats_reset()
        for q, ch in enumerate(chunks):
            if len(ch) == 1:
                i = ch[0]
                group.pack(h_prompts[i], [h_resps[i][offs[k]:offs[k + 1]] for k in range(G)], c["max_seq"])
            else:
                group.pack_multi([h_prompts[i] for i in ch],
                                 [[h_resps[i][offs[k]:offs[k + 1]] for k in range(G)] for i in ch], c["max_seq"])
            if world > 1 and q == len(chunks) - 1:
                grads.allreduce_overlap()
            P.train_microbatch(tm, group, grads, hyper, rewards=rew_ch[q], want_stats=False)
        if world > 1:
            grads.allreduce()
            ctx.stats_allreduce()
        return ctx.stats()

    clk = ClockSampler(local).start()  # running through the warm-up: its first line takes ~0.3 s
    for _ in range(args.warmup):
        step_device()
    ctx.sync()
    if args.launch_list:
        clk.stop()  # one step inside an NVTX range for `ncu --nvtx --nvtx-include step/`
        torch.cuda.nvtx.range_push("step")
        step_device()
        ctx.sync()
        torch.cuda.nvtx.range_pop()
        return

    # ---- device-resident timed region (CUDA events on the library's stream)
    l0 = ctx.launches
    barrier(pg)
    ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk.mark()
    e0.record(stream)
    for _ in range(args.steps):
        step_device()
    e1.record(stream)
    ctx.sync()
    clk.stop()
    launches = (ctx.launches - l0) // max(args.steps, 1)
    ms = e0.elapsed_time(e1)
    barrier(pg)
    ms_max = allmax(pg, ms)

    # ---- end-to-end through the public API with host buffers, right after the device-resident
    # leg so both timed legs run under the same conditions (clocks drift under sustained load)
    for _ in range(2):
        step_e2e()
    barrier(pg)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step_e2e()
    e2e_s = time.perf_counter() - t0
    e2e_max = allmax(pg, e2e_s)

    # ---- the SGD update, timed separately (outside the metric): divisor = the
    # global batch's N*G samples (pipeline.cpp:346-351), snapshot old <- policy, apply_update
    upd0, upd1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    upd0.record(stream)
    grads.set_micro_step_count(n_global * G)
    tm.snapshot_old_policy()
    try:
        tm.policy.apply_update(grads, 1e-4)
        upd1.record(stream)
        ctx.sync()
        update_ms = upd0.elapsed_time(upd1)
    except P.ConfigError as e:  # C3 / C4: no device fp64 master at 7B (61 GB); the update is not timed
        ctx.sync()
        update_ms = f"not timed: {e}"

    # ---- again with per-launch CUDA events on the launch stream for every kernel class
    # (roofline), over min(K, 4) steps; kept out of `value`.
    prof_steps = min(args.steps, 4)
    ctx.profile(True)
    ctx.sync()
    for _ in range(prof_steps):
        step_device()
    ctx.sync()
    ctx.profile(False)
    prof = {k: ctx.profile_read(k) for k in ctx.KC}

    if rank != 0:
        return
    tokens_per_step = n_global * T
    value = tokens_per_step * args.steps / (ms_max / 1000.0)
    e2e_val = tokens_per_step * args.steps / e2e_max
    hbm, bf16, bf16_sus, src = peaks()
    # dominant tensor-core class
    tc = {k: v for k, v in prof.items() if k in ("gemm", "head", "attn_fwd", "attn_bwd") and v["ms"] > 0}
    dom = max(tc, key=lambda k: tc[k]["ms"]) if tc else "gemm"
    dp = prof[dom]
    achieved = dp["work"] / (dp["ms"] / 1000.0) / 1e12 if dp["ms"] > 0 else 0.0
    step_ms = ms_max / args.steps
    traffic, traffic_src = measured_traffic(dom)
    if args.config != "c2":  # the committed capture is of a C2 step: no traffic figure for other configs
        traffic, traffic_src = None, "no ncu capture of this config"
    if c["prec"] == "fp32":  # the fp32 build runs SIMT (FFMA): its roofline is the FP32 pipe, not the tensor core
        peak_t, peak_kind = 148 * 128 * 2 * (sm_max_mhz() or 1965.0) * 1e6 / 1e12, \
            "nominal fp32 FFMA (148 SMs x 128 lanes x 2 x max SM clock; the fp32 build runs SIMT)"
    else:
        peak_t, peak_kind = bf16_sus, f"{src} bf16 sustained"
    share = {k: round(v["ms"] / prof_steps / step_ms, 4) for k, v in prof.items() if v["ms"] > 0}
    c["name"] = args.config
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:  # one measured step of the reference on the host cores (after both timed regions)
            rb = RefBaseline(c)
            secs = [rb.step()]
            rb.close()
            cpu = rb.describe(c, secs)
        except (FileNotFoundError, MemoryError):
            cpu = None
    out = {
        "metric": "packed tokens/s, tri-model logprob+GRPO loss at 1/2/4/8 B200 vs CPU ref",
        "value": value, "unit": "packed tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": c["prec"], "data": "synthetic (random-init weights, uniform tokens in [4,V), U[0,1) rewards)",
        "config": {"workload": f"{args.config}: d={c['d']} H={c['H']} L={c['L']} F={c['F']} V={c['vocab']}, "
                               f"P={Pn} G={G} R={c['R'] or lens.tolist()} (T={T}); global batch {n_global} groups "
                               f"per step, {ng} on rank 0",
                   "global_groups": n_global, "groups_per_rank": ng, "packed_tokens_per_group": T,
                   "groups_per_packed_sequence": K,
                   "l2": "working set (weights+activations, GBs) exceeds the 126 MB L2; no explicit flush",
                   "roofline_timing": f"per-launch CUDA events over {prof_steps} further identical steps",
                   "update_ms": update_ms,
                   "parallelism": f"dp{world} over prompt groups"},
        "e2e": {"value": e2e_val, "unit": "packed tokens/s", "h2d_bytes_per_step": ng * (T * 4 + G * 8 + G * 4),
                "d2h_bytes_per_step": 40},
        "gpu_launches": int(launches),
        "roofline": {"bound": "tensor" if c["prec"] != "fp32" else "fp32", "kernel_class": dom, "achieved": achieved,
                     "peak": peak_t, "unit": "TFLOP/s", "frac": achieved / peak_t, "peak_kind": peak_kind,
                     "traffic": traffic, "traffic_unit": "DRAM bytes per launch (ncu, read + write)",
                     "traffic_source": traffic_src, "share_of_step": share},
        "kernel_classes": {k: {"ms_per_step": v["ms"] / prof_steps, "launches_per_step": v["launches"] / prof_steps,
                               "achieved": (v["work"] / (v["ms"] / 1e3) / (1e12 if k in tc else 1e9))
                               if v["ms"] > 0 else None,
                               "unit": "TFLOP/s" if k in ("gemm", "head", "attn_fwd", "attn_bwd") else "GB/s"}
                           for k, v in prof.items()},
        "flops_per_group": flops_per_group(c, Pn, lens.tolist()),
        "model_tflops": flops_per_group(c, Pn, lens.tolist()) * ng * world / (step_ms / 1e3) / 1e12,
        "clocks": clk.summary(),
    }
    if cpu is not None:
        out["cpu_baseline"] = {"value": cpu["value"], "unit": "packed tokens/s", "cores": cpu["cores"],
                               "kind": "reference", "sample": cpu["sample"], "same_config": cpu["same_config"]}
        if "extrapolated_to_workload" in cpu:
            out["cpu_baseline"]["extrapolated_to_workload"] = cpu["extrapolated_to_workload"]
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--groups", type=int, default=0, help="global batch: prompt groups per step (all ranks)")
    ap.add_argument("--pack", type=int, default=0,
                    help="prompt groups packed into one sequence per micro-step (0: the config's default)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--launch-list", action="store_true",
                    help="run one step inside an NVTX range 'step' (for ncu launch lists) and exit")
    args = ap.parse_args()
    c = dict(CONFIGS[args.config])
    if args.impl == "reference":
        run_reference(args, c)
    else:
        run_ours(args, c)


if __name__ == "__main__":
    main()
