"""Calibrate the event simulator's train_cost_per_microstep from measured GPU micro-steps.

The reference's virtual-clock model charges every trained micro-step a constant cost
(PipelineSettings::train_cost_per_microstep, pipeline.hpp:81; simulate_iteration,
event_sim.cpp:89-127), "a constant from config or measured-and-frozen from a calibration
run".  This measures it on the device path: one shared-prompt micro-step
(pack -> tri-model forward -> GRPO loss -> policy backward -> accumulate) of the given
shape, CUDA-event timed on the library's stream after warm-up, and writes the config
fragment the reference's harness reads (config.cpp:200-208):

    python -m paper_2511_18871_b200.calibrate --config c2 [--steps 10] [--out calib.json]
    -> {"run": {"train_cost_per_microstep": <seconds>}, "calibration": {...}}

`--seconds-per-virtual` rescales when the simulator's virtual clock is not in seconds.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def measure_microstep(vocab, d, L, H, F, P, lens, precision="bf16", steps=10, warmup=3, seed=7, device=0):
    """Mean device seconds of one micro-step of this shape (m = G: one packed group)."""
    import torch

    from paper_2511_18871_b200 import parl as PL

    ctx = PL.Context(device, PL.PREC_BF16 if precision == "bf16" else PL.PREC_FP32)
    T = P + int(sum(lens))
    cfg = PL.ModelConfig(vocab, d, L, H, F, max(T, 8))
    pol = PL.ModelParams.init_device(cfg, seed, ctx)
    tm = PL.TriModel(pol, pol.clone(seed=seed + 4, noise=0.01), pol.clone())
    grads = PL.GradBuffer(pol)
    rng = np.random.default_rng(seed)
    d_prompt = torch.from_numpy(rng.integers(4, vocab, P).astype(np.int32)).cuda(device)
    d_resp = torch.from_numpy(rng.integers(4, vocab, T - P).astype(np.int32)).cuda(device)
    rewards = rng.random(len(lens))
    group = PL.Group(T, len(lens), ctx)
    lens = np.asarray(lens, np.int32)
    stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{device}")

    def step():
        group.pack_device(d_prompt.data_ptr(), P, d_resp.data_ptr(), lens, cfg.max_seq_len)
        PL.train_microbatch(tm, group, grads, PL.HyperParams(), rewards=rewards, want_stats=False)

    for _ in range(warmup):
        step()
    ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    ctx.sync()
    return e0.elapsed_time(e1) / 1000.0 / steps


def main():
    sys.path.insert(0, ROOT)
    from bench import CONFIGS, group_lens

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seconds-per-virtual", type=float, default=1.0)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    c = CONFIGS[args.config]
    lens = group_lens(c)
    secs = measure_microstep(c["vocab"], c["d"], c["L"], c["H"], c["F"], c["P"], lens, c["prec"], args.steps,
                             args.warmup)
    out = {"run": {"train_cost_per_microstep": secs / args.seconds_per_virtual},
           "calibration": {"config": args.config, "device_seconds_per_microstep": secs, "steps": args.steps,
                           "micro_step": f"m=G={len(lens)} shared-prompt group, P={c['P']}, T={c['P'] + sum(lens)}",
                           "precision": c["prec"], "source": "CUDA events on the library stream (calibrate.py)"}}
    s = json.dumps(out, indent=1)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s + "\n")
    print(s)


if __name__ == "__main__":
    main()
