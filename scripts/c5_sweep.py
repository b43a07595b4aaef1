"""BASELINE configs[4] (C5): mask-efficiency sweep at 32k packed tokens, shared-prompt
packing vs the replicated-prompt baseline.

For each prompt fraction f and group size G: P = floor(f * 32768), R = floor((32768 - P) / G).
  shared     : one packed group (prompt once, G responses, shared-prompt mask) through
               Pipeline::train_microbatch's shared-prompt branch (pipeline.cpp:97-141)
  replicated : the reference's non-packed branch (pipeline.cpp:142-170): G causal sequences
               prompt || response_k, each its own tri-model forward + GRPO + backward
Both report time per micro-step and "useful" tokens/s = (P + G R) / time, plus the
FLOP-model ratio of SURVEY.md §8d.  C2 model dims (Qwen2.5-0.5B-shaped, bf16), random init.

    python scripts/c5_sweep.py [--fractions 0.1,0.5,0.9] [--groups 2,8,64] > profiles/rNN_c5_sweep.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS, flops_per_group  # noqa: E402


def causal_flops(c, T, scored):
    """SURVEY.md §8d FLOP model for one causal sequence of T tokens with `scored` head rows."""
    d, L, F, V = c["d"], c["L"], c["F"], c["vocab"]
    gemm = 2.0 * T * L * (4 * d * d + 2 * d * F)
    attn = 4.0 * (T * (T + 1) / 2) * d * L
    head = 2.0 * scored * d * V
    return 3 * (gemm + attn + head) + 2 * gemm + 2.5 * attn + 2 * head


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fractions", default="0.1,0.3,0.5,0.7,0.9")
    ap.add_argument("--groups", default="2,4,8,16,32,64")
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()

    import torch

    from paper_2511_18871_b200 import parl as P

    c = dict(CONFIGS["c2"])
    ctx = P.Context(0, P.PREC_BF16)
    cfg = P.ModelConfig(c["vocab"], c["d"], c["L"], c["H"], c["F"], max(c["max_seq"], args.tokens))
    pol = P.ModelParams.init_device(cfg, 7, ctx)
    tm = P.TriModel(pol, pol.clone(seed=11, noise=0.01), pol.clone())
    grads = P.GradBuffer(pol)
    hyper = P.HyperParams(0.2, 0.04, "token")
    stream = torch.cuda.ExternalStream(ctx.stream)
    rng = np.random.default_rng(123)

    def timed(fn):
        fn()  # warm-up (allocations, schedules)
        ctx.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.reps):
            fn()
        e1.record(stream)
        ctx.sync()
        return e0.elapsed_time(e1) / args.reps / 1e3

    for f in [float(x) for x in args.fractions.split(",")]:
        for G in [int(x) for x in args.groups.split(",")]:
            Pn = int(f * args.tokens)
            R = (args.tokens - Pn) // G
            if R < 1:
                continue
            prompt = rng.integers(4, c["vocab"], Pn).astype(np.int32)
            resps = [rng.integers(4, c["vocab"], R).astype(np.int32) for _ in range(G)]
            rewards = rng.random(G)
            adv = (rewards - rewards.mean()) / max(rewards.std(), 1e-8)
            T = Pn + G * R

            group = P.Group(T, G, ctx)
            group.pack(prompt, resps, cfg.max_seq_len)

            def shared():
                grads.reset()
                P.train_microbatch(tm, group, grads, hyper, advantages=adv, want_stats=False)

            t_sh = timed(shared)
            print(f"f={f} G={G} shared {t_sh:.3f}s", file=sys.stderr, flush=True)

            # replicated prompt: G causal sequences prompt || response (pipeline.cpp:79-88, 142-170)
            L = Pn + R
            rep = P.Group(L, 1, ctx)
            toks = [np.concatenate([prompt, r]).astype(np.int32) for r in resps]
            pos = np.arange(L, dtype=np.int32)
            labels = [np.concatenate([np.full(Pn, -1, np.int32), r]).astype(np.int32) for r in resps]

            def replicated():
                grads.reset()
                for k in range(G):
                    rep.set_sequence(toks[k], pos, labels[k], P.AttentionMaskSpec.causal(), cfg.vocab_size,
                                     cfg.max_seq_len)
                    P.train_microbatch(tm, rep, grads, hyper, advantages=[adv[k]], want_stats=False)

            t_rep = timed(replicated)
            fl_sh = flops_per_group(c, Pn, [R] * G)
            fl_rep = G * causal_flops(c, Pn + R, R)
            print(json.dumps({"prompt_fraction": f, "G": G, "P": Pn, "R": R, "packed_tokens": T,
                              "shared_s": t_sh, "replicated_s": t_rep, "speedup": t_rep / t_sh,
                              "flop_ratio": fl_rep / fl_sh, "shared_tok_s": T / t_sh, "replicated_tok_s": T / t_rep}),
                  flush=True)
            del group, rep


if __name__ == "__main__":
    main()
