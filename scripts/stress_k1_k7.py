"""K1 (packer) and K7 (GRPO loss) at a stress size (>= 2^24 scored tokens),
where they move hundreds of MB instead of the ~0.25 MB of one C2 micro-step.

    python scripts/stress_k1_k7.py [--tokens 16777216] [--reps 20] [--only k1|k7]

Prints one JSON line: per kernel, algorithmic bytes per launch, CUDA-event time per launch
(on the library's stream, after warm-up) and achieved GB/s against the measured HBM peak.
Algorithmic bytes (our output layout, kernels.cuh PackedDev):
  K1: reads the T token ids (4 B) and writes tokens, labels, positions, seg, pred, row_ptr
      (6 x 4 B per packed position) plus scored_pos, scored_label, pred_pos, sample_of,
      row_idx (5 x 4 B per scored token)           -> 28 B / position + 20 B / scored token
  K7: reads lp, old, ref (3 x 4 B) and sample_of (4 B), writes upstream (4 B)
                                                    -> 20 B / scored token (+ 16 B / sample)
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=1 << 24, help="scored tokens")
    ap.add_argument("--G", type=int, default=64)
    ap.add_argument("--P", type=int, default=512)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    import torch

    from paper_2511_18871_b200 import parl as P

    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        hbm = json.load(f)["hbm_gbs"]
    ctx = P.Context(0, P.PREC_BF16)
    G, Pn = args.G, args.P
    R = args.tokens // G
    S = R * G
    T = Pn + S
    stream = torch.cuda.ExternalStream(ctx.stream)
    rng = np.random.default_rng(0)
    d_prompt = torch.from_numpy(rng.integers(4, 151936, Pn).astype(np.int32)).cuda()
    d_resp = torch.from_numpy(rng.integers(4, 151936, S).astype(np.int32)).cuda()
    g = P.Group(T, G, ctx)
    lens = np.full(G, R, np.int32)
    out = {"tokens_scored": S, "tokens_packed": T, "G": G, "hbm_peak_gbs": hbm}

    def timed(fn, n):
        for _ in range(3):
            fn()
        ctx.sync()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(n):
            fn()
        b.record(stream)
        ctx.sync()
        return a.elapsed_time(b) / n

    g.pack_device(d_prompt.data_ptr(), Pn, d_resp.data_ptr(), lens, T)
    if args.only in ("", "k1"):
        ms = timed(lambda: g.pack_device(d_prompt.data_ptr(), Pn, d_resp.data_ptr(), lens, T), args.reps)
        byts = 28.0 * T + 20.0 * S
        out["k1_pack"] = {"bytes_per_launch": byts, "ms_per_launch": ms, "gbs": byts / ms / 1e6,
                          "frac_hbm": byts / ms / 1e6 / hbm,
                          "note": "includes the host-side launch prologue (segment bounds / schedule upload, "
                                  "cached for a repeated shape)"}
    if args.only in ("", "k7"):
        for slot in range(3):
            g.set_logprobs(slot, -3.0 * rng.random(S) + (0.05 * rng.standard_normal(S) if slot else 0.0))
        adv = P._f64(rng.standard_normal(G))
        hyper = P.HyperParams().c()

        def k7():  # parl_grpo_loss without reading the stats back (no stream sync)
            P._check(P.LIB.parl_grpo_loss(ctx.h, g.h, None, P._pd(adv), P.C.byref(hyper), None), ctx.h)

        ms = timed(k7, args.reps)
        byts = 20.0 * S + 16.0 * G
        out["k7_grpo"] = {"bytes_per_launch": byts, "ms_per_launch": ms, "gbs": byts / ms / 1e6,
                          "frac_hbm": byts / ms / 1e6 / hbm,
                          "note": "one parl_grpo_loss call: k_grpo_tokens + k_grpo_finish (+ advantages upload)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
