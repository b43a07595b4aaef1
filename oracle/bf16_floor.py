"""Measure the bf16 rounding floor of the hot path at the BASELINE layer widths
(SURVEY.md §8c method), with the pinned torch restatement (oracle/torch_ref.py):
exact fp64 against bf16-rounded MMA inputs with fp64 accumulation, on the same
weights (ModelParams::init bit-exact, old / ref perturbed) and inputs.

    python -m oracle.bf16_floor            # writes tests/golden/bf16_floor.json

Cases (L=1 except C1; one ragged shared-prompt group, P=64, responses 96/80/131, not
tile aligned):
  c1  : BASELINE configs[0] exactly (d=256, H=4, L=2, F=1024, V=4096; P=64, G=4, R=128)
  c2w : d=896,  H=14, F=4864,  V=151936 (Qwen2.5-0.5B widths, the real vocabulary)
  c4w : d=1536, H=12, F=8960,  V=151936 (Qwen2.5-1.5B)
  c3w : d=3584, H=28, F=18944, V=152064 (Qwen2.5-7B)
Floors: log-prob max / mean |delta|; backward at the exact upstream seed: per-tensor
relative Frobenius error (worst, excluding attn.bk), global relative error and cosine;
attn.bk max |grad| (analytically 0); GRPO objective relative error of the full loop.
The GPU tolerances (tests/test_gpu_widths.py) are a fixed multiple of these floors.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

from oracle import Cfg, Oracle, layout
from oracle import torch_ref as TR

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "bf16_floor.json")

CASES = {
    "c1": (Cfg(4096, 256, 2, 4, 1024, 576), 64, [128, 128, 128, 128]),
    "c2w": (Cfg(151936, 896, 1, 14, 4864, 512), 64, [96, 80, 131]),
    "c4w": (Cfg(151936, 1536, 1, 12, 8960, 512), 64, [96, 80, 131]),
    "c3w": (Cfg(152064, 3584, 1, 28, 18944, 512), 64, [96, 80, 131]),
}


def case_inputs(name, cfg, P, lens, seed=7):
    """Deterministic weights / tokens / rewards of a case (also rebuilt by the GPU test)."""
    w = Oracle("c").init_params(cfg, seed)
    rng = np.random.default_rng([17, len(name)])
    w_old = w + 0.01 * rng.standard_normal(len(w))
    w_ref = w - 0.01 * rng.standard_normal(len(w))
    rng = np.random.default_rng([23, cfg.d_model])
    prompt = rng.integers(4, cfg.vocab, P).astype(np.int32)
    resp = [rng.integers(4, cfg.vocab, n).astype(np.int32) for n in lens]
    adv = TR.group_advantages(rng.random(len(lens)))
    return w, w_old, w_ref, prompt, resp, adv


def compare(cfg, lp3_a, g_a, st_a, lp3_b, g_b, st_b):
    """Error metrics of (a) against the exact (b)."""
    d = np.abs(lp3_a - lp3_b)
    per, bk = {}, 0.0
    for name, off, r, c in layout(cfg):
        x, y = g_a[off:off + r * c], g_b[off:off + r * c]
        if name.endswith("attn.bk"):
            bk = max(bk, float(np.abs(x).max()))
            continue
        ny = np.linalg.norm(y)
        per[name] = float(np.linalg.norm(x - y) / ny) if ny > 0 else float(np.linalg.norm(x))
    worst = max(per, key=per.get)
    mask = np.ones(len(g_a), bool)
    for name, off, r, c in layout(cfg):
        if name.endswith("attn.bk"):
            mask[off:off + r * c] = False
    ga, gb = g_a[mask], g_b[mask]
    return {"lp_max": float(d.max()), "lp_mean": float(d.mean()),
            "grad_rel_worst": per[worst], "grad_rel_worst_tensor": worst,
            "grad_rel_global": float(np.linalg.norm(ga - gb) / np.linalg.norm(gb)),
            "grad_cos": float(ga @ gb / (np.linalg.norm(ga) * np.linalg.norm(gb))),
            "bk_abs": bk, "obj_rel": float(abs(st_a[0] - st_b[0]) / max(abs(st_b[0]), 1e-12))}


def measure(name, device="cpu"):
    cfg, P, lens = CASES[name]
    w, wo, wr, prompt, resp, adv = case_inputs(name, cfg, P, lens)
    t0 = time.time()
    lp3_x, g_x, st_x = TR.microstep(cfg, w, wo, wr, prompt, resp, adv, rnd=False, device=device)
    up_x, _ = TR.grpo_terms(lp3_x[0], lp3_x[1], lp3_x[2], lens, adv)
    # backward floor at the exact upstream seed; objective floor of the full emulated loop
    lp3_b, g_b, _ = TR.microstep(cfg, w, wo, wr, prompt, resp, adv, rnd=True, device=device, upstream=up_x)
    _, st_b = TR.grpo_terms(lp3_b[0], lp3_b[1], lp3_b[2], lens, adv)
    out = compare(cfg, lp3_b, g_b, st_b, lp3_x, g_x, st_x)
    out["seconds"] = time.time() - t0
    out["cfg"] = [cfg.vocab, cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.d_ff, cfg.max_seq]
    out["P"], out["lens"] = P, lens
    return out


def main():
    """python -m oracle.bf16_floor [case ...] [--device cuda] [--out path]: the widest case (c3w)
    needs ~60 GB for its fp64 weights and gradients and runs on a GPU box's fp64 torch."""
    args, device, out = [], "cpu", OUT
    argv = sys.argv[1:]
    while argv:
        a = argv.pop(0)
        if a == "--device":
            device = argv.pop(0)
        elif a == "--out":
            out = argv.pop(0)
        else:
            args.append(a)
    names = args or list(CASES)
    res = {}
    if os.path.exists(out):
        with open(out) as f:
            res = json.load(f)
    for n in names:
        res[n] = measure(n, device)
        res[n]["device"] = device
        print(n, json.dumps(res[n]), flush=True)
        with open(out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
