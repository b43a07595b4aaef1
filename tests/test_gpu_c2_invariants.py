"""Invariants at the full headline shape (BASELINE configs[1], C2), on the tcgen05 path.

The shape is L=24, d=896, H=14, F=4864, V=151,936, with P=512 and G=8 responses of R=1024 (T=8,704), and random-init weights. These are SURVEY.md §8c's GPU-internal checks for C2-C5, run at C2:

  * shared == replicated (test_packing.cpp:123-200, at the headline shape, bf16). The packed group's log-probs match those of the G causal sequences [prompt + response_k]. Its policy gradient, for one upstream, matches the sum of the G per-sequence gradients.
    - The identity is exact in real arithmetic.
    - With P and R multiples of the 128-row tile, the log-probs see the same key tiles in the same order and the same per-row GEMM reductions, so they are compared to 1e-3.
    - The gradients differ only by fp32 summation order over the responses, plus the bf16 rounding of the prompt rows' per-sequence dX. They are held to 1e-2 per tensor and a 0.9999 cosine.
  * fp32 build ~ bf16 build. The same weights and group go through the fp32 path (SIMT, fp32 everywhere) and the bf16 tcgen05 path.
    - Rounding error accumulates over the layers as a random walk.
    - The tolerance is 3x the measured single-layer bf16 floor at C2's widths (tests/golden/bf16_floor.json, c2w) times sqrt(L): log-probs max / mean, global gradient relative error, and 1 - cosine times L.
"""
import json
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN
from tests.gpu_helpers import ocfg, per_tensor_rel

pytestmark = pytest.mark.gpu

P_LEN, G, R = 512, 8, 1024


@pytest.fixture(scope="module")
def P():
    from paper_2511_18871_b200 import parl

    return parl


def c2(P):
    return P.ModelConfig(151936, 896, 24, 14, 4864, P_LEN + G * R)


def inputs(seed=3):
    rng = np.random.default_rng(seed)
    prompt = rng.integers(4, 151936, P_LEN).astype(np.int32)
    resp = [rng.integers(4, 151936, R).astype(np.int32) for _ in range(G)]
    up = rng.uniform(-1.0, 1.0, G * R) / (G * R)
    return prompt, resp, up


def test_c2_shared_equals_replicated_bf16(P):
    ctx = P.Context(0, P.PREC_BF16)
    cfg = c2(P)
    pm = P.ModelParams.init_device(cfg, 11, ctx)
    prompt, resp, up = inputs()
    pk = P.pack_group(prompt, resp, cfg.max_seq_len, ctx)
    f = P.forward_logprobs(pm, pk.tokens, pk.positions, pk.mask, pk.labels, True)
    lp_shared = np.array(f.logprobs)
    g_shared = P.backward(pm, f, up).flat()
    del f
    gr = P.GradBuffer(pm)
    dmax = 0.0
    for k, r in enumerate(resp):
        toks = np.concatenate([prompt, r])
        fr = P.forward_logprobs(pm, toks, np.arange(len(toks)), P.AttentionMaskSpec.causal(),
                                np.concatenate([np.full(P_LEN, -1), r]), True)
        d = np.abs(np.array(fr.logprobs) - lp_shared[k * R:(k + 1) * R])
        dmax = max(dmax, float(d.max()))
        P.backward(pm, fr, up[k * R:(k + 1) * R], gr)
        del fr
    g_rep = gr.flat()
    rel = per_tensor_rel(ocfg(cfg), g_shared, g_rep)
    worst = max((v, k) for k, v in rel.items() if not k.endswith("attn.bk"))
    cos = float(g_shared @ g_rep / (np.linalg.norm(g_shared) * np.linalg.norm(g_rep)))
    print("C2 shared vs replicated: lp max |delta|", dmax, "grad worst rel", worst, "cos", cos)
    assert dmax <= 1e-3
    assert worst[0] <= 1e-2, worst
    assert cos >= 0.9999


def test_c2_fp32_build_vs_bf16_build(P):
    with open(os.path.join(GOLDEN, "bf16_floor.json")) as fh:
        floor = json.load(fh)["c2w"]
    L = 24
    grow = 3.0 * np.sqrt(L)
    prompt, resp, up = inputs(5)
    out = {}
    for prec in ("bf16", "fp32"):
        ctx = P.Context(0, P.PREC_BF16 if prec == "bf16" else P.PREC_FP32)
        cfg = c2(P)
        pm = P.ModelParams.init_device(cfg, 13, ctx)
        pk = P.pack_group(prompt, resp, cfg.max_seq_len, ctx)
        f = P.forward_logprobs(pm, pk.tokens, pk.positions, pk.mask, pk.labels, True)
        out[prec] = (np.array(f.logprobs), P.backward(pm, f, up).flat())
        del f, pm, pk
    (lb, gb), (lf, gf) = out["bf16"], out["fp32"]
    d = np.abs(lb - lf)
    grel = float(np.linalg.norm(gb - gf) / np.linalg.norm(gf))
    cos = float(gb @ gf / (np.linalg.norm(gb) * np.linalg.norm(gf)))
    print("C2 bf16 vs fp32 build: lp max", float(d.max()), "mean", float(d.mean()), "grad rel", grel, "cos", cos,
          "| bounds", grow * floor["lp_max"], grow * floor["lp_mean"], grow * floor["grad_rel_global"],
          1 - 3 * L * (1 - floor["grad_cos"]))
    assert np.isfinite(lb).all() and np.isfinite(gb).all()
    assert d.max() <= grow * floor["lp_max"]
    assert d.mean() <= grow * floor["lp_mean"]
    assert grel <= grow * floor["grad_rel_global"]
    assert 1 - cos <= 3 * L * (1 - floor["grad_cos"])
