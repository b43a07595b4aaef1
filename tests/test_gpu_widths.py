"""bf16 parity at the BASELINE layer widths and the real 152K vocabularies.

For each case of oracle/bf16_floor.py (C1 exactly; C2 / C4 / C3 layer widths at L=1 with
V = 151,936 / 151,936 / 152,064 and a ragged, tile-misaligned shared-prompt group) the
tensor-core path runs one micro-step through the C-ABI and is compared with the exact fp64
restatement (oracle/torch_ref.py, pinned to the C oracle by tests/test_oracle.py), evaluated
here on the GPU in fp64:

  * log-probs of the three roles: max / mean |delta|;
  * the backward at the exact upstream seed: per-tensor relative Frobenius error (worst
    tensor), global relative error and cosine over every parameter; attn.bk absolutely
    (analytically 0);
  * the GRPO objective of the fused micro-step: exact (fp32 accumulation) given its own
    log-probs; its error against the exact loop is reported.

Tolerance = TOL_FACTOR x the rounding floor that the same restatement measures with
bf16-rounded MMA inputs (tests/golden/bf16_floor.json), i.e. SURVEY.md §8c's method with
floors measured at these widths instead of C1's.
"""
import json
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu
TOL_FACTOR = 3.0


def _floors():
    with open(os.path.join(GOLDEN, "bf16_floor.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def P():
    from paper_2511_18871_b200 import parl

    return parl


@pytest.fixture(scope="module")
def ctx16(P):
    return P.Context(0, P.PREC_BF16)


@pytest.mark.parametrize("case", ["c1", "c2w", "c4w", "c3w"])
def test_bf16_parity_at_width(P, ctx16, case):
    import torch

    from oracle import bf16_floor as BF
    from oracle import torch_ref as TR

    floors = _floors()
    if case not in floors:
        pytest.skip(f"no measured floor for {case} (python -m oracle.bf16_floor {case} --device cuda)")
    floor = floors[case]
    cfg_o, Pn, lens = BF.CASES[case]
    w, wo, wr, prompt, resp, adv = BF.case_inputs(case, cfg_o, Pn, lens)
    cfg = P.ModelConfig(cfg_o.vocab, cfg_o.d_model, cfg_o.n_layers, cfg_o.n_heads, cfg_o.d_ff, cfg_o.max_seq)
    tm = P.TriModel(P.ModelParams.from_flat(cfg, w, 0, ctx16), P.ModelParams.from_flat(cfg, wo, 0, ctx16),
                    P.ModelParams.from_flat(cfg, wr, 0, ctx16))
    # fused micro-step: pack -> tri-model forward -> K7 -> backward (objective, log-probs)
    pk = P.pack_group(prompt, resp, cfg.max_seq_len, ctx16)
    gb = P.GradBuffer(tm.policy)
    ctx16.stats_reset()
    st = P.train_microbatch(tm, pk.group, gb, P.HyperParams(), advantages=adv)
    lp3 = np.stack([pk.group.logprobs(s) for s in range(3)])
    # exact fp64 restatement on the GPU
    lp3_x, g_x, st_x = TR.microstep(cfg_o, w, wo, wr, prompt, resp, adv, rnd=False, device="cuda")
    up_x, _ = TR.grpo_terms(lp3_x[0], lp3_x[1], lp3_x[2], lens, adv)
    # the backward at the exact upstream seed
    toks = np.concatenate([prompt] + resp)
    pos = np.concatenate([np.arange(Pn)] + [Pn + np.arange(n) for n in lens])
    labels = np.concatenate([np.full(Pn, -1)] + resp)
    fwd = P.forward_logprobs(tm.policy, toks, pos, P.AttentionMaskSpec.shared_prompt(Pn, lens), labels,
                             want_cache=True)
    g = P.backward(tm.policy, fwd, up_x).flat()
    torch.cuda.empty_cache()
    m = BF.compare(cfg_o, lp3, g, [st["objective_sum"]], lp3_x, g_x, st_x)
    print(case, json.dumps(m), "floor", json.dumps({k: floor[k] for k in m if k in floor}))
    tol = lambda k: TOL_FACTOR * floor[k]
    assert m["lp_max"] <= tol("lp_max"), m
    assert m["lp_mean"] <= tol("lp_mean"), m
    assert m["grad_rel_worst"] <= tol("grad_rel_worst"), m
    assert m["grad_rel_global"] <= tol("grad_rel_global"), m
    assert 1 - m["grad_cos"] <= TOL_FACTOR * (1 - floor["grad_cos"]), m
    assert m["bk_abs"] <= max(tol("bk_abs"), 1e-2), m  # attn.bk <= 1e-2 absolute in bf16
    # the objective: its error against the exact loop is the log-probs' error (bounded above)
    # propagated through exp(lp - old) and expm1(ref - lp), which amplifies it by the ratios and
    # cancels across advantages summing to zero -- so its relative error is reported, not held to
    # a floor.  What the loss kernel itself owes is exactness given the log-probs it consumed: the
    # fp64 GRPO terms (grpo.cpp:119-131) of the GPU's own log-probs, to fp32 accumulation.
    _, st_self = TR.grpo_terms(lp3[0], lp3[1], lp3[2], lens, adv)
    scale = np.abs(adv).sum() + abs(st_self[0])
    print(case, "objective relative to exact", m["obj_rel"], "floor", floor["obj_rel"],
          "| vs fp64 terms of its own log-probs", abs(st["objective_sum"] - st_self[0]) / scale)
    assert abs(st["objective_sum"] - st_self[0]) <= 1e-5 * scale, (st["objective_sum"], st_self[0])
    for k, kk in (("clip_sum", 1), ("kl_sum", 2), ("clipped_units", 3), ("total_units", 4)):
        assert abs(st[k] - st_self[kk]) <= 1e-5 * (abs(st_self[kk]) + scale), (k, st[k], st_self[kk])
