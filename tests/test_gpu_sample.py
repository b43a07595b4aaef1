"""GPU: sample_tokens (model.cpp:843-900) against the reference's own sampled tokens
(tests/golden/sample_tokens.npz, written by oracle/make_golden.py from oracle/_ref)."""
import numpy as np
import pytest

from tests.gpu_helpers import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2511_18871_b200 import parl

    return parl


CFGS = {"tiny": (16, 16, 2, 2, 24, 64), "c1": (4096, 256, 2, 4, 1024, 576)}


def test_sample_tokens_match_reference_fp32(P):
    """fp32 forward + the reference's fp64 choice and RNG stream: the same tokens, greedy and
    at temperatures 0.8 / 1.5 (stops after kEosToken like the reference)."""
    ctx = P.Context(0, P.PREC_FP32)
    z = load("sample_tokens.npz")
    models = {}
    for k in range(len(z["names"])):
        name, wseed = str(z["names"][k]), int(z["wseeds"][k])
        if name not in models:
            models[name] = P.ModelParams.init(P.ModelConfig(*CFGS[name]), wseed, ctx)
        want = z["tokens"][k][z["tokens"][k] >= 0]
        got = P.sample_tokens(models[name], z["prompts"][k], 24, float(z["temps"][k]), int(z["seeds"][k]))
        assert np.array_equal(got, want), (name, float(z["temps"][k]), got, want)


def test_sample_tokens_bf16_and_errors(P):
    ctx = P.Context(0, P.PREC_BF16)
    pm = P.ModelParams.init(P.ModelConfig(*CFGS["c1"]), 7, ctx)
    prompt = [5, 9, 100, 4000, 17, 8]
    a = P.sample_tokens(pm, prompt, 16, 0.0, 0)
    b = P.sample_tokens(pm, prompt, 16, 0.0, 0)
    assert np.array_equal(a, b) and len(a) >= 1 and (a >= 0).all() and (a < 4096).all()
    with pytest.raises(P.ShapeError):
        P.sample_tokens(pm, [], 4)
    with pytest.raises(P.ConfigError):
        P.sample_tokens(pm, prompt, -1)
    with pytest.raises(P.ConfigError):
        P.sample_tokens(pm, prompt, 4, -0.5)
    with pytest.raises(P.ShapeError):
        P.sample_tokens(pm, prompt, 576)
    with pytest.raises(P.VocabError):
        P.sample_tokens(pm, [4096], 2)


def test_score_logprobs_matches_oracle(P, orc):
    """score_logprobs (rollout.cpp:52-66) of a sampled response against the oracle's causal forward."""
    from oracle import Cfg

    ctx = P.Context(0, P.PREC_FP32)
    pm = P.ModelParams.init(P.ModelConfig(*CFGS["tiny"]), 41, ctx)
    prompt = [5, 9, 11, 4, 7]
    resp = P.sample_tokens(pm, prompt, 10, 0.8, 3)
    lp = P.score_logprobs(pm, prompt, resp)
    toks = np.concatenate([prompt, resp])
    labels = np.full(len(toks), -1)
    labels[len(prompt):] = resp
    want = orc.forward(Cfg(*CFGS["tiny"]), pm.flat(), toks, np.arange(len(toks)), labels)
    assert len(lp) == len(resp) and np.abs(lp - want).max() < 2e-5


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_kv_cached_group_decoder(P, prec):
    """parl_sample_group: the G rollouts of one prompt on one shared prompt cache give, sequence
    by sequence, what sample_tokens gives with that sequence's seed (fp32: the reference's own
    tokens, checked above); the returned log-probs are score_logprobs of the sampled tokens."""
    ctx = P.Context(0, P.PREC_FP32 if prec == "fp32" else P.PREC_BF16)
    cfg = CFGS["tiny"] if prec == "fp32" else CFGS["c1"]
    z = load("sample_tokens.npz")
    name = "tiny" if prec == "fp32" else "c1"
    pm = P.ModelParams.init(P.ModelConfig(*cfg), 41 if name == "tiny" else 7, ctx)
    prompt = [5, 9, 11, 4, 7, 3, 12]
    seeds = [11, 12, 13, 99, 7]
    for temp in (0.0, 0.8):
        toks, lps = P.sample_group(pm, prompt, len(seeds), 20, temp, seeds, want_logprobs=True)
        for k, s in enumerate(seeds):
            want = P.sample_tokens(pm, prompt, 20, temp, s)
            if prec == "fp32":
                assert np.array_equal(toks[k], want), (temp, k, toks[k], want)
            ref_lp = P.score_logprobs(pm, prompt, toks[k])
            tol = 1e-4 if prec == "fp32" else 0.1
            assert np.abs(lps[k] - ref_lp).max() < tol
    if prec == "fp32":  # the fixture's reference runs, now through the cached decoder
        for k in range(len(z["names"])):
            if str(z["names"][k]) != "tiny" or int(z["wseeds"][k]) != 41:
                continue
            want = z["tokens"][k][z["tokens"][k] >= 0]
            got = P.sample_group(pm, z["prompts"][k], 1, 24, float(z["temps"][k]), [int(z["seeds"][k])])[0]
            assert np.array_equal(got, want)
