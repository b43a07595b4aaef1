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
