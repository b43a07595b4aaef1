"""GPU: the optimizer step and the GRPO operator API through the C-ABI.

* a full training iteration (pipeline.cpp:263-352: accumulate the micro-batches,
  divisor N*G, snapshot, apply_update) against the reference's own TriModel /
  GradBuffer / apply_update (oracle/_ref) or, without it, the C restatement;
* the micro-batch partition does not change the update (test_pipeline.cpp:292-308);
* rollout_weights mode: ratio exactly 1 at step 0 (test_pipeline.cpp:243-252);
* advantages incl. mean-only (test_grpo.cpp:29-60), the clip / KL closed forms and
  the microbatch loss (test_grpo.cpp:62-202) through the K7 kernels;
* non-finite updates refused with the weights untouched (test_model.cpp:207-212);
* token ids outside the vocabulary rejected before any kernel reads them.
"""
import math

import numpy as np
import pytest

from tests.gpu_helpers import FP32_TOL, ocfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2511_18871_b200 import parl

    return parl


@pytest.fixture(scope="module")
def ctx32(P):
    return P.Context(0, P.PREC_FP32)


@pytest.fixture(scope="module")
def ctx16(P):
    return P.Context(0, P.PREC_BF16)


def _oracle():
    import os

    from oracle import LIB_REF, Oracle

    return Oracle("ref") if os.path.exists(LIB_REF) else Oracle("c")


def _batch(rng, n_groups, G, V, plen=(2, 9), rlen=(1, 9)):
    out = []
    for _ in range(n_groups):
        prompt = rng.integers(4, V, int(rng.integers(*plen)))
        resp = [rng.integers(4, V, int(rng.integers(*rlen))) for _ in range(G)]
        rewards = rng.random(G)
        out.append((prompt, resp, rewards))
    return out


def _tri(P, ctx, cfg, seed=7, noise=0.01):
    tm = P.TriModel.init(cfg, seed, ctx)
    rng = np.random.default_rng(seed)
    w = tm.policy.flat()
    tm.old_policy.upload(w + noise * rng.standard_normal(len(w)))
    tm.reference.upload(w - noise * rng.standard_normal(len(w)))
    return tm


def _groups(P, ctx, cfg, batch, m, orc):
    """Shared-prompt micro-batches of m responses (G % m == 0) with the group's advantages."""
    mbs, host = [], []
    for prompt, resp, rewards in batch:
        adv = orc.group_advantages(rewards)
        for s in range(0, len(resp), m):
            pk = P.pack_group(prompt, resp[s:s + m], cfg.max_seq_len, ctx)
            mbs.append((pk.group, adv[s:s + m], None))
            host.append((prompt, resp[s:s + m], adv[s:s + m]))
    return mbs, host


@pytest.mark.parametrize("m", [4, 2])
def test_full_iteration_matches_reference(P, ctx32, m):
    """N=2 groups x G=4 through the drop-in, update divisor N*G (pipeline.cpp:346-351)."""
    orc = _oracle()
    cfg = P.ModelConfig(16, 16, 2, 2, 24, 64)
    tm = _tri(P, ctx32, cfg)
    w0, wo0, wr0 = tm.policy.flat(), tm.old_policy.flat(), tm.reference.flat()
    batch = _batch(np.random.default_rng(5), 2, 4, cfg.vocab_size)
    mbs, host = _groups(P, ctx32, cfg, batch, m, orc)
    hp = P.HyperParams()
    st = P.train_iteration(tm, mbs, hp, lr=0.1)
    w_new, w_old_new, st_ref = orc.train_iteration(ocfg(cfg), w0, wo0, wr0, host, 0.1)
    # snapshot_old_policy is the pre-update policy, bit for bit (pipeline.cpp:350)
    assert np.array_equal(tm.old_policy.flat(), w_old_new)
    assert tm.policy.version() == 1 and tm.old_policy.version() == 0
    d_gpu, d_ref = tm.policy.flat() - w0, w_new - w0
    rel = np.linalg.norm(d_gpu - d_ref) / np.linalg.norm(d_ref)
    assert rel < FP32_TOL["grad_rel"], rel
    assert abs(st["objective_sum"] - st_ref[0]) <= FP32_TOL["obj_rel"] * max(1.0, abs(st_ref[0]))
    assert st["total_units"] == st_ref[4] and st["clipped_units"] == st_ref[3]


def test_update_independent_of_micro_batch_size(P, ctx32):
    """Non-packed branch (pipeline.cpp:142-170): one causal forward per sample, canonical order;
    m in {1, 2, 4} gives bit-identical weights (test_pipeline.cpp:292-308)."""
    orc = _oracle()
    cfg = P.ModelConfig(16, 16, 1, 2, 16, 48)
    batch = _batch(np.random.default_rng(9), 2, 4, cfg.vocab_size, rlen=(1, 6))
    hp = P.HyperParams()
    results = []
    for m in (1, 2, 4):
        tm = _tri(P, ctx32, cfg, seed=77)
        gb = P.GradBuffer(tm.policy)
        gb.reset()
        samples = []
        for prompt, resp, rewards in batch:
            adv = orc.group_advantages(rewards)
            for j, r in enumerate(resp):
                samples.append((prompt, r, adv[j]))
        groups = []
        for prompt, r, a in samples:  # causal scoring inputs, pipeline.cpp:79-88
            toks = np.concatenate([prompt, r]).astype(np.int32)
            labels = np.full(len(toks), -1, np.int32)
            labels[len(prompt):] = r
            g = P.Group(len(toks), 1, ctx32)
            g.set_sequence(toks, np.arange(len(toks)), labels, P.AttentionMaskSpec.causal(), cfg.vocab_size,
                           cfg.max_seq_len)
            groups.append((g, [a]))
        for s in range(0, len(groups), m):  # micro-batches of m samples, trained in order
            for g, a in groups[s:s + m]:
                P.train_microbatch(tm, g, gb, hp, advantages=a, want_stats=False)
        gb.set_micro_step_count(len(samples))
        tm.snapshot_old_policy()
        tm.policy.apply_update(gb, 0.1)
        results.append(tm.policy.flat())
    assert np.array_equal(results[0], results[1]) and np.array_equal(results[0], results[2])


def test_shared_prompt_equals_unpacked_update(P, ctx32):
    """test_pipeline.cpp:254-270 at fp32 tolerance: packed (m=G) and per-sample causal updates."""
    orc = _oracle()
    cfg = P.ModelConfig(16, 16, 1, 2, 16, 48)
    batch = _batch(np.random.default_rng(13), 2, 4, cfg.vocab_size, rlen=(1, 6))
    hp = P.HyperParams()
    tm_p = _tri(P, ctx32, cfg, seed=77)
    w0 = tm_p.policy.flat()
    mbs, _ = _groups(P, ctx32, cfg, batch, 4, orc)
    P.train_iteration(tm_p, mbs, hp, lr=0.1)
    tm_u = _tri(P, ctx32, cfg, seed=77)
    gb = P.GradBuffer(tm_u.policy)
    for prompt, resp, rewards in batch:
        adv = orc.group_advantages(rewards)
        for j, r in enumerate(resp):
            toks = np.concatenate([prompt, r]).astype(np.int32)
            labels = np.full(len(toks), -1, np.int32)
            labels[len(prompt):] = r
            g = P.Group(len(toks), 1, ctx32)
            g.set_sequence(toks, np.arange(len(toks)), labels, P.AttentionMaskSpec.causal(), cfg.vocab_size,
                           cfg.max_seq_len)
            P.train_microbatch(tm_u, g, gb, hp, advantages=[adv[j]], want_stats=False)
    gb.set_micro_step_count(8)
    tm_u.snapshot_old_policy()
    tm_u.policy.apply_update(gb, 0.1)
    d_p, d_u = tm_p.policy.flat() - w0, tm_u.policy.flat() - w0
    assert np.linalg.norm(d_p - d_u) / np.linalg.norm(d_u) < FP32_TOL["grad_rel"]


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_rollout_weights_ratio_one(P, ctx32, ctx16, prec):
    """rollout_weights mode at step 0 (policy == old == ref): clip fraction 0 and KL 0
    (test_pipeline.cpp:243-252).  Old log-probs come from the rollout-side causal scoring."""
    ctx = ctx32 if prec == "fp32" else ctx16
    cfg = P.ModelConfig(16, 16, 2, 2, 24, 64) if prec == "fp32" else P.ModelConfig(512, 128, 2, 2, 256, 256)
    tm = P.TriModel.init(cfg, 77, ctx)
    rng = np.random.default_rng(3)
    prompt = rng.integers(4, cfg.vocab_size, 6)
    resp = [rng.integers(4, cfg.vocab_size, int(n)) for n in (5, 9, 3, 7)]
    old = np.concatenate([P.score_logprobs(tm.policy, prompt, r) for r in resp])
    pk = P.pack_group(prompt, resp, cfg.max_seq_len, ctx)
    gb = P.GradBuffer(tm.policy)
    ctx.stats_reset()
    st = P.train_microbatch(tm, pk.group, gb, P.HyperParams(), rewards=rng.random(4), rollout_old_logprobs=old)
    assert st["clipped_units"] == 0 and st["total_units"] == sum(len(r) for r in resp)
    assert st["kl_sum"] == 0.0  # policy and reference run identical kernels on identical weights
    assert np.array_equal(pk.group.logprobs(0), pk.group.logprobs(2))


def test_advantages_and_mean_only(P, ctx32, orc):
    """group_advantages[_mean_only] on the device (test_grpo.cpp:29-60)."""
    a = P.group_advantages([1.0, 0.0, 0.0, 1.0], ctx32)
    assert np.allclose(a, [1, -1, -1, 1], rtol=0, atol=1e-12)
    assert np.all(P.group_advantages([1.0] * 4, ctx32) == 0.0)
    with pytest.raises(P.ConfigError):
        P.group_advantages([0.5], ctx32)
    rng = np.random.default_rng(99)
    for trial in range(20):
        r = rng.random(2 + trial % 7) * 3 - 1
        for mo in (False, True):
            got = P.group_advantages(r, ctx32, mean_only=mo)
            assert np.allclose(got, orc.group_advantages(r, mean_only=mo), rtol=0, atol=1e-13)
        assert abs(P.group_advantages(r, ctx32).sum()) < 1e-12
        assert np.allclose(P.group_advantages(r + 17.25, ctx32), P.group_advantages(r, ctx32), atol=1e-12)
    # mean-only through the fused micro-step: the per-sample advantage table K7 used
    cfg = P.ModelConfig(16, 16, 2, 2, 24, 64)
    tm = _tri(P, ctx32, cfg)
    prompt = rng.integers(4, 16, 5)
    resp = [rng.integers(4, 16, int(n)) for n in (3, 4, 2, 5)]
    rewards = rng.random(4)
    pk = P.pack_group(prompt, resp, 64, ctx32)
    for mo in (False, True):
        gb = P.GradBuffer(tm.policy)
        ctx32.stats_reset()
        st = P.train_microbatch(tm, pk.group, gb, P.HyperParams(advantage_mean_only=mo), rewards=rewards)
        adv = orc.group_advantages(rewards, mean_only=mo)
        _, st_ref, _ = orc.train_microbatch(ocfg(cfg), tm.policy.flat(), tm.old_policy.flat(), tm.reference.flat(),
                                            prompt, resp, adv)
        assert abs(st["objective_sum"] - st_ref[0]) < 1e-5 and abs(st["kl_sum"] - st_ref[2]) < 1e-6


def test_grpo_closed_forms(P, ctx32):
    """test_grpo.cpp:62-202 through K7 (fp64 operator path)."""
    c = ctx32
    assert P.clipped_term(math.log(1.5), 0.0, 1.0, 0.2, c) == pytest.approx(1.2, rel=1e-12)
    assert P.clipped_term(math.log(0.5), 0.0, -1.0, 0.2, c) == pytest.approx(-0.8, rel=1e-12)
    for adv in (-2.0, 0.0, 0.7):
        assert P.clipped_term(-1.3, -1.3, adv, 0.2, c) == pytest.approx(adv, rel=1e-12, abs=1e-300)
    with pytest.raises(P.ConfigError):
        P.clipped_term(0.0, 0.0, 1.0, 1.5, c)
    with pytest.raises(P.NumericError):
        P.clipped_term(float("nan"), 0.0, 1.0, 0.2, c)
    assert P.kl_term(-1.7, -1.7, c) == 0.0
    assert P.kl_term(-2.0, -2.0 + math.log(2.0), c) == pytest.approx(2.0 - math.log(2.0) - 1.0, rel=1e-12)
    # identity-weights microbatch loss
    samples, lps = [], []
    advs = [1.0, -0.5, 0.25, 2.0]
    for j in range(4):
        v = [-1.0 - j, -0.5, -2.0 + 0.3 * j]
        samples.append(P.Sample(response=[6, 6, 6], advantage=advs[j], old_logprobs=v, ref_logprobs=v))
        lps.append(v)
    ml = P.grpo_microbatch_loss(samples, lps, 0.2, 0.04, "token", c)
    expect = -(1.0 - 0.5 + 0.25 + 2.0) / 4.0
    assert ml.loss == pytest.approx(expect, rel=1e-12)
    assert ml.report.clip_fraction == 0.0 and ml.report.kl_mean == 0.0 and ml.report.token_count == 12
    assert P.grpo_microbatch_loss(samples, lps, 0.2, 0.04, "sequence", c).loss == pytest.approx(expect, rel=1e-12)
    # clipped-branch upstream closed forms (test_grpo.cpp:169-202)
    eps, beta = 0.2, 0.04
    s = P.Sample(response=[6], advantage=1.0, old_logprobs=[-1.0 - math.log(1.5)], ref_logprobs=[-1.0 + 0.1])
    ml = P.grpo_microbatch_loss([s], [[-1.0]], eps, beta, "token", c)
    assert ml.upstream[0][0] == pytest.approx(-(0.0 - beta * -math.expm1(0.1)), rel=1e-15)
    assert ml.report.clip_fraction == 1.0
    s = P.Sample(response=[6], advantage=-1.0, old_logprobs=[-1.0 - math.log(0.5)], ref_logprobs=[-1.0 - 0.2])
    ml = P.grpo_microbatch_loss([s], [[-1.0]], eps, beta, "token", c)
    assert ml.upstream[0][0] == pytest.approx(-(0.0 - beta * -math.expm1(-0.2)), rel=1e-15)
    s = P.Sample(response=[6], advantage=-1.0, old_logprobs=[-1.0 - math.log(1.5)], ref_logprobs=[-1.0])
    ml = P.grpo_microbatch_loss([s], [[-1.0]], eps, beta, "token", c)
    assert ml.upstream[0][0] == pytest.approx(1.5, rel=1e-12) and ml.report.clip_fraction == 1.0


def test_microbatch_loss_matches_oracle_terms(P, ctx32, orc):
    """Multi-chunk K7 (several 2048-token blocks, samples straddling them) vs per_sample_terms."""
    rng = np.random.default_rng(4)
    lens = [700, 1, 3000, 5, 2100, 64]
    for gran in ("token", "sequence"):
        samples, lps = [], []
        for n in lens:
            lp = -3 * rng.random(n)
            samples.append(P.Sample(response=[6] * n, advantage=float(rng.standard_normal()),
                                    old_logprobs=lp + 0.3 * rng.standard_normal(n),
                                    ref_logprobs=lp + 0.1 * rng.standard_normal(n)))
            lps.append(lp)
        ml = P.grpo_microbatch_loss(samples, lps, 0.2, 0.04, gran, ctx32)
        obj = 0.0
        for s, lp, up in zip(samples, lps, ml.upstream):
            t = orc.sample_terms(lp, s.old_logprobs, s.ref_logprobs, s.advantage, 0.2, 0.04,
                                 0 if gran == "token" else 1)
            # sequence granularity differentiates sums over up to 3,000 log-probs, added in a fixed
            # tree order here and sequentially in the reference: ~1e-13 relative on the sums
            rtol = 1e-12 if gran == "token" else 1e-9
            assert np.allclose(up, -t["upstream"] / len(lens), rtol=rtol, atol=1e-15)
            obj += t["clip_term"] - 0.04 * t["kl"]
            pst = P.per_sample_terms(s, lp, 0.2, 0.04, gran, ctx32)
            assert pst.total_units == t["total_units"] and pst.clipped_units == t["clipped_units"]
            assert pst.clip_term == pytest.approx(t["clip_term"], rel=1e-9)
        assert ml.report.objective == pytest.approx(obj / len(lens), rel=1e-9)


@pytest.mark.parametrize("gran", ["token", "sequence"])
def test_microbatch_loss_ragged_at_scale(P, ctx32, gran):
    """K7 with 3M scored tokens (several spans per warp range, runs carried across them) and
    hundreds of 1-3 token samples (more samples than fit one warp's sample table), vs the fp64
    GRPO terms of torch_ref (grpo.cpp:111-184)."""
    from oracle import torch_ref as TR

    rng = np.random.default_rng(11)
    lens = [1] * 300 + [2, 3] * 100 + [1_000_003, 77, 1_400_000, 1] + [int(x) for x in rng.integers(1, 9, 200)] \
        + [600_000]
    S = sum(lens)
    lp = -3 * rng.random(S)
    cu = np.concatenate([[0], np.cumsum(lens)])
    # sequence granularity exponentiates differences of sums: per-token noise ~ 1/sqrt(n_j) there
    sc = 1.0 if gran == "token" else np.repeat(1.0 / np.sqrt(lens), lens)
    old = lp + 0.3 * sc * rng.standard_normal(S)
    ref = lp + 0.1 * sc * rng.standard_normal(S)
    adv = rng.standard_normal(len(lens))
    samples = [P.Sample(response=np.full(n, 6, np.int32), advantage=float(adv[j]),
                        old_logprobs=old[cu[j]:cu[j + 1]], ref_logprobs=ref[cu[j]:cu[j + 1]])
               for j, n in enumerate(lens)]
    ml = P.grpo_microbatch_loss(samples, [lp[cu[j]:cu[j + 1]] for j in range(len(lens))], 0.2, 0.04, gran, ctx32)
    n = len(lens)
    if gran == "token":
        up, st = TR.grpo_terms(lp, old, ref, lens, adv)
        assert np.allclose(np.concatenate(ml.upstream), up / n, rtol=1e-12, atol=1e-18)
        assert ml.report.objective == pytest.approx(st[0] / n, rel=1e-10)
        assert ml.report.clip_fraction == pytest.approx(st[3] / st[4], rel=1e-12)
    else:  # one evaluation per sample on the summed log-probs (grpo.cpp:134-149)
        sl, so, sr = (np.add.reduceat(x, cu[:-1]) for x in (lp, old, ref))
        up, st = TR.grpo_terms(sl, so, sr, [1] * n, adv)
        got = np.array([u[0] for u in ml.upstream])
        assert np.allclose(got, up / n, rtol=1e-8, atol=1e-18)
        for u in ml.upstream:
            assert np.all(u == u[0])
        assert ml.report.objective == pytest.approx(st[0] / n, rel=1e-8)


def test_shared_prompt_mask(P, ctx32):  # test_packing.cpp:79-107
    m = P.build_shared_prompt_mask(2, [1, 1], ctx32)
    assert m.astype(int).ravel().tolist() == [1, 0, 0, 0, 1, 1, 0, 0, 1, 1, 1, 0, 1, 1, 0, 1]
    m1 = P.build_shared_prompt_mask(2, [3], ctx32)
    assert np.array_equal(m1, np.tril(np.ones((5, 5), bool)))


def test_nonfinite_update_refused(P, ctx32):  # test_model.cpp:175-216
    cfg = P.ModelConfig(16, 16, 2, 2, 24, 32)
    p = P.ModelParams.init(cfg, 9, ctx32)
    before = p.flat()
    bad = P.GradBuffer(p)
    g = np.zeros(cfg.param_count())
    g[3] = np.nan
    bad.upload(g)
    bad.set_micro_step_count(1)
    assert not bad.all_finite()
    with pytest.raises(P.NumericError):
        p.apply_update(bad, 0.1)
    assert np.array_equal(p.flat(), before) and p.version() == 0
    huge = P.GradBuffer(p)
    g[3] = 3e38
    huge.upload(g)
    huge.set_micro_step_count(1)
    with pytest.raises(P.NumericError):  # result would be non-finite (model.cpp:213-216)
        p.apply_update(huge, 1e300)
    assert np.array_equal(p.flat(), before) and p.all_finite()
    with pytest.raises(P.ConfigError):
        p.apply_update(P.GradBuffer(p), 0.1)  # micro_step_count 0
    # one accumulation with count 1 == two with count 2, bit for bit
    g1 = P.GradBuffer(p)
    g1.upload(0.25 * (np.arange(cfg.param_count()) % 5))
    g1.set_micro_step_count(1)
    a, b = p.clone(), p.clone()
    a.apply_update(g1, 0.3)
    g2 = P.GradBuffer(p)
    g2.accumulate(g1)
    g2.accumulate(g1)
    assert g2.micro_step_count() == 2
    b.apply_update(g2, 0.3)
    assert np.array_equal(a.flat(), b.flat())


def test_vocab_checked_before_kernels(P, ctx32):
    cfg = P.ModelConfig(16, 16, 1, 2, 16, 64)
    tm = P.TriModel.init(cfg, 3, ctx32)
    gb = P.GradBuffer(tm.policy)
    for bad in (16, 99, -1):
        pk = P.pack_group([1, 5, 3], [[7, bad], [9]], 64, ctx32)
        with pytest.raises(P.VocabError):
            P.train_microbatch(tm, pk.group, gb, P.HyperParams(), rewards=[0.1, 0.9])
    # device-packed inputs: K1's id range is checked before the forward
    import torch

    pr = torch.tensor([1, 5, 3], dtype=torch.int32, device="cuda")
    rs = torch.tensor([7, 8, 40], dtype=torch.int32, device="cuda")
    g = P.Group(8, 2, ctx32)
    g.pack_device(pr.data_ptr(), 3, rs.data_ptr(), [2, 1], 64)
    torch.cuda.synchronize()
    with pytest.raises(P.VocabError):
        P.train_microbatch(tm, g, gb, P.HyperParams(), rewards=[0.1, 0.9])
    with pytest.raises(P.ConfigError):
        g.set_logprobs(3, np.zeros(g.S))
    assert gb.micro_step_count() == 0


def test_bf16_trimodel_identical_weights_bitwise(P, ctx16):
    """test_pipeline.cpp:118-136 on the grouped tcgen05 path: the three role outputs are identical."""
    cfg = P.ModelConfig(4096, 256, 2, 4, 1024, 576)
    tm = P.TriModel.init(cfg, 7, ctx16)
    rng = np.random.default_rng(1)
    prompt = rng.integers(4, 4096, 64)
    resp = [rng.integers(4, 4096, 128) for _ in range(4)]
    pk = P.pack_group(prompt, resp, 576, ctx16)
    gb = P.GradBuffer(tm.policy)
    P.train_microbatch(tm, pk.group, gb, P.HyperParams(), rewards=rng.random(4))
    lp = [pk.group.logprobs(s) for s in range(3)]
    assert np.array_equal(lp[0], lp[1]) and np.array_equal(lp[0], lp[2])
    assert np.all(np.isfinite(lp[0]))


def test_model_copy_keeps_init_seed(P, ctx32, tmp_path):
    cfg = P.ModelConfig(16, 16, 2, 2, 24, 64)
    p = P.ModelParams.init(cfg, 41, ctx32)
    q = p.clone()
    assert q.init_seed() == 41
    p.save(str(tmp_path / "a.ckpt"))
    q.save(str(tmp_path / "b.ckpt"))
    assert (tmp_path / "a.ckpt").read_bytes() == (tmp_path / "b.ckpt").read_bytes()


def test_logprob_rows_normalized(P, ctx32):
    """test_model.cpp:72-93 at fp32: rows normalised, log-probs <= 0, and a forward_logprobs value
    equals its forward_logprob_rows entry bit for bit (the same LSE kernel and rounding)."""
    cfg = P.ModelConfig(16, 16, 2, 2, 24, 32)
    p = P.ModelParams.init(cfg, 3, ctx32)
    tokens = [1, 5, 9, 4, 2]
    rows = P.forward_logprob_rows(p, tokens, np.arange(5), P.AttentionMaskSpec.causal())
    assert np.abs(np.exp(rows).sum(1) - 1).max() < 1e-5 and rows.max() <= 0
    labels = [-1, -1, 9, -1, -1]
    out = P.forward_logprobs(p, tokens, np.arange(5), P.AttentionMaskSpec.causal(), labels)
    assert out.logprobs[0] == rows[1, 9]


@pytest.mark.parametrize("mean_only", [False, True])
def test_grpo_device_path_rewards_at_scale(P, ctx32, mean_only):
    """K7 on the device path (fp32 log-probs in the group, advantages rebuilt in-kernel from the
    rewards per prompt group, grpo.cpp:24-48) over ~0.8M scored tokens of 24 groups x 8 ragged
    responses packed into one sequence, against the fp64 GRPO terms of the same fp32 inputs."""
    from oracle import torch_ref as TR

    rng = np.random.default_rng(21)
    n, G = 24, 8
    prompts = [rng.integers(4, 4096, int(rng.integers(1, 64))).astype(np.int32) for _ in range(n)]
    resps = [[rng.integers(4, 4096, int(rng.integers(1, 8000))).astype(np.int32) for _ in range(G)] for _ in range(n)]
    T = sum(len(p) + sum(len(r) for r in rs) for p, rs in zip(prompts, resps))
    g = P.Group(T, n * G, ctx32).pack_multi(prompts, resps, 1 << 16)
    S = g.S
    lens = [len(r) for rs in resps for r in rs]
    lp = (-3 * rng.random(S)).astype(np.float32).astype(np.float64)  # the group holds fp32 log-probs
    old = (lp + 0.3 * rng.standard_normal(S)).astype(np.float32).astype(np.float64)
    ref = (lp + 0.1 * rng.standard_normal(S)).astype(np.float32).astype(np.float64)
    for slot, v in enumerate((lp, old, ref)):
        g.set_logprobs(slot, v)
    rewards = rng.random(n * G)
    ctx32.stats_reset()
    st = P.grpo_loss(ctx32, g, P.HyperParams(0.2, 0.04, "token", mean_only), rewards=rewards)
    adv = np.concatenate([TR.group_advantages(rewards[q * G:(q + 1) * G], mean_only) for q in range(n)])
    up, st_x = TR.grpo_terms(lp, old, ref, lens, adv)
    # the clipped gradient is discontinuous at r = 1 +- eps: a ratio within fp32 rounding of the
    # boundary may take the other branch (the clipped value itself is continuous there)
    r = np.exp(lp - old)
    edge = (np.abs(r - 0.8) < 2e-6) | (np.abs(r - 1.2) < 2e-6)
    assert edge.sum() <= max(8, 1e-5 * S)
    assert np.allclose(g.upstream()[~edge], up[~edge], rtol=2e-5, atol=1e-10)
    scale = np.abs(adv).sum() + abs(st_x[0])
    assert abs(st["objective_sum"] - st_x[0]) <= 1e-5 * scale
    assert abs(st["kl_sum"] - st_x[2]) <= 1e-5 * (abs(st_x[2]) + 1)
    assert abs(st["clipped_units"] - st_x[3]) <= edge.sum() and st["total_units"] == st_x[4]
