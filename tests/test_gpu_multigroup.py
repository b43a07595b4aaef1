"""Several prompt groups in one packed sequence (SPEC.md:278 lifted).

One packed forward / backward over groups [P_0 R_0.. | P_1 R_1.. | ...] must give each group
what its own pack_group forward gives: attention never crosses groups, positions restart
per group, the loss takes per-group advantages.  Checked against per-group micro-steps on
the device (fp32: log-probs bit-identical, the summed gradient at fp32 tolerance; bf16: at
the bf16 tolerances) and against the C oracle.
"""
import numpy as np
import pytest

from tests.gpu_helpers import FP32_TOL, ocfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2511_18871_b200 import parl

    return parl


def _groups(rng, V, n, G, plen=(3, 150), rlen=(1, 170)):
    prompts = [rng.integers(4, V, int(rng.integers(*plen))) for _ in range(n)]
    resps = [[rng.integers(4, V, int(rng.integers(*rlen))) for _ in range(G)] for _ in range(n)]
    return prompts, resps


def test_multi_pack_layout(P, orc):
    ctx = P.Context(0, P.PREC_FP32)
    rng = np.random.default_rng(0)
    prompts, resps = _groups(rng, 100, 3, 4)
    T = sum(len(p) + sum(len(r) for r in rs) for p, rs in zip(prompts, resps))
    g = P.Group(T, 12, ctx).pack_multi(prompts, resps, 4096)
    d = g.download()
    off = 0
    for p, rs in zip(prompts, resps):
        o = orc.pack(p, rs, 4096)
        n = len(o["tokens"])
        for k in ("tokens", "labels", "positions"):
            assert np.array_equal(d[k][off:off + n], o[k]), k
        off += n
    assert off == g.T and g.S == sum(len(r) for rs in resps for r in rs)


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_multi_group_equals_per_group(P, orc, prec):
    ctx = P.Context(0, P.PREC_FP32 if prec == "fp32" else P.PREC_BF16)
    cfg = P.ModelConfig(64, 32, 2, 2, 64, 512) if prec == "fp32" else P.ModelConfig(512, 128, 2, 2, 256, 1024)
    rng = np.random.default_rng(1)
    tm = P.TriModel.init(cfg, 7, ctx)
    w = tm.policy.flat()
    tm.old_policy.upload(w + 0.01 * rng.standard_normal(len(w)))
    tm.reference.upload(w - 0.01 * rng.standard_normal(len(w)))
    n, G = 3, 4
    prompts, resps = _groups(rng, cfg.vocab_size, n, G)
    rewards = [rng.random(G) for _ in range(n)]
    hp = P.HyperParams()
    # one packed sequence over the three groups
    T = sum(len(p) + sum(len(r) for r in rs) for p, rs in zip(prompts, resps))
    gm = P.Group(T, n * G, ctx).pack_multi(prompts, resps, cfg.max_seq_len)
    gb_m = P.GradBuffer(tm.policy)
    ctx.stats_reset()
    st_m = P.train_microbatch(tm, gm, gb_m, hp, rewards=np.concatenate(rewards))
    lp_m = [gm.logprobs(s) for s in range(3)]
    # per group
    gb_s = P.GradBuffer(tm.policy)
    ctx.stats_reset()
    lp_s = [[], [], []]
    for q in range(n):
        pk = P.pack_group(prompts[q], resps[q], cfg.max_seq_len, ctx)
        P.train_microbatch(tm, pk.group, gb_s, hp, rewards=rewards[q], want_stats=False)
        for s in range(3):
            lp_s[s].append(pk.group.logprobs(s))
    st_s = ctx.stats()
    lp_s = [np.concatenate(x) for x in lp_s]
    g_m, g_s = gb_m.flat(), gb_s.flat()
    rel = np.linalg.norm(g_m - g_s) / np.linalg.norm(g_s)
    if prec == "fp32":
        for s in range(3):
            assert np.array_equal(lp_m[s], lp_s[s])
        assert rel < FP32_TOL["grad_rel"], rel
        assert abs(st_m["objective_sum"] - st_s["objective_sum"]) < 1e-6
        # and against the oracle, group by group
        oc = ocfg(cfg)
        g_ref = np.zeros(len(w))
        for q in range(n):
            orc.train_microbatch(oc, w, tm.old_policy.flat(), tm.reference.flat(), prompts[q], resps[q],
                                 orc.group_advantages(rewards[q]), grad_acc=g_ref)
        assert np.linalg.norm(g_m - g_ref) / np.linalg.norm(g_ref) < FP32_TOL["grad_rel"]
    else:
        for s in range(3):
            assert np.abs(lp_m[s] - lp_s[s]).max() < 0.05
        assert rel < 2e-2, rel
    assert st_m["total_units"] == st_s["total_units"]


def test_multi_pack_every_array_bit_exact(P):
    """All eleven K1 arrays of a several-group sequence with ragged group sizes and prompt lengths
    of every residue mod 4: each group is laid out exactly as a single pack_group of its own,
    shifted by its packed offset (positions restart; segments, scored rows, head-row CSR and the
    sample ids continue across groups; a group's first position has no predecessor)."""
    import ctypes as C

    from tests.test_gpu_parity import _pack_arrays_np

    f = P.LIB.parl_debug_group_arrays
    f.restype, f.argtypes = C.c_int, [C.c_void_p, C.c_void_p]
    ctx = P.Context(0, P.PREC_FP32)
    rng = np.random.default_rng(9)
    for trial in range(4):
        n = int(rng.integers(2, 7))
        sizes = [int(rng.integers(1, 7)) for _ in range(n)]
        prompts = [rng.integers(4, 151936, int(rng.integers(1, 200))).astype(np.int32) for _ in range(n)]
        resps = [[rng.integers(4, 151936, int(rng.integers(1, 300))).astype(np.int32) for _ in range(G)] for G in sizes]
        T = sum(len(p) + sum(len(r) for r in rs) for p, rs in zip(prompts, resps))
        g = P.Group(T, sum(sizes), ctx).pack_multi(prompts, resps, 4096)
        S = g.S
        exp = {k: [] for k in ("tokens", "labels", "positions", "seg", "pred", "row_ptr", "scored_pos", "scored_label",
                               "pred_pos", "sample_of", "row_idx")}
        gs = s0 = k0 = 0
        for q, (p, rs) in enumerate(zip(prompts, resps)):
            ref, Tq, Sq = _pack_arrays_np(p, rs)
            exp["tokens"].append(ref["tokens"])
            exp["labels"].append(ref["labels"])
            exp["positions"].append(ref["positions"])
            exp["seg"].append(ref["seg"] + q + k0)
            exp["pred"].append(np.where(ref["pred"] < 0, -1, ref["pred"] + gs))
            exp["row_ptr"].append(ref["row_ptr"][:Tq] + s0)
            exp["scored_pos"].append(ref["scored_pos"] + gs)
            exp["scored_label"].append(ref["scored_label"])
            exp["pred_pos"].append(ref["pred_pos"] + gs)
            exp["sample_of"].append(ref["sample_of"] + k0)
            exp["row_idx"].append(ref["row_idx"] + s0)
            gs, s0, k0 = gs + Tq, s0 + Sq, k0 + len(rs)
        exp["row_ptr"].append(np.array([S]))
        exp = {k: np.concatenate(v) for k, v in exp.items()}
        buf = np.zeros(6 * T + 1 + 5 * S, np.int32)
        assert f(g.h, buf.ctypes.data) == 0
        off = 0
        for name, m in (("tokens", T), ("labels", T), ("positions", T), ("seg", T), ("pred", T), ("row_ptr", T + 1),
                        ("scored_pos", S), ("scored_label", S), ("pred_pos", S), ("sample_of", S), ("row_idx", S)):
            assert np.array_equal(buf[off:off + m], exp[name]), (trial, name)
            off += m
