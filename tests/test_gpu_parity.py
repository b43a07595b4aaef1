"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
golden fixtures generated from the reference build.

Integer work (packing, segments, predecessors) is bit-exact; floating point
is held to the SURVEY.md §8c tolerances written in tests/gpu_helpers.py.
"""
import numpy as np
import pytest

from tests.gpu_helpers import BF16_TOL, FP32_TOL, load, ocfg, per_tensor_rel, split_resp

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


def tiny(P):
    return P.ModelConfig(16, 16, 2, 2, 24, 64)


def c1(P):
    return P.ModelConfig(4096, 256, 2, 4, 1024, 576)


# --------------------------------------------------------------------------- K1 packer
def test_pack_bit_exact_vs_oracle(P, ctx32, orc):
    rng = np.random.default_rng(3)
    for trial in range(30):
        Pn = int(rng.integers(1, 40))
        G = int(rng.integers(1, 9))
        resp = [rng.integers(4, 100, int(rng.integers(1, 50))) for _ in range(G)]
        prompt = rng.integers(4, 100, Pn)
        pk = P.pack_group(prompt, resp, 4096, ctx32)
        d = pk.group.download()
        o = orc.pack(prompt, resp, 4096)
        for k in ("tokens", "labels", "positions", "seg", "pred", "span_start"):
            assert np.array_equal(d[k], o[k]), (trial, k)
        assert np.array_equal(d["scored_pos"], np.arange(Pn, Pn + sum(len(r) for r in resp)))


def test_pack_golden_lists_and_errors(P, ctx32):  # test_packing.cpp:46-76
    pk = P.pack_group([1, 5, 3], [[7, 8], [9, 10]], 64, ctx32)
    assert pk.tokens.tolist() == [1, 5, 3, 7, 8, 9, 10]
    assert pk.positions.tolist() == [0, 1, 2, 3, 4, 3, 4]
    assert pk.spans == [(3, 2), (5, 2)]
    pk = P.pack_group([1, 5, 3], [[7], [8, 9, 10]], 64, ctx32)
    assert pk.positions.tolist() == [0, 1, 2, 3, 3, 4, 5]
    with pytest.raises(P.ShapeError, match="max_seq_len"):
        P.pack_group([1, 5, 3], [[7, 8], [9, 10]], 6, ctx32)
    for bad in (([], [[7]]), ([1, 5, 3], [[7], []])):
        with pytest.raises(P.ShapeError):
            P.pack_group(bad[0], bad[1], 64, ctx32)


def test_pack_large_bit_exact(P, ctx32, orc):
    rng = np.random.default_rng(4)
    prompt = rng.integers(4, 151936, 512)
    resp = [rng.integers(4, 151936, 1024) for _ in range(8)]
    d = P.pack_group(prompt, resp, 16384, ctx32).group.download()
    o = orc.pack(prompt, resp, 16384)
    for k in ("tokens", "labels", "positions", "seg", "pred"):
        assert np.array_equal(d[k], o[k]), k


def _pack_arrays_np(prompt, resp):
    """Every K1 array restated (packing.cpp:7-45, model.cpp:230-253; head-row CSR of kernels.cuh)."""
    Pn, G = len(prompt), len(resp)
    lens = np.array([len(r) for r in resp])
    cu = np.concatenate([[0], np.cumsum(lens)])
    S, T = int(cu[-1]), Pn + int(cu[-1])
    k = np.repeat(np.arange(G), lens)
    s = np.arange(S)
    i = s - cu[k]
    rt = np.concatenate(resp) if S else np.zeros(0, int)
    t = Pn + s
    pred_r = np.where(i == 0, Pn - 1, t - 1)
    out = {"tokens": np.concatenate([prompt, rt]), "labels": np.concatenate([np.full(Pn, -1), rt]),
           "positions": np.concatenate([np.arange(Pn), Pn + i]), "seg": np.concatenate([np.zeros(Pn), k + 1]),
           "pred": np.concatenate([np.arange(Pn) - 1, pred_r]),
           "row_ptr": np.concatenate([np.zeros(Pn), G + s - k, [S]]),
           "scored_pos": t, "scored_label": rt, "pred_pos": pred_r, "sample_of": k}
    row_idx = np.zeros(S, np.int64)
    row_idx[:G] = cu[:G]
    nl = i != lens[k] - 1
    row_idx[(G + s - k)[nl]] = (s + 1)[nl]
    out["row_idx"] = row_idx
    return out, T, S


@pytest.mark.parametrize("Pn", [1, 2, 3, 4, 5, 511, 513, 1023])
def test_pack_every_array_bit_exact(P, ctx32, Pn):
    """All eleven K1 arrays (incl. the scored-row gathers and the head-row CSR) against a numpy
    restatement, for every prompt length mod 4 (the 16-byte store paths), over several blocks of
    the grid-stride loop and with many short responses."""
    import ctypes as C

    f = P.LIB.parl_debug_group_arrays
    f.restype, f.argtypes = C.c_int, [C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(Pn)
    for G, hi in ((1, 300), (3, 2000), (64, 40), (200, 9000)):
        prompt = rng.integers(4, 151936, Pn).astype(np.int32)
        resp = [rng.integers(4, 151936, int(rng.integers(1, hi))).astype(np.int32) for _ in range(G)]
        pk = P.pack_group(prompt, resp, 1 << 22, ctx32)
        ref, T, S = _pack_arrays_np(prompt, resp)
        buf = np.zeros(6 * T + 1 + 5 * S, np.int32)
        assert f(pk.group.h, buf.ctypes.data) == 0
        off = 0
        for name, n in (("tokens", T), ("labels", T), ("positions", T), ("seg", T), ("pred", T), ("row_ptr", T + 1),
                        ("scored_pos", S), ("scored_label", S), ("pred_pos", S), ("sample_of", S), ("row_idx", S)):
            assert np.array_equal(buf[off:off + n], ref[name]), (Pn, G, name)
            off += n


# --------------------------------------------------------------------------- init parity
def test_init_bit_exact(P, ctx32, orc):
    cfg = tiny(P)
    w = P.ModelParams.init(cfg, 41, ctx32).flat()
    assert np.array_equal(w, orc.init_params(ocfg(cfg), 41))


# --------------------------------------------------------------------------- forward / backward (fp32)
def test_tiny_packed_fp32(P, ctx32):
    z = load("tiny_packed.npz")
    cfg = tiny(P)
    pm = P.ModelParams.init(cfg, int(z["seed"]), ctx32)
    mask = P.AttentionMaskSpec.shared_prompt(len(z["prompt"]), z["lens"])
    f = P.forward_logprobs(pm, z["tokens"], z["positions"], mask, z["labels"], want_cache=True)
    assert np.abs(f.logprobs - z["logprobs"]).max() < FP32_TOL["lp_abs"]
    g = P.backward(pm, f, z["upstream"]).flat()
    rel = per_tensor_rel(ocfg(cfg), g, z["grad"])
    worst = max((v, k) for k, v in rel.items() if not k.endswith("attn.bk"))
    assert worst[0] < FP32_TOL["grad_rel"], worst
    assert max(v for k, v in rel.items() if k.endswith("attn.bk")) < FP32_TOL["bk_abs"]


def test_tiny_causal_fp32(P, ctx32):
    z = load("tiny_causal.npz")
    cfg = tiny(P)
    pm = P.ModelParams.init(cfg, int(z["seed"]), ctx32)
    f = P.forward_logprobs(pm, z["tokens"], z["positions"], P.AttentionMaskSpec.causal(), z["labels"], True)
    assert np.abs(f.logprobs - z["logprobs"]).max() < FP32_TOL["lp_abs"]
    g = P.backward(pm, f, z["upstream"]).flat()
    rel = per_tensor_rel(ocfg(cfg), g, z["grad"])
    assert max(v for k, v in rel.items() if not k.endswith("attn.bk")) < FP32_TOL["grad_rel"]
    rows = P.forward_logprob_rows(pm, z["tokens"], z["positions"], P.AttentionMaskSpec.causal())
    assert np.abs(rows - z["rows"]).max() < FP32_TOL["lp_abs"]


@pytest.mark.parametrize("gran", [0, 1])
def test_tiny_microbatch_fp32(P, ctx32, gran):
    from oracle.make_golden import perturb

    z = load("tiny_micro.npz")
    cfg = tiny(P)
    pol = P.ModelParams.init(cfg, int(z["seed"]), ctx32)
    w = pol.flat()
    tm = P.TriModel(pol, P.ModelParams.from_flat(cfg, perturb(w, int(z["old_seed"]), float(z["scale"])), ctx=ctx32),
                    P.ModelParams.from_flat(cfg, perturb(w, int(z["ref_seed"]), float(z["scale"])), ctx=ctx32))
    pk = P.pack_group(z["prompt"], split_resp(z), cfg.max_seq_len, ctx32)
    gb = P.GradBuffer(pol)
    ctx32.stats_reset()
    hyper = P.HyperParams(0.2, 0.04, "token" if gran == 0 else "sequence")
    st = P.train_microbatch(tm, pk.group, gb, hyper, rewards=z["rewards"])
    ref_st = z[f"stats_g{gran}"]
    lp3 = z[f"lp3_g{gran}"]
    for slot in range(3):
        assert np.abs(pk.group.logprobs(slot) - lp3[slot]).max() < FP32_TOL["lp_abs"]
    got = np.array([st[k] for k in ("objective_sum", "clip_sum", "kl_sum", "clipped_units", "total_units")])
    assert abs(got[0] - ref_st[0]) <= FP32_TOL["obj_rel"] * max(abs(ref_st[0]), 1e-3)
    assert got[4] == ref_st[4]
    rel = per_tensor_rel(ocfg(cfg), gb.flat(), z[f"grad_g{gran}"])
    assert max(v for k, v in rel.items() if not k.endswith("attn.bk")) < FP32_TOL["grad_rel"]
    assert gb.micro_step_count() == 1


def c2w(P):
    return P.ModelConfig(4096, 896, 1, 14, 4864, 512)


def _c1_setup(P, ctx, name="c1_micro.npz", cfg_of=c1):
    from oracle.make_golden import perturb

    z = load(name)
    cfg = cfg_of(P)
    pol = P.ModelParams.init(cfg, int(z["seed"]), ctx)
    w = pol.flat()
    tm = P.TriModel(pol, P.ModelParams.from_flat(cfg, perturb(w, int(z["old_seed"]), float(z["scale"])), ctx=ctx),
                    P.ModelParams.from_flat(cfg, perturb(w, int(z["ref_seed"]), float(z["scale"])), ctx=ctx))
    pk = P.pack_group(z["prompt"], split_resp(z), cfg.max_seq_len, ctx)
    return z, cfg, tm, pk


def _grad_summaries(cfg, g, z):
    from oracle import layout

    rels = {}
    for (name, off, r, c), l2 in zip(layout(ocfg(cfg)), z["grad_l2"]):
        if name.endswith("attn.bk"):
            continue
        rels[name] = abs(np.linalg.norm(g[off:off + r * c]) - l2) / max(l2, 1e-30)
    return rels


def test_c1_microbatch_fp32(P, ctx32):
    z, cfg, tm, pk = _c1_setup(P, ctx32)
    gb = P.GradBuffer(tm.policy)
    ctx32.stats_reset()
    st = P.train_microbatch(tm, pk.group, gb, P.HyperParams(), advantages=z["advantages"])
    for slot in range(3):
        assert np.abs(pk.group.logprobs(slot) - z["lp3"][slot]).max() < FP32_TOL["lp_abs"]
    assert abs(st["objective_sum"] - z["stats"][0]) <= FP32_TOL["obj_rel"] * abs(z["stats"][0]) + 1e-9
    g = gb.flat()
    sampled = g[z["grad_idx"]]
    ref = z["grad_vals"]
    assert np.linalg.norm(sampled - ref) / np.linalg.norm(ref) < FP32_TOL["grad_rel"]
    rels = _grad_summaries(cfg, g, z)
    assert max(rels.values()) < FP32_TOL["grad_rel"], max(rels.items(), key=lambda kv: kv[1])


def _fixture_upstream(z, orc):
    """Backward seed of the golden micro-batch, recomputed in fp64 from its log-probs."""
    lp3, up, c = z["lp3"], [], 0
    for j, n in enumerate(z["lens"]):
        t = orc.sample_terms(lp3[0][c:c + n], lp3[1][c:c + n], lp3[2][c:c + n], z["advantages"][j], 0.2, 0.04)
        up.append(-t["upstream"])
        c += n
    return np.concatenate(up)


def test_c1_forward_bf16(P, ctx16):
    z, cfg, tm, pk = _c1_setup(P, ctx16)
    act = P.C.c_void_p()
    P._check(P.LIB.parl_trimodel_forward(ctx16.h, tm.policy.h, tm.old_policy.h, tm.reference.h, pk.group.h,
                                         P.C.byref(act)), ctx16.h)
    P.LIB.parl_act_destroy(act)
    for slot in range(3):
        d = np.abs(pk.group.logprobs(slot) - z["lp3"][slot])
        assert d.max() < BF16_TOL["lp_max"] and d.mean() < BF16_TOL["lp_mean"], (slot, d.max(), d.mean())


def test_c1_backward_bf16(P, ctx16, orc):
    """bf16 backward against the reference gradient for the same upstream seed."""
    z, cfg, tm, pk = _c1_setup(P, ctx16)
    f = P.forward_logprobs(tm.policy, pk.tokens, pk.positions, pk.mask, pk.labels, want_cache=True)
    g = P.backward(tm.policy, f, _fixture_upstream(z, orc)).flat()
    sampled, ref = g[z["grad_idx"]], z["grad_vals"]
    cos = sampled @ ref / (np.linalg.norm(sampled) * np.linalg.norm(ref))
    assert cos > BF16_TOL["cos"], cos
    rels = _grad_summaries(cfg, g, z)
    assert max(rels.values()) < BF16_TOL["grad_rel"], max(rels.items(), key=lambda kv: kv[1])


def test_c1_microbatch_bf16_stats(P, ctx16):
    z, cfg, tm, pk = _c1_setup(P, ctx16)
    gb = P.GradBuffer(tm.policy)
    ctx16.stats_reset()
    st = P.train_microbatch(tm, pk.group, gb, P.HyperParams(), advantages=z["advantages"])
    assert abs(st["objective_sum"] - z["stats"][0]) <= BF16_TOL["obj_rel"] * abs(z["stats"][0]) + 1e-3
    assert st["total_units"] == z["stats"][4]
    assert gb.micro_step_count() == 1


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_c2_width_microbatch(P, ctx32, ctx16, orc, prec):
    """C2's layer width (d=896, H=14, F=4864) on a ragged group: the kernels' wide-row
    paths (LayerNorm backward, padded activations, head) against the reference."""
    ctx = ctx32 if prec == "fp32" else ctx16
    # Rounding grows with the contraction widths (d=896, F=4864 vs C1's 256 / 1024), so the
    # SURVEY.md 8c bounds (calibrated at C1) are scaled: 2x for fp32; 1.5x for the bf16 log-prob
    # bounds (two independent kernel generations measure the same 0.116 max / 0.021 mean here)
    if prec == "fp32":
        tol = {k: 2 * v for k, v in FP32_TOL.items()}
    else:
        tol = dict(BF16_TOL, lp_max=1.5 * BF16_TOL["lp_max"], lp_mean=1.5 * BF16_TOL["lp_mean"],
                   obj_rel=5 * BF16_TOL["obj_rel"])  # the objective inherits the log-prob rounding
    z, cfg, tm, pk = _c1_setup(P, ctx, "c2w_micro.npz", c2w)
    gb = P.GradBuffer(tm.policy)
    ctx.stats_reset()
    st = P.train_microbatch(tm, pk.group, gb, P.HyperParams(), advantages=z["advantages"])
    for slot in range(3):
        d = np.abs(pk.group.logprobs(slot) - z["lp3"][slot])
        if prec == "fp32":
            assert d.max() < tol["lp_abs"], (slot, d.max())
        else:
            assert d.max() < tol["lp_max"] and d.mean() < tol["lp_mean"], (slot, d.max(), d.mean())
    assert abs(st["objective_sum"] - z["stats"][0]) <= tol["obj_rel"] * abs(z["stats"][0]) + 1e-3
    g = gb.flat()
    if prec == "bf16":  # the bf16 upstream inherits the log-prob rounding: check the backward at the reference's seed
        f = P.forward_logprobs(tm.policy, pk.tokens, pk.positions, pk.mask, pk.labels, want_cache=True)
        g = P.backward(tm.policy, f, _fixture_upstream(z, orc)).flat()
    sampled, ref = g[z["grad_idx"]], z["grad_vals"]
    if prec == "fp32":
        assert np.linalg.norm(sampled - ref) / np.linalg.norm(ref) < tol["grad_rel"]
    else:
        assert sampled @ ref / (np.linalg.norm(sampled) * np.linalg.norm(ref)) > tol["cos"]
    rels = _grad_summaries(cfg, g, z)
    assert max(rels.values()) < tol["grad_rel"], max(rels.items(), key=lambda kv: kv[1])


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("fixture", ["c1_micro.npz", "c2w_micro.npz"])
def test_recompute_bitwise(P, ctx32, ctx16, prec, fixture):
    """Activation recomputation (only x_0..x_L kept, layers and bf16 logits rebuilt in
    the backward) runs the same kernels on the same inputs: log-probs, stats and
    gradients are bit-identical to the keep-everything mode."""
    ctx = ctx32 if prec == "fp32" else ctx16
    z, cfg, tm, pk = _c1_setup(P, ctx, fixture, c1 if fixture.startswith("c1") else c2w)
    out = []
    try:
        for mode in (2, 1, 2):
            ctx.set_recompute(mode)
            gb = P.GradBuffer(tm.policy)
            ctx.stats_reset()
            st = P.train_microbatch(tm, pk.group, gb, P.HyperParams(), advantages=z["advantages"])
            out.append((gb.flat(), [pk.group.logprobs(s) for s in range(3)], st["objective_sum"]))
    finally:
        ctx.set_recompute(0)
    for g, lps, obj in out[1:]:
        assert np.array_equal(g, out[0][0])
        for a, b in zip(lps, out[0][1]):
            assert np.array_equal(a, b)
        assert obj == out[0][2]
    assert np.abs(out[1][0]).sum() > 0


# --------------------------------------------------------------------------- reference contracts
def test_determinism_bitwise(P, ctx32):  # test_model.cpp:251-265
    cfg = tiny(P)
    pm = P.ModelParams.init(cfg, 17, ctx32)
    toks, labs = [1, 4, 9, 6, 2], [-1, 4, 9, 6, 2]
    u = [1.0, -0.5, 0.25, 2.0]
    out = []
    for _ in range(2):
        f = P.forward_logprobs(pm, toks, range(5), P.AttentionMaskSpec.causal(), labs, True)
        out.append((f.logprobs, P.backward(pm, f, u).flat()))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


def test_backward_linearity_exact(P, ctx32):  # test_model.cpp:131-153
    cfg = tiny(P)
    pm = P.ModelParams.init(cfg, 5, ctx32)
    toks, labs = [1, 5, 6, 7], [-1, 5, 9, 2]
    f = P.forward_logprobs(pm, toks, range(4), P.AttentionMaskSpec.causal(), labs, True)
    assert (P.backward(pm, f, [0.0, 0.0, 0.0]).flat() == 0).all()
    f = P.forward_logprobs(pm, toks, range(4), P.AttentionMaskSpec.causal(), labs, True)
    g1 = P.backward(pm, f, [0.3, -1.1, 0.7]).flat()
    f = P.forward_logprobs(pm, toks, range(4), P.AttentionMaskSpec.causal(), labs, True)
    g2 = P.backward(pm, f, [0.6, -2.2, 1.4]).flat()
    assert np.array_equal(g2, 2 * g1)


def test_no_leakage_bitwise(P, ctx32):  # test_packing.cpp:202-223
    cfg = tiny(P)
    pm = P.ModelParams.init(cfg, 53, ctx32)
    prompt = [1, 12, 3]
    base = [[5, 6], [7, 8], [9, 10]]
    mut = [[5, 6], [13, 14], [9, 10]]
    outs = []
    for resp in (base, mut):
        pk = P.pack_group(prompt, resp, cfg.max_seq_len, ctx32)
        f = P.forward_logprobs(pm, pk.tokens, pk.positions, pk.mask, pk.labels)
        outs.append(P.extract_response_logprobs(f.logprobs, pk))
    for j in (0, 2):
        assert np.array_equal(outs[0][j], outs[1][j])


def test_single_response_equals_causal(P, ctx32):  # test_packing.cpp:153-162
    cfg = tiny(P)
    pm = P.ModelParams.init(cfg, 43, ctx32)
    prompt, resp = [1, 6, 9, 3], [5, 7, 2]
    pk = P.pack_group(prompt, [resp], 64, ctx32)
    a = P.forward_logprobs(pm, pk.tokens, pk.positions, pk.mask, pk.labels).logprobs
    toks = prompt + resp
    b = P.forward_logprobs(pm, toks, range(7), P.AttentionMaskSpec.causal(), [-1] * 4 + resp).logprobs
    assert np.array_equal(a, b)


def test_shared_equals_replicated(P, ctx32):  # test_packing.cpp:123-200
    cfg = tiny(P)
    pm = P.ModelParams.init(cfg, 47, ctx32)
    rng = np.random.default_rng(29)
    prompt = [1, 8, 4]
    resp = [[5, 6], [7], [9, 10, 11]]
    pk = P.pack_group(prompt, resp, cfg.max_seq_len, ctx32)
    u = rng.uniform(-1, 1, 6)
    f = P.forward_logprobs(pm, pk.tokens, pk.positions, pk.mask, pk.labels, True)
    gp = P.backward(pm, f, u).flat()
    gs = P.GradBuffer(pm)
    c = 0
    for r in resp:
        toks = prompt + r
        fr = P.forward_logprobs(pm, toks, range(len(toks)), P.AttentionMaskSpec.causal(), [-1] * 3 + r, True)
        assert np.abs(fr.logprobs - f.logprobs[c:c + len(r)]).max() < FP32_TOL["lp_abs"]
        P.backward(pm, fr, u[c:c + len(r)], gs)
        c += len(r)
    gsum = gs.flat()
    assert np.linalg.norm(gp - gsum) / np.linalg.norm(gsum) < FP32_TOL["grad_rel"]


def test_trimodel_identical_weights(P, ctx32):  # test_pipeline.cpp:118-136
    cfg = tiny(P)
    tm = P.TriModel.init(cfg, 5, ctx32)
    tri = P.trimodel_forward(tm, [1, 6, 3, 7, 8], range(5), P.AttentionMaskSpec.causal(), [-1, -1, -1, 7, 8])
    assert np.array_equal(tri.policy.logprobs, tri.old_logprobs)
    assert np.array_equal(tri.policy.logprobs, tri.ref_logprobs)


def test_errors_map_to_reference_types(P, ctx32):  # test_model.cpp:107-173
    cfg = tiny(P)
    pm = P.ModelParams.init(cfg, 1, ctx32)
    with pytest.raises(P.ShapeError):
        P.forward_logprobs(pm, [1, 2, 3], [0, 1], P.AttentionMaskSpec.causal(), [-1, 2, 2])
    with pytest.raises(P.VocabError):
        P.forward_logprobs(pm, [1, 99, 3], range(3), P.AttentionMaskSpec.causal(), [-1, 2, 2])
    with pytest.raises(P.ShapeError):
        P.forward_logprobs(pm, [1, 2, 3], range(3), P.AttentionMaskSpec.causal(), [3, -1, -1])
    f = P.forward_logprobs(pm, [1, 5, 6], range(3), P.AttentionMaskSpec.causal(), [-1, 5, 9], True)
    P.forward_logprobs(pm, [1, 5, 6], range(3), P.AttentionMaskSpec.causal(), [-1, 5, 9])
    with pytest.raises(P.LifecycleError):
        P.backward(pm, f, [1.0, 1.0])
    f2 = P.forward_logprobs(pm, [1, 5, 6], range(3), P.AttentionMaskSpec.causal(), [-1, 5, 9], True)
    with pytest.raises(P.ShapeError):
        P.backward(pm, f2, [1.0] * 5)
    with pytest.raises(P.ConfigError):
        P.ModelParams(P.ModelConfig(16, 30, 2, 4, 24, 64), ctx32)


def test_apply_update_semantics(P, ctx32):  # test_model.cpp:175-216
    cfg = tiny(P)
    pm = P.ModelParams.init(cfg, 9, ctx32)
    w0 = pm.flat()
    f = P.forward_logprobs(pm, [1, 5, 6, 7], range(4), P.AttentionMaskSpec.causal(), [-1, 5, 9, 2], True)
    g = P.backward(pm, f, [0.3, -1.1, 0.7])
    pm.apply_update(g, 0.5)
    assert pm.version() == 1
    assert np.allclose(pm.flat(), w0 - 0.5 * g.flat(), rtol=0, atol=1e-12)


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("d,H", [(1536, 12), (3584, 28)])
def test_wide_rows_vs_oracle(P, ctx32, ctx16, orc, d, H, prec):
    """C4 / C3 model widths (d = 1536 / 3584, Dh = 128) at L = 1 on a ragged packed group:
    the wide-row LayerNorm forward / backward kernels and the Dh = 128 attention against
    the C oracle (fp64) on the same inputs, at tolerances scaled to the measured rounding
    floor of these widths (below)."""
    from oracle import Cfg

    ctx = ctx32 if prec == "fp32" else ctx16
    cfg = P.ModelConfig(256, d, 1, H, 512, 128)
    oc = Cfg(256, d, 1, H, 512, 128)
    pm = P.ModelParams.init(cfg, 5, ctx)
    rng = np.random.default_rng(9)
    prompt = rng.integers(4, 256, 20)
    lens = [30, 17, 25]
    pk = P.pack_group(prompt, [rng.integers(4, 256, n) for n in lens], cfg.max_seq_len, ctx)
    f = P.forward_logprobs(pm, pk.tokens, pk.positions, pk.mask, pk.labels, want_cache=True)
    up = rng.uniform(-1, 1, len(f.logprobs))
    lp_ref, g_ref = orc.forward(oc, pm.flat(), pk.tokens, pk.positions, pk.labels, len(prompt), lens, up)
    d_lp = np.abs(f.logprobs - lp_ref)
    g = P.backward(pm, f, up).flat()
    rel = per_tensor_rel(ocfg(cfg), g, g_ref)
    worst = max((v, k) for k, v in rel.items() if not k.endswith("attn.bk"))
    if prec == "fp32":
        # fp32 rounding grows with the contraction widths: bounds scaled by d / 448 (2x at
        # C2 width); the previous kernel generation measures the same 1e-4 at d = 3584
        sc = d / 448
        assert d_lp.max() < sc * FP32_TOL["lp_abs"], d_lp.max()
        assert worst[0] < sc * FP32_TOL["grad_rel"], worst
    else:
        # bf16 rounding floor at these widths (0.08-scale init: logits grow with sqrt(d)): the
        # previous kernel generation (commit eca3549, other attention and LayerNorm kernels)
        # measures the same 0.182 / 0.0325 / cos 0.99952 (d = 1536) and 0.340 / 0.072 /
        # 0.99830 (d = 3584) on this case; the bounds sit ~25% above that floor
        lp_max, lp_mean, cos = {1536: (0.23, 0.041, 0.9993), 3584: (0.43, 0.09, 0.9978)}[d]
        assert d_lp.max() < lp_max and d_lp.mean() < lp_mean, (d_lp.max(), d_lp.mean())
        assert g @ g_ref / (np.linalg.norm(g) * np.linalg.norm(g_ref)) > cos
        assert worst[0] < 2 * BF16_TOL["grad_rel"], worst
