"""CPU tests: pin the oracle (oracle/parl_oracle.c) before trusting it.

1. the reference's own known-answer tests for the hot path
   (proj/tests/test_packing.cpp, test_grpo.cpp, test_model.cpp), restated;
2. the golden fixtures generated from the reference build (tests/golden/,
   oracle/make_golden.py) — bit-exact;
3. live cross-check against oracle/_ref when it is present.
"""
import math
import os

import numpy as np
import pytest

from oracle import Cfg, OracleError, layout
from tests.conftest import GOLDEN

TINY = Cfg(16, 16, 2, 2, 24, 64)
C1 = Cfg(4096, 256, 2, 4, 1024, 576)


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


# --------------------------------------------------------------------------- packing
def test_pack_golden_lists(orc):  # test_packing.cpp:46-63
    pk = orc.pack([1, 5, 3], [[7, 8], [9, 10]], 64)
    assert pk["tokens"].tolist() == [1, 5, 3, 7, 8, 9, 10]
    assert pk["positions"].tolist() == [0, 1, 2, 3, 4, 3, 4]
    assert pk["span_start"].tolist() == [3, 5]
    assert pk["labels"].tolist() == [-1, -1, -1, 7, 8, 9, 10]
    assert pk["seg"].tolist() == [0, 0, 0, 1, 1, 2, 2]
    assert pk["pred"].tolist() == [-1, 0, 1, 2, 3, 2, 5]


def test_pack_unequal_and_errors(orc):  # test_packing.cpp:64-76
    pk = orc.pack([1, 5, 3], [[7], [8, 9, 10]], 64)
    assert pk["positions"].tolist() == [0, 1, 2, 3, 3, 4, 5]
    assert pk["span_start"].tolist() == [3, 4]
    for args in (([1, 5, 3], [[7, 8], [9, 10]], 6), ([], [[7]], 64), ([1, 5, 3], [], 64),
                 ([1, 5, 3], [[7], []], 64)):
        with pytest.raises(OracleError) as e:
            orc.pack(*args)
        assert e.value.kind == "ShapeError"


def test_mask_enumeration():  # test_packing.cpp:79-107
    import ctypes as C

    from oracle import LIB_C

    lib = C.CDLL(LIB_C)
    lens = (C.c_int * 2)(1, 1)
    m = (C.c_ubyte * 16)()
    assert lib.orc_shared_prompt_mask(2, lens, 2, m) == 4
    assert list(m) == [1, 0, 0, 0, 1, 1, 0, 0, 1, 1, 1, 0, 1, 1, 0, 1]
    single = (C.c_int * 1)(3)
    m1 = (C.c_ubyte * 25)()
    lib.orc_shared_prompt_mask(2, single, 1, m1)
    assert all(m1[i * 5 + j] == (j <= i) for i in range(5) for j in range(5))


# --------------------------------------------------------------------------- GRPO
def test_group_advantages(orc):  # test_grpo.cpp:29-60
    a = orc.group_advantages([1.0, 0.0, 0.0, 1.0])
    assert np.allclose(a, [1, -1, -1, 1], rtol=0, atol=1e-12)
    assert (orc.group_advantages([1.0] * 4) == 0).all()
    with pytest.raises(OracleError):
        orc.group_advantages([0.5])
    rng = np.random.default_rng(99)
    for trial in range(50):
        r = rng.random(2 + trial % 7) * 3 - 1
        adv = orc.group_advantages(r)
        assert abs(adv.sum()) < 1e-12
        assert np.abs(adv - orc.group_advantages(r + 17.25)).max() < 1e-12
    assert np.allclose(orc.group_advantages([1.0, 2.0, 6.0], mean_only=True), [-2, -1, 3])


def test_clip_and_kl_closed_forms(orc):  # test_grpo.cpp:62-99
    assert orc.clipped_term(math.log(1.5), 0.0, 1.0, 0.2) == pytest.approx(1.2, abs=1e-12)
    assert orc.clipped_term(math.log(0.5), 0.0, -1.0, 0.2) == pytest.approx(-0.8, abs=1e-12)
    for adv in (-2.0, 0.0, 0.7):
        assert orc.clipped_term(-1.3, -1.3, adv, 0.2) == pytest.approx(adv, abs=1e-12)
    assert orc.kl_term(-1.7, -1.7) == 0.0
    assert orc.kl_term(-2.0, -2.0 + math.log(2.0)) == pytest.approx(2.0 - math.log(2.0) - 1.0, abs=1e-12)
    rng = np.random.default_rng(11)
    for a, b in rng.uniform(-8, 0, (2000, 2)):
        assert orc.kl_term(a, b) >= 0.0


def test_clipped_branch_upstream(orc):  # test_grpo.cpp:169-202
    eps, beta = 0.2, 0.04
    t = orc.sample_terms([-1.0], [-1.0 - math.log(1.5)], [-0.9], 1.0, eps, beta)
    assert t["upstream"][0] == pytest.approx(beta * math.expm1(0.1), abs=1e-15)
    assert t["clipped_units"] == 1
    t = orc.sample_terms([-1.0], [-1.0 - math.log(1.5)], [-1.0], -1.0, eps, beta)
    assert t["upstream"][0] == pytest.approx(-1.5, abs=1e-12)


def test_identity_weights_loss(orc):  # test_grpo.cpp:101-129
    advs = [1.0, -0.5, 0.25, 2.0]
    obj = 0.0
    for j, a in enumerate(advs):
        v = [-1.0 - j, -0.5, -2.0 + 0.3 * j]
        for gran in (0, 1):
            t = orc.sample_terms(v, v, v, a, 0.2, 0.04, gran)
            assert t["clip_term"] == pytest.approx(a, abs=1e-12)
            assert t["kl"] == 0.0 and t["clipped_units"] == 0
        obj += a
    assert obj / 4 == pytest.approx((1.0 - 0.5 + 0.25 + 2.0) / 4)


def test_upstream_matches_fd(orc):  # test_grpo.cpp:131-167
    rng = np.random.default_rng(31)
    for gran in (0, 1):
        n = 4
        pol = -2.5 * rng.random(n) - 0.1
        old = pol - np.array([0.02, -0.03, 0.015, -0.025])
        ref = pol + np.array([-0.02, 0.01, 0.03, -0.015])
        a = 1.4
        base = orc.sample_terms(pol, old, ref, a, 0.2, 0.04, gran)

        def J(p):
            t = orc.sample_terms(p, old, ref, a, 0.2, 0.04, gran)
            return t["clip_term"] - 0.04 * t["kl"]

        h = 1e-3
        for t in range(n):
            e = np.zeros(n)
            e[t] = 1
            fd = (8 * (J(pol + h * e) - J(pol - h * e)) - (J(pol + 2 * h * e) - J(pol - 2 * h * e))) / (12 * h)
            assert abs(fd - base["upstream"][t]) / max(abs(fd), 1e-3) < 1e-8


# --------------------------------------------------------------------------- model
def test_init_parity_with_reference_fixture(orc):
    z = load("c1_micro.npz")
    w = orc.init_params(C1, 7)
    assert len(w) == 3_828_736
    assert w[:64].tobytes() == z["param_head"].tobytes()
    assert w.sum() == z["param_sum"]


def test_tiny_packed_fixture_bit_exact(orc):
    z = load("tiny_packed.npz")
    w = orc.init_params(TINY, int(z["seed"]))
    pk = orc.pack(z["prompt"], np.split(z["resp_flat"], np.cumsum(z["lens"])[:-1]), TINY.max_seq)
    for k in ("tokens", "labels", "positions", "span_start"):
        assert np.array_equal(pk[k], z[k]), k
    lp, g = orc.forward(TINY, w, pk["tokens"], pk["positions"], pk["labels"], len(z["prompt"]), z["lens"],
                        z["upstream"])
    assert np.array_equal(lp, z["logprobs"])
    assert np.array_equal(g, z["grad"])


def test_tiny_causal_fixture_bit_exact(orc):
    z = load("tiny_causal.npz")
    w = orc.init_params(TINY, int(z["seed"]))
    lp, g = orc.forward(TINY, w, z["tokens"], z["positions"], z["labels"], 0, (), z["upstream"])
    assert np.array_equal(lp, z["logprobs"]) and np.array_equal(g, z["grad"])
    rows = orc.logprob_rows(TINY, w, z["tokens"], z["positions"])
    assert np.array_equal(rows, z["rows"])
    assert np.allclose(np.exp(rows).sum(1), 1.0, atol=1e-12)  # test_model.cpp:72-93


def test_tiny_micro_fixture_bit_exact(orc):
    from oracle.make_golden import perturb

    z = load("tiny_micro.npz")
    w = orc.init_params(TINY, int(z["seed"]))
    wo, wr = perturb(w, int(z["old_seed"]), float(z["scale"])), perturb(w, int(z["ref_seed"]), float(z["scale"]))
    resp = np.split(z["resp_flat"], np.cumsum(z["lens"])[:-1])
    assert np.array_equal(orc.group_advantages(z["rewards"]), z["advantages"])
    for gran in (0, 1):
        g, st, lp3 = orc.train_microbatch(TINY, w, wo, wr, z["prompt"], resp, z["advantages"], 0.2, 0.04, gran)
        assert np.array_equal(g, z[f"grad_g{gran}"])
        assert np.array_equal(st, z[f"stats_g{gran}"])
        assert np.array_equal(lp3, z[f"lp3_g{gran}"])


def test_packed_equals_unpacked(orc):  # test_packing.cpp:123-151, 164-200
    w = orc.init_params(TINY, 41)
    rng = np.random.default_rng(17)
    for _ in range(10):
        prompt = rng.integers(0, 16, rng.integers(1, 6))
        resp = [rng.integers(0, 16, rng.integers(1, 6)) for _ in range(rng.integers(1, 5))]
        pk = orc.pack(prompt, resp, 64)
        up = rng.uniform(-1, 1, int(pk["lens"].sum()))
        lp, g = orc.forward(TINY, w, pk["tokens"], pk["positions"], pk["labels"], len(prompt), pk["lens"], up)
        gsum = np.zeros_like(g)
        off = 0
        for r in resp:
            toks = np.concatenate([prompt, r])
            labs = np.concatenate([np.full(len(prompt), -1), r])
            l1, _ = orc.forward(TINY, w, toks, np.arange(len(toks)), labs, 0, (), up[off:off + len(r)], gsum)
            assert np.abs(l1 - lp[off:off + len(r)]).max() < 1e-10
            off += len(r)
        denom = np.maximum(np.maximum(np.abs(g), np.abs(gsum)), 1e-6)
        assert (np.abs(g - gsum) / denom).max() < 1e-9


def test_forward_validation_order(orc):  # test_model.cpp:107-123
    w = orc.init_params(TINY, 1)
    with pytest.raises(OracleError) as e:
        orc.forward(TINY, w, [1, 99, 3], [0, 1, 2], [-1, 2, 2])
    assert e.value.kind == "VocabError"
    with pytest.raises(OracleError) as e:
        orc.forward(TINY, w, [1, 2, 3], [0, 1, 2], [3, -1, -1])
    assert e.value.kind == "ShapeError"


def test_attn_bk_grad_is_zero(orc):
    z = load("tiny_packed.npz")
    for name, off, r, c in layout(TINY):
        if name.endswith("attn.bk"):
            assert np.abs(z["grad"][off:off + r * c]).max() < 1e-12


# --------------------------------------------------------------------------- live reference
def test_oracle_matches_reference_live(orc, ref_orc):
    rng = np.random.default_rng(5)
    cfg = Cfg(32, 16, 2, 4, 40, 96)
    w = ref_orc.init_params(cfg, 9)
    assert np.array_equal(w, orc.init_params(cfg, 9))
    prompt = rng.integers(4, 32, 7)
    resp = [rng.integers(4, 32, n) for n in (5, 9, 2)]
    adv = orc.group_advantages(rng.random(3))
    wo, wr = w + 0.01 * rng.standard_normal(len(w)), w - 0.01 * rng.standard_normal(len(w))
    for gran in (0, 1):
        a = orc.train_microbatch(cfg, w, wo, wr, prompt, resp, adv, 0.2, 0.04, gran)
        b = ref_orc.train_microbatch(cfg, w, wo, wr, prompt, resp, adv, 0.2, 0.04, gran)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


# --------------------------------------------------------------------------- PARLCKP1 (model.cpp:907-987)
TINY_CKPT = Cfg(vocab=16, d_model=16, n_layers=2, n_heads=2, d_ff=24, max_seq=64)


def test_parlckp1_golden_layout_and_values(orc):
    """The reference-written golden checkpoint: header, tensor names / shapes in
    build_layout order (model.cpp:86-114), and the init(seed 41) weights bit-exact."""
    from oracle import read_parlckp1

    cfg, version, seed, names, flat = read_parlckp1(os.path.join(GOLDEN, "tiny_seed41.parlckp1"))
    assert cfg == TINY_CKPT and version == 0 and seed == 41
    assert [(n, r, c) for n, _, r, c in layout(cfg)] == names
    assert np.array_equal(flat, orc.init_params(cfg, 41))


def test_parlckp1_reference_round_trip(ref_orc, tmp_path):
    from oracle import read_parlckp1

    w = ref_orc.init_params(TINY_CKPT, 5) * 1.5
    path = str(tmp_path / "w.parlckp1")
    ref_orc.save_checkpoint(TINY_CKPT, w, 5, path)
    cfg, version, seed, w2 = ref_orc.load_checkpoint(path)
    assert cfg == TINY_CKPT and version == 0 and seed == 5 and np.array_equal(w, w2)
    assert np.array_equal(read_parlckp1(path)[4], w)


def test_torch_ref_pinned(orc):
    """oracle/torch_ref.py (exact mode) == the C restatement on a shared-prompt micro-step:
    log-probs of the three roles, the gradient and the loss stats, to fp64 rounding."""
    from oracle import Cfg
    from oracle import torch_ref as TR

    for cfg, P, lens in ((Cfg(16, 16, 2, 2, 24, 64), 5, [3, 4, 1, 2]), (Cfg(64, 32, 1, 4, 48, 64), 9, [7, 1, 12])):
        w = orc.init_params(cfg, 41)
        rng = np.random.default_rng(0)
        wo, wr = w + 0.01 * rng.standard_normal(len(w)), w - 0.01 * rng.standard_normal(len(w))
        prompt = rng.integers(4, cfg.vocab, P)
        resp = [rng.integers(4, cfg.vocab, n) for n in lens]
        adv = orc.group_advantages(rng.random(len(lens)))
        g, st, lp3 = orc.train_microbatch(cfg, w, wo, wr, prompt, resp, adv)
        lp3_t, g_t, st_t = TR.microstep(cfg, w, wo, wr, prompt, resp, adv)
        assert np.abs(lp3 - lp3_t).max() < 1e-13
        assert np.abs(g - g_t).max() <= 1e-12 * np.abs(g).max()
        assert np.abs(st - st_t).max() < 1e-13


def test_torch_ref_pinned_c2_width_fixture():
    """The restatement at C2's layer width against the reference-generated fixture
    (tests/golden/c2w_micro.npz: log-probs, per-tensor gradient sums / norms, 4096 sampled entries)."""
    from oracle import Cfg, Oracle
    from oracle import torch_ref as TR
    from oracle.make_golden import C2W, perturb

    z = np.load(os.path.join(GOLDEN, "c2w_micro.npz"))
    w = Oracle("c").init_params(C2W, int(z["seed"]))
    wo, wr = perturb(w, int(z["old_seed"]), float(z["scale"])), perturb(w, int(z["ref_seed"]), float(z["scale"]))
    resp = np.split(z["resp_flat"], np.cumsum(z["lens"])[:-1])
    lp3, g, st = TR.microstep(C2W, w, wo, wr, z["prompt"], resp, z["advantages"])
    assert np.abs(lp3 - z["lp3"]).max() < 1e-11
    assert np.abs(st - z["stats"]).max() < 1e-11
    assert np.allclose(g[z["grad_idx"]], z["grad_vals"], rtol=1e-9, atol=1e-14)
