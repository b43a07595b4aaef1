"""Generate tests/golden/*.npz from the reference itself (oracle/_ref/libparl_ref.so).

Run here (where /root/reference exists):  python -m oracle.make_golden
The fixtures are committed; the GPU box only reads them.

Cases
-----
tiny_*   : the reference tests' small config (V=16, d=16, L=2, H=2, F=24; test_packing.cpp:14-23)
c1_*     : BASELINE configs[0] (d=256, H=4, L=2, F=1024, V=4096; P=64, G=4, R=128; T=576)
c2w_*    : C2's layer width (d=896, H=14, F=4864) at L=1, V=4096; P=64, G=3, R=[96, 80, 131]

Weights come from ModelParams::init (model.cpp:142-164) and, for old/ref, from
`perturb(w, seed, scale)` below, which is reproducible with numpy alone so the GPU
tests can rebuild identical inputs without the reference.
"""
from __future__ import annotations

import os

import numpy as np

from oracle import Cfg, Oracle, layout

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

TINY = Cfg(vocab=16, d_model=16, n_layers=2, n_heads=2, d_ff=24, max_seq=64)
C1 = Cfg(vocab=4096, d_model=256, n_layers=2, n_heads=4, d_ff=1024, max_seq=576)
# C2 width (Qwen2.5-0.5B: d=896, H=14, F=4864) at L=1, a 4096-token vocab and a small
# ragged group whose response boundaries are not tile aligned
C2W = Cfg(vocab=4096, d_model=896, n_layers=1, n_heads=14, d_ff=4864, max_seq=512)


def perturb(w: np.ndarray, seed: int, scale: float) -> np.ndarray:
    """Old/ref weights: w + scale * N(0,1) from numpy's PCG64(seed)."""
    return w + scale * np.random.default_rng(seed).standard_normal(len(w))


def group_inputs(seed: int, vocab: int, P: int, lens):
    rng = np.random.default_rng(seed)
    prompt = rng.integers(4, vocab, P).astype(np.int32)
    responses = [rng.integers(4, vocab, n).astype(np.int32) for n in lens]
    rewards = rng.random(len(lens))
    return prompt, responses, rewards


def grad_summary(cfg: Cfg, g: np.ndarray, n_samples: int = 4096, seed: int = 5):
    names, sums, l2 = [], [], []
    for name, off, r, c in layout(cfg):
        names.append(name)
        sl = g[off: off + r * c]
        sums.append(sl.sum())
        l2.append(np.sqrt((sl * sl).sum()))
    idx = np.sort(np.random.default_rng(seed).choice(len(g), n_samples, replace=False))
    return np.array(names), np.array(sums), np.array(l2), idx, g[idx]


def main(only=None):
    os.makedirs(GOLDEN, exist_ok=True)
    ref = Oracle("ref")
    if only == "c2w":
        return _c2w(ref)
    if only == "ckpt":
        return _ckpt(ref)
    if only == "sample":
        return _sample(ref)

    # ---- tiny: packed forward/backward with an arbitrary upstream -------------
    w = ref.init_params(TINY, 41)
    prompt, responses, rewards = group_inputs(1, TINY.vocab, 5, [3, 4, 1, 2])
    pk = ref.pack(prompt, responses, TINY.max_seq)
    S = int(pk["lens"].sum())
    upstream = np.random.default_rng(2).uniform(-1, 1, S)
    lp, grad = ref.forward(TINY, w, pk["tokens"], pk["positions"], pk["labels"], len(prompt), pk["lens"], upstream)
    np.savez_compressed(os.path.join(GOLDEN, "tiny_packed.npz"), seed=41, prompt=prompt,
                        resp_flat=np.concatenate(responses), lens=pk["lens"], tokens=pk["tokens"],
                        labels=pk["labels"], positions=pk["positions"], span_start=pk["span_start"],
                        upstream=upstream, logprobs=lp, grad=grad)

    # ---- tiny: causal sequence ------------------------------------------------
    toks = np.array([1, 4, 9, 6, 2, 11, 7], dtype=np.int32)
    labs = np.array([-1, 4, 9, 6, 2, 11, 7], dtype=np.int32)
    pos = np.arange(len(toks), dtype=np.int32)
    up_c = np.array([1.0, -0.5, 0.25, 2.0, -1.5, 0.75])
    lp_c, g_c = ref.forward(TINY, w, toks, pos, labs, 0, (), up_c)
    rows = ref.logprob_rows(TINY, w, toks, pos)
    np.savez_compressed(os.path.join(GOLDEN, "tiny_causal.npz"), seed=41, tokens=toks, labels=labs,
                        positions=pos, upstream=up_c, logprobs=lp_c, grad=g_c, rows=rows)

    # ---- tiny: full micro-batch (tri-model + GRPO + backward), both granularities
    w_old = perturb(w, 11, 0.02)
    w_ref = perturb(w, 12, 0.02)
    adv = ref.group_advantages(rewards)
    out = {}
    for gran in (0, 1):
        g, st, lp3 = ref.train_microbatch(TINY, w, w_old, w_ref, prompt, responses, adv, 0.2, 0.04, gran)
        out[f"grad_g{gran}"], out[f"stats_g{gran}"], out[f"lp3_g{gran}"] = g, st, lp3
    np.savez_compressed(os.path.join(GOLDEN, "tiny_micro.npz"), seed=41, old_seed=11, ref_seed=12, scale=0.02,
                        prompt=prompt, resp_flat=np.concatenate(responses), lens=pk["lens"], rewards=rewards,
                        advantages=adv, **out)

    # ---- C1 micro-batch ---------------------------------------------------------
    w1 = ref.init_params(C1, 7)
    prompt, responses, rewards = group_inputs(123, C1.vocab, 64, [128] * 4)
    w1_old = perturb(w1, 21, 0.01)
    w1_ref = perturb(w1, 22, 0.01)
    adv = ref.group_advantages(rewards)
    g, st, lp3 = ref.train_microbatch(C1, w1, w1_old, w1_ref, prompt, responses, adv, 0.2, 0.04, 0)
    names, sums, l2, idx, vals = grad_summary(C1, g)
    np.savez_compressed(os.path.join(GOLDEN, "c1_micro.npz"), seed=7, old_seed=21, ref_seed=22, scale=0.01,
                        prompt=prompt, resp_flat=np.concatenate(responses), lens=np.array([128] * 4, np.int32),
                        rewards=rewards, advantages=adv, stats=st, lp3=lp3, grad_names=names, grad_sums=sums,
                        grad_l2=l2, grad_idx=idx, grad_vals=vals, param_sum=w1.sum(), param_head=w1[:64])
    _c2w(ref)


def _sample(ref):
    """sample_tokens (model.cpp:843-900) of the reference: tiny model (init seed 41) and C1
    width (seed 7), greedy and temperature runs."""
    runs = []
    for name, cfg, wseed in (("tiny", TINY, 41), ("c1", C1, 7)):
        w = ref.init_params(cfg, wseed)
        prompt = np.random.default_rng(5).integers(4, cfg.vocab, 6).astype(np.int32)
        for temp, seed in ((0.0, 0), (0.8, 11), (1.5, 12)):
            toks = ref.sample_tokens(cfg, w, prompt, 24, temp, seed)
            runs.append((name, wseed, temp, seed, prompt, toks))
    np.savez_compressed(os.path.join(GOLDEN, "sample_tokens.npz"),
                        names=np.array([r[0] for r in runs]), wseeds=np.array([r[1] for r in runs]),
                        temps=np.array([r[2] for r in runs]), seeds=np.array([r[3] for r in runs]),
                        prompts=np.stack([r[4] for r in runs]),
                        tokens=np.array([np.pad(r[5], (0, 24 - len(r[5])), constant_values=-1) for r in runs]))
    print("wrote sample_tokens.npz", [len(r[5]) for r in runs])


def _ckpt(ref):
    """PARLCKP1 file written by the reference's own save_checkpoint (model.cpp:924-946) for
    the tiny config, init seed 41 (version 0)."""
    ref.save_checkpoint(TINY, ref.init_params(TINY, 41), 41, os.path.join(GOLDEN, "tiny_seed41.parlckp1"))
    print("wrote tiny_seed41.parlckp1")


def _c2w(ref):
    if True:  # ---- C2-width micro-batch
        lens = [96, 80, 131]
        w2 = ref.init_params(C2W, 7)
        prompt, responses, rewards = group_inputs(321, C2W.vocab, 64, lens)
        w2_old = perturb(w2, 31, 0.01)
        w2_ref = perturb(w2, 32, 0.01)
        adv = ref.group_advantages(rewards)
        g, st, lp3 = ref.train_microbatch(C2W, w2, w2_old, w2_ref, prompt, responses, adv, 0.2, 0.04, 0)
        names, sums, l2, idx, vals = grad_summary(C2W, g)
        np.savez_compressed(os.path.join(GOLDEN, "c2w_micro.npz"), seed=7, old_seed=31, ref_seed=32, scale=0.01,
                            prompt=prompt, resp_flat=np.concatenate(responses), lens=np.array(lens, np.int32),
                            rewards=rewards, advantages=adv, stats=st, lp3=lp3, grad_names=names, grad_sums=sums,
                            grad_l2=l2, grad_idx=idx, grad_vals=vals, param_sum=w2.sum(), param_head=w2[:64])
    print("wrote", sorted(os.listdir(GOLDEN)))


if __name__ == "__main__":
    import sys

    main(sys.argv[1] if len(sys.argv) > 1 else None)
