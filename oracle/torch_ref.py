"""ORACLE — test infrastructure only.  A torch restatement of the reference's
forward / backward / GRPO micro-step, used

  * in fp64 ("exact") as a checker at the headline widths (C2-C4 layer widths and
    the real 152K vocabularies), where the C restatement (parl_oracle.c) needs
    minutes per case on the host; it runs on whatever torch device it is given;
  * with bf16-rounded MMA inputs and fp64 accumulation ("bf16") to measure the
    rounding floor of a bf16 tensor-core path at those widths, from which the
    tolerances of tests/test_gpu_widths.py are set (SURVEY.md §8c method).

It is pinned to the C restatement (and through it to the reference, which the C
restatement matches bit for bit) by tests/test_oracle.py::test_torch_ref_pinned.

Reference math (proj/src/model.cpp):
  embeddings 449-455; layer_norm 317-343 (population variance, eps 1e-5, 132);
  linear 301-314 (W stored [in x out]); attention 468-501 (scale 1/sqrt(Dh), 441;
  shared-prompt rule 242-245); GELU 255; head + predecessor rows 518-556;
  backward 587-838 (here by autograd); GRPO grpo.cpp:24-151, pipeline.cpp:127-139.

bf16 emulation follows the device path: every contraction rounds both operands to
bf16 (activations, weights, attention P and dS, the backward's incoming gradients)
and accumulates in fp64; biases, LayerNorm, softmax statistics and the residual
stream stay unrounded; the policy's softmax backward reads bf16-rounded logits
(the device keeps them in bf16) against the unrounded log-sum-exp.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from oracle import layout


def _r(x, on):
    return x.to(torch.bfloat16).to(x.dtype) if on else x


class _Linear(torch.autograd.Function):
    """y = R(a) R(W) + b; dA = R(g) R(W)^T, dW = R(a)^T R(g), db = 1^T R(g)."""

    @staticmethod
    def forward(ctx, a, w, b, rnd):
        ar, wr = _r(a, rnd), _r(w, rnd)
        ctx.save_for_backward(ar, wr)
        ctx.rnd = rnd
        return ar @ wr + b

    @staticmethod
    def backward(ctx, g):
        ar, wr = ctx.saved_tensors
        gr = _r(g, ctx.rnd)
        return gr @ wr.T, ar.T @ gr, gr.sum(0), None


class _Attention(torch.autograd.Function):
    """One head, dense allowed mask; flash-style rounding of P / dS / dO (k_attn_tc.cu)."""

    @staticmethod
    def forward(ctx, q, k, v, allowed, scale, rnd):
        qr, kr, vr = _r(q, rnd), _r(k, rnd), _r(v, rnd)
        s = (qr @ kr.T) * scale
        s = s.masked_fill(~allowed, -math.inf)
        m = s.max(1, keepdim=True).values
        p_un = torch.exp(s - m)
        l = p_un.sum(1, keepdim=True)
        o = (_r(p_un, rnd) @ vr) / l
        lse = (m + torch.log(l)).squeeze(1)
        ctx.save_for_backward(qr, kr, vr, _r(o, rnd), lse, allowed)
        ctx.scale, ctx.rnd = scale, rnd
        return o

    @staticmethod
    def backward(ctx, do):
        qr, kr, vr, orr, lse, allowed = ctx.saved_tensors
        rnd, scale = ctx.rnd, ctx.scale
        dor = _r(do, rnd)
        s = ((qr @ kr.T) * scale).masked_fill(~allowed, -math.inf)
        p = torch.exp(s - lse[:, None])
        dp = dor @ vr.T
        D = (dor * orr).sum(1, keepdim=True)
        ds = p * (dp - D)
        dsr = _r(ds, rnd)
        dq = (dsr @ kr) * scale
        dk = (dsr.T @ qr) * scale
        dv = _r(p, rnd).T @ dor
        return dq, dk, dv, None, None, None


class _HeadLogprob(torch.autograd.Function):
    """lp = z[label] - lse(z), z = R(h) R(W) + b over the predecessor rows; the backward's
    softmax reads R(z) (bf16-kept logits) against the unrounded lse, dZ rounded for dH / dW."""

    @staticmethod
    def forward(ctx, h, w, b, labels, rnd):
        hr, wr = _r(h, rnd), _r(w, rnd)
        z = hr @ wr + b
        lse = torch.logsumexp(z, 1)
        lp = z.gather(1, labels[:, None]).squeeze(1) - lse
        ctx.save_for_backward(hr, wr, _r(z, rnd), lse, labels)
        ctx.rnd = rnd
        return lp

    @staticmethod
    def backward(ctx, u):
        hr, wr, zr, lse, labels = ctx.saved_tensors
        dz = -u[:, None] * torch.exp(zr - lse[:, None])
        dz.scatter_add_(1, labels[:, None], u[:, None])
        dzr = _r(dz, ctx.rnd)
        return dzr @ wr.T, hr.T @ dzr, dzr.sum(0), None, None


def _ln(x, g, b):
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) / torch.sqrt(var + 1e-5) * g + b


def params_from_flat(cfg, w, device="cpu", requires_grad=False):
    flat = torch.as_tensor(np.ascontiguousarray(w), dtype=torch.float64, device=device)
    out = {}
    for name, off, r, c in layout(cfg):
        t = flat[off:off + r * c].view(r, c) if r > 1 else flat[off:off + r * c]
        out[name] = t.clone().requires_grad_(requires_grad)
    return out


def grads_to_flat(cfg, params):
    n = sum(r * c for _, _, r, c in layout(cfg))
    g = np.zeros(n, np.float64)
    for name, off, r, c in layout(cfg):
        t = params[name].grad
        if t is not None:
            g[off:off + r * c] = t.detach().reshape(-1).cpu().numpy()
    return g


def packed_meta(P, lens):
    """seg / pred / allowed of the shared-prompt packing (model.cpp:230-253)."""
    T = P + int(sum(lens))
    seg = np.zeros(T, np.int64)
    t = P
    for k, n in enumerate(lens):
        seg[t:t + n] = k + 1
        t += n
    pred = np.arange(T) - 1
    starts = P + np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    pred[starts] = P - 1
    i, j = np.arange(T)[:, None], np.arange(T)[None, :]
    allowed = np.where(seg[:, None] == 0, (seg[None, :] == 0) & (j <= i),
                       (seg[None, :] == 0) | ((seg[None, :] == seg[:, None]) & (j <= i)))
    return seg, pred, allowed


def forward_logprobs(cfg, params, tokens, positions, labels, P, lens, rnd=False):
    """Log-probs of the scored tokens in position order (model.cpp:534-567)."""
    dev = params["tok_emb"].device
    tok = torch.as_tensor(np.asarray(tokens, np.int64), device=dev)
    pos = torch.as_tensor(np.asarray(positions, np.int64), device=dev)
    lab = np.asarray(labels, np.int64)
    _, pred, allowed = packed_meta(P, lens)
    allowed_t = torch.as_tensor(allowed, device=dev)
    d, H = cfg.d_model, cfg.n_heads
    Dh = d // H
    scale = 1.0 / math.sqrt(Dh)
    x = params["tok_emb"][tok] + params["pos_emb"][pos]
    for l in range(cfg.n_layers):
        p = lambda n: params[f"layers.{l}.{n}"]
        a = _ln(x, p("ln1.gamma"), p("ln1.beta"))
        q = _Linear.apply(a, p("attn.wq"), p("attn.bq"), rnd)
        k = _Linear.apply(a, p("attn.wk"), p("attn.bk"), rnd)
        v = _Linear.apply(a, p("attn.wv"), p("attn.bv"), rnd)
        heads = [_Attention.apply(q[:, h * Dh:(h + 1) * Dh], k[:, h * Dh:(h + 1) * Dh], v[:, h * Dh:(h + 1) * Dh],
                                  allowed_t, scale, rnd) for h in range(H)]
        ctx = torch.cat(heads, 1)
        xm = x + _Linear.apply(ctx, p("attn.wo"), p("attn.bo"), rnd)
        u = _Linear.apply(_ln(xm, p("ln2.gamma"), p("ln2.beta")), p("ffn.w1"), p("ffn.b1"), rnd)
        act = 0.5 * u * torch.erfc(-u / math.sqrt(2.0))
        x = xm + _Linear.apply(act, p("ffn.w2"), p("ffn.b2"), rnd)
    scored = np.nonzero(lab != -1)[0]
    rows = torch.as_tensor(pred[scored], device=dev)
    hf = _ln(x[rows], params["ln_f.gamma"], params["ln_f.beta"])
    return _HeadLogprob.apply(hf, params["head.w"], params["head.b"],
                              torch.as_tensor(lab[scored], device=dev), rnd)


def group_advantages(rewards, mean_only=False):
    r = np.asarray(rewards, np.float64)
    mean = r.mean()
    sd = math.sqrt(((r - mean) ** 2).mean())
    if mean_only:
        return r - mean
    return np.zeros_like(r) if sd < 1e-8 else (r - mean) / sd


def grpo_terms(lp, old, ref, lens, adv, eps=0.2, beta=0.04):
    """Token granularity (grpo.cpp:119-131): upstream = -g per token and the 5 stats."""
    lp, old, ref = (np.asarray(x, np.float64) for x in (lp, old, ref))
    up = np.zeros_like(lp)
    st = np.zeros(5)
    c = 0
    for j, n in enumerate(lens):
        s = slice(c, c + n)
        r = np.exp(lp[s] - old[s])
        cl = np.clip(r, 1 - eps, 1 + eps)
        un, cv = r * adv[j], cl * adv[j]
        val = np.where(un <= cv, un, cv)
        grad = np.where(un <= cv, r * adv[j], np.where((r > 1 - eps) & (r < 1 + eps), r * adv[j], 0.0))
        d = ref[s] - lp[s]
        em = np.expm1(d)
        up[s] = -(grad + beta * em) / n
        L, KL = val.mean(), (em - d).mean()
        st += [L - beta * KL, L, KL, ((r < 1 - eps) | (r > 1 + eps)).sum(), n]
        c += n
    return up, st


def microstep(cfg, w_pol, w_old, w_ref, prompt, responses, advantages, rnd=False, device="cpu", upstream=None):
    """Pipeline::train_microbatch shared-prompt branch: (lp3 [3, S], grad flat, stats5).
    `upstream` given: the backward is seeded with it instead of the emulated loss's own
    (isolates the backward's rounding from the log-probs' rounding)."""
    P = len(prompt)
    lens = [len(r) for r in responses]
    tokens = np.concatenate([prompt] + list(responses))
    positions = np.concatenate([np.arange(P)] + [P + np.arange(n) for n in lens])
    labels = np.concatenate([np.full(P, -1)] + list(responses))
    lp3 = []
    with torch.no_grad():
        for w in (w_old, w_ref):
            prm = params_from_flat(cfg, w, device)
            lp3.append(forward_logprobs(cfg, prm, tokens, positions, labels, P, lens, rnd).cpu().numpy())
    prm = params_from_flat(cfg, w_pol, device, requires_grad=True)
    lp = forward_logprobs(cfg, prm, tokens, positions, labels, P, lens, rnd)
    lp_np = lp.detach().cpu().numpy()
    up, st = grpo_terms(lp_np, lp3[0], lp3[1], lens, np.asarray(advantages))
    if upstream is not None:
        up = np.asarray(upstream, np.float64)
    lp.backward(torch.as_tensor(up, device=lp.device))
    return np.stack([lp_np, lp3[0], lp3[1]]), grads_to_flat(cfg, prm), st
