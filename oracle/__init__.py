"""ORACLE — test infrastructure only.

numpy/ctypes front-end over two CPU checkers of the hot path
(`Pipeline::train_microbatch`, /root/reference/proj/src/pipeline.cpp:97-141):

* ``Oracle("c")``   -> oracle/liboracle.so, the plain-C fp64 restatement
  (oracle/parl_oracle.c);
* ``Oracle("ref")`` -> oracle/_ref/libparl_ref.so, the reference's own sources
  compiled by oracle/Makefile behind oracle/ref_shim.cpp.

Both expose the same methods, so tests can pin one against the other.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import this
package; the product path (paper_2511_18871_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_C = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libparl_ref.so")
REF_SRC = "/root/reference/proj"


def build(ref: bool = True) -> None:
    """Compile the C restatement, and the reference shim when the reference is mounted."""
    subprocess.check_call(["make", "-s", "-C", HERE, "liboracle.so"])
    if ref and os.path.isdir(REF_SRC):
        subprocess.check_call(["make", "-s", "-j8", "-C", HERE, "ref"])


@dataclass(frozen=True)
class Cfg:
    """ModelConfig, proj/include/parl/model.hpp:26-36."""

    vocab: int = 64
    d_model: int = 32
    n_layers: int = 2
    n_heads: int = 2
    d_ff: int = 64
    max_seq: int = 256

    def c(self):
        return (C.c_int * 6)(self.vocab, self.d_model, self.n_layers, self.n_heads, self.d_ff, self.max_seq)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        names = {1: "ConfigError", 2: "ShapeError", 3: "VocabError", 4: "LifecycleError", 5: "NumericError"}
        self.code = code
        self.kind = names.get(code, "Error")
        super().__init__(f"{self.kind} in {what}")


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class Oracle:
    def __init__(self, kind: str = "c"):
        self.kind = kind
        path = LIB_C if kind == "c" else LIB_REF
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.px = "orc_" if kind == "c" else "ref_"
        for name in ("clipped_term", "kl_term"):
            f = getattr(self.lib, self.px + name)
            f.restype = C.c_double
            f.argtypes = [C.c_double] * (4 if name == "clipped_term" else 2)
        if kind == "ref":
            self.lib.ref_save_checkpoint.argtypes = [C.c_void_p, C.c_void_p, C.c_ulonglong, C.c_char_p]
            self.lib.ref_load_checkpoint.restype = C.c_long
            self.lib.ref_load_checkpoint.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            self.lib.ref_bench_microbatch.restype = C.c_double
            self.lib.ref_bench_microbatch.argtypes = [C.c_void_p, C.c_ulonglong] + [C.c_int] * 5
            self.lib.ref_param_count.restype = C.c_long
            self.lib.ref_bench_open.restype = C.c_void_p
            self.lib.ref_bench_open.argtypes = [C.c_void_p, C.c_ulonglong, C.c_int]
            self.lib.ref_bench_run.restype = C.c_double
            self.lib.ref_bench_run.argtypes = [C.c_void_p] + [C.c_int] * 4
            self.lib.ref_bench_close.argtypes = [C.c_void_p]
        else:
            self.lib.orc_param_count.restype = C.c_size_t
        self.lib[self.px + "init_params"].argtypes = [C.c_void_p, C.c_ulonglong, C.c_void_p]

    def _f(self, name):
        return getattr(self.lib, self.px + name)

    @staticmethod
    def _chk(rc, what):
        if rc < 0:
            raise OracleError(-rc, what)
        return rc

    def save_checkpoint(self, cfg: Cfg, w, seed: int, path: str):
        """The reference's save_checkpoint (model.cpp:924-946) of weights w (version 0)."""
        assert self.kind == "ref"
        c = cfg.c()
        self._chk(self.lib.ref_save_checkpoint(C.byref(c), _p(_f64(w)), C.c_ulonglong(seed), os.fsencode(path)),
                  "save_checkpoint")

    def sample_tokens(self, cfg: Cfg, w, prompt, max_new: int, temperature: float, seed: int):
        """The reference's sample_tokens (model.cpp:843-900)."""
        assert self.kind == "ref"
        c = cfg.c()
        out = np.zeros(max(max_new, 1), dtype=np.int32)
        pr = _i32(prompt)
        self.lib.ref_sample_tokens.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_double,
                                               C.c_ulonglong, C.c_void_p]
        n = self._chk(self.lib.ref_sample_tokens(C.byref(c), _p(_f64(w)), _p(pr), len(pr), max_new, temperature,
                                                 C.c_ulonglong(seed), _p(out)), "sample_tokens")
        return out[:n]

    def load_checkpoint(self, path: str):
        """The reference's load_checkpoint (model.cpp:948-987): (Cfg, version, seed, flat)."""
        assert self.kind == "ref"
        c, ver, seed = (C.c_int * 6)(), C.c_ulonglong(), C.c_ulonglong()
        n = self._chk(self.lib.ref_load_checkpoint(os.fsencode(path), C.byref(c), None, C.byref(ver),
                                                   C.byref(seed)), "load_checkpoint")
        w = np.zeros(n, dtype=np.float64)
        self.lib.ref_load_checkpoint(os.fsencode(path), C.byref(c), _p(w), C.byref(ver), C.byref(seed))
        return Cfg(*list(c)), ver.value, seed.value, w

    def param_count(self, cfg: Cfg) -> int:
        c = cfg.c()
        return int(self._f("param_count")(C.byref(c)))

    def init_params(self, cfg: Cfg, seed: int) -> np.ndarray:
        w = np.zeros(self.param_count(cfg), dtype=np.float64)
        c = cfg.c()
        self._chk(self._f("init_params")(C.byref(c), C.c_ulonglong(seed), _p(w)), "init_params")
        return w

    def pack(self, prompt, responses, max_seq):
        prompt = _i32(prompt)
        lens = _i32([len(r) for r in responses])
        flat = _i32(np.concatenate([np.asarray(r, dtype=np.int32) for r in responses]) if len(responses) else [])
        T = len(prompt) + int(lens.sum())
        out = {k: np.zeros(max(T, 1), dtype=np.int32) for k in ("tokens", "labels", "positions", "seg", "pred")}
        spans = np.zeros(max(len(responses), 1), dtype=np.int32)
        if self.kind == "c":
            rc = self.lib.orc_pack(_p(prompt), len(prompt), _p(flat), _p(lens), len(responses), max_seq,
                                   _p(out["tokens"]), _p(out["labels"]), _p(out["positions"]), _p(spans),
                                   _p(out["seg"]), _p(out["pred"]))
        else:
            rc = self.lib.ref_pack(_p(prompt), len(prompt), _p(flat), _p(lens), len(responses), max_seq,
                                   _p(out["tokens"]), _p(out["labels"]), _p(out["positions"]), _p(spans))
        self._chk(rc, "pack")
        res = {k: v[:rc] for k, v in out.items()}
        res["span_start"] = spans[: len(responses)]
        res["lens"] = lens
        if self.kind != "c":
            res.pop("seg")
            res.pop("pred")
        return res

    def forward(self, cfg: Cfg, w, tokens, positions, labels, prompt_len=0, resp_lens=(), upstream=None,
                grad_acc=None):
        """forward_logprobs (+ backward into grad_acc when upstream is given)."""
        tokens, positions, labels = _i32(tokens), _i32(positions), _i32(labels)
        lens = _i32(resp_lens if len(resp_lens) else [0])
        T = len(tokens)
        lp = np.zeros(max(T, 1), dtype=np.float64)
        c = cfg.c()
        w = _f64(w)
        up = _f64(upstream) if upstream is not None else None
        if up is not None and grad_acc is None:
            grad_acc = np.zeros(len(w), dtype=np.float64)
        if self.kind == "c":
            rc = self.lib.orc_forward(C.byref(c), _p(w), _p(tokens), _p(positions), T, prompt_len, _p(lens),
                                      len(resp_lens), _p(labels), _p(lp), None, _p(up), _p(grad_acc), None)
        else:
            rc = self.lib.ref_forward(C.byref(c), _p(w), _p(tokens), _p(positions), T, prompt_len, _p(lens),
                                      len(resp_lens), _p(labels), _p(lp), _p(up), _p(grad_acc))
        self._chk(rc, "forward")
        return (lp[:rc], grad_acc) if up is not None else lp[:rc]

    def logprob_rows(self, cfg: Cfg, w, tokens, positions, prompt_len=0, resp_lens=()):
        tokens, positions = _i32(tokens), _i32(positions)
        lens = _i32(resp_lens if len(resp_lens) else [0])
        T = len(tokens)
        rows = np.zeros(T * cfg.vocab, dtype=np.float64)
        c = cfg.c()
        w = _f64(w)
        if self.kind == "c":
            rc = self.lib.orc_forward(C.byref(c), _p(w), _p(tokens), _p(positions), T, prompt_len, _p(lens),
                                      len(resp_lens), None, None, None, None, None, _p(rows))
        else:
            rc = self.lib.ref_logprob_rows(C.byref(c), _p(w), _p(tokens), _p(positions), T, prompt_len,
                                           _p(lens), len(resp_lens), _p(rows))
        self._chk(rc, "logprob_rows")
        return rows.reshape(T, cfg.vocab)

    def group_advantages(self, rewards, mean_only=False):
        r = _f64(rewards)
        a = np.zeros(len(r), dtype=np.float64)
        self._chk(self._f("group_advantages")(_p(r), len(r), int(mean_only), _p(a)), "group_advantages")
        return a

    def clipped_term(self, lp, old, adv, eps):
        return self._f("clipped_term")(lp, old, adv, eps)

    def kl_term(self, lp, ref):
        return self._f("kl_term")(lp, ref)

    def sample_terms(self, lp, old, ref, adv, eps, beta, granularity=0):
        lp, old, ref = _f64(lp), _f64(old), _f64(ref)
        up = np.zeros(len(lp), dtype=np.float64)
        out4 = np.zeros(4, dtype=np.float64)
        self._chk(self._f("sample_terms")(_p(lp), _p(old), _p(ref), len(lp), C.c_double(adv), C.c_double(eps),
                                          C.c_double(beta), granularity, _p(up), _p(out4)), "sample_terms")
        return {"clip_term": out4[0], "kl": out4[1], "clipped_units": int(out4[2]), "total_units": int(out4[3]),
                "upstream": up}

    def train_microbatch(self, cfg: Cfg, w_pol, w_old, w_ref, prompt, responses, advantages, eps=0.2,
                         beta=0.04, granularity=0, grad_acc=None):
        """Pipeline::train_microbatch shared-prompt branch.  Returns (grad, stats5, lp3[3,S])."""
        prompt = _i32(prompt)
        lens = _i32([len(r) for r in responses])
        flat = _i32(np.concatenate([np.asarray(r, dtype=np.int32) for r in responses]))
        adv = _f64(advantages)
        S = int(lens.sum())
        if grad_acc is None:
            grad_acc = np.zeros(len(w_pol), dtype=np.float64)
        stats = np.zeros(5, dtype=np.float64)
        lp3 = np.zeros(3 * S, dtype=np.float64)
        c = cfg.c()
        w_pol, w_old, w_ref = _f64(w_pol), _f64(w_old), _f64(w_ref)
        rc = self._f("train_microbatch")(C.byref(c), _p(w_pol), _p(w_old), _p(w_ref), _p(prompt), len(prompt),
                                         _p(flat), _p(lens), len(responses), _p(adv), *(
                                             [None] if self.kind == "c" else []),
                                         C.c_double(eps), C.c_double(beta), granularity, _p(grad_acc), _p(stats),
                                         _p(lp3))
        self._chk(rc, "train_microbatch")
        return grad_acc, stats, lp3.reshape(3, S)

    def train_iteration(self, cfg: Cfg, w_pol, w_old, w_ref, microbatches, lr, eps=0.2, beta=0.04,
                        granularity=0, rollout_old=None, total_samples=None):
        """pipeline.cpp:263-352 (training half): micro-batches [(prompt, responses, advantages)],
        accumulate, divisor N*G, snapshot, apply_update.  Returns (new_policy, new_old, stats5).
        The C restatement composes orc_train_microbatch with ModelParams::apply_update's
        arithmetic (model.cpp:202-219); the reference runs its own TriModel / GradBuffer."""
        total = total_samples if total_samples is not None else sum(len(mb[2]) for mb in microbatches)
        w_pol, w_old, w_ref = _f64(w_pol).copy(), _f64(w_old).copy(), _f64(w_ref)
        stats = np.zeros(5, dtype=np.float64)
        if self.kind == "ref":
            pflat = _i32(np.concatenate([np.asarray(mb[0], np.int32) for mb in microbatches]))
            plens = _i32([len(mb[0]) for mb in microbatches])
            rlist = [r for mb in microbatches for r in mb[1]]
            rflat = _i32(np.concatenate([np.asarray(r, np.int32) for r in rlist]))
            lens = _i32([len(r) for r in rlist])
            off = _i32(np.concatenate([[0], np.cumsum([len(mb[1]) for mb in microbatches])]))
            adv = _f64(np.concatenate([np.asarray(mb[2], np.float64) for mb in microbatches]))
            ro = _f64(rollout_old) if rollout_old is not None else None
            c = cfg.c()
            rc = self.lib.ref_train_iteration(C.byref(c), _p(w_pol), _p(w_old), _p(w_ref), len(microbatches),
                                              _p(pflat), _p(plens), _p(rflat), _p(lens), _p(off), _p(adv), _p(ro),
                                              C.c_double(eps), C.c_double(beta), granularity, C.c_double(lr),
                                              int(total), _p(stats))
            self._chk(rc, "train_iteration")
            return w_pol, w_old, stats
        if rollout_old is not None:
            raise NotImplementedError("rollout_weights iteration: use the reference build")
        g = np.zeros(len(w_pol), dtype=np.float64)
        for prompt, responses, adv in microbatches:
            _, st, _ = self.train_microbatch(cfg, w_pol, w_old, w_ref, prompt, responses, adv, eps, beta,
                                             granularity, grad_acc=g)
            stats += st
        new_old = w_pol.copy()  # snapshot_old_policy before the update (pipeline.cpp:350-351)
        w_new = w_pol - (lr / float(total)) * g
        return w_new, new_old, stats

    def bench_open(self, cfg: Cfg, seed: int, threads: int):
        """Persistent CPU-baseline workers (one TriModel each, built once, outside any timing)."""
        assert self.kind == "ref"
        c = cfg.c()
        return self.lib.ref_bench_open(C.byref(c), C.c_ulonglong(seed), threads)

    def bench_run(self, h, P, G, R, reps) -> float:
        """Max wall seconds over the workers for `reps` shared-prompt micro-batches each."""
        return float(self.lib.ref_bench_run(h, P, G, R, reps))

    def bench_close(self, h):
        self.lib.ref_bench_close(h)

    def bench_microbatch(self, cfg: Cfg, seed, P, G, R, reps, threads) -> float:
        assert self.kind == "ref"
        c = cfg.c()
        return float(self.lib.ref_bench_microbatch(C.byref(c), C.c_ulonglong(seed), P, G, R, reps, threads))


def read_parlckp1(path: str):
    """PARLCKP1 reader (save_checkpoint, model.cpp:924-946; docs/formats.md): header, then
    per tensor u32 name length, name, u32 rows, u32 cols, rows * cols f64.  Returns
    (Cfg, version, init_seed, [(name, rows, cols)], flat fp64)."""
    import struct

    with open(path, "rb") as f:
        b = f.read()
    if b[:8] != b"PARLCKP1":
        raise ValueError("bad checkpoint magic")
    V, d, L, H, F, S = struct.unpack_from("<6I", b, 8)
    version, seed = struct.unpack_from("<2Q", b, 32)
    (n,) = struct.unpack_from("<I", b, 48)
    o, names, parts = 52, [], []
    for _ in range(n):
        (nl,) = struct.unpack_from("<I", b, o)
        name = b[o + 4:o + 4 + nl].decode()
        o += 4 + nl
        r, c = struct.unpack_from("<2I", b, o)
        o += 8
        parts.append(np.frombuffer(b, dtype="<f8", count=r * c, offset=o))
        o += 8 * r * c
        names.append((name, r, c))
    if o != len(b):
        raise ValueError("trailing bytes in checkpoint")
    return Cfg(V, d, L, H, F, S), version, seed, names, np.concatenate(parts)


def layout(cfg: Cfg):
    """Named (offset, rows, cols) slices of the flat parameter array, model.cpp:86-114."""
    d, F, V = cfg.d_model, cfg.d_ff, cfg.vocab
    out = []
    o = 0

    def add(name, r, c):
        nonlocal o
        out.append((name, o, r, c))
        o += r * c

    add("tok_emb", V, d)
    add("pos_emb", cfg.max_seq, d)
    for l in range(cfg.n_layers):
        p = f"layers.{l}."
        for n, r, c in (("ln1.gamma", 1, d), ("ln1.beta", 1, d), ("attn.wq", d, d), ("attn.bq", 1, d),
                        ("attn.wk", d, d), ("attn.bk", 1, d), ("attn.wv", d, d), ("attn.bv", 1, d),
                        ("attn.wo", d, d), ("attn.bo", 1, d), ("ln2.gamma", 1, d), ("ln2.beta", 1, d),
                        ("ffn.w1", d, F), ("ffn.b1", 1, F), ("ffn.w2", F, d), ("ffn.b2", 1, d)):
            add(p + n, r, c)
    add("ln_f.gamma", 1, d)
    add("ln_f.beta", 1, d)
    add("head.w", d, V)
    add("head.b", 1, V)
    return out
