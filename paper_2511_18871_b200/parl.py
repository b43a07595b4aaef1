"""Python front-end over the C-ABI (include/parl_gpu.h) of libparl_gpu.so.

Mirrors the reference operator interface of the hot path — same names,
argument meaning and exception types:

    pack_group                 proj/src/packing.cpp:7-45
    extract_response_logprobs  proj/src/packing.cpp:74-89
    forward_logprobs           proj/src/model.cpp:534-567
    forward_logprob_rows       proj/src/model.cpp:569-585
    backward                   proj/src/model.cpp:587-838
    GradBuffer.accumulate      proj/src/model.cpp:189-194
    ModelParams.apply_update   proj/src/model.cpp:202-219
    trimodel_forward           proj/src/pipeline.cpp:22-30
    train_microbatch           proj/src/pipeline.cpp:97-141 (shared-prompt branch)

There is no CPU fallback: importing this module loads the CUDA library and
raises if it is missing; every call runs on the device.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PARL_LIB", os.path.join(_HERE, "libparl_gpu.so"))  # PARL_LIB: A/B runs of another build

kIgnoreLabel = -1


# --------------------------------------------------------------------------- errors (errors.hpp:9-46)
class ParlError(RuntimeError):
    pass


class ConfigError(ParlError):
    pass


class ShapeError(ParlError):
    pass


class VocabError(ParlError):
    pass


class LifecycleError(ParlError):
    pass


class NumericError(ParlError):
    pass


class BarrierError(ParlError):
    pass


class StallError(ParlError):
    pass


class IoError(ParlError):
    pass


class CudaError(ParlError):
    pass


class NcclError(ParlError):
    pass


_ERRORS = {1: ConfigError, 2: ShapeError, 3: VocabError, 4: LifecycleError, 5: NumericError, 6: BarrierError,
           7: StallError, 8: IoError, 9: CudaError, 10: NcclError}

PREC_FP32, PREC_BF16 = 0, 1


class _Config(C.Structure):
    _fields_ = [("vocab_size", C.c_int), ("d_model", C.c_int), ("n_layers", C.c_int), ("n_heads", C.c_int),
                ("d_ff", C.c_int), ("max_seq_len", C.c_int)]


class _Hyper(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("beta", C.c_double), ("granularity", C.c_int),
                ("advantage_mean_only", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("objective_sum", C.c_double), ("clip_sum", C.c_double), ("kl_sum", C.c_double),
                ("clipped_units", C.c_double), ("total_units", C.c_double)]


class _SampleTerms(C.Structure):
    _fields_ = [("clip_term", C.c_double), ("kl", C.c_double), ("clipped_units", C.c_int),
                ("total_units", C.c_int)]


class _LossReport(C.Structure):
    _fields_ = [("objective", C.c_double), ("clip_term_mean", C.c_double), ("kl_mean", C.c_double),
                ("clip_fraction", C.c_double), ("token_count", C.c_long)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    vp, i32p, f64p = C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_double)
    sig = {
        "parl_ctx_create": [C.c_int, C.c_int, C.POINTER(vp)],
        "parl_ctx_destroy": [vp], "parl_ctx_sync": [vp],
        "parl_model_create": [vp, C.POINTER(_Config), C.POINTER(vp)], "parl_model_destroy": [vp],
        "parl_model_upload": [vp, f64p, C.c_size_t, C.c_uint64], "parl_model_init": [vp, C.c_uint64],
        "parl_model_init_device": [vp, C.c_uint64, C.c_double],
        "parl_model_copy": [vp, vp, C.c_uint64, C.c_double], "parl_model_download": [vp, f64p, C.c_size_t],
        "parl_group_create": [vp, C.c_int, C.c_int, C.POINTER(vp)], "parl_group_destroy": [vp],
        "parl_pack": [vp, i32p, C.c_int, i32p, i32p, C.c_int, C.c_int],
        "parl_pack_device": [vp, vp, C.c_int, vp, i32p, C.c_int, C.c_int],
        "parl_pack_multi": [vp, i32p, i32p, i32p, i32p, i32p, C.c_int, C.c_int],
        "parl_pack_multi_device": [vp, vp, i32p, vp, i32p, i32p, C.c_int, C.c_int],
        "parl_set_sequence": [vp, i32p, i32p, i32p, C.c_int, C.c_int, i32p, C.c_int, C.c_int, C.c_int],
        "parl_group_download": [vp, i32p, i32p, i32p, i32p, i32p, i32p, i32p],
        "parl_forward": [vp, vp, vp, C.c_int, C.POINTER(vp)],
        "parl_trimodel_forward": [vp, vp, vp, vp, vp, C.POINTER(vp)],
        "parl_group_logprobs": [vp, C.c_int, f64p], "parl_group_set_logprobs": [vp, C.c_int, f64p],
        "parl_logprob_rows": [vp, vp, vp, f64p], "parl_act_destroy": [vp],
        "parl_grpo_loss": [vp, vp, f64p, f64p, C.POINTER(_Hyper), C.POINTER(_Stats)],
        "parl_group_upstream": [vp, f64p], "parl_group_set_upstream": [vp, f64p],
        "parl_stats_download": [vp, C.POINTER(_Stats)], "parl_stats_reset": [vp],
        "parl_grad_create": [vp, vp, C.POINTER(vp)], "parl_grad_destroy": [vp], "parl_grad_reset": [vp],
        "parl_backward": [vp, vp, vp, vp, vp], "parl_grad_download": [vp, f64p, C.c_size_t],
        "parl_grad_accumulate": [vp, vp],
        "parl_train_microbatch": [vp, vp, vp, vp, vp, f64p, f64p, C.POINTER(_Hyper), vp, C.POINTER(_Stats)],
        "parl_apply_update": [vp, vp, C.c_double],
        "parl_comm_unique_id": [C.c_char_p], "parl_comm_init": [vp, C.c_char_p, C.c_int, C.c_int],
        "parl_grad_allreduce": [vp, vp], "parl_stats_allreduce": [vp], "parl_grad_allreduce_overlap": [vp, vp],
        "parl_checkpoint_save": [vp, C.c_char_p], "parl_checkpoint_load": [vp, C.c_char_p, C.POINTER(vp)],
        "parl_model_config": [vp, C.POINTER(_Config)],
        "parl_sample_tokens": [vp, vp, vp, C.c_int, C.c_int, C.c_double, C.c_uint64, vp, C.POINTER(C.c_int)],
        "parl_sample_group": [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_double, vp, vp, vp, vp],
        "parl_ctx_profile": [vp, C.c_int], "parl_ctx_set_recompute": [vp, C.c_int], "parl_act_recompute": [vp],
        "parl_ctx_profile_read": [vp, C.c_int, f64p, f64p, C.POINTER(C.c_long)],
        "parl_grad_set_micro_steps": [vp, C.c_int], "parl_grad_add_micro_steps": [vp, C.c_int],
        "parl_grad_all_finite": [vp, C.POINTER(C.c_int)], "parl_grad_upload": [vp, f64p, C.c_size_t],
        "parl_model_all_finite": [vp, C.POINTER(C.c_int)], "parl_model_set_init_seed": [vp, C.c_uint64],
        "parl_group_advantages": [vp, f64p, C.c_int, C.c_int, f64p],
        "parl_clipped_term": [vp, C.c_double, C.c_double, C.c_double, C.c_double, f64p],
        "parl_kl_term": [vp, C.c_double, C.c_double, f64p],
        "parl_per_sample_terms": [vp, f64p, f64p, f64p, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                  f64p, C.POINTER(_SampleTerms)],
        "parl_grpo_microbatch_loss": [vp, C.c_int, i32p, f64p, f64p, f64p, f64p, C.c_double, C.c_double, C.c_int,
                                      f64p, C.POINTER(_LossReport), f64p],
        "parl_shared_prompt_mask": [vp, C.c_int, i32p, C.c_int, C.POINTER(C.c_uint8)],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    lib.parl_last_error.argtypes = [vp]
    lib.parl_last_error.restype = C.c_char_p
    lib.parl_param_count.argtypes = [C.POINTER(_Config)]
    lib.parl_param_count.restype = C.c_size_t
    lib.parl_group_tokens.argtypes = [vp]
    lib.parl_group_scored.argtypes = [vp]
    lib.parl_grad_micro_steps.argtypes = [vp]
    lib.parl_model_version.argtypes = [vp]
    lib.parl_model_version.restype = C.c_uint64
    lib.parl_model_init_seed.argtypes = [vp]
    lib.parl_model_init_seed.restype = C.c_uint64
    lib.parl_ctx_stream.argtypes = [vp]
    lib.parl_ctx_stream.restype = C.c_void_p
    lib.parl_ctx_launches.argtypes = [vp]
    lib.parl_ctx_launches.restype = C.c_uint64
    lib.parl_version.restype = C.c_char_p
    return lib


LIB = _load()


def _check(rc: int, ctx=None):
    if rc != 0:
        msg = LIB.parl_last_error(ctx).decode(errors="replace")
        raise _ERRORS.get(rc, ParlError)(msg)


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _pi(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32)) if a is not None else None


def _pd(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


# --------------------------------------------------------------------------- context
class Context:
    """Device + stream + workspaces (+ optional NCCL communicator)."""

    def __init__(self, device: int = 0, precision: int = PREC_FP32):
        h = C.c_void_p()
        _check(LIB.parl_ctx_create(device, precision, C.byref(h)))
        self.h = h
        self.device = device
        self.precision = precision

    def sync(self):
        _check(LIB.parl_ctx_sync(self.h), self.h)

    @property
    def stream(self) -> int:
        return LIB.parl_ctx_stream(self.h)

    @property
    def launches(self) -> int:
        return LIB.parl_ctx_launches(self.h)

    KC = {"gemm": 0, "head": 1, "attn_fwd": 2, "attn_bwd": 3, "loss": 4, "pack": 5, "norm": 6, "seed": 7}

    def set_recompute(self, mode: int):
        """Activation recomputation: 0 auto, 1 always, 2 never (parl_ctx_set_recompute)."""
        _check(LIB.parl_ctx_set_recompute(self.h, int(mode)), self.h)

    def profile(self, enable: bool):
        _check(LIB.parl_ctx_profile(self.h, int(enable)), self.h)

    def profile_read(self, cls: str) -> dict:
        ms, work, n = C.c_double(), C.c_double(), C.c_long()
        _check(LIB.parl_ctx_profile_read(self.h, self.KC[cls], C.byref(ms), C.byref(work), C.byref(n)), self.h)
        return {"ms": ms.value, "work": work.value, "launches": n.value}

    def comm_init(self, uid: bytes, rank: int, nranks: int):
        _check(LIB.parl_comm_init(self.h, uid, rank, nranks), self.h)

    @staticmethod
    def comm_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(LIB.parl_comm_unique_id(buf))
        return buf.raw

    def stats(self) -> dict:
        s = _Stats()
        _check(LIB.parl_stats_download(self.h, C.byref(s)), self.h)
        return {k: getattr(s, k) for k, _ in _Stats._fields_}

    def stats_reset(self):
        _check(LIB.parl_stats_reset(self.h), self.h)

    def stats_allreduce(self):
        _check(LIB.parl_stats_allreduce(self.h), self.h)

    def __del__(self):
        try:
            LIB.parl_ctx_destroy(self.h)
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context(precision: int = PREC_FP32) -> Context:
    global _default_ctx
    if _default_ctx is None or _default_ctx.precision != precision:
        _default_ctx = Context(0, precision)
    return _default_ctx


# --------------------------------------------------------------------------- model
@dataclass(frozen=True)
class ModelConfig:
    """proj/include/parl/model.hpp:26-36."""

    vocab_size: int = 64
    d_model: int = 32
    n_layers: int = 2
    n_heads: int = 2
    d_ff: int = 64
    max_seq_len: int = 256

    def c(self):
        return _Config(self.vocab_size, self.d_model, self.n_layers, self.n_heads, self.d_ff, self.max_seq_len)

    def param_count(self) -> int:
        c = self.c()
        return int(LIB.parl_param_count(C.byref(c)))


class ModelParams:
    """Device-resident weight set (replaces ModelParams, model.hpp:64-106)."""

    def __init__(self, config: ModelConfig, ctx: Optional[Context] = None, _handle=None):
        self.ctx = ctx or default_context()
        self.config = config
        if _handle is not None:
            self.h = _handle
            return
        h = C.c_void_p()
        c = config.c()
        _check(LIB.parl_model_create(self.ctx.h, C.byref(c), C.byref(h)), self.ctx.h)
        self.h = h

    @classmethod
    def init(cls, config: ModelConfig, seed: int, ctx: Optional[Context] = None) -> "ModelParams":
        p = cls(config, ctx)
        _check(LIB.parl_model_init(p.h, seed), p.ctx.h)
        return p

    @classmethod
    def init_device(cls, config: ModelConfig, seed: int, ctx: Optional[Context] = None,
                    scale: float = 0.08) -> "ModelParams":
        p = cls(config, ctx)
        _check(LIB.parl_model_init_device(p.h, seed, scale), p.ctx.h)
        return p

    @classmethod
    def from_flat(cls, config: ModelConfig, flat, version: int = 0, ctx: Optional[Context] = None):
        p = cls(config, ctx)
        p.upload(flat, version)
        return p

    def upload(self, flat, version: int = 0):
        w = _f64(flat)
        _check(LIB.parl_model_upload(self.h, _pd(w), len(w), version), self.ctx.h)

    def flat(self) -> np.ndarray:
        out = np.zeros(self.config.param_count(), dtype=np.float64)
        _check(LIB.parl_model_download(self.h, _pd(out), len(out)), self.ctx.h)
        return out

    def clone(self, seed: int = 0, noise: float = 0.0) -> "ModelParams":
        p = ModelParams(self.config, self.ctx)
        _check(LIB.parl_model_copy(p.h, self.h, seed, noise), self.ctx.h)
        return p

    def copy_from(self, other: "ModelParams"):
        _check(LIB.parl_model_copy(self.h, other.h, 0, 0.0), self.ctx.h)

    def version(self) -> int:
        return int(LIB.parl_model_version(self.h))

    def init_seed(self) -> int:
        return int(LIB.parl_model_init_seed(self.h))

    def set_init_seed(self, seed: int):
        _check(LIB.parl_model_set_init_seed(self.h, int(seed)), self.ctx.h)

    def all_finite(self) -> bool:
        """ModelParams::all_finite (model.cpp:183-187)."""
        v = C.c_int()
        _check(LIB.parl_model_all_finite(self.h, C.byref(v)), self.ctx.h)
        return bool(v.value)

    def apply_update(self, grads: "GradBuffer", lr: float):
        _check(LIB.parl_apply_update(self.h, grads.h, lr), self.ctx.h)

    def save(self, path: str):
        """save_checkpoint (model.cpp:924-946): PARLCKP1 file of the fp64 weights."""
        _check(LIB.parl_checkpoint_save(self.h, os.fsencode(path)), self.ctx.h)

    @classmethod
    def load(cls, path: str, ctx: Optional[Context] = None) -> "ModelParams":
        """load_checkpoint (model.cpp:948-987)."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(LIB.parl_checkpoint_load(ctx.h, os.fsencode(path), C.byref(h)), ctx.h)
        c = _Config()
        _check(LIB.parl_model_config(h, C.byref(c)), ctx.h)
        cfg = ModelConfig(c.vocab_size, c.d_model, c.n_layers, c.n_heads, c.d_ff, c.max_seq_len)
        return cls(cfg, ctx, _handle=h)

    def __del__(self):
        try:
            LIB.parl_model_destroy(self.h)
        except Exception:
            pass


class GradBuffer:
    """fp32 device accumulator in the reference flat layout (GradBuffer, model.hpp:109-134)."""

    def __init__(self, like: ModelParams):
        self.ctx = like.ctx
        self.config = like.config
        h = C.c_void_p()
        _check(LIB.parl_grad_create(self.ctx.h, like.h, C.byref(h)), self.ctx.h)
        self.h = h

    def flat(self) -> np.ndarray:
        out = np.zeros(self.config.param_count(), dtype=np.float64)
        _check(LIB.parl_grad_download(self.h, _pd(out), len(out)), self.ctx.h)
        return out

    def reset(self):
        _check(LIB.parl_grad_reset(self.h), self.ctx.h)

    def micro_step_count(self) -> int:
        return int(LIB.parl_grad_micro_steps(self.h))

    def set_micro_step_count(self, n: int):
        """GradBuffer::set_micro_step_count (model.hpp:126): the update divisor."""
        _check(LIB.parl_grad_set_micro_steps(self.h, int(n)), self.ctx.h)

    def add_micro_steps(self, n: int):
        _check(LIB.parl_grad_add_micro_steps(self.h, int(n)), self.ctx.h)

    def all_finite(self) -> bool:
        v = C.c_int()
        _check(LIB.parl_grad_all_finite(self.h, C.byref(v)), self.ctx.h)
        return bool(v.value)

    def upload(self, flat):
        """Host fp64 values into the device accumulator (a GradBuffer::flat_mut() write)."""
        g = _f64(flat)
        _check(LIB.parl_grad_upload(self.h, _pd(g), len(g)), self.ctx.h)

    def allreduce(self):
        _check(LIB.parl_grad_allreduce(self.ctx.h, self.h), self.ctx.h)

    def allreduce_overlap(self):
        """Arm before the step's last micro-batch: its backward streams each finished gradient
        slice to NCCL (parl_grad_allreduce_overlap); allreduce() then completes the exchange."""
        _check(LIB.parl_grad_allreduce_overlap(self.ctx.h, self.h), self.ctx.h)

    def accumulate(self, other: "GradBuffer"):
        """GradBuffer::accumulate (model.cpp:189-194)."""
        _check(LIB.parl_grad_accumulate(self.h, other.h), self.ctx.h)

    def __del__(self):
        try:
            LIB.parl_grad_destroy(self.h)
        except Exception:
            pass


# --------------------------------------------------------------------------- packing
@dataclass
class AttentionMaskSpec:
    """proj/include/parl/model.hpp:41-55."""

    kind: str = "causal"
    prompt_len: int = 0
    response_lens: tuple = ()

    @staticmethod
    def causal():
        return AttentionMaskSpec()

    @staticmethod
    def shared_prompt(prompt_len: int, response_lens):
        return AttentionMaskSpec("shared_prompt", int(prompt_len), tuple(int(x) for x in response_lens))


class Group:
    """A device-resident packed sequence (PackedGroup + K1 outputs)."""

    def __init__(self, max_tokens: int, max_responses: int = 1, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        _check(LIB.parl_group_create(self.ctx.h, max_tokens, max(1, max_responses), C.byref(h)), self.ctx.h)
        self.h = h
        self.max_tokens = max_tokens
        self.max_responses = max(1, max_responses)
        self.prompt_len = 0
        self.response_lens: tuple = ()

    @property
    def T(self) -> int:
        return LIB.parl_group_tokens(self.h)

    @property
    def S(self) -> int:
        return LIB.parl_group_scored(self.h)

    def pack(self, prompt, responses, max_seq_len: int):
        p = _i32(prompt)
        lens = _i32([len(r) for r in responses])
        flat = _i32(np.concatenate([np.asarray(r, dtype=np.int32) for r in responses]) if len(responses) else [])
        _check(LIB.parl_pack(self.h, _pi(p), len(p), _pi(flat), _pi(lens), len(lens), max_seq_len), self.ctx.h)
        self.prompt_len, self.response_lens = len(p), tuple(int(x) for x in lens)
        return self

    def pack_device(self, d_prompt: int, P: int, d_resp: int, lens, max_seq_len: int):
        lens = _i32(lens)
        _check(LIB.parl_pack_device(self.h, C.c_void_p(d_prompt), P, C.c_void_p(d_resp), _pi(lens), len(lens),
                                    max_seq_len), self.ctx.h)
        self.prompt_len, self.response_lens = P, tuple(int(x) for x in lens)
        return self

    def pack_multi(self, prompts, groups, max_seq_len: int):
        """Several prompt groups in one packed sequence (parl_pack_multi): prompts[q] with its
        responses groups[q]; each group laid out as pack_group, no attention across groups."""
        pl = _i32([len(p) for p in prompts])
        gs = _i32([len(r) for r in groups])
        rl = _i32([len(x) for r in groups for x in r])
        pf = _i32(np.concatenate([np.asarray(p, np.int32) for p in prompts]))
        rf = _i32(np.concatenate([np.asarray(x, np.int32) for r in groups for x in r]))
        _check(LIB.parl_pack_multi(self.h, _pi(pf), _pi(pl), _pi(rf), _pi(rl), _pi(gs), len(pl), max_seq_len),
               self.ctx.h)
        self.prompt_len, self.response_lens = int(pl[0]), tuple(int(x) for x in rl)
        return self

    def pack_multi_device(self, d_prompts: int, prompt_lens, d_resp: int, resp_lens, group_sizes, max_seq_len: int):
        pl, rl, gs = _i32(prompt_lens), _i32(resp_lens), _i32(group_sizes)
        _check(LIB.parl_pack_multi_device(self.h, C.c_void_p(d_prompts), _pi(pl), C.c_void_p(d_resp), _pi(rl),
                                          _pi(gs), len(pl), max_seq_len), self.ctx.h)
        self.prompt_len, self.response_lens = int(pl[0]), tuple(int(x) for x in rl)
        return self

    def set_sequence(self, tokens, positions, labels, mask: AttentionMaskSpec, vocab_size: int, max_seq_len: int):
        t, p = _i32(tokens), _i32(positions)
        lab = _i32(labels) if labels is not None else None
        if len(t) != len(p) or (lab is not None and len(lab) != len(t)):
            raise ShapeError("tokens/positions/labels lengths differ")
        lens = _i32(mask.response_lens if mask.kind == "shared_prompt" else [0])
        P = mask.prompt_len if mask.kind == "shared_prompt" else 0
        if mask.kind == "shared_prompt" and P < 1:
            raise ShapeError("shared_prompt mask needs prompt_len >= 1")
        _check(LIB.parl_set_sequence(self.h, _pi(t), _pi(p), _pi(lab), len(t), P, _pi(lens),
                                     len(mask.response_lens) if P else 0, vocab_size, max_seq_len), self.ctx.h)
        self.prompt_len, self.response_lens = P, tuple(mask.response_lens) if P else ()
        return self

    def download(self) -> dict:
        T, S = self.T, self.S
        out = {k: np.zeros(max(T, 1), np.int32) for k in ("tokens", "labels", "positions", "seg", "pred")}
        span = np.zeros(max(len(self.response_lens), 1), np.int32)
        sp = np.zeros(max(S, 1), np.int32)
        _check(LIB.parl_group_download(self.h, _pi(out["tokens"]), _pi(out["labels"]), _pi(out["positions"]),
                                       _pi(out["seg"]), _pi(out["pred"]), _pi(span), _pi(sp)), self.ctx.h)
        res = {k: v[:T] for k, v in out.items()}
        res["span_start"] = span[: len(self.response_lens)]
        res["scored_pos"] = sp[:S]
        return res

    def logprobs(self, slot: int = 0) -> np.ndarray:
        out = np.zeros(max(self.S, 1), np.float64)
        _check(LIB.parl_group_logprobs(self.h, slot, _pd(out)), self.ctx.h)
        return out[: self.S]

    def set_logprobs(self, slot: int, values):
        v = _f64(values)
        if len(v) != self.S:
            raise ShapeError("logprob vector does not match the scored count")
        _check(LIB.parl_group_set_logprobs(self.h, slot, _pd(v)), self.ctx.h)

    def upstream(self) -> np.ndarray:
        out = np.zeros(max(self.S, 1), np.float64)
        _check(LIB.parl_group_upstream(self.h, _pd(out)), self.ctx.h)
        return out[: self.S]

    def set_upstream(self, values):
        v = _f64(values)
        if len(v) != self.S:
            raise ShapeError(f"upstream gradient count {len(v)} != scored position count {self.S}")
        _check(LIB.parl_group_set_upstream(self.h, _pd(v)), self.ctx.h)

    def __del__(self):
        try:
            LIB.parl_group_destroy(self.h)
        except Exception:
            pass


@dataclass
class PackedGroup:
    """packing.hpp:13-23 (host view) + the device group it was packed into."""

    tokens: np.ndarray
    labels: np.ndarray
    positions: np.ndarray
    mask: AttentionMaskSpec
    spans: list
    group: Group = field(repr=False, default=None)


def pack_group(prompt, responses, max_seq_len: int, ctx: Optional[Context] = None,
               group: Optional[Group] = None) -> PackedGroup:
    """pack_group (packing.cpp:7-45), executed by the device packer K1."""
    T = len(prompt) + sum(len(r) for r in responses)
    if group is None:
        group = Group(max(T, 1), max(len(responses), 1), ctx)
    group.pack(prompt, responses, max_seq_len)
    d = group.download()
    spans = [(int(s), int(n)) for s, n in zip(d["span_start"], group.response_lens)]
    return PackedGroup(d["tokens"], d["labels"], d["positions"],
                       AttentionMaskSpec.shared_prompt(len(prompt), group.response_lens), spans, group)


def sample_tokens(params: "ModelParams", prompt, max_new_tokens: int, temperature: float = 0.0,
                  rng_seed: int = 0) -> np.ndarray:
    """sample_tokens (model.cpp:843-900) on the device forward; token choice on the host with the
    reference's fp64 arithmetic and RNG stream."""
    pr = np.ascontiguousarray(np.asarray(prompt, dtype=np.int32))
    out = np.zeros(max(int(max_new_tokens), 1), dtype=np.int32)
    n = C.c_int(0)
    _check(LIB.parl_sample_tokens(params.ctx.h, params.h, pr.ctypes.data_as(C.c_void_p), len(pr), int(max_new_tokens),
                                  float(temperature), int(rng_seed), out.ctypes.data_as(C.c_void_p), C.byref(n)),
           params.ctx.h)
    return out[:n.value]


def sample_group(params: "ModelParams", prompt, n_seq: int, max_new_tokens: int, temperature: float, seeds,
                 want_logprobs: bool = False):
    """The G rollouts of one prompt on the KV-cached decoder (parl_sample_group): sequence k is
    sample_tokens(prompt, max_new_tokens, temperature, seeds[k]); with want_logprobs also each
    sampled token's log-prob (the rollout-side old_logprobs).  Returns a list of token arrays
    (and of log-prob arrays)."""
    pr = np.ascontiguousarray(np.asarray(prompt, dtype=np.int32))
    sd = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
    if len(sd) != n_seq:
        raise ShapeError("one seed per sequence")
    mx = max(int(max_new_tokens), 1)
    out = np.zeros(n_seq * mx, np.int32)
    n = np.zeros(n_seq, np.int32)
    lp = np.zeros(n_seq * mx, np.float64) if want_logprobs else None
    _check(LIB.parl_sample_group(params.ctx.h, params.h, pr.ctypes.data_as(C.c_void_p), len(pr), int(n_seq),
                                 int(max_new_tokens), float(temperature), sd.ctypes.data_as(C.c_void_p),
                                 out.ctypes.data_as(C.c_void_p), n.ctypes.data_as(C.c_void_p),
                                 lp.ctypes.data_as(C.c_void_p) if lp is not None else None), params.ctx.h)
    toks = [out[k * mx:k * mx + n[k]] for k in range(n_seq)]
    if not want_logprobs:
        return toks
    return toks, [lp[k * mx:k * mx + n[k]] for k in range(n_seq)]


def extract_response_logprobs(logprobs, packed: PackedGroup):
    """packing.cpp:74-89."""
    expected = sum(n for _, n in packed.spans)
    if len(logprobs) != expected:
        raise ShapeError(f"logprob vector of length {len(logprobs)} does not match {expected} response tokens")
    out, c = [], 0
    for _, n in packed.spans:
        out.append(np.asarray(logprobs[c:c + n]))
        c += n
    return out


# --------------------------------------------------------------------------- forward / backward
class Activations:
    """ForwardResult::cache — device activations of one cached policy forward."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            LIB.parl_act_destroy(self.h)
        except Exception:
            pass


@dataclass
class ForwardResult:
    logprobs: np.ndarray
    scored_positions: np.ndarray
    cache: Optional[Activations] = None
    group: Optional[Group] = None


def _group_for(params: ModelParams, tokens, positions, mask, labels) -> Group:
    n = len(tokens)
    g = Group(max(n, 1), max(len(mask.response_lens), 1), params.ctx)
    g.set_sequence(tokens, positions, labels, mask, params.config.vocab_size, params.config.max_seq_len)
    return g


def forward_logprobs(params: ModelParams, tokens, positions, mask: AttentionMaskSpec, labels,
                     want_cache: bool = False, slot: int = 0) -> ForwardResult:
    """model.cpp:534-567 on the device."""
    if labels is None:
        raise ShapeError("forward_logprobs requires labels")
    g = _group_for(params, tokens, positions, mask, labels)
    act = C.c_void_p()
    _check(LIB.parl_forward(params.ctx.h, params.h, g.h, slot, C.byref(act) if want_cache else None), params.ctx.h)
    d = g.download()
    return ForwardResult(g.logprobs(slot), d["scored_pos"], Activations(act) if want_cache else None, g)


def score_logprobs(params: ModelParams, prompt, response) -> np.ndarray:
    """RolloutService::score_logprobs (rollout.cpp:52-66): log-probs of the response tokens
    under a causal forward over prompt || response (the rollout-side old log-probs)."""
    if len(response) == 0:
        return np.zeros(0)
    toks = np.concatenate([np.asarray(prompt, np.int32), np.asarray(response, np.int32)])
    labels = np.full(len(toks), -1, np.int32)
    labels[len(prompt):] = np.asarray(response, np.int32)
    return forward_logprobs(params, toks, np.arange(len(toks), dtype=np.int32), AttentionMaskSpec.causal(),
                            labels).logprobs


def forward_logprob_rows(params: ModelParams, tokens, positions, mask: AttentionMaskSpec) -> np.ndarray:
    """model.cpp:569-585: [T x V] log-softmax rows."""
    g = _group_for(params, tokens, positions, mask, None)
    T, V = len(tokens), params.config.vocab_size
    rows = np.zeros(T * V, np.float64)
    _check(LIB.parl_logprob_rows(params.ctx.h, params.h, g.h, _pd(rows)), params.ctx.h)
    return rows.reshape(T, V)


def backward(params: ModelParams, fwd: ForwardResult, upstream, grads: Optional[GradBuffer] = None) -> GradBuffer:
    """model.cpp:587-838: gradient of sum_i upstream[i] * logprobs[i]; accumulates into `grads`."""
    if fwd.cache is None:
        raise LifecycleError("backward requires a cached forward result")
    up = _f64(upstream)
    if len(up) != len(fwd.logprobs):
        raise ShapeError(f"upstream gradient count {len(up)} != scored position count {len(fwd.logprobs)}")
    fwd.group.set_upstream(up)
    gb = grads if grads is not None else GradBuffer(params)
    _check(LIB.parl_backward(params.ctx.h, params.h, fwd.cache.h, fwd.group.h, gb.h), params.ctx.h)
    return gb


@dataclass
class TriModel:
    """pipeline.hpp:41-48."""

    policy: ModelParams
    old_policy: ModelParams
    reference: ModelParams

    @staticmethod
    def init(config: ModelConfig, seed: int, ctx: Optional[Context] = None) -> "TriModel":
        pol = ModelParams.init(config, seed, ctx)
        return TriModel(pol, pol.clone(), pol.clone())

    def snapshot_old_policy(self):
        self.old_policy.copy_from(self.policy)


@dataclass
class TriForwardResult:
    policy: ForwardResult
    old_logprobs: np.ndarray
    ref_logprobs: np.ndarray


def trimodel_forward(tm: TriModel, tokens, positions, mask: AttentionMaskSpec, labels) -> TriForwardResult:
    """pipeline.cpp:22-30."""
    ctx = tm.policy.ctx
    g = _group_for(tm.policy, tokens, positions, mask, labels)
    act = C.c_void_p()
    _check(LIB.parl_trimodel_forward(ctx.h, tm.policy.h, tm.old_policy.h, tm.reference.h, g.h, C.byref(act)), ctx.h)
    d = g.download()
    return TriForwardResult(ForwardResult(g.logprobs(0), d["scored_pos"], Activations(act), g), g.logprobs(1),
                            g.logprobs(2))


@dataclass
class HyperParams:
    """pipeline.hpp:29-37 (loss subset)."""

    epsilon: float = 0.2
    beta: float = 0.04
    granularity: str = "token"
    advantage_mean_only: bool = False

    def c(self):
        return _Hyper(self.epsilon, self.beta, 0 if self.granularity == "token" else 1, int(self.advantage_mean_only))


def grpo_loss(ctx: Context, group: Group, hyper: HyperParams, rewards=None, advantages=None) -> dict:
    """group_advantages + per_sample_terms over the group's responses; stats accumulate on the device."""
    h = hyper.c()
    s = _Stats()
    r = _f64(rewards) if rewards is not None else None
    a = _f64(advantages) if advantages is not None else None
    _check(LIB.parl_grpo_loss(ctx.h, group.h, _pd(r), _pd(a), C.byref(h), C.byref(s)), ctx.h)
    return {k: getattr(s, k) for k, _ in _Stats._fields_}


def train_microbatch(tm: TriModel, group: Group, grads: GradBuffer, hyper: HyperParams, rewards=None,
                     advantages=None, rollout_old_logprobs=None, want_stats: bool = True) -> Optional[dict]:
    """Pipeline::train_microbatch, shared-prompt branch (pipeline.cpp:97-141), fully on the device.

    rollout_old_logprobs != None selects the rollout_weights mode (no old-policy forward)."""
    ctx = tm.policy.ctx
    h = hyper.c()
    s = _Stats()
    r = _f64(rewards) if rewards is not None else None
    a = _f64(advantages) if advantages is not None else None
    old = tm.old_policy.h
    if rollout_old_logprobs is not None:
        group.set_logprobs(1, rollout_old_logprobs)
        old = None
    _check(LIB.parl_train_microbatch(ctx.h, tm.policy.h, old, tm.reference.h, group.h, _pd(r), _pd(a), C.byref(h),
                                     grads.h, C.byref(s) if want_stats else None), ctx.h)
    return {k: getattr(s, k) for k, _ in _Stats._fields_} if want_stats else None


# --------------------------------------------------------------------------- GRPO operator API (grpo.hpp:50-83)
def group_advantages(rewards, ctx: Optional[Context] = None, mean_only: bool = False) -> np.ndarray:
    """grpo.cpp:24-38 (mean_only: 40-48), evaluated by K7 on the device."""
    ctx = ctx or default_context()
    r = _f64(rewards)
    out = np.zeros(max(len(r), 1), np.float64)
    _check(LIB.parl_group_advantages(ctx.h, _pd(r), len(r), int(mean_only), _pd(out)), ctx.h)
    return out[:len(r)]


def group_advantages_mean_only(rewards, ctx: Optional[Context] = None) -> np.ndarray:
    return group_advantages(rewards, ctx, mean_only=True)


def clipped_term(lp_new: float, lp_old: float, advantage: float, epsilon: float,
                 ctx: Optional[Context] = None) -> float:
    """grpo.cpp:95-101."""
    ctx = ctx or default_context()
    v = C.c_double()
    _check(LIB.parl_clipped_term(ctx.h, lp_new, lp_old, advantage, epsilon, C.byref(v)), ctx.h)
    return v.value


def kl_term(lp_new: float, lp_ref: float, ctx: Optional[Context] = None) -> float:
    """grpo.cpp:103-107."""
    ctx = ctx or default_context()
    v = C.c_double()
    _check(LIB.parl_kl_term(ctx.h, lp_new, lp_ref, C.byref(v)), ctx.h)
    return v.value


@dataclass
class Sample:
    """grpo.hpp:14-27 (fields the loss reads)."""

    response: Sequence[int]
    advantage: float = 0.0
    old_logprobs: Sequence[float] = ()
    ref_logprobs: Sequence[float] = ()
    prompt: Sequence[int] = ()
    reward: float = 0.0
    group_id: int = 0
    rollout_index: int = 0


@dataclass
class SampleTerms:
    clip_term: float
    kl: float
    clipped_units: int
    total_units: int
    upstream: np.ndarray


def per_sample_terms(sample: Sample, policy_logprobs, epsilon: float, beta: float, granularity: str = "token",
                     ctx: Optional[Context] = None) -> SampleTerms:
    """grpo.cpp:111-151."""
    ctx = ctx or default_context()
    n = len(sample.response)
    lp, old, ref = _f64(policy_logprobs), _f64(sample.old_logprobs), _f64(sample.ref_logprobs)
    if len(lp) != n or len(old) != n or len(ref) != n:
        raise ShapeError(f"logprob vectors not aligned with response length {n}")
    up = np.zeros(max(n, 1), np.float64)
    st = _SampleTerms()
    _check(LIB.parl_per_sample_terms(ctx.h, _pd(lp), _pd(old), _pd(ref), n, float(sample.advantage), epsilon, beta,
                                     0 if granularity == "token" else 1, _pd(up), C.byref(st)), ctx.h)
    return SampleTerms(st.clip_term, st.kl, st.clipped_units, st.total_units, up[:n])


@dataclass
class LossReport:
    objective: float
    clip_term_mean: float
    kl_mean: float
    clip_fraction: float
    token_count: int


@dataclass
class MicrobatchLoss:
    loss: float
    upstream: list
    report: LossReport


def grpo_microbatch_loss(samples: Sequence[Sample], policy_logprobs, epsilon: float, beta: float,
                         granularity: str = "token", ctx: Optional[Context] = None) -> MicrobatchLoss:
    """grpo.cpp:153-184."""
    ctx = ctx or default_context()
    if len(samples) == 0:
        raise ShapeError("empty micro-batch")
    if len(policy_logprobs) != len(samples):
        raise ShapeError("policy logprob count != sample count")
    lens = _i32([len(s.response) for s in samples])
    for s, lp in zip(samples, policy_logprobs):
        n = len(s.response)
        if len(lp) != n or len(s.old_logprobs) != n or len(s.ref_logprobs) != n:
            raise ShapeError(f"logprob vectors not aligned with response length {n}")
    cat = lambda xs: _f64(np.concatenate([np.asarray(x, np.float64) for x in xs]) if len(xs) else [])
    lp, old = cat(policy_logprobs), cat([s.old_logprobs for s in samples])
    ref, adv = cat([s.ref_logprobs for s in samples]), _f64([s.advantage for s in samples])
    up = np.zeros(max(len(lp), 1), np.float64)
    rep, loss = _LossReport(), C.c_double()
    _check(LIB.parl_grpo_microbatch_loss(ctx.h, len(samples), _pi(lens), _pd(lp), _pd(old), _pd(ref), _pd(adv),
                                         epsilon, beta, 0 if granularity == "token" else 1, _pd(up), C.byref(rep),
                                         C.byref(loss)), ctx.h)
    ups = np.split(up[:len(lp)], np.cumsum(lens)[:-1])
    return MicrobatchLoss(loss.value, ups, LossReport(rep.objective, rep.clip_term_mean, rep.kl_mean,
                                                      rep.clip_fraction, int(rep.token_count)))


def build_shared_prompt_mask(prompt_len: int, response_lens, ctx: Optional[Context] = None) -> np.ndarray:
    """packing.cpp:47-72: dense [n x n] allowed-pair matrix (row i attends to column j)."""
    ctx = ctx or default_context()
    lens = _i32(response_lens)
    n = int(prompt_len) + int(lens.sum())
    out = np.zeros(max(n * n, 1), np.uint8)
    _check(LIB.parl_shared_prompt_mask(ctx.h, int(prompt_len), _pi(lens), len(lens),
                                       out.ctypes.data_as(C.POINTER(C.c_uint8))), ctx.h)
    return out[:n * n].reshape(n, n).astype(bool)


def train_iteration(tm: "TriModel", groups, hyper: "HyperParams", lr: float, grads: Optional[GradBuffer] = None,
                    old_policy: str = "one_step_delayed", world_samples: Optional[int] = None,
                    allreduce: bool = False) -> dict:
    """The training half of Pipeline::run_iteration (pipeline.cpp:263-352), device-resident.

    groups: list of (Group, advantages[m], rollout_old_logprobs or None) micro-batches of this rank, in
    consumption order.  Accumulates every micro-batch (train_microbatch), then, as pipeline.cpp:346-351:
    divisor = N*G samples (world_samples when the batch is sharded over ranks), snapshot old <- policy,
    apply_update.  Returns the summed stats (allreduced across ranks when `allreduce`)."""
    ctx = tm.policy.ctx
    gb = grads if grads is not None else GradBuffer(tm.policy)
    gb.reset()
    ctx.stats_reset()
    n_samples = 0
    for group, adv, old_lp in groups:
        train_microbatch(tm, group, gb, hyper, advantages=adv,
                         rollout_old_logprobs=old_lp if old_policy == "rollout_weights" else None, want_stats=False)
        n_samples += len(adv)
    if allreduce:
        gb.allreduce()
        ctx.stats_allreduce()
    gb.set_micro_step_count(world_samples if world_samples is not None else n_samples)
    tm.snapshot_old_policy()
    tm.policy.apply_update(gb, lr)
    return ctx.stats()


def version() -> str:
    return LIB.parl_version().decode()
