"""Shared helpers for the -m gpu parity tests (inputs rebuilt from tests/golden/)."""
import os

import numpy as np

from oracle import layout as flat_layout
from tests.conftest import GOLDEN

# Tolerances (~2.5-5x the measured noise floors)
FP32_TOL = dict(lp_abs=2e-5, grad_rel=1e-5, obj_rel=1e-6, bk_abs=1e-5)
BF16_TOL = dict(lp_max=1e-1, lp_mean=2e-2, grad_rel=5e-2, cos=0.9995, obj_rel=1e-2, bk_abs=1e-2)


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def split_resp(z):
    return np.split(z["resp_flat"], np.cumsum(z["lens"])[:-1])


def per_tensor_rel(cfg_o, got, ref, skip_bk=True):
    """{tensor: ||got-ref||_F / ||ref||_F} over the reference layout."""
    out = {}
    for name, off, r, c in flat_layout(cfg_o):
        a, b = got[off:off + r * c], ref[off:off + r * c]
        if skip_bk and name.endswith("attn.bk"):
            out[name] = float(np.abs(a - b).max())
            continue
        nb = np.linalg.norm(b)
        out[name] = float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a))
    return out


def ocfg(cfg):
    from oracle import Cfg

    return Cfg(cfg.vocab_size, cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.d_ff, cfg.max_seq_len)
