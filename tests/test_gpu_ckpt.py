"""GPU: PARLCKP1 checkpoints (save_checkpoint / load_checkpoint, model.cpp:907-987)
through the C-ABI, against the file the reference itself writes."""
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

GOLD = os.path.join(GOLDEN, "tiny_seed41.parlckp1")


@pytest.fixture(scope="module")
def P():
    from paper_2511_18871_b200 import parl

    return parl


@pytest.fixture(scope="module")
def ctx32(P):
    return P.Context(0, P.PREC_FP32)


def tiny(P):
    return P.ModelConfig(16, 16, 2, 2, 24, 64)


def test_save_is_byte_identical_to_reference(P, ctx32, tmp_path):
    """init(seed 41) then save: the same bytes as the reference's save_checkpoint."""
    pm = P.ModelParams.init(tiny(P), 41, ctx32)
    path = str(tmp_path / "a.parlckp1")
    pm.save(path)
    with open(path, "rb") as a, open(GOLD, "rb") as b:
        assert a.read() == b.read()


def test_load_reference_checkpoint(P, ctx32, orc):
    from oracle import Cfg

    pm = P.ModelParams.load(GOLD, ctx32)
    assert pm.config == tiny(P) and pm.version() == 0
    assert np.array_equal(pm.flat(), orc.init_params(Cfg(16, 16, 2, 2, 24, 64), 41))


def test_round_trip_version_and_values(P, ctx32, tmp_path):
    from oracle import read_parlckp1

    w = np.random.default_rng(3).normal(0, 0.1, tiny(P).param_count())
    pm = P.ModelParams.from_flat(tiny(P), w, version=7, ctx=ctx32)
    path = str(tmp_path / "b.parlckp1")
    pm.save(path)
    cfg, version, seed, names, flat = read_parlckp1(path)
    assert version == 7 and np.array_equal(flat, w)
    back = P.ModelParams.load(path, ctx32)
    assert back.version() == 7 and np.array_equal(back.flat(), w)


def test_load_errors(P, ctx32, tmp_path):
    with pytest.raises(P.IoError):
        P.ModelParams.load(str(tmp_path / "missing.parlckp1"), ctx32)
    raw = open(GOLD, "rb").read()
    bad = tmp_path / "bad.parlckp1"
    bad.write_bytes(b"XARLCKP1" + raw[8:])
    with pytest.raises(P.IoError):
        P.ModelParams.load(str(bad), ctx32)
    bad.write_bytes(raw[:-100])  # truncated in the last tensor
    with pytest.raises(P.IoError):
        P.ModelParams.load(str(bad), ctx32)
    nan = bytearray(raw)
    nan[-8:] = np.array([np.nan]).tobytes()  # last head.b entry
    bad.write_bytes(bytes(nan))
    with pytest.raises(P.NumericError):
        P.ModelParams.load(str(bad), ctx32)
