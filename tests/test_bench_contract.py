"""bench.py's reference arm (the one arm that runs on this CPU-only host): one JSON line with the
contract's keys, on the same metric / unit / direction as the GPU arm (BASELINE.json; bench.py).
Runs BASELINE configs[0] (C1) for one short step through oracle/_ref (the reference built from its
own sources by `__graft_entry__.build()`)."""
import json
import os
import subprocess
import sys

import pytest

from tests.conftest import ROOT


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libparl_ref.so")),
                    reason="oracle/_ref not built (run __graft_entry__.build())")
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["metric"].startswith("packed tokens/s") and d["unit"] == "packed tokens/s"
    assert d["higher_is_better"] is True and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["same_config"] is True  # C1 runs exactly BASELINE configs[0]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
