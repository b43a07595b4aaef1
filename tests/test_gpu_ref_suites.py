"""The reference's own hot-path suites, compiled UNMODIFIED against the drop-in.

proj/tests/test_packing.cpp, test_model.cpp, test_grpo.cpp and test_pipeline.cpp
(with the reference caller code they exercise: pipeline.cpp, rollout.cpp, tasks.cpp,
gradcheck.cpp) are compiled where they lie against include/parl/*.hpp and a doctest
shim by paper_2511_18871_b200._build.build_ref_suites(), and run here on the GPU.
Every test case must pass except the ones listed in FP64_ONLY: those assert fp64
tolerances (finite differences at h = 1e-5, 1e-9 / 1e-10 / 1e-12 agreement) that no
fp32 device path can meet; their restated versions at the §8c
tolerances live in tests/test_gpu_parity.py and tests/test_gpu_train.py.
"""
import os
import re
import subprocess

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu
SUITE_DIR = os.path.join(ROOT, "paper_2511_18871_b200", "build", "ref_suites")
SUITES = ["test_packing", "test_grpo", "test_model", "test_pipeline"]

# test case -> the assertion sites (reference file:line) allowed to fail, each an fp64-only
# tolerance that an fp32 device path cannot meet, with the restated check
FP64_ONLY = {
    # sum_v exp(row) == 1 within 1e-12: fp32 logits / LSE give ~1e-7 (restated at fp32:
    # test_gpu_train.py::test_logprob_rows_normalized)
    "softmax rows are normalized and logprobs nonpositive": {"test_model.cpp:84"},
    # central finite differences at h = 1e-5 against 1e-6 relative error: meaningless below fp64;
    # the analytic backward is compared with the FD-verified oracle backward instead
    # (test_gpu_parity.py::test_tiny_microbatch_fp32, 1e-5 rel)
    "backward matches central finite differences on the default config": {"test_model.cpp:128"},
    # packed grad == sum of per-response grads within 1e-9 per element (test_gpu_parity.py::
    # test_shared_equals_replicated, fp32 tolerance)
    "gradient packing equivalence: packed backward equals summed per-response backwards": {"test_packing.cpp:198"},
    # packed and unpacked training reach the same weights within 1e-9 (test_gpu_train.py::
    # test_shared_prompt_equals_unpacked_update, fp32 tolerance)
    "shared-prompt packing trains to the same weights as unpacked": {"test_pipeline.cpp:269"},
}


def _run(name):
    exe = os.path.join(SUITE_DIR, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    env = dict(os.environ, PARL_PRECISION="fp32")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1200, env=env)
    cases, cur = {}, None
    for line in r.stdout.splitlines():
        m = re.match(r"^CASE (PASS|FAIL) (\d+) (\d+) (.*)$", line)
        if m:
            cur = m.group(4)
            cases[cur] = (m.group(1), int(m.group(2)), int(m.group(3)), set())
            continue
        m = re.match(r"^\s+FAILED_AT (\S+):(\d+) x\d+$", line)
        if m and cur:
            cases[cur][3].add(f"{os.path.basename(m.group(1))}:{m.group(2)}")
    print(r.stdout[-6000:])
    return cases, r


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_dropin(suite):
    cases, r = _run(suite)
    assert cases, r.stdout + r.stderr
    bad = [c for c, (st, _, _, sites) in cases.items() if st == "FAIL" and not sites <= FP64_ONLY.get(c, set())]
    assert not bad, f"{suite}: {bad}\n{r.stdout[-6000:]}"
    n_pass = sum(1 for st, *_ in cases.values() if st == "PASS")
    print(f"{suite}: {n_pass}/{len(cases)} test cases pass unmodified")
