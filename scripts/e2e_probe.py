"""Host-side timing of the C2 bench step, packing 4 groups per sequence: wall time per step, and
per micro-batch the host time of the pack call and of the train_microbatch call (a call that
takes ~ a micro-step's GPU time means the host blocked on the stream; a few ms means it only
enqueued).  Both the device-resident path (pack_multi_device) and the host-input path
(pack_multi from pinned host arrays).   python scripts/e2e_probe.py [micro_steps]"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2511_18871_b200 import parl as P  # noqa: E402

c = CONFIGS["c2"]
NM = int(sys.argv[1]) if len(sys.argv) > 1 else 4
K = 4
ctx = P.Context(0, P.PREC_BF16)
cfg = P.ModelConfig(c["vocab"], c["d"], c["L"], c["H"], c["F"], c["max_seq"])
pol = P.ModelParams.init_device(cfg, 7, ctx)
tm = P.TriModel(pol, pol.clone(seed=11, noise=0.01), pol.clone())
grads = P.GradBuffer(pol)
hyper = P.HyperParams(0.2, 0.04, "token")
Pn, G, R = c["P"], c["G"], c["R"]
T1 = Pn + G * R
rng = np.random.default_rng(123)
pr = [torch.from_numpy(rng.integers(4, c["vocab"], Pn).astype(np.int32)).pin_memory().numpy() for _ in range(K)]
rs = [torch.from_numpy(rng.integers(4, c["vocab"], G * R).astype(np.int32)).pin_memory().numpy() for _ in range(K)]
d_pr = torch.from_numpy(np.concatenate(pr)).cuda()
d_rs = torch.from_numpy(np.concatenate(rs)).cuda()
rw = rng.random(K * G)
group = P.Group(K * T1, K * G, ctx)


def step(tt, device):
    t0 = time.perf_counter()
    grads.reset()
    ctx.stats_reset()
    for _ in range(NM):
        a = time.perf_counter()
        if device:
            group.pack_multi_device(d_pr.data_ptr(), [Pn] * K, d_rs.data_ptr(), [R] * (K * G), [G] * K, c["max_seq"])
        else:
            group.pack_multi(pr, [[r[k * R:(k + 1) * R] for k in range(G)] for r in rs], c["max_seq"])
        b = time.perf_counter()
        P.train_microbatch(tm, group, grads, hyper, rewards=rw, want_stats=False)
        cc = time.perf_counter()
        tt.append((b - a, cc - b))
    ctx.stats()
    return time.perf_counter() - t0


for device in (True, False):
    for _ in range(2):
        step([], device)
    for _ in range(3):
        tt = []
        w = step(tt, device)
        print("%s step %.1f ms (%.1f ms / micro-step) | pack ms %s | train_microbatch ms %s" % (
            "device" if device else "host  ", w * 1e3, w * 1e3 / NM, " ".join("%.1f" % (x[0] * 1e3) for x in tt),
            " ".join("%.1f" % (x[1] * 1e3) for x in tt)), flush=True)
