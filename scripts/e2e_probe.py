"""Host-side timing of the end-to-end bench step (C2): wall time per step, pack and launch-issue
time per micro-batch.  python scripts/e2e_probe.py"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2511_18871_b200 import parl as P
from bench import CONFIGS
c = CONFIGS["c2"]
ctx = P.Context(0, P.PREC_BF16)
cfg = P.ModelConfig(c["vocab"], c["d"], c["L"], c["H"], c["F"], c["max_seq"])
pol = P.ModelParams.init_device(cfg, 7, ctx); tm = P.TriModel(pol, pol.clone(seed=11, noise=0.01), pol.clone())
grads = P.GradBuffer(pol); hyper = P.HyperParams(0.2, 0.04, "token")
Pn, G, R = c["P"], c["G"], c["R"]; T = Pn + G * R
rng = np.random.default_rng(123)
pr = [torch.from_numpy(rng.integers(4, c["vocab"], Pn).astype(np.int32)).pin_memory().numpy() for _ in range(2)]
rs = [torch.from_numpy(rng.integers(4, c["vocab"], G * R).astype(np.int32)).pin_memory().numpy() for _ in range(2)]
rw = [rng.random(G) for _ in range(2)]
group = P.Group(T, G, ctx)
def step(tt):
    t0 = time.perf_counter(); grads.reset(); ctx.stats_reset()
    for i in range(2):
        a = time.perf_counter()
        group.pack(pr[i], [rs[i][k * R:(k + 1) * R] for k in range(G)], c["max_seq"])
        b = time.perf_counter()
        P.train_microbatch(tm, group, grads, hyper, rewards=rw[i], want_stats=False)
        cc = time.perf_counter()
        tt.append((b - a, cc - b))
    st = ctx.stats()
    return time.perf_counter() - t0
for _ in range(3): step([])
for _ in range(8):
    tt = []
    w = step(tt)
    print("step %.1f ms  pack %.2f/%.2f ms  issue %.1f/%.1f ms" % (w * 1e3, tt[0][0] * 1e3, tt[1][0] * 1e3, tt[0][1] * 1e3, tt[1][1] * 1e3), flush=True)
