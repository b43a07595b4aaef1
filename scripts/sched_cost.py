"""Host cost of packing a ragged C4-shaped group whose segment structure changes every call (the
attention tile schedule is rebuilt on the host then): python scripts/sched_cost.py"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2511_18871_b200 import parl as P
ctx = P.Context(0, P.PREC_BF16)
rng = np.random.default_rng(1)
Pn = 2048
g = P.Group(2048 + 8 * 16384, 8, ctx)
times = []
for it in range(12):
    lens = rng.integers(1024, 16385, 8)
    prompt = rng.integers(4, 151936, Pn).astype(np.int32)
    resp = [rng.integers(4, 151936, int(n)).astype(np.int32) for n in lens]
    ctx.sync()
    t0 = time.perf_counter()
    g.pack(prompt, resp, 1 << 17)
    t1 = time.perf_counter()
    ctx.sync()
    times.append((t1 - t0) * 1e3)
    print("T=%d pack host %.2f ms (new segment structure each time)" % (Pn + lens.sum(), (t1 - t0) * 1e3))
print("median ms", np.median(times[2:]))
