"""Per-tensor bf16-vs-fp32 gradient error at C1 (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2511_18871_b200 import parl as P
from tests.gpu_helpers import load, split_resp, ocfg
from oracle import layout
from oracle.make_golden import perturb
z = load("c1_micro.npz")
cfg = P.ModelConfig(4096, 256, 2, 4, 1024, 576)
res = {}
for prec in (P.PREC_FP32, P.PREC_BF16):
    ctx = P.Context(0, prec)
    pol = P.ModelParams.init(cfg, 7, ctx); w = pol.flat()
    tm = P.TriModel(pol, P.ModelParams.from_flat(cfg, perturb(w, 21, 0.01), ctx=ctx), P.ModelParams.from_flat(cfg, perturb(w, 22, 0.01), ctx=ctx))
    pk = P.pack_group(z["prompt"], split_resp(z), cfg.max_seq_len, ctx)
    gb = P.GradBuffer(pol)
    st = P.train_microbatch(tm, pk.group, gb, P.HyperParams(), advantages=z["advantages"])
    res[prec] = (gb.flat(), [pk.group.logprobs(s) for s in range(3)], pk.group.upstream(), st)
g32, lp32, up32, _ = res[0]; g16, lp16, up16, _ = res[1]
for s in range(3): print("lp slot", s, "max", np.abs(lp32[s]-lp16[s]).max(), "mean", np.abs(lp32[s]-lp16[s]).mean())
print("upstream rel", np.linalg.norm(up32-up16)/np.linalg.norm(up32))
for name, off, r, c in layout(ocfg(cfg)):
    a, b = g16[off:off+r*c], g32[off:off+r*c]
    nb = np.linalg.norm(b)
    print(f"{name:28s} rel {np.linalg.norm(a-b)/max(nb,1e-30):.3e}  |ref| {nb:.3e}")
print("global rel", np.linalg.norm(g16-g32)/np.linalg.norm(g32), "cos", g16@g32/np.linalg.norm(g16)/np.linalg.norm(g32))
