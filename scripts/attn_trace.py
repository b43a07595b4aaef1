"""Phase timeline of the attention forward's CTA 0 (needs a -DPARL_ATTN_TRACE build,
loaded through PARL_LIB).  Prints per-tile cycle offsets for the two softmax groups
(wait S, S ready, S loaded, exps done, PV(prev) done, P handed over) and the two
MMA issuers (S issued, PV wait begin, PV issued)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_18871_b200 import parl as P

f = P.LIB.parl_debug_attn_bf16
f.restype = C.c_int
f.argtypes = [C.c_int] * 5 + [C.c_void_p] * 6
# ATTN_SHAPE=c3: the C3 shape (Dh = 128)
Pl, G, R, H, Dh = (1024, 16, 4096, 28, 128) if os.environ.get("ATTN_SHAPE") == "c3" else (512, 8, 1024, 14, 64)
T = Pl + G * R
seg = torch.zeros(T, dtype=torch.int32)
st, en = [0], [Pl]
t = Pl
for k in range(G):
    seg[t:t + R] = k + 1
    st.append(t)
    en.append(t + R)
    t += R
seg, st, en = seg.cuda(), torch.tensor(st, dtype=torch.int32).cuda(), torch.tensor(en, dtype=torch.int32).cuda()
qkv = torch.randn(T, 3 * H * Dh, device="cuda").bfloat16()
out = torch.zeros(T, H * Dh, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(H, T, device="cuda")
args = (2, T, H, Dh, Pl, seg.data_ptr(), st.data_ptr(), en.data_ptr(), qkv.data_ptr(), out.data_ptr(), lse.data_ptr())
for _ in range(3):
    f(*args)
torch.cuda.synchronize()
if len(sys.argv) > 1 and sys.argv[1] == "bwd":  # trace the dK/dV kernel instead
    fb = P.LIB.parl_debug_attn_bwd_bf16
    fb.restype = C.c_int
    fb.argtypes = [C.c_int] * 5 + [C.c_void_p] * 9
    dout = torch.randn(T, H * Dh, device="cuda").bfloat16()
    dsum = torch.zeros(H, T, device="cuda")
    dqkv = torch.zeros(T, 3 * H * Dh, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        fb(2, T, H, Dh, Pl, seg.data_ptr(), st.data_ptr(), en.data_ptr(), qkv.data_ptr(), out.data_ptr(),
           dout.data_ptr(), lse.data_ptr(), dsum.data_ptr(), dqkv.data_ptr())
    torch.cuda.synchronize()
buf = np.zeros((16, 64, 8), dtype=np.uint64)
assert P.LIB.parl_debug_attn_trace(buf.ctypes.data_as(C.c_void_p)) == 0
b = buf.astype(np.int64)
span = b[12:15].reshape(-1, 8)[:, :2]
span = span[span[:, 0] > 0]
if len(span):
    s0 = span[:, 0].min()
    st, en = (span[:, 0] - s0) / 1e3, (span[:, 1] - s0) / 1e3
    print(f"CTA spans (us, {len(span)} CTAs): start max {st.max():.1f}, end min {en.min():.1f} / median "
          f"{np.median(en):.1f} / max {en.max():.1f}; busy median {np.median(en - st):.1f}")
    b[12:15] = 0
t0 = b[b > 0].min()
np.set_printoptions(linewidth=200)
if len(sys.argv) > 1 and sys.argv[1] == "bwd":
    t0 = b[4:12][b[4:12] > 0].min()
    print("per element-wise warp: P handed (k=5) and S loaded (k=2) of tiles 2..8, minus t0")
    for wp in range(8):
        print(wp, "S loaded", b[4 + wp, 2:9, 2] - t0, "P handed", b[4 + wp, 2:9, 5] - t0)
    print("mma: S issued", b[2, 2:10, 0] - t0, "PV wait", b[2, 2:10, 1] - t0, "PV issued", b[2, 2:10, 2] - t0)
    print("issue_sd: enter", b[3, 2:10, 0] - t0, "a_full ok", b[3, 2:10, 1] - t0, "b_full ok", b[3, 2:10, 2] - t0,
          "s_free ok", b[3, 2:10, 3] - t0)
    sys.exit(0)
for w in range(2):
    print(f"element-wise group {w}: [wait S, S ready, S loaded, exps done, MMA(prev) done, P handed] - t0")
    for n in range(40):
        if b[w, n, 0] == 0:
            break
        r = b[w, n, :6] - t0
        print(n, r, "dur", r[5] - r[0], "waitS", r[1] - r[0], "load", r[2] - r[1], "exp", r[3] - r[2],
              "waitPV", r[4] - r[3], "store", r[5] - r[4],
              ("item end: O ready %d, out written %d" % (b[w, n, 6] - t0, b[w, n, 7] - t0)) if b[w, n, 6] else "")
for w in range(2 if not (len(sys.argv) > 1 and sys.argv[1] == "bwd") else 1):
    print(f"mma {w}: [S issued, PV wait begin, PV issued] - t0")
    for n in range(40):
        if b[2 + w, n, 0] == 0 and b[2 + w, n, 1] == 0:
            break
        print(n, b[2 + w, n, :3] - t0)
