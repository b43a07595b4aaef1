"""tcgen05 vs FFMA attention forward / backward at C2 / C3-like shapes (CUDA events).
   python scripts/attn_bench.py [c2|c3]   (default: both; the FFMA reference only where T < 20k)"""
import ctypes as C, os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
# the library directly (PARL_LIB: A/B of another build; no dependency on parl.py's symbol list)
LIB = C.CDLL(os.environ.get("PARL_LIB") or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                          "paper_2511_18871_b200", "libparl_gpu.so"))
LIB.parl_last_error.restype = C.c_char_p
class P:  # noqa: N801
    LIB = LIB
f = P.LIB.parl_debug_attn_bf16
f.restype = C.c_int
f.argtypes = [C.c_int] * 5 + [C.c_void_p] * 6
SHAPES = {"c2": (512, 8, 1024, 14, 64), "c3": (1024, 16, 4096, 28, 128)}
SEL = [SHAPES[a] for a in sys.argv[1:]] or list(SHAPES.values())
for (Pl, G, R, H, Dh) in SEL:
    lens = [R] * G
    T = Pl + G * R
    seg = torch.zeros(T, dtype=torch.int32)
    st, en = [0], [Pl]
    t = Pl
    for k, n in enumerate(lens):
        seg[t:t+n] = k + 1; st.append(t); en.append(t + n); t += n
    seg, st, en = seg.cuda(), torch.tensor(st, dtype=torch.int32).cuda(), torch.tensor(en, dtype=torch.int32).cuda()
    qkv = torch.randn(T, 3 * H * Dh, device="cuda").bfloat16()
    out = torch.zeros(T, H * Dh, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(H, T, device="cuda")
    pairs = Pl * (Pl + 1) / 2 + sum(r * Pl + r * (r + 1) / 2 for r in lens)
    flops = 4 * pairs * H * Dh
    for path in ((0, 1) if T < 20000 else (0,)):
        args = (path, T, H, Dh, Pl, seg.data_ptr(), st.data_ptr(), en.data_ptr(), qkv.data_ptr(), out.data_ptr(), lse.data_ptr())
        assert f(*args) == 0, P.LIB.parl_last_error(None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 30 if path == 0 else 1
        args2 = ((2,) + args[1:]) if path == 0 else args
        e0.record()
        for _ in range(n):
            f(*args2)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(f"attn fwd {'tc' if path == 0 else 'ffma'} T={T} H={H} Dh={Dh}: {ms:.3f} ms  {flops/ms/1e9:.1f} TFLOP/s", flush=True)
fb = P.LIB.parl_debug_attn_bwd_bf16
fb.restype = C.c_int
fb.argtypes = [C.c_int] * 5 + [C.c_void_p] * 9
SHAPES = {"c2": (512, 8, 1024, 14, 64), "c3": (1024, 16, 4096, 28, 128)}
SEL = [SHAPES[a] for a in sys.argv[1:]] or list(SHAPES.values())
for (Pl, G, R, H, Dh) in SEL:
    lens = [R] * G
    T = Pl + G * R
    seg = torch.zeros(T, dtype=torch.int32)
    st, en = [0], [Pl]
    t = Pl
    for k, n in enumerate(lens):
        seg[t:t+n] = k + 1; st.append(t); en.append(t + n); t += n
    seg, st, en = seg.cuda(), torch.tensor(st, dtype=torch.int32).cuda(), torch.tensor(en, dtype=torch.int32).cuda()
    d = H * Dh
    qkv = torch.randn(T, 3 * d, device="cuda").bfloat16()
    out = torch.randn(T, d, device="cuda").bfloat16()
    dout = torch.randn(T, d, device="cuda").bfloat16()
    lse = torch.full((H, T), 5.0, device="cuda")
    dsum = torch.zeros(H, T, device="cuda")
    dqkv = torch.zeros(T, 3 * d, device="cuda", dtype=torch.bfloat16)
    pairs = Pl * (Pl + 1) / 2 + sum(r * Pl + r * (r + 1) / 2 for r in lens)
    flops = 10 * pairs * d
    for path in ((0, 1) if T < 20000 else (0,)):
        args = (path, T, H, Dh, Pl, seg.data_ptr(), st.data_ptr(), en.data_ptr(), qkv.data_ptr(), out.data_ptr(),
                dout.data_ptr(), lse.data_ptr(), dsum.data_ptr(), dqkv.data_ptr())
        assert fb(*args) == 0, P.LIB.parl_last_error(None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 30 if path == 0 else 1
        args2 = ((2,) + args[1:]) if path == 0 else args
        e0.record()
        for _ in range(n):
            fb(*args2)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(f"attn bwd {'tc' if path == 0 else 'ffma'} T={T} H={H} Dh={Dh}: {ms:.3f} ms  {flops/ms/1e9:.1f} TFLOP/s", flush=True)
