"""Throughput of the tcgen05 GEMM at the C2 hot-path shapes with their real
fused epilogues (CUDA events, 10 back-to-back launches after warm-up), next to cuBLAS
(torch.matmul, bf16 out, no epilogue) on the same operands.
    python scripts/gemm_bench.py [--rows-mult 4] [name filters]   (rows x4: 4 groups per sequence)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_18871_b200 import parl as P

f = P.LIB.parl_debug_gemm_bf16
f.restype = C.c_int
f.argtypes = [C.c_int] * 4 + [C.c_void_p, C.c_long, C.c_long, C.c_void_p, C.c_long, C.c_long, C.c_int, C.c_void_p,
                              C.c_void_p, C.c_long, C.c_void_p, C.c_void_p, C.c_long, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
argv = sys.argv[1:]
mult = 1
if "--rows-mult" in argv:
    i = argv.index("--rows-mult")
    mult = int(argv[i + 1])
    del argv[i:i + 2]
T, d, F, V, S = 8704 * mult, 896, 4864, 151936, 8192 * mult
EPI = dict(F32=0, ACC=1, ACT=2, RESID=3, GELU=4, GELU_BWD=5, LSE=6, GELU_ACT=7)
cases = [
    ("qkv fwd", T, 3 * d, d, 0, 0, "ACT"), ("o fwd", T, d, d, 0, 0, "RESID"), ("w1 fwd", T, F, d, 0, 0, "GELU"),
    ("w2 fwd", T, d, F, 0, 0, "RESID"), ("head fwd", S, V, d, 0, 0, "LSE"), ("w2 dX", T, F, d, 0, 1, "GELU_BWD"),
    ("w1 dX", T, d, F, 0, 1, "F32"), ("head dX", S, d, V, 0, 1, "F32"), ("w1 dW", d, F, T, 1, 1, "ACC"),
    ("qkv dW", d, d, T, 1, 1, "ACC"), ("head dW", d, V, S, 1, 1, "ACC"), ("big 8192^3", 8192, 8192, 8192, 0, 0, "F32"),
    # the GELU epilogues' cost: the same shapes with the plain bf16 store
    ("w1 fwd/act", T, F, d, 0, 0, "ACT"), ("w2 dX/act", T, F, d, 0, 1, "ACT"), ("w1 fwd/gelu_act", T, F, d, 0, 0, "GELU_ACT"),
]
sel = argv or None
for name, M, N, K, amn, bmn, epi in cases:
    if sel and not any(s in name for s in sel):
        continue
    A = torch.randn(K, M, device="cuda").bfloat16() if amn else torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16() if bmn else torch.randn(N, K, device="cuda").bfloat16()
    sam, sak = (1, M) if amn else (K, 1)
    sbn, sbk = (1, N) if bmn else (K, 1)
    outf = torch.zeros(M, N, device="cuda") if epi in ("F32", "ACC", "RESID") else None
    resid = torch.zeros(M, N, device="cuda") if epi == "RESID" else None
    outa = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if epi in ("ACT", "GELU", "GELU_BWD", "GELU_ACT") else None
    aux = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if epi in ("GELU", "GELU_BWD") else None
    bias = torch.zeros(N, device="cuda")
    labels = torch.randint(0, N, (M,), device="cuda", dtype=torch.int32) if epi == "LSE" else None
    n_parts = (N + 127) // 128
    part = torch.empty(M, n_parts, 2, device="cuda") if epi == "LSE" else None
    target = torch.empty(M, device="cuda") if epi == "LSE" else None
    p = lambda t: None if t is None else t.data_ptr()
    args = (0, M, N, K, A.data_ptr(), sam, sak, B.data_ptr(), sbn, sbk, EPI[epi], p(bias), p(outf), N, p(resid),
            p(outa), N, p(aux), p(aux), p(labels), p(part), p(target), None, n_parts)
    for _ in range(2):
        assert f(*args) == 0, P.LIB.parl_last_error(None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    args2 = (2,) + args[1:]
    for _ in range(n):
        f(*args2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    # cuBLAS on the same operands: C[M x N] = A(m,k) B(n,k)
    Am = A.t() if amn else A            # [M x K]
    Bm = B if bmn else B.t()            # [K x N]
    for _ in range(2):
        torch.matmul(Am, Bm)
    e0.record()
    for _ in range(n):
        torch.matmul(Am, Bm)
    e1.record()
    torch.cuda.synchronize()
    ms_cb = e0.elapsed_time(e1) / n
    print(f"{name:12s} {epi:8s} M={M:6d} N={N:6d} K={K:6d}  {ms:8.3f} ms  {2*M*N*K/ms/1e9:8.1f} TFLOP/s"
          f"   cuBLAS {ms_cb:8.3f} ms  {2*M*N*K/ms_cb/1e9:8.1f} TFLOP/s", flush=True)
    del A, B, outf, outa, aux, resid, part
    torch.cuda.empty_cache()
