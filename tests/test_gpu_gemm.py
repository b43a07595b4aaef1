"""GPU unit tests of the tcgen05 contraction kernel (through the debug hook in
include/parl_gpu_debug.h) against an fp32 torch reference of the same op:
every operand layout the hot path uses (K/K forward, K/MN dX, MN/MN dW),
ragged M/N/K tails, split-K, and every fused epilogue."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EPI = dict(F32=0, F32_ACC=1, ACT=2, RESID=3, GELU=4, GELU_BWD=5, LSE=6, GELU_ACT=7)


@pytest.fixture(scope="module")
def env():
    import torch

    from paper_2511_18871_b200 import parl as P

    lib = P.LIB
    f = lib.parl_debug_gemm_bf16
    f.restype = C.c_int
    f.argtypes = [C.c_int] * 4 + [C.c_void_p, C.c_long, C.c_long, C.c_void_p, C.c_long, C.c_long, C.c_int,
                                  C.c_void_p, C.c_void_p, C.c_long, C.c_void_p, C.c_void_p, C.c_long, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
    torch.backends.cuda.matmul.allow_tf32 = False
    return torch, P, f


def ptr(t):
    return None if t is None else t.data_ptr()


def run(env, path, A, sam, sak, B, sbn, sbk, M, N, K, epi, bias=None, Cf=None, ldc=0, resid=None, Ca=None, ldca=0,
        Caux=None, aux=None, labels=None, part=None, target=None, logits=None, n_parts=0):
    torch, P, f = env
    rc = f(path, M, N, K, ptr(A), sam, sak, ptr(B), sbn, sbk, epi, ptr(bias), ptr(Cf), ldc, ptr(resid), ptr(Ca), ldca,
           ptr(Caux), ptr(aux), ptr(labels), ptr(part), ptr(target), ptr(logits), n_parts)
    assert rc == 0, P.LIB.parl_last_error(None)


def operands(torch, M, N, K, a_mn, b_mn, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    ref = A.float() @ B.float().T
    # storage: K-major = [rows x K] row-major; MN-major = [K x rows] row-major
    As = A.t().contiguous() if a_mn else A.contiguous()
    Bs = B.t().contiguous() if b_mn else B.contiguous()
    sam, sak = (1, M) if a_mn else (K, 1)
    sbn, sbk = (1, N) if b_mn else (K, 1)
    return As, sam, sak, Bs, sbn, sbk, ref


LAYOUTS = [(0, 0), (0, 1), (1, 1)]
SHAPES = [(128, 256, 64), (256, 512, 192), (296, 200, 104), (128, 896, 896), (1000, 384, 520), (64, 40, 24),
          # large enough for the CTA-pair (cta_group::2) kernel, with M/K tails
          (4096, 1024, 512), (4000, 1152, 520), (8704, 896, 896), (4096, 2688, 200)]


@pytest.mark.parametrize("lay", LAYOUTS)
@pytest.mark.parametrize("shape", SHAPES)
def test_layouts_f32(env, lay, shape):
    torch = env[0]
    M, N, K = shape
    A, sam, sak, B, sbn, sbk, ref = operands(torch, M, N, K, *lay)
    bias = torch.randn(N, device="cuda")
    out = torch.zeros(M, N, device="cuda")
    run(env, 0, A, sam, sak, B, sbn, sbk, M, N, K, EPI["F32"], bias=bias, Cf=out, ldc=N)
    err = (out - (ref + bias)).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


def test_split_k_accumulate_pair(env):
    torch = env[0]
    M, N, K = 896, 4864, 8704  # dW shape: pair kernel + split-K
    A, sam, sak, B, sbn, sbk, ref = operands(torch, M, N, K, 1, 1, seed=9)
    out = torch.zeros(M, N, device="cuda")
    run(env, 0, A, sam, sak, B, sbn, sbk, M, N, K, EPI["F32_ACC"], Cf=out, ldc=N)
    err = (out - ref).abs().max().item() / ref.abs().max().item()
    assert err < 3e-5, err  # fp32 accumulation over K = 8704 in a different order than torch


def test_split_k_accumulate(env):
    torch = env[0]
    M, N, K = 256, 384, 8704  # dW shape class: small M x N, K = tokens
    A, sam, sak, B, sbn, sbk, ref = operands(torch, M, N, K, 1, 1)
    out = torch.randn(M, N, device="cuda")
    base = out.clone()
    run(env, 0, A, sam, sak, B, sbn, sbk, M, N, K, EPI["F32_ACC"], Cf=out, ldc=N)
    err = (out - base - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err
    out2 = base.clone()
    run(env, 0, A, sam, sak, B, sbn, sbk, M, N, K, EPI["F32_ACC"], Cf=out2, ldc=N)
    assert torch.equal(out, out2)  # deterministic split order


@pytest.mark.parametrize("shape", [(384, 512, 256), (4096, 1024, 512), (2000, 896, 200),
                                   # 224-wide CTA-pair tiles (N = 896, 2688)
                                   (4096, 896, 512), (3000, 2688, 256)])
def test_epilogues(env, shape):
    torch = env[0]
    M, N, K = shape
    A, sam, sak, B, sbn, sbk, ref = operands(torch, M, N, K, 0, 0, seed=3)
    bias = torch.randn(N, device="cuda")
    # ACT
    Ca = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    run(env, 0, A, sam, sak, B, sbn, sbk, M, N, K, EPI["ACT"], bias=bias, Ca=Ca, ldca=N)
    assert torch.allclose(Ca.float(), (ref + bias).bfloat16().float(), rtol=1e-2, atol=1e-2)
    # RESID
    resid = torch.randn(M, N, device="cuda")
    out = torch.empty(M, N, device="cuda")
    run(env, 0, A, sam, sak, B, sbn, sbk, M, N, K, EPI["RESID"], bias=bias, Cf=out, ldc=N, resid=resid)
    assert (out - (resid + ref + bias)).abs().max().item() < 1e-3
    # GELU (pre and act)
    u = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    act = torch.empty_like(u)
    run(env, 0, A, sam, sak, B, sbn, sbk, M, N, K, EPI["GELU"], bias=bias, Ca=u, ldca=N, Caux=act)
    uref = (ref + bias).bfloat16()
    assert torch.allclose(u.float(), uref.float(), rtol=1e-2, atol=1e-2)
    gref = torch.nn.functional.gelu(u.float()).bfloat16()
    assert torch.allclose(act.float(), gref.float(), rtol=1e-2, atol=1e-2)
    # GELU_ACT (activation only)
    act2 = torch.empty_like(u)
    run(env, 0, A, sam, sak, B, sbn, sbk, M, N, K, EPI["GELU_ACT"], bias=bias, Ca=act2, ldca=N)
    assert torch.equal(act2, act)
    # GELU_BWD
    aux = torch.randn(M, N, device="cuda").bfloat16()
    d = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    run(env, 0, A, sam, sak, B, sbn, sbk, M, N, K, EPI["GELU_BWD"], Ca=d, ldca=N, aux=aux)
    x = aux.float().requires_grad_(True)
    gp = torch.autograd.grad(torch.nn.functional.gelu(x).sum(), x)[0]
    assert torch.allclose(d.float(), (ref * gp).bfloat16().float(), rtol=2e-2, atol=2e-2)


def test_lse_epilogue(env):
    torch = env[0]
    M, N, K = 300, 151936 // 16 + 37, 128  # ragged vocab, partial last tile
    A, sam, sak, B, sbn, sbk, ref = operands(torch, M, N, K, 0, 0, seed=5)
    bias = torch.randn(N, device="cuda") * 0.1
    z = ref + bias
    labels = torch.randint(0, N, (M,), device="cuda", dtype=torch.int32)
    n_parts = (N + 127) // 128
    part = torch.zeros(M, n_parts, 2, device="cuda")
    target = torch.zeros(M, device="cuda")
    logits = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    run(env, 0, A, sam, sak, B, sbn, sbk, M, N, K, EPI["LSE"], bias=bias, labels=labels, part=part, target=target,
        logits=logits, ldca=N, n_parts=n_parts)
    m = part[:, :, 0]
    lse = m.max(1).values + torch.log((part[:, :, 1] * torch.exp(m - m.max(1, keepdim=True).values)).sum(1))
    assert (lse - torch.logsumexp(z, 1)).abs().max().item() < 1e-3
    assert (target - z.gather(1, labels.long()[:, None])[:, 0]).abs().max().item() < 1e-3
    assert torch.allclose(logits.float(), z.bfloat16().float(), rtol=1e-2, atol=1e-2)
