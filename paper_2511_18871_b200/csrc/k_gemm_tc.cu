// tcgen05 GEMM for sm_100a: C[M x N] = sum_k A(m,k) B(n,k), bf16 operands,
// fp32 accumulation in TMEM, fused epilogues of the hot path.
//
// Persistent, warp-specialised CTA (one per SM, 256 threads):
//   warp 0      TMA producer   (cp.async.bulk.tensor, SWIZZLE_128B, mbarrier ring)
//   warp 1      MMA issuer     (one thread issues tcgen05.mma 128 x BN x 16)
//   warp 2      TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4..7  epilogue       (tcgen05.ld 32x32b: thread i owns tile row i)
// A and B may each be K-major or MN-major in global memory; the layout is
// carried by the TMA box orientation, the UMMA smem descriptor (LBO/SBO) and
// the instruction descriptor's major bits, so no transposes are ever
// materialised (forward: K/K, dX: K/MN, dW: MN/MN).
// Weight-gradient GEMMs (K = tokens) use a deterministic split-K: partials go
// to a workspace and are summed in split order by a second kernel.
//
// Replaces `linear` (proj/src/model.cpp:301-314), the head (model.cpp:520)
// with its logsumexp (model.cpp:523-556) fused into the epilogue, and the
// dX/dW loops of `backward` (model.cpp:652-817).
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

#include "internal.cuh"
#include "tc_util.cuh"

namespace parl_gpu {

namespace {

constexpr int BM = 128, BK = 64;
constexpr int EPI_WARPS = 8;                      // two per TMEM lane quadrant, each half the columns
constexpr int NTHREADS = 128 + 32 * EPI_WARPS;    // warps 0-3 producer/MMA/TMEM/spare, 4.. epilogue
constexpr int STG_BYTES = 4096;                   // epilogue staging buffer: 32 rows x 128 B
constexpr int NBUF = 3;                           // staging buffers per epilogue warp
constexpr int EPI_SMEM = EPI_WARPS * NBUF * STG_BYTES;

struct TcArgs {
    int M, N, K, nkb, tiles_m, tiles_n, splits, kbs, epi;
    const float* bias;
    int bias_vec;          // bias is 16-byte aligned
    const int32_t* labels;
    float* part;
    float* target;
    int n_parts;
    int store_logits;      // EPI_LSE: also store bf16 logits (policy, for the backward) by TMA
    bf16* logits_direct;   // EPI_LSE: ... or by plain stores when the row stride is not 16-byte aligned
    long ldl;
    int raster;            // CTA-pair kernels: 1 = n-tiles fastest (B small, stays in L2; A read once)
};

template <int BN>
struct Cfg {
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int STAGES = BN == 256 ? 2 : 4;
    static constexpr int STG_OFF = STAGES * STAGE;  // 1024-aligned
    static constexpr int BAR_OFF = STG_OFF + EPI_SMEM;
    static constexpr int SMEM = BAR_OFF + 512 + 1024;
};

// Phi(x) = 0.5 (1 + erf(x / sqrt 2)) with erf(z) ~= tanh(z (a0 + a1 z^2 + a2 z^4))
// (minimax fit on [0, 6]: |erf err| <= 3.7e-5, plus the hardware tanh.approx's
// ~2^-11 relative error, both far below the bf16 rounding of the outputs).
// One MUFU op per GELU, two per GELU'.
__device__ __forceinline__ float tanh_approx(float x) {
    float r;
    asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float erf_arg(float x, float x2) {  // y with erf(x / sqrt 2) ~= tanh(y)
    x2 = fminf(x2, 72.f);  // the fit's range |x| <= 6 sqrt 2; beyond it tanh(y) saturates at +-1
    return x * fmaf(x2, fmaf(x2, -0.000315806263f, 0.0367982576f), 0.797717834f);
}
__device__ __forceinline__ float gelu_dev(float x) {  // x * Phi(x)  (model.cpp:255)
    const float h = 0.5f * x;
    return fmaf(h, tanh_approx(erf_arg(x, x * x)), h);
}
__device__ __forceinline__ float gelu_grad_dev(float x) {  // Phi(x) + x phi(x)  (model.cpp:257-260)
    const float x2 = x * x;
    const float phi = fmaf(0.5f, tanh_approx(erf_arg(x, x2)), 0.5f);
    const float e = tc::ex2_approx(x2 * -0.72134752044448170368f);  // exp(-x^2 / 2)
    return fmaf(x * 0.39894228040143267794f, e, phi);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&t);
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// The same GELU / GELU' on a pair in packed fp32 arithmetic (FFMA2 / FMUL2: the per-lane
// operations and rounding of gelu_dev / gelu_grad_dev, half the issue slots)
__device__ __forceinline__ float2 erf_arg2(float2 x, float2 x2) {
    x2.x = fminf(x2.x, 72.f);
    x2.y = fminf(x2.y, 72.f);
    const float2 p = tc::ffma2(x2, tc::ffma2(x2, make_float2(-0.000315806263f, -0.000315806263f),
                                             make_float2(0.0367982576f, 0.0367982576f)),
                               make_float2(0.797717834f, 0.797717834f));
    return tc::fmul2(x, p);
}
__device__ __forceinline__ float2 gelu_dev2(float2 x) {
    const float2 h = tc::fmul2(make_float2(0.5f, 0.5f), x);
    const float2 y = erf_arg2(x, tc::fmul2(x, x));
    return tc::ffma2(h, make_float2(tanh_approx(y.x), tanh_approx(y.y)), h);
}
__device__ __forceinline__ float2 gelu_grad_dev2(float2 x) {
    const float2 x2 = tc::fmul2(x, x);
    const float2 y = erf_arg2(x, x2);
    const float2 phi = tc::ffma2(make_float2(0.5f, 0.5f), make_float2(tanh_approx(y.x), tanh_approx(y.y)),
                                 make_float2(0.5f, 0.5f));
    const float2 ea = tc::fmul2(x2, make_float2(-0.72134752044448170368f, -0.72134752044448170368f));
    const float2 e = make_float2(tc::ex2_approx(ea.x), tc::ex2_approx(ea.y));
    return tc::ffma2(tc::fmul2(x, make_float2(0.39894228040143267794f, 0.39894228040143267794f)), e, phi);
}
// byte offset of 16-byte chunk j of row r in a [32 x 128 B] SWIZZLE_128B / [32 x 64 B] SWIZZLE_64B tile
__device__ __forceinline__ uint32_t sw128(int r, int j) { return r * 128 + ((j ^ (r & 7)) << 4); }
__device__ __forceinline__ uint32_t sw64(int r, int j) { return r * 64 + ((j ^ ((r >> 1) & 3)) << 4); }

// The CTA's sequence of output tiles (both kernels share the epilogue).
struct EpiSeq {
    int first, stride, n_items, tiles_me;  // items first, first+stride, ...; m-tiles per n column
    int mrows;                             // rows per m-tile (128, or 256 for a CTA pair)
    int rank;                              // CTA rank within the pair
    int tpp;                               // items per problem (grouped launches of equal-shape problems)
};

// Epilogue warps (4..11).  Thread = accumulator row (TMEM lane); warp w owns
// lane quadrant w%4 and half of the tile's columns, in 32-column chunks:
//   tcgen05.ld 32 columns -> registers -> fused math (bias, residual, GELU,
//   GELU', log-sum-exp) -> swizzled smem staging -> one TMA bulk store per
//   chunk (reduce-add for in-place gradient accumulation).
// Inputs of the epilogue (fp32 residual, bf16 GELU pre-activation) arrive by
// TMA into the same staging buffer two chunks ahead.  Three staging buffers per
// warp let the stores of chunks k-1, k-2 drain while chunk k is computed.
// Grouped launches (NP > 1 equal-shape problems, e.g. the three models' copies
// of one layer GEMM): item = problem * tpp + tile; av / mo / mo2 / mi are per
// problem.  The epilogue class (input, number of outputs) is the same for all.
template <int BNT, class Release>
__device__ __forceinline__ void epilogue_warps(const TcArgs* av, const CUtensorMap* mo, const CUtensorMap* mo2,
                                               const CUtensorMap* mi, uint8_t* stg_all, uint64_t* inbar_all,
                                               uint64_t* tfull, uint32_t tbase, const EpiSeq& e, Release release) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ew = warp & 3, half = (warp - 4) >> 2, wi = warp - 4;
    // the two warp halves own columns [0, H0) and [H0, BNT) of the tile (224-wide pair
    // tiles split 128 + 96 so every chunk is a full 32 columns)
    constexpr int H0 = BNT == 224 ? 128 : BNT / 2;
    const int hcol = half ? H0 : 0;
    const int NCH = (half ? BNT - H0 : H0) / 32;
    uint8_t* stg = stg_all + wi * NBUF * STG_BYTES;
    const uint32_t stg_s = tc::smem_u32(stg);
    uint64_t* inbar = inbar_all + wi * NBUF;
    const TcArgs& a0 = av[0];
    const bool has_in = a0.epi == EPI_RESID || a0.epi == EPI_GELU_BWD;
    const uint32_t in_bytes = a0.epi == EPI_RESID ? 4096u : 2048u;
    const bool do_store = a0.epi != EPI_LSE || a0.store_logits;

    auto coords_calc = [&](int item, int& row, int& col, int& sp) {
        const int t = item % e.tpp;
        int mt, nt;
        if (a0.raster) {
            nt = t % a0.tiles_n;
            const int rest = t / a0.tiles_n;
            mt = rest % e.tiles_me;
            sp = rest / e.tiles_me;
        } else {
            mt = t % e.tiles_me;
            const int rest = t / e.tiles_me;
            nt = rest % a0.tiles_n;
            sp = rest / a0.tiles_n;
        }
        row = mt * e.mrows + e.rank * BM + ew * 32;
        col = nt * BNT + hcol;
    };
    // the chunk streams (prefetch, bias, current) ask for the same item NCH times in a row, and the
    // integer divisions above cost ~60 instructions: keep the last two items' coordinates
    int ci0 = -1, cr0 = 0, cc0 = 0, cs0 = 0, ci1 = -1, cr1 = 0, cc1 = 0, cs1 = 0;
    bool c_next = false;
    auto coords = [&](int item, int& row, int& col, int& sp) {
        if (ci0 == item) {
            row = cr0; col = cc0; sp = cs0;
            return;
        }
        if (ci1 == item) {
            row = cr1; col = cc1; sp = cs1;
            return;
        }
        coords_calc(item, row, col, sp);
        if (c_next) {
            ci1 = item; cr1 = row; cc1 = col; cs1 = sp;
        } else {
            ci0 = item; cr0 = row; cc0 = col; cs0 = sp;
        }
        c_next = !c_next;
    };
    // chunk stream: (item, c) -> the next chunk; item >= n_items when exhausted
    auto next = [&](int& item, int& c) {
        if (++c == NCH) {
            c = 0;
            item += e.stride;
        }
    };
    auto issue_in = [&](int item, int c, int b) {
        int row, col, sp;
        coords(item, row, col, sp);
        tc::mbar_expect_tx(&inbar[b], in_bytes);
        tc::tma_load_2d(stg + b * STG_BYTES, mi + item / e.tpp, &inbar[b], col + c * 32, row);
    };
    // bias of a chunk, loaded one chunk ahead (broadcast loads: every lane reads the same columns)
    float bn[32];
    auto load_bias = [&](int item, int c) {
        if (item >= e.n_items) return;
        const TcArgs& a = av[item / e.tpp];
        if (!a.bias) return;
        int row, col, sp;
        coords(item, row, col, sp);
        col += c * 32;
        if (a.bias_vec && col + 32 <= a.N) {
            const float4* bp = reinterpret_cast<const float4*>(a.bias + col);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float4 t = __ldg(bp + j);
                bn[4 * j] = t.x; bn[4 * j + 1] = t.y; bn[4 * j + 2] = t.z; bn[4 * j + 3] = t.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) bn[j] = col + j < a.N ? __ldg(a.bias + col + j) : 0.f;
        }
    };

    uint32_t k = 0, local = 0;
    // input prefetch runs two chunks ahead (NBUF = 3 staging buffers)
    int pf_item = e.first, pf_c = 0;
    if (has_in && lane == 0) {
        for (int q = 0; q < 2 && pf_item < e.n_items; ++q) {
            issue_in(pf_item, pf_c, q);
            next(pf_item, pf_c);
        }
    }
    load_bias(e.first, 0);
    for (int item = e.first; item < e.n_items; item += e.stride, ++local) {
        const uint32_t acc = local & 1, use = local >> 1;
        const int prob = item / e.tpp;
        const TcArgs& a = av[prob];
        const int epi = a.epi;
        tc::mbar_wait(&tfull[acc], use & 1);
        tc::tc_fence_after();
        int row0, colh, sp;
        coords(item, row0, colh, sp);
        const int row = row0 + lane;
        const int label = (epi == EPI_LSE && row < a.M) ? a.labels[row] : -1;
        float lm = -INFINITY, ls = 0.f;
#pragma unroll 1
        for (int c = 0; c < NCH; ++c, ++k) {
            const int col = colh + c * 32;
            const uint32_t b = k % NBUF;
            const uint32_t sb = stg_s + b * STG_BYTES;
            float v[32];
            tc::tmem_ld32(tbase + acc * BNT + hcol + c * 32 + ((uint32_t)(ew * 32) << 16), v);
            if (c == NCH - 1) {  // accumulator fully read: hand it back to the MMA warp
                tc::tc_fence_before();
                release(acc);
            }
            if (a.bias) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] += bn[j];
                int ni = item, nc = c;
                next(ni, nc);
                load_bias(ni, nc);
            }
            if (has_in) {
                tc::mbar_wait(&inbar[b], (k / NBUF) & 1);
            } else if (do_store) {  // the store issued from this buffer NBUF chunks ago has read it
                if (lane == 0) tc::bulk_wait_read<NBUF - 1>();
                __syncwarp();
            }
            switch (epi) {
                case EPI_F32:
                case EPI_F32_ACC:
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        tc::sts128(sb + sw128(lane, j), __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                                   __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
                    break;
                case EPI_RESID: {  // all inputs first: the shared loads are ordered behind the stores
                    uint32_t r[32];
#pragma unroll
                    for (int j = 0; j < 8; ++j) tc::lds128(sb + sw128(lane, j), r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float2 s0 = tc::fadd2(make_float2(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1])),
                                                    make_float2(v[4 * j], v[4 * j + 1]));
                        const float2 s1 = tc::fadd2(make_float2(__uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])),
                                                    make_float2(v[4 * j + 2], v[4 * j + 3]));
                        tc::sts128(sb + sw128(lane, j), __float_as_uint(s0.x), __float_as_uint(s0.y), __float_as_uint(s1.x),
                                   __float_as_uint(s1.y));
                    }
                    break;
                }
                case EPI_ACT:
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        tc::sts128(sb + sw64(lane, j), pack_bf16(v[8 * j], v[8 * j + 1]),
                                   pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                                   pack_bf16(v[8 * j + 6], v[8 * j + 7]));
                    break;
                case EPI_GELU: {  // 16 independent pairs, then the stores
                    uint32_t u[16], g[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        u[q] = pack_bf16(v[2 * q], v[2 * q + 1]);
                        const float2 gg = gelu_dev2(make_float2(bf_lo(u[q]), bf_hi(u[q])));
                        g[q] = pack_bf16(gg.x, gg.y);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        tc::sts128(sb + sw64(lane, j), u[4 * j], u[4 * j + 1], u[4 * j + 2], u[4 * j + 3]);
                        tc::sts128(sb + 2048 + sw64(lane, j), g[4 * j], g[4 * j + 1], g[4 * j + 2], g[4 * j + 3]);
                    }
                    break;
                }
                case EPI_GELU_ACT: {  // activation only (no backward will need the pre-activation)
                    uint32_t g[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const uint32_t u = pack_bf16(v[2 * q], v[2 * q + 1]);
                        const float2 gg = gelu_dev2(make_float2(bf_lo(u), bf_hi(u)));
                        g[q] = pack_bf16(gg.x, gg.y);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) tc::sts128(sb + sw64(lane, j), g[4 * j], g[4 * j + 1], g[4 * j + 2], g[4 * j + 3]);
                    break;
                }
                case EPI_GELU_BWD: {  // all inputs first, then 16 independent pairs, then the stores
                    uint32_t x[16];
#pragma unroll
                    for (int j = 0; j < 4; ++j) tc::lds128(sb + sw64(lane, j), x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const float2 gd = tc::fmul2(make_float2(v[2 * q], v[2 * q + 1]),
                                                    gelu_grad_dev2(make_float2(bf_lo(x[q]), bf_hi(x[q]))));
                        x[q] = pack_bf16(gd.x, gd.y);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) tc::sts128(sb + sw64(lane, j), x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
                    break;
                }
                case EPI_LSE: {
                    const int ncol = min(32, a.N - col);
                    float cm = -INFINITY;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < ncol) cm = fmaxf(cm, v[j]);
                    const float nm = fmaxf(lm, cm);
                    const float nml = nm * 1.4426950408889634f;
                    float s = 0.f;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < ncol) s += tc::ex2_approx(fmaf(v[j], 1.4426950408889634f, -nml));
                    ls = ls * tc::ex2_approx((lm - nm) * 1.4426950408889634f) + s;
                    lm = nm;
                    const int lj = label - col;
                    if ((unsigned)lj < 32u) {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (j == lj) a.target[row] = v[j];
                    }
                    if (a.logits_direct && row < a.M) {
                        bf16* dst = a.logits_direct + (long)row * a.ldl + col;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (j < ncol) dst[j] = __float2bfloat16_rn(v[j]);
                    }
                    if (a.store_logits) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            tc::sts128(sb + sw64(lane, j), pack_bf16(v[8 * j], v[8 * j + 1]),
                                       pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                                       pack_bf16(v[8 * j + 6], v[8 * j + 7]));
                    }
                    break;
                }
                default:
                    break;
            }
            if (do_store) {
                tc::fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (epi == EPI_F32_ACC) {
                        if (a.splits > 1) tc::tma_store_3d(mo + prob, sb, col, row0, sp);
                        else tc::tma_reduce_add_2d(mo + prob, sb, col, row0);
                    } else if (epi == EPI_LSE) {  // the policy's logits: written once, read by the backward
                        tc::tma_store_2d_hint(mo + prob, sb, col, row0, tc::l2_evict_first_policy());
                    } else {
                        tc::tma_store_2d(mo + prob, sb, col, row0);
                        if (epi == EPI_GELU) tc::tma_store_2d(mo2 + prob, sb + 2048, col, row0);
                    }
                    tc::bulk_commit();
                    if (has_in && pf_item < e.n_items) {
                        // chunk k+2 goes into the buffer chunk k-1 used: its store has read it
                        tc::bulk_wait_read<1>();
                        issue_in(pf_item, pf_c, (k + 2) % NBUF);
                        next(pf_item, pf_c);
                    }
                }
            }
        }
        if (epi == EPI_LSE && row < a.M) {  // one (max, sumexp) partial per 128 columns
            float* p = a.part + ((long)row * a.n_parts + colh / 128) * 2;
            p[0] = lm;
            p[1] = ls;
        }
    }
    if (lane == 0) tc::bulk_wait<0>();
    __syncwarp();
}

template <int BN, int A_MN, int B_MN>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmO2,
              const __grid_constant__ CUtensorMap tmI, TcArgs a) {
    using C = Cfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* inbar = tempty + 2;  // [EPI_WARPS x NBUF]
    uint32_t* tbase_s = reinterpret_cast<uint32_t*>(inbar + NBUF * EPI_WARPS);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_items = a.tiles_m * a.tiles_n * a.splits;

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&tfull[s], 1);
            tc::mbar_init(&tempty[s], 32 * EPI_WARPS);
        }
        for (int s = 0; s < NBUF * EPI_WARPS; ++s) tc::mbar_init(&inbar[s], 1);
        tc::fence_barrier_init();
        tc::tma_prefetch(&tmA);
        tc::tma_prefetch(&tmB);
    }
    if (warp == 2) tc::tmem_alloc<2 * BN>(tbase_s);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tbase = *tbase_s;
    pdl_wait();  // operands come from the previous kernel
    pdl_trigger();

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer
        uint32_t cnt = 0;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
            const int mt = item % a.tiles_m, rest = item / a.tiles_m;
            const int nt = rest % a.tiles_n, sp = rest / a.tiles_n;
            const int kb0 = sp * a.kbs, kb1 = min(a.nkb, kb0 + a.kbs);
            for (int kb = kb0; kb < kb1; ++kb, ++cnt) {
                const int s = cnt % C::STAGES;
                const uint32_t ph = (cnt / C::STAGES) & 1;
                tc::mbar_wait(&empty[s], ph ^ 1);
                uint8_t* sa = smem + s * C::STAGE;
                uint8_t* sb = sa + C::A_BYTES;
                tc::mbar_expect_tx(&full[s], C::STAGE);
                if (!A_MN) {
                    tc::tma_load_2d(sa, &tmA, &full[s], kb * BK, mt * BM);
                } else {
                    tc::tma_load_2d(sa, &tmA, &full[s], mt * BM, kb * BK);
                    tc::tma_load_2d(sa + 8192, &tmA, &full[s], mt * BM + 64, kb * BK);
                }
                if (!B_MN) {
                    tc::tma_load_2d(sb, &tmB, &full[s], kb * BK, nt * BN);
                } else {
#pragma unroll
                    for (int q = 0; q < BN / 64; ++q) tc::tma_load_2d(sb + q * 8192, &tmB, &full[s], nt * BN + q * 64, kb * BK);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (whole warp; one elected lane issues)
        constexpr uint32_t idesc = tc::idesc_bf16(BM, BN, A_MN, B_MN);
        uint32_t cnt = 0, local = 0;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
            const int rest = item / a.tiles_m;
            const int sp = rest / a.tiles_n;
            const int kb0 = sp * a.kbs, kb1 = min(a.nkb, kb0 + a.kbs);
            const uint32_t acc = local & 1, use = local >> 1;
            tc::mbar_wait(&tempty[acc], (use & 1) ^ 1);
            tc::tc_fence_after();
            const uint32_t dcol = tbase + acc * BN;
            for (int kb = kb0; kb < kb1; ++kb, ++cnt) {
                const int s = cnt % C::STAGES;
                const uint32_t ph = (cnt / C::STAGES) & 1;
                tc::mbar_wait(&full[s], ph);
                tc::tc_fence_after();
                const uint32_t sa = tc::smem_u32(smem + s * C::STAGE);
                const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
                for (int ks = 0; ks < BK / 16; ++ks) {
                    const uint64_t ad = A_MN ? tc::sdesc(sa + ks * 2048, 8192, 1024) : tc::sdesc(sa + ks * 32, 16, 1024);
                    const uint64_t bd = B_MN ? tc::sdesc(sb + ks * 2048, 8192, 1024) : tc::sdesc(sb + ks * 32, 16, 1024);
                    tc::mma_bf16_e(dcol, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
                }
                tc::mma_commit_e(&empty[s]);
            }
            tc::mma_commit_e(&tfull[acc]);
        }
    } else if (warp >= 4) {
        const EpiSeq e{(int)blockIdx.x, (int)gridDim.x, n_items, a.tiles_m, BM, 0, n_items};
        epilogue_warps<BN>(&a, &tmO, &tmO2, &tmI, smem + C::STG_OFF, inbar, tfull, tbase, e,
                           [&](uint32_t acc) { tc::mbar_arrive_relaxed(&tempty[acc]); });
    }
    __syncthreads();
    if (warp == 2) {
        tc::tc_fence_after();
        tc::tmem_dealloc<2 * BN>(tbase);
    }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a 256 x 256 output tile per SM pair.  Each
// CTA loads its 128 rows of A and its 128 columns of B; the leader CTA issues
// tcgen05.mma.cta_group::2 (M = 256) which reads both CTAs' shared memory and
// writes each CTA's 128 accumulator rows into its own TMEM.  Per SM this halves
// the operand bytes per MMA cycle relative to the 1-CTA 128 x 256 tile.
constexpr int BN2 = 256;
// NB = tile width of the pair (256, or 224 for N = 896 / 2688-like problems so no
// half-empty tile column is computed); each CTA holds NB / 2 columns of B.
template <int NB>
struct Cfg2T {
    static constexpr int A_BYTES = BM * BK * 2;          // 128 rows of A
    static constexpr int B_BYTES = 128 * BK * 2;         // NB / 2 <= 128 columns of B (MN-major loads two 64-wide boxes)
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int STAGES = 4;
    static constexpr int STG_OFF = STAGES * STAGE;
    static constexpr int BAR_OFF = STG_OFF + EPI_SMEM;
    static constexpr int SMEM = BAR_OFF + 512 + 1024;
};
using Cfg2 = Cfg2T<256>;

template <int NP>
struct PairMaps {
    CUtensorMap a[NP], b[NP], o[NP], o2[NP], i[NP];
};
template <int NP>
struct PairArgs {
    TcArgs a[NP];
};

// NP equal-shape problems per launch (item = problem * tiles-per-problem + tile)
template <int A_MN, int B_MN, int NP, int NB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    k_gemm_tc2(const __grid_constant__ PairMaps<NP> mp, const __grid_constant__ PairArgs<NP> pa) {
    const TcArgs& a = pa.a[0];  // shape / K-split fields are common to the problems
    using C = Cfg2T<NB>;
    // expected bytes per stage and CTA: A + the B half actually transferred
    constexpr uint32_t STAGE_TX = C::A_BYTES + (B_MN ? 128 : NB / 2) * BK * 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* inbar = tempty + 2;  // [EPI_WARPS x NBUF]
    uint32_t* tbase_s = reinterpret_cast<uint32_t*>(inbar + NBUF * EPI_WARPS);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const int tiles_m2 = (a.M + 2 * BM - 1) / (2 * BM);
    const int tpp = tiles_m2 * a.tiles_n * a.splits;
    const int n_items = tpp * NP;

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&tfull[s], 1);
            tc::mbar_init(&tempty[s], 2 * 32 * EPI_WARPS);  // both CTAs' epilogue threads
        }
        for (int s = 0; s < NBUF * EPI_WARPS; ++s) tc::mbar_init(&inbar[s], 1);
        tc::fence_barrier_init();
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            tc::tma_prefetch(&mp.a[q]);
            tc::tma_prefetch(&mp.b[q]);
        }
    }
    if (warp == 2) tc::tmem_alloc_pair<512>(tbase_s);
    tc::tc_fence_before();
    __syncthreads();
    tc::cluster_sync();  // peer barriers initialised before any remote arrive / complete_tx
    tc::tc_fence_after();
    const uint32_t tbase = *tbase_s;
    pdl_wait();
    pdl_trigger();

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer (both CTAs, completing on the leader's barrier)
        const uint64_t pol_keep = tc::l2_evict_last_policy();
        uint32_t cnt = 0;
        for (int item = cid; item < n_items; item += ncl) {
            const int prob = item / tpp, t = item % tpp;
            const CUtensorMap* tA = &mp.a[prob];
            const CUtensorMap* tB = &mp.b[prob];
            const int mt = a.raster ? (t / a.tiles_n) % tiles_m2 : t % tiles_m2;
            const int nt = a.raster ? t % a.tiles_n : (t / tiles_m2) % a.tiles_n;
            const int sp = t / (tiles_m2 * a.tiles_n);
            const int kb0 = sp * a.kbs, kb1 = min(a.nkb, kb0 + a.kbs);
            const int m0 = mt * 2 * BM + (int)rank * BM, n0 = nt * NB + (int)rank * (NB / 2);
            for (int kb = kb0; kb < kb1; ++kb, ++cnt) {
                const int s = cnt % C::STAGES;
                const uint32_t ph = (cnt / C::STAGES) & 1;
                tc::mbar_wait(&empty[s], ph ^ 1);
                const uint32_t fb = tc::mapa(&full[s], 0);
                if (rank == 0) tc::mbar_expect_tx(&full[s], 2 * STAGE_TX);
                uint8_t* sa = smem + s * C::STAGE;
                uint8_t* sb = sa + C::A_BYTES;
                if (!A_MN) {
                    // m-fastest sweeps re-read all of A once per n-tile column: keep it in L2 (the LM head,
                    // where the 10 GB logits stream would otherwise evict it)
                    if (a.epi == EPI_LSE && !a.raster) tc::tma_load_2d_pair_hint(sa, tA, fb, kb * BK, m0, pol_keep);
                    else tc::tma_load_2d_pair(sa, tA, fb, kb * BK, m0);
                } else {
                    tc::tma_load_2d_pair(sa, tA, fb, m0, kb * BK);
                    tc::tma_load_2d_pair(sa + 8192, tA, fb, m0 + 64, kb * BK);
                }
                if (!B_MN) {
                    tc::tma_load_2d_pair(sb, tB, fb, kb * BK, n0);
                } else {
                    tc::tma_load_2d_pair(sb, tB, fb, n0, kb * BK);
                    tc::tma_load_2d_pair(sb + 8192, tB, fb, n0 + 64, kb * BK);
                }
            }
        }
    } else if (warp == 1 && rank == 0) {
        // ---------------- MMA issuer (leader CTA only; whole warp, one elected lane issues)
        constexpr uint32_t idesc = tc::idesc_bf16(2 * BM, NB, A_MN, B_MN);
        uint32_t cnt = 0, local = 0;
        for (int item = cid; item < n_items; item += ncl, ++local) {
            const int rest = (item % tpp) / tiles_m2;
            const int sp = rest / a.tiles_n;
            const int kb0 = sp * a.kbs, kb1 = min(a.nkb, kb0 + a.kbs);
            const uint32_t acc = local & 1, use = local >> 1;
            tc::mbar_wait(&tempty[acc], (use & 1) ^ 1);
            tc::tc_fence_after();
            const uint32_t dcol = tbase + acc * NB;
            for (int kb = kb0; kb < kb1; ++kb, ++cnt) {
                const int s = cnt % C::STAGES;
                const uint32_t ph = (cnt / C::STAGES) & 1;
                tc::mbar_wait(&full[s], ph);
                tc::tc_fence_after();
                const uint32_t sa = tc::smem_u32(smem + s * C::STAGE);
                const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
                for (int ks = 0; ks < BK / 16; ++ks) {
                    const uint64_t ad = A_MN ? tc::sdesc(sa + ks * 2048, 8192, 1024) : tc::sdesc(sa + ks * 32, 16, 1024);
                    const uint64_t bd = B_MN ? tc::sdesc(sb + ks * 2048, 8192, 1024) : tc::sdesc(sb + ks * 32, 16, 1024);
                    tc::mma_bf16_pair_e(dcol, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
                }
                tc::mma_commit_pair_e(&empty[s], 0x3);
            }
            tc::mma_commit_pair_e(&tfull[acc], 0x3);
        }
    } else if (warp >= 4) {
        // ---------------- epilogue (both CTAs: this CTA's 128 rows x all 256 columns)
        const EpiSeq e{cid, ncl, n_items, tiles_m2, 2 * BM, (int)rank, tpp};
        const uint32_t leader_tempty0 = tc::mapa(&tempty[0], 0);
        epilogue_warps<NB>(pa.a, mp.o, mp.o2, mp.i, smem + C::STG_OFF, inbar, tfull, tbase, e, [&](uint32_t acc) {
            tc::mbar_arrive_cluster_relaxed(leader_tempty0 + acc * 8);
        });
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::cluster_sync();
    if (warp == 2) {
        tc::tc_fence_after();
        tc::tmem_dealloc_pair<512>(tbase);
    }
}


// ---------------------------------------------------------------------------
// Grouped weight-gradient GEMM (CTA pair, A and B MN-major, K shared):
//   for each problem p:  C_p[M_p x N_p] += A_p^T B_p   (fp32, TMA reduce-add)
// One persistent launch covers all dW / db GEMMs of a layer, so the tile count
// fills the machine without split-K (every output element has exactly one
// writer: deterministic) and one problem's last wave overlaps the next's.
constexpr int GROUP_MAX = 8;
struct GroupMaps {
    CUtensorMap a[GROUP_MAX], b[GROUP_MAX], o[GROUP_MAX];
};
struct GroupArgs {
    int n_prob, nkb;
    int M[GROUP_MAX], tiles_m2[GROUP_MAX], tiles_n[GROUP_MAX], start[GROUP_MAX + 1];  // start: first pair-tile of p
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    k_gemm_group2(const __grid_constant__ GroupMaps mp, const __grid_constant__ GroupArgs g) {
    using C = Cfg2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tbase_s = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const int n_items = g.start[g.n_prob];
    // item -> (problem, m pair-tile, n tile)
    auto decode = [&](int item, int& p, int& mt, int& nt) {
        p = 0;
        while (p + 1 < g.n_prob && item >= g.start[p + 1]) ++p;
        const int t = item - g.start[p];
        mt = t % g.tiles_m2[p];
        nt = t / g.tiles_m2[p];
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&tfull[s], 1);
            tc::mbar_init(&tempty[s], 2 * 32 * EPI_WARPS);
        }
        tc::fence_barrier_init();
    }
    if (warp == 2) tc::tmem_alloc_pair<2 * BN2>(tbase_s);
    tc::tc_fence_before();
    __syncthreads();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tbase = *tbase_s;
    pdl_wait();
    pdl_trigger();

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer
        uint32_t cnt = 0;
        for (int item = cid; item < n_items; item += ncl) {
            int p, mt, nt;
            decode(item, p, mt, nt);
            const int m0 = mt * 2 * BM + (int)rank * BM, n0 = nt * BN2 + (int)rank * (BN2 / 2);
            for (int kb = 0; kb < g.nkb; ++kb, ++cnt) {
                const int s = cnt % C::STAGES;
                const uint32_t ph = (cnt / C::STAGES) & 1;
                tc::mbar_wait(&empty[s], ph ^ 1);
                const uint32_t fb = tc::mapa(&full[s], 0);
                if (rank == 0) tc::mbar_expect_tx(&full[s], 2 * C::STAGE);
                uint8_t* sa = smem + s * C::STAGE;
                uint8_t* sb = sa + C::A_BYTES;
                tc::tma_load_2d_pair(sa, &mp.a[p], fb, m0, kb * BK);
                tc::tma_load_2d_pair(sa + 8192, &mp.a[p], fb, m0 + 64, kb * BK);
                tc::tma_load_2d_pair(sb, &mp.b[p], fb, n0, kb * BK);
                tc::tma_load_2d_pair(sb + 8192, &mp.b[p], fb, n0 + 64, kb * BK);
            }
        }
    } else if (warp == 1 && rank == 0) {
        // ---------------- MMA issuer (leader CTA; whole warp, one elected lane issues)
        constexpr uint32_t idesc = tc::idesc_bf16(2 * BM, BN2, 1, 1);
        uint32_t cnt = 0, local = 0;
        for (int item = cid; item < n_items; item += ncl, ++local) {
            const uint32_t acc = local & 1, use = local >> 1;
            tc::mbar_wait(&tempty[acc], (use & 1) ^ 1);
            tc::tc_fence_after();
            const uint32_t dcol = tbase + acc * BN2;
            for (int kb = 0; kb < g.nkb; ++kb, ++cnt) {
                const int s = cnt % C::STAGES;
                const uint32_t ph = (cnt / C::STAGES) & 1;
                tc::mbar_wait(&full[s], ph);
                tc::tc_fence_after();
                const uint32_t sa = tc::smem_u32(smem + s * C::STAGE);
                const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
                for (int ks = 0; ks < BK / 16; ++ks)
                    tc::mma_bf16_pair_e(dcol, tc::sdesc(sa + ks * 2048, 8192, 1024), tc::sdesc(sb + ks * 2048, 8192, 1024),
                                      idesc, (kb > 0 || ks > 0) ? 1u : 0u);
                tc::mma_commit_pair_e(&empty[s], 0x3);
            }
            tc::mma_commit_pair_e(&tfull[acc], 0x3);
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: fp32 accumulator -> swizzled staging -> TMA reduce-add
        const int ew = warp & 3, half = (warp - 4) >> 2, wi = warp - 4;
        const uint32_t stg = tc::smem_u32(smem + C::STG_OFF + wi * NBUF * STG_BYTES);
        const uint32_t leader_tempty0 = tc::mapa(&tempty[0], 0);
        uint32_t k = 0, local = 0;
        for (int item = cid; item < n_items; item += ncl, ++local) {
            int p, mt, nt;
            decode(item, p, mt, nt);
            const uint32_t acc = local & 1, use = local >> 1;
            tc::mbar_wait(&tfull[acc], use & 1);
            tc::tc_fence_after();
            const int row0 = mt * 2 * BM + (int)rank * BM + ew * 32;
            const bool rows_live = row0 < g.M[p];
#pragma unroll 1
            for (int c = 0; c < 4; ++c, ++k) {
                const int col = nt * BN2 + half * 128 + c * 32;
                const uint32_t sb = stg + (k % NBUF) * STG_BYTES;
                float v[32];
                tc::tmem_ld32(tbase + acc * BN2 + half * 128 + c * 32 + ((uint32_t)(ew * 32) << 16), v);
                if (c == 3) {
                    tc::tc_fence_before();
                    tc::mbar_arrive_cluster_relaxed(leader_tempty0 + acc * 8);
                }
                if (!rows_live) continue;  // the whole 32-row slab is past M (e.g. beyond a bias row)
                if (lane == 0) tc::bulk_wait_read<NBUF - 1>();
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    tc::sts128(sb + sw128(lane, j), __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                               __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
                tc::fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tc::tma_reduce_add_2d(&mp.o[p], sb, col, row0);
                    tc::bulk_commit();
                }
            }
        }
        if (lane == 0) tc::bulk_wait<0>();
        __syncwarp();
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::cluster_sync();
    if (warp == 2) {
        tc::tc_fence_after();
        tc::tmem_dealloc_pair<2 * BN2>(tbase);
    }
}

__global__ void k_splitk_reduce(const float* __restrict__ ws, int splits, int M, int N, float* __restrict__ C, long ldc) {
    const long n = (long)M * N;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        float acc = 0.f;
        for (int s = 0; s < splits; ++s) acc += ws[(long)s * n + e];
        const int m = (int)(e / N), c = (int)(e % N);
        C[(long)m * ldc + c] += acc;
    }
}

// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// bf16 2D operand map: inner (contiguous) extent, outer extent, outer stride (elements), box.
bool make_map(CUtensorMap* m, const void* base, long inner, long outer, long stride_elems, int box_inner,
              int box_outer) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)stride_elems * 2};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Epilogue tile map: [rows x cols] (optionally x `planes`) row-major with row
// stride ld (elements); 32 x 32 boxes; fp32 rows use SWIZZLE_128B, bf16 rows
// SWIZZLE_64B (matching sw128 / sw64 in the epilogue).
bool make_epi_map(CUtensorMap* m, const void* base, bool f32, long cols, long rows, long ld, int planes = 1) {
    auto fn = encode_fn();
    if (!fn || !base || !aligned16(base)) return false;
    const int es = f32 ? 4 : 2;
    if ((ld * es) % 16) return false;
    cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)ld * es, (cuuint64_t)ld * es * rows};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t el[3] = {1, 1, 1};
    CUresult r = fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, planes > 1 ? 3 : 2,
                    const_cast<void*>(base), dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

struct Workspace {
    float* p = nullptr;
    size_t bytes = 0;
    float* get(size_t need) {
        if (need > bytes) {
            if (p) cudaFree(p);
            p = nullptr;
            if (cudaMalloc(&p, need) != cudaSuccess) {
                p = nullptr;
                bytes = 0;
                return nullptr;
            }
            bytes = need;
        }
        return p;
    }
};
Workspace g_ws;

struct Maps {
    CUtensorMap a, b, o, o2, i;
};

template <int BN, int A_MN, int B_MN>
void launch(const Maps& m, const TcArgs& a, int grid, cudaStream_t st) {
    auto k = k_gemm_tc<BN, A_MN, B_MN>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM);
        attr = true;
    }
    launch_pdl(k, dim3(grid), dim3(NTHREADS), Cfg<BN>::SMEM, st, m.a, m.b, m.o, m.o2, m.i, a);
    PARL_LAUNCHED();
}

template <int A_MN, int B_MN, int NP, int NB = 256>
void launch2(const Maps* m, const TcArgs* a, int grid, cudaStream_t st) {
    auto k = k_gemm_tc2<A_MN, B_MN, NP, NB>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2T<NB>::SMEM);
        attr = true;
    }
    PairMaps<NP> pm;
    PairArgs<NP> pa;
    for (int q = 0; q < NP; ++q) {
        pm.a[q] = m[q].a; pm.b[q] = m[q].b; pm.o[q] = m[q].o; pm.o2[q] = m[q].o2; pm.i[q] = m[q].i;
        pa.a[q] = a[q];
    }
    launch_pdl(k, dim3(grid), dim3(NTHREADS), Cfg2T<NB>::SMEM, st, pm, pa);
}

// PARL_GEMM_PAIR=0 disables the CTA-pair kernel (diagnostics)
bool pair_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("PARL_GEMM_PAIR");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

}  // namespace

// C_p += A_p^T B_p for every problem (A_p: [K x M_p], B_p: [K x N_p] bf16 row-major,
// i.e. MN-major operands; C_p fp32 [M_p x N_p] with row stride ldc_p).  All
// problems share K.  Returns false when a problem is unsupported (the caller
// then runs them one by one).
bool gemm_tc_group_dw(const GemmArgs* gs, int n, cudaStream_t st) {
    if (n <= 0 || n > GROUP_MAX || !pair_enabled() || !encode_fn()) return false;
    static GroupMaps maps;  // host staging of the kernel parameter (copied at launch)
    GroupArgs ga{};
    ga.n_prob = n;
    const int K = gs[0].K;
    ga.nkb = (K + BK - 1) / BK;
    int tiles = 0;
    for (int p = 0; p < n; ++p) {
        const GemmArgs& g = gs[p];
        if (g.K != K || g.sam != 1 || g.sbn != 1 || g.epi != EPI_F32_ACC || g.N % 128 != 0) return false;
        if ((g.sak * 2) % 16 || (g.sbk * 2) % 16 || !aligned16(g.A) || !aligned16(g.B)) return false;
        if (!make_map(&maps.a[p], g.A, g.M, g.K, g.sak, 64, BK)) return false;
        if (!make_map(&maps.b[p], g.B, g.N, g.K, g.sbk, 64, BK)) return false;
        if (!make_epi_map(&maps.o[p], g.Cf, true, g.N, g.M, g.ldc)) return false;
        ga.M[p] = g.M;
        ga.tiles_m2[p] = (g.M + 2 * BM - 1) / (2 * BM);
        ga.tiles_n[p] = (g.N + BN2 - 1) / BN2;
        ga.start[p] = tiles;
        tiles += ga.tiles_m2[p] * ga.tiles_n[p];
    }
    ga.start[n] = tiles;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_gemm_group2, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2::SMEM);
        attr = true;
    }
    const int grid = 2 * std::min(tiles, num_sms() / 2);
    launch_pdl(k_gemm_group2, dim3(grid), dim3(NTHREADS), Cfg2::SMEM, st, maps, ga);
    PARL_LAUNCHED();
    return true;
}

namespace {
// Launch plan of one GEMM: kernel variant, tiling, tensor maps, device args.
struct Plan {
    bool pair = false;
    int BN = 256, variant = 0, items = 0;  // variant: 0 K/K, 1 K/MN, 2 MN/MN; BN: tile width (pair: 256 or 224)
    Maps mp;
    TcArgs a{};
    float* ws = nullptr;
};

// false if the shape / layout is not supported by the tcgen05 kernels
bool plan_gemm(const GemmArgs& g, Plan& P) {
    const bool a_k = g.sak == 1, a_mn = g.sam == 1 && !a_k;
    const bool b_k = g.sbk == 1, b_mn = g.sbn == 1 && !b_k;
    if (!(a_k || a_mn) || !(b_k || b_mn)) return false;
    const long lda = a_k ? g.sam : g.sak, ldb = b_k ? g.sbn : g.sbk;
    if ((lda * 2) % 16 || (ldb * 2) % 16 || !aligned16(g.A) || !aligned16(g.B)) return false;
    if (a_mn && !b_mn) return false;  // combination not instantiated
    if (!encode_fn()) return false;
    P.variant = a_k && b_k ? 0 : (a_k ? 1 : 2);

    // tile width: 128 when N is a multiple of 128 but not of 256, or N is small
    // (the LSE epilogue writes one (max, sumexp) partial per 128 columns: n_parts = ceil(N / 128))
    // CTA pair (256 x 256 tiles) when the problem has enough of them; N must be a
    // multiple of 128 so each CTA's half-tile of B is full-width aligned.
    const int sms = num_sms();
    const bool pair = pair_enabled() && g.M > 128 && g.N >= 256 && (g.N % 128) == 0 &&
                      (long)((g.M + 255) / 256) * ((g.N + 255) / 256) >= sms / 4 && (a_k || b_mn);
    // pair tiles are 224 wide when that covers N exactly and 256 does not (N = 896, 2688, ...)
    const int NB = (g.N % 256 != 0 && g.N % 224 == 0 && g.epi != EPI_LSE) ? 224 : 256;
    const int BN = pair ? NB : (g.epi == EPI_LSE ? 256 : ((g.N % 256 != 0 && g.N % 128 == 0) || g.N <= 128 ? 128 : 256));
    P.pair = pair;
    P.BN = BN;
    Maps& mp = P.mp;
    std::memset(&mp, 0, sizeof(mp));
    bool ok;
    if (a_k) ok = make_map(&mp.a, g.A, g.K, g.M, lda, BK, BM);
    else ok = make_map(&mp.a, g.A, g.M, g.K, lda, 64, BK);
    if (!ok) return false;
    const int bbox = pair ? BN / 2 : BN;  // rows of B per CTA
    if (b_k) ok = make_map(&mp.b, g.B, g.K, g.N, ldb, BK, bbox);
    else ok = make_map(&mp.b, g.B, g.N, g.K, ldb, 64, BK);
    if (!ok) return false;

    TcArgs& a = P.a;
    a = TcArgs{};
    a.M = g.M; a.N = g.N; a.K = g.K;
    a.nkb = (g.K + BK - 1) / BK;
    a.tiles_m = (g.M + BM - 1) / BM;
    a.tiles_n = (g.N + BN - 1) / BN;
    a.epi = g.epi;
    a.bias = g.bias;
    a.bias_vec = g.bias && aligned16(g.bias);
    a.labels = g.labels; a.part = g.part; a.target = g.target;
    a.n_parts = g.n_parts;
    a.store_logits = g.logits_act != nullptr;
    const int tiles = pair ? ((g.M + 255) / 256) * a.tiles_n : a.tiles_m * a.tiles_n;
    // n-fastest tile order when the N-side operand is small (weights: it stays in L2 while the
    // concurrently running tiles share each A row block, so A streams from HBM once); else
    // m-fastest (the LM head's 270 MB weight would be re-read per m block).  PARL_GEMM_RASTER=0/1
    static const int raster_env = [] {
        const char* e = getenv("PARL_GEMM_RASTER");
        return e ? atoi(e) : -1;
    }();
    const double b_bytes = (double)g.N * g.K * 2, a_bytes = (double)g.M * g.K * 2;
    a.raster = pair && (raster_env >= 0 ? raster_env == 1 : (b_bytes <= 16e6 && a_bytes >= b_bytes));
    a.splits = 1;
    a.kbs = a.nkb;
    const int slots = pair ? sms / 2 : sms;  // concurrently running tiles
    if (g.epi == EPI_F32_ACC && tiles < slots && a.nkb >= 4) {
        int want = std::min((slots + tiles - 1) / tiles, a.nkb / 2);
        want = std::max(want, 1);
        a.kbs = (a.nkb + want - 1) / want;
        a.splits = (a.nkb + a.kbs - 1) / a.kbs;
    }
    P.ws = nullptr;
    if (a.splits > 1) {
        P.ws = g_ws.get((size_t)a.splits * g.M * g.N * sizeof(float));
        if (!P.ws) return false;
    }
    // epilogue maps
    switch (g.epi) {
        case EPI_F32:
            ok = make_epi_map(&mp.o, g.Cf, true, g.N, g.M, g.ldc);
            break;
        case EPI_F32_ACC:
            ok = a.splits > 1 ? make_epi_map(&mp.o, P.ws, true, g.N, g.M, g.N, a.splits)
                              : make_epi_map(&mp.o, g.Cf, true, g.N, g.M, g.ldc);
            break;
        case EPI_RESID:
            ok = make_epi_map(&mp.o, g.Cf, true, g.N, g.M, g.ldc) && make_epi_map(&mp.i, g.resid, true, g.N, g.M, g.ldc);
            break;
        case EPI_ACT:
            ok = make_epi_map(&mp.o, g.Ca, false, g.N, g.M, g.ldca);
            break;
        case EPI_GELU:
            ok = make_epi_map(&mp.o, g.Ca, false, g.N, g.M, g.ldca) && make_epi_map(&mp.o2, g.Caux, false, g.N, g.M, g.ldca);
            break;
        case EPI_GELU_ACT:
            ok = make_epi_map(&mp.o, g.Ca, false, g.N, g.M, g.ldca);
            break;
        case EPI_GELU_BWD:
            ok = make_epi_map(&mp.o, g.Ca, false, g.N, g.M, g.ldca) &&
                 make_epi_map(&mp.i, g.aux_in, false, g.N, g.M, g.ldca);
            break;
        case EPI_LSE:
            ok = true;
            if (g.logits_act && !make_epi_map(&mp.o, g.logits_act, false, g.N, g.M, g.ldca)) {
                a.store_logits = 0;
                a.logits_direct = static_cast<bf16*>(g.logits_act);
                a.ldl = g.ldca;
            }
            break;
        default:
            ok = false;
    }
    if (!ok) return false;
    P.items = tiles * a.splits;
    return true;
}

void run_plan(const Plan& P, const GemmArgs& g, cudaStream_t st) {
    const int sms = num_sms();
    const int v = P.variant;
    if (P.pair) {
        const int grid = 2 * std::min(P.items, sms / 2);
        if (P.BN == 224) {
            if (v == 0) launch2<0, 0, 1, 224>(&P.mp, &P.a, grid, st);
            else if (v == 1) launch2<0, 1, 1, 224>(&P.mp, &P.a, grid, st);
            else launch2<1, 1, 1, 224>(&P.mp, &P.a, grid, st);
        } else {
            if (v == 0) launch2<0, 0, 1>(&P.mp, &P.a, grid, st);
            else if (v == 1) launch2<0, 1, 1>(&P.mp, &P.a, grid, st);
            else launch2<1, 1, 1>(&P.mp, &P.a, grid, st);
        }
    } else if (P.BN == 256) {
        const int grid = std::min(P.items, sms);
        if (v == 0) launch<256, 0, 0>(P.mp, P.a, grid, st);
        else if (v == 1) launch<256, 0, 1>(P.mp, P.a, grid, st);
        else launch<256, 1, 1>(P.mp, P.a, grid, st);
    } else {
        const int grid = std::min(P.items, sms);
        if (v == 0) launch<128, 0, 0>(P.mp, P.a, grid, st);
        else if (v == 1) launch<128, 0, 1>(P.mp, P.a, grid, st);
        else launch<128, 1, 1>(P.mp, P.a, grid, st);
    }
    if (P.a.splits > 1) {
        const long n = (long)g.M * g.N;
        const int blocks = (int)std::min<long>((n + 255) / 256, 148L * 8);
        k_splitk_reduce<<<blocks, 256, 0, st>>>(P.ws, P.a.splits, g.M, g.N, g.Cf, g.ldc);
        PARL_LAUNCHED();
    }
}
}  // namespace

bool gemm_tc(const GemmArgs& g, cudaStream_t st) {
    if (g.M <= 0 || g.N <= 0 || g.K <= 0) return true;
    Plan P;
    if (!plan_gemm(g, P)) return false;
    run_plan(P, g, st);
    return true;
}

// Equal-shape GEMMs (the three models' copies of one layer GEMM) in one CTA-pair
// launch; falls back to one launch per problem when they cannot be grouped.
bool gemm_tc_multi(const GemmArgs* gs, int n, cudaStream_t st) {
    if (n <= 0) return true;
    static Plan P[3];
    bool group = (n == 2 || n == 3) && pair_enabled();
    for (int q = 0; q < n; ++q) {
        if (gs[q].M <= 0 || gs[q].N <= 0 || gs[q].K <= 0) return n == 1;
        if (!plan_gemm(gs[q], P[q < 3 ? q : 0])) return false;
        if (q >= 3) group = false;
    }
    if (group) {
        for (int q = 0; q < n; ++q)
            group = group && P[q].pair && P[q].a.splits == 1 && P[q].variant == P[0].variant && P[q].BN == P[0].BN &&
                    P[q].a.M == P[0].a.M && P[q].a.N == P[0].a.N && P[q].a.K == P[0].a.K &&
                    P[q].a.store_logits == P[0].a.store_logits && P[q].a.logits_direct == nullptr &&
                    ((P[q].a.epi == EPI_RESID || P[q].a.epi == EPI_GELU_BWD) ==
                     (P[0].a.epi == EPI_RESID || P[0].a.epi == EPI_GELU_BWD));
    }
    if (!group) {
        for (int q = 0; q < n; ++q) {
            if (q >= 3 && !plan_gemm(gs[q], P[0])) return false;
            run_plan(P[q < 3 ? q : 0], gs[q], st);
        }
        return true;
    }
    Maps m3[3] = {P[0].mp, P[1].mp, P[2].mp};
    TcArgs a3[3] = {P[0].a, P[1].a, P[2].a};
    const int grid = 2 * std::min(n * P[0].items, num_sms() / 2);
    const int v = P[0].variant;
    if (n == 3 && P[0].BN == 224) {
        if (v == 0) launch2<0, 0, 3, 224>(m3, a3, grid, st);
        else if (v == 1) launch2<0, 1, 3, 224>(m3, a3, grid, st);
        else launch2<1, 1, 3, 224>(m3, a3, grid, st);
    } else if (n == 3) {
        if (v == 0) launch2<0, 0, 3>(m3, a3, grid, st);
        else if (v == 1) launch2<0, 1, 3>(m3, a3, grid, st);
        else launch2<1, 1, 3>(m3, a3, grid, st);
    } else if (P[0].BN == 224) {
        if (v == 0) launch2<0, 0, 2, 224>(m3, a3, grid, st);
        else if (v == 1) launch2<0, 1, 2, 224>(m3, a3, grid, st);
        else launch2<1, 1, 2, 224>(m3, a3, grid, st);
    } else {
        if (v == 0) launch2<0, 0, 2>(m3, a3, grid, st);
        else if (v == 1) launch2<0, 1, 2>(m3, a3, grid, st);
        else launch2<1, 1, 2>(m3, a3, grid, st);
    }
    return true;
}

}  // namespace parl_gpu
