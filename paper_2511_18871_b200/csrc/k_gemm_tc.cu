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

#include <mutex>

#include "internal.cuh"
#include "tc_util.cuh"

namespace parl_gpu {

namespace {

constexpr int BM = 128, BK = 64;
constexpr int EPI_WARPS = 8;                      // two per TMEM lane quadrant, each half the columns
constexpr int NTHREADS = 128 + 32 * EPI_WARPS;    // warps 0-3 producer/MMA/TMEM/spare, 4.. epilogue

struct TcArgs {
    int M, N, K, nkb, tiles_m, tiles_n, splits, kbs, epi, vec_ok;
    const float* bias;
    float* Cf;
    long ldc;
    const float* resid;
    bf16* Ca;
    long ldca;
    bf16* Caux;
    const bf16* aux_in;
    const int32_t* labels;
    float* part;
    float* target;
    bf16* logits_act;
    int n_parts;
    float* ws;  // split-K partials [splits x M x N]
};

template <int BN>
struct Cfg {
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int STAGES = BN == 256 ? 4 : 6;
    static constexpr int EPI_OFF = STAGES * STAGE + 256;                  // after the barriers
    static constexpr int SMEM = EPI_OFF + EPI_WARPS * 32 * 33 * 4 + 1024;  // + per-warp epilogue tiles + align
};

// Phi(x) = 0.5 (1 + erf(x / sqrt 2)) with Abramowitz-Stegun 7.1.26 (|erf err| <= 1.5e-7,
// far below the bf16 rounding of the outputs); returns exp(-x^2/2) for GELU' too.
__device__ __forceinline__ float phi_fast(float x, float& e) {
    const float z = fabsf(x) * 0.70710678118654752f;
    const float t = __frcp_rn(fmaf(0.3275911f, z, 1.f));
    e = __expf(-z * z);
    const float poly = t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 1.061405429f, -1.453152027f), 1.421413741f), -0.284496736f),
                                0.254829592f);
    const float erf_abs = 1.f - poly * e;
    return 0.5f * (1.f + copysignf(erf_abs, x));
}
__device__ __forceinline__ float gelu_dev(float x) {  // x * Phi(x)  (model.cpp:255)
    float e;
    return x * phi_fast(x, e);
}
__device__ __forceinline__ float gelu_grad_dev(float x) {  // Phi(x) + x phi(x)  (model.cpp:257-260)
    float e;
    const float p = phi_fast(x, e);
    return p + x * 0.39894228040143267794f * e;
}

// Epilogue of one 32-row x 32-column chunk.  v[] arrives in the TMEM layout
// (lane = tile row).  Element-wise epilogues are transposed through a padded
// per-warp smem tile so that lane = column and every global access is a
// coalesced row segment; the LSE epilogue reduces along its own row first.
__device__ __forceinline__ void epilogue_chunk(const TcArgs& a, int row0, int col0, float* v, int split,
                                               float* sm /* [32][33] */, float& lse_m, float& lse_s, int label) {
    const int lane = threadIdx.x & 31;
    const int row = row0 + lane;
    if (a.epi == EPI_LSE) {
        const int ncol = min(32, a.N - col0);
        if (row < a.M && ncol > 0) {
            float cm = -INFINITY;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                v[j] += (j < ncol && a.bias) ? a.bias[col0 + j] : 0.f;
                if (j < ncol) cm = fmaxf(cm, v[j]);
            }
            const float nm = fmaxf(lse_m, cm);
            float s = lse_s * __expf(lse_m - nm);
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (j < ncol) s += __expf(v[j] - nm);
            lse_m = nm;
            lse_s = s;
            const int lj = label - col0;
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (j == lj) a.target[row] = v[j];
        }
        if (!a.logits_act) return;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) sm[lane * 33 + j] = v[j];
    __syncwarp();
    const int col = col0 + lane;
    if (col < a.N) {
        const float b = (a.bias && a.epi != EPI_LSE) ? a.bias[col] : 0.f;
        const int rmax = min(32, a.M - row0);
        switch (a.epi) {
            case EPI_F32:
                for (int r = 0; r < rmax; ++r) a.Cf[(long)(row0 + r) * a.ldc + col] = sm[r * 33 + lane] + b;
                break;
            case EPI_F32_ACC:
                if (a.splits > 1) {
                    for (int r = 0; r < rmax; ++r)
                        a.ws[((long)split * a.M + row0 + r) * a.N + col] = sm[r * 33 + lane];
                } else {
                    // batch the loads first: stores may alias, so the compiler
                    // would otherwise serialise every load behind a store
#pragma unroll
                    for (int h = 0; h < 32; h += 16) {
                        float old[16];
#pragma unroll
                        for (int r = 0; r < 16; ++r)
                            old[r] = h + r < rmax ? a.Cf[(long)(row0 + h + r) * a.ldc + col] : 0.f;
#pragma unroll
                        for (int r = 0; r < 16; ++r)
                            if (h + r < rmax)
                                a.Cf[(long)(row0 + h + r) * a.ldc + col] = old[r] + sm[(h + r) * 33 + lane];
                    }
                }
                break;
            case EPI_ACT:
                for (int r = 0; r < rmax; ++r)
                    a.Ca[(long)(row0 + r) * a.ldca + col] = __float2bfloat16_rn(sm[r * 33 + lane] + b);
                break;
            case EPI_RESID: {
#pragma unroll
                for (int h = 0; h < 32; h += 16) {
                    float rv[16];
#pragma unroll
                    for (int r = 0; r < 16; ++r)
                        rv[r] = h + r < rmax ? a.resid[(long)(row0 + h + r) * a.ldc + col] : 0.f;
#pragma unroll
                    for (int r = 0; r < 16; ++r)
                        if (h + r < rmax) a.Cf[(long)(row0 + h + r) * a.ldc + col] = rv[r] + (sm[(h + r) * 33 + lane] + b);
                }
                break;
            }
            case EPI_GELU:
                for (int r = 0; r < rmax; ++r) {
                    const long o = (long)(row0 + r) * a.ldca + col;
                    const bf16 u = __float2bfloat16_rn(sm[r * 33 + lane] + b);
                    a.Ca[o] = u;
                    a.Caux[o] = __float2bfloat16_rn(gelu_dev(__bfloat162float(u)));
                }
                break;
            case EPI_GELU_BWD: {
#pragma unroll
                for (int h = 0; h < 32; h += 16) {
                    bf16 uv[16];
#pragma unroll
                    for (int r = 0; r < 16; ++r)
                        uv[r] = h + r < rmax ? a.aux_in[(long)(row0 + h + r) * a.ldca + col] : __float2bfloat16_rn(0.f);
#pragma unroll
                    for (int r = 0; r < 16; ++r)
                        if (h + r < rmax)
                            a.Ca[(long)(row0 + h + r) * a.ldca + col] =
                                __float2bfloat16_rn(sm[(h + r) * 33 + lane] * gelu_grad_dev(__bfloat162float(uv[r])));
                }
                break;
            }
            case EPI_LSE:
                for (int r = 0; r < rmax; ++r)
                    a.logits_act[(long)(row0 + r) * a.ldca + col] = __float2bfloat16_rn(sm[r * 33 + lane]);
                break;
            default:
                break;
        }
    }
    __syncwarp();
}

template <int BN, int A_MN, int B_MN>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcArgs a) {
    using C = Cfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tbase_s = reinterpret_cast<uint32_t*>(tempty + 2);

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
        tc::fence_barrier_init();
        tc::tma_prefetch(&tmA);
        tc::tma_prefetch(&tmB);
    }
    if (warp == 2) tc::tmem_alloc<2 * BN>(tbase_s);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tbase = *tbase_s;

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
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer
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
                    tc::mma_bf16(dcol, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
                }
                tc::mma_commit(&empty[s]);
            }
            tc::mma_commit(&tfull[acc]);
        }
    } else if (warp >= 4) {
        // ---------------- epilogue
        const int ew = warp & 3;           // TMEM lane quadrant (a warp may only touch lanes 32*(warp%4)..)
        const int half = (warp - 4) >> 2;  // which half of the tile's columns
        float* esm = reinterpret_cast<float*>(smem + C::EPI_OFF) + (warp - 4) * 32 * 33;
        uint32_t local = 0;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
            const int mt = item % a.tiles_m, rest = item / a.tiles_m;
            const int nt = rest % a.tiles_n, sp = rest / a.tiles_n;
            const uint32_t acc = local & 1, use = local >> 1;
            tc::mbar_wait(&tfull[acc], use & 1);
            tc::tc_fence_after();
            const int row0 = mt * BM + ew * 32, row = row0 + lane;
            const int label = (a.epi == EPI_LSE && row < a.M) ? a.labels[row] : -1;
            float lm = -INFINITY, ls = 0.f;
            constexpr int HALF = BN / 2;
#pragma unroll 1
            for (int c = 0; c < HALF / 32; ++c) {
                float v[32];
                const int col = half * HALF + c * 32;
                tc::tmem_ld32(tbase + acc * BN + col + ((uint32_t)(ew * 32) << 16), v);
                epilogue_chunk(a, row0, nt * BN + col, v, sp, esm, lm, ls, label);
            }
            if (a.epi == EPI_LSE && row < a.M) {  // partials per 128 columns
                float* p = a.part + ((long)row * a.n_parts + (nt * BN + half * HALF) / 128) * 2;
                p[0] = lm;
                p[1] = ls;
            }
            tc::tc_fence_before();
            tc::mbar_arrive_relaxed(&tempty[acc]);
        }
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
// the operand bytes per MMA cycle relative to the 1-CTA 128 x 256 tile, so the
// 6-stage ring covers the TMA latency.
constexpr int BN2 = 256;
struct Cfg2 {
    static constexpr int A_BYTES = BM * BK * 2;          // 128 rows of A
    static constexpr int B_BYTES = (BN2 / 2) * BK * 2;   // 128 columns of B
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int STAGES = 6;
    static constexpr int EPI_OFF = STAGES * STAGE + 256;
    static constexpr int SMEM = EPI_OFF + EPI_WARPS * 32 * 33 * 4 + 1024;
};

template <int A_MN, int B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    k_gemm_tc2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcArgs a) {
    using C = Cfg2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tbase_s = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const int tiles_m2 = (a.M + 2 * BM - 1) / (2 * BM);
    const int n_items = tiles_m2 * a.tiles_n * a.splits;

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&tfull[s], 1);
            tc::mbar_init(&tempty[s], 2 * 32 * EPI_WARPS);  // both CTAs' epilogue threads
        }
        tc::fence_barrier_init();
        tc::tma_prefetch(&tmA);
        tc::tma_prefetch(&tmB);
    }
    if (warp == 2) tc::tmem_alloc_pair<2 * BN2>(tbase_s);
    tc::tc_fence_before();
    __syncthreads();
    tc::cluster_sync();  // peer barriers initialised before any remote arrive / complete_tx
    tc::tc_fence_after();
    const uint32_t tbase = *tbase_s;

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer (both CTAs, completing on the leader's barrier)
        uint32_t cnt = 0;
        for (int item = cid; item < n_items; item += ncl) {
            const int mt = item % tiles_m2, rest = item / tiles_m2;
            const int nt = rest % a.tiles_n, sp = rest / a.tiles_n;
            const int kb0 = sp * a.kbs, kb1 = min(a.nkb, kb0 + a.kbs);
            const int m0 = mt * 2 * BM + (int)rank * BM, n0 = nt * BN2 + (int)rank * (BN2 / 2);
            for (int kb = kb0; kb < kb1; ++kb, ++cnt) {
                const int s = cnt % C::STAGES;
                const uint32_t ph = (cnt / C::STAGES) & 1;
                tc::mbar_wait(&empty[s], ph ^ 1);
                const uint32_t fb = tc::mapa(&full[s], 0);
                if (rank == 0) tc::mbar_expect_tx(&full[s], 2 * C::STAGE);
                uint8_t* sa = smem + s * C::STAGE;
                uint8_t* sb = sa + C::A_BYTES;
                if (!A_MN) {
                    tc::tma_load_2d_pair(sa, &tmA, fb, kb * BK, m0);
                } else {
                    tc::tma_load_2d_pair(sa, &tmA, fb, m0, kb * BK);
                    tc::tma_load_2d_pair(sa + 8192, &tmA, fb, m0 + 64, kb * BK);
                }
                if (!B_MN) {
                    tc::tma_load_2d_pair(sb, &tmB, fb, kb * BK, n0);
                } else {
                    tc::tma_load_2d_pair(sb, &tmB, fb, n0, kb * BK);
                    tc::tma_load_2d_pair(sb + 8192, &tmB, fb, n0 + 64, kb * BK);
                }
            }
        }
    } else if (warp == 1 && lane == 0 && rank == 0) {
        // ---------------- MMA issuer (leader CTA only)
        constexpr uint32_t idesc = tc::idesc_bf16(2 * BM, BN2, A_MN, B_MN);
        uint32_t cnt = 0, local = 0;
        for (int item = cid; item < n_items; item += ncl, ++local) {
            const int rest = item / tiles_m2;
            const int sp = rest / a.tiles_n;
            const int kb0 = sp * a.kbs, kb1 = min(a.nkb, kb0 + a.kbs);
            const uint32_t acc = local & 1, use = local >> 1;
            tc::mbar_wait(&tempty[acc], (use & 1) ^ 1);
            tc::tc_fence_after();
            const uint32_t dcol = tbase + acc * BN2;
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
                    tc::mma_bf16_pair(dcol, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
                }
                tc::mma_commit_pair(&empty[s], 0x3);
            }
            tc::mma_commit_pair(&tfull[acc], 0x3);
        }
    } else if (warp >= 4) {
        // ---------------- epilogue (both CTAs: this CTA's 128 rows x all 256 columns)
        const int ew = warp & 3;
        const int half = (warp - 4) >> 2;
        float* esm = reinterpret_cast<float*>(smem + C::EPI_OFF) + (warp - 4) * 32 * 33;
        uint32_t local = 0;
        for (int item = cid; item < n_items; item += ncl, ++local) {
            const int mt = item % tiles_m2, rest = item / tiles_m2;
            const int nt = rest % a.tiles_n, sp = rest / a.tiles_n;
            const uint32_t acc = local & 1, use = local >> 1;
            tc::mbar_wait(&tfull[acc], use & 1);
            tc::tc_fence_after();
            const int row0 = mt * 2 * BM + (int)rank * BM + ew * 32, row = row0 + lane;
            const int label = (a.epi == EPI_LSE && row < a.M) ? a.labels[row] : -1;
            float lm = -INFINITY, ls = 0.f;
            constexpr int HALF = BN2 / 2;
#pragma unroll 1
            for (int c = 0; c < HALF / 32; ++c) {
                float v[32];
                const int col = half * HALF + c * 32;
                tc::tmem_ld32(tbase + acc * BN2 + col + ((uint32_t)(ew * 32) << 16), v);
                epilogue_chunk(a, row0, nt * BN2 + col, v, sp, esm, lm, ls, label);
            }
            if (a.epi == EPI_LSE && row < a.M) {
                float* p = a.part + ((long)row * a.n_parts + (nt * BN2 + half * HALF) / 128) * 2;
                p[0] = lm;
                p[1] = ls;
            }
            tc::tc_fence_before();
            tc::mbar_arrive_cluster_relaxed(tc::mapa(&tempty[acc], 0));
        }
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

// bf16 2D map: inner (contiguous) extent, outer extent, outer stride (elements), box.
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

template <int BN, int A_MN, int B_MN>
void launch(const CUtensorMap& ma, const CUtensorMap& mb, const TcArgs& a, int grid, cudaStream_t st) {
    auto k = k_gemm_tc<BN, A_MN, B_MN>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM);
        attr = true;
    }
    k<<<grid, NTHREADS, Cfg<BN>::SMEM, st>>>(ma, mb, a);
    PARL_LAUNCHED();
}

template <int A_MN, int B_MN>
void launch2(const CUtensorMap& ma, const CUtensorMap& mb, const TcArgs& a, int grid, cudaStream_t st) {
    auto k = k_gemm_tc2<A_MN, B_MN>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2::SMEM);
        attr = true;
    }
    k<<<grid, NTHREADS, Cfg2::SMEM, st>>>(ma, mb, a);
    PARL_LAUNCHED();
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

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

bool gemm_tc(const GemmArgs& g, cudaStream_t st) {
    if (g.M <= 0 || g.N <= 0 || g.K <= 0) return true;
    const bool a_k = g.sak == 1, a_mn = g.sam == 1 && !a_k;
    const bool b_k = g.sbk == 1, b_mn = g.sbn == 1 && !b_k;
    if (!(a_k || a_mn) || !(b_k || b_mn)) return false;
    const long lda = a_k ? g.sam : g.sak, ldb = b_k ? g.sbn : g.sbk;
    if ((lda * 2) % 16 || (ldb * 2) % 16 || !aligned16(g.A) || !aligned16(g.B)) return false;
    if (a_mn && !b_mn) return false;  // combination not instantiated
    if (!encode_fn()) return false;

    // tile width: 128 when N is a multiple of 128 but not of 256, or N is small
    // (the LSE epilogue writes one (max, sumexp) partial per 128 columns: n_parts = ceil(N / 128))
    // CTA pair (256 x 256 tiles) when the problem has enough of them; N must be a
    // multiple of 128 so each CTA's half-tile of B is full-width aligned.
    const int sms0 = num_sms();
    const bool pair = pair_enabled() && g.M > 128 && g.N >= 256 && (g.N % 128) == 0 &&
                      (long)((g.M + 255) / 256) * ((g.N + 255) / 256) >= sms0 / 4 && (a_k || b_mn);
    const int BN = pair ? 256 : (g.epi == EPI_LSE ? 256 : ((g.N % 256 != 0 && g.N % 128 == 0) || g.N <= 128 ? 128 : 256));
    CUtensorMap ma, mb;
    bool ok;
    if (a_k) ok = make_map(&ma, g.A, g.K, g.M, lda, BK, BM);
    else ok = make_map(&ma, g.A, g.M, g.K, lda, 64, BK);
    if (!ok) return false;
    const int bbox = pair ? BN / 2 : BN;  // rows of B per CTA
    if (b_k) ok = make_map(&mb, g.B, g.K, g.N, ldb, BK, bbox);
    else ok = make_map(&mb, g.B, g.N, g.K, ldb, 64, BK);
    if (!ok) return false;

    TcArgs a{};
    a.M = g.M; a.N = g.N; a.K = g.K;
    a.nkb = (g.K + BK - 1) / BK;
    a.tiles_m = (g.M + BM - 1) / BM;
    a.tiles_n = (g.N + BN - 1) / BN;
    a.epi = g.epi;
    a.bias = g.bias; a.Cf = g.Cf; a.ldc = g.ldc; a.resid = g.resid;
    a.Ca = static_cast<bf16*>(g.Ca); a.ldca = g.ldca; a.Caux = static_cast<bf16*>(g.Caux);
    a.aux_in = static_cast<const bf16*>(g.aux_in);
    a.labels = g.labels; a.part = g.part; a.target = g.target;
    a.logits_act = static_cast<bf16*>(g.logits_act);
    a.n_parts = g.n_parts;
    const int sms = num_sms();
    const int tiles = pair ? ((g.M + 255) / 256) * a.tiles_n : a.tiles_m * a.tiles_n;
    a.splits = 1;
    a.kbs = a.nkb;
    const int slots = pair ? sms / 2 : sms;  // concurrently running tiles
    if (g.epi == EPI_F32_ACC && tiles < slots && a.nkb >= 4) {
        int want = std::min((slots + tiles - 1) / tiles, a.nkb / 2);
        want = std::max(want, 1);
        a.kbs = (a.nkb + want - 1) / want;
        a.splits = (a.nkb + a.kbs - 1) / a.kbs;
        if (a.splits > 1) {
            a.ws = g_ws.get((size_t)a.splits * g.M * g.N * sizeof(float));
            if (!a.ws) return false;
        }
    }
    a.vec_ok = ((g.ldc % 4) == 0 && (g.ldca % 8) == 0 && (g.N % 4) == 0) ? 1 : 0;
    if (g.Cf && !aligned16(g.Cf)) a.vec_ok = 0;
    if (g.Ca && !aligned16(g.Ca)) a.vec_ok = 0;
    if (g.Caux && !aligned16(g.Caux)) a.vec_ok = 0;
    if (g.aux_in && !aligned16(g.aux_in)) a.vec_ok = 0;
    if (g.resid && !aligned16(g.resid)) a.vec_ok = 0;
    if (g.logits_act && !aligned16(g.logits_act)) a.vec_ok = 0;
    if (a.splits > 1 && (g.N % 4) != 0) a.vec_ok = 0;

    const int items = tiles * a.splits;
    if (pair) {
        const int grid = 2 * std::min(items, sms / 2);
        if (a_k && b_k) launch2<0, 0>(ma, mb, a, grid, st);
        else if (a_k && b_mn) launch2<0, 1>(ma, mb, a, grid, st);
        else launch2<1, 1>(ma, mb, a, grid, st);
    } else if (BN == 256) {
        const int grid = std::min(items, sms);
        if (a_k && b_k) launch<256, 0, 0>(ma, mb, a, grid, st);
        else if (a_k && b_mn) launch<256, 0, 1>(ma, mb, a, grid, st);
        else launch<256, 1, 1>(ma, mb, a, grid, st);
    } else {
        const int grid = std::min(items, sms);
        if (a_k && b_k) launch<128, 0, 0>(ma, mb, a, grid, st);
        else if (a_k && b_mn) launch<128, 0, 1>(ma, mb, a, grid, st);
        else launch<128, 1, 1>(ma, mb, a, grid, st);
    }
    if (a.splits > 1) {
        const long n = (long)g.M * g.N;
        const int blocks = (int)std::min<long>((n + 255) / 256, 148L * 8);
        k_splitk_reduce<<<blocks, 256, 0, st>>>(a.ws, a.splits, g.M, g.N, g.Cf, g.ldc);
        PARL_LAUNCHED();
    }
    return true;
}

}  // namespace parl_gpu
