// Varlen shared-prompt attention, FFMA path (one warp per (row, head)).
//
// Replaces the attention loops of run_forward (proj/src/model.cpp:468-501)
// and backward (model.cpp:751-786).  The shared-prompt rule
// (model.cpp:242-245) makes every row's allowed set a union of at most two
// contiguous ranges, so masked pairs are never visited (no -inf masking, no
// leakage: a response's result cannot depend on another response's values).
//   query i in a prompt            : keys [group start, i]
//   query i in response k          : keys [its group's prompt) and [start_k, i]
//   key j in a prompt              : queries [j, group end)
//   key j in response k            : queries [j, end_k)
// (AttnArgs::seg_info; one group: the prompt is [0, P) and the group ends at T)
// Forward saves only the per-row log-sum-exp (no T x T probabilities); the
// backward recomputes probabilities and is deterministic (dQ and dK/dV are
// produced by separate row-owning passes, no float atomics).
#include "internal.cuh"
#include "kernels.cuh"

namespace parl_gpu {

namespace {

constexpr int WPB = 8;    // warps per block
constexpr int MAXE = 4;   // per-lane head-dim elements (Dh <= 128)

struct Ranges {
    int b0, e0, b1, e1;  // [b0, e0) and [b1, e1), inclusive-exclusive
};

__device__ __forceinline__ Ranges key_ranges(const AttnArgs& a, int i) {
    const int4 f = a.seg_info[a.seg[i]];
    Ranges r;
    if (f.y < 0) {  // prompt row: its group's prompt prefix
        r.b0 = f.x; r.e0 = i + 1; r.b1 = 0; r.e1 = 0;
    } else {        // response row: its group's prompt, then its own prefix
        r.b0 = f.x; r.e0 = f.y; r.b1 = f.z; r.e1 = i + 1;
    }
    return r;
}

template <class T>
__global__ void __launch_bounds__(WPB * 32) k_attn_fwd(AttnArgs a, const T* __restrict__ qkv, T* __restrict__ out,
                                                      float* __restrict__ lse) {
    extern __shared__ float qs_all[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long gw = (long)blockIdx.x * WPB + wib;
    if (gw >= (long)a.T * a.H) return;
    const int h = (int)(gw / a.T), i = (int)(gw % a.T);
    const int Dh = a.Dh, ld = 3 * a.d;
    float* qs = qs_all + wib * Dh;
    const T* qrow = qkv + (long)i * ld + h * Dh;
    for (int e = lane; e < Dh; e += 32) qs[e] = to_f<T>(qrow[e]);
    __syncwarp();

    float o[MAXE] = {0.f, 0.f, 0.f, 0.f};
    float m = -INFINITY, l = 0.f;
    // Keys are walked in the row's *virtual* order: prompt keys, then the own
    // response's prefix -- exactly the unpacked causal sequence of that
    // response, so packed and unpacked scores are bit-identical.
    const Ranges R = key_ranges(a, i);
    const int n0 = R.e0 - R.b0, nv = n0 + (R.e1 - R.b1);
    for (int v0 = 0; v0 < nv; v0 += 32) {
        const int v = v0 + lane;
        const int j = v < n0 ? R.b0 + v : R.b1 + (v - n0);
        float s = -INFINITY;
        if (v < nv) {
            const T* kr = qkv + (long)j * ld + a.d + h * Dh;
            float acc = 0.f;
            for (int e = 0; e < Dh; ++e) acc = fmaf(qs[e], to_f<T>(kr[e]), acc);
            s = acc * a.scale;
        }
        const float mn = fmaxf(m, warp_max(s));
        const float p = (v < nv) ? __expf(s - mn) : 0.f;
        const float corr = __expf(m - mn);  // m == -inf on the first chunk -> 0
        l = l * corr + warp_sum(p);
#pragma unroll
        for (int q = 0; q < MAXE; ++q) o[q] *= corr;
        m = mn;
        const int nj = min(32, nv - v0);
        for (int t = 0; t < nj; ++t) {
            const float pt = __shfl_sync(0xffffffffu, p, t);
            const int jt = __shfl_sync(0xffffffffu, j, t);
            const T* vr = qkv + (long)jt * ld + 2 * a.d + h * Dh;
#pragma unroll
            for (int q = 0; q < MAXE; ++q) {
                const int e = lane + 32 * q;
                if (e < Dh) o[q] = fmaf(pt, to_f<T>(vr[e]), o[q]);
            }
        }
    }
    const float inv = 1.f / l;
    T* orow = out + (long)i * (a.ldo ? a.ldo : a.d) + h * Dh;
#pragma unroll
    for (int q = 0; q < MAXE; ++q) {
        const int e = lane + 32 * q;
        if (e < Dh) orow[e] = from_f<T>(o[q] * inv);
    }
    if (lane == 0) lse[(long)h * a.T + i] = m + logf(l);
}

// D[h][i] = sum_e dO[i,h,e] * O[i,h,e]
template <class T>
__global__ void k_attn_dsum(AttnArgs a, const T* __restrict__ out, const T* __restrict__ dout,
                            float* __restrict__ dsum) {
    const int lane = threadIdx.x & 31;
    const long gw = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw >= (long)a.T * a.H) return;
    const int h = (int)(gw / a.T), i = (int)(gw % a.T);
    float acc = 0.f;
    for (int e = lane; e < a.Dh; e += 32) {
        const long off = (long)i * a.d + h * a.Dh + e;
        acc += to_f<T>(out[(long)i * (a.ldo ? a.ldo : a.d) + h * a.Dh + e]) * to_f<T>(dout[off]);
    }
    acc = warp_sum(acc);
    if (lane == 0) dsum[(long)h * a.T + i] = acc;
}

// dQ: one warp per (query row, head), walking the row's allowed keys.
template <class T>
__global__ void __launch_bounds__(WPB * 32) k_attn_bwd_dq(AttnArgs a, const T* __restrict__ qkv,
                                                         const T* __restrict__ dout, const float* __restrict__ lse,
                                                         const float* __restrict__ dsum, T* __restrict__ dqkv) {
    extern __shared__ float sm_all[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long gw = (long)blockIdx.x * WPB + wib;
    if (gw >= (long)a.T * a.H) return;
    const int h = (int)(gw / a.T), i = (int)(gw % a.T);
    const int Dh = a.Dh, ld = 3 * a.d;
    float* qs = sm_all + wib * 2 * Dh;
    float* dos = qs + Dh;
    for (int e = lane; e < Dh; e += 32) {
        qs[e] = to_f<T>(qkv[(long)i * ld + h * Dh + e]);
        dos[e] = to_f<T>(dout[(long)i * a.d + h * Dh + e]);
    }
    __syncwarp();
    const float L = lse[(long)h * a.T + i], Di = dsum[(long)h * a.T + i];
    float dq[MAXE] = {0.f, 0.f, 0.f, 0.f};
    const Ranges R = key_ranges(a, i);
    const int n0 = R.e0 - R.b0, nv = n0 + (R.e1 - R.b1);
    for (int v0 = 0; v0 < nv; v0 += 32) {
        const int v = v0 + lane;
        const int j = v < n0 ? R.b0 + v : R.b1 + (v - n0);
        float ds = 0.f;
        if (v < nv) {
            const T* kr = qkv + (long)j * ld + a.d + h * Dh;
            const T* vr = qkv + (long)j * ld + 2 * a.d + h * Dh;
            float s = 0.f, dp = 0.f;
            for (int e = 0; e < Dh; ++e) {
                s = fmaf(qs[e], to_f<T>(kr[e]), s);
                dp = fmaf(dos[e], to_f<T>(vr[e]), dp);
            }
            const float p = __expf(s * a.scale - L);
            ds = p * (dp - Di);
        }
        const int nj = min(32, nv - v0);
        for (int t = 0; t < nj; ++t) {
            const float dst = __shfl_sync(0xffffffffu, ds, t);
            const int jt = __shfl_sync(0xffffffffu, j, t);
            const T* kr = qkv + (long)jt * ld + a.d + h * Dh;
#pragma unroll
            for (int q = 0; q < MAXE; ++q) {
                const int e = lane + 32 * q;
                if (e < Dh) dq[q] = fmaf(dst, to_f<T>(kr[e]), dq[q]);
            }
        }
    }
    T* drow = dqkv + (long)i * ld + h * Dh;
#pragma unroll
    for (int q = 0; q < MAXE; ++q) {
        const int e = lane + 32 * q;
        if (e < Dh) drow[e] = from_f<T>(dq[q] * a.scale);
    }
}

// dK, dV: one warp per (key row, head), walking the key's allowed queries.
template <class T>
__global__ void __launch_bounds__(WPB * 32) k_attn_bwd_dkv(AttnArgs a, const T* __restrict__ qkv,
                                                          const T* __restrict__ dout, const float* __restrict__ lse,
                                                          const float* __restrict__ dsum, T* __restrict__ dqkv) {
    extern __shared__ float sm_all[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long gw = (long)blockIdx.x * WPB + wib;
    if (gw >= (long)a.T * a.H) return;
    const int h = (int)(gw / a.T), j = (int)(gw % a.T);
    const int Dh = a.Dh, ld = 3 * a.d;
    float* ks = sm_all + wib * 2 * Dh;
    float* vs = ks + Dh;
    for (int e = lane; e < Dh; e += 32) {
        ks[e] = to_f<T>(qkv[(long)j * ld + a.d + h * Dh + e]);
        vs[e] = to_f<T>(qkv[(long)j * ld + 2 * a.d + h * Dh + e]);
    }
    __syncwarp();
    const int ie = a.seg_info[a.seg[j]].w;  // queries [j, ie) see key j
    float dk[MAXE] = {0.f, 0.f, 0.f, 0.f}, dv[MAXE] = {0.f, 0.f, 0.f, 0.f};
    for (int i0 = j; i0 < ie; i0 += 32) {
        const int i = i0 + lane;
        float p = 0.f, ds = 0.f;
        if (i < ie) {
            const T* qr = qkv + (long)i * ld + h * Dh;
            const T* dor = dout + (long)i * a.d + h * Dh;
            float s = 0.f, dp = 0.f;
            for (int e = 0; e < Dh; ++e) {
                s = fmaf(to_f<T>(qr[e]), ks[e], s);
                dp = fmaf(to_f<T>(dor[e]), vs[e], dp);
            }
            p = __expf(s * a.scale - lse[(long)h * a.T + i]);
            ds = p * (dp - dsum[(long)h * a.T + i]);
        }
        const int ni = min(32, ie - i0);
        for (int t = 0; t < ni; ++t) {
            const float pt = __shfl_sync(0xffffffffu, p, t), dst = __shfl_sync(0xffffffffu, ds, t);
            const T* qr = qkv + (long)(i0 + t) * ld + h * Dh;
            const T* dor = dout + (long)(i0 + t) * a.d + h * Dh;
#pragma unroll
            for (int q = 0; q < MAXE; ++q) {
                const int e = lane + 32 * q;
                if (e < Dh) {
                    dv[q] = fmaf(pt, to_f<T>(dor[e]), dv[q]);
                    dk[q] = fmaf(dst, to_f<T>(qr[e]), dk[q]);
                }
            }
        }
    }
    T* krow = dqkv + (long)j * ld + a.d + h * Dh;
    T* vrow = dqkv + (long)j * ld + 2 * a.d + h * Dh;
#pragma unroll
    for (int q = 0; q < MAXE; ++q) {
        const int e = lane + 32 * q;
        if (e < Dh) {
            krow[e] = from_f<T>(dk[q] * a.scale);
            vrow[e] = from_f<T>(dv[q]);
        }
    }
}

}  // namespace

template <class T>
void launch_attn_fwd(const AttnArgs& a, const T* qkv, T* out, float* lse, cudaStream_t st) {
    const long warps = (long)a.T * a.H;
    k_attn_fwd<T><<<cdiv(warps, WPB), WPB * 32, WPB * a.Dh * sizeof(float), st>>>(a, qkv, out, lse);
    PARL_LAUNCHED();
}

template <class T>
void launch_attn_dsum(const AttnArgs& a, const T* out, const T* dout, float* dsum, cudaStream_t st) {
    const long warps = (long)a.T * a.H;
    k_attn_dsum<T><<<cdiv(warps * 32, 256), 256, 0, st>>>(a, out, dout, dsum);
    PARL_LAUNCHED();
}
template void launch_attn_dsum<float>(const AttnArgs&, const float*, const float*, float*, cudaStream_t);
template void launch_attn_dsum<bf16>(const AttnArgs&, const bf16*, const bf16*, float*, cudaStream_t);

template <class T>
void launch_attn_bwd(const AttnArgs& a, const T* qkv, const T* out, const T* dout, const float* lse, float* dsum,
                     T* dqkv, cudaStream_t st) {
    const long warps = (long)a.T * a.H;
    launch_attn_dsum<T>(a, out, dout, dsum, st);
    const size_t sm = WPB * 2 * a.Dh * sizeof(float);
    k_attn_bwd_dq<T><<<cdiv(warps, WPB), WPB * 32, sm, st>>>(a, qkv, dout, lse, dsum, dqkv);
    PARL_LAUNCHED();
    k_attn_bwd_dkv<T><<<cdiv(warps, WPB), WPB * 32, sm, st>>>(a, qkv, dout, lse, dsum, dqkv);
    PARL_LAUNCHED();
}

// ---------------------------------------------------------------------------
// KV-cached decoding (the rollout side, sample_tokens model.cpp:843-900): one new query row
// per sequence against the shared prompt's cached K/V (prefilled once for all sequences of
// a group) and the sequence's own generated K/V.  Block = (sequence, head), 4 warps stride
// over the keys with an online softmax each, combined at the end; lane holds Dh/32 elements.
template <class T>
__global__ void __launch_bounds__(128) k_decode_attn(const T* __restrict__ q, long ldq, const T* __restrict__ kv_prompt,
                                                     const T* __restrict__ kv_own, long own_stride, int P, int n_own,
                                                     int d, int Dh, float scale, T* __restrict__ out, long ldo) {
    __shared__ float sm_m[4], sm_l[4], sm_o[4][128];
    const int seq = blockIdx.x, h = blockIdx.y, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float qv[MAXE], o[MAXE] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < MAXE; ++k) {
        const int e = lane + 32 * k;
        qv[k] = e < Dh ? to_f<T>(q[(long)seq * ldq + h * Dh + e]) : 0.f;
    }
    float m = -INFINITY, l = 0.f;
    for (int j = w; j < P + n_own; j += 4) {
        const T* kr = j < P ? kv_prompt + (long)j * 2 * d + h * Dh : kv_own + seq * own_stride + (long)(j - P) * 2 * d + h * Dh;
        const T* vr = kr + d;
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < MAXE; ++k) {
            const int e = lane + 32 * k;
            if (e < Dh) s = fmaf(qv[k], to_f<T>(kr[e]), s);
        }
        s = warp_sum(s) * scale;
        const float mn = fmaxf(m, s), corr = __expf(m - mn), p = __expf(s - mn);
        l = l * corr + p;
#pragma unroll
        for (int k = 0; k < MAXE; ++k) {
            const int e = lane + 32 * k;
            o[k] = o[k] * corr + (e < Dh ? p * to_f<T>(vr[e]) : 0.f);
        }
        m = mn;
    }
    if (lane == 0) {
        sm_m[w] = m;
        sm_l[w] = l;
    }
#pragma unroll
    for (int k = 0; k < MAXE; ++k)
        if (lane + 32 * k < Dh) sm_o[w][lane + 32 * k] = o[k];
    __syncthreads();
    if (w != 0) return;
    const float mm = fmaxf(fmaxf(sm_m[0], sm_m[1]), fmaxf(sm_m[2], sm_m[3]));
    float lt = 0.f, c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        c[u] = sm_m[u] == -INFINITY ? 0.f : __expf(sm_m[u] - mm);
        lt += sm_l[u] * c[u];
    }
#pragma unroll
    for (int k = 0; k < MAXE; ++k) {
        const int e = lane + 32 * k;
        if (e >= Dh) continue;
        float v = 0.f;
#pragma unroll
        for (int u = 0; u < 4; ++u) v += sm_o[u][e] * c[u];
        out[(long)seq * ldo + h * Dh + e] = from_f<T>(v / lt);
    }
}

template <class T>
void launch_decode_attn(const T* q, long ldq, const T* kv_prompt, const T* kv_own, long own_stride, int P, int n_own,
                        int n_seq, int H, int d, float scale, T* out, long ldo, cudaStream_t st) {
    k_decode_attn<T><<<dim3(n_seq, H), 128, 0, st>>>(q, ldq, kv_prompt, kv_own, own_stride, P, n_own, d, d / H, scale,
                                                     out, ldo);
    PARL_LAUNCHED();
}
template void launch_decode_attn<float>(const float*, long, const float*, const float*, long, int, int, int, int, int,
                                        float, float*, long, cudaStream_t);
template void launch_decode_attn<bf16>(const bf16*, long, const bf16*, const bf16*, long, int, int, int, int, int,
                                       float, bf16*, long, cudaStream_t);

template void launch_attn_fwd<float>(const AttnArgs&, const float*, float*, float*, cudaStream_t);
template void launch_attn_fwd<bf16>(const AttnArgs&, const bf16*, bf16*, float*, cudaStream_t);
template void launch_attn_bwd<float>(const AttnArgs&, const float*, const float*, const float*, const float*, float*,
                                     float*, cudaStream_t);
template void launch_attn_bwd<bf16>(const AttnArgs&, const bf16*, const bf16*, const bf16*, const float*, float*,
                                    bf16*, cudaStream_t);

}  // namespace parl_gpu
