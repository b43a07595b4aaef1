// HBM-bound / integer kernels of the hot path:
//   K1  packer                 pack_group + build_segments/predecessor (packing.cpp:7-45, model.cpp:230-253)
//   K2  embedding gather       model.cpp:449-455
//   K5  LayerNorm fwd / bwd    model.cpp:317-369
//   K6b vocab LSE + gather     model.cpp:523-556 (FFMA mode; the tcgen05 head fuses this)
//   K8a softmax backward seed  model.cpp:637-650
//   K11 embedding-grad reduce  model.cpp:825-834 (deterministic: stable sort + segmented sum)
// plus column reductions (bias / LN parameter grads), weight conversion,
// device init, SGD update.
#include <cstdlib>
#include <type_traits>
#include <algorithm>
#include <cub/cub.cuh>

#include "internal.cuh"
#include "kernels.cuh"

namespace parl_gpu {

// ---------------------------------------------------------------------------
// K1: device packer.  One thread per packed position t.  cu[k] = scored offset
// of response k (exclusive prefix of resp_lens), cu[G] = S.
// `id_max` receives max over tokens of (unsigned)id: an id outside [0, V) is exactly
// one with (unsigned)id >= V (VocabError, model.cpp:413-417), checked before the forward.
__device__ __forceinline__ void st4(int32_t* p, const int* v) {
    *reinterpret_cast<int4*>(p) = make_int4(v[0], v[1], v[2], v[3]);
}

// One thread per 4 consecutive positions (P a multiple of 4, so the [T] and [S] arrays are
// both 16-byte aligned): one binary search over cu[] per thread (the following positions
// advance the response index), 16-byte stores of all the arrays.
__global__ void k_pack(const int32_t* __restrict__ prompt, int P, const int32_t* __restrict__ resp_flat,
                       const int32_t* __restrict__ cu, int G, PackedDev pk, unsigned* __restrict__ id_max) {
    const int T = P + cu[G];
    const bool vt = ((reinterpret_cast<uintptr_t>(pk.tokens) | reinterpret_cast<uintptr_t>(pk.labels) |
                      reinterpret_cast<uintptr_t>(pk.positions) | reinterpret_cast<uintptr_t>(pk.seg) |
                      reinterpret_cast<uintptr_t>(pk.pred) | reinterpret_cast<uintptr_t>(pk.row_ptr)) & 15) == 0;
    const bool vs = (P & 3) == 0 &&
                    ((reinterpret_cast<uintptr_t>(pk.scored_pos) | reinterpret_cast<uintptr_t>(pk.scored_label) |
                      reinterpret_cast<uintptr_t>(pk.pred_pos) | reinterpret_cast<uintptr_t>(pk.sample_of)) & 15) == 0;
    unsigned umax = 0;
    for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; 4 * q < T; q += (long)gridDim.x * blockDim.x) {
        const int t0 = (int)(4 * q);
        int tk[4], lb[4], ps[4], sg[4], pr[4], rp[4], sp[4], sk[4];
        int k = -1;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int t = t0 + u;
            tk[u] = lb[u] = ps[u] = sg[u] = pr[u] = rp[u] = sp[u] = sk[u] = 0;
            if (t >= T) continue;
            if (t < P) {
                const int tok = prompt[t];
                umax = max(umax, (unsigned)tok);
                tk[u] = tok;
                lb[u] = -1;
                ps[u] = t;
                pr[u] = t - 1;
            } else {
                const int s = t - P;
                if (k < 0) {  // response k with cu[k] <= s < cu[k+1]
                    int lo = 0, hi = G - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (cu[mid] <= s) lo = mid; else hi = mid - 1;
                    }
                    k = lo;
                } else {
                    while (cu[k + 1] <= s) ++k;
                }
                const int i = s - cu[k];
                const int tok = resp_flat[s];
                umax = max(umax, (unsigned)tok);
                tk[u] = tok;
                lb[u] = tok;  // self-aligned labels, packing.cpp:37
                ps[u] = P + i;
                sg[u] = k + 1;
                pr[u] = (i == 0) ? P - 1 : t - 1;  // model.cpp:251
                // position -> gathered head rows (CSR): P-1 owns the G response starts, every
                // non-final response token owns row t+1-P
                rp[u] = G + s - k;
                sp[u] = t;
                sk[u] = k;
                const bool last = (i == cu[k + 1] - cu[k] - 1);
                if (!last) pk.row_idx[G + s - k] = s + 1;
            }
            if (t == P - 1)
                for (int r = 0; r < G; ++r) pk.row_idx[r] = cu[r];
            if (t == T - 1) pk.row_ptr[T] = cu[G];
        }
        if (vt && t0 + 4 <= T) {
            st4(pk.tokens + t0, tk);
            st4(pk.labels + t0, lb);
            st4(pk.positions + t0, ps);
            st4(pk.seg + t0, sg);
            st4(pk.pred + t0, pr);
            st4(pk.row_ptr + t0, rp);
        } else {
            for (int u = 0; u < 4 && t0 + u < T; ++u) {
                pk.tokens[t0 + u] = tk[u];
                pk.labels[t0 + u] = lb[u];
                pk.positions[t0 + u] = ps[u];
                pk.seg[t0 + u] = sg[u];
                pk.pred[t0 + u] = pr[u];
                pk.row_ptr[t0 + u] = rp[u];
            }
        }
        if (vs && t0 >= P && t0 + 4 <= T) {  // s0 = t0 - P is a multiple of 4
            const int s0 = t0 - P;
            st4(pk.scored_pos + s0, sp);
            st4(pk.scored_label + s0, tk);
            st4(pk.pred_pos + s0, pr);
            st4(pk.sample_of + s0, sk);
        } else {
            for (int u = 0; u < 4; ++u) {
                const int t = t0 + u;
                if (t < P || t >= T) continue;
                pk.scored_pos[t - P] = sp[u];
                pk.scored_label[t - P] = tk[u];
                pk.pred_pos[t - P] = pr[u];
                pk.sample_of[t - P] = sk[u];
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) umax = max(umax, __shfl_xor_sync(0xffffffffu, umax, o));
    if ((threadIdx.x & 31) == 0 && id_max) atomicMax(id_max, umax);
}

// K1 when P is not a multiple of 4 (the [T] and [S] arrays cannot both be 16-byte aligned):
// one thread per position, every store instruction 128 contiguous bytes of one array.
__global__ void k_pack_scalar(const int32_t* __restrict__ prompt, int P, const int32_t* __restrict__ resp_flat,
                       const int32_t* __restrict__ cu, int G, PackedDev pk, unsigned* __restrict__ id_max) {
    const int T = P + cu[G];
    unsigned umax = 0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
        if (t < P) {
            umax = max(umax, (unsigned)prompt[t]);
            pk.tokens[t] = prompt[t];
            pk.labels[t] = -1;
            pk.positions[t] = t;
            pk.seg[t] = 0;
            pk.pred[t] = t - 1;
            pk.row_ptr[t] = 0;
        } else {
            const int s = t - P;
            int lo = 0, hi = G - 1;  // response k with cu[k] <= s < cu[k+1]
            while (lo < hi) {
                int mid = (lo + hi + 1) >> 1;
                if (cu[mid] <= s) lo = mid; else hi = mid - 1;
            }
            const int k = lo, i = s - cu[k];
            const int tok = resp_flat[s];
            umax = max(umax, (unsigned)tok);
            pk.tokens[t] = tok;
            pk.labels[t] = tok;  // self-aligned labels, packing.cpp:37
            pk.positions[t] = P + i;
            pk.seg[t] = k + 1;
            const int pr = (i == 0) ? P - 1 : t - 1;  // model.cpp:251
            pk.pred[t] = pr;
            pk.scored_pos[s] = t;
            pk.scored_label[s] = tok;
            pk.pred_pos[s] = pr;
            pk.sample_of[s] = k;
            // position -> gathered head rows (CSR): P-1 owns the G response
            // starts, every non-final response token owns row t+1-P.
            pk.row_ptr[t] = G + s - k;
            const bool last = (i == cu[k + 1] - cu[k] - 1);
            if (!last) pk.row_idx[G + s - k] = s + 1;
        }
        if (t == P - 1)
            for (int k = 0; k < G; ++k) pk.row_idx[k] = cu[k];
        if (t == T - 1) pk.row_ptr[T] = cu[G];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) umax = max(umax, __shfl_xor_sync(0xffffffffu, umax, o));
    if ((threadIdx.x & 31) == 0 && id_max) atomicMax(id_max, umax);
}

// K1, several prompt groups in one packed sequence (f4: several prompts per launch):
// [P_0 | R_0,0 .. R_0,G0-1 | P_1 | R_1,0 ..], each group laid out as pack_group lays out
// one (packing.cpp:27-43): positions restart at 0 for every group, the responses of a group
// restart at its P, labels self-aligned, the first token of a response scored from its
// group's last prompt position.  Segments: group g's prompt is segment g + r0[g] (r0 =
// first response of the group), its responses follow.  One thread per packed position;
// the group by binary search over gstart[n + 1], the response over rcu (scored offsets).
__global__ void k_pack_multi(const int32_t* __restrict__ prompts, const int32_t* __restrict__ resp_flat,
                             const int32_t* __restrict__ gstart, const int32_t* __restrict__ pstart,
                             const int32_t* __restrict__ r0, const int32_t* __restrict__ rcu,
                             const int32_t* __restrict__ rstart, int n, PackedDev pk, unsigned* __restrict__ id_max) {
    const int T = gstart[n], S = rcu[r0[n]];
    unsigned umax = 0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
        int lo = 0, hi = n - 1;  // group g with gstart[g] <= t < gstart[g + 1]
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (gstart[mid] <= t) lo = mid; else hi = mid - 1;
        }
        const int g = lo, gs = gstart[g], kr0 = r0[g], kr1 = r0[g + 1];
        const int P = (kr1 > kr0 ? rstart[kr0] : gstart[g + 1]) - gs;
        const int pe = gs + P - 1;                     // the group's last prompt position
        const int S_before = rcu[kr0];                 // rows owned by earlier groups' positions
        const int sp = g + kr0;                        // the group's prompt segment
        if (t < gs + P) {
            const int tok = prompts[pstart[g] + (t - gs)];
            umax = max(umax, (unsigned)tok);
            pk.tokens[t] = tok;
            pk.labels[t] = -1;
            pk.positions[t] = t - gs;
            pk.seg[t] = sp;
            pk.pred[t] = t > gs ? t - 1 : -1;
            pk.row_ptr[t] = S_before;
            if (t == pe)
                for (int k = kr0; k < kr1; ++k) pk.row_idx[S_before + (k - kr0)] = rcu[k];
        } else {
            int a = kr0, b = kr1 - 1;  // response k with rstart[k] <= t
            while (a < b) {
                const int mid = (a + b + 1) >> 1;
                if (rstart[mid] <= t) a = mid; else b = mid - 1;
            }
            const int k = a, i = t - rstart[k], s = rcu[k] + i;
            const int tok = resp_flat[s];
            umax = max(umax, (unsigned)tok);
            pk.tokens[t] = tok;
            pk.labels[t] = tok;
            pk.positions[t] = P + i;
            pk.seg[t] = sp + 1 + (k - kr0);
            const int pr = i == 0 ? pe : t - 1;
            pk.pred[t] = pr;
            pk.scored_pos[s] = t;
            pk.scored_label[s] = tok;
            pk.pred_pos[s] = pr;
            pk.sample_of[s] = k;
            const int rp = S_before + (kr1 - kr0) + (s - rcu[kr0]) - (k - kr0);
            pk.row_ptr[t] = rp;
            if (i != rcu[k + 1] - rcu[k] - 1) pk.row_idx[rp] = s + 1;
        }
        if (t == T - 1) pk.row_ptr[T] = S;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) umax = max(umax, __shfl_xor_sync(0xffffffffu, umax, o));
    if ((threadIdx.x & 31) == 0 && id_max) atomicMax(id_max, umax);
}

// ---------------------------------------------------------------------------
// K2: x[t] = tok_emb[tokens[t]] + pos_emb[positions[t]]  (fp32 residual stream)
__global__ void k_embed(const float* __restrict__ tok_emb, const float* __restrict__ pos_emb,
                        const int32_t* __restrict__ tokens, const int32_t* __restrict__ positions, int T,
                        int D, float* __restrict__ x) {
    const long n = (long)T * D;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const int t = (int)(e / D), i = (int)(e % D);
        x[e] = tok_emb[(long)tokens[t] * D + i] + pos_emb[(long)positions[t] * D + i];
    }
}

// float4 variant (D % 4 == 0, 16-byte aligned rows): one warp per token row, no per-element
// index division
__global__ void __launch_bounds__(256) k_embed4(const float4* __restrict__ tok_emb, const float4* __restrict__ pos_emb,
                                                const int32_t* __restrict__ tokens,
                                                const int32_t* __restrict__ positions, int T, int D4,
                                                float4* __restrict__ x) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (t >= T) return;
    const float4* a = tok_emb + (long)tokens[t] * D4;
    const float4* b = pos_emb + (long)positions[t] * D4;
    float4* y = x + (long)t * D4;
    for (int c = lane; c < D4; c += 32) {
        const float4 u = a[c], v = b[c];
        y[c] = make_float4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w);
    }
}

// ---------------------------------------------------------------------------
// K5: LayerNorm forward, one warp per row; rows optionally gathered through
// `rows` (final LN over the head's predecessor rows).  Two-pass mean/variance
// (population), eps 1e-5 (model.cpp:132, 317-343).
template <class T, int PER>
__global__ void k_layernorm(const float* __restrict__ x, const int32_t* __restrict__ rows, int R, int D,
                            const float* __restrict__ gamma, const float* __restrict__ beta,
                            T* __restrict__ y, long ldy, float* __restrict__ mean_out, float* __restrict__ rstd_out) {
    // PER > 0: the row stays in registers (PER floats per lane, D <= 32 * PER); 0: strided passes
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= R) return;
    const int src = rows ? rows[warp] : warp;
    const float* xr = x + (long)src * D;
    T* yr = y + (long)warp * ldy;
    float mean, rstd;
    if constexpr (PER > 0) {
        float v[PER];
        float s = 0.f;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int i = lane + 32 * q;
            v[q] = i < D ? xr[i] : 0.f;
            s += v[q];
        }
        mean = warp_sum(s) / D;
        float var = 0.f;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int i = lane + 32 * q;
            const float c = i < D ? v[q] - mean : 0.f;
            var += c * c;
        }
        rstd = rsqrtf(warp_sum(var) / D + 1e-5f);
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int i = lane + 32 * q;
            if (i < D) yr[i] = from_f<T>((v[q] - mean) * rstd * gamma[i] + beta[i]);
        }
    } else {
        float s = 0.f;
        for (int i = lane; i < D; i += 32) s += xr[i];
        mean = warp_sum(s) / D;
        float v = 0.f;
        for (int i = lane; i < D; i += 32) {
            const float c = xr[i] - mean;
            v += c * c;
        }
        rstd = rsqrtf(warp_sum(v) / D + 1e-5f);
        for (int i = lane; i < D; i += 32) yr[i] = from_f<T>((xr[i] - mean) * rstd * gamma[i] + beta[i]);
    }
    if (lane == 0) {
        mean_out[warp] = mean;
        rstd_out[warp] = rstd;
    }
}

// LayerNorm backward (input part), one warp per row:
//   dx[r] = (res ? res[r] : 0) + rstd * (dxh - mean(dxh) - xhat * mean(dxh*xhat)),  dxh = dy*gamma
// x rows gathered through `rows` when given (stats are per output row).
__global__ void k_layernorm_bwd(const float* __restrict__ dy, const float* __restrict__ x,
                                const int32_t* __restrict__ rows, const float* __restrict__ mean,
                                const float* __restrict__ rstd, const float* __restrict__ gamma, int R, int D,
                                const float* __restrict__ res, float* __restrict__ dx) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= R) return;
    const float* xr = x + (long)(rows ? rows[warp] : warp) * D;
    const float* dyr = dy + (long)warp * D;
    const float mu = mean[warp], rs = rstd[warp];
    float a = 0.f, b = 0.f;
    for (int i = lane; i < D; i += 32) {
        const float dxh = dyr[i] * gamma[i];
        a += dxh;
        b += dxh * (xr[i] - mu) * rs;
    }
    a = warp_sum(a) / D;
    b = warp_sum(b) / D;
    float* o = dx + (long)warp * D;
    const float* rr = res ? res + (long)warp * D : nullptr;
    for (int i = lane; i < D; i += 32) {
        const float xh = (xr[i] - mu) * rs;
        const float v = rs * (dyr[i] * gamma[i] - a - xh * b);
        o[i] = rr ? rr[i] + v : v;
    }
}

// Column reductions, deterministic two-stage: block (col chunk, row split)
// sums its rows in fixed stripe order into partial[split][col]; stage 2 adds
// the splits in order.
//   mode 0: out[c] += sum_r X[r][c]                                      (bias grads)
//   mode 1: out[c] += sum_r dy[r][c]*xhat[r][c], out2[c] += sum_r dy[r][c] (LN gamma/beta)
template <class T>
struct Pair2;
template <>
struct Pair2<float> {
    using V = float2;
    static __device__ __forceinline__ float2 f(V v) { return v; }
};
template <>
struct Pair2<bf16> {
    using V = __nv_bfloat162;
    static __device__ __forceinline__ float2 f(V v) { return __bfloat1622float2(v); }
};

// Block = 8 warps over 64 columns (2 per lane, one contiguous segment per row
// per warp); warps stripe the block's row range with 4-row ILP.  Requires even
// N and ldx (else the scalar kernel below is used).
template <class T>
__global__ void __launch_bounds__(256) k_colsum_part(const T* __restrict__ X, long ldx, int R, int N,
                                                     int rows_per_split, const float* __restrict__ xs,
                                                     const int32_t* __restrict__ rows, const float* __restrict__ mean,
                                                     const float* __restrict__ rstd, int mode,
                                                     float* __restrict__ part_a, float* __restrict__ part_b) {
    pdl_wait();
    __shared__ float2 sa[8][32], sb[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int c = blockIdx.x * 64 + 2 * lane;
    const int r0 = blockIdx.y * rows_per_split, r1 = min(R, r0 + rows_per_split);
    float2 a = make_float2(0.f, 0.f), b = make_float2(0.f, 0.f);
    if (c < N) {
        int r = r0 + w;
        for (; r + 24 < r1; r += 32) {
            float2 v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                v[q] = Pair2<T>::f(*reinterpret_cast<const typename Pair2<T>::V*>(X + (long)(r + 8 * q) * ldx + c));
            if (mode == 0) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    a.x += v[q].x;
                    a.y += v[q].y;
                }
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int rr = r + 8 * q;
                    const float2 xv = *reinterpret_cast<const float2*>(xs + (long)(rows ? rows[rr] : rr) * N + c);
                    const float mu = mean[rr], rs = rstd[rr];
                    a.x += v[q].x * (xv.x - mu) * rs;
                    a.y += v[q].y * (xv.y - mu) * rs;
                    b.x += v[q].x;
                    b.y += v[q].y;
                }
            }
        }
        for (; r < r1; r += 8) {
            const float2 v = Pair2<T>::f(*reinterpret_cast<const typename Pair2<T>::V*>(X + (long)r * ldx + c));
            if (mode == 0) {
                a.x += v.x;
                a.y += v.y;
            } else {
                const float2 xv = *reinterpret_cast<const float2*>(xs + (long)(rows ? rows[r] : r) * N + c);
                a.x += v.x * (xv.x - mean[r]) * rstd[r];
                a.y += v.y * (xv.y - mean[r]) * rstd[r];
                b.x += v.x;
                b.y += v.y;
            }
        }
    }
    sa[w][lane] = a;
    sb[w][lane] = b;
    __syncthreads();
    if (w == 0 && c < N) {
        float2 ta = make_float2(0.f, 0.f), tb = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            ta.x += sa[i][lane].x;
            ta.y += sa[i][lane].y;
            tb.x += sb[i][lane].x;
            tb.y += sb[i][lane].y;
        }
        part_a[(long)blockIdx.y * N + c] = ta.x;
        part_a[(long)blockIdx.y * N + c + 1] = ta.y;
        if (mode == 1) {
            part_b[(long)blockIdx.y * N + c] = tb.x;
            part_b[(long)blockIdx.y * N + c + 1] = tb.y;
        }
    }
}

// scalar variant (odd N / ldx)
template <class T>
__global__ void k_colsum_part1(const T* __restrict__ X, long ldx, int R, int N, int rows_per_split,
                               const float* __restrict__ xs, const int32_t* __restrict__ rows,
                               const float* __restrict__ mean, const float* __restrict__ rstd, int mode,
                               float* __restrict__ part_a, float* __restrict__ part_b) {
    __shared__ float sa[8][33], sb[8][33];
    const int c = blockIdx.x * 32 + threadIdx.x;
    const int ty = threadIdx.y;
    const int r0 = blockIdx.y * rows_per_split, r1 = min(R, r0 + rows_per_split);
    float a = 0.f, b = 0.f;
    if (c < N) {
        for (int r = r0 + ty; r < r1; r += 8) {
            const float v = to_f<T>(X[(long)r * ldx + c]);
            if (mode == 0) {
                a += v;
            } else {
                const float xv = xs[(long)(rows ? rows[r] : r) * N + c];
                a += v * (xv - mean[r]) * rstd[r];
                b += v;
            }
        }
    }
    sa[ty][threadIdx.x] = a;
    sb[ty][threadIdx.x] = b;
    __syncthreads();
    if (ty == 0 && c < N) {
        float ta = 0.f, tb = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            ta += sa[i][threadIdx.x];
            tb += sb[i][threadIdx.x];
        }
        part_a[(long)blockIdx.y * N + c] = ta;
        if (mode == 1) part_b[(long)blockIdx.y * N + c] = tb;
    }
}

__global__ void k_colsum_final(const float* __restrict__ part_a, const float* __restrict__ part_b, int splits, int N,
                               float* __restrict__ out, float* __restrict__ out2, int mode) {
    pdl_wait();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= N) return;
    // loads issued 8 at a time, added in split order (deterministic)
    float a = 0.f, b = 0.f;
    int s0 = 0;
    for (; s0 + 8 <= splits; s0 += 8) {
        float va[8], vb[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            va[q] = part_a[(long)(s0 + q) * N + c];
            vb[q] = mode == 1 ? part_b[(long)(s0 + q) * N + c] : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            a += va[q];
            b += vb[q];
        }
    }
    for (; s0 < splits; ++s0) {
        a += part_a[(long)s0 * N + c];
        if (mode == 1) b += part_b[(long)s0 * N + c];
    }
    out[c] += a;
    if (mode == 1) out2[c] += b;
}

namespace {
struct Scratch {
    float* p = nullptr;
    size_t n = 0;
    float* get(size_t need) {
        if (need > n) {
            if (p) cudaFree(p);
            if (cudaMalloc(&p, need * sizeof(float)) != cudaSuccess) throw Error{PARL_E_CUDA, "scratch alloc"};
            n = need;
        }
        return p;
    }
} g_colsum_scratch;

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
}  // namespace

template <class T>
static void colsum_impl(const T* X, long ldx, int R, int N, float* out, const float* xs, const int32_t* rows,
                        const float* mean, const float* rstd, float* out2, int mode, cudaStream_t st) {
    const bool vec = (N % 2 == 0) && (ldx % 2 == 0) && ((reinterpret_cast<uintptr_t>(X) & 7) == 0);
    const int cw = vec ? 64 : 32;
    const int col_blocks = cdiv(N, cw);
    int splits = std::max(1, std::min(cdiv(R, 128), cdiv(4 * 148, col_blocks)));
    const int rps = cdiv(R, splits);
    splits = cdiv(R, rps);
    float* pa = g_colsum_scratch.get((size_t)2 * splits * N);
    float* pb = pa + (size_t)splits * N;
    if (vec)
        launch_pdl(k_colsum_part<T>, dim3(col_blocks, splits), dim3(256), 0, st, X, ldx, R, N, rps, xs, rows, mean, rstd,
                   mode, pa, pb);
    else
        k_colsum_part1<T><<<dim3(col_blocks, splits), dim3(32, 8), 0, st>>>(X, ldx, R, N, rps, xs, rows, mean, rstd,
                                                                           mode, pa, pb);
    PARL_LAUNCHED();
    launch_pdl(k_colsum_final, dim3(cdiv(N, 256)), dim3(256), 0, st, (const float*)pa, (const float*)pb, splits, N, out,
               out2, mode);
    PARL_LAUNCHED();
}

// ---------------------------------------------------------------------------
// K6b (FFMA mode): per head row s: lse = logsumexp(z[s,:]); lp[s] = z[s,label] - lse.
__global__ void k_row_lse(const float* __restrict__ z, int V, const int32_t* __restrict__ labels,
                          float* __restrict__ lse_out, float* __restrict__ lp_out) {
    __shared__ float sm[32], ss[32];
    const int s = blockIdx.x;
    const float* row = z + (long)s * V;
    float m = -INFINITY, sum = 0.f;
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
        const float x = row[v];
        if (x > m) {
            sum = sum * __expf(m - x) + 1.f;
            m = x;
        } else {
            sum += __expf(x - m);
        }
    }
    // warp then block combine of (m, sum)
    for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
        const float mm = fmaxf(m, m2);
        sum = (m == -INFINITY ? 0.f : sum * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
        m = mm;
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sm[w] = m;
        ss[w] = sum;
    }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        m = lane < nw ? sm[lane] : -INFINITY;
        sum = lane < nw ? ss[lane] : 0.f;
        for (int o = 16; o > 0; o >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
            const float mm = fmaxf(m, m2);
            sum = (m == -INFINITY ? 0.f : sum * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
            m = mm;
        }
        if (lane == 0) {
            const float lse = m + logf(sum);
            lse_out[s] = lse;
            if (lp_out) lp_out[s] = row[labels[s]] - lse;
        }
    }
}

// Combine the tcgen05 head's per-tile (max, sumexp) partials: lse and lp.
// one warp per head row: lanes stride over the row's (max, sumexp) partials with
// 8-byte coalesced loads, keep an online (max, sum), then combine in a fixed
// shuffle tree (deterministic)
__global__ void k_lse_combine(const float* __restrict__ part, int n_parts, const float* __restrict__ target,
                              int S, float* __restrict__ lse_out, float* __restrict__ lp_out) {
    pdl_wait();
    const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (s >= S) return;
    const float2* p = reinterpret_cast<const float2*>(part + (long)s * n_parts * 2);
    // two independent online chains per lane (parts i and i + 32), merged before the shuffles
    float m = -INFINITY, sum = 0.f, m1 = -INFINITY, sum1 = 0.f;
    int i = lane;
    for (; i + 32 < n_parts; i += 64) {
        const float2 v = p[i], w = p[i + 32];
        const float nm = fmaxf(m, v.x), nm1 = fmaxf(m1, w.x);
        if (nm > -INFINITY) sum = sum * __expf(m - nm) + v.y * __expf(v.x - nm);
        if (nm1 > -INFINITY) sum1 = sum1 * __expf(m1 - nm1) + w.y * __expf(w.x - nm1);
        m = nm;
        m1 = nm1;
    }
    if (i < n_parts) {
        const float2 v = p[i];
        const float nm = fmaxf(m, v.x);
        if (nm > -INFINITY) sum = sum * __expf(m - nm) + v.y * __expf(v.x - nm);
        m = nm;
    }
    {
        const float nm = fmaxf(m, m1);
        sum = nm > -INFINITY ? sum * __expf(m - nm) + sum1 * __expf(m1 - nm) : 0.f;
        m = nm;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, sum, o);
        const float nm = fmaxf(m, om);
        sum = nm > -INFINITY ? sum * __expf(m - nm) + os * __expf(om - nm) : 0.f;
        m = nm;
    }
    if (lane == 0) {
        const float lse = m + logf(sum);
        lse_out[s] = lse;
        lp_out[s] = target[s] - lse;
    }
}

// K8a: dZ[s, v] = u[s] * (onehot(label[s]) - exp(z[s, v] - lse[s]))   (model.cpp:637-650)
// grid: (column chunks, rows); 8 columns per thread.
template <class Tin, class Tout>
__global__ void k_softmax_bwd(const Tin* __restrict__ z, long ldz, Tout* __restrict__ dz, long lddz, int S, int V,
                              const float* __restrict__ lse, const float* __restrict__ u,
                              const int32_t* __restrict__ labels) {
    const int s = blockIdx.x;
    const float us = u[s], L = lse[s];
    const int lab = labels[s];
    const Tin* zr = z + (long)s * ldz;
    Tout* dr = dz + (long)s * lddz;
    for (int v0 = (blockIdx.y * blockDim.x + threadIdx.x) * 8; v0 < V; v0 += gridDim.y * blockDim.x * 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int v = v0 + q;
            if (v < V) dr[v] = from_f<Tout>(us * ((v == lab ? 1.f : 0.f) - __expf(to_f<Tin>(zr[v]) - L)));
        }
    }
}

// bf16 -> bf16 variant with 16-byte loads / stores (ldz, lddz, V multiples of 8)
__global__ void k_softmax_bwd_v8(const bf16* z, long ldz, bf16* dz,  // may alias (in place)
                                 long lddz, int S, int V,
                                 const float* __restrict__ lse, const float* __restrict__ u,
                                 const int32_t* __restrict__ labels) {
    pdl_wait();
    const int s = blockIdx.x;
    const float us = u[s], L2 = lse[s] * 1.4426950408889634f;
    const int lab = labels[s];
    const uint4* zr = reinterpret_cast<const uint4*>(z + (long)s * ldz);
    uint4* dr = reinterpret_cast<uint4*>(dz + (long)s * lddz);
    const int n8 = V >> 3;
    for (int c = blockIdx.y * blockDim.x + threadIdx.x; c < n8; c += gridDim.y * blockDim.x) {
        const uint4 in = zr[c];
        const uint32_t w[4] = {in.x, in.y, in.z, in.w};
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int v = 8 * c + 2 * q;
            const float z0 = __uint_as_float(w[q] << 16), z1 = __uint_as_float(w[q] & 0xffff0000u);
            float d0 = -us * exp2f(fmaf(z0, 1.4426950408889634f, -L2));
            float d1 = -us * exp2f(fmaf(z1, 1.4426950408889634f, -L2));
            if (v == lab) d0 += us;
            if (v + 1 == lab) d1 += us;
            __nv_bfloat162 b = __floats2bfloat162_rn(d0, d1);
            o[q] = *reinterpret_cast<uint32_t*>(&b);
        }
        dr[c] = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

// ---------------------------------------------------------------------------
// dx[t] = sum over gathered head rows r owned by position t of dxg[r]  (CSR;
// rows of positions without scored successors are zero).
__global__ void k_scatter_rows(const float* __restrict__ dxg, const int32_t* __restrict__ row_ptr,
                               const int32_t* __restrict__ row_idx, int T, int D, float* __restrict__ dx) {
    const long n = (long)T * D;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const int t = (int)(e / D), i = (int)(e % D);
        float acc = 0.f;
        for (int r = row_ptr[t]; r < row_ptr[t + 1]; ++r) acc += dxg[(long)row_idx[r] * D + i];
        dx[e] = acc;
    }
}

// float4 variant: one warp per position row, its head rows summed in CSR order (as above)
__global__ void __launch_bounds__(256) k_scatter_rows4(const float4* __restrict__ dxg, const int32_t* __restrict__ row_ptr,
                                                       const int32_t* __restrict__ row_idx, int T, int D4,
                                                       float4* __restrict__ dx) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (t >= T) return;
    const int r0 = row_ptr[t], r1 = row_ptr[t + 1];
    for (int c = lane; c < D4; c += 32) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = r0; r < r1; ++r) {
            const float4 v = dxg[(long)row_idx[r] * D4 + c];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        dx[(long)t * D4 + c] = acc;
    }
}

// K11: segmented sum of dx rows over runs of equal keys (keys sorted stably,
// so each run lists its rows in position order): grad[key] += sum dx[idx].
__global__ void k_embed_grad(const int32_t* __restrict__ keys, const int32_t* __restrict__ idx, int T,
                             const float* __restrict__ dx, int D, float* __restrict__ grad) {
    const int i = blockIdx.x;
    if (i >= T) return;
    const int key = keys[i];
    if (i > 0 && keys[i - 1] == key) return;  // not a run start
    int end = i + 1;
    while (end < T && keys[end] == key) ++end;
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
        float acc = 0.f;
        for (int r = i; r < end; ++r) acc += dx[(long)idx[r] * D + c];
        grad[(long)key * D + c] += acc;
    }
}

// ---------------------------------------------------------------------------
// conversions
template <class T>
__global__ void k_f32_to_act(const float* __restrict__ x, T* __restrict__ y, long n) {
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x)
        y[e] = from_f<T>(x[e]);
}

// src fp64 [rows x cols] (row-major) -> dst [rows x cols] (transposed=0) or
// [cols x rows] (transposed=1) in dtype T, with dst leading dimension ldd.
template <class T>
__global__ void k_convert_w(const double* __restrict__ src, int rows, int cols, T* __restrict__ dst, long ldd,
                            int transposed) {
    __shared__ float tile[32][33];
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = (float)src[(long)r * cols + c];
    }
    __syncthreads();
    if (!transposed) {
        for (int i = threadIdx.y; i < 32; i += blockDim.y) {
            const int r = r0 + i, c = c0 + threadIdx.x;
            if (r < rows && c < cols) dst[(long)r * ldd + c] = from_f<T>(tile[i][threadIdx.x]);
        }
    } else {
        for (int i = threadIdx.y; i < 32; i += blockDim.y) {
            const int c = c0 + i, r = r0 + threadIdx.x;
            if (r < rows && c < cols) dst[(long)c * ldd + r] = from_f<T>(tile[threadIdx.x][i]);
        }
    }
}

// reverse of the above into fp64 (model download)
template <class T>
__global__ void k_export_w(const T* __restrict__ src, long lds, int rows, int cols, int transposed,
                           double* __restrict__ dst) {
    const long n = (long)rows * cols;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const int r = (int)(e / cols), c = (int)(e % cols);
        dst[e] = (double)to_f<T>(transposed ? src[(long)c * lds + r] : src[(long)r * lds + c]);
    }
}

__global__ void k_f32_to_f64(const float* __restrict__ x, double* __restrict__ y, long n) {
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) y[e] = x[e];
}

// Philox-based N(0,1) * scale (+ base): device init of large configs.
__device__ __forceinline__ uint2 philox(uint2 ctr, uint32_t key_lo, uint32_t key_hi, uint32_t c2) {
    uint32_t c0 = ctr.x, c1 = ctr.y, k0 = key_lo, k1 = key_hi, cc2 = c2, c3 = 0;
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * cc2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        cc2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return make_uint2(c0, cc2);
}

__global__ void k_randn(double* out, long n, uint64_t seed, uint32_t stream, double scale,
                        const double* base) {
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const uint2 r = philox(make_uint2((uint32_t)e, (uint32_t)(e >> 32)), (uint32_t)seed, (uint32_t)(seed >> 32),
                               stream);
        const double u1 = ((r.x >> 8) + 1.0) * (1.0 / 16777217.0), u2 = (r.y >> 8) * (1.0 / 16777216.0);
        const double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
        out[e] = (base ? base[e] : 0.0) + scale * z;
    }
}

__global__ void k_fill_f64(double* __restrict__ out, long n, double v) {
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) out[e] = v;
}

__global__ void k_axpy(const float* __restrict__ x, float* __restrict__ y, long n) {
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) y[e] += x[e];
}

// apply_update (model.cpp:202-219): flag non-finite gradients / results.
__global__ void k_sgd_check(const float* __restrict__ g, const double* __restrict__ w, long n, double scale,
                            int* __restrict__ flags) {
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        if (!isfinite(g[e])) atomicOr(flags, 1);
        else if (!isfinite(w[e] - scale * (double)g[e])) atomicOr(flags, 2);
    }
}
__global__ void k_sgd_apply(const float* __restrict__ g, double* __restrict__ w, long n, double scale) {
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x)
        w[e] -= scale * (double)g[e];
}

// ---------------------------------------------------------------------------
// launchers
static int grid_for(long n, int bs = 256) {
    long g = (n + bs - 1) / bs;
    return (int)(g < 148L * 16 ? (g < 1 ? 1 : g) : 148L * 16);
}

// dense shared-prompt mask (build_shared_prompt_mask, packing.cpp:47-72) from the segment ids
__global__ void k_allowed_mask(const int32_t* __restrict__ seg, int n, uint8_t* __restrict__ mask) {
    const long nn = (long)n * n;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < nn; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e / n), j = (int)(e % n);
        const int si = seg[i], sj = seg[j];
        mask[e] = si == 0 ? (sj == 0 && j <= i) : (sj == 0 || (sj == si && j <= i));
    }
}

void launch_allowed_mask(const int32_t* seg, int n, uint8_t* mask, cudaStream_t st) {
    k_allowed_mask<<<grid_for((long)n * n), 256, 0, st>>>(seg, n, mask);
    PARL_LAUNCHED();
}

void launch_pack_multi(const int32_t* prompts, const int32_t* resp, const int32_t* tables, int n, int n_resp, int T,
                       const PackedDev& pk, unsigned* id_max, cudaStream_t st) {
    // tables: gstart [n + 1] | pstart [n] | r0 [n + 1] | rcu [n_resp + 1] | rstart [n_resp]
    const int32_t* gstart = tables;
    const int32_t* pstart = gstart + n + 1;
    const int32_t* r0 = pstart + n;
    const int32_t* rcu = r0 + n + 1;
    const int32_t* rstart = rcu + n_resp + 1;
    if (id_max) PARL_CUDA(cudaMemsetAsync(id_max, 0, sizeof(unsigned), st));
    k_pack_multi<<<grid_for(T), 256, 0, st>>>(prompts, resp, gstart, pstart, r0, rcu, rstart, n, pk, id_max);
    PARL_LAUNCHED();
}

void launch_pack(const int32_t* prompt, int P, const int32_t* resp, const int32_t* cu, int G, int T,
                 const PackedDev& pk, unsigned* id_max, cudaStream_t st) {
    if (id_max) PARL_CUDA(cudaMemsetAsync(id_max, 0, sizeof(unsigned), st));
    if (P & 3) k_pack_scalar<<<grid_for(T), 256, 0, st>>>(prompt, P, resp, cu, G, pk, id_max);
    else k_pack<<<grid_for(cdiv(T, 4)), 256, 0, st>>>(prompt, P, resp, cu, G, pk, id_max);
    PARL_LAUNCHED();
}

void launch_embed(const float* tok, const float* pos, const int32_t* tokens, const int32_t* positions, int T, int D,
                  float* x, cudaStream_t st) {
    const bool v4 = D % 4 == 0 && ((reinterpret_cast<uintptr_t>(tok) | reinterpret_cast<uintptr_t>(pos) |
                                    reinterpret_cast<uintptr_t>(x)) & 15) == 0;
    if (v4)
        k_embed4<<<cdiv(T, 8), 256, 0, st>>>(reinterpret_cast<const float4*>(tok), reinterpret_cast<const float4*>(pos),
                                             tokens, positions, T, D / 4, reinterpret_cast<float4*>(x));
    else
        k_embed<<<grid_for((long)T * D), 256, 0, st>>>(tok, pos, tokens, positions, T, D, x);
    PARL_LAUNCHED();
}

// float4 variant (D % 4 == 0): every load of the row is issued before any use
template <class T>
__device__ __forceinline__ void store4(T* p, float4 v);
template <>
__device__ __forceinline__ void store4<float>(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
template <>
__device__ __forceinline__ void store4<bf16>(bf16* p, float4 v) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(p) = u;
}

// float4 variant of the forward (D % 4 == 0, 16-byte aligned rows): one warp per row
template <class T, int P4>
__device__ __forceinline__ void ln4_row(const float* __restrict__ x, const int32_t* __restrict__ rows, int r, int D,
                                        const float* __restrict__ gamma, const float* __restrict__ beta,
                                        T* __restrict__ y, long ldy, float* __restrict__ mean_out,
                                        float* __restrict__ rstd_out) {
    const int lane = threadIdx.x & 31;
    const int D4 = D >> 2;
    const float4* xr = reinterpret_cast<const float4*>(x + (long)(rows ? rows[r] : r) * D);
    float4 v[P4];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < P4; ++k) {
        const int c = lane + 32 * k;
        v[k] = c < D4 ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
        s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
    }
    const float mean = warp_sum(s) / D;
    float var = 0.f;
#pragma unroll
    for (int k = 0; k < P4; ++k) {
        const int c = lane + 32 * k;
        if (c < D4) {
            const float a = v[k].x - mean, b = v[k].y - mean, cc = v[k].z - mean, d = v[k].w - mean;
            var += (a * a + b * b) + (cc * cc + d * d);
        }
    }
    const float rstd = rsqrtf(warp_sum(var) / D + 1e-5f);
    T* yr = y + (long)r * ldy;
#pragma unroll
    for (int k = 0; k < P4; ++k) {
        const int c = lane + 32 * k;
        if (c < D4) {
            const float4 g = __ldg(reinterpret_cast<const float4*>(gamma) + c);
            const float4 b = __ldg(reinterpret_cast<const float4*>(beta) + c);
            float4 o;
            o.x = (v[k].x - mean) * rstd * g.x + b.x;
            o.y = (v[k].y - mean) * rstd * g.y + b.y;
            o.z = (v[k].z - mean) * rstd * g.z + b.z;
            o.w = (v[k].w - mean) * rstd * g.w + b.w;
            store4<T>(yr + 4 * c, o);
        }
    }
    if (lane == 0) {
        mean_out[r] = mean;
        rstd_out[r] = rstd;
    }
}

template <class T, int P4>
__global__ void __launch_bounds__(256) k_layernorm4(const float* __restrict__ x, const int32_t* __restrict__ rows,
                                                    int R, int D, const float* __restrict__ gamma,
                                                    const float* __restrict__ beta, T* __restrict__ y, long ldy,
                                                    float* __restrict__ mean_out, float* __restrict__ rstd_out) {
    pdl_wait();
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= R) return;
    ln4_row<T, P4>(x, rows, r, D, gamma, beta, y, ldy, mean_out, rstd_out);
}

// the same LayerNorm of up to three models (tri-model forward) in one launch: blockIdx.y = model
template <class T>
struct LnMulti {
    const float* x[3];
    const float *g[3], *b[3];
    T* y[3];
    float *mean[3], *rstd[3];
};
template <class T, int P4>
__global__ void __launch_bounds__(256) k_layernorm4_multi(const __grid_constant__ LnMulti<T> a, int R, int D, long ldy) {
    pdl_wait();
    // persistent warps over rows; the next row is pulled into L2 while this one is normalised
    const int m = blockIdx.y, lane = threadIdx.x & 31, rstep = gridDim.x * 8;
    for (int r = blockIdx.x * 8 + (threadIdx.x >> 5); r < R; r += rstep) {
        if (r + rstep < R) {
            const float* nx = a.x[m] + (long)(r + rstep) * D;
            for (int c = lane * 32; c < D; c += 32 * 32) prefetch_l2(nx + c);
        }
        ln4_row<T, P4>(a.x[m], nullptr, r, D, a.g[m], a.b[m], a.y[m], ldy, a.mean[m], a.rstd[m]);
    }
}

// resident blocks per SM of k_layernorm4_multi<T, P4>
template <class T, int P4>
int ln_multi_occupancy() {
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_layernorm4_multi<T, P4>, 256, 0);
        if (occ <= 0) occ = 1;
    }
    return occ;
}

template <class T>
void launch_layernorm(const float* x, const int32_t* rows, int R, int D, const float* g, const float* b, T* y,
                      long ldy, float* mean, float* rstd, cudaStream_t st) {
    if (R <= 0) return;
    const bool v4 = D % 4 == 0 && (ldy * (long)sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0;
    if (v4 && D <= 512) launch_pdl(k_layernorm4<T, 4>, dim3(cdiv(R, 8)), dim3(256), 0, st, x, rows, R, D, g, b, y, ldy, mean, rstd);
    else if (v4 && D <= 896) launch_pdl(k_layernorm4<T, 7>, dim3(cdiv(R, 8)), dim3(256), 0, st, x, rows, R, D, g, b, y, ldy, mean, rstd);
    else if (v4 && D <= 1024) launch_pdl(k_layernorm4<T, 8>, dim3(cdiv(R, 8)), dim3(256), 0, st, x, rows, R, D, g, b, y, ldy, mean, rstd);
    else if (v4 && D <= 1536) launch_pdl(k_layernorm4<T, 12>, dim3(cdiv(R, 8)), dim3(256), 0, st, x, rows, R, D, g, b, y, ldy, mean, rstd);
    else if (v4 && D <= 2048) launch_pdl(k_layernorm4<T, 16>, dim3(cdiv(R, 8)), dim3(256), 0, st, x, rows, R, D, g, b, y, ldy, mean, rstd);
    else if (v4 && D <= 3584) launch_pdl(k_layernorm4<T, 28>, dim3(cdiv(R, 8)), dim3(256), 0, st, x, rows, R, D, g, b, y, ldy, mean, rstd);
    else if (v4 && D <= 4096) launch_pdl(k_layernorm4<T, 32>, dim3(cdiv(R, 8)), dim3(256), 0, st, x, rows, R, D, g, b, y, ldy, mean, rstd);
    else if (D <= 256) k_layernorm<T, 8><<<cdiv(R, 8), 256, 0, st>>>(x, rows, R, D, g, b, y, ldy, mean, rstd);
    else if (D <= 1024) k_layernorm<T, 32><<<cdiv(R, 8), 256, 0, st>>>(x, rows, R, D, g, b, y, ldy, mean, rstd);
    else if (D <= 2048) k_layernorm<T, 64><<<cdiv(R, 8), 256, 0, st>>>(x, rows, R, D, g, b, y, ldy, mean, rstd);
    else k_layernorm<T, 0><<<cdiv(R, 8), 256, 0, st>>>(x, rows, R, D, g, b, y, ldy, mean, rstd);
    PARL_LAUNCHED();
}
template void launch_layernorm<float>(const float*, const int32_t*, int, int, const float*, const float*, float*,
                                      long, float*, float*, cudaStream_t);
template void launch_layernorm<bf16>(const float*, const int32_t*, int, int, const float*, const float*, bf16*,
                                     long, float*, float*, cudaStream_t);

// LayerNorm backward (model.cpp:319-343 reversed), input part: one warp per row
// with the row held in registers: dx = (res) + rstd (dxh - mean(dxh) - xhat mean(dxh xhat)),
// dxh = dy gamma, plus an optional compute-dtype copy of dx (the next GEMM's
// operand).  The gamma / beta gradients are column sums done by colsum_impl
// (mode 1) in a fixed order.
template <class T, int PER>
__global__ void __launch_bounds__(256) k_ln_bwd_rows(const float* __restrict__ dy, const float* __restrict__ x,
                                                     const int32_t* __restrict__ rows, const float* __restrict__ mean,
                                                     const float* __restrict__ rstd, const float* __restrict__ gamma,
                                                     int R, int D, const float* __restrict__ res,
                                                     float* __restrict__ dx, T* __restrict__ dx_act) {
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (r >= R) return;
    const float* xr = x + (long)(rows ? rows[r] : r) * D;
    const float* dyr = dy + (long)r * D;
    const float mu = mean[r], rs = rstd[r];
    float vy[PER], xh[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int i = lane + 32 * q;
        vy[q] = i < D ? dyr[i] * __ldg(gamma + i) : 0.f;
        xh[q] = i < D ? (xr[i] - mu) * rs : 0.f;
    }
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        sa += vy[q];
        sb += vy[q] * xh[q];
    }
    sa = warp_sum(sa) / D;
    sb = warp_sum(sb) / D;
    float* o = dx + (long)r * D;
    const float* rr = res ? res + (long)r * D : nullptr;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int i = lane + 32 * q;
        if (i < D) {
            float v = rs * (vy[q] - sa - xh[q] * sb);
            if (rr) v += rr[i];
            o[i] = v;
            if (dx_act) dx_act[(long)r * D + i] = from_f<T>(v);
        }
    }
}

template <class T>
void launch_layernorm_multi(int nm, const float* const* x, const float* const* g, const float* const* b, T* const* y,
                            long ldy, float* const* mean, float* const* rstd, int R, int D, cudaStream_t st) {
    if (R <= 0) return;
    bool v4 = D % 4 == 0 && (ldy * (long)sizeof(T)) % 16 == 0 && nm >= 1 && nm <= 3;
    for (int k = 0; k < nm; ++k) v4 = v4 && (reinterpret_cast<uintptr_t>(y[k]) & 15) == 0;
    if (!v4 || D > 4096) {
        for (int k = 0; k < nm; ++k) launch_layernorm<T>(x[k], nullptr, R, D, g[k], b[k], y[k], ldy, mean[k], rstd[k], st);
        return;
    }
    LnMulti<T> a;
    for (int k = 0; k < nm; ++k) {
        a.x[k] = x[k]; a.g[k] = g[k]; a.b[k] = b[k]; a.y[k] = y[k]; a.mean[k] = mean[k]; a.rstd[k] = rstd[k];
    }
    // all blocks resident at once, split evenly over the models
#define PARL_LN_MULTI(P4)                                                                                  \
    do {                                                                                                   \
        const int gx = std::min(cdiv(R, 8), std::max(1, ln_multi_occupancy<T, P4>() * num_sms() / nm)); \
        launch_pdl(k_layernorm4_multi<T, P4>, dim3(gx, nm), dim3(256), 0, st, a, R, D, ldy);            \
    } while (0)
    if (D <= 512) PARL_LN_MULTI(4);
    else if (D <= 896) PARL_LN_MULTI(7);
    else if (D <= 1024) PARL_LN_MULTI(8);
    else if (D <= 1536) PARL_LN_MULTI(12);
    else if (D <= 2048) PARL_LN_MULTI(16);
    else if (D <= 3584) PARL_LN_MULTI(28);
    else PARL_LN_MULTI(32);
#undef PARL_LN_MULTI
    PARL_LAUNCHED();
}
template void launch_layernorm_multi<float>(int, const float* const*, const float* const*, const float* const*,
                                            float* const*, long, float* const*, float* const*, int, int, cudaStream_t);
template void launch_layernorm_multi<bf16>(int, const float* const*, const float* const*, const float* const*,
                                           bf16* const*, long, float* const*, float* const*, int, int, cudaStream_t);

template <class T, int P4>
__global__ void __launch_bounds__(256) k_ln_bwd_rows4(const float* __restrict__ dy, const float* __restrict__ x,
                                                      const int32_t* __restrict__ rows, const float* __restrict__ mean,
                                                      const float* __restrict__ rstd, const float* __restrict__ gamma,
                                                      int R, int D, const float* __restrict__ res,
                                                      float* __restrict__ dx, T* __restrict__ dx_act) {
    pdl_wait();
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (r >= R) return;
    const int D4 = D >> 2;
    const float4* xr = reinterpret_cast<const float4*>(x + (long)(rows ? rows[r] : r) * D);
    const float4* dyr = reinterpret_cast<const float4*>(dy + (long)r * D);
    const float4* rr = res ? reinterpret_cast<const float4*>(res + (long)r * D) : nullptr;
    const float4* g4 = reinterpret_cast<const float4*>(gamma);
    float4 vy[P4], vx[P4], vr[P4];
#pragma unroll
    for (int k = 0; k < P4; ++k) {
        const int c = lane + 32 * k;
        const bool ok = c < D4;
        vy[k] = ok ? dyr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
        vx[k] = ok ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
        vr[k] = (ok && rr) ? rr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float mu = mean[r], rs = rstd[r];
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int k = 0; k < P4; ++k) {
        const int c = lane + 32 * k;
        const float4 g = c < D4 ? __ldg(g4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        vy[k].x *= g.x; vy[k].y *= g.y; vy[k].z *= g.z; vy[k].w *= g.w;  // dxh
        vx[k].x = (vx[k].x - mu) * rs; vx[k].y = (vx[k].y - mu) * rs;     // xhat
        vx[k].z = (vx[k].z - mu) * rs; vx[k].w = (vx[k].w - mu) * rs;
        sa += (vy[k].x + vy[k].y) + (vy[k].z + vy[k].w);
        sb += (vy[k].x * vx[k].x + vy[k].y * vx[k].y) + (vy[k].z * vx[k].z + vy[k].w * vx[k].w);
    }
    sa = warp_sum(sa) / D;
    sb = warp_sum(sb) / D;
#pragma unroll
    for (int k = 0; k < P4; ++k) {
        const int c = lane + 32 * k;
        if (c < D4) {
            float4 v;
            v.x = rs * (vy[k].x - sa - vx[k].x * sb) + vr[k].x;
            v.y = rs * (vy[k].y - sa - vx[k].y * sb) + vr[k].y;
            v.z = rs * (vy[k].z - sa - vx[k].z * sb) + vr[k].z;
            v.w = rs * (vy[k].w - sa - vx[k].w * sb) + vr[k].w;
            reinterpret_cast<float4*>(dx + (long)r * D)[c] = v;
            if (dx_act) store4<T>(dx_act + (long)r * D + 4 * c, v);
        }
    }
}

// LayerNorm backward with the gamma / beta gradients fused (d <= 1024): persistent warps
// over rows accumulate dgamma = sum dy * xhat and dbeta = sum dy for their lane's columns
// in registers; each block then reduces its 8 warps in shared memory and writes one
// partial row (k_colsum_final adds the partials in block order: deterministic).
template <class T, int P4>
__global__ void __launch_bounds__(256) k_ln_bwd_rows4_cs(const float* __restrict__ dy, const float* __restrict__ x,
                                                       const int32_t* __restrict__ rows, const float* __restrict__ mean,
                                                       const float* __restrict__ rstd, const float* __restrict__ gamma,
                                                       int R, int D, const float* __restrict__ res,
                                                       float* __restrict__ dx, T* __restrict__ dx_act,
                                                       float* __restrict__ part_a, float* __restrict__ part_b) {
    // per-warp column partials in shared memory: [2][8 warps][D / 4] float4 (each element owned by one lane)
    extern __shared__ float4 red[];
    pdl_wait();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int D4 = D >> 2;
    float4* sga = red + wib * D4;
    float4* sgb = red + (8 + wib) * D4;
    for (int c = lane; c < D4; c += 32) sga[c] = sgb[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* g4 = reinterpret_cast<const float4*>(gamma);
    const int rstep = gridDim.x * 8;
    for (int r = blockIdx.x * 8 + wib; r < R; r += rstep) {
        const float4* xr = reinterpret_cast<const float4*>(x + (long)(rows ? rows[r] : r) * D);
        const float4* dyr = reinterpret_cast<const float4*>(dy + (long)r * D);
        // L2 prefetch of this row's residual gradient (read after the row reduction) and of
        // the next row's dy / x: one DRAM latency per row overlaps the current row's work
        if (res) {
            const float* rp = res + (long)r * D;
            for (int c = lane * 32; c < D; c += 32 * 32) prefetch_l2(rp + c);
        }
        if (r + rstep < R) {
            const float* np = dy + (long)(r + rstep) * D;
            const float* nx = x + (long)(rows ? rows[r + rstep] : r + rstep) * D;
            for (int c = lane * 32; c < D; c += 32 * 32) {
                prefetch_l2(np + c);
                prefetch_l2(nx + c);
            }
        }
        float4 vy[P4], vx[P4];
#pragma unroll
        for (int k = 0; k < P4; ++k) {
            const int c = lane + 32 * k;
            const bool ok = c < D4;
            vy[k] = ok ? dyr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
            vx[k] = ok ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        const float mu = mean[r], rs = rstd[r];
        float sa = 0.f, sb = 0.f;
#pragma unroll
        for (int k = 0; k < P4; ++k) {
            const int c = lane + 32 * k;
            vx[k].x = (vx[k].x - mu) * rs; vx[k].y = (vx[k].y - mu) * rs;     // xhat
            vx[k].z = (vx[k].z - mu) * rs; vx[k].w = (vx[k].w - mu) * rs;
            if (c < D4) {
                const float4 g = __ldg(g4 + c);
                float4 a = sga[c], b = sgb[c];
                a.x += vy[k].x * vx[k].x; a.y += vy[k].y * vx[k].y;           // dgamma
                a.z += vy[k].z * vx[k].z; a.w += vy[k].w * vx[k].w;
                b.x += vy[k].x; b.y += vy[k].y; b.z += vy[k].z; b.w += vy[k].w;  // dbeta
                sga[c] = a;
                sgb[c] = b;
                vy[k].x *= g.x; vy[k].y *= g.y; vy[k].z *= g.z; vy[k].w *= g.w;  // dxh
            }
            sa += (vy[k].x + vy[k].y) + (vy[k].z + vy[k].w);
            sb += (vy[k].x * vx[k].x + vy[k].y * vx[k].y) + (vy[k].z * vx[k].z + vy[k].w * vx[k].w);
        }
        sa = warp_sum(sa) / D;
        sb = warp_sum(sb) / D;
        const float4* rr = res ? reinterpret_cast<const float4*>(res + (long)r * D) : nullptr;
#pragma unroll
        for (int k = 0; k < P4; ++k) {
            const int c = lane + 32 * k;
            if (c < D4) {
                const float4 rv = rr ? rr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
                float4 v;
                v.x = rs * (vy[k].x - sa - vx[k].x * sb) + rv.x;
                v.y = rs * (vy[k].y - sa - vx[k].y * sb) + rv.y;
                v.z = rs * (vy[k].z - sa - vx[k].z * sb) + rv.z;
                v.w = rs * (vy[k].w - sa - vx[k].w * sb) + rv.w;
                reinterpret_cast<float4*>(dx + (long)r * D)[c] = v;
                if (dx_act) store4<T>(dx_act + (long)r * D + 4 * c, v);
            }
        }
    }
    __syncthreads();
    // block reduction over the 8 warps, in warp order
    for (int c = threadIdx.x; c < 2 * D4; c += 256) {
        const int pass = c >= D4, cc = c - pass * D4;
        const float4* src = red + pass * 8 * D4 + cc;
        float4 t = src[0];
#pragma unroll
        for (int q = 1; q < 8; ++q) {
            const float4 u = src[q * D4];
            t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
        }
        reinterpret_cast<float4*>((pass ? part_b : part_a) + (long)blockIdx.x * D)[cc] = t;
    }
}

// resident blocks per SM of the fused kernel (registers / shared memory bound)
template <class T, int P4>
int ln_bwd_cs_occupancy(int D) {
    static int occ[2] = {0, 0};
    static int last_d = -1;
    if (last_d != D) {
        cudaFuncSetAttribute(k_ln_bwd_rows4_cs<T, P4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 8 * 256 * 16);
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_ln_bwd_rows4_cs<T, P4>, 256, (size_t)2 * 8 * (D / 4) * 16);
        occ[0] = n > 0 ? n : 1;
        last_d = D;
    }
    return occ[0];
}

// out[c] += sum_s part_a[s][c] (out2 likewise) for many partial rows: 8 columns x 32 row
// groups per block (enough blocks to cover the SMs at d ~ 1k), the groups combined in a
// fixed order (deterministic)
__global__ void __launch_bounds__(256) k_colsum_final8(const float* __restrict__ part_a, const float* __restrict__ part_b,
                                                      int splits, int N, float* __restrict__ out, float* __restrict__ out2) {
    __shared__ float sa[32][9], sb[32][9];
    pdl_wait();
    const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
    const int c = blockIdx.x * 8 + tx;
    float a = 0.f, b = 0.f;
    if (c < N) {
#pragma unroll 4
        for (int s0 = ty; s0 < splits; s0 += 32) {
            a += part_a[(long)s0 * N + c];
            b += part_b[(long)s0 * N + c];
        }
    }
    sa[ty][tx] = a;
    sb[ty][tx] = b;
    __syncthreads();
    if (ty == 0 && c < N) {
        float ta = 0.f, tb = 0.f;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            ta += sa[q][tx];
            tb += sb[q][tx];
        }
        out[c] += ta;
        out2[c] += tb;
    }
}

template <class T, int P4>
void launch_ln_bwd_cs(const float* dy, const float* x, const int32_t* rows, const float* mean, const float* rstd,
                      const float* gamma, int R, int D, const float* res, float* dx, T* dx_act, float* pa, float* pb,
                      int grid, cudaStream_t st) {
    const size_t smem = (size_t)2 * 8 * (D / 4) * 16;
    launch_pdl(k_ln_bwd_rows4_cs<T, P4>, dim3(grid), dim3(256), smem, st, dy, x, rows, mean, rstd, gamma, R, D, res, dx,
               dx_act, pa, pb);
    PARL_LAUNCHED();
}

// Wide rows (d > 1024: C3 / C4): the same math in two passes over the row (sums, then
// outputs), so nothing is held in registers; the second pass re-reads dy / x from L2.
template <class T>
__global__ void __launch_bounds__(256) k_ln_bwd_rows4_2p(const float* __restrict__ dy, const float* __restrict__ x,
                                                         const int32_t* __restrict__ rows, const float* __restrict__ mean,
                                                         const float* __restrict__ rstd, const float* __restrict__ gamma,
                                                         int R, int D, const float* __restrict__ res,
                                                         float* __restrict__ dx, T* __restrict__ dx_act) {
    pdl_wait();
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (r >= R) return;
    const int D4 = D >> 2;
    const float4* xr = reinterpret_cast<const float4*>(x + (long)(rows ? rows[r] : r) * D);
    const float4* dyr = reinterpret_cast<const float4*>(dy + (long)r * D);
    const float4* rr = res ? reinterpret_cast<const float4*>(res + (long)r * D) : nullptr;
    const float4* g4 = reinterpret_cast<const float4*>(gamma);
    const float mu = mean[r], rs = rstd[r];
    float sa = 0.f, sb = 0.f;
#pragma unroll 4
    for (int c = lane; c < D4; c += 32) {
        const float4 g = __ldg(g4 + c), yv = dyr[c], xv = xr[c];
        const float a0 = yv.x * g.x, a1 = yv.y * g.y, a2 = yv.z * g.z, a3 = yv.w * g.w;
        sa += (a0 + a1) + (a2 + a3);
        sb += (a0 * (xv.x - mu) + a1 * (xv.y - mu)) + (a2 * (xv.z - mu) + a3 * (xv.w - mu));
    }
    sa = warp_sum(sa) / D;
    sb = warp_sum(sb) * rs / D;
#pragma unroll 4
    for (int c = lane; c < D4; c += 32) {
        const float4 g = __ldg(g4 + c), yv = dyr[c], xv = xr[c];
        const float4 rv = rr ? rr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 v;
        v.x = rs * (yv.x * g.x - sa - (xv.x - mu) * rs * sb) + rv.x;
        v.y = rs * (yv.y * g.y - sa - (xv.y - mu) * rs * sb) + rv.y;
        v.z = rs * (yv.z * g.z - sa - (xv.z - mu) * rs * sb) + rv.z;
        v.w = rs * (yv.w * g.w - sa - (xv.w - mu) * rs * sb) + rv.w;
        reinterpret_cast<float4*>(dx + (long)r * D)[c] = v;
        if (dx_act) store4<T>(dx_act + (long)r * D + 4 * c, v);
    }
}

template <class T>
void launch_layernorm_bwd(const float* dy, const float* x, const int32_t* rows, const float* mean, const float* rstd,
                          const float* gamma, int R, int D, const float* res, float* dx, T* dx_act, float* dgamma,
                          float* dbeta, cudaStream_t st) {
    if (R <= 0) return;
    const int blocks = cdiv(R, 8);
    static const bool fused = [] {
        const char* e = std::getenv("PARL_LN_FUSED");
        return !(e && e[0] == '0');
    }();
    if (fused && D % 4 == 0 && D <= 1024) {
        // fused dgamma / dbeta: persistent blocks (all resident at once), one partial row per block
        const int occ = D <= 512 ? ln_bwd_cs_occupancy<T, 4>(D) : D <= 896 ? ln_bwd_cs_occupancy<T, 7>(D)
                                                                            : ln_bwd_cs_occupancy<T, 8>(D);
        const int grid = std::min(blocks, occ * num_sms());
        float* pa = g_colsum_scratch.get((size_t)2 * grid * D);
        float* pb = pa + (size_t)grid * D;
        if (D <= 512) launch_ln_bwd_cs<T, 4>(dy, x, rows, mean, rstd, gamma, R, D, res, dx, dx_act, pa, pb, grid, st);
        else if (D <= 896) launch_ln_bwd_cs<T, 7>(dy, x, rows, mean, rstd, gamma, R, D, res, dx, dx_act, pa, pb, grid, st);
        else launch_ln_bwd_cs<T, 8>(dy, x, rows, mean, rstd, gamma, R, D, res, dx, dx_act, pa, pb, grid, st);
        launch_pdl(k_colsum_final8, dim3(cdiv(D, 8)), dim3(256), 0, st, (const float*)pa, (const float*)pb, grid, D,
                   dgamma, dbeta);
        PARL_LAUNCHED();
        return;
    }
    if (D % 4 == 0 && D <= 1024) {
        if (D <= 512) launch_pdl(k_ln_bwd_rows4<T, 4>, dim3(blocks), dim3(256), 0, st, dy, x, rows, mean, rstd, gamma, R, D, res, dx, dx_act);
        else if (D <= 896) launch_pdl(k_ln_bwd_rows4<T, 7>, dim3(blocks), dim3(256), 0, st, dy, x, rows, mean, rstd, gamma, R, D, res, dx, dx_act);
        else launch_pdl(k_ln_bwd_rows4<T, 8>, dim3(blocks), dim3(256), 0, st, dy, x, rows, mean, rstd, gamma, R, D, res, dx, dx_act);
    } else if (D % 4 == 0) {
        launch_pdl(k_ln_bwd_rows4_2p<T>, dim3(blocks), dim3(256), 0, st, dy, x, rows, mean, rstd, gamma, R, D, res, dx,
                   dx_act);
    } else if (D <= 256) k_ln_bwd_rows<T, 8><<<blocks, 256, 0, st>>>(dy, x, rows, mean, rstd, gamma, R, D, res, dx, dx_act);
    else if (D <= 512) k_ln_bwd_rows<T, 16><<<blocks, 256, 0, st>>>(dy, x, rows, mean, rstd, gamma, R, D, res, dx, dx_act);
    else if (D <= 768) k_ln_bwd_rows<T, 24><<<blocks, 256, 0, st>>>(dy, x, rows, mean, rstd, gamma, R, D, res, dx, dx_act);
    else if (D <= 896) k_ln_bwd_rows<T, 28><<<blocks, 256, 0, st>>>(dy, x, rows, mean, rstd, gamma, R, D, res, dx, dx_act);
    else if (D <= 1024) k_ln_bwd_rows<T, 32><<<blocks, 256, 0, st>>>(dy, x, rows, mean, rstd, gamma, R, D, res, dx, dx_act);
    else {
        k_layernorm_bwd<<<blocks, 256, 0, st>>>(dy, x, rows, mean, rstd, gamma, R, D, res, dx);
        PARL_LAUNCHED();
        if (dx_act) launch_f32_to_act<T>(dx, dx_act, (size_t)R * D, st);
        colsum_impl<float>(dy, D, R, D, dgamma, x, rows, mean, rstd, dbeta, 1, st);
        return;
    }
    PARL_LAUNCHED();
    colsum_impl<float>(dy, D, R, D, dgamma, x, rows, mean, rstd, dbeta, 1, st);
}
template void launch_layernorm_bwd<float>(const float*, const float*, const int32_t*, const float*, const float*,
                                          const float*, int, int, const float*, float*, float*, float*, float*,
                                          cudaStream_t);
template void launch_layernorm_bwd<bf16>(const float*, const float*, const int32_t*, const float*, const float*,
                                         const float*, int, int, const float*, float*, bf16*, float*, float*,
                                         cudaStream_t);

// pad columns [D, ld) of every row: 1 at column D (bias row of a weight-gradient
// GEMM), 0 after it
template <class T>
__global__ void k_fill_pad(T* __restrict__ y, long rows, int D, long ld) {
    const long n = rows * (ld - D);
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const long r = e / (ld - D);
        const int c = (int)(e % (ld - D));
        y[r * ld + D + c] = from_f<T>(c == 0 ? 1.f : 0.f);
    }
}
template <class T>
void launch_fill_pad(T* y, long rows, int D, long ld, cudaStream_t st) {
    if (rows <= 0 || ld <= D) return;
    k_fill_pad<T><<<grid_for(rows * (ld - D)), 256, 0, st>>>(y, rows, D, ld);
    PARL_LAUNCHED();
}
template void launch_fill_pad<float>(float*, long, int, long, cudaStream_t);
template void launch_fill_pad<bf16>(bf16*, long, int, long, cudaStream_t);

template <class T>
void launch_colsum(const T* X, long ldx, int R, int N, float* out, cudaStream_t st) {
    if (R <= 0) return;
    colsum_impl<T>(X, ldx, R, N, out, nullptr, nullptr, nullptr, nullptr, nullptr, 0, st);
}
template void launch_colsum<float>(const float*, long, int, int, float*, cudaStream_t);
template void launch_colsum<bf16>(const bf16*, long, int, int, float*, cudaStream_t);

void launch_row_lse(const float* z, int S, int V, const int32_t* labels, float* lse, float* lp, cudaStream_t st) {
    if (S <= 0) return;
    k_row_lse<<<S, 256, 0, st>>>(z, V, labels, lse, lp);
    PARL_LAUNCHED();
}

void launch_lse_combine(const float* part, int n_parts, const float* target, int S, float* lse, float* lp,
                        cudaStream_t st) {
    if (S <= 0) return;
    launch_pdl(k_lse_combine, dim3(cdiv(S, 8)), dim3(256), 0, st, (const float*)part, n_parts, target, S, lse, lp);
    PARL_LAUNCHED();
}

template <class Tin, class Tout>
void launch_softmax_bwd(const Tin* z, long ldz, Tout* dz, long lddz, int S, int V, const float* lse, const float* u,
                        const int32_t* labels, cudaStream_t st) {
    if (S <= 0) return;
    const int cx = std::max(1, std::min(cdiv(V, 256 * 8), 8));
    if constexpr (std::is_same_v<Tin, bf16> && std::is_same_v<Tout, bf16>) {
        if (V % 8 == 0 && ldz % 8 == 0 && lddz % 8 == 0 && (reinterpret_cast<uintptr_t>(z) & 15) == 0 &&
            (reinterpret_cast<uintptr_t>(dz) & 15) == 0) {
            launch_pdl(k_softmax_bwd_v8, dim3(S, cx), dim3(256), 0, st, z, ldz, dz, lddz, S, V, lse, u, labels);
            PARL_LAUNCHED();
            return;
        }
    }
    k_softmax_bwd<Tin, Tout><<<dim3(S, cx), 256, 0, st>>>(z, ldz, dz, lddz, S, V, lse, u, labels);
    PARL_LAUNCHED();
}
template void launch_softmax_bwd<float, float>(const float*, long, float*, long, int, int, const float*,
                                               const float*, const int32_t*, cudaStream_t);
template void launch_softmax_bwd<float, bf16>(const float*, long, bf16*, long, int, int, const float*, const float*,
                                              const int32_t*, cudaStream_t);
template void launch_softmax_bwd<bf16, bf16>(const bf16*, long, bf16*, long, int, int, const float*, const float*,
                                             const int32_t*, cudaStream_t);
template void launch_softmax_bwd<bf16, float>(const bf16*, long, float*, long, int, int, const float*, const float*,
                                              const int32_t*, cudaStream_t);

void launch_scatter_rows(const float* dxg, const int32_t* row_ptr, const int32_t* row_idx, int T, int D, float* dx,
                         cudaStream_t st) {
    if (D % 4 == 0 && ((reinterpret_cast<uintptr_t>(dxg) | reinterpret_cast<uintptr_t>(dx)) & 15) == 0)
        k_scatter_rows4<<<cdiv(T, 8), 256, 0, st>>>(reinterpret_cast<const float4*>(dxg), row_ptr, row_idx, T, D / 4,
                                                    reinterpret_cast<float4*>(dx));
    else
        k_scatter_rows<<<grid_for((long)T * D), 256, 0, st>>>(dxg, row_ptr, row_idx, T, D, dx);
    PARL_LAUNCHED();
}

size_t sort_temp_bytes(int n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, n);
    return bytes;
}

void launch_sort_pairs(void* temp, size_t temp_bytes, const int32_t* keys_in, int32_t* keys_out,
                       const int32_t* vals_in, int32_t* vals_out, int n, int end_bit, cudaStream_t st) {
    const cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, n,
                                                          0, end_bit, st);
    if (e != cudaSuccess) throw Error{PARL_E_CUDA, std::string("radix sort: ") + cudaGetErrorString(e)};
    PARL_LAUNCHED();
}

__global__ void k_iota(int32_t* x, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = i;
}
void launch_iota(int32_t* x, int n, cudaStream_t st) {
    k_iota<<<cdiv(n, 256), 256, 0, st>>>(x, n);
    PARL_LAUNCHED();
}

void launch_embed_grad(const int32_t* keys, const int32_t* idx, int T, const float* dx, int D, float* grad,
                       cudaStream_t st) {
    if (T <= 0) return;
    k_embed_grad<<<T, 128, 0, st>>>(keys, idx, T, dx, D, grad);
    PARL_LAUNCHED();
}

template <class T>
void launch_f32_to_act(const float* x, T* y, long n, cudaStream_t st) {
    k_f32_to_act<T><<<grid_for(n), 256, 0, st>>>(x, y, n);
    PARL_LAUNCHED();
}
template void launch_f32_to_act<float>(const float*, float*, long, cudaStream_t);
template void launch_f32_to_act<bf16>(const float*, bf16*, long, cudaStream_t);

template <class T>
void launch_convert_w(const double* src, int rows, int cols, T* dst, long ldd, int transposed, cudaStream_t st) {
    dim3 grid(cdiv(cols, 32), cdiv(rows, 32));
    k_convert_w<T><<<grid, dim3(32, 8), 0, st>>>(src, rows, cols, dst, ldd, transposed);
    PARL_LAUNCHED();
}
template void launch_convert_w<float>(const double*, int, int, float*, long, int, cudaStream_t);
template void launch_convert_w<bf16>(const double*, int, int, bf16*, long, int, cudaStream_t);

template <class T>
void launch_export_w(const T* src, long lds, int rows, int cols, int transposed, double* dst, cudaStream_t st) {
    k_export_w<T><<<grid_for((long)rows * cols), 256, 0, st>>>(src, lds, rows, cols, transposed, dst);
    PARL_LAUNCHED();
}
template void launch_export_w<float>(const float*, long, int, int, int, double*, cudaStream_t);
template void launch_export_w<bf16>(const bf16*, long, int, int, int, double*, cudaStream_t);

void launch_f32_to_f64(const float* x, double* y, long n, cudaStream_t st) {
    k_f32_to_f64<<<grid_for(n), 256, 0, st>>>(x, y, n);
    PARL_LAUNCHED();
}

void launch_randn(double* out, long n, uint64_t seed, uint32_t stream, double scale, const double* base,
                  cudaStream_t st) {
    k_randn<<<grid_for(n), 256, 0, st>>>(out, n, seed, stream, scale, base);
    PARL_LAUNCHED();
}

void launch_fill_f64(double* out, long n, double v, cudaStream_t st) {
    k_fill_f64<<<grid_for(n), 256, 0, st>>>(out, n, v);
    PARL_LAUNCHED();
}

// ---- sparse token-embedding allreduce helpers (rows of tok_emb touched by any rank)
__global__ void k_mark_rows(const int32_t* __restrict__ ids, int n, uint8_t* __restrict__ flags) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) flags[ids[i]] = 1;
}
void launch_mark_rows(const int32_t* ids, int n, uint8_t* flags, cudaStream_t st) {
    if (n <= 0) return;
    k_mark_rows<<<std::min(cdiv(n, 256), 1024), 256, 0, st>>>(ids, n, flags);
    PARL_LAUNCHED();
}
__global__ void k_or_bytes(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] |= src[i];
}
void launch_or_bytes(const uint8_t* src, uint8_t* dst, int n, cudaStream_t st) {
    if (n <= 0) return;
    k_or_bytes<<<std::min(cdiv(n, 256), 1024), 256, 0, st>>>(src, dst, n);
    PARL_LAUNCHED();
}
// idx[0 .. *count) = the flagged row ids, ascending
void select_flagged_rows(const uint8_t* flags, int n, int32_t* idx, int* count, cudaStream_t st) {
    static void* temp = nullptr;
    static size_t temp_bytes = 0;
    cub::CountingInputIterator<int32_t> it(0);
    size_t need = 0;
    cub::DeviceSelect::Flagged(nullptr, need, it, flags, idx, count, n, st);
    if (need > temp_bytes) {
        if (temp) cudaFree(temp);
        PARL_CUDA(cudaMalloc(&temp, need));
        temp_bytes = need;
    }
    PARL_CUDA(cub::DeviceSelect::Flagged(temp, temp_bytes, it, flags, idx, count, n, st));
}
// dir 0: dst[i] = src[idx[i]] (gather rows); 1: dst[idx[i]] = src[i] (scatter back)
__global__ void k_rows_copy(const float* __restrict__ src, const int32_t* __restrict__ idx, int n, int d, int dir,
                            float* __restrict__ dst) {
    const int d4 = d >> 2;
    const long total = (long)n * d4;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e / d4), c = (int)(e % d4);
        const long r = idx[i];
        if (dir == 0) reinterpret_cast<float4*>(dst)[(long)i * d4 + c] = reinterpret_cast<const float4*>(src)[r * d4 + c];
        else reinterpret_cast<float4*>(dst)[r * d4 + c] = reinterpret_cast<const float4*>(src)[(long)i * d4 + c];
    }
}
void launch_rows_copy(const float* src, const int32_t* idx, int n, int d, int dir, float* dst, cudaStream_t st) {
    if (n <= 0) return;
    k_rows_copy<<<grid_for((long)n * (d / 4)), 256, 0, st>>>(src, idx, n, d, dir, dst);
    PARL_LAUNCHED();
}

void launch_axpy(const float* x, float* y, long n, cudaStream_t st) {
    k_axpy<<<grid_for(n), 256, 0, st>>>(x, y, n);
    PARL_LAUNCHED();
}

__global__ void k_f64_to_f32(const double* __restrict__ x, float* __restrict__ y, long n) {
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x)
        y[e] = (float)x[e];
}
void launch_f64_to_f32(const double* x, float* y, long n, cudaStream_t st) {
    k_f64_to_f32<<<grid_for(n), 256, 0, st>>>(x, y, n);
    PARL_LAUNCHED();
}

template <class T>
__global__ void k_finite_check(const T* __restrict__ x, long n, int* __restrict__ flags) {
    bool bad = false;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x)
        bad |= !isfinite(x[e]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1);
}
void launch_finite_check_f32(const float* x, long n, int* flags, cudaStream_t st) {
    k_finite_check<float><<<grid_for(n), 256, 0, st>>>(x, n, flags);
    PARL_LAUNCHED();
}
void launch_finite_check_f64(const double* x, long n, int* flags, cudaStream_t st) {
    k_finite_check<double><<<grid_for(n), 256, 0, st>>>(x, n, flags);
    PARL_LAUNCHED();
}

void launch_sgd(const float* g, double* w, long n, double scale, int* flags, int phase, cudaStream_t st) {
    if (phase == 0) k_sgd_check<<<grid_for(n), 256, 0, st>>>(g, w, n, scale, flags);
    else k_sgd_apply<<<grid_for(n), 256, 0, st>>>(g, w, n, scale);
    PARL_LAUNCHED();
}

}  // namespace parl_gpu
