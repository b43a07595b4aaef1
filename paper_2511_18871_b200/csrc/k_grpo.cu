// K7: the GRPO loss over every scored token of a micro-batch, one coalesced,
// vectorised pass (grpo.cpp:24-151 + pipeline.cpp:127-139).
//
//   k_grpo_tokens  grid over the S scored tokens, CHUNK tokens per block (4 per
//                  thread, 16-byte loads of the three log-prob vectors and the
//                  token -> sample map).  Group advantages (grpo.cpp:24-48) are
//                  rebuilt in shared memory by every block for the samples its
//                  chunk touches, so the rewards never take a separate launch.
//                  Token granularity writes the backward seed
//                      upstream[t] = up_scale * (1/n_j) (clip_grad - beta kl_grad)
//                  (pipeline.cpp:138 pushes up_scale = -1) and reduces the
//                  per-sample sums {clip value, kl value, clipped} with a
//                  segmented block scan; each (sample, block) partial goes to
//                  its own slot (index sample + block), so the finisher adds them
//                  in a fixed order: deterministic, no atomics.
//   k_grpo_finish  one block: per-sample terms (SampleTerms, grpo.hpp:64-70) and
//                  the running stats (pipeline.cpp:131-137), fixed-order tree.
//   k_grpo_bcast   sequence granularity only: broadcast g_j to every token.
//
// Hot path inputs are the fp32 device log-probs: the ratio / KL terms are then
// evaluated in fp32 (expf / expm1f, full precision) and every sum in fp64, which
// keeps the pass on the HBM roofline (fp64 exp + expm1 per token would bound it
// on the fp64 pipe at stress sizes).  The operator API
// (parl_per_sample_terms / parl_grpo_microbatch_loss) passes fp64 inputs and runs
// the same kernels with fp64 arithmetic throughout.
#include <cub/block/block_scan.cuh>

#include "internal.cuh"
#include "kernels.cuh"

namespace parl_gpu {

namespace {

constexpr int GR_THREADS = 256, GR_ITEMS = 4, GR_CHUNK = GR_THREADS * GR_ITEMS;

// eval_clip (grpo.cpp:64-80) in the arithmetic of R
template <class R>
__device__ __forceinline__ void clip_eval(R lp, R old, R A, R eps, R& val, R& grad, int& clipped) {
    const R r = exp(lp - old), lo = R(1) - eps, hi = R(1) + eps;
    const R cl = fmin(fmax(r, lo), hi);
    const R un = r * A, cv = cl * A;
    clipped = (r < lo || r > hi);
    if (un <= cv) {
        val = un;
        grad = r * A;
    } else {
        val = cv;
        grad = (r > lo && r < hi) ? r * A : R(0);
    }
}

struct SegAgg {
    double a, b, c;
    int reset;  // a segment boundary lies in (or at the start of) this span: earlier values do not carry in
};

struct SegOp {
    __device__ __forceinline__ SegAgg operator()(const SegAgg& x, const SegAgg& y) const {
        if (y.reset) return y;
        return {x.a + y.a, x.b + y.b, x.c + y.c, x.reset};
    }
};

template <class LP, class R>
__device__ __forceinline__ void load8(const LP* __restrict__ p, long t, long S, R* v) {
    if constexpr (std::is_same_v<LP, float>) {
        if (t + GR_ITEMS <= S && ((reinterpret_cast<uintptr_t>(p + t) & 15) == 0)) {
#pragma unroll
            for (int q = 0; q < GR_ITEMS; q += 4) {
                const float4 x = *reinterpret_cast<const float4*>(p + t + q);
                v[q] = x.x; v[q + 1] = x.y; v[q + 2] = x.z; v[q + 3] = x.w;
            }
            return;
        }
    }
#pragma unroll
    for (int i = 0; i < GR_ITEMS; ++i) v[i] = (t + i < S) ? (R)p[t + i] : R(0);
}

template <class LP>
__global__ void __launch_bounds__(GR_THREADS, 4) k_grpo_tokens(const GrpoArgs a) {
    using Scan = cub::BlockScan<SegAgg, GR_THREADS>;
    using R = std::conditional_t<std::is_same_v<LP, float>, float, double>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ R s_adv[GR_CHUNK], s_inv[GR_CHUNK];
    __shared__ int s_first[GR_THREADS], s_last[GR_THREADS];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long c0 = (long)blockIdx.x * GR_CHUNK;
    const long c1 = min((long)a.S, c0 + GR_CHUNK);
    // this thread's tokens first: their loads are in flight while the prologue below walks its
    // chain of dependent loads (sample range -> advantages / lengths)
    const long t0 = c0 + (long)tid * GR_ITEMS;
    int s[GR_ITEMS];
    R x0[GR_ITEMS], x1[GR_ITEMS], x2[GR_ITEMS];  // per-token values in the arithmetic type (fp32 hot path)
    if (t0 + GR_ITEMS <= c1 && ((reinterpret_cast<uintptr_t>(a.sample_of + t0) & 15) == 0)) {
#pragma unroll
        for (int q = 0; q < GR_ITEMS; q += 4) {
            const int4 v = *reinterpret_cast<const int4*>(a.sample_of + t0 + q);
            s[q] = v.x; s[q + 1] = v.y; s[q + 2] = v.z; s[q + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < GR_ITEMS; ++i) s[i] = (t0 + i < c1) ? a.sample_of[t0 + i] : -1;
    }
    load8(static_cast<const LP*>(a.lp), t0, c1, x0);
    load8(static_cast<const LP*>(a.old), t0, c1, x1);
    load8(static_cast<const LP*>(a.ref), t0, c1, x2);
    const int j_lo = a.sample_of[c0], j_hi = a.sample_of[c1 - 1];
    // per-sample advantage and 1/n_j for the samples this chunk touches
    if (a.adv_in) {
        for (int j = j_lo + tid; j <= j_hi; j += GR_THREADS) s_adv[j - j_lo] = (R)a.adv_in[j];
    } else {
        const int G = a.group_size, g_lo = j_lo / G, g_hi = j_hi / G;
        for (int grp = g_lo + wid; grp <= g_hi; grp += GR_THREADS / 32) {  // group_advantages[_mean_only]
            const double* r = a.rewards + (long)grp * G;
            double s = 0.0;
            for (int i = lane; i < G; i += 32) s += r[i];
            const double mean = warp_sum_d(s) / G;
            double v = 0.0;
            for (int i = lane; i < G; i += 32) v += (r[i] - mean) * (r[i] - mean);
            const double sd = sqrt(warp_sum_d(v) / G);
            for (int i = lane; i < G; i += 32) {
                const int j = grp * G + i;
                if (j < j_lo || j > j_hi) continue;
                s_adv[j - j_lo] = (R)(a.mean_only ? r[i] - mean : (sd < 1e-8 ? 0.0 : (r[i] - mean) / sd));
            }
        }
    }
    for (int j = j_lo + tid; j <= j_hi; j += GR_THREADS) {
        s_inv[j - j_lo] = R(1) / (R)(a.cu[j + 1] - a.cu[j]);
        if (a.adv_out && a.cu[j] >= c0) {  // one writer: the sample's first chunk (fp64 advantage)
            if (a.adv_in) a.adv_out[j] = a.adv_in[j];
            else {
                const int G = a.group_size, grp = j / G;
                const double* r = a.rewards + (long)grp * G;
                double s = 0.0, v = 0.0;
                for (int i = 0; i < G; ++i) s += r[i];
                const double mean = s / G;
                for (int i = 0; i < G; ++i) v += (r[i] - mean) * (r[i] - mean);
                const double sd = sqrt(v / G), rj = r[j - grp * G];
                a.adv_out[j] = a.mean_only ? rj - mean : (sd < 1e-8 ? 0.0 : (rj - mean) / sd);
            }
        }
    }
    __syncthreads();

    const int nv = (int)max(0L, min((long)GR_ITEMS, c1 - t0));  // valid items of this thread
    const R eps = (R)a.eps, beta = (R)a.beta;
    if (a.gran == 0) {  // token granularity (grpo.cpp:119-131)
        float up4[GR_ITEMS];
#pragma unroll
        for (int i = 0; i < GR_ITEMS; ++i) {
            if (i >= nv) {
                x0[i] = x1[i] = x2[i] = R(0);
                up4[i] = 0.f;
                continue;
            }
            const R lp = x0[i], old = x1[i], ref = x2[i];
            const int jl = s[i] - j_lo;
            R cv, cg;
            int c;
            clip_eval<R>(lp, old, (R)s_adv[jl], eps, cv, cg, c);
            const R d = ref - lp, em = expm1(d);  // eval_kl, grpo.cpp:89-93
            const R g = s_inv[jl] * (cg + beta * em);
            x0[i] = cv;
            x1[i] = em - d;
            x2[i] = (R)c;
            up4[i] = (float)((R)a.up_scale * g);
            if (a.up_f64) a.up_f64[t0 + i] = a.up_scale * (double)g;
        }
        if (a.up_f32) {
            if (nv == GR_ITEMS && ((reinterpret_cast<uintptr_t>(a.up_f32 + t0) & 15) == 0)) {
#pragma unroll
                for (int q = 0; q < GR_ITEMS; q += 4)
                    *reinterpret_cast<float4*>(a.up_f32 + t0 + q) = make_float4(up4[q], up4[q + 1], up4[q + 2], up4[q + 3]);
            } else {
                for (int i = 0; i < nv; ++i) a.up_f32[t0 + i] = up4[i];
            }
        }
    }  // sequence granularity: sum the raw log-probs (grpo.cpp:134-140)

    // segmented reduction of (x0, x1, x2) by sample over the block's chunk
    const int first = nv > 0 ? s[0] : -1, last = nv > 0 ? s[nv - 1] : -1;
    s_first[tid] = first;
    s_last[tid] = last;
    __syncthreads();
    const int prev_last = tid > 0 ? s_last[tid - 1] : -2;
    const int next_first = tid + 1 < GR_THREADS ? s_first[tid + 1] : -2;
    // the thread's last run (in R, at most 8 terms), widened once
    R t0a = 0, t0b = 0, t0c = 0;
    for (int i = 0; i < nv; ++i)
        if (s[i] == last) {
            t0a += x0[i];
            t0b += x1[i];
            t0c += x2[i];
        }
    SegAgg agg{(double)t0a, (double)t0b, (double)t0c, (tid == 0 || first != prev_last || first != last) ? 1 : 0};
    SegAgg carry;
    Scan(scan_tmp).ExclusiveScan(agg, carry, SegOp());
    double c0a = 0.0, c0b = 0.0, c0c = 0.0;  // carried into the thread's first run
    if (tid > 0 && nv > 0 && first == prev_last) {
        c0a = carry.a;
        c0b = carry.b;
        c0c = carry.c;
    }
    R r0 = 0, r1 = 0, r2 = 0;
    for (int i = 0; i < nv; ++i) {
        r0 += x0[i];
        r1 += x1[i];
        r2 += x2[i];
        const bool end = (i + 1 < nv) ? (s[i + 1] != s[i]) : (next_first != s[i]);
        if (end) {
            double* o = a.slots + 3 * ((long)s[i] + blockIdx.x);
            o[0] = c0a + (double)r0;
            o[1] = c0b + (double)r1;
            o[2] = c0c + (double)r2;
            r0 = r1 = r2 = 0;
            c0a = c0b = c0c = 0.0;
        }
    }
}

// Per-sample terms + stats, one block: warp w takes samples w, w + 32, ...; its lanes add the
// sample's (sample, block) partials in a fixed strided order (a sample spanning many chunks is
// not a serial chain of dependent loads), then a fixed-order tree over the warps.
__global__ void __launch_bounds__(1024) k_grpo_finish(const GrpoArgs a) {
    __shared__ double red[5][32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    double acc[5] = {0, 0, 0, 0, 0};
    for (int j = wid; j < a.n; j += nw) {
        const int b = a.cu[j], e = a.cu[j + 1], n = e - b;
        const int b0 = b / GR_CHUNK, b1 = (e - 1) / GR_CHUNK;
        double s0 = 0, s1 = 0, s2 = 0;
        for (int k = b0 + lane; k <= b1; k += 32) {
            const double* o = a.slots + 3 * ((long)j + k);
            s0 += o[0];
            s1 += o[1];
            s2 += o[2];
        }
        s0 = warp_sum_d(s0);
        s1 = warp_sum_d(s1);
        s2 = warp_sum_d(s2);
        if (lane != 0) continue;
        double t[4];
        if (a.gran == 0) {
            const double inv = 1.0 / n;
            t[0] = s0 * inv;
            t[1] = s1 * inv;
            t[2] = s2;
            t[3] = n;
        } else {  // one evaluation on the summed log-probs (grpo.cpp:134-149)
            double cv, cg;
            int c;
            clip_eval<double>(s0, s1, a.adv_out[j], a.eps, cv, cg, c);
            const double d = s2 - s0, em = expm1(d);
            t[0] = cv;
            t[1] = em - d;
            t[2] = c;
            t[3] = 1;
            a.g_seq[j] = a.up_scale * (cg + a.beta * em);
        }
        if (a.per_sample)
            for (int q = 0; q < 4; ++q) a.per_sample[4 * (long)j + q] = t[q];
        acc[0] += t[0] - a.beta * t[1];
        acc[1] += t[0];
        acc[2] += t[1];
        acc[3] += t[2];
        acc[4] += t[3];
    }
    if (lane == 0)
        for (int q = 0; q < 5; ++q) red[q][wid] = acc[q];
    __syncthreads();
    if (tid == 0 && a.stats) {
        for (int q = 0; q < 5; ++q) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += red[q][w];
            a.stats[q] += s;
        }
    }
}

__global__ void __launch_bounds__(256) k_grpo_bcast(const GrpoArgs a) {
    for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < a.S; t += (long)gridDim.x * blockDim.x) {
        const double g = a.g_seq[a.sample_of[t]];
        if (a.up_f32) a.up_f32[t] = (float)g;
        if (a.up_f64) a.up_f64[t] = g;
    }
}

}  // namespace

size_t grpo_slot_count(long S, int n) { return 3 * ((size_t)n + (size_t)((S + GR_CHUNK - 1) / GR_CHUNK) + 1); }

void launch_grpo(const GrpoArgs& a, cudaStream_t st) {
    if (a.S <= 0 || a.n <= 0) return;
    const int grid = (int)((a.S + GR_CHUNK - 1) / GR_CHUNK);
    if (a.lp_f64) k_grpo_tokens<double><<<grid, GR_THREADS, 0, st>>>(a);
    else k_grpo_tokens<float><<<grid, GR_THREADS, 0, st>>>(a);
    PARL_LAUNCHED();
    k_grpo_finish<<<1, 1024, 0, st>>>(a);
    PARL_LAUNCHED();
    if (a.gran == 1) {
        k_grpo_bcast<<<std::min(cdiv(a.S, 256), 148 * 8), 256, 0, st>>>(a);
        PARL_LAUNCHED();
    }
}

}  // namespace parl_gpu
