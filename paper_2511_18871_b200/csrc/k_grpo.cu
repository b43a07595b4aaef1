// K7: the GRPO loss over every scored token of a micro-batch, one coalesced,
// vectorised pass (grpo.cpp:24-151 + pipeline.cpp:127-139).
//
//   k_grpo_tokens  warp-autonomous: each warp walks a contiguous range of
//                  warp_tokens scored tokens in spans of 128 (4 per lane,
//                  16-byte loads of the three log-prob vectors and the
//                  token -> sample map); no block barrier anywhere.  The group
//                  advantages (grpo.cpp:24-48) and 1/n_j of the samples a span
//                  touches are rebuilt by the warp's lanes into a per-warp
//                  table only when the span leaves the samples already there
//                  (once per sample boundary), so the rewards take no separate
//                  launch.  Token granularity writes the backward seed
//                      upstream[t] = up_scale * (1/n_j) (clip_grad + beta kl_grad)
//                  (pipeline.cpp:138 pushes up_scale = -1) and reduces the
//                  per-sample sums {clip value, kl value, clipped} with a
//                  segmented warp scan whose open run carries from span to span;
//                  each (sample, warp range) partial goes to its own slot (index
//                  sample + range), so the finisher adds them in a fixed order:
//                  deterministic, no atomics.
//   k_grpo_finish  warp (long samples) or thread (short ones) per sample: per-sample terms
//                  (SampleTerms, grpo.hpp:64-70); block partials of the running stats, added
//                  in index order by the last block (pipeline.cpp:131-137).
//   k_grpo_bcast   sequence granularity only: broadcast g_j to every token.
//
// Hot path inputs are the fp32 device log-probs: the ratio / KL terms are then
// evaluated in fp32 (expf / expm1f, full precision) and every cross-lane sum in
// fp64, which keeps the pass on the HBM roofline (fp64 exp + expm1 per token would
// bound it on the fp64 pipe at stress sizes).  The operator API
// (parl_per_sample_terms / parl_grpo_microbatch_loss) passes fp64 inputs and runs
// the same kernels with fp64 arithmetic throughout.
#include "internal.cuh"
#include "kernels.cuh"

namespace parl_gpu {

namespace {

constexpr int GR_ITEMS = 4, GR_SPAN = 32 * GR_ITEMS, GR_WARPS = 8, GR_MAX_ITERS = 8;

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

// GR_ITEMS consecutive values from t (zero beyond the range end e); one or two 16-byte loads
template <class LP, class R>
__device__ __forceinline__ void load_items(const LP* __restrict__ p, long t, long e, R* v) {
    if (t + GR_ITEMS <= e && ((reinterpret_cast<uintptr_t>(p + t) & 15) == 0)) {
        if constexpr (std::is_same_v<LP, float>) {
            const float4 x = __ldcs(reinterpret_cast<const float4*>(p + t));
            v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        } else {
            const double2 x = __ldcs(reinterpret_cast<const double2*>(p + t));
            const double2 y = __ldcs(reinterpret_cast<const double2*>(p + t + 2));
            v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y;
        }
        return;
    }
#pragma unroll
    for (int i = 0; i < GR_ITEMS; ++i) v[i] = (t + i < e) ? (R)p[t + i] : R(0);
}

// the advantage of sample j (grpo.cpp:24-48: group mean / population std, mean-only variant)
__device__ __forceinline__ double sample_advantage(const GrpoArgs& a, int j) {
    if (a.adv_in) return a.adv_in[j];
    const int G = a.group_size, grp = j / G;
    const double* r = a.rewards + (long)grp * G;
    double s = 0.0, v = 0.0;
    for (int i = 0; i < G; ++i) s += r[i];
    const double mean = s / G;
    for (int i = 0; i < G; ++i) v += (r[i] - mean) * (r[i] - mean);
    const double sd = sqrt(v / G), rj = r[j - grp * G];
    return a.mean_only ? rj - mean : (sd < 1e-8 ? 0.0 : (rj - mean) / sd);
}

// The per-token part of one span: loads (FULL: one 16-byte load per vector and lane, no
// bounds), the sample table refresh, the GRPO terms (token granularity, grpo.cpp:119-131) and
// the upstream store.  On return x0 / x1 / x2 hold the values to reduce per sample (zero past
// the range end): {clip value, kl value, clipped} or, for sequence granularity, the raw
// {lp, old, ref} (grpo.cpp:134-140).
template <class LP, class R, int GRAN, bool FULL>
__device__ __forceinline__ void span_terms(const GrpoArgs& a, long b, long e, long r0, long r1, int lane,
                                           R (*tab)[2], int& tab_lo, int& tab_hi, int* s, R* x0, R* x1, R* x2,
                                           int& nv, int& j_first, int& j_last, int& last_lane, int& first,
                                           int& last) {
    const long t0 = b + lane * GR_ITEMS;
    if constexpr (FULL) {
        const int4 v = __ldcs(reinterpret_cast<const int4*>(a.sample_of + t0));
        s[0] = v.x; s[1] = v.y; s[2] = v.z; s[3] = v.w;
        nv = GR_ITEMS;
        last_lane = 31;
        first = s[0];
        last = s[GR_ITEMS - 1];
    } else {
#pragma unroll
        for (int i = 0; i < GR_ITEMS; ++i) s[i] = (t0 + i < e) ? a.sample_of[t0 + i] : -1;
        nv = (int)max(0L, min((long)GR_ITEMS, e - t0));
        last_lane = (int)((e - b - 1) / GR_ITEMS);
        first = nv > 0 ? s[0] : -1;
        last = first;
#pragma unroll
        for (int i = 1; i < GR_ITEMS; ++i) last = i < nv ? s[i] : last;
    }
    load_items<LP, R>(static_cast<const LP*>(a.lp), t0, FULL ? t0 + GR_ITEMS : e, x0);
    load_items<LP, R>(static_cast<const LP*>(a.old), t0, FULL ? t0 + GR_ITEMS : e, x1);
    load_items<LP, R>(static_cast<const LP*>(a.ref), t0, FULL ? t0 + GR_ITEMS : e, x2);
    j_first = __shfl_sync(0xffffffffu, first, 0);
    j_last = __shfl_sync(0xffffffffu, last, last_lane);
    if constexpr (GRAN == 0) {
        if (j_first < tab_lo || j_last > tab_hi) {  // refresh the sample table (warp-uniform)
            __syncwarp();
            // [j_first, j_last] is at most GR_SPAN samples (every sample holds >= 1 token); one lane
            // round fills up to 32 of them, so short samples refresh once per 32
            tab_lo = j_first;
            tab_hi = max(j_last, min(a.n - 1, j_first + 31));
            for (int j = tab_lo + lane; j <= tab_hi; j += 32) {
                const double adv = sample_advantage(a, j);
                const int cj = a.cu[j];
                tab[j - tab_lo][0] = (R)adv;
                tab[j - tab_lo][1] = R(1) / (R)(a.cu[j + 1] - cj);
                if (a.adv_out && cj >= r0 && cj < r1) a.adv_out[j] = adv;  // the range holding the first token
            }
            __syncwarp();
        }
        const R eps = (R)a.eps, beta = (R)a.beta, ups = (R)a.up_scale;
        R up4[GR_ITEMS];
#pragma unroll
        for (int i = 0; i < GR_ITEMS; ++i) {
            const bool ok = FULL || i < nv;
            const int jl = ok ? s[i] - tab_lo : 0;
            R cv, cg;
            int c;
            clip_eval<R>(x0[i], x1[i], tab[jl][0], eps, cv, cg, c);
            const R d = x2[i] - x0[i], em = expm1(d);  // eval_kl, grpo.cpp:89-93
            const R g = tab[jl][1] * (cg + beta * em);
            x0[i] = ok ? cv : R(0);
            x1[i] = ok ? em - d : R(0);
            x2[i] = ok ? (R)c : R(0);
            up4[i] = ups * g;
        }
        if (a.up_f32) {
            if (FULL || nv == GR_ITEMS) {
                __stcs(reinterpret_cast<float4*>(a.up_f32 + t0),
                       make_float4((float)up4[0], (float)up4[1], (float)up4[2], (float)up4[3]));
            } else {
                for (int i = 0; i < nv; ++i) a.up_f32[t0 + i] = (float)up4[i];
            }
        }
        if (a.up_f64)
            for (int i = 0; i < nv; ++i) a.up_f64[t0 + i] = (double)up4[i];
    } else if (a.adv_out) {  // sequence granularity: the advantage, written by the span holding the first token
        for (int j = j_first + lane; j <= j_last; j += 32) {
            const int cj = a.cu[j];
            if (cj >= b && cj < e) a.adv_out[j] = sample_advantage(a, j);
        }
    }
}

// Warp-autonomous pass over the range [r0, r1) of scored tokens.  The open run (sample cs,
// the one the previous span ended in) is held as per-lane fp64 partials la / lb / lc: a span
// wholly inside it (the common case: samples are hundreds of tokens) only adds each lane's
// items, with no cross-lane traffic.  A span holding a sample boundary folds the partials
// into a carry, runs a segmented warp scan, writes every run that ends inside it to its
// (sample, range) slot and leaves the new open run's total in lane 0.
template <class LP, int GRAN>
__global__ void __launch_bounds__(GR_WARPS * 32) k_grpo_tokens(const GrpoArgs a) {
    using R = std::conditional_t<std::is_same_v<LP, float>, float, double>;
    __shared__ R s_tab[GR_WARPS][GR_SPAN][2];  // per warp: {advantage, 1/n} of samples [tab_lo, tab_hi]
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long rng = (long)blockIdx.x * GR_WARPS + wid;  // this warp's range of scored tokens
    const long r0 = rng * a.warp_tokens, r1 = min((long)a.S, r0 + a.warp_tokens);
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.ticket = 0u;  // k_grpo_finish's ticket (stream-ordered)
    if (r0 >= r1) return;
    // 16-byte vector loads / stores need 16-byte aligned bases (t0 is a multiple of 4 elements)
    const bool aligned = ((reinterpret_cast<uintptr_t>(a.lp) | reinterpret_cast<uintptr_t>(a.old) |
                           reinterpret_cast<uintptr_t>(a.ref) | reinterpret_cast<uintptr_t>(a.sample_of) |
                           reinterpret_cast<uintptr_t>(a.up_f32)) & 15) == 0;
    R(*tab)[2] = s_tab[wid];
    int tab_lo = 0, tab_hi = -1;
    int cs = -1;                    // the open run's sample
    double la = 0.0, lb = 0.0, lc = 0.0;  // its per-lane partials
    for (long b = r0; b < r1; b += GR_SPAN) {
        const long e = min(r1, b + GR_SPAN);
        int s[GR_ITEMS], nv, j_first, j_last, last_lane, first, last;
        R x0[GR_ITEMS], x1[GR_ITEMS], x2[GR_ITEMS];
        if (aligned && e - b == GR_SPAN)
            span_terms<LP, R, GRAN, true>(a, b, e, r0, r1, lane, tab, tab_lo, tab_hi, s, x0, x1, x2, nv, j_first,
                                          j_last, last_lane, first, last);
        else
            span_terms<LP, R, GRAN, false>(a, b, e, r0, r1, lane, tab, tab_lo, tab_hi, s, x0, x1, x2, nv, j_first,
                                           j_last, last_lane, first, last);
        if (j_first == j_last && (cs == j_first || cs < 0)) {  // inside the open run (warp-uniform)
            cs = j_first;
            if constexpr (GRAN == 0) {  // token terms: a 4-term fp32 sum per lane, then fp64
                la += (double)((x0[0] + x0[1]) + (x0[2] + x0[3]));
                lb += (double)((x1[0] + x1[1]) + (x1[2] + x1[3]));
                lc += (double)((x2[0] + x2[1]) + (x2[2] + x2[3]));
            } else {  // raw log-probs: exact fp64 sums
#pragma unroll
                for (int i = 0; i < GR_ITEMS; ++i) {
                    la += (double)x0[i];
                    lb += (double)x1[i];
                    lc += (double)x2[i];
                }
            }
            continue;
        }
        // a sample boundary: the open run's total, flushed if the span does not continue it
        double ca = warp_sum_d(la), cb = warp_sum_d(lb), cc = warp_sum_d(lc);
        if (cs >= 0 && j_first != cs) {
            if (lane == 0) {
                double* o = a.slots + 3 * ((long)cs + rng);
                o[0] = ca;
                o[1] = cb;
                o[2] = cc;
            }
            cs = -1;
            ca = cb = cc = 0.0;
        }
        const int up_last = __shfl_up_sync(0xffffffffu, last, 1);
        const int prev_last = lane == 0 ? cs : up_last;
        const int next_first = __shfl_down_sync(0xffffffffu, first, 1);
        double ta = 0, tb = 0, tc = 0;  // the lane's last run
#pragma unroll
        for (int i = 0; i < GR_ITEMS; ++i)
            if (i < nv && s[i] == last) {
                ta += (double)x0[i];
                tb += (double)x1[i];
                tc += (double)x2[i];
            }
        double va = ta, vb = tb, vc = tc;
        int reset = (lane == 0 || first != prev_last || first != last) ? 1 : 0;
        if (lane == 0 && nv > 0 && first == last && first == cs) {  // the carried run continues through lane 0
            va += ca;
            vb += cb;
            vc += cc;
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {  // inclusive segmented scan over the lanes
            const double ua = __shfl_up_sync(0xffffffffu, va, o), ub = __shfl_up_sync(0xffffffffu, vb, o),
                         uc = __shfl_up_sync(0xffffffffu, vc, o);
            const int ur = __shfl_up_sync(0xffffffffu, reset, o);
            if (lane >= o && !reset) {
                va += ua;
                vb += ub;
                vc += uc;
                reset = ur;
            }
        }
        // carried into the lane's first run: the previous lane's inclusive value (lane 0: the open run)
        const double pa = __shfl_up_sync(0xffffffffu, va, 1), pb = __shfl_up_sync(0xffffffffu, vb, 1),
                     pc = __shfl_up_sync(0xffffffffu, vc, 1);
        double c0a = 0.0, c0b = 0.0, c0c = 0.0;
        if (nv > 0 && first == prev_last) {
            c0a = lane == 0 ? ca : pa;
            c0b = lane == 0 ? cb : pb;
            c0c = lane == 0 ? cc : pc;
        }
        double q0 = 0, q1 = 0, q2 = 0;
#pragma unroll
        for (int i = 0; i < GR_ITEMS; ++i) {
            if (i >= nv) break;
            q0 += (double)x0[i];
            q1 += (double)x1[i];
            q2 += (double)x2[i];
            const bool open = (lane == last_lane) && (i == nv - 1);  // continues into the next span
            const bool end = (i + 1 < nv) ? (s[i + 1] != s[i]) : (!open && next_first != s[i]);
            if (end) {
                double* o = a.slots + 3 * ((long)s[i] + rng);
                o[0] = c0a + q0;
                o[1] = c0b + q1;
                o[2] = c0c + q2;
                q0 = q1 = q2 = 0;
                c0a = c0b = c0c = 0.0;
            }
        }
        // the span's last run stays open: its inclusive value, held by lane 0
        cs = j_last;
        ca = __shfl_sync(0xffffffffu, va, last_lane);
        cb = __shfl_sync(0xffffffffu, vb, last_lane);
        cc = __shfl_sync(0xffffffffu, vc, last_lane);
        la = lane == 0 ? ca : 0.0;
        lb = lane == 0 ? cb : 0.0;
        lc = lane == 0 ? cc : 0.0;
    }
    // flush the open run at the range end
    const double ca = warp_sum_d(la), cb = warp_sum_d(lb), cc = warp_sum_d(lc);
    if (lane == 0) {
        double* o = a.slots + 3 * ((long)cs + rng);
        o[0] = ca;
        o[1] = cb;
        o[2] = cc;
    }
}

// Per-sample terms (SampleTerms, grpo.hpp:64-70) from the (sample, range) partials, then the
// running stats (pipeline.cpp:131-137).  Two shapes, chosen per launch from S / n:
//   WPS (long samples, many partials each): warp w takes sample w, its lanes add the partials in
//        a fixed strided order, then a fixed butterfly;
//   TPS (short samples, a few partials): thread t takes sample t and adds them in order.
// Each block reduces its samples' stats contributions in a fixed tree into a block partial; the
// last block to finish (a ticket k_grpo_tokens zeroed) adds the block partials in index order.
// Deterministic for a given (S, n): the shape and both trees depend on nothing else.
template <bool WPS>
__global__ void __launch_bounds__(WPS ? 1024 : 256) k_grpo_finish(const GrpoArgs a) {
    __shared__ double red[5][32];
    __shared__ unsigned ticket;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int j = WPS ? (int)(((long)blockIdx.x * blockDim.x + tid) >> 5) : blockIdx.x * blockDim.x + tid;
    double acc[5] = {0, 0, 0, 0, 0};
    if (j < a.n) {
        const int b = a.cu[j], e = a.cu[j + 1], n = e - b;
        const int b0 = b / a.warp_tokens, b1 = (e - 1) / a.warp_tokens;
        double s0 = 0, s1 = 0, s2 = 0;
        if constexpr (WPS) {
#pragma unroll 4
            for (int k = b0 + lane; k <= b1; k += 32) {
                const double* o = a.slots + 3 * ((long)j + k);
                s0 += o[0];
                s1 += o[1];
                s2 += o[2];
            }
            s0 = warp_sum_d(s0);
            s1 = warp_sum_d(s1);
            s2 = warp_sum_d(s2);
        } else {
            for (int k = b0; k <= b1; ++k) {
                const double* o = a.slots + 3 * ((long)j + k);
                s0 += o[0];
                s1 += o[1];
                s2 += o[2];
            }
        }
        if (!WPS || lane == 0) {
            double tm[4];
            if (a.gran == 0) {
                const double inv = 1.0 / n;
                tm[0] = s0 * inv;
                tm[1] = s1 * inv;
                tm[2] = s2;
                tm[3] = n;
            } else {  // one evaluation on the summed log-probs (grpo.cpp:134-149)
                double cv, cg;
                int c;
                clip_eval<double>(s0, s1, a.adv_out[j], a.eps, cv, cg, c);
                const double d = s2 - s0, em = expm1(d);
                tm[0] = cv;
                tm[1] = em - d;
                tm[2] = c;
                tm[3] = 1;
                a.g_seq[j] = a.up_scale * (cg + a.beta * em);
            }
            if (a.per_sample)
                for (int q = 0; q < 4; ++q) a.per_sample[4 * (long)j + q] = tm[q];
            acc[0] = tm[0] - a.beta * tm[1];
            acc[1] = tm[0];
            acc[2] = tm[1];
            acc[3] = tm[2];
            acc[4] = tm[3];
        }
    }
    if (!a.stats) return;
    // the block's contribution: a fixed tree (lanes, then warps in order)
    if constexpr (!WPS) {
#pragma unroll
        for (int q = 0; q < 5; ++q) acc[q] = warp_sum_d(acc[q]);
    }
    if (lane == 0)
        for (int q = 0; q < 5; ++q) red[q][wid] = acc[q];
    __syncthreads();
    if (tid < 5) {
        double s = 0.0;
        for (int w = 0; w < nw; ++w) s += red[tid][w];
        a.terms[5 * (long)blockIdx.x + tid] = s;  // block partials
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) ticket = atomicAdd(a.ticket, 1u);
    __syncthreads();
    if (ticket != gridDim.x - 1) return;
    double tot[5] = {0, 0, 0, 0, 0};
    for (int k = tid; k < (int)gridDim.x; k += blockDim.x)
        for (int q = 0; q < 5; ++q) tot[q] += __ldcg(a.terms + 5 * (long)k + q);
#pragma unroll
    for (int q = 0; q < 5; ++q) tot[q] = warp_sum_d(tot[q]);
    __syncthreads();
    if (lane == 0)
        for (int q = 0; q < 5; ++q) red[q][wid] = tot[q];
    __syncthreads();
    if (tid < 5) {
        double s = 0.0;
        for (int w = 0; w < nw; ++w) s += red[tid][w];
        a.stats[tid] += s;
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

// slots for the finest warp range (one span): enough for any range length launch_grpo picks
// (+ 5 per finisher block of at most 32 samples: the block partials, + 1: k_grpo_finish's ticket)
size_t grpo_slot_count(long S, int n) {
    return 3 * ((size_t)n + (size_t)((S + GR_SPAN - 1) / GR_SPAN) + 1) + 5 * (size_t)((n + 31) / 32) + 1;
}

void launch_grpo(const GrpoArgs& a_in, cudaStream_t st) {
    if (a_in.S <= 0 || a_in.n <= 0) return;
    GrpoArgs a = a_in;
    a.terms = a.slots + 3 * ((size_t)a.n + (size_t)((a.S + GR_SPAN - 1) / GR_SPAN) + 1);
    a.ticket = reinterpret_cast<unsigned*>(a.terms + 5 * (size_t)((a.n + 31) / 32));
    // spans per warp: as many as keep >= ~48 warps per SM busy (fewer slots, longer carried runs)
    const long spans = (a.S + GR_SPAN - 1) / GR_SPAN;
    const int iters = (int)std::max(1L, std::min((long)GR_MAX_ITERS, spans / (148L * 48)));
    a.warp_tokens = GR_SPAN * iters;
    const long warps = (a.S + a.warp_tokens - 1) / a.warp_tokens;
    const int grid = (int)((warps + GR_WARPS - 1) / GR_WARPS);
    if (a.lp_f64) {
        if (a.gran == 0) k_grpo_tokens<double, 0><<<grid, GR_WARPS * 32, 0, st>>>(a);
        else k_grpo_tokens<double, 1><<<grid, GR_WARPS * 32, 0, st>>>(a);
    } else {
        if (a.gran == 0) k_grpo_tokens<float, 0><<<grid, GR_WARPS * 32, 0, st>>>(a);
        else k_grpo_tokens<float, 1><<<grid, GR_WARPS * 32, 0, st>>>(a);
    }
    PARL_LAUNCHED();
    // a thread per sample while samples hold a few (sample, range) partials, else a warp
    if (a.S / a.n > 4L * a.warp_tokens) k_grpo_finish<true><<<cdiv(a.n, 32), 1024, 0, st>>>(a);
    else k_grpo_finish<false><<<cdiv(a.n, 256), 256, 0, st>>>(a);
    PARL_LAUNCHED();
    if (a.gran == 1) {
        k_grpo_bcast<<<std::min(cdiv(a.S, 256), 148 * 8), 256, 0, st>>>(a);
        PARL_LAUNCHED();
    }
}

}  // namespace parl_gpu
