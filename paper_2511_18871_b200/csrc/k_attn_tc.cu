// tcgen05 varlen shared-prompt attention (bf16 in, fp32 accumulate).
//
// Forward (k_attn_fwd_pair): persistent CTAs, work item = (pair of adjacent 128-row
// query tiles, head) taken from a global queue; replaces the attention loops of
// run_forward (proj/src/model.cpp:468-501) under the shared-prompt rule of
// model.cpp:242-245.  TMA-staged Q/K/V, S = QK^T and O += PV on tcgen05 with TMEM
// accumulators (P written back to TMEM as the A operand of the PV MMA), online
// softmax in the log2 domain with a conditional O rescale.  Key tiles are visited
// only when some row of a query tile can see them: response-to-response tiles of
// different responses are skipped, and only tiles straddling a boundary apply the
// per-element mask.  The forward saves only the row log-sum-exp.
//
// Backward (k_attn_prep_v8 + k_attn_bwd2<DKV> + k_attn_bwd2<DQ>): D = rowsum(dO*O),
// then dK/dV per key tile and dQ per query tile, deterministic (no atomics).
#include <cudaTypedefs.h>

#include <cuda_fp16.h>

#include "internal.cuh"
#include "kernels.cuh"
#include "tc_util.cuh"

namespace parl_gpu {

namespace {

constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&t);
}

// ===========================================================================
// Forward, two query tiles per CTA (Dh = 64 / 128).  Work item = (pair of adjacent
// 128-row query tiles, head); the pair's key tiles are the union of both
// tiles' visible lists, flagged per tile (visible / full).  Roles:
//   warps 0-3  softmax of query tile 0, warps 4-7 softmax of query tile 1
//              (thread = query row; two warps per SM sub-partition so the
//              exp/max/pack stream of one tile overlaps the other's)
//   warp 8     TMA: Q pair (double-buffered across items at Dh = 64), K/V ring (3 / 2 stages)
//   warps 9,10 MMA, one issuer per query tile: S_w = Q_w K^T (TMEM, one buffer per tile, re-issued as soon
//              as the softmax has pulled the previous S into registers), then
//              O_w += P_w V with P_w read from TMEM (tcgen05 "TS" form)
//   setmaxnreg moves registers from the TMA/MMA group to the softmax groups so
//   a whole 128-key score row stays in registers.
// TMEM: S0 | S1 | O0 | O1 | P0 | P1  (128 | 128 | 64 | 64 | 64 | 64 columns) at Dh = 64;
// S0 | S1 | O0 | O1 (128 each, P_w over S_w) at Dh = 128.
struct AttnPairArgs {
    int T, H, d, grid;
    const int32_t* seg;
    const int4* seg_info;
    const int32_t *p_ptr, *p_list;
    const int32_t *w_ptr, *w_items;  // per-CTA item lists (item = pair * H + head)
    // dynamic work queue (dyn): CTAs take items from `order` (n_items, longest or head-major
    // first) through one global counter: item = atomicAdd(ctr, 1) - base
    int dyn, n_items;
    const int32_t* order;
    unsigned* ctr;
    unsigned base;
    // grouped launch over nm models (same schedule, the tri-model forward): item =
    // model * n_base + pair * H + head, n_base = n_pairs * H; tensor maps per model
    int nm, n_base;
    float* lse[3];
    float scale_log2;
    long ldo;
};

struct AttnPairMaps {
    CUtensorMap qkv[3], out[3];
};

constexpr int PAIR_NTHR = 384;  // 3 warp groups: softmax 0, softmax 1, TMA/MMA
constexpr int KV_STAGES = 3;
constexpr uint32_t VIS0 = 1u << 24, FULL0 = 1u << 25, VIS1 = 1u << 26, FULL1 = 1u << 27;

template <int DH>
struct PairSmem {
    static constexpr int TILE = 128 * DH * 2;
    static constexpr int QB = DH == 128 ? 1 : 2;             // Q pair buffers (across items)
    static constexpr int KVS = DH == 128 ? 2 : KV_STAGES;    // K/V ring stages
    static constexpr int OFF_Q = 0;                          // [QB buffers][2 tiles]
    static constexpr int OFF_K = OFF_Q + 2 * QB * TILE;      // [KVS]
    static constexpr int OFF_V = OFF_K + KVS * TILE;         // [KVS]
    static constexpr int OFF_OST = OFF_V + KVS * TILE;       // [8 softmax warps][32 rows x 128 B] output staging
    static constexpr int OFF_BAR = OFF_OST + 8 * 4096;
    static constexpr int OFF_RING = OFF_BAR + 256;           // [4] item ids of the dynamic queue
    static constexpr int OFF_L0 = OFF_RING + 64;             // Dh 64: [2 items][256 softmax threads] row range start
    static constexpr int TOTAL = OFF_L0 + (DH == 64 ? 2 * 256 * 4 : 0) + 1024;
};

#ifndef ATTN_POLY_PAIRS
// of every 8 exp pairs of a full tile, how many run on the FMA pipe (packed-pair math).  With the
// FFMA2 / FADD2 softmax the Dh 64 forward is MUFU-bound: 1 pair +0.8%, 2 pairs +2.3% at C2
// (profiles/r02_ab_attn_poly_pairs.txt).  Off by default: a tile's exps then depend on whether it is
// full, so regrouping sequences (several prompt groups per sequence) would no longer be bit-identical.
#define ATTN_POLY_PAIRS 0
#endif

__device__ __forceinline__ float fmax3(float a, float b, float c) { return fmaxf(fmaxf(a, b), c); }

// bits [lo, hi) of the 32-column word starting at column c0 (lo / hi relative to the tile)
__device__ __forceinline__ uint32_t range_bits(int lo, int hi, int c0) {
    const int a = min(max(lo - c0, 0), 32), b = min(max(hi - c0, 0), 32);
    const uint32_t ub = b >= 32 ? 0xffffffffu : ((1u << b) - 1u), ua = a >= 32 ? 0xffffffffu : ((1u << a) - 1u);
    return ub & ~ua;
}

#ifdef PARL_ATTN_TRACE
// phase timestamps of CTA 0 (build with -DPARL_ATTN_TRACE; read by parl_debug_attn_trace)
__device__ unsigned long long g_attn_trace[16][64][8];
#define ATTN_TRACE(role, n, k)                                                                  \
    do {                                                                                        \
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (n) < 64) g_attn_trace[role][n][k] = clock64(); \
    } while (0)
// per-CTA [start, end] global time (ns) of the traced launch: roles 12.. hold CTA / 64
#define ATTN_SPAN(k)                                                                                  \
    do {                                                                                              \
        if (threadIdx.x == 0) {                                                                       \
            unsigned long long t_;                                                                    \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                    \
            g_attn_trace[12 + blockIdx.x / 64][blockIdx.x % 64][k] = t_;                              \
        }                                                                                             \
    } while (0)
#else
#define ATTN_SPAN(k) \
    do {             \
    } while (0)
#define ATTN_TRACE(role, n, k) \
    do {                       \
    } while (0)
#endif

template <int DH>
__global__ void __launch_bounds__(PAIR_NTHR, 1)
    k_attn_fwd_pair(const __grid_constant__ AttnPairMaps maps, AttnPairArgs a) {
    static_assert(DH == 64 || DH == 128, "head dim");
    using L = PairSmem<DH>;
    // TMEM: Dh = 64: S0 | S1 | O0 | O1 | P0 | P1; Dh = 128: S0 | S1 | O0 | O1 with P_w written
    // over S_w (the S of a tile's next key tile is then issued only behind its PV, which the
    // tensor pipe executes in issue order)
    constexpr bool P_IN_S = DH == 128;
    constexpr int KVS = L::KVS, QB = L::QB, PCOL = P_IN_S ? 128 : 64;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
    uint64_t* q_full = bar + 0;                   // [2]
    uint64_t* q_empty = bar + 2;                  // [2]
    uint64_t* kv_full = bar + 4;                  // [3]
    uint64_t* kv_empty = bar + 7;                 // [3]
    uint64_t* s_full = bar + 10;                  // [2 tiles][2 S buffers] (Dh = 64: buffer 0 only)
    uint64_t* s_free = bar + 14;                  // [2]
    uint64_t* p_full = bar + 16;                  // [2]
    uint64_t* o_done = bar + 18;                  // [2]
    uint64_t* o_free = bar + 20;                  // [2]
    uint32_t* tbase_s = reinterpret_cast<uint32_t*>(bar + 22);
    uint64_t* ring_full = bar + 24;               // [4] dynamic queue: item id published
    uint64_t* ring_empty = bar + 28;              // [4] released by the 2 MMA + 8 softmax warps
    volatile int* ring = reinterpret_cast<volatile int*>(smem + L::OFF_RING);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int H = a.H;

    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&q_full[s], 1);
            tc::mbar_init(&q_empty[s], 2);  // one release per MMA issuer
            tc::mbar_init(&s_full[2 * s], 1);
            tc::mbar_init(&s_full[2 * s + 1], 1);
            tc::mbar_init(&s_free[s], 4);
            tc::mbar_init(&p_full[s], 4);
            tc::mbar_init(&o_done[s], 1);
            tc::mbar_init(&o_free[s], 4);
        }
        for (int s = 0; s < KVS; ++s) {
            tc::mbar_init(&kv_full[s], 1);
            tc::mbar_init(&kv_empty[s], 2);
        }
        for (int s = 0; s < 4; ++s) {
            tc::mbar_init(&ring_full[s], 1);
            tc::mbar_init(&ring_empty[s], 10);
        }
        tc::fence_barrier_init();
        for (int m = 0; m < a.nm; ++m) tc::tma_prefetch(&maps.qkv[m]);
    }
    if (warp == 9) tc::tmem_alloc<512>(tbase_s);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tbase = *tbase_s;
    const uint32_t t_s = tbase, t_o = tbase + 256, t_p = P_IN_S ? tbase : tbase + 256 + 2 * DH;
    pdl_wait();
    pdl_trigger();
    ATTN_SPAN(0);

    // The li-th item of this CTA (-1: none left).  Static lists, or the dynamic queue: the TMA
    // thread publishes item li + 1 before it loads item li, so a consumer working on item li
    // may always look at li + 1; consumers release an item's slot when done with it.
    auto item_at = [&](int li) -> int {
        if (!a.dyn) {
            const int k = a.w_ptr[blockIdx.x] + li;
            return k < a.w_ptr[blockIdx.x + 1] ? a.w_items[k] : -1;
        }
        tc::mbar_wait(&ring_full[li & 3], (li >> 2) & 1);
        return ring[li & 3];
    };
    auto item_done = [&](int li) {
        if (a.dyn && lane == 0) tc::mbar_arrive(&ring_empty[li & 3]);
    };

    // Per-row metadata of a softmax item (prefetched one item ahead): pair p, head h, row i,
    // the row's allowed key ranges [l0, e0) u [b1, e1) (model.cpp:242-245), the pair's entry
    // range and its first entry
    struct ItemMeta {
        int p, h, i, l0, e0, b1, e1, ea, eb;
        uint32_t f0;
        int mdl;
    };
    auto fetch_item = [&](int li, int w, int r) -> ItemMeta {  // p < 0: no item li
        ItemMeta m{-1, 0, a.T, 0, 0, 0, 0, 0, 0, 0u, 0};
        const int it = item_at(li);
        if (it < 0) return m;
        m.mdl = it / a.n_base;
        m.p = (it % a.n_base) / H;
        m.h = it % H;
        m.i = (2 * m.p + w) * 128 + r;
        const bool row_ok = m.i < a.T;
        const int4 f = row_ok ? a.seg_info[a.seg[m.i]] : make_int4(0, 0, 0, 0);
        const bool resp = row_ok && f.y >= 0;
        m.l0 = f.x;
        // Dh 64: the score row leaves no register for it; kept in shared memory by item parity
        if constexpr (DH == 64) reinterpret_cast<int*>(smem + L::OFF_L0)[(li & 1) * 256 + warp * 32 + lane] = f.x;
        m.e0 = !row_ok ? 0 : (resp ? f.y : m.i + 1);
        m.b1 = resp ? f.z : 0;
        m.e1 = resp ? m.i + 1 : 0;
        m.ea = a.p_ptr[m.p];
        m.eb = a.p_ptr[m.p + 1];
        m.f0 = m.ea < m.eb ? (uint32_t)a.p_list[m.ea] : 0u;
        return m;
    };

    // Item epilogue of a softmax warp: O / l (fp32, TMEM) -> bf16 rows of `out`, staged per
    // warp through a 128B-swizzled 32 x 64 smem slab and written by TMA (coalesced; the
    // rows past T are clipped by the tensor map), then lse.  Releases O after the last load.
    auto store_out = [&](uint32_t t_ow, int w, int q4, int mdl, int p, int h, int i, bool row_ok, float l,
                         float m_used) {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        const uint32_t slab = tc::smem_u32(smem + L::OFF_OST + warp * 4096);
#pragma unroll
        for (int hc = 0; hc < DH / 64; ++hc) {
            float o[64];
            tc::tmem_ld32_nowait(t_ow + hc * 64, reinterpret_cast<uint32_t*>(o));
            tc::tmem_ld32_nowait(t_ow + hc * 64 + 32, reinterpret_cast<uint32_t*>(o) + 32);
            tc::tmem_ld_wait();
            if (hc == DH / 64 - 1) {
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&o_free[w]);
            }
            if (lane == 0) tc::bulk_wait_read<0>();  // the slab's previous store has been read
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 8; ++c)
                tc::sts128(slab + lane * 128 + ((c ^ (lane & 7)) << 4), pack2(o[8 * c] * inv, o[8 * c + 1] * inv),
                           pack2(o[8 * c + 2] * inv, o[8 * c + 3] * inv), pack2(o[8 * c + 4] * inv, o[8 * c + 5] * inv),
                           pack2(o[8 * c + 6] * inv, o[8 * c + 7] * inv));
            tc::fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                tc::tma_store_2d(&maps.out[mdl], slab, h * DH + hc * 64, (2 * p + w) * 128 + q4 * 32);
                tc::bulk_commit();
            }
        }
        if (row_ok) a.lse[mdl][(long)h * a.T + i] = (m_used + log2f(l)) * 0.69314718055994531f;
    };

    // ---- Dh = 128: key tiles are processed as two 64-key chunks so that each query tile
    // has two S buffers (64 TMEM columns each) next to its 128-column O: the S MMA of the
    // next chunk runs while the softmax works on the current one.  P (bf16, 32 columns)
    // is written over its chunk's S buffer, which the S MMA two chunks later reuses only
    // behind this chunk's PV (in-order tensor pipe).  s_full has one barrier per buffer.
    auto mma_issuer_dh128 = [&]() {
      if constexpr (DH == 128) {
        const int w = warp - 9;
        const uint32_t VIS = w ? VIS1 : VIS0;
        constexpr uint32_t id_s = tc::idesc_bf16(128, 64, 0, 0);
        constexpr uint32_t id_o = tc::idesc_bf16(128, DH, 0, 1);
        const uint32_t t_sw = t_s + w * 128, t_ow = t_o + w * DH;
        int cS = 0, cP = 0, nI = 0;  // chunk counters
        int s_it = item_at(0), s_li = 0, s_e = 0, s_end = 0, gS = 0, s_h = 0;
        auto s_load_item = [&]() {
            if (s_it >= 0) {
                const int p = (s_it % a.n_base) / H;
                s_e = a.p_ptr[p];
                s_end = a.p_ptr[p + 1];
            }
        };
        // next visible (entry, chunk) of this tile, at most QB - 1 items past li_now
        auto s_seek = [&](int li_now) -> bool {
            while (s_it >= 0) {
                if (s_e >= s_end) {
                    if (s_li + 1 > li_now + QB - 1) return false;
                    s_it = item_at(++s_li);
                    s_load_item();
                    continue;
                }
                if ((uint32_t)a.p_list[s_e] & VIS) return true;
                ++s_e;
                ++gS;
            }
            return false;
        };
        s_load_item();
        auto issue_s = [&]() {
            const int st = gS % KVS, qb = s_li % QB;
            tc::mbar_wait(&q_full[qb], (s_li / QB) & 1);
            tc::mbar_wait(&kv_full[st], (gS / KVS) & 1);
            tc::tc_fence_after();
            const uint32_t sk = tc::smem_u32(smem + L::OFF_K + st * L::TILE) + s_h * (64 * 128);
            const uint32_t sq = tc::smem_u32(smem + L::OFF_Q + (qb * 2 + w) * L::TILE);
#pragma unroll
            for (int ks = 0; ks < DH / 16; ++ks) {
                const uint32_t off = (ks >> 2) * (128 * 128) + (ks & 3) * 32;
                tc::mma_bf16_e(t_sw + (cS & 1) * 64, tc::sdesc(sq + off, 16, 1024), tc::sdesc(sk + off, 16, 1024),
                               id_s, ks > 0);
            }
            tc::mma_commit_e(&s_full[2 * w + (cS & 1)]);
            ATTN_TRACE(2 + w, cS, 0);
            ++cS;
            if (++s_h == 2) {
                s_h = 0;
                ++s_e;
                ++gS;
                // last S of this tile in the item: Q is no longer read (PV does not use it), so
                // its buffer goes back to the TMA producer now, not after the item's last PV
                bool more = false;
                for (int e2 = s_e; e2 < s_end && !more; ++e2) more = ((uint32_t)a.p_list[e2] & VIS) != 0;
                if (!more) tc::mma_commit_e(&q_empty[qb]);
            }
        };
        // S of chunk n reuses the buffer of chunk n - 2: issued after PV(n - 2) (cS < cP + 2);
        // within the K/V ring window and the Q buffers this issuer has released
        auto advance_s = [&](int g_now, int li_now) {
            while (cS < cP + 2 && s_seek(li_now) && gS <= g_now + KVS - 1 && s_li <= li_now + QB - 1) issue_s();
        };
        int g = 0;
        for (int li = 0;; ++li) {
            const int itm = item_at(li);
            if (itm < 0) break;
            const int p = (itm % a.n_base) / H, qb = li % QB;
            const int ea = a.p_ptr[p], eb = a.p_ptr[p + 1];
            bool started = false;
            for (int e = ea; e < eb; ++e, ++g) {
                const uint32_t f = (uint32_t)a.p_list[e];
                const int st = g % KVS;
                advance_s(g, li);
                if (!(f & VIS)) {
                    tc::mbar_wait(&kv_full[st], (g / KVS) & 1);
                    if (lane == 0) tc::mbar_arrive(&kv_empty[st]);
                    continue;
                }
                const uint32_t sv = tc::smem_u32(smem + L::OFF_V + st * L::TILE);
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    advance_s(g, li);
                    ATTN_TRACE(2 + w, cP, 1);
                    tc::mbar_wait(&p_full[w], cP & 1);
                    if (!started && nI > 0) tc::mbar_wait(&o_free[w], (nI - 1) & 1);
                    tc::tc_fence_after();
                    ATTN_TRACE(2 + w, cP, 2);
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        tc::mma_bf16_ts_e(t_ow, t_sw + (cP & 1) * 64 + ks * 8,
                                          tc::sdesc(sv + h * (64 * 128) + ks * 2048, 128 * 128, 1024), id_o,
                                          (started || ks > 0) ? 1u : 0u);
                    tc::mma_commit_e(&o_done[w]);
                    if (h == 1) tc::mma_commit_e(&kv_empty[st]);
                    ++cP;
                    if (!started) {
                        started = true;
                        ++nI;
                    }
                }
                advance_s(g, li);
            }
            if (!started) {  // (released after the last S otherwise)
                tc::mbar_wait(&q_full[qb], (li / QB) & 1);
                if (lane == 0) tc::mbar_arrive(&q_empty[qb]);
            }
            item_done(li);
        }
      }
    };
    auto softmax_dh128 = [&]() {
      if constexpr (DH == 128) {
        const int w = warp >> 2, q4 = warp & 3;
        const int r = q4 * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
        const uint32_t VIS = w ? VIS1 : VIS0, FULL = w ? FULL1 : FULL0;
        const uint32_t t_sw = t_s + w * 128 + lane_off, t_ow = t_o + w * DH + lane_off;
        const float c2 = a.scale_log2;
        int cS = 0;
        ItemMeta nx = fetch_item(0, w, r);
        for (int k = 0; nx.p >= 0; ++k) {
            const ItemMeta cur = nx;
            nx = fetch_item(k + 1, w, r);  // the next item's chain of dependent loads, off the critical path
            const int p = cur.p, h = cur.h, i = cur.i, l0 = cur.l0, e0 = cur.e0, b1 = cur.b1, e1 = cur.e1;
            const bool row_ok = i < a.T;
            float m_used = -INFINITY, l = 0.f;
            bool first = true;
            for (int e = cur.ea; e < cur.eb; ++e) {
                const uint32_t f = e == cur.ea ? cur.f0 : (uint32_t)a.p_list[e];
                if (!(f & VIS)) continue;
#pragma unroll 1
                for (int hc = 0; hc < 2; ++hc) {
                    const int buf = cS & 1;
                    if (q4 == 0) ATTN_TRACE(w, cS, 0);
                    tc::mbar_wait(&s_full[2 * w + buf], (cS >> 1) & 1);
                    tc::tc_fence_after();
                    if (q4 == 0) ATTN_TRACE(w, cS, 1);
                    float sv[64];
                    tc::tmem_ld32_nowait(t_sw + buf * 64, reinterpret_cast<uint32_t*>(sv));
                    tc::tmem_ld32_nowait(t_sw + buf * 64 + 32, reinterpret_cast<uint32_t*>(sv) + 32);
                    tc::tmem_ld_wait();
                    if (q4 == 0) ATTN_TRACE(w, cS, 2);
                    if (!(f & FULL)) {
                        // allowed keys [l0, e0) u [b1, e1) as a column bitmask (no per-element range math)
                        const int j0 = (int)(f & 0xffffff) * 128 + hc * 64;
                        uint32_t mw[2];
#pragma unroll
                        for (int q = 0; q < 2; ++q)
                            mw[q] = range_bits(l0 - j0, e0 - j0, 32 * q) | range_bits(b1 - j0, e1 - j0, 32 * q);
#pragma unroll
                        for (int j = 0; j < 64; ++j) sv[j] = ((mw[j >> 5] >> (j & 31)) & 1u) ? sv[j] : -INFINITY;
                    }
                    float mq[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) mq[q] = fmaxf(sv[q], sv[q + 4]);
#pragma unroll
                    for (int j = 8; j < 64; j += 8) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) mq[q] = fmax3(mq[q], sv[j + 2 * q], sv[j + 2 * q + 1]);
                    }
                    const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
                    const float mxl = mx * c2;
                    const bool need = mxl > m_used + 8.f;
                    const float m_new = need ? mxl : m_used;
                    const float alpha = need ? tc::ex2_approx(m_used - m_new) : 1.f;
                    const float mb = m_new == -INFINITY ? 0.f : m_new;
                    float sm0 = 0.f, sm1 = 0.f, sm2 = 0.f, sm3 = 0.f;
                    uint32_t pk[32];
                    {  // packed fp32 pairs (FFMA2 / FADD2), the same per-lane arithmetic and sum order
                        const float2 c22 = make_float2(c2, c2), mb2 = make_float2(-mb, -mb);
                        float2 s01 = make_float2(0.f, 0.f), s23 = make_float2(0.f, 0.f);
#pragma unroll
                        for (int j = 0; j < 64; j += 4) {
                            const float2 a01 = tc::ffma2(make_float2(sv[j], sv[j + 1]), c22, mb2);
                            const float2 a23 = tc::ffma2(make_float2(sv[j + 2], sv[j + 3]), c22, mb2);
                            const float2 p01 = make_float2(tc::ex2_approx(a01.x), tc::ex2_approx(a01.y));
                            const float2 p23 = make_float2(tc::ex2_approx(a23.x), tc::ex2_approx(a23.y));
                            s01 = tc::fadd2(s01, p01);
                            s23 = tc::fadd2(s23, p23);
                            pk[j / 2] = pack2(p01.x, p01.y);
                            pk[j / 2 + 1] = pack2(p23.x, p23.y);
                        }
                        sm0 = s01.x; sm1 = s01.y; sm2 = s23.x; sm3 = s23.y;
                    }
                    if (q4 == 0) ATTN_TRACE(w, cS, 3);
                    // the previous chunk's PV has finished writing O
                    if (cS > 0) {
                        tc::mbar_wait(&o_done[w], (cS - 1) & 1);
                        tc::tc_fence_after();
                    }
                    if (q4 == 0) ATTN_TRACE(w, cS, 4);
                    if (!first && __any_sync(0xffffffffu, need)) {
#pragma unroll
                        for (int c = 0; c < DH / 32; ++c) {
                            float o[32];
                            tc::tmem_ld32(t_ow + c * 32, o);
                            uint32_t wv[32];
#pragma unroll
                            for (int q = 0; q < 32; ++q) wv[q] = __float_as_uint(o[q] * alpha);
                            tc::tmem_st16(t_ow + c * 32, wv);
                            tc::tmem_st16(t_ow + c * 32 + 16, wv + 16);
                        }
                    }
                    tc::tmem_st16(t_sw + buf * 64, pk);
                    tc::tmem_st16(t_sw + buf * 64 + 16, pk + 16);
                    tc::tmem_st_wait();
                    tc::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive(&p_full[w]);
                    if (q4 == 0) ATTN_TRACE(w, cS, 5);
                    l = l * alpha + ((sm0 + sm1) + (sm2 + sm3));
                    m_used = m_new;
                    first = false;
                    ++cS;
                }
            }
            if (first) {  // no key tile for this query tile (past the end)
                item_done(k);
                continue;
            }
            tc::mbar_wait(&o_done[w], (cS - 1) & 1);
            tc::tc_fence_after();
            if (q4 == 0) ATTN_TRACE(w, cS - 1, 6);
            store_out(t_ow, w, q4, cur.mdl, p, h, i, row_ok, l, m_used);
            if (q4 == 0) ATTN_TRACE(w, cS - 1, 7);
            item_done(k);
        }
      }
    };

    if (warp >= 8) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
      if (warp == 8) {
        if (lane == 0) {  // ---------------- TMA
            int g = 0;
            int published = -1;  // dynamic queue: last published slot index
            bool ended = false;
            auto publish = [&](int n) {  // fetch item n of this CTA from the global counter
                tc::mbar_wait(&ring_empty[n & 3], ((n >> 2) & 1) ^ 1);
                const unsigned v = atomicAdd(a.ctr, 1u) - a.base;
                // queue position v: base item order[v / nm] (longest / head-major first) of model v % nm
                const int it = v < (unsigned)a.n_items ? (int)(v % a.nm) * a.n_base + a.order[v / a.nm] : -1;
                ring[n & 3] = it;
                tc::mbar_arrive(&ring_full[n & 3]);
                published = n;
                ended = it < 0;
            };
            if (a.dyn) publish(0);
            for (int li = 0;; ++li) {
                const int it = a.dyn ? ring[li & 3] : item_at(li);
                if (it < 0) break;
                if (a.dyn && !ended && published == li) publish(li + 1);
                const int mdl = it / a.n_base, p = (it % a.n_base) / H, h = it % H, qb = li % QB;
                const CUtensorMap* tm_qkv = &maps.qkv[mdl];
                tc::mbar_wait(&q_empty[qb], ((li / QB) & 1) ^ 1);
                tc::mbar_expect_tx(&q_full[qb], 2 * L::TILE);
#pragma unroll
                for (int w = 0; w < 2; ++w)
#pragma unroll
                    for (int r = 0; r < DH / 64; ++r)
                        tc::tma_load_2d(smem + L::OFF_Q + (qb * 2 + w) * L::TILE + r * 128 * 128, tm_qkv, &q_full[qb],
                                        h * DH + r * 64, (2 * p + w) * 128);
                for (int e = a.p_ptr[p]; e < a.p_ptr[p + 1]; ++e, ++g) {
                    const int j0 = (a.p_list[e] & 0xffffff) * 128;
                    const int st = g % KVS;
                    tc::mbar_wait(&kv_empty[st], ((g / KVS) & 1) ^ 1);
                    tc::mbar_expect_tx(&kv_full[st], 2 * L::TILE);
#pragma unroll
                    for (int r = 0; r < DH / 64; ++r) {
                        tc::tma_load_2d(smem + L::OFF_K + st * L::TILE + r * 128 * 128, tm_qkv, &kv_full[st],
                                        a.d + h * DH + r * 64, j0);
                        tc::tma_load_2d(smem + L::OFF_V + st * L::TILE + r * 128 * 128, tm_qkv, &kv_full[st],
                                        2 * a.d + h * DH + r * 64, j0);
                    }
                }
            }
        }
    } else if ((warp == 9 || warp == 10) && DH == 128) {
        mma_issuer_dh128();
    } else if (warp == 9 || warp == 10) {  // whole warp; one elected lane issues
        // ---------------- MMA issuers: warp 9 serves query tile 0, warp 10 tile 1,
        // so neither softmax group waits on the other's progress.  K/V stages and
        // the Q pair are released when both issuers are done with them.
        const int w = warp - 9;
        const uint32_t VIS = w ? VIS1 : VIS0;
        constexpr uint32_t id_s = tc::idesc_bf16(128, 128, 0, 0);
        constexpr uint32_t id_o = tc::idesc_bf16(128, DH, 0, 1);
        int cS = 0, cP = 0, nI = 0;
        // S look-ahead over the entries visible to this tile.  A look-ahead S may only
        // wait for a K/V stage that cannot depend on this thread's own later releases:
        // its entry must lie within KV_STAGES - 1 of the entry being processed (a tile
        // whose pair partner sees many more key tiles skips long runs of entries).
        int s_it = item_at(0), s_li = 0, s_e = 0, s_end = 0, gS = 0;
        auto s_load_item = [&]() {
            if (s_it >= 0) {
                const int p = (s_it % a.n_base) / H;
                s_e = a.p_ptr[p];
                s_end = a.p_ptr[p + 1];
            }
        };
        // move the iterator to the next entry visible to this tile (global index gS), at most
        // QB - 1 items past li_now; false at the end
        auto s_seek = [&](int li_now) -> bool {
            while (s_it >= 0) {
                if (s_e >= s_end) {
                    if (s_li + 1 > li_now + QB - 1) return false;
                    s_it = item_at(++s_li);
                    s_load_item();
                    continue;
                }
                if ((uint32_t)a.p_list[s_e] & VIS) return true;
                ++s_e;
                ++gS;
            }
            return false;
        };
        s_load_item();
        auto issue_s = [&]() {  // S for the iterator's entry (visible, gS)
            const int g = gS, st = g % KVS, qb = s_li % QB;
            tc::mbar_wait(&q_full[qb], (s_li / QB) & 1);
            tc::mbar_wait(&kv_full[st], (g / KVS) & 1);
            if (cS > 0) tc::mbar_wait(&s_free[w], (cS - 1) & 1);
            tc::tc_fence_after();
            const uint32_t sk = tc::smem_u32(smem + L::OFF_K + st * L::TILE);
            const uint32_t sq = tc::smem_u32(smem + L::OFF_Q + (qb * 2 + w) * L::TILE);
#pragma unroll
            for (int ks = 0; ks < DH / 16; ++ks) {
                const uint32_t off = (ks >> 2) * (128 * 128) + (ks & 3) * 32;
                tc::mma_bf16_e(t_s + w * 128, tc::sdesc(sq + off, 16, 1024), tc::sdesc(sk + off, 16, 1024), id_s,
                               ks > 0);
            }
            tc::mma_commit_e(&s_full[2 * w]);
            ATTN_TRACE(2 + w, cS, 0);
            ++cS;
            ++s_e;
            ++gS;
        };
        // issue pending S (at most one beyond the tile being processed) within the stage window
        // (and at most QB - 1 items ahead: the Q buffer of a later item is freed by this
        // issuer's own end-of-item release)
        auto advance_s = [&](int g_now, int li_now) {
            while (cS < cP + (P_IN_S ? 1 : 2) && s_seek(li_now) && gS <= g_now + KVS - 1 && s_li <= li_now + QB - 1)
                issue_s();
        };
        int g = 0;
        for (int li = 0;; ++li) {
            const int itm = item_at(li);
            if (itm < 0) break;
            const int p = (itm % a.n_base) / H, qb = li % QB;
            const int ea = a.p_ptr[p], eb = a.p_ptr[p + 1];
            bool started = false;
            for (int e = ea; e < eb; ++e, ++g) {
                const uint32_t f = (uint32_t)a.p_list[e];
                const int st = g % KVS;
                advance_s(g, li);  // S of this entry (if not yet issued) and of the next visible one
                if (!(f & VIS)) {  // not ours: release the stage once it holds this entry
                    tc::mbar_wait(&kv_full[st], (g / KVS) & 1);
                    if (lane == 0) tc::mbar_arrive(&kv_empty[st]);
                    continue;
                }
                ATTN_TRACE(2 + w, cP, 1);
                tc::mbar_wait(&p_full[w], cP & 1);
                if (!started && nI > 0) tc::mbar_wait(&o_free[w], (nI - 1) & 1);
                tc::tc_fence_after();
                ATTN_TRACE(2 + w, cP, 2);
                const uint32_t sv = tc::smem_u32(smem + L::OFF_V + st * L::TILE);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    tc::mma_bf16_ts_e(t_o + w * DH, t_p + w * PCOL + ks * 8, tc::sdesc(sv + ks * 2048, 128 * 128, 1024),
                                      id_o, (started || ks > 0) ? 1u : 0u);
                tc::mma_commit_e(&o_done[w]);
                tc::mma_commit_e(&kv_empty[st]);
                ++cP;
                if (!started) {
                    started = true;
                    ++nI;
                }
                advance_s(g, li);  // look ahead right after handing this PV off
            }
            if (started) {
                tc::mma_commit_e(&q_empty[qb]);
            } else {
                tc::mbar_wait(&q_full[qb], (li / QB) & 1);
                if (lane == 0) tc::mbar_arrive(&q_empty[qb]);
            }
            item_done(li);
        }
      }
    } else if (DH == 128) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
        softmax_dh128();
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
        // ---------------- softmax: warp group w = query tile w of the pair
        const int w = warp >> 2, q4 = warp & 3;
        const int r = q4 * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
        const uint32_t VIS = w ? VIS1 : VIS0, FULL = w ? FULL1 : FULL0;
        const float c2 = a.scale_log2;
        int cS = 0;
        ItemMeta nx = fetch_item(0, w, r);
        for (int k = 0; nx.p >= 0; ++k) {
            const ItemMeta cur = nx;
            nx = fetch_item(k + 1, w, r);  // the next item's chain of dependent loads, off the critical path
            const int p = cur.p, h = cur.h, i = cur.i, e0 = cur.e0, b1 = cur.b1, e1 = cur.e1;
            const int* l0_slot = reinterpret_cast<const int*>(smem + L::OFF_L0) + (k & 1) * 256 + warp * 32 + lane;
            const bool row_ok = i < a.T;
            float m_used = -INFINITY, l = 0.f;
            bool first = true;
            for (int e = cur.ea; e < cur.eb; ++e) {
                const uint32_t f = e == cur.ea ? cur.f0 : (uint32_t)a.p_list[e];
                if (!(f & VIS)) continue;
                if (q4 == 0) ATTN_TRACE(w, cS, 0);
                tc::mbar_wait(&s_full[2 * w], cS & 1);
                tc::tc_fence_after();
                if (q4 == 0) ATTN_TRACE(w, cS, 1);
                float sv[128];
                tc::tmem_ld128(t_s + w * 128 + lane_off, sv);
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&s_free[w]);  // the next S of this tile may be issued
                if (q4 == 0) ATTN_TRACE(w, cS, 2);
                if (!(f & FULL)) {
                    // allowed keys [l0, e0) u [b1, e1) as a column bitmask (no per-element range math)
                    const int j0 = (int)(f & 0xffffff) * 128, l0 = *l0_slot;
                    uint32_t mw[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        mw[q] = range_bits(l0 - j0, e0 - j0, 32 * q) | range_bits(b1 - j0, e1 - j0, 32 * q);
#pragma unroll
                    for (int j = 0; j < 128; ++j) sv[j] = ((mw[j >> 5] >> (j & 31)) & 1u) ? sv[j] : -INFINITY;
                }
                float mq[4];  // four independent max chains
#pragma unroll
                for (int q = 0; q < 4; ++q) mq[q] = fmaxf(sv[q], sv[q + 4]);
#pragma unroll
                for (int j = 8; j < 128; j += 8) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) mq[q] = fmax3(mq[q], sv[j + 2 * q], sv[j + 2 * q + 1]);
                }
                const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
                const float mxl = mx * c2;
                const bool need = mxl > m_used + 8.f;
                const float m_new = need ? mxl : m_used;
                const float alpha = need ? tc::ex2_approx(m_used - m_new) : 1.f;
                const float mb = m_new == -INFINITY ? 0.f : m_new;
                // P = exp2(S * c - m) -> bf16 (registers)
                float sm0 = 0.f, sm1 = 0.f, sm2 = 0.f, sm3 = 0.f;
                uint32_t pk[64];
                if (ATTN_POLY_PAIRS != 0 && (f & FULL)) {
                    // FA4-style: the last ATTN_POLY_PAIRS pairs of every 16 exps on the FMA pipe, the rest on
                    // MUFU (full tiles only: masked -inf scores need MUFU's exact zero)
                    const float2 c22 = make_float2(c2, c2), mb2 = make_float2(-mb, -mb);
                    float2 s01 = make_float2(0.f, 0.f), s23 = make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < 128; j += 16) {
#pragma unroll
                        for (int q = 0; q < 16; q += 4) {
                            const float2 a01 = tc::ffma2(make_float2(sv[j + q], sv[j + q + 1]), c22, mb2);
                            const float2 a23 = tc::ffma2(make_float2(sv[j + q + 2], sv[j + q + 3]), c22, mb2);
                            const bool poly01 = (q / 2) >= 8 - ATTN_POLY_PAIRS, poly23 = (q / 2 + 1) >= 8 - ATTN_POLY_PAIRS;
                            const float2 p01 = poly01 ? tc::exp2_fma2(a01)
                                                      : make_float2(tc::ex2_approx(a01.x), tc::ex2_approx(a01.y));
                            const float2 p23 = poly23 ? tc::exp2_fma2(a23)
                                                      : make_float2(tc::ex2_approx(a23.x), tc::ex2_approx(a23.y));
                            s01 = tc::fadd2(s01, p01);
                            s23 = tc::fadd2(s23, p23);
                            pk[(j + q) / 2] = pack2(p01.x, p01.y);
                            pk[(j + q) / 2 + 1] = pack2(p23.x, p23.y);
                        }
                    }
                    sm0 = s01.x; sm1 = s01.y; sm2 = s23.x; sm3 = s23.y;
                } else {  // masked scores are -inf: MUFU gives their exact zero
                    // packed fp32 pairs: one FFMA2 per two arguments, one FADD2 per two row-sum terms
                    const float2 c22 = make_float2(c2, c2), mb2 = make_float2(-mb, -mb);
                    float2 s01 = make_float2(0.f, 0.f), s23 = make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < 128; j += 4) {
                        const float2 a01 = tc::ffma2(make_float2(sv[j], sv[j + 1]), c22, mb2);
                        const float2 a23 = tc::ffma2(make_float2(sv[j + 2], sv[j + 3]), c22, mb2);
                        const float2 p01 = make_float2(tc::ex2_approx(a01.x), tc::ex2_approx(a01.y));
                        const float2 p23 = make_float2(tc::ex2_approx(a23.x), tc::ex2_approx(a23.y));
                        s01 = tc::fadd2(s01, p01);
                        s23 = tc::fadd2(s23, p23);
                        pk[j / 2] = pack2(p01.x, p01.y);
                        pk[j / 2 + 1] = pack2(p23.x, p23.y);
                    }
                    sm0 = s01.x; sm1 = s01.y; sm2 = s23.x; sm3 = s23.y;
                }
                if (q4 == 0) ATTN_TRACE(w, cS, 3);
                // the previous PV of this tile has finished reading P and writing O
                if (cS > 0) {
                    tc::mbar_wait(&o_done[w], (cS - 1) & 1);
                    tc::tc_fence_after();
                }
                if (q4 == 0) ATTN_TRACE(w, cS, 4);
                if (!first && __any_sync(0xffffffffu, need)) {
#pragma unroll
                    for (int c = 0; c < DH / 32; ++c) {
                        float o[32];
                        tc::tmem_ld32(t_o + w * DH + c * 32 + lane_off, o);
                        uint32_t wv[32];
#pragma unroll
                        for (int q = 0; q < 32; ++q) wv[q] = __float_as_uint(o[q] * alpha);
                        tc::tmem_st16(t_o + w * DH + c * 32 + lane_off, wv);
                        tc::tmem_st16(t_o + w * DH + c * 32 + 16 + lane_off, wv + 16);
                    }
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) tc::tmem_st16(t_p + w * PCOL + c * 16 + lane_off, pk + 16 * c);
                tc::tmem_st_wait();
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&p_full[w]);
                if (q4 == 0) ATTN_TRACE(w, cS, 5);
                l = l * alpha + ((sm0 + sm1) + (sm2 + sm3));
                m_used = m_new;
                first = false;
                ++cS;
            }
            if (first) {  // no key tile for this query tile (past the end)
                item_done(k);
                continue;
            }
            // item epilogue: O / l -> out (bf16), lse; then release O to the next item
            tc::mbar_wait(&o_done[w], (cS - 1) & 1);
            tc::tc_fence_after();
            store_out(t_o + w * DH + lane_off, w, q4, cur.mdl, p, h, i, row_ok, l, m_used);
            item_done(k);
        }
    }
    if (warp < 8 && lane == 0) tc::bulk_wait<0>();  // output stores complete before the CTA exits
    tc::tc_fence_before();
    __syncthreads();
    ATTN_SPAN(1);
    if (warp == 9) {
        tc::tc_fence_after();
        tc::tmem_dealloc<512>(tbase);
    }
}


// Backward prologue for the v2 kernels: D = rowsum(dO * O) per (head, row),
// lse in log2 units, and per-row visibility bounds {qhi, b1, l0, e0} (b1 = -1
// for prompt rows): key j is seen by queries [j, qhi_j); query i sees keys
// [l0, e0) u [b1, i] with e0 = i + 1 (prompt row) or its group's prompt end.
__device__ __forceinline__ int4 row_meta(const int4 f) {
    return make_int4(f.w, f.y < 0 ? -1 : f.z, f.x, f.y);
}

__global__ void k_attn_prep(int T, int H, int d, int Dh, long ldo, const int32_t* __restrict__ seg,
                            const int4* __restrict__ seg_info, const bf16* __restrict__ out,
                            const bf16* __restrict__ dout, const float* __restrict__ lse, float* __restrict__ dsum,
                            float* __restrict__ lse2, int4* __restrict__ meta) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const long gw = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw >= (long)T * H) return;
    const int h = (int)(gw / T), i = (int)(gw % T);
    float acc = 0.f;
    for (int c = 2 * lane; c < Dh; c += 64) {
        const __nv_bfloat162 o2 = *reinterpret_cast<const __nv_bfloat162*>(out + (long)i * ldo + h * Dh + c);
        const __nv_bfloat162 g2 = *reinterpret_cast<const __nv_bfloat162*>(dout + (long)i * d + h * Dh + c);
        acc += __bfloat162float(o2.x) * __bfloat162float(g2.x) + __bfloat162float(o2.y) * __bfloat162float(g2.y);
    }
    acc = warp_sum(acc);
    if (lane == 0) {
        dsum[(long)h * T + i] = acc;
        lse2[(long)h * T + i] = lse[(long)h * T + i] * LOG2E;
    }
    if (h == 0 && lane == 1) meta[i] = row_meta(seg_info[seg[i]]);
}

// The same prologue with 16-byte loads: thread = 8 consecutive columns of one row, the
// G = Dh / 8 threads of a head reduce by shuffles (G <= 32, aligned groups of a warp);
// a block covers whole rows, so every warp streams 512 contiguous bytes of O and dO.
template <int G>
__global__ void __launch_bounds__(256) k_attn_prep_v8(int T, int H, int d, long ldo, const int32_t* __restrict__ seg,
                                                      const int4* __restrict__ seg_info, const bf16* __restrict__ out,
                                                      const bf16* __restrict__ dout, const float* __restrict__ lse,
                                                      float* __restrict__ dsum, float* __restrict__ lse2,
                                                      int4* __restrict__ meta) {
    pdl_wait();
    const int d8 = d >> 3;
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool ok = t < (long)T * d8;
    const int i = ok ? (int)(t / d8) : 0, c8 = ok ? (int)(t % d8) : 0;
    float acc = 0.f;
    if (ok) {
        const uint4 o = *reinterpret_cast<const uint4*>(out + (long)i * ldo + 8 * c8);
        const uint4 g = *reinterpret_cast<const uint4*>(dout + (long)i * d + 8 * c8);
        const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&o);
        const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 a = __bfloat1622float2(o2[q]), b = __bfloat1622float2(g2[q]);
            acc = fmaf(a.x, b.x, acc);
            acc = fmaf(a.y, b.y, acc);
        }
    }
#pragma unroll
    for (int m = G / 2; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (ok && c8 % G == 0) {
        const long hi = (long)(c8 / G) * T + i;
        dsum[hi] = acc;
        lse2[hi] = lse[hi] * LOG2E;
    }
    if (ok && c8 == 0) meta[i] = row_meta(seg_info[seg[i]]);
}

struct BwdWs {
    void* p = nullptr;
    size_t bytes = 0;
    void* get(size_t need) {
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
BwdWs g_bwd_ws;

// ===========================================================================
// Backward v2 (Dh = 64): persistent CTAs over LPT-balanced work lists.
//   MODE_DKV: item = (key tile, head); streams the query tiles that see it:
//             S^T = K Q^T, dP^T = V dO^T, P^T = exp2(S^T c - lse), dS^T = P^T (dP^T - D),
//             dV += P^T dO, dK += dS^T Q           (thread = key row)
//   MODE_DQ:  item = (query tile, head); streams its visible key tiles:
//             S = Q K^T, dP = dO V^T, dS = P (dP - D), dQ += dS K   (thread = query row)
// Roles (12 warps): 0-7 element-wise (warp w: TMEM lane quadrant w%4, 64 of the
// tile's 128 columns), 8 TMA (+ the per-query lse / D vectors for MODE_DKV),
// 9 MMA issuer.  P and dS go to TMEM and feed the gradient MMAs as the A
// operand (TS form).  S/dP of the next streamed tile (possibly of the next
// item) are issued as soon as the element-wise warps have read the current
// ones.  No atomics: every output row is written by exactly one CTA.
// TMEM: S | dP | acc1 | acc2 | P | dS = 128 | 128 | 64 | 64 | 64 | 64 columns.
enum { MODE_DKV = 0, MODE_DQ = 1 };

struct AttnBwd2Args {
    int T, H, d;
    const int32_t *lst_ptr, *lst;    // per item tile: partner tiles (k_ptr/k_list or q_ptr/q_list)
    const int32_t *w_ptr, *w_items;  // per-CTA items (tile * H + head)
    float scale, scale_log2;
    const float* lse2;  // [H x T] log-sum-exp in log2 units
    const float* dsum;  // [H x T]
    const int4* meta;   // [T] {qhi, b1, l0, e0} (k_attn_prep)
    bf16* dqkv;         // [T x 3d]
};

constexpr int BWD_NTHR = 384;
constexpr int BWD_ST = 4;

template <int DH>
struct Bwd2Smem {
    static constexpr int TILE = 128 * DH * 2;
    static constexpr int AB = DH == 128 ? 1 : 2;             // item operand buffers
    static constexpr int BST = DH == 128 ? 2 : BWD_ST;       // streamed operand stages
    static constexpr int OFF_A = 0;                          // item operands [AB][2 tiles]
    static constexpr int OFF_B = OFF_A + 2 * AB * TILE;      // streamed operands [BST][2 tiles]
    static constexpr int OFF_VEC = OFF_B + 2 * BST * TILE;   // [BST][lse*log2e | D][128] (MODE_DKV)
    static constexpr int OFF_BAR = OFF_VEC + BST * 2 * 128 * 4;
    static constexpr int TOTAL = OFF_BAR + 256 + 1024;
};

template <int DH, int MODE>
__global__ void __launch_bounds__(BWD_NTHR, 1)
    k_attn_bwd2(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                AttnBwd2Args a) {
    static_assert(DH == 64 || DH == 128, "head dim");
    using L = Bwd2Smem<DH>;
    constexpr int AB = L::AB, BST = L::BST;
    // TMEM (512 columns): S | dP | acc1 | acc2 | P | dS at Dh = 64 (128|128|64|64|64|64).
    // Dh = 128, MODE_DKV: S | dP | dV | dK, with P written over S and dS over dP (each half
    // of the element-wise warps packs its 64 columns into the first 32 of its own half), so
    // the next tile's S / dP MMAs are issued behind this tile's gradient MMAs (in-order pipe).
    // Dh = 128, MODE_DQ: S | dP | dQ | dS.
    constexpr bool ALIAS = DH == 128 && MODE == MODE_DKV;
    constexpr int HSTR = ALIAS ? 64 : 32;  // TMEM column stride between the halves' packed P / dS
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
    uint64_t* a_full = bar + 0;    // [2]
    uint64_t* a_empty = bar + 2;   // [2]
    uint64_t* b_full = bar + 4;              // [BWD_ST]
    uint64_t* b_empty = b_full + BST;        // [BST]
    uint64_t* s_full = b_empty + BST;
    uint64_t* s_free = s_full + 1;
    uint64_t* p_full = s_full + 2;
    uint64_t* g_done = s_full + 3;
    uint64_t* acc_full = s_full + 4;
    uint64_t* dp_full = s_full + 5;  // dP of the current tile (S is committed first, on s_full)
    uint32_t* tbase_s = reinterpret_cast<uint32_t*>(s_full + 6);
    float* vec = reinterpret_cast<float*>(smem + L::OFF_VEC);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int H = a.H;
    const int k_begin = a.w_ptr[blockIdx.x], k_end = a.w_ptr[blockIdx.x + 1];
    // item operand columns in qkv/dout: MODE_DKV fixes K, V and streams Q, dO; MODE_DQ the reverse
    const int fix_col0 = MODE == MODE_DKV ? a.d : 0, fix_col1 = MODE == MODE_DKV ? 2 * a.d : 0;
    const int str_col0 = MODE == MODE_DKV ? 0 : a.d, str_col1 = MODE == MODE_DKV ? 0 : 2 * a.d;
    const CUtensorMap* fix_map1 = MODE == MODE_DKV ? &tm_qkv : &tm_do;  // V | dO
    const CUtensorMap* str_map1 = MODE == MODE_DKV ? &tm_do : &tm_qkv;  // dO | V

    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&a_full[s], 1);
            tc::mbar_init(&a_empty[s], 1);
        }
        for (int s = 0; s < BST; ++s) {
            tc::mbar_init(&b_full[s], 1 + 32);  // TMA bytes + one cp.async completion per lane of warp 8
            tc::mbar_init(&b_empty[s], 1);
        }
        tc::mbar_init(s_full, 1);
        tc::mbar_init(dp_full, 1);
        tc::mbar_init(s_free, 8);
        tc::mbar_init(p_full, 8);
        tc::mbar_init(g_done, 1);
        tc::mbar_init(acc_full, 1);
        tc::fence_barrier_init();
        tc::tma_prefetch(&tm_qkv);
        tc::tma_prefetch(&tm_do);
    }
    if (warp == 9) tc::tmem_alloc<512>(tbase_s);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tbase = *tbase_s;
    const uint32_t t_s = tbase, t_dp = tbase + 128, t_acc1 = tbase + 256, t_acc2 = tbase + 256 + DH;
    pdl_wait();
    pdl_trigger();
    if (MODE == MODE_DKV) ATTN_SPAN(0);
    const uint32_t t_p = ALIAS ? t_s : tbase + 384;
    const uint32_t t_ds = ALIAS ? t_dp : (DH == 128 ? tbase + 384 : tbase + 448);

    if (warp >= 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
        if (warp == 8) {  // ---------------- TMA (whole warp: lane 0 issues, all lanes write vectors)
            int g = 0, li = 0;
            for (int k = k_begin; k < k_end; ++k, ++li) {
                const int it = a.w_items[k], t = it / H, h = it % H, ab = li % AB;
                tc::mbar_wait(&a_empty[ab], ((li / AB) & 1) ^ 1);
                if (lane == 0) {
                    tc::mbar_expect_tx(&a_full[ab], 2 * L::TILE);
                    uint8_t* A0 = smem + L::OFF_A + (ab * 2) * L::TILE;
#pragma unroll
                    for (int r = 0; r < DH / 64; ++r) {
                        tc::tma_load_2d(A0 + r * 128 * 128, &tm_qkv, &a_full[ab], fix_col0 + h * DH + r * 64, t * 128);
                        tc::tma_load_2d(A0 + L::TILE + r * 128 * 128, fix_map1, &a_full[ab], fix_col1 + h * DH + r * 64,
                                        t * 128);
                    }
                }
                for (int e = a.lst_ptr[t]; e < a.lst_ptr[t + 1]; ++e, ++g) {
                    const int u = a.lst[e] & 0x3fffffff;
                    const int st = g % BST;
                    tc::mbar_wait(&b_empty[st], ((g / BST) & 1) ^ 1);
                    if (lane == 0) {
                        tc::mbar_expect_tx(&b_full[st], 2 * L::TILE);
                        uint8_t* B0 = smem + L::OFF_B + (st * 2) * L::TILE;
#pragma unroll
                        for (int r = 0; r < DH / 64; ++r) {
                            tc::tma_load_2d(B0 + r * 128 * 128, &tm_qkv, &b_full[st], str_col0 + h * DH + r * 64, u * 128);
                            tc::tma_load_2d(B0 + L::TILE + r * 128 * 128, str_map1, &b_full[st],
                                            str_col1 + h * DH + r * 64, u * 128);
                        }
                    }
                    if (MODE == MODE_DKV) {  // lse2 and D of the streamed query tile (zero-filled past T)
                        const uint32_t vl = tc::smem_u32(vec + st * 256);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int i = u * 128 + q * 32 + lane;
                            const uint32_t n = i < a.T ? 4u : 0u;
                            const long gi = (long)h * a.T + min(i, a.T - 1);
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(vl + (q * 32 + lane) * 4),
                                         "l"(a.lse2 + gi), "r"(n) : "memory");
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(vl + (128 + q * 32 + lane) * 4),
                                         "l"(a.dsum + gi), "r"(n) : "memory");
                        }
                    }
                    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&b_full[st]))
                                 : "memory");
                }
            }
        } else if (warp == 9) {  // ---------------- MMA (whole warp; one elected lane issues)
            constexpr uint32_t id_s = tc::idesc_bf16(128, 128, 0, 0);
            constexpr uint32_t id_g = tc::idesc_bf16(128, DH, 0, 1);
            int cS = 0, cP = 0;
            // S/dP look-ahead iterator over (item, streamed tile)
            int s_k = k_begin, s_li = 0, s_e = 0, s_end = 0, s_first = 0, gS = 0;
            auto s_load = [&]() {
                while (s_k < k_end) {
                    const int t = a.w_items[s_k] / H;
                    s_e = s_first = a.lst_ptr[t];
                    s_end = a.lst_ptr[t + 1];
                    if (s_e < s_end) return;
                    ++s_k;
                    ++s_li;
                }
            };
            s_load();
            auto issue_sd = [&]() {
                if (s_k >= k_end) return;
                const int st = gS % BST, ab = s_li % AB;
                if (MODE == MODE_DKV) ATTN_TRACE(3, cS, 0);
                if (s_e == s_first) tc::mbar_wait(&a_full[ab], (s_li / AB) & 1);
                if (MODE == MODE_DKV) ATTN_TRACE(3, cS, 1);
                tc::mbar_wait(&b_full[st], (gS / BST) & 1);
                if (MODE == MODE_DKV) ATTN_TRACE(3, cS, 2);
                if (cS > 0) tc::mbar_wait(s_free, (cS - 1) & 1);
                if (MODE == MODE_DKV) ATTN_TRACE(3, cS, 3);
                tc::tc_fence_after();
                const uint32_t f0 = tc::smem_u32(smem + L::OFF_A + (ab * 2) * L::TILE);
                const uint32_t s0 = tc::smem_u32(smem + L::OFF_B + (st * 2) * L::TILE);
                // Dh 128: S first, on its own barrier, so the element-wise warps start the exponentials
                // while dP is still in the tensor pipe
#pragma unroll
                for (int ks = 0; ks < DH / 16; ++ks) {
                    const uint32_t off = (ks >> 2) * (128 * 128) + (ks & 3) * 32;
                    tc::mma_bf16_e(t_s, tc::sdesc(f0 + off, 16, 1024), tc::sdesc(s0 + off, 16, 1024), id_s, ks > 0);
                }
                if (DH == 128) tc::mma_commit_e(s_full);
#pragma unroll
                for (int ks = 0; ks < DH / 16; ++ks) {
                    const uint32_t off = (ks >> 2) * (128 * 128) + (ks & 3) * 32;
                    tc::mma_bf16_e(t_dp, tc::sdesc(f0 + L::TILE + off, 16, 1024),
                                 tc::sdesc(s0 + L::TILE + off, 16, 1024), id_s, ks > 0);
                }
                tc::mma_commit_e(DH == 128 ? dp_full : s_full);  // Dh 64: S and dP on one barrier
                if (MODE == MODE_DKV) ATTN_TRACE(2, cS, 0);
                ++cS;
                ++gS;
                if (++s_e == s_end) {
                    ++s_k;
                    ++s_li;
                    s_load();
                }
            };
            // S / dP issue window: one tile ahead of the gradient MMAs (none when P / dS live
            // in S / dP's columns), and never into an item whose operand buffer this warp
            // has not released yet
            auto advance_sd = [&](int li_now) {
                while (s_k < k_end && cS < cP + (ALIAS ? 1 : 2) && s_li <= li_now + AB - 1) issue_sd();
            };
            int g = 0, li = 0;
            for (int k = k_begin; k < k_end; ++k, ++li) {
                const int t = a.w_items[k] / H, ab = li % AB;
                const int ea = a.lst_ptr[t], eb = a.lst_ptr[t + 1];
                if (ea == eb) {  // nothing streams into this item: release its operands
                    tc::mbar_wait(&a_full[ab], (li / AB) & 1);
                    if (lane == 0) tc::mbar_arrive(&a_empty[ab]);
                    continue;
                }
                for (int e = ea; e < eb; ++e, ++g) {
                    const int st = g % BST;
                    advance_sd(li);
                    if (MODE == MODE_DKV) ATTN_TRACE(2, cP, 1);
                    tc::mbar_wait(p_full, cP & 1);
                    tc::tc_fence_after();
                    if (MODE == MODE_DKV) ATTN_TRACE(2, cP, 2);
                    const uint32_t s0 = tc::smem_u32(smem + L::OFF_B + (st * 2) * L::TILE);
                    const uint32_t acc = (e > ea) ? 1u : 0u;
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks) {
                        const uint64_t b0 = tc::sdesc(s0 + ks * 2048, 128 * 128, 1024);
                        const uint64_t b1 = tc::sdesc(s0 + L::TILE + ks * 2048, 128 * 128, 1024);
                        const uint32_t pc = (ks >> 2) * HSTR + (ks & 3) * 8;  // packed P / dS columns of this K step
                        if (MODE == MODE_DKV) {
                            tc::mma_bf16_ts_e(t_acc1, t_p + pc, b1, id_g, (acc || ks > 0) ? 1u : 0u);   // dV += P^T dO
                            tc::mma_bf16_ts_e(t_acc2, t_ds + pc, b0, id_g, (acc || ks > 0) ? 1u : 0u);  // dK += dS^T Q
                        } else {
                            tc::mma_bf16_ts_e(t_acc1, t_ds + pc, b0, id_g, (acc || ks > 0) ? 1u : 0u);  // dQ += dS K
                        }
                    }
                    tc::mma_commit_e(g_done);
                    tc::mma_commit_e(&b_empty[st]);
                    ++cP;
                    if (e == eb - 1) {
                        // item done: release the accumulators to the epilogue and the item operands
                        // before looking ahead (the element-wise warps reach the next item's S only
                        // after their epilogue)
                        tc::mma_commit_e(acc_full);
                        tc::mma_commit_e(&a_empty[ab]);
                        advance_sd(li + 1);
                    } else {
                        advance_sd(li);
                    }
                }
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
        // ---------------- element-wise: row = TMEM lane, 64 of the 128 streamed columns
        const int q4 = warp & 3, half = warp >> 2;
        const int r = q4 * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
        const float c2 = a.scale_log2;
        int cS = 0, na = 0, g = 0;
        // per-row data of an item (prefetched one item ahead)
        int4 nmeta = make_int4(0, -1, 0, 0);
        float nlr = 0.f, ndr = 0.f;
        auto fetch = [&](int k) {
            if (k >= k_end) return;
            const int it = a.w_items[k], x = (it / H) * 128 + r, h = it % H;
            if (x < a.T) {
                nmeta = a.meta[x];
                if (MODE == MODE_DQ) {
                    nlr = a.lse2[(long)h * a.T + x];
                    ndr = a.dsum[(long)h * a.T + x];
                }
            }
        };
        fetch(k_begin);
        for (int k = k_begin; k < k_end; ++k) {
            const int it = a.w_items[k], t = it / H, h = it % H;
            const int x = t * 128 + r;  // this thread's row: key j (DKV) or query i (DQ)
            const bool row_ok = x < a.T;
            const int4 meta = nmeta;
            const float lr = nlr, dr = ndr;
            fetch(k + 1);
            // DKV: queries that see key j are [j, qhi); DQ: keys seen by query i are [l0, e0) u [b1, e1)
            const int qhi = row_ok ? meta.x : 0;
            const int l0 = meta.z;
            const int e0 = !row_ok ? 0 : (meta.y < 0 ? x + 1 : meta.w);
            const int b1 = meta.y < 0 ? 0 : meta.y, e1 = (row_ok && meta.y >= 0) ? x + 1 : 0;
            const int ea = a.lst_ptr[t], eb = a.lst_ptr[t + 1];
            for (int e = ea; e < eb; ++e, ++g) {
                const uint32_t fl = (uint32_t)a.lst[e];
                const int u0 = (int)(fl & 0x3fffffff) * 128;  // first row of the streamed tile
                const bool full = (fl >> 30) & 1;
                const uint32_t vl = tc::smem_u32(vec + (g % BST) * 256);
                if (MODE == MODE_DKV) ATTN_TRACE(4 + warp, cS, 0);
                tc::mbar_wait(s_full, cS & 1);
                tc::tc_fence_after();
                if (MODE == MODE_DKV) ATTN_TRACE(4 + warp, cS, 1);
                uint32_t pp[32], pd[32];  // packed bf16 P / dS of this thread's 64 columns
                if constexpr (DH == 128) {  // measured: +4% at Dh 128, -7% at Dh 64 (profiles/r02_ab_attn_bwd_split.txt)
                // S (both 32-column chunks) first; P = exp2(S c - lse) runs while dP is still being
                // computed; then dP, after which S / dP are released so the next tile's MMAs overlap
                float pv[64], dall[64];
                tc::tmem_ld32_nowait(t_s + half * 64 + lane_off, reinterpret_cast<uint32_t*>(pv));
                tc::tmem_ld32_nowait(t_s + half * 64 + 32 + lane_off, reinterpret_cast<uint32_t*>(pv) + 32);
                tc::tmem_ld_wait();
                if (MODE == MODE_DKV) ATTN_TRACE(4 + warp, cS, 2);
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int cb = half * 64 + c * 32;  // first tile column of the chunk
                    float* sv = pv + 32 * c;
                    // exponent argument (log2 units); -inf where the pair is masked
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        float l4[4];
                        if (MODE == MODE_DKV) {
                            uint32_t w0, w1, w2, w3;
                            tc::lds128(vl + (cb + j) * 4, w0, w1, w2, w3);
                            l4[0] = __uint_as_float(w0); l4[1] = __uint_as_float(w1);
                            l4[2] = __uint_as_float(w2); l4[3] = __uint_as_float(w3);
                        } else {
                            l4[0] = l4[1] = l4[2] = l4[3] = lr;
                        }
                        const float2 c22 = make_float2(c2, c2);
                        const float2 a01 = tc::ffma2(make_float2(sv[j], sv[j + 1]), c22, make_float2(-l4[0], -l4[1]));
                        const float2 a23 = tc::ffma2(make_float2(sv[j + 2], sv[j + 3]), c22, make_float2(-l4[2], -l4[3]));
                        sv[j] = a01.x; sv[j + 1] = a01.y; sv[j + 2] = a23.x; sv[j + 3] = a23.y;
                    }
                    if (!full) {
                        const int cu = u0 + cb;
                        int lo, hi, l2, h2;
                        if (MODE == MODE_DKV) {
                            lo = min(max(x - cu, 0), 32);
                            hi = min(max(qhi - cu, 0), 32);
                            l2 = h2 = 32;
                        } else {
                            lo = min(max(l0 - cu, 0), 32);
                            hi = min(max(e0 - cu, 0), 32);
                            l2 = min(max(b1 - cu, 0), 32);
                            h2 = min(max(e1 - cu, 0), 32);
                        }
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const bool ok = ((j >= lo) & (j < hi)) | ((j >= l2) & (j < h2));
                            sv[j] = ok ? sv[j] : -INFINITY;
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 32; j += 2) {
                        sv[j] = tc::ex2_approx(sv[j]);
                        sv[j + 1] = tc::ex2_approx(sv[j + 1]);
                        pp[c * 16 + j / 2] = pack2(sv[j], sv[j + 1]);
                    }
                }
                tc::mbar_wait(dp_full, cS & 1);
                tc::tc_fence_after();
                tc::tmem_ld32_nowait(t_dp + half * 64 + lane_off, reinterpret_cast<uint32_t*>(dall));
                tc::tmem_ld32_nowait(t_dp + half * 64 + 32 + lane_off, reinterpret_cast<uint32_t*>(dall) + 32);
                tc::tmem_ld_wait();
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(s_free);
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int cb = half * 64 + c * 32;
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        float d4[4];
                        if (MODE == MODE_DKV) {
                            uint32_t w0, w1, w2, w3;
                            tc::lds128(vl + (128 + cb + j) * 4, w0, w1, w2, w3);
                            d4[0] = __uint_as_float(w0); d4[1] = __uint_as_float(w1);
                            d4[2] = __uint_as_float(w2); d4[3] = __uint_as_float(w3);
                        } else {
                            d4[0] = d4[1] = d4[2] = d4[3] = dr;
                        }
#pragma unroll
                        for (int q = 0; q < 4; q += 2) {
                            const int jj = 32 * c + j + q;
                            const float2 dd = tc::fadd2(make_float2(dall[jj], dall[jj + 1]), make_float2(-d4[q], -d4[q + 1]));
                            const float2 ds = tc::fmul2(make_float2(pv[jj], pv[jj + 1]), dd);
                            pd[jj / 2] = pack2(ds.x, ds.y);
                        }
                    }
                }
                } else {
                // all four TMEM loads (S and dP, both 32-column chunks) in flight at once, then
                // S/dP are released so the next tile's S/dP MMAs overlap this tile's math
                float sall[64], dall[64];
                tc::tmem_ld32_nowait(t_s + half * 64 + lane_off, reinterpret_cast<uint32_t*>(sall));
                tc::tmem_ld32_nowait(t_dp + half * 64 + lane_off, reinterpret_cast<uint32_t*>(dall));
                tc::tmem_ld32_nowait(t_s + half * 64 + 32 + lane_off, reinterpret_cast<uint32_t*>(sall) + 32);
                tc::tmem_ld32_nowait(t_dp + half * 64 + 32 + lane_off, reinterpret_cast<uint32_t*>(dall) + 32);
                tc::tmem_ld_wait();
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(s_free);
                if (MODE == MODE_DKV) ATTN_TRACE(4 + warp, cS, 2);
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int cb = half * 64 + c * 32;  // first tile column of the chunk
                    const float* sv = sall + 32 * c;
                    const float* dp = dall + 32 * c;
                    // exponent argument (log2 units); -inf where the pair is masked
                    float arg[32], dd[32];
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        float l4[4], d4[4];
                        if (MODE == MODE_DKV) {
                            uint32_t w0, w1, w2, w3;
                            tc::lds128(vl + (cb + j) * 4, w0, w1, w2, w3);
                            l4[0] = __uint_as_float(w0); l4[1] = __uint_as_float(w1);
                            l4[2] = __uint_as_float(w2); l4[3] = __uint_as_float(w3);
                            tc::lds128(vl + (128 + cb + j) * 4, w0, w1, w2, w3);
                            d4[0] = __uint_as_float(w0); d4[1] = __uint_as_float(w1);
                            d4[2] = __uint_as_float(w2); d4[3] = __uint_as_float(w3);
                        } else {
                            l4[0] = l4[1] = l4[2] = l4[3] = lr;
                            d4[0] = d4[1] = d4[2] = d4[3] = dr;
                        }
                        const float2 c22 = make_float2(c2, c2);
                        const float2 a01 = tc::ffma2(make_float2(sv[j], sv[j + 1]), c22, make_float2(-l4[0], -l4[1]));
                        const float2 a23 = tc::ffma2(make_float2(sv[j + 2], sv[j + 3]), c22, make_float2(-l4[2], -l4[3]));
                        const float2 d01 = tc::fadd2(make_float2(dp[j], dp[j + 1]), make_float2(-d4[0], -d4[1]));
                        const float2 d23 = tc::fadd2(make_float2(dp[j + 2], dp[j + 3]), make_float2(-d4[2], -d4[3]));
                        arg[j] = a01.x; arg[j + 1] = a01.y; arg[j + 2] = a23.x; arg[j + 3] = a23.y;
                        dd[j] = d01.x; dd[j + 1] = d01.y; dd[j + 2] = d23.x; dd[j + 3] = d23.y;
                    }
                    if (!full) {
                        const int cu = u0 + cb;
                        int lo, hi, l2, h2;
                        if (MODE == MODE_DKV) {
                            lo = min(max(x - cu, 0), 32);
                            hi = min(max(qhi - cu, 0), 32);
                            l2 = h2 = 32;
                        } else {
                            lo = min(max(l0 - cu, 0), 32);
                            hi = min(max(e0 - cu, 0), 32);
                            l2 = min(max(b1 - cu, 0), 32);
                            h2 = min(max(e1 - cu, 0), 32);
                        }
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const bool ok = ((j >= lo) & (j < hi)) | ((j >= l2) & (j < h2));
                            arg[j] = ok ? arg[j] : -INFINITY;
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 32; j += 2) {
                        const float2 p = make_float2(tc::ex2_approx(arg[j]), tc::ex2_approx(arg[j + 1]));
                        const float2 ds = tc::fmul2(p, make_float2(dd[j], dd[j + 1]));
                        pp[c * 16 + j / 2] = pack2(p.x, p.y);
                        pd[c * 16 + j / 2] = pack2(ds.x, ds.y);
                    }
                }
                }
                if (MODE == MODE_DKV) ATTN_TRACE(4 + warp, cS, 3);
                // the previous tile's gradient MMAs have read P / dS
                if (cS > 0) {
                    tc::mbar_wait(g_done, (cS - 1) & 1);
                    tc::tc_fence_after();
                }
                if (MODE == MODE_DKV) ATTN_TRACE(4 + warp, cS, 4);
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    if (MODE == MODE_DKV) tc::tmem_st16(t_p + half * HSTR + c * 16 + lane_off, pp + 16 * c);
                    tc::tmem_st16(t_ds + half * HSTR + c * 16 + lane_off, pd + 16 * c);
                }
                tc::tmem_st_wait();
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(p_full);
                if (MODE == MODE_DKV) ATTN_TRACE(4 + warp, cS, 5);
                ++cS;
            }
            // item epilogue: accumulators -> bf16 rows of dqkv (MODE_DKV: half 0 dV -> 2d + h DH,
            // half 1 dK * scale -> d + h DH; MODE_DQ: dQ * scale, half h -> columns [32 h, 32 h + 32))
            constexpr int NC = MODE == MODE_DKV ? DH : DH / 2;
            constexpr int CH = NC < 64 ? NC : 64;  // columns per TMEM load batch
            bf16* dst = a.dqkv + (long)x * 3 * a.d + h * DH +
                        (MODE == MODE_DKV ? (half ? a.d : 2 * a.d) : half * (DH / 2));
            if (eb > ea) {
                tc::mbar_wait(acc_full, na & 1);
                tc::tc_fence_after();
                ++na;
                const uint32_t src = MODE == MODE_DKV ? (half ? t_acc2 : t_acc1) : t_acc1 + half * (DH / 2);
                const float mul = (MODE == MODE_DQ || half) ? a.scale : 1.f;
#pragma unroll
                for (int cb = 0; cb < NC; cb += CH) {
                    float o[CH];
#pragma unroll
                    for (int c = 0; c < CH / 32; ++c)
                        tc::tmem_ld32_nowait(src + cb + c * 32 + lane_off, reinterpret_cast<uint32_t*>(o) + 32 * c);
                    tc::tmem_ld_wait();
                    if (row_ok) {
#pragma unroll
                        for (int q = 0; q < CH; q += 8) {
                            uint4 v4;
                            v4.x = pack2(o[q] * mul, o[q + 1] * mul);
                            v4.y = pack2(o[q + 2] * mul, o[q + 3] * mul);
                            v4.z = pack2(o[q + 4] * mul, o[q + 5] * mul);
                            v4.w = pack2(o[q + 6] * mul, o[q + 7] * mul);
                            *reinterpret_cast<uint4*>(dst + cb + q) = v4;
                        }
                    }
                }
            } else if (row_ok) {
#pragma unroll
                for (int q = 0; q < NC; q += 8) *reinterpret_cast<uint4*>(dst + q) = make_uint4(0, 0, 0, 0);
            }
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (MODE == MODE_DKV) ATTN_SPAN(1);
    if (warp == 9) {
        tc::tc_fence_after();
        tc::tmem_dealloc<512>(tbase);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}


int device_sms_attn() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <int DH>
void launch_fwd_pair(const AttnPairMaps& maps, const AttnPairArgs& a, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_attn_fwd_pair<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, PairSmem<DH>::TOTAL);
        attr = true;
    }
    launch_pdl(k_attn_fwd_pair<DH>, dim3(a.grid), dim3(PAIR_NTHR), PairSmem<DH>::TOTAL, st, maps, a);
    PARL_LAUNCHED();
}

bool make_qkv_map(CUtensorMap* m, const bf16* base, long cols, long rows) {
    auto fn = encode();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<bf16*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}


}  // namespace

template <int DH, int MODE>
void launch_bwd2(const CUtensorMap& mq, const CUtensorMap& md, const AttnBwd2Args& a, int grid, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_attn_bwd2<DH, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, Bwd2Smem<DH>::TOTAL);
        attr = true;
    }
    launch_pdl(k_attn_bwd2<DH, MODE>, dim3(grid), dim3(BWD_NTHR), Bwd2Smem<DH>::TOTAL, st, mq, md, a);
    PARL_LAUNCHED();
}

// dqkv <- attention backward given dO = dout [T x d], the forward's lse and
// D = rowsum(dO * O) (dsum).  false if unsupported.
bool attn_bwd_tc(const AttnArgs& aa, const bf16* qkv, const bf16* out, const bf16* dout, const float* lse,
                 float* dsum, bf16* dqkv, cudaStream_t st) {
    if (!(aa.Dh == 64 || aa.Dh == 128)) return false;
    if (((long)aa.d * 2) % 16 || (reinterpret_cast<uintptr_t>(qkv) & 15) || (reinterpret_cast<uintptr_t>(dout) & 15) ||
        (reinterpret_cast<uintptr_t>(dqkv) & 15))
        return false;
    CUtensorMap mq, md;
    if (!make_qkv_map(&mq, qkv, 3L * aa.d, aa.T) || !make_qkv_map(&md, dout, aa.d, aa.T)) return false;
    if (!aa.sched.q_ptr || !aa.sched.k_ptr || !aa.sched.bk_ptr || !aa.sched.bq_ptr || !out) return false;
    {
        const size_t ht = (size_t)aa.H * aa.T;
        float* lse2 = static_cast<float*>(g_bwd_ws.get(ht * 4 + (size_t)aa.T * 16 + 16));
        if (!lse2) return false;
        int4* meta = reinterpret_cast<int4*>(lse2 + ((ht + 3) & ~size_t(3)));
        const long warps = (long)aa.T * aa.H, ldo = aa.ldo ? aa.ldo : aa.d;
        const bool v8 = (aa.Dh == 64 || aa.Dh == 128) && aa.d % 8 == 0 && ldo % 8 == 0 &&
                        (reinterpret_cast<uintptr_t>(out) & 15) == 0 && (reinterpret_cast<uintptr_t>(dout) & 15) == 0;
        const long thr = (long)aa.T * (aa.d / 8);
        if (v8 && aa.Dh == 64)
            launch_pdl(k_attn_prep_v8<8>, dim3((int)((thr + 255) / 256)), dim3(256), 0, st, aa.T, aa.H, aa.d, ldo,
                       aa.seg, aa.seg_info, out, dout, lse, dsum, lse2, meta);
        else if (v8)
            launch_pdl(k_attn_prep_v8<16>, dim3((int)((thr + 255) / 256)), dim3(256), 0, st, aa.T, aa.H, aa.d, ldo,
                       aa.seg, aa.seg_info, out, dout, lse, dsum, lse2, meta);
        else
            launch_pdl(k_attn_prep, dim3((int)((warps * 32 + 255) / 256)), dim3(256), 0, st, aa.T, aa.H, aa.d, aa.Dh,
                       ldo, aa.seg, aa.seg_info, out, dout, lse, dsum, lse2, meta);
        PARL_LAUNCHED();
        AttnBwd2Args b;
        b.T = aa.T; b.H = aa.H; b.d = aa.d;
        b.scale = aa.scale; b.scale_log2 = aa.scale * LOG2E;
        b.lse2 = lse2; b.dsum = dsum; b.meta = meta; b.dqkv = dqkv;
        b.lst_ptr = aa.sched.k_ptr; b.lst = aa.sched.k_list;
        b.w_ptr = aa.sched.bk_ptr; b.w_items = aa.sched.bk_items;
        if (aa.Dh == 64) launch_bwd2<64, MODE_DKV>(mq, md, b, aa.sched.bk_grid, st);
        else launch_bwd2<128, MODE_DKV>(mq, md, b, aa.sched.bk_grid, st);
        b.lst_ptr = aa.sched.q_ptr; b.lst = aa.sched.q_list;
        b.w_ptr = aa.sched.bq_ptr; b.w_items = aa.sched.bq_items;
        if (aa.Dh == 64) launch_bwd2<64, MODE_DQ>(mq, md, b, aa.sched.bq_grid, st);
        else launch_bwd2<128, MODE_DQ>(mq, md, b, aa.sched.bq_grid, st);
    }
    return true;
}

// qkv: [T x 3d] bf16 per model; the nm models (same packed group, e.g. the tri-model forward)
// run as one launch when the dynamic queue is on.  false when the head dim / alignment is
// unsupported.
bool attn_fwd_tc_multi(const AttnArgs& aa, const bf16* const* qkv, bf16* const* out, float* const* lse, int nm,
                       cudaStream_t st) {
    if (!(aa.Dh == 64 || aa.Dh == 128) || nm < 1 || nm > 3) return false;
    const long ldo = aa.ldo ? aa.ldo : aa.d;
    if (((3L * aa.d * 2) % 16) || ((ldo * 2) % 16)) return false;
    for (int k = 0; k < nm; ++k)
        if ((reinterpret_cast<uintptr_t>(qkv[k]) & 15) || (reinterpret_cast<uintptr_t>(out[k]) & 15)) return false;
    auto fn = encode();
    if (!fn) return false;
    cuuint32_t es[2] = {1, 1};
    auto qkv_map = [&](CUtensorMap* m, const bf16* p) {
        cuuint64_t dims[2] = {(cuuint64_t)(3 * aa.d), (cuuint64_t)aa.T};
        cuuint64_t strides[1] = {(cuuint64_t)(3 * aa.d) * 2};
        cuuint32_t box[2] = {64, 128};
        return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<bf16*>(p), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    // output tensor map: [T x d] bf16 with row stride ldo, 32 x 64 boxes, 128B swizzle
    auto out_map = [&](CUtensorMap* m, bf16* p) {
        cuuint64_t odims[2] = {(cuuint64_t)aa.d, (cuuint64_t)aa.T};
        cuuint64_t ostr[1] = {(cuuint64_t)ldo * 2};
        cuuint32_t obox[2] = {64, 32};
        return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, odims, ostr, obox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
               CUDA_SUCCESS;
    };
    if (!aa.sched.q_ptr) return false;
    if (!aa.sched.p_ptr || !aa.sched.w_ptr) return false;
    {
        // dynamic work queue (PARL_ATTN_DYN=0: the static per-CTA lists, one launch per model)
        static const bool dyn_ok = [] {
            const char* e = getenv("PARL_ATTN_DYN");
            return !(e && e[0] == '0');
        }();
        const bool dyn = dyn_ok && aa.item_ctr && aa.item_base && aa.sched.w_order;
        const int per_launch = dyn ? nm : 1;
        for (int k0 = 0; k0 < nm; k0 += per_launch) {
            AttnPairArgs pa;
            AttnPairMaps maps;
            pa.T = aa.T; pa.H = aa.H; pa.d = aa.d;
            pa.seg = aa.seg; pa.seg_info = aa.seg_info;
            pa.p_ptr = aa.sched.p_ptr; pa.p_list = aa.sched.p_list;
            pa.w_ptr = aa.sched.w_ptr; pa.w_items = aa.sched.w_items;
            pa.scale_log2 = aa.scale * LOG2E;
            pa.ldo = ldo;
            pa.nm = per_launch;
            pa.n_base = aa.sched.w_n > 0 ? aa.sched.w_n : (1 << 30);
            for (int k = 0; k < per_launch; ++k) {
                if (!qkv_map(&maps.qkv[k], qkv[k0 + k]) || !out_map(&maps.out[k], out[k0 + k])) return false;
                pa.lse[k] = lse[k0 + k];
            }
            pa.dyn = dyn;
            pa.n_items = per_launch * aa.sched.w_n;
            pa.order = aa.sched.w_order;
            pa.ctr = aa.item_ctr;
            // the static lists' grid, or (queue) enough CTAs for all models' items
            pa.grid = dyn ? std::min(pa.n_items, std::max(aa.sched.w_grid, device_sms_attn())) : aa.sched.w_grid;
            pa.base = dyn ? *aa.item_base : 0u;
            if (dyn) *aa.item_base += (unsigned)(pa.n_items + pa.grid);  // every CTA's last fetch finds the end
            if (aa.Dh == 64) launch_fwd_pair<64>(maps, pa, st);
            else launch_fwd_pair<128>(maps, pa, st);
        }
        return true;
    }
    return true;
}

bool attn_fwd_tc(const AttnArgs& aa, const bf16* qkv, bf16* out, float* lse, cudaStream_t st) {
    return attn_fwd_tc_multi(aa, &qkv, &out, &lse, 1, st);
}

#ifdef PARL_ATTN_TRACE
bool attn_trace_read(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, g_attn_trace, sizeof(g_attn_trace)) == cudaSuccess;
}
#else
bool attn_trace_read(unsigned long long*) { return false; }
#endif

}  // namespace parl_gpu
