// C-ABI implementation: context, device-resident models, packed groups,
// activation handles, gradient accumulators, and the orchestration of the
// hot path (forward_logprobs / trimodel_forward / GRPO loss / backward /
// accumulate) over the kernels in k_*.cu.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <memory>
#include <mutex>
#include <queue>
#include <random>
#include <type_traits>
#include <vector>

#include "internal.cuh"
#include "kernels.cuh"

namespace parl_gpu {
uint64_t g_launches = 0;
bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("PARL_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}
}

using namespace parl_gpu;

// ---------------------------------------------------------------------------
// device memory: grow-only named buffers
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void* get(size_t need) {
        if (need > bytes) {
            if (p) cudaFree(p);
            p = nullptr;
            PARL_CUDA(cudaMalloc(&p, need));
            bytes = need;
        }
        return p;
    }
    template <class T>
    T* as(size_t n) { return static_cast<T*>(get(std::max<size_t>(n, 1) * sizeof(T))); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    ~DevBuf() { release(); }
};

// pinned host staging for small async uploads: the buffer is reused only once the
// previous copy out of it has completed (event), so no stream synchronisation
struct HostStage {
    void* p = nullptr;
    size_t bytes = 0;
    cudaEvent_t ev = nullptr;
    bool pending = false;
    void upload(void* dst, const void* src, size_t n, cudaStream_t st) {
        if (pending) PARL_CUDA(cudaEventSynchronize(ev));
        if (n > bytes) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            PARL_CUDA(cudaMallocHost(&p, n));
            bytes = n;
        }
        if (!ev) PARL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        std::memcpy(p, src, n);
        PARL_CUDA(cudaMemcpyAsync(dst, p, n, cudaMemcpyHostToDevice, st));
        PARL_CUDA(cudaEventRecord(ev, st));
        pending = true;
    }
    // two host ranges into one pinned buffer, two copies, one completion event
    void upload2(void* dst1, const void* src1, size_t n1, void* dst2, const void* src2, size_t n2, cudaStream_t st) {
        if (pending) PARL_CUDA(cudaEventSynchronize(ev));
        const size_t n1a = (n1 + 15) & ~size_t(15), n = n1a + n2;
        if (n > bytes) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            PARL_CUDA(cudaMallocHost(&p, n));
            bytes = n;
        }
        if (!ev) PARL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        std::memcpy(p, src1, n1);
        std::memcpy(static_cast<char*>(p) + n1a, src2, n2);
        if (n1) PARL_CUDA(cudaMemcpyAsync(dst1, p, n1, cudaMemcpyHostToDevice, st));
        if (n2) PARL_CUDA(cudaMemcpyAsync(dst2, static_cast<char*>(p) + n1a, n2, cudaMemcpyHostToDevice, st));
        PARL_CUDA(cudaEventRecord(ev, st));
        pending = true;
    }
    ~HostStage() {
        if (pending) cudaEventSynchronize(ev);
        if (ev) cudaEventDestroy(ev);
        if (p) cudaFreeHost(p);
    }
};

struct SchedHost {
    std::vector<int32_t> q_ptr, k_ptr, p_ptr;
    std::vector<int32_t> p_cost;  // forward pair items: 2 per key tile both query tiles see, 1 per one-sided
};

struct NcclApi {
    void* h = nullptr;
    int (*getUniqueId)(void*) = nullptr;
    int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*commDestroy)(void*) = nullptr;
    const char* (*getErrorString)(int) = nullptr;
};

struct parl_ctx_s {
    int device = 0;
    parl_precision prec = PARL_PREC_FP32;
    cudaStream_t st = nullptr;
    std::string err;
    // forward workspaces of cache-less forwards, one set per role slot (models of a
    // layer-interleaved tri-model forward are live at the same time)
    struct FwdScratch {
        DevBuf x, xmid, a, qkv, ctxo, bn, actv, stats, lse_attn, hf, lnf_mean, lnf_rstd, lse_head, logits;
    } scr[3];
    DevBuf part, target;
    // dynamic attention work queue: monotonic device counter, host copy of its next base
    DevBuf item_ctr;
    unsigned item_base = 0;
    // backward workspaces
    DevBuf dx, dx2, dx_act, dpre, dbn, dmid, dmid_act, dctx, dqkv, da, dsum, dhf, dxg, dz;
    DevBuf stats, per_sample, staging, flags, grpo_slots, g_seq;
    // KV-cached decoder (parl_sample_group): prompt / per-sequence caches and one step's rows
    DevBuf kv_prompt, kv_own, dec_x, dec_x2, dec_xm, dec_a, dec_qkv, dec_ctx, dec_act, dec_st, dec_logits, dec_tok;
    // one caller at a time per context (the reference allows distinct ModelParams on distinct
    // threads; they share this context's stream and workspaces)
    std::recursive_mutex mu;
    // kernel-class profiler (parl_ctx_profile)
    struct ProfRec {
        int cls;
        cudaEvent_t a, b;
        double work;
    };
    bool prof_on = false;
    std::vector<ProfRec> prof_pending;
    std::vector<cudaEvent_t> ev_pool;
    double prof_ms[PARL_KC_COUNT] = {}, prof_work[PARL_KC_COUNT] = {};
    long prof_n[PARL_KC_COUNT] = {};
    cudaEvent_t ev() {
        if (ev_pool.empty()) {
            cudaEvent_t e;
            PARL_CUDA(cudaEventCreate(&e));
            return e;
        }
        cudaEvent_t e = ev_pool.back();
        ev_pool.pop_back();
        return e;
    }
    void prof_collect() {
        if (prof_pending.empty()) return;
        PARL_CUDA(cudaStreamSynchronize(st));
        for (auto& r : prof_pending) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, r.a, r.b);
            prof_ms[r.cls] += ms;
            prof_work[r.cls] += r.work;
            prof_n[r.cls] += 1;
            ev_pool.push_back(r.a);
            ev_pool.push_back(r.b);
        }
        prof_pending.clear();
    }
    // activation recomputation: 0 auto (when the stacks do not fit), 1 always, 2 never
    int recompute = 0;
    // the policy's bf16 logits: 0 keep them for the backward's softmax seed (S x V x 2 B of HBM,
    // written once, read once), 1 never write them and rebuild them in the backward with the same
    // head GEMM into dZ (one more 2 S V d contraction); activation recomputation implies 1.
    // $PARL_HEAD_RECOMPUTE (the A/B of DESIGN.md §4, K8)
    int head_recompute = 0;
    // activation handle reused by parl_train_microbatch (no per-call allocation)
    parl_act_s* act_cache = nullptr;
    // lifetime: objects created on this context keep it alive
    int refs = 0;
    bool closing = false;
    // NCCL (data-parallel over prompt groups); every collective of the communicator runs on
    // comm_st, ordered against the compute stream by events
    void* comm = nullptr;
    int rank = 0, nranks = 1;
    cudaStream_t comm_st = nullptr;
    cudaEvent_t ev_comm = nullptr, ev_comm_done = nullptr;
};

struct parl_model_s {
    parl_ctx_s* ctx = nullptr;
    parl_config cfg{};
    FlatLayout L{};
    ModelW W{};
    std::vector<LayerW> layers;
    DevBuf f32, act, master;
    bool has_master = false;
    uint64_t version = 0, forward_gen = 0;
    uint64_t init_seed = 0;  // ModelParams::init_seed (checkpoint header)
    uint64_t epoch = 0;  // bumped by every write of the weights (host mirrors of the drop-in key on it)
};

// Segment layout of one packed sequence (host): contiguous token ranges, each a prompt or a
// response of some prompt group, with the shared-prompt visibility rule (model.cpp:242-245)
// generalised to several groups per sequence: rows of a prompt segment see [A, i], rows of a
// response see their group's prompt [A, B) and their own prefix [C, i]; keys of a segment are
// seen by queries up to Q (the group's end for a prompt, the response's end for a response).
// One group: segment 0 = prompt [0, P), segments 1..G = responses; causal: one prompt [0, T).
struct SegLayout {
    std::vector<int> start, end;
    std::vector<int4> info;  // {A, B (-1: prompt segment), C, Q} == AttnArgs::seg_info
    int n_groups = 0;
    void clear() {
        start.clear();
        end.clear();
        info.clear();
        n_groups = 0;
    }
    // appends one group: prompt [p0, p0 + P), then the responses back to back
    void add_group(int p0, int P, const int* lens, int G) {
        int t = p0 + P;
        for (int k = 0; k < G; ++k) t += lens[k];
        const int gend = t;
        start.push_back(p0);
        end.push_back(p0 + P);
        info.push_back(make_int4(p0, -1, p0, gend));
        t = p0 + P;
        for (int k = 0; k < G; ++k) {
            start.push_back(t);
            end.push_back(t + lens[k]);
            info.push_back(make_int4(p0, p0 + P, t, t + lens[k]));
            t += lens[k];
        }
        ++n_groups;
    }
    int T() const { return end.empty() ? 0 : end.back(); }
    int max_group_len() const {  // the longest prompt group (info.w of a prompt segment = group end)
        int m = 0;
        for (size_t k = 0; k < info.size(); ++k)
            if (info[k].y < 0) m = std::max(m, info[k].w - info[k].x);
        return m;
    }
    // allowed (query, key) pairs: the algorithmic attention work
    double pairs() const {
        double s = 0;
        for (size_t k = 0; k < start.size(); ++k) {
            const double n = end[k] - start[k];
            s += n * (n + 1) / 2;
            if (info[k].y >= 0) s += n * (info[k].y - info[k].x);
        }
        return s;
    }
};

struct parl_group_s {
    parl_ctx_s* ctx = nullptr;
    int max_T = 0, max_G = 0;
    int T = 0, P = 0, G = 0, S = 0, n_samples = 0;
    int Peff = 0;  // end of segment 0 (prompt, or the whole causal sequence)
    double pairs = 0;  // allowed attention pairs (algorithmic attention work)
    uint64_t epoch = 0;
    PackedDev pk{};
    DevBuf ints, seg_info, cu_d, in_prompt, in_resp, lp, upstream, rewards, adv;
    SegLayout segs;
    DevBuf tok_keys, tok_idx, pos_keys, pos_idx, iota, sort_tmp, sched_buf, work_buf;
    HostStage sched_stage, work_stage, adv_stage, multi_stage;  // pinned staging: async uploads, no host block
    // host token inputs (parl_pack / parl_pack_multi): a pageable copy above 64 KB would block the
    // host until the stream drains; two pinned stages let the host run a micro-batch ahead
    HostStage in_stage[2];
    int in_flip = 0;
    int n_groups = 1, group_G = 0;  // prompt groups in the sequence; responses per group (0: not uniform)
    DevBuf multi_tab, multi_prompts, multi_resp;
    AttnSched sched;
    SchedHost sched_h;  // host copies of the schedule's tile pointers (work lists)
    int work_H = -1, work_d = -1;
    uint64_t work_epoch = ~0ull;
    uint64_t sorted_epoch = ~0ull;
    std::vector<int> lens, span_start, cu;
    std::vector<int> sched_key;  // segment structure (starts) the schedule was built for
    int max_seq = 0, vocab = 0;
    // token-id range of the packed tokens (validate_forward_inputs, model.cpp:413-417): known on
    // the host for host-packed groups, read once from K1's device reduction for device-packed ones
    int tok_min = 0, tok_max = 0;
    bool tok_range_dev = false;  // pending on the device (parl_pack_device)
    DevBuf tok_range;
};

struct parl_act_s {
    parl_model_s* owner = nullptr;
    parl_group_s* group = nullptr;
    uint64_t version = 0, gen = 0, epoch = 0;
    int T = 0, S = 0;
    DevBuf xs, xmid, a, qkv, ctxo, bn, pre, actv, stats, lse_attn;  // per-layer stacks
    DevBuf hf, lnf_mean, lnf_rstd, logits, lse_head;
    bool logits_bf16 = false;  // logits stored bf16 by the fused tcgen05 head
    bool logits_rc = false;    // logits not kept: the backward rebuilds them into dZ (head recompute)
    bool recompute = false;    // only x_0..x_L kept; layers (and bf16 logits) rebuilt in the backward
    int rc_key[3] = {-1, -1, -1};  // shape the automatic recompute decision was made for
    uintptr_t pad_sig[8] = {};  // buffers / sizes the bias columns were filled for
};

struct parl_grad_s {
    parl_ctx_s* ctx = nullptr;
    parl_config cfg{};
    FlatLayout L{};
    DevBuf g;
    int micro_steps = 0;
    // after a data-parallel allreduce the count is the sum over ranks, held on the device until
    // apply_update (which synchronises anyway) reads it
    DevBuf count_dev;
    bool count_on_device = false;
    // tok_emb rows touched by this buffer's backward passes (the other rows are exactly 0), so
    // the data-parallel exchange of the V x d token-embedding gradient sends only those rows
    DevBuf touched, sel_idx, sel_rows, sel_count;
    bool overlap = false;  // armed: the next backward allreduces each layer as soon as it is final
    bool streamed = false; // that backward has run: layers and head are in flight on comm_st
};

static void ctx_release(parl_ctx_s* ctx) {
    if (--ctx->refs > 0 || !ctx->closing) return;
    cudaStreamSynchronize(ctx->st);
    if (ctx->comm_st) {
        cudaStreamSynchronize(ctx->comm_st);
        cudaStreamDestroy(ctx->comm_st);
        cudaEventDestroy(ctx->ev_comm);
        cudaEventDestroy(ctx->ev_comm_done);
    }
    delete ctx->act_cache;
    cudaStreamDestroy(ctx->st);
    delete ctx;
}

// RAII: bracket the launches of one kernel class with events when profiling.
struct ProfScope {
    parl_ctx_s* c;
    int cls;
    double work;
    cudaEvent_t a = nullptr;
    ProfScope(parl_ctx_s* c_, int cls_, double work_) : c(c_), cls(cls_), work(work_) {
        if (c->prof_on) {
            a = c->ev();
            cudaEventRecord(a, c->st);
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEvent_t b = c->ev();
            cudaEventRecord(b, c->st);
            c->prof_pending.push_back({cls, a, b, work});
            if (c->prof_pending.size() > 4096) c->prof_collect();
        }
    }
};

namespace {

thread_local std::string tl_err;

// Every entry point runs under its context's lock and the process lock: the reference lets
// distinct ModelParams instances run on distinct threads (rollout.cpp:178), and
// contexts share a few process-wide workspaces (the split-K and attention-backward scratch).
std::recursive_mutex& process_mutex() {
    static std::recursive_mutex m;
    return m;
}

template <class F>
parl_status guarded(parl_ctx_s* c, F&& f) {
    std::lock_guard<std::recursive_mutex> glk(process_mutex());
    std::unique_lock<std::recursive_mutex> lk;
    if (c) lk = std::unique_lock<std::recursive_mutex>(c->mu);
    try {
        f();
        return PARL_OK;
    } catch (const Error& e) {
        if (c) c->err = e.msg;
        tl_err = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        if (c) c->err = e.what();
        tl_err = e.what();
        return PARL_E_CUDA;
    }
}

void check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error{PARL_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e)};
}

void validate_config(const parl_config& c) {  // ModelConfig::validate, model.cpp:19-31
    if (c.vocab_size < 4)
        throw Error{PARL_E_CONFIG, "vocab_size must be >= 4 (ids 0..3 are reserved), got " + std::to_string(c.vocab_size)};
    if (c.d_model <= 0) throw Error{PARL_E_CONFIG, "d_model must be positive"};
    if (c.n_layers <= 0) throw Error{PARL_E_CONFIG, "n_layers must be positive"};
    if (c.n_heads <= 0) throw Error{PARL_E_CONFIG, "n_heads must be positive"};
    if (c.d_ff <= 0) throw Error{PARL_E_CONFIG, "d_ff must be positive"};
    if (c.max_seq_len <= 0) throw Error{PARL_E_CONFIG, "max_seq_len must be positive"};
    if (c.d_model % c.n_heads != 0)
        throw Error{PARL_E_CONFIG, "d_model (" + std::to_string(c.d_model) + ") not divisible by n_heads (" +
                                       std::to_string(c.n_heads) + ")"};
    if (c.d_model / c.n_heads > 128) throw Error{PARL_E_CONFIG, "head dim > 128 not supported by the device path"};
}

// per-array stride of the group's [T] vectors: a multiple of 4 elements keeps every array
// 16-byte aligned for the vectorised kernels (K7)
size_t group_stride(const parl_group_s* g) { return ((size_t)g->max_T + 3) & ~(size_t)3; }
float* group_lp(parl_group_s* g, int slot) { return static_cast<float*>(g->lp.p) + (size_t)slot * group_stride(g); }

bool same_cfg(const parl_config& a, const parl_config& b) { return std::memcmp(&a, &b, sizeof(a)) == 0; }

size_t act_size(parl_precision p) { return p == PARL_PREC_BF16 ? 2 : 4; }

// One weight tensor's place in the compute copy.
struct TensorMap {
    size_t src_off;  // offset in the reference flat layout
    int rows, cols;  // reference shape
    bool matrix;     // act dtype, stored transposed ([cols x rows])
    void* dst;       // f32 (vector/embedding) or act-dtype destination
    long ldd;
    int kind;        // 0 normal(0.08), 1 ones, 2 zeros  (model.cpp:152-162)
};

std::vector<TensorMap> tensor_maps(parl_model_s* m) {
    const auto& c = m->cfg;
    const int d = c.d_model, F = c.d_ff, V = c.vocab_size;
    std::vector<TensorMap> v;
    const size_t es = act_size(m->ctx->prec);
    auto actp = [&](void* base, size_t elems) { return static_cast<char*>(base) + elems * es; };
    v.push_back({m->L.tok_emb, V, d, false, m->W.tok_emb, d, 0});
    v.push_back({m->L.pos_emb, c.max_seq_len, d, false, m->W.pos_emb, d, 0});
    for (int l = 0; l < c.n_layers; ++l) {
        auto o = m->L.layer(l, d, F);
        LayerW& w = m->layers[l];
        v.push_back({o.ln1g, 1, d, false, w.ln1_g, d, 1});
        v.push_back({o.ln1b, 1, d, false, w.ln1_b, d, 2});
        v.push_back({o.wq, d, d, true, actp(w.wqkv_t, 0), d, 0});
        v.push_back({o.bq, 1, d, false, w.bqkv, d, 2});
        v.push_back({o.wk, d, d, true, actp(w.wqkv_t, (size_t)d * d), d, 0});
        v.push_back({o.bk, 1, d, false, w.bqkv + d, d, 2});
        v.push_back({o.wv, d, d, true, actp(w.wqkv_t, (size_t)2 * d * d), d, 0});
        v.push_back({o.bv, 1, d, false, w.bqkv + 2 * d, d, 2});
        v.push_back({o.wo, d, d, true, w.wo_t, d, 0});
        v.push_back({o.bo, 1, d, false, w.bo, d, 2});
        v.push_back({o.ln2g, 1, d, false, w.ln2_g, d, 1});
        v.push_back({o.ln2b, 1, d, false, w.ln2_b, d, 2});
        v.push_back({o.w1, d, F, true, w.w1_t, d, 0});
        v.push_back({o.b1, 1, F, false, w.b1, F, 2});
        v.push_back({o.w2, F, d, true, w.w2_t, F, 0});
        v.push_back({o.b2, 1, d, false, w.b2, d, 2});
    }
    v.push_back({m->L.lnf_g, 1, d, false, m->W.lnf_g, d, 1});
    v.push_back({m->L.lnf_b, 1, d, false, m->W.lnf_b, d, 2});
    v.push_back({m->L.head_w, d, V, true, m->W.head_w_t, d, 0});
    v.push_back({m->L.head_b, 1, V, false, m->W.head_b, V, 2});
    return v;
}

void convert_tensor(parl_model_s* m, const TensorMap& t, const double* dsrc) {
    cudaStream_t st = m->ctx->st;
    if (!t.matrix) {
        launch_convert_w<float>(dsrc, t.rows, t.cols, static_cast<float*>(t.dst), t.cols, 0, st);
    } else if (m->ctx->prec == PARL_PREC_BF16) {
        launch_convert_w<bf16>(dsrc, t.rows, t.cols, static_cast<bf16*>(t.dst), t.ldd, 1, st);
    } else {
        launch_convert_w<float>(dsrc, t.rows, t.cols, static_cast<float*>(t.dst), t.ldd, 1, st);
    }
}

// compute copy of one tensor -> fp64 (flat reference layout)
void export_tensor(parl_model_s* m, const TensorMap& t, double* stg, cudaStream_t st) {
    if (!t.matrix) launch_export_w<float>(static_cast<float*>(t.dst), t.cols, t.rows, t.cols, 0, stg, st);
    else if (m->ctx->prec == PARL_PREC_BF16)
        launch_export_w<bf16>(static_cast<bf16*>(t.dst), t.ldd, t.rows, t.cols, 1, stg, st);
    else launch_export_w<float>(static_cast<float*>(t.dst), t.ldd, t.rows, t.cols, 1, stg, st);
}

// Rebuild the compute copy from the device fp64 master.
void convert_from_master(parl_model_s* m) {
    const double* base = static_cast<const double*>(m->master.p);
    for (const auto& t : tensor_maps(m)) convert_tensor(m, t, base + t.src_off);
    check_launch();
}

// Contractions: bf16 runs on the tcgen05 kernels only (a shape they reject is an
// error, never a silent SIMT fallback); fp32 (BASELINE configs[0]) is the FFMA kernel.
template <class T>
void gemm(parl_ctx_s* c, const GemmArgs& g, int cls = PARL_KC_GEMM) {
    ProfScope ps(c, cls, 2.0 * g.M * (double)g.N * g.K);
    if constexpr (std::is_same_v<T, bf16>) {
        PARL_REQUIRE(gemm_tc(g, c->st), PARL_E_CONFIG,
                     "tcgen05 GEMM rejected shape " + std::to_string(g.M) + "x" + std::to_string(g.N) + "x" +
                         std::to_string(g.K) + " (bf16 needs 16-byte aligned rows)");
    } else {
        gemm_simt<T>(g, c->st);
    }
}

GemmArgs mk(int M, int N, int K, const void* A, long sam, long sak, const void* B, long sbn, long sbk) {
    GemmArgs g;
    g.M = M; g.N = N; g.K = K;
    g.A = A; g.sam = sam; g.sak = sak;
    g.B = B; g.sbn = sbn; g.sbk = sbk;
    return g;
}

void ensure_sorted(parl_group_s* g) {
    if (g->sorted_epoch == g->epoch) return;
    cudaStream_t st = g->ctx->st;
    const int T = g->T;
    int32_t* iota = g->iota.as<int32_t>(T);
    launch_iota(iota, T, st);
    const size_t tb = sort_temp_bytes(T);
    void* tmp = g->sort_tmp.get(std::max<size_t>(tb, 16));
    auto bits = [](int n) {
        int b = 1;
        while ((1L << b) < n) ++b;
        return b;
    };
    launch_sort_pairs(tmp, tb, g->pk.tokens, g->tok_keys.as<int32_t>(T), iota, g->tok_idx.as<int32_t>(T), T,
                      bits(g->vocab), st);
    launch_sort_pairs(tmp, tb, g->pk.positions, g->pos_keys.as<int32_t>(T), iota, g->pos_idx.as<int32_t>(T), T,
                      bits(g->max_seq), st);
    g->sorted_epoch = g->epoch;
}

void ensure_attn_work(parl_group_s* g, int H, int d);

// ---------------------------------------------------------------------------
// forward (forward_logprobs, model.cpp:534-567; run_forward 430-521)
//
// Several models over the same packed group (trimodel_forward, pipeline.cpp:22-30)
// run layer-interleaved: the three models' copies of each layer GEMM go out as one
// grouped launch (3x the tiles: full waves, one prologue), with per-model kernels
// for LayerNorm, attention and the head.  Every model runs the same kernels, so
// identical weights still give bit-identical outputs (test_pipeline.cpp:126-127).
// Model 0 may keep its activations (`act`, the policy); the others use per-slot
// scratch that holds one layer at a time.
template <class T>
void gemm_multi(parl_ctx_s* c, const GemmArgs* gs, int n) {
    double fl = 0;
    for (int q = 0; q < n; ++q) fl += 2.0 * gs[q].M * (double)gs[q].N * gs[q].K;
    ProfScope ps(c, PARL_KC_GEMM, fl);
    if constexpr (std::is_same_v<T, bf16>) {
        if (gemm_tc_multi(gs, n, c->st)) return;
        for (int q = 0; q < n; ++q)
            PARL_REQUIRE(gemm_tc(gs[q], c->st), PARL_E_CONFIG, "tcgen05 GEMM rejected a layer shape");
    } else {
        for (int q = 0; q < n; ++q) gemm_simt<T>(gs[q], c->st);
    }
}

// Per-layer activation buffers of one model in a forward.  With `stack_layers`
// every layer's tensors are kept for the backward; without it one layer's set is
// reused (cache-less forwards, and the policy under activation recomputation,
// where only the residual stream x_0..x_L is kept: `stack_x`).
template <class T>
struct FwdBufs {
    bool stack_x = false, stack_layers = false;
    float* xs = nullptr;    // residual stream: layer inputs x_0..x_L (stack) or ping-pong
    float* xmid = nullptr;  // x_mid
    T *a = nullptr, *qkv = nullptr, *ctxo = nullptr, *bn = nullptr, *pre = nullptr, *actv = nullptr;
    float *stats = nullptr, *lse_attn = nullptr;
    T* kv = nullptr;  // prefill of the KV-cached decoder: every layer's K | V rows kept, [L][T][2d]
    size_t lay(size_t per, int l) const { return stack_layers ? per * (size_t)l : 0; }
    float* xin(size_t TD, int l) const { return xs + (stack_x ? TD * l : TD * (l & 1)); }
};

AttnArgs attn_args(parl_group_s* g, const parl_config& cf) {
    AttnArgs aa;
    aa.T = g->T; aa.H = cf.n_heads; aa.Dh = cf.d_model / cf.n_heads; aa.d = cf.d_model;
    aa.seg = g->pk.seg;
    aa.seg_info = static_cast<const int4*>(g->seg_info.p);
    aa.scale = 1.0f / std::sqrt((float)aa.Dh);
    aa.sched = g->sched;
    aa.ldo = cf.d_model + PAD_COLS;
    aa.item_ctr = static_cast<unsigned*>(g->ctx->item_ctr.p);
    aa.item_base = &g->ctx->item_base;
    return aa;
}

// One decoder layer (model.cpp:458-516) for nm models at once (grouped GEMMs).
// `recompute`: rebuild the layer's activations for the backward; the W2 GEMM
// (whose output x_{l+1} is already kept) is skipped.
template <class T>
void layer_forward(parl_ctx_s* c, parl_model_s* const* ms, int nm, const FwdBufs<T>* B, int l, parl_group_s* g,
                   const AttnArgs& aa, bool recompute) {
    cudaStream_t st = c->st;
    const auto& cf = ms[0]->cfg;
    const int Tn = g->T, D = cf.d_model, H = cf.n_heads, F = cf.d_ff;
    const size_t TD = (size_t)Tn * D;
    const int Dp = D + PAD_COLS, Fp = F + PAD_COLS;
    const size_t TDp = (size_t)Tn * Dp, TFp = (size_t)Tn * Fp;
    GemmArgs gs[3];
    // LayerNorm of the nm models in one launch
    auto ln_multi = [&](int which) {
        const float* x[3];
        const float *gg[3], *bb[3];
        T* y[3];
        float *mu[3], *rs[3];
        for (int k = 0; k < nm; ++k) {
            const FwdBufs<T>& b = B[k];
            const LayerW& w = ms[k]->layers[l];
            float* st4 = b.stats + b.lay((size_t)4 * Tn, l) + (which ? 2 * Tn : 0);
            x[k] = which ? b.xmid + b.lay(TD, l) : b.xin(TD, l);
            gg[k] = which ? w.ln2_g : w.ln1_g;
            bb[k] = which ? w.ln2_b : w.ln1_b;
            y[k] = which ? b.bn + b.lay(TDp, l) : b.a + b.lay(TDp, l);
            mu[k] = st4;
            rs[k] = st4 + Tn;
        }
        launch_layernorm_multi<T>(nm, x, gg, bb, y, Dp, mu, rs, Tn, D, st);
    };
    {
        ProfScope ps(c, PARL_KC_NORM, (double)Tn * D * (4 + sizeof(T)) * nm);
        ln_multi(0);
    }
    for (int k = 0; k < nm; ++k) {  // fused Q|K|V projection (model.cpp:464-466)
        const FwdBufs<T>& b = B[k];
        const LayerW& w = ms[k]->layers[l];
        gs[k] = mk(Tn, 3 * D, D, b.a + b.lay(TDp, l), Dp, 1, w.wqkv_t, D, 1);
        gs[k].epi = EPI_ACT; gs[k].bias = w.bqkv; gs[k].Ca = b.qkv + b.lay(3 * TD, l); gs[k].ldca = 3 * D;
    }
    gemm_multi<T>(c, gs, nm);
    if (B[0].kv)  // K | V columns of this layer's projection into the decoder's cache
        PARL_CUDA(cudaMemcpy2DAsync(B[0].kv + (size_t)l * Tn * 2 * D, (size_t)2 * D * sizeof(T),
                                    B[0].qkv + B[0].lay(3 * TD, l) + D, (size_t)3 * D * sizeof(T),
                                    (size_t)2 * D * sizeof(T), Tn, cudaMemcpyDeviceToDevice, st));
    {
        ProfScope ps(c, PARL_KC_ATTN_FWD, 4.0 * g->pairs * D * nm);
        T* ql[3];
        T* cl[3];
        float* la[3];
        for (int k = 0; k < nm; ++k) {
            const FwdBufs<T>& b = B[k];
            ql[k] = b.qkv + b.lay(3 * TD, l);
            cl[k] = b.ctxo + b.lay(TDp, l);
            la[k] = b.lse_attn + b.lay((size_t)H * Tn, l);
        }
        if constexpr (std::is_same_v<T, bf16>) {  // the models' attention as one tcgen05 launch
            PARL_REQUIRE(attn_fwd_tc_multi(aa, ql, cl, la, nm, st), PARL_E_CONFIG,
                         "tcgen05 attention rejected the head dim / alignment");
        } else {
            for (int k = 0; k < nm; ++k) launch_attn_fwd<T>(aa, ql[k], cl[k], la[k], st);
        }
    }
    for (int k = 0; k < nm; ++k) {  // O projection + residual (model.cpp:504-506)
        const FwdBufs<T>& b = B[k];
        const LayerW& w = ms[k]->layers[l];
        gs[k] = mk(Tn, D, D, b.ctxo + b.lay(TDp, l), Dp, 1, w.wo_t, D, 1);
        gs[k].epi = EPI_RESID; gs[k].bias = w.bo; gs[k].resid = b.xin(TD, l);
        gs[k].Cf = b.xmid + b.lay(TD, l); gs[k].ldc = D;
    }
    gemm_multi<T>(c, gs, nm);
    {
        ProfScope ps(c, PARL_KC_NORM, (double)Tn * D * (4 + sizeof(T)) * nm);
        ln_multi(1);
    }
    for (int k = 0; k < nm; ++k) {  // W1 + bias + GELU (model.cpp:509-511)
        const FwdBufs<T>& b = B[k];
        const LayerW& w = ms[k]->layers[l];
        gs[k] = mk(Tn, F, D, b.bn + b.lay(TDp, l), Dp, 1, w.w1_t, D, 1);
        gs[k].bias = w.b1; gs[k].ldca = Fp;
        if (b.pre) {  // the backward needs the pre-activation u (GELU') and the activation
            gs[k].epi = EPI_GELU; gs[k].Ca = b.pre + b.lay(TFp, l); gs[k].Caux = b.actv + b.lay(TFp, l);
        } else {
            gs[k].epi = EPI_GELU_ACT; gs[k].Ca = b.actv;
        }
    }
    gemm_multi<T>(c, gs, nm);
    if (recompute) return;
    for (int k = 0; k < nm; ++k) {  // W2 + bias + residual (model.cpp:513-515)
        const FwdBufs<T>& b = B[k];
        const LayerW& w = ms[k]->layers[l];
        gs[k] = mk(Tn, D, F, b.actv + b.lay(TFp, l), Fp, 1, w.w2_t, F, 1);
        gs[k].epi = EPI_RESID; gs[k].bias = w.b2; gs[k].resid = b.xmid + b.lay(TD, l);
        gs[k].Cf = b.xin(TD, l + 1); gs[k].ldc = D;
    }
    gemm_multi<T>(c, gs, nm);
}

// Bytes of the per-layer activation stacks (all layers) and of the backward's
// workspaces, for the recompute decision.
size_t layer_act_bytes(const parl_config& cf, int Tn, size_t es) {
    const size_t D = cf.d_model, F = cf.d_ff, H = cf.n_heads, Dp = D + PAD_COLS, Fp = F + PAD_COLS;
    return (size_t)Tn * (4 * D + es * (3 * Dp + 3 * D + 2 * Fp) + 16 + 4 * H);
}

// Activation recomputation (c->recompute: 0 auto, 1 always, 2 never).  Auto keeps
// every layer's activations when they fit next to the backward's workspaces;
// otherwise only the residual stream is kept and each layer is rebuilt in the
// backward (C3 / C4 sizes: 150-280 GB of stacks).
template <class T>
bool want_recompute(parl_ctx_s* c, parl_act_s* act, const parl_config& cf, int Tn, int S) {
    if (c->recompute == 1) return true;
    if (c->recompute == 2) return false;
    // decided once per activation handle and shape (cudaMemGetInfo is a driver round trip)
    if (act->rc_key[0] == Tn && act->rc_key[1] == S && act->rc_key[2] == cf.d_model) return act->recompute;
    const size_t es = sizeof(T), D = cf.d_model, F = cf.d_ff, V = cf.vocab_size, H = cf.n_heads;
    const size_t stacks = layer_act_bytes(cf, Tn, es) * cf.n_layers + (size_t)S * V * es;
    const size_t held = act->xmid.bytes + act->a.bytes + act->qkv.bytes + act->ctxo.bytes + act->bn.bytes +
                        act->pre.bytes + act->actv.bytes + act->stats.bytes + act->lse_attn.bytes + act->logits.bytes;
    const size_t TD = (size_t)Tn * D;
    const size_t ws = (size_t)S * V * es + (size_t)Tn * (F + PAD_COLS) * es + 5 * TD * 4 + 6 * TD * es +
                      H * Tn * 4 + 2 * (size_t)S * D * 4;
    const size_t ws_held = c->dz.bytes + c->dpre.bytes + c->dx.bytes + c->dx2.bytes + c->dbn.bytes + c->dmid.bytes +
                           c->da.bytes + c->dx_act.bytes + c->dmid_act.bytes + c->dctx.bytes + c->dqkv.bytes +
                           c->dsum.bytes + c->dhf.bytes + c->dxg.bytes;
    size_t free_b = 0, total_b = 0;
    PARL_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const size_t avail = free_b + held, need = stacks + (ws > ws_held ? ws - ws_held : 0) + ((size_t)3 << 30);
    act->rc_key[0] = Tn;
    act->rc_key[1] = S;
    act->rc_key[2] = cf.d_model;
    return need > avail;
}

// LM head with the fused vocab log-sum-exp / target gather epilogue (bf16 path);
// `logits`: where the bf16 logits go (the policy's backward), or null
GemmArgs head_lse_args(parl_ctx_s* c, parl_model_s* m, parl_group_s* g, const bf16* hf, bf16* logits) {
    const int S = g->S, V = m->cfg.vocab_size, D = m->cfg.d_model;
    const int n_parts = (V + 127) / 128;
    GemmArgs ga = mk(S, V, D, hf, D + PAD_COLS, 1, m->W.head_w_t, D, 1);
    ga.epi = EPI_LSE; ga.bias = m->W.head_b; ga.labels = g->pk.scored_label;
    ga.part = c->part.as<float>((size_t)S * n_parts * 2);
    ga.target = c->target.as<float>(S);
    ga.n_parts = n_parts; ga.part_cols = 128;
    ga.logits_act = logits;
    ga.ldca = V;
    return ga;
}

template <class T>
void forward_impl(parl_ctx_s* c, parl_model_s* const* ms, const int* slots, int nm, parl_group_s* g,
                  parl_act_s* act, bool full_logits = false, T* kv_out = nullptr) {
    cudaStream_t st = c->st;
    const auto& cf = ms[0]->cfg;
    const int Tn = g->T, D = cf.d_model, H = cf.n_heads, F = cf.d_ff, V = cf.vocab_size, S = g->S;
    const int NL = cf.n_layers;
    const size_t TD = (size_t)Tn * D;
    // GEMM-operand activations carry PAD extra columns: column D (F) is 1.0 so the
    // weight-gradient GEMM of the backward also produces the bias gradient
    // (the bias row follows the weight in the flat layout, model.cpp:86-114)
    const int Dp = D + PAD_COLS, Fp = F + PAD_COLS;
    const size_t TDp = (size_t)Tn * Dp, TFp = (size_t)Tn * Fp;

    FwdBufs<T> B[3];
    for (int k = nm - 1; k >= 0; --k) {  // the policy's (k = 0) last: its recompute decision sees the rest
        FwdBufs<T>& b = B[k];
        if (k == 0 && act) {
            const bool rc = want_recompute<T>(c, act, cf, Tn, S);
            const int nl = rc ? 1 : NL;
            act->recompute = rc;
            b.stack_x = true;
            b.stack_layers = !rc;
            b.xs = act->xs.as<float>(TD * (NL + 1));
            b.xmid = act->xmid.as<float>(TD * nl);
            b.a = act->a.as<T>(TDp * nl);
            b.qkv = act->qkv.as<T>(3 * TD * nl);
            b.ctxo = act->ctxo.as<T>(TDp * nl);
            b.bn = act->bn.as<T>(TDp * nl);
            b.pre = rc ? nullptr : act->pre.as<T>(TFp * nl);
            b.actv = act->actv.as<T>(TFp * nl);
            b.stats = act->stats.as<float>((size_t)4 * Tn * nl);
            b.lse_attn = act->lse_attn.as<float>((size_t)H * Tn * nl);
        } else {
            auto& r = c->scr[slots[k]];
            b.xs = r.x.as<float>(TD * 2);
            b.xmid = r.xmid.as<float>(TD);
            b.a = r.a.as<T>(TDp);
            b.qkv = r.qkv.as<T>(3 * TD);
            b.ctxo = r.ctxo.as<T>(TDp);
            b.bn = r.bn.as<T>(TDp);
            b.pre = nullptr;
            b.actv = r.actv.as<T>(TFp);
            b.stats = r.stats.as<float>((size_t)4 * Tn);
            b.lse_attn = r.lse_attn.as<float>((size_t)H * Tn);
        }
    }

    B[0].kv = kv_out;
    if constexpr (std::is_same_v<T, bf16>) ensure_attn_work(g, H, D);
    const AttnArgs aa = attn_args(g, cf);
    {
        ProfScope ps(c, PARL_KC_NORM, (double)Tn * D * 12 * nm);
        for (int k = 0; k < nm; ++k)
            launch_embed(ms[k]->W.tok_emb, ms[k]->W.pos_emb, g->pk.tokens, g->pk.positions, Tn, D, B[k].xin(TD, 0),
                         st);
    }
    for (int l = 0; l < NL; ++l) layer_forward<T>(c, ms, nm, B, l, g, aa, false);
    // final LN + head only on the scored tokens' predecessor rows (model.cpp:518-556)
    for (int k = 0; k < nm; ++k) {
        const FwdBufs<T>& b = B[k];
        parl_model_s* m = ms[k];
        parl_act_s* ak = (k == 0) ? act : nullptr;
        auto& r = c->scr[slots[k]];
        float* xfin = b.xin(TD, NL);
        T* hf = ak ? ak->hf.as<T>((size_t)S * Dp) : r.hf.as<T>((size_t)S * Dp);
        if (ak) {  // bias columns of the weight-gradient operands (refilled when the buffers move)
            const long rows = (long)Tn * (b.stack_layers ? NL : 1);
            const uintptr_t sig[8] = {(uintptr_t)b.a, (uintptr_t)b.ctxo, (uintptr_t)b.bn, (uintptr_t)b.actv,
                                      (uintptr_t)hf, (uintptr_t)Tn, (uintptr_t)S, (uintptr_t)rows};
            if (std::memcmp(sig, ak->pad_sig, sizeof(sig)) != 0) {
                launch_fill_pad<T>(b.a, rows, D, Dp, st);
                launch_fill_pad<T>(b.ctxo, rows, D, Dp, st);
                launch_fill_pad<T>(b.bn, rows, D, Dp, st);
                launch_fill_pad<T>(b.actv, rows, F, Fp, st);
                launch_fill_pad<T>(hf, (long)S, D, Dp, st);
                std::memcpy(ak->pad_sig, sig, sizeof(sig));
            }
        }
        float* lnf_mean = ak ? ak->lnf_mean.as<float>(S) : r.lnf_mean.as<float>(S);
        float* lnf_rstd = ak ? ak->lnf_rstd.as<float>(S) : r.lnf_rstd.as<float>(S);
        float* lse_head = ak ? ak->lse_head.as<float>(S) : r.lse_head.as<float>(S);
        float* lp = group_lp(g, slots[k]);
        if (S > 0) {
            launch_layernorm<T>(xfin, g->pk.pred_pos, S, D, m->W.lnf_g, m->W.lnf_b, hf, Dp, lnf_mean, lnf_rstd, st);
            bool fused = false;
            if constexpr (std::is_same_v<T, bf16>) if (!full_logits) {
                // tcgen05 head with the vocab log-sum-exp and target gather fused
                // into the epilogue: logits reach HBM only for the policy (bf16,
                // kept for the backward unless it recomputes them), never for old/ref.
                if (ak) ak->logits_rc = ak->recompute || c->head_recompute;
                bf16* keep = (ak && !ak->logits_rc) ? ak->logits.as<bf16>((size_t)S * V) : nullptr;
                GemmArgs ga = head_lse_args(c, m, g, hf, keep);
                {
                    ProfScope ps(c, PARL_KC_HEAD, 2.0 * S * (double)V * D);
                    fused = gemm_tc(ga, st);
                    if (fused) launch_lse_combine(ga.part, ga.n_parts, ga.target, S, lse_head, lp, st);
                }
            }
            if (!fused) {
                float* logits = ak ? ak->logits.as<float>((size_t)S * V) : r.logits.as<float>((size_t)S * V);
                GemmArgs ga = mk(S, V, D, hf, Dp, 1, m->W.head_w_t, D, 1);
                ga.epi = EPI_F32; ga.bias = m->W.head_b; ga.Cf = logits; ga.ldc = V;
                gemm<T>(c, ga, PARL_KC_HEAD);
                launch_row_lse(logits, S, V, g->pk.scored_label, lse_head, lp, st);
            }
            if (ak) ak->logits_bf16 = fused;
        }
    }
    check_launch();
}

}  // namespace
int nccl_allreduce_raw(void* p, size_t n, int dtype, int op, void* comm, cudaStream_t st);
namespace {
// Allreduce (sum) of n elements at p on the communicator's stream, after everything the
// compute stream has issued so far.  dtype: ncclFloat32 = 7, ncclFloat64 = 8.
void comm_allreduce(parl_ctx_s* c, void* p, size_t n, int dtype, int op = 0 /* ncclSum */) {
    PARL_CUDA(cudaEventRecord(c->ev_comm, c->st));
    PARL_CUDA(cudaStreamWaitEvent(c->comm_st, c->ev_comm, 0));
    const int r = nccl_allreduce_raw(p, n, dtype, op, c->comm, c->comm_st);
    PARL_REQUIRE(r == 0, PARL_E_NCCL, "ncclAllReduce failed");
}

// backward (model.cpp:587-838) + GradBuffer::accumulate (model.cpp:189-194)
template <class T>
void backward_impl(parl_ctx_s* c, parl_model_s* m, parl_act_s* act, parl_group_s* g, parl_grad_s* gr) {
    cudaStream_t st = c->st;
    const auto& cf = m->cfg;
    const int Tn = g->T, D = cf.d_model, H = cf.n_heads, F = cf.d_ff, V = cf.vocab_size, S = g->S;
    const int NL = cf.n_layers;
    const int Dp = D + PAD_COLS, Fp = F + PAD_COLS;
    const size_t TD = (size_t)Tn * D, TDp = (size_t)Tn * Dp, TFp = (size_t)Tn * Fp;
    float* G = static_cast<float*>(gr->g.p);
    const FlatLayout& L = gr->L;
    const float* u = static_cast<const float*>(g->upstream.p);

    float* dx = c->dx.as<float>(TD);
    T* dx_act = c->dx_act.as<T>(TD);
    if (S > 0) {
        // dZ = u (onehot - softmax) at the head rows (model.cpp:637-650)
        T* dz = c->dz.as<T>((size_t)S * V);
        {
            if (act->logits_bf16 && act->logits_rc) {
                if constexpr (std::is_same_v<T, bf16>) {
                    // logits were not kept: the same head GEMM rebuilds them (bit-identical)
                    // into dZ, which the softmax backward then overwrites in place
                    GemmArgs ga = head_lse_args(c, m, g, static_cast<const bf16*>(act->hf.p), dz);
                    {
                        ProfScope ps_h(c, PARL_KC_HEAD, 2.0 * S * (double)V * D);
                        PARL_REQUIRE(gemm_tc(ga, st), PARL_E_CUDA, "head recompute: tcgen05 GEMM unavailable");
                    }
                    ProfScope ps_sm(c, PARL_KC_SEED, 4.0 * S * (double)V);  // bf16 z in, bf16 dZ out
                    launch_softmax_bwd<bf16, T>(dz, V, dz, V, S, V, static_cast<float*>(act->lse_head.p), u,
                                                g->pk.scored_label, st);
                }
            } else if (act->logits_bf16) {
                ProfScope ps_sm(c, PARL_KC_SEED, 4.0 * S * (double)V);
                launch_softmax_bwd<bf16, T>(static_cast<bf16*>(act->logits.p), V, dz, V, S, V,
                                            static_cast<float*>(act->lse_head.p), u, g->pk.scored_label, st);
            } else {
                ProfScope ps_sm(c, PARL_KC_SEED, (4.0 + sizeof(T)) * S * (double)V);
                launch_softmax_bwd<float, T>(static_cast<float*>(act->logits.p), V, dz, V, S, V,
                                             static_cast<float*>(act->lse_head.p), u, g->pk.scored_label, st);
            }
        }
        T* hf = static_cast<T*>(act->hf.p);
        float* dhf = c->dhf.as<float>((size_t)S * D);
        {  // dH = dZ W_head^T (model.cpp:654-666)
            GemmArgs ga = mk(S, D, V, dz, V, 1, m->W.head_w_t, 1, D);
            ga.epi = EPI_F32; ga.Cf = dhf; ga.ldc = D;
            gemm<T>(c, ga);
        }
        {  // [dW_head; db_head] += [H 1]^T dZ  (hf's column D is 1)
            GemmArgs ga = mk(D + 1, V, S, hf, 1, Dp, dz, 1, V);
            ga.epi = EPI_F32_ACC; ga.Cf = G + L.head_w; ga.ldc = V;
            gemm<T>(c, ga);
        }
        // final LN backward on the gathered rows, then scatter to positions
        float* dxg = c->dxg.as<float>((size_t)S * D);
        float* xfin = static_cast<float*>(act->xs.p) + TD * NL;
        {
            // algorithmic bytes: final-LN backward over the S gathered rows (dH, x in, dX out, fp32),
            // the scatter onto positions (dX rows in, dx out) and the compute-dtype copy of dx
            ProfScope ps_(c, PARL_KC_NORM,
                          (double)S * D * 12 + (double)S * D * 4 + (double)Tn * D * 4 + (double)Tn * D * (4 + sizeof(T)));
            launch_layernorm_bwd<T>(dhf, xfin, g->pk.pred_pos, static_cast<float*>(act->lnf_mean.p),
                                    static_cast<float*>(act->lnf_rstd.p), m->W.lnf_g, S, D, nullptr, dxg,
                                    static_cast<T*>(nullptr), G + L.lnf_g, G + L.lnf_b, st);
            launch_scatter_rows(dxg, g->pk.row_ptr, g->pk.row_idx, Tn, D, dx, st);
            launch_f32_to_act<T>(dx, dx_act, TD, st);
        }
    } else {
        PARL_CUDA(cudaMemsetAsync(dx, 0, TD * sizeof(float), st));
        PARL_CUDA(cudaMemsetAsync(dx_act, 0, TD * sizeof(T), st));
    }
    // overlapped data-parallel allreduce (armed by parl_grad_allreduce_overlap on the last
    // micro-batch): each gradient slice goes out as soon as this backward has finished it,
    // the final LN + head now, every layer after its LN1 backward, the embeddings last
    const bool stream_ar = gr->overlap && c->comm && c->nranks > 1;
    if (stream_ar) comm_allreduce(c, G + L.lnf_g, L.total - L.lnf_g, 7);

    T* dpre = c->dpre.as<T>(TFp);
    float* dbn = c->dbn.as<float>(TD);
    float* dmid = c->dmid.as<float>(TD);
    T* dmid_act = c->dmid_act.as<T>(TD);
    T* dctx = c->dctx.as<T>(TD);
    T* dqkv = c->dqkv.as<T>(3 * TD);
    float* da = c->da.as<float>(TD);
    float* dsum = c->dsum.as<float>((size_t)H * Tn);
    float* dx2 = c->dx2.as<float>(TD);

    if constexpr (std::is_same_v<T, bf16>) ensure_attn_work(g, H, D);
    const AttnArgs aa = attn_args(g, cf);
    // recompute mode: one layer's activation set, rebuilt from x_l before its backward
    const bool rc = act->recompute;
    FwdBufs<T> RB;
    RB.stack_x = true;
    RB.xs = static_cast<float*>(act->xs.p);
    RB.xmid = static_cast<float*>(act->xmid.p);
    RB.a = static_cast<T*>(act->a.p);
    RB.qkv = static_cast<T*>(act->qkv.p);
    RB.ctxo = static_cast<T*>(act->ctxo.p);
    RB.bn = static_cast<T*>(act->bn.p);
    RB.pre = rc ? act->pre.as<T>(TFp) : static_cast<T*>(act->pre.p);
    RB.actv = static_cast<T*>(act->actv.p);
    RB.stats = static_cast<float*>(act->stats.p);
    RB.lse_attn = static_cast<float*>(act->lse_attn.p);
    const int ll = rc ? 0 : 1;  // layer stride multiplier of the stacks

    // weight-gradient GEMMs of a layer are collected and run as one grouped launch
    // (bf16); the fp32 path runs them as they come
    std::vector<GemmArgs> dw;
    auto add_dw = [&](const GemmArgs& ga) {
        if constexpr (std::is_same_v<T, bf16>) dw.push_back(ga);
        else gemm<T>(c, ga);
    };
    auto flush_dw = [&]() {
        if (dw.empty()) return;
        bool done = false;
        if constexpr (std::is_same_v<T, bf16>) {
            double fl = 0;
            for (const auto& ga : dw) fl += 2.0 * ga.M * (double)ga.N * ga.K;
            ProfScope ps(c, PARL_KC_GEMM, fl);
            done = gemm_tc_group_dw(dw.data(), (int)dw.size(), st);
        }
        if (!done)  // one tcgen05 launch per problem (N not a multiple of 128)
            for (const auto& ga : dw) gemm<T>(c, ga);
        dw.clear();
    };
    for (int l = NL - 1; l >= 0; --l) {
        const LayerW& w = m->layers[l];
        const auto o = L.layer(l, D, F);
        if (rc) layer_forward<T>(c, &m, 1, &RB, l, g, aa, true);
        const int li = l * ll;
        float* xin = RB.xs + TD * l;
        float* xm = RB.xmid + TD * li;
        T* al = RB.a + TDp * li;
        T* ql = RB.qkv + 3 * TD * li;
        T* cl = RB.ctxo + TDp * li;
        T* bl = RB.bn + TDp * li;
        T* pl = RB.pre + TFp * li;
        T* vl = RB.actv + TFp * li;
        float* st4 = RB.stats + (size_t)4 * Tn * li;
        float* la = RB.lse_attn + (size_t)H * Tn * li;

        // FFN (model.cpp:688-727); dx_act holds the compute-dtype copy of dx
        {
            GemmArgs ga = mk(Tn, F, D, dx_act, D, 1, w.w2_t, 1, F);
            ga.epi = EPI_GELU_BWD; ga.aux_in = pl; ga.Ca = dpre; ga.ldca = Fp;
            gemm<T>(c, ga);
        }
        {  // [dW2; db2] += [act 1]^T dx
            GemmArgs ga = mk(F + 1, D, Tn, vl, 1, Fp, dx_act, 1, D);
            ga.epi = EPI_F32_ACC; ga.Cf = G + o.w2; ga.ldc = D;
            add_dw(ga);
        }
        {
            GemmArgs ga = mk(Tn, D, F, dpre, Fp, 1, w.w1_t, 1, D);
            ga.epi = EPI_F32; ga.Cf = dbn; ga.ldc = D;
            gemm<T>(c, ga);
        }
        {  // [dW1; db1] += [LN2 1]^T dpre
            GemmArgs ga = mk(D + 1, F, Tn, bl, 1, Dp, dpre, 1, Fp);
            ga.epi = EPI_F32_ACC; ga.Cf = G + o.w1; ga.ldc = F;
            add_dw(ga);
        }
        // LN2 (model.cpp:729-730): dmid = dx + LN2^T(dbn), plus its compute-dtype copy
        {  // bytes: dy, x, residual grad in (fp32), dx out (fp32) + its compute-dtype copy, per row
            ProfScope ps_(c, PARL_KC_NORM, (double)Tn * D * (16 + sizeof(T)));
            launch_layernorm_bwd<T>(dbn, xm, nullptr, st4 + 2 * Tn, st4 + 3 * Tn, w.ln2_g, Tn, D, dx, dmid, dmid_act,
                                    G + o.ln2g, G + o.ln2b, st);
        }
        // O projection (model.cpp:733-749)
        {
            GemmArgs ga = mk(Tn, D, D, dmid_act, D, 1, w.wo_t, 1, D);
            ga.epi = EPI_ACT; ga.Ca = dctx; ga.ldca = D;
            gemm<T>(c, ga);
        }
        {  // [dWo; dbo] += [ctx 1]^T dmid
            GemmArgs ga = mk(D + 1, D, Tn, cl, 1, Dp, dmid_act, 1, D);
            ga.epi = EPI_F32_ACC; ga.Cf = G + o.wo; ga.ldc = D;
            add_dw(ga);
        }
        // attention (model.cpp:752-786)
        {
            ProfScope ps(c, PARL_KC_ATTN_BWD, 10.0 * g->pairs * D);
            if constexpr (std::is_same_v<T, bf16>) {  // computes D = rowsum(dO O) itself
                PARL_REQUIRE(attn_bwd_tc(aa, ql, cl, dctx, la, dsum, dqkv, st), PARL_E_CONFIG,
                             "tcgen05 attention backward rejected the head dim / alignment");
            } else {
                launch_attn_bwd<T>(aa, ql, cl, dctx, la, dsum, dqkv, st);
            }
        }
        // Q/K/V projections (model.cpp:789-817)
        {
            GemmArgs ga = mk(Tn, D, 3 * D, dqkv, 3 * D, 1, w.wqkv_t, 1, D);
            ga.epi = EPI_F32; ga.Cf = da; ga.ldc = D;
            gemm<T>(c, ga);
        }
        const size_t woff[3] = {o.wq, o.wk, o.wv};
        for (int p = 0; p < 3; ++p) {  // [dWp; dbp] += [LN1 1]^T dqkv_p
            GemmArgs ga = mk(D + 1, D, Tn, al, 1, Dp, dqkv + (size_t)p * D, 1, 3 * D);
            ga.epi = EPI_F32_ACC; ga.Cf = G + woff[p]; ga.ldc = D;
            add_dw(ga);
        }
        flush_dw();  // dx_act is overwritten next
        // LN1 (model.cpp:820-822): dx <- dmid + LN1^T(da), plus the next layer's compute-dtype copy
        {
            ProfScope ps_(c, PARL_KC_NORM, (double)Tn * D * (16 + sizeof(T)));
            launch_layernorm_bwd<T>(da, xin, nullptr, st4, st4 + Tn, w.ln1_g, Tn, D, dmid, dx2, dx_act, G + o.ln1g,
                                    G + o.ln1b, st);
        }
        std::swap(dx, dx2);
        if (stream_ar) comm_allreduce(c, G + o.ln1g, L.layer_stride, 7);
    }
    // embeddings (model.cpp:826-834), deterministic segmented sums
    ensure_sorted(g);
    launch_mark_rows(g->pk.tokens, Tn, static_cast<uint8_t*>(gr->touched.p), st);
    launch_embed_grad(static_cast<int32_t*>(g->tok_keys.p), static_cast<int32_t*>(g->tok_idx.p), Tn, dx, D,
                      G + L.tok_emb, st);
    launch_embed_grad(static_cast<int32_t*>(g->pos_keys.p), static_cast<int32_t*>(g->pos_idx.p), Tn, dx, D,
                      G + L.pos_emb, st);
    check_launch();
    gr->micro_steps += 1;
    if (stream_ar) {
        gr->overlap = false;
        gr->streamed = true;
    }
}

// Host-side attention tile schedule (see AttnSched in kernels.cuh): the visibility rule of
// SegLayout (model.cpp:242-245, per prompt group) at 128 x 128 tile level.  The rows of a
// query tile fall into at most a few segments ("pieces"); a key tile is visible when some
// piece sees one of its keys and full (no per-element mask) when every row sees all of them.
AttnSched build_schedule(const SegLayout& L, DevBuf& buf, HostStage& stage, cudaStream_t st,
                         SchedHost* host_out = nullptr) {
    const int T = L.T();
    const int nt = (T + 127) / 128;
    struct Piece {
        int s, r0, r1;  // segment, rows [r0, r1)
    };
    std::vector<std::vector<Piece>> pieces(nt);
    for (size_t s = 0; s < L.start.size(); ++s)
        for (int r = L.start[s]; r < L.end[s];) {
            const int qt = r / 128, r1 = std::min(L.end[s], (qt + 1) * 128);
            pieces[qt].push_back({(int)s, r, r1});
            r = r1;
        }
    // rows [r0, r1) of segment s against keys [j0, j1)
    auto piece_visible = [&](const Piece& p, int j0, int j1) {
        const int4 f = L.info[p.s];
        if (f.y < 0) return std::max(f.x, j0) <= std::min(p.r1 - 1, j1 - 1);  // [A, i]
        return std::max(f.x, j0) < std::min(f.y, j1) || std::max(f.z, j0) <= std::min(p.r1 - 1, j1 - 1);
    };
    auto piece_full = [&](const Piece& p, int j0, int j1) {  // the piece's first row sees the least
        const int4 f = L.info[p.s];
        if (f.y < 0) return f.x <= j0 && j1 - 1 <= p.r0;
        if (f.z <= f.y)  // prompt and own prefix touch: one range [A, max(B, r0 + 1))
            return f.x <= j0 && j1 <= std::max(f.y, p.r0 + 1);
        return (f.x <= j0 && j1 <= f.y) || (f.z <= j0 && j1 - 1 <= p.r0);
    };
    auto visible = [&](int qt, int j0, int j1) {
        for (const auto& p : pieces[qt])
            if (piece_visible(p, j0, j1)) return true;
        return false;
    };
    auto full = [&](int qt, int j0) {
        const int j1 = j0 + 128;
        if (j1 > T || (qt + 1) * 128 > T) return false;
        for (const auto& p : pieces[qt])
            if (!piece_full(p, j0, j1)) return false;
        return true;
    };
    std::vector<int32_t> q_ptr(nt + 1, 0), q_list, k_ptr(nt + 1, 0), k_list;
    std::vector<std::vector<int32_t>> per_k(nt);
    for (int qt = 0; qt < nt; ++qt) {
        const int i0 = qt * 128, i1 = std::min(T, i0 + 128);
        for (int kt = 0; kt <= (i1 - 1) / 128; ++kt) {
            const int j0 = kt * 128, j1 = std::min(T, j0 + 128);
            if (!visible(qt, j0, j1)) continue;
            const int32_t e = (full(qt, j0) ? (1 << 30) : 0);
            q_list.push_back(kt | e);
            per_k[kt].push_back(qt | e);
        }
        q_ptr[qt + 1] = (int32_t)q_list.size();
    }
    for (int kt = 0; kt < nt; ++kt) {
        k_list.insert(k_list.end(), per_k[kt].begin(), per_k[kt].end());
        k_ptr[kt + 1] = (int32_t)k_list.size();
    }
    std::vector<int32_t> q_order(nt), k_order(nt);
    for (int t = 0; t < nt; ++t) q_order[t] = k_order[t] = t;
    std::stable_sort(q_order.begin(), q_order.end(),
                     [&](int x, int y) { return q_ptr[x + 1] - q_ptr[x] > q_ptr[y + 1] - q_ptr[y]; });
    std::stable_sort(k_order.begin(), k_order.end(),
                     [&](int x, int y) { return k_ptr[x + 1] - k_ptr[x] > k_ptr[y + 1] - k_ptr[y]; });
    // query-tile pairs: merged key lists with per-tile visibility / fullness flags
    const int np = (nt + 1) / 2;
    std::vector<int32_t> p_ptr(np + 1, 0), p_list, p_order(np);
    for (int p = 0; p < np; ++p) {
        int a0 = q_ptr[2 * p], a1 = q_ptr[2 * p + 1];
        int b0 = 2 * p + 1 < nt ? q_ptr[2 * p + 1] : 0, b1 = 2 * p + 1 < nt ? q_ptr[2 * p + 2] : 0;
        while (a0 < a1 || b0 < b1) {
            const int ka = a0 < a1 ? (q_list[a0] & 0x3fffffff) : INT32_MAX;
            const int kb = b0 < b1 ? (q_list[b0] & 0x3fffffff) : INT32_MAX;
            const int kt = std::min(ka, kb);
            int32_t e = kt;
            if (ka == kt) {
                e |= (1 << 24) | ((q_list[a0] >> 30) & 1) << 25;
                ++a0;
            }
            if (kb == kt) {
                e |= (1 << 26) | ((q_list[b0] >> 30) & 1) << 27;
                ++b0;
            }
            p_list.push_back(e);
        }
        p_ptr[p + 1] = (int32_t)p_list.size();
        p_order[p] = p;
    }
    std::stable_sort(p_order.begin(), p_order.end(),
                     [&](int x, int y) { return p_ptr[x + 1] - p_ptr[x] > p_ptr[y + 1] - p_ptr[y]; });
    std::vector<int32_t> all;
    all.reserve(4 * (nt + 1) + q_list.size() + k_list.size() + 2 * (np + 1) + p_list.size());
    size_t o_qp = all.size(); all.insert(all.end(), q_ptr.begin(), q_ptr.end());
    size_t o_ql = all.size(); all.insert(all.end(), q_list.begin(), q_list.end());
    size_t o_qo = all.size(); all.insert(all.end(), q_order.begin(), q_order.end());
    size_t o_kp = all.size(); all.insert(all.end(), k_ptr.begin(), k_ptr.end());
    size_t o_kl = all.size(); all.insert(all.end(), k_list.begin(), k_list.end());
    size_t o_ko = all.size(); all.insert(all.end(), k_order.begin(), k_order.end());
    size_t o_pp = all.size(); all.insert(all.end(), p_ptr.begin(), p_ptr.end());
    size_t o_pl = all.size(); all.insert(all.end(), p_list.begin(), p_list.end());
    size_t o_po = all.size(); all.insert(all.end(), p_order.begin(), p_order.end());
    int32_t* d = buf.as<int32_t>(all.size());
    stage.upload(d, all.data(), all.size() * 4, st);
    if (host_out) {
        host_out->q_ptr = q_ptr;
        host_out->k_ptr = k_ptr;
        host_out->p_ptr = p_ptr;
        // a key tile seen by both query tiles of a pair runs both softmax groups (sharing the
        // SM's exponential units); a one-sided one runs one, in about half the time
        host_out->p_cost.assign(np, 0);
        for (int p = 0; p < np; ++p)
            for (int e = p_ptr[p]; e < p_ptr[p + 1]; ++e)
                host_out->p_cost[p] += ((p_list[e] >> 24) & 1) + ((p_list[e] >> 26) & 1);
    }
    AttnSched s;
    s.q_ptr = d + o_qp; s.q_list = d + o_ql; s.q_order = d + o_qo;
    s.k_ptr = d + o_kp; s.k_list = d + o_kl; s.k_order = d + o_ko;
    s.p_ptr = d + o_pp; s.p_list = d + o_pl; s.p_order = d + o_po;
    s.n_pairs = np;
    return s;
}

// Longest-processing-time assignment of attention work items (tile * H + head)
// to one persistent CTA per SM; cost = partner tiles + 1 (per-item overhead).
// Appends [ptr (grid + 1) | items] to `all`; returns the grid.
// PARL_ATTN_ORDER=lpt: longest-first order (diagnostics); default head-major
bool attn_order_lpt() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("PARL_ATTN_ORDER");
        v = (e && std::strcmp(e, "lpt") == 0) ? 1 : 0;
    }
    return v == 1;
}

int lpt_lists(const std::vector<int32_t>& ptr, int H, std::vector<int32_t>& all, bool locality,
              const std::vector<int32_t>* tile_cost = nullptr, std::vector<int32_t>* order_out = nullptr) {
    const int nt = (int)ptr.size() - 1;
    const int n = nt * H;
    int sms = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int grid = std::max(1, std::min(n, sms));
    std::vector<int32_t> order(n);
    // per item: partner tiles (or the given per-tile cost) + the per-item overhead
    auto cost = [&](int it) {
        return tile_cost ? (*tile_cost)[it / H] + 2 : ptr[it / H + 1] - ptr[it / H] + 1;
    };
    if (!locality || attn_order_lpt()) {
        for (int i = 0; i < n; ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return cost(x) > cost(y); });
    } else {
        // head-major, tiles ascending: the items in flight at any time belong to one or two
        // heads, whose K/V (or Q/dO) tiles then stay in L2 (C3: 34 MB per head) instead of
        // being re-read from HBM by every tile of every head.  Items far above the mean
        // cost (prompt key tiles of the dK/dV pass, seen by every query tile) go first,
        // longest first, so the greedy least-loaded assignment below stays balanced.
        long tot = 0;
        for (int t = 0; t < nt; ++t) tot += (long)cost(t * H) * H;
        const double big = 2.0 * (double)tot / std::max(n, 1);
        int k = 0;
        for (int i = 0; i < n; ++i)
            if (cost(i) > big) order[k++] = i;
        std::stable_sort(order.begin(), order.begin() + k, [&](int x, int y) { return cost(x) > cost(y); });
        for (int i = 0; i < n; ++i) {
            const int it = (i % nt) * H + i / nt;
            if (cost(it) <= big) order[k++] = it;
        }
    }
    if (order_out) *order_out = order;
    std::vector<std::vector<int32_t>> per(grid);
    using L = std::pair<long, int>;
    std::priority_queue<L, std::vector<L>, std::greater<L>> heap;
    for (int b = 0; b < grid; ++b) heap.push({0, b});
    for (int it : order) {
        auto [load, b] = heap.top();
        heap.pop();
        per[b].push_back(it);
        heap.push({load + cost(it), b});
    }
    int32_t acc = 0;
    all.push_back(0);
    for (int b = 0; b < grid; ++b) all.push_back(acc += (int32_t)per[b].size());
    for (int b = 0; b < grid; ++b) all.insert(all.end(), per[b].begin(), per[b].end());
    return grid;
}

// forward (query-tile pairs), dK/dV (key tiles) and dQ (query tiles) work lists
// (forward: head-major order only when the K/V of all heads overflow about half the L2;
// below that, longest-first balances better; the backward streams two operands per tile
// and gains from head-major order at every size measured)
void build_attn_work(AttnSched& s, const SchedHost& hs, int H, int dm, DevBuf& buf, HostStage& stage,
                     cudaStream_t st) {
    std::vector<int32_t> all;
    const double kv_bytes = 128.0 * ((double)hs.q_ptr.size() - 1) * dm * 4;
    const size_t o_f = all.size();
    std::vector<int32_t> forder;
    const int gf = lpt_lists(hs.p_ptr, H, all, kv_bytes > 64e6, hs.p_cost.empty() ? nullptr : &hs.p_cost, &forder);
    const size_t o_k = all.size();
    const int gk = lpt_lists(hs.k_ptr, H, all, true);
    const size_t o_q = all.size();
    const int gq = lpt_lists(hs.q_ptr, H, all, true);
    const size_t o_o = all.size();
    all.insert(all.end(), forder.begin(), forder.end());
    int32_t* d = buf.as<int32_t>(all.size());
    stage.upload(d, all.data(), all.size() * 4, st);
    s.w_ptr = d + o_f; s.w_items = d + o_f + gf + 1; s.w_grid = gf;
    s.w_order = d + o_o; s.w_n = (int)forder.size();
    s.bk_ptr = d + o_k; s.bk_items = d + o_k + gk + 1; s.bk_grid = gk;
    s.bq_ptr = d + o_q; s.bq_items = d + o_q + gq + 1; s.bq_grid = gq;
}

void ensure_attn_work(parl_group_s* g, int H, int d) {
    if (g->work_H == H && g->work_d == d) return;
    build_attn_work(g->sched, g->sched_h, H, d, g->work_buf, g->work_stage, g->ctx->st);
    g->work_H = H;
    g->work_d = d;
}

void alloc_group_arrays(parl_group_s* g) {
    const size_t T = group_stride(g);
    const int G = g->max_G;
    // tokens labels positions seg pred [T] ; scored_pos scored_label pred_pos sample_of [T];
    // row_ptr [T+1]; row_idx [T]
    int32_t* base = g->ints.as<int32_t>((size_t)T * 10 + 1);
    g->pk.tokens = base;
    g->pk.labels = base + T;
    g->pk.positions = base + 2 * (size_t)T;
    g->pk.seg = base + 3 * (size_t)T;
    g->pk.pred = base + 4 * (size_t)T;
    g->pk.scored_pos = base + 5 * (size_t)T;
    g->pk.scored_label = base + 6 * (size_t)T;
    g->pk.pred_pos = base + 7 * (size_t)T;
    g->pk.sample_of = base + 8 * (size_t)T;
    g->pk.row_idx = base + 9 * (size_t)T;
    g->seg_info.as<int4>((size_t)G + 1);                       // per-segment visibility (SegLayout)
    g->pk.row_ptr = g->cu_d.as<int32_t>((size_t)g->max_T + 1 + (G + 1));  // row_ptr [T+1] | cu [G+1]
    g->lp.as<float>((size_t)3 * T);
    g->upstream.as<float>(T);
    g->rewards.as<double>(G);
    g->adv.as<double>(G);
}

int32_t* group_cu(parl_group_s* g) { return static_cast<int32_t*>(g->cu_d.p) + g->max_T + 1; }

// upload the segment layout / response offsets computed on the host
void upload_meta(parl_group_s* g) {
    const SegLayout& L = g->segs;
    int4* si = g->seg_info.as<int4>(L.info.size());
    PARL_CUDA(cudaMemcpyAsync(si, L.info.data(), L.info.size() * sizeof(int4), cudaMemcpyHostToDevice, g->ctx->st));
    PARL_CUDA(cudaMemcpyAsync(group_cu(g), g->cu.data(), g->cu.size() * 4, cudaMemcpyHostToDevice, g->ctx->st));
    // the tile schedule and the attention work lists depend only on the segment structure:
    // a group re-packed with the same lengths (every step of a fixed-shape run) keeps them
    std::vector<int> key = L.start;
    key.insert(key.end(), L.end.begin(), L.end.end());
    for (const auto& f : L.info) key.insert(key.end(), {f.x, f.y, f.z, f.w});
    if (key == g->sched_key && g->sched.q_ptr) return;
    g->sched = build_schedule(L, g->sched_buf, g->sched_stage, g->ctx->st, &g->sched_h);
    g->sched_key = std::move(key);
    g->work_H = -1;
}

void check_pack_inputs(parl_group_s* g, int P, const int32_t* lens, int G, int max_seq) {
    if (P < 1) throw Error{PARL_E_SHAPE, "pack_group: empty prompt"};          // packing.cpp:9
    if (G < 1) throw Error{PARL_E_SHAPE, "pack_group: no responses"};          // packing.cpp:10
    long total = P;
    for (int k = 0; k < G; ++k) {
        if (lens[k] < 1) throw Error{PARL_E_SHAPE, "pack_group: empty response"};
        total += lens[k];
    }
    if (total > max_seq)                                                         // packing.cpp:16-19
        throw Error{PARL_E_SHAPE, "pack_group: packed length " + std::to_string(total) + " for group of " +
                                      std::to_string(G) + " responses exceeds max_seq_len " + std::to_string(max_seq)};
    if (total > g->max_T || G > g->max_G)
        throw Error{PARL_E_SHAPE, "packed group exceeds the capacity this group was created with"};
}

void set_pack_meta(parl_group_s* g, int P, const int32_t* lens, int G, int max_seq) {
    g->P = P;
    g->G = G;
    g->n_samples = G;
    g->lens.assign(lens, lens + G);
    g->span_start.resize(G);
    g->cu.assign(G + 1, 0);
    int t = P;
    for (int k = 0; k < G; ++k) {
        g->span_start[k] = t;
        g->cu[k + 1] = g->cu[k] + lens[k];
        t += lens[k];
    }
    g->T = t;
    g->S = t - P;
    g->Peff = P;
    g->n_groups = 1;
    g->group_G = G;
    g->segs.clear();
    g->segs.add_group(0, P, lens, G);
    g->pairs = g->segs.pairs();
    g->max_seq = max_seq;
    g->epoch++;
}

}  // namespace

// ===========================================================================
extern "C" {

const char* parl_version(void) { return "parl_gpu 0.1 (sm_100a)"; }

const char* parl_last_error(parl_ctx_t ctx) { return ctx ? ctx->err.c_str() : tl_err.c_str(); }

parl_status parl_ctx_create(int device, parl_precision prec, parl_ctx_t* out) {
    return guarded(nullptr, [&] {
        auto c = std::make_unique<parl_ctx_s>();
        c->device = device;
        c->prec = prec;
        PARL_CUDA(cudaSetDevice(device));
        PARL_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
        double* s = c->stats.as<double>(8);
        PARL_CUDA(cudaMemsetAsync(s, 0, 8 * sizeof(double), c->st));
        PARL_CUDA(cudaMemsetAsync(c->item_ctr.as<unsigned>(4), 0, 4 * sizeof(unsigned), c->st));
        if (const char* e = std::getenv("PARL_RECOMPUTE")) c->recompute = std::atoi(e);
        if (const char* e = std::getenv("PARL_HEAD_RECOMPUTE")) c->head_recompute = std::atoi(e) != 0;
        PARL_REQUIRE(c->recompute >= 0 && c->recompute <= 2, PARL_E_CONFIG, "PARL_RECOMPUTE must be 0, 1 or 2");
        *out = c.release();
    });
}


parl_status parl_ctx_destroy(parl_ctx_t ctx) {
    if (!ctx) return PARL_OK;
    ctx->closing = true;
    ctx->refs++;
    ctx_release(ctx);
    return PARL_OK;
}

parl_status parl_ctx_sync(parl_ctx_t ctx) {
    return guarded(ctx, [&] { PARL_CUDA(cudaStreamSynchronize(ctx->st)); });
}

void* parl_ctx_stream(parl_ctx_t ctx) { return ctx ? (void*)ctx->st : nullptr; }

parl_status parl_ctx_profile(parl_ctx_t ctx, int enable) {
    return guarded(ctx, [&] {
        ctx->prof_collect();
        ctx->prof_on = enable != 0;
    });
}

parl_status parl_ctx_profile_read(parl_ctx_t ctx, int cls, double* ms, double* work, long* n) {
    return guarded(ctx, [&] {
        PARL_REQUIRE(cls >= 0 && cls < PARL_KC_COUNT, PARL_E_CONFIG, "unknown kernel class");
        ctx->prof_collect();
        if (ms) *ms = ctx->prof_ms[cls];
        if (work) *work = ctx->prof_work[cls];
        if (n) *n = ctx->prof_n[cls];
        ctx->prof_ms[cls] = ctx->prof_work[cls] = 0;
        ctx->prof_n[cls] = 0;
    });
}
uint64_t parl_ctx_launches(parl_ctx_t) { return g_launches; }

size_t parl_param_count(const parl_config* cfg) { return make_layout(*cfg).total; }

parl_status parl_model_create(parl_ctx_t ctx, const parl_config* cfg, parl_model_t* out) {
    return guarded(ctx, [&] {
        validate_config(*cfg);
        if (ctx->prec == PARL_PREC_BF16) {  // shapes the tcgen05 kernels take (no SIMT fallback in bf16)
            const int dh = cfg->d_model / cfg->n_heads;
            PARL_REQUIRE(dh == 64 || dh == 128, PARL_E_CONFIG,
                         "bf16 path needs head dim 64 or 128, got " + std::to_string(dh));
            PARL_REQUIRE(cfg->d_model % 8 == 0 && cfg->d_ff % 8 == 0 && cfg->vocab_size % 8 == 0, PARL_E_CONFIG,
                         "bf16 path needs d_model, d_ff and vocab_size divisible by 8 (16-byte TMA rows)");
        }
        auto m = std::make_unique<parl_model_s>();
        m->ctx = ctx;
        ctx->refs++;
        m->cfg = *cfg;
        m->L = make_layout(*cfg);
        const size_t d = cfg->d_model, F = cfg->d_ff, V = cfg->vocab_size, NL = cfg->n_layers;
        const size_t n32 = V * d + (size_t)cfg->max_seq_len * d + NL * (4 * d + 3 * d + d + F + d) + 2 * d + V;
        const size_t nact = NL * (3 * d * d + d * d + F * d + d * F) + V * d;
        float* f = m->f32.as<float>(n32);
        char* a = static_cast<char*>(m->act.get(std::max<size_t>(nact, 1) * act_size(ctx->prec)));
        const size_t es = act_size(ctx->prec);
        auto takef = [&](size_t n) { float* p = f; f += n; return p; };
        auto takea = [&](size_t n) { void* p = a; a += n * es; return p; };
        m->W.tok_emb = takef(V * d);
        m->W.pos_emb = takef((size_t)cfg->max_seq_len * d);
        m->layers.resize(NL);
        for (auto& w : m->layers) {
            w.ln1_g = takef(d); w.ln1_b = takef(d); w.ln2_g = takef(d); w.ln2_b = takef(d);
            w.bqkv = takef(3 * d); w.bo = takef(d); w.b1 = takef(F); w.b2 = takef(d);
            w.wqkv_t = takea(3 * d * d); w.wo_t = takea(d * d); w.w1_t = takea(F * d); w.w2_t = takea(d * F);
        }
        m->W.lnf_g = takef(d);
        m->W.lnf_b = takef(d);
        m->W.head_b = takef(V);
        m->W.head_w_t = takea(V * d);
        m->W.layers = m->layers.data();
        // fp64 master copy (apply_update / snapshots) when it fits comfortably
        m->has_master = m->L.total * sizeof(double) <= (size_t)24 << 30;
        if (m->has_master) m->master.as<double>(m->L.total);
        *out = m.release();
    });
}

parl_status parl_model_destroy(parl_model_t m) {
    if (m) {
        parl_ctx_s* c = m->ctx;
        {
            std::lock_guard<std::recursive_mutex> lk(c->mu);
            cudaStreamSynchronize(c->st);
            delete m;
        }
        ctx_release(c);
    }
    return PARL_OK;
}

uint64_t parl_model_version(parl_model_t m) { return m->version; }
uint64_t parl_model_init_seed(parl_model_t m) { return m->init_seed; }
uint64_t parl_model_epoch(parl_model_t m) { return m->epoch; }
uint64_t parl_model_forward_gen(parl_model_t m) { return m->forward_gen; }
parl_status parl_model_set_init_seed(parl_model_t m, uint64_t seed) {
    return guarded(m->ctx, [&] { m->init_seed = seed; });
}

parl_status parl_model_all_finite(parl_model_t m, int* out) {
    return guarded(m->ctx, [&] {
        PARL_REQUIRE(m->has_master, PARL_E_CONFIG, "all_finite needs the fp64 master copy");
        cudaStream_t st = m->ctx->st;
        int* flags = m->ctx->flags.as<int>(1);
        PARL_CUDA(cudaMemsetAsync(flags, 0, 4, st));
        launch_finite_check_f64(static_cast<const double*>(m->master.p), (long)m->L.total, flags, st);
        int h = 0;
        PARL_CUDA(cudaMemcpyAsync(&h, flags, 4, cudaMemcpyDeviceToHost, st));
        PARL_CUDA(cudaStreamSynchronize(st));
        *out = h == 0;
    });
}

parl_status parl_model_upload(parl_model_t m, const double* flat, size_t n, uint64_t version) {
    return guarded(m->ctx, [&] {
        PARL_REQUIRE(n == m->L.total, PARL_E_SHAPE, "weight array size does not match the model layout");
        cudaStream_t st = m->ctx->st;
        if (m->has_master) {
            PARL_CUDA(cudaMemcpyAsync(m->master.p, flat, n * sizeof(double), cudaMemcpyHostToDevice, st));
            convert_from_master(m);
        } else {
            for (const auto& t : tensor_maps(m)) {
                const size_t cnt = (size_t)t.rows * t.cols;
                double* stg = m->ctx->staging.as<double>(cnt);
                PARL_CUDA(cudaMemcpyAsync(stg, flat + t.src_off, cnt * sizeof(double), cudaMemcpyHostToDevice, st));
                convert_tensor(m, t, stg);
            }
        }
        PARL_CUDA(cudaStreamSynchronize(st));
        m->version = version;
        ++m->epoch;
    });
}

parl_status parl_model_init(parl_model_t m, uint64_t seed) {
    // ModelParams::init (model.cpp:142-164) with the reference RNG
    // (rng.hpp: splitmix64-whitened std::mt19937_64, Box-Muller normals).
    std::vector<double> w;
    parl_status s = guarded(m->ctx, [&] {
        auto sm64 = [](uint64_t x) {
            x += 0x9e3779b97f4a7c15ull;
            x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
            x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
            return x ^ (x >> 31);
        };
        const uint64_t mixed = sm64(sm64(seed) ^ (0x9e3779b97f4a7c15ull + 0x6d6f64656cull));
        std::mt19937_64 eng(sm64(mixed));
        bool has_spare = false;
        double spare = 0.0;
        auto normal = [&]() {
            if (has_spare) {
                has_spare = false;
                return spare;
            }
            const double u1 = 1.0 - (double)(eng() >> 11) * 0x1.0p-53;
            const double u2 = (double)(eng() >> 11) * 0x1.0p-53;
            const double r = std::sqrt(-2.0 * std::log(u1)), a = 6.283185307179586476925286766559 * u2;
            spare = r * std::sin(a);
            has_spare = true;
            return r * std::cos(a);
        };
        w.assign(m->L.total, 0.0);
        for (const auto& t : tensor_maps(m)) {
            double* dst = w.data() + t.src_off;
            const size_t cnt = (size_t)t.rows * t.cols;
            if (t.kind == 1) std::fill(dst, dst + cnt, 1.0);
            else if (t.kind == 0)
                for (size_t i = 0; i < cnt; ++i) dst[i] = 0.08 * normal();
        }
    });
    if (s != PARL_OK) return s;
    // tensor_maps lists tensors in layout order, so draws follow model.cpp:153-162
    m->init_seed = seed;
    return parl_model_upload(m, w.data(), w.size(), 0);
}

parl_status parl_model_init_device(parl_model_t m, uint64_t seed, double scale) {
    return guarded(m->ctx, [&] {
        cudaStream_t st = m->ctx->st;
        uint32_t stream = 0;
        for (const auto& t : tensor_maps(m)) {
            const size_t cnt = (size_t)t.rows * t.cols;
            double* dst = m->has_master ? static_cast<double*>(m->master.p) + t.src_off
                                        : m->ctx->staging.as<double>(cnt);
            if (t.kind == 0) launch_randn(dst, (long)cnt, seed, stream++, scale, nullptr, st);
            else launch_fill_f64(dst, (long)cnt, t.kind == 1 ? 1.0 : 0.0, st);
            if (!m->has_master) convert_tensor(m, t, dst);
        }
        if (m->has_master) convert_from_master(m);
        check_launch();
        PARL_CUDA(cudaStreamSynchronize(st));
        m->version = 0;
        m->init_seed = seed;
        ++m->epoch;
    });
}

parl_status parl_model_copy(parl_model_t dst, parl_model_t src, uint64_t seed, double scale) {
    return guarded(dst->ctx, [&] {
        PARL_REQUIRE(same_cfg(dst->cfg, src->cfg), PARL_E_SHAPE, "model copy between different configs");
        cudaStream_t st = dst->ctx->st;
        if (src->has_master && dst->has_master) {
            if (scale != 0.0)
                launch_randn(static_cast<double*>(dst->master.p), (long)dst->L.total, seed, 0xC0FFEEu, scale,
                             static_cast<const double*>(src->master.p), st);
            else
                PARL_CUDA(cudaMemcpyAsync(dst->master.p, src->master.p, dst->L.total * sizeof(double),
                                          cudaMemcpyDeviceToDevice, st));
            convert_from_master(dst);
        } else if (scale != 0.0) {
            // no fp64 master (large models): perturb tensor by tensor through the fp64 staging
            // buffer, from the source's compute copy
            const auto ts = tensor_maps(src), td = tensor_maps(dst);
            uint32_t stream = 0xC0FFEEu;
            for (size_t i = 0; i < ts.size(); ++i) {
                const auto& t = ts[i];
                const size_t cnt = (size_t)t.rows * t.cols;
                double* stg = dst->ctx->staging.as<double>(cnt);
                export_tensor(src, t, stg, st);
                launch_randn(stg, (long)cnt, seed, stream++, scale, stg, st);
                convert_tensor(dst, td[i], stg);
            }
            check_launch();
        } else {
            PARL_CUDA(cudaMemcpyAsync(dst->f32.p, src->f32.p, src->f32.bytes, cudaMemcpyDeviceToDevice, st));
            PARL_CUDA(cudaMemcpyAsync(dst->act.p, src->act.p, src->act.bytes, cudaMemcpyDeviceToDevice, st));
        }
        PARL_CUDA(cudaStreamSynchronize(st));
        dst->version = src->version;
        dst->init_seed = src->init_seed;  // ModelParams::clone keeps init_seed_ (model.cpp:172-181)
        ++dst->epoch;
    });
}

parl_status parl_model_download(parl_model_t m, double* flat, size_t n) {
    return guarded(m->ctx, [&] {
        PARL_REQUIRE(n == m->L.total, PARL_E_SHAPE, "weight array size does not match the model layout");
        cudaStream_t st = m->ctx->st;
        if (m->has_master) {
            PARL_CUDA(cudaMemcpyAsync(flat, m->master.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
        } else {
            for (const auto& t : tensor_maps(m)) {
                const size_t cnt = (size_t)t.rows * t.cols;
                double* stg = m->ctx->staging.as<double>(cnt);
                export_tensor(m, t, stg, st);
                PARL_CUDA(cudaMemcpyAsync(flat + t.src_off, stg, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
                PARL_CUDA(cudaStreamSynchronize(st));
            }
        }
        PARL_CUDA(cudaStreamSynchronize(st));
    });
}

// ---- checkpoints: PARLCKP1 (save_checkpoint / load_checkpoint, model.cpp:907-987) --------
// magic "PARLCKP1"; u32 vocab, d_model, n_layers, n_heads, d_ff, max_seq_len; u64 version,
// init_seed; u32 n_tensors; per tensor in layout order: u32 name length, name bytes,
// u32 rows, u32 cols, rows * cols f64 (the reference flat layout, model.cpp:86-114).
extern "C++" {
namespace {
constexpr char kCkptMagic[8] = {'P', 'A', 'R', 'L', 'C', 'K', 'P', '1'};

std::vector<std::string> tensor_names(const parl_config& c) {  // build_layout, model.cpp:86-114
    std::vector<std::string> v = {"tok_emb", "pos_emb"};
    static const char* per_layer[] = {"ln1.gamma", "ln1.beta", "attn.wq", "attn.bq", "attn.wk", "attn.bk",
                                      "attn.wv",   "attn.bv",  "attn.wo", "attn.bo", "ln2.gamma", "ln2.beta",
                                      "ffn.w1",    "ffn.b1",   "ffn.w2",  "ffn.b2"};
    for (int l = 0; l < c.n_layers; ++l)
        for (const char* n : per_layer) v.push_back("layers." + std::to_string(l) + "." + n);
    for (const char* n : {"ln_f.gamma", "ln_f.beta", "head.w", "head.b"}) v.push_back(n);
    return v;
}

template <class T>
void put(std::ostream& os, T v) {
    os.write(reinterpret_cast<const char*>(&v), sizeof(T));
}

template <class T>
T get(std::istream& is) {
    T v{};
    is.read(reinterpret_cast<char*>(&v), sizeof(T));
    PARL_REQUIRE(bool(is), PARL_E_IO, "checkpoint truncated");
    return v;
}
}  // namespace
}  // extern "C++"

parl_status parl_model_config(parl_model_t m, parl_config* out) {
    if (!m || !out) return PARL_E_CONFIG;
    *out = m->cfg;
    return PARL_OK;
}

parl_status parl_checkpoint_save(parl_model_t m, const char* path) {
    return guarded(m->ctx, [&] {
        std::ofstream os(path, std::ios::binary | std::ios::trunc);
        PARL_REQUIRE(bool(os), PARL_E_IO, std::string("cannot open checkpoint for writing: ") + path);
        os.write(kCkptMagic, sizeof(kCkptMagic));
        const auto& c = m->cfg;
        for (int v : {c.vocab_size, c.d_model, c.n_layers, c.n_heads, c.d_ff, c.max_seq_len}) put<uint32_t>(os, v);
        put<uint64_t>(os, m->version);
        put<uint64_t>(os, m->init_seed);
        const auto maps = tensor_maps(m);
        const auto names = tensor_names(c);
        put<uint32_t>(os, (uint32_t)maps.size());
        cudaStream_t st = m->ctx->st;
        std::vector<double> h;
        for (size_t i = 0; i < maps.size(); ++i) {
            const auto& t = maps[i];
            const size_t cnt = (size_t)t.rows * t.cols;
            h.resize(cnt);
            const double* src = m->has_master ? static_cast<const double*>(m->master.p) + t.src_off : nullptr;
            if (!src) {
                double* stg = m->ctx->staging.as<double>(cnt);
                export_tensor(m, t, stg, st);
                src = stg;
            }
            PARL_CUDA(cudaMemcpyAsync(h.data(), src, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
            PARL_CUDA(cudaStreamSynchronize(st));
            put<uint32_t>(os, (uint32_t)names[i].size());
            os.write(names[i].data(), (std::streamsize)names[i].size());
            put<uint32_t>(os, (uint32_t)t.rows);
            put<uint32_t>(os, (uint32_t)t.cols);
            os.write(reinterpret_cast<const char*>(h.data()), (std::streamsize)(cnt * sizeof(double)));
        }
        PARL_REQUIRE(bool(os), PARL_E_IO, std::string("write failed: ") + path);
    });
}

parl_status parl_checkpoint_load(parl_ctx_t ctx, const char* path, parl_model_t* out) {
    parl_model_t m = nullptr;
    const parl_status s = guarded(ctx, [&] {
        std::ifstream is(path, std::ios::binary);
        PARL_REQUIRE(bool(is), PARL_E_IO, std::string("cannot open checkpoint: ") + path);
        char magic[8];
        is.read(magic, sizeof(magic));
        PARL_REQUIRE(is && std::memcmp(magic, kCkptMagic, sizeof(magic)) == 0, PARL_E_IO,
                     std::string("bad checkpoint magic in ") + path);
        parl_config c{};
        c.vocab_size = (int)get<uint32_t>(is);
        c.d_model = (int)get<uint32_t>(is);
        c.n_layers = (int)get<uint32_t>(is);
        c.n_heads = (int)get<uint32_t>(is);
        c.d_ff = (int)get<uint32_t>(is);
        c.max_seq_len = (int)get<uint32_t>(is);
        const uint64_t version = get<uint64_t>(is), seed = get<uint64_t>(is);
        const uint32_t n_tensors = get<uint32_t>(is);
        const parl_status cs = parl_model_create(ctx, &c, &m);  // ConfigError on a bad header
        if (cs != PARL_OK) throw Error{cs, ctx->err};
        const auto maps = tensor_maps(m);
        const auto names = tensor_names(c);
        PARL_REQUIRE(n_tensors == maps.size(), PARL_E_IO, std::string("checkpoint tensor count mismatch in ") + path);
        cudaStream_t st = ctx->st;
        std::vector<double> h;
        for (size_t i = 0; i < maps.size(); ++i) {
            const auto& t = maps[i];
            const uint32_t nl = get<uint32_t>(is);
            std::string name(nl, '\0');
            is.read(name.data(), nl);
            const uint32_t rows = get<uint32_t>(is), cols = get<uint32_t>(is);
            PARL_REQUIRE(is && name == names[i] && rows == (uint32_t)t.rows && cols == (uint32_t)t.cols, PARL_E_IO,
                         "checkpoint tensor '" + name + "' does not match expected layout");
            const size_t cnt = (size_t)rows * cols;
            h.resize(cnt);
            is.read(reinterpret_cast<char*>(h.data()), (std::streamsize)(cnt * sizeof(double)));
            PARL_REQUIRE(bool(is), PARL_E_IO, "checkpoint truncated in tensor " + name);
            for (double v : h)
                PARL_REQUIRE(std::isfinite(v), PARL_E_NUMERIC,
                             std::string("checkpoint contains non-finite values: ") + path);
            double* dst = m->has_master ? static_cast<double*>(m->master.p) + t.src_off
                                        : ctx->staging.as<double>(cnt);
            PARL_CUDA(cudaMemcpyAsync(dst, h.data(), cnt * sizeof(double), cudaMemcpyHostToDevice, st));
            if (!m->has_master) convert_tensor(m, t, dst);
            PARL_CUDA(cudaStreamSynchronize(st));  // h is reused
        }
        if (m->has_master) convert_from_master(m);
        check_launch();
        PARL_CUDA(cudaStreamSynchronize(st));
        m->version = version;
        m->init_seed = seed;
    });
    if (s != PARL_OK) {
        if (m) parl_model_destroy(m);
        return s;
    }
    *out = m;
    return PARL_OK;
}

// ---- groups -----------------------------------------------------------------
parl_status parl_group_create(parl_ctx_t ctx, int max_tokens, int max_responses, parl_group_t* out) {
    return guarded(ctx, [&] {
        PARL_REQUIRE(max_tokens > 0 && max_responses > 0, PARL_E_CONFIG, "group capacity must be positive");
        auto g = std::make_unique<parl_group_s>();
        g->ctx = ctx;
        ctx->refs++;
        g->max_T = max_tokens;
        g->max_G = max_responses;
        alloc_group_arrays(g.get());
        *out = g.release();
    });
}

parl_status parl_group_destroy(parl_group_t g) {
    if (g) {
        parl_ctx_s* c = g->ctx;
        {
            std::lock_guard<std::recursive_mutex> lk(c->mu);
            cudaStreamSynchronize(c->st);
            delete g;
        }
        ctx_release(c);
    }
    return PARL_OK;
}

int parl_group_tokens(parl_group_t g) { return g->T; }
int parl_group_scored(parl_group_t g) { return g->S; }

parl_status parl_pack(parl_group_t g, const int32_t* prompt, int P, const int32_t* resp_flat, const int32_t* lens,
                      int G, int max_seq) {
    return guarded(g->ctx, [&] {
        check_pack_inputs(g, P, lens, G, max_seq);
        set_pack_meta(g, P, lens, G, max_seq);
        unsigned umax = 0;  // (unsigned)id >= V <=> id outside [0, V)
        for (int i = 0; i < P; ++i) umax = std::max(umax, (unsigned)prompt[i]);
        for (int i = 0; i < g->S; ++i) umax = std::max(umax, (unsigned)resp_flat[i]);
        g->tok_max = (int)std::min<unsigned>(umax, INT32_MAX);
        g->tok_range_dev = false;
        cudaStream_t st = g->ctx->st;
        int32_t* dp = g->in_prompt.as<int32_t>(g->max_T);
        int32_t* dr = g->in_resp.as<int32_t>(g->max_T);
        g->in_flip ^= 1;
        g->in_stage[g->in_flip].upload2(dp, prompt, (size_t)P * 4, dr, resp_flat, (size_t)g->S * 4, st);
        upload_meta(g);
        ProfScope ps(g->ctx, PARL_KC_PACK, 24.0 * g->T + 24.0 * g->S);
        launch_pack(dp, P, dr, group_cu(g), G, g->T, g->pk, nullptr, st);
        check_launch();
    });
}

// ---- several prompt groups per packed sequence (f4) -------------------------------
namespace {
// validate each group as pack_group does (packing.cpp:7-19; positions restart per group, so
// max_seq_len bounds every group's own packed length), then set the host meta and return the
// K1 tables gstart [n+1] | pstart [n] | r0 [n+1] | rcu [R+1] | rstart [R]
std::vector<int32_t> set_multi_meta(parl_group_s* g, const int32_t* prompt_lens, const int32_t* resp_lens,
                                    const int32_t* group_sizes, int n, int max_seq) {
    PARL_REQUIRE(n >= 1, PARL_E_SHAPE, "pack: no prompt groups");
    long T = 0;
    int R = 0, uniform = group_sizes[0];
    for (int q = 0; q < n; ++q) {
        const int P = prompt_lens[q], G = group_sizes[q];
        PARL_REQUIRE(P >= 1, PARL_E_SHAPE, "pack_group: empty prompt");
        PARL_REQUIRE(G >= 1, PARL_E_SHAPE, "pack_group: no responses");
        long tg = P;
        for (int k = 0; k < G; ++k) {
            PARL_REQUIRE(resp_lens[R + k] >= 1, PARL_E_SHAPE, "pack_group: empty response");
            tg += resp_lens[R + k];
        }
        PARL_REQUIRE(tg <= max_seq, PARL_E_SHAPE,
                     "pack_group: packed length " + std::to_string(tg) + " for group of " + std::to_string(G) +
                         " responses exceeds max_seq_len " + std::to_string(max_seq));
        T += tg;
        R += G;
        if (G != uniform) uniform = 0;
    }
    PARL_REQUIRE(T <= g->max_T && R <= g->max_G, PARL_E_SHAPE,
                 "packed groups exceed the capacity this group was created with");
    std::vector<int32_t> gstart(n + 1), pstart(n), r0(n + 1), rcu(R + 1), rstart(R);
    g->segs.clear();
    g->lens.assign(resp_lens, resp_lens + R);
    g->span_start.assign(R, 0);
    int t = 0, po = 0, k = 0;
    rcu[0] = 0;
    for (int q = 0; q < n; ++q) {
        gstart[q] = t;
        pstart[q] = po;
        r0[q] = k;
        g->segs.add_group(t, prompt_lens[q], resp_lens + k, group_sizes[q]);
        t += prompt_lens[q];
        po += prompt_lens[q];
        for (int j = 0; j < group_sizes[q]; ++j, ++k) {
            rstart[k] = t;
            g->span_start[k] = t;
            rcu[k + 1] = rcu[k] + resp_lens[k];
            t += resp_lens[k];
        }
    }
    gstart[n] = t;
    r0[n] = R;
    g->T = t;
    g->S = rcu[R];
    g->P = prompt_lens[0];
    g->G = R;
    g->n_samples = R;
    g->n_groups = n;
    g->group_G = uniform;
    g->Peff = n == 1 ? prompt_lens[0] : 0;
    g->cu.assign(rcu.begin(), rcu.end());
    g->pairs = g->segs.pairs();
    g->max_seq = max_seq;
    g->epoch++;
    std::vector<int32_t> tab;
    for (const auto* v : {&gstart, &pstart, &r0, &rcu, &rstart}) tab.insert(tab.end(), v->begin(), v->end());
    return tab;
}

void pack_multi_launch(parl_group_s* g, const int32_t* d_prompts, const int32_t* d_resp, const std::vector<int32_t>& tab,
                       unsigned* id_max) {
    upload_meta(g);
    int32_t* d_tab = g->multi_tab.as<int32_t>(tab.size());
    g->multi_stage.upload(d_tab, tab.data(), tab.size() * 4, g->ctx->st);
    ProfScope ps(g->ctx, PARL_KC_PACK, 28.0 * g->T + 20.0 * g->S);
    launch_pack_multi(d_prompts, d_resp, d_tab, g->n_groups, g->G, g->T, g->pk, id_max, g->ctx->st);
    check_launch();
}
}  // namespace

parl_status parl_pack_multi(parl_group_t g, const int32_t* prompts, const int32_t* prompt_lens,
                            const int32_t* resp_flat, const int32_t* resp_lens, const int32_t* group_sizes, int n,
                            int max_seq) {
    return guarded(g->ctx, [&] {
        auto tab = set_multi_meta(g, prompt_lens, resp_lens, group_sizes, n, max_seq);
        long np = 0;
        for (int q = 0; q < n; ++q) np += prompt_lens[q];
        unsigned umax = 0;
        for (long i = 0; i < np; ++i) umax = std::max(umax, (unsigned)prompts[i]);
        for (long i = 0; i < g->S; ++i) umax = std::max(umax, (unsigned)resp_flat[i]);
        g->tok_max = (int)std::min<unsigned>(umax, INT32_MAX);
        g->tok_range_dev = false;
        cudaStream_t st = g->ctx->st;
        int32_t* dp = g->multi_prompts.as<int32_t>(np);
        int32_t* dr = g->multi_resp.as<int32_t>(g->S);
        g->in_flip ^= 1;
        g->in_stage[g->in_flip].upload2(dp, prompts, (size_t)np * 4, dr, resp_flat, (size_t)g->S * 4, st);
        pack_multi_launch(g, dp, dr, tab, nullptr);
    });
}

parl_status parl_pack_multi_device(parl_group_t g, const int32_t* d_prompts, const int32_t* prompt_lens,
                                   const int32_t* d_resp, const int32_t* resp_lens, const int32_t* group_sizes, int n,
                                   int max_seq) {
    return guarded(g->ctx, [&] {
        auto tab = set_multi_meta(g, prompt_lens, resp_lens, group_sizes, n, max_seq);
        pack_multi_launch(g, d_prompts, d_resp, tab, g->tok_range.as<unsigned>(1));
        g->tok_range_dev = true;
    });
}

parl_status parl_pack_device(parl_group_t g, const int32_t* d_prompt, int P, const int32_t* d_resp,
                             const int32_t* lens, int G, int max_seq) {
    return guarded(g->ctx, [&] {
        check_pack_inputs(g, P, lens, G, max_seq);
        set_pack_meta(g, P, lens, G, max_seq);
        upload_meta(g);
        ProfScope ps(g->ctx, PARL_KC_PACK, 24.0 * g->T + 24.0 * g->S);
        launch_pack(d_prompt, P, d_resp, group_cu(g), G, g->T, g->pk, g->tok_range.as<unsigned>(1), g->ctx->st);
        g->tok_range_dev = true;  // read (once) by the first forward over this packing
        check_launch();
    });
}

parl_status parl_set_sequence(parl_group_t g, const int32_t* tokens, const int32_t* positions, const int32_t* labels,
                              int T, int prompt_len, const int32_t* resp_lens, int G, int vocab, int max_seq) {
    return guarded(g->ctx, [&] {
        // validate_forward_inputs (model.cpp:404-426), same order
        PARL_REQUIRE(T > 0, PARL_E_SHAPE, "empty token sequence");
        PARL_REQUIRE(T <= max_seq, PARL_E_SHAPE,
                     "sequence length " + std::to_string(T) + " exceeds max_seq_len " + std::to_string(max_seq));
        for (int t = 0; t < T; ++t)
            PARL_REQUIRE(tokens[t] >= 0 && tokens[t] < vocab, PARL_E_VOCAB,
                         "token id " + std::to_string(tokens[t]) + " outside vocab of size " + std::to_string(vocab));
        g->tok_max = 0;
        for (int t = 0; t < T; ++t) g->tok_max = std::max(g->tok_max, (int)tokens[t]);
        g->tok_range_dev = false;
        for (int t = 0; t < T; ++t)
            PARL_REQUIRE(positions[t] >= 0 && positions[t] < max_seq, PARL_E_SHAPE,
                         "position id " + std::to_string(positions[t]) + " outside [0, max_seq_len)");
        if (labels)
            for (int t = 0; t < T; ++t)
                PARL_REQUIRE(labels[t] == -1 || (labels[t] >= 0 && labels[t] < vocab), PARL_E_VOCAB,
                             "label id " + std::to_string(labels[t]) + " outside vocab");
        if (prompt_len > 0) {  // AttentionMaskSpec::validate (model.cpp:53-61)
            PARL_REQUIRE(G >= 1, PARL_E_SHAPE, "shared_prompt mask needs >= 1 response");
            long tot = prompt_len;
            for (int k = 0; k < G; ++k) {
                PARL_REQUIRE(resp_lens[k] >= 1, PARL_E_SHAPE, "shared_prompt mask response lengths must be >= 1");
                tot += resp_lens[k];
            }
            PARL_REQUIRE(tot == T, PARL_E_SHAPE, "mask total length does not match sequence length");
        }
        PARL_REQUIRE(T <= g->max_T && G <= g->max_G, PARL_E_SHAPE, "sequence exceeds the group capacity");
        const int Peff = prompt_len > 0 ? prompt_len : T;
        std::vector<int32_t> seg(T, 0), pred(T), sp, sl, pp, so, rp(T + 1, 0), ri;
        g->lens.clear();
        g->span_start.clear();
        if (prompt_len > 0) {
            int t = prompt_len;
            for (int k = 0; k < G; ++k) {
                g->span_start.push_back(t);
                g->lens.push_back(resp_lens[k]);
                for (int i = 0; i < resp_lens[k]; ++i) seg[t++] = k + 1;
            }
        }
        for (int t = 0; t < T; ++t)
            pred[t] = (prompt_len > 0 && seg[t] != 0 && seg[t - 1] != seg[t]) ? prompt_len - 1 : t - 1;
        std::vector<int> nsample(std::max(G, 1), 0);
        if (labels)
            for (int t = 0; t < T; ++t) {
                if (labels[t] == -1) continue;
                PARL_REQUIRE(pred[t] >= 0, PARL_E_SHAPE, "position 0 has no predecessor to score its label from");
                sp.push_back(t);
                sl.push_back(labels[t]);
                pp.push_back(pred[t]);
                const int k = seg[t] > 0 ? seg[t] - 1 : 0;
                so.push_back(k);
                nsample[k]++;
            }
        const int S = (int)sp.size();
        // position -> gathered rows CSR (rows listed in scored order)
        std::vector<std::vector<int>> owned(T);
        for (int s = 0; s < S; ++s) owned[pp[s]].push_back(s);
        for (int t = 0; t < T; ++t) {
            rp[t + 1] = rp[t] + (int)owned[t].size();
            for (int s : owned[t]) ri.push_back(s);
        }
        g->T = T;
        g->P = prompt_len;
        g->G = prompt_len > 0 ? G : 0;
        g->segs.clear();
        g->segs.add_group(0, Peff, prompt_len > 0 ? resp_lens : nullptr, g->G);
        g->pairs = g->segs.pairs();
        g->n_groups = 1;
        g->group_G = std::max(g->G, 1);
        g->S = S;
        g->Peff = Peff;
        g->n_samples = std::max(G, 1);
        g->cu.assign(g->n_samples + 1, 0);
        for (int k = 0; k < g->n_samples; ++k) g->cu[k + 1] = g->cu[k] + nsample[k];
        g->max_seq = max_seq;
        g->vocab = vocab;
        g->epoch++;
        cudaStream_t st = g->ctx->st;
        auto up = [&](int32_t* dst, const void* src, size_t n) {
            if (n) PARL_CUDA(cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyHostToDevice, st));
        };
        up(g->pk.tokens, tokens, T);
        up(g->pk.positions, positions, T);
        if (labels) up(g->pk.labels, labels, T);
        up(g->pk.seg, seg.data(), T);
        up(g->pk.pred, pred.data(), T);
        up(g->pk.scored_pos, sp.data(), S);
        up(g->pk.scored_label, sl.data(), S);
        up(g->pk.pred_pos, pp.data(), S);
        up(g->pk.sample_of, so.data(), S);
        up(g->pk.row_ptr, rp.data(), T + 1);
        up(g->pk.row_idx, ri.data(), S);
        upload_meta(g);
        PARL_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope
    });
}

parl_status parl_group_download(parl_group_t g, int32_t* tokens, int32_t* labels, int32_t* positions, int32_t* seg,
                                int32_t* pred, int32_t* span_start, int32_t* scored_pos) {
    return guarded(g->ctx, [&] {
        cudaStream_t st = g->ctx->st;
        auto dn = [&](void* dst, const int32_t* src, size_t n) {
            if (dst && n) PARL_CUDA(cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyDeviceToHost, st));
        };
        dn(tokens, g->pk.tokens, g->T);
        dn(labels, g->pk.labels, g->T);
        dn(positions, g->pk.positions, g->T);
        dn(seg, g->pk.seg, g->T);
        dn(pred, g->pk.pred, g->T);
        dn(scored_pos, g->pk.scored_pos, g->S);
        PARL_CUDA(cudaStreamSynchronize(st));
        if (span_start) std::copy(g->span_start.begin(), g->span_start.end(), span_start);
    });
}

// ---- forward ------------------------------------------------------------------
// forwards of nm models over one group (model k -> log-prob slot slots[k]); the
// first model's activations go to *act_out when given
static void do_forward_n(parl_ctx_s* c, parl_model_s* const* ms, const int* slots, int nm, parl_group_s* g,
                         parl_act_t* act_out) {
    PARL_REQUIRE(g->T > 0, PARL_E_SHAPE, "group is empty (pack or set a sequence first)");
    for (int k = 0; k < nm; ++k) {
        PARL_REQUIRE(slots[k] >= 0 && slots[k] < 3, PARL_E_CONFIG, "slot must be 0, 1 or 2");
        // positions restart per prompt group: max_seq_len bounds each group's own length
        PARL_REQUIRE(g->segs.max_group_len() <= ms[k]->cfg.max_seq_len, PARL_E_SHAPE,
                     "sequence length exceeds max_seq_len");
        PARL_REQUIRE(same_cfg(ms[k]->cfg, ms[0]->cfg), PARL_E_CONFIG, "models of one forward must share a config");
    }
    g->vocab = ms[0]->cfg.vocab_size;
    if (g->tok_range_dev) {  // device-packed: K1's (unsigned) id maximum, read once per packing
        unsigned u = 0;
        PARL_CUDA(cudaMemcpyAsync(&u, g->tok_range.p, sizeof(u), cudaMemcpyDeviceToHost, c->st));
        PARL_CUDA(cudaStreamSynchronize(c->st));
        g->tok_max = (int)std::min<unsigned>(u, INT32_MAX);
        g->tok_range_dev = false;
    }
    // validate_forward_inputs (model.cpp:413-417): token (and self-aligned label) ids in [0, V)
    PARL_REQUIRE(g->tok_max < g->vocab, PARL_E_VOCAB,
                 "token id " + std::to_string(g->tok_max) + " outside vocab of size " + std::to_string(g->vocab));
    parl_act_s* act = nullptr;
    if (act_out) {
        act = *act_out ? *act_out : new parl_act_s();
        *act_out = act;
    }
    if (c->prec == PARL_PREC_BF16) forward_impl<bf16>(c, ms, slots, nm, g, act);
    else forward_impl<float>(c, ms, slots, nm, g, act);
    for (int k = 0; k < nm; ++k) {
        const uint64_t gen = ++ms[k]->forward_gen;  // bump_forward_generation, model.cpp:559
        if (k == 0 && act) {
            act->owner = ms[0];
            act->group = g;
            act->version = ms[0]->version;
            act->gen = gen;
            act->epoch = g->epoch;
            act->T = g->T;
            act->S = g->S;
        }
    }
}

static void do_forward(parl_ctx_s* c, parl_model_s* m, parl_group_s* g, int slot, parl_act_t* act_out) {
    do_forward_n(c, &m, &slot, 1, g, act_out);
}

parl_status parl_forward(parl_ctx_t ctx, parl_model_t m, parl_group_t g, int slot, parl_act_t* act_out) {
    return guarded(ctx, [&] { do_forward(ctx, m, g, slot, act_out); });
}

parl_status parl_trimodel_forward(parl_ctx_t ctx, parl_model_t pol, parl_model_t old, parl_model_t ref,
                                  parl_group_t g, parl_act_t* act_out) {
    return guarded(ctx, [&] {
        parl_model_s* ms[3] = {pol, old ? old : ref, ref};
        int slots[3] = {0, old ? 1 : 2, 2};
        do_forward_n(ctx, ms, slots, old ? 3 : 2, g, act_out);
    });
}

parl_status parl_group_logprobs(parl_group_t g, int slot, double* out) {
    return guarded(g->ctx, [&] {
        PARL_REQUIRE(slot >= 0 && slot < 3, PARL_E_CONFIG, "slot must be 0, 1 or 2");
        std::vector<float> h(g->S);
        if (g->S)
            PARL_CUDA(cudaMemcpyAsync(h.data(), group_lp(g, slot), g->S * 4,
                                      cudaMemcpyDeviceToHost, g->ctx->st));
        PARL_CUDA(cudaStreamSynchronize(g->ctx->st));
        for (int s = 0; s < g->S; ++s) out[s] = h[s];
    });
}

parl_status parl_group_set_logprobs(parl_group_t g, int slot, const double* in) {
    return guarded(g->ctx, [&] {
        PARL_REQUIRE(slot >= 0 && slot < 3, PARL_E_CONFIG, "slot must be 0, 1 or 2");
        for (int s = 0; s < g->S; ++s) PARL_REQUIRE(std::isfinite(in[s]), PARL_E_NUMERIC, "log-prob is not finite");
        std::vector<float> h(in, in + g->S);
        if (g->S)
            PARL_CUDA(cudaMemcpyAsync(group_lp(g, slot), h.data(), g->S * 4,
                                      cudaMemcpyHostToDevice, g->ctx->st));
        PARL_CUDA(cudaStreamSynchronize(g->ctx->st));
    });
}

parl_status parl_logprob_rows(parl_ctx_t ctx, parl_model_t m, parl_group_t g, double* rows) {
    // forward_logprob_rows: every position is a head row.
    return guarded(ctx, [&] {
        const int T = g->T, V = m->cfg.vocab_size;
        std::vector<int32_t> tok(T), pos(T);
        PARL_CUDA(cudaMemcpyAsync(tok.data(), g->pk.tokens, T * 4, cudaMemcpyDeviceToHost, ctx->st));
        PARL_CUDA(cudaMemcpyAsync(pos.data(), g->pk.positions, T * 4, cudaMemcpyDeviceToHost, ctx->st));
        PARL_CUDA(cudaStreamSynchronize(ctx->st));
        // rows: score label 0 at every position from the position itself
        std::vector<int32_t> lens(g->lens.begin(), g->lens.end());
        parl_group_s tmp;
        tmp.ctx = ctx;
        tmp.max_T = std::max(T, 1);
        tmp.max_G = std::max(g->max_G, 1);
        alloc_group_arrays(&tmp);
        // a T+1 long sequence would change attention; instead gather every row as a predecessor
        std::vector<int32_t> seg(T), pred(T), sp(T), sl(T, 0), pp(T), so(T, 0), rp(T + 1), ri(T);
        PARL_CUDA(cudaMemcpyAsync(seg.data(), g->pk.seg, T * 4, cudaMemcpyDeviceToHost, ctx->st));
        PARL_CUDA(cudaStreamSynchronize(ctx->st));
        for (int t = 0; t < T; ++t) {
            sp[t] = t; pp[t] = t; rp[t] = t; ri[t] = t;
        }
        rp[T] = T;
        tmp.T = T; tmp.P = g->P; tmp.G = g->G; tmp.S = T; tmp.Peff = g->Peff; tmp.n_samples = 1;
        tmp.lens = g->lens; tmp.span_start = g->span_start; tmp.cu = {0, T};
        tmp.segs = g->segs;
        tmp.vocab = V; tmp.max_seq = m->cfg.max_seq_len;
        auto up = [&](int32_t* dst, const void* src, size_t n) {
            PARL_CUDA(cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyHostToDevice, ctx->st));
        };
        up(tmp.pk.tokens, tok.data(), T);
        up(tmp.pk.positions, pos.data(), T);
        up(tmp.pk.seg, seg.data(), T);
        up(tmp.pk.scored_pos, sp.data(), T);
        up(tmp.pk.scored_label, sl.data(), T);
        up(tmp.pk.pred_pos, pp.data(), T);
        up(tmp.pk.row_ptr, rp.data(), T + 1);
        up(tmp.pk.row_idx, ri.data(), T);
        upload_meta(&tmp);
        int slot0 = 0;
        // every row's full distribution: the unfused head (fp32 logits + row log-sum-exp)
        if (ctx->prec == PARL_PREC_BF16) forward_impl<bf16>(ctx, &m, &slot0, 1, &tmp, nullptr, true);
        else forward_impl<float>(ctx, &m, &slot0, 1, &tmp, nullptr, true);
        ++m->forward_gen;
        std::vector<float> z((size_t)T * V), lse(T);
        PARL_CUDA(cudaMemcpyAsync(z.data(), ctx->scr[0].logits.p, z.size() * 4, cudaMemcpyDeviceToHost, ctx->st));
        PARL_CUDA(cudaMemcpyAsync(lse.data(), ctx->scr[0].lse_head.p, T * 4, cudaMemcpyDeviceToHost, ctx->st));
        PARL_CUDA(cudaStreamSynchronize(ctx->st));
        for (int t = 0; t < T; ++t)
            for (int v = 0; v < V; ++v)  // the LSE kernel's own rounding: lp = z - lse in fp32, so a row
                rows[(size_t)t * V + v] = (double)(z[(size_t)t * V + v] - lse[t]);  // entry == forward_logprobs
    });
}

parl_status parl_ctx_set_recompute(parl_ctx_t ctx, int mode) {
    return guarded(ctx, [&] {
        PARL_REQUIRE(mode >= 0 && mode <= 2, PARL_E_CONFIG, "recompute mode must be 0, 1 or 2");
        ctx->recompute = mode;
    });
}

int parl_act_recompute(parl_act_t a) { return a && a->recompute ? 1 : 0; }

// ---- rollout side: the KV-cached decoder ------------------------------------------------
// sample_tokens (model.cpp:843-900) for n sequences that share one prompt (the G rollouts of
// a group): the prompt runs once through the causal forward with every layer's K | V kept
// (prefill), then each step embeds the n newest tokens, runs every layer on those n rows
// (tensor-core GEMMs with M = n, decode attention over the shared prompt cache plus each
// sequence's own cache) and the LM head on n rows.  Token choice stays with the reference's
// own fp64 arithmetic and RNG stream per sequence (Rng(mix_seed(seed, "sample")), rng.hpp):
// greedy argmax (lowest id on ties) at temperature 0, else inverse-CDF sampling of
// softmax(logits / temperature); a sequence stops after kEosToken.  Optionally returns each
// sampled token's log-prob under the model (what score_logprobs recomputes, rollout.cpp:52-66).
extern "C++" {
namespace {
struct Sampler {
    std::mt19937_64 eng;
    explicit Sampler(uint64_t seed) {
        auto sm64 = [](uint64_t x) {
            x += 0x9e3779b97f4a7c15ull;
            x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
            x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
            return x ^ (x >> 31);
        };
        eng.seed(sm64(sm64(sm64(seed) ^ (0x9e3779b97f4a7c15ull + 0x73616d706c65ull))));
    }
    // model.cpp:868-893 on one fp32 logit row; *lp = log softmax(row)[chosen]
    int32_t choose(const float* row, int V, double temperature, std::vector<double>& w, double* lp) {
        int32_t chosen = 0;
        double maxv = row[0];
        for (int v = 1; v < V; ++v) maxv = std::max(maxv, (double)row[v]);
        if (temperature == 0.0) {
            double best = row[0];
            for (int v = 1; v < V; ++v)
                if ((double)row[v] > best) {  // strict: lowest id wins ties
                    best = row[v];
                    chosen = v;
                }
        } else {
            double z = 0.0;
            for (int v = 0; v < V; ++v) {
                w[v] = std::exp(((double)row[v] - maxv) / temperature);
                z += w[v];
            }
            const double target = (double)(eng() >> 11) * 0x1.0p-53 * z;
            double acc = 0.0;
            chosen = V - 1;
            for (int v = 0; v < V; ++v) {
                acc += w[v];
                if (target < acc) {
                    chosen = v;
                    break;
                }
            }
        }
        if (lp) {
            double s = 0.0;
            for (int v = 0; v < V; ++v) s += std::exp((double)row[v] - maxv);
            *lp = (double)row[chosen] - maxv - std::log(s);
        }
        return chosen;
    }
};

template <class T>
void sample_group_impl(parl_ctx_s* c, parl_model_s* m, const int32_t* prompt, int P, int n, int max_new,
                       double temperature, const uint64_t* seeds, int32_t* out, int* n_out, double* lp_out) {
    const auto& cf = m->cfg;
    const int V = cf.vocab_size, D = cf.d_model, F = cf.d_ff, H = cf.n_heads, NL = cf.n_layers;
    cudaStream_t st = c->st;
    for (int k = 0; k < n; ++k) n_out[k] = 0;
    if (max_new == 0) return;
    // prefill: the causal forward over the prompt, K | V of every layer kept, logits of row P - 1
    parl_group_s g;
    g.ctx = c;
    g.max_T = P;
    g.max_G = 1;
    alloc_group_arrays(&g);
    std::vector<int32_t> pos(P), zeros(P, 0);
    for (int t = 0; t < P; ++t) pos[t] = t;
    const int32_t last = P - 1;
    PARL_CUDA(cudaMemcpyAsync(g.pk.tokens, prompt, (size_t)P * 4, cudaMemcpyHostToDevice, st));
    PARL_CUDA(cudaMemcpyAsync(g.pk.positions, pos.data(), (size_t)P * 4, cudaMemcpyHostToDevice, st));
    PARL_CUDA(cudaMemcpyAsync(g.pk.seg, zeros.data(), (size_t)P * 4, cudaMemcpyHostToDevice, st));
    PARL_CUDA(cudaMemcpyAsync(g.pk.scored_label, zeros.data(), 4, cudaMemcpyHostToDevice, st));
    PARL_CUDA(cudaMemcpyAsync(g.pk.pred_pos, &last, 4, cudaMemcpyHostToDevice, st));
    g.T = P; g.P = P; g.G = 0; g.S = 1; g.Peff = P; g.n_samples = 1;
    g.cu = {0, 1};
    g.segs.add_group(0, P, nullptr, 0);
    g.pairs = g.segs.pairs();
    g.vocab = V; g.max_seq = cf.max_seq_len;
    ++g.epoch;
    upload_meta(&g);
    const size_t row2 = (size_t)2 * D;
    T* kvp = c->kv_prompt.as<T>((size_t)NL * P * row2);
    int slot = 0;
    forward_impl<T>(c, &m, &slot, 1, &g, nullptr, true, kvp);
    ++m->forward_gen;
    // decode state: n rows
    const long own_stride = (long)max_new * row2;  // per sequence, per layer
    T* kvo = c->kv_own.as<T>((size_t)NL * n * own_stride);
    float* x = c->dec_x.as<float>((size_t)n * D);
    float* x2 = c->dec_x2.as<float>((size_t)n * D);
    float* xm = c->dec_xm.as<float>((size_t)n * D);
    T* a = c->dec_a.as<T>((size_t)n * D);
    T* qkv = c->dec_qkv.as<T>((size_t)n * 3 * D);
    T* cx = c->dec_ctx.as<T>((size_t)n * D);
    T* act = c->dec_act.as<T>((size_t)n * F);
    float* stv = c->dec_st.as<float>((size_t)2 * n);
    float* logits = c->dec_logits.as<float>((size_t)n * V);
    int32_t* dtok = c->dec_tok.as<int32_t>((size_t)2 * n);
    std::vector<float> rows((size_t)n * V);
    PARL_CUDA(cudaMemcpyAsync(rows.data(), c->scr[0].logits.p, (size_t)V * 4, cudaMemcpyDeviceToHost, st));
    PARL_CUDA(cudaStreamSynchronize(st));
    for (int k = 1; k < n; ++k) std::copy(rows.begin(), rows.begin() + V, rows.begin() + (size_t)k * V);
    std::vector<Sampler> smp;
    for (int k = 0; k < n; ++k) smp.emplace_back(seeds[k]);
    std::vector<double> w(V);
    std::vector<char> done(n, 0);
    std::vector<int32_t> tok(n), tpos(n);
    const float scale = 1.0f / std::sqrt((float)(D / H));
    for (int step = 0;; ++step) {
        bool any = false;
        for (int k = 0; k < n; ++k) {
            if (done[k]) continue;
            double lp = 0.0;
            tok[k] = smp[k].choose(rows.data() + (size_t)k * V, V, temperature, w, lp_out ? &lp : nullptr);
            if (lp_out) lp_out[(size_t)k * max_new + step] = lp;
            out[(size_t)k * max_new + step] = tok[k];
            n_out[k] = step + 1;
            if (tok[k] == 2 || step + 1 == max_new) done[k] = 1;  // kEosToken (model.hpp:18)
            else any = true;
        }
        if (!any) break;
        // one decode step over the n newest tokens at position P + step
        for (int k = 0; k < n; ++k) tpos[k] = P + step;
        std::vector<int32_t> io(tok);
        io.insert(io.end(), tpos.begin(), tpos.end());
        PARL_CUDA(cudaMemcpyAsync(dtok, io.data(), io.size() * 4, cudaMemcpyHostToDevice, st));
        launch_embed(m->W.tok_emb, m->W.pos_emb, dtok, dtok + n, n, D, x, st);
        for (int l = 0; l < NL; ++l) {
            const LayerW& lw = m->layers[l];
            launch_layernorm<T>(x, nullptr, n, D, lw.ln1_g, lw.ln1_b, a, D, stv, stv + n, st);
            GemmArgs gq = mk(n, 3 * D, D, a, D, 1, lw.wqkv_t, D, 1);
            gq.epi = EPI_ACT; gq.bias = lw.bqkv; gq.Ca = qkv; gq.ldca = 3 * D;
            gemm<T>(c, gq);
            T* own = kvo + (size_t)l * n * own_stride;
            PARL_CUDA(cudaMemcpy2DAsync(own + (size_t)step * row2, own_stride * sizeof(T), qkv + D, 3 * D * sizeof(T),
                                        row2 * sizeof(T), n, cudaMemcpyDeviceToDevice, st));
            launch_decode_attn<T>(qkv, 3 * D, kvp + (size_t)l * P * row2, own, own_stride, P, step + 1, n, H, D, scale,
                                  cx, D, st);
            GemmArgs go = mk(n, D, D, cx, D, 1, lw.wo_t, D, 1);
            go.epi = EPI_RESID; go.bias = lw.bo; go.resid = x; go.Cf = xm; go.ldc = D;
            gemm<T>(c, go);
            launch_layernorm<T>(xm, nullptr, n, D, lw.ln2_g, lw.ln2_b, a, D, stv, stv + n, st);
            GemmArgs g1 = mk(n, F, D, a, D, 1, lw.w1_t, D, 1);
            g1.epi = EPI_GELU_ACT; g1.bias = lw.b1; g1.Ca = act; g1.ldca = F;
            gemm<T>(c, g1);
            GemmArgs g2 = mk(n, D, F, act, F, 1, lw.w2_t, F, 1);
            g2.epi = EPI_RESID; g2.bias = lw.b2; g2.resid = xm; g2.Cf = x2; g2.ldc = D;
            gemm<T>(c, g2);
            std::swap(x, x2);
        }
        launch_layernorm<T>(x, nullptr, n, D, m->W.lnf_g, m->W.lnf_b, a, D, stv, stv + n, st);
        GemmArgs gh = mk(n, V, D, a, D, 1, m->W.head_w_t, D, 1);
        gh.epi = EPI_F32; gh.bias = m->W.head_b; gh.Cf = logits; gh.ldc = V;
        gemm<T>(c, gh, PARL_KC_HEAD);
        check_launch();
        PARL_CUDA(cudaMemcpyAsync(rows.data(), logits, (size_t)n * V * 4, cudaMemcpyDeviceToHost, st));
        PARL_CUDA(cudaStreamSynchronize(st));
    }
    ++m->forward_gen;  // bump_forward_generation (model.cpp:865)
}

void check_sample_args(const parl_config& c, const int32_t* prompt, int P, int max_new, double temperature) {
    PARL_REQUIRE(P > 0, PARL_E_SHAPE, "empty prompt");
    PARL_REQUIRE(max_new >= 0, PARL_E_CONFIG, "max_new_tokens must be >= 0");
    PARL_REQUIRE(temperature >= 0.0, PARL_E_CONFIG, "temperature must be >= 0");
    PARL_REQUIRE(P + max_new <= c.max_seq_len, PARL_E_SHAPE, "prompt + max_new_tokens exceeds max_seq_len");
    for (int t = 0; t < P; ++t)
        PARL_REQUIRE(prompt[t] >= 0 && prompt[t] < c.vocab_size, PARL_E_VOCAB, "token id out of vocabulary");
}
}  // namespace
}  // extern "C++"

parl_status parl_sample_tokens(parl_ctx_t ctx, parl_model_t m, const int32_t* prompt, int P, int max_new_tokens,
                               double temperature, uint64_t rng_seed, int32_t* out, int* n_out) {
    return guarded(ctx, [&] {
        check_sample_args(m->cfg, prompt, P, max_new_tokens, temperature);
        if (ctx->prec == PARL_PREC_BF16)
            sample_group_impl<bf16>(ctx, m, prompt, P, 1, max_new_tokens, temperature, &rng_seed, out, n_out, nullptr);
        else
            sample_group_impl<float>(ctx, m, prompt, P, 1, max_new_tokens, temperature, &rng_seed, out, n_out, nullptr);
    });
}

parl_status parl_sample_group(parl_ctx_t ctx, parl_model_t m, const int32_t* prompt, int P, int n_seq,
                              int max_new_tokens, double temperature, const uint64_t* seeds, int32_t* out, int* n_out,
                              double* logprobs_out) {
    return guarded(ctx, [&] {
        check_sample_args(m->cfg, prompt, P, max_new_tokens, temperature);
        PARL_REQUIRE(n_seq >= 1, PARL_E_CONFIG, "n_seq must be >= 1");
        if (ctx->prec == PARL_PREC_BF16)
            sample_group_impl<bf16>(ctx, m, prompt, P, n_seq, max_new_tokens, temperature, seeds, out, n_out,
                                    logprobs_out);
        else
            sample_group_impl<float>(ctx, m, prompt, P, n_seq, max_new_tokens, temperature, seeds, out, n_out,
                                     logprobs_out);
    });
}

parl_status parl_act_destroy(parl_act_t a) {
    delete a;
    return PARL_OK;
}

// ---- loss ---------------------------------------------------------------------
parl_status parl_grpo_loss(parl_ctx_t ctx, parl_group_t g, const double* rewards, const double* advantages,
                           const parl_hyper* hp, parl_loss_stats* out) {
    return guarded(ctx, [&] {
        const int G = g->n_samples;
        PARL_REQUIRE(hp->epsilon > 0.0 && hp->epsilon < 1.0, PARL_E_CONFIG, "epsilon must be in (0, 1)");
        PARL_REQUIRE(hp->beta >= 0.0, PARL_E_CONFIG, "beta must be >= 0");
        PARL_REQUIRE(rewards || advantages, PARL_E_CONFIG, "grpo loss needs rewards or advantages");
        for (int k = 0; k < G; ++k)
            PARL_REQUIRE(g->cu[k + 1] > g->cu[k], PARL_E_SHAPE, "sample has empty response");
        cudaStream_t st = ctx->st;
        GrpoArgs a;
        a.lp = group_lp(g, 0);
        a.old = group_lp(g, 1);
        a.ref = group_lp(g, 2);
        a.sample_of = g->pk.sample_of;
        a.cu = group_cu(g);
        a.S = g->S;
        a.n = G;
        if (rewards) {  // group_advantages[_mean_only] over each group's rewards (grpo.cpp:24-48)
            const int gs = g->n_groups > 1 ? g->group_G : G;
            PARL_REQUIRE(gs > 0, PARL_E_CONFIG, "rewards need groups of equal size; pass advantages instead");
            PARL_REQUIRE(gs >= 2, PARL_E_CONFIG, "group_advantages needs G >= 2 rewards");
            double* r = g->rewards.as<double>(G);
            g->adv_stage.upload(r, rewards, G * sizeof(double), st);
            a.rewards = r;
            a.group_size = gs;
            a.mean_only = hp->advantage_mean_only;
        } else {
            for (int k = 0; k < G; ++k)  // per_sample_terms: require_finite(advantage), grpo.cpp:117
                PARL_REQUIRE(std::isfinite(advantages[k]), PARL_E_NUMERIC, "advantage is not finite");
            double* ad = g->rewards.as<double>(G);
            g->adv_stage.upload(ad, advantages, G * sizeof(double), st);
            a.adv_in = ad;
        }
        a.eps = hp->epsilon;
        a.beta = hp->beta;
        a.gran = hp->granularity;
        a.up_scale = -1.0;  // the pipeline backpropagates -d(L - beta KL)/d lp (pipeline.cpp:138)
        a.up_f32 = static_cast<float*>(g->upstream.p);
        a.adv_out = g->adv.as<double>(G);
        a.slots = ctx->grpo_slots.as<double>(grpo_slot_count(a.S, G));
        a.per_sample = ctx->per_sample.as<double>(4 * (size_t)G);
        a.g_seq = ctx->g_seq.as<double>(G);
        a.stats = ctx->stats.as<double>(8);
        {
            ProfScope ps(ctx, PARL_KC_LOSS, 20.0 * g->S + 16.0 * G);
            launch_grpo(a, st);
        }
        check_launch();
        if (out) {
            double h[5];
            PARL_CUDA(cudaMemcpyAsync(h, a.stats, 5 * sizeof(double), cudaMemcpyDeviceToHost, st));
            PARL_CUDA(cudaStreamSynchronize(st));
            out->objective_sum = h[0];
            out->clip_sum = h[1];
            out->kl_sum = h[2];
            out->clipped_units = h[3];
            out->total_units = h[4];
        }
    });
}

// ---- GRPO operator API (grpo.hpp:50-83) over host arrays: the same K7 kernels in fp64 ------
namespace {
// m samples of lengths lens[] (log-prob vectors concatenated) through K7; upstream (scaled by
// up_scale), per-sample terms and the summed stats back on the host
void grpo_host(parl_ctx_s* c, int m, const int32_t* lens, const double* lp, const double* old, const double* ref,
               const double* rewards, const double* adv, int group_size, int mean_only, double eps, double beta,
               int gran, double up_scale, double* upstream, double* per_sample, double* stats, double* adv_out) {
    PARL_REQUIRE(m >= 1, PARL_E_SHAPE, "empty micro-batch");
    std::vector<int32_t> cu(m + 1, 0);
    for (int j = 0; j < m; ++j) {
        PARL_REQUIRE(lens[j] >= 1, PARL_E_SHAPE, "sample has empty response");
        cu[j + 1] = cu[j] + lens[j];
    }
    const long S = cu[m];
    std::vector<int32_t> so(S);
    for (int j = 0; j < m; ++j)
        for (int t = cu[j]; t < cu[j + 1]; ++t) so[t] = j;
    cudaStream_t st = c->st;
    // one scratch block: lp | old | ref | upstream (S each) | adv_in / rewards (m) | adv_out (m) |
    // per_sample (4m) | g_seq (m) | stats (8) | slots, then ints: cu (m+1) | sample_of (S)
    const size_t nslot = grpo_slot_count(S, m);
    const size_t nd = 4 * (size_t)S + 8 * (size_t)m + 8 + nslot;
    double* d = c->staging.as<double>(nd + ((size_t)(m + 1 + S) + 1) / 2 + 1);
    double *d_lp = d, *d_old = d + S, *d_ref = d + 2 * S, *d_up = d + 3 * S, *d_in = d + 4 * S;
    double *d_adv = d_in + m, *d_ps = d_adv + m, *d_gs = d_ps + 4 * (size_t)m, *d_st = d_gs + m, *d_sl = d_st + 8;
    int32_t* d_cu = reinterpret_cast<int32_t*>(d_sl + nslot);
    int32_t* d_so = d_cu + m + 1;
    auto up = [&](void* dst, const void* src, size_t bytes) {
        if (bytes) PARL_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    };
    up(d_lp, lp, S * 8);
    up(d_old, old, S * 8);
    up(d_ref, ref, S * 8);
    up(d_in, rewards ? rewards : adv, (size_t)m * 8);
    up(d_cu, cu.data(), (size_t)(m + 1) * 4);
    up(d_so, so.data(), (size_t)S * 4);
    PARL_CUDA(cudaMemsetAsync(d_st, 0, 8 * sizeof(double), st));
    GrpoArgs a;
    a.lp = d_lp; a.old = d_old; a.ref = d_ref; a.lp_f64 = 1;
    a.sample_of = d_so; a.cu = d_cu; a.S = S; a.n = m;
    if (rewards) {
        a.rewards = d_in;
        a.group_size = group_size;
        a.mean_only = mean_only;
    } else {
        a.adv_in = d_in;
    }
    a.eps = eps; a.beta = beta; a.gran = gran; a.up_scale = up_scale;
    a.up_f64 = d_up; a.adv_out = d_adv; a.slots = d_sl; a.per_sample = d_ps; a.g_seq = d_gs; a.stats = d_st;
    launch_grpo(a, st);
    check_launch();
    auto dn = [&](void* dst, const void* src, size_t bytes) {
        if (dst && bytes) PARL_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    };
    dn(upstream, d_up, S * 8);
    dn(per_sample, d_ps, (size_t)m * 32);
    dn(stats, d_st, 5 * 8);
    dn(adv_out, d_adv, (size_t)m * 8);
    PARL_CUDA(cudaStreamSynchronize(st));
}

void require_finite(double v, const char* what) {  // grpo.cpp:56-58
    PARL_REQUIRE(std::isfinite(v), PARL_E_NUMERIC, std::string(what) + " is not finite");
}
}  // namespace

parl_status parl_group_advantages(parl_ctx_t ctx, const double* rewards, int G, int mean_only, double* adv) {
    return guarded(ctx, [&] {
        PARL_REQUIRE(G >= 2, PARL_E_CONFIG, "group_advantages needs G >= 2 rewards");
        // the G rewards as one group of G one-token samples with zero log-probs
        std::vector<int32_t> lens(G, 1);
        std::vector<double> z(G, 0.0);
        grpo_host(ctx, G, lens.data(), z.data(), z.data(), z.data(), rewards, nullptr, G, mean_only, 0.2, 0.0, 0,
                  1.0, nullptr, nullptr, nullptr, adv);
    });
}

parl_status parl_clipped_term(parl_ctx_t ctx, double lp_new, double lp_old, double adv, double eps, double* out) {
    return guarded(ctx, [&] {
        require_finite(lp_new, "logp_new");
        require_finite(lp_old, "logp_old");
        require_finite(adv, "advantage");
        PARL_REQUIRE(eps > 0.0 && eps < 1.0, PARL_E_CONFIG, "epsilon must be in (0, 1)");
        const int32_t one = 1;
        double ps[4];
        grpo_host(ctx, 1, &one, &lp_new, &lp_old, &lp_new, nullptr, &adv, 0, 0, eps, 0.0, 0, 1.0, nullptr, ps,
                  nullptr, nullptr);
        *out = ps[0];
    });
}

parl_status parl_kl_term(parl_ctx_t ctx, double lp_new, double lp_ref, double* out) {
    return guarded(ctx, [&] {
        require_finite(lp_new, "logp_new");
        require_finite(lp_ref, "logp_ref");
        const int32_t one = 1;
        const double zero = 0.0;
        double ps[4];
        grpo_host(ctx, 1, &one, &lp_new, &lp_new, &lp_ref, nullptr, &zero, 0, 0, 0.2, 0.0, 0, 1.0, nullptr, ps,
                  nullptr, nullptr);
        *out = ps[1];
    });
}

parl_status parl_per_sample_terms(parl_ctx_t ctx, const double* lp, const double* old, const double* ref, int n,
                                  double adv, double eps, double beta, int granularity, double* upstream,
                                  parl_sample_terms* out) {
    return guarded(ctx, [&] {
        PARL_REQUIRE(n >= 1, PARL_E_SHAPE, "sample has empty response");
        require_finite(adv, "advantage");
        double ps[4];
        const int32_t len = n;
        grpo_host(ctx, 1, &len, lp, old, ref, nullptr, &adv, 0, 0, eps, beta, granularity, 1.0, upstream, ps,
                  nullptr, nullptr);
        out->clip_term = ps[0];
        out->kl = ps[1];
        out->clipped_units = (int)ps[2];
        out->total_units = (int)ps[3];
    });
}

parl_status parl_grpo_microbatch_loss(parl_ctx_t ctx, int m, const int32_t* lens, const double* lp,
                                      const double* old, const double* ref, const double* advantages, double eps,
                                      double beta, int granularity, double* upstream, parl_loss_report* report,
                                      double* loss) {
    return guarded(ctx, [&] {
        PARL_REQUIRE(m >= 1, PARL_E_SHAPE, "empty micro-batch");
        for (int j = 0; j < m; ++j) require_finite(advantages[j], "advantage");
        const double inv_m = 1.0 / m;
        double st[5];
        grpo_host(ctx, m, lens, lp, old, ref, nullptr, advantages, 0, 0, eps, beta, granularity, -inv_m, upstream,
                  nullptr, st, nullptr);
        long tokens = 0;
        for (int j = 0; j < m; ++j) tokens += lens[j];
        if (loss) *loss = -inv_m * st[0];  // grpo.cpp:177-182
        if (report) {
            report->objective = inv_m * st[0];
            report->clip_term_mean = inv_m * st[1];
            report->kl_mean = inv_m * st[2];
            report->clip_fraction = st[4] > 0 ? st[3] / st[4] : 0.0;
            report->token_count = tokens;
        }
    });
}

// build_shared_prompt_mask (packing.cpp:47-72): the dense allowed-pair matrix, evaluated on the
// device by the rule the attention kernels apply tile by tile (model.cpp:242-245)
parl_status parl_shared_prompt_mask(parl_ctx_t ctx, int P, const int32_t* lens, int G, uint8_t* mask) {
    return guarded(ctx, [&] {
        PARL_REQUIRE(P >= 1, PARL_E_SHAPE, "prompt_len must be >= 1");  // packing.cpp:48-50
        long n = P;
        for (int k = 0; k < G; ++k) {
            PARL_REQUIRE(lens[k] >= 1, PARL_E_SHAPE, "response lengths must be >= 1");
            n += lens[k];
        }
        std::vector<int32_t> seg(n, 0);
        long t = P;
        for (int k = 0; k < G; ++k)
            for (int i = 0; i < lens[k]; ++i) seg[t++] = k + 1;
        int32_t* d_seg = static_cast<int32_t*>(ctx->staging.get((size_t)n * 4 + (size_t)n * n + 16));
        uint8_t* d_mask = reinterpret_cast<uint8_t*>(d_seg + n);
        PARL_CUDA(cudaMemcpyAsync(d_seg, seg.data(), (size_t)n * 4, cudaMemcpyHostToDevice, ctx->st));
        launch_allowed_mask(d_seg, (int)n, d_mask, ctx->st);
        PARL_CUDA(cudaMemcpyAsync(mask, d_mask, (size_t)n * n, cudaMemcpyDeviceToHost, ctx->st));
        PARL_CUDA(cudaStreamSynchronize(ctx->st));
    });
}

parl_status parl_group_upstream(parl_group_t g, double* out) {
    return guarded(g->ctx, [&] {
        std::vector<float> h(g->S);
        if (g->S)
            PARL_CUDA(cudaMemcpyAsync(h.data(), g->upstream.p, g->S * 4, cudaMemcpyDeviceToHost, g->ctx->st));
        PARL_CUDA(cudaStreamSynchronize(g->ctx->st));
        for (int s = 0; s < g->S; ++s) out[s] = h[s];
    });
}

parl_status parl_group_set_upstream(parl_group_t g, const double* in) {
    return guarded(g->ctx, [&] {
        std::vector<float> h(in, in + g->S);
        if (g->S)
            PARL_CUDA(cudaMemcpyAsync(g->upstream.p, h.data(), g->S * 4, cudaMemcpyHostToDevice, g->ctx->st));
        PARL_CUDA(cudaStreamSynchronize(g->ctx->st));
    });
}

parl_status parl_stats_download(parl_ctx_t ctx, parl_loss_stats* out) {
    return guarded(ctx, [&] {
        double h[5];
        PARL_CUDA(cudaMemcpyAsync(h, ctx->stats.as<double>(8), 5 * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
        PARL_CUDA(cudaStreamSynchronize(ctx->st));
        out->objective_sum = h[0];
        out->clip_sum = h[1];
        out->kl_sum = h[2];
        out->clipped_units = h[3];
        out->total_units = h[4];
    });
}

parl_status parl_stats_reset(parl_ctx_t ctx) {
    return guarded(ctx, [&] { PARL_CUDA(cudaMemsetAsync(ctx->stats.as<double>(8), 0, 8 * sizeof(double), ctx->st)); });
}

// ---- backward -----------------------------------------------------------------
parl_status parl_grad_create(parl_ctx_t ctx, parl_model_t like, parl_grad_t* out) {
    return parl_grad_create_config(ctx, &like->cfg, out);
}

parl_status parl_grad_create_config(parl_ctx_t ctx, const parl_config* cfg, parl_grad_t* out) {
    return guarded(ctx, [&] {
        validate_config(*cfg);
        auto gr = std::make_unique<parl_grad_s>();
        gr->ctx = ctx;
        ctx->refs++;
        gr->cfg = *cfg;
        gr->L = make_layout(*cfg);
        float* p = gr->g.as<float>(gr->L.total);
        PARL_CUDA(cudaMemsetAsync(p, 0, gr->L.total * sizeof(float), ctx->st));
        PARL_CUDA(cudaMemsetAsync(gr->touched.as<uint8_t>(gr->cfg.vocab_size), 0, gr->cfg.vocab_size, ctx->st));
        PARL_CUDA(cudaStreamSynchronize(ctx->st));
        *out = gr.release();
    });
}

parl_status parl_grad_destroy(parl_grad_t gr) {
    if (gr) {
        parl_ctx_s* c = gr->ctx;
        {
            std::lock_guard<std::recursive_mutex> lk(c->mu);
            cudaStreamSynchronize(c->st);
            delete gr;
        }
        ctx_release(c);
    }
    return PARL_OK;
}

parl_status parl_grad_reset(parl_grad_t gr) {
    return guarded(gr->ctx, [&] {
        PARL_CUDA(cudaMemsetAsync(gr->g.p, 0, gr->L.total * sizeof(float), gr->ctx->st));
        PARL_CUDA(cudaMemsetAsync(gr->touched.p, 0, gr->cfg.vocab_size, gr->ctx->st));
        gr->micro_steps = 0;
        gr->count_on_device = false;
    });
}

int parl_grad_micro_steps(parl_grad_t gr) {
    if (gr->count_on_device) {  // the data-parallel sum over ranks (parl_grad_allreduce)
        std::lock_guard<std::recursive_mutex> lk(gr->ctx->mu);
        double c = 0;
        if (cudaMemcpyAsync(&c, gr->count_dev.p, sizeof(c), cudaMemcpyDeviceToHost, gr->ctx->st) == cudaSuccess &&
            cudaStreamSynchronize(gr->ctx->st) == cudaSuccess) {
            gr->micro_steps = (int)c;
            gr->count_on_device = false;
        }
    }
    return gr->micro_steps;
}

// GradBuffer::set_micro_step_count / add_micro_steps (model.hpp:126-127): the pipeline sets the
// update divisor to the batch's N*G samples before apply_update (pipeline.cpp:346-351)
parl_status parl_grad_set_micro_steps(parl_grad_t gr, int n) {
    return guarded(gr->ctx, [&] {
        gr->micro_steps = n;
        gr->count_on_device = false;
    });
}

parl_status parl_grad_add_micro_steps(parl_grad_t gr, int n) {
    return guarded(gr->ctx, [&] {
        parl_grad_micro_steps(gr);
        gr->micro_steps += n;
    });
}

// GradBuffer::all_finite / ModelParams::all_finite
parl_status parl_grad_all_finite(parl_grad_t gr, int* out) {
    return guarded(gr->ctx, [&] {
        cudaStream_t st = gr->ctx->st;
        int* flags = gr->ctx->flags.as<int>(1);
        PARL_CUDA(cudaMemsetAsync(flags, 0, 4, st));
        launch_finite_check_f32(static_cast<const float*>(gr->g.p), (long)gr->L.total, flags, st);
        int h = 0;
        PARL_CUDA(cudaMemcpyAsync(&h, flags, 4, cudaMemcpyDeviceToHost, st));
        PARL_CUDA(cudaStreamSynchronize(st));
        *out = h == 0;
    });
}

parl_status parl_grad_accumulate(parl_grad_t dst, parl_grad_t src) {
    return guarded(dst->ctx, [&] {
        parl_grad_micro_steps(dst);
        parl_grad_micro_steps(src);
        PARL_REQUIRE(same_cfg(dst->cfg, src->cfg), PARL_E_SHAPE, "gradient buffers have incongruent layouts");
        launch_axpy(static_cast<const float*>(src->g.p), static_cast<float*>(dst->g.p), (long)dst->L.total,
                    dst->ctx->st);
        launch_or_bytes(static_cast<const uint8_t*>(src->touched.p), static_cast<uint8_t*>(dst->touched.p),
                        dst->cfg.vocab_size, dst->ctx->st);
        check_launch();
        dst->micro_steps += src->micro_steps;
    });
}

parl_status parl_backward(parl_ctx_t ctx, parl_model_t pol, parl_act_t act, parl_group_t g, parl_grad_t gr) {
    return guarded(ctx, [&] {
        // lifecycle checks, model.cpp:590-598
        PARL_REQUIRE(act != nullptr && act->owner != nullptr, PARL_E_LIFECYCLE,
                     "backward requires a cached forward result");
        PARL_REQUIRE(act->owner == pol && act->version == pol->version && act->gen == pol->forward_gen &&
                         act->group == g && act->epoch == g->epoch,
                     PARL_E_LIFECYCLE, "stale activation handle: a newer forward or update invalidated this cache");
        PARL_REQUIRE(same_cfg(gr->cfg, pol->cfg), PARL_E_SHAPE, "gradient buffers have incongruent layouts");
        if (ctx->prec == PARL_PREC_BF16) backward_impl<bf16>(ctx, pol, act, g, gr);
        else backward_impl<float>(ctx, pol, act, g, gr);
    });
}

parl_status parl_grad_upload(parl_grad_t gr, const double* flat, size_t n) {
    return guarded(gr->ctx, [&] {
        PARL_REQUIRE(n == gr->L.total, PARL_E_SHAPE, "gradient array size does not match the layout");
        cudaStream_t st = gr->ctx->st;
        const size_t chunk = (size_t)64 << 20;
        for (size_t o = 0; o < n; o += chunk) {
            const size_t cnt = std::min(chunk, n - o);
            double* stg = gr->ctx->staging.as<double>(cnt);
            PARL_CUDA(cudaMemcpyAsync(stg, flat + o, cnt * sizeof(double), cudaMemcpyHostToDevice, st));
            launch_f64_to_f32(stg, static_cast<float*>(gr->g.p) + o, (long)cnt, st);
            PARL_CUDA(cudaStreamSynchronize(st));
        }
        // rows of the token embedding that may now be non-zero (sparse data-parallel exchange)
        PARL_CUDA(cudaMemsetAsync(gr->touched.p, 1, gr->cfg.vocab_size, st));
    });
}

parl_status parl_grad_download(parl_grad_t gr, double* flat, size_t n) {
    return guarded(gr->ctx, [&] {
        PARL_REQUIRE(n == gr->L.total, PARL_E_SHAPE, "gradient array size does not match the layout");
        cudaStream_t st = gr->ctx->st;
        const size_t chunk = (size_t)64 << 20;
        for (size_t o = 0; o < n; o += chunk) {
            const size_t cnt = std::min(chunk, n - o);
            double* stg = gr->ctx->staging.as<double>(cnt);
            launch_f32_to_f64(static_cast<float*>(gr->g.p) + o, stg, (long)cnt, st);
            PARL_CUDA(cudaMemcpyAsync(flat + o, stg, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
            PARL_CUDA(cudaStreamSynchronize(st));
        }
    });
}

parl_status parl_train_microbatch(parl_ctx_t ctx, parl_model_t pol, parl_model_t old, parl_model_t ref,
                                  parl_group_t g, const double* rewards, const double* advantages,
                                  const parl_hyper* hp, parl_grad_t gr, parl_loss_stats* stats_out) {
    // Pipeline::train_microbatch shared-prompt branch (pipeline.cpp:97-141).
    // The activation handle is context-owned and reused across micro-batches.
    parl_act_t act = ctx->act_cache;
    parl_status s = parl_trimodel_forward(ctx, pol, old, ref, g, &act);
    ctx->act_cache = act;
    if (s == PARL_OK) s = parl_grpo_loss(ctx, g, rewards, advantages, hp, stats_out);
    if (s == PARL_OK) s = parl_backward(ctx, pol, act, g, gr);
    return s;
}

parl_status parl_apply_update(parl_model_t m, parl_grad_t gr, double lr) {
    // ModelParams::apply_update, model.cpp:202-219
    return guarded(m->ctx, [&] {
        PARL_REQUIRE(same_cfg(gr->cfg, m->cfg), PARL_E_SHAPE, "gradient layout not congruent with parameters");
        parl_grad_micro_steps(gr);
        PARL_REQUIRE(gr->micro_steps > 0, PARL_E_CONFIG, "apply_update requires micro_step_count > 0");
        PARL_REQUIRE(lr >= 0.0 && std::isfinite(lr), PARL_E_CONFIG, "learning rate must be finite and >= 0");
        PARL_REQUIRE(m->has_master, PARL_E_CONFIG, "apply_update needs the fp64 master copy");
        cudaStream_t st = m->ctx->st;
        int* flags = m->ctx->flags.as<int>(1);
        PARL_CUDA(cudaMemsetAsync(flags, 0, 4, st));
        const double scale = lr / gr->micro_steps;
        launch_sgd(static_cast<float*>(gr->g.p), static_cast<double*>(m->master.p), (long)m->L.total, scale, flags, 0, st);
        int h = 0;
        PARL_CUDA(cudaMemcpyAsync(&h, flags, 4, cudaMemcpyDeviceToHost, st));
        PARL_CUDA(cudaStreamSynchronize(st));
        PARL_REQUIRE(!(h & 1), PARL_E_NUMERIC, "refusing update: gradient contains NaN/Inf");
        PARL_REQUIRE(!(h & 2), PARL_E_NUMERIC, "refusing update: result would be non-finite");
        launch_sgd(static_cast<float*>(gr->g.p), static_cast<double*>(m->master.p), (long)m->L.total, scale, flags, 1, st);
        convert_from_master(m);
        PARL_CUDA(cudaStreamSynchronize(st));
        ++m->version;
        ++m->epoch;
    });
}

// ---- NCCL (loaded at run time; data-parallel gradient/stat allreduce) -------------
static NcclApi& nccl();

extern "C++" int nccl_allreduce_raw(void* p, size_t n, int dtype, int op, void* comm, cudaStream_t st) {
    return nccl().allReduce(p, p, n, dtype, op, comm, st);
}

static NcclApi& nccl() {
    static NcclApi api;
    if (!api.h) {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names)
            if ((api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
        if (api.h) {
            api.getUniqueId = (int (*)(void*))dlsym(api.h, "ncclGetUniqueId");
            api.allReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(api.h, "ncclAllReduce");
            api.commDestroy = (int (*)(void*))dlsym(api.h, "ncclCommDestroy");
            api.getErrorString = (const char* (*)(int))dlsym(api.h, "ncclGetErrorString");
        }
    }
    if (!api.h || !api.getUniqueId) throw Error{PARL_E_NCCL, "libnccl.so.2 not loadable"};
    return api;
}

struct NcclId {
    char b[PARL_NCCL_ID_BYTES];
};

parl_status parl_comm_unique_id(char id[PARL_NCCL_ID_BYTES]) {
    return guarded(nullptr, [&] {
        int r = nccl().getUniqueId(id);
        PARL_REQUIRE(r == 0, PARL_E_NCCL, "ncclGetUniqueId failed");
    });
}

parl_status parl_comm_init(parl_ctx_t ctx, const char id[PARL_NCCL_ID_BYTES], int rank, int nranks) {
    return guarded(ctx, [&] {
        auto& api = nccl();
        using InitFn = int (*)(void**, int, NcclId, int);
        auto init = (InitFn)dlsym(api.h, "ncclCommInitRank");
        PARL_REQUIRE(init != nullptr, PARL_E_NCCL, "ncclCommInitRank missing");
        NcclId uid;
        std::memcpy(uid.b, id, PARL_NCCL_ID_BYTES);
        PARL_CUDA(cudaSetDevice(ctx->device));
        int r = init(&ctx->comm, nranks, uid, rank);
        PARL_REQUIRE(r == 0, PARL_E_NCCL, std::string("ncclCommInitRank: ") + (api.getErrorString ? api.getErrorString(r) : "?"));
        ctx->rank = rank;
        ctx->nranks = nranks;
        if (!ctx->comm_st) {
            PARL_CUDA(cudaStreamCreateWithFlags(&ctx->comm_st, cudaStreamNonBlocking));
            PARL_CUDA(cudaEventCreateWithFlags(&ctx->ev_comm, cudaEventDisableTiming));
            PARL_CUDA(cudaEventCreateWithFlags(&ctx->ev_comm_done, cudaEventDisableTiming));
        }
    });
}

parl_status parl_grad_allreduce(parl_ctx_t ctx, parl_grad_t gr) {
    return guarded(ctx, [&] {
        gr->overlap = false;
        if (!ctx->comm || ctx->nranks == 1) {
            gr->streamed = false;
            return;
        }
        float* G = static_cast<float*>(gr->g.p);
        // PARL_SPARSE_EMB=1: exchange only the token-embedding rows some rank touched (a union of
        // row flags, then a compacted allreduce).  Its row count must reach the host to size the
        // NCCL call, a stream synchronisation mid-exchange, so the default is one dense allreduce
        // of the whole buffer (no host round trip; the rows are ~28% of the C2 gradient).
        static const bool sparse = [] {
            const char* e = std::getenv("PARL_SPARSE_EMB");
            return e && e[0] == '1';
        }();
        const int V = gr->cfg.vocab_size, D = gr->cfg.d_model;
        size_t dense0 = 0;  // first element exchanged densely
        if (sparse && gr->L.tok_emb == 0 && D % 4 == 0) {
            // union of the touched rows over the ranks (max of 0/1 bytes), then only those rows
            cudaStream_t st = ctx->st;
            uint8_t* flags = static_cast<uint8_t*>(gr->touched.p);
            comm_allreduce(ctx, flags, V, 1 /* ncclUint8 */, 2 /* ncclMax */);
            PARL_CUDA(cudaEventRecord(ctx->ev_comm_done, ctx->comm_st));
            PARL_CUDA(cudaStreamWaitEvent(st, ctx->ev_comm_done, 0));
            int32_t* idx = gr->sel_idx.as<int32_t>(V);
            int* cnt = gr->sel_count.as<int>(1);
            select_flagged_rows(flags, V, idx, cnt, st);
            int n = 0;
            PARL_CUDA(cudaMemcpyAsync(&n, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
            PARL_CUDA(cudaStreamSynchronize(st));
            float* rows = gr->sel_rows.as<float>((size_t)std::max(n, 1) * D);
            launch_rows_copy(G + gr->L.tok_emb, idx, n, D, 0, rows, st);
            comm_allreduce(ctx, rows, (size_t)n * D, 7, 0);
            PARL_CUDA(cudaEventRecord(ctx->ev_comm_done, ctx->comm_st));
            PARL_CUDA(cudaStreamWaitEvent(st, ctx->ev_comm_done, 0));
            launch_rows_copy(rows, idx, n, D, 1, G + gr->L.tok_emb, st);
            check_launch();
            dense0 = (size_t)V * D;
        }
        if (gr->streamed) {  // the layers and the head went out during the backward
            if (gr->L.layer0 > dense0) comm_allreduce(ctx, G + dense0, gr->L.layer0 - dense0, 7);
        } else {
            comm_allreduce(ctx, G + dense0, gr->L.total - dense0, 7);
        }
        gr->streamed = false;
        // counts add across ranks like GradBuffer::accumulate (read back lazily by apply_update)
        double* cnt_d = gr->count_dev.as<double>(1);
        const double cnt_h = (double)gr->micro_steps;
        PARL_CUDA(cudaMemcpyAsync(cnt_d, &cnt_h, sizeof(double), cudaMemcpyHostToDevice, ctx->st));
        comm_allreduce(ctx, cnt_d, 1, 8);
        gr->count_on_device = true;
        // the compute stream continues once every slice is reduced
        PARL_CUDA(cudaEventRecord(ctx->ev_comm_done, ctx->comm_st));
        PARL_CUDA(cudaStreamWaitEvent(ctx->st, ctx->ev_comm_done, 0));
    });
}

parl_status parl_grad_allreduce_overlap(parl_ctx_t ctx, parl_grad_t gr) {
    // Off unless PARL_AR_OVERLAP=1: NCCL's CTAs then run beside full-grid persistent kernels,
    // whose CTAs on the SMs NCCL holds start late; measured neutral at N = 2 with NCCL's default
    // channels (108.1 vs 108.4 ms per step) and slower with the channels capped to leave SMs free.
    static const bool enabled = [] {
        const char* e = std::getenv("PARL_AR_OVERLAP");
        return e && e[0] == '1';
    }();
    return guarded(ctx, [&] {
        gr->overlap = enabled && ctx->comm && ctx->nranks > 1;
        gr->streamed = false;
    });
}

parl_status parl_stats_allreduce(parl_ctx_t ctx) {
    return guarded(ctx, [&] {
        if (!ctx->comm || ctx->nranks == 1) return;
        comm_allreduce(ctx, ctx->stats.p, 5, 8);
        PARL_CUDA(cudaEventRecord(ctx->ev_comm_done, ctx->comm_st));
        PARL_CUDA(cudaStreamWaitEvent(ctx->st, ctx->ev_comm_done, 0));
    });
}

}  // extern "C"

// ---- test hooks (include/parl_gpu_debug.h) -------------------------------------
#include "parl_gpu_debug.h"
extern "C" parl_status parl_debug_gemm_bf16(int path, int M, int N, int K, const void* A, long sam, long sak,
                                            const void* B, long sbn, long sbk, int epi, const float* bias, float* Cf,
                                            long ldc, const float* resid, void* Ca, long ldca, void* Caux,
                                            const void* aux_in, const int32_t* labels, float* part, float* target,
                                            void* logits_act, int n_parts) {
    return guarded(nullptr, [&] {
        GemmArgs g = mk(M, N, K, A, sam, sak, B, sbn, sbk);
        g.epi = epi; g.bias = bias; g.Cf = Cf; g.ldc = ldc; g.resid = resid; g.Ca = Ca; g.ldca = ldca;
        g.Caux = Caux; g.aux_in = aux_in; g.labels = labels; g.part = part; g.target = target;
        g.logits_act = logits_act; g.n_parts = n_parts; g.part_cols = 128;
        if (path == 0 || path == 2) {  // 2: tcgen05, no device sync (timing loops)
            PARL_REQUIRE(gemm_tc(g, 0), PARL_E_CONFIG, "shape/layout not supported by the tcgen05 kernel");
        } else {
            gemm_simt<bf16>(g, 0);
        }
        PARL_CUDA(cudaGetLastError());
        if (path != 2) PARL_CUDA(cudaDeviceSynchronize());
    });
}

namespace {
// The debug hooks' layout: one group from the device seg_start / seg_end arrays the tests pass
// ([prompt, r1, ..] when Peff < T, else a causal sequence), its seg_info and tile schedule /
// work lists (cached across the timing loops' repeated calls of one shape).
struct DebugLayout {
    DevBuf info, sched, work;
    HostStage stage, wstage;
    AttnSched cached;
    long key[5] = {-1, -1, -1, -1, -1};
};

void debug_layout(DebugLayout& D, AttnArgs& aa, int path, int T, int H, int Dh, int Peff, const int32_t* seg_start,
                  const int32_t* seg_end) {
    const long k5[5] = {T, Peff, (long)(uintptr_t)seg_start, (long)(uintptr_t)seg_end, H};
    if (path == 2 && std::memcmp(D.key, k5, sizeof(k5)) == 0) {  // timing loops reuse the schedule
        aa.sched = D.cached;
        aa.seg_info = static_cast<const int4*>(D.info.p);
        return;
    }
    std::vector<int> lens;
    if (Peff < T) {  // count the responses: walk the segment ends until T
        std::vector<int32_t> s1(T + 1), e1(T + 1);
        int n = 1;
        while (true) {
            PARL_CUDA(cudaMemcpy(e1.data() + n - 1, seg_end + n - 1, 4, cudaMemcpyDeviceToHost));
            if (e1[n - 1] >= T) break;
            ++n;
        }
        PARL_CUDA(cudaMemcpy(s1.data(), seg_start, 4 * n, cudaMemcpyDeviceToHost));
        for (int k = 1; k < n; ++k) lens.push_back(e1[k] - s1[k]);
    }
    SegLayout L;
    L.add_group(0, Peff, lens.data(), (int)lens.size());
    int4* si = D.info.as<int4>(L.info.size());
    PARL_CUDA(cudaMemcpy(si, L.info.data(), L.info.size() * sizeof(int4), cudaMemcpyHostToDevice));
    aa.seg_info = si;
    SchedHost hs;
    aa.sched = build_schedule(L, D.sched, D.stage, 0, &hs);
    build_attn_work(aa.sched, hs, H, H * Dh, D.work, D.wstage, 0);
    D.cached = aa.sched;
    std::memcpy(D.key, k5, sizeof(k5));
}
}  // namespace

extern "C" parl_status parl_debug_attn_bf16(int path, int T, int H, int Dh, int Peff, const int32_t* seg,
                                            const int32_t* seg_start, const int32_t* seg_end, const void* qkv,
                                            void* out, float* lse) {
    return guarded(nullptr, [&] {
        AttnArgs aa;
        aa.T = T; aa.H = H; aa.Dh = Dh; aa.d = H * Dh;
        aa.seg = seg;
        aa.scale = 1.0f / std::sqrt((float)Dh);
        static DevBuf dbg_ctr;
        static unsigned dbg_base = 0;
        if (!dbg_ctr.p) PARL_CUDA(cudaMemset(dbg_ctr.as<unsigned>(4), 0, 4 * sizeof(unsigned)));
        aa.item_ctr = static_cast<unsigned*>(dbg_ctr.p);
        aa.item_base = &dbg_base;
        static DebugLayout D;
        debug_layout(D, aa, path, T, H, Dh, Peff, seg_start, seg_end);
        if (path == 0 || path == 2) {  // 2: no device sync (timing loops)
            PARL_REQUIRE(attn_fwd_tc(aa, static_cast<const bf16*>(qkv), static_cast<bf16*>(out), lse, 0), PARL_E_CONFIG,
                         "head dim not supported by the tcgen05 attention");
        } else {
            launch_attn_fwd<bf16>(aa, static_cast<const bf16*>(qkv), static_cast<bf16*>(out), lse, 0);
        }
        PARL_CUDA(cudaGetLastError());
        if (path != 2) PARL_CUDA(cudaDeviceSynchronize());
    });
}

extern "C" parl_status parl_debug_attn_bwd_bf16(int path, int T, int H, int Dh, int Peff, const int32_t* seg,
                                                const int32_t* seg_start, const int32_t* seg_end, const void* qkv,
                                                const void* out, const void* dout, const float* lse, float* dsum,
                                                void* dqkv) {
    return guarded(nullptr, [&] {
        AttnArgs aa;
        aa.T = T; aa.H = H; aa.Dh = Dh; aa.d = H * Dh;
        aa.seg = seg;
        aa.scale = 1.0f / std::sqrt((float)Dh);
        static DebugLayout D;
        debug_layout(D, aa, path, T, H, Dh, Peff, seg_start, seg_end);
        const bf16* q = static_cast<const bf16*>(qkv);
        if (path == 0 || path == 2) {  // 2: no device sync (timing loops)
            PARL_REQUIRE(attn_bwd_tc(aa, q, static_cast<const bf16*>(out), static_cast<const bf16*>(dout), lse, dsum,
                                     static_cast<bf16*>(dqkv), 0),
                         PARL_E_CONFIG, "head dim not supported by the tcgen05 attention");
        } else {
            launch_attn_bwd<bf16>(aa, q, static_cast<const bf16*>(out), static_cast<const bf16*>(dout), lse, dsum,
                                  static_cast<bf16*>(dqkv), 0);
        }
        PARL_CUDA(cudaGetLastError());
        if (path != 2) PARL_CUDA(cudaDeviceSynchronize());
    });
}

namespace parl_gpu {
bool attn_trace_read(unsigned long long* out);
}
// phase timestamps of the attention forward's CTA 0 (builds with -DPARL_ATTN_TRACE only)
extern "C" parl_status parl_debug_group_arrays(parl_group_t g, int32_t* out) {
    return guarded(g->ctx, [&] {
        const long T = g->T, S = g->S;
        const int32_t* src[11] = {g->pk.tokens, g->pk.labels, g->pk.positions, g->pk.seg, g->pk.pred, g->pk.row_ptr,
                                  g->pk.scored_pos, g->pk.scored_label, g->pk.pred_pos, g->pk.sample_of,
                                  g->pk.row_idx};
        const long n[11] = {T, T, T, T, T, T + 1, S, S, S, S, S};
        for (int a = 0; a < 11; ++a) {
            if (n[a]) PARL_CUDA(cudaMemcpyAsync(out, src[a], n[a] * 4, cudaMemcpyDeviceToHost, g->ctx->st));
            out += n[a];
        }
        PARL_CUDA(cudaStreamSynchronize(g->ctx->st));
    });
}

extern "C" parl_status parl_debug_attn_trace(unsigned long long* out) {
    return parl_gpu::attn_trace_read(out) ? PARL_OK : PARL_E_CONFIG;
}
