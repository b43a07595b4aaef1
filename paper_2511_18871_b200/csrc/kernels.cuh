// Device data layouts and kernel launchers shared across translation units.
#pragma once

#include "internal.cuh"

namespace parl_gpu {

// K1 outputs for one packed sequence (device pointers).
struct PackedDev {
    int32_t *tokens, *labels, *positions, *seg, *pred;  // [T]
    int32_t *scored_pos, *scored_label, *pred_pos;      // [S] (gathered head rows follow scored order)
    int32_t* sample_of;                                 // [S] response index of each scored token
    int32_t *row_ptr, *row_idx;                         // position -> gathered rows CSR: [T+1], [S]
};

// Reference flat layout offsets (model.cpp:86-114).
// Activations that feed weight-gradient GEMMs carry PAD_COLS extra columns
// (1, 0, ..., 0): the GEMM over in+1 rows then yields the bias gradient too.
constexpr int PAD_COLS = 64;  // keeps padded rows 128-byte aligned (bf16) for TMA

struct FlatLayout {
    size_t tok_emb, pos_emb, layer0, layer_stride, lnf_g, lnf_b, head_w, head_b, total;
    struct Layer {
        size_t ln1g, ln1b, wq, bq, wk, bk, wv, bv, wo, bo, ln2g, ln2b, w1, b1, w2, b2;
    };
    Layer layer(int l, int d, int F) const {
        Layer r;
        size_t o = layer0 + layer_stride * (size_t)l;
        const size_t dd = (size_t)d, FF = (size_t)F;
        r.ln1g = o; o += dd;
        r.ln1b = o; o += dd;
        r.wq = o; o += dd * dd;
        r.bq = o; o += dd;
        r.wk = o; o += dd * dd;
        r.bk = o; o += dd;
        r.wv = o; o += dd * dd;
        r.bv = o; o += dd;
        r.wo = o; o += dd * dd;
        r.bo = o; o += dd;
        r.ln2g = o; o += dd;
        r.ln2b = o; o += dd;
        r.w1 = o; o += dd * FF;
        r.b1 = o; o += FF;
        r.w2 = o; o += FF * dd;
        r.b2 = o; o += dd;
        return r;
    }
};

inline FlatLayout make_layout(const parl_config& c) {
    FlatLayout L;
    size_t o = 0;
    const size_t d = (size_t)c.d_model, F = (size_t)c.d_ff, V = (size_t)c.vocab_size;
    L.tok_emb = o; o += V * d;
    L.pos_emb = o; o += (size_t)c.max_seq_len * d;
    L.layer0 = o;
    L.layer_stride = 2 * d + 4 * (d * d + d) + 2 * d + (d * F + F) + (F * d + d);
    o += L.layer_stride * (size_t)c.n_layers;
    L.lnf_g = o; o += d;
    L.lnf_b = o; o += d;
    L.head_w = o; o += d * V;
    L.head_b = o; o += V;
    L.total = o;
    return L;
}

// Compute copy of one weight set.  Matrices are stored out-major ("W^T",
// [out x in]) so every forward contraction is K-major on both operands
// (the tcgen05 / TMA-friendly layout); backward dX contractions read the
// same arrays as MN-major operands.  Q, K, V are fused into one [3d x d].
struct LayerW {
    float *ln1_g, *ln1_b, *ln2_g, *ln2_b, *bqkv, *bo, *b1, *b2;
    void *wqkv_t, *wo_t, *w1_t, *w2_t;  // act dtype
};
struct ModelW {
    float *tok_emb, *pos_emb, *lnf_g, *lnf_b, *head_b;
    void* head_w_t;  // [V x d]
    LayerW* layers;  // host array of device pointers
};

// launchers (k_elem.cu)
void launch_pack(const int32_t* prompt, int P, const int32_t* resp, const int32_t* cu, int G, int T,
                 const PackedDev& pk, unsigned* id_max, cudaStream_t st);
// several prompt groups per sequence; tables: gstart [n+1] | pstart [n] | r0 [n+1] | rcu [R+1] | rstart [R]
void launch_pack_multi(const int32_t* prompts, const int32_t* resp, const int32_t* tables, int n, int n_resp, int T,
                       const PackedDev& pk, unsigned* id_max, cudaStream_t st);
void launch_allowed_mask(const int32_t* seg, int n, uint8_t* mask, cudaStream_t st);
void launch_embed(const float* tok, const float* pos, const int32_t* tokens, const int32_t* positions, int T, int D,
                  float* x, cudaStream_t st);
template <class T>
void launch_layernorm(const float* x, const int32_t* rows, int R, int D, const float* g, const float* b, T* y,
                      long ldy, float* mean, float* rstd, cudaStream_t st);
// the same LayerNorm of nm <= 3 models (tri-model forward) in one launch
template <class T>
void launch_layernorm_multi(int nm, const float* const* x, const float* const* g, const float* const* b, T* const* y,
                            long ldy, float* const* mean, float* const* rstd, int R, int D, cudaStream_t st);
template <class T>
void launch_layernorm_bwd(const float* dy, const float* x, const int32_t* rows, const float* mean, const float* rstd,
                          const float* gamma, int R, int D, const float* res, float* dx, T* dx_act, float* dgamma,
                          float* dbeta, cudaStream_t st);
template <class T>
void launch_fill_pad(T* y, long rows, int D, long ld, cudaStream_t st);
template <class T>
void launch_colsum(const T* X, long ldx, int R, int N, float* out, cudaStream_t st);
void launch_row_lse(const float* z, int S, int V, const int32_t* labels, float* lse, float* lp, cudaStream_t st);
void launch_lse_combine(const float* part, int n_parts, const float* target, int S, float* lse, float* lp,
                        cudaStream_t st);
template <class Tin, class Tout>
void launch_softmax_bwd(const Tin* z, long ldz, Tout* dz, long lddz, int S, int V, const float* lse, const float* u,
                        const int32_t* labels, cudaStream_t st);
// K7 GRPO loss (k_grpo.cu): advantages + per-token terms + per-sample sums + stats
struct GrpoArgs {
    const void *lp = nullptr, *old = nullptr, *ref = nullptr;  // [S] each, fp32 or (lp_f64) fp64
    int lp_f64 = 0;
    const int32_t* sample_of = nullptr;  // [S] sample of each scored token (non-decreasing)
    const int32_t* cu = nullptr;         // [n + 1] token offsets of the samples
    long S = 0;
    int n = 0;
    const double* rewards = nullptr;  // [n]: advantages per group of group_size samples (grpo.cpp:24-48)
    const double* adv_in = nullptr;   // [n]: given advantages (rewards == nullptr)
    int group_size = 0, mean_only = 0;
    double eps = 0.2, beta = 0.04;
    int gran = 0;             // 0 token, 1 sequence
    double up_scale = -1.0;   // upstream = up_scale * d(L_j - beta KL_j)/d lp  (pipeline.cpp:138: -1)
    float* up_f32 = nullptr;  // [S] upstream out (one of up_f32 / up_f64 may be null)
    double* up_f64 = nullptr;
    double* adv_out = nullptr;     // [n] advantages used (required)
    double* slots = nullptr;       // grpo_slot_count(S, n) doubles
    double* per_sample = nullptr;  // [n x 4] {clip_term, kl, clipped_units, total_units} or null
    double* g_seq = nullptr;       // [n] (sequence granularity)
    double* stats = nullptr;       // [5] += {objective, clip, kl, clipped, units} or null
    int warp_tokens = 0;           // set by launch_grpo: tokens per warp range (slot granularity)
    double* terms = nullptr;       // set by launch_grpo: the finisher's block partials of the stats (slots block)
    unsigned* ticket = nullptr;    // set by launch_grpo: k_grpo_finish's last-block ticket (in the slots block)
};
size_t grpo_slot_count(long S, int n);
void launch_grpo(const GrpoArgs& a, cudaStream_t st);
void launch_scatter_rows(const float* dxg, const int32_t* row_ptr, const int32_t* row_idx, int T, int D, float* dx,
                         cudaStream_t st);
size_t sort_temp_bytes(int n);
void launch_sort_pairs(void* temp, size_t temp_bytes, const int32_t* keys_in, int32_t* keys_out,
                       const int32_t* vals_in, int32_t* vals_out, int n, int end_bit, cudaStream_t st);
void launch_iota(int32_t* x, int n, cudaStream_t st);
void launch_embed_grad(const int32_t* keys, const int32_t* idx, int T, const float* dx, int D, float* grad,
                       cudaStream_t st);
template <class T>
void launch_f32_to_act(const float* x, T* y, long n, cudaStream_t st);
template <class T>
void launch_convert_w(const double* src, int rows, int cols, T* dst, long ldd, int transposed, cudaStream_t st);
template <class T>
void launch_export_w(const T* src, long lds, int rows, int cols, int transposed, double* dst, cudaStream_t st);
void launch_f32_to_f64(const float* x, double* y, long n, cudaStream_t st);
void launch_f64_to_f32(const double* x, float* y, long n, cudaStream_t st);
void launch_randn(double* out, long n, uint64_t seed, uint32_t stream, double scale, const double* base,
                  cudaStream_t st);
void launch_fill_f64(double* out, long n, double v, cudaStream_t st);
void launch_axpy(const float* x, float* y, long n, cudaStream_t st);  // y += x
// sparse token-embedding gradient exchange (rows touched by any rank)
void launch_mark_rows(const int32_t* ids, int n, uint8_t* flags, cudaStream_t st);
void launch_or_bytes(const uint8_t* src, uint8_t* dst, int n, cudaStream_t st);
void select_flagged_rows(const uint8_t* flags, int n, int32_t* idx, int* count, cudaStream_t st);
void launch_rows_copy(const float* src, const int32_t* idx, int n, int d, int dir, float* dst, cudaStream_t st);
void launch_finite_check_f32(const float* x, long n, int* flags, cudaStream_t st);  // flags |= 1 on NaN/Inf
void launch_finite_check_f64(const double* x, long n, int* flags, cudaStream_t st);
void launch_sgd(const float* g, double* w, long n, double scale, int* flags, int phase, cudaStream_t st);

// attention (k_attn.cu).  qkv: [T x 3d] (q | k | v, head h at columns h*Dh);
// seg/seg_start/seg_end describe the shared-prompt structure (seg 0 = prompt).
// Attention tile schedule (128 x 128 tiles), built once per packed sequence on
// the host: for every query tile the visible key tiles, for every key tile the
// query tiles that see it; entries are tile | (full << 30), where full means
// every (row, key) pair of the tile is allowed (no per-element mask).  Orders
// list the tiles heaviest-first for load balance.
struct AttnSched {
    const int32_t *q_ptr = nullptr, *q_list = nullptr, *q_order = nullptr;
    const int32_t *k_ptr = nullptr, *k_list = nullptr, *k_order = nullptr;
    // pairs of adjacent query tiles (2p, 2p+1): union of their key tiles, each
    // entry kt | VIS0 << 24 | FULL0 << 25 | VIS1 << 26 | FULL1 << 27
    const int32_t *p_ptr = nullptr, *p_list = nullptr, *p_order = nullptr;
    int n_pairs = 0;
    // forward work lists: CTA b processes items w_items[w_ptr[b] .. w_ptr[b+1]),
    // item = pair * H + head, balanced over w_grid CTAs (LPT on key-tile counts)
    const int32_t *w_ptr = nullptr, *w_items = nullptr;
    int w_grid = 0;
    // the same items as one queue (longest / head-major first) for the dynamic work queue
    const int32_t* w_order = nullptr;
    int w_n = 0;
    // backward work lists: dK/dV items = key tile * H + head, dQ items = query tile * H + head
    const int32_t *bk_ptr = nullptr, *bk_items = nullptr, *bq_ptr = nullptr, *bq_items = nullptr;
    int bk_grid = 0, bq_grid = 0;
};

struct AttnArgs {
    AttnSched sched;
    int T, H, Dh, d;
    long ldo = 0;              // row stride of the attention output O (0: d)
    const int32_t* seg;        // [T] segment of each position
    // per segment {A, B, C, Q}: rows of a prompt segment (B = -1) see keys [A, i]; rows of a
    // response segment see their group's prompt [A, B) and their own prefix [C, i]; keys of the
    // segment are seen by queries [j, Q) (model.cpp:242-245, several prompt groups per sequence)
    const int4* seg_info;
    float scale;
    // dynamic work queue of the forward: a device counter and the host-side running base
    // (each launch consumes n_items + grid counter values); null: static per-CTA lists
    unsigned* item_ctr = nullptr;
    unsigned* item_base = nullptr;
};
// tcgen05 forward (k_attn_tc.cu); false if the head dim / alignment is unsupported
bool attn_fwd_tc(const AttnArgs& a, const bf16* qkv, bf16* out, float* lse, cudaStream_t st);
// nm models of one group (tri-model forward) in one launch where possible
bool attn_fwd_tc_multi(const AttnArgs& a, const bf16* const* qkv, bf16* const* out, float* const* lse, int nm,
                       cudaStream_t st);
template <class T>
void launch_attn_fwd(const AttnArgs& a, const T* qkv, T* out, float* lse, cudaStream_t st);
// tcgen05 backward (k_attn_tc.cu): dqkv from dO, lse and D = rowsum(dO*O)
bool attn_bwd_tc(const AttnArgs& a, const bf16* qkv, const bf16* out, const bf16* dout, const float* lse, float* dsum,
                 bf16* dqkv, cudaStream_t st);
// KV-cached decode attention: n_seq query rows (q, row stride ldq, head h at h*Dh) against
// the shared prompt cache kv_prompt [P x 2d] (K | V) and each sequence's own cache
// kv_own + seq * own_stride [n_own x 2d]
template <class T>
void launch_decode_attn(const T* q, long ldq, const T* kv_prompt, const T* kv_own, long own_stride, int P, int n_own,
                        int n_seq, int H, int d, float scale, T* out, long ldo, cudaStream_t st);
template <class T>
void launch_attn_dsum(const AttnArgs& a, const T* out, const T* dout, float* dsum, cudaStream_t st);
template <class T>
void launch_attn_bwd(const AttnArgs& a, const T* qkv, const T* out, const T* dout, const float* lse, float* dsum,
                     T* dqkv, cudaStream_t st);

}  // namespace parl_gpu
