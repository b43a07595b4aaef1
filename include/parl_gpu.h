/*
 * parl_gpu.h — C-ABI of the B200-native hot path of arXiv 2511.18871:
 * shared-prompt packing -> tri-model log-prob -> GRPO loss -> policy backward
 * -> gradient accumulate (+ NCCL allreduce across ranks).
 *
 * Plain C types only (no torch, no C++).  Every entry point returns a
 * parl_status; the codes map 1:1 onto the reference's exception types
 * (proj/include/parl/errors.hpp:9-46) plus CUDA/NCCL failures, and
 * parl_last_error() returns the message.  The C++ drop-in layer
 * (include/parl_gpu.hpp) converts them back into the same exception types.
 *
 * Each function cites the reference interface it replaces.  Device buffers
 * stay resident: weights are uploaded once per version, and only per-token
 * vectors and scalars cross host<->device on the measured path.
 */
#ifndef PARL_GPU_H
#define PARL_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PARL_OK = 0,
    PARL_E_CONFIG = 1,    /* ConfigError    errors.hpp:9  */
    PARL_E_SHAPE = 2,     /* ShapeError     errors.hpp:14 */
    PARL_E_VOCAB = 3,     /* VocabError     errors.hpp:19 */
    PARL_E_LIFECYCLE = 4, /* LifecycleError errors.hpp:24 */
    PARL_E_NUMERIC = 5,   /* NumericError   errors.hpp:29 */
    PARL_E_BARRIER = 6,   /* BarrierError   errors.hpp:34 */
    PARL_E_STALL = 7,     /* StallError     errors.hpp:39 */
    PARL_E_IO = 8,        /* IoError        errors.hpp:44 */
    PARL_E_CUDA = 9,
    PARL_E_NCCL = 10
} parl_status;

/* Arithmetic of the device path.  FP32: fp32 storage, FFMA contractions
 * (the BASELINE configs[0] precision).  BF16: bf16 operands on tcgen05
 * tensor cores with fp32 accumulation, fp32 residual stream/statistics. */
typedef enum { PARL_PREC_FP32 = 0, PARL_PREC_BF16 = 1 } parl_precision;

/* ModelConfig, proj/include/parl/model.hpp:26-36 */
typedef struct {
    int vocab_size, d_model, n_layers, n_heads, d_ff, max_seq_len;
} parl_config;

/* HyperParams subset used by the loss, proj/include/parl/pipeline.hpp:29-37 */
typedef struct {
    double epsilon;         /* clip range, (0,1) */
    double beta;            /* KL weight, >= 0 */
    int granularity;        /* 0 = token, 1 = sequence (LossGranularity) */
    int advantage_mean_only;/* 0 = (r-mean)/std_pop, 1 = r-mean (grpo.cpp:24-48) */
} parl_hyper;

/* Pipeline::MicrobatchStats, proj/include/parl/pipeline.hpp:109-116 */
typedef struct {
    double objective_sum, clip_sum, kl_sum, clipped_units, total_units;
} parl_loss_stats;

/* SampleTerms (scalar part), proj/include/parl/grpo.hpp:64-70 */
typedef struct {
    double clip_term, kl;
    int clipped_units, total_units;
} parl_sample_terms;

/* LossReport, proj/include/parl/grpo.hpp:41-47 */
typedef struct {
    double objective, clip_term_mean, kl_mean, clip_fraction;
    long token_count;
} parl_loss_report;

typedef struct parl_ctx_s* parl_ctx_t;     /* device, stream, workspaces, optional NCCL comm */
typedef struct parl_model_s* parl_model_t; /* one device weight set (ModelParams) */
typedef struct parl_group_s* parl_group_t; /* one packed sequence (PackedGroup + K1 outputs) */
typedef struct parl_act_s* parl_act_t;     /* policy activations (ForwardResult::cache) */
typedef struct parl_grad_s* parl_grad_t;   /* fp32 gradient accumulator (GradBuffer) */

/* ---- context ------------------------------------------------------------ */
parl_status parl_ctx_create(int device, parl_precision prec, parl_ctx_t* out);
parl_status parl_ctx_destroy(parl_ctx_t ctx);
const char* parl_last_error(parl_ctx_t ctx);
parl_status parl_ctx_sync(parl_ctx_t ctx);
/* cudaStream_t the context launches on (for callers timing with events). */
void* parl_ctx_stream(parl_ctx_t ctx);
/* Number of kernels this context launched since creation (bench evidence). */
uint64_t parl_ctx_launches(parl_ctx_t ctx);
const char* parl_version(void);

/* Kernel-class profiler (bench evidence): when enabled, every launch of the
 * classes below is bracketed by CUDA events on the context stream and its
 * algorithmic work (FLOPs or bytes) is recorded.  Reading syncs the stream. */
typedef enum {
    PARL_KC_GEMM = 0,      /* all tensor-core / FFMA contractions */
    PARL_KC_HEAD = 1,      /* LM-head forward contraction (+LSE epilogue) */
    PARL_KC_ATTN_FWD = 2,
    PARL_KC_ATTN_BWD = 3,
    PARL_KC_LOSS = 4,      /* K7 GRPO loss */
    PARL_KC_PACK = 5,      /* K1 packer */
    PARL_KC_NORM = 6,      /* LayerNorm fwd/bwd, embeddings, reductions */
    PARL_KC_SEED = 7,      /* softmax backward seed dZ = u (onehot - softmax) over the policy logits */
    PARL_KC_COUNT = 8
} parl_kernel_class;
parl_status parl_ctx_profile(parl_ctx_t ctx, int enable);
/* ms = summed event time, work = summed algorithmic FLOPs (or bytes for HBM
 * classes), launches = count; then resets the class. */
parl_status parl_ctx_profile_read(parl_ctx_t ctx, int kernel_class, double* ms, double* work, long* launches);

/* Activation recomputation of the policy forward (B200 memory policy, no
 * reference counterpart): 0 = auto (keep every layer's activations when they
 * fit in HBM next to the backward's workspaces, else keep only the residual
 * stream and rebuild each layer in the backward), 1 = always, 2 = never.
 * Results are bit-identical in all modes.  Default 0, or $PARL_RECOMPUTE. */
parl_status parl_ctx_set_recompute(parl_ctx_t ctx, int mode);
/* 1 if the activation handle was produced in recompute mode, else 0 */
int parl_act_recompute(parl_act_t act);

/* ---- models: ModelParams (model.hpp:64-106) ---------------------------- */
parl_status parl_model_create(parl_ctx_t ctx, const parl_config* cfg, parl_model_t* out);
parl_status parl_model_destroy(parl_model_t m);
/* Replaces ModelParams::flat() as the weight source: fp64 flat array in the
 * reference layout (model.cpp:86-114).  `version` keys staleness. */
parl_status parl_model_upload(parl_model_t m, const double* flat, size_t n, uint64_t version);
/* ModelParams::init (model.cpp:142-164) bit-exact on the host, then upload. */
parl_status parl_model_init(parl_model_t m, uint64_t seed);
/* Device-side random init (Philox; same distribution, not the same stream)
 * for the large configs whose fp64 host copy is impractical. */
parl_status parl_model_init_device(parl_model_t m, uint64_t seed, double scale);
/* dst <- src (+ scale * N(0,1) from seed when scale != 0): snapshot_old_policy,
 * pipeline.cpp:20 / model copies for synthetic old/ref weights. */
parl_status parl_model_copy(parl_model_t dst, parl_model_t src, uint64_t seed, double scale);
/* Download weights into the reference fp64 layout (checkpoint path). */
parl_status parl_model_download(parl_model_t m, double* flat, size_t n);
size_t parl_param_count(const parl_config* cfg);
uint64_t parl_model_version(parl_model_t m);
/* ModelParams::init_seed (model.hpp:71): kept by init / copy / checkpoint load; set by callers that
 * upload weights drawn elsewhere (checkpoint header field). */
uint64_t parl_model_init_seed(parl_model_t m);
/* Write counter of the device weights (upload / init / copy / update / load): host mirrors key on it. */
uint64_t parl_model_epoch(parl_model_t m);
/* ModelParams::forward_generation (model.hpp:100-101): bumped by every forward on this model. */
uint64_t parl_model_forward_gen(parl_model_t m);
parl_status parl_model_set_init_seed(parl_model_t m, uint64_t seed);
/* ModelParams::all_finite (model.cpp:183-187): *out = 1 when every weight is finite. */
parl_status parl_model_all_finite(parl_model_t m, int* out);

/* Checkpoints in the reference's PARLCKP1 format (docs/formats.md): save_checkpoint /
 * load_checkpoint (model.cpp:924-987).  IoError on open / magic / truncation / layout
 * mismatch, NumericError on non-finite weights, ConfigError on an invalid header config.
 * load creates a new model on ctx holding the stored weights and version. */
/* sample_tokens (model.cpp:843-900): up to max_new_tokens sampled after `prompt` (greedy at
 * temperature 0, else softmax(logits / temperature) with the reference RNG stream), stopping
 * after kEosToken; out[max_new_tokens], *n_out = tokens written.  Same errors as the
 * reference (ShapeError / ConfigError / VocabError). */
parl_status parl_sample_tokens(parl_ctx_t ctx, parl_model_t m, const int32_t* prompt, int prompt_len,
                               int max_new_tokens, double temperature, uint64_t rng_seed, int32_t* out, int* n_out);
/* The G rollouts of one prompt at once (RolloutService::run's sample_tokens calls,
 * rollout.cpp:140-160) on a KV-cached decoder: the prompt is prefilled once and its K/V shared
 * by the n_seq sequences; sequence k follows sample_tokens(prompt, max_new_tokens, temperature,
 * seeds[k]) exactly (the reference's token choice and RNG stream).  out[k * max_new_tokens ..],
 * n_out[k]; logprobs_out (may be NULL) gets each sampled token's log-prob under the model, the
 * old_logprobs of rollout_weights mode (score_logprobs, rollout.cpp:52-66). */
parl_status parl_sample_group(parl_ctx_t ctx, parl_model_t m, const int32_t* prompt, int prompt_len, int n_seq,
                              int max_new_tokens, double temperature, const uint64_t* seeds, int32_t* out, int* n_out,
                              double* logprobs_out);
parl_status parl_checkpoint_save(parl_model_t m, const char* path);
parl_status parl_model_config(parl_model_t m, parl_config* out);
parl_status parl_checkpoint_load(parl_ctx_t ctx, const char* path, parl_model_t* out);

/* ---- packing: pack_group (packing.cpp:7-45) + segments/predecessors
 *      (model.cpp:230-253), K1 on the device ------------------------------ */
parl_status parl_group_create(parl_ctx_t ctx, int max_tokens, int max_responses, parl_group_t* out);
parl_status parl_group_destroy(parl_group_t g);
/* Host inputs: prompt[P], responses concatenated in resp_flat with lengths
 * resp_lens[G].  Same validation and errors as pack_group. */
parl_status parl_pack(parl_group_t g, const int32_t* prompt, int P, const int32_t* resp_flat,
                      const int32_t* resp_lens, int G, int max_seq_len);
/* Device-resident inputs (same meaning; pointers are device pointers). */
parl_status parl_pack_device(parl_group_t g, const int32_t* d_prompt, int P,
                             const int32_t* d_resp_flat, const int32_t* resp_lens_host, int G,
                             int max_seq_len);
/* Several prompt groups in ONE packed sequence (f4; SPEC.md:278 lifted): group q is
 * prompt q (prompt_lens[q] tokens, concatenated in `prompts`) followed by its group_sizes[q]
 * responses (concatenated in resp_flat, lengths resp_lens[]), each group laid out as
 * pack_group lays out one (positions restart per group, max_seq_len bounds each group);
 * attention never crosses groups.  One forward / backward then covers every group; the
 * GRPO loss takes per-group rewards (equal group sizes) or per-sample advantages. */
parl_status parl_pack_multi(parl_group_t g, const int32_t* prompts, const int32_t* prompt_lens,
                            const int32_t* resp_flat, const int32_t* resp_lens, const int32_t* group_sizes, int n,
                            int max_seq_len);
/* Device-resident token arrays (lengths on the host). */
parl_status parl_pack_multi_device(parl_group_t g, const int32_t* d_prompts, const int32_t* prompt_lens,
                                   const int32_t* d_resp, const int32_t* resp_lens, const int32_t* group_sizes, int n,
                                   int max_seq_len);
/* General forward_logprobs input (model.hpp:153-158): arbitrary tokens,
 * positions and self-aligned labels (-1 = unscored) under a causal mask
 * (prompt_len == 0) or a shared-prompt mask (prompt_len, resp_lens[G]).
 * Validation order and errors follow validate_forward_inputs (model.cpp:404-426). */
parl_status parl_set_sequence(parl_group_t g, const int32_t* tokens, const int32_t* positions,
                              const int32_t* labels, int T, int prompt_len,
                              const int32_t* resp_lens, int G, int vocab_size, int max_seq_len);
/* Packed outputs back to the host (any pointer may be NULL). */
parl_status parl_group_download(parl_group_t g, int32_t* tokens, int32_t* labels,
                                int32_t* positions, int32_t* seg, int32_t* pred,
                                int32_t* span_start, int32_t* scored_pos);
int parl_group_tokens(parl_group_t g);
int parl_group_scored(parl_group_t g);

/* ---- forward: forward_logprobs (model.cpp:534-567), trimodel_forward
 *      (pipeline.cpp:22-30) -------------------------------------------------
 * slot: 0 = policy, 1 = old, 2 = reference.  Log-probs stay on the device in
 * the group (slot-indexed) unless copied out with parl_group_logprobs. */
parl_status parl_forward(parl_ctx_t ctx, parl_model_t m, parl_group_t g, int slot,
                         parl_act_t* act_out /* NULL = no activation cache */);
/* old == NULL: rollout_weights mode (pipeline.cpp:113-119); old log-probs
 * come from parl_group_set_logprobs(slot 1). */
parl_status parl_trimodel_forward(parl_ctx_t ctx, parl_model_t pol, parl_model_t old,
                                  parl_model_t ref, parl_group_t g, parl_act_t* act_out);
parl_status parl_group_logprobs(parl_group_t g, int slot, double* out /* [scored] */);
parl_status parl_group_set_logprobs(parl_group_t g, int slot, const double* in);
/* forward_logprob_rows (model.cpp:569-585): [T x V] log-softmax rows. */
parl_status parl_logprob_rows(parl_ctx_t ctx, parl_model_t m, parl_group_t g, double* rows);
parl_status parl_act_destroy(parl_act_t a);

/* ---- GRPO loss: group_advantages (grpo.cpp:24-48) + per_sample_terms
 *      (grpo.cpp:111-151) over every response of the group --------------
 * rewards[G] (host) -> advantages on the device, or advantages given
 * directly (rewards == NULL).  Writes the backward seed upstream = -g
 * (pipeline.cpp:138) into the group and ADDS this micro-batch's stats. */
parl_status parl_grpo_loss(parl_ctx_t ctx, parl_group_t g, const double* rewards,
                           const double* advantages, const parl_hyper* hp,
                           parl_loss_stats* stats_out /* NULL = keep on device */);
parl_status parl_group_upstream(parl_group_t g, double* out);
parl_status parl_group_set_upstream(parl_group_t g, const double* in);
/* Device-side running stats (accumulated by parl_grpo_loss). */
parl_status parl_stats_download(parl_ctx_t ctx, parl_loss_stats* out);
parl_status parl_stats_reset(parl_ctx_t ctx);

/* ---- backward: backward (model.cpp:587-838) + GradBuffer::accumulate
 *      (model.cpp:189-194); uses the group's upstream seed --------------- */
parl_status parl_grad_create(parl_ctx_t ctx, parl_model_t like, parl_grad_t* out);
parl_status parl_grad_create_config(parl_ctx_t ctx, const parl_config* cfg, parl_grad_t* out);
parl_status parl_grad_destroy(parl_grad_t gr);
parl_status parl_grad_reset(parl_grad_t gr);
parl_status parl_backward(parl_ctx_t ctx, parl_model_t pol, parl_act_t act, parl_group_t g,
                          parl_grad_t gr);
parl_status parl_grad_download(parl_grad_t gr, double* flat, size_t n);
/* GradBuffer::accumulate (model.cpp:189-194): dst += src, counts add. */
parl_status parl_grad_accumulate(parl_grad_t dst, parl_grad_t src);
/* GradBuffer::micro_step_count / set_micro_step_count / add_micro_steps (model.hpp:124-127).
 * parl_backward adds 1 per call (backward returns a count-1 buffer that accumulate adds);
 * the pipeline sets the batch's N*G before apply_update (pipeline.cpp:346-351). */
int parl_grad_micro_steps(parl_grad_t gr);
parl_status parl_grad_set_micro_steps(parl_grad_t gr, int n);
parl_status parl_grad_add_micro_steps(parl_grad_t gr, int n);
/* GradBuffer::all_finite (model.cpp:196-200) */
parl_status parl_grad_all_finite(parl_grad_t gr, int* out);
/* Host fp64 gradient -> device accumulator (GradBuffer::flat_mut() writes of a drop-in caller). */
parl_status parl_grad_upload(parl_grad_t gr, const double* flat, size_t n);

/* ---- whole micro-step: Pipeline::train_microbatch shared-prompt branch
 *      (pipeline.cpp:97-141) in one call ------------------------------------ */
parl_status parl_train_microbatch(parl_ctx_t ctx, parl_model_t pol, parl_model_t old,
                                  parl_model_t ref, parl_group_t g, const double* rewards,
                                  const double* advantages, const parl_hyper* hp,
                                  parl_grad_t gr, parl_loss_stats* stats_out);

/* ---- GRPO operator API (grpo.hpp:50-83) on host arrays, evaluated by the K7 kernels in fp64 ----
 * group_advantages / group_advantages_mean_only (grpo.cpp:24-48): ConfigError for G < 2. */
parl_status parl_group_advantages(parl_ctx_t ctx, const double* rewards, int G, int mean_only, double* adv);
/* clipped_term / kl_term (grpo.cpp:95-108): NumericError on non-finite input, ConfigError on eps. */
parl_status parl_clipped_term(parl_ctx_t ctx, double lp_new, double lp_old, double adv, double eps, double* out);
parl_status parl_kl_term(parl_ctx_t ctx, double lp_new, double lp_ref, double* out);
/* per_sample_terms (grpo.cpp:111-151) for one sample of n tokens: upstream[n] = d(L - beta KL)/d lp. */
parl_status parl_per_sample_terms(parl_ctx_t ctx, const double* lp, const double* old, const double* ref, int n,
                                  double adv, double eps, double beta, int granularity, double* upstream,
                                  parl_sample_terms* out);
/* grpo_microbatch_loss (grpo.cpp:153-184) over m samples of lengths lens[m] (log-prob vectors and
 * upstream concatenated in sample order): upstream = -(1/m) per-sample upstream. */
parl_status parl_grpo_microbatch_loss(parl_ctx_t ctx, int m, const int32_t* lens, const double* lp,
                                      const double* old, const double* ref, const double* advantages, double eps,
                                      double beta, int granularity, double* upstream, parl_loss_report* report,
                                      double* loss);
/* build_shared_prompt_mask (packing.cpp:47-72): row-major [n x n] 0/1, n = P + sum(lens). */
parl_status parl_shared_prompt_mask(parl_ctx_t ctx, int P, const int32_t* lens, int G, uint8_t* mask);

/* ---- apply_update (model.cpp:202-219) on the device: W -= lr*g/count,
 *      refusing non-finite gradients/results (weights untouched). ---------- */
parl_status parl_apply_update(parl_model_t m, parl_grad_t gr, double lr);

/* ---- multi-GPU: data parallel over prompt groups (NCCL over NVLink) -------- */
#define PARL_NCCL_ID_BYTES 128
parl_status parl_comm_unique_id(char id[PARL_NCCL_ID_BYTES]);
parl_status parl_comm_init(parl_ctx_t ctx, const char id[PARL_NCCL_ID_BYTES], int rank, int nranks);
parl_status parl_grad_allreduce(parl_ctx_t ctx, parl_grad_t gr);
parl_status parl_stats_allreduce(parl_ctx_t ctx);
/* Arm an overlapped gradient allreduce: the next parl_backward into `grad` (the last
 * micro-batch of the optimizer step) hands every gradient slice to NCCL on a second stream
 * as soon as it is final (head + final LN first, each layer after its LN1 backward), so the
 * exchange overlaps the rest of the backward; parl_grad_allreduce then reduces the
 * embeddings and joins the streams.  Same sum as one allreduce of the whole buffer. */
parl_status parl_grad_allreduce_overlap(parl_ctx_t ctx, parl_grad_t grad);

#ifdef __cplusplus
}
#endif
#endif /* PARL_GPU_H */
