/* ORACLE — test infrastructure only (see parl_oracle.c header). */
#pragma once
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes mirror proj/include/parl/errors.hpp:9-46 and include/parl_gpu.h. */
enum { ORC_E_CONFIG = 1, ORC_E_SHAPE = 2, ORC_E_VOCAB = 3, ORC_E_LIFECYCLE = 4, ORC_E_NUMERIC = 5 };

/* ModelConfig, proj/include/parl/model.hpp:26-36 */
typedef struct {
    int vocab, d_model, n_layers, n_heads, d_ff, max_seq;
} orc_cfg;

typedef struct {
    size_t tok_emb, pos_emb, layer0, layer_stride, lnf_g, lnf_b, head_w, head_b, total;
} orc_layout_t;

uint64_t orc_mix_seed(uint64_t a, uint64_t b);
void orc_rng_stream(uint64_t seed, int n, int kind, double* out);
void orc_layout(const orc_cfg* c, orc_layout_t* L);
size_t orc_param_count(const orc_cfg* c);
int orc_init_params(const orc_cfg* c, uint64_t seed, double* w);
int orc_pack(const int* prompt, int P, const int* resp_flat, const int* resp_lens, int G,
             int max_seq, int* tokens, int* labels, int* positions, int* span_start, int* seg,
             int* pred);
int orc_shared_prompt_mask(int P, const int* resp_lens, int G, unsigned char* mask);
int orc_forward(const orc_cfg* c, const double* w, const int* tokens, const int* positions, int T,
                int P, const int* resp_lens, int G, const int* labels, double* logprobs_out,
                int* scored_pos_out, const double* upstream, double* grad_acc, double* rows_out);
int orc_group_advantages(const double* r, int G, int mean_only, double* a);
double orc_clipped_term(double lp, double old, double A, double eps);
double orc_kl_term(double lp, double ref);
int orc_sample_terms(const double* lp, const double* old, const double* ref, int n, double A,
                     double eps, double beta, int granularity, double* upstream, double* out4);
int orc_train_microbatch(const orc_cfg* c, const double* w_pol, const double* w_old,
                         const double* w_ref, const int* prompt, int P, const int* resp_flat,
                         const int* resp_lens, int G, const double* advantages,
                         const double* old_lp_in, double eps, double beta, int granularity,
                         double* grad_acc, double* stats5, double* lp3);

#ifdef __cplusplus
}
#endif
