// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference sources (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libparl_ref.so).
// It is used (a) to pin the C restatement in parl_oracle.c, (b) to generate
// the golden fixtures in tests/golden/, and (c) as the CPU baseline in
// bench.py (`cpu_baseline.kind = "reference"`).  Nothing here is product code.
#include <atomic>
#include <chrono>
#include <cstring>
#include <thread>
#include <vector>

#include "parl/grpo.hpp"
#include "parl/model.hpp"
#include "parl/packing.hpp"
#include "parl/pipeline.hpp"
#include "parl/rng.hpp"

using namespace parl;

namespace {

struct CCfg {
    int vocab, d_model, n_layers, n_heads, d_ff, max_seq;
};

ModelConfig to_cfg(const CCfg* c) {
    ModelConfig m;
    m.vocab_size = c->vocab;
    m.d_model = c->d_model;
    m.n_layers = c->n_layers;
    m.n_heads = c->n_heads;
    m.d_ff = c->d_ff;
    m.max_seq_len = c->max_seq;
    return m;
}

// Error convention of the C-ABI: errors.hpp types -> small positive codes.
template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const ConfigError&) {
        return -1;
    } catch (const ShapeError&) {
        return -2;
    } catch (const VocabError&) {
        return -3;
    } catch (const LifecycleError&) {
        return -4;
    } catch (const NumericError&) {
        return -5;
    } catch (...) {
        return -99;
    }
}

ModelParams params_from(const CCfg* c, const double* w) {
    ModelParams p = ModelParams::init(to_cfg(c), 0);
    if (w) std::memcpy(p.flat_mut().data(), w, p.flat().size() * sizeof(double));
    return p;
}

AttentionMaskSpec mask_from(int P, const int* lens, int G) {
    if (P <= 0) return AttentionMaskSpec::causal();
    return AttentionMaskSpec::shared_prompt(P, std::vector<int>(lens, lens + G));
}

}  // namespace

extern "C" {

long ref_param_count(const CCfg* c) {
    return guarded([&] { return (int)ModelParams::init(to_cfg(c), 0).flat().size(); });
}

int ref_init_params(const CCfg* c, unsigned long long seed, double* out) {
    return guarded([&] {
        ModelParams p = ModelParams::init(to_cfg(c), seed);
        std::memcpy(out, p.flat().data(), p.flat().size() * sizeof(double));
        return 0;
    });
}

// pack_group (packing.cpp:7-45).  Returns T.
int ref_pack(const int* prompt, int P, const int* resp_flat, const int* lens, int G, int max_seq,
             int* tokens, int* labels, int* positions, int* span_start) {
    return guarded([&] {
        std::vector<TokenId> pr(prompt, prompt + P);
        std::vector<std::vector<TokenId>> rs;
        int off = 0;
        for (int g = 0; g < G; ++g) {
            rs.emplace_back(resp_flat + off, resp_flat + off + lens[g]);
            off += lens[g];
        }
        PackedGroup pg = pack_group(pr, rs, max_seq);
        std::copy(pg.tokens.begin(), pg.tokens.end(), tokens);
        std::copy(pg.labels.begin(), pg.labels.end(), labels);
        std::copy(pg.positions.begin(), pg.positions.end(), positions);
        for (size_t g = 0; g < pg.spans.size(); ++g) span_start[g] = pg.spans[g].start;
        return (int)pg.tokens.size();
    });
}

// forward_logprobs (+ backward when upstream != nullptr; grad ADDED to grad_acc).
int ref_forward(const CCfg* c, const double* w, const int* tokens, const int* positions, int T,
                int P, const int* lens, int G, const int* labels, double* lp_out,
                const double* upstream, double* grad_acc) {
    return guarded([&] {
        ModelParams p = params_from(c, w);
        auto mask = mask_from(P, lens, G);
        std::span<const TokenId> tk(tokens, T);
        std::span<const int> ps(positions, T);
        std::span<const std::int32_t> lb(labels, T);
        ForwardResult f = forward_logprobs(p, tk, ps, mask, lb, upstream != nullptr);
        std::copy(f.logprobs.begin(), f.logprobs.end(), lp_out);
        if (upstream) {
            GradBuffer g = backward(p, f, std::span<const double>(upstream, f.logprobs.size()));
            for (size_t i = 0; i < g.flat().size(); ++i) grad_acc[i] += g.flat()[i];
        }
        return (int)f.logprobs.size();
    });
}

int ref_logprob_rows(const CCfg* c, const double* w, const int* tokens, const int* positions,
                     int T, int P, const int* lens, int G, double* rows) {
    return guarded([&] {
        ModelParams p = params_from(c, w);
        auto r = forward_logprob_rows(p, std::span<const TokenId>(tokens, T),
                                      std::span<const int>(positions, T), mask_from(P, lens, G));
        std::copy(r.begin(), r.end(), rows);
        return 0;
    });
}

int ref_group_advantages(const double* r, int G, int mean_only, double* a) {
    return guarded([&] {
        auto v = mean_only ? group_advantages_mean_only(std::span<const double>(r, G))
                           : group_advantages(std::span<const double>(r, G));
        std::copy(v.begin(), v.end(), a);
        return 0;
    });
}

int ref_sample_terms(const double* lp, const double* old, const double* ref, int n, double A,
                     double eps, double beta, int gran, double* upstream, double* out4) {
    return guarded([&] {
        Sample s;
        s.response.assign(n, 4);
        s.old_logprobs.assign(old, old + n);
        s.ref_logprobs.assign(ref, ref + n);
        s.advantage = A;
        SampleTerms st = per_sample_terms(s, std::span<const double>(lp, n), eps, beta,
                                          gran ? LossGranularity::sequence : LossGranularity::token);
        std::copy(st.upstream.begin(), st.upstream.end(), upstream);
        out4[0] = st.clip_term;
        out4[1] = st.kl;
        out4[2] = st.clipped_units;
        out4[3] = st.total_units;
        return 0;
    });
}

double ref_clipped_term(double lp, double old, double A, double eps) {
    return clipped_term(lp, old, A, eps);
}
double ref_kl_term(double lp, double r) { return kl_term(lp, r); }

}  // extern "C"

namespace {

// Pipeline::train_microbatch shared-prompt branch (pipeline.cpp:97-141),
// replayed through the reference's public operator API.
void microbatch(TriModel& tm, const std::vector<TokenId>& prompt,
                const std::vector<std::vector<TokenId>>& responses,
                const std::vector<double>& advantages, double eps, double beta,
                LossGranularity gran, GradBuffer& grads, double* stats5, double* lp3,
                const double* rollout_old = nullptr) {
    PackedGroup packed = pack_group(prompt, responses, tm.policy.config().max_seq_len);
    TriForwardResult tri;
    if (!rollout_old) {  // one_step_delayed (pipeline.cpp:110-112)
        tri = trimodel_forward(tm, packed.tokens, packed.positions, packed.mask, packed.labels);
    } else {  // rollout_weights: policy + reference only, old log-probs from the rollout (pipeline.cpp:113-119)
        tri.policy = forward_logprobs(tm.policy, packed.tokens, packed.positions, packed.mask, packed.labels, true);
        tri.ref_logprobs =
            forward_logprobs(tm.reference, packed.tokens, packed.positions, packed.mask, packed.labels).logprobs;
        tri.old_logprobs.assign(rollout_old, rollout_old + tri.policy.logprobs.size());
    }
    auto pol = extract_response_logprobs(tri.policy.logprobs, packed);
    auto ref = extract_response_logprobs(tri.ref_logprobs, packed);
    auto old = extract_response_logprobs(tri.old_logprobs, packed);
    std::vector<double> upstream;
    for (size_t j = 0; j < responses.size(); ++j) {
        Sample s;
        s.prompt = prompt;
        s.response = responses[j];
        s.advantage = advantages[j];
        s.old_logprobs = old[j];
        s.ref_logprobs = ref[j];
        SampleTerms st = per_sample_terms(s, pol[j], eps, beta, gran);
        if (stats5) {
            stats5[0] += st.clip_term - beta * st.kl;
            stats5[1] += st.clip_term;
            stats5[2] += st.kl;
            stats5[3] += st.clipped_units;
            stats5[4] += st.total_units;
        }
        for (double u : st.upstream) upstream.push_back(-u);
    }
    GradBuffer gb = backward(tm.policy, tri.policy, upstream);
    grads.accumulate(gb);
    if (lp3) {
        size_t S = tri.policy.logprobs.size();
        std::copy(tri.policy.logprobs.begin(), tri.policy.logprobs.end(), lp3);
        std::copy(tri.old_logprobs.begin(), tri.old_logprobs.end(), lp3 + S);
        std::copy(tri.ref_logprobs.begin(), tri.ref_logprobs.end(), lp3 + 2 * S);
    }
}

}  // namespace

extern "C" {

// One shared-prompt micro-batch through the reference.  grad_acc += gradient.
int ref_train_microbatch(const CCfg* c, const double* w_pol, const double* w_old,
                         const double* w_ref, const int* prompt, int P, const int* resp_flat,
                         const int* lens, int G, const double* adv, double eps, double beta,
                         int gran, double* grad_acc, double* stats5, double* lp3) {
    return guarded([&] {
        TriModel tm = TriModel::init(to_cfg(c), 0);
        const size_t n = tm.policy.flat().size();
        std::memcpy(tm.policy.flat_mut().data(), w_pol, n * sizeof(double));
        std::memcpy(tm.old_policy.flat_mut().data(), w_old, n * sizeof(double));
        std::memcpy(tm.reference.flat_mut().data(), w_ref, n * sizeof(double));
        std::vector<TokenId> pr(prompt, prompt + P);
        std::vector<std::vector<TokenId>> rs;
        int off = 0;
        for (int g = 0; g < G; ++g) {
            rs.emplace_back(resp_flat + off, resp_flat + off + lens[g]);
            off += lens[g];
        }
        GradBuffer grads(tm.policy);
        microbatch(tm, pr, rs, std::vector<double>(adv, adv + G), eps, beta,
                   gran ? LossGranularity::sequence : LossGranularity::token, grads, stats5, lp3);
        for (size_t i = 0; i < n; ++i) grad_acc[i] += grads.flat()[i];
        return (int)(P + off);
    });
}

// The training half of Pipeline::run_iteration (pipeline.cpp:263-352) through the reference API:
// n_mb shared-prompt micro-batches (micro-batch b: prompt b, lens[mb_off[b] .. mb_off[b+1]),
// advantages alongside, optional rollout old log-probs), accumulated in order, then
// set_micro_step_count(N*G) -> snapshot_old_policy -> apply_update(lr).  w_pol / w_old are
// replaced by the updated policy / snapshot; stats5 summed.
int ref_train_iteration(const CCfg* c, double* w_pol, double* w_old, const double* w_ref, int n_mb,
                        const int* prompt_flat, const int* prompt_lens, const int* resp_flat, const int* lens,
                        const int* mb_off, const double* adv, const double* rollout_old, double eps, double beta,
                        int gran, double lr, int total_samples, double* stats5) {
    return guarded([&] {
        TriModel tm = TriModel::init(to_cfg(c), 0);
        const size_t n = tm.policy.flat().size();
        std::memcpy(tm.policy.flat_mut().data(), w_pol, n * sizeof(double));
        std::memcpy(tm.old_policy.flat_mut().data(), w_old, n * sizeof(double));
        std::memcpy(tm.reference.flat_mut().data(), w_ref, n * sizeof(double));
        GradBuffer grad_acc(tm.policy);
        int po = 0, ro = 0, so = 0;
        for (int b = 0; b < n_mb; ++b) {
            std::vector<TokenId> pr(prompt_flat + po, prompt_flat + po + prompt_lens[b]);
            po += prompt_lens[b];
            std::vector<std::vector<TokenId>> rs;
            std::vector<double> a;
            int S = 0;
            for (int k = mb_off[b]; k < mb_off[b + 1]; ++k) {
                rs.emplace_back(resp_flat + ro, resp_flat + ro + lens[k]);
                ro += lens[k];
                S += lens[k];
                a.push_back(adv[k]);
            }
            microbatch(tm, pr, rs, a, eps, beta, gran ? LossGranularity::sequence : LossGranularity::token, grad_acc,
                       stats5, nullptr, rollout_old ? rollout_old + so : nullptr);
            so += S;
        }
        grad_acc.set_micro_step_count(total_samples);
        tm.snapshot_old_policy();
        tm.policy.apply_update(grad_acc, lr);
        std::memcpy(w_pol, tm.policy.flat().data(), n * sizeof(double));
        std::memcpy(w_old, tm.old_policy.flat().data(), n * sizeof(double));
        return 0;
    });
}

// save_checkpoint / load_checkpoint (model.cpp:924-987) of the reference itself:
// golden PARLCKP1 files and the check that the reference reads the GPU path's files.
int ref_save_checkpoint(const CCfg* c, const double* w, unsigned long long seed, const char* path) {
    return guarded([&] {
        ModelParams p = ModelParams::init(to_cfg(c), seed);
        if (w) std::memcpy(p.flat_mut().data(), w, p.flat().size() * sizeof(double));
        save_checkpoint(path, p);
        return 0;
    });
}

// Returns the parameter count; fills cfg, version, seed and (if w) the weights.
long ref_load_checkpoint(const char* path, CCfg* c, double* w, unsigned long long* version,
                         unsigned long long* seed) {
    try {
        ModelParams p = load_checkpoint(path);
        const auto& m = p.config();
        *c = CCfg{m.vocab_size, m.d_model, m.n_layers, m.n_heads, m.d_ff, m.max_seq_len};
        *version = p.version();
        *seed = p.init_seed();
        if (w) std::memcpy(w, p.flat().data(), p.flat().size() * sizeof(double));
        return (long)p.flat().size();
    } catch (const IoError&) {
        return -8;
    } catch (const NumericError&) {
        return -5;
    } catch (...) {
        return -99;
    }
}

// sample_tokens (model.cpp:843-900).  Returns the number of tokens written to out.
int ref_sample_tokens(const CCfg* c, const double* w, const int* prompt, int P, int max_new, double temperature,
                      unsigned long long seed, int* out) {
    return guarded([&] {
        ModelParams p = params_from(c, w);
        auto toks = sample_tokens(p, std::span<const TokenId>(prompt, P), max_new, temperature, seed);
        std::copy(toks.begin(), toks.end(), out);
        return (int)toks.size();
    });
}

// CPU baseline: `threads` independent workers, each with its own TriModel
// (SPEC.md:113 allows distinct instances concurrently), each running `reps`
// shared-prompt micro-batches of P + G x R tokens with random tokens in
// [4, V).  Model init is excluded: workers initialise, meet at a barrier, and
// the returned wall seconds cover only the micro-batch loops (max over workers).
double ref_bench_microbatch(const CCfg* c, unsigned long long seed, int P, int G, int R, int reps,
                            int threads) {
    std::vector<std::thread> pool;
    std::vector<double> secs(threads, 0.0);
    std::atomic<int> ready{0};
    for (int th = 0; th < threads; ++th) {
        pool.emplace_back([=, &ready, &secs] {
            ModelConfig mc = to_cfg(c);
            TriModel tm = TriModel::init(mc, seed);
            Rng rng(mix_seed(seed, 123 + th));
            std::vector<std::vector<TokenId>> prompts, resps_flat;
            ready.fetch_add(1);
            while (ready.load() < threads) std::this_thread::yield();
            auto t0 = std::chrono::steady_clock::now();
            for (int rep = 0; rep < reps; ++rep) {
                std::vector<TokenId> prompt(P);
                for (auto& t : prompt) t = rng.uniform_int(4, mc.vocab_size - 1);
                std::vector<std::vector<TokenId>> rs(G, std::vector<TokenId>(R));
                for (auto& r : rs)
                    for (auto& t : r) t = rng.uniform_int(4, mc.vocab_size - 1);
                std::vector<double> rewards(G);
                for (auto& r : rewards) r = rng.uniform();
                std::vector<double> adv = group_advantages(rewards);
                GradBuffer grads(tm.policy);
                microbatch(tm, prompt, rs, adv, 0.2, 0.04, LossGranularity::token, grads, nullptr,
                           nullptr);
            }
            secs[th] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        });
    }
    for (auto& t : pool) t.join();
    double mx = 0.0;
    for (double v : secs) mx = v > mx ? v : mx;
    return mx;
}

// Persistent CPU-baseline workers (bench.py --impl reference): the TriModels are built once
// (ref_bench_open, in parallel), then every ref_bench_run times `reps` shared-prompt
// micro-batches per worker, all workers concurrently; returns the max wall seconds.
struct RefBench {
    ModelConfig mc;
    std::vector<std::unique_ptr<TriModel>> tms;
    std::vector<Rng> rngs;
};

void* ref_bench_open(const CCfg* c, unsigned long long seed, int threads) {
    auto* b = new RefBench();
    b->mc = to_cfg(c);
    b->tms.resize(threads);
    for (int th = 0; th < threads; ++th) b->rngs.emplace_back(mix_seed(seed, 123 + th));
    std::vector<std::thread> pool;
    for (int th = 0; th < threads; ++th)
        pool.emplace_back([b, th, seed] { b->tms[th] = std::make_unique<TriModel>(TriModel::init(b->mc, seed)); });
    for (auto& t : pool) t.join();
    return b;
}

double ref_bench_run(void* h, int P, int G, int R, int reps) {
    auto* b = static_cast<RefBench*>(h);
    const int threads = (int)b->tms.size();
    std::vector<std::thread> pool;
    std::vector<double> secs(threads, 0.0);
    std::atomic<int> ready{0};
    for (int th = 0; th < threads; ++th) {
        pool.emplace_back([=, &ready, &secs] {
            TriModel& tm = *b->tms[th];
            Rng& rng = b->rngs[th];
            const ModelConfig& mc = b->mc;
            ready.fetch_add(1);
            while (ready.load() < threads) std::this_thread::yield();
            auto t0 = std::chrono::steady_clock::now();
            for (int rep = 0; rep < reps; ++rep) {
                std::vector<TokenId> prompt(P);
                for (auto& t : prompt) t = rng.uniform_int(4, mc.vocab_size - 1);
                std::vector<std::vector<TokenId>> rs(G, std::vector<TokenId>(R));
                for (auto& r : rs)
                    for (auto& t : r) t = rng.uniform_int(4, mc.vocab_size - 1);
                std::vector<double> rewards(G);
                for (auto& r : rewards) r = rng.uniform();
                std::vector<double> adv = group_advantages(rewards);
                GradBuffer grads(tm.policy);
                microbatch(tm, prompt, rs, adv, 0.2, 0.04, LossGranularity::token, grads, nullptr, nullptr);
            }
            secs[th] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        });
    }
    for (auto& t : pool) t.join();
    double mx = 0.0;
    for (double v : secs) mx = v > mx ? v : mx;
    return mx;
}

void ref_bench_close(void* h) { delete static_cast<RefBench*>(h); }

}  // extern "C"
