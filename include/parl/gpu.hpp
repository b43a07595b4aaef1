// parl/gpu.hpp — the fused device micro-step, for callers that replace the body
// of Pipeline::train_microbatch (proj/src/pipeline.cpp:92-172) and the update of
// run_iteration (pipeline.cpp:346-352); see INTEGRATION.md.  Namespace
// parl::gpu, so it links beside the reference's own TriModel (pipeline.hpp:41-60).
//
//   TriModel / trimodel_forward : the three roles as one layer-interleaved device
//                                 forward (grouped GEMM / attention launches)
//   train_microbatch            : pack -> tri-model forward -> K7 loss -> backward ->
//                                 accumulate, one call, only the loss scalars return;
//                                 both old-policy modes (pipeline.cpp:107-119), both
//                                 branches (shared-prompt packed / per-sample causal)
//   finish_iteration            : divisor N*G, snapshot old <- policy, apply_update
#pragma once

#include <span>
#include <vector>

#include "parl/grpo.hpp"
#include "parl/model.hpp"
#include "parl/packing.hpp"

namespace parl::gpu {

enum class OldPolicyMode { rollout_weights, one_step_delayed };  // pipeline.hpp:16-19

struct HyperParams {  // pipeline.hpp:29-37
    double lr = 0.1;
    double epsilon = 0.2;
    double beta = 0.04;
    LossGranularity granularity = LossGranularity::token;
    OldPolicyMode old_policy = OldPolicyMode::one_step_delayed;
    bool advantage_mean_only = false;
    parl_hyper c() const {
        return {epsilon, beta, granularity == LossGranularity::token ? 0 : 1, advantage_mean_only ? 1 : 0};
    }
};

struct MicrobatchStats {  // Pipeline::MicrobatchStats, pipeline.hpp:109-116
    double objective_sum = 0.0, clip_sum = 0.0, kl_sum = 0.0;
    long clipped_units = 0, total_units = 0;
    int micro_batches = 0;
};

struct TriModel {  // pipeline.hpp:41-48
    ModelParams policy, old_policy, reference;
    static TriModel init(const ModelConfig& cfg, std::uint64_t seed, Device& dev = Device::get()) {
        ModelParams p = ModelParams::init(cfg, seed, dev);
        return TriModel{p.clone(), p.clone(), std::move(p)};
    }
    void snapshot_old_policy() {  // pipeline.cpp:20, a device copy
        detail::check(parl_model_copy(old_policy.handle(), policy.handle(), 0, 0.0), policy.device().ctx());
        old_policy.refresh();
    }
};

struct TriForwardResult {
    ForwardResult policy;
    std::vector<double> old_logprobs, ref_logprobs;
};

// pipeline.cpp:22-30 as one grouped device forward (identical weights give identical outputs)
inline TriForwardResult trimodel_forward(const TriModel& tm, std::span<const TokenId> tokens,
                                         std::span<const int> positions, const AttentionMaskSpec& mask,
                                         std::span<const std::int32_t> labels) {
    auto g = detail::sequence(tm.policy, tokens, positions, mask, labels);
    if (!labels.data()) throw ShapeError("forward_logprobs requires labels");
    parl_ctx_t ctx = tm.policy.device().ctx();
    parl_act_t act = nullptr;
    detail::check(parl_trimodel_forward(ctx, tm.policy.handle(), tm.old_policy.handle(), tm.reference.handle(), g.get(),
                                        &act),
                  ctx);
    TriForwardResult r;
    const int S = parl_group_scored(g.get());
    r.policy.logprobs.resize(S);
    r.old_logprobs.resize(S);
    r.ref_logprobs.resize(S);
    detail::check(parl_group_logprobs(g.get(), 0, r.policy.logprobs.data()), ctx);
    detail::check(parl_group_logprobs(g.get(), 1, r.old_logprobs.data()), ctx);
    detail::check(parl_group_logprobs(g.get(), 2, r.ref_logprobs.data()), ctx);
    std::vector<std::int32_t> sp(S);
    detail::check(parl_group_download(g.get(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, sp.data()), ctx);
    r.policy.scored_positions.assign(sp.begin(), sp.end());
    r.policy.cache = std::make_shared<ForwardCache>();
    r.policy.cache->group = g;
    r.policy.cache->act = std::shared_ptr<parl_act_s>(act, [](parl_act_t x) { parl_act_destroy(x); });
    r.policy.cache->owner = &tm.policy;
    return r;
}

namespace detail2 {
inline void add_stats(MicrobatchStats& stats, const parl_loss_stats& s) {
    stats.objective_sum += s.objective_sum;
    stats.clip_sum += s.clip_sum;
    stats.kl_sum += s.kl_sum;
    stats.clipped_units += (long)s.clipped_units;
    stats.total_units += (long)s.total_units;
}

// one device micro-step over a packed / causal sequence: loss scalars of this call only
inline parl_loss_stats fused_step(TriModel& tm, parl_group_t g, const std::vector<double>& adv,
                                  const std::vector<double>* rollout_old, const HyperParams& hp, GradBuffer& grads) {
    parl_ctx_t ctx = tm.policy.device().ctx();
    detail::check(parl_stats_reset(ctx), ctx);
    parl_model_t old = tm.old_policy.handle();
    if (hp.old_policy == OldPolicyMode::rollout_weights) {  // policy + reference only (pipeline.cpp:113-119)
        if (!rollout_old || (int)rollout_old->size() != parl_group_scored(g))
            throw ShapeError("rollout_weights mode needs the samples' old_logprobs");
        detail::check(parl_group_set_logprobs(g, 1, rollout_old->data()), ctx);
        old = nullptr;
    }
    parl_hyper h = hp.c();
    parl_loss_stats s{};
    detail::check(parl_train_microbatch(ctx, tm.policy.handle(), old, tm.reference.handle(), g, nullptr, adv.data(), &h,
                                        grads.handle(), &s),
                  ctx);
    grads.touched();
    return s;
}
}  // namespace detail2

// Pipeline::train_microbatch (pipeline.cpp:92-172) on the device.  `samples` carry their
// group advantage (and, in rollout_weights mode, old_logprobs); the shared-prompt branch
// packs them into one sequence (all samples of one group), the other scores each sample
// under a causal mask.  grads accumulates -upstream-seeded gradients, one micro-step count
// per backward call (the caller sets N*G before the update, pipeline.cpp:350).
inline void train_microbatch(TriModel& tm, std::vector<Sample>& samples, GradBuffer& grads, MicrobatchStats& stats,
                             const HyperParams& hp, bool shared_prompt) {
    const int max_seq = tm.policy.config().max_seq_len;
    if (shared_prompt) {
        for (const auto& s : samples)
            if (s.group_id != samples[0].group_id) throw BarrierError("packed micro-batch mixes groups");
        std::vector<std::vector<TokenId>> responses;
        std::vector<double> adv, old;
        for (const auto& s : samples) {
            responses.push_back(s.response);
            adv.push_back(s.advantage);
            old.insert(old.end(), s.old_logprobs.begin(), s.old_logprobs.end());
        }
        PackedGroup packed = pack_group(samples[0].prompt, responses, max_seq, tm.policy.device());
        detail2::add_stats(stats, detail2::fused_step(tm, packed.device.get(), adv, &old, hp, grads));
    } else {
        for (auto& s : samples) {  // causal_scoring_inputs, pipeline.cpp:79-88
            std::vector<TokenId> tokens(s.prompt.begin(), s.prompt.end());
            tokens.insert(tokens.end(), s.response.begin(), s.response.end());
            std::vector<int> positions(tokens.size());
            for (std::size_t i = 0; i < tokens.size(); ++i) positions[i] = static_cast<int>(i);
            std::vector<std::int32_t> labels(tokens.size(), kIgnoreLabel);
            for (std::size_t i = 0; i < s.response.size(); ++i) labels[s.prompt.size() + i] = s.response[i];
            auto g = detail::sequence(tm.policy, tokens, positions, AttentionMaskSpec::causal(), labels);
            const std::vector<double> adv{s.advantage};
            detail2::add_stats(stats, detail2::fused_step(tm, g.get(), adv, &s.old_logprobs, hp, grads));
        }
    }
    ++stats.micro_batches;
}

// Convenience: one shared-prompt group with its rewards (advantages from the whole group).
inline MicrobatchStats train_microbatch(TriModel& tm, std::span<const TokenId> prompt,
                                        const std::vector<std::vector<TokenId>>& responses,
                                        std::span<const double> rewards, const HyperParams& hp, GradBuffer& grads,
                                        MicrobatchStats& stats) {
    if (rewards.size() != responses.size()) throw ShapeError("one reward per response required");
    const std::vector<double> adv = hp.advantage_mean_only ? group_advantages_mean_only(rewards) : group_advantages(rewards);
    std::vector<Sample> samples(responses.size());
    for (std::size_t j = 0; j < responses.size(); ++j) {
        samples[j].prompt.assign(prompt.begin(), prompt.end());
        samples[j].response = responses[j];
        samples[j].advantage = adv[j];
        samples[j].reward = rewards[j];
    }
    MicrobatchStats m;
    train_microbatch(tm, samples, grads, m, hp, true);
    stats.objective_sum += m.objective_sum;
    stats.clip_sum += m.clip_sum;
    stats.kl_sum += m.kl_sum;
    stats.clipped_units += m.clipped_units;
    stats.total_units += m.total_units;
    stats.micro_batches += m.micro_batches;
    return m;
}

// run_iteration's update (pipeline.cpp:346-352): divisor = the batch's N*G samples (all
// ranks' samples when the batch is sharded and `grads` was allreduced), snapshot, update.
inline void finish_iteration(TriModel& tm, GradBuffer& grads, int total_samples, double lr) {
    grads.set_micro_step_count(total_samples);
    tm.snapshot_old_policy();
    tm.policy.apply_update(grads, lr);
}

// The G rollouts of one prompt on the KV-cached decoder (parl_sample_group): the prompt's K/V
// prefilled once and shared; sequence k == sample_tokens(params, prompt, max_new_tokens,
// temperature, seeds[k]).  old_logprobs (optional): each sampled token's log-prob under params.
inline std::vector<std::vector<TokenId>> sample_group(const ModelParams& params, std::span<const TokenId> prompt,
                                                      int max_new_tokens, double temperature,
                                                      std::span<const std::uint64_t> seeds,
                                                      std::vector<std::vector<double>>* old_logprobs = nullptr) {
    const int n = (int)seeds.size(), mx = std::max(max_new_tokens, 1);
    std::vector<TokenId> out((std::size_t)n * mx);
    std::vector<int> lens(n);
    std::vector<double> lp(old_logprobs ? (std::size_t)n * mx : 0);
    detail::check(parl_sample_group(params.device().ctx(), params.handle(), prompt.data(), (int)prompt.size(), n,
                                    max_new_tokens, temperature, seeds.data(), out.data(), lens.data(),
                                    old_logprobs ? lp.data() : nullptr),
                  params.device().ctx());
    std::vector<std::vector<TokenId>> r(n);
    if (old_logprobs) old_logprobs->assign(n, {});
    for (int k = 0; k < n; ++k) {
        r[k].assign(out.begin() + (std::size_t)k * mx, out.begin() + (std::size_t)k * mx + lens[k]);
        if (old_logprobs)
            (*old_logprobs)[k].assign(lp.begin() + (std::size_t)k * mx, lp.begin() + (std::size_t)k * mx + lens[k]);
    }
    return r;
}

// RolloutService::score_logprobs (rollout.cpp:52-66): response log-probs under a causal forward
inline std::vector<double> score_logprobs(const ModelParams& params, std::span<const TokenId> prompt,
                                          std::span<const TokenId> response) {
    if (response.empty()) return {};
    std::vector<TokenId> tokens(prompt.begin(), prompt.end());
    tokens.insert(tokens.end(), response.begin(), response.end());
    std::vector<int> positions(tokens.size());
    for (std::size_t i = 0; i < tokens.size(); ++i) positions[i] = static_cast<int>(i);
    std::vector<std::int32_t> labels(tokens.size(), kIgnoreLabel);
    for (std::size_t i = 0; i < response.size(); ++i) labels[prompt.size() + i] = response[i];
    return forward_logprobs(params, tokens, positions, AttentionMaskSpec::causal(), labels).logprobs;
}

}  // namespace parl::gpu
