// parl/grpo.hpp — drop-in for proj/include/parl/grpo.hpp (grpo.hpp:12-98).
// The loss math (group advantages, clipped / KL terms, per-sample terms and the
// micro-batch loss) runs on the device in the K7 kernels, with fp64 arithmetic
// on this host-array API; the batch plumbing (BatchSpec, split_microbatches) is
// host bookkeeping as in the reference (grpo.cpp:9-22, 186-213).
#pragma once

#include <algorithm>
#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "parl/errors.hpp"
#include "parl/model.hpp"

namespace parl {

struct Sample {
    std::int64_t prompt_id = 0;
    int group_slot = 0;
    int rollout_index = 0;
    std::int64_t group_id = 0;
    std::vector<TokenId> prompt;
    std::vector<TokenId> response;
    double reward = 0.0;
    double advantage = 0.0;
    std::vector<double> old_logprobs;
    std::vector<double> ref_logprobs;
    double completion_time = 0.0;
};

struct BatchSpec {
    int prompts_per_batch = 0;   // N
    int rollouts_per_group = 0;  // G
    int microbatch_size = 0;     // m

    int batch_samples() const { return prompts_per_batch * rollouts_per_group; }
    int micro_count() const { return batch_samples() / microbatch_size; }
    void validate() const {  // grpo.cpp:9-22
        if (prompts_per_batch < 1) throw ConfigError("prompts_per_batch must be >= 1");
        if (rollouts_per_group < 2) throw ConfigError("rollouts_per_group must be >= 2 (group advantages need G >= 2)");
        if (microbatch_size < 1) throw ConfigError("microbatch_size must be >= 1");
        const int total = batch_samples();
        if (total % microbatch_size != 0) {
            std::string valid;
            for (int m = 1; m <= total; ++m)
                if (total % m == 0) valid += (valid.empty() ? "" : ", ") + std::to_string(m);
            throw ConfigError("N*G = " + std::to_string(total) + " not divisible by m = " +
                              std::to_string(microbatch_size) + "; valid m values: " + valid);
        }
    }
};

enum class LossGranularity { token, sequence };

struct LossReport {
    double objective = 0.0;
    double clip_term_mean = 0.0;
    double kl_mean = 0.0;
    double clip_fraction = 0.0;
    long token_count = 0;
};

// grpo.cpp:24-38 / 40-48
inline std::vector<double> group_advantages(std::span<const double> rewards) {
    Device& dev = Device::get();
    std::vector<double> a(rewards.size());
    detail::check(parl_group_advantages(dev.ctx(), rewards.data(), (int)rewards.size(), 0, a.data()), dev.ctx());
    return a;
}
inline std::vector<double> group_advantages_mean_only(std::span<const double> rewards) {
    Device& dev = Device::get();
    std::vector<double> a(rewards.size());
    detail::check(parl_group_advantages(dev.ctx(), rewards.data(), (int)rewards.size(), 1, a.data()), dev.ctx());
    return a;
}

// grpo.cpp:95-108
inline double clipped_term(double logp_new, double logp_old, double advantage, double epsilon) {
    Device& dev = Device::get();
    double v = 0.0;
    detail::check(parl_clipped_term(dev.ctx(), logp_new, logp_old, advantage, epsilon, &v), dev.ctx());
    return v;
}
inline double kl_term(double logp_new, double logp_ref) {
    Device& dev = Device::get();
    double v = 0.0;
    detail::check(parl_kl_term(dev.ctx(), logp_new, logp_ref, &v), dev.ctx());
    return v;
}

struct SampleTerms {
    double clip_term = 0.0;
    double kl = 0.0;
    int clipped_units = 0;
    int total_units = 0;
    std::vector<double> upstream;
};

// grpo.cpp:111-151
inline SampleTerms per_sample_terms(const Sample& sample, std::span<const double> policy_logprobs, double epsilon,
                                    double beta, LossGranularity granularity) {
    const std::size_t T = sample.response.size();
    if (policy_logprobs.size() != T || sample.old_logprobs.size() != T || sample.ref_logprobs.size() != T)
        throw ShapeError("logprob vectors not aligned with response length " + std::to_string(T));
    if (T == 0) throw ShapeError("sample has empty response");
    Device& dev = Device::get();
    SampleTerms st;
    st.upstream.assign(T, 0.0);
    parl_sample_terms c{};
    detail::check(parl_per_sample_terms(dev.ctx(), policy_logprobs.data(), sample.old_logprobs.data(),
                                        sample.ref_logprobs.data(), (int)T, sample.advantage, epsilon, beta,
                                        granularity == LossGranularity::token ? 0 : 1, st.upstream.data(), &c),
                  dev.ctx());
    st.clip_term = c.clip_term;
    st.kl = c.kl;
    st.clipped_units = c.clipped_units;
    st.total_units = c.total_units;
    return st;
}

struct MicrobatchLoss {
    double loss = 0.0;
    std::vector<std::vector<double>> upstream;
    LossReport report;
};

// grpo.cpp:153-184
inline MicrobatchLoss grpo_microbatch_loss(std::span<const Sample> samples,
                                           const std::vector<std::vector<double>>& policy_logprobs, double epsilon,
                                           double beta, LossGranularity granularity) {
    if (samples.empty()) throw ShapeError("empty micro-batch");
    if (policy_logprobs.size() != samples.size()) throw ShapeError("policy logprob count != sample count");
    std::vector<std::int32_t> lens;
    std::vector<double> lp, old, ref, adv;
    for (std::size_t j = 0; j < samples.size(); ++j) {
        const Sample& s = samples[j];
        const std::size_t T = s.response.size();
        if (policy_logprobs[j].size() != T || s.old_logprobs.size() != T || s.ref_logprobs.size() != T)
            throw ShapeError("logprob vectors not aligned with response length " + std::to_string(T));
        if (T == 0) throw ShapeError("sample has empty response");
        lens.push_back((std::int32_t)T);
        lp.insert(lp.end(), policy_logprobs[j].begin(), policy_logprobs[j].end());
        old.insert(old.end(), s.old_logprobs.begin(), s.old_logprobs.end());
        ref.insert(ref.end(), s.ref_logprobs.begin(), s.ref_logprobs.end());
        adv.push_back(s.advantage);
    }
    Device& dev = Device::get();
    std::vector<double> up(lp.size());
    parl_loss_report rep{};
    MicrobatchLoss out;
    detail::check(parl_grpo_microbatch_loss(dev.ctx(), (int)samples.size(), lens.data(), lp.data(), old.data(),
                                            ref.data(), adv.data(), epsilon, beta,
                                            granularity == LossGranularity::token ? 0 : 1, up.data(), &rep, &out.loss),
                  dev.ctx());
    std::size_t c = 0;
    for (int n : lens) {
        out.upstream.emplace_back(up.begin() + c, up.begin() + c + n);
        c += n;
    }
    out.report.objective = rep.objective;
    out.report.clip_term_mean = rep.clip_term_mean;
    out.report.kl_mean = rep.kl_mean;
    out.report.clip_fraction = rep.clip_fraction;
    out.report.token_count = rep.token_count;
    return out;
}

enum class SplitPolicy { arrival_order, group_major };

// grpo.cpp:186-213 (host batch plumbing)
inline std::vector<std::vector<Sample>> split_microbatches(std::vector<Sample> batch, int m, SplitPolicy policy) {
    if (m < 1) throw ConfigError("microbatch size must be >= 1");
    const int total = static_cast<int>(batch.size());
    if (total % m != 0) {
        std::string valid;
        for (int k = 1; k <= total; ++k)
            if (total % k == 0) valid += (valid.empty() ? "" : ", ") + std::to_string(k);
        throw ConfigError("batch of " + std::to_string(total) + " samples not divisible by m = " + std::to_string(m) +
                          "; valid m values: " + valid);
    }
    if (policy == SplitPolicy::group_major)
        std::stable_sort(batch.begin(), batch.end(), [](const Sample& a, const Sample& b) {
            if (a.group_id != b.group_id) return a.group_id < b.group_id;
            return a.rollout_index < b.rollout_index;
        });
    std::vector<std::vector<Sample>> out;
    out.reserve(total / m);
    for (int i = 0; i < total; i += m) out.emplace_back(batch.begin() + i, batch.begin() + i + m);
    return out;
}

}  // namespace parl
