// parl_gpu.hpp — C++ drop-in layer over the C-ABI (parl_gpu.h).
//
// Mirrors the reference operator interface of the hot path, in namespace
// `parl`, with the same names, argument meaning and exception types:
//
//   errors            proj/include/parl/errors.hpp:9-46
//   ModelConfig       proj/include/parl/model.hpp:26-36
//   AttentionMaskSpec proj/include/parl/model.hpp:41-55
//   ModelParams       proj/include/parl/model.hpp:64-106  (device-resident weights)
//   GradBuffer        proj/include/parl/model.hpp:109-134 (device fp32 accumulator)
//   forward_logprobs  proj/include/parl/model.hpp:153-158
//   backward          proj/include/parl/model.hpp:162-163
//   forward_logprob_rows  model.hpp:168-171
//   PackedGroup / pack_group / extract_response_logprobs  packing.hpp:13-35
//   TriModel / trimodel_forward  pipeline.hpp:41-60
//   train_microbatch  Pipeline::train_microbatch shared-prompt branch, pipeline.cpp:97-141
//
// Differences a caller sees: weights live on the GPU (ModelParams::flat()
// returns a host copy), log-probs are computed in fp32 (PARL_PREC_FP32) or
// with bf16 tensor-core operands (PARL_PREC_BF16), and train_microbatch keeps
// the whole micro-step on the device (only the loss scalars come back).
// Header-only; link with libparl_gpu.so.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "parl_gpu.h"

namespace parl {

using TokenId = std::int32_t;
constexpr TokenId kPadToken = 0, kBosToken = 1, kEosToken = 2, kSepToken = 3, kFirstPayloadToken = 4;
constexpr std::int32_t kIgnoreLabel = -1;

// ---- errors (errors.hpp:9-46) ---------------------------------------------
#define PARL_GPU_ERROR_TYPE(Name) \
    struct Name : std::runtime_error { explicit Name(const std::string& m) : std::runtime_error(m) {} };
PARL_GPU_ERROR_TYPE(ConfigError)
PARL_GPU_ERROR_TYPE(ShapeError)
PARL_GPU_ERROR_TYPE(VocabError)
PARL_GPU_ERROR_TYPE(LifecycleError)
PARL_GPU_ERROR_TYPE(NumericError)
PARL_GPU_ERROR_TYPE(BarrierError)
PARL_GPU_ERROR_TYPE(StallError)
PARL_GPU_ERROR_TYPE(IoError)
PARL_GPU_ERROR_TYPE(DeviceError)
#undef PARL_GPU_ERROR_TYPE

inline void check(parl_status s, parl_ctx_t ctx = nullptr) {
    if (s == PARL_OK) return;
    const std::string m = parl_last_error(ctx);
    switch (s) {
        case PARL_E_CONFIG: throw ConfigError(m);
        case PARL_E_SHAPE: throw ShapeError(m);
        case PARL_E_VOCAB: throw VocabError(m);
        case PARL_E_LIFECYCLE: throw LifecycleError(m);
        case PARL_E_NUMERIC: throw NumericError(m);
        case PARL_E_BARRIER: throw BarrierError(m);
        case PARL_E_STALL: throw StallError(m);
        case PARL_E_IO: throw IoError(m);
        default: throw DeviceError(m);
    }
}

// ---- device context ------------------------------------------------------------
class Device {
public:
    static Device& get(int device = 0, parl_precision prec = PARL_PREC_FP32) {
        static std::shared_ptr<Device> d[2];
        auto& slot = d[prec == PARL_PREC_BF16 ? 1 : 0];
        if (!slot) slot = std::shared_ptr<Device>(new Device(device, prec));
        return *slot;
    }
    parl_ctx_t ctx() const { return ctx_; }
    void sync() const { check(parl_ctx_sync(ctx_), ctx_); }
    ~Device() { parl_ctx_destroy(ctx_); }

private:
    Device(int device, parl_precision prec) { check(parl_ctx_create(device, prec, &ctx_)); }
    parl_ctx_t ctx_ = nullptr;
};

// ---- model (model.hpp:26-106) ------------------------------------------------------
struct ModelConfig {
    int vocab_size = 64, d_model = 32, n_layers = 2, n_heads = 2, d_ff = 64, max_seq_len = 256;
    parl_config c() const { return {vocab_size, d_model, n_layers, n_heads, d_ff, max_seq_len}; }
    bool operator==(const ModelConfig&) const = default;
};

struct AttentionMaskSpec {
    enum class Kind { causal, shared_prompt };
    Kind kind = Kind::causal;
    int prompt_len = 0;
    std::vector<int> response_lens;
    static AttentionMaskSpec causal() { return {}; }
    static AttentionMaskSpec shared_prompt(int p, std::vector<int> lens) {
        return {Kind::shared_prompt, p, std::move(lens)};
    }
    int total_len() const {
        if (kind == Kind::causal) return 0;
        int t = prompt_len;
        for (int r : response_lens) t += r;
        return t;
    }
};

class GradBuffer;

class ModelParams {
public:
    static ModelParams init(const ModelConfig& cfg, std::uint64_t seed, Device& dev = Device::get()) {
        ModelParams p(cfg, dev);
        check(parl_model_init(p.h_.get(), seed), dev.ctx());
        return p;
    }
    static ModelParams from_flat(const ModelConfig& cfg, std::span<const double> flat, std::uint64_t version = 0,
                                 Device& dev = Device::get()) {
        ModelParams p(cfg, dev);
        check(parl_model_upload(p.h_.get(), flat.data(), flat.size(), version), dev.ctx());
        return p;
    }
    const ModelConfig& config() const { return cfg_; }
    std::uint64_t version() const { return parl_model_version(h_.get()); }
    std::vector<double> flat() const {
        std::vector<double> w(param_count());
        check(parl_model_download(h_.get(), w.data(), w.size()), dev_->ctx());
        return w;
    }
    std::size_t param_count() const {
        parl_config c = cfg_.c();
        return parl_param_count(&c);
    }
    ModelParams clone() const {
        ModelParams p(cfg_, *dev_);
        check(parl_model_copy(p.h_.get(), h_.get(), 0, 0.0), dev_->ctx());
        return p;
    }
    inline void apply_update(const GradBuffer& grads, double lr);
    parl_model_t handle() const { return h_.get(); }
    Device& device() const { return *dev_; }

    // save_checkpoint / load_checkpoint (model.cpp:924-987), PARLCKP1 format
    void save(const std::string& path) const { check(parl_checkpoint_save(h_.get(), path.c_str()), dev_->ctx()); }
    static ModelParams load(const std::string& path, Device& dev = Device::get()) {
        parl_model_t m = nullptr;
        check(parl_checkpoint_load(dev.ctx(), path.c_str(), &m), dev.ctx());
        parl_config c{};
        parl_model_config(m, &c);
        return ModelParams(ModelConfig{c.vocab_size, c.d_model, c.n_layers, c.n_heads, c.d_ff, c.max_seq_len}, dev, m);
    }

private:
    ModelParams(const ModelConfig& cfg, Device& dev, parl_model_t m) : cfg_(cfg), dev_(&dev) {
        h_ = std::shared_ptr<parl_model_s>(m, [](parl_model_t x) { parl_model_destroy(x); });
    }
    ModelParams(const ModelConfig& cfg, Device& dev) : cfg_(cfg), dev_(&dev) {
        parl_config c = cfg.c();
        parl_model_t m = nullptr;
        check(parl_model_create(dev.ctx(), &c, &m), dev.ctx());
        h_ = std::shared_ptr<parl_model_s>(m, [](parl_model_t x) { parl_model_destroy(x); });
    }
    ModelConfig cfg_;
    Device* dev_;
    std::shared_ptr<parl_model_s> h_;
};

class GradBuffer {
public:
    explicit GradBuffer(const ModelParams& like) : dev_(&like.device()), n_(like.param_count()) {
        parl_grad_t g = nullptr;
        check(parl_grad_create(dev_->ctx(), like.handle(), &g), dev_->ctx());
        h_ = std::shared_ptr<parl_grad_s>(g, [](parl_grad_t x) { parl_grad_destroy(x); });
    }
    void reset() { check(parl_grad_reset(h_.get()), dev_->ctx()); }
    void accumulate(const GradBuffer& other) { check(parl_grad_accumulate(h_.get(), other.h_.get()), dev_->ctx()); }
    std::vector<double> flat() const {
        std::vector<double> g(n_);
        check(parl_grad_download(h_.get(), g.data(), g.size()), dev_->ctx());
        return g;
    }
    int micro_step_count() const { return parl_grad_micro_steps(h_.get()); }
    void allreduce() { check(parl_grad_allreduce(dev_->ctx(), h_.get()), dev_->ctx()); }
    parl_grad_t handle() const { return h_.get(); }

private:
    Device* dev_;
    std::size_t n_;
    std::shared_ptr<parl_grad_s> h_;
};

// sample_tokens (model.cpp:843-900)
inline std::vector<TokenId> sample_tokens(const ModelParams& params, std::span<const TokenId> prompt,
                                          int max_new_tokens, double temperature, std::uint64_t rng_seed) {
    std::vector<TokenId> out(std::max(max_new_tokens, 1));
    int n = 0;
    check(parl_sample_tokens(params.device().ctx(), params.handle(), prompt.data(), (int)prompt.size(),
                             max_new_tokens, temperature, rng_seed, out.data(), &n),
          params.device().ctx());
    out.resize(n);
    return out;
}

inline void save_checkpoint(const std::string& path, const ModelParams& params) { params.save(path); }
inline ModelParams load_checkpoint(const std::string& path, Device& dev = Device::get()) {
    return ModelParams::load(path, dev);
}

inline void ModelParams::apply_update(const GradBuffer& grads, double lr) {
    check(parl_apply_update(h_.get(), grads.handle(), lr), dev_->ctx());
}

// ---- packed sequences ----------------------------------------------------------------
namespace detail {
inline std::shared_ptr<parl_group_s> make_group(Device& dev, int max_tokens, int max_resp) {
    parl_group_t g = nullptr;
    check(parl_group_create(dev.ctx(), std::max(max_tokens, 1), std::max(max_resp, 1), &g), dev.ctx());
    return std::shared_ptr<parl_group_s>(g, [](parl_group_t x) { parl_group_destroy(x); });
}
}  // namespace detail

struct PackedGroup {
    std::vector<TokenId> tokens;
    std::vector<std::int32_t> labels;
    std::vector<int> positions;
    AttentionMaskSpec mask;
    struct Span {
        int start = 0;
        int len = 0;
    };
    std::vector<Span> spans;
    std::shared_ptr<parl_group_s> device;  // packed on the GPU by K1
};

// pack_group (packing.cpp:7-45), run by the device packer; host views downloaded.
inline PackedGroup pack_group(std::span<const TokenId> prompt, const std::vector<std::vector<TokenId>>& responses,
                              int max_seq_len, Device& dev = Device::get()) {
    std::vector<std::int32_t> flat, lens;
    for (const auto& r : responses) {
        lens.push_back((std::int32_t)r.size());
        flat.insert(flat.end(), r.begin(), r.end());
    }
    PackedGroup pg;
    const int T = (int)(prompt.size() + flat.size());
    pg.device = detail::make_group(dev, T, (int)responses.size());
    check(parl_pack(pg.device.get(), prompt.data(), (int)prompt.size(), flat.data(), lens.data(), (int)lens.size(),
                    max_seq_len),
          dev.ctx());
    pg.tokens.resize(T);
    pg.labels.resize(T);
    pg.positions.resize(T);
    std::vector<std::int32_t> starts(responses.size());
    check(parl_group_download(pg.device.get(), pg.tokens.data(), pg.labels.data(), pg.positions.data(), nullptr,
                              nullptr, starts.data(), nullptr),
          dev.ctx());
    for (std::size_t k = 0; k < responses.size(); ++k) pg.spans.push_back({starts[k], lens[k]});
    pg.mask = AttentionMaskSpec::shared_prompt((int)prompt.size(), std::vector<int>(lens.begin(), lens.end()));
    return pg;
}

// packing.cpp:74-89
inline std::vector<std::vector<double>> extract_response_logprobs(std::span<const double> lp, const PackedGroup& p) {
    std::size_t expected = 0;
    for (const auto& s : p.spans) expected += (std::size_t)s.len;
    if (lp.size() != expected)
        throw ShapeError("logprob vector of length " + std::to_string(lp.size()) + " does not match " +
                         std::to_string(expected) + " response tokens");
    std::vector<std::vector<double>> out;
    std::size_t c = 0;
    for (const auto& s : p.spans) {
        out.emplace_back(lp.begin() + c, lp.begin() + c + s.len);
        c += (std::size_t)s.len;
    }
    return out;
}

// ---- forward / backward ------------------------------------------------------------------
struct ForwardCache {
    std::shared_ptr<parl_group_s> group;
    std::shared_ptr<parl_act_s> act;
};

struct ForwardResult {
    std::vector<double> logprobs;
    std::vector<int> scored_positions;
    std::shared_ptr<ForwardCache> cache;  // null unless want_cache
};

namespace detail {
inline std::shared_ptr<parl_group_s> sequence(const ModelParams& p, std::span<const TokenId> tokens,
                                              std::span<const int> positions, const AttentionMaskSpec& mask,
                                              std::span<const std::int32_t> labels) {
    const auto& c = p.config();
    if (tokens.size() != positions.size() || (labels.data() && tokens.size() != labels.size()))
        throw ShapeError("tokens/positions/labels lengths differ");
    auto g = make_group(p.device(), (int)tokens.size(), (int)mask.response_lens.size());
    const int P = mask.kind == AttentionMaskSpec::Kind::shared_prompt ? mask.prompt_len : 0;
    if (mask.kind == AttentionMaskSpec::Kind::shared_prompt && P < 1)
        throw ShapeError("shared_prompt mask needs prompt_len >= 1");
    std::vector<std::int32_t> lens(mask.response_lens.begin(), mask.response_lens.end());
    check(parl_set_sequence(g.get(), tokens.data(), positions.data(), labels.data(), (int)tokens.size(), P,
                            lens.data(), P ? (int)lens.size() : 0, c.vocab_size, c.max_seq_len),
          p.device().ctx());
    return g;
}
}  // namespace detail

// model.cpp:534-567
inline ForwardResult forward_logprobs(const ModelParams& params, std::span<const TokenId> tokens,
                                      std::span<const int> positions, const AttentionMaskSpec& mask,
                                      std::span<const std::int32_t> labels, bool want_cache = false) {
    if (!labels.data()) throw ShapeError("forward_logprobs requires labels");
    auto g = detail::sequence(params, tokens, positions, mask, labels);
    parl_act_t act = nullptr;
    parl_ctx_t ctx = params.device().ctx();
    check(parl_forward(ctx, params.handle(), g.get(), 0, want_cache ? &act : nullptr), ctx);
    ForwardResult r;
    const int S = parl_group_scored(g.get());
    r.logprobs.resize(S);
    std::vector<std::int32_t> sp(S);
    check(parl_group_logprobs(g.get(), 0, r.logprobs.data()), ctx);
    check(parl_group_download(g.get(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, sp.data()), ctx);
    r.scored_positions.assign(sp.begin(), sp.end());
    if (want_cache) {
        r.cache = std::make_shared<ForwardCache>();
        r.cache->group = g;
        r.cache->act = std::shared_ptr<parl_act_s>(act, [](parl_act_t x) { parl_act_destroy(x); });
    }
    return r;
}

// model.cpp:587-838: gradient of sum_i upstream[i] * logprobs[i]
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

inline GradBuffer backward(const ModelParams& params, const ForwardResult& fwd, std::span<const double> upstream) {
    if (!fwd.cache) throw LifecycleError("backward requires a cached forward result");
    if (upstream.size() != fwd.logprobs.size())
        throw ShapeError("upstream gradient count " + std::to_string(upstream.size()) +
                         " != scored position count " + std::to_string(fwd.logprobs.size()));
    parl_ctx_t ctx = params.device().ctx();
    check(parl_group_set_upstream(fwd.cache->group.get(), upstream.data()), ctx);
    GradBuffer gb(params);
    check(parl_backward(ctx, params.handle(), fwd.cache->act.get(), fwd.cache->group.get(), gb.handle()), ctx);
    return gb;
}

// model.cpp:569-585: [T x V] log-softmax rows
inline std::vector<double> forward_logprob_rows(const ModelParams& params, std::span<const TokenId> tokens,
                                                std::span<const int> positions, const AttentionMaskSpec& mask) {
    auto g = detail::sequence(params, tokens, positions, mask, {});
    std::vector<double> rows(tokens.size() * (std::size_t)params.config().vocab_size);
    check(parl_logprob_rows(params.device().ctx(), params.handle(), g.get(), rows.data()), params.device().ctx());
    return rows;
}

// ---- tri-model and the fused micro-step (pipeline.hpp:41-60, pipeline.cpp:97-141) -------
struct TriModel {
    ModelParams policy, old_policy, reference;
    static TriModel init(const ModelConfig& cfg, std::uint64_t seed, Device& dev = Device::get()) {
        ModelParams p = ModelParams::init(cfg, seed, dev);
        return TriModel{p, p.clone(), p.clone()};
    }
    void snapshot_old_policy() { check(parl_model_copy(old_policy.handle(), policy.handle(), 0, 0.0)); }
};

struct TriForwardResult {
    ForwardResult policy;
    std::vector<double> old_logprobs, ref_logprobs;
};

inline TriForwardResult trimodel_forward(const TriModel& tm, std::span<const TokenId> tokens,
                                         std::span<const int> positions, const AttentionMaskSpec& mask,
                                         std::span<const std::int32_t> labels) {
    auto g = detail::sequence(tm.policy, tokens, positions, mask, labels);
    parl_ctx_t ctx = tm.policy.device().ctx();
    parl_act_t act = nullptr;
    check(parl_trimodel_forward(ctx, tm.policy.handle(), tm.old_policy.handle(), tm.reference.handle(), g.get(), &act),
          ctx);
    TriForwardResult r;
    const int S = parl_group_scored(g.get());
    r.policy.logprobs.resize(S);
    r.old_logprobs.resize(S);
    r.ref_logprobs.resize(S);
    check(parl_group_logprobs(g.get(), 0, r.policy.logprobs.data()), ctx);
    check(parl_group_logprobs(g.get(), 1, r.old_logprobs.data()), ctx);
    check(parl_group_logprobs(g.get(), 2, r.ref_logprobs.data()), ctx);
    std::vector<std::int32_t> sp(S);
    check(parl_group_download(g.get(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, sp.data()), ctx);
    r.policy.scored_positions.assign(sp.begin(), sp.end());
    r.policy.cache = std::make_shared<ForwardCache>();
    r.policy.cache->group = g;
    r.policy.cache->act = std::shared_ptr<parl_act_s>(act, [](parl_act_t x) { parl_act_destroy(x); });
    return r;
}

enum class LossGranularity { token, sequence };

struct HyperParams {  // pipeline.hpp:29-37 (loss subset)
    double epsilon = 0.2;
    double beta = 0.04;
    LossGranularity granularity = LossGranularity::token;
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

// One shared-prompt micro-batch: pack -> tri-model forward -> GRPO terms
// (advantages from `rewards`) -> backward of -upstream -> grads += (all on the
// device).  Returns this micro-batch's stats and adds them into `stats`.
inline MicrobatchStats train_microbatch(TriModel& tm, std::span<const TokenId> prompt,
                                        const std::vector<std::vector<TokenId>>& responses,
                                        std::span<const double> rewards, const HyperParams& hp, GradBuffer& grads,
                                        MicrobatchStats& stats) {
    PackedGroup pg = pack_group(prompt, responses, tm.policy.config().max_seq_len, tm.policy.device());
    parl_ctx_t ctx = tm.policy.device().ctx();
    if (rewards.size() != responses.size()) throw ShapeError("one reward per response required");
    check(parl_stats_reset(ctx), ctx);
    parl_hyper h = hp.c();
    parl_loss_stats s{};
    check(parl_train_microbatch(ctx, tm.policy.handle(), tm.old_policy.handle(), tm.reference.handle(),
                                pg.device.get(), rewards.data(), nullptr, &h, grads.handle(), &s),
          ctx);
    MicrobatchStats m;
    m.objective_sum = s.objective_sum;
    m.clip_sum = s.clip_sum;
    m.kl_sum = s.kl_sum;
    m.clipped_units = (long)s.clipped_units;
    m.total_units = (long)s.total_units;
    m.micro_batches = 1;
    stats.objective_sum += m.objective_sum;
    stats.clip_sum += m.clip_sum;
    stats.kl_sum += m.kl_sum;
    stats.clipped_units += m.clipped_units;
    stats.total_units += m.total_units;
    stats.micro_batches += 1;
    return m;
}

}  // namespace parl
