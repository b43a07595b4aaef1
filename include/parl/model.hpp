// parl/model.hpp — drop-in for proj/include/parl/model.hpp, backed by the
// B200 device path (libparl_gpu.so, C-ABI include/parl_gpu.h).
//
// Same names, signatures, argument meaning and exception types as the
// reference (model.hpp:12-193); what changes is where the work runs:
//   * ModelParams owns a device weight set (fp64 master + the compute copy);
//     flat() is a host mirror refreshed whenever the device weights change
//     (parl_model_epoch).  After flat_mut() the host copy is authoritative, as the
//     reference's w_ is: a span the caller keeps may be written at any time, so
//     every device use first uploads the host copy when its contents changed;
//   * GradBuffer owns the device fp32 accumulator; flat()/flat_mut() likewise;
//   * forward_logprobs / backward / forward_logprob_rows / sample_tokens run the
//     device kernels (validation order and errors of model.cpp:404-426, 587-598).
// Arithmetic: fp32 (FFMA kernels) by default, bf16 tensor-core operands with
// PARL_PRECISION=bf16 (or an explicit Device); the reference computes in fp64,
// so fp64-tolerance assertions hold at the SURVEY.md §8c tolerances instead.
// Header-only; link with libparl_gpu.so.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "parl/errors.hpp"
#include "parl_gpu.h"

namespace parl {

using TokenId = std::int32_t;

// Reserved token ids (model.hpp:15-20)
constexpr TokenId kPadToken = 0;
constexpr TokenId kBosToken = 1;
constexpr TokenId kEosToken = 2;
constexpr TokenId kSepToken = 3;
constexpr TokenId kFirstPayloadToken = 4;
constexpr std::int32_t kIgnoreLabel = -1;

// ---- device context (no reference counterpart) ---------------------------------
// One process-wide context per precision; the reference API has no device
// argument, so its calls run on Device::get() (device 0, $PARL_PRECISION).
class Device {
public:
    static Device& get(int device = 0) { return get(device, default_precision()); }
    static Device& get(int device, parl_precision prec) {
        static std::shared_ptr<Device> d[2];
        auto& slot = d[prec == PARL_PREC_BF16 ? 1 : 0];
        if (!slot) slot = std::shared_ptr<Device>(new Device(device, prec));
        return *slot;
    }
    static parl_precision default_precision() {
        const char* e = std::getenv("PARL_PRECISION");
        return (e && std::strcmp(e, "bf16") == 0) ? PARL_PREC_BF16 : PARL_PREC_FP32;
    }
    parl_ctx_t ctx() const { return ctx_; }
    parl_precision precision() const { return prec_; }
    void sync() const { detail::check(parl_ctx_sync(ctx_), ctx_); }
    ~Device() { parl_ctx_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

private:
    Device(int device, parl_precision prec) : prec_(prec) { detail::check(parl_ctx_create(device, prec, &ctx_)); }
    parl_ctx_t ctx_ = nullptr;
    parl_precision prec_;
};

// ---- config and mask (model.hpp:26-55, model.cpp:19-61) ------------------------
struct ModelConfig {
    int vocab_size = 64;
    int d_model = 32;
    int n_layers = 2;
    int n_heads = 2;
    int d_ff = 64;
    int max_seq_len = 256;

    void validate() const {  // model.cpp:19-31
        if (vocab_size < 4)
            throw ConfigError("vocab_size must be >= 4 (ids 0..3 are reserved), got " + std::to_string(vocab_size));
        if (d_model <= 0) throw ConfigError("d_model must be positive");
        if (n_layers <= 0) throw ConfigError("n_layers must be positive");
        if (n_heads <= 0) throw ConfigError("n_heads must be positive");
        if (d_ff <= 0) throw ConfigError("d_ff must be positive");
        if (max_seq_len <= 0) throw ConfigError("max_seq_len must be positive");
        if (d_model % n_heads != 0)
            throw ConfigError("d_model (" + std::to_string(d_model) + ") not divisible by n_heads (" +
                              std::to_string(n_heads) + ")");
    }
    bool operator==(const ModelConfig&) const = default;
    parl_config c() const { return {vocab_size, d_model, n_layers, n_heads, d_ff, max_seq_len}; }
};

struct AttentionMaskSpec {
    enum class Kind { causal, shared_prompt };

    Kind kind = Kind::causal;
    int prompt_len = 0;
    std::vector<int> response_lens;

    static AttentionMaskSpec causal() { return {}; }
    static AttentionMaskSpec shared_prompt(int prompt_len, std::vector<int> response_lens) {
        AttentionMaskSpec m;
        m.kind = Kind::shared_prompt;
        m.prompt_len = prompt_len;
        m.response_lens = std::move(response_lens);
        return m;
    }
    int total_len() const {
        if (kind == Kind::causal) return 0;
        int total = prompt_len;
        for (int r : response_lens) total += r;
        return total;
    }
    void validate(int seq_len, int max_seq_len) const {  // model.cpp:53-61
        if (kind == Kind::causal) return;
        if (prompt_len < 1) throw ShapeError("shared_prompt mask needs prompt_len >= 1");
        if (response_lens.empty()) throw ShapeError("shared_prompt mask needs >= 1 response");
        for (int r : response_lens)
            if (r < 1) throw ShapeError("shared_prompt mask response lengths must be >= 1");
        if (total_len() != seq_len)
            throw ShapeError("shared_prompt mask covers " + std::to_string(total_len()) +
                             " tokens but sequence has " + std::to_string(seq_len));
        if (seq_len > max_seq_len)
            throw ShapeError("packed length " + std::to_string(seq_len) + " exceeds max_seq_len " +
                             std::to_string(max_seq_len));
    }
};

struct TensorInfo {
    std::string name;
    std::size_t offset = 0;
    int rows = 0;
    int cols = 0;
    std::size_t size() const { return static_cast<std::size_t>(rows) * cols; }
};

namespace detail {
// the reference flat layout (model.cpp:86-114) and its signature (model.cpp:66-128)
inline std::vector<TensorInfo> build_layout(const ModelConfig& c) {
    std::vector<TensorInfo> v;
    std::size_t total = 0;
    auto add = [&](const std::string& n, int r, int k) {
        v.push_back({n, total, r, k});
        total += static_cast<std::size_t>(r) * k;
    };
    add("tok_emb", c.vocab_size, c.d_model);
    add("pos_emb", c.max_seq_len, c.d_model);
    for (int l = 0; l < c.n_layers; ++l) {
        const std::string p = "layers." + std::to_string(l) + ".";
        add(p + "ln1.gamma", 1, c.d_model);
        add(p + "ln1.beta", 1, c.d_model);
        add(p + "attn.wq", c.d_model, c.d_model);
        add(p + "attn.bq", 1, c.d_model);
        add(p + "attn.wk", c.d_model, c.d_model);
        add(p + "attn.bk", 1, c.d_model);
        add(p + "attn.wv", c.d_model, c.d_model);
        add(p + "attn.bv", 1, c.d_model);
        add(p + "attn.wo", c.d_model, c.d_model);
        add(p + "attn.bo", 1, c.d_model);
        add(p + "ln2.gamma", 1, c.d_model);
        add(p + "ln2.beta", 1, c.d_model);
        add(p + "ffn.w1", c.d_model, c.d_ff);
        add(p + "ffn.b1", 1, c.d_ff);
        add(p + "ffn.w2", c.d_ff, c.d_model);
        add(p + "ffn.b2", 1, c.d_model);
    }
    add("ln_f.gamma", 1, c.d_model);
    add("ln_f.beta", 1, c.d_model);
    add("head.w", c.d_model, c.vocab_size);
    add("head.b", 1, c.vocab_size);
    return v;
}

inline std::uint64_t fnv1a(const void* data, std::size_t n, std::uint64_t h = 0xcbf29ce484222325ull) {
    const auto* p = static_cast<const unsigned char*>(data);
    for (std::size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

inline std::uint64_t layout_hash(const ModelConfig& c, const std::vector<TensorInfo>& layout) {
    std::uint64_t h = fnv1a(&c.vocab_size, sizeof(int));
    for (const int* f : {&c.d_model, &c.n_layers, &c.n_heads, &c.d_ff, &c.max_seq_len}) h = fnv1a(f, sizeof(int), h);
    for (const auto& t : layout) {
        h = fnv1a(t.name.data(), t.name.size(), h);
        h = fnv1a(&t.rows, sizeof(int), h);
        h = fnv1a(&t.cols, sizeof(int), h);
    }
    return h;
}

struct ModelDel {
    void operator()(parl_model_t m) const { parl_model_destroy(m); }
};
struct GradDel {
    void operator()(parl_grad_t g) const { parl_grad_destroy(g); }
};
}  // namespace detail

class GradBuffer;

// ---- ModelParams (model.hpp:64-106) ---------------------------------------------
class ModelParams {
public:
    static ModelParams init(const ModelConfig& config, std::uint64_t seed) { return init(config, seed, Device::get()); }
    static ModelParams init(const ModelConfig& config, std::uint64_t seed, Device& dev) {
        config.validate();
        ModelParams p(config, dev);
        detail::check(parl_model_init(p.h_.get(), seed), dev.ctx());  // model.cpp:142-164, bit-exact
        return p;
    }
    // weights drawn elsewhere (fp64, reference layout)
    static ModelParams from_flat(const ModelConfig& config, std::span<const double> flat, std::uint64_t version = 0,
                                 Device& dev = Device::get()) {
        config.validate();
        ModelParams p(config, dev);
        detail::check(parl_model_upload(p.h_.get(), flat.data(), flat.size(), version), dev.ctx());
        return p;
    }

    const ModelConfig& config() const { return cfg_; }
    std::uint64_t version() const { return parl_model_version(h_.get()); }
    std::uint64_t init_seed() const { return parl_model_init_seed(h_.get()); }

    std::span<const double> flat() const { return mirror(); }
    std::span<double> flat_mut() {
        mirror();
        host_owned_ = true;
        return host_;
    }
    const std::vector<TensorInfo>& layout() const { return layout_; }
    std::span<const double> tensor(const std::string& name) const {
        for (const auto& t : layout_)
            if (t.name == name) return mirror().subspan(t.offset, t.size());
        throw ConfigError("unknown tensor name: " + name);
    }
    std::uint64_t layout_signature() const { return layout_sig_; }

    ModelParams clone() const {  // model.cpp:172-181 (init_seed kept, version kept)
        ModelParams p(cfg_, *dev_);
        detail::check(parl_model_copy(p.h_.get(), handle(), 0, 0.0), dev_->ctx());
        if (host_valid_) {
            p.host_ = host_;
            p.host_epoch_ = parl_model_epoch(p.h_.get());
            p.host_valid_ = true;
        }
        return p;
    }
    // after a device write through this object: keep an authoritative host copy in step
    void refresh() const {
        if (!host_owned_) return;
        detail::check(parl_model_download(h_.get(), host_.data(), host_.size()), dev_->ctx());
        host_epoch_ = parl_model_epoch(h_.get());
        host_hash_ = detail::fnv1a(host_.data(), host_.size() * sizeof(double));
    }
    ModelParams(const ModelParams& o) : ModelParams(o.clone()) {}
    ModelParams& operator=(const ModelParams& o) {
        if (this != &o) *this = o.clone();
        return *this;
    }
    ModelParams(ModelParams&&) noexcept = default;
    ModelParams& operator=(ModelParams&&) noexcept = default;

    // W <- W - lr * grad_sum / micro_step_count; bumps version; refuses non-finite (model.cpp:202-219)
    inline void apply_update(const GradBuffer& grads, double lr);

    bool all_finite() const {
        int ok = 0;
        detail::check(parl_model_all_finite(handle(), &ok), dev_->ctx());
        return ok != 0;
    }

    // ForwardCache staleness counter (model.hpp:100-101), kept on the device and bumped by every forward
    std::uint64_t forward_generation() const { return parl_model_forward_gen(h_.get()); }

    // device handle; host writes made through flat_mut() are uploaded first (same version)
    parl_model_t handle() const {
        if (host_owned_) {
            const std::uint64_t hsh = detail::fnv1a(host_.data(), host_.size() * sizeof(double));
            if (hsh != host_hash_) {
                const std::uint64_t v = version(), seed = init_seed();
                detail::check(parl_model_upload(h_.get(), host_.data(), host_.size(), v), dev_->ctx());
                detail::check(parl_model_set_init_seed(h_.get(), seed), dev_->ctx());
                host_hash_ = hsh;
                host_epoch_ = parl_model_epoch(h_.get());
            }
        }
        return h_.get();
    }
    Device& device() const { return *dev_; }

    ModelParams(const ModelConfig& cfg, Device& dev, parl_model_t adopt = nullptr)
        : cfg_(cfg), dev_(&dev), layout_(detail::build_layout(cfg)) {
        layout_sig_ = detail::layout_hash(cfg_, layout_);
        parl_model_t m = adopt;
        if (!m) {
            parl_config c = cfg.c();
            detail::check(parl_model_create(dev.ctx(), &c, &m), dev.ctx());
        }
        h_.reset(m);
    }

private:
    std::span<const double> mirror() const {
        if (host_owned_) return host_;
        const std::uint64_t e = parl_model_epoch(h_.get());
        if (!host_valid_ || host_epoch_ != e) {
            host_.resize(layout_.empty() ? 0 : layout_.back().offset + layout_.back().size());
            detail::check(parl_model_download(h_.get(), host_.data(), host_.size()), dev_->ctx());
            host_epoch_ = e;
            host_valid_ = true;
        }
        return host_;
    }

    ModelConfig cfg_;
    Device* dev_;
    std::vector<TensorInfo> layout_;
    std::uint64_t layout_sig_ = 0;
    std::unique_ptr<parl_model_s, detail::ModelDel> h_;
    mutable std::vector<double> host_;
    mutable std::uint64_t host_epoch_ = ~0ull, host_hash_ = 0;
    mutable bool host_valid_ = false;
    bool host_owned_ = false;
};

// ---- GradBuffer (model.hpp:109-134): device fp32 accumulator ----------------------
class GradBuffer {
public:
    explicit GradBuffer(const ModelParams& ref)
        : dev_(&ref.device()), cfg_(ref.config()), n_(ref.layout().back().offset + ref.layout().back().size()),
          layout_sig_(ref.layout_signature()) {
        parl_grad_t g = nullptr;
        detail::check(parl_grad_create(dev_->ctx(), ref.handle(), &g), dev_->ctx());
        h_.reset(g);
    }
    GradBuffer(const GradBuffer& o) : dev_(o.dev_), cfg_(o.cfg_), n_(o.n_), layout_sig_(o.layout_sig_) {
        parl_grad_t g = nullptr;
        const parl_config c = cfg_.c();
        detail::check(parl_grad_create_config(dev_->ctx(), &c, &g), dev_->ctx());
        h_.reset(g);
        detail::check(parl_grad_accumulate(g, o.handle()), dev_->ctx());  // counts add: 0 + o's
    }
    GradBuffer& operator=(const GradBuffer& o) {
        if (this != &o) {
            reset();
            accumulate(o);
        }
        return *this;
    }
    GradBuffer(GradBuffer&&) noexcept = default;
    GradBuffer& operator=(GradBuffer&&) noexcept = default;

    void reset() {
        detail::check(parl_grad_reset(h_.get()), dev_->ctx());
        touched();
    }
    // elementwise += other; counts add (model.cpp:189-194)
    void accumulate(const GradBuffer& other) {
        if (other.layout_sig_ != layout_sig_ || other.n_ != n_)
            throw ShapeError("gradient buffers have incongruent layouts");
        detail::check(parl_grad_accumulate(handle(), other.handle()), dev_->ctx());
        touched();
    }
    std::span<const double> flat() const { return mirror(); }
    std::span<double> flat_mut() {
        mirror();
        host_owned_ = true;
        return host_;
    }
    int micro_step_count() const { return parl_grad_micro_steps(h_.get()); }
    void set_micro_step_count(int n) { detail::check(parl_grad_set_micro_steps(h_.get(), n), dev_->ctx()); }
    void add_micro_steps(int n) { detail::check(parl_grad_add_micro_steps(h_.get(), n), dev_->ctx()); }
    std::uint64_t layout_signature() const { return layout_sig_; }
    bool all_finite() const {
        int ok = 0;
        detail::check(parl_grad_all_finite(handle(), &ok), dev_->ctx());
        return ok != 0;
    }
    // data-parallel exchange (NCCL allreduce of the accumulator, counts summed)
    void allreduce() {
        detail::check(parl_grad_allreduce(dev_->ctx(), handle()), dev_->ctx());
        touched();
    }

    // device handle; host writes made through flat_mut() are uploaded first
    parl_grad_t handle() const {
        if (host_owned_) {
            const std::uint64_t hsh = detail::fnv1a(host_.data(), host_.size() * sizeof(double));
            if (hsh != host_hash_) {
                detail::check(parl_grad_upload(h_.get(), host_.data(), host_.size()), dev_->ctx());
                host_hash_ = hsh;
            }
        }
        return h_.get();
    }
    // the device accumulator changed (backward / accumulate / reset / allreduce)
    void touched() {
        ++dev_epoch_;
        if (host_owned_) {  // keep the authoritative host copy in step
            detail::check(parl_grad_download(h_.get(), host_.data(), host_.size()), dev_->ctx());
            host_hash_ = detail::fnv1a(host_.data(), host_.size() * sizeof(double));
            host_epoch_ = dev_epoch_;
        }
    }
    Device& device() const { return *dev_; }

private:
    std::span<const double> mirror() const {
        if (host_owned_) return host_;
        if (host_epoch_ != dev_epoch_) {
            host_.resize(n_);
            detail::check(parl_grad_download(h_.get(), host_.data(), host_.size()), dev_->ctx());
            host_epoch_ = dev_epoch_;
        }
        return host_;
    }

    Device* dev_;
    ModelConfig cfg_;
    std::size_t n_;
    std::uint64_t layout_sig_;
    std::unique_ptr<parl_grad_s, detail::GradDel> h_;
    std::uint64_t dev_epoch_ = 0;
    mutable std::vector<double> host_;
    mutable std::uint64_t host_epoch_ = ~0ull, host_hash_ = 0;
    bool host_owned_ = false;
};

inline void ModelParams::apply_update(const GradBuffer& grads, double lr) {
    if (grads.layout_signature() != layout_sig_) throw ShapeError("gradient layout not congruent with parameters");
    detail::check(parl_apply_update(handle(), grads.handle(), lr), dev_->ctx());
    refresh();
}

// ---- forward / backward (model.hpp:136-193) ----------------------------------------------
// The activation handle of a cached forward: the device packed sequence and the
// policy activations, with the owner / version / generation checks of
// model.cpp:590-598 enforced by parl_backward.
struct ForwardCache {
    std::shared_ptr<parl_group_s> group;
    std::shared_ptr<parl_act_s> act;
    const ModelParams* owner = nullptr;
};

struct ForwardResult {
    std::vector<double> logprobs;
    std::vector<int> scored_positions;
    std::shared_ptr<ForwardCache> cache;  // null unless want_cache
};

namespace detail {
inline std::shared_ptr<parl_group_s> make_group(Device& dev, int max_tokens, int max_resp) {
    parl_group_t g = nullptr;
    check(parl_group_create(dev.ctx(), std::max(max_tokens, 1), std::max(max_resp, 1), &g), dev.ctx());
    return std::shared_ptr<parl_group_s>(g, [](parl_group_t x) { parl_group_destroy(x); });
}

// validate_forward_inputs (model.cpp:404-426) runs in parl_set_sequence, same order
inline std::shared_ptr<parl_group_s> sequence(const ModelParams& p, std::span<const TokenId> tokens,
                                              std::span<const int> positions, const AttentionMaskSpec& mask,
                                              std::span<const std::int32_t> labels) {
    const auto& c = p.config();
    if (tokens.size() != positions.size() || (labels.data() && tokens.size() != labels.size()))
        throw ShapeError("tokens/positions/labels lengths differ");
    auto g = make_group(p.device(), (int)tokens.size(), (int)mask.response_lens.size());
    const bool sp = mask.kind == AttentionMaskSpec::Kind::shared_prompt;
    if (sp && mask.prompt_len < 1) {  // checked after the per-element validation, as mask.validate is
        check(parl_set_sequence(g.get(), tokens.data(), positions.data(), labels.data(), (int)tokens.size(), 0,
                                nullptr, 0, c.vocab_size, c.max_seq_len),
              p.device().ctx());
        throw ShapeError("shared_prompt mask needs prompt_len >= 1");
    }
    std::vector<std::int32_t> lens(mask.response_lens.begin(), mask.response_lens.end());
    check(parl_set_sequence(g.get(), tokens.data(), positions.data(), labels.data(), (int)tokens.size(),
                            sp ? mask.prompt_len : 0, lens.data(), sp ? (int)lens.size() : 0, c.vocab_size,
                            c.max_seq_len),
          p.device().ctx());
    return g;
}
}  // namespace detail

// model.cpp:534-567
inline ForwardResult forward_logprobs(const ModelParams& params, std::span<const TokenId> tokens,
                                      std::span<const int> positions, const AttentionMaskSpec& mask,
                                      std::span<const std::int32_t> labels, bool want_cache = false) {
    auto g = detail::sequence(params, tokens, positions, mask, labels);
    if (!labels.data()) throw ShapeError("forward_logprobs requires labels");
    parl_ctx_t ctx = params.device().ctx();
    parl_act_t act = nullptr;
    detail::check(parl_forward(ctx, params.handle(), g.get(), 0, want_cache ? &act : nullptr), ctx);
    ForwardResult r;
    const int S = parl_group_scored(g.get());
    r.logprobs.resize(S);
    std::vector<std::int32_t> sp(S);
    detail::check(parl_group_logprobs(g.get(), 0, r.logprobs.data()), ctx);
    detail::check(parl_group_download(g.get(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, sp.data()), ctx);
    r.scored_positions.assign(sp.begin(), sp.end());
    if (want_cache) {
        r.cache = std::make_shared<ForwardCache>();
        r.cache->group = g;
        r.cache->act = std::shared_ptr<parl_act_s>(act, [](parl_act_t x) { parl_act_destroy(x); });
        r.cache->owner = &params;
    }
    return r;
}

// model.cpp:587-838: gradient of sum_i upstream[i] * logprobs[i]; micro_step_count 1
inline GradBuffer backward(const ModelParams& params, const ForwardResult& fwd, std::span<const double> upstream) {
    const ForwardCache* fc = fwd.cache.get();
    if (!fc || !fc->act) throw LifecycleError("backward requires a cached forward result");
    if (fc->owner != &params)
        throw LifecycleError("stale activation handle: a newer forward or update invalidated this cache");
    if (upstream.size() != fwd.scored_positions.size())
        throw ShapeError("upstream gradient count " + std::to_string(upstream.size()) + " != scored position count " +
                         std::to_string(fwd.scored_positions.size()));
    parl_ctx_t ctx = params.device().ctx();
    detail::check(parl_group_set_upstream(fc->group.get(), upstream.data()), ctx);
    GradBuffer gb(params);
    detail::check(parl_backward(ctx, params.handle(), fc->act.get(), fc->group.get(), gb.handle()), ctx);
    gb.touched();
    return gb;
}

// model.cpp:569-585: [seq_len x vocab] log-softmax rows
inline std::vector<double> forward_logprob_rows(const ModelParams& params, std::span<const TokenId> tokens,
                                                std::span<const int> positions, const AttentionMaskSpec& mask) {
    auto g = detail::sequence(params, tokens, positions, mask, {});
    std::vector<double> rows(tokens.size() * (std::size_t)params.config().vocab_size);
    detail::check(parl_logprob_rows(params.device().ctx(), params.handle(), g.get(), rows.data()),
                  params.device().ctx());
    return rows;
}

// model.cpp:843-900 (the forward on the device, the token choice with the reference RNG stream)
inline std::vector<TokenId> sample_tokens(const ModelParams& params, std::span<const TokenId> prompt,
                                          int max_new_tokens, double temperature, std::uint64_t rng_seed) {
    std::vector<TokenId> out(std::max(max_new_tokens, 1));
    int n = 0;
    detail::check(parl_sample_tokens(params.device().ctx(), params.handle(), prompt.data(), (int)prompt.size(),
                                     max_new_tokens, temperature, rng_seed, out.data(), &n),
                  params.device().ctx());
    out.resize(n);
    return out;
}

// model.cpp:907-987, PARLCKP1 (byte-identical to the reference's files)
inline void save_checkpoint(const std::string& path, const ModelParams& params) {
    detail::check(parl_checkpoint_save(params.handle(), path.c_str()), params.device().ctx());
}
inline ModelParams load_checkpoint(const std::string& path) {
    Device& dev = Device::get();
    parl_model_t m = nullptr;
    detail::check(parl_checkpoint_load(dev.ctx(), path.c_str(), &m), dev.ctx());
    parl_config c{};
    parl_model_config(m, &c);
    return ModelParams(ModelConfig{c.vocab_size, c.d_model, c.n_layers, c.n_heads, c.d_ff, c.max_seq_len}, dev, m);
}

}  // namespace parl
