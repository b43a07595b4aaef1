// C++ parity tests of the drop-in layer (include/parl_gpu.hpp) on the GPU,
// written like the reference's own suites (proj/tests/test_packing.cpp,
// test_model.cpp, test_pipeline.cpp) and checked against the C oracle
// (oracle/parl_oracle.c, test infrastructure only).  Built by
// __graft_entry__.build(); run by tests/test_gpu_cpp.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <functional>
#include <random>
#include <string>

#include "../../oracle/parl_oracle.h"
#include "parl_gpu.hpp"

using namespace parl;

static int g_checks = 0, g_fail = 0;
#define CHECK(c)                                                             \
    do {                                                                     \
        ++g_checks;                                                          \
        if (!(c)) {                                                          \
            ++g_fail;                                                        \
            std::fprintf(stderr, "%s:%d CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
        }                                                                    \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                     \
    do {                                             \
        bool thrown_ = false;                        \
        try {                                        \
            (void)(expr);                            \
        } catch (const T&) {                         \
            thrown_ = true;                          \
        } catch (...) {                              \
        }                                            \
        CHECK(thrown_ && #T);                        \
    } while (0)

static std::vector<std::pair<std::string, std::function<void()>>>& cases() {
    static std::vector<std::pair<std::string, std::function<void()>>> c;
    return c;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { cases().emplace_back(n, std::move(f)); }
};
#define TEST_CASE(name) static void name(); static Reg reg_##name(#name, name); static void name()

static ModelConfig small_config() {  // test_packing.cpp:14-23
    ModelConfig c;
    c.vocab_size = 16; c.d_model = 16; c.n_layers = 2; c.n_heads = 2; c.d_ff = 24; c.max_seq_len = 64;
    return c;
}
static orc_cfg ocfg(const ModelConfig& c) { return {c.vocab_size, c.d_model, c.n_layers, c.n_heads, c.d_ff, c.max_seq_len}; }
static std::vector<int> iota(int n) {
    std::vector<int> p(n);
    for (int i = 0; i < n; ++i) p[i] = i;
    return p;
}

TEST_CASE(pack_group_positions_labels_spans) {  // test_packing.cpp:46-76
    std::vector<TokenId> prompt{1, 5, 3};
    PackedGroup pg = pack_group(prompt, {{7, 8}, {9, 10}}, 64);
    CHECK((pg.tokens == std::vector<TokenId>{1, 5, 3, 7, 8, 9, 10}));
    CHECK((pg.positions == std::vector<int>{0, 1, 2, 3, 4, 3, 4}));
    CHECK(pg.spans.size() == 2 && pg.spans[0].start == 3 && pg.spans[1].start == 5 && pg.spans[1].len == 2);
    for (int i = 0; i < 3; ++i) CHECK(pg.labels[i] == kIgnoreLabel);
    for (int i = 3; i < 7; ++i) CHECK(pg.labels[i] == pg.tokens[i]);
    PackedGroup uneq = pack_group(prompt, {{7}, {8, 9, 10}}, 64);
    CHECK((uneq.positions == std::vector<int>{0, 1, 2, 3, 3, 4, 5}));
    bool named = false;
    try {
        pack_group(prompt, {{7, 8}, {9, 10}}, 6);
    } catch (const ShapeError& e) {
        named = std::string(e.what()).find("max_seq_len") != std::string::npos;
    }
    CHECK(named);
    CHECK_THROWS_AS(pack_group(std::vector<TokenId>{}, {{7}}, 64), ShapeError);
    CHECK_THROWS_AS(pack_group(prompt, {}, 64), ShapeError);
    CHECK_THROWS_AS(pack_group(prompt, {{7}, {}}, 64), ShapeError);
}

TEST_CASE(extract_response_logprobs_slices) {  // test_packing.cpp:109-121
    PackedGroup pg = pack_group(std::vector<TokenId>{1, 5}, {{7}, {8, 9}}, 64);
    std::vector<double> lp{-0.5, -1.0, -1.5};
    auto s = extract_response_logprobs(lp, pg);
    CHECK(s.size() == 2 && s[0] == std::vector<double>{-0.5} && (s[1] == std::vector<double>{-1.0, -1.5}));
    std::vector<double> bad{-0.5, -1.0};
    CHECK_THROWS_AS(extract_response_logprobs(bad, pg), ShapeError);
}

TEST_CASE(init_bit_exact_with_oracle) {  // model.cpp:142-164
    ModelConfig c = small_config();
    ModelParams p = ModelParams::init(c, 41);
    orc_cfg oc = ocfg(c);
    std::vector<double> w(orc_param_count(&oc));
    orc_init_params(&oc, 41, w.data());
    CHECK(std::ranges::equal(p.flat(), w));
}

TEST_CASE(packed_logprobs_and_grads_match_oracle) {  // test_packing.cpp:123-200 vs the oracle
    ModelConfig c = small_config();
    ModelParams params = ModelParams::init(c, 41);
    orc_cfg oc = ocfg(c);
    std::vector<double> w(params.flat().begin(), params.flat().end());
    std::mt19937 rng(17);
    for (int trial = 0; trial < 10; ++trial) {
        std::vector<TokenId> prompt(1 + rng() % 5);
        for (auto& t : prompt) t = rng() % 16;
        std::vector<std::vector<TokenId>> resp(1 + rng() % 4);
        for (auto& r : resp) {
            r.resize(1 + rng() % 5);
            for (auto& t : r) t = rng() % 16;
        }
        PackedGroup pg = pack_group(prompt, resp, c.max_seq_len);
        std::vector<double> up;
        for (const auto& s : pg.spans)
            for (int i = 0; i < s.len; ++i) up.push_back(std::uniform_real_distribution<double>(-1, 1)(rng));
        auto fwd = forward_logprobs(params, pg.tokens, pg.positions, pg.mask, pg.labels, true);
        std::vector<double> gref(w.size(), 0.0), lref(up.size());
        std::vector<int> lens(pg.mask.response_lens);
        int n = orc_forward(&oc, w.data(), pg.tokens.data(), pg.positions.data(), (int)pg.tokens.size(),
                            pg.mask.prompt_len, lens.data(), (int)lens.size(), pg.labels.data(), lref.data(), nullptr,
                            up.data(), gref.data(), nullptr);
        CHECK(n == (int)up.size());
        double lp_err = 0;
        for (int i = 0; i < n; ++i) lp_err = std::max(lp_err, std::fabs(fwd.logprobs[i] - lref[i]));
        CHECK(lp_err < 2e-5);
        GradBuffer gb = backward(params, fwd, up);
        std::vector<double> g(gb.flat().begin(), gb.flat().end());
        double num = 0, den = 0;
        for (std::size_t i = 0; i < g.size(); ++i) {
            num += (g[i] - gref[i]) * (g[i] - gref[i]);
            den += gref[i] * gref[i];
        }
        CHECK(std::sqrt(num / den) < 1e-5);
    }
}

TEST_CASE(single_response_packed_equals_causal_bitwise) {  // test_packing.cpp:153-162
    ModelParams params = ModelParams::init(small_config(), 43);
    std::vector<TokenId> prompt{1, 6, 9, 3}, resp{5, 7, 2};
    PackedGroup pg = pack_group(prompt, {resp}, 64);
    auto packed = forward_logprobs(params, pg.tokens, pg.positions, pg.mask, pg.labels);
    std::vector<TokenId> toks{1, 6, 9, 3, 5, 7, 2};
    std::vector<std::int32_t> labs{-1, -1, -1, -1, 5, 7, 2};
    auto causal = forward_logprobs(params, toks, iota(7), AttentionMaskSpec::causal(), labs);
    CHECK(packed.logprobs == causal.logprobs);
}

TEST_CASE(no_leakage_bitwise) {  // test_packing.cpp:202-223
    ModelConfig c = small_config();
    ModelParams params = ModelParams::init(c, 53);
    std::vector<TokenId> prompt{1, 12, 3};
    PackedGroup base = pack_group(prompt, {{5, 6}, {7, 8}, {9, 10}}, c.max_seq_len);
    PackedGroup mut = pack_group(prompt, {{5, 6}, {13, 14}, {9, 10}}, c.max_seq_len);
    auto b = extract_response_logprobs(forward_logprobs(params, base.tokens, base.positions, base.mask, base.labels).logprobs, base);
    auto m = extract_response_logprobs(forward_logprobs(params, mut.tokens, mut.positions, mut.mask, mut.labels).logprobs, mut);
    CHECK(b[0] == m[0]);
    CHECK(b[2] == m[2]);
}

TEST_CASE(forward_input_validation) {  // test_model.cpp:107-123
    ModelParams p = ModelParams::init(small_config(), 1);
    std::vector<TokenId> tokens{1, 2, 3};
    std::vector<std::int32_t> labels{kIgnoreLabel, 2, 2};
    std::vector<int> short_pos{0, 1};
    CHECK_THROWS_AS(forward_logprobs(p, tokens, short_pos, AttentionMaskSpec::causal(), labels), ShapeError);
    std::vector<TokenId> bad{1, 99, 3};
    CHECK_THROWS_AS(forward_logprobs(p, bad, iota(3), AttentionMaskSpec::causal(), labels), VocabError);
    std::vector<std::int32_t> label0{3, kIgnoreLabel, kIgnoreLabel};
    CHECK_THROWS_AS(forward_logprobs(p, tokens, iota(3), AttentionMaskSpec::causal(), label0), ShapeError);
}

TEST_CASE(backward_linearity_and_lifecycle) {  // test_model.cpp:131-173
    ModelParams p = ModelParams::init(small_config(), 5);
    std::vector<TokenId> tokens{1, 5, 6, 7};
    std::vector<std::int32_t> labels{kIgnoreLabel, 5, 9, 2};
    auto f0 = forward_logprobs(p, tokens, iota(4), AttentionMaskSpec::causal(), labels, true);
    GradBuffer gz = backward(p, f0, std::vector<double>{0, 0, 0});
    for (double v : gz.flat()) CHECK(v == 0.0);
    auto f1 = forward_logprobs(p, tokens, iota(4), AttentionMaskSpec::causal(), labels, true);
    GradBuffer gb1 = backward(p, f1, std::vector<double>{0.3, -1.1, 0.7});
    auto g1 = gb1.flat();
    auto f2 = forward_logprobs(p, tokens, iota(4), AttentionMaskSpec::causal(), labels, true);
    GradBuffer gb2 = backward(p, f2, std::vector<double>{0.6, -2.2, 1.4});
    auto g2 = gb2.flat();
    bool exact = true;
    for (std::size_t i = 0; i < g1.size(); ++i) exact = exact && g2[i] == 2 * g1[i];
    CHECK(exact);
    auto f3 = forward_logprobs(p, tokens, iota(4), AttentionMaskSpec::causal(), labels, true);
    forward_logprobs(p, tokens, iota(4), AttentionMaskSpec::causal(), labels);  // invalidates f3
    CHECK_THROWS_AS(backward(p, f3, std::vector<double>{1, 1, 1}), LifecycleError);
    auto f4 = forward_logprobs(p, tokens, iota(4), AttentionMaskSpec::causal(), labels, true);
    CHECK_THROWS_AS(backward(p, f4, std::vector<double>(5, 1.0)), ShapeError);
    auto nc = forward_logprobs(p, tokens, iota(4), AttentionMaskSpec::causal(), labels);
    CHECK_THROWS_AS(backward(p, nc, std::vector<double>{1, 1, 1}), LifecycleError);
}

TEST_CASE(gradbuffer_accumulate_and_update) {  // test_model.cpp:175-216
    ModelParams p = ModelParams::init(small_config(), 9);
    std::vector<double> w0(p.flat().begin(), p.flat().end());
    std::vector<TokenId> tokens{1, 5, 6, 7};
    std::vector<std::int32_t> labels{kIgnoreLabel, 5, 9, 2};
    auto f = forward_logprobs(p, tokens, iota(4), AttentionMaskSpec::causal(), labels, true);
    GradBuffer g = backward(p, f, std::vector<double>{0.3, -1.1, 0.7});
    GradBuffer acc(p);
    acc.accumulate(g);
    acc.accumulate(g);
    CHECK(acc.micro_step_count() == 2);
    std::vector<double> gf(g.flat().begin(), g.flat().end());
    p.apply_update(acc, 0.5);  // W -= 0.5 * (2g) / 2
    CHECK(p.version() == 1);
    auto w1 = p.flat();
    double err = 0;
    for (std::size_t i = 0; i < w1.size(); ++i) err = std::max(err, std::fabs(w1[i] - (w0[i] - 0.5 * gf[i])));
    CHECK(err < 1e-9);
    GradBuffer empty(p);
    CHECK_THROWS_AS(p.apply_update(empty, 0.1), ConfigError);
}

TEST_CASE(trimodel_identical_weights) {  // test_pipeline.cpp:118-136
    ModelConfig c = small_config();
    TriModel tm = TriModel::init(c, 5);
    std::vector<TokenId> tokens{1, 6, 3, 7, 8};
    std::vector<std::int32_t> labels{kIgnoreLabel, kIgnoreLabel, kIgnoreLabel, 7, 8};
    auto tri = trimodel_forward(tm, tokens, iota(5), AttentionMaskSpec::causal(), labels);
    CHECK(tri.policy.logprobs.size() == 2);
    CHECK(tri.policy.logprobs == tri.old_logprobs);
    CHECK(tri.policy.logprobs == tri.ref_logprobs);
}

TEST_CASE(train_microbatch_matches_oracle) {  // pipeline.cpp:97-141
    ModelConfig c = small_config();
    TriModel tm = TriModel::init(c, 41);
    std::vector<TokenId> prompt{1, 8, 4, 9};
    std::vector<std::vector<TokenId>> resp{{5, 6, 2}, {7}, {9, 10, 11, 3}};
    std::vector<double> rewards{0.2, 0.9, 0.4};
    GradBuffer grads(tm.policy);
    MicrobatchStats stats;
    train_microbatch(tm, prompt, resp, rewards, HyperParams{}, grads, stats);
    orc_cfg oc = ocfg(c);
    std::vector<double> w(tm.policy.flat().begin(), tm.policy.flat().end());
    std::vector<double> adv(3), g(w.size(), 0.0), st(5, 0.0);
    orc_group_advantages(rewards.data(), 3, 0, adv.data());
    std::vector<int> flat{5, 6, 2, 7, 9, 10, 11, 3}, lens{3, 1, 4};
    orc_train_microbatch(&oc, w.data(), w.data(), w.data(), prompt.data(), 4, flat.data(), lens.data(), 3, adv.data(),
                         nullptr, 0.2, 0.04, 0, g.data(), st.data(), nullptr);
    auto gg = grads.flat();
    double num = 0, den = 0;
    for (std::size_t i = 0; i < gg.size(); ++i) {
        num += (gg[i] - g[i]) * (gg[i] - g[i]);
        den += g[i] * g[i];
    }
    CHECK(std::sqrt(num / den) < 1e-5);
    CHECK(std::fabs(stats.objective_sum - st[0]) < 1e-6);
    CHECK(stats.total_units == (long)st[4]);
    CHECK(grads.micro_step_count() == 1);
}

TEST_CASE(checkpoint_round_trip_and_errors) {  // model.cpp:907-987
    ModelConfig c = small_config();
    ModelParams p = ModelParams::init(c, 41);
    const std::string path = "/tmp/parl_dropin_ckpt.parlckp1";
    save_checkpoint(path, p);
    ModelParams q = load_checkpoint(path);
    CHECK(q.config() == c);
    CHECK(std::ranges::equal(q.flat(), p.flat()));
    CHECK(q.version() == p.version());
    CHECK_THROWS_AS(load_checkpoint("/tmp/parl_dropin_missing.parlckp1"), IoError);
}

TEST_CASE(sample_tokens_and_score_logprobs) {  // model.cpp:843-900, rollout.cpp:52-66
    ModelConfig c = small_config();
    ModelParams p = ModelParams::init(c, 41);
    std::vector<TokenId> prompt{5, 9, 11, 4, 7};
    auto a = sample_tokens(p, prompt, 12, 0.8, 3);
    auto b = sample_tokens(p, prompt, 12, 0.8, 3);
    CHECK(a == b);
    CHECK(!a.empty() && a.size() <= 12);
    auto lp = score_logprobs(p, prompt, a);
    CHECK(lp.size() == a.size());
    for (double v : lp) CHECK(v <= 0.0);
    CHECK_THROWS_AS(sample_tokens(p, std::vector<TokenId>{}, 4, 0.0, 0), ShapeError);
    CHECK_THROWS_AS(sample_tokens(p, prompt, -1, 0.0, 0), ConfigError);
}

int main() {
    for (auto& [name, fn] : cases()) {
        const int before = g_fail;
        try {
            fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::fprintf(stderr, "%s: unexpected exception %s\n", name.c_str(), e.what());
        }
        std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name.c_str());
    }
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
