// parl/packing.hpp — drop-in for proj/include/parl/packing.hpp (packing.hpp:13-35):
// pack_group runs the device packer K1 (the host vectors are its downloaded
// outputs, and the packed device sequence rides along for the fused forward);
// build_shared_prompt_mask is evaluated on the device.
#pragma once

#include <span>
#include <vector>

#include "parl/model.hpp"

namespace parl {

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
    std::shared_ptr<parl_group_s> device;  // the K1 outputs on the GPU (no reference counterpart)
};

// packing.cpp:7-45, same validation and errors
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
    detail::check(parl_pack(pg.device.get(), prompt.data(), (int)prompt.size(), flat.data(), lens.data(),
                            (int)lens.size(), max_seq_len),
                  dev.ctx());
    pg.tokens.resize(T);
    pg.labels.resize(T);
    pg.positions.resize(T);
    std::vector<std::int32_t> starts(responses.size());
    detail::check(parl_group_download(pg.device.get(), pg.tokens.data(), pg.labels.data(), pg.positions.data(),
                                      nullptr, nullptr, starts.data(), nullptr),
                  dev.ctx());
    for (std::size_t k = 0; k < responses.size(); ++k) pg.spans.push_back({starts[k], lens[k]});
    pg.mask = AttentionMaskSpec::shared_prompt((int)prompt.size(), std::vector<int>(lens.begin(), lens.end()));
    return pg;
}

// packing.cpp:47-72: row-major [n x n], row i attends to column j
inline std::vector<bool> build_shared_prompt_mask(int prompt_len, std::span<const int> response_lens) {
    Device& dev = Device::get();
    std::vector<std::int32_t> lens(response_lens.begin(), response_lens.end());
    long n = prompt_len;
    for (int r : response_lens) n += r;
    std::vector<std::uint8_t> m(n > 0 ? (std::size_t)n * n : 1);
    detail::check(parl_shared_prompt_mask(dev.ctx(), prompt_len, lens.data(), (int)lens.size(), m.data()), dev.ctx());
    return std::vector<bool>(m.begin(), m.begin() + (std::size_t)n * n);
}

// packing.cpp:74-89
inline std::vector<std::vector<double>> extract_response_logprobs(std::span<const double> logprobs,
                                                                  const PackedGroup& packed) {
    std::size_t expected = 0;
    for (const auto& s : packed.spans) expected += static_cast<std::size_t>(s.len);
    if (logprobs.size() != expected)
        throw ShapeError("logprob vector of length " + std::to_string(logprobs.size()) + " does not match " +
                         std::to_string(expected) + " response tokens");
    std::vector<std::vector<double>> out;
    out.reserve(packed.spans.size());
    std::size_t cursor = 0;
    for (const auto& s : packed.spans) {
        out.emplace_back(logprobs.begin() + cursor, logprobs.begin() + cursor + s.len);
        cursor += static_cast<std::size_t>(s.len);
    }
    return out;
}

}  // namespace parl
