// sinkr/cuda/analysis.hpp — proxy-reliability analysis:
// the reference's analysis.hpp oracle-label / PR API plus the GPU's
// full-attention BOS mass and attention_weights (attention.cpp:75-99).
#pragma once

#include <span>
#include <stdexcept>
#include <vector>

#include "router.hpp"

namespace sinkr::cuda {

enum class OracleMode { Head, GroupMean };

struct OracleLabel {
    double alpha0 = 0.0;
    bool is_sink = false;
};

// analysis.hpp:17-19: rows must sum to 1 within 1e-4.
inline std::vector<OracleLabel> oracle_labels(std::span<const float> weights, std::size_t heads,
                                              std::size_t len, double gamma, OracleMode mode) {
    if (weights.size() != heads * len) throw std::invalid_argument("weights must be heads x len");
    std::vector<double> a0(heads);
    for (std::size_t h = 0; h < heads; ++h) {
        double s = 0.0;
        for (std::size_t i = 0; i < len; ++i) s += weights[h * len + i];
        if (s < 1.0 - 1e-4 || s > 1.0 + 1e-4)
            throw std::invalid_argument("attention weight rows must sum to 1 within 1e-4");
        a0[h] = weights[h * len];
    }
    const int m = mode == OracleMode::Head ? 0 : 1;
    const std::size_t n = m == 0 ? heads : 1;
    std::vector<double> la(n);
    std::vector<std::uint8_t> sk(n);
    check(sinkr_oracle_labels(a0.data(), heads, heads, gamma, m, la.data(), sk.data()));
    std::vector<OracleLabel> out(n);
    for (std::size_t i = 0; i < n; ++i) out[i] = {la[i], sk[i] != 0};
    return out;
}

struct PrPoint {
    double threshold = 0.0;
    double precision = 0.0;
    double recall = 0.0;
    double f1 = 0.0;
};

struct PrCurve {
    std::vector<PrPoint> points;
    double auprc = 0.0;
};

inline PrCurve pr_curve(std::span<const double> scores, std::span<const std::uint8_t> labels) {
    if (scores.size() != labels.size()) throw std::invalid_argument("scores/labels length mismatch");
    std::vector<double> pts(4 * (scores.size() ? scores.size() : 1));
    std::size_t n = 0;
    PrCurve c;
    check(sinkr_pr_curve(scores.data(), labels.data(), scores.size(), pts.data(), &n, &c.auprc));
    for (std::size_t i = 0; i < n; ++i) c.points.push_back({pts[4 * i], pts[4 * i + 1], pts[4 * i + 2], pts[4 * i + 3]});
    return c;
}

// GPU: alpha0 of every query head of all B sequences ([B][H_q]).
inline std::vector<double> attention_bos_mass(const KvCache& cache, std::span<const float> queries,
                                              std::size_t layer) {
    const auto& c = cache.config();
    std::vector<double> a0(c.num_seqs * c.num_q_heads);
    check(sinkr_attention_bos_mass(cache.handle(), queries.data(), layer, a0.data()));
    return a0;
}

// GPU attention_weights for one GQA group: [r][len] over the slot's rows.
inline std::vector<float> attention_weights(const KvCache& cache, std::span<const float> group_q,
                                            std::size_t layer, std::size_t kv_head,
                                            std::size_t seq = 0) {
    const std::size_t L = cache.length(layer, kv_head, seq);
    std::vector<float> w(cache.config().group_width() * L);
    check(sinkr_attention_weights(cache.handle(), group_q.data(), seq, layer, kv_head, w.data()));
    return w;
}

// Device time of the last attention_bos_mass / attention_weights call's kernels.
inline double last_kernel_seconds(const KvCache& cache) {
    double s = 0.0;
    check(sinkr_attention_last_kernel_seconds(cache.handle(), &s));
    return s;
}

}  // namespace sinkr::cuda
