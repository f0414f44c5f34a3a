// sinkr/cuda/calibration.hpp — the reference's calibration.hpp API (threshold
// calibration) over the C-ABI.  Statistics and the cubic fit
// are the library's host C++ (bit-identical to the reference); score
// populations can come from the GPU's routing-phase-only collector.
#pragma once

#include <algorithm>
#include <filesystem>
#include <functional>
#include <set>
#include <stdexcept>
#include <span>
#include <utility>
#include <vector>

#include "router.hpp"

namespace sinkr::cuda {

struct ScoreSample {
    double score = 0.0;
    std::size_t layer = 0;
    std::size_t length = 0;
};

struct ScorePopulation {  // calibration.hpp:43-50
    std::vector<ScoreSample> samples;
    void add(double score, std::size_t layer, std::size_t length) {
        samples.push_back({score, layer, length});
    }
    std::size_t size() const { return samples.size(); }
    bool empty() const { return samples.empty(); }
    std::vector<double> scores() const {
        std::vector<double> out;
        out.reserve(samples.size());
        for (const auto& s : samples) out.push_back(s.score);
        return out;
    }
};

inline std::vector<std::pair<double, double>> sweep(const ScorePopulation& pop,
                                                    std::span<const double> thresholds) {
    const auto s = pop.scores();
    std::vector<double> r(thresholds.size());
    check(sinkr_sweep(s.data(), s.size(), thresholds.data(), thresholds.size(), r.data()));
    std::vector<std::pair<double, double>> out;
    for (std::size_t i = 0; i < r.size(); ++i) out.emplace_back(thresholds[i], r[i]);
    return out;
}

inline double skip_ratio_at(const ScorePopulation& pop, double threshold) {
    const auto s = pop.scores();
    double out = 0.0;
    check(sinkr_skip_ratio_at(s.data(), s.size(), threshold, &out));
    return out;
}

inline double solve_threshold(const ScorePopulation& pop, double target_skip) {
    const auto s = pop.scores();
    double out = 0.0;
    check(sinkr_solve_threshold(s.data(), s.size(), target_skip, &out));
    return out;
}

struct CubicFit {
    std::array<double, 4> coeffs{0.0, 0.0, 0.0, 0.0};
    double residual = 0.0;
};

inline CubicFit fit_cubic(std::span<const std::pair<double, double>> points) {
    std::vector<double> x, y;
    for (const auto& [a, b] : points) {
        x.push_back(a);
        y.push_back(b);
    }
    CubicFit f;
    check(sinkr_fit_cubic(x.data(), y.data(), x.size(), f.coeffs.data(), &f.residual));
    return f;
}

using ScoreCollector = std::function<ScorePopulation(std::size_t length)>;

namespace detail {
inline ThresholdProfile from_c(const sinkr_profile& p) {
    ThresholdProfile t;
    for (int i = 0; i < 4; ++i) t.coeffs[i] = p.threshold.coeffs[i];
    t.length_normalizer = p.threshold.length_normalizer;
    t.clamp_lo = p.threshold.clamp_lo;
    t.clamp_hi = p.threshold.clamp_hi;
    t.target_skip = p.target_skip;
    t.gamma = p.gamma;
    t.excluded_layers.assign(p.excluded_layers, p.excluded_layers + p.num_excluded_layers);
    t.points.clear();
    for (std::size_t i = 0; i < p.num_points; ++i)
        t.points.push_back({p.points[i].length, p.points[i].tau, p.points[i].skip});
    return t;
}
inline sinkr_profile to_c(const ThresholdProfile& t) {
    sinkr_profile p{};
    p.threshold = t.c();
    p.target_skip = t.target_skip;
    p.gamma = t.gamma;
    if (t.excluded_layers.size() > SINKR_MAX_EXCLUDED_LAYERS ||
        t.points.size() > SINKR_MAX_CALIBRATION_POINTS)
        throw std::invalid_argument("profile too large for the C-ABI");
    p.num_excluded_layers = t.excluded_layers.size();
    for (std::size_t i = 0; i < t.excluded_layers.size(); ++i) p.excluded_layers[i] = t.excluded_layers[i];
    p.num_points = t.points.size();
    for (std::size_t i = 0; i < t.points.size(); ++i)
        p.points[i] = sinkr_calibration_point{t.points[i].length, t.points[i].tau, t.points[i].skip};
    return p;
}
}  // namespace detail

// calibration.hpp:79-83: the collector runs once per distinct length.
inline ThresholdProfile calibrate(const ScoreCollector& collect,
                                  std::span<const std::size_t> lengths, double target_skip,
                                  double gamma,
                                  const std::vector<std::size_t>& excluded_layers = {0, 1}) {
    std::set<std::size_t> distinct(lengths.begin(), lengths.end());
    if (distinct.size() < 4) throw std::invalid_argument("calibration needs at least 4 distinct lengths");
    std::vector<std::size_t> lens, layers, offsets{0};
    std::vector<double> scores;
    for (std::size_t L : distinct) {
        const ScorePopulation pop = collect(L);
        for (const auto& s : pop.samples) {
            scores.push_back(s.score);
            layers.push_back(s.layer);
        }
        lens.push_back(L);
        offsets.push_back(scores.size());
    }
    sinkr_profile out{};
    check(sinkr_calibrate(lens.data(), lens.size(), scores.data(), layers.data(), offsets.data(),
                          target_skip, gamma, excluded_layers.data(), excluded_layers.size(), &out));
    return detail::from_c(out);
}

inline void save_profile(const std::filesystem::path& path, const ThresholdProfile& profile) {
    const auto p = detail::to_c(profile);
    check(sinkr_save_profile(path.string().c_str(), &p));
}

inline ThresholdProfile load_profile(const std::filesystem::path& path) {
    sinkr_profile p{};
    check(sinkr_load_profile(path.string().c_str(), &p));
    return detail::from_c(p);
}

// Score-collection mode on the GPU (routing phase alone): group scores of all
// B sequences of `layer` for one query block [B][H_q][D].
inline std::vector<double> collect_group_scores(const KvCache& cache,
                                                std::span<const float> queries,
                                                std::size_t layer) {
    const auto& c = cache.config();
    std::vector<double> gs(c.num_seqs * c.num_kv_heads);
    check(sinkr_collect_scores(cache.handle(), queries.data(), layer, nullptr, nullptr, gs.data(),
                               nullptr));
    return gs;
}

// The same for n query blocks [n][B][H_q][D] over one layer in one launch
// (a calibration length's samples): group scores [n][B*H_kv], bit-identical
// to n collect_group_scores calls.
inline std::vector<double> collect_group_scores_batch(const KvCache& cache,
                                                      std::span<const float> queries,
                                                      std::size_t layer) {
    const auto& c = cache.config();
    const std::size_t per = c.num_seqs * c.num_q_heads * c.head_dim;
    if (per == 0 || queries.size() % per != 0)
        throw std::invalid_argument("queries must be n x B x H_q x D for one layer");
    const std::size_t n = queries.size() / per;
    std::vector<double> gs(n * c.num_seqs * c.num_kv_heads);
    if (n)
        check(sinkr_collect_scores_batch(cache.handle(), queries.data(), n, layer, nullptr, nullptr,
                                         gs.data(), nullptr));
    return gs;
}

}  // namespace sinkr::cuda
