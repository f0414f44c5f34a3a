// C++ caller of the drop-in API (include/sinkr/cuda/router.hpp): the same
// code a user of sinkr::routed_decode_step writes, with sinkr:: -> sinkr::cuda::.
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <vector>

#include "sinkr/cuda/analysis.hpp"
#include "sinkr/cuda/calibration.hpp"
#include "sinkr/cuda/router.hpp"

namespace sc = sinkr::cuda;

#define REQUIRE(c)                                                       \
    do {                                                                 \
        if (!(c)) {                                                      \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
            return 1;                                                    \
        }                                                                \
    } while (0)

template <class E, class F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    const std::size_t L = 777, D = 128, hq = 32, hkv = 8;
    sc::KvCache cache(sc::CacheConfig{2, hq, hkv, D, 1024, 1});
    std::mt19937 rng(7);
    std::normal_distribution<float> n01;
    std::vector<float> q(hq * D);
    for (auto& x : q) x = n01(rng);
    REQUIRE(throws<std::runtime_error>([&] {
        sc::routed_decode_step(q, 0, cache, sc::RoutingConfig{});
    }));  // empty cache (router.cpp:90)
    for (std::size_t layer = 0; layer < 2; ++layer)
        for (std::size_t g = 0; g < hkv; ++g) {
            std::vector<float> k(L * D), v(L * D);
            for (auto& x : k) x = n01(rng);
            for (auto& x : v) x = n01(rng);
            cache.append(layer, g, k, v);
        }
    REQUIRE(cache.token_count() == L);
    REQUIRE(std::fabs(cache.anchor(0, 0).k0_norm) > 0.0f);

    std::fprintf(stderr, "step: dense layer 1\n");
    // routing disabled: every group attends the whole cache
    auto cfg = sc::RoutingConfig::from_profile(sc::ThresholdProfile::constant(2.0));
    auto r = sc::routed_decode_step(q, 1, cache, cfg);
    REQUIRE(r.counters.groups_active == hkv && r.counters.groups_skipped == 0);
    REQUIRE(r.counters.kv_floats_loaded == hkv * 2 * L * D);
    for (auto& g : r.groups) REQUIRE(!g.decision.sink && g.decision.head_scores.size() == 4);

    // full skip on a routable layer: bitwise-zero outputs, no KV traffic
    sc::RoutingConfig skip;
    skip.profile = sc::ThresholdProfile::constant(-2.0);
    skip.excluded_layers = {0};  // layer 1 routable, layer 0 excluded
    std::fprintf(stderr, "step: full skip layer 1\n");
    auto s = sc::routed_decode_step(q, 1, cache, skip);
    REQUIRE(s.counters.groups_skipped == hkv && s.counters.kv_floats_loaded == 0);
    for (float x : s.outputs) REQUIRE(x == 0.0f && !std::signbit(x));
    // ... but never on an excluded layer (router.hpp:19)
    std::fprintf(stderr, "step: excluded layer 0\n");
    auto e = sc::routed_decode_step(q, 0, cache, skip);
    REQUIRE(e.counters.groups_active == hkv);

    REQUIRE(throws<std::out_of_range>([&] { sc::routed_decode_step(q, 2, cache, cfg); }));
    REQUIRE(throws<std::invalid_argument>([&] {
        sc::routed_decode_step(std::span<const float>(q.data(), 5), 0, cache, cfg);
    }));
    REQUIRE(throws<std::invalid_argument>([&] { sc::split_ranges(3, 4); }));
    const auto sr = sc::split_ranges(10, 3);
    REQUIRE(sr[1].first == 4 && sr[1].second == 7);
    REQUIRE(sc::threshold_for_length(5, sc::ThresholdProfile{{1, 0, 0, 0}, 10.0, 0.0, 1.0}) ==
            0.125);

    // calibration.hpp: a collector over the GPU's routing-phase-only scores
    std::fprintf(stderr, "calibrate\n");
    const std::vector<std::size_t> lens{100, 200, 400, 600, 777};
    std::vector<std::size_t> seen;
    auto collect = [&](std::size_t len) {
        seen.push_back(len);
        sc::ScorePopulation pop;
        std::normal_distribution<float> shift(0.02f * (float)len / 100.0f, 1.0f);
        std::vector<float> qs(8 * hq * D);  // the length's 8 samples
        for (auto& x : qs) x = shift(rng);
        // one launch for all samples, bit-identical to one call per sample
        const auto batch = sc::collect_group_scores_batch(cache, qs, 1);
        for (int sample = 0; sample < 8; ++sample) {
            const auto one = sc::collect_group_scores(
                cache, std::span<const float>(qs.data() + sample * hq * D, hq * D), 1);
            for (std::size_t g = 0; g < one.size(); ++g) {
                if (one[g] != batch[sample * one.size() + g])
                    throw std::runtime_error("collect_group_scores_batch != collect_group_scores");
                pop.add(one[g], 1, len);
            }
        }
        return pop;
    };
    auto prof = sc::calibrate(collect, lens, 0.6, 0.65, {0});
    REQUIRE(seen == lens && prof.points.size() == lens.size());
    REQUIRE(prof.length_normalizer == 777.0);
    const auto path = std::filesystem::temp_directory_path() / "sinkr_shim_profile.json";
    sc::save_profile(path, prof);
    const auto back = sc::load_profile(path);
    REQUIRE(back.coeffs == prof.coeffs && back.points.size() == prof.points.size());
    REQUIRE(throws<std::invalid_argument>([&] {
        sc::calibrate(collect, std::vector<std::size_t>{1, 2, 3}, 0.6, 0.65);
    }));

    // attention.hpp:76-85: splitk_attention of one cached group
    const auto sk = sc::splitk_attention(cache, std::span<const float>(q.data(), 4 * D), 1, 0, 2);
    REQUIRE(sk.out.size() == 4 * D && sk.counters.kv_floats_loaded == 2 * L * D);
    REQUIRE(throws<std::invalid_argument>([&] {
        sc::splitk_attention(cache, std::span<const float>(q.data(), 4 * D), 1, 0, 0);
    }));

    // attention.hpp:14-85 over host spans, as a reference caller writes it
    std::fprintf(stderr, "span operators\n");
    {
        const std::size_t n = 1500, d = 80, h = 3;
        std::vector<float> kk(n * d), vv(n * d), qq(h * d);
        for (auto& x : kk) x = n01(rng);
        for (auto& x : vv) x = n01(rng);
        for (auto& x : qq) x = 2.0f * n01(rng);
        const auto qg = sc::QueryGroup::over(qq, h, d);
        REQUIRE(qg.scale == 1.0f / std::sqrt(80.0f));
        sc::ThreadPool pool(4);
        const auto spk = sc::splitk_attention(qg, kk, vv, n, 3, &pool);
        REQUIRE(spk.counters.kv_floats_loaded == 2 * n * d);
        const auto on = sc::online_attention(qg, kk, vv, n);
        const auto de = sc::dense_attention(qg, kk, vv, n);
        std::vector<sc::SplitPartial> parts;
        for (auto [a, b] : sc::split_ranges(n, 4))
            parts.push_back(sc::attend_chunk(qg, std::span<const float>(kk).subspan(a * d, (b - a) * d),
                                             std::span<const float>(vv).subspan(a * d, (b - a) * d), b - a));
        parts.insert(parts.begin() + 1, sc::SplitPartial{});  // empty: skipped by the merge
        REQUIRE(parts[0].tokens == 375 && parts[0].m.size() == h && parts[0].acc.size() == h * d);
        const auto mg = sc::merge_partials(parts, h, d);
        float dm = 0.0f;
        for (std::size_t i = 0; i < h * d; ++i) {
            dm = std::fmax(dm, std::fabs(mg[i] - spk.out[i]));
            dm = std::fmax(dm, std::fabs(on[i] - de[i]));
            dm = std::fmax(dm, std::fabs(on[i] - spk.out[i]));
        }
        REQUIRE(dm <= 1e-6f);
        std::vector<sc::SplitPartial> none(2);
        REQUIRE(throws<std::invalid_argument>([&] { sc::merge_partials(none, h, d); }));
        REQUIRE(throws<std::invalid_argument>([&] { sc::attend_chunk(qg, kk, vv, n, 0); }));
        REQUIRE(throws<std::invalid_argument>([&] { sc::splitk_attention(qg, kk, vv, n, 0); }));
        REQUIRE(throws<std::invalid_argument>([&] {
            sc::dense_attention(qg, std::span<const float>(kk).first(d * 3), vv, n);
        }));
        // attend_chunk over a cached range == over the same rows as a span
        const auto [hk, hv] = cache.historical(1, 2, 100, 600);
        const std::span<const float> gq(q.data() + 8 * D, 4 * D);
        const auto pc = sc::attend_chunk(cache, gq, 1, 2, 100, 600);
        const auto ps = sc::attend_chunk(sc::QueryGroup::over(gq, 4, D), hk, hv, 500);
        REQUIRE(pc.tokens == 500 && pc.m == ps.m);  // logits are bit-exact: maxima equal
        for (std::size_t i = 0; i < 4 * D; ++i)
            REQUIRE(std::fabs(pc.acc[i] - ps.acc[i]) <= 1e-12 * (1.0 + std::fabs(ps.acc[i])));
        REQUIRE(throws<std::out_of_range>([&] { sc::attend_chunk(cache, gq, 1, 2, 100, L + 1); }));
    }

    // analysis.hpp: GPU BOS mass, oracle labels, PR curve
    const auto a0 = sc::attention_bos_mass(cache, q, 1);
    for (double a : a0) REQUIRE(a > 0.0 && a < 1.0);
    const auto w = sc::attention_weights(cache, std::span<const float>(q.data(), 4 * D), 1, 0);
    REQUIRE(w.size() == 4 * L && std::fabs(w[0] - a0[0]) < 1e-6);
    REQUIRE(sc::last_kernel_seconds(cache) > 0.0);
    const auto labs = sc::oracle_labels(w, 4, L, 0.65, sc::OracleMode::GroupMean);
    REQUIRE(labs.size() == 1 && !labs[0].is_sink);
    const std::vector<double> sco{0.9, 0.8, 0.3, 0.1};
    const std::vector<std::uint8_t> lab{1, 1, 0, 0};
    REQUIRE(sc::pr_curve(sco, lab).auprc == 1.0);

    // kv_cache.hpp:72-80: snapshot round trip
    std::fprintf(stderr, "snapshot\n");
    const auto dir = std::filesystem::temp_directory_path() / "sinkr_shim_snapshot";
    cache.save_snapshot(dir);
    auto loaded = sc::KvCache::load_snapshot(dir);
    REQUIRE(loaded.token_count() == L && loaded.config().num_layers == 2);
    REQUIRE(loaded.historical(1, 5, 0, L).first == cache.historical(1, 5, 0, L).first);
    auto r2 = sc::routed_decode_step(q, 1, loaded, cfg);
    float md = 0.0f;  // Split-K partials merge in claim order: equal within tolerance
    for (std::size_t i = 0; i < r.outputs.size(); ++i) md = std::fmax(md, std::fabs(r2.outputs[i] - r.outputs[i]));
    REQUIRE(md <= 1e-5f);
    std::filesystem::remove_all(dir);
    std::filesystem::remove(path);
    std::printf("shim OK (%.1f us attention)\n", r.counters.attention_seconds * 1e6);
    return 0;
}
