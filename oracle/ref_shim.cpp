// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/).  It
// lets the Python tests and bench.py's reference arm call the reference's own
// sinkr:: API through ctypes.  No reference source is copied here: this file
// only includes the reference headers and forwards arguments.
//
// Error convention (mirrors include/sinkr_cuda.h's sinkr_status):
//   0 ok, 1 invalid_argument, 2 out_of_range, 3 runtime_error, 4 logic_error,
//   5 other exception.  The message is kept in a thread-local buffer.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "sinkr/attention.hpp"
#include "sinkr/calibration.hpp"
#include "sinkr/kv_cache.hpp"
#include "sinkr/parallel.hpp"
#include "sinkr/router.hpp"
#include "sinkr/tensor.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

sinkr::ThresholdProfile make_profile(const double* coeffs, double normalizer, double lo,
                                     double hi) {
    sinkr::ThresholdProfile p;
    for (int i = 0; i < 4; ++i) p.coeffs[i] = coeffs[i];
    p.length_normalizer = normalizer;
    p.clamp_lo = lo;
    p.clamp_hi = hi;
    return p;
}

sinkr::QueryGroup group_of(const float* q, std::size_t heads, std::size_t dim) {
    return sinkr::QueryGroup::over(std::span<const float>(q, heads * dim), heads, dim);
}

void copy_partial(const sinkr::SplitPartial& p, double* m, double* l, double* acc,
                  std::size_t* tokens) {
    std::memcpy(m, p.m.data(), p.m.size() * sizeof(double));
    std::memcpy(l, p.l.data(), p.l.size() * sizeof(double));
    std::memcpy(acc, p.acc.data(), p.acc.size() * sizeof(double));
    *tokens = p.tokens;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- scalar routing helpers (router.hpp:41-54,78) -------------------------
int ref_proxy_score(const float* q, const float* k0, float k0_norm, std::size_t d,
                    double* score, int* degenerate) {
    return guard([&] {
        sinkr::GroupAnchor a;
        a.k0.assign(k0, k0 + d);
        a.k0_norm = k0_norm;
        const auto s = sinkr::proxy_score(std::span<const float>(q, d), a);
        *score = s.value;
        *degenerate = s.degenerate ? 1 : 0;
    });
}

int ref_group_score(const double* scores, std::size_t n, std::size_t width, double* out) {
    return guard([&] { *out = sinkr::group_score(std::span<const double>(scores, n), width); });
}

int ref_threshold_for_length(std::size_t len, const double* coeffs, double normalizer,
                             double lo, double hi, double* out) {
    return guard([&] {
        *out = sinkr::threshold_for_length(len, make_profile(coeffs, normalizer, lo, hi));
    });
}

int ref_profile_constant(double tau, double* coeffs, double* normalizer, double* lo,
                         double* hi) {
    return guard([&] {
        const auto p = sinkr::ThresholdProfile::constant(tau);
        for (int i = 0; i < 4; ++i) coeffs[i] = p.coeffs[i];
        *normalizer = p.length_normalizer;
        *lo = p.clamp_lo;
        *hi = p.clamp_hi;
    });
}

int ref_route(std::size_t layer, double score, std::size_t len, const double* coeffs,
              double normalizer, double lo, double hi, const std::size_t* excluded,
              std::size_t n_excluded, int sink_on_tie, int* sink, double* threshold) {
    return guard([&] {
        sinkr::RoutingConfig cfg;
        cfg.profile = make_profile(coeffs, normalizer, lo, hi);
        cfg.excluded_layers.assign(excluded, excluded + n_excluded);
        cfg.sink_on_tie = sink_on_tie != 0;
        const auto d = sinkr::route(layer, score, len, cfg);
        *sink = d.sink ? 1 : 0;
        *threshold = d.threshold;
    });
}

std::size_t ref_auto_num_splits(std::size_t len) { return sinkr::auto_num_splits(len); }

int ref_split_ranges(std::size_t len, std::size_t n, std::size_t* from_to) {
    return guard([&] {
        const auto r = sinkr::split_ranges(len, n);
        for (std::size_t i = 0; i < r.size(); ++i) {
            from_to[2 * i] = r[i].first;
            from_to[2 * i + 1] = r[i].second;
        }
    });
}

// ---- attention engine (attention.hpp:38-85) --------------------------------
int ref_dense_attention(const float* q, std::size_t heads, std::size_t dim, const float* k,
                        const float* v, std::size_t len, float* out) {
    return guard([&] {
        const auto o = sinkr::dense_attention(group_of(q, heads, dim),
                                              std::span<const float>(k, len * dim),
                                              std::span<const float>(v, len * dim), len);
        std::memcpy(out, o.data(), o.size() * sizeof(float));
    });
}

int ref_online_attention(const float* q, std::size_t heads, std::size_t dim, const float* k,
                         const float* v, std::size_t len, std::size_t block, float* out) {
    return guard([&] {
        const auto o = sinkr::online_attention(group_of(q, heads, dim),
                                               std::span<const float>(k, len * dim),
                                               std::span<const float>(v, len * dim), len,
                                               block);
        std::memcpy(out, o.data(), o.size() * sizeof(float));
    });
}

int ref_attention_weights(const float* q, std::size_t heads, std::size_t dim, const float* k,
                          std::size_t len, float* out) {
    return guard([&] {
        const auto o = sinkr::attention_weights(group_of(q, heads, dim),
                                                std::span<const float>(k, len * dim), len);
        std::memcpy(out, o.data(), o.size() * sizeof(float));
    });
}

int ref_attend_chunk(const float* q, std::size_t heads, std::size_t dim, const float* k,
                     const float* v, std::size_t len, std::size_t block, double* m, double* l,
                     double* acc, std::size_t* tokens) {
    return guard([&] {
        const auto p = sinkr::attend_chunk(group_of(q, heads, dim),
                                           std::span<const float>(k, len * dim),
                                           std::span<const float>(v, len * dim), len, block);
        copy_partial(p, m, l, acc, tokens);
    });
}

// parts laid out as n_parts x {m[heads], l[heads], acc[heads*dim], tokens}
int ref_merge_partials(std::size_t n_parts, const double* m, const double* l, const double* acc,
                       const std::size_t* tokens, std::size_t heads, std::size_t dim,
                       float* out) {
    return guard([&] {
        std::vector<sinkr::SplitPartial> parts(n_parts);
        for (std::size_t i = 0; i < n_parts; ++i) {
            parts[i].m.assign(m + i * heads, m + (i + 1) * heads);
            parts[i].l.assign(l + i * heads, l + (i + 1) * heads);
            parts[i].acc.assign(acc + i * heads * dim, acc + (i + 1) * heads * dim);
            parts[i].tokens = tokens[i];
        }
        const auto o = sinkr::merge_partials(parts, heads, dim);
        std::memcpy(out, o.data(), o.size() * sizeof(float));
    });
}

void* ref_pool_create(unsigned workers) { return new sinkr::ThreadPool(workers); }
void ref_pool_destroy(void* p) { delete static_cast<sinkr::ThreadPool*>(p); }

int ref_splitk_attention(const float* q, std::size_t heads, std::size_t dim, const float* k,
                         const float* v, std::size_t len, std::size_t splits, void* pool,
                         std::size_t block, float* out, std::uint64_t* kv_floats) {
    return guard([&] {
        const auto r = sinkr::splitk_attention(
            group_of(q, heads, dim), std::span<const float>(k, len * dim),
            std::span<const float>(v, len * dim), len, splits,
            static_cast<sinkr::ThreadPool*>(pool), block);
        std::memcpy(out, r.out.data(), r.out.size() * sizeof(float));
        *kv_floats = r.counters.kv_floats_loaded;
    });
}

// ---- KvCache (kv_cache.hpp:42-80) -------------------------------------------
int ref_cache_create(std::size_t layers, std::size_t hq, std::size_t hkv, std::size_t dim,
                     std::size_t capacity, void** out) {
    return guard([&] {
        *out = new sinkr::KvCache(sinkr::CacheConfig{layers, hq, hkv, dim, capacity});
    });
}

void ref_cache_destroy(void* c) { delete static_cast<sinkr::KvCache*>(c); }

// Appends `rows` rows (row-major rows x dim) one row at a time through the
// reference's KvCache::append, so anchor capture follows kv_cache.cpp:61-84.
int ref_cache_append_rows(void* c, std::size_t layer, std::size_t head, const float* k,
                          const float* v, std::size_t rows) {
    return guard([&] {
        auto* cache = static_cast<sinkr::KvCache*>(c);
        const std::size_t d = cache->config().head_dim;
        for (std::size_t i = 0; i < rows; ++i)
            cache->append(layer, head, std::span<const float>(k + i * d, d),
                          std::span<const float>(v + i * d, d));
    });
}

int ref_cache_anchor(void* c, std::size_t layer, std::size_t head, float* k0, float* norm) {
    return guard([&] {
        auto* cache = static_cast<sinkr::KvCache*>(c);
        sinkr::LoadCounters ctr;
        const auto& a = cache->anchor(layer, head, ctr);
        std::memcpy(k0, a.k0.data(), a.k0.size() * sizeof(float));
        *norm = a.k0_norm;
    });
}

int ref_cache_token_count(void* c, std::size_t* out) {
    return guard([&] { *out = static_cast<sinkr::KvCache*>(c)->token_count(); });
}

// ---- routed_decode_step (router.hpp:84-86) ----------------------------------
// Per-group outputs: score, threshold, sink, degenerate, kv_floats; head scores
// are H_q doubles in query-head order.  counters_u64 = {kv_floats,
// anchor_floats, groups_active, groups_skipped}; seconds = {routing,
// attention, merge}.
int ref_routed_decode_step(void* c, const float* queries, std::size_t layer,
                           const double* coeffs, double normalizer, double lo, double hi,
                           const std::size_t* excluded, std::size_t n_excluded,
                           int sink_on_tie, std::size_t num_splits, std::size_t block,
                           void* pool, int observe_only, float* outputs, double* group_scores,
                           double* thresholds, int* sink, int* degenerate,
                           std::uint64_t* group_kv_floats, double* head_scores,
                           std::uint64_t* counters_u64, double* seconds) {
    return guard([&] {
        auto* cache = static_cast<sinkr::KvCache*>(c);
        const auto& cc = cache->config();
        sinkr::RoutingConfig cfg;
        cfg.profile = make_profile(coeffs, normalizer, lo, hi);
        cfg.excluded_layers.assign(excluded, excluded + n_excluded);
        cfg.sink_on_tie = sink_on_tie != 0;
        sinkr::EngineOptions opt;
        opt.num_splits = num_splits;
        opt.block_size = block;
        opt.pool = static_cast<sinkr::ThreadPool*>(pool);
        opt.observe_only = observe_only != 0;
        const auto r = sinkr::routed_decode_step(
            std::span<const float>(queries, cc.num_q_heads * cc.head_dim), layer, *cache, cfg,
            opt);
        std::memcpy(outputs, r.outputs.data(), r.outputs.size() * sizeof(float));
        const std::size_t rw = cc.group_width();
        for (std::size_t g = 0; g < r.groups.size(); ++g) {
            const auto& d = r.groups[g].decision;
            group_scores[g] = d.group_score;
            thresholds[g] = d.threshold;
            sink[g] = d.sink ? 1 : 0;
            degenerate[g] = d.degenerate ? 1 : 0;
            group_kv_floats[g] = r.groups[g].kv_floats_loaded;
            for (std::size_t i = 0; i < rw; ++i) head_scores[g * rw + i] = d.head_scores[i];
        }
        counters_u64[0] = r.counters.kv_floats_loaded;
        counters_u64[1] = r.counters.anchor_floats_loaded;
        counters_u64[2] = r.counters.groups_active;
        counters_u64[3] = r.counters.groups_skipped;
        seconds[0] = r.counters.routing_seconds;
        seconds[1] = r.counters.attention_seconds;
        seconds[2] = r.counters.merge_seconds;
    });
}

// ---- calibration (calibration.hpp:36-90) -------------------------------------
namespace {
sinkr::ScorePopulation pop_of(const double* s, const std::size_t* layers, std::size_t n,
                              std::size_t length) {
    sinkr::ScorePopulation p;
    for (std::size_t i = 0; i < n; ++i) p.add(s[i], layers ? layers[i] : 0, length);
    return p;
}
// profile <-> flat arrays: coeffs[4], norm, lo, hi, target, gamma | excluded | points (len,tau,skip)
void profile_out(const sinkr::ThresholdProfile& p, double* f8, std::size_t* excluded,
                 std::size_t* n_excl, double* points, std::size_t* n_points) {
    for (int i = 0; i < 4; ++i) f8[i] = p.coeffs[i];
    f8[4] = p.length_normalizer;
    f8[5] = p.clamp_lo;
    f8[6] = p.clamp_hi;
    f8[7] = p.target_skip;
    f8[8] = p.gamma;
    *n_excl = p.excluded_layers.size();
    for (std::size_t i = 0; i < p.excluded_layers.size(); ++i) excluded[i] = p.excluded_layers[i];
    *n_points = p.points.size();
    for (std::size_t i = 0; i < p.points.size(); ++i) {
        points[3 * i] = (double)p.points[i].length;
        points[3 * i + 1] = p.points[i].tau;
        points[3 * i + 2] = p.points[i].skip;
    }
}
}  // namespace

int ref_sweep(const double* s, std::size_t n, const double* t, std::size_t m, double* out) {
    return guard([&] {
        const auto r = sinkr::sweep(pop_of(s, nullptr, n, 0), std::span<const double>(t, m));
        for (std::size_t i = 0; i < r.size(); ++i) out[i] = r[i].second;
    });
}

int ref_skip_ratio_at(const double* s, std::size_t n, double t, double* out) {
    return guard([&] { *out = sinkr::skip_ratio_at(pop_of(s, nullptr, n, 0), t); });
}

int ref_solve_threshold(const double* s, std::size_t n, double target, double* out) {
    return guard([&] { *out = sinkr::solve_threshold(pop_of(s, nullptr, n, 0), target); });
}

int ref_fit_cubic(const double* x, const double* y, std::size_t n, double* coeffs,
                  double* residual) {
    return guard([&] {
        std::vector<std::pair<double, double>> pts;
        for (std::size_t i = 0; i < n; ++i) pts.emplace_back(x[i], y[i]);
        const auto f = sinkr::fit_cubic(pts);
        for (int i = 0; i < 4; ++i) coeffs[i] = f.coeffs[i];
        *residual = f.residual;
    });
}

// calibrate with a collector replaying caller-given populations (one per length)
int ref_calibrate(const std::size_t* lengths, std::size_t n_lengths, const double* scores,
                  const std::size_t* layers, const std::size_t* offsets, double target,
                  double gamma, const std::size_t* excluded, std::size_t n_excl, double* f8,
                  std::size_t* excl_out, std::size_t* n_excl_out, double* points,
                  std::size_t* n_points, std::size_t* calls) {
    return guard([&] {
        *calls = 0;
        sinkr::ScoreCollector collect = [&](std::size_t len) {
            ++*calls;
            for (std::size_t i = 0; i < n_lengths; ++i)
                if (lengths[i] == len)
                    return pop_of(scores + offsets[i], layers + offsets[i],
                                  offsets[i + 1] - offsets[i], len);
            return sinkr::ScorePopulation{};
        };
        const auto p = sinkr::calibrate(collect, std::span<const std::size_t>(lengths, n_lengths),
                                        target, gamma,
                                        std::vector<std::size_t>(excluded, excluded + n_excl));
        profile_out(p, f8, excl_out, n_excl_out, points, n_points);
    });
}

int ref_save_profile(const char* path, const double* f8, const std::size_t* excluded,
                     std::size_t n_excl, const double* points, std::size_t n_points) {
    return guard([&] {
        sinkr::ThresholdProfile p;
        for (int i = 0; i < 4; ++i) p.coeffs[i] = f8[i];
        p.length_normalizer = f8[4];
        p.clamp_lo = f8[5];
        p.clamp_hi = f8[6];
        p.target_skip = f8[7];
        p.gamma = f8[8];
        p.excluded_layers.assign(excluded, excluded + n_excl);
        for (std::size_t i = 0; i < n_points; ++i)
            p.points.push_back({(std::size_t)points[3 * i], points[3 * i + 1], points[3 * i + 2]});
        sinkr::save_profile(path, p);
    });
}

int ref_load_profile(const char* path, double* f8, std::size_t* excluded, std::size_t* n_excl,
                     double* points, std::size_t* n_points) {
    return guard([&] { profile_out(sinkr::load_profile(path), f8, excluded, n_excl, points, n_points); });
}

// ---- SNKT + snapshots (tensor.hpp:86-96, kv_cache.hpp:72-80) -----------------
int ref_write_tensor(const char* path, const std::uint64_t* dims, std::size_t ndim,
                     const float* data) {
    return guard([&] {
        sinkr::Tensor t;
        t.dims.assign(dims, dims + ndim);
        t.data.assign(data, data + sinkr::element_count(t.dims));
        sinkr::write_tensor(path, t);
    });
}

int ref_read_tensor(const char* path, std::uint64_t* dims, std::size_t* ndim, float* data,
                    std::size_t capacity) {
    return guard([&] {
        const auto t = sinkr::read_tensor(path);
        *ndim = t.dims.size();
        for (std::size_t i = 0; i < t.dims.size(); ++i) dims[i] = t.dims[i];
        if (data) {
            if (t.data.size() > capacity) throw std::invalid_argument("buffer too small");
            std::memcpy(data, t.data.data(), t.data.size() * sizeof(float));
        }
    });
}

std::uint64_t ref_snkt_file_size(const std::uint64_t* dims, std::size_t ndim) {
    return sinkr::snkt_file_size(std::span<const std::uint64_t>(dims, ndim));
}

int ref_cache_save_snapshot(void* c, const char* dir) {
    return guard([&] { static_cast<sinkr::KvCache*>(c)->save_snapshot(dir); });
}

int ref_cache_load_snapshot(const char* dir, void** out) {
    return guard([&] { *out = new sinkr::KvCache(sinkr::KvCache::load_snapshot(dir)); });
}

int ref_cache_historical(void* c, std::size_t layer, std::size_t head, std::size_t from,
                         std::size_t to, float* k, float* v) {
    return guard([&] {
        auto* cache = static_cast<sinkr::KvCache*>(c);
        sinkr::LoadCounters ctr;
        const auto h = cache->historical(layer, head, from, to, ctr);
        std::memcpy(k, h.k.data(), h.k.size() * sizeof(float));
        std::memcpy(v, h.v.data(), h.v.size() * sizeof(float));
    });
}

}  // extern "C"
