// sinkr/cuda/router.hpp — header-only C++20 shim over the C-ABI
// (include/sinkr_cuda.h) with the reference's own operator API:
//
//   reference (/root/reference/proj/include/sinkr/...)   here (namespace sinkr::cuda)
//   CacheConfig, KvCache            kv_cache.hpp:13-80    CacheConfig, KvCache (HBM, bf16)
//   GroupAnchor                     kv_cache.hpp:27-30    GroupAnchor
//   ThresholdProfile::constant      calibration.hpp:21-34 ThresholdProfile::constant
//   RoutingConfig                   router.hpp:16-26      RoutingConfig
//   RouteDecision, GroupStepInfo,   router.hpp:28-67      same names, same fields
//   LayerStepResult
//   LoadCounters                    counters.hpp:9-28     LoadCounters
//   EngineOptions                   router.hpp:69-76      EngineOptions (no ThreadPool*;
//                                                         + global_context_len)
//   threshold_for_length, route,    router.hpp:47-54,78   same
//   auto_num_splits
//   split_ranges                    attention.hpp:82-85   same
//   QueryGroup, SplitPartial        attention.hpp:14-33   same names, same fields
//   attend_chunk, merge_partials,   attention.hpp:38-85   same signatures over host spans
//   splitk_attention, dense_/       (span overloads)      (GPU span kernels, fp64 state);
//   online_attention                                      + overloads over a cached group
//   ThreadPool                      parallel.hpp:20-44    accepted and unused (the GPU splits)
//   routed_decode_step              router.hpp:84-86      same signature
//   KvCache::save/load_snapshot     kv_cache.hpp:72-80    same (SNKT + manifest.json)
//   calibration / analysis APIs     calibration.hpp, analysis.hpp -> sinkr/cuda/calibration.hpp,
//                                                         sinkr/cuda/analysis.hpp
//
// Status codes are rethrown as the reference's exception classes
// (std::invalid_argument / out_of_range / runtime_error / logic_error), so a
// caller of the reference sees identical error behaviour.  A caller switches
// by replacing `sinkr::` with `sinkr::cuda::` and linking libsinkr_cuda.so.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstddef>
#include <filesystem>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../sinkr_cuda.h"

namespace sinkr::cuda {

inline void check(sinkr_status s) {
    if (s == SINKR_OK) return;
    const std::string msg = sinkr_last_error();
    switch (s) {
        case SINKR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SINKR_OUT_OF_RANGE: throw std::out_of_range(msg);
        case SINKR_LOGIC_ERROR: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

constexpr std::size_t kDefaultBlockSize = 128;

struct CacheConfig {
    std::size_t num_layers = 0;
    std::size_t num_q_heads = 0;
    std::size_t num_kv_heads = 0;
    std::size_t head_dim = 0;
    std::size_t capacity = 0;
    std::size_t num_seqs = 1;  // B independent caches served by one launch
    std::size_t group_width() const { return num_q_heads / num_kv_heads; }
};

struct GroupAnchor {
    std::vector<float> k0;
    float k0_norm = 0.0f;
};

struct CalibrationPoint {  // calibration.hpp:14-18
    std::size_t length = 0;
    double tau = 0.0;
    double skip = 0.0;
};

struct ThresholdProfile {
    std::array<double, 4> coeffs{0.0, 0.0, 0.0, 0.0};
    double length_normalizer = 1.0;
    double clamp_lo = 0.0;
    double clamp_hi = 1.0;
    double target_skip = 0.60;
    double gamma = 0.65;
    std::vector<std::size_t> excluded_layers{0, 1};
    std::vector<CalibrationPoint> points;

    static ThresholdProfile constant(double tau) {  // calibration.cpp:29-35
        ThresholdProfile p;
        p.coeffs = {0.0, 0.0, 0.0, tau};
        p.clamp_lo = tau < 0.0 ? tau : 0.0;
        p.clamp_hi = 1.0 < tau ? tau : 1.0;
        return p;
    }
    sinkr_threshold_profile c() const {
        sinkr_threshold_profile p{};
        for (int i = 0; i < 4; ++i) p.coeffs[i] = coeffs[i];
        p.length_normalizer = length_normalizer;
        p.clamp_lo = clamp_lo;
        p.clamp_hi = clamp_hi;
        return p;
    }
};

struct RoutingConfig {
    double gamma = 0.65;
    ThresholdProfile profile;
    std::vector<std::size_t> excluded_layers{0, 1};
    bool sink_on_tie = false;

    static RoutingConfig from_profile(ThresholdProfile profile) {  // router.cpp:23-29
        RoutingConfig c;
        c.gamma = profile.gamma;
        c.excluded_layers = profile.excluded_layers;
        c.profile = std::move(profile);
        return c;
    }
    bool layer_excluded(std::size_t layer) const {
        for (auto l : excluded_layers)
            if (l == layer) return true;
        return false;
    }
    sinkr_routing_config c() const {
        sinkr_routing_config r{};
        r.gamma = gamma;
        r.profile = profile.c();
        r.excluded_layers = excluded_layers.data();
        r.num_excluded_layers = excluded_layers.size();
        r.sink_on_tie = sink_on_tie ? 1 : 0;
        return r;
    }
};

struct RouteDecision {
    double group_score = 0.0;
    double threshold = 0.0;
    bool sink = false;
    bool degenerate = false;
    std::vector<double> head_scores;
};

struct LoadCounters {
    std::uint64_t kv_floats_loaded = 0;
    std::uint64_t anchor_floats_loaded = 0;
    std::uint64_t groups_active = 0;
    std::uint64_t groups_skipped = 0;
    double routing_seconds = 0.0;
    double attention_seconds = 0.0;
    double merge_seconds = 0.0;
};

struct GroupStepInfo {
    std::size_t layer = 0;
    std::size_t kv_head = 0;
    RouteDecision decision;
    std::uint64_t kv_floats_loaded = 0;
    std::uint64_t tokens_loaded = 0;  // rows the decode kernel streamed
};

struct LayerStepResult {
    std::vector<float> outputs;  // B x H_q x D, query-head order
    std::vector<GroupStepInfo> groups;
    LoadCounters counters;
};

struct EngineOptions {
    std::size_t num_splits = 0;
    std::size_t block_size = kDefaultBlockSize;
    bool observe_only = false;
    std::size_t global_context_len = 0;
    sinkr_engine_options c() const {
        return sinkr_engine_options{num_splits, block_size, observe_only ? 1 : 0,
                                    global_context_len};
    }
};

class KvCache {
public:
    explicit KvCache(CacheConfig config, int device = 0) : config_(config) {
        const sinkr_cache_config c{config.num_layers, config.num_q_heads, config.num_kv_heads,
                                   config.head_dim,   config.capacity,    config.num_seqs};
        check(sinkr_engine_create(&c, device, &e_));
    }
    ~KvCache() { sinkr_engine_destroy(e_); }
    KvCache(const KvCache&) = delete;
    KvCache& operator=(const KvCache&) = delete;
    KvCache(KvCache&& o) noexcept : config_(o.config_), e_(o.e_) { o.e_ = nullptr; }

    // kv_cache.hpp:72-80 — SNKT files + manifest.json, one sequence per snapshot
    void save_snapshot(const std::filesystem::path& dir, std::size_t seq = 0) const {
        check(sinkr_save_snapshot(e_, seq, dir.string().c_str()));
    }
    static KvCache load_snapshot(const std::filesystem::path& dir, int device = 0) {
        sinkr_engine* e = nullptr;
        check(sinkr_load_snapshot(dir.string().c_str(), device, &e));
        return KvCache(e);
    }

    const CacheConfig& config() const { return config_; }
    sinkr_engine* handle() const { return e_; }

    void append(std::size_t layer, std::size_t kv_head, std::span<const float> k,
                std::span<const float> v, std::size_t seq = 0) {
        const std::size_t d = config_.head_dim;
        if (k.size() != v.size() || k.empty() || k.size() % d != 0)
            throw std::invalid_argument("k/v row size does not match head_dim");
        check(sinkr_kv_append(e_, seq, layer, kv_head, k.data(), v.data(), k.size() / d));
    }
    std::size_t length(std::size_t layer, std::size_t kv_head, std::size_t seq = 0) const {
        std::size_t n = 0;
        check(sinkr_kv_length(e_, seq, layer, kv_head, &n));
        return n;
    }
    std::size_t token_count(std::size_t seq = 0) const {
        std::size_t n = 0;
        check(sinkr_kv_token_count(e_, seq, &n));
        return n;
    }
    GroupAnchor anchor(std::size_t layer, std::size_t kv_head, std::size_t seq = 0) const {
        GroupAnchor a;
        a.k0.resize(config_.head_dim);
        check(sinkr_kv_anchor(e_, seq, layer, kv_head, a.k0.data(), &a.k0_norm));
        return a;
    }
    // KvCache::historical as a copy (exact f32 upcast of the stored bf16 rows)
    std::pair<std::vector<float>, std::vector<float>> historical(std::size_t layer,
                                                                 std::size_t kv_head,
                                                                 std::size_t from, std::size_t to,
                                                                 std::size_t seq = 0) const {
        std::vector<float> k((to > from ? to - from : 0) * config_.head_dim), v(k.size());
        check(sinkr_kv_read(e_, seq, layer, kv_head, from, to, k.data(), v.data()));
        return {std::move(k), std::move(v)};
    }

private:
    explicit KvCache(sinkr_engine* e) : e_(e) {
        sinkr_cache_config c{};
        check(sinkr_engine_config(e, &c));
        config_ = CacheConfig{c.num_layers, c.num_q_heads, c.num_kv_heads,
                              c.head_dim,   c.capacity,    c.num_seqs};
    }
    CacheConfig config_;
    sinkr_engine* e_ = nullptr;
};

inline double threshold_for_length(std::size_t context_len, const ThresholdProfile& profile) {
    const auto p = profile.c();
    double out = 0.0;
    check(sinkr_threshold_for_length(context_len, &p, &out));
    return out;
}

inline RouteDecision route(std::size_t layer, double score, std::size_t context_len,
                           const RoutingConfig& config) {
    const auto c = config.c();
    int sink = 0;
    RouteDecision d;
    d.group_score = score;
    check(sinkr_route(layer, score, context_len, &c, &sink, &d.threshold));
    d.sink = sink != 0;
    return d;
}

inline std::size_t auto_num_splits(std::size_t context_len) {
    return sinkr_auto_num_splits(context_len);
}

inline std::vector<std::pair<std::size_t, std::size_t>> split_ranges(std::size_t len,
                                                                     std::size_t num_splits) {
    std::vector<std::size_t> buf(2 * (num_splits ? num_splits : 1));
    check(sinkr_split_ranges(len, num_splits, buf.data()));
    std::vector<std::pair<std::size_t, std::size_t>> out;
    for (std::size_t i = 0; i < num_splits; ++i) out.emplace_back(buf[2 * i], buf[2 * i + 1]);
    return out;
}

// SplitkResult / splitk_attention (attention.hpp:71-85) of one cached group on
// the GPU: the group's r query heads over all of its rows.  num_splits is
// validated like split_ranges; the kernel picks its own split.
struct SplitkResult {
    std::vector<float> out;  // heads x dim
    LoadCounters counters;
};

inline SplitkResult splitk_attention(const KvCache& cache, std::span<const float> group_q,
                                     std::size_t layer, std::size_t kv_head,
                                     std::size_t num_splits, std::size_t seq = 0) {
    const CacheConfig& cc = cache.config();
    if (group_q.size() != cc.group_width() * cc.head_dim)
        throw std::invalid_argument("query span size does not match heads x dim");
    SplitkResult res;
    res.out.resize(group_q.size());
    sinkr_load_counters ctr{};
    check(sinkr_group_attention(cache.handle(), group_q.data(), seq, layer, kv_head, num_splits,
                                res.out.data(), &ctr));
    res.counters.kv_floats_loaded = ctr.kv_floats_loaded;
    return res;
}

// dense_attention / online_attention (attention.cpp:42-73,144-157) of one
// cached group: the same GPU group attention (block_size checked like
// attend_chunk, attention.cpp:107).
inline std::vector<float> dense_attention(const KvCache& cache, std::span<const float> group_q,
                                          std::size_t layer, std::size_t kv_head,
                                          std::size_t seq = 0) {
    return splitk_attention(cache, group_q, layer, kv_head, 1, seq).out;
}

inline std::vector<float> online_attention(const KvCache& cache, std::span<const float> group_q,
                                           std::size_t layer, std::size_t kv_head,
                                           std::size_t block_size = kDefaultBlockSize,
                                           std::size_t seq = 0) {
    if (block_size == 0) throw std::invalid_argument("block_size must be positive");
    return splitk_attention(cache, group_q, layer, kv_head, 1, seq).out;
}

// ---- span-level operators (attention.hpp:14-85) ------------------------------
// QueryGroup / SplitPartial with the reference's fields; the operators run on
// the GPU of the calling thread (include/sinkr_cuda.h, span section).

struct QueryGroup {  // attention.hpp:14-21
    std::span<const float> q;
    std::size_t heads = 0;
    std::size_t dim = 0;
    float scale = 0.0f;

    static QueryGroup over(std::span<const float> q, std::size_t heads, std::size_t dim) {
        QueryGroup qg{q, heads, dim, 0.0f};  // attention.cpp:33-40
        if (dim == 0) throw std::invalid_argument("head_dim must be positive");
        qg.scale = 1.0f / std::sqrt(static_cast<float>(dim));
        if (q.size() != heads * dim)
            throw std::invalid_argument("query span size does not match heads x dim");
        return qg;
    }
};

struct SplitPartial {  // attention.hpp:26-33
    std::vector<double> m;    // heads
    std::vector<double> l;    // heads
    std::vector<double> acc;  // heads x dim
    std::size_t tokens = 0;

    bool empty() const { return tokens == 0; }
};

// The reference's CPU pool (parallel.hpp).  Accepted where the reference takes
// a ThreadPool*, so callers compile unchanged; the split itself runs on the GPU.
class ThreadPool {
public:
    explicit ThreadPool(std::size_t threads = 0) : n_(threads ? threads : 1) {}
    std::size_t size() const { return n_; }

private:
    std::size_t n_;
};

namespace detail {
// attention.cpp:13-23 (span sizes are only known on this side of the C-ABI)
inline void check_shapes(const QueryGroup& qg, std::span<const float> keys,
                         std::span<const float> values, std::size_t len, bool with_values) {
    if (qg.heads == 0 || qg.dim == 0) throw std::invalid_argument("empty query group");
    if (qg.q.size() != qg.heads * qg.dim)
        throw std::invalid_argument("query span size does not match heads x dim");
    if (len == 0) throw std::invalid_argument("attention needs at least one token");
    if (keys.size() != len * qg.dim)
        throw std::invalid_argument("key span size does not match len x dim");
    if (with_values && values.size() != len * qg.dim)
        throw std::invalid_argument("value span size does not match len x dim");
}
}  // namespace detail

// attend_chunk (attention.hpp:55-60): the chunk's fp64 online-softmax state.
inline SplitPartial attend_chunk(const QueryGroup& qg, std::span<const float> keys,
                                 std::span<const float> values, std::size_t len,
                                 std::size_t block_size = kDefaultBlockSize) {
    detail::check_shapes(qg, keys, values, len, true);
    SplitPartial p;
    p.m.resize(qg.heads);
    p.l.resize(qg.heads);
    p.acc.resize(qg.heads * qg.dim);
    std::uint64_t tok = 0;
    check(sinkr_attend_chunk(qg.q.data(), qg.heads, qg.dim, keys.data(), values.data(), len,
                             block_size, p.m.data(), p.l.data(), p.acc.data(), &tok));
    p.tokens = tok;
    return p;
}

// attend_chunk over the cached rows [from, to) of one group (historical +
// attend_chunk, router.cpp:149-160), read in place from HBM.
inline SplitPartial attend_chunk(const KvCache& cache, std::span<const float> group_q,
                                 std::size_t layer, std::size_t kv_head, std::size_t from,
                                 std::size_t to, std::size_t seq = 0,
                                 std::size_t block_size = kDefaultBlockSize) {
    const CacheConfig& cc = cache.config();
    const std::size_t r = cc.group_width(), d = cc.head_dim;
    if (group_q.size() != r * d) throw std::invalid_argument("query span size does not match heads x dim");
    SplitPartial p;
    p.m.resize(r);
    p.l.resize(r);
    p.acc.resize(r * d);
    std::uint64_t tok = 0;
    check(sinkr_attend_chunk_cached(cache.handle(), group_q.data(), seq, layer, kv_head, from, to,
                                    block_size, p.m.data(), p.l.data(), p.acc.data(), &tok));
    p.tokens = tok;
    return p;
}

// merge_partials (attention.hpp:62-64): LSE combine on the GPU.
inline std::vector<float> merge_partials(std::span<const SplitPartial> parts, std::size_t heads,
                                         std::size_t dim) {
    std::vector<double> m(parts.size() * heads), l(m.size()), acc(m.size() * dim);
    std::vector<std::uint64_t> tok(parts.size());
    for (std::size_t i = 0; i < parts.size(); ++i) {
        const SplitPartial& p = parts[i];
        tok[i] = p.tokens;
        if (p.empty()) continue;
        if (p.m.size() != heads || p.l.size() != heads || p.acc.size() != heads * dim)
            throw std::invalid_argument("partial shape does not match heads x dim");
        std::copy(p.m.begin(), p.m.end(), m.begin() + i * heads);
        std::copy(p.l.begin(), p.l.end(), l.begin() + i * heads);
        std::copy(p.acc.begin(), p.acc.end(), acc.begin() + i * heads * dim);
    }
    std::vector<float> out(heads * dim);
    check(sinkr_merge_partials(parts.size(), m.data(), l.data(), acc.data(), tok.data(), heads,
                               dim, out.data()));
    return out;
}

// splitk_attention (attention.hpp:76-85) over host spans.
inline SplitkResult splitk_attention(const QueryGroup& qg, std::span<const float> keys,
                                     std::span<const float> values, std::size_t len,
                                     std::size_t num_splits, ThreadPool* pool = nullptr,
                                     std::size_t block_size = kDefaultBlockSize) {
    (void)pool;
    detail::check_shapes(qg, keys, values, len, true);
    SplitkResult res;
    res.out.resize(qg.heads * qg.dim);
    sinkr_load_counters ctr{};
    check(sinkr_splitk_attention(qg.q.data(), qg.heads, qg.dim, keys.data(), values.data(), len,
                                 num_splits, block_size, res.out.data(), &ctr));
    res.counters.kv_floats_loaded = ctr.kv_floats_loaded;
    return res;
}

// dense_attention / online_attention (attention.hpp:38-53) over host spans.
inline std::vector<float> dense_attention(const QueryGroup& qg, std::span<const float> keys,
                                          std::span<const float> values, std::size_t len) {
    detail::check_shapes(qg, keys, values, len, true);
    std::vector<float> out(qg.heads * qg.dim);
    check(sinkr_dense_attention(qg.q.data(), qg.heads, qg.dim, keys.data(), values.data(), len,
                                out.data()));
    return out;
}

inline std::vector<float> online_attention(const QueryGroup& qg, std::span<const float> keys,
                                           std::span<const float> values, std::size_t len,
                                           std::size_t block_size = kDefaultBlockSize) {
    detail::check_shapes(qg, keys, values, len, true);
    std::vector<float> out(qg.heads * qg.dim);
    check(sinkr_online_attention(qg.q.data(), qg.heads, qg.dim, keys.data(), values.data(), len,
                                 block_size, out.data()));
    return out;
}

// router.hpp:84-86 — one decode step for one layer (all B sequences).
inline LayerStepResult routed_decode_step(std::span<const float> queries, std::size_t layer,
                                          const KvCache& cache, const RoutingConfig& config,
                                          const EngineOptions& options = {}) {
    const CacheConfig& cc = cache.config();
    const std::size_t B = cc.num_seqs ? cc.num_seqs : 1;
    if (queries.size() != B * cc.num_q_heads * cc.head_dim)
        throw std::invalid_argument("queries span must be H_q x D for one layer");
    const auto rc = config.c();
    const auto oc = options.c();
    LayerStepResult r;
    r.outputs.resize(queries.size());
    std::vector<sinkr_group_info> gi(B * cc.num_kv_heads);
    std::vector<double> hs(B * cc.num_q_heads);
    sinkr_load_counters ctr{};
    check(sinkr_routed_decode_batch(cache.handle(), queries.data(), layer, &rc, &oc,
                                    r.outputs.data(), gi.data(), hs.data(), &ctr));
    const std::size_t w = cc.group_width();
    r.groups.resize(gi.size());
    for (std::size_t u = 0; u < gi.size(); ++u) {
        auto& g = r.groups[u];
        g.layer = gi[u].layer;
        g.kv_head = gi[u].kv_head;
        g.decision.group_score = gi[u].group_score;
        g.decision.threshold = gi[u].threshold;
        g.decision.sink = gi[u].sink != 0;
        g.decision.degenerate = gi[u].degenerate != 0;
        g.decision.head_scores.assign(hs.begin() + u * w, hs.begin() + (u + 1) * w);
        g.kv_floats_loaded = gi[u].kv_floats_loaded;
        g.tokens_loaded = gi[u].tokens_loaded;
    }
    r.counters = LoadCounters{ctr.kv_floats_loaded, ctr.anchor_floats_loaded,
                              ctr.groups_active,    ctr.groups_skipped,
                              ctr.routing_seconds,  ctr.attention_seconds,
                              ctr.merge_seconds};
    return r;
}

}  // namespace sinkr::cuda
