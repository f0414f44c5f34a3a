// span.cu — C-ABI of the reference's span-level attention operators
// (attention.hpp:38-85) on the GPU: attend_chunk, merge_partials,
// splitk_attention, dense_attention, online_attention over host spans, and
// attend_chunk over a cached bf16 range of an engine (engine.cu calls
// sinkr::span::attend_device).  Kernels: span.cuh.
//
// Free functions like the reference's: each call runs on the calling
// thread's current CUDA device, on a per-device context (stream + scratch
// grown on demand) serialised by a mutex, and blocks until its results are
// in host memory.  Validation follows attention.cpp's check_shapes (13-23),
// attend_chunk (107), merge_partials (159-170) and split_ranges (185-190),
// with the reference's messages.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sinkr_cuda.h"
#include "host_util.hpp"
#include "span.cuh"
#include "span.hpp"

namespace {

using sinkr::host::fail;
using sinkr::host::guard;
namespace sp = sinkr::span;

#define SPAN_CK(x)                                                                     \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            fail(SINKR_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_));    \
    } while (0)

constexpr size_t kMaxSpanDim = 8192;

struct SpanCtx {
    std::mutex mu;
    int device = 0;
    cudaStream_t stream = nullptr;
    uint8_t* d_buf = nullptr;
    size_t d_bytes = 0;
    uint8_t* grow(size_t need) {
        if (need > d_bytes) {
            SPAN_CK(cudaStreamSynchronize(stream));
            cudaFree(d_buf);
            d_buf = nullptr;
            d_bytes = 0;
            SPAN_CK(cudaMalloc(&d_buf, need));
            d_bytes = need;
        }
        return d_buf;
    }
};

// one context per device, created on first use and kept for the process
SpanCtx& ctx_for_current_device() {
    static std::mutex reg_mu;
    static std::map<int, std::unique_ptr<SpanCtx>> reg;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        fail(SINKR_NO_DEVICE, "no CUDA device visible (the span operators have no CPU fallback)");
    }
    int dev = 0;
    SPAN_CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(reg_mu);
    auto it = reg.find(dev);
    if (it != reg.end()) return *it->second;
    cudaDeviceProp prop;
    SPAN_CK(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10) fail(SINKR_NO_DEVICE, std::string("sm_100 device required, found ") + prop.name);
    auto c = std::make_unique<SpanCtx>();
    c->device = dev;
    SPAN_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    for (const void* fn : {(const void*)sp::span_attend_kernel<float>,
                           (const void*)sp::span_attend_kernel<__nv_bfloat16>})
        SPAN_CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    return *reg.emplace(dev, std::move(c)).first->second;
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

// attention.cpp:13-23
void check_shapes(const float* q, size_t heads, size_t dim, const float* keys, const float* values,
                  size_t len, bool with_values) {
    if (heads == 0 || dim == 0) fail(SINKR_INVALID_ARGUMENT, "empty query group");
    if (!q) fail(SINKR_INVALID_ARGUMENT, "query span size does not match heads x dim");
    if (len == 0) fail(SINKR_INVALID_ARGUMENT, "attention needs at least one token");
    if (!keys) fail(SINKR_INVALID_ARGUMENT, "key span size does not match len x dim");
    if (with_values && !values) fail(SINKR_INVALID_ARGUMENT, "value span size does not match len x dim");
    if (dim > kMaxSpanDim)
        fail(SINKR_INVALID_ARGUMENT, "head_dim above 8192 is not supported by the GPU span operators");
}

float logit_scale(size_t dim) { return 1.0f / std::sqrt(static_cast<float>(dim)); }  // attention.cpp:36

// CTA partials per chunk: enough CTAs to cover the SMs, >= one tile each
uint32_t parts_for(size_t len, size_t nhb, int T, int sms) {
    const size_t want = std::max<size_t>(1, (size_t)(2 * sms) / std::max<size_t>(1, nhb));
    const size_t tiles = (len + T - 1) / T;
    return (uint32_t)std::min(want, tiles);
}

}  // namespace

namespace sinkr {
namespace span {

// Online softmax of q [heads][dim] over the device span K, V [len][dim] into
// one fp64 partial per CTA range, then their LSE combine into the chunk's
// partial (d_m [heads], d_l [heads], d_acc [heads][dim]) -- attend_chunk.
template <class E>
static void attend_device_impl(cudaStream_t st, const float* d_q, size_t heads, size_t dim,
                               const E* d_k, const E* d_v, size_t len, uint8_t* scratch,
                               double* d_m, double* d_l, double* d_acc, int sms) {
    const TileGeom g = tile_geom(heads, dim);
    const size_t nhb = (heads + g.HB - 1) / g.HB;
    const uint32_t np = parts_for(len, nhb, g.T, sms);
    double* pm = reinterpret_cast<double*>(scratch);
    double* pl = pm + (size_t)np * heads;
    double* pa = pl + (size_t)np * heads;
    const size_t smem = tile_smem(dim, g);
    span_attend_kernel<E><<<dim3(np, (unsigned)nhb), kSpanThreads, smem, st>>>(
        d_q, (uint32_t)heads, (uint32_t)dim, logit_scale(dim), d_k, d_v, len, np, g.T, g.HB, pm, pl, pa);
    SPAN_CK(cudaGetLastError());
    const unsigned blocks = (unsigned)((heads * dim + kSpanThreads - 1) / kSpanThreads);
    span_merge_kernel<<<blocks, kSpanThreads, 0, st>>>(pm, pl, pa, nullptr, np, (uint32_t)heads,
                                                       (uint32_t)dim, nullptr, d_m, d_l, d_acc);
    SPAN_CK(cudaGetLastError());
}

size_t attend_scratch_bytes(size_t heads, size_t dim, size_t len, int sms) {
    const TileGeom g = tile_geom(heads, dim);
    const size_t nhb = (heads + g.HB - 1) / g.HB;
    const uint32_t np = parts_for(len, nhb, g.T, sms);
    return align256((size_t)np * heads * (dim + 2) * 8);
}

void attend_device(cudaStream_t st, const float* d_q, size_t heads, size_t dim,
                   const __nv_bfloat16* d_k, const __nv_bfloat16* d_v, size_t len,
                   uint8_t* scratch, double* d_m, double* d_l, double* d_acc, int sms) {
    static bool attr = [] {
        cudaFuncSetAttribute(span_attend_kernel<__nv_bfloat16>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        return true;
    }();
    (void)attr;
    attend_device_impl(st, d_q, heads, dim, d_k, d_v, len, scratch, d_m, d_l, d_acc, sms);
}

}  // namespace span
}  // namespace sinkr

namespace {

int sm_count(int dev) {
    int n = 0;
    SPAN_CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
}

// Uploads q and the K/V span, runs attend_chunk over each of the `ranges`
// (one fp64 partial each, left in device memory at *d_parts), returns the
// device pointers.  Layout: q | K | V | partials m[n][h] l[n][h] acc[n][h][d] | tokens[n] | out | scratch
struct Staged {
    double *m, *l, *acc;
    uint64_t* tok;
    float* out;
};

Staged stage_and_attend(SpanCtx& c, const float* q, size_t heads, size_t dim, const float* keys,
                        const float* values, size_t len,
                        const std::vector<std::pair<size_t, size_t>>& ranges) {
    const int sms = sm_count(c.device);
    const size_t n = ranges.size();
    const size_t qb = align256(heads * dim * 4), kvb = align256(len * dim * 4);
    const size_t pb = align256(n * heads * (dim + 2) * 8), tb = align256(n * 8),
                 ob = align256(heads * dim * 4);
    size_t sb = 0;
    for (auto [a, b] : ranges) sb = std::max(sb, sp::attend_scratch_bytes(heads, dim, b - a, sms));
    uint8_t* base = c.grow(qb + 2 * kvb + pb + tb + ob + sb);
    float* d_q = reinterpret_cast<float*>(base);
    float* d_k = reinterpret_cast<float*>(base + qb);
    float* d_v = reinterpret_cast<float*>(base + qb + kvb);
    Staged s;
    s.m = reinterpret_cast<double*>(base + qb + 2 * kvb);
    s.l = s.m + n * heads;
    s.acc = s.l + n * heads;
    s.tok = reinterpret_cast<uint64_t*>(base + qb + 2 * kvb + pb);
    s.out = reinterpret_cast<float*>(base + qb + 2 * kvb + pb + tb);
    uint8_t* scratch = base + qb + 2 * kvb + pb + tb + ob;
    SPAN_CK(cudaMemcpyAsync(d_q, q, heads * dim * 4, cudaMemcpyHostToDevice, c.stream));
    SPAN_CK(cudaMemcpyAsync(d_k, keys, len * dim * 4, cudaMemcpyHostToDevice, c.stream));
    if (values) SPAN_CK(cudaMemcpyAsync(d_v, values, len * dim * 4, cudaMemcpyHostToDevice, c.stream));
    std::vector<uint64_t> tok(n);
    for (size_t i = 0; i < n; ++i) {
        const auto [a, b] = ranges[i];
        tok[i] = b - a;
        // chunks run one after another on the stream and share the scratch
        sp::attend_device_impl<float>(c.stream, d_q, heads, dim, d_k + a * dim, d_v + a * dim, b - a,
                                      scratch, s.m + i * heads, s.l + i * heads,
                                      s.acc + i * heads * dim, sms);
    }
    SPAN_CK(cudaMemcpyAsync(s.tok, tok.data(), n * 8, cudaMemcpyHostToDevice, c.stream));
    SPAN_CK(cudaStreamSynchronize(c.stream));  // `tok` is a host temporary
    return s;
}

void merge_to_host(SpanCtx& c, const Staged& s, size_t n, size_t heads, size_t dim, float* out) {
    const unsigned blocks = (unsigned)((heads * dim + sp::kSpanThreads - 1) / sp::kSpanThreads);
    sp::span_merge_kernel<<<blocks, sp::kSpanThreads, 0, c.stream>>>(
        s.m, s.l, s.acc, s.tok, (uint32_t)n, (uint32_t)heads, (uint32_t)dim, s.out, nullptr, nullptr,
        nullptr);
    SPAN_CK(cudaGetLastError());
    SPAN_CK(cudaMemcpyAsync(out, s.out, heads * dim * 4, cudaMemcpyDeviceToHost, c.stream));
    SPAN_CK(cudaStreamSynchronize(c.stream));
}

std::vector<std::pair<size_t, size_t>> split_ranges(size_t len, size_t num_splits) {
    if (num_splits == 0 || num_splits > len)  // attention.cpp:187-190
        fail(SINKR_INVALID_ARGUMENT, "num_splits must be in [1, len], got " + std::to_string(num_splits) +
                                         " for len " + std::to_string(len));
    std::vector<std::pair<size_t, size_t>> r;
    const size_t base = len / num_splits, rem = len % num_splits;
    size_t start = 0;
    for (size_t c = 0; c < num_splits; ++c) {
        const size_t sz = base + (c < rem ? 1 : 0);
        r.emplace_back(start, start + sz);
        start += sz;
    }
    return r;
}

}  // namespace

extern "C" {

sinkr_status sinkr_attend_chunk(const float* q, size_t heads, size_t dim, const float* keys,
                                const float* values, size_t len, size_t block_size, double* m,
                                double* l, double* acc, uint64_t* tokens) {
    return guard([&] {
        check_shapes(q, heads, dim, keys, values, len, true);
        if (block_size == 0) fail(SINKR_INVALID_ARGUMENT, "block_size must be positive");
        if (!m || !l || !acc) fail(SINKR_INVALID_ARGUMENT, "null argument");
        SpanCtx& c = ctx_for_current_device();
        std::lock_guard<std::mutex> lk(c.mu);
        const Staged s = stage_and_attend(c, q, heads, dim, keys, values, len, {{0, len}});
        SPAN_CK(cudaMemcpyAsync(m, s.m, heads * 8, cudaMemcpyDeviceToHost, c.stream));
        SPAN_CK(cudaMemcpyAsync(l, s.l, heads * 8, cudaMemcpyDeviceToHost, c.stream));
        SPAN_CK(cudaMemcpyAsync(acc, s.acc, heads * dim * 8, cudaMemcpyDeviceToHost, c.stream));
        SPAN_CK(cudaStreamSynchronize(c.stream));
        if (tokens) *tokens = len;
    });
}

sinkr_status sinkr_merge_partials(size_t n, const double* m, const double* l, const double* acc,
                                  const uint64_t* tokens, size_t heads, size_t dim, float* out) {
    return guard([&] {
        if (!out || (n && (!m || !l || !acc || !tokens))) fail(SINKR_INVALID_ARGUMENT, "null argument");
        size_t live = 0;
        for (size_t i = 0; i < n; ++i) live += tokens[i] != 0;
        if (live == 0) fail(SINKR_INVALID_ARGUMENT, "merge needs at least one non-empty partial");
        if (heads == 0 || dim == 0)
            fail(SINKR_INVALID_ARGUMENT, "partial shape does not match heads x dim");
        SpanCtx& c = ctx_for_current_device();
        std::lock_guard<std::mutex> lk(c.mu);
        const size_t pb = align256(n * heads * (dim + 2) * 8), tb = align256(n * 8);
        uint8_t* base = c.grow(pb + tb + align256(heads * dim * 4));
        Staged s;
        s.m = reinterpret_cast<double*>(base);
        s.l = s.m + n * heads;
        s.acc = s.l + n * heads;
        s.tok = reinterpret_cast<uint64_t*>(base + pb);
        s.out = reinterpret_cast<float*>(base + pb + tb);
        SPAN_CK(cudaMemcpyAsync(s.m, m, n * heads * 8, cudaMemcpyHostToDevice, c.stream));
        SPAN_CK(cudaMemcpyAsync(s.l, l, n * heads * 8, cudaMemcpyHostToDevice, c.stream));
        SPAN_CK(cudaMemcpyAsync(s.acc, acc, n * heads * dim * 8, cudaMemcpyHostToDevice, c.stream));
        SPAN_CK(cudaMemcpyAsync(s.tok, tokens, n * 8, cudaMemcpyHostToDevice, c.stream));
        merge_to_host(c, s, n, heads, dim, out);
    });
}

sinkr_status sinkr_merge_partials_async(size_t n, const double* d_m, const double* d_l,
                                        const double* d_acc, const uint64_t* d_tokens, size_t heads,
                                        size_t dim, float* d_out, void* stream) {
    return guard([&] {
        if (!d_m || !d_l || !d_acc || !d_out || n == 0 || heads == 0 || dim == 0)
            fail(SINKR_INVALID_ARGUMENT, "null argument");
        const unsigned blocks = (unsigned)((heads * dim + sp::kSpanThreads - 1) / sp::kSpanThreads);
        sp::span_merge_kernel<<<blocks, sp::kSpanThreads, 0, static_cast<cudaStream_t>(stream)>>>(
            d_m, d_l, d_acc, d_tokens, (uint32_t)n, (uint32_t)heads, (uint32_t)dim, d_out, nullptr,
            nullptr, nullptr);
        SPAN_CK(cudaGetLastError());
    });
}

sinkr_status sinkr_splitk_attention(const float* q, size_t heads, size_t dim, const float* keys,
                                    const float* values, size_t len, size_t num_splits,
                                    size_t block_size, float* out, sinkr_load_counters* counters) {
    return guard([&] {
        check_shapes(q, heads, dim, keys, values, len, true);
        const auto ranges = split_ranges(len, num_splits);
        if (block_size == 0) fail(SINKR_INVALID_ARGUMENT, "block_size must be positive");
        if (!out) fail(SINKR_INVALID_ARGUMENT, "null argument");
        SpanCtx& c = ctx_for_current_device();
        std::lock_guard<std::mutex> lk(c.mu);
        const Staged s = stage_and_attend(c, q, heads, dim, keys, values, len, ranges);
        merge_to_host(c, s, ranges.size(), heads, dim, out);
        if (counters) {
            *counters = sinkr_load_counters{};
            counters->kv_floats_loaded = 2ull * len * dim;  // attention.cpp:219
        }
    });
}

sinkr_status sinkr_online_attention(const float* q, size_t heads, size_t dim, const float* keys,
                                    const float* values, size_t len, size_t block_size, float* out) {
    return guard([&] {
        check_shapes(q, heads, dim, keys, values, len, true);
        if (block_size == 0) fail(SINKR_INVALID_ARGUMENT, "block_size must be positive");
        if (!out) fail(SINKR_INVALID_ARGUMENT, "null argument");
        SpanCtx& c = ctx_for_current_device();
        std::lock_guard<std::mutex> lk(c.mu);
        const Staged s = stage_and_attend(c, q, heads, dim, keys, values, len, {{0, len}});
        merge_to_host(c, s, 1, heads, dim, out);  // acc / l (attention.cpp:149-156)
    });
}

sinkr_status sinkr_dense_attention(const float* q, size_t heads, size_t dim, const float* keys,
                                   const float* values, size_t len, float* out) {
    return guard([&] {
        check_shapes(q, heads, dim, keys, values, len, true);
        if (!out) fail(SINKR_INVALID_ARGUMENT, "null argument");
        SpanCtx& c = ctx_for_current_device();
        std::lock_guard<std::mutex> lk(c.mu);
        const Staged s = stage_and_attend(c, q, heads, dim, keys, values, len, {{0, len}});
        merge_to_host(c, s, 1, heads, dim, out);
    });
}

}  // extern "C"
