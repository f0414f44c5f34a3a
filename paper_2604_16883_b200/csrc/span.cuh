// span.cuh — the reference's span-level attention operators
// (attention.hpp:38-85) as sm_100a kernels: attend_chunk's online softmax
// over an arbitrary [len][dim] K/V span and merge_partials' LSE combine.
//
// These serve the drop-in boundary for callers of attend_chunk /
// merge_partials / splitk_attention / dense_attention / online_attention
// with host spans (or a cached bf16 range).  They are not the decode hot path
// (step.cuh streams the cache at the HBM roofline); they are built for
// fidelity: every logit is the reference's dot -- f32 x f32 products summed
// sequentially in fp64 in index order (attention.cpp:25-29), scaled by the
// float 1/sqrt(dim) -- so logits and block maxima are bit-identical, and the
// softmax state (m, l, acc) is fp64 like SplitPartial (attention.hpp:26-33).
//
// Work split: CTA (c, hb) runs the online softmax of heads [hb*HB, hb*HB+HB)
// over the token range c of the span in tiles of T tokens (K and V tiles
// staged in shared memory, rows padded to dim+1 floats so the per-token dot
// threads do not collide on banks) and writes one fp64 partial; the partials
// of a span are then LSE-merged by span_merge_kernel, which is also
// merge_partials itself.
#pragma once

#include <cuda_bf16.h>
#include <cstdint>

namespace sinkr {
namespace span {

constexpr int kSpanThreads = 256;

struct TileGeom {
    int T;   // tokens per tile
    int HB;  // heads per CTA
};

// tiles sized so the staged K/V (2 x T x (dim+1) f32) stay around 128 KB or less
inline TileGeom tile_geom(size_t heads, size_t dim) {
    int T = (int)(8192 / (dim + 1));
    T = T < 1 ? 1 : (T > 32 ? 32 : T);
    int HB = (int)(2048 / dim);
    HB = HB < 1 ? 1 : (HB > 8 ? 8 : HB);
    if ((size_t)HB > heads) HB = (int)heads;
    return {T, HB};
}

inline size_t tile_smem(size_t dim, TileGeom g) {
    return 8 * (size_t)g.HB * dim           // acc (fp64)
           + 8 * 3 * (size_t)g.HB           // m, l, rescale
           + 8 * (size_t)g.HB * g.T         // z / p (fp64)
           + 4 * (size_t)g.HB * dim         // q (f32)
           + 4 * 2 * (size_t)g.T * (dim + 1);  // K, V tiles (f32, padded rows)
}

__device__ __forceinline__ float load_elem(const float* p) { return __ldg(p); }
__device__ __forceinline__ float load_elem(const __nv_bfloat16* p) { return __bfloat162float(*p); }

// One CTA: heads [h0, h0 + nh) over tokens [t0, t1) of the span.
//   q [heads][dim] f32; K, V [len][dim] (f32 span or bf16 cache rows)
//   out_m / out_l [part][heads], out_acc [part][heads][dim] (fp64), part = blockIdx.x
template <class E>
__global__ void __launch_bounds__(kSpanThreads)
    span_attend_kernel(const float* __restrict__ q, uint32_t heads, uint32_t dim, float scale,
                       const E* __restrict__ K, const E* __restrict__ V, uint64_t len,
                       uint32_t nparts, int T, int HB, double* __restrict__ out_m,
                       double* __restrict__ out_l, double* __restrict__ out_acc) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t c = blockIdx.x, h0 = blockIdx.y * HB;
    const uint32_t nh = min((uint32_t)HB, heads - h0);
    const uint32_t tid = threadIdx.x;
    const uint64_t t0 = len * c / nparts, t1 = len * (c + 1) / nparts;
    const uint32_t P = dim + 1;  // padded K/V row
    double* acc = reinterpret_cast<double*>(smem);
    double* sm_m = acc + (size_t)HB * dim;
    double* sm_l = sm_m + HB;
    double* sm_r = sm_l + HB;
    double* z = sm_r + HB;  // [HB][T]
    float* qs = reinterpret_cast<float*>(z + (size_t)HB * T);
    float* ks = qs + (size_t)HB * dim;
    float* vs = ks + (size_t)T * P;

    for (uint32_t i = tid; i < nh * dim; i += kSpanThreads) {
        qs[i] = __ldg(q + (size_t)h0 * dim + i);
        acc[i] = 0.0;
    }
    for (uint32_t h = tid; h < nh; h += kSpanThreads) {
        sm_m[h] = -INFINITY;
        sm_l[h] = 0.0;
    }
    const double sc = (double)scale;
    for (uint64_t b0 = t0; b0 < t1; b0 += T) {
        const uint32_t nt = (uint32_t)min((uint64_t)T, t1 - b0);
        __syncthreads();  // previous tile consumed
        for (uint32_t i = tid; i < nt * dim; i += kSpanThreads) {
            const uint32_t r = i / dim, j = i % dim;
            ks[r * P + j] = load_elem(K + (b0 + r) * dim + j);
            vs[r * P + j] = load_elem(V + (b0 + r) * dim + j);
        }
        __syncthreads();
        // z = scale * dot(q_h, k_i): the reference's sequential fp64 sum of
        // exact f32 x f32 products (attention.cpp:25-29, 124)
        for (uint32_t pi = tid; pi < nh * nt; pi += kSpanThreads) {
            const uint32_t h = pi / nt, i = pi % nt;
            const float* qa = qs + h * dim;
            const float* kb = ks + i * P;
            double s = 0.0;
            for (uint32_t j = 0; j < dim; ++j) s = __dadd_rn(s, __dmul_rn((double)qa[j], (double)kb[j]));
            z[h * T + i] = __dmul_rn(sc, s);
        }
        __syncthreads();
        // block max -> new running max, rescale of (l, acc)
        for (uint32_t h = tid; h < nh; h += kSpanThreads) {
            double bm = -INFINITY;
            for (uint32_t i = 0; i < nt; ++i) bm = fmax(bm, z[h * T + i]);
            const double nm = fmax(sm_m[h], bm);
            sm_r[h] = exp(sm_m[h] - nm);  // 0 on the first tile (exp(-inf))
            sm_m[h] = nm;
        }
        __syncthreads();
        for (uint32_t pi = tid; pi < nh * nt; pi += kSpanThreads) {
            const uint32_t h = pi / nt, i = pi % nt;
            z[h * T + i] = exp(z[h * T + i] - sm_m[h]);
        }
        __syncthreads();
        for (uint32_t h = tid; h < nh; h += kSpanThreads) {
            double l = __dmul_rn(sm_l[h], sm_r[h]);
            for (uint32_t i = 0; i < nt; ++i) l = __dadd_rn(l, z[h * T + i]);
            sm_l[h] = l;
        }
        for (uint32_t e = tid; e < nh * dim; e += kSpanThreads) {
            const uint32_t h = e / dim, j = e % dim;
            // acc *= rescale; acc += p * v in token order, no contraction
            // (attention.cpp:128-139)
            double a = __dmul_rn(acc[e], sm_r[h]);
            for (uint32_t i = 0; i < nt; ++i) a = __dadd_rn(a, __dmul_rn(z[h * T + i], (double)vs[i * P + j]));
            acc[e] = a;
        }
    }
    __syncthreads();
    for (uint32_t h = tid; h < nh; h += kSpanThreads) {
        out_m[(size_t)c * heads + h0 + h] = sm_m[h];
        out_l[(size_t)c * heads + h0 + h] = sm_l[h];
    }
    for (uint32_t e = tid; e < nh * dim; e += kSpanThreads)
        out_acc[((size_t)c * heads + h0) * dim + e] = acc[e];
}

// merge_partials (attention.cpp:159-183) over n fp64 partials laid out
// m/l [n][heads], acc [n][heads][dim], tokens [n] (NULL: all live): one
// thread per (head, dim) output, the partials visited in order, empty ones
// (tokens == 0) skipped, m* = max, l* = sum l e^(m - m*), out = sum acc
// e^(m - m*) / l*.  Writes the f32 output (out_f32) or the combined fp64
// partial (out_m / out_l / out_acc: a chunk's state from its CTA partials).
__global__ void __launch_bounds__(kSpanThreads)
    span_merge_kernel(const double* __restrict__ m, const double* __restrict__ l,
                      const double* __restrict__ acc, const uint64_t* __restrict__ tokens,
                      uint32_t n, uint32_t heads, uint32_t dim, float* __restrict__ out_f32,
                      double* __restrict__ out_m, double* __restrict__ out_l,
                      double* __restrict__ out_acc) {
    const uint64_t e = (uint64_t)blockIdx.x * kSpanThreads + threadIdx.x;
    if (e >= (uint64_t)heads * dim) return;
    const uint32_t g = (uint32_t)(e / dim);
    double ms = -INFINITY;
    for (uint32_t p = 0; p < n; ++p)
        if (!tokens || tokens[p]) ms = fmax(ms, m[(size_t)p * heads + g]);
    double ls = 0.0, s = 0.0;
    for (uint32_t p = 0; p < n; ++p) {
        if (tokens && !tokens[p]) continue;
        const double w = exp(m[(size_t)p * heads + g] - ms);
        ls = __dadd_rn(ls, __dmul_rn(l[(size_t)p * heads + g], w));
        s = __dadd_rn(s, __dmul_rn(acc[(size_t)p * heads * dim + e], w));
    }
    if (out_f32) out_f32[e] = (float)(s / ls);
    if (out_acc) {
        out_acc[e] = s;
        if (e % dim == 0) {
            out_m[g] = ms;
            out_l[g] = ls;
        }
    }
}

}  // namespace span
}  // namespace sinkr
