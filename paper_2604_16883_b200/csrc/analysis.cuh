// analysis.cuh — full-attention BOS mass on the GPU: the
// oracle side of the routing proxy.  attention_weights (attention.cpp:75-99)
// normalises softmax(scale * q.K^T) over the whole cached context; the oracle
// sink label needs only its token-0 entry alpha0 (analysis.hpp:12-22,
// SPEC.md oracle_labels).  One K-only streaming pass per layer:
//
//   bos_partial_kernel  grid (chunks, units): each CTA streams a token chunk
//                       of one unit's K rows (bf16, 16-byte vector loads), one
//                       token per thread, r head logits per row from the
//                       unit's queries in smem; per-head online (max, sum) in
//                       the log2 domain, reduced over the CTA -> partial.
//   bos_finish_kernel   per head: LSE-merge of the chunk partials and
//                       alpha0 = 2^(z0 - M) / L (z0 = token 0's logit).
//   weights_kernel      attention_weights rows: 2^(z_t - M) / L per token.
//
// K traffic: 2 * L * D bytes per unit (half a decode step's), so the pass is
// HBM bound like the decode stream.  Arithmetic is fp32 (q fp32, K bf16);
// the reference computes in fp64 — alpha0 agrees to ~1e-6 (tests).
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace sinkr {
namespace dev {

constexpr int kBosThreads = 256;
constexpr int kBosHeads = 8;  // heads per pass (a GQA group; more -> several passes)

struct BosArgs {
    const __nv_bfloat16* k;   // cache K base
    const float* q;           // [B*Hq][D] queries
    const uint32_t* len;      // [U] rows per unit (this layer)
    float* part;              // [U][chunks][r][2]: m, l (log2 domain)
    float* z0;                // [U*r] token-0 logit (log2 domain)
    float* stats;             // [U*r][2]: M, L after finish
    double* alpha0;           // [U*r]
    float* weights;           // weights_kernel: [r][len] of unit u_first
    uint32_t U, r, Hkv, cap, chunks, slot0;  // slot0 = layer * U
    uint32_t u_first;         // first unit of the launch (grid.y offset)
    float qscale;             // log2(e) / sqrt(D)
};

template <int D>
__device__ __forceinline__ void load_row(const __nv_bfloat16* row, float (&k)[D]) {
#pragma unroll
    for (int c = 0; c < D / 8; ++c) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(row) + c);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            k[8 * c + 2 * e] = __uint_as_float(w[e] << 16);
            k[8 * c + 2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
        }
    }
}

template <int D>
__global__ void __launch_bounds__(kBosThreads) bos_partial_kernel(BosArgs a, uint32_t h0) {
    __shared__ float sq[kBosHeads][D];
    __shared__ float red[kBosThreads / 32][kBosHeads][2];
    const uint32_t u = a.u_first + blockIdx.y, chunk = blockIdx.x;
    const uint32_t nh = min((uint32_t)kBosHeads, a.r - h0);
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint32_t i = tid; i < kBosHeads * D; i += kBosThreads) {
        const uint32_t h = i / D, j = i % D;
        sq[h][j] = h < nh ? a.q[(size_t(u) * a.r + h0 + h) * D + j] * a.qscale : 0.f;
    }
    __syncthreads();
    const uint32_t L = a.len[u];
    const uint32_t per = (L + a.chunks - 1) / a.chunks;
    const uint32_t t0 = min(L, chunk * per), t1 = min(L, t0 + per);
    const __nv_bfloat16* base = a.k + size_t(a.slot0 + u) * a.cap * D;
    float m[kBosHeads], l[kBosHeads];
#pragma unroll
    for (int h = 0; h < kBosHeads; ++h) {
        m[h] = -INFINITY;
        l[h] = 0.f;
    }
    for (uint32_t t = t0 + tid; t < t1; t += kBosThreads) {
        float k[D];
        load_row<D>(base + size_t(t) * D, k);
#pragma unroll
        for (int h = 0; h < kBosHeads; ++h) {
            if (h < (int)nh) {
                float z = 0.f;
#pragma unroll
                for (int j = 0; j < D; ++j) z = fmaf(sq[h][j], k[j], z);
                if (t == 0) a.z0[size_t(u) * a.r + h0 + h] = z;
                if (z > m[h]) {
                    l[h] = l[h] * exp2f(m[h] - z) + 1.f;
                    m[h] = z;
                } else {
                    l[h] += exp2f(z - m[h]);
                }
            }
        }
    }
    // CTA reduction of (m, l) per head
#pragma unroll
    for (int h = 0; h < kBosHeads; ++h) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float mo = __shfl_xor_sync(0xffffffffu, m[h], o);
            const float lo = __shfl_xor_sync(0xffffffffu, l[h], o);
            const float mx = fmaxf(m[h], mo);
            l[h] = (mx == -INFINITY) ? 0.f : l[h] * exp2f(m[h] - mx) + lo * exp2f(mo - mx);
            m[h] = mx;
        }
        if (lane == 0) {
            red[warp][h][0] = m[h];
            red[warp][h][1] = l[h];
        }
    }
    __syncthreads();
    if (tid < nh) {
        float M = -INFINITY;
        for (int w = 0; w < kBosThreads / 32; ++w) M = fmaxf(M, red[w][tid][0]);
        float S = 0.f;
        if (M != -INFINITY)
            for (int w = 0; w < kBosThreads / 32; ++w) S += red[w][tid][1] * exp2f(red[w][tid][0] - M);
        float* P = a.part + ((size_t(u) * a.chunks + chunk) * a.r + h0 + tid) * 2;
        P[0] = M;
        P[1] = S;
    }
}

__global__ void bos_finish_kernel(BosArgs a, uint32_t n_units) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;  // head index within the launch
    if (i >= n_units * a.r) return;
    const uint32_t u = a.u_first + i / a.r, h = i % a.r;
    double M = -INFINITY;
    for (uint32_t c = 0; c < a.chunks; ++c)
        M = fmax(M, (double)a.part[((size_t(u) * a.chunks + c) * a.r + h) * 2]);
    double S = 0.0;
    for (uint32_t c = 0; c < a.chunks; ++c) {
        const float* P = a.part + ((size_t(u) * a.chunks + c) * a.r + h) * 2;
        if (P[0] != -INFINITY) S += (double)P[1] * exp2((double)P[0] - M);
    }
    const size_t gi = size_t(u) * a.r + h;
    a.stats[gi * 2] = (float)M;
    a.stats[gi * 2 + 1] = (float)S;
    a.alpha0[gi] = exp2((double)a.z0[gi] - M) / S;
}

template <int D>
__global__ void __launch_bounds__(kBosThreads) weights_kernel(BosArgs a) {
    __shared__ float sq[kBosHeads][D];
    const uint32_t u = a.u_first;
    const uint32_t h0 = blockIdx.y * kBosHeads, nh = min((uint32_t)kBosHeads, a.r - h0);
    for (uint32_t i = threadIdx.x; i < kBosHeads * D; i += kBosThreads) {
        const uint32_t h = i / D, j = i % D;
        sq[h][j] = h < nh ? a.q[(size_t(u) * a.r + h0 + h) * D + j] * a.qscale : 0.f;
    }
    __syncthreads();
    const uint32_t L = a.len[u];
    const __nv_bfloat16* base = a.k + size_t(a.slot0 + u) * a.cap * D;
    for (uint32_t t = blockIdx.x * kBosThreads + threadIdx.x; t < L; t += gridDim.x * kBosThreads) {
        float k[D];
        load_row<D>(base + size_t(t) * D, k);
#pragma unroll
        for (int h = 0; h < kBosHeads; ++h) {
            if (h < (int)nh) {
                float z = 0.f;
#pragma unroll
                for (int j = 0; j < D; ++j) z = fmaf(sq[h][j], k[j], z);
                const size_t gi = size_t(u) * a.r + h0 + h;
                a.weights[size_t(h0 + h) * L + t] =
                    (float)(exp2((double)z - (double)a.stats[gi * 2]) / (double)a.stats[gi * 2 + 1]);
            }
        }
    }
}

}  // namespace dev
}  // namespace sinkr
