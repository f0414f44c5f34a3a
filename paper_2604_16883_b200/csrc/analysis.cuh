// analysis.cuh — full-attention BOS mass on the GPU: the
// oracle side of the routing proxy.  attention_weights (attention.cpp:75-99)
// normalises softmax(scale * q.K^T) over the whole cached context; the oracle
// sink label needs only its token-0 entry alpha0 (analysis.hpp:12-22,
// SPEC.md oracle_labels).  One K-only streaming pass per layer:
//
//   bos_stream_kernel   one CTA per SM; the units' K rows are one flat token
//                       space, claimed by guided self-scheduling.  A TMA producer
//                       warp streams 64-token K tiles (128B-swizzled, the
//                       decode stream's layout) into a smem ring; 4 consumer
//                       warps take 16 tokens each and compute the head logits
//                       on the tensor cores: z = Q.K^T with the fp32 query
//                       split three ways into bf16 (hi, lo, lo2; ~24 mantissa
//                       bits, products exact in fp32) — A1 = [hi; lo] and
//                       A2 = [lo2; 0] as 16-row mma.sync operands.  Per-head
//                       online (max, sum) in the log2 domain; one partial per
//                       (unit, CTA) the CTA's claims touched.
//   bos_finish_kernel   one warp per head: LSE-merge of the unit's partials
//                       (fp64) and alpha0 = 2^(z0 - M) / L (z0 = token 0's
//                       logit).  (Merging in the stream kernel, by the last CTA
//                       or by each unit's last flusher, measured 10 us slower.)
//   weights_kernel      attention_weights rows: 2^(z_t - M) / L per token, from
//                       the logits the stream pass wrote (same z, to the bit).
//
// K traffic: 2 * L * D bytes per unit (half a decode step's), so the pass is
// HBM bound like the decode stream.  The reference computes in fp64 — alpha0
// agrees to ~1e-7 (tests).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "kernels.cuh"
#include "ptx.cuh"

namespace sinkr {
namespace dev {

constexpr int kBosCWarps = 8;                  // consumer warps, 16 tokens each
constexpr int kBosThreads = 32 * (1 + kBosCWarps);
constexpr int kBosTok = kWarpTok * kBosCWarps;  // tokens per stage (2 per SMSP in flight)
constexpr int kBosBoxes = kBosTok / kStageTok;  // 64-row TMA boxes per stage and half
constexpr int kBosHeads = 16;                  // heads per unit: up to two 8-head mma tiles
static_assert(kBosHeads >= kMaxRWide, "one stream pass covers a GQA group");

struct BosArgs {
    const uint32_t* pre;      // [n_units + 1] token prefix over the launch's units
    const float* q;           // [B*Hq][D] queries
    float* part;              // [n_units][G][r][2]: m, l (log2 domain), slot-indexed
    uint32_t* ctr;            // [1 + n_units]: token cursor, partial slots per unit; zero
                              // on entry (two sets used alternately, see bos_finish_kernel)
    uint32_t* ctr_next;       // the other set: zeroed by bos_finish_kernel for the next call
    uint32_t ctr_len;         // entries per set
    float* z0;                // [U*r] token-0 logit (log2 domain)
    float* stats;             // [U*r][2]: M, L after finish
    double* alpha0;           // [U*r]
    float* zout;              // logits [r][L] of the launch's only unit, or null
    float* weights;           // weights_kernel: [r][L] of unit u_first
    uint32_t r, cap, slot0;     // slot0 = layer * (units per layer)
    uint32_t u_first, n_units;  // units of this launch
    uint32_t G;                 // stream CTAs
    float qscale;               // log2(e) / sqrt(D)
};

template <int D>
struct BosCfg {
    static constexpr int kHalves = Cfg<D>::kHalves;
    static constexpr int kBoxDim = Cfg<D>::kBoxDim;
    static constexpr int kStageBytes = kBosTok * D * 2;     // K only
    static constexpr int kStages = (192 * 1024) / kStageBytes > 16 ? 16 : (192 * 1024) / kStageBytes;
    static constexpr int kNK = D / 16;
    static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kStages * (16 + 16) +
                                      kBosCWarps * kBosHeads * 2 * 4 + 16;  // + the flush's slot index
};

// byte offset of (token, 16-byte chunk) in a K stage: swz<D> with kBosTok rows per half
template <int D>
__device__ __forceinline__ uint32_t bos_swz(uint32_t tok, uint32_t chunk) {
    if constexpr (D >= 64) {
        const uint32_t half = chunk >> 3, c = chunk & 7;
        return half * (kBosTok * 128) + tok * 128 + ((c ^ (tok & 7)) << 4);
    } else {
        const uint32_t o = tok * 64 + chunk * 16;
        return o ^ (((o >> 7) & 3) << 4);
    }
}

__device__ __forceinline__ uint32_t bos_ld_volatile(const uint32_t* p) {
    return *reinterpret_cast<const volatile uint32_t*>(p);
}

// one warp per head: the lanes fold the unit's partials (one per CTA that
// streamed part of it; at most G), read from L2
__device__ __forceinline__ void bos_finish_head(const BosArgs& a, uint32_t i, uint32_t h, uint32_t lane) {
    const uint32_t n = min(__ldcg(&a.ctr[1 + i]), a.G);
    double M = -INFINITY;
    for (uint32_t j = lane; j < n; j += 32)
        M = fmax(M, (double)__ldcg(&a.part[((size_t(i) * a.G + j) * a.r + h) * 2]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
    double S = 0.0;
    for (uint32_t j = lane; j < n; j += 32) {
        const float* P = a.part + ((size_t(i) * a.G + j) * a.r + h) * 2;
        const float pm = __ldcg(P);
        if (pm != -INFINITY) S += (double)__ldcg(P + 1) * exp2((double)pm - M);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
    if (lane == 0) {
        const size_t gi = size_t(a.u_first + i) * a.r + h;
        a.stats[gi * 2] = (float)M;
        a.stats[gi * 2 + 1] = (float)S;
        a.alpha0[gi] = exp2((double)__ldcg(&a.z0[gi]) - M) / S;
    }
}

// NT: 8-head query tiles per group (1: r <= 8; 2: r <= 16, each K fragment
// feeds both tiles' MMAs)
template <int D, int NT>
__global__ void __launch_bounds__(kBosThreads, 1)
    bos_stream_kernel(const __grid_constant__ CUtensorMap tmk, BosArgs a) {
    using C = BosCfg<D>;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* ring = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;
    StageMeta* meta = reinterpret_cast<StageMeta*>(empty + C::kStages);
    float* sm_ml = reinterpret_cast<float*>(meta + C::kStages);  // [kBosCWarps][kBosHeads][2]
    uint32_t* sm_slot = reinterpret_cast<uint32_t*>(sm_ml + kBosCWarps * kBosHeads * 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t c = blockIdx.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], kBosCWarps);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();

    if (warp == 0) {
        // ------------------------------ producer ------------------------------
        if (lane == 0) {
            ptx::tma_prefetch_desc(&tmk);
            const uint64_t pol = ptx::policy_evict_first();
            // guided self-scheduling over the flat token space (the units laid
            // end to end): a static first range of 2T/(3G) tokens per CTA, then
            // claims from one cursor whose size shrinks with the remaining
            // tokens, (T - pos)/(2G), down to one stage, so all SMs finish
            // within about a stage of each other.  Claims only move forward, so
            // a CTA meets each unit in one run and flushes it at most once.
            const uint32_t T = a.pre[a.n_units], G = gridDim.x;
            const uint32_t S0 = (uint32_t)((uint64_t)T * 2 / (3ull * G)) / kBosTok * kBosTok;
            const uint32_t base = (uint32_t)min((uint64_t)S0 * G, (uint64_t)T);
            const uint32_t cap_tok = max(S0, (uint32_t)kBosTok);
            auto guided = [&](uint32_t pos) {
                const uint32_t rem = T > pos ? T - pos : 0u;
                const uint32_t sz = rem / (2 * G) / kBosTok * kBosTok;
                return sz < (uint32_t)kBosTok ? (uint32_t)kBosTok : (sz > cap_tok ? cap_tok : sz);
            };
            int stage = 0;
            uint32_t phase = 0;
            uint32_t i = 0;  // launch-relative unit of g0
            uint32_t g0 = min(c * S0, base), g1 = min(g0 + S0, base);
            for (;;) {
                // prefetch the next claim, sized from the live cursor
                const uint32_t sz = guided(base + bos_ld_volatile(a.ctr));
                const uint32_t n0 = base + atomicAdd(a.ctr, sz);
                while (g0 < g1) {
                    if (a.pre[i + 1] <= g0) {  // binary search forward
                        uint32_t lo = i + 1, hi = a.n_units;
                        while (hi - lo > 1) {
                            const uint32_t mid = (lo + hi) >> 1;
                            if (a.pre[mid] <= g0) lo = mid; else hi = mid;
                        }
                        i = lo;
                    }
                    const uint32_t ub = a.pre[i], ue = min(a.pre[i + 1], g1);
                    const int32_t row0 = (int32_t)(size_t(a.slot0 + a.u_first + i) * a.cap);
                    for (uint32_t tk = g0 - ub; tk < ue - ub; tk += kBosTok) {
                        ptx::mbar_wait(&empty[stage], phase ^ 1u);
                        meta[stage].unit = i;
                        meta[stage].tok0 = tk;
                        meta[stage].ntok = min((uint32_t)kBosTok, ue - ub - tk);
                        ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                        uint8_t* kd = ring + stage * C::kStageBytes;
#pragma unroll
                        for (int hh = 0; hh < C::kHalves; ++hh)
#pragma unroll
                            for (int bx = 0; bx < kBosBoxes; ++bx)
                                ptx::tma_load_2d(kd + (hh * kBosTok + bx * kStageTok) * (D >= 64 ? 128 : 2 * D),
                                                 &tmk, hh * C::kBoxDim, row0 + (int32_t)(tk + bx * kStageTok),
                                                 &full[stage], pol);
                        if (++stage == C::kStages) {
                            stage = 0;
                            phase ^= 1u;
                        }
                    }
                    g0 = ue;
                }
                if (n0 >= T) break;
                g0 = n0;
                g1 = min(n0 + sz, T);
            }
            ptx::mbar_wait(&empty[stage], phase ^ 1u);
            meta[stage].unit = kEnd;
            ptx::mbar_arrive(&full[stage]);
        }
    } else {
        // ------------------------------ consumers ------------------------------
        const int cw = warp - 1;
        const uint32_t ctid = threadIdx.x - 32;
        const int tb = cw * kWarpTok;
        const int grp = lane >> 2, qd = lane & 3;
        const int lj = lane >> 3, li = lane & 7;
        const uint32_t k_tok = tb + ((lj >> 1) << 3) + li, k_csel = lj & 1;
        const uint32_t nh = a.r;  // <= 8 * NT: one pass covers the group

        // per tile: A1 = [hi; lo], A2 = [lo2; 0] of heads 8 ht + grp
        uint32_t q1[NT][C::kNK][4], q2[NT][C::kNK][2];
        float m[NT], l[NT];
        uint32_t cur = kEnd;

        auto load_q = [&](uint32_t i) {
#pragma unroll
            for (int ht = 0; ht < NT; ++ht) {
                const bool live = 8 * ht + grp < (int)nh;
                const float* qrow = a.q + (size_t(a.u_first + i) * a.r + (live ? 8 * ht + grp : 0)) * D;
#pragma unroll
                for (int kk = 0; kk < C::kNK; ++kk) {
#pragma unroll
                    for (int hv = 0; hv < 2; ++hv) {
                        float2 x = make_float2(0.f, 0.f);
                        if (live) x = *reinterpret_cast<const float2*>(qrow + 16 * kk + 8 * hv + 2 * qd);
                        x.x *= a.qscale;
                        x.y *= a.qscale;
                        const uint32_t hi = ptx::pack_bf16(x.x, x.y);
                        const float r0 = x.x - ptx::bf16_lo_as_f32(hi), r1 = x.y - ptx::bf16_hi_as_f32(hi);
                        const uint32_t lo = ptx::pack_bf16(r0, r1);
                        q1[ht][kk][2 * hv] = hi;
                        q1[ht][kk][2 * hv + 1] = lo;
                        q2[ht][kk][hv] = ptx::pack_bf16(r0 - ptx::bf16_lo_as_f32(lo), r1 - ptx::bf16_hi_as_f32(lo));
                    }
                }
            }
        };
        auto flush = [&](uint32_t i) {
#pragma unroll
            for (int ht = 0; ht < NT; ++ht) {
                float mo = __shfl_xor_sync(0xffffffffu, m[ht], 1), lo = __shfl_xor_sync(0xffffffffu, l[ht], 1);
                float mx = fmaxf(m[ht], mo);
                l[ht] = mx == -INFINITY ? 0.f : l[ht] * exp2f(m[ht] - mx) + lo * exp2f(mo - mx);
                m[ht] = mx;
                mo = __shfl_xor_sync(0xffffffffu, m[ht], 2);
                lo = __shfl_xor_sync(0xffffffffu, l[ht], 2);
                mx = fmaxf(m[ht], mo);
                l[ht] = mx == -INFINITY ? 0.f : l[ht] * exp2f(m[ht] - mx) + lo * exp2f(mo - mx);
                m[ht] = mx;
                if (qd == 0) {
                    sm_ml[(cw * kBosHeads + 8 * ht + grp) * 2] = m[ht];
                    sm_ml[(cw * kBosHeads + 8 * ht + grp) * 2 + 1] = l[ht];
                }
            }
            if (ctid == 0) sm_slot[0] = atomicAdd(&a.ctr[1 + i], 1u);
            ptx::named_bar_sync(1, kBosCWarps * 32);
            if (ctid < nh) {
                float M = -INFINITY;
#pragma unroll
                for (int w = 0; w < kBosCWarps; ++w) M = fmaxf(M, sm_ml[(w * kBosHeads + ctid) * 2]);
                float S = 0.f;
                if (M != -INFINITY)
#pragma unroll
                    for (int w = 0; w < kBosCWarps; ++w)
                        S += sm_ml[(w * kBosHeads + ctid) * 2 + 1] * exp2f(sm_ml[(w * kBosHeads + ctid) * 2] - M);
                float* P = a.part + ((size_t(i) * a.G + sm_slot[0]) * a.r + ctid) * 2;
                P[0] = M;
                P[1] = S;
            }
            ptx::named_bar_sync(1, kBosCWarps * 32);
        };

        int stage = 0;
        uint32_t phase = 0;
        for (;;) {
            ptx::mbar_wait(&full[stage], phase);
            const uint32_t unit = meta[stage].unit;
            if (unit == kEnd) break;
            if (unit != cur) {
                if (cur != kEnd) flush(cur);
                cur = unit;
                load_q(unit);
#pragma unroll
                for (int ht = 0; ht < NT; ++ht) {
                    m[ht] = -INFINITY;
                    l[ht] = 0.f;
                }
            }
            const uint32_t tok0 = meta[stage].tok0;
            const int n = (int)meta[stage].ntok - tb;
            if (n > 0) {
                const uint32_t kbase = ptx::smem_u32(ring + stage * C::kStageBytes);
                float s1[NT][2][2][4], s2[NT][2][4];
#pragma unroll
                for (int ht = 0; ht < NT; ++ht)
#pragma unroll
                    for (int x = 0; x < 2; ++x) {
                        s2[ht][x][0] = s2[ht][x][1] = s2[ht][x][2] = s2[ht][x][3] = 0.f;
#pragma unroll
                        for (int y = 0; y < 2; ++y)
                            s1[ht][x][y][0] = s1[ht][x][y][1] = s1[ht][x][y][2] = s1[ht][x][y][3] = 0.f;
                    }
#pragma unroll
                for (int kk = 0; kk < C::kNK; ++kk) {
                    uint32_t b[4];
                    ptx::ldsm_x4(b, kbase + bos_swz<D>(k_tok, 2 * kk + k_csel));
#pragma unroll
                    for (int ht = 0; ht < NT; ++ht) {
                        const uint32_t a2[4] = {q2[ht][kk][0], 0u, q2[ht][kk][1], 0u};
                        ptx::mma_bf16(s1[ht][0][kk & 1], q1[ht][kk], b[0], b[1]);
                        ptx::mma_bf16(s1[ht][1][kk & 1], q1[ht][kk], b[2], b[3]);
                        ptx::mma_bf16(s2[ht][0], a2, b[0], b[1]);
                        ptx::mma_bf16(s2[ht][1], a2, b[2], b[3]);
                    }
                }
#pragma unroll
                for (int ht = 0; ht < NT; ++ht) {
                    const int head = 8 * ht + grp;
                    const bool live = head < (int)nh;
                    float z[4];
                    float bm = -INFINITY;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int nt = j >> 1, col = j & 1;
                        const float hi = s1[ht][nt][0][col] + s1[ht][nt][1][col];
                        const float lo = s1[ht][nt][0][col + 2] + s1[ht][nt][1][col + 2];
                        const int tok = nt * 8 + 2 * qd + col;
                        z[j] = tok < n ? (hi + lo) + s2[ht][nt][col] : -INFINITY;
                        bm = fmaxf(bm, z[j]);
                    }
                    if (tok0 + tb == 0 && live && qd == 0)  // token 0 of the unit: j = 0 of lane quad 0
                        a.z0[size_t(a.u_first + unit) * a.r + head] = z[0];
                    if (a.zout != nullptr && live) {  // attention_weights: keep every logit
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int tok = (j >> 1) * 8 + 2 * qd + (j & 1);
                            if (tok < n) a.zout[size_t(head) * a.pre[1] + tok0 + tb + tok] = z[j];
                        }
                    }
                    if (bm != -INFINITY) {
                        const float mn = fmaxf(m[ht], bm);
                        l[ht] = (m[ht] == -INFINITY ? 0.f : l[ht] * exp2f(m[ht] - mn)) +
                                ((exp2f(z[0] - mn) + exp2f(z[1] - mn)) + (exp2f(z[2] - mn) + exp2f(z[3] - mn)));
                        m[ht] = mn;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&empty[stage]);
            if (++stage == C::kStages) {
                stage = 0;
                phase ^= 1u;
            }
        }
        if (cur != kEnd) flush(cur);
    }

}

// one warp per head (grid-wide), then zero the counter set of the next call
__global__ void __launch_bounds__(256) bos_finish_kernel(BosArgs a) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t idx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < a.ctr_len; j += gridDim.x * blockDim.x)
        a.ctr_next[j] = 0;
    if (idx < a.n_units * a.r) bos_finish_head(a, idx / a.r, idx % a.r, lane);
}

// attention_weights of unit u_first from the stream pass's logits
__global__ void weights_kernel(BosArgs a) {
    const uint32_t L = a.pre[1];
    const size_t n = size_t(a.r) * L;
    for (size_t idx = size_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < n;
         idx += size_t(gridDim.x) * blockDim.x) {
        const uint32_t h = (uint32_t)(idx / L);
        const size_t gi = size_t(a.u_first) * a.r + h;
        a.weights[idx] =
            (float)(exp2((double)a.zout[idx] - (double)a.stats[gi * 2]) / (double)a.stats[gi * 2 + 1]);
    }
}

}  // namespace dev
}  // namespace sinkr
