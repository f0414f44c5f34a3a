// kernels.cuh — the three sm_100a kernels of one SinkRouter decode step.
//
//   probe_kernel   router.cpp:100-125 (proxy_score router.cpp:36-48,
//                  group_score 50-57, route 67-75) + the task build of
//                  router.cpp:131-145, as a device-side compacted work list.
//   decode_kernel  attend_chunk (attention.cpp:101-142) over the Active
//                  groups only, persistent over all SMs.
//   combine_kernel merge_partials (attention.cpp:159-183) + output assembly
//                  with the zero surrogate (router.cpp:96-98,168-186).
//
// HBM layout: K and V are bf16 [layer][seq][kv_head][cap][D]
// (the reference slot layout kv_cache.cpp:41-49,79-80 with a batch axis);
// anchors f32 [layer][seq][kv_head][D] + k0_norm f32.  A "unit" is one
// (seq, kv_head) pair of the layer being decoded: u = seq * H_kv + g.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "ptx.cuh"

namespace sinkr {
namespace dev {

constexpr int kStageTok = 64;                         // tokens per TMA stage
constexpr int kWarpTok = 16;                          // tokens per consumer warp per stage
constexpr int kCWarps = kStageTok / kWarpTok;         // consumer warps
constexpr int kThreads = 32 * (1 + kCWarps);          // + 1 TMA producer warp
constexpr int kMaxR = 8;                              // GQA width per MMA row tile (hi/lo split)
constexpr int kMaxRWide = 16;                         // step kernel WIDE form: two 8-head tiles per group
constexpr uint32_t kEnd = 0xFFFFFFFFu;
constexpr int kProbeThreads = 256;
constexpr int kChunksPerCta = 128;                    // dynamic-scheduling granularity target
constexpr int kMinChunkTok = 256;                     // >= claim latency of one chunk

// unit_flags bits
constexpr uint32_t kSink = 1u, kDegenerate = 2u, kActive = 4u;
// hdr flags
constexpr uint32_t kObserveOnly = 1u, kSinkOnTie = 2u, kLayerExcluded = 4u;

// Host -> device copy of the pinned (mapped) staging block by a small kernel.
// As a graph node it is ~8 us shorter than a cudaMemcpy node of the same 16 KB
// (copy-engine start latency; scripts/micro/e2e_floor.cu), which is most of
// what separates a blocking step from its device time.
__global__ void upload_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, uint32_t n16) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x)
        dst[i] = src[i];
}

struct StepHdr {
    uint32_t layer;
    uint32_t flags;
    uint32_t pad[2];
};

// Per-step scalars handed to the probe by value (kernel parameters live in the
// constant bank: no global-memory round trip before routing can start).  The
// engine patches them into the captured graph node each step.
constexpr int kParamSeqs = 8;  // keeps the launch parameter block small (launch latency)
struct ProbeParams {
    uint32_t layer;
    uint32_t flags;
    uint32_t inline_seqs;  // 1: tau/len below; 0: B > kParamSeqs, read DevTables.tau/len
    uint32_t only_unit;    // 0: route; u + 1: unit u Active, every other unit Sink
                           // (sinkr_group_attention: splitk_attention of one group)
    double tau[kParamSeqs];
    uint32_t len[kParamSeqs];
};

// ProbeParams.only_unit: the route decision replaced by "unit only_unit - 1
// Active, every other unit Sink" (applied after the scores are formed)
__device__ __forceinline__ void force_route(uint32_t only_unit, uint32_t u, bool& sink, bool& active) {
    if (only_unit) {
        active = u + 1 == only_unit;
        sink = !active;
    }
}

struct WorkState {
    unsigned int n_active;
    unsigned int chunk_tokens;
    unsigned int error;
    unsigned int probe_done;
    unsigned int pad[4];
};

struct StageMeta {
    uint32_t unit;
    uint32_t tok0;
    uint32_t ntok;
    uint32_t pad;
};

struct DevTables {
    const StepHdr* hdr;
    const double* tau;           // [B]
    const uint32_t* len;         // [B] rows to attend per seq
    const float* q;              // [B][Hq][D]
    const float* anchors;        // [layers][B][Hkv][D]
    const float* anchor_norm;    // [layers][B][Hkv]
    double* head_scores;         // [B*Hq]
    uint32_t* head_degen;        // [B*Hq]
    double* group_scores;        // [U]
    uint32_t* unit_flags;        // [U]
    unsigned long long* tokens;  // [U] rows streamed by decode (measured)
    WorkState* ws;
    uint4* act_info;             // [U] compacted Active units {unit, L, nchunks, slot}
    uint32_t* unit_next;         // [U] chunk cursor per active-list entry
    uint32_t* slot_count;        // [U]
    float* partials;             // [U][S][r*(D+2)]
    uint32_t B, Hq, Hkv, r, D, cap, S, grid;
    float qscale;                // (1/sqrt(D)) * log2(e)
    uint32_t* done;              // probe: optional completion word in mapped host memory (set last)
};

// ============================================================================
// score_batch: the score-collection mode over n query samples
// of one cache layer in one launch -- proxy_score (router.cpp:36-48),
// group_score (50-57) and the route compare (67-75,113-120), bit-exact with
// the probe kernel (the same products, sequential chains and IEEE
// sqrt/div/clamp).  CTA c takes units_per_cta whole units of the n x U
// (sample, unit) space, so a group's mean needs no other CTA.
// ============================================================================
struct ScoreBatchArgs {
    const float* q;             // [n][B*Hq][D]
    const float* anchors;       // this layer's [U][D]
    const float* anchor_norm;   // this layer's [U]
    const double* tau;          // [B] (cfg only)
    double* head_scores;        // [n][B*Hq]
    double* group_scores;       // [n][U]
    int32_t* sink;              // [n][U]
    uint32_t n, U, Hkv, r, units_per_cta, flags, has_cfg;
};
constexpr int kScoreThreads = 128;
constexpr int kScoreHeads = 64;  // heads per CTA (whole units)

template <int D>
__global__ void __launch_bounds__(kScoreThreads) score_batch_kernel(const ScoreBatchArgs a) {
    constexpr int DP = D + 1;
    extern __shared__ double s_prod[];  // [2][kScoreHeads][D+1]: q*k0, q*q
    __shared__ double s_sc[kScoreHeads];
    __shared__ uint32_t s_dg[kScoreHeads];
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t r = a.r, NH = a.U * r;
    const uint32_t gu0 = blockIdx.x * a.units_per_cta;  // first (sample, unit) of this CTA
    const uint32_t nu = min(a.units_per_cta, a.n * a.U - gu0);
    const uint32_t nh = nu * r;
    // exact fp64 products (f32 x f32 fits in 53 bits) into odd-stride rows
    for (uint32_t hl = warp; hl < nh; hl += kScoreThreads / 32) {
        const uint32_t gu = gu0 + hl / r, smp = gu / a.U, u = gu % a.U;
        const float* qrow = a.q + (size_t(smp) * NH + u * r + hl % r) * D;
        const float* krow = a.anchors + size_t(u) * D;
        for (uint32_t j = lane; j < (uint32_t)D; j += 32) {
            const double qj = (double)__ldg(qrow + j);
            s_prod[hl * DP + j] = __dmul_rn(qj, (double)__ldg(krow + j));
            s_prod[(kScoreHeads + hl) * DP + j] = __dmul_rn(qj, qj);
        }
    }
    __syncthreads();
    // thread h: the dot chain of head h; thread 64+h: its |q|^2 chain -- each a
    // sequential sum in index order (router.cpp:40-43)
    const uint32_t hl = tid % kScoreHeads;
    double acc = 0.0;
    if (hl < nh) {
        const double* pr = s_prod + ((tid < (uint32_t)kScoreHeads ? 0 : kScoreHeads) + hl) * DP;
#pragma unroll 16
        for (uint32_t j = 0; j < (uint32_t)D; ++j) acc = __dadd_rn(acc, pr[j]);
    }
    __syncthreads();  // products dead: reuse row 0 of the second half for the |q|^2 sums
    double* s_qq = s_prod + kScoreHeads * DP;
    if (tid >= (uint32_t)kScoreHeads && hl < nh) s_qq[hl] = acc;
    __syncthreads();
    if (tid < nh) {
        const uint32_t gu = gu0 + tid / r, smp = gu / a.U, u = gu % a.U;
        const double qn = __dsqrt_rn(s_qq[tid]);
        double sc = 0.0;
        uint32_t dg = 0;
        if (qn < 1e-12) {
            dg = 1;
        } else {
            sc = __ddiv_rn(acc, __dmul_rn(qn, (double)__ldg(&a.anchor_norm[u])));
            sc = sc < -1.0 ? -1.0 : (1.0 < sc ? 1.0 : sc);  // std::clamp
        }
        s_sc[tid] = sc;
        s_dg[tid] = dg;
        a.head_scores[size_t(smp) * NH + u * r + tid % r] = sc;
    }
    __syncthreads();
    if (tid < nu) {
        const uint32_t gu = gu0 + tid, smp = gu / a.U, u = gu % a.U;
        double sum = 0.0;
        uint32_t degen = 0;
        for (uint32_t i = 0; i < r; ++i) {
            sum = __dadd_rn(sum, s_sc[tid * r + i]);
            degen |= s_dg[tid * r + i];
        }
        const double S = __ddiv_rn(sum, (double)r);
        a.group_scores[size_t(smp) * a.U + u] = S;
        bool sink = false;
        if (a.has_cfg) {
            const double tau = a.tau[u / a.Hkv];
            const bool over = (a.flags & kSinkOnTie) ? (S >= tau) : (S > tau);
            sink = over && !(a.flags & kLayerExcluded) && !degen;
        }
        a.sink[size_t(smp) * a.U + u] = sink ? 1 : 0;
    }
}

// ============================================================================
// probe: bit-exact with router.cpp:36-75.  Each CTA scores a tile of
// kProbeHeads query heads: all threads form the exact fp64 products
// (f32 x f32 is exact in fp64) into shared memory, then one thread per head
// sums them sequentially in index order (the reference's order — a tree
// reduction would change ~75% of the bit patterns) and takes
// IEEE sqrt/div and the clamp.  The last CTA (the only one for <= 64 heads)
// does group_score (sequential mean), the tau compare (strict '>' or '>=' under
// sink_on_tie; tau computed on the host with the reference's own expression)
// and builds the compacted Active work list for the decode kernel.  All global
// inputs are fetched in one batch of independent loads.
// ============================================================================
constexpr int kProbeHeads = 64;

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <int D>
__global__ void __launch_bounds__(kProbeThreads, 1) probe_kernel(DevTables t, const ProbeParams p) {
    using Scan = cub::BlockScan<uint32_t, kProbeThreads>;
    using Reduce = cub::BlockReduce<unsigned long long, kProbeThreads>;
    __shared__ union {
        typename Scan::TempStorage scan;
        typename Reduce::TempStorage reduce;
    } tmp;
    __shared__ unsigned long long s_tokens;
    __shared__ uint32_t s_last;
    __shared__ double s_score[kProbeHeads];
    __shared__ uint32_t s_degen[kProbeHeads];
    constexpr int DP = D + 1;
    extern __shared__ double s_prod[];                      // [2][kProbeHeads][D+1]

    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    pdl_launch();
    const uint32_t U = t.B * t.Hkv, NH = t.B * t.Hq;

    // ---- proxy_score for this CTA's head tile (router.cpp:36-48).  Warp w
    // takes heads w, w+8, ...; lanes take dims.  Head i belongs to unit i / r
    // (heads of a GQA group are contiguous, router.cpp:109).
    constexpr int kHW = kProbeHeads / (kProbeThreads / 32);  // heads per warp
    constexpr int kJL = (D + 31) / 32;                        // dims per lane
    const uint32_t h_base = blockIdx.x * kProbeHeads;
    const uint32_t nh = min((uint32_t)kProbeHeads, NH - h_base);
    float qv[kHW][kJL];
#pragma unroll
    for (int a = 0; a < kHW; ++a) {
        const uint32_t i = h_base + warp + a * (kProbeThreads / 32);
#pragma unroll
        for (int b = 0; b < kJL; ++b) {
            const uint32_t j = lane + 32 * b;
            qv[a][b] = (i < NH && j < D) ? __ldg(t.q + size_t(i) * D + j) : 0.f;
        }
    }
    const uint32_t layer = p.layer, flags = p.flags;
    float kv[kHW][kJL];
#pragma unroll
    for (int a = 0; a < kHW; ++a) {
        const uint32_t i = h_base + warp + a * (kProbeThreads / 32);
        const size_t slot = size_t(layer) * U + (i < NH ? i / t.r : 0);
#pragma unroll
        for (int b = 0; b < kJL; ++b) {
            const uint32_t j = lane + 32 * b;
            kv[a][b] = (i < NH && j < D) ? __ldg(t.anchors + slot * D + j) : 0.f;
        }
    }
    double kn = 1.0;
    if (tid < nh) kn = (double)__ldg(&t.anchor_norm[size_t(layer) * U + (h_base + tid) / t.r]);
#pragma unroll
    for (int a = 0; a < kHW; ++a) {
        const uint32_t hl = warp + a * (kProbeThreads / 32);
#pragma unroll
        for (int b = 0; b < kJL; ++b) {
            const uint32_t j = lane + 32 * b;
            if (j < D) {
                const double qj = (double)qv[a][b];
                s_prod[hl * DP + j] = __dmul_rn(qj, (double)kv[a][b]);
                s_prod[(kProbeHeads + hl) * DP + j] = __dmul_rn(qj, qj);
            }
        }
    }
    __syncthreads();
    if (tid < nh) {
        const uint32_t i = h_base + tid;
        const double* pd = s_prod + tid * DP;
        const double* pq = s_prod + (kProbeHeads + tid) * DP;
        double dot = 0.0, qsq = 0.0;
#pragma unroll 16
        for (uint32_t j = 0; j < D; ++j) {
            dot = __dadd_rn(dot, pd[j]);
            qsq = __dadd_rn(qsq, pq[j]);
        }
        const double qn = __dsqrt_rn(qsq);
        double sc = 0.0;
        uint32_t dg = 0;
        if (qn < 1e-12) {
            dg = 1;
        } else {
            sc = __ddiv_rn(dot, __dmul_rn(qn, kn));
            sc = sc < -1.0 ? -1.0 : (1.0 < sc ? 1.0 : sc);  // std::clamp
        }
        t.head_scores[i] = sc;
        t.head_degen[i] = dg;
        s_score[tid] = sc;
        s_degen[tid] = dg;
    }

    // ---- last CTA: group_score / route / work list
    const bool single = gridDim.x == 1;
    if (!single) {
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = atomicAdd(&t.ws->probe_done, 1u) == gridDim.x - 1;
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        if (tid == 0) t.ws->probe_done = 0;
    }
    __syncthreads();

    // group_score + route (router.cpp:50-57,67-75,113-120).  Units are
    // processed in contiguous runs per thread so the scan below keeps order.
    const uint32_t per = (U + kProbeThreads - 1) / kProbeThreads;
    const uint32_t u0 = min(U, tid * per), u1 = min(U, u0 + per);
    uint32_t my_active = 0, my_flags = 0;
    unsigned long long my_tokens = 0;
    for (uint32_t u = u0; u < u1; ++u) {
        const uint32_t seq = u / t.Hkv;
        const uint32_t h0 = u * t.r;
        double sum = 0.0;
        uint32_t degen = 0;
        for (uint32_t i = 0; i < t.r; ++i) {
            const double hs = single ? s_score[h0 + i] : __ldcg(&t.head_scores[h0 + i]);
            sum = __dadd_rn(sum, hs);
            degen |= single ? s_degen[h0 + i] : __ldcg(&t.head_degen[h0 + i]);
        }
        const double S = __ddiv_rn(sum, (double)t.r);
        const double tau = p.inline_seqs ? p.tau[seq] : __ldg(&t.tau[seq]);
        const bool over = (flags & kSinkOnTie) ? (S >= tau) : (S > tau);
        bool sink = over && !(flags & kLayerExcluded);
        if (degen) sink = false;  // router.cpp:114-117 fail-safe toward exact
        bool active = (flags & kObserveOnly) || !sink;
        force_route(p.only_unit, u, sink, active);
        const uint32_t fl =
            (sink ? kSink : 0u) | (degen ? kDegenerate : 0u) | (active ? kActive : 0u);
        t.group_scores[u] = S;
        t.unit_flags[u] = fl;
        t.slot_count[u] = 0;
        t.tokens[u] = 0ull;
        if (active) {
            ++my_active;
            my_tokens += p.inline_seqs ? p.len[seq] : __ldg(&t.len[seq]);
        }
        if (u - u0 < 32) my_flags |= (active ? 1u : 0u) << (u - u0);
    }
    const unsigned long long T_all = Reduce(tmp.reduce).Sum(my_tokens);
    if (tid == 0) s_tokens = T_all;
    __syncthreads();
    uint32_t a_off, a_tot;
    Scan(tmp.scan).ExclusiveSum(my_active, a_off, a_tot);
    // chunk size: ~kChunksPerCta chunks per persistent CTA, multiple of a stage
    const unsigned long long T = s_tokens;
    unsigned long long cc = (T + (unsigned long long)t.grid * kChunksPerCta - 1) /
                            ((unsigned long long)t.grid * kChunksPerCta);
    cc = ((cc + kStageTok - 1) / kStageTok) * kStageTok;
    if (cc < kMinChunkTok) cc = kMinChunkTok;
    const uint32_t Ck = (uint32_t)cc;
    for (uint32_t u = u0; u < u1; ++u) {
        const bool act = (u - u0 < 32) ? ((my_flags >> (u - u0)) & 1u) : (t.unit_flags[u] & kActive);
        if (!act) continue;
        const uint32_t L = p.inline_seqs ? p.len[u / t.Hkv] : __ldg(&t.len[u / t.Hkv]);
        // decode CTAs c with c % a_tot == a_off take chunk c / a_tot statically
        t.unit_next[a_off] = a_off < t.grid ? (t.grid - a_off + a_tot - 1) / a_tot : 0u;
        t.act_info[a_off] = make_uint4(u, L, (L + Ck - 1) / Ck, layer * U + u);
        ++a_off;
    }
    if (tid == 0) {
        t.ws->n_active = a_tot;
        t.ws->chunk_tokens = Ck;
        t.ws->error = 0;
    }
    if (t.done) {
        // score collection: the scores went to mapped host memory; make the
        // whole CTA's writes visible system-wide, then set the word the host
        // spins on (no kernel-retire -> stream-sync round trip)
        __syncthreads();
        if (tid == 0) {
            __threadfence_system();
            ptx::st_release_sys(t.done, 1u);
        }
    }
}

// ============================================================================
// decode: persistent Split-K flash-decode over the Active work list.
//
// Warp 0 (one lane) is the TMA producer: it claims chunks (unit, token range)
// from a global atomic counter and streams K/V rows in 64-token stages into
// a kStages-deep shared-memory ring (cp.async.bulk.tensor, 128B swizzle,
// L2 evict_first).  Warps 1..4 each take 16 tokens of every stage:
//   S^T-free QK:   S[16 x 16] = Qhl[16 x D] . K^T      (mma.sync m16n8k16)
//                  rows 0-7 = q_hi of heads 0-7, rows 8-15 = q_lo, so the fp32
//                  query is carried at ~16 mantissa bits; s = S[h] + S[h+8]
//   online softmax fp32, log2 domain, lazy rescale (threshold 8)
//   PV:            O[16 x D] += Phl[16 x 16] . V      (same hi/lo split of P)
// A CTA keeps one running state per unit and flushes a partial (m, l, acc)
// when its stream moves to another unit.
// ============================================================================
template <int D>
struct Cfg {
    static constexpr int kHalves = D >= 64 ? D / 64 : 1;       // 128B-swizzled boxes per row
    static constexpr int kBoxDim = D >= 64 ? 64 : D;
    static constexpr int kTileBytes = kStageTok * D * 2;       // one of K or V per stage
    static constexpr int kStageBytes = 2 * kTileBytes;
    static constexpr int kStages = D >= 128 ? 6 : (D == 64 ? 10 : 16);
    static constexpr int kNK = D / 16;                         // k-steps of QK / n-pairs of PV
    static constexpr int kOStride = D + 4;
    static constexpr int kScratchBytes = kCWarps * kMaxR * (kOStride + 2) * 4 + 16;
    static constexpr int kSmemBytes =
        1024 + kStages * kStageBytes + kStages * 16 + kStages * 16 + kScratchBytes;
};

// byte offset of (token, first dim of a 16-byte chunk) inside a K or V tile
template <int D>
__device__ __forceinline__ uint32_t swz(uint32_t tok, uint32_t chunk) {
    if constexpr (D >= 64) {
        const uint32_t half = chunk >> 3, c = chunk & 7;
        return half * (kStageTok * 128) + tok * 128 + ((c ^ (tok & 7)) << 4);
    } else {  // D == 32: 64-byte rows, SWIZZLE_64B (bits 4-5 ^= bits 7-8)
        const uint32_t o = tok * 64 + chunk * 16;
        return o ^ (((o >> 7) & 3) << 4);
    }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    decode_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                  DevTables t) {
    using C = Cfg<D>;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;
    StageMeta* meta = reinterpret_cast<StageMeta*>(empty + C::kStages);
    float* sm_o = reinterpret_cast<float*>(meta + C::kStages);     // [kCWarps][kMaxR][kOStride]
    float* sm_ml = sm_o + kCWarps * kMaxR * C::kOStride;            // [kCWarps][kMaxR][2]
    uint32_t* sm_slot = reinterpret_cast<uint32_t*>(sm_ml + kCWarps * kMaxR * 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], kCWarps);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmk);
        ptx::tma_prefetch_desc(&tmv);
    }
    pdl_launch();  // let the combine grid get resident early; it waits on us
    pdl_wait();    // the probe's work list must be complete and visible
    const uint32_t PS = t.r * (D + 2);

    if (warp == 0) {
        // ------------------------------ producer ------------------------------
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_first();
            // Unit-affine dynamic scheduling: CTA c starts on active unit
            // c mod n_active and claims chunks from that unit's cursor; when
            // the unit is exhausted it moves on to the next one, so every CTA
            // keeps streaming until all Active units are done while touching
            // only ~1-2 units (few Split-K partials per unit).
            const uint32_t nact = t.ws->n_active, Ck = t.ws->chunk_tokens;
            int stage = 0;
            uint32_t phase = 0;
            if (nact > 0) {
                // first claim is static (chunk blockIdx / nact of entry blockIdx % nact;
                // the probe pre-advanced the cursors past these), later ones dynamic
                uint32_t a = blockIdx.x % nact, visited = 1;
                uint32_t k = blockIdx.x / nact;
                uint4 ai = t.act_info[a];  // {unit, L, nch, slot}
                for (;;) {
                    const uint32_t u = ai.x, L = ai.y, nch = ai.z;
                    if (k >= nch) {
                        if (visited == nact) break;
                        ++visited;
                        a = (a + 1 == nact) ? 0 : a + 1;
                        ai = t.act_info[a];
                        k = atomicAdd(&t.unit_next[a], 1u);
                        continue;
                    }
                    const uint32_t k_next = atomicAdd(&t.unit_next[a], 1u);  // prefetch claim
                    const uint32_t t0 = k * Ck;
                    const uint32_t t1 = min(t0 + Ck, L);
                    const int32_t row0 = (int32_t)(size_t(ai.w) * t.cap);
                    for (uint32_t tk = t0; tk < t1; tk += kStageTok) {
                        ptx::mbar_wait(&empty[stage], phase ^ 1u);
                        meta[stage].unit = u;
                        meta[stage].tok0 = tk;
                        meta[stage].ntok = min((uint32_t)kStageTok, t1 - tk);
                        ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                        uint8_t* kd = ring + stage * C::kStageBytes;
                        uint8_t* vd = kd + C::kTileBytes;
#pragma unroll
                        for (int h = 0; h < C::kHalves; ++h) {
                            ptx::tma_load_2d(kd + h * kStageTok * 128, &tmk, h * C::kBoxDim,
                                             row0 + (int32_t)tk, &full[stage], pol);
                            ptx::tma_load_2d(vd + h * kStageTok * 128, &tmv, h * C::kBoxDim,
                                             row0 + (int32_t)tk, &full[stage], pol);
                        }
                        if (++stage == C::kStages) {
                            stage = 0;
                            phase ^= 1u;
                        }
                    }
                    k = k_next;
                }
            }
            ptx::mbar_wait(&empty[stage], phase ^ 1u);
            meta[stage].unit = kEnd;
            ptx::mbar_arrive(&full[stage]);
        }
        return;
    }

    // ------------------------------ consumers ------------------------------
    const int cw = warp - 1;
    const uint32_t ctid = threadIdx.x - 32;  // 0..127
    const int tb = cw * kWarpTok;            // this warp's token offset in a stage
    const int grp = lane >> 2, qd = lane & 3;
    const int lj = lane >> 3, li = lane & 7;
    // ldmatrix lane roles (see DESIGN.md §4 for the fragment mapping)
    const uint32_t k_tok = tb + ((lj >> 1) << 3) + li, k_csel = lj & 1;
    const uint32_t v_tok = tb + ((lj & 1) << 3) + li, v_csel = lj >> 1;

    uint32_t qa[C::kNK][4];
    float o[2 * C::kNK][4];
    float m_used = -INFINITY, l_acc = 0.f;
    uint32_t cur = kEnd, run_tokens = 0;

    auto reset_state = [&]() {
#pragma unroll
        for (int i = 0; i < 2 * C::kNK; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
        m_used = -INFINITY;
        l_acc = 0.f;
    };
    auto load_q = [&](uint32_t u) {
        const uint32_t seq = u / t.Hkv, g = u % t.Hkv;
        const bool live = grp < (int)t.r;
        const float* qrow = t.q + (size_t(seq) * t.Hq + g * t.r + (live ? grp : 0)) * D;
#pragma unroll
        for (int kk = 0; kk < C::kNK; ++kk) {
            float2 x = make_float2(0.f, 0.f), y = make_float2(0.f, 0.f);
            if (live) {
                x = *reinterpret_cast<const float2*>(qrow + 16 * kk + 2 * qd);
                y = *reinterpret_cast<const float2*>(qrow + 16 * kk + 8 + 2 * qd);
            }
            x.x *= t.qscale; x.y *= t.qscale; y.x *= t.qscale; y.y *= t.qscale;
            const uint32_t xh = ptx::pack_bf16(x.x, x.y), yh = ptx::pack_bf16(y.x, y.y);
            qa[kk][0] = xh;
            qa[kk][1] = ptx::pack_bf16(x.x - ptx::bf16_lo_as_f32(xh), x.y - ptx::bf16_hi_as_f32(xh));
            qa[kk][2] = yh;
            qa[kk][3] = ptx::pack_bf16(y.x - ptx::bf16_lo_as_f32(yh), y.y - ptx::bf16_hi_as_f32(yh));
        }
    };
    auto flush = [&](uint32_t u) {
        float l_tot = l_acc + __shfl_xor_sync(0xffffffffu, l_acc, 1);
        l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 2);
        if (grp < (int)t.r) {
            float* so = sm_o + (cw * kMaxR + grp) * C::kOStride;
#pragma unroll
            for (int nt = 0; nt < 2 * C::kNK; ++nt) {
                so[8 * nt + 2 * qd] = o[nt][0] + o[nt][2];
                so[8 * nt + 2 * qd + 1] = o[nt][1] + o[nt][3];
            }
            if (qd == 0) {
                sm_ml[(cw * kMaxR + grp) * 2] = m_used;
                sm_ml[(cw * kMaxR + grp) * 2 + 1] = l_tot;
            }
        }
        if (ctid == 0) {
            *sm_slot = atomicAdd(&t.slot_count[u], 1u);
            atomicAdd(&t.tokens[u], (unsigned long long)run_tokens);
        }
        ptx::named_bar_sync(1, kCWarps * 32);
        const uint32_t slot = *sm_slot;
        if (slot < t.S) {
            float* P = t.partials + (size_t(u) * t.S + slot) * PS;
            for (uint32_t idx = ctid; idx < t.r * D; idx += kCWarps * 32) {
                const uint32_t h = idx / D, d = idx % D;
                float mx = -INFINITY;
#pragma unroll
                for (int w = 0; w < kCWarps; ++w) mx = fmaxf(mx, sm_ml[(w * kMaxR + h) * 2]);
                float acc = 0.f, lsum = 0.f;
#pragma unroll
                for (int w = 0; w < kCWarps; ++w) {
                    const float sc = ptx::ex2(sm_ml[(w * kMaxR + h) * 2] - mx);
                    acc += sm_o[(w * kMaxR + h) * C::kOStride + d] * sc;
                    lsum += sm_ml[(w * kMaxR + h) * 2 + 1] * sc;
                }
                P[2 * t.r + h * D + d] = acc;
                if (d == 0) {
                    P[h] = mx;
                    P[t.r + h] = lsum;
                }
            }
        } else if (ctid == 0) {
            atomicExch(&t.ws->error, 1u);
        }
        ptx::named_bar_sync(1, kCWarps * 32);
    };

    int stage = 0;
    uint32_t phase = 0;
    for (;;) {
        ptx::mbar_wait(&full[stage], phase);
        const uint32_t unit = meta[stage].unit;
        if (unit == kEnd) break;
        const uint32_t ntok = meta[stage].ntok;
        if (unit != cur) {
            if (cur != kEnd) flush(cur);
            cur = unit;
            run_tokens = 0;
            load_q(unit);
            reset_state();
        }
        run_tokens += ntok;
        const int n = (int)ntok - tb;
        if (n > 0) {
            const uint32_t kbase = ptx::smem_u32(ring + stage * C::kStageBytes);
            const uint32_t vbase = kbase + C::kTileBytes;
            // ---- S = Qhl . K^T  (two 8-token n-tiles, two k-parity chains each)
            float sacc[2][2][4];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 2; ++b) sacc[a][b][0] = sacc[a][b][1] = sacc[a][b][2] = sacc[a][b][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < C::kNK; ++kk) {
                uint32_t b[4];
                ptx::ldsm_x4(b, kbase + swz<D>(k_tok, 2 * kk + k_csel));
                ptx::mma_bf16(sacc[0][kk & 1], qa[kk], b[0], b[1]);
                ptx::mma_bf16(sacc[1][kk & 1], qa[kk], b[2], b[3]);
            }
            float sc[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int nt = j >> 1, col = j & 1;
                const float v = (sacc[nt][0][col] + sacc[nt][1][col]) +
                                (sacc[nt][0][col + 2] + sacc[nt][1][col + 2]);
                const int tok = nt * 8 + 2 * qd + col;
                sc[j] = tok < n ? v : -INFINITY;
            }
            // ---- online softmax (log2 domain), lazy rescale
            float bm = fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3]));
            bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 1));
            bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 2));
            const bool need = bm > m_used + 8.0f;
            if (__any_sync(0xffffffffu, need)) {
                const float m_new = need ? bm : m_used;
                const float alpha = need ? ptx::ex2(m_used - m_new) : 1.0f;
                l_acc *= alpha;
#pragma unroll
                for (int i = 0; i < 2 * C::kNK; ++i) {
                    o[i][0] *= alpha; o[i][1] *= alpha; o[i][2] *= alpha; o[i][3] *= alpha;
                }
                m_used = m_new;
            }
            float p[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) p[j] = ptx::ex2(sc[j] - m_used);
            l_acc += (p[0] + p[1]) + (p[2] + p[3]);
            uint32_t pa[4];
            pa[0] = ptx::pack_bf16(p[0], p[1]);
            pa[1] = ptx::pack_bf16(p[0] - ptx::bf16_lo_as_f32(pa[0]), p[1] - ptx::bf16_hi_as_f32(pa[0]));
            pa[2] = ptx::pack_bf16(p[2], p[3]);
            pa[3] = ptx::pack_bf16(p[2] - ptx::bf16_lo_as_f32(pa[2]), p[3] - ptx::bf16_hi_as_f32(pa[2]));
            // ---- O += Phl . V
#pragma unroll
            for (int nn = 0; nn < C::kNK; ++nn) {
                uint32_t b[4];
                ptx::ldsm_x4_t(b, vbase + swz<D>(v_tok, 2 * nn + v_csel));
                ptx::mma_bf16(o[2 * nn], pa, b[0], b[1]);
                ptx::mma_bf16(o[2 * nn + 1], pa, b[2], b[3]);
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

// ============================================================================
// combine: attention.cpp:159-183 on the device.  grid = (U, r, D/32), block =
// 32 * kCombineGroups: warp sg folds every kCombineGroups-th partial for the
// 32 output dims of this CTA (loads issued before the max is known), then the
// warps are reduced in shared memory.
// mode 0: normalised outputs [B][Hq][D] (Sink units -> bitwise 0,
//         router.cpp:97);
// mode 1: one un-normalised partial per unit ("rank partial", for the NCCL
//         sequence-shard merge), laid out m[r], l[r], acc[r][D];
// Partial j of unit u lives at src + u*unit_stride + j*slot_stride, and the
// slot count is slot_count[u] (fixed_n == 0) or fixed_n.
// ============================================================================
constexpr int kCombineGroups = 8;
constexpr int kCombineUnroll = 19;        // 8 * 19 = 152 >= 148 partial slots in one round trip
constexpr int kCombineMaxWarpSlots = 5;   // 5 * 32 = 160 m values held by warp 0

__global__ void __launch_bounds__(32 * kCombineGroups)
    combine_kernel(DevTables t, const float* __restrict__ src, uint32_t unit_stride,
                   uint32_t slot_stride, uint32_t fixed_n, float* __restrict__ dst, int mode) {
    extern __shared__ float s_w[];  // [n] partial weights
    __shared__ float s_acc[kCombineGroups][33];
    __shared__ float s_l[kCombineGroups];
    __shared__ float s_mx;
    const uint32_t u = blockIdx.x, h = blockIdx.y;
    const uint32_t D = t.D, r = t.r;
    const uint32_t lane = threadIdx.x & 31, sg = threadIdx.x >> 5;
    const uint32_t d = blockIdx.z * 32 + lane;
    const uint32_t seq = u / t.Hkv, g = u % t.Hkv;
    const uint32_t cap_n = fixed_n ? fixed_n : t.S;  // slots that may hold a partial
    const float* base = src + size_t(u) * unit_stride;
    pdl_wait();  // decode partials complete and visible
    // one round trip: flags, count and every candidate partial are fetched
    // together (slots beyond the count hold stale but finite data and are
    // masked below; the partial buffer is zeroed at engine creation)
    const uint32_t flag = __ldcg(&t.unit_flags[u]);
    const uint32_t cnt = fixed_n ? fixed_n : __ldcg(&t.slot_count[u]);
    float vals[kCombineUnroll], ls[kCombineUnroll], mv[kCombineMaxWarpSlots];
#pragma unroll
    for (int k = 0; k < kCombineUnroll; ++k) {
        const uint32_t j = sg + k * kCombineGroups;
        vals[k] = j < cap_n ? __ldcg(base + j * slot_stride + 2 * r + h * D + d) : 0.f;
        ls[k] = j < cap_n ? __ldcg(base + j * slot_stride + r + h) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < kCombineMaxWarpSlots; ++k) {
        const uint32_t j = lane + 32 * k;
        mv[k] = (sg == 0 && j < cap_n) ? __ldcg(base + j * slot_stride + h) : -INFINITY;
    }
    const uint32_t n = (flag & kActive) ? cnt : 0u;
    if (n == 0) {
        if (sg != 0) return;
        if (mode == 0) {
            dst[(size_t(seq) * t.Hq + g * r + h) * D + d] = 0.0f;  // zero surrogate, bitwise +0
        } else {
            float* P = dst + size_t(u) * r * (D + 2);
            if (d == 0) {
                P[h] = -INFINITY;
                P[r + h] = 0.f;
            }
            P[2 * r + h * D + d] = 0.f;
        }
        return;
    }
    // max over the partials' m (warp 0), weights into smem
    if (sg == 0) {
        float mx = -INFINITY;
#pragma unroll
        for (int k = 0; k < kCombineMaxWarpSlots; ++k)
            if (lane + 32 * k < n) mx = fmaxf(mx, mv[k]);
        for (uint32_t j = lane + 32 * kCombineMaxWarpSlots; j < n; j += 32)
            mx = fmaxf(mx, __ldcg(base + j * slot_stride + h));
        for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
#pragma unroll
        for (int k = 0; k < kCombineMaxWarpSlots; ++k) {
            const uint32_t j = lane + 32 * k;
            if (j < n) s_w[j] = mv[k] == -INFINITY ? 0.f : ptx::ex2(mv[k] - mx);
        }
        for (uint32_t j = lane + 32 * kCombineMaxWarpSlots; j < n; j += 32) {
            const float m = __ldcg(base + j * slot_stride + h);
            s_w[j] = m == -INFINITY ? 0.f : ptx::ex2(m - mx);
        }
        if (lane == 0) s_mx = mx;
    }
    __syncthreads();
    float acc = 0.f, lsum = 0.f;
#pragma unroll
    for (int k = 0; k < kCombineUnroll; ++k) {
        const uint32_t j = sg + k * kCombineGroups;
        if (j < n) {
            acc += vals[k] * s_w[j];
            lsum += ls[k] * s_w[j];
        }
    }
    for (uint32_t j = sg + kCombineUnroll * kCombineGroups; j < n; j += kCombineGroups) {
        acc += __ldcg(base + j * slot_stride + 2 * r + h * D + d) * s_w[j];
        lsum += __ldcg(base + j * slot_stride + r + h) * s_w[j];
    }
    s_acc[sg][lane] = acc;
    if (lane == 0) s_l[sg] = lsum;
    __syncthreads();
    if (sg != 0) return;
#pragma unroll
    for (int k = 1; k < kCombineGroups; ++k) {
        acc += s_acc[k][lane];
        lsum += s_l[k];
    }
    if (mode == 0) {
        dst[(size_t(seq) * t.Hq + g * r + h) * D + d] = acc / lsum;
    } else {
        float* P = dst + size_t(u) * r * (D + 2);
        if (d == 0) {
            P[h] = s_mx;
            P[r + h] = lsum;
        }
        P[2 * r + h * D + d] = acc;
    }
}

// ============================================================================
// Cache maintenance kernels (prefill side, not on the step path).
// ============================================================================
// anchor capture from a stored bf16 row (kv_cache.cpp:19-23,71-77):
// k0 = upcast row, k0_norm = (float)sqrt(sum (double)k^2) in index order.
__global__ void anchor_capture_kernel(const __nv_bfloat16* __restrict__ row, uint32_t D,
                                      float* __restrict__ k0, float* __restrict__ k0_norm,
                                      double* __restrict__ norm64) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double s = 0.0;
    for (uint32_t j = 0; j < D; ++j) {
        const float x = __bfloat162float(row[j]);
        k0[j] = x;
        s = __dadd_rn(s, __dmul_rn((double)x, (double)x));
    }
    const double n = __dsqrt_rn(s);
    *norm64 = n;
    *k0_norm = (float)n;
}

// device prefill: f32 rows -> bf16 (RNE) slot rows, 4 elements per thread
__global__ void f32_to_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                   size_t n) {
    const size_t n4 = n / 4;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
         i += (size_t)gridDim.x * blockDim.x) {
        const float4 x = reinterpret_cast<const float4*>(src)[i];
        __nv_bfloat162 a = __floats2bfloat162_rn(x.x, x.y), b = __floats2bfloat162_rn(x.z, x.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&a);
        pk.y = *reinterpret_cast<uint32_t*>(&b);
        reinterpret_cast<uint2*>(dst)[i] = pk;
    }
    for (size_t i = n4 * 4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        dst[i] = __float2bfloat16_rn(src[i]);
}

// One decode token appended to every (seq, kv_head) slot of a layer
// (KvCache::append, kv_cache.cpp:61-84, for the step's new row), stream
// ordered: CTA u writes the f32 rows knew/vnew [U][D] as bf16 (RNE) at row
// len[slot] of slot layer*U + u and advances the device length table.  The
// engine tracks the same lengths on the host (they feed the step's params)
// and keeps first rows (anchor capture, degenerate check) on the host path.
__global__ void append_token_kernel(const float* __restrict__ knew, const float* __restrict__ vnew,
                                    __nv_bfloat16* __restrict__ K, __nv_bfloat16* __restrict__ V,
                                    uint32_t* __restrict__ dlen, uint32_t slot0, uint32_t D,
                                    uint32_t cap) {
    const uint32_t u = blockIdx.x, slot = slot0 + u;
    const uint32_t row = dlen[slot];
    const size_t off = ((size_t)slot * cap + row) * D;
    for (uint32_t j = threadIdx.x; j < D; j += blockDim.x) {
        K[off + j] = __float2bfloat16_rn(knew[(size_t)u * D + j]);
        V[off + j] = __float2bfloat16_rn(vnew[(size_t)u * D + j]);
    }
    __syncthreads();
    if (threadIdx.x == 0) dlen[slot] = row + 1;
}

// synthetic rows: value = bf16(scale * gauss12(key, row*D + j)), the exact
// restatement of oracle/sinkr_oracle.c:orc_fill_rows (counter-based access to
// the reference's SplitMix64 stream, tensor.hpp:15-25).
__device__ __forceinline__ uint64_t sm64_draw(uint64_t key, uint64_t n) {
    uint64_t z = key + (n + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ float gauss12(uint64_t key, uint64_t e) {
    uint64_t s = 0;
#pragma unroll
    for (uint64_t j = 0; j < 6; ++j) {
        const uint64_t h = sm64_draw(key, e * 6 + j);
        s += (h >> 40) + ((h >> 16) & 0xFFFFFFull);
    }
    return (float)__dadd_rn((double)s * 0x1.0p-24, -6.0);
}
__global__ void synth_rows_kernel(__nv_bfloat16* __restrict__ k, __nv_bfloat16* __restrict__ v,
                                  uint64_t key_k, uint64_t key_v, float k_scale, float v_scale,
                                  uint64_t row0, uint64_t rows, uint32_t D) {
    const uint64_t n = rows * D;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t e = row0 * D + i;
        k[i] = __float2bfloat16_rn(__fmul_rn(k_scale, gauss12(key_k, e)));
        v[i] = __float2bfloat16_rn(__fmul_rn(v_scale, gauss12(key_v, e)));
    }
}

// exact bf16 -> f32 upcast (KvCache::historical as a copy)
__global__ void upcast_kernel(const __nv_bfloat16* __restrict__ src, float* __restrict__ dst,
                              uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = __bfloat162float(src[i]);
}

}  // namespace dev
}  // namespace sinkr
