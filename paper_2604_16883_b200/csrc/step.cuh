// step.cuh — the whole SinkRouter decode step in ONE persistent, cooperative
// sm_100a kernel (one CTA per SM):
//
//   phase R  routing (router.cpp:36-75,100-125).  Single-sequence steps: every
//            CTA scores the query heads against the cached token-0 keys itself
//            (no inter-CTA traffic) -- an fp32 estimate decides when every
//            group clears tau by kRouteMargin, else the exact fp64 scores
//            (products exact, sequential sums, IEEE sqrt/div: bit-exact with
//            the reference) decide first.  Batched steps: each CTA scores its
//            share of the groups, one grid barrier.  The exact record (head and
//            group scores) is always published; the Active groups form a work
//            list in every CTA's shared memory.
//   phase S  Split-K flash-decode (attend_chunk, attention.cpp:101-142) over the
//            Active groups only: TMA producer warp + 4 mma.sync consumer warps
//            per CTA, unit-affine guided claims (or guided claims over one
//            global token space when there are more Active groups than SMs).
//   phase M  LSE merge (merge_partials, attention.cpp:159-183): with few Active
//            groups the (group, head, 32-dim) slices are claimed by warps once
//            a group's last row has been counted; with many groups the CTA that
//            streams a group's last rows merges it.  Mode 3 writes the rank
//            partials into every rank's exchange block instead, as LL words
//            tagged with the step, and merges all ranks' partials as soon as
//            their tags show up (no fence, no arrival counter).
//
// The cross-CTA counters come in two sets used by alternate launches (each
// launch zeroes its successor's set), so the launch needs no memset and
// replays as a single graph node.
//
// Instantiations: <D, LEAN, WIDE>.  LEAN = single-sequence shapes (routing
// in every CTA, its scratch in the idle flush staging so the ring is free);
// WIDE = GQA width 9-16 (each consumer warp takes one 8-head tile and 32
// tokens per stage).  Single-sequence steps also (a) let CTA G-1 dry-run the
// stream/flush/merge code before routing so a cold step finds it in L2
// ("code prewarm"), and (b) prefetch each CTA's first static stages into L2
// under the layer's previous Active set while warp 0 routes ("speculative
// prefetch"); both are hints that never change a result.
#pragma once

#include "kernels.cuh"

namespace sinkr {
namespace dev {

constexpr int kMaxUnits = 1280;      // B * H_kv per step (LLaVA-13B B=32 x 40)
constexpr int kMaxStepHeads = 4096;  // B * H_q per step
constexpr int kRouteTile = 64;       // heads per routing tile
constexpr uint32_t kFlatMinTok = 512;  // smallest claim of the global token-space scheduler
// an fp32 estimate of a group score decides the route when it clears tau by
// this much (its own error is ~1e-6); closer calls wait for the exact score
constexpr double kRouteMargin = 1e-4;
constexpr unsigned long long kPrewarmLateNs = 12000;  // a dry pass longer than this ran cold
// a late CTA joins the stream only above this many unclaimed rows (all
// units): ~2 us of the whole grid's stream at 7 TB/s and 512 B per row
constexpr unsigned long long kLateJoinTok = 32768;
// the speculative L2 prefetch runs when the Active rows per CTA reach this
// (64K per unit at 3 of 8 groups Active: 1,328; 32K: 664)
constexpr uint32_t kSpecMinFairTok = 1024;
constexpr uint32_t kMaxEstHeads = 2048;  // distributed form: per-CTA estimate slots (s_score overlay)
// LEAN routing scratch in sm_o (bytes): est [2][64] f32, s_score [64] f64,
// s_degen [64] u8, s_tau [64] f64, s_len [64] u32 (B*H_q <= 64)
constexpr int kLsScore = 512, kLsDegen = 1024, kLsTau = 1088, kLsLen = 1600, kLsBytes = 1856;

// Cross-CTA counters of one step.  Two sets, used by alternate launches
// (parity of the per-CTA launch count, StepTables.cta_epoch): a launch zeroes
// the set its predecessor used, which the next launch will use, so no CTA has
// to restore anything at exit (the per-unit arrays cursor / slot_count /
// tokens_done / ovf are double-buffered the same way).
struct StepCounters {
    unsigned int flat_counter;
    unsigned int merge_next;
    unsigned int exit_count;  // only counted when a last CTA has work (the host completion word)
    unsigned int error;
    unsigned int route_done;  // CTAs that published their units' decisions (distributed routing)
    unsigned int pad[3];
};
struct StepState {
    StepCounters c[2];
    unsigned int pad[8];
};

struct StepTables {
    // TMA descriptors live in global memory (written once at engine creation):
    // keeping 256 B of descriptors out of the parameter block halves the
    // launch latency of this kernel (scripts/micro/launch_cost2.cu)
    const CUtensorMap* tmk;
    const CUtensorMap* tmv;
    const float* q;                // [B][Hq][D]
    const float* anchors;          // [layers][B][Hkv][D]
    const float* anchor_norm;      // [layers][B][Hkv]
    const double* tau_g;           // [B] (when params are not inline)
    const uint32_t* len_g;         // [B]
    double* head_scores;           // result [B*Hq]
    double* group_scores;          // result [U]
    uint32_t* unit_flags;          // result [U]
    uint32_t* route_flags;         // [U] device scratch: decisions for the distributed routing
    uint32_t* route_sum;           // [grid] distributed routing: each CTA's Active bitmask of its units
    unsigned long long* tokens;    // result [U] rows streamed (the skipped-block record)
    uint32_t* status;              // result: nonzero = partial-slot overflow
    StepState* ss;
    uint32_t* cursor;              // [2][U] chunk cursor per active-list entry (two sets: parity)
    uint32_t* slot_count;          // [2][U]
    uint32_t* tokens_done;         // [2][U]
    uint32_t* ovf;                 // [2][U] spill-slot lock (bit0) + valid (bit1)
    uint32_t* cta_epoch;           // [2][grid]: launches seen by each CTA slot (counter-set parity),
                                   // then mode-3 steps seen by each CTA slot (the exchange's step tag)
    float* partials;               // [U][S][r*(D+2)]: m[r], l[r], acc[r][D]
    float* out;                    // mode 0: [B][Hq][D]; mode 1: [U][r][D+2]
    uint32_t B, Hq, Hkv, r, cap, S, mode;  // mode 0 outputs, 1 rank partial, 3 peer merge
    // mode 3 (sequence-sharded peer merge over NVLink): every rank's exchange
    // block holds [2][world][U][r*(D+2)] rank partials (step parity) as LL
    // words {value, step tag} (ptx::st_ll)
    unsigned long long* const* peer_xchg;  // [world] exchange blocks of every rank
    const unsigned long long* xchg_local;  // this rank's block
    uint32_t world, rank;
    float qscale;                  // (1/sqrt(D)) * log2(e)
    uint32_t static_pct;           // static share of the unit-affine schedule (0: one Ck chunk)
    uint32_t prewarm;              // single-sequence steps: the last CTAs dry-run code regions first
    uint32_t* spec_mask;           // [layers] single-sequence steps: Active units of the layer's last step
    uint32_t spec_stages;          // stages of its first static range a CTA prefetches into L2 (0: off)
    unsigned long long* trace;     // optional [grid][4] per-CTA globaltimer stamps
    uint32_t* done;                // optional completion word in mapped host memory (set to 1 last)
};

template <int D>
struct StepCfg {
    using C = Cfg<D>;
    static constexpr int kRing = C::kStages * C::kStageBytes;
    static constexpr int kOffBars = kRing;
    static constexpr int kOffMeta = kOffBars + 2 * C::kStages * 8;
    static constexpr int kOffO = kOffMeta + C::kStages * 16;
    static constexpr int kOffML = kOffO + kCWarps * kMaxR * C::kOStride * 4;
    static constexpr int kOffMisc = kOffML + (kCWarps * kMaxR + kMaxRWide) * 2 * 4;  // + spill staging [16][2]
    static constexpr int kOffAct = kOffMisc + 64;
    static constexpr int kOffPrefix = kOffAct + kMaxUnits * 2;
    static constexpr int kOffLen = kOffPrefix + (kMaxUnits + 1) * 4;
    static constexpr int kBytes = kOffLen + kMaxUnits * 4;
    static constexpr int kSmemBytes = 1024 + kBytes;
    // routing overlay (inside the ring, before streaming starts)
    static constexpr int kDP = D + 1;
    static constexpr int kOvProd = 0;  // q, k0 [2][kRouteTile][D+1] f32 + chains [2][kRouteTile] f64
    static constexpr int kOvScore = (2 * kRouteTile * kDP * 8 + 2 * kRouteTile * 8 + 15) / 16 * 16;
    static constexpr int kOvDegen = kOvScore + kMaxStepHeads * 8;         // [kMaxStepHeads] u8
    static constexpr int kOvSeq = kOvDegen + kMaxStepHeads;             // tau f64 [B], len u32 [B]
    static_assert(kOvSeq + 12 * kMaxUnits <= kRing, "routing overlay exceeds the ring");
    static_assert(kSmemBytes <= 232448, "step kernel shared memory");
    static_assert(kLsBytes <= kCWarps * kMaxR * C::kOStride * 4, "LEAN routing scratch exceeds sm_o");
};

// misc smem words
enum : int { kMiscNact = 0, kMiscChunk, kMiscSlot, kMiscLast, kMiscTask, kMiscFlat, kMiscFast,
             kMiscStatic };

// Unit-affine scheduling: the static first range of a CTA is static_pct % of
// its fair share T/G of the Active tokens (64-token multiple, at least one
// stage); the rest is claimed from per-unit cursors (guided, capped at Ck).
__device__ __forceinline__ uint32_t static_chunk(unsigned long long T, uint32_t G, uint32_t pct,
                                                 uint32_t Ck) {
    if (pct == 0) return Ck;
    unsigned long long c = (T * pct + 100ull * G - 1) / (100ull * G);
    c = (c + kStageTok - 1) / kStageTok * kStageTok;
    return c < (unsigned long long)kStageTok ? (uint32_t)kStageTok : (uint32_t)c;
}


__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
    return *reinterpret_cast<const volatile uint32_t*>(p);
}

// One warp LSE-merges the n Split-K partials of (unit, head h) for the 32
// dims d0 .. d0+31 (merge_partials, attention.cpp:159-183): partials come in
// groups of 64 -- lane j holds (m, l) of partials j, j+32, every lane holds its
// dim of all 64 acc rows, all loads of a group in flight at once -- and the
// weights 2^(m_j - max) reach the lanes by shuffle.  One L2 round trip per 64
// partials.  Writes the normalised row (mode 0), an un-normalised rank partial
// (mode 1), or that partial into every rank's exchange block (mode 3).
// Slots past the count enter warp_merge's FMA chains with weight 0.  A
// non-finite value left there by an earlier step (a NaN query, an inf K/V
// row) would make 0 * x NaN, so a non-finite merge result is recomputed over
// the count's slots only: this step's own non-finite partials stay NaN, an
// earlier step's do not leak into it.  Rare, so out of line.
template <int D, int R>
__device__ __noinline__ float merge_valid_slots(const float* base, uint32_t n, uint32_t h, uint32_t d, float mx) {
    constexpr uint32_t PS = R * (D + 2);
    float acc = 0.f;
    for (uint32_t j = 0; j < n; ++j) {
        const float m = __ldcg(base + size_t(j) * PS + h);
        const float w = m == -INFINITY ? 0.f : ptx::ex2(m - mx);
        acc = fmaf(__ldcg(base + size_t(j) * PS + 2 * R + h * D + d), w, acc);
    }
    return acc;
}

template <int D, int R>
__device__ __forceinline__ void warp_merge(const StepTables& t, uint32_t u, uint32_t h, uint32_t d0,
                                           uint32_t lane, size_t xoff, uint32_t tag, float* wsm, bool dry) {
    // R = t.r at compile time: the partial stride is an immediate, so each of
    // the 64 acc loads is one LDG with an immediate offset.  This loop is cold
    // code at the end of every step, and instruction fetch from DRAM costs
    // (DESIGN.md §4).  Loads past slot_count are unpredicated: the partial
    // block is padded by 64 slots and zero-initialised, every slot holds
    // finite values, and their weights are 0.
    constexpr uint32_t r = R, PS = R * (D + 2);
    // dry: one group over slot 0 (finite, stale) and no stores -- fetches this
    // code into L2 before the real merge needs it
    const uint32_t n = dry ? 1u : min(ld_volatile(&t.slot_count[u]), t.S);
    const float* base = t.partials + size_t(u) * t.S * PS;
    const uint32_t d = d0 + lane;
    float mx = -INFINITY, lsum = 0.f, acc = 0.f;
    for (uint32_t j0 = 0; j0 < n; j0 += 64) {
        float mv[2], lv[2], av[64];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const uint32_t j = j0 + 32 * c + lane;
            mv[c] = j < n ? __ldcg(base + size_t(j) * PS + h) : -INFINITY;
            lv[c] = j < n ? __ldcg(base + size_t(j) * PS + r + h) : 0.f;
        }
        const float* pa = base + size_t(j0) * PS + 2 * r + h * D + d;
#pragma unroll
        for (int k = 0; k < 64; ++k) av[k] = __ldcg(pa + k * PS);
        float cm = fmaxf(mv[0], mv[1]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
        const float nm = fmaxf(mx, cm);
        if (nm != mx) {  // rescale the running sums to the new max
            const float sc = mx == -INFINITY ? 0.f : ptx::ex2(mx - nm);
            acc *= sc;
            lsum *= sc;
            mx = nm;
        }
        float w[2], lw = 0.f;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            w[c] = mv[c] == -INFINITY ? 0.f : ptx::ex2(mv[c] - mx);
            lw += lv[c] * w[c];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lw += __shfl_xor_sync(0xffffffffu, lw, o);
        lsum += lw;
        // the 64 weights reach every lane through the warp's shared scratch
        // (16 broadcast 16-byte loads instead of 64 shuffles: a shorter cold
        // tail), into 4 independent FMA chains
        wsm[lane] = w[0];
        wsm[32 + lane] = w[1];
        __syncwarp();
        float a4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k4 = 0; k4 < 16; ++k4) {
            const float4 wv = reinterpret_cast<const float4*>(wsm)[k4];
            a4[0] = fmaf(av[4 * k4], wv.x, a4[0]);
            a4[1] = fmaf(av[4 * k4 + 1], wv.y, a4[1]);
            a4[2] = fmaf(av[4 * k4 + 2], wv.z, a4[2]);
            a4[3] = fmaf(av[4 * k4 + 3], wv.w, a4[3]);
        }
        acc += (a4[0] + a4[1]) + (a4[2] + a4[3]);
        __syncwarp();  // scratch reused by the next group / task
    }
    if (dry) return;
    if (!isfinite(acc)) acc = merge_valid_slots<D, R>(base, n, h, d, mx);
    if (t.mode == 0) {
        t.out[(size_t(u) * r + h) * D + d] = acc / lsum;
    } else if (t.mode == 1) {
        float* P = t.out + size_t(u) * PS;
        if (d == 0) {
            P[h] = mx;
            P[r + h] = lsum;
        }
        P[2 * r + h * D + d] = acc;
    } else {  // mode 3: this rank's partial straight into every rank's exchange block
        // as LL words tagged with the step: no fence, no arrival counter --
        // an owner that reads the tag reads the value (one 8-byte store)
        for (uint32_t q = 0; q < t.world; ++q) {
            unsigned long long* P = t.peer_xchg[q] + xoff + size_t(u) * PS;
            if (d == 0) {
                ptx::st_ll(P + h, mx, tag);
                ptx::st_ll(P + r + h, lsum, tag);
            }
            ptx::st_ll(P + 2 * r + h * D + d, acc, tag);
        }
    }
}

// warp_merge for the runtime GQA width (WIDE kernels: 9 <= r <= 16)
template <int D, bool WIDE>
__device__ __forceinline__ void warp_merge_r(const StepTables& t, uint32_t u, uint32_t h, uint32_t d0,
                                             uint32_t lane, size_t xoff, uint32_t tag, float* wsm,
                                             bool dry = false) {
    if constexpr (WIDE) {
        switch (t.r) {
            case 9: warp_merge<D, 9>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
            case 10: warp_merge<D, 10>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
            case 11: warp_merge<D, 11>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
            case 12: warp_merge<D, 12>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
            case 13: warp_merge<D, 13>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
            case 14: warp_merge<D, 14>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
            case 15: warp_merge<D, 15>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
            default: warp_merge<D, 16>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
        }
        return;
    }
    switch (t.r) {
        case 1: warp_merge<D, 1>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
        case 2: warp_merge<D, 2>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
        case 3: warp_merge<D, 3>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
        case 4: warp_merge<D, 4>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
        case 5: warp_merge<D, 5>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
        case 6: warp_merge<D, 6>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
        case 7: warp_merge<D, 7>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
        default: warp_merge<D, 8>(t, u, h, d0, lane, xoff, tag, wsm, dry); break;
    }
}

// A step-kernel error: kept in the launch's counter set and stored straight
// into the result block's status word (zeroed by CTA 0 at launch; every error
// source is a >= 2 s watchdog or CTA 0 itself, so the zeroing comes first).
__device__ __forceinline__ void raise_error(const StepTables& t, StepCounters* sc, uint32_t code) {
    atomicExch(&sc->error, code);
    *reinterpret_cast<volatile uint32_t*>(t.status) = code;
}

// LEAN: the single-sequence instantiation (B*H_q <= 64, B*H_kv <= 32: every
// single-sequence shape of the configs) -- estimate-first routing in every CTA,
// unit-affine scheduling; the distributed routing, the global-token-space
// scheduler and their exact record are compiled out, so the binary a step
// fetches (cold, from DRAM, at the start of every step in a model) is smaller.
// The engine picks the instantiation once, from its shape (engine.cu step_fn).
// WIDE: GQA width 9-16 (e.g. 128 q / 8 kv heads): consumer warp cw takes the
// head half cw & 1 (two 8-head hi/lo MMA tiles per group) and 32 tokens of
// each stage as two 16-token sub-tiles, so every warp keeps one 8-head tile
// of online-softmax state and the per-stage work is unchanged.
template <int D, bool LEAN, bool WIDE>
__global__ void __launch_bounds__(kThreads, 1)
    step_kernel(const StepTables t_in, const ProbeParams p) {
    using C = Cfg<D>;
    using SC = StepCfg<D>;
    using Scan = cub::BlockScan<uint32_t, kThreads>;
    using Reduce = cub::BlockReduce<unsigned long long, kThreads>;
    __shared__ union {
        typename Scan::TempStorage scan;
        typename Reduce::TempStorage reduce;
    } tmp;
    __shared__ unsigned long long s_tok_total;

    extern __shared__ __align__(16) uint8_t smem_raw[];
    // 1024-B alignment for the 128B-swizzled TMA tiles, by offsetting the
    // shared array itself so the compiler keeps shared-space (LDS/STS) access
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + SC::kOffBars);
    uint64_t* empty = full + C::kStages;
    StageMeta* meta = reinterpret_cast<StageMeta*>(smem + SC::kOffMeta);
    float* sm_o = reinterpret_cast<float*>(smem + SC::kOffO);
    float* sm_ml = reinterpret_cast<float*>(smem + SC::kOffML);
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + SC::kOffMisc);
    uint16_t* act_unit = reinterpret_cast<uint16_t*>(smem + SC::kOffAct);
    uint32_t* act_prefix = reinterpret_cast<uint32_t*>(smem + SC::kOffPrefix);
    uint32_t* act_len = reinterpret_cast<uint32_t*>(smem + SC::kOffLen);  // rows per Active entry
    // routing scratch: the single-sequence (LEAN) form keeps its ~2 KB in the
    // flush staging sm_o (idle until the first flush), so the ring stays free
    // during routing; the distributed form overlays the ring
    uint8_t* const ls = reinterpret_cast<uint8_t*>(sm_o);
    double* s_score = LEAN ? reinterpret_cast<double*>(ls + kLsScore) : reinterpret_cast<double*>(ring + SC::kOvScore);
    uint8_t* s_degen = LEAN ? ls + kLsDegen : ring + SC::kOvDegen;
    double* s_tau = LEAN ? reinterpret_cast<double*>(ls + kLsTau) : reinterpret_cast<double*>(ring + SC::kOvSeq);  // [B]
    uint32_t* s_len = LEAN ? reinterpret_cast<uint32_t*>(ls + kLsLen)
                           : reinterpret_cast<uint32_t*>(ring + SC::kOvSeq + 8 * kMaxUnits);  // [B]

    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t G = gridDim.x, bid = blockIdx.x;
    const uint32_t U = t_in.B * t_in.Hkv, NH = t_in.B * t_in.Hq, r = t_in.r;
    // prologue that touches no memory the previous kernel may write: with a
    // programmatic (PDL) launch it runs while the previous step drains
    if (tid == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], kCWarps);
        }
        ptx::fence_mbar_init();
        ptx::tma_prefetch_desc(t_in.tmk);
        ptx::tma_prefetch_desc(t_in.tmv);
    }
    pdl_wait();              // no-op unless launched with programmatic serialization
    pdl_launch();  // the next step's CTAs may take SMs as this grid's CTAs exit
    // counter-set parity: every CTA of a launch reads the same count (the
    // grid is fixed per engine and CTA b's count is written only by CTA b,
    // after its final barrier); this launch uses set `par` and zeroes the
    // other, which the previous launch used and the next one will use
    const uint32_t cta_ep = ld_volatile(&t_in.cta_epoch[bid]), par = cta_ep & 1u;
    StepTables t = t_in;
    t.cursor += par * U;
    t.slot_count += par * U;
    t.tokens_done += par * U;
    t.ovf += par * U;
    StepCounters* const sc = &t_in.ss->c[par];
    {
        const uint32_t oth = (par ^ 1u) * U;
        for (uint32_t i = bid * kThreads + tid; i < U; i += G * kThreads) {
            t_in.cursor[oth + i] = 0u;
            t_in.slot_count[oth + i] = 0u;
            t_in.tokens_done[oth + i] = 0u;
            t_in.ovf[oth + i] = 0u;
        }
        if (bid == 0 && tid == 0) {
            StepCounters* o = &t_in.ss->c[par ^ 1u];
            o->flat_counter = o->merge_next = o->exit_count = o->error = o->route_done = 0u;
            *t.status = 0u;  // (errors are raised by watchdogs >= 2 s later, or by this CTA)
        }
    }
    const uint32_t layer = p.layer, flags = p.flags;
    const bool lead = bid == 0;
    unsigned long long* clk = reinterpret_cast<unsigned long long*>(t.status + 4);
    if (lead && tid == 0) clk[0] = globaltimer();
    if (t.trace && tid == 0) t.trace[bid * 8 + 4] = globaltimer();
    unsigned long long* dbg = clk + 4;  // debug cycle stamps (lead CTA, thread 0)
#define STAMP(i) do { if (lead && tid == 0) dbg[i] = clock64(); } while (0)
    STAMP(0);
    STAMP(1);
    // Code prewarm (single-sequence steps).  A decode step in a model runs
    // with a cold L2, so every code region a step enters for the first time
    // is fetched from DRAM -- by all 148 SMs at once, on the critical path
    // (cold code).  The last CTA(s) first run code regions DRY
    // (no waits, no claims, no stores): one consumer iteration over stale
    // shared memory, one flush, one merge task per warp over slot 0.  That
    // brings the regions' code into L2 while the other CTAs route; the dry
    // CTAs then route and stream on dynamic claims only (no static range), so
    // their late start costs no tail.  The dry and the real pass are one loop
    // over the same code, so they execute the same instructions.  Default
    // (engine): all three regions in CTA G-1 -- splitting them over three
    // CTAs fetched faster but cost 2.5 us back to back at 512K
    // (profiles/r02_prewarm_ab.txt).
    // t.prewarm: bit mask of the regions (bit 0 consumer body, 1 flush, 2
    // merge), the k-th set bit to CTA G-1-k; bit 3: all three in CTA G-1;
    // bits 8+: the cold-pass threshold in us (A/B; 0 = kPrewarmLateNs)
    const uint32_t pw_mask = (LEAN && G >= 64u) ? (t.prewarm & 15u) : 0u;
    const uint32_t n_pw = (pw_mask & 8u) ? 1u : __popc(pw_mask);
    const bool pw_on = n_pw != 0u;
    const bool prewarm = pw_on && bid >= G - n_pw;
    uint32_t dry_regions = 0;  // prewarm CTAs: bit 0 consumer body, 1 flush, 2 merge
    if (prewarm) {
        uint32_t m = pw_mask;
        for (uint32_t k = G - 1u - bid; k > 0; --k) m &= m - 1u;
        dry_regions = (pw_mask & 8u) ? 7u : 1u << (__ffs(m) - 1);
    }
    unsigned long long t_stream_end = 0;
    const unsigned long long t_cta_start = prewarm ? globaltimer() : 0ull;
    constexpr bool lean = LEAN;
    bool exact_later = false;  // distributed form: exact record after streaming starts
    // mode 3: this CTA slot's mode-3 step count (the same in every CTA) tags
    // the exchange words of this step
    const uint32_t epoch = t.mode == 3 ? ld_volatile(&t.cta_epoch[G + bid]) : 0u;
    uint32_t nact = 0, Ck = 0, Cs = 0;
    bool flat = false, queue_mode = true, lean_fast = false;
    size_t xoff = 0;
#pragma unroll 1
    for (uint32_t pass = prewarm ? 0u : 1u; pass < 2u; ++pass) {
    const bool dry = pass == 0u;
    if (!dry) {
    // per-sequence tau / length into smem once (no dynamic indexing of the
    // parameter block in the loops below; after the dry pass, which uses sm_o)
    if (p.inline_seqs) {
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < kParamSeqs; ++k) {  // compile-time indices: plain LDC
                s_tau[k] = p.tau[k];
                s_len[k] = p.len[k];
            }
        }
    } else {
        for (uint32_t sq = tid; sq < t.B; sq += kThreads) {
            s_tau[sq] = __ldg(&t.tau_g[sq]);
            s_len[sq] = __ldg(&t.len_g[sq]);
        }
    }
    // ======================= phase R: routing ================================
    // proxy_score (router.cpp:36-48), group_score (50-57), route (67-75) and the
    // task build (131-145).  Two forms with identical results:
    //  * lean (B*H_q <= 64, B*H_kv <= 32: every single-sequence shape): all
    //    warps form the exact fp64 products (a product of two floats is exact
    //    in fp64, so s + p is bit-identical to the reference's
    //    `s += (double)q[i] * k0[i]`); thread h then runs its head's dot and
    //    |q|^2 chains interleaved (sequential DADDs in index order: ~8 cycles
    //    each, the floor of this phase) and scores it.  Warp 0 routes one unit
    //    per lane and builds the Active list with a ballot: two block barriers
    //    in all, and a short code path (the phase is latency bound).
    //  * distributed (batched steps): each CTA scores its share of the units,
    //    one grid barrier, then every CTA scans the published decisions.
    if (lean) {
        // Fast decision first: an fp32 estimate of every head score (warp
        // dot products of the rows already in registers).  If every group's
        // estimate clears tau by kRouteMargin -- far above the estimate's
        // error of ~1e-6 -- the decisions are exact already and streaming
        // starts now; the lead CTA's consumer warps then compute the exact
        // fp64 scores for the record (and check the decisions) while their
        // first stages are in flight.  Otherwise the exact scores come first:
        // all warps form the exact fp64 products (a product of two floats is
        // exact in fp64, so s + p is bit-identical to the reference's
        // `s += (double)q[i] * k0[i]`), thread h runs its head's dot and |q|^2
        // chains (sequential DADDs in index order), and warp 0 routes.
        float* est = reinterpret_cast<float*>(ls);  // [2][kRouteTile] fp32 dot, |q|^2
        // the layer's previous Active set (speculative prefetch below), loaded
        // by the thread that issues the prefetch while warp 0 routes
        const bool spec = t.spec_stages && p.inline_seqs && bid != 0 && !prewarm && warp == 1;
        const uint32_t smask = spec ? ld_volatile(&t.spec_mask[layer]) : 0u;
        constexpr int kW = kThreads / 32;
        constexpr int kHPW = (kRouteTile + kW - 1) / kW;
        constexpr int kV = D / 32;
        float qv[kHPW][kV], kv[kHPW][kV];
        // warp 0 lane u: k0_norm of unit u, loaded with the rows (off the
        // decision's critical path)
        const float kn_lane = (warp == 0 && lane < U)
                                  ? ptx::ldg_last(&t.anchor_norm[size_t(layer) * U + lane], ptx::policy_evict_last())
                                  : 1.f;
        {
            const uint64_t keep = ptx::policy_evict_last();
            const uint32_t rmagic = 0xFFFFFFFFu / r + 1u;  // i / r == umulhi(i, rmagic) for i < 2^16
            const float* kbase = t.anchors + size_t(layer) * U * D + kV * lane;
#pragma unroll
            for (int a = 0; a < kHPW; ++a) {
                const uint32_t h = min(warp + a * kW, NH - 1);
                const float* qrow = t.q + size_t(h) * D + kV * lane;
                const float* krow = kbase + size_t(r == 1 ? h : __umulhi(h, rmagic)) * D;
                if constexpr (kV == 4) {
                    const float4 x = ptx::ldg_last4(qrow, keep);
                    const float4 y = ptx::ldg_last4(krow, keep);
                    qv[a][0] = x.x; qv[a][1] = x.y; qv[a][2] = x.z; qv[a][3] = x.w;
                    kv[a][0] = y.x; kv[a][1] = y.y; kv[a][2] = y.z; kv[a][3] = y.w;
                } else if constexpr (kV == 2) {
                    const float2 x = ptx::ldg_last2(qrow, keep);
                    const float2 y = ptx::ldg_last2(krow, keep);
                    qv[a][0] = x.x; qv[a][1] = x.y;
                    kv[a][0] = y.x; kv[a][1] = y.y;
                } else {
                    qv[a][0] = ptx::ldg_last(qrow, keep);
                    kv[a][0] = ptx::ldg_last(krow, keep);
                }
            }
            if (tid == 0) STAMP(13);
#pragma unroll
            for (int a = 0; a < kHPW; ++a) {
                const uint32_t h = warp + a * kW;
                float d = 0.f, qq = 0.f;
#pragma unroll
                for (int e = 0; e < kV; ++e) {
                    d = fmaf(qv[a][e], kv[a][e], d);
                    qq = fmaf(qv[a][e], qv[a][e], qq);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    d += __shfl_xor_sync(0xffffffffu, d, o);
                    qq += __shfl_xor_sync(0xffffffffu, qq, o);
                }
                if (lane == 0 && h < NH) {
                    est[h] = d;
                    est[kRouteTile + h] = qq;
                }
            }
        }
        __syncthreads();
        STAMP(15);
        // Speculative L2 prefetch of this CTA's first static range under the
        // layer's previous Active set (sink heads are stable across decode
        // steps), issued by warp 1 (a box per lane) while warp 0 routes: DRAM streams
        // during the rest of routing and the first stages come from L2.  A
        // hint only -- the plan comes from this step's routing; a changed set
        // costs a few idle-time DRAM reads, never a result.  (Issued together
        // with the routing loads, the prefetches delayed them: +1.7 us at 32K.)
        if (spec) {
            const uint32_t ns = __popc(smask);
            if (ns != 0u && bid < G - n_pw) {
                uint32_t T = 0, u = 0;
                const uint32_t a = bid % ns;
                uint32_t m = smask;
                for (uint32_t i = 0; m; ++i, m &= m - 1u) {
                    const uint32_t uu = __ffs(m) - 1;
                    T += s_len[uu / t.Hkv];
                    if (i == a) u = uu;
                }
                // long steps only: at 32K per unit the prefetches cost more than
                // they hide (+0.7 us back to back, +1.4 L2-flushed)
                const bool go = T >= G * kSpecMinFairTok;
                // the chunk plan route_units builds (below) for this set
                const uint32_t gdiv = G * kChunksPerCta;
                uint32_t cc = (T + gdiv - 1) / gdiv;
                cc = (cc + kStageTok - 1) / kStageTok * kStageTok;
                const uint32_t Cs = static_chunk(T, G, t.static_pct, cc < kMinChunkTok ? kMinChunkTok : cc);
                const uint32_t L = s_len[u / t.Hkv];
                const uint32_t t0 = (bid / ns - (a == 0 ? 1u : 0u)) * Cs;
                const uint32_t t1 = min(min(t0 + Cs, L), t0 + t.spec_stages * (uint32_t)kStageTok);
                const int32_t row0 = (int32_t)((size_t(layer) * U + u) * t.cap);
                // one box per lane (every lane of warp 1 computed the plan)
                const uint32_t nbox = go && t1 > t0 ? (t1 - t0 + kStageTok - 1) / kStageTok * 2 * C::kHalves : 0u;
                for (uint32_t i = lane; i < nbox; i += 32) {
                    const uint32_t st = i / (2 * C::kHalves), hf = (i / 2) % C::kHalves;
                    ptx::tma_prefetch_l2_2d((i & 1) ? t.tmv : t.tmk, (int32_t)hf * C::kBoxDim,
                                            row0 + (int32_t)(t0 + st * kStageTok));
                }
            }
        }

        // warp 0: one unit per lane -> decisions (from the estimates, or from the
        // exact scores on the second pass), then the Active list by ballot
        auto route_units = [&](bool exact) -> bool {
            const uint32_t u = lane;
            bool active = false, certain = true;
            uint32_t L = 0;
            if (u < U) {
                const uint32_t seq = u / t.Hkv;
                const double tau = s_tau[seq];
                double S;
                uint32_t degen = 0;
                if (exact) {
                    double sum = 0.0;
                    for (uint32_t i = 0; i < r; ++i) {
                        sum = __dadd_rn(sum, s_score[u * r + i]);
                        degen |= s_degen[u * r + i];
                    }
                    // sum / r (router.cpp:56); for power-of-two r the product
                    // with 1/r is the same correctly rounded value
                    S = (r & (r - 1)) == 0 ? __dmul_rn(sum, 1.0 / (double)r) : __ddiv_rn(sum, (double)r);
                } else {
                    // fast-math estimate (rsqrt, reciprocal): its error stays far
                    // below kRouteMargin
                    const float inv_kn = __frcp_rn(kn_lane);
                    float sum = 0.f;
                    for (uint32_t i = 0; i < r; ++i) {
                        const float qq = est[kRouteTile + u * r + i];
                        certain &= qq > 1e-20f;  // near-degenerate query: decide exactly
                        sum += qq > 0.f ? est[u * r + i] * rsqrtf(qq) * inv_kn : 0.f;
                    }
                    const float Sf = sum * __frcp_rn((float)r);
                    certain &= fabsf(Sf - (float)tau) > (float)kRouteMargin;
                    S = (double)Sf;
                }
                const bool over = (flags & kSinkOnTie) ? (S >= tau) : (S > tau);
                bool sink = over && !(flags & kLayerExcluded);
                if (degen) sink = false;  // router.cpp:114-117 fail-safe toward exact
                active = (flags & kObserveOnly) || !sink;
                if ((flags & kObserveOnly) || (flags & kLayerExcluded) || p.only_unit) certain = true;
                force_route(p.only_unit, u, sink, active);
                L = s_len[seq];
                if (!exact) act_prefix[u] = active ? 1u : 0u;  // estimate decisions, checked later
                if (lead && exact) {  // (fast path: the consumers publish the record)
                    t.group_scores[u] = S;
                    t.unit_flags[u] =
                        (sink ? kSink : 0u) | (degen ? kDegenerate : 0u) | (active ? kActive : 0u);
                    if (!active) {
                        t.tokens[u] = 0ull;
                        if (t.mode == 1) {  // rank partial of a skipped group: empty
                            float* P = t.out + size_t(u) * r * (D + 2);
                            for (uint32_t h = 0; h < r; ++h) {
                                P[h] = -INFINITY;
                                P[r + h] = 0.f;
                            }
                            for (uint32_t k = 0; k < r * D; ++k) P[2 * r + k] = 0.f;
                        }
                    }
                }
            }
            if (!exact && !__all_sync(0xffffffffu, certain)) return false;
            const uint32_t mask = __ballot_sync(0xffffffffu, active);
            const uint32_t nact = __popc(mask);
            const uint32_t pos = __popc(mask & ((1u << lane) - 1u));
            if (active) {
                act_unit[pos] = (uint16_t)u;
                act_len[pos] = L;
            }
            // chunk size from the Active token total (32-bit: U <= 32 slots)
            uint32_t T = active ? L : 0u;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) T += __shfl_xor_sync(0xffffffffu, T, o);
            if (lane == 0) {
                const uint32_t gdiv = G * kChunksPerCta;
                uint32_t cc = (T + gdiv - 1) / gdiv;
                cc = (cc + kStageTok - 1) / kStageTok * kStageTok;
                misc[kMiscNact] = nact;
                misc[kMiscChunk] = cc < kMinChunkTok ? kMinChunkTok : cc;
                misc[kMiscStatic] = static_chunk(T, G, t.static_pct, misc[kMiscChunk]);
                misc[kMiscFlat] = 0u;  // U <= 32 < #SMs: unit-affine scheduling
                if (lead && t.spec_stages) t.spec_mask[layer] = mask;  // the next step's guess
            }
            return true;
        };
        if (warp == 0) {
            const bool fast = route_units(false);
            if (lane == 0) misc[kMiscFast] = fast ? 1u : 0u;
        }
        STAMP(14);
        __syncthreads();
        STAMP(16);
        if (!misc[kMiscFast]) {
            // exact scores before any decision: thread h runs its head's dot
            // and |q|^2 chains over its q row and its group's k0 row (in L2:
            // the estimate just loaded them), the products exact in fp64 off
            // the chain, each a sequential fp64 sum in index order
            // (router.cpp:40-43) -- no shared-memory staging, so the ring
            // stays free for the speculative stages
            if (tid < NH) {
                const uint32_t u = tid / r;
                const float4* qrow = reinterpret_cast<const float4*>(t.q + size_t(tid) * D);
                const float4* krow = reinterpret_cast<const float4*>(t.anchors + (size_t(layer) * U + u) * D);
                const float kn = ptx::ldg_last(&t.anchor_norm[size_t(layer) * U + u], ptx::policy_evict_last());
                double dot = 0.0, qq = 0.0;
#pragma unroll 8
                for (int c = 0; c < D / 4; ++c) {
                    const float4 x = __ldg(qrow + c), y = __ldg(krow + c);
                    const float qf[4] = {x.x, x.y, x.z, x.w}, kf[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const double qd = (double)qf[e];
                        dot = __dadd_rn(dot, __dmul_rn(qd, (double)kf[e]));
                        qq = __dadd_rn(qq, __dmul_rn(qd, qd));
                    }
                }
                const double qn = __dsqrt_rn(qq);
                double sc = 0.0;
                uint8_t dg = 0;
                if (qn < 1e-12) {
                    dg = 1;
                } else {
                    sc = __ddiv_rn(dot, __dmul_rn(qn, (double)kn));
                    sc = sc < -1.0 ? -1.0 : (1.0 < sc ? 1.0 : sc);  // std::clamp
                }
                s_score[tid] = sc;
                s_degen[tid] = dg;
                if (lead) t.head_scores[tid] = sc;
            }
            __syncthreads();  // scores visible
            if (warp == 0) route_units(true);
        }
        STAMP(3);
    } else {
        // distributed (batched steps): CTA c scores units [u_lo, u_hi) -- all r
        // heads of each, so it also takes their group means and decisions --
        // publishes them, and after one grid barrier every CTA builds the Active
        // list from the published decisions.  Head i belongs to unit i / r.  The
        // exact fp64 products of 64-head tiles are staged in smem; then thread h
        // runs the dot chain and thread 64+h the |q|^2 chain, each a sequential
        // fp64 sum in index order.
        const uint32_t up = (U + G - 1) / G;
        const uint32_t u_lo = min(U, bid * up), u_hi = min(U, u_lo + up);
        const uint32_t h_lo = u_lo * r, h_hi = u_hi * r;
        // fp32 estimates of this CTA's head scores first (warp dot products);
        // if all its groups clear tau by kRouteMargin the decisions are
        // published now and the exact fp64 record is computed by the consumer
        // warps after streaming starts (as in the lean form)
        {
            float* est = reinterpret_cast<float*>(s_score);  // [2][kMaxEstHeads]
            constexpr int kV = D / 32;
            const uint64_t keep = ptx::policy_evict_last();
            for (uint32_t h = h_lo + warp; h < h_hi; h += kThreads / 32) {
                const float* qrow = t.q + size_t(h) * D + kV * lane;
                const float* krow = t.anchors + (size_t(layer) * U + h / r) * D + kV * lane;
                float d = 0.f, qq = 0.f;
#pragma unroll
                for (int e = 0; e < kV; ++e) {
                    const float x = ptx::ldg_last(qrow + e, keep), y = ptx::ldg_last(krow + e, keep);
                    d = fmaf(x, y, d);
                    qq = fmaf(x, x, qq);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    d += __shfl_xor_sync(0xffffffffu, d, o);
                    qq += __shfl_xor_sync(0xffffffffu, qq, o);
                }
                if (lane == 0) {
                    est[h - h_lo] = d;
                    est[kMaxEstHeads + h - h_lo] = qq;
                }
            }
            __syncthreads();
            bool certain = true;
            for (uint32_t u = u_lo + tid; u < u_hi; u += kThreads) {
                const float inv_kn = __frcp_rn(__ldg(&t.anchor_norm[size_t(layer) * U + u]));
                const uint32_t hb = (u - u_lo) * r;
                float sum = 0.f;
                for (uint32_t i = 0; i < r; ++i) {
                    const float qq = est[kMaxEstHeads + hb + i];
                    certain &= qq > 1e-20f;
                    sum += qq > 0.f ? est[hb + i] * rsqrtf(qq) * inv_kn : 0.f;
                }
                const float Sf = sum * __frcp_rn((float)r);
                const double tau = s_tau[u / t.Hkv];
                certain &= fabsf(Sf - (float)tau) > (float)kRouteMargin ||
                           (flags & (kObserveOnly | kLayerExcluded)) != 0;
                if (p.only_unit) certain = true;  // forced route: scores only for the record
                s_score[kMaxEstHeads + (u - u_lo)] = (double)Sf;  // estimate, for the decision below
            }
            exact_later = __syncthreads_and(certain) != 0 && (h_hi - h_lo) <= (uint32_t)(kThreads - 32);
        }
        STAMP(15);
        if (!exact_later) {
            double* sq = reinterpret_cast<double*>(ring + SC::kOvProd);  // [kRouteTile][D+1] f64
            double* sk = sq + kRouteTile * SC::kDP;
            double* s_chain = sk + kRouteTile * SC::kDP;  // [2][kRouteTile]
            for (uint32_t h_base = h_lo; h_base < h_hi; h_base += kRouteTile) {
                const uint32_t nh = min((uint32_t)kRouteTile, h_hi - h_base);
                // warp w loads heads w, w+5, ...; lane l loads kV = D/32 consecutive
                // floats of the row with one vector load.  The products go to smem
                // rows of odd stride (D+1 doubles, conflict-free for the chains)
                // with a lane-rotated element order, so the stores are conflict-free
                // as well.
                constexpr int kW = kThreads / 32;
                constexpr int kHPW = (kRouteTile + kW - 1) / kW;
                constexpr int kV = D / 32;
                float qv[kHPW][kV], kv[kHPW][kV];
                const uint64_t keep = ptx::policy_evict_last();
#pragma unroll
                for (int a = 0; a < kHPW; ++a) {
                    const uint32_t hl = warp + a * kW;
                    const bool ok = hl < nh;
                    const uint32_t i = h_base + (ok ? hl : 0);
                    const float* qrow = t.q + size_t(i) * D + kV * lane;
                    const float* krow = t.anchors + (size_t(layer) * U + i / r) * D + kV * lane;
                    if constexpr (kV == 4) {
                        float4 x = make_float4(0.f, 0.f, 0.f, 0.f), y = x;
                        if (ok) {
                            x = ptx::ldg_last4(qrow, keep);
                            y = ptx::ldg_last4(krow, keep);
                        }
                        qv[a][0] = x.x; qv[a][1] = x.y; qv[a][2] = x.z; qv[a][3] = x.w;
                        kv[a][0] = y.x; kv[a][1] = y.y; kv[a][2] = y.z; kv[a][3] = y.w;
                    } else if constexpr (kV == 2) {
                        float2 x = make_float2(0.f, 0.f), y = x;
                        if (ok) {
                            x = ptx::ldg_last2(qrow, keep);
                            y = ptx::ldg_last2(krow, keep);
                        }
                        qv[a][0] = x.x; qv[a][1] = x.y;
                        kv[a][0] = y.x; kv[a][1] = y.y;
                    } else {
                        qv[a][0] = ok ? ptx::ldg_last(qrow, keep) : 0.f;
                        kv[a][0] = ok ? ptx::ldg_last(krow, keep) : 0.f;
                    }
                }
                double kn = 1.0;
                if (tid < nh)
                    kn = (double)ptx::ldg_last(&t.anchor_norm[size_t(layer) * U + (h_base + tid) / r], keep);
                // exact fp64 products (f32 x f32 fits in 53 bits), off the chain
#pragma unroll
                for (int a = 0; a < kHPW; ++a) {
                    const uint32_t hl = warp + a * kW;
                    if (hl < nh) {
#pragma unroll
                        for (int e = 0; e < kV; ++e) {
                            const uint32_t idx = (e + lane) % kV;
                            float qf = qv[a][0], kf = kv[a][0];
#pragma unroll
                            for (int c = 1; c < kV; ++c)
                                if (idx == (uint32_t)c) {
                                    qf = qv[a][c];
                                    kf = kv[a][c];
                                }
                            const double qd = (double)qf;
                            sq[hl * SC::kDP + kV * lane + idx] = __dmul_rn(qd, (double)kf);
                            sk[hl * SC::kDP + kV * lane + idx] = __dmul_rn(qd, qd);
                        }
                    }
                }
                __syncthreads();
                if (tid < 2 * kRouteTile && (tid % kRouteTile) < nh) {
                    const uint32_t hl = tid % kRouteTile;
                    // thread h: the dot chain; thread 64+h: the |q|^2 chain, each a
                    // sequential sum in index order (router.cpp:40-43)
                    const double* a = (tid < (uint32_t)kRouteTile ? sq : sk) + hl * SC::kDP;
                    double acc = 0.0;
#pragma unroll 16
                    for (uint32_t j = 0; j < D; ++j) acc = __dadd_rn(acc, a[j]);
                    s_chain[tid] = acc;
                }
                __syncthreads();
                if (tid < nh) {
                    const double dot = s_chain[tid], qsq = s_chain[kRouteTile + tid];
                    const double qn = __dsqrt_rn(qsq);
                    double sc = 0.0;
                    uint8_t dg = 0;
                    if (qn < 1e-12) {
                        dg = 1;
                    } else {
                        sc = __ddiv_rn(dot, __dmul_rn(qn, kn));
                        sc = sc < -1.0 ? -1.0 : (1.0 < sc ? 1.0 : sc);  // std::clamp
                    }
                    s_score[h_base - h_lo + tid] = sc;
                    s_degen[h_base - h_lo + tid] = dg;
                }
                __syncthreads();
            }
        }  // !exact_later

        // group_score + route (router.cpp:50-57,67-75,113-120) of this CTA's units
        bool my_act = false;  // (up <= 32: thread i decides unit u_lo + i)
        for (uint32_t u = u_lo + tid; u < u_hi; u += kThreads) {
            const uint32_t seq = u / t.Hkv;
            const uint32_t hb = (u - u_lo) * r;
            double S;
            uint32_t degen = 0;
            if (exact_later) {
                S = s_score[kMaxEstHeads + (u - u_lo)];  // the estimate: it cleared the margin
            } else {
                double sum = 0.0;
                for (uint32_t i = 0; i < r; ++i) {
                    sum = __dadd_rn(sum, s_score[hb + i]);
                    degen |= s_degen[hb + i];
                }
                // sum / r (router.cpp:56); for power-of-two r the product with
                // 1/r is the same correctly rounded value
                S = (r & (r - 1)) == 0 ? __dmul_rn(sum, 1.0 / (double)r) : __ddiv_rn(sum, (double)r);
            }
            const double tau = s_tau[seq];
            const bool over = (flags & kSinkOnTie) ? (S >= tau) : (S > tau);
            bool sink = over && !(flags & kLayerExcluded);
            if (degen) sink = false;  // router.cpp:114-117 fail-safe toward exact
            bool active = (flags & kObserveOnly) || !sink;
            force_route(p.only_unit, u, sink, active);
            const uint32_t fl = (sink ? kSink : 0u) | (degen ? kDegenerate : 0u) | (active ? kActive : 0u);
            my_act = active;
            t.route_flags[u] = fl;
            if (!exact_later) t.group_scores[u] = S;
            t.unit_flags[u] = fl;
            if (!active) {
                t.tokens[u] = 0ull;
                if (t.mode == 1) {  // rank partial of a skipped group: empty
                    float* P = t.out + size_t(u) * r * (D + 2);
                    for (uint32_t h = 0; h < r; ++h) {
                        P[h] = -INFINITY;
                        P[r + h] = 0.f;
                    }
                    for (uint32_t k = 0; k < r * D; ++k) P[2 * r + k] = 0.f;
                }
            }
        }
        if (!exact_later)
            for (uint32_t h = h_lo + tid; h < h_hi; h += kThreads) t.head_scores[h] = s_score[h - h_lo];
        // this CTA's decisions as one word (bit i: unit u_lo + i Active), so
        // every CTA reads one word per CTA after the barrier, not one per unit
        const bool use_sum = up <= 32u;
        if (use_sum && warp == 0) {
            const uint32_t m = __ballot_sync(0xffffffffu, my_act && tid < u_hi - u_lo);
            if (lane == 0) t.route_sum[bid] = m;
        }
        STAMP(14);
        // grid barrier: every unit's decision is published (cooperative launch,
        // all CTAs resident; a 2 s watchdog turns a bug into an error, not a hang)
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            atomicAdd(&sc->route_done, 1u);
            const unsigned long long t_spin = globaltimer();
            while (ld_volatile(&sc->route_done) < G) {
                if (globaltimer() - t_spin > 2000000000ull) {
                    raise_error(t, sc, 3u);
                    break;
                }
            }
            __threadfence();
        }
        __syncthreads();
        STAMP(16);

        // the Active list from the published decisions: contiguous unit runs
        // per thread, then an order-preserving scan.
        // With the per-CTA words, thread t takes CTA t's units (one load);
        // else contiguous runs of per-unit flags.
        const uint32_t per = use_sum ? up : (U + kThreads - 1) / kThreads;
        const uint32_t u0 = min(U, tid * per), u1 = min(U, u0 + per);
        uint32_t my_active = 0;
        unsigned long long my_tok = 0;
        uint64_t my_bits = 0;  // active bits of this thread's run (per <= 64 guaranteed)
        if (use_sum && u0 < u1) {
            const uint32_t m = __ldcg(&t.route_sum[tid]);
            my_bits = m;
            my_active = __popc(m);
            for (uint32_t b = m; b; b &= b - 1u) my_tok += s_len[(u0 + __ffs(b) - 1) / t.Hkv];
        }
        // (per-unit flags: all of this thread's flags in flight at once, runs
        // are <= 8 units for U <= 1280, then the bookkeeping)
        for (uint32_t ub = u0; !use_sum && ub < u1; ub += 8) {
            uint32_t fl[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) fl[k] = (ub + k < u1) ? __ldcg(&t.route_flags[ub + k]) : 0u;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (fl[k] & kActive) {
                    const uint32_t u = ub + k;
                    ++my_active;
                    my_tok += s_len[u / t.Hkv];
                    my_bits |= 1ull << (u - u0);
                }
            }
        }
        STAMP(17);
        const unsigned long long tok_all = Reduce(tmp.reduce).Sum(my_tok);
        if (tid == 0) s_tok_total = tok_all;
        __syncthreads();
        STAMP(18);
        uint32_t a_off, nact;
        Scan(tmp.scan).ExclusiveSum(my_active, a_off, nact);
        STAMP(19);
        // chunk size: ~kChunksPerCta chunks per CTA, >= kMinChunkTok, stage multiple
        const unsigned long long T = s_tok_total;
        const uint32_t gdiv = G * kChunksPerCta;
        unsigned long long cc = T < (1ull << 32)
                                    ? (unsigned long long)(((uint32_t)T + gdiv - 1) / gdiv)
                                    : (T + gdiv - 1) / gdiv;
        cc = ((cc + kStageTok - 1) / kStageTok) * kStageTok;
        if (cc < kMinChunkTok) cc = kMinChunkTok;
        const uint32_t Ck = (uint32_t)cc;
        const bool flat = nact > G;
        uint32_t my_chunks = 0;  // flat mode: this thread's Active tokens (token prefix)
        {
            uint32_t a = a_off;
            for (uint32_t u = u0; u < u1; ++u) {
                if (!((my_bits >> (u - u0)) & 1ull)) continue;
                const uint32_t L = s_len[u / t.Hkv];
                act_len[a] = L;
                act_unit[a++] = (uint16_t)u;
                if (flat) my_chunks += L;
            }
        }
        STAMP(20);
        if (flat) {
            __syncthreads();
            uint32_t c_off, c_tot;
            Scan(tmp.scan).ExclusiveSum(my_chunks, c_off, c_tot);
            uint32_t a = a_off;
            for (uint32_t u = u0; u < u1; ++u) {
                if (!((my_bits >> (u - u0)) & 1ull)) continue;
                act_prefix[a] = c_off;
                c_off += act_len[a++];
            }
            if (tid == 0) act_prefix[nact] = c_tot;
        }
        STAMP(21);
        if (tid == 0) {
            misc[kMiscNact] = nact;
            misc[kMiscChunk] = Ck;
            misc[kMiscStatic] = static_chunk(T, G, t.static_pct, Ck);
            misc[kMiscFlat] = flat ? 1u : 0u;
        }
    }
    __syncthreads();  // Active list, chunk plan and misc visible to all threads
    STAMP(7);
    nact = misc[kMiscNact];
    Ck = misc[kMiscChunk];
    Cs = misc[kMiscStatic];
    flat = !LEAN && misc[kMiscFlat] != 0;
    // up to ~4 merge tasks (unit, head, 32 dims) per consumer warp: the tasks
    // are spread over every warp once its stream ends; more: the CTA that
    // streams a group's last rows merges it in line.  A/B (r01f, back to back):
    // queue mode for all takes C3-dense (2,048 tasks) 959 -> 941 us and
    // C5-routed (1,920) 309 -> 305 us, but C5-dense (5,120) 757 -> 761 us.
    queue_mode = LEAN || nact * r * (D / 32) <= 16u * G;  // (LEAN: nact <= 32; correct either way)
    lean_fast = lean && misc[kMiscFast] != 0;
    // mode 3: partial slots double-buffered by step parity (a rank one step
    // ahead never overwrites partials a slower rank is still merging).  The
    // step number is each CTA slot's own count of mode-3 launches
    // (cta_epoch[G + bid], advanced by that CTA at exit), so the graph needs
    // no per-step parameter patch.
    xoff = (size_t((epoch & 1u) * t.world + t.rank)) * U * (r * (D + 2));
    __syncthreads();  // routing overlay dead from here on; the ring is free
    STAMP(8);
    if (t.trace && tid == 0) t.trace[bid * 8 + 0] = globaltimer();
    if (lead && tid == 0) clk[1] = globaltimer();
    } else {
        // dry pass: one Active entry (unit 0), no routing
        if (tid == 0) {
            act_unit[0] = 0;
            act_len[0] = 0;
        }
        nact = 1;
        __syncthreads();
    }

    // ======================= phase S: stream + attend ==========================
    if (warp == 0) {
        if (lane == 0 && !dry) {
            const uint64_t pol = ptx::policy_evict_first();
            int stage = 0;
            uint32_t phase = 0;
            uint32_t n_emit = 0, tok_emit = 0;  // trace only
            auto emit = [&](uint32_t u, uint32_t L, uint32_t t0, uint32_t t1) {
                ++n_emit;
                tok_emit += t1 > t0 ? t1 - t0 : 0u;
                const int32_t row0 = (int32_t)((size_t(layer) * U + u) * t.cap);
                for (uint32_t tk = t0; tk < t1; tk += kStageTok) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1u);
                    meta[stage].unit = u;
                    meta[stage].tok0 = tk;
                    meta[stage].ntok = min((uint32_t)kStageTok, t1 - tk);
                    meta[stage].pad = L;
                    ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                    uint8_t* kd = ring + stage * C::kStageBytes;
                    uint8_t* vd = kd + C::kTileBytes;
#pragma unroll
                    for (int h = 0; h < C::kHalves; ++h) {
                        ptx::tma_load_2d(kd + h * kStageTok * 128, t.tmk, h * C::kBoxDim,
                                         row0 + (int32_t)tk, &full[stage], pol);
                        ptx::tma_load_2d(vd + h * kStageTok * 128, t.tmv, h * C::kBoxDim,
                                         row0 + (int32_t)tk, &full[stage], pol);
                    }
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            };
            if (nact > 0 && !flat) {
                // Unit-affine guided self-scheduling over TOKEN cursors.  CTA c
                // starts on Active entry c mod nact with the static range
                // [k*Cs, (k+1)*Cs), k = c / nact.  Later claims take tokens past
                // the statically covered prefix base(a)*Cs; their size shrinks
                // with the unit's remaining rows (guided), down to one 64-token
                // stage, so all SMs finish within about one stage of each other.
                // An exhausted unit hands the CTA on to the unit with the most
                // unclaimed rows (all cursors read in parallel, 16 loads in
                // flight), so the tail is spent streaming, not probing.
                // The lead CTA (bid 0) has no static range: its consumers are
                // busy with the routing record for the first microseconds, so
                // it starts on dynamic claims; entry 0's static ranges go to
                // CTAs nact, 2 nact, ... (chunk k - 1).
                // (the prewarm CTAs, the last ones, have no static range either)
                const uint32_t cpu = (G + nact - 1) / nact;  // CTAs per unit
                const uint32_t Gs = G - n_pw;  // CTAs [0, Gs) hold static ranges
                // (static CTAs interleaved over the entries: contiguous blocks of
                // CTAs per entry ran 1-1.8 us slower back to back, r02 A/B)
                auto static_end = [&](uint32_t e) {        // statically covered prefix of entry e
                    return (e < Gs ? ((Gs - e + nact - 1) / nact) - (e == 0 ? 1u : 0u) : 0u) * Cs;
                };
                uint32_t a = bid % nact;
                uint32_t u = act_unit[a], L = act_len[a];
                uint32_t first = static_end(a);
                const uint32_t k0 = bid / nact - (a == 0 ? 1u : 0u);  // bid 0: wraps, no static range
                uint32_t t0 = (bid == 0 || prewarm) ? L : k0 * Cs, t1 = min(t0 + Cs, L);
                auto guided = [&](uint32_t hint) {
                    const uint32_t rem = L > hint ? L - hint : 0u;
                    uint32_t sz = rem / (3 * cpu);
                    sz = sz / kStageTok * kStageTok;
                    return sz < (uint32_t)kStageTok ? (uint32_t)kStageTok : (sz > Ck ? Ck : sz);
                };
                // the prewarm CTA arrives late (after its dry pass): it joins
                // only while there is more than ~2 us of stream left for the
                // whole grid, else its first stage would land after the others
                // finish and make it the tail
                bool late_join = prewarm;
                for (;;) {
                    if (t0 >= L) {
                        uint32_t best = 0, best_rem = 0;
                        unsigned long long all_rem = 0;
                        for (uint32_t b0 = 0; b0 < nact; b0 += 16) {
                            uint32_t cur[16];
#pragma unroll
                            for (int k = 0; k < 16; ++k)
                                cur[k] = (b0 + k < nact) ? ld_volatile(&t.cursor[b0 + k]) : 0u;
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                const uint32_t b = b0 + k;
                                if (b < nact) {
                                    const uint32_t pos = static_end(b) + cur[k];
                                    const uint32_t rem = act_len[b] > pos ? act_len[b] - pos : 0u;
                                    all_rem += rem;
                                    if (rem > best_rem) {
                                        best_rem = rem;
                                        best = b;
                                    }
                                }
                            }
                        }
                        if (best_rem == 0) break;
                        if (late_join && all_rem < kLateJoinTok) break;
                        late_join = false;
                        a = best;
                        u = act_unit[a];
                        L = act_len[a];
                        first = static_end(a);
                        // a hand-off claim is sized from the unit's live remainder
                        const uint32_t sz = guided(L - best_rem);
                        t0 = first + atomicAdd(&t.cursor[a], sz);
                        t1 = min(t0 + sz, L);
                        continue;
                    }
                    // prefetch the next claim of this unit (sized from our position)
                    const uint32_t sz = guided(max(t0, first));
                    const uint32_t n0 = first + atomicAdd(&t.cursor[a], sz);
                    emit(u, L, t0, t1);
                    t0 = n0;
                    t1 = min(n0 + sz, L);
                }
            } else if (nact > 0) {
                // many Active groups (batched steps): guided self-scheduling over
                // ONE global token space, the Active units laid end to end
                // (act_prefix = token prefix).  A static first claim of T/(3G)
                // tokens per CTA, then claims from one cursor whose size shrinks
                // with the remaining tokens (T - pos)/(2G), down to one stage.
                // Early claims cover about a unit, so a CTA flushes a partial
                // every few units rather than every chunk; a claim that crosses
                // a unit boundary is emitted piecewise.
                const uint32_t T = act_prefix[nact];
                uint32_t S0 = T / (3 * G);
                S0 = max((uint32_t)kStageTok, S0 / kStageTok * kStageTok);
                const uint32_t base = min(G * S0, T);  // dynamic region start
                // claims never shrink below kFlatMinTok: consecutive claims of
                // one CTA land in different units, so each costs a partial flush
                // (~3 L2 round trips); a 512-token floor bounds the tail at
                // ~256 KB per SM instead of paying a flush per 64 tokens
                const uint32_t cap_tok = max(S0, kFlatMinTok);
                auto guided = [&](uint32_t pos) {
                    const uint32_t rem = T > pos ? T - pos : 0u;
                    uint32_t sz = rem / (2 * G) / kStageTok * kStageTok;
                    return sz < kFlatMinTok ? kFlatMinTok : (sz > cap_tok ? cap_tok : sz);
                };
                uint32_t g0 = min(bid * S0, base), g1 = min(g0 + S0, base);
                uint32_t a = 0;
                for (;;) {
                    // prefetch the next claim, sized from the LIVE cursor: our own
                    // position lags it by about one claim per CTA, which would
                    // keep late claims large and leave a long tail
                    const uint32_t sz = guided(base + ld_volatile(&sc->flat_counter));
                    const uint32_t n0 = base + atomicAdd(&sc->flat_counter, sz);
                    while (g0 < g1) {
                        // act_prefix is sorted and claims of one CTA increase
                        if (act_prefix[a + 1] <= g0) {
                            uint32_t lo = a + 1, hi = nact;
                            while (hi - lo > 1) {
                                const uint32_t mid = (lo + hi) >> 1;
                                if (act_prefix[mid] <= g0) lo = mid; else hi = mid;
                            }
                            a = lo;
                        }
                        const uint32_t pa = act_prefix[a], pe = min(act_prefix[a + 1], g1);
                        emit(act_unit[a], act_len[a], g0 - pa, pe - pa);
                        g0 = pe;
                    }
                    if (n0 >= T) break;
                    g0 = n0;
                    g1 = min(n0 + sz, T);
                }
            }
            if (t.trace) {
                t.trace[bid * 8 + 6] = ((unsigned long long)n_emit << 32) | tok_emit;
                t.trace[bid * 8 + 7] = globaltimer();
            }
            ptx::mbar_wait(&empty[stage], phase ^ 1u);
            meta[stage].unit = kEnd;
            ptx::mbar_arrive(&full[stage]);
        }
        __syncwarp();
    } else {
        // ------------------------------ consumers ------------------------------
        const int cw = warp - 1;
        const uint32_t ctid = tid - 32;
        // zero surrogate rows of Sink groups (router.cpp:97), written while the
        // first stages are in flight: single-sequence steps, CTA u mod G for
        // unit u (binary search of the sorted Active list); batched steps, the
        // CTA that routed the unit
        if (!dry && t.mode != 1 && nact < U) {
            uint32_t z_lo = bid, z_step = G, z_hi = U;
            if (!lean) {
                const uint32_t up = (U + G - 1) / G;
                z_lo = min(U, bid * up);
                z_hi = min(U, z_lo + up);
                z_step = 1;
            }
            for (uint32_t u = z_lo; u < z_hi; u += z_step) {
                bool sink;
                if (lean) {
                    uint32_t lo = 0, hi = nact;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (act_unit[mid] < u) lo = mid + 1; else hi = mid;
                    }
                    sink = !(lo < nact && act_unit[lo] == u);
                } else {
                    sink = !(__ldcg(&t.route_flags[u]) & kActive);
                }
                if (!sink) continue;
                float4* row = reinterpret_cast<float4*>(t.out + size_t(u) * r * D);
                for (uint32_t k = ctid; k < r * D / 4; k += kCWarps * 32) row[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        if (!dry && ((lean_fast && lead) || exact_later)) {
            // the routing record's exact fp64 scores (the decisions were taken
            // from fp32 estimates that cleared tau by kRouteMargin), computed
            // while the first stages are in flight: thread h streams q row h and
            // its group's k0 row through registers, exact products off the
            // chain, sequential DADD chains in index order (router.cpp:40-43).
            // Lean form: the lead CTA, all heads; distributed form: every CTA,
            // its own units.
            uint32_t xu_lo = 0, xu_hi = U;
            if (!lean) {
                const uint32_t up = (U + G - 1) / G;
                xu_lo = min(U, bid * up);
                xu_hi = min(U, xu_lo + up);
            }
            const uint32_t xh_lo = xu_lo * r, nxh = (xu_hi - xu_lo) * r;
            double* xs = reinterpret_cast<double*>(sm_o);  // flush staging is idle until the first flush
            uint8_t* xd = reinterpret_cast<uint8_t*>(xs + (kThreads - 32));
            if (ctid < nxh) {
                const uint32_t h = xh_lo + ctid, u = h / r;
                const float4* qrow = reinterpret_cast<const float4*>(t.q + size_t(h) * D);
                const float4* krow = reinterpret_cast<const float4*>(t.anchors + (size_t(layer) * U + u) * D);
                const float kn = __ldg(&t.anchor_norm[size_t(layer) * U + u]);
                double dot = 0.0, qq = 0.0;
#pragma unroll 8
                for (int c = 0; c < D / 4; ++c) {
                    const float4 x = __ldg(qrow + c), y = __ldg(krow + c);
                    const float qf[4] = {x.x, x.y, x.z, x.w}, kf[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const double qd = (double)qf[e];
                        dot = __dadd_rn(dot, __dmul_rn(qd, (double)kf[e]));
                        qq = __dadd_rn(qq, __dmul_rn(qd, qd));
                    }
                }
                const double qn = __dsqrt_rn(qq);
                double sc = 0.0;
                uint8_t dg = 0;
                if (qn < 1e-12) {
                    dg = 1;
                } else {
                    sc = __ddiv_rn(dot, __dmul_rn(qn, (double)kn));
                    sc = sc < -1.0 ? -1.0 : (1.0 < sc ? 1.0 : sc);  // std::clamp
                }
                xs[ctid] = sc;
                xd[ctid] = dg;
                t.head_scores[h] = sc;
            }
            ptx::named_bar_sync(1, kCWarps * 32);
            for (uint32_t u = xu_lo + ctid; u < xu_hi; u += kCWarps * 32) {
                const uint32_t seq = u / t.Hkv, hb = (u - xu_lo) * r;
                double sum = 0.0;
                uint32_t degen = 0;
                for (uint32_t i = 0; i < r; ++i) {
                    sum = __dadd_rn(sum, xs[hb + i]);
                    degen |= xd[hb + i];
                }
                const double S = (r & (r - 1)) == 0 ? __dmul_rn(sum, 1.0 / (double)r) : __ddiv_rn(sum, (double)r);
                double tau = 0.0;  // the ring overlay (s_tau) is gone: re-read the step's tau
                if (p.inline_seqs) {
#pragma unroll
                    for (int k = 0; k < kParamSeqs; ++k)
                        if ((uint32_t)k == seq) tau = p.tau[k];
                } else {
                    tau = __ldg(&t.tau_g[seq]);
                }
                const bool over = (flags & kSinkOnTie) ? (S >= tau) : (S > tau);
                bool sink = over && !(flags & kLayerExcluded);
                if (degen) sink = false;
                bool active = (flags & kObserveOnly) || !sink;
                force_route(p.only_unit, u, sink, active);
                t.group_scores[u] = S;
                // the exact flags (the estimate pass cannot see a degenerate head
                // when observe-only or an excluded layer made every decision certain)
                t.unit_flags[u] = (sink ? kSink : 0u) | (degen ? kDegenerate : 0u) | (active ? kActive : 0u);
                if (lean && !active) {
                    t.tokens[u] = 0ull;
                    if (t.mode == 1) {  // rank partial of a skipped group: empty
                        float* P = t.out + size_t(u) * r * (D + 2);
                        for (uint32_t h = 0; h < r; ++h) {
                            P[h] = -INFINITY;
                            P[r + h] = 0.f;
                        }
                        for (uint32_t k = 0; k < r * D; ++k) P[2 * r + k] = 0.f;
                    }
                }
                const bool taken = lean ? act_prefix[u] != 0u : (t.route_flags[u] & kActive) != 0u;
                if (active != taken) raise_error(t, sc, 4u);  // never: margin >> error
            }
            ptx::named_bar_sync(1, kCWarps * 32);
        }
        // this warp's tokens of a stage (kSub 16-token sub-tiles from tb0) and
        // query heads (hbase .. hbase+7; WIDE: the group's head half cw & 1)
        constexpr int kSub = WIDE ? 2 : 1;
        const int tb0 = WIDE ? (cw >> 1) * (2 * kWarpTok) : cw * kWarpTok;
        const uint32_t hbase = WIDE ? 8u * (cw & 1) : 0u;
        const int grp = lane >> 2, qd = lane & 3;
        const int lj = lane >> 3, li = lane & 7;
        const uint32_t k_csel = lj & 1, v_csel = lj >> 1;
        const uint32_t PS = r * (D + 2);

        uint32_t qa[C::kNK][4];
        float o[2 * C::kNK][4];
        float m_used = -INFINITY, l_acc = 0.f;
        uint32_t cur = kEnd, cur_len = 0, run_tokens = 0;
        uint32_t my_slot = 0;  // ctid 0: partial slot of the current visit, claimed at its start

        auto reset_state = [&]() {
#pragma unroll
            for (int i = 0; i < 2 * C::kNK; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
            m_used = -INFINITY;
            l_acc = 0.f;
        };
        auto load_q = [&](uint32_t u) {
            const bool live = hbase + grp < r;
            const float* qrow = t.q + (size_t(u) * r + (live ? hbase + grp : 0)) * D;
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
        // merge every partial of unit u (consumers only; few partials)
        auto merge_unit = [&](uint32_t u, uint32_t L) {
            for (uint32_t task = cw; task < r * (D / 32); task += kCWarps)
                warp_merge_r<D, WIDE>(t, u, task / (D / 32), (task % (D / 32)) * 32, lane, xoff, epoch + 1u,
                                      sm_o + warp * 64);
            if (ctid == 0) t.tokens[u] = L;
        };
        auto flush = [&](uint32_t u, uint32_t L) {
            float l_tot = l_acc + __shfl_xor_sync(0xffffffffu, l_acc, 1);
            l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 2);
            if (hbase + grp < r) {
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
            if (ctid == 0) misc[kMiscSlot] = my_slot;
            ptx::named_bar_sync(1, kCWarps * 32);
            const uint32_t slot = misc[kMiscSlot];
            // slots [0, S-1) take one partial each; every later partial of the
            // unit (only a long, many-handed tail gets there) is LSE-combined
            // into slot S-1 under a per-unit lock (ovf: bit0 lock, bit1 valid)
            const bool spill = !dry && slot >= t.S - 1;
            if (spill) {
                if (ctid == 0) {
                    uint32_t old_v;
                    const unsigned long long t_spin = globaltimer();
                    while ((old_v = atomicOr(&t.ovf[u], 1u)) & 1u) {
                        if (globaltimer() - t_spin > 2000000000ull) {
                            raise_error(t, sc, 1u);
                            break;
                        }
                    }
                    __threadfence();
                    misc[kMiscTask] = old_v & 2u;  // slot S-1 already holds a partial
                }
                ptx::named_bar_sync(1, kCWarps * 32);
            }
            const bool combine = spill && misc[kMiscTask] != 0;
            float* P = t.partials + (size_t(u) * t.S + (spill ? t.S - 1 : slot)) * PS;
            float* old_ml = sm_ml + kCWarps * kMaxR * 2;  // [kMaxR][2] staged (m, l) of slot S-1
            if (combine) {
                if (ctid < r) {
                    old_ml[2 * ctid] = __ldcg(P + ctid);
                    old_ml[2 * ctid + 1] = __ldcg(P + r + ctid);
                }
                ptx::named_bar_sync(1, kCWarps * 32);
            }
            for (uint32_t idx = ctid; idx < r * D; idx += kCWarps * 32) {
                const uint32_t h = idx / D, d = idx % D;
                // the warps holding head h, and its row in their tiles (WIDE:
                // warps h/8 and h/8 + 2, row h % 8; else all warps, row h)
                constexpr int kHW = WIDE ? 2 : kCWarps;
                const uint32_t w0 = WIDE ? h / 8 : 0u, hr = WIDE ? h % 8 : h;
                constexpr uint32_t kWs = WIDE ? 2u : 1u;
                float mx = -INFINITY;
                // (dry: everything but the stores below)
#pragma unroll
                for (int i = 0; i < kHW; ++i) mx = fmaxf(mx, sm_ml[((w0 + i * kWs) * kMaxR + hr) * 2]);
                float acc = 0.f, lsum = 0.f;
#pragma unroll
                for (int i = 0; i < kHW; ++i) {
                    const uint32_t row = (w0 + i * kWs) * kMaxR + hr;
                    const float sc = ptx::ex2(sm_ml[row * 2] - mx);
                    acc += sm_o[row * C::kOStride + d] * sc;
                    lsum += sm_ml[row * 2 + 1] * sc;
                }
                if (combine) {
                    const float mo = old_ml[2 * h], mn = fmaxf(mo, mx);
                    const float so = mo == -INFINITY ? 0.f : ptx::ex2(mo - mn);
                    const float sn = mx == -INFINITY ? 0.f : ptx::ex2(mx - mn);
                    acc = __ldcg(P + 2 * r + h * D + d) * so + acc * sn;
                    lsum = old_ml[2 * h + 1] * so + lsum * sn;
                    mx = mn;
                }
                if (!dry) {
                    P[2 * r + h * D + d] = acc;
                    if (d == 0) {
                        P[h] = mx;
                        P[r + h] = lsum;
                    }
                }
            }
            if (spill) {
                __threadfence();
                ptx::named_bar_sync(1, kCWarps * 32);
                if (ctid == 0) atomicExch(&t.ovf[u], 2u);  // release; slot S-1 now valid
            }
            // the partial is visible before this run's rows are counted: the
            // barrier orders the CTA's writes before ctid 0's gpu-scope release
            ptx::named_bar_sync(1, kCWarps * 32);
            if (ctid == 0) {
                const uint32_t done =
                    dry ? 0u
                        : (queue_mode ? ptx::atom_add_release(&t.tokens_done[u], run_tokens)
                                      : ptx::atom_add_acq_rel(&t.tokens_done[u], run_tokens)) +
                              run_tokens;
                misc[kMiscLast] = (!dry && done == L) ? 1u : 0u;
            }
            ptx::named_bar_sync(1, kCWarps * 32);
            if (misc[kMiscLast] && !queue_mode) merge_unit(u, L);
            ptx::named_bar_sync(1, kCWarps * 32);
        };

        int stage = 0;
        uint32_t phase = 0;
        // dry pass: iteration 0 runs the body on unit 0 over stale shared
        // memory, iteration 1 the flush (no stores), then out
        uint32_t dry_it = 0;
        for (;;) {
            if (dry && !(dry_regions & 3u)) break;  // merge only
            if (!dry) ptx::mbar_wait(&full[stage], phase);
            const uint32_t unit = dry ? (dry_it++ == 0 ? 0u : kEnd) : meta[stage].unit;
            if (unit != cur || unit == kEnd) {  // kEnd == cur when a CTA had no work
                if (cur != kEnd && !(dry && !(dry_regions & 2u))) flush(cur, cur_len);  // the only flush site
                if (unit == kEnd) break;
                cur = unit;
                if (ctid == 0 && !dry) my_slot = atomicAdd(&t.slot_count[unit], 1u);  // hidden by the stream
                cur_len = dry ? 0u : meta[stage].pad;
                run_tokens = 0;
                load_q(unit);
                reset_state();
            }
            const uint32_t ntok = dry ? ((dry_regions & 1u) ? (uint32_t)kStageTok : 0u) : meta[stage].ntok;
            run_tokens += ntok;
            if constexpr (WIDE) {
                // the warp's 32 tokens as ONE online-softmax step: both 16-token
                // sub-tiles' QK chains interleaved, one max / rescale / exp pass,
                // then both PV products (two independent k16 slices)
                const int n = (int)ntok - tb0;
                if (n > 0) {
                    const uint32_t kbase = ptx::smem_u32(ring + stage * C::kStageBytes);
                    const uint32_t vbase = kbase + C::kTileBytes;
                    float sacc[2][2][2][4];  // [sub][8-token n-tile][chain][4]
#pragma unroll
                    for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
                        for (int a = 0; a < 2; ++a)
#pragma unroll
                            for (int b = 0; b < 2; ++b)
                                sacc[s2][a][b][0] = sacc[s2][a][b][1] = sacc[s2][a][b][2] = sacc[s2][a][b][3] = 0.f;
#pragma unroll
                    for (int kk = 0; kk < C::kNK; ++kk) {
#pragma unroll
                        for (int s2 = 0; s2 < 2; ++s2) {
                            const uint32_t k_tok = tb0 + s2 * kWarpTok + ((lj >> 1) << 3) + li;
                            uint32_t b[4];
                            ptx::ldsm_x4(b, kbase + swz<D>(k_tok, 2 * kk + k_csel));
                            ptx::mma_bf16(sacc[s2][0][kk & 1], qa[kk], b[0], b[1]);
                            ptx::mma_bf16(sacc[s2][1][kk & 1], qa[kk], b[2], b[3]);
                        }
                    }
                    float sc[2][4];
#pragma unroll
                    for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int nt = j >> 1, col = j & 1;
                            const float v = (sacc[s2][nt][0][col] + sacc[s2][nt][1][col]) +
                                            (sacc[s2][nt][0][col + 2] + sacc[s2][nt][1][col + 2]);
                            const int tok = s2 * kWarpTok + nt * 8 + 2 * qd + col;
                            sc[s2][j] = tok < n ? v : -INFINITY;
                        }
                    float bm = fmaxf(fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[0][2], sc[0][3])),
                                     fmaxf(fmaxf(sc[1][0], sc[1][1]), fmaxf(sc[1][2], sc[1][3])));
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
                    uint32_t pa[2][4];
#pragma unroll
                    for (int s2 = 0; s2 < 2; ++s2) {
                        float pr[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) pr[j] = ptx::ex2(sc[s2][j] - m_used);
                        l_acc += (pr[0] + pr[1]) + (pr[2] + pr[3]);
                        pa[s2][0] = ptx::pack_bf16(pr[0], pr[1]);
                        pa[s2][1] = ptx::pack_bf16(pr[0] - ptx::bf16_lo_as_f32(pa[s2][0]),
                                                   pr[1] - ptx::bf16_hi_as_f32(pa[s2][0]));
                        pa[s2][2] = ptx::pack_bf16(pr[2], pr[3]);
                        pa[s2][3] = ptx::pack_bf16(pr[2] - ptx::bf16_lo_as_f32(pa[s2][2]),
                                                   pr[3] - ptx::bf16_hi_as_f32(pa[s2][2]));
                    }
#pragma unroll
                    for (int nn = 0; nn < C::kNK; ++nn) {
#pragma unroll
                        for (int s2 = 0; s2 < 2; ++s2) {
                            const uint32_t v_tok = tb0 + s2 * kWarpTok + ((lj & 1) << 3) + li;
                            uint32_t b[4];
                            ptx::ldsm_x4_t(b, vbase + swz<D>(v_tok, 2 * nn + v_csel));
                            ptx::mma_bf16(o[2 * nn], pa[s2], b[0], b[1]);
                            ptx::mma_bf16(o[2 * nn + 1], pa[s2], b[2], b[3]);
                        }
                    }
                }
            } else {
#pragma unroll
            for (int sub = 0; sub < kSub; ++sub) {
            const int tb = tb0 + sub * kWarpTok;
            const uint32_t k_tok = tb + ((lj >> 1) << 3) + li;
            const uint32_t v_tok = tb + ((lj & 1) << 3) + li;
            const int n = (int)ntok - tb;
            if (n > 0) {
                const uint32_t kbase = ptx::smem_u32(ring + stage * C::kStageBytes);
                const uint32_t vbase = kbase + C::kTileBytes;
                float sacc[2][2][4];
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int b = 0; b < 2; ++b)
                        sacc[a][b][0] = sacc[a][b][1] = sacc[a][b][2] = sacc[a][b][3] = 0.f;
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
                float pr[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) pr[j] = ptx::ex2(sc[j] - m_used);
                l_acc += (pr[0] + pr[1]) + (pr[2] + pr[3]);
                uint32_t pa[4];
                pa[0] = ptx::pack_bf16(pr[0], pr[1]);
                pa[1] = ptx::pack_bf16(pr[0] - ptx::bf16_lo_as_f32(pa[0]), pr[1] - ptx::bf16_hi_as_f32(pa[0]));
                pa[2] = ptx::pack_bf16(pr[2], pr[3]);
                pa[3] = ptx::pack_bf16(pr[2] - ptx::bf16_lo_as_f32(pa[2]), pr[3] - ptx::bf16_hi_as_f32(pa[2]));
#pragma unroll
                for (int nn = 0; nn < C::kNK; ++nn) {
                    uint32_t b[4];
                    ptx::ldsm_x4_t(b, vbase + swz<D>(v_tok, 2 * nn + v_csel));
                    ptx::mma_bf16(o[2 * nn], pa, b[0], b[1]);
                    ptx::mma_bf16(o[2 * nn + 1], pa, b[2], b[3]);
                }
            }
            }  // sub
            }  // !WIDE
            __syncwarp();
            if (lane == 0 && !dry) ptx::mbar_arrive(&empty[stage]);
            if (++stage == C::kStages) {
                stage = 0;
                phase ^= 1u;
            }
        }
    }
    __syncthreads();
    if (!dry) {
        STAMP(9);
        t_stream_end = globaltimer();
        if (t.trace && tid == 0) t.trace[bid * 8 + 1] = t_stream_end;
    } else if (t.trace && tid == 0) {
        t.trace[bid * 8 + 3] = globaltimer();  // dry stream pass done (trace only)
    }

    // ======================= phase M: distributed merge ========================
    // Tasks (active entry, head, 32-dim slice) are claimed by WARPS: a warp
    // waits until its unit's last rows are counted, then merges the slice with
    // warp_merge (one L2 round trip per 64 partials, no block barrier).
    if (queue_mode && nact > 0 && !(dry && !(dry_regions & 4u))) {
        constexpr uint32_t nd = D / 32;
        const uint32_t ntasks = nact * r * nd;
        for (;;) {
            uint32_t task = 0;
            if (lane == 0) task = dry ? warp : atomicAdd(&sc->merge_next, 1u);
            task = __shfl_sync(0xffffffffu, task, 0);
            if (task >= ntasks) break;
            const uint32_t a = task / (r * nd), rem = task % (r * nd);
            const uint32_t h = rem / nd, d = (rem % nd) * 32 + lane;
            const uint32_t u = act_unit[a];
            const uint32_t L = act_len[a];
            if (lane == 0 && !dry) {
                // watchdog: a unit that never completes (a bug) must not hang
                // the GPU; after 2 s report an error and give up the task
                const unsigned long long t_spin = globaltimer();
                while (ptx::ld_acquire(&t.tokens_done[u]) < L) {
                    if (globaltimer() - t_spin > 2000000000ull) {
                        raise_error(t, sc, 2u);
                        break;
                    }
                }
                if (t.trace) t.trace[bid * 8 + 3] = globaltimer();
            }
            __syncwarp();
            warp_merge_r<D, WIDE>(t, u, h, d - lane, lane, xoff, epoch + 1u, sm_o + warp * 64, dry);
            if (dry) break;
            if (h == 0 && d == 0) t.tokens[u] = L;
            // every warp of the grid claims once, so with no more tasks than
            // warps a second claim finds nothing: skip its L2 round trip (the
            // dry pass claims nothing; every CTA claims in its real pass)
            if (ntasks <= (G - n_pw) * (kThreads / 32)) break;
        }
    }
    if (dry) {
        // A dry pass this slow ran from a cold L2 (~20 us against ~6 warm):
        // by now the other CTAs have claimed the work and this CTA would
        // only be the last to route and exit, so it leaves (the others'
        // merge claims suffice: ntasks <= (G - n_pw) warps).  Warm, it joins
        // the stream on dynamic claims.
        if (tid == 0) {
            const unsigned long long now = globaltimer();
            const unsigned long long late_ns = (t.prewarm >> 8) ? (t.prewarm >> 8) * 1000ull : kPrewarmLateNs;
            misc[kMiscTask] = (now - t_cta_start > late_ns) ? 1u : 0u;
            if (t.trace) t.trace[bid * 8 + 5] = now;  // dry pass done (trace only)
        }
        __syncthreads();  // (also: scratch sm_o free before the stream)
        if (misc[kMiscTask]) break;
    }
    }  // pass

    // ======================= mode 3: merge every rank's partials ===============
    // Every rank's merge warps stored its partial into this rank's exchange
    // block as LL words tagged with the step (warp_merge): an owner thread
    // polls the three words it needs from each rank -- (m, l) of its head and
    // its acc element -- until all carry this step's tag, then merges.  No
    // fence and no arrival counter on the critical path; a word of an older
    // step (same parity two steps back) has another tag.  The owners finish
    // BEFORE they count out below, so the status a last CTA publishes covers
    // their waits.  A rank that never delivers is a watchdog error: the
    // owners then write NaN rather than a merge of incomplete partials.
    __syncthreads();
    STAMP(10);
    if (t.mode == 3 && bid * kThreads < nact * r * D) {
        const uint32_t PSx = r * (D + 2), tag = epoch + 1u, world = t.world;
        const unsigned long long* X = t.xchg_local + size_t((epoch & 1u) * world) * U * PSx;
        const unsigned long long t_spin = globaltimer();
        for (uint32_t e = bid * kThreads + tid; e < nact * r * D; e += G * kThreads) {
            const uint32_t a = e / (r * D), h = (e / D) % r, d = e % D;
            const uint32_t u = act_unit[a];
            float mq[8], aq[8], lq[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                mq[q] = -INFINITY;
                lq[q] = 0.f;
                aq[q] = 0.f;
            }
            uint32_t pending = (1u << world) - 1u;
            bool late = false;
            while (pending) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if ((pending >> q) & 1u) {
                        const unsigned long long* Pq = X + (size_t(q) * U + u) * PSx;
                        const unsigned long long wm = ptx::ld_ll(Pq + h), wl = ptx::ld_ll(Pq + r + h),
                                                 wa = ptx::ld_ll(Pq + 2 * r + h * D + d);
                        if (ptx::ll_tag(wm) == tag && ptx::ll_tag(wl) == tag && ptx::ll_tag(wa) == tag) {
                            mq[q] = ptx::ll_val(wm);
                            lq[q] = ptx::ll_val(wl);
                            aq[q] = ptx::ll_val(wa);
                            pending &= ~(1u << q);
                        }
                    }
                }
                if (pending && globaltimer() - t_spin > 2000000000ull) {
                    raise_error(t, sc, 5u);
                    late = true;
                    break;
                }
            }
            float mx = mq[0];
#pragma unroll
            for (int q = 1; q < 8; ++q) mx = fmaxf(mx, mq[q]);
            float acc = 0.f, lsum = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float w = mq[q] == -INFINITY ? 0.f : ptx::ex2(mq[q] - mx);
                acc += aq[q] * w;
                lsum += lq[q] * w;
            }
            t.out[(size_t(u) * r + h) * D + d] = late ? __int_as_float(0x7fc00000) : acc / lsum;
        }
    }

    // ======================= exit =============================================
    // Nothing to restore (the next launch zeroes this launch's counter set).
    // A last CTA is found only when it has work: the host completion word
    // (zero-copy results).
    __syncthreads();
    if (t.trace && tid == 0) t.trace[bid * 8 + 2] = globaltimer();
    if (tid == 0) {
        t_in.cta_epoch[bid] = cta_ep + 1u;  // after every thread of the CTA read it
        if (t.mode == 3) t_in.cta_epoch[G + bid] = epoch + 1u;  // this slot's mode-3 step count
    }
    if (t.done) {
        if (tid == 0) {
            // acq_rel count: releases this CTA's writes (ordered before tid 0
            // by the barrier) and, for the last CTA, acquires everyone's.
            // System scope when results go to mapped host memory and a host
            // thread waits on the completion word instead of the stream.
            const uint32_t prev = ptx::atom_add_acq_rel_sys(&sc->exit_count, 1u);
            if (prev == G - 1) {
                if (t.trace) t.trace[bid * 8 + 5] = globaltimer();
                clk[2] = t_stream_end;
                clk[3] = globaltimer();
                // every CTA's results (outputs, routing record, status) are
                // visible system-wide before the host sees the word
                __threadfence_system();
                ptx::st_release_sys(t.done, 1u);
            }
        }
    } else if (tid == 0) {
        // phase stamps: the latest stream end and exit (globaltimer only grows,
        // so a max over this launch's CTAs needs no reset)
        atomicMax(&clk[2], t_stream_end);
        atomicMax(&clk[3], globaltimer());
    }
}

}  // namespace dev
}  // namespace sinkr
