// stream_ab.cu -- A/B of the decode stream loop's contraction (SURVEY §8(d),
// BASELINE north_star: "the GQA group's query rows are packed into a small
// tcgen05/mma tile only if ncu shows it beats CUDA-core FMA").
//
// One kernel per variant streams the bf16 K/V of `nact` Active groups (D=128,
// GQA width R) through a TMA shared-memory ring and computes the Split-K
// online-softmax partial (m, l, acc) of every CTA's token range -- exactly the
// step kernel's phase S (attend_chunk, attention.cpp:101-142) with a static
// split instead of guided claims, so the three contraction schemes see the
// same memory stream:
//
//   hmma   the product path: 4 consumer warps, mma.sync m16n8k16, the fp32
//          query carried as hi/lo bf16 rows, P as hi/lo bf16 (step.cuh)
//   fma    CUDA-core fp32 FMA: QK with a thread per (token, half row), PV with
//          a thread per (head, 4 dims); exact bf16 K/V, fp32 q and P
//   tc05   tcgen05: S^T[128 tok x 16] = K[128 x 128] . Qhl^T (M = tokens,
//          N = hi/lo heads) into TMEM; softmax warps tcgen05.ld their token
//          lane, write P^T (hi/lo bf16) to smem; O^T[128 dims x 16] += V^T . P^T
//          (A = V tile read MN-major) accumulated in TMEM; lazy rescale of O in
//          TMEM (tcgen05.ld/st) when a head's max grows by > 8 (log2 domain)
//
// Checks every variant against an fp64 CPU reference (merged partials) at a
// small L, then times each at the requested L (back-to-back CUDA events).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -o stream_ab stream_ab.cu -lcuda
//   ./stream_ab [L=524288] [nact=3] [variant=all|hmma|hmma128|fma|tc05] [R=4|8]
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../paper_2604_16883_b200/csrc/ptx.cuh"

using namespace sinkr;
#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);    \
            exit(1);                                                                     \
        }                                                                                \
    } while (0)

constexpr int D = 128;
constexpr int kMaxR = 8;
constexpr int kPartFloats = 2 * kMaxR + kMaxR * D;  // m[8], l[8], acc[8][128]

struct Args {
    const CUtensorMap* tmk;
    const CUtensorMap* tmv;
    const float* q;  // [nact][R][D] f32
    float* part;     // [G][kPartFloats]
    uint32_t nact, L, stage_tok;
    float qscale;  // log2(e) / sqrt(D)
};

// static split: CTA c -> unit c % nact, part c / nact of that unit's tokens
__device__ __forceinline__ void cta_range(const Args& a, uint32_t& u, uint32_t& t0, uint32_t& t1) {
    const uint32_t G = gridDim.x, c = blockIdx.x;
    u = c % a.nact;
    const uint32_t np = (G - u + a.nact - 1) / a.nact, k = c / a.nact;
    uint32_t chunk = (a.L + np - 1) / np;
    chunk = (chunk + a.stage_tok - 1) / a.stage_tok * a.stage_tok;
    t0 = min(a.L, k * chunk);
    t1 = min(a.L, t0 + chunk);
}

__device__ __forceinline__ void write_empty(const Args& a) {
    float* P = a.part + size_t(blockIdx.x) * kPartFloats;
    for (int i = threadIdx.x; i < kPartFloats; i += blockDim.x) P[i] = i < kMaxR ? -INFINITY : 0.f;
}

// ---------------------------------------------------------------------------
// shared producer: 64-dim boxes of `box_tok` rows, K then V, per stage
template <int STAGES, int BOX_TOK>
__device__ __forceinline__ void produce(const Args& a, uint8_t* ring, uint64_t* full, uint64_t* empty,
                                        uint32_t u, uint32_t t0, uint32_t t1) {
    constexpr uint32_t kTile = BOX_TOK * D * 2, kStage = 2 * kTile;
    const uint64_t pol = ptx::policy_evict_first();
    int s = 0;
    uint32_t ph = 0;
    for (uint32_t tk = t0; tk < t1; tk += BOX_TOK) {
        ptx::mbar_wait(&empty[s], ph ^ 1u);
        ptx::mbar_arrive_expect_tx(&full[s], kStage);
        uint8_t* kd = ring + s * kStage;
        const int32_t row = (int32_t)(u * a.L + tk);
        for (int h = 0; h < 2; ++h) {
            ptx::tma_load_2d(kd + h * BOX_TOK * 128, a.tmk, h * 64, row, &full[s], pol);
            ptx::tma_load_2d(kd + kTile + h * BOX_TOK * 128, a.tmv, h * 64, row, &full[s], pol);
        }
        if (++s == STAGES) {
            s = 0;
            ph ^= 1u;
        }
    }
}

// byte offset of (token, 16-byte chunk of the 256-byte row) in a 64-row-box tile
template <int BOX_TOK>
__device__ __forceinline__ uint32_t swz(uint32_t tok, uint32_t chunk) {
    const uint32_t half = chunk >> 3, c = chunk & 7;
    return half * (BOX_TOK * 128) + tok * 128 + ((c ^ (tok & 7)) << 4);
}

// ============================ variant hmma ==================================
// HTOK = 64: the product's ring (6 x 32 KB, 4 consumer warps); HTOK = 128:
// tc05's ring shape (3 x 64 KB) with 8 consumer warps -- separates the stage
// size from the contraction in the A/B
template <int HTOK>
constexpr int hmma_smem() {
    return 1024 + (HTOK == 64 ? 6 : 3) * 2 * HTOK * D * 2 + 2 * 6 * 8 + (HTOK / 16) * kMaxR * (D + 4) * 4 +
           (HTOK / 16) * kMaxR * 2 * 4 + 256;
}

template <int R, int HTOK>
__global__ void __launch_bounds__(32 + 2 * HTOK, 1) k_hmma(const Args a) {
    constexpr int kHTok = HTOK, kHStages = HTOK == 64 ? 6 : 3, kCW = HTOK / 16;
    extern __shared__ __align__(16) uint8_t sraw[];
    uint8_t* ring = sraw + ((1024u - (ptx::smem_u32(sraw) & 1023u)) & 1023u);
    constexpr uint32_t kTile = kHTok * D * 2, kStage = 2 * kTile;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + kHStages * kStage);
    uint64_t* empty = full + kHStages;
    float* so = reinterpret_cast<float*>(empty + kHStages);  // [kCW][8][D+4]
    float* sml = so + kCW * kMaxR * (D + 4);                 // [kCW][8][2]
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint32_t u, t0, t1;
    cta_range(a, u, t0, t1);
    if (t0 >= t1) {
        write_empty(a);
        return;
    }
    if (tid == 0) {
        for (int s = 0; s < kHStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], kCW);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) produce<kHStages, kHTok>(a, ring, full, empty, u, t0, t1);
    } else {
        const int cw = warp - 1, tb = cw * 16;
        const int grp = lane >> 2, qd = lane & 3, lj = lane >> 3, li = lane & 7;
        const uint32_t k_tok = tb + ((lj >> 1) << 3) + li, k_csel = lj & 1;
        const uint32_t v_tok = tb + ((lj & 1) << 3) + li, v_csel = lj >> 1;
        uint32_t qa[8][4];
        {
            const bool live = grp < R;
            const float* qrow = a.q + (size_t(u) * R + (live ? grp : 0)) * D;
            for (int kk = 0; kk < 8; ++kk) {
                float2 x = make_float2(0.f, 0.f), y = make_float2(0.f, 0.f);
                if (live) {
                    x = *reinterpret_cast<const float2*>(qrow + 16 * kk + 2 * qd);
                    y = *reinterpret_cast<const float2*>(qrow + 16 * kk + 8 + 2 * qd);
                }
                x.x *= a.qscale; x.y *= a.qscale; y.x *= a.qscale; y.y *= a.qscale;
                const uint32_t xh = ptx::pack_bf16(x.x, x.y), yh = ptx::pack_bf16(y.x, y.y);
                qa[kk][0] = xh;
                qa[kk][1] = ptx::pack_bf16(x.x - ptx::bf16_lo_as_f32(xh), x.y - ptx::bf16_hi_as_f32(xh));
                qa[kk][2] = yh;
                qa[kk][3] = ptx::pack_bf16(y.x - ptx::bf16_lo_as_f32(yh), y.y - ptx::bf16_hi_as_f32(yh));
            }
        }
        float o[16][4];
        for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
        float m_used = -INFINITY, l_acc = 0.f;
        int s = 0;
        uint32_t ph = 0;
        for (uint32_t tk = t0; tk < t1; tk += kHTok) {
            ptx::mbar_wait(&full[s], ph);
            const uint32_t kbase = ptx::smem_u32(ring + s * kStage), vbase = kbase + kTile;
            float sacc[2][2][4];
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
                for (int y = 0; y < 2; ++y) sacc[x][y][0] = sacc[x][y][1] = sacc[x][y][2] = sacc[x][y][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                uint32_t b[4];
                ptx::ldsm_x4(b, kbase + swz<kHTok>(k_tok, 2 * kk + k_csel));
                ptx::mma_bf16(sacc[0][kk & 1], qa[kk], b[0], b[1]);
                ptx::mma_bf16(sacc[1][kk & 1], qa[kk], b[2], b[3]);
            }
            float sc[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int nt = j >> 1, col = j & 1;
                sc[j] = (sacc[nt][0][col] + sacc[nt][1][col]) + (sacc[nt][0][col + 2] + sacc[nt][1][col + 2]);
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
                for (int i = 0; i < 16; ++i) {
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
            for (int nn = 0; nn < 8; ++nn) {
                uint32_t b[4];
                ptx::ldsm_x4_t(b, vbase + swz<kHTok>(v_tok, 2 * nn + v_csel));
                ptx::mma_bf16(o[2 * nn], pa, b[0], b[1]);
                ptx::mma_bf16(o[2 * nn + 1], pa, b[2], b[3]);
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&empty[s]);
            if (++s == kHStages) {
                s = 0;
                ph ^= 1u;
            }
        }
        float l_tot = l_acc + __shfl_xor_sync(0xffffffffu, l_acc, 1);
        l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 2);
        if (grp < R) {
            float* w = so + (cw * kMaxR + grp) * (D + 4);
            for (int nt = 0; nt < 16; ++nt) {
                w[8 * nt + 2 * qd] = o[nt][0] + o[nt][2];
                w[8 * nt + 2 * qd + 1] = o[nt][1] + o[nt][3];
            }
            if (qd == 0) {
                sml[(cw * kMaxR + grp) * 2] = m_used;
                sml[(cw * kMaxR + grp) * 2 + 1] = l_tot;
            }
        }
    }
    __syncthreads();
    float* P = a.part + size_t(blockIdx.x) * kPartFloats;
    for (uint32_t idx = tid; idx < (uint32_t)(kMaxR * D); idx += blockDim.x) {
        const uint32_t h = idx / D, d = idx % D;
        if (h >= (uint32_t)R) {
            P[2 * kMaxR + idx] = 0.f;
            if (d == 0) { P[h] = -INFINITY; P[kMaxR + h] = 0.f; }
            continue;
        }
        float mx = -INFINITY;
        for (int w = 0; w < kCW; ++w) mx = fmaxf(mx, sml[(w * kMaxR + h) * 2]);
        float acc = 0.f, ls = 0.f;
        for (int w = 0; w < kCW; ++w) {
            const float m = sml[(w * kMaxR + h) * 2];
            const float sc = m == -INFINITY ? 0.f : ptx::ex2(m - mx);
            acc += so[(w * kMaxR + h) * (D + 4) + d] * sc;
            ls += sml[(w * kMaxR + h) * 2 + 1] * sc;
        }
        P[2 * kMaxR + idx] = acc;
        if (d == 0) { P[h] = mx; P[kMaxR + h] = ls; }
    }
}

// ============================ variant fma ===================================
// QK: thread t -> token t/2 of the 64-token stage, dims [64 (t%2), +64);
// PV: thread t -> dims [4 (t%32), +4) of heads t/32 (+4).  Two named barriers
// per stage.  Exact bf16 -> fp32 K/V, fp32 q, fp32 P.
constexpr int kFStages = 6, kFTok = 64;
constexpr int kFSmem = 1024 + kFStages * 2 * kFTok * D * 2 + 2 * kFStages * 8 + kMaxR * 2 * (64 + 4) * 4 +
                       kFTok * kMaxR * 4 + 4 * kMaxR * 4 + 4 * kMaxR * 4 + 256;

__device__ __forceinline__ void bf8_to_f(const uint4 v, float (&f)[8]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}

template <int R>
__global__ void __launch_bounds__(160, 1) k_fma(const Args a) {
    extern __shared__ __align__(16) uint8_t sraw[];
    uint8_t* ring = sraw + ((1024u - (ptx::smem_u32(sraw) & 1023u)) & 1023u);
    constexpr uint32_t kTile = kFTok * D * 2, kStage = 2 * kTile;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + kFStages * kStage);
    uint64_t* empty = full + kFStages;
    float* qs = reinterpret_cast<float*>(empty + kFStages);  // [R][2][64+4]
    float* ps = qs + kMaxR * 2 * 68;                          // [64 tok][8]
    float* wmax = ps + kFTok * kMaxR;                          // [4 warps][8]
    float* lsh = wmax + 4 * kMaxR;                             // [4 warps][8]
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint32_t u, t0, t1;
    cta_range(a, u, t0, t1);
    if (t0 >= t1) {
        write_empty(a);
        return;
    }
    if (tid == 0) {
        for (int s = 0; s < kFStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::fence_mbar_init();
    }
    for (uint32_t i = tid; i < (uint32_t)(R * D); i += blockDim.x) {
        const uint32_t h = i / D, d = i % D;
        qs[(h * 2 + d / 64) * 68 + d % 64] = a.q[size_t(u) * R * D + i] * a.qscale;
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) produce<kFStages, kFTok>(a, ring, full, empty, u, t0, t1);
        return;
    }
    const uint32_t ct = tid - 32, cw = warp - 1;
    const uint32_t tok = ct >> 1, half = ct & 1;  // QK role
    constexpr int kHP = R > 4 ? 2 : 1;             // PV role: heads per thread
    const uint32_t pd = 4 * (ct & 31), ph0 = ct >> 5;
    float acc[kHP][4];
    for (int i = 0; i < kHP; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    float m_used[R], l_thr[R];
    for (int h = 0; h < R; ++h) { m_used[h] = -INFINITY; l_thr[h] = 0.f; }
    int s = 0;
    uint32_t ph = 0;
    for (uint32_t tk = t0; tk < t1; tk += kFTok) {
        ptx::mbar_wait(&full[s], ph);
        const uint8_t* kt = ring + s * kStage;
        const uint8_t* vt = kt + kTile;
        // QK: dot of my half row with every head
        float kf[64];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const uint4 v = *reinterpret_cast<const uint4*>(kt + half * (kFTok * 128) + tok * 128 + ((c ^ (tok & 7)) << 4));
            float f[8];
            bf8_to_f(v, f);
#pragma unroll
            for (int e = 0; e < 8; ++e) kf[8 * c + e] = f[e];
        }
        float z[R];
#pragma unroll
        for (int h = 0; h < R; ++h) {
            const float4* qr = reinterpret_cast<const float4*>(qs + (h * 2 + half) * 68);
            float d0 = 0.f, d1 = 0.f;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const float4 qv = qr[c];
                d0 = fmaf(qv.x, kf[4 * c], d0);
                d1 = fmaf(qv.y, kf[4 * c + 1], d1);
                d0 = fmaf(qv.z, kf[4 * c + 2], d0);
                d1 = fmaf(qv.w, kf[4 * c + 3], d1);
            }
            z[h] = d0 + d1;
            z[h] += __shfl_xor_sync(0xffffffffu, z[h], 1);
        }
        // tile max per head over the 64 tokens (16 per warp), shared
#pragma unroll
        for (int h = 0; h < R; ++h) {
            float mx = z[h];
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
            if (lane == 0) wmax[cw * kMaxR + h] = mx;
        }
        ptx::named_bar_sync(1, 128);
        float alpha[R];
#pragma unroll
        for (int h = 0; h < R; ++h) {
            const float tmax = fmaxf(fmaxf(wmax[h], wmax[kMaxR + h]), fmaxf(wmax[2 * kMaxR + h], wmax[3 * kMaxR + h]));
            alpha[h] = 1.f;
            if (tmax > m_used[h] + 8.f) {  // uniform over the CTA
                alpha[h] = m_used[h] == -INFINITY ? 0.f : ptx::ex2(m_used[h] - tmax);
                m_used[h] = tmax;
            }
            const float p = ptx::ex2(z[h] - m_used[h]);
            if (half == 0) {
                ps[tok * kMaxR + h] = p;
                l_thr[h] = l_thr[h] * alpha[h] + p;
            }
        }
#pragma unroll
        for (int i = 0; i < kHP; ++i) {
            float al = 1.f;
#pragma unroll
            for (int h = 0; h < R; ++h)
                if ((uint32_t)h == ph0 + 4 * i) al = alpha[h];
            acc[i][0] *= al; acc[i][1] *= al; acc[i][2] *= al; acc[i][3] *= al;
        }
        ptx::named_bar_sync(1, 128);
        // PV: my 4 dims of my head(s) over the 64 tokens
        const uint32_t vb = (pd >> 6) * (kFTok * 128), vc = (pd & 63) >> 3, vo = (pd & 7) * 2;
#pragma unroll 8
        for (uint32_t t = 0; t < (uint32_t)kFTok; ++t) {
            const uint2 v = *reinterpret_cast<const uint2*>(vt + vb + t * 128 + ((vc ^ (t & 7)) << 4) + vo);
            const float v0 = __uint_as_float(v.x << 16), v1 = __uint_as_float(v.x & 0xFFFF0000u);
            const float v2 = __uint_as_float(v.y << 16), v3 = __uint_as_float(v.y & 0xFFFF0000u);
#pragma unroll
            for (int i = 0; i < kHP; ++i) {
                const uint32_t h = ph0 + 4 * i;
                if (h < (uint32_t)R) {
                    const float p = ps[t * kMaxR + h];
                    acc[i][0] = fmaf(p, v0, acc[i][0]);
                    acc[i][1] = fmaf(p, v1, acc[i][1]);
                    acc[i][2] = fmaf(p, v2, acc[i][2]);
                    acc[i][3] = fmaf(p, v3, acc[i][3]);
                }
            }
        }
        ptx::named_bar_sync(1, 128);  // ps / wmax reused next stage; stage consumed
        if (ct == 0) ptx::mbar_arrive(&empty[s]);
        if (++s == kFStages) {
            s = 0;
            ph ^= 1u;
        }
    }
    // l: sum over the token threads (half 0) of each head
#pragma unroll
    for (int h = 0; h < R; ++h) {
        float l = half == 0 ? l_thr[h] : 0.f;
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
        if (lane == 0) lsh[cw * kMaxR + h] = l;
    }
    ptx::named_bar_sync(1, 128);
    float* P = a.part + size_t(blockIdx.x) * kPartFloats;
#pragma unroll
    for (int i = 0; i < kHP; ++i) {
        const uint32_t h = ph0 + 4 * i;
        if (h < (uint32_t)R) {
            float* pa = P + 2 * kMaxR + h * D + pd;
            pa[0] = acc[i][0]; pa[1] = acc[i][1]; pa[2] = acc[i][2]; pa[3] = acc[i][3];
        }
    }
    if (ct == 0) {
#pragma unroll
        for (int h = 0; h < R; ++h) {
            P[h] = m_used[h];
            P[kMaxR + h] = lsh[h] + lsh[kMaxR + h] + lsh[2 * kMaxR + h] + lsh[3 * kMaxR + h];
        }
        for (int h = R; h < kMaxR; ++h) { P[h] = -INFINITY; P[kMaxR + h] = 0.f; }
    }
    for (uint32_t i = ct; i < (uint32_t)((kMaxR - R) * D); i += 128) P[2 * kMaxR + R * D + i] = 0.f;
}

// ============================ variant tc05 ==================================
constexpr int kTStages = 3, kTTok = 128;
constexpr uint32_t kTTile = kTTok * D * 2, kTStage = 2 * kTTile;  // 32 KB + 32 KB
// smem: ring | Qhl (2 boxes of 16 rows x 128 B) | P^T x2 (2 boxes of 16 x 128 B) | bars | misc
constexpr int kTOffQ = kTStages * kTStage;
constexpr int kTOffP = kTOffQ + 4096;
constexpr int kTOffBar = kTOffP + 2 * 4096;
constexpr int kTOffMisc = kTOffBar + 32 * 8;
constexpr int kTSmem = 1024 + kTOffMisc + 1024;

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    // tcgen05 shared-memory matrix descriptor, SWIZZLE_128B, version 1
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     ptx::smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
        "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
        "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// bf16 of (n, k) in a K-major SW128 operand made of 64-wide boxes of `rows` rows
__device__ __forceinline__ uint32_t kmaj_off(uint32_t n, uint32_t k, uint32_t rows) {
    const uint32_t box = k >> 6, kk = k & 63;
    return box * rows * 128 + n * 128 + ((((kk >> 3) ^ (n & 7)) << 4) | ((kk & 7) << 1));
}

template <int R>
__global__ void __launch_bounds__(256, 1) k_tc05(const Args a) {
    extern __shared__ __align__(16) uint8_t sraw[];
    uint8_t* sm = sraw + ((1024u - (ptx::smem_u32(sraw) & 1023u)) & 1023u);
    uint8_t* ring = sm;
    uint8_t* qb = sm + kTOffQ;
    uint8_t* pb = sm + kTOffP;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kTOffBar);
    uint64_t* full = bars;            // [3] TMA -> MMA
    uint64_t* empty = bars + 3;       // [3] MMA (PV commit) -> TMA
    uint64_t* sfull = bars + 6;       // [2] MMA (QK commit) -> softmax
    uint64_t* sfree = bars + 8;       // [2] softmax read S -> MMA
    uint64_t* pfull = bars + 10;      // [2] softmax wrote P -> MMA
    uint64_t* pfree = bars + 12;      // [2] MMA (PV commit) -> softmax
    uint32_t* misc = reinterpret_cast<uint32_t*>(sm + kTOffMisc);  // [0] tmem base
    float* wmax = reinterpret_cast<float*>(misc + 4);               // [4][8]
    float* lsh = wmax + 32;                                         // [4][8]
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint32_t u, t0, t1;
    cta_range(a, u, t0, t1);
    if (t0 >= t1) {
        write_empty(a);
        return;
    }
    const uint32_t nst = (t1 - t0) / kTTok;  // ranges are stage multiples
    if (tid == 0) {
        for (int s = 0; s < kTStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&sfull[b], 1);
            ptx::mbar_init(&sfree[b], 4);
            ptx::mbar_init(&pfull[b], 4);
            ptx::mbar_init(&pfree[b], 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) {  // TMEM: S0 cols 0-15, S1 16-31, O 32-47
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(ptx::smem_u32(misc)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // Qhl^T operand (B of QK): rows n = 0..7 hi, 8..15 lo of heads (0 past R),
    // K-major over the 128 dims; P^T buffers: rows past R stay 0
    for (uint32_t i = tid; i < 16 * D; i += blockDim.x) {
        const uint32_t n = i / D, k = i % D, h = n & 7;
        float x = 0.f;
        if (h < (uint32_t)R) x = a.q[(size_t(u) * R + h) * D + k] * a.qscale;
        const __nv_bfloat16 hi = __float2bfloat16_rn(x);
        const __nv_bfloat16 v = n < 8 ? hi : __float2bfloat16_rn(x - __bfloat162float(hi));
        *reinterpret_cast<__nv_bfloat16*>(qb + kmaj_off(n, k, 16)) = v;
    }
    for (uint32_t i = tid; i < 2 * 4096 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(pb)[i] = 0u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = misc[0];
    // instruction descriptors: bf16 x bf16 -> f32, M = 128, N = 16
    constexpr uint32_t kIdBase = (1u << 4) | (1u << 7) | (1u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
    constexpr uint32_t kIdQK = kIdBase;              // A (K tile) K-major, B (Qhl) K-major
    constexpr uint32_t kIdPV = kIdBase | (1u << 15);  // A (V tile as V^T) MN-major, B (P^T) K-major

    if (warp == 0) {
        if (lane == 0) produce<kTStages, kTTok>(a, ring, full, empty, u, t0, t1);
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t qaddr = ptx::smem_u32(qb);
            auto issue_qk = [&](uint32_t i) {
                const uint32_t s = i % kTStages, sb = i & 1;
                ptx::mbar_wait(&full[s], (i / kTStages) & 1u);
                if (i >= 2) ptx::mbar_wait(&sfree[sb], ((i >> 1) - 1) & 1u);
                tc_fence_after();
                const uint32_t kaddr = ptx::smem_u32(ring + s * kTStage);
#pragma unroll
                for (uint32_t k = 0; k < 8; ++k) {  // 16 dims per MMA
                    const uint32_t ko = (k >> 2) * (kTTok * 128) + (k & 3) * 32;
                    const uint32_t qo = (k >> 2) * (16 * 128) + (k & 3) * 32;
                    umma_f16(tmem + sb * 16, sdesc(kaddr + ko, 16, 1024), sdesc(qaddr + qo, 16, 1024), kIdQK, k > 0);
                }
                umma_commit(&sfull[sb]);
            };
            if (nst > 0) issue_qk(0);
            for (uint32_t i = 0; i < nst; ++i) {
                const uint32_t s = i % kTStages, sb = i & 1;
                if (i + 1 < nst) issue_qk(i + 1);
                ptx::mbar_wait(&pfull[sb], (i >> 1) & 1u);
                tc_fence_after();
                const uint32_t vaddr = ptx::smem_u32(ring + s * kTStage + kTTile);
                const uint32_t paddr = ptx::smem_u32(pb + sb * 4096);
#pragma unroll
                for (uint32_t k = 0; k < 8; ++k) {  // 16 tokens per MMA
                    const uint32_t vo = k * 16 * 128;                          // 16 rows of 128 B
                    const uint32_t po = (k >> 2) * (16 * 128) + (k & 3) * 32;  // P^T: 64-token boxes
                    umma_f16(tmem + 32, sdesc(vaddr + vo, kTTok * 128, 1024), sdesc(paddr + po, 16, 1024), kIdPV,
                             (i > 0 || k > 0) ? 1u : 0u);
                }
                umma_commit(&empty[s]);
                umma_commit(&pfree[sb]);
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        const uint32_t qw = warp & 3;  // TMEM lane quarter
        const uint32_t row = 32 * qw + lane;  // token within the stage (S), dim (O)
        float m_used[R], l_thr[R];
#pragma unroll
        for (int h = 0; h < R; ++h) { m_used[h] = -INFINITY; l_thr[h] = 0.f; }
        for (uint32_t i = 0; i < nst; ++i) {
            const uint32_t sb = i & 1;
            ptx::mbar_wait(&sfull[sb], (i >> 1) & 1u);
            tc_fence_after();
            float sv[16];
            tmem_ld16(tmem + ((32 * qw) << 16) + sb * 16, sv);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&sfree[sb]);
            float z[R];
#pragma unroll
            for (int h = 0; h < R; ++h) {
                z[h] = sv[h] + sv[h + 8];
                float mx = z[h];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                if (lane == 0) wmax[qw * 8 + h] = mx;
            }
            ptx::named_bar_sync(1, 128);
            float alpha[R];
            bool resc = false;
#pragma unroll
            for (int h = 0; h < R; ++h) {
                const float tmax = fmaxf(fmaxf(wmax[h], wmax[8 + h]), fmaxf(wmax[16 + h], wmax[24 + h]));
                alpha[h] = 1.f;
                if (tmax > m_used[h] + 8.f) {  // uniform over the 128 threads
                    alpha[h] = m_used[h] == -INFINITY ? 0.f : ptx::ex2(m_used[h] - tmax);
                    m_used[h] = tmax;
                    resc = true;
                }
                l_thr[h] *= alpha[h];
            }
            ptx::named_bar_sync(1, 128);  // wmax reused next stage
            // the P buffer of stage i was last read by PV(i - 2); O is stable
            // once PV(i - 1) completed (needed for a rescale)
            if (i >= 1) {
                const uint32_t pi = i - 1;
                ptx::mbar_wait(&pfree[pi & 1], (pi >> 1) & 1u);
            }
            tc_fence_after();
            if (resc && i > 0) {
                float ov[16];
                const uint32_t oaddr = tmem + ((32 * qw) << 16) + 32;
                tmem_ld16(oaddr, ov);
#pragma unroll
                for (int h = 0; h < R; ++h) {
                    ov[h] *= alpha[h];
                    ov[h + 8] *= alpha[h];
                }
                tmem_st16(oaddr, ov);
            }
            uint8_t* pbuf = pb + sb * 4096;
#pragma unroll
            for (int h = 0; h < R; ++h) {
                const float p = ptx::ex2(z[h] - m_used[h]);
                l_thr[h] += p;
                const __nv_bfloat16 hi = __float2bfloat16_rn(p);
                const __nv_bfloat16 lo = __float2bfloat16_rn(p - __bfloat162float(hi));
                *reinterpret_cast<__nv_bfloat16*>(pbuf + kmaj_off(h, row, 16)) = hi;
                *reinterpret_cast<__nv_bfloat16*>(pbuf + kmaj_off(8 + h, row, 16)) = lo;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&pfull[sb]);
        }
        // final: O^T lanes = dims, columns h (hi) + h + 8 (lo)
        if (nst > 0) {
            const uint32_t li = nst - 1;
            ptx::mbar_wait(&pfree[li & 1], (li >> 1) & 1u);
        }
        tc_fence_after();
        float ov[16];
        tmem_ld16(tmem + ((32 * qw) << 16) + 32, ov);
        float* P = a.part + size_t(blockIdx.x) * kPartFloats;
#pragma unroll
        for (int h = 0; h < kMaxR; ++h) P[2 * kMaxR + h * D + row] = h < R ? ov[h] + ov[h + 8] : 0.f;
#pragma unroll
        for (int h = 0; h < R; ++h) {
            float l = l_thr[h];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
            if (lane == 0) lsh[qw * 8 + h] = l;
        }
        ptx::named_bar_sync(1, 128);
        if (qw == 0 && lane == 0) {
#pragma unroll
            for (int h = 0; h < kMaxR; ++h) {
                P[h] = h < R ? m_used[h < R ? h : 0] : -INFINITY;
                P[kMaxR + h] = h < R ? lsh[h] + lsh[8 + h] + lsh[16 + h] + lsh[24 + h] : 0.f;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------
__global__ void fill_bf16(__nv_bfloat16* p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t x = (uint32_t)i * 2654435761u ^ seed;
        x ^= x >> 15; x *= 0x2c1b3c6du; x ^= x >> 12; x *= 0x297a2d39u; x ^= x >> 15;
        const float uni = (x & 0xFFFFFF) * (1.0f / 16777216.0f) - 0.5f;  // U(-0.5, 0.5)
        p[i] = __float2bfloat16_rn(uni * 3.4641016f);                   // unit variance
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}
static void make_map(CUtensorMap* m, void* base, size_t rows, uint32_t box_rows) {
    const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)(D * 2)};
    const cuuint32_t box[2] = {64, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult rc = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) { printf("tensor map encode failed %d\n", (int)rc); exit(1); }
}

static float bf2f(uint16_t b) { uint32_t x = (uint32_t)b << 16; float f; memcpy(&f, &x, 4); return f; }

struct Run {
    std::string name;
    int R;
};

int main(int argc, char** argv) {
    const uint32_t L = argc > 1 ? atoi(argv[1]) : 524288;
    const uint32_t nact = argc > 2 ? atoi(argv[2]) : 3;
    const std::string which = argc > 3 ? argv[3] : "all";
    const int Rsel = argc > 4 ? atoi(argv[4]) : 0;
    const bool once = argc > 5 && std::string(argv[5]) == "once";  // one launch per variant (ncu)
    int G;
    CK(cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, 0));
    const uint32_t Lchk = 8192;
    const size_t rows = size_t(nact) * L;
    __nv_bfloat16 *dk, *dv;
    CK(cudaMalloc(&dk, rows * D * 2));
    CK(cudaMalloc(&dv, rows * D * 2));
    fill_bf16<<<1024, 256>>>(dk, rows * D, 0x1234u);
    fill_bf16<<<1024, 256>>>(dv, rows * D, 0x9876u);
    float* dq;
    CK(cudaMalloc(&dq, nact * kMaxR * D * 4));
    std::vector<float> hq(nact * kMaxR * D);
    for (size_t i = 0; i < hq.size(); ++i) hq[i] = (float)((std::sin(0.37 * i + 1.1) + std::cos(0.011 * i)) * 0.9);
    CK(cudaMemcpy(dq, hq.data(), hq.size() * 4, cudaMemcpyHostToDevice));
    float* dpart;
    CK(cudaMalloc(&dpart, size_t(G) * kPartFloats * 4));
    CUtensorMap maps[4];
    make_map(&maps[0], dk, rows, 64);
    make_map(&maps[1], dv, rows, 64);
    make_map(&maps[2], dk, rows, 128);
    make_map(&maps[3], dv, rows, 128);
    CUtensorMap* dmaps;
    CK(cudaMalloc(&dmaps, sizeof(maps)));
    CK(cudaMemcpy(dmaps, maps, sizeof(maps), cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(k_hmma<4, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, hmma_smem<64>()));
    CK(cudaFuncSetAttribute(k_hmma<8, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, hmma_smem<64>()));
    CK(cudaFuncSetAttribute(k_hmma<4, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, hmma_smem<128>()));
    CK(cudaFuncSetAttribute(k_hmma<8, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, hmma_smem<128>()));
    CK(cudaFuncSetAttribute(k_fma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmem));
    CK(cudaFuncSetAttribute(k_fma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmem));
    CK(cudaFuncSetAttribute(k_tc05<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTSmem));
    CK(cudaFuncSetAttribute(k_tc05<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTSmem));
    CK(cudaDeviceSynchronize());

    auto launch = [&](const std::string& v, int R, uint32_t Lrun) {
        Args a{};
        a.q = dq;
        a.part = dpart;
        a.nact = nact;
        a.L = Lrun;
        a.qscale = (float)(1.4426950408889634 / std::sqrt((double)D));
        // the kernels address unit u at rows [u * Lrun, ...): use the first
        // nact * Lrun rows of the same buffers
        if (v == "tc05") {
            a.tmk = dmaps + 2; a.tmv = dmaps + 3; a.stage_tok = kTTok;
            if (R == 4) k_tc05<4><<<G, 256, kTSmem>>>(a); else k_tc05<8><<<G, 256, kTSmem>>>(a);
        } else if (v == "fma") {
            a.tmk = dmaps; a.tmv = dmaps + 1; a.stage_tok = kFTok;
            if (R == 4) k_fma<4><<<G, 160, kFSmem>>>(a); else k_fma<8><<<G, 160, kFSmem>>>(a);
        } else if (v == "hmma128") {
            a.tmk = dmaps + 2; a.tmv = dmaps + 3; a.stage_tok = 128;
            if (R == 4) k_hmma<4, 128><<<G, 288, hmma_smem<128>()>>>(a);
            else k_hmma<8, 128><<<G, 288, hmma_smem<128>()>>>(a);
        } else {
            a.tmk = dmaps; a.tmv = dmaps + 1; a.stage_tok = 64;
            if (R == 4) k_hmma<4, 64><<<G, 160, hmma_smem<64>()>>>(a);
            else k_hmma<8, 64><<<G, 160, hmma_smem<64>()>>>(a);
        }
        CK(cudaGetLastError());
    };
    // fp64 reference at Lchk: unit u = rows [u * Lchk, (u + 1) * Lchk)
    std::vector<uint16_t> hk(size_t(nact) * Lchk * D), hv(hk.size());
    CK(cudaMemcpy(hk.data(), dk, hk.size() * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hv.data(), dv, hv.size() * 2, cudaMemcpyDeviceToHost));
    std::vector<std::string> vars;
    for (const char* v : {"hmma", "hmma128", "fma", "tc05"})
        if (which == "all" || which == v) vars.push_back(v);
    std::vector<int> Rs;
    if (Rsel == 4 || Rsel == 0) Rs.push_back(4);
    if (Rsel == 8 || Rsel == 0) Rs.push_back(8);
    if (once) {
        for (int R : Rs)
            for (const auto& v : vars) launch(v, R, L);
        CK(cudaDeviceSynchronize());
        return 0;
    }
    for (int R : Rs) {
        // reference
        std::vector<double> ref(size_t(nact) * R * D);
        const double scale = 1.0 / std::sqrt((double)D);
        for (uint32_t u = 0; u < nact; ++u)
            for (int h = 0; h < R; ++h) {
                const float* q = &hq[(size_t(u) * R + h) * D];
                std::vector<double> z(Lchk);
                double mx = -1e300;
                for (uint32_t t = 0; t < Lchk; ++t) {
                    double s = 0;
                    for (int d = 0; d < D; ++d) s += (double)q[d] * bf2f(hk[(size_t(u) * Lchk + t) * D + d]);
                    z[t] = s * scale;
                    mx = std::max(mx, z[t]);
                }
                double l = 0;
                std::vector<double> o(D, 0.0);
                for (uint32_t t = 0; t < Lchk; ++t) {
                    const double p = std::exp(z[t] - mx);
                    l += p;
                    for (int d = 0; d < D; ++d) o[d] += p * bf2f(hv[(size_t(u) * Lchk + t) * D + d]);
                }
                for (int d = 0; d < D; ++d) ref[(size_t(u) * R + h) * D + d] = o[d] / l;
            }
        for (const auto& v : vars) {
            launch(v, R, Lchk);
            CK(cudaDeviceSynchronize());
            std::vector<float> part(size_t(G) * kPartFloats);
            CK(cudaMemcpy(part.data(), dpart, part.size() * 4, cudaMemcpyDeviceToHost));
            double maxerr = 0, num = 0, den = 0;
            for (uint32_t u = 0; u < nact; ++u)
                for (int h = 0; h < R; ++h) {
                    double M = -1e300;
                    for (int c = u; c < G; c += nact) M = std::max(M, (double)part[size_t(c) * kPartFloats + h]);
                    double l = 0;
                    std::vector<double> o(D, 0.0);
                    for (int c = u; c < G; c += nact) {
                        const float* P = &part[size_t(c) * kPartFloats];
                        if (P[h] == -INFINITY) continue;
                        const double w = std::exp2((double)P[h] - M);
                        l += P[kMaxR + h] * w;
                        for (int d = 0; d < D; ++d) o[d] += P[2 * kMaxR + h * D + d] * w;
                    }
                    for (int d = 0; d < D; ++d) {
                        const double g = o[d] / l, r = ref[(size_t(u) * R + h) * D + d];
                        maxerr = std::max(maxerr, std::fabs(g - r));
                        num += (g - r) * (g - r);
                        den += r * r;
                    }
                }
            const double rel = std::sqrt(num / den);
            printf("check R=%d %-5s L=%u: max-abs %.3e rel-L2 %.3e %s\n", R, v.c_str(), Lchk, maxerr, rel,
                   (maxerr <= 2e-3 && rel <= 1e-3) ? "ok" : "FAIL");
        }
        // timing at L
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        for (const auto& v : vars) {
            for (int i = 0; i < 3; ++i) launch(v, R, L);
            CK(cudaDeviceSynchronize());
            const int n = 20;
            CK(cudaEventRecord(e0));
            for (int i = 0; i < n; ++i) launch(v, R, L);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double us = ms * 1e3 / n, bytes = double(nact) * L * D * 2 * 2;
            printf("time  R=%d %-5s L=%u nact=%u: %8.2f us  %7.1f GB/s (K+V bf16 %.0f MB)\n", R, v.c_str(), L,
                   nact, us, bytes / (us * 1e-6) / 1e9, bytes / 1e6);
        }
    }
    return 0;
}
