// microbenchmark: how long a pure TMA-style read stream of S bytes takes on B200
// from a COLD L2 (256 MiB read-only flush kernel before each timed launch) and
// back to back, for S from 25 MB to 800 MB.  Same streaming skeleton as
// read_bw.cu (1 CTA/SM, 6 x 32 KB cp.async.bulk ring, evict_first), plus an
// empty kernel for the event/launch floor.  Calibrates the decode step's
// short-context (C1 32K, 64K-per-rank) cold numbers against the hardware.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/stream_ramp stream_ramp.cu
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(s32(b)), "r"(c)); }
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(s32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(s32(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" :: "r"(s32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 :: "r"(s32(dst)), "l"(src), "r"(n), "r"(s32(b)), "l"(pol) : "memory");
}
constexpr int STAGES = 6, BYTES = 32768;
__global__ void __launch_bounds__(160, 1) stream(const uint8_t* buf, size_t per_cta, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * BYTES);
    uint64_t* empty = full + STAGES;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    if (tid == 0) { for (int s = 0; s < STAGES; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], 4); } asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    const uint8_t* base = buf + blockIdx.x * per_cta;
    const size_t n = per_cta / BYTES;
    if (warp == 0) {
        if (lane == 0) {
            uint64_t pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            for (size_t i = 0; i < n; ++i) {
                const int s = i % STAGES; const uint32_t ph = (i / STAGES) & 1;
                mb_wait(&empty[s], ph ^ 1);
                mb_expect(&full[s], BYTES);
                bulk(sm + s * BYTES, base + i * BYTES, BYTES, &full[s], pol);
            }
        }
    } else {
        unsigned long long acc = 0;
        for (size_t i = 0; i < n; ++i) {
            const int s = i % STAGES; const uint32_t ph = (i / STAGES) & 1;
            mb_wait(&full[s], ph);
            acc += sm[s * BYTES + tid * 8];
            __syncwarp();
            if (lane == 0) mb_arrive(&empty[s]);
        }
        if (acc == 0xdeadbeef) *sink = acc;
    }
}
__global__ void flush_kernel(const int4* p, size_t n, unsigned long long* sink) {
    int4 a = make_int4(0, 0, 0, 0);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int4 v = __ldcs(p + i);
        a.x ^= v.x; a.y ^= v.y;
    }
    if (a.x == 0x12345 && a.y == 0x777) *sink = 1;
}
__global__ void empty_kernel() {}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t maxb = 1024ull << 20, fl = 256ull << 20;
    uint8_t *buf, *fb; cudaMalloc(&buf, maxb); cudaMalloc(&fb, fl);
    cudaMemset(buf, 1, maxb); cudaMemset(fb, 2, fl);
    unsigned long long* sink; cudaMalloc(&sink, 8);
    const int smem = STAGES * BYTES + 2 * STAGES * 8;
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timed = [&](auto&& fn, bool cold) {
        std::vector<float> ts;
        for (int it = 0; it < 15; ++it) {
            if (cold) flush_kernel<<<sms * 4, 512>>>((const int4*)fb, fl / 16, sink);
            cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); ts.push_back(ms * 1e3f);
        }
        std::sort(ts.begin(), ts.end());
        return ts[ts.size() / 2];
    };
    printf("empty kernel: warm %.2f us, after flush %.2f us\n",
           timed([&] { empty_kernel<<<sms, 160>>>(); }, false), timed([&] { empty_kernel<<<sms, 160>>>(); }, true));
    for (size_t mb : {25, 50, 100, 200, 400, 800}) {
        const size_t per = ((mb << 20) / sms) / BYTES * BYTES;
        auto fn = [&] { stream<<<sms, 160, smem>>>(buf, per, sink); };
        const float w = timed(fn, false), c = timed(fn, true);
        const double bytes = (double)per * sms;
        printf("%4zu MB: warm %7.2f us (%6.0f GB/s)  cold %7.2f us (%6.0f GB/s)\n", mb, w, bytes / (w * 1e-6) / 1e9, c,
               bytes / (c * 1e-6) / 1e9);
    }
    cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
}
