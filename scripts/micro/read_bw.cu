// microbenchmark: HBM read ceiling on B200 for a TMA-style streaming kernel.
// Each CTA streams a contiguous slice of a large buffer through a smem ring of
// `stages` x `bytes` with cp.async.bulk (1-D bulk copies) + mbarriers; the
// consumer warps only wait and release.  Reports GB/s for several shapes.
#include <cstdio>
#include <cstdint>
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
template <int STAGES, int BYTES>
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
template <int STAGES, int BYTES>
void run(const uint8_t* buf, size_t total, unsigned long long* sink, int ctas_per_sm) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * ctas_per_sm;
    const size_t per = (total / grid) / BYTES * BYTES;
    const int smem = STAGES * BYTES + 2 * STAGES * 8;
    cudaFuncSetAttribute(stream<STAGES, BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int it = 0; it < 6; ++it) {
        cudaEventRecord(a);
        stream<STAGES, BYTES><<<grid, 160, smem>>>(buf, per, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("stages %2d x %6d B, %d CTA/SM: %.1f GB/s (%.3f ms for %.2f GB)\n", STAGES, BYTES, ctas_per_sm,
           per * grid / (best * 1e-3) / 1e9, best, per * grid / 1e9);
}
int main() {
    const size_t total = 4ull << 30;
    uint8_t* buf; cudaMalloc(&buf, total); cudaMemset(buf, 1, total);
    unsigned long long* sink; cudaMalloc(&sink, 8);
    run<6, 32768>(buf, total, sink, 1);
    run<12, 16384>(buf, total, sink, 1);
    run<3, 65536>(buf, total, sink, 1);
    run<24, 8192>(buf, total, sink, 1);
    run<3, 32768>(buf, total, sink, 2);
    run<6, 16384>(buf, total, sink, 2);
    cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
}
