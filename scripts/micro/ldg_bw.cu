// microbenchmark: HBM read ceiling with plain vector loads (LDG.128 / LDG.E.ENL2.256
// where available) vs the TMA bulk ring of read_bw.cu.  A grid-stride XOR-reduce
// over a 4 GiB buffer; blocks x threads and unroll are swept.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int UNROLL>
__global__ void ldg_read(const uint4* __restrict__ p, size_t n, unsigned* sink) {
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (UNROLL - 1) * stride < n; i += UNROLL * stride) {
        uint4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n; i += stride) { const uint4 v = __ldcs(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
    if (acc == 0x12345678u) *sink = acc;
}

template <int UNROLL>
float run(const uint4* p, size_t n, unsigned* sink, int blocks, int threads) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) ldg_read<UNROLL><<<blocks, threads>>>(p, n, sink);
    cudaEventRecord(a);
    const int it = 10;
    for (int k = 0; k < it; ++k) ldg_read<UNROLL><<<blocks, threads>>>(p, n, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return (float)(n * 16.0 * it / (ms * 1e-3) / 1e9);
}

int main() {
    const size_t bytes = 4ull << 30, n = bytes / 16;
    uint4* p; unsigned* sink;
    cudaMalloc(&p, bytes); cudaMalloc(&sink, 4);
    cudaMemset(p, 1, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int bpsm[] = {1, 2, 4, 8};
    const int thr[] = {256, 512, 1024};
    for (int t : thr)
        for (int k : bpsm) {
            if (k * t > 2048) continue;
            printf("threads %4d blocks/SM %d: unroll4 %7.1f GB/s  unroll8 %7.1f GB/s  unroll16 %7.1f GB/s\n", t, k,
                   run<4>(p, n, sink, k * sms, t), run<8>(p, n, sink, k * sms, t), run<16>(p, n, sink, k * sms, t));
        }
    return 0;
}
