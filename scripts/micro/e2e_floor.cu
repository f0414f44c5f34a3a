// microbenchmark: the host round-trip floor of a blocking decode call on this
// box, next to the engine's own blocking call (sinkr_routed_decode_step).
//   empty kernel + cudaStreamSynchronize
//   empty kernel writing a mapped completion word, host spins on it
//   graph [16 KB pinned H2D copy -> kernel writing the word], host spins
//   the engine: all-sink step (no KV streamed) and a routed step, blocking,
//   and the same steps back to back on the device (CUDA events)
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../include \
//        e2e_floor.cu -L../../paper_2604_16883_b200/_lib -lsinkr_cuda \
//        -Xlinker -rpath -Xlinker '$ORIGIN/../../paper_2604_16883_b200/_lib' -o e2e_floor
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "sinkr_cuda.h"
using clk = std::chrono::steady_clock;
#define OK(x) do { if ((x) != SINKR_OK) { printf("err %s\n", sinkr_last_error()); return 1; } } while (0)

__global__ void empty_kernel() {}
// every CTA reads the whole 16 KB query block from mapped host memory
__global__ void zc_read_kernel(const float4* hq, float* out, volatile unsigned* done, unsigned* cnt) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = threadIdx.x; i < 1040; i += blockDim.x) {
        const float4 v = hq[i];
        acc.x += v.x; acc.y += v.y;
    }
    if (acc.x == 1234.5f) out[1] = acc.y;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(cnt, 1u) == gridDim.x - 1) {
            *cnt = 0;
            __threadfence_system();
            *done = 1u;
        }
    }
}
// one CTA copies the 16 KB block from mapped host memory into device memory
__global__ void zc_copy_kernel(const float4* hq, float4* dq) {
    for (int i = threadIdx.x; i < 1040; i += blockDim.x) dq[i] = hq[i];
}
__global__ void done_kernel(const float* q, float* out, volatile unsigned* done) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        out[0] = q[0];
        __threadfence_system();
        *done = 1u;
    }
}

template <class F>
double time_us(F&& f, int n = 400) {
    for (int i = 0; i < 50; ++i) f();
    std::vector<double> ts;
    for (int i = 0; i < n; ++i) {
        auto a = clk::now();
        f();
        ts.push_back(std::chrono::duration<double, std::micro>(clk::now() - a).count());
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

int main(int argc, char** argv) {
    const size_t L = argc > 1 ? atol(argv[1]) : 524288;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    unsigned* h_done;
    cudaHostAlloc(&h_done, 64, cudaHostAllocMapped);
    unsigned* d_done;
    cudaHostGetDevicePointer(&d_done, h_done, 0);
    float *h_q, *d_q, *d_out;
    cudaHostAlloc(&h_q, 16640, cudaHostAllocDefault);
    cudaMalloc(&d_q, 16640);
    cudaMalloc(&d_out, 64);
    auto spin = [&] { while (!*(volatile unsigned*)h_done) {} std::atomic_thread_fence(std::memory_order_acquire); };
    printf("empty kernel (%d CTAs) + stream sync:        %7.2f us\n", sms,
           time_us([&] { empty_kernel<<<sms, 160, 0, s>>>(); cudaStreamSynchronize(s); }));
    printf("kernel writing a mapped word, host spin:    %7.2f us\n", time_us([&] {
               *(volatile unsigned*)h_done = 0;
               done_kernel<<<sms, 160, 0, s>>>(d_q, d_out, d_done);
               spin();
           }));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    cudaMemcpyAsync(d_q, h_q, 16640, cudaMemcpyHostToDevice, s);
    done_kernel<<<sms, 160, 0, s>>>(d_q, d_out, d_done);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    printf("graph [16 KB H2D -> kernel] + host spin:    %7.2f us\n", time_us([&] {
               *(volatile unsigned*)h_done = 0;
               cudaGraphLaunch(ge, s);
               spin();
           }));
    {
        unsigned* cnt;
        cudaMalloc(&cnt, 4);
        cudaMemset(cnt, 0, 4);
        float* hq_dev;
        cudaHostGetDevicePointer(&hq_dev, h_q, 0);
        printf("all CTAs read 16 KB zero-copy, host spin:   %7.2f us\n", time_us([&] {
                   *(volatile unsigned*)h_done = 0;
                   zc_read_kernel<<<sms, 160, 0, s>>>((const float4*)hq_dev, d_out, d_done, cnt);
                   spin();
               }));
        cudaGraph_t g2;
        cudaGraphExec_t ge2;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        zc_copy_kernel<<<1, 512, 0, s>>>((const float4*)hq_dev, (float4*)d_q);
        done_kernel<<<sms, 160, 0, s>>>(d_q, d_out, d_done);
        cudaStreamEndCapture(s, &g2);
        cudaGraphInstantiate(&ge2, g2, 0);
        printf("graph [1-CTA zero-copy upload -> kernel]:   %7.2f us\n", time_us([&] {
                   *(volatile unsigned*)h_done = 0;
                   cudaGraphLaunch(ge2, s);
                   spin();
               }));
        cudaGraph_t g3;
        cudaGraphExec_t ge3;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        cudaMemcpyAsync(d_q, h_q, 16640, cudaMemcpyHostToDevice, s);
        cudaStreamEndCapture(s, &g3);
        cudaGraphInstantiate(&ge3, g3, 0);
        printf("graph [16 KB H2D] + stream sync:            %7.2f us\n", time_us([&] {
                   cudaGraphLaunch(ge3, s);
                   cudaStreamSynchronize(s);
               }));
    }
    printf("cudaGraphLaunch API call alone:             %7.2f us\n", time_us([&] {
               *(volatile unsigned*)h_done = 0;
               auto a = clk::now();
               cudaGraphLaunch(ge, s);
               (void)a;
               cudaStreamSynchronize(s);
           }));

    sinkr_cache_config c{1, 32, 8, 128, L, 1};
    sinkr_engine* e;
    OK(sinkr_engine_create(&c, 0, &e));
    for (size_t gi = 0; gi < 8; ++gi) OK(sinkr_kv_append_synthetic(e, 0, 0, gi, 11 + gi, 99 + gi, 1.f, 1.f, 0, L));
    sinkr_set_timing(e, 0);
    std::vector<float> q(32 * 128, 0.3f), out(32 * 128);
    std::vector<double> hs(32);
    std::vector<sinkr_group_info> gi(8);
    sinkr_load_counters ctr;
    float *dq, *dout;
    cudaMalloc(&dq, q.size() * 4);
    cudaMalloc(&dout, q.size() * 4);
    cudaMemcpy(dq, q.data(), q.size() * 4, cudaMemcpyHostToDevice);
    cudaStream_t es = (cudaStream_t)sinkr_engine_stream(e);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (double tau : {-2.0, 2.0}) {
        sinkr_routing_config rc{};
        rc.profile.coeffs[3] = tau;
        rc.profile.length_normalizer = 1.0;
        rc.profile.clamp_lo = tau < 0 ? tau : 0.0;
        rc.profile.clamp_hi = tau > 1 ? tau : 1.0;
        int bad = 0;
        const double blk = time_us([&] {
            bad |= sinkr_routed_decode_step(e, q.data(), 0, &rc, nullptr, out.data(), gi.data(), hs.data(), &ctr);
        });
        for (int i = 0; i < 20; ++i) sinkr_routed_decode_async(e, dq, 0, &rc, nullptr, dout);
        cudaStreamSynchronize(es);
        cudaEventRecord(e0, es);
        for (int i = 0; i < 100; ++i) sinkr_routed_decode_async(e, dq, 0, &rc, nullptr, dout);
        cudaEventRecord(e1, es);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("engine %-8s blocking C-ABI step %8.2f us | device back to back %8.2f us | overhead %6.2f us%s\n",
               tau < 0 ? "all-sink" : "dense", blk, ms * 10.0, blk - ms * 10.0, bad ? " (errors)" : "");
    }
    sinkr_engine_destroy(e);
    return 0;
}
