// microbenchmark: host-side cost of the blocking C-ABI step (no Python).
// build: g++ -O2 -std=c++17 e2e_cabi.cpp -I../../include -L../../paper_2604_16883_b200/_lib
//        -lsinkr_cuda -lcudart -L/usr/local/cuda/lib64 -Wl,-rpath,...
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "sinkr_cuda.h"
using clk = std::chrono::steady_clock;
#define OK(x) do { if ((x) != SINKR_OK) { printf("err %s\n", sinkr_last_error()); return 1; } } while (0)
int main(int argc, char** argv) {
    const size_t L = argc > 1 ? atol(argv[1]) : 32768;
    sinkr_cache_config c{1, 32, 8, 128, L, 1};
    sinkr_engine* e;
    OK(sinkr_engine_create(&c, 0, &e));
    for (size_t g = 0; g < 8; ++g) OK(sinkr_kv_append_synthetic(e, 0, 0, g, 11 + g, 99 + g, 1.f, 1.f, 0, L));
    std::vector<float> q(32 * 128, 0.3f), out(32 * 128);
    std::vector<double> hs(32);
    std::vector<sinkr_group_info> gi(8);
    sinkr_load_counters ctr;
    sinkr_set_timing(e, 0);
    for (double tau : {-2.0, 2.0}) {
        sinkr_routing_config rc{};
        rc.profile.coeffs[3] = tau;
        rc.profile.length_normalizer = 1.0;
        rc.profile.clamp_lo = tau < 0 ? tau : 0.0;
        rc.profile.clamp_hi = tau > 1 ? tau : 1.0;
        for (int i = 0; i < 50; ++i)
            OK(sinkr_routed_decode_step(e, q.data(), 0, &rc, nullptr, out.data(), gi.data(), hs.data(), &ctr));
        const int n = 500;
        auto t0 = clk::now();
        for (int i = 0; i < n; ++i)
            OK(sinkr_routed_decode_step(e, q.data(), 0, &rc, nullptr, out.data(), gi.data(), hs.data(), &ctr));
        auto t1 = clk::now();
        // async path with device buffers: launch + sync only
        float *dq, *dout;
        cudaMalloc(&dq, q.size() * 4); cudaMalloc(&dout, q.size() * 4);
        cudaMemcpy(dq, q.data(), q.size() * 4, cudaMemcpyHostToDevice);
        cudaStream_t s = (cudaStream_t)sinkr_engine_stream(e);
        for (int i = 0; i < 50; ++i) { OK(sinkr_routed_decode_async(e, dq, 0, &rc, nullptr, dout)); cudaStreamSynchronize(s); }
        double launch = 0;
        auto t2 = clk::now();
        for (int i = 0; i < n; ++i) {
            auto a = clk::now();
            OK(sinkr_routed_decode_async(e, dq, 0, &rc, nullptr, dout));
            launch += std::chrono::duration<double, std::micro>(clk::now() - a).count();
            cudaStreamSynchronize(s);
        }
        auto t3 = clk::now();
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        for (int i = 0; i < n; ++i) OK(sinkr_routed_decode_async(e, dq, 0, &rc, nullptr, dout));
        cudaEventRecord(e1, s); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("tau=%5.1f  step(host bufs) %.2f us | async launch %.2f us + sync -> %.2f us | device b2b %.2f us\n", tau,
               std::chrono::duration<double, std::micro>(t1 - t0).count() / n, launch / n,
               std::chrono::duration<double, std::micro>(t3 - t2).count() / n, ms * 1e3 / n);
        cudaFree(dq); cudaFree(dout);
    }
    sinkr_engine_destroy(e);
}
