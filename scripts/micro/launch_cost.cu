// Microbenchmark: cost of back-to-back small kernels in a CUDA graph on B200,
// with/without PDL and with a large dynamic-smem persistent kernel.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__global__ void k_small(int* p) { pdl_launch(); pdl_wait(); if (threadIdx.x == 0) atomicAdd(p, 1); }
__global__ void k_big(int* p) {
    extern __shared__ char sm[];
    pdl_launch(); pdl_wait();
    if (threadIdx.x == 0) { sm[blockIdx.x & 1023] = 1; atomicAdd(p + 1, sm[0]); }
}
__global__ void k_loads(const float* q, float* out, int n) {  // 1 CTA, one round trip of loads
    pdl_launch(); pdl_wait();
    float acc = 0; for (int i = threadIdx.x; i < n; i += blockDim.x) acc += q[i];
    if (acc == 12345.f) out[0] = acc;
}
int main() {
    int* p; cudaMalloc(&p, 64); float* q; cudaMalloc(&q, 1 << 20); cudaMemset(q, 0, 1 << 20);
    cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto launch = [&](void* fn, dim3 g, dim3 b, size_t smem, bool pdl, void** args) {
        cudaLaunchConfig_t cfg{}; cfg.gridDim = g; cfg.blockDim = b; cfg.dynamicSmemBytes = smem; cfg.stream = s;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = a; cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelExC(&cfg, fn, args);
    };
    int n = 4096;
    void* a_small[] = {&p}; void* a_loads[] = {&q, &q, &n};
    const char* names[] = {"1 small", "3 small", "small+big+small", "small+big+small PDL", "loads+big+small PDL", "big only", "big only x3 PDL"};
    for (int variant = 0; variant < 7; ++variant) {
        cudaGraph_t g; cudaGraphExec_t ex;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        bool pdl = variant == 3 || variant == 4 || variant == 6;
        if (variant == 0) launch((void*)k_small, 1, 256, 0, false, a_small);
        if (variant == 1) for (int i = 0; i < 3; ++i) launch((void*)k_small, 1, 256, 0, false, a_small);
        if (variant >= 2 && variant <= 4) {
            launch(variant == 4 ? (void*)k_loads : (void*)k_small, 1, 256, 0, false, variant == 4 ? a_loads : a_small);
            launch((void*)k_big, 148, 160, 210 * 1024, pdl, a_small);
            launch((void*)k_small, dim3(8, 4), 256, 0, pdl, a_small);
        }
        if (variant == 5) launch((void*)k_big, 148, 160, 210 * 1024, false, a_small);
        if (variant == 6) for (int i = 0; i < 3; ++i) launch((void*)k_big, 148, 160, 210 * 1024, i > 0, a_small);
        cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ex, g, 0);
        for (int i = 0; i < 20; ++i) cudaGraphLaunch(ex, s);
        cudaStreamSynchronize(s);
        cudaEventRecord(e0, s);
        for (int i = 0; i < 200; ++i) cudaGraphLaunch(ex, s);
        cudaEventRecord(e1, s); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-28s %7.2f us/graph\n", names[variant], ms * 1e3 / 200);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
