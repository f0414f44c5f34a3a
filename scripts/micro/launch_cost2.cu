// Inter-kernel gap for a persistent kernel shaped like step_kernel:
// 148 CTAs x 160 threads, ~224 KB dynamic smem, large by-value params,
// TMA descriptors as __grid_constant__, atomics + writes at exit.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
struct Big { char pad[1100]; };
__global__ void __launch_bounds__(160, 1) k_step(const __grid_constant__ CUtensorMap a, const __grid_constant__ CUtensorMap b, Big p, int* ctr, unsigned long long* t) {
    extern __shared__ char sm[];
    if (threadIdx.x == 0) { sm[threadIdx.x] = p.pad[blockIdx.x % 1000]; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long g; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
        if (blockIdx.x == 0) t[0] = g;
        if (atomicAdd(ctr, 1) == gridDim.x - 1) { *ctr = 0; unsigned long long e; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(e)); t[1] = e; }
    }
}
__global__ void __launch_bounds__(160, 1) k_plain(int* ctr) {
    extern __shared__ char sm[];
    if (threadIdx.x == 0) { sm[0] = 1; if (atomicAdd(ctr, sm[0]) == gridDim.x - 1) *ctr = 0; }
}
int main() {
    int* ctr; cudaMalloc(&ctr, 64); cudaMemset(ctr, 0, 64);
    unsigned long long* t; cudaMallocManaged(&t, 64);
    CUtensorMap ma{}, mb{}; Big p{};
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int smem : {16 * 1024, 100 * 1024, 200 * 1024, 224 * 1024}) {
        cudaFuncSetAttribute(k_step, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int variant = 0; variant < 2; ++variant) {
            cudaGraph_t g; cudaGraphExec_t ex;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
            if (variant == 0) k_step<<<148, 160, smem, s>>>(ma, mb, p, ctr, t);
            else k_plain<<<148, 160, smem, s>>>(ctr);
            cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ex, g, 0);
            for (int i = 0; i < 20; ++i) cudaGraphLaunch(ex, s);
            cudaStreamSynchronize(s);
            cudaEventRecord(e0, s);
            for (int i = 0; i < 200; ++i) cudaGraphLaunch(ex, s);
            cudaEventRecord(e1, s); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("smem %3d KB %-6s %6.2f us/launch\n", smem / 1024, variant ? "plain" : "step", ms * 1e3 / 200);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
