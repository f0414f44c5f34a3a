// Back-to-back launch cost of a near-empty 148 x 160 kernel on B200 vs its
// dynamic shared memory, by-value parameter size and the cooperative
// attribute (one CUDA graph per launch, replayed 400 times; us per launch).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)
struct Small { int x[4]; };
struct Big { int x[280]; };  // ~1.1 KB, like StepTables
template <class Pm>
__global__ void __launch_bounds__(160, 1) k_empty(Pm p, int* ctr) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0) { sm[0] = p.x[blockIdx.x & 3]; if (sm[0] == 12345) *ctr = 1; }
}
int main() {
    int* ctr; cudaMalloc(&ctr, 64);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int big = 0; big < 2; ++big)
    for (int coop = 0; coop < 2; ++coop)
    for (int kb : {1, 16, 64, 128, 192, 224}) {
        const void* fn = big ? (const void*)k_empty<Big> : (const void*)k_empty<Small>;
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024));
        Small ps{}; Big pb{};
        void* args[2] = {big ? (void*)&pb : (void*)&ps, &ctr};
        cudaLaunchConfig_t cfg{}; cfg.gridDim = 148; cfg.blockDim = 160; cfg.dynamicSmemBytes = kb * 1024; cfg.stream = s;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeCooperative; a[0].val.cooperative = 1;
        cfg.attrs = a; cfg.numAttrs = coop;
        cudaGraph_t g; cudaGraphExec_t ex;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        CK(cudaLaunchKernelExC(&cfg, fn, args));
        CK(cudaStreamEndCapture(s, &g)); CK(cudaGraphInstantiate(&ex, g, 0));
        for (int i = 0; i < 50; ++i) cudaGraphLaunch(ex, s);
        CK(cudaStreamSynchronize(s));
        cudaEventRecord(e0, s);
        for (int i = 0; i < 400; ++i) cudaGraphLaunch(ex, s);
        cudaEventRecord(e1, s); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        // the same kernel launched directly (no graph)
        cudaEventRecord(e0, s);
        for (int i = 0; i < 400; ++i) cudaLaunchKernelExC(&cfg, fn, args);
        cudaEventRecord(e1, s); cudaEventSynchronize(e1);
        float ms2; cudaEventElapsedTime(&ms2, e0, e1);
        printf("params %-5s coop %d smem %3d KB: graph %5.2f us/launch, direct %5.2f\n", big ? "1.1KB" : "16B", coop, kb,
               ms * 1e3 / 400, ms2 * 1e3 / 400);
        cudaGraphExecDestroy(ex); cudaGraphDestroy(g);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
