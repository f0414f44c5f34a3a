// Probe helpers (ctypes): does the step's cold launch pay an SM shared-memory
// carveout switch after a small-smem kernel (the bench's torch L2 flush)?
//   touch_bigsmem(stream): 148 CTAs x 160 threads with ~223 KB dynamic smem
//   that do nothing (an SM configured like the step kernel's).
//   stamp(ptr, stream): one thread writes %globaltimer.
#include <cuda_runtime.h>
__global__ void __launch_bounds__(160, 1) k_touch(int* p) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0) { sm[0] = blockIdx.x; if (sm[0] == -1) *p = 1; }
}
__global__ void k_stamp(unsigned long long* p) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    *p = g;
}
extern "C" int touch_bigsmem(void* stream, int smem_kb) {
    static int* p = nullptr;
    if (!p) cudaMalloc(&p, 64);
    cudaFuncSetAttribute(k_touch, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
    k_touch<<<148, 160, (size_t)smem_kb * 1024, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}
extern "C" int stamp(void* ptr, void* stream) {
    k_stamp<<<1, 1, 0, (cudaStream_t)stream>>>((unsigned long long*)ptr);
    return (int)cudaGetLastError();
}
