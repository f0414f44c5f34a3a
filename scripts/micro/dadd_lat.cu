// microbenchmark: dependent fp64 add latency, smem-fed sequential sum
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n) {
    __shared__ double s[2][128];
    for (int j = threadIdx.x; j < 128; j += blockDim.x) { s[0][j] = j * 0.5; s[1][j] = j * 0.25; }
    __syncthreads();
    if (threadIdx.x) return;
    long long t0 = clock64();
    double a = 0, b = 0;
    for (int i = 0; i < n; ++i) a = __dadd_rn(a, (double)i);
    long long t1 = clock64();
#pragma unroll 8
    for (int j = 0; j < 128; ++j) { b = __dadd_rn(b, s[0][j]); a = __dadd_rn(a, s[1][j]); }
    long long t2 = clock64();
    double q = __dsqrt_rn(b); double r = __ddiv_rn(a, q);
    long long t3 = clock64();
    out[0] = a + b + r; cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8); cudaMallocManaged(&c, 64);
    for (int it = 0; it < 3; ++it) { k<<<1, 128>>>(o, c, 1024); cudaDeviceSynchronize(); }
    printf("dadd chain 1024: %lld cyc (%.1f/op); smem seq sum 128x2: %lld cyc; sqrt+div: %lld cyc\n", c[0], c[0] / 1024.0, c[1], c[2]);
}
