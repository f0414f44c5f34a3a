// microbenchmark: B200 FP64 latency/throughput for the routing chain design.
// 64 threads (2 warps), one CTA; cycles per element of a 128-long chain.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double f2d_int(float f) {  // exact float->double with integer ops (normal/zero)
    const unsigned b = __float_as_uint(f);
    const unsigned long long s = (unsigned long long)(b >> 31) << 63;
    const unsigned e = (b >> 23) & 0xff, m = b & 0x7fffff;
    const unsigned long long bits = e == 0 ? s : (s | ((unsigned long long)(e + 896) << 52) | ((unsigned long long)m << 29));
    return __longlong_as_double((long long)bits);
}
template <int MODE>
__global__ void k(const float* q, const float* kk, double* out, long long* cyc) {
    const int t = threadIdx.x;
    float qv[128], kv[128];
#pragma unroll
    for (int j = 0; j < 128; ++j) { qv[j] = q[(t * 131 + j) & 4095]; kv[j] = kk[(t * 17 + j) & 4095]; }
    __syncthreads();
    long long t0 = clock64();
    double a = 0, b = 0;
#pragma unroll
    for (int j = 0; j < 128; ++j) {
        if (MODE == 0) { const double qd = qv[j]; a = __fma_rn(qd, (double)kv[j], a); b = __fma_rn(qd, qd, b); }
        if (MODE == 1) { const double qd = qv[j]; a = __dadd_rn(a, __dmul_rn(qd, (double)kv[j])); b = __dadd_rn(b, __dmul_rn(qd, qd)); }
        if (MODE == 2) { const double qd = f2d_int(qv[j]); const double kd = f2d_int(kv[j]); a = __fma_rn(qd, kd, a); b = __fma_rn(qd, qd, b); }
        if (MODE == 3) { a = __dadd_rn(a, (double)j); }                 // dadd latency
        if (MODE == 4) { a = __fma_rn(a, 1.0000001, 0.5); }             // dfma latency
        if (MODE == 5) { a = __dadd_rn(a, (double)qv[j]); b = __dadd_rn(b, (double)kv[j]); }  // f2f + dadd
    }
    long long t1 = clock64();
    out[t] = a + b;
    if (t == 0) cyc[MODE] = t1 - t0;
}
int main() {
    float *q, *kk; double* o; long long* c;
    cudaMalloc(&q, 16384); cudaMalloc(&kk, 16384); cudaMalloc(&o, 4096); cudaMallocManaged(&c, 64);
    cudaMemset(q, 0x3f, 16384); cudaMemset(kk, 0x3e, 16384);
    for (int nt : {32, 64, 128}) {
        for (int it = 0; it < 3; ++it) {
            k<0><<<1, nt>>>(q, kk, o, c); k<1><<<1, nt>>>(q, kk, o, c); k<2><<<1, nt>>>(q, kk, o, c);
            k<3><<<1, nt>>>(q, kk, o, c); k<4><<<1, nt>>>(q, kk, o, c); k<5><<<1, nt>>>(q, kk, o, c);
            cudaDeviceSynchronize();
        }
        printf("threads %3d cyc/elem: fma-chains %.1f  dmul+dadd %.1f  intcvt+fma %.1f  dadd-lat %.1f  dfma-lat %.1f  f2f+dadd x2 %.1f\n",
               nt, c[0] / 128.0, c[1] / 128.0, c[2] / 128.0, c[3] / 128.0, c[4] / 128.0, c[5] / 128.0);
    }
}
