// FP64 pipe microbenchmark: DFMA throughput vs warps/SM and independent chains/thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k(long iters, double *sink) {
    double a[C];
#pragma unroll
    for (int c = 0; c < C; c++) a[c] = threadIdx.x * 1e-9 + c;
    for (long i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 16; u++)
#pragma unroll
            for (int c = 0; c < C; c++) a[c] = __fma_rn(a[c], 0.999999999, 1e-12);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; c++) s += a[c];
    if (s == 1.2345) sink[0] = s;
}
template <int C>
void run(int warps_per_sm, double *sink) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long iters = 4000 / C + 1;
    int threads = 32 * warps_per_sm;  // one block per SM
    k<C><<<sms, threads>>>(10, sink);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k<C><<<sms, threads>>>(iters, sink); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double inst = (double)sms * threads * iters * 16 * C;
    printf("chains %d warps/SM %2d : %.2f T DFMA/s\n", C, warps_per_sm, inst / (ms * 1e-3) / 1e12);
}
int main() {
    double *sink; cudaMalloc(&sink, 8);
    for (int w : {4, 8, 12, 16, 32}) { run<1>(w, sink); run<2>(w, sink); run<4>(w, sink); run<8>(w, sink); }
    return 0;
}
