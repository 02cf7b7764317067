// DFMA throughput vs operand pattern (register-file read bandwidth test).
#include <cstdio>
#include <cuda_runtime.h>
// mode 0: a[c] = fma(a[c], k1, k2) (constants)
// mode 1: a[c] = fma(u[c], w, a[c])   one shared register operand (reuse-able)
// mode 2: a[c] = fma(u[c], v[c], a[c]) three distinct register pairs
template <int MODE>
__global__ void k(long iters, double *sink, double seed) {
    double a[8], u[8], v[8];
#pragma unroll
    for (int c = 0; c < 8; c++) { a[c] = threadIdx.x * 1e-9 + c; u[c] = 1.0 + c * 1e-3 + seed; v[c] = 0.5 - c * 1e-3 + seed; }
    double w = 0.999 + seed;
    for (long i = 0; i < iters; i++) {
#pragma unroll
        for (int r = 0; r < 8; r++) {
#pragma unroll
            for (int c = 0; c < 8; c++) {
                if (MODE == 0) a[c] = __fma_rn(a[c], 0.999999999, 1e-12);
                else if (MODE == 1) a[c] = __fma_rn(u[c], w, a[c]);
                else a[c] = __fma_rn(u[c], v[c], a[c]);
            }
            w = w * 0.9999999 + 1e-9;  // a new "row" operand (1 DMUL-ish)
#pragma unroll
            for (int c = 0; c < 8; c++) { u[c] = u[c] * 0.999999999; }
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; c++) s += a[c] + u[c] + v[c];
    if (s == 1.2345) sink[0] = s;
}
template <int MODE>
void run(int warps_per_sm, double *sink) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long iters = 300;
    int threads = 32 * warps_per_sm;
    k<MODE><<<sms, threads>>>(10, sink, 0.0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k<MODE><<<sms, threads>>>(iters, sink, 0.0); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    // per r: 8 DFMA + 1 (w) + 8 (u) FP64 ops
    double fma = (double)sms * threads * iters * 8 * 8, all = (double)sms * threads * iters * 8 * 17;
    printf("mode %d warps/SM %2d : %.2f T DFMA/s (%.2f T FP64 instr/s)\n", MODE, warps_per_sm, fma / (ms * 1e-3) / 1e12, all / (ms * 1e-3) / 1e12);
}
int main() {
    double *sink; cudaMalloc(&sink, 8);
    for (int w : {8, 12, 16}) { run<0>(w, sink); run<1>(w, sink); run<2>(w, sink); }
    return 0;
}
