// Is FP64 DMMA a separate pipe from DFMA on B200?  Per warp-iteration: NM
// independent mma.m8n8k4.f64 and ND independent DFMA per thread; compare the
// time of both streams together with each alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_mix dmma_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NM, int ND>
__global__ void mix(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0001;
    double c[4][2] = {};
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < NM; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
#pragma unroll
        for (int i = 0; i < ND; ++i) x[i] = fma(x[i], 1.0000001, 1e-9);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
    if (s == 1234.5) out[0] = s;
}

template <int NM, int ND> float run(double* d, int grid) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mix<NM, ND><<<grid, 256>>>(d, 10);
    cudaEventRecord(e0);
    mix<NM, ND><<<grid, 256>>>(d, 20000);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    double* d;
    cudaMalloc(&d, 64);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 8;
    const double warps = (double)grid * 8 * 20000;
    float tm = run<4, 0>(d, grid), tf = run<0, 8>(d, grid), tb = run<4, 8>(d, grid);
    printf("DMMA only (4 mma/warp-iter):  %.3f ms  %.2f TFLOP/s\n", tm, warps * 4 * 512 / tm / 1e9);
    printf("DFMA only (8 fma/thread-iter): %.3f ms  %.2f TFLOP/s\n", tf, warps * 8 * 64 / tf / 1e9);
    printf("both:                          %.3f ms  (sum %.3f, max %.3f) -> %.2f TFLOP/s combined\n", tb, tm + tf,
           tm > tf ? tm : tf, warps * (4 * 512 + 8 * 64) / tb / 1e9);
    return 0;
}
