// Micro-probes for the roofline denominators this path needs that the driver
// does not measure: FP64/FP32 issue rate (DFMA, DADD), FP64 DMMA, L2 read
// bandwidth on a resident buffer, HBM copy.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <typename T, int OP>
__global__ void alu_loop(T* out, int iters, T a, T b) {
    T x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (T)(threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) x[i] = fma(x[i], a, b);
            else x[i] = x[i] + b;
        }
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == (T)1234.5) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0001;
    double c[2][2] = {{0, 0}, {0, 0}};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 2; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
    if (c[0][0] + c[1][1] == 1234.5) out[0] = c[0][0];
}

__global__ void l2_read(const double2* __restrict__ p, size_t n, int reps, double* out) {
    double acc = 0;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            double2 v = __ldcg(p + i);
            acc += v.x + v.y;
        }
    if (acc == 1234.5) out[0] = acc;
}

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    printf("device %s SMs %d L2 %d MB clock %d kHz\n", prop.name, prop.multiProcessorCount, prop.l2CacheSize >> 20, prop.clockRate);
    double* dout; CK(cudaMalloc(&dout, 64));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms = prop.multiProcessorCount;
    float ms;
    const int iters = 20000;
    for (int blocks_per_sm : {4, 8}) {
        int grid = sms * blocks_per_sm, thr = 256;
        alu_loop<double, 0><<<grid, thr>>>(dout, 100, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        alu_loop<double, 0><<<grid, thr>>>(dout, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)grid * thr * iters * 8;
        printf("DFMA  bps=%d: %.2f Tinstr/s = %.2f TFLOP/s (per SM per clk at 1965MHz: %.1f)\n", blocks_per_sm, ops / ms / 1e9, 2 * ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
        cudaEventRecord(e0);
        alu_loop<double, 1><<<grid, thr>>>(dout, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("DADD  bps=%d: %.2f Tinstr/s\n", blocks_per_sm, ops / ms / 1e9);
        cudaEventRecord(e0);
        alu_loop<float, 0><<<grid, thr>>>((float*)dout, iters, 1.0000001f, 1e-9f);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("FFMA  bps=%d: %.2f Tinstr/s = %.2f TFLOP/s\n", blocks_per_sm, ops / ms / 1e9, 2 * ops / ms / 1e9);
    }
    {
        int grid = sms * 8, thr = 256, it2 = 5000;
        dmma_loop<<<grid, thr>>>(dout, 10);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        dmma_loop<<<grid, thr>>>(dout, it2);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        double flops = (double)grid * (thr / 32) * it2 * 2 * (8 * 8 * 4 * 2);
        printf("DMMA m8n8k4: %.2f TFLOP/s\n", flops / ms / 1e9);
    }
    for (size_t mb : {16, 32, 64, 96}) {
        size_t n = mb * (1 << 20) / 16;
        double2* p; CK(cudaMalloc(&p, n * 16)); cudaMemset(p, 0, n * 16);
        int reps = 20;
        l2_read<<<sms * 8, 256>>>(p, n, 2, dout);
        cudaEventRecord(e0);
        l2_read<<<sms * 8, 256>>>(p, n, reps, dout);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("L2-resident read %zu MiB: %.1f GB/s\n", mb, (double)n * 16 * reps / ms / 1e6);
        cudaFree(p);
    }
    {
        size_t n = (size_t)2 << 30 >> 4;
        double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
        cudaMemset(a, 0, n * 16);
        copy_k<<<sms * 8, 256>>>(a, b, n);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) copy_k<<<sms * 8, 256>>>(a, b, n);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("HBM copy 2 GiB: %.1f GB/s (read+write)\n", 2.0 * n * 16 * 5 / ms / 1e6);
    }
    CK(cudaGetLastError());
    return 0;
}
