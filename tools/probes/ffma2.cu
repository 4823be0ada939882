// Probe: packed fp32 (fma.rn.f32x2 -> FFMA2, add.rn.f32x2 -> FADD2) issue rate
// on sm_100a against scalar FFMA, alone and next to shared-memory loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2 ffma2.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ float2 up(u64 v) { float2 r; asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }

// MODE 0: 16 scalar FFMA / iter; 1: 8 FFMA2 / iter (same flops); 2: 8 FADD2; 3: 16 FADD
// LDS > 0: that many LDS.64 per iteration as well
template <int MODE, int LDS>
__global__ void loop(float* out, int iters, float a, float b) {
    __shared__ float2 sh[1024];
    sh[threadIdx.x] = make_float2(a, b);
    sh[threadIdx.x + 512] = make_float2(b, a);
    __syncthreads();
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = (float)(threadIdx.x + i);
    u64 p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = pk(x[2 * i], x[2 * i + 1]);
    const u64 pa = pk(a, a), pb = pk(b, b);
    float2 acc = make_float2(0, 0);
    int idx = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
        } else if (MODE == 3) {
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = x[i] + b;
        } else if (MODE == 1) {
#pragma unroll
            for (int i = 0; i < 8; ++i) p[i] = fma2(p[i], pa, pb);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) p[i] = add2(p[i], pb);
        }
#pragma unroll
        for (int l = 0; l < LDS; ++l) {
            float2 v = sh[(idx + l * 32) & 1023];
            acc.x += v.x;
            idx += (int)v.y;
        }
    }
    float s = acc.x + acc.y;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) { float2 v = up(p[i]); s += v.x + v.y; }
    if (s == 1234.5f) out[0] = s;
}

template <int MODE, int LDS> void run(const char* name, float* d, int sms) {
    const int iters = 20000, grid = sms * 4, thr = 512;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    loop<MODE, LDS><<<grid, thr>>>(d, 100, 1.0000001f, 0.f);
    cudaEventRecord(e0);
    loop<MODE, LDS><<<grid, thr>>>(d, iters, 1.0000001f, 0.f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double lane_ops = (double)grid * thr * iters * 16;
    printf("%-28s %.3f ms  %.2f T lane-ops/s (%s)\n", name, ms, lane_ops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
    float* d; cudaMalloc(&d, 64);
    int sms = prop.multiProcessorCount;
    run<0, 0>("16 FFMA", d, sms);
    run<1, 0>("8 FFMA2", d, sms);
    run<3, 0>("16 FADD", d, sms);
    run<2, 0>("8 FADD2", d, sms);
    run<0, 2>("16 FFMA + 2 LDS.64(+2 FADD,I2F)", d, sms);
    run<1, 2>("8 FFMA2 + 2 LDS.64", d, sms);
    run<0, 4>("16 FFMA + 4 LDS.64", d, sms);
    run<1, 4>("8 FFMA2 + 4 LDS.64", d, sms);
    return 0;
}
