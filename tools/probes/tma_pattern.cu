// Memory-pattern ceiling of the strided pass: persistent CTAs stage
// [R rows x W cols] tiles (row stride C) with one 3-D TMA box each, double
// buffered, and write every element back with STG from registers -- the
// pass kernel's data movement without its arithmetic.  Also a contiguous
// variant (1-D bulk copies).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_pattern tma_pattern.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int R, int W, int RB>
__global__ void __launch_bounds__(1024, 1) pattern(const __grid_constant__ CUtensorMap map, double2* dst, long long tiles,
                                                  int C, int tpp, int mode) {
    extern __shared__ __align__(128) unsigned char sm[];
    double2* buf = (double2*)sm;
    unsigned long long* bar = (unsigned long long*)(sm + (2 * R * W * 16 + 127) / 128 * 128);
    const int t = threadIdx.x;
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto stage = [&](long long tile, int b) {
        const long long p = tile / tpp;
        const int col = (int)(tile - p * tpp) * W;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[b])), "r"(R * W * 16));
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(sa(buf + b * R * W)), "l"(&map), "r"(2 * col), "r"(0), "r"((int)(p * (R / RB))), "r"(sa(&bar[b])) : "memory");
    };
    if (t == 0) {
        if (blockIdx.x < tiles) stage(blockIdx.x, 0);
        if (blockIdx.x + gridDim.x < tiles) stage(blockIdx.x + gridDim.x, 1);
    }
    int it = 0;
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
        const int b = it & 1;
        unsigned ok;
        do {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(ok) : "r"(sa(&bar[b])), "r"((it >> 1) & 1) : "memory");
        } while (!ok);
        const long long p = tile / tpp;
        const int col = (int)(tile - p * tpp) * W;
        double2* g = dst + p * (long long)R * C + col;
        if (mode == 3) {
            __syncthreads();
            if (t == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                             ::"l"(&map), "r"(2 * col), "r"(0), "r"((int)(p * (R / RB))), "r"(sa(buf + b * R * W)) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
        } else if (mode != 1) {
            for (int e = t; e < R * W; e += blockDim.x) {
                const int row = e / W, c = e % W;
                g[(long long)row * C + c] = buf[b * R * W + e];
            }
        } else if (buf[b * R * W + t].x == 12345.0) {
            g[t] = buf[b * R * W];
        }
        __syncthreads();
        if (t == 0 && tile + 2 * gridDim.x < tiles) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            stage(tile + 2 * gridDim.x, b);
        }
    }
}

template <int R, int W, int RB>
void run(double2* x, double2* y, long long N, long long batch, int C, PFN_cuTensorMapEncodeTiled_v12000 enc) {
    const size_t bytes = N * batch * 16;
    const unsigned long long rows = N * batch / C;
    cuuint64_t dims[3] = {(cuuint64_t)2 * C, (cuuint64_t)RB, rows / RB};
    cuuint64_t strides[2] = {(cuuint64_t)C * 16, (cuuint64_t)RB * C * 16};
    cuuint32_t box[3] = {2 * W, RB, R / RB}, es[3] = {1, 1, 1};
    CUtensorMap m;
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n");
        return;
    }
    const int tpp = C / W + (C % W ? 1 : 0);
    const long long tiles = (N * batch / (R * (long long)C)) * tpp;
    const int smem = (2 * R * W * 16 + 127) / 128 * 128 + 16;
    auto k = pattern<R, W, RB>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode : {0, 1, 2, 3})
        for (int nt : {256, 512}) {
            k<<<148, nt, smem>>>(m, y, tiles, C, tpp, mode);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            for (int r = 0; r < 5; ++r) k<<<148, nt, smem>>>(m, y, tiles, C, tpp, mode);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("R=%d W=%d RB=%d C=%d mode=%s thr=%d: %.3f ms, %.0f GB/s\n", R, W, RB, C,
                   mode == 0 ? "ld+stg" : mode == 1 ? "ld    " : mode == 2 ? "stg   " : "ld+tma", nt, ms / 5,
                   (mode == 0 || mode == 3 ? 2.0 : 1.0) * bytes / (ms / 5 * 1e-3) / 1e9);
        }
}

int main() {
    const long long N = 1594323, batch = 64;
    const size_t bytes = N * batch * 16;
    double2 *x, *y;
    CK(cudaMalloc(&x, bytes));
    CK(cudaMalloc(&y, bytes));
    cudaMemset(x, 0, bytes);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
    run<729, 8, 243>(x, y, N, batch, 2187, enc);
    run<243, 16, 243>(x, y, N, batch, 6561, enc);
    run<729, 4, 243>(x, y, N, batch, 2187, enc);
    return 0;
}
