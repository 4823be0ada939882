// DSMEM (distributed shared memory) exchange bandwidth on B200, the number
// that decides whether a single-pass cluster convolution (SURVEY.md 2.1 K5:
// a whole signal resident across a thread-block cluster, stage groups
// exchanged through DSMEM instead of HBM) can beat the three-pass design.
//
// Each CTA of a cluster of C holds `kb` KB of shared memory and scatters it
// all-to-all (the exchange between the strided and the contiguous stage
// groups): chunk j of CTA r (C equal contiguous chunks) goes to CTA
// (r + j) % C, each warp storing contiguous 512-byte runs (16-byte
// st.shared::cluster per lane), repeated `reps` times between cluster
// barriers; the same kernel with C = 1 is the local shared-memory reference.  Reported: bytes moved per cluster barrier round / time, chip-wide
// and per SM, next to the HBM copy peak (MEASURED_PEAKS.json, ~6.55 TB/s).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bw dsmem_bw.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void exchange(int words, int reps, double* out) {
    extern __shared__ double2 buf[];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned C = cl.num_blocks(), r = cl.block_rank();
    for (int i = threadIdx.x; i < words; i += blockDim.x) buf[i] = make_double2(r, i);
    cl.sync();
    for (int it = 0; it < reps; ++it) {
        for (int i = threadIdx.x; i < words; i += blockDim.x) {
            const unsigned dst = (unsigned)(i / ((words + C - 1) / C) + r) % C;  // chunk -> CTA; C = 1: local
            double2* rem = cl.map_shared_rank(buf, dst);
            const double2 v = buf[i];
            rem[i] = make_double2(v.x + 1.0, v.y);
        }
        cl.sync();
    }
    if (threadIdx.x == 0 && buf[0].x == -1.0) out[0] = buf[1].y;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double* out;
    CK(cudaMalloc(&out, 64));
    CK(cudaFuncSetAttribute(exchange, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const int kbs[] = {64, 150};
    const int cls[] = {1, 2, 4, 8, 16};
    for (int kb : kbs) {
        CK(cudaFuncSetAttribute(exchange, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024));
        for (int C : cls) {
            const int words = kb * 1024 / 16, reps = 200, threads = 512;
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = C;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            cfg.blockDim = dim3(threads);
            cfg.dynamicSmemBytes = kb * 1024;
            int maxc = 0;
            cfg.gridDim = dim3(C);
            if (cudaOccupancyMaxActiveClusters(&maxc, exchange, &cfg) != cudaSuccess || maxc < 1) {
                printf("kb=%d C=%d: not launchable\n", kb, C);
                cudaGetLastError();
                continue;
            }
            cfg.gridDim = dim3(maxc * C);
            cudaEvent_t e0, e1;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(cudaLaunchKernelEx(&cfg, exchange, words, 2, out));  // warm-up
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0));
            CK(cudaLaunchKernelEx(&cfg, exchange, words, reps, out));
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double bytes = (double)maxc * C * words * 16.0 * reps;  // every CTA moves its buffer once per round
            const double remote = C > 1 ? 1.0 : 0.0;
            printf("kb=%3d cluster=%2d: %3d clusters (%3d CTAs on %d SMs), %.1f GB/s chip-wide, %.1f GB/s per CTA%s\n", kb,
                   C, maxc, maxc * C, sms, bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9 / (maxc * C),
                   remote ? " (DSMEM all-to-all)" : " (local shared memory)");
        }
    }
    return 0;
}
