// Kernel-boundary cost inside a CUDA graph on B200: a chain of dependent
// launches of an almost empty persistent-shaped kernel (444 CTAs x 256
// threads, 64 KB dynamic shared memory, one global store per CTA), captured
// into one graph and replayed; reported per launch.  This is the floor a
// batch-1 call of three dependent passes pays at its two internal boundaries
// (BASELINE config 1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_gap launch_gap.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void touch(float* p, int n) {
    extern __shared__ float s[];
    s[threadIdx.x] = (float)threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0) p[blockIdx.x % n] += s[7];
}

int main() {
    float* p;
    CK(cudaMalloc(&p, 1 << 20));
    CK(cudaFuncSetAttribute(touch, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const int grids[] = {148, 296, 444};
    for (int g : grids) {
        for (int chain : {3, 300}) {
            cudaGraph_t graph;
            cudaGraphExec_t exec;
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
            for (int i = 0; i < chain; ++i) touch<<<g, 256, 64 * 1024, st>>>(p, 1 << 16);
            CK(cudaStreamEndCapture(st, &graph));
            CK(cudaGraphInstantiate(&exec, graph, 0));
            CK(cudaGraphLaunch(exec, st));
            CK(cudaStreamSynchronize(st));
            cudaEvent_t e0, e1;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            const int reps = 20;
            CK(cudaEventRecord(e0, st));
            for (int r = 0; r < reps; ++r) CK(cudaGraphLaunch(exec, st));
            CK(cudaEventRecord(e1, st));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            printf("grid %3d x 256 thr, 64 KB smem, chain of %3d launches per graph: %.2f us per launch\n", g, chain,
                   1e3 * ms / (reps * chain));
            CK(cudaGraphExecDestroy(exec));
            CK(cudaGraphDestroy(graph));
        }
    }
    return 0;
}
