// Micro-benchmark: 10 dependent tiny kernels per "step": plain stream
// launches vs a CUDA graph vs programmatic dependent launch (PDL).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_a(int* p) { if (threadIdx.x == 0) p[blockIdx.x] += 1; }
__global__ void k_pdl(int* p) {
    cudaGridDependencySynchronize();
    if (threadIdx.x == 0) p[blockIdx.x] += 1;
    cudaTriggerProgrammaticLaunchCompletion();
}

int main() {
    int* p; cudaMalloc(&p, 1 << 20); cudaMemset(p, 0, 1 << 20);
    cudaStream_t st; cudaStreamCreate(&st);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int K = 10, N = 200;
    auto step = [&](int grid, int blk) { for (int i = 0; i < K; ++i) k_a<<<grid, blk, 0, st>>>(p); };
    for (int cfg = 0; cfg < 2; ++cfg) {
        const int grid = cfg ? 296 : 1, blk = cfg ? 256 : 1024;
        for (int i = 0; i < 5; ++i) step(grid, blk);
        cudaEventRecord(a, st);
        for (int i = 0; i < N; ++i) step(grid, blk);
        cudaEventRecord(b, st); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("stream  grid %d: %.2f us per kernel\n", grid, ms * 1000 / (N * K));
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        step(grid, blk);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        for (int i = 0; i < 5; ++i) cudaGraphLaunch(ge, st);
        cudaEventRecord(a, st);
        for (int i = 0; i < N; ++i) cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("graph   grid %d: %.2f us per kernel\n", grid, ms * 1000 / (N * K));
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cudaLaunchConfig_t lc = {};
        lc.gridDim = grid; lc.blockDim = blk; lc.stream = st; lc.attrs = at; lc.numAttrs = 1;
        auto pstep = [&]() { for (int i = 0; i < K; ++i) cudaLaunchKernelEx(&lc, k_pdl, p); };
        for (int i = 0; i < 5; ++i) pstep();
        cudaEventRecord(a, st);
        for (int i = 0; i < N; ++i) pstep();
        cudaEventRecord(b, st); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("pdl     grid %d: %.2f us per kernel\n", grid, ms * 1000 / (N * K));
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        pstep();
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        for (int i = 0; i < 5; ++i) cudaGraphLaunch(ge, st);
        cudaEventRecord(a, st);
        for (int i = 0; i < N; ++i) cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("pdl+graph grid %d: %.2f us per kernel\n", grid, ms * 1000 / (N * K));
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
