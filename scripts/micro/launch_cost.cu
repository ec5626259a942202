// Micro-benchmark: per-launch cost of small kernels (1 CTA x 1024 threads)
// with / without static shared memory, alone and interleaved with a
// large-smem kernel.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 launch_cost.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_plain(int* p) { if (threadIdx.x == 0) p[blockIdx.x] += 1; }
__global__ void k_static16(int* p) {
    __shared__ unsigned sh[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sh[i] = i;
    __syncthreads();
    if (threadIdx.x == 0) p[blockIdx.x] += sh[5];
}
__global__ void k_atom(int* p) {
    __shared__ unsigned sh[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sh[i] = i;
    __syncthreads();
    for (int b = threadIdx.x; b < 2048; b += blockDim.x) atomicAdd(p + 64 + b, (int)sh[b]);
}
__global__ void k_big(int* p) {
    extern __shared__ unsigned dyn[];
    dyn[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0) p[blockIdx.x % 64] += dyn[3];
}

template <typename F>
float timeit(F f, int iters, cudaStream_t st) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 10; ++i) f();
    cudaEventRecord(a, st);
    for (int i = 0; i < iters; ++i) f();
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms * 1000.f / iters;
}

int main() {
    int* p; cudaMalloc(&p, 1 << 20); cudaMemset(p, 0, 1 << 20);
    cudaStream_t st; cudaStreamCreate(&st);
    cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int N = 200;
    printf("plain        %.2f us\n", timeit([&] { k_plain<<<1, 1024, 0, st>>>(p); }, N, st));
    printf("static16     %.2f us\n", timeit([&] { k_static16<<<1, 1024, 0, st>>>(p); }, N, st));
    printf("atom2048     %.2f us\n", timeit([&] { k_atom<<<1, 1024, 0, st>>>(p); }, N, st));
    printf("big          %.2f us\n", timeit([&] { k_big<<<296, 512, 100 * 1024, st>>>(p); }, N, st));
    printf("big+plain    %.2f us\n", timeit([&] { k_big<<<296, 512, 100 * 1024, st>>>(p); k_plain<<<1, 1024, 0, st>>>(p); }, N, st));
    printf("big+static16 %.2f us\n", timeit([&] { k_big<<<296, 512, 100 * 1024, st>>>(p); k_static16<<<1, 1024, 0, st>>>(p); }, N, st));
    printf("big+atom     %.2f us\n", timeit([&] { k_big<<<296, 512, 100 * 1024, st>>>(p); k_atom<<<1, 1024, 0, st>>>(p); }, N, st));
    printf("plain x2     %.2f us\n", timeit([&] { k_plain<<<1, 1024, 0, st>>>(p); k_plain<<<1, 1024, 0, st>>>(p); }, N, st));
    printf("grid296 plain %.2f us\n", timeit([&] { k_plain<<<296, 256, 0, st>>>(p); }, N, st));
    cudaDeviceSynchronize();
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
