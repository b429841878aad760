// FP64 tensor-core (mma.sync m8n8k4 f64, DMMA) throughput vs DFMA on this B200.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void dmma_chain(double* out, int iters) {
    double a = 1e-3 * threadIdx.x, b = 2e-3;
    double c[8][2];
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma(c[j][0], c[j][1], a, b);
    }
    double s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    int blocks = p.multiProcessorCount * 4, threads = 256, iters = 2048;
    double* out; cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    dmma_chain<<<blocks, threads>>>(out, 16); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0); dmma_chain<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double warps = double(blocks) * threads / 32;
    double flops = warps * iters * 8 * 2.0 * 8 * 8 * 4;
    printf("{\"dmma_m8n8k4_tflops\": %.3f, \"ms\": %.3f, \"err\": \"%s\"}\n", flops / best / 1e9, best, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
