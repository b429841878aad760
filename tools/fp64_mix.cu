// Do DMMA (mma.sync m8n8k4 f64) and DFMA share one issue pipe on this B200?
// Runs, per warp, 8 independent DMMA chains, R independent DFMA chains, or both interleaved,
// and prints the times: if the pipes are separate, "both" takes ~max(dmma, dfma), else ~sum.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_mix tools/fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <bool DM, int NF>
__global__ void mix(double* out, int iters) {
    double a = 1e-3 * threadIdx.x, b = 2e-3;
    double c[8][2], f[NF > 0 ? NF : 1];
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = j;
    for (int j = 0; j < (NF > 0 ? NF : 1); ++j) f[j] = j * 1e-3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (DM) dmma(c[j][0], c[j][1], a, b);
#pragma unroll
            for (int q = 0; q < NF / 8; ++q) f[j * (NF / 8) + q] = fma(f[j * (NF / 8) + q], b, a);
        }
    }
    double s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
    for (int j = 0; j < (NF > 0 ? NF : 1); ++j) s += f[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <class K>
float run(K kern, int blocks, int threads, double* out, int iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, threads>>>(out, 16);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}
int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int blocks = p.multiProcessorCount * 4, threads = 256, iters = 2048;
    double* out;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    const double dm_fl = 512.0 * 8 * iters * blocks * (threads / 32);  // flops of the DMMAs
    const double f16 = 2.0 * 16 * iters * blocks * threads, f32 = 2.0 * 32 * iters * blocks * threads;
    const float t_d = run(mix<true, 0>, blocks, threads, out, iters);
    const float t_f16 = run(mix<false, 16>, blocks, threads, out, iters);
    const float t_b16 = run(mix<true, 16>, blocks, threads, out, iters);
    const float t_f32 = run(mix<false, 32>, blocks, threads, out, iters);
    const float t_b32 = run(mix<true, 32>, blocks, threads, out, iters);
    std::printf("{\"dmma_ms\": %.3f, \"dmma_tflops\": %.2f, \"dfma16_ms\": %.3f, \"dfma16_tflops\": %.2f, "
                "\"both16_ms\": %.3f, \"dfma32_ms\": %.3f, \"dfma32_tflops\": %.2f, \"both32_ms\": %.3f, "
                "\"err\": \"%s\"}\n",
                t_d, dm_fl / t_d * 1e-9, t_f16, f16 / t_f16 * 1e-9, t_b16, t_f32, f32 / t_f32 * 1e-9, t_b32,
                cudaGetErrorString(cudaGetLastError()));
    return 0;
}
