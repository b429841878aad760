// How well do unsynchronised warps share the FP64 pipe? Each warp alternates a burst of 12
// DMMAs (3 accumulator chains x 4 k-steps, the 2-pipe tile of tc_common.cuh) with a gap of G
// dependent FP32 FMAs (~4 cycles each, another pipe) that stands for the epilogue / group
// work of the tensor-core kernels. With W warps per sub-partition a work-conserving pipe
// would be busy min(1, W * 192 / (192 + gap cycles)); the measured DMMA rate against that
// bound is what queueing behind the other warps' bursts costs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_burst tools/dmma_burst.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int G>
__global__ void __launch_bounds__(128) burst(double* out, long long* cyc, int iters) {
    double a = 1e-3 * threadIdx.x, b = 2e-3;
    double c[3][2] = {{0, 0}, {1, 1}, {2, 2}};
    float f = 1.0f + threadIdx.x;
    // de-synchronise the warps of a sub-partition
    for (int i = 0; i < int((threadIdx.x >> 5) + blockIdx.x % 7) * 13; ++i) f = fmaf(f, 1.0001f, 0.5f);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int q = 0; q < 3; ++q) dmma(c[q][0], c[q][1], a, b);
#pragma unroll 1
        for (int g = 0; g < G; ++g) f = fmaf(f, 1.0001f, 0.5f);
        a += double(f) * 1e-30;  // the next burst depends on the gap
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = c[0][0] + c[1][1] + c[2][0] + f;
}

template <int G>
void run(double* out, long long* cyc, int ctas_per_sm, int sms) {
    const int iters = 4096, blocks = sms * ctas_per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    burst<G><<<blocks, 128>>>(out, cyc, 16);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        burst<G><<<blocks, 128>>>(out, cyc, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    long long h = 0;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double tf = 12.0 * 512.0 * iters * double(blocks) * 4 / (best * 1e-3) * 1e-12;
    std::printf("{\"warps_per_subpartition\": %d, \"gap_fmas\": %d, \"cycles_per_iteration_warp0\": %.0f, "
                "\"dmma_tflops\": %.2f, \"frac_of_36.9\": %.3f}\n",
                ctas_per_sm, G, double(h) / iters, tf, tf / 36.9);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * p.multiProcessorCount * 8 * 128);
    cudaMalloc(&cyc, sizeof(long long));
    for (int w : {1, 2, 4}) {  // CTAs of 4 warps per SM = warps per sub-partition
        run<0>(out, cyc, w, p.multiProcessorCount);
        run<25>(out, cyc, w, p.multiProcessorCount);
        run<50>(out, cyc, w, p.multiProcessorCount);
        run<100>(out, cyc, w, p.multiProcessorCount);
        run<200>(out, cyc, w, p.multiProcessorCount);
        run<400>(out, cyc, w, p.multiProcessorCount);
    }
    return 0;
}
