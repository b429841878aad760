// FP64 mma.sync shapes on this B200: throughput with NACC independent accumulator chains per
// warp (8: throughput, 1-2: latency-bound), m8n8k4 vs m16n8k4 / m16n8k8 / m16n8k16.
#include <cstdio>
#include <cuda_runtime.h>

template <int SH>
struct Shape;
template <>
struct Shape<0> {  // m8n8k4
    static constexpr int NA = 1, NB = 1, NC = 2, M = 8, N = 8, K = 4;
    __device__ static void mma(double* c, const double* a, const double* b) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[0]), "+d"(c[1]) : "d"(a[0]), "d"(b[0]));
    }
};
template <>
struct Shape<1> {  // m16n8k4
    static constexpr int NA = 2, NB = 1, NC = 4, M = 16, N = 8, K = 4;
    __device__ static void mma(double* c, const double* a, const double* b) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
    }
};
template <>
struct Shape<2> {  // m16n8k8
    static constexpr int NA = 4, NB = 2, NC = 4, M = 16, N = 8, K = 8;
    __device__ static void mma(double* c, const double* a, const double* b) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
    }
};
template <>
struct Shape<3> {  // m16n8k16
    static constexpr int NA = 8, NB = 4, NC = 4, M = 16, N = 8, K = 16;
    __device__ static void mma(double* c, const double* a, const double* b) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
            "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
            : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
            : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
              "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
};

template <int SH, int NACC>
__global__ void chain(double* out, int iters) {
    using S = Shape<SH>;
    double a[S::NA], b[S::NB], c[NACC][S::NC];
    for (int i = 0; i < S::NA; ++i) a[i] = 1e-3 * (threadIdx.x + i);
    for (int i = 0; i < S::NB; ++i) b[i] = 2e-3 * (i + 1);
    for (int j = 0; j < NACC; ++j)
        for (int i = 0; i < S::NC; ++i) c[j][i] = j + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < NACC; ++j) S::mma(c[j], a, b);
    }
    double s = 0;
    for (int j = 0; j < NACC; ++j)
        for (int i = 0; i < S::NC; ++i) s += c[j][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int SH, int NACC>
void run(const char* name, int blocks_per_sm, int threads) {
    using S = Shape<SH>;
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int blocks = p.multiProcessorCount * blocks_per_sm, iters = 4096 / (S::M * S::N * S::K / 256);
    double* out;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    chain<SH, NACC><<<blocks, threads>>>(out, 4);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        chain<SH, NACC><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double warps = double(blocks) * threads / 32;
    const double flops = warps * iters * NACC * 2.0 * S::M * S::N * S::K;
    printf("{\"shape\": \"%s\", \"nacc\": %d, \"warps_per_sm\": %d, \"tflops\": %.3f, \"err\": \"%s\"}\n", name, NACC,
           blocks_per_sm * threads / 32, flops / best / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    for (int wps : {4, 16}) {
        const int bps = wps / 4;
        run<0, 8>("m8n8k4", bps, 128);
        run<0, 4>("m8n8k4", bps, 128);
        run<0, 1>("m8n8k4", bps, 128);
        run<1, 4>("m16n8k4", bps, 128);
        run<1, 1>("m16n8k4", bps, 128);
        run<2, 4>("m16n8k8", bps, 128);
        run<2, 1>("m16n8k8", bps, 128);
        run<3, 4>("m16n8k16", bps, 128);
        run<3, 1>("m16n8k16", bps, 128);
    }
    return 0;
}
