// Where does the per-segment parent kernel's tile loop spend its time? A replica of
// parent_tc.cu's inner loop (tc_common.cuh's own tile code: A slots from warp shared memory,
// 12 DMMAs for 2 pipes, the T(phi) gather, the re-centring product and the shared accumulator
// update) with no global traffic at all, at the kernel's occupancy (4 CTAs x 4 warps per SM,
// 48.9 KB shared per CTA), in variants that drop or restructure one part each:
//   0 as the product      1 no accumulator update      2 no epilogue at all (DMMAs + A loads)
//   3 two tiles per step: both tiles' DMMAs, then both epilogues
//   4 DMMAs only (A from registers; the compiler hoists loop-invariant tiles: ignore)
//   5 next tile's A slots loaded ahead   6 DMMAs of tile t before the epilogue of tile t-1
//   7 / 8 as 0 plus the per-group geometry rows (fill_row + factors + barrier) from registers
// Prints the DMMA rate of each as a fraction of the 36.9 TF/s peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr \
//        -Ipaper_2112_06316_b200/csrc/cuda -o tools/tile_probe tools/tile_probe.cu
#include <cstdio>

#include "tc_common.cuh"

using namespace ifgfb200;
using namespace ifgfb200::tc;
using namespace ifgfb200::dev;

constexpr int kWarps = 4, NPC = 2, NPP = 2;
constexpr int kRow = kRowLen + 8, kNode = kRowLen + 6;
constexpr int kGeoSz = 32 * kRow;
constexpr int kAcc = 2 * kNP * NPP * 2;

template <int V>
__global__ void __launch_bounds__(32 * kWarps, 4) probe(const double* __restrict__ bsrc, double2* __restrict__ out,
                                                        int groups, int tiles) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* geo = smem + warp * (kGeoSz + kAcc);
    double2* acc = reinterpret_cast<double2*>(geo + kGeoSz);
    const int r = lane >> 2, tig = lane & 3;
    using LY = Layout<NPC>;
    for (int e = lane; e < kAcc / 2; e += 32) acc[e] = make_double2(0.0, 0.0);
    {
        double* row = geo + lane * kRow;
        fill_row(0.1 + 0.01 * lane, -0.2 + 0.02 * lane, 0.3 - 0.01 * lane, row);
        for (int pc = 0; pc < 3; ++pc) {
            row[kRowLen + 2 * pc] = 0.5 + 0.01 * pc;
            row[kRowLen + 2 * pc + 1] = 0.25;
        }
        row[kNode] = __longlong_as_double((long long)((lane * 7) % 150));
    }
    __syncwarp();
    double2 sink = make_double2(0.0, 0.0);
    for (int g = 0; g < groups; ++g) {
        double bq[LY::NB];
#pragma unroll
        for (int i = 0; i < LY::NB; ++i) bq[i] = bsrc[(g * 37 + i * 32 + lane) & 4095];
        if constexpr (V == 7 || V == 8) {
            // the per-group geometry step of the template path without its global loads: the
            // row's A slots, T(phi), factors and node written by each lane, then the barrier
            if (V == 7 || lane < 8 * tiles) {
                double* row = geo + lane * kRow;
                const double x = 1e-3 * g;
                fill_row(0.1 + 0.01 * lane + x, -0.2 + 0.02 * lane - x, 0.3 - 0.01 * lane + x, row);
#pragma unroll
                for (int pc = 0; pc < NPC; ++pc) {
                    row[kRowLen + 2 * pc] = 0.5 + x;
                    row[kRowLen + 2 * pc + 1] = 0.25 - x;
                }
                row[kNode] = __longlong_as_double((long long)((lane * 7 + g) % 150));
            }
            __syncwarp();
        }
        auto mma = [&](int t0, double (&d)[LY::NQ][2]) {
            if constexpr (V == 4) {
#pragma unroll
                for (int q = 0; q < LY::NQ; ++q) d[q][0] = d[q][1] = 0.0;
#pragma unroll
                for (int j = 0; j < kKS; ++j)
#pragma unroll
                    for (int q = 0; q < LY::NQ; ++q) dmma884(d[q][0], d[q][1], bq[j], bq[q * kKS + j]);
            } else {
                tile_mma_row<NPC>(geo + (t0 + r) * kRow, true, tig, bq, d);
            }
        };
        auto epilogue = [&](int t0, const double (&d)[LY::NQ][2]) {
            if constexpr (V == 2 || V == 4) {
#pragma unroll
                for (int q = 0; q < LY::NQ; ++q) {
                    sink.x += d[q][0];
                    sink.y += d[q][1];
                }
                return;
            }
            const double* gp = geo + (t0 + r) * kRow;
            const double2 val = tile_gather_row<NPC>(gp, lane, d);
            const int fp = tig < NPC ? tig : 0;
            const double2 ctb = cmul(make_double2(gp[kRowLen + 2 * fp], gp[kRowLen + 2 * fp + 1]), val);
            if constexpr (V == 1) {
                sink = cadd(sink, ctb);
            } else if (tig < NPC) {
                double2& a = acc[int(__double_as_longlong(gp[kNode])) * NPP + tig];
                a = cadd(a, ctb);
            }
        };
        if constexpr (V == 5) {
            // the next tile's A slots are loaded before this tile's DMMAs
            double an[kKS];
#pragma unroll
            for (int j = 0; j < kKS; ++j) an[j] = geo[r * kRow + 4 * j + tig];
            for (int t = 0; t < tiles; ++t) {
                double a[kKS], d[LY::NQ][2];
#pragma unroll
                for (int j = 0; j < kKS; ++j) a[j] = an[j];
                const int tn = ((t + 1) & 3) * 8;
#pragma unroll
                for (int j = 0; j < kKS; ++j) an[j] = geo[(tn + r) * kRow + 4 * j + tig];
#pragma unroll
                for (int q = 0; q < LY::NQ; ++q) d[q][0] = d[q][1] = 0.0;
#pragma unroll
                for (int j = 0; j < kKS; ++j)
#pragma unroll
                    for (int q = 0; q < LY::NQ; ++q) dmma884(d[q][0], d[q][1], a[j], bq[q * kKS + j]);
                epilogue((t & 3) * 8, d);
            }
        } else if constexpr (V == 6) {
            // tile t's DMMAs are issued before tile t-1's epilogue
            double dp[LY::NQ][2];
            mma(0, dp);
            for (int t = 1; t < tiles; ++t) {
                double d[LY::NQ][2];
                mma((t & 3) * 8, d);
                epilogue(((t - 1) & 3) * 8, dp);
#pragma unroll
                for (int q = 0; q < LY::NQ; ++q) dp[q][0] = d[q][0], dp[q][1] = d[q][1];
            }
            epilogue(((tiles - 1) & 3) * 8, dp);
        } else if constexpr (V == 3) {
            for (int t = 0; t < tiles; t += 2) {
                double d0[LY::NQ][2], d1[LY::NQ][2];
                mma((t & 3) * 8, d0);
                mma(((t + 1) & 3) * 8, d1);
                epilogue((t & 3) * 8, d0);
                epilogue(((t + 1) & 3) * 8, d1);
            }
        } else {
            for (int t = 0; t < tiles; ++t) {
                double d[LY::NQ][2];
                mma((t & 3) * 8, d);
                epilogue((t & 3) * 8, d);
            }
        }
        __syncwarp();
    }
    if (sink.x == 12345.678) out[0] = sink;
    if (lane == 0) out[blockIdx.x * kWarps + warp] = cadd(acc[lane], sink);
}

template <int V>
void run(const double* bsrc, double2* out, int blocks, int groups, int tiles, const char* what) {
    const size_t smem = size_t(kWarps) * (kGeoSz + kAcc) * sizeof(double);
    cudaFuncSetAttribute(probe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe<V><<<blocks, 32 * kWarps, smem>>>(bsrc, out, 2, tiles);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        probe<V><<<blocks, 32 * kWarps, smem>>>(bsrc, out, groups, tiles);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double dm = 12.0 * tiles * groups * double(blocks) * kWarps;  // DMMAs
    const double tf = dm * 512.0 / (best * 1e-3) * 1e-12;
    std::printf("{\"variant\": %d, \"what\": \"%s\", \"tiles_per_group\": %d, \"ms\": %.3f, \"dmma_tflops\": %.2f, "
                "\"frac_of_36.9\": %.3f, \"err\": \"%s\"}\n",
                V, what, tiles, best, tf, tf / 36.9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int blocks = p.multiProcessorCount * 4 * 8;
    double* bsrc;
    double2* out;
    cudaMalloc(&bsrc, 4096 * sizeof(double));
    cudaMemset(bsrc, 0, 4096 * sizeof(double));
    cudaMalloc(&out, sizeof(double2) * blocks * kWarps);
    for (int tiles : {2, 4, 16}) {
        const int groups = 4096 / tiles;
        run<0>(bsrc, out, blocks, groups, tiles, "product tile loop");
        run<1>(bsrc, out, blocks, groups, tiles, "no accumulator update");
        run<2>(bsrc, out, blocks, groups, tiles, "no epilogue");
        run<3>(bsrc, out, blocks, groups, tiles, "two tiles per step");
        run<4>(bsrc, out, blocks, groups, tiles, "DMMAs only");
        run<7>(bsrc, out, blocks, groups, tiles, "product loop + the group's geometry rows (32 lanes)");
        run<8>(bsrc, out, blocks, groups, tiles, "product loop + the group's geometry rows (8 x tiles lanes)");
        run<5>(bsrc, out, blocks, groups, tiles, "next tile's A slots loaded ahead");
        run<6>(bsrc, out, blocks, groups, tiles, "DMMAs of tile t before the epilogue of t-1");
    }
    return 0;
}
