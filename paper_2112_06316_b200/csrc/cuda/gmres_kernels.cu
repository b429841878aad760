// Vector kernels of the device-resident restarted GMRES (solver.cpp:177-300): the Krylov
// basis lives in HBM and only the Hessenberg column (j + 2 complex numbers) crosses to the
// host per iteration. Reductions are two-pass with a fixed grid and a fixed tree, so every
// run (and every rank of a replicated solve) produces the same bits.
#include "dev_common.cuh"
#include "kernels.cuh"

namespace ifgfb200 {
namespace {

using namespace dev;

constexpr int kRedThreads = 256;

__device__ __forceinline__ double2 block_sum(double2 v, double2* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_down_sync(0xffffffffu, v.x, o);
        v.y += __shfl_down_sync(0xffffffffu, v.y, o);
    }
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double2 t = make_double2(0.0, 0.0);
    if (threadIdx.x == 0)
        for (int w = 0; w < int(blockDim.x) / 32; ++w) t = cadd(t, sh[w]);
    return t;  // valid in thread 0
}

// partial[b] = sum over the block's grid-stride share of conj(a) b
__global__ void __launch_bounds__(kRedThreads) cdot_partial_kernel(std::int64_t n, const double2* __restrict__ a,
                                                                   const double2* __restrict__ b,
                                                                   double2* __restrict__ partial) {
    __shared__ double2 sh[kRedThreads / 32];
    double2 acc = make_double2(0.0, 0.0);
    for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < n;
         i += std::int64_t(gridDim.x) * blockDim.x) {
        const double2 x = a[i], y = b[i];
        acc.x = fma(x.x, y.x, fma(x.y, y.y, acc.x));  // conj(x) y
        acc.y = fma(x.x, y.y, fma(-x.y, y.x, acc.y));
    }
    const double2 t = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// dst = sum of the partials (fixed order); with as_norm, dst = (sqrt(re), 0)
__global__ void cdot_final_kernel(int nb, const double2* __restrict__ partial, double2* __restrict__ dst,
                                  int as_norm) {
    __shared__ double2 sh[kRedThreads / 32];
    double2 acc = make_double2(0.0, 0.0);
    for (int i = threadIdx.x; i < nb; i += blockDim.x) acc = cadd(acc, partial[i]);
    const double2 t = block_sum(acc, sh);
    if (threadIdx.x == 0) *dst = as_norm ? make_double2(sqrt(t.x), 0.0) : t;
}

// w -= h v (h read on the device)
__global__ void caxpy_dev_kernel(std::int64_t n, const double2* __restrict__ h, double2* __restrict__ w,
                                 const double2* __restrict__ v) {
    const std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const double2 c = *h, x = v[i];
    double2 y = w[i];
    y.x -= c.x * x.x - c.y * x.y;
    y.y -= c.x * x.y + c.y * x.x;
    w[i] = y;
}

// v = w / |h| (h = (norm, 0) on the device)
__global__ void cscale_inv_kernel(std::int64_t n, const double2* __restrict__ h, const double2* __restrict__ w,
                                  double2* __restrict__ v) {
    const std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const double s = h->x;
    const double2 x = w[i];
    v[i] = make_double2(x.x / s, x.y / s);
}

// r = b - ax
__global__ void csub_kernel(std::int64_t n, const double2* __restrict__ b, const double2* __restrict__ ax,
                            double2* __restrict__ r) {
    const std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    r[i] = make_double2(b[i].x - ax[i].x, b[i].y - ax[i].y);
}

// x += sum_{i < m} y_i V_i (V rows of length n, stride ld), fixed order in i
__global__ void cupdate_kernel(std::int64_t n, int m, const double2* __restrict__ y, const double2* __restrict__ V,
                               std::int64_t ld, double2* __restrict__ x) {
    const std::int64_t t = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
    if (t >= n) return;
    double2 acc = x[t];
    for (int i = 0; i < m; ++i) {
        const double2 c = y[i], v = V[i * ld + t];
        acc.x += c.x * v.x - c.y * v.y;
        acc.y += c.x * v.y + c.y * v.x;
    }
    x[t] = acc;
}

int blocks_for(std::int64_t n, int threads) { return int((n + threads - 1) / threads); }

}  // namespace

int gmres_reduce_blocks() { return 2 * 148; }

void launch_cdot(std::int64_t n, const double2* a, const double2* b, double2* partial, double2* dst, bool as_norm,
                 cudaStream_t st) {
    const int nb = gmres_reduce_blocks();
    cdot_partial_kernel<<<nb, kRedThreads, 0, st>>>(n, a, b, partial);
    cdot_final_kernel<<<1, kRedThreads, 0, st>>>(nb, partial, dst, as_norm ? 1 : 0);
    IFGF_CUDA(cudaGetLastError());
}

void launch_caxpy_dev(std::int64_t n, const double2* h, double2* w, const double2* v, cudaStream_t st) {
    caxpy_dev_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, h, w, v);
    IFGF_CUDA(cudaGetLastError());
}

void launch_cscale_inv(std::int64_t n, const double2* h, const double2* w, double2* v, cudaStream_t st) {
    cscale_inv_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, h, w, v);
    IFGF_CUDA(cudaGetLastError());
}

void launch_csub(std::int64_t n, const double2* b, const double2* ax, double2* r, cudaStream_t st) {
    csub_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, b, ax, r);
    IFGF_CUDA(cudaGetLastError());
}

void launch_cupdate(std::int64_t n, int m, const double2* y, const double2* V, std::int64_t ld, double2* x,
                    cudaStream_t st) {
    if (m <= 0) return;
    cupdate_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, m, y, V, ld, x);
    IFGF_CUDA(cudaGetLastError());
}

}  // namespace ifgfb200
