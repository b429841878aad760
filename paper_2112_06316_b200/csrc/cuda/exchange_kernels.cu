// Layout kernels around the per-apply NCCL exchange of a multi-GPU operator (SURVEY.md
// §8(e)) and the Morton-sharded GMRES vectors. NCCL's reduce-scatter and all-gather move
// equal chunks per rank, while the Morton ranges of the ranks differ in length, so every
// rank's range is padded to the longest one (C entries):
//
//   reduce-scatter send  [rank r][S | D][C]   (pack_ranges)  -> recv [S | D][C] (unpack_owned)
//   all-gather           send [C] (copy_pad)  -> recv [rank r][C]  -> original order
//                        (unpermute_padded: out[perm[t]] = recv[r(t) C + t - bounds[r(t)]])
#include "dev_common.cuh"
#include "kernels.cuh"

namespace ifgfb200 {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ int rank_of(std::uint32_t t, const std::uint32_t* __restrict__ bounds, int world) {
    int r = 0;
    while (r + 1 < world && t >= bounds[r + 1]) ++r;
    return r;
}

__global__ void pack_ranges_kernel(const double2* __restrict__ Sp, const double2* __restrict__ Dp,
                                   const std::uint32_t* __restrict__ bounds, int world, std::int64_t C,
                                   double2* __restrict__ send) {
    const std::int64_t total = std::int64_t(world) * 2 * C;
    for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < total;
         i += std::int64_t(gridDim.x) * blockDim.x) {
        const int r = int(i / (2 * C));
        const std::int64_t rem = i - std::int64_t(r) * 2 * C;
        const bool dbl = rem >= C;
        const std::int64_t t = std::int64_t(bounds[r]) + (dbl ? rem - C : rem);
        send[i] = t < std::int64_t(bounds[r + 1]) ? (dbl ? Dp[t] : Sp[t]) : make_double2(0.0, 0.0);
    }
}

__global__ void unpack_owned_kernel(const double2* __restrict__ recv, std::int64_t lo, std::int64_t cnt,
                                    std::int64_t C, double2* __restrict__ Sp, double2* __restrict__ Dp) {
    for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < cnt;
         i += std::int64_t(gridDim.x) * blockDim.x) {
        Sp[lo + i] = recv[i];
        Dp[lo + i] = recv[C + i];
    }
}

__global__ void copy_pad_kernel(const double2* __restrict__ src, std::int64_t cnt, std::int64_t C,
                                double2* __restrict__ dst) {
    for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < C;
         i += std::int64_t(gridDim.x) * blockDim.x)
        dst[i] = i < cnt ? src[i] : make_double2(0.0, 0.0);
}

__global__ void unpermute_padded_kernel(std::int64_t n, const std::uint32_t* __restrict__ perm,
                                        const std::uint32_t* __restrict__ bounds, int world, std::int64_t C,
                                        const double2* __restrict__ recv, double2* __restrict__ out) {
    for (std::int64_t t = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; t < n;
         t += std::int64_t(gridDim.x) * blockDim.x) {
        const int r = rank_of(std::uint32_t(t), bounds, world);
        out[perm[t]] = recv[std::int64_t(r) * C + (t - std::int64_t(bounds[r]))];
    }
}

__global__ void gather_local_kernel(const std::uint32_t* __restrict__ perm, std::int64_t lo, std::int64_t cnt,
                                    const double2* __restrict__ in, double2* __restrict__ out) {
    for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < cnt;
         i += std::int64_t(gridDim.x) * blockDim.x)
        out[i] = in[perm[lo + i]];
}

__global__ void csqrt_re_kernel(double2* h) { *h = make_double2(sqrt(h->x), 0.0); }

int grid_for(std::int64_t n) { return int(std::min<std::int64_t>((n + kThreads - 1) / kThreads, 148 * 16)); }

}  // namespace

void launch_pack_ranges(const double2* Sp, const double2* Dp, const std::uint32_t* bounds, int world,
                        std::int64_t C, double2* send, cudaStream_t st) {
    const std::int64_t total = std::int64_t(world) * 2 * C;
    if (total == 0) return;
    pack_ranges_kernel<<<grid_for(total), kThreads, 0, st>>>(Sp, Dp, bounds, world, C, send);
    IFGF_CUDA(cudaGetLastError());
}

void launch_unpack_owned(const double2* recv, std::int64_t lo, std::int64_t cnt, std::int64_t C, double2* Sp,
                         double2* Dp, cudaStream_t st) {
    if (cnt == 0) return;
    unpack_owned_kernel<<<grid_for(cnt), kThreads, 0, st>>>(recv, lo, cnt, C, Sp, Dp);
    IFGF_CUDA(cudaGetLastError());
}

void launch_copy_pad(const double2* src, std::int64_t cnt, std::int64_t C, double2* dst, cudaStream_t st) {
    if (C == 0) return;
    copy_pad_kernel<<<grid_for(C), kThreads, 0, st>>>(src, cnt, C, dst);
    IFGF_CUDA(cudaGetLastError());
}

void launch_unpermute_padded(std::int64_t n, const std::uint32_t* perm, const std::uint32_t* bounds, int world,
                             std::int64_t C, const double2* recv, double2* out, cudaStream_t st) {
    if (n == 0) return;
    unpermute_padded_kernel<<<grid_for(n), kThreads, 0, st>>>(n, perm, bounds, world, C, recv, out);
    IFGF_CUDA(cudaGetLastError());
}

void launch_gather_local(const std::uint32_t* perm, std::int64_t lo, std::int64_t cnt, const double2* in,
                         double2* out, cudaStream_t st) {
    if (cnt == 0) return;
    gather_local_kernel<<<grid_for(cnt), kThreads, 0, st>>>(perm, lo, cnt, in, out);
    IFGF_CUDA(cudaGetLastError());
}

void launch_csqrt_re(double2* h, cudaStream_t st) {
    csqrt_re_kernel<<<1, 1, 0, st>>>(h);
    IFGF_CUDA(cudaGetLastError());
}

}  // namespace ifgfb200
