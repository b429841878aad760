// Batched golden-section closest points of classify_pairs (reference rp.cpp:122-137,
// 194-289) on the GPU: one thread per (target, patch) search, the shared host/device
// routine of host/closest_point.hpp compiled with --fmad=false (Makefile rule), so every
// (u, v, dist) equals the host's -- and the reference's -- bit for bit.
#include <vector>

#include "../host/closest_point.hpp"
#include "../host/proximity.hpp"
#include "dev_common.cuh"
#include "kernels.cuh"

namespace ifgfb200 {
namespace {

struct CpJob {
    double x, y, z, u0, v0;
    std::int32_t q;
    std::int32_t pad;
};

__global__ void closest_point_kernel(int n, const CpJob* __restrict__ jobs, const double* __restrict__ series,
                                     const std::int64_t* __restrict__ soff, const int* __restrict__ dims,
                                     double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const CpJob j = jobs[i];
    const double* c = series + soff[j.q];
    const int du = dims[2 * j.q], dv = dims[2 * j.q + 1];
    const cp::PatchSeries ps{c, c + std::size_t(du) * dv, c + 2 * std::size_t(du) * dv, du, dv};
    double u, v, d;
    cp::solve(ps, j.x, j.y, j.z, j.u0, j.v0, u, v, d);
    out[3 * i] = u;
    out[3 * i + 1] = v;
    out[3 * i + 2] = d;
}

}  // namespace

void gpu_closest_points(const Surface& s, const std::vector<ClosestPointRequest>& req, std::vector<ClosestPoint>& res,
                        int device) {
    IFGF_CUDA(cudaSetDevice(device));
    const std::size_t nq = s.patches.size();
    std::vector<double> series;
    std::vector<std::int64_t> soff(nq);
    std::vector<int> dims(2 * nq);
    for (std::size_t q = 0; q < nq; ++q) {
        const Patch& p = s.patches[q];
        if (p.du > cp::kMaxExtent || p.dv > cp::kMaxExtent)
            throw InvalidArgument("closest point: series extent above 64");
        soff[q] = std::int64_t(series.size());
        dims[2 * q] = p.du;
        dims[2 * q + 1] = p.dv;
        for (int a = 0; a < 3; ++a) series.insert(series.end(), p.pos_c[a].begin(), p.pos_c[a].end());
    }
    std::vector<CpJob> jobs;
    std::vector<std::size_t> where;
    for (std::size_t i = 0; i < req.size(); ++i) {
        if (req[i].own) continue;
        const Vec3& x = s.pos[req[i].target];
        jobs.push_back({x.x, x.y, x.z, req[i].u0, req[i].v0, req[i].q, 0});
        where.push_back(i);
    }
    res.assign(req.size(), ClosestPoint{});
    if (jobs.empty()) return;
    double* d_series = nullptr;
    std::int64_t* d_soff = nullptr;
    int* d_dims = nullptr;
    CpJob* d_jobs = nullptr;
    double* d_out = nullptr;
    auto release = [&] {
        cudaFree(d_series);
        cudaFree(d_soff);
        cudaFree(d_dims);
        cudaFree(d_jobs);
        cudaFree(d_out);
    };
    try {
        IFGF_CUDA(cudaMalloc(&d_series, series.size() * sizeof(double)));
        IFGF_CUDA(cudaMalloc(&d_soff, soff.size() * sizeof(std::int64_t)));
        IFGF_CUDA(cudaMalloc(&d_dims, dims.size() * sizeof(int)));
        IFGF_CUDA(cudaMalloc(&d_jobs, jobs.size() * sizeof(CpJob)));
        IFGF_CUDA(cudaMalloc(&d_out, 3 * jobs.size() * sizeof(double)));
        IFGF_CUDA(cudaMemcpy(d_series, series.data(), series.size() * sizeof(double), cudaMemcpyHostToDevice));
        IFGF_CUDA(cudaMemcpy(d_soff, soff.data(), soff.size() * sizeof(std::int64_t), cudaMemcpyHostToDevice));
        IFGF_CUDA(cudaMemcpy(d_dims, dims.data(), dims.size() * sizeof(int), cudaMemcpyHostToDevice));
        IFGF_CUDA(cudaMemcpy(d_jobs, jobs.data(), jobs.size() * sizeof(CpJob), cudaMemcpyHostToDevice));
        const int n = int(jobs.size());
        closest_point_kernel<<<(n + 127) / 128, 128>>>(n, d_jobs, d_series, d_soff, d_dims, d_out);
        IFGF_CUDA(cudaGetLastError());
        std::vector<double> out(3 * jobs.size());
        IFGF_CUDA(cudaMemcpy(out.data(), d_out, out.size() * sizeof(double), cudaMemcpyDeviceToHost));
        for (std::size_t k = 0; k < where.size(); ++k) res[where[k]] = {out[3 * k], out[3 * k + 1], out[3 * k + 2]};
    } catch (...) {
        release();
        throw;
    }
    release();
}

}  // namespace ifgfb200
