// Golden-section closest point on a patch (reference rp.cpp:22-43, 122-137), written once
// for the host (proximity.cpp, g++ -ffp-contract=off) and the device
// (cuda/proximity_kernels.cu, nvcc --fmad=false): the same IEEE operations in the same
// order, so both produce the reference's (u, v, dist) bit for bit. The pair decisions
// (dist > delta) and the (ubar, vbar) fed to the beta tables depend on it.
#pragma once

#include <cmath>
#include <cstddef>

#ifdef __CUDACC__
#define IFGF_HD __host__ __device__
#else
#define IFGF_HD
#endif

namespace ifgfb200 {
namespace cp {

constexpr double kInvGolden = 0.6180339887498949;
constexpr double kSearchTol = 1e-12;
constexpr int kSweeps = 50;
constexpr int kMaxExtent = 64;

// Clenshaw of each u-line, then of the v-column (chebyshev.cpp:12-25, 63-74)
IFGF_HD inline double series_at(const double* c, int du, int dv, double u, double v) {
    double row[kMaxExtent];
    row[0] = 0.0;
    for (int j = 0; j < dv; ++j) {
        const double* a = c + std::size_t(du) * j;
        double b1 = 0, b2 = 0;
        for (int i = du - 1; i >= 1; --i) {
            const double b0 = a[i] + 2.0 * u * b1 - b2;
            b2 = b1;
            b1 = b0;
        }
        row[j] = a[0] + u * b1 - b2;
    }
    double b1 = 0, b2 = 0;
    for (int j = dv - 1; j >= 1; --j) {
        const double b0 = row[j] + 2.0 * v * b1 - b2;
        b2 = b1;
        b1 = b0;
    }
    return row[0] + v * b1 - b2;
}

struct PatchSeries {
    const double *cx, *cy, *cz;  // position series, u fastest
    int du, dv;
};

// |x - y(u, v)|^2 with the association of len2(x - y) = (dx dx + dy dy) + dz dz
IFGF_HD inline double dist2(const PatchSeries& p, double x, double y, double z, double u, double v) {
    const double ex = x - series_at(p.cx, p.du, p.dv, u, v);
    const double ey = y - series_at(p.cy, p.du, p.dv, u, v);
    const double ez = z - series_at(p.cz, p.du, p.dv, u, v);
    return ex * ex + ey * ey + ez * ez;
}

template <class F>
IFGF_HD inline double golden(const F& f, double a, double b) {
    double c = b - (b - a) * kInvGolden;
    double d = a + (b - a) * kInvGolden;
    double fc = f(c), fd = f(d);
    while (b - a > kSearchTol) {
        if (fc < fd) {
            b = d;
            d = c;
            fd = fc;
            c = b - (b - a) * kInvGolden;
            fc = f(c);
        } else {
            a = c;
            c = d;
            fc = fd;
            d = a + (b - a) * kInvGolden;
            fd = f(d);
        }
    }
    return 0.5 * (a + b);
}

IFGF_HD inline double clamp_unit(double t) { return t < -1.0 ? -1.0 : (1.0 < t ? 1.0 : t); }

// alternating golden-section sweeps in u and v from (u0, v0) (rp.cpp:122-137)
IFGF_HD inline void solve(const PatchSeries& p, double x, double y, double z, double u0, double v0, double& u_out,
                          double& v_out, double& dist_out) {
    double u = clamp_unit(u0), v = clamp_unit(v0);
    for (int sweep = 0; sweep < kSweeps; ++sweep) {
        const double u_prev = u, v_prev = v;
        u = golden([&](double q) { return dist2(p, x, y, z, q, v); }, -1.0, 1.0);
        v = golden([&](double q) { return dist2(p, x, y, z, u, q); }, -1.0, 1.0);
        if (std::fabs(u - u_prev) < kSearchTol && std::fabs(v - v_prev) < kSearchTol) break;
    }
    u_out = u;
    v_out = v;
    dist_out = std::sqrt(dist2(p, x, y, z, u, v));
}

}  // namespace cp
}  // namespace ifgfb200
