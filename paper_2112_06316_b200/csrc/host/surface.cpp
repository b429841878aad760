#include "surface.hpp"

#include <algorithm>
#include <cstdint>
#include <exception>
#include <functional>
#include <limits>

#include "chebyshev.hpp"

namespace ifgfb200 {

namespace {

// patches are independent: loops over them run in parallel; the exception of the lowest
// failing patch is rethrown, as the serial loop would have thrown it
template <class F>
void for_each_patch(std::size_t n, F&& body) {
    std::exception_ptr err;
    std::size_t err_at = n;
#pragma omp parallel for schedule(dynamic, 16)
    for (std::int64_t q = 0; q < std::int64_t(n); ++q) {
        try {
            body(std::size_t(q));
        } catch (...) {
#pragma omp critical(ifgf_surface_error)
            if (std::size_t(q) < err_at) {
                err_at = std::size_t(q);
                err = std::current_exception();
            }
        }
    }
    if (err) std::rethrow_exception(err);
}

void derive_series(Patch& p) {
    for (int c = 0; c < 3; ++c) {
        p.du_c[c] = cheb::deriv_u(p.pos_c[c], p.du, p.dv);
        p.dv_c[c] = cheb::deriv_v(p.pos_c[c], p.du, p.dv);
    }
}

// Increasing-degree tensor fit until the sampled residual is below tol (geometry.cpp:29-61).
Patch fit(const std::function<Vec3(double, double)>& f, int nu, int nv, double tol) {
    Patch p;
    p.nu = nu;
    p.nv = nv;
    const int start = std::max({12, nu, nv});
    const int stop = std::max(48, start);
    for (int deg = start; deg <= stop; deg += 6) {
        const std::vector<double> xs = cheb::gauss_nodes(deg);
        std::array<std::vector<double>, 3> smp;
        for (auto& s : smp) s.assign(std::size_t(deg) * deg, 0.0);
        for (int j = 0; j < deg; ++j)
            for (int i = 0; i < deg; ++i) {
                const Vec3 y = f(xs[i], xs[j]);
                const std::size_t at = i + std::size_t(deg) * j;
                smp[0][at] = y.x;
                smp[1][at] = y.y;
                smp[2][at] = y.z;
            }
        p.du = p.dv = deg;
        for (int c = 0; c < 3; ++c) p.pos_c[c] = cheb::coeffs_2d(smp[c].data(), deg, deg);
        const std::vector<double> probe = cheb::gauss_nodes(deg + 3);
        double worst = 0.0;
        for (int j = 0; j < deg + 3; j += 2)
            for (int i = 0; i < deg + 3; i += 2) {
                const Vec3 want = f(probe[i], probe[j]);
                const Vec3 got{cheb::eval_2d(p.pos_c[0].data(), deg, deg, probe[i], probe[j]),
                               cheb::eval_2d(p.pos_c[1].data(), deg, deg, probe[i], probe[j]),
                               cheb::eval_2d(p.pos_c[2].data(), deg, deg, probe[i], probe[j])};
                worst = std::max(worst, len(want - got));
            }
        if (worst < tol) break;
    }
    derive_series(p);
    return p;
}

}  // namespace

Vec3 patch_point(const Patch& p, double u, double v) {
    return {cheb::eval_2d(p.pos_c[0].data(), p.du, p.dv, u, v),
            cheb::eval_2d(p.pos_c[1].data(), p.du, p.dv, u, v),
            cheb::eval_2d(p.pos_c[2].data(), p.du, p.dv, u, v)};
}

void patch_tangent_frame(const Patch& p, double u, double v, Vec3& tu, Vec3& tv, Vec3& n,
                         double& jac) {
    tu = {cheb::eval_2d(p.du_c[0].data(), p.du, p.dv, u, v),
          cheb::eval_2d(p.du_c[1].data(), p.du, p.dv, u, v),
          cheb::eval_2d(p.du_c[2].data(), p.du, p.dv, u, v)};
    tv = {cheb::eval_2d(p.dv_c[0].data(), p.du, p.dv, u, v),
          cheb::eval_2d(p.dv_c[1].data(), p.du, p.dv, u, v),
          cheb::eval_2d(p.dv_c[2].data(), p.du, p.dv, u, v)};
    const Vec3 cr = cross3(tu, tv);
    jac = len(cr);
    if (jac < 1e-14) throw DegenerateGeometry("patch frame: vanishing Jacobian");
    n = cr * (p.orient / jac);
}

std::vector<double> Surface::spacing() const {
    std::vector<double> out(patches.size(), 0.0);
    for (std::size_t q = 0; q < patches.size(); ++q) {
        const int nu = patches[q].nu, nv = patches[q].nv;
        double m = 0.0;
        for (int j = 0; j < nv; ++j)
            for (int i = 0; i < nu; ++i) {
                const Vec3 a = pos[node(int(q), i, j)];
                if (i + 1 < nu) m = std::max(m, len(a - pos[node(int(q), i + 1, j)]));
                if (j + 1 < nv) m = std::max(m, len(a - pos[node(int(q), i, j + 1)]));
            }
        out[q] = m;
    }
    return out;
}

double Surface::extent() const {
    constexpr double big = std::numeric_limits<double>::max();
    Vec3 lo{big, big, big}, hi{-big, -big, -big};
    for (const Vec3& p : pos) {
        lo = {std::min(lo.x, p.x), std::min(lo.y, p.y), std::min(lo.z, p.z)};
        hi = {std::max(hi.x, p.x), std::max(hi.y, p.y), std::max(hi.z, p.z)};
    }
    return std::max({hi.x - lo.x, hi.y - lo.y, hi.z - lo.z});
}

Surface assemble_surface(std::vector<Patch> patches, const Vec3& interior) {
    Surface s;
    s.patches = std::move(patches);
    s.interior = interior;
    for_each_patch(s.patches.size(), [&](std::size_t q) {
        Patch& p = s.patches[q];
        if (p.nu < 1 || p.nv < 1 || p.du < 1 || p.dv < 1)
            throw InvalidArgument("assemble_surface: nonpositive patch dimensions");
        if (p.du_c[0].empty()) derive_series(p);
        p.orient = 1.0;
        Vec3 tu, tv, n;
        double jac;
        try {
            patch_tangent_frame(p, 0.0, 0.0, tu, tv, n, jac);
        } catch (const DegenerateGeometry&) {
            throw DegenerateGeometry("degenerate Jacobian at patch center (patch " +
                                     std::to_string(q) + ")");
        }
        if (dot3(n, patch_point(p, 0.0, 0.0) - interior) < 0.0) p.orient = -1.0;
    });
    s.patch_start.assign(s.patches.size() + 1, 0);
    for (std::size_t q = 0; q < s.patches.size(); ++q)
        s.patch_start[q + 1] = s.patch_start[q] + std::size_t(s.patches[q].nu) * s.patches[q].nv;
    const std::size_t n = s.patch_start.back();
    s.pos.resize(n);
    s.nrm.resize(n);
    s.jac.resize(n);
    s.wt.resize(n);
    s.pu.resize(n);
    s.pv.resize(n);
    s.patch_of.resize(n);
    for_each_patch(s.patches.size(), [&](std::size_t q) {
        const Patch& p = s.patches[q];
        std::vector<double> un, uw, vn, vw;
        cheb::fejer(p.nu, un, uw);
        cheb::fejer(p.nv, vn, vw);
        for (int j = 0; j < p.nv; ++j)
            for (int i = 0; i < p.nu; ++i) {
                const std::size_t l = s.node(int(q), i, j);
                s.pos[l] = patch_point(p, un[i], vn[j]);
                Vec3 tu, tv;
                try {
                    patch_tangent_frame(p, un[i], vn[j], tu, tv, s.nrm[l], s.jac[l]);
                } catch (const DegenerateGeometry&) {
                    throw DegenerateGeometry("degenerate Jacobian at node (patch " +
                                             std::to_string(q) + ")");
                }
                s.wt[l] = uw[i] * vw[j];
                s.pu[l] = un[i];
                s.pv[l] = vn[j];
                s.patch_of[l] = int(q);
            }
    });
    return s;
}

namespace {

std::vector<Patch> cube_sphere_patches(double radius, int splits, int nu, int nv) {
    if (radius <= 0.0) throw InvalidArgument("make_sphere: radius must be positive");
    if (splits < 0 || nu < 1 || nv < 1) throw InvalidArgument("make_sphere: bad counts");
    // face = (axis, sign) in the reference's order (geometry.cpp:188)
    const int axis[6] = {0, 0, 1, 1, 2, 2};
    const double sign[6] = {1, -1, 1, -1, 1, -1};
    const int m = 1 << splits;
    std::vector<Patch> out(6 * std::size_t(m) * m);
    for_each_patch(out.size(), [&](std::size_t idx) {
                const int f = int(idx / (std::size_t(m) * m)), a = int(idx / m % m), b = int(idx % m);
                const double alo = -1.0 + 2.0 * a / m, ahi = alo + 2.0 / m;
                const double blo = -1.0 + 2.0 * b / m, bhi = blo + 2.0 / m;
                const int ax = axis[f];
                const double sg = sign[f];
                auto map = [=](double u, double v) -> Vec3 {
                    const double s = alo + (u + 1.0) * 0.5 * (ahi - alo);
                    const double t = blo + (v + 1.0) * 0.5 * (bhi - blo);
                    const Vec3 c = ax == 0 ? Vec3{sg, s, t} : (ax == 1 ? Vec3{t, sg, s} : Vec3{s, t, sg});
                    return c * (radius / len(c));
                };
                out[idx] = fit(map, nu, nv, 1e-12);
    });
    return out;
}

}  // namespace

Surface make_sphere(double radius, int splits, int nu, int nv) {
    return assemble_surface(cube_sphere_patches(radius, splits, nu, nv), Vec3{0, 0, 0});
}

Surface make_spheroid(int splits, int nu, int nv, double ax, double ay, double az) {
    std::vector<Patch> ps = cube_sphere_patches(1.0, splits, nu, nv);
    const double sc[3] = {ax, ay, az};
    for (Patch& p : ps)
        for (int c = 0; c < 3; ++c) {
            for (double& v : p.pos_c[c]) v *= sc[c];
            p.du_c[c].clear();
            p.dv_c[c].clear();
        }
    return assemble_surface(std::move(ps), Vec3{0, 0, 0});
}

}  // namespace ifgfb200
