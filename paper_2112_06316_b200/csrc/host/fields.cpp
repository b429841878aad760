#include "fields.hpp"

#include <algorithm>
#include <cmath>

#include "chebyshev.hpp"

namespace ifgfb200 {

FineQuad oversample_for_fields(const Surface& s, const cplx* density, double k) {
    FineQuad out;
    std::vector<double> nodes, weights, are, aim;
    for (std::size_t q = 0; q < s.patches.size(); ++q) {
        const Patch& p = s.patches[q];
        const std::size_t b = s.patch_start[q], e = s.patch_start[q + 1];
        Vec3 lo = s.pos[b], hi = lo;
        for (std::size_t l = b; l < e; ++l) {
            lo = {std::min(lo.x, s.pos[l].x), std::min(lo.y, s.pos[l].y), std::min(lo.z, s.pos[l].z)};
            hi = {std::max(hi.x, s.pos[l].x), std::max(hi.y, s.pos[l].y), std::max(hi.z, s.pos[l].z)};
        }
        const double diam = len(hi - lo);
        const int m = std::min(24, std::max({p.nu, p.nv, 8 + int(std::ceil(0.75 * k * diam))}));
        // density coefficients of the patch (u fastest), real and imaginary series
        const std::vector<cplx> a = cheb::coeffs_2d(density + b, p.nu, p.nv);
        are.resize(a.size());
        aim.resize(a.size());
        for (std::size_t i = 0; i < a.size(); ++i) {
            are[i] = a[i].real();
            aim[i] = a[i].imag();
        }
        cheb::fejer(m, nodes, weights);
        for (int j = 0; j < m; ++j)
            for (int i = 0; i < m; ++i) {
                const double u = nodes[i], v = nodes[j];
                Vec3 tu, tv, nrm;
                double jac = 0;
                patch_tangent_frame(p, u, v, tu, tv, nrm, jac);
                const Vec3 y = patch_point(p, u, v);
                out.x.push_back(y.x);
                out.y.push_back(y.y);
                out.z.push_back(y.z);
                out.nx.push_back(nrm.x);
                out.ny.push_back(nrm.y);
                out.nz.push_back(nrm.z);
                out.jw.push_back(jac * weights[i] * weights[j]);
                out.density.emplace_back(cheb::eval_2d(are.data(), p.nu, p.nv, u, v),
                                         cheb::eval_2d(aim.data(), p.nu, p.nv, u, v));
            }
    }
    return out;
}

std::vector<Vec3> far_field_directions(int n_phi, int n_theta) {
    if (n_phi < 2 || n_theta < 2) throw InvalidArgument("FarFieldGrid: need at least 2 points per direction");
    const double dphi = kPi / (n_phi - 1), dtheta = 2.0 * kPi / (n_theta - 1);
    std::vector<Vec3> d(std::size_t(n_phi) * n_theta);
    for (int n = 0; n < n_theta; ++n)
        for (int m = 0; m < n_phi; ++m) {
            const double ph = m * dphi, th = n * dtheta;  // polar angle, azimuth
            d[m + std::size_t(n_phi) * n] = {std::cos(th) * std::sin(ph), std::sin(th) * std::sin(ph), std::cos(ph)};
        }
    return d;
}

namespace {

// j_0..j_L(x) (Miller's downward recurrence, normalised by j_0 or j_1 whichever is larger)
// and y_0..y_L(x) (upward recurrence, stable for y)
void sph_bessel(int L, double x, std::vector<double>& j, std::vector<double>& y) {
    if (x <= 0) throw InvalidArgument("spherical_bessel: x must be positive");
    const double sx = std::sin(x), cx = std::cos(x);
    const int top = L + 24 + int(std::ceil(std::sqrt(40.0 * (L + 1))));
    std::vector<double> f(top + 2, 0.0);
    f[top] = 1e-280;
    for (int l = top; l >= 1; --l) {
        f[l - 1] = (2.0 * l + 1.0) / x * f[l] - f[l + 1];
        if (std::abs(f[l - 1]) > 1e250)
            for (int t = l - 1; t <= top + 1; ++t) f[t] *= 1e-250;
    }
    const double j0 = sx / x, j1 = sx / (x * x) - cx / x;
    const double scale = std::abs(j0) >= std::abs(j1) ? j0 / f[0] : j1 / f[1];
    j.resize(L + 1);
    y.resize(L + 1);
    for (int l = 0; l <= L; ++l) j[l] = f[l] * scale;
    y[0] = -cx / x;
    if (L >= 1) y[1] = -cx / (x * x) - sx / x;
    for (int l = 2; l <= L; ++l) y[l] = (2.0 * l - 1.0) / x * y[l - 1] - y[l - 2];
}

}  // namespace

std::vector<cplx> mie_far_field(double radius, double k, const Vec3& direction, const std::vector<Vec3>& dirs,
                                int extra_terms) {
    if (radius <= 0 || k <= 0) throw InvalidArgument("mie_far_field: need kR > 0");
    const double x = k * radius;
    const int L = int(std::ceil(x + 6.0 * std::cbrt(x) + 20.0)) + extra_terms;
    std::vector<double> jl, yl;
    sph_bessel(L, x, jl, yl);
    std::vector<cplx> coef(L + 1);  // (2l + 1) j_l / h_l
    for (int l = 0; l <= L; ++l) coef[l] = (2.0 * l + 1.0) * jl[l] / cplx(jl[l], yl[l]);
    const double dn = len(direction);
    if (dn == 0) throw InvalidArgument("mie_far_field: zero incidence direction");
    const Vec3 dh = direction * (1.0 / dn);
    std::vector<cplx> out(dirs.size());
    for (std::size_t t = 0; t < dirs.size(); ++t) {
        const Vec3 e = dirs[t] * (1.0 / len(dirs[t]));
        const double mu = std::clamp(dot3(e, dh), -1.0, 1.0);
        double pm = 1.0, pc = mu;  // P_{l-1}, P_l
        cplx acc = coef[0];
        if (L >= 1) acc += coef[1] * mu;
        for (int l = 2; l <= L; ++l) {
            const double pn = ((2.0 * l - 1.0) * mu * pc - (l - 1.0) * pm) / l;
            acc += coef[l] * pn;
            pm = pc;
            pc = pn;
        }
        out[t] = cplx(0.0, 1.0 / k) * acc;
    }
    return out;
}

double eps_metric(const cplx* ref, const cplx* apx, std::size_t n, int* skipped) {
    double worst = 0.0;
    int skip = 0;
    for (std::size_t i = 0; i < n; ++i) {
        const double r = std::abs(ref[i]);
        if (r == 0.0) {
            ++skip;
            continue;
        }
        worst = std::max(worst, std::abs(r - std::abs(apx[i])) / r);
    }
    if (skipped) *skipped = skip;
    return worst;
}

}  // namespace ifgfb200
