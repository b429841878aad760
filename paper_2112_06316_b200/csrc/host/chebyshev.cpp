#include "chebyshev.hpp"

#include <algorithm>

namespace ifgfb200::cheb {

std::vector<double> gauss_nodes(int n) {
    if (n < 1) throw InvalidArgument("cheb: node count must be >= 1");
    std::vector<double> x(n);
    for (int k = 0; k < n; ++k) x[k] = std::cos((2.0 * k + 1.0) * kPi / (2.0 * n));
    return x;
}

void basis(int n, double x, double* out) {
    out[0] = 1.0;
    if (n > 1) out[1] = x;
    for (int i = 2; i < n; ++i) out[i] = 2.0 * x * out[i - 1] - out[i - 2];
}

namespace {

template <class T>
std::vector<T> transform_line(const T* s, int n) {
    if (n < 1) throw InvalidArgument("cheb: empty sample line");
    const std::vector<double> xs = gauss_nodes(n);
    std::vector<double> tk(n);
    std::vector<T> a(n, T{});
    for (int k = 0; k < n; ++k) {
        basis(n, xs[k], tk.data());
        for (int i = 0; i < n; ++i) a[i] += s[k] * tk[i];
    }
    for (int i = 0; i < n; ++i) a[i] *= (i == 0 ? 1.0 : 2.0) / n;
    return a;
}

template <class T>
std::vector<T> transform_grid(const T* s, int nu, int nv) {
    if (nu < 1 || nv < 1) throw InvalidArgument("cheb: bad 2d grid");
    std::vector<T> rows(std::size_t(nu) * nv), out(std::size_t(nu) * nv), col(nv);
    for (int j = 0; j < nv; ++j) {
        const auto a = transform_line(s + std::size_t(nu) * j, nu);
        std::copy(a.begin(), a.end(), rows.begin() + std::size_t(nu) * j);
    }
    for (int i = 0; i < nu; ++i) {
        for (int j = 0; j < nv; ++j) col[j] = rows[i + std::size_t(nu) * j];
        const auto a = transform_line(col.data(), nv);
        for (int j = 0; j < nv; ++j) out[i + std::size_t(nu) * j] = a[j];
    }
    return out;
}

double clenshaw_r(const double* a, int n, double x) {
    double b1 = 0, b2 = 0;
    for (int i = n - 1; i >= 1; --i) {
        const double b0 = a[i] + 2.0 * x * b1 - b2;
        b2 = b1;
        b1 = b0;
    }
    return a[0] + x * b1 - b2;
}

double clamp_unit(double x) {
    constexpr double tol = 1e-12;
    if (x > 1.0 + tol || x < -1.0 - tol)
        throw InvalidArgument("chebyshev evaluation point out of [-1,1]: x=" + std::to_string(x));
    return x > 1.0 ? 1.0 : (x < -1.0 ? -1.0 : x);
}

}  // namespace

std::vector<double> coeffs_1d(const double* s, int n) { return transform_line(s, n); }
std::vector<cplx> coeffs_1d(const cplx* s, int n) { return transform_line(s, n); }
std::vector<double> coeffs_2d(const double* s, int nu, int nv) { return transform_grid(s, nu, nv); }
std::vector<cplx> coeffs_2d(const cplx* s, int nu, int nv) { return transform_grid(s, nu, nv); }

double eval_2d(const double* c, int nu, int nv, double u, double v) {
    const double uc = clamp_unit(u), vc = clamp_unit(v);
    std::vector<double> row(nv);
    for (int j = 0; j < nv; ++j) row[j] = clenshaw_r(c + std::size_t(nu) * j, nu, uc);
    return clenshaw_r(row.data(), nv, vc);
}

std::vector<double> deriv_u(const std::vector<double>& c, int nu, int nv) {
    std::vector<double> out(c.size(), 0.0);
    if (nu == 1) return out;
    for (int j = 0; j < nv; ++j) {
        const double* a = c.data() + std::size_t(nu) * j;
        double* d = out.data() + std::size_t(nu) * j;
        d[nu - 1] = 0.0;
        d[nu - 2] = 2.0 * (nu - 1) * a[nu - 1];
        for (int i = nu - 3; i >= 0; --i) d[i] = d[i + 2] + 2.0 * (i + 1) * a[i + 1];
        d[0] *= 0.5;
    }
    return out;
}

std::vector<double> deriv_v(const std::vector<double>& c, int nu, int nv) {
    std::vector<double> out(c.size(), 0.0);
    if (nv == 1) return out;
    std::vector<double> a(nv), d(nv);
    for (int i = 0; i < nu; ++i) {
        for (int j = 0; j < nv; ++j) a[j] = c[i + std::size_t(nu) * j];
        d[nv - 1] = 0.0;
        d[nv - 2] = 2.0 * (nv - 1) * a[nv - 1];
        for (int j = nv - 3; j >= 0; --j) d[j] = d[j + 2] + 2.0 * (j + 1) * a[j + 1];
        d[0] *= 0.5;
        for (int j = 0; j < nv; ++j) out[i + std::size_t(nu) * j] = d[j];
    }
    return out;
}

void fejer(int J, std::vector<double>& nodes, std::vector<double>& weights) {
    nodes = gauss_nodes(J);
    weights.assign(J, 0.0);
    for (int j = 0; j < J; ++j) {
        double acc = 0.0;
        for (int l = 1; l <= J / 2; ++l)
            acc += std::cos(l * kPi * (2.0 * j + 1.0) / J) / (4.0 * l * l - 1.0);
        weights[j] = (2.0 / J) * (1.0 - 2.0 * acc);
    }
}

std::vector<double> transform(int n) {
    const std::vector<double> xs = gauss_nodes(n);
    std::vector<double> M(std::size_t(n) * n), tk(n);
    for (int k = 0; k < n; ++k) {
        basis(n, xs[k], tk.data());
        for (int i = 0; i < n; ++i) M[std::size_t(i) * n + k] = (i == 0 ? 1.0 : 2.0) / n * tk[i];
    }
    return M;
}

}  // namespace ifgfb200::cheb
