#include "gmres.hpp"

#include <algorithm>

namespace ifgfb200 {

namespace {

double norm2v(const std::vector<cplx>& v) {
    double s = 0;
    for (const cplx& z : v) s += std::norm(z);
    return std::sqrt(s);
}

// one Arnoldi cycle from x (solver.cpp:177-266)
GmresOutcome cycle(const ApplyFn& apply, const std::vector<cplx>& rhs, std::vector<cplx> x,
                   double tol, int m, double bnorm) {
    const std::size_t n = rhs.size();
    GmresOutcome res;
    std::vector<cplx> r = rhs, w(n);
    bool nonzero = false;
    for (const cplx& v : x) nonzero |= (v != cplx{});
    if (nonzero) {
        apply(x.data(), w.data());
        for (std::size_t i = 0; i < n; ++i) r[i] -= w[i];
    }
    const double beta = norm2v(r);
    if (beta / bnorm <= tol) {
        res.x = std::move(x);
        res.converged = true;
        return res;
    }
    std::vector<std::vector<cplx>> V(1, std::vector<cplx>(n));
    for (std::size_t i = 0; i < n; ++i) V[0][i] = r[i] / beta;
    std::vector<std::vector<cplx>> H;
    std::vector<cplx> cs(m), sn(m), g(m + 1, cplx{});
    g[0] = beta;
    for (int j = 0; j < m; ++j) {
        apply(V[j].data(), w.data());
        H.emplace_back(j + 2, cplx{});
        for (int i = 0; i <= j; ++i) {
            cplx h{};
            for (std::size_t t = 0; t < n; ++t) h += std::conj(V[i][t]) * w[t];
            H[j][i] = h;
            for (std::size_t t = 0; t < n; ++t) w[t] -= h * V[i][t];
        }
        const double hn = norm2v(w);
        H[j][j + 1] = hn;
        ++res.iterations;
        for (int i = 0; i < j; ++i) {
            const cplx t = std::conj(cs[i]) * H[j][i] + std::conj(sn[i]) * H[j][i + 1];
            H[j][i + 1] = -sn[i] * H[j][i] + cs[i] * H[j][i + 1];
            H[j][i] = t;
        }
        const double den = std::sqrt(std::norm(H[j][j]) + hn * hn);
        if (den < 1e-300) {
            res.history.push_back(std::abs(g[j]) / bnorm);
            throw ConvergenceFailure("gmres: Arnoldi breakdown", res.history);
        }
        cs[j] = H[j][j] / den;
        sn[j] = cplx(hn / den, 0.0);
        H[j][j] = std::conj(cs[j]) * H[j][j] + std::conj(sn[j]) * hn;
        H[j][j + 1] = 0.0;
        g[j + 1] = -sn[j] * g[j];
        g[j] = std::conj(cs[j]) * g[j];
        const double rel = std::abs(g[j + 1]) / bnorm;
        res.history.push_back(rel);
        if (rel <= tol || j == m - 1 || hn < 1e-14) {
            std::vector<cplx> y(j + 1);
            for (int i = j; i >= 0; --i) {
                cplx acc = g[i];
                for (int t = i + 1; t <= j; ++t) acc -= H[t][i] * y[t];
                y[i] = acc / H[i][i];
            }
            for (int i = 0; i <= j; ++i)
                for (std::size_t t = 0; t < n; ++t) x[t] += y[i] * V[i][t];
            res.x = std::move(x);
            res.converged = rel <= tol;
            return res;
        }
        V.emplace_back(n);
        for (std::size_t t = 0; t < n; ++t) V[j + 1][t] = w[t] / hn;
    }
    res.x = std::move(x);
    return res;
}

}  // namespace

GmresOutcome gmres(const ApplyFn& apply, const std::vector<cplx>& rhs, double tol, int max_iter,
                   int restart) {
    if (tol <= 0) throw InvalidArgument("gmres_solve: tolerance must be positive");
    const double bnorm = norm2v(rhs);
    if (bnorm == 0.0) {
        GmresOutcome r;
        r.x.assign(rhs.size(), cplx{});
        r.converged = true;
        return r;
    }
    if (restart <= 0) return cycle(apply, rhs, std::vector<cplx>(rhs.size()), tol, max_iter, bnorm);
    GmresOutcome total;
    std::vector<cplx> x(rhs.size(), cplx{});
    while (total.iterations < max_iter) {
        const int len = std::min(restart, max_iter - total.iterations);
        GmresOutcome r = cycle(apply, rhs, x, tol, len, bnorm);
        x = std::move(r.x);
        total.iterations += r.iterations;
        total.history.insert(total.history.end(), r.history.begin(), r.history.end());
        if (r.converged) {
            total.converged = true;
            break;
        }
    }
    total.x = std::move(x);
    return total;
}

}  // namespace ifgfb200
