// ifgf_b200.hpp — header-only C++ face of the B200 operator, a drop-in for the
// reference's ifgf::CombinedOperator (/root/reference/proj/include/ifgf/solver.hpp:50-84).
//
//   ifgf::SurfaceMesh mesh = ifgf::build_sphere(1, 4, 16, 16);     // reference geometry
//   ifgf::SolveConfig cfg; cfg.k = 16 * M_PI;
//   ifgfb200::GpuCombinedOperator op(mesh, cfg);                    // same ctor arguments
//   std::vector<std::complex<double>> out = op.apply(phi);          // same apply
//   auto res = ifgf::gmres_solve([&](auto x) { return op.apply(x); }, rhs, 1e-4, 300, 50);
//
// Only plain C crosses the library boundary (include/ifgf_b200.h). Errors come back as the
// reference's exception types when its headers are included first (IFGF_B200_WITH_REFERENCE
// is defined automatically then), otherwise as ifgfb200::Error with the status code.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <span>
#include <vector>

#include "ifgf_b200.h"

#if defined(IFGF_COMMON_HPP) || __has_include("ifgf/common.hpp")
#if __has_include("ifgf/solver.hpp")
#include "ifgf/solver.hpp"
#define IFGF_B200_WITH_REFERENCE 1
#endif
#endif

namespace ifgfb200 {

using cplx = std::complex<double>;

struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void raise(int status, const char* what) {
    const std::string msg = std::string(what) + ": " + ifgf_last_error();
#ifdef IFGF_B200_WITH_REFERENCE
    switch (status) {  // the reference's taxonomy (common.hpp:40-66)
        case 1: throw ifgf::InvalidArgument(msg);
        case 2: throw ifgf::ParseError(msg, 0);
        case 3: throw ifgf::DegenerateGeometry(msg, -1);
        case 4: throw ifgf::ConvergenceFailure(msg, {});
        case 5: throw ifgf::InternalError(msg);
        default: break;
    }
#endif
    throw Error(status, msg);
}

inline void check(int rc, const char* what) {
    if (rc != 0) raise(rc < 0 ? -rc : rc, what);
}

// RAII surface handle
class Surface {
  public:
    Surface() = default;
    explicit Surface(ifgf_surface* h) : h_(h) {}
    Surface(const Surface&) = delete;
    Surface& operator=(const Surface&) = delete;
    Surface(Surface&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    ~Surface() { ifgf_surface_free(h_); }
    ifgf_surface* get() const { return h_; }
    std::size_t size() const { return std::size_t(ifgf_surface_size(h_)); }

    static Surface sphere(double radius, int splits, int nu, int nv) {
        ifgf_surface* h = nullptr;
        check(ifgf_surface_sphere(radius, splits, nu, nv, &h), "ifgf_surface_sphere");
        return Surface(h);
    }

#ifdef IFGF_B200_WITH_REFERENCE
    // exact import of the reference's assembled mesh (geometry.hpp:36-57)
    static Surface from_reference(const ifgf::SurfaceMesh& m) {
        std::vector<std::int32_t> dims;
        std::vector<double> orient, c, cu, cv, pos, nrm;
        for (const auto& p : m.patches) {
            dims.insert(dims.end(), {p.nu, p.nv, p.du, p.dv});
            orient.push_back(p.orient);
            for (int k = 0; k < 3; ++k) {
                c.insert(c.end(), p.coeff[k].begin(), p.coeff[k].end());
                cu.insert(cu.end(), p.coeff_u[k].begin(), p.coeff_u[k].end());
                cv.insert(cv.end(), p.coeff_v[k].begin(), p.coeff_v[k].end());
            }
        }
        for (std::size_t i = 0; i < m.size(); ++i) {
            pos.insert(pos.end(), {m.pos[i].x, m.pos[i].y, m.pos[i].z});
            nrm.insert(nrm.end(), {m.normal[i].x, m.normal[i].y, m.normal[i].z});
        }
        const double interior[3] = {m.interior_point.x, m.interior_point.y, m.interior_point.z};
        ifgf_surface* h = nullptr;
        check(ifgf_surface_import(int(m.patches.size()), dims.data(), orient.data(), c.data(), cu.data(),
                                  cv.data(), interior, std::int64_t(m.size()), pos.data(), nrm.data(),
                                  m.jac.data(), m.weight.data(), m.pu.data(), m.pv.data(), &h),
              "ifgf_surface_import");
        return Surface(h);
    }
#endif

  private:
    ifgf_surface* h_ = nullptr;
};

class GpuCombinedOperator {
  public:
    GpuCombinedOperator(const Surface& s, const ifgf_config& cfg) { build(s, cfg); }

#ifdef IFGF_B200_WITH_REFERENCE
    // same constructor arguments as ifgf::CombinedOperator (solver.hpp:52)
    GpuCombinedOperator(const ifgf::SurfaceMesh& mesh, const ifgf::SolveConfig& sc, int device = 0)
        : surf_(Surface::from_reference(mesh)) {
        ifgf_config c;
        ifgf_config_default(&c);
        c.k = sc.k;
        c.gamma = sc.gamma;
        c.strategy = sc.dl_strategy == ifgf::DlStrategy::W4 ? 0 : (sc.dl_strategy == ifgf::DlStrategy::W2W3 ? 1 : 2);
        c.finest_box_lambda = sc.finest_box_lambda;
        c.n_c0 = sc.cone.n_c0;
        c.n_s0 = sc.cone.n_s0;
        c.ps = sc.cone.ps;
        c.pang = sc.cone.pang;
        c.delta_rel = sc.rp.delta_rel;
        c.delta_abs = sc.rp.delta_abs;
        c.n_beta = sc.rp.n_beta;
        c.cov_d = sc.rp.cov_d;
        c.workers = sc.workers;
        c.device = device;
        // the reference ctor's cache policy (solver.cpp:64-74): load when it matches, else
        // compute on the GPU and save
        c.beta_cache_path = sc.beta_cache_path.empty() ? nullptr : sc.beta_cache_path.c_str();
        build(surf_, c);
    }
#endif

    GpuCombinedOperator(const GpuCombinedOperator&) = delete;
    GpuCombinedOperator& operator=(const GpuCombinedOperator&) = delete;
    ~GpuCombinedOperator() { ifgf_operator_free(op_); }

    std::size_t size() const { return n_; }
    double gamma() const { return ifgf_operator_gamma(op_); }

    // CombinedOperator::apply (solver.cpp:149-157)
    template <class Span>
    std::vector<cplx> apply(const Span& density) const {
        if (std::size_t(density.size()) != n_) raise(1, "apply: density size mismatch");
        std::vector<cplx> out(n_);
        check(ifgf_operator_apply(op_, reinterpret_cast<const double*>(density.data()),
                                  reinterpret_cast<double*>(out.data())),
              "apply");
        return out;
    }

    // CombinedOperator::layer_potentials (solver.cpp:78-147)
    template <class Span>
    void layer_potentials(const Span& density, std::vector<cplx>& S, std::vector<cplx>& D) const {
        if (std::size_t(density.size()) != n_) raise(1, "layer_potentials: density size mismatch");
        S.assign(n_, cplx{});
        D.assign(n_, cplx{});
        check(ifgf_operator_layer_potentials(op_, reinterpret_cast<const double*>(density.data()),
                                             reinterpret_cast<double*>(S.data()), reinterpret_cast<double*>(D.data())),
              "layer_potentials");
    }

    // CombinedOperator::apply_direct (solver.cpp:159-167)
    template <class Span>
    std::vector<cplx> apply_direct(const Span& density) const {
        std::vector<cplx> out(n_);
        check(ifgf_operator_apply_direct(op_, reinterpret_cast<const double*>(density.data()),
                                         reinterpret_cast<double*>(out.data())),
              "apply_direct");
        return out;
    }

    ifgf_operator* handle() const { return op_; }
    bool beta_cache_was_reused() const { return ifgf_operator_beta_cache_hit(op_) == 1; }

#ifdef IFGF_B200_WITH_REFERENCE
    // solve(mesh, incident, cfg) (solver.hpp:111-112) on this operator: rhs = -u^i for either
    // IncidentField kind, restarted MGS-GMRES with the Krylov basis in HBM
    ifgf::SolveResult solve(const ifgf::IncidentField& inc, const ifgf::SolveConfig& sc) const {
        std::vector<double> src;
        if (inc.kind == ifgf::IncidentField::Kind::PointSources)
            for (const auto& y : inc.sources) src.insert(src.end(), {y.x, y.y, y.z});
        ifgf::SolveResult r;
        r.density.resize(n_);
        r.residual_history.resize(std::size_t(sc.max_iter) + 1);
        int it = 0, cv = 0;
        const int rc = ifgf_solve_incident(op_, inc.theta, inc.phi, src.empty() ? nullptr : src.data(),
                                           int64_t(src.size() / 3), sc.tol, sc.max_iter, sc.restart,
                                           reinterpret_cast<double*>(r.density.data()), r.residual_history.data(),
                                           int(r.residual_history.size()), &it, &cv);
        r.iterations = it;
        r.converged = cv != 0;
        r.residual_history.resize(std::size_t(std::max(it, 0)));
        r.gamma = gamma();
        r.k = sc.k;
        // not converged (or Arnoldi breakdown): the reference's solve() throws
        // ConvergenceFailure carrying the residual history (solver.cpp:334-338)
        if (rc == 4) throw ifgf::ConvergenceFailure(std::string("solve: ") + ifgf_last_error(), r.residual_history);
        check(rc, "solve");
        return r;
    }
#endif

  private:
    void build(const Surface& s, const ifgf_config& c) {
        check(ifgf_operator_create(s.get(), &c, &op_), "GpuCombinedOperator");
        n_ = std::size_t(ifgf_operator_size(op_));
    }
    Surface surf_;
    ifgf_operator* op_ = nullptr;
    std::size_t n_ = 0;
};

#ifdef IFGF_B200_WITH_REFERENCE
// far_field(mesh, density, gamma, k, n_phi, n_theta) (postprocess.hpp:34-37), the dense sum
// on GPU `device`
inline ifgf::FarFieldGrid gpu_far_field(const ifgf::SurfaceMesh& mesh, std::span<const cplx> density, double gamma,
                                       double k, int n_phi, int n_theta, int device = 0) {
    Surface s = Surface::from_reference(mesh);
    ifgf::FarFieldGrid g = ifgf::FarFieldGrid::make(n_phi, n_theta);
    std::vector<double> dirs(3 * g.directions.size());
    check(ifgf_far_field(s.get(), reinterpret_cast<const double*>(density.data()), gamma, k, n_phi, n_theta, device,
                         dirs.data(), reinterpret_cast<double*>(g.values.data())),
          "far_field");
    return g;
}
#endif

}  // namespace ifgfb200
