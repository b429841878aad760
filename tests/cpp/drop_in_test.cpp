// Drop-in check, written like the reference's own doctest suites (test_solver.cpp): the
// reference's CombinedOperator and ifgfb200::GpuCombinedOperator are built from the SAME
// ifgf::SurfaceMesh and ifgf::SolveConfig, and the GPU operator is handed unchanged to the
// reference's own gmres_solve through std::function. Exit code 0 = all checks passed.
// Built by oracle/Makefile into oracle/_ref/drop_in_test (links the reference = test infra).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numbers>
#include <random>

#include "ifgf/postprocess.hpp"
#include "ifgf/solver.hpp"
#include "../../include/ifgf_b200.hpp"

using namespace ifgf;

static std::vector<cplx> random_density(std::size_t n, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1, 1);
    std::vector<cplx> a(n);
    for (auto& v : a) v = cplx(u(rng), u(rng));
    return a;
}

static double rel_l2(const std::vector<cplx>& a, const std::vector<cplx>& b) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        num += std::norm(a[i] - b[i]);
        den += std::norm(b[i]);
    }
    return std::sqrt(num / den);
}

int main() {
    int failures = 0;
    auto check = [&](const char* name, bool ok, double v) {
        std::printf("[%s] %s (%.3e)\n", ok ? "pass" : "FAIL", name, v);
        if (!ok) ++failures;
    };
    const auto mesh = build_sphere(1.0, 1, 6, 6);  // 864 unknowns (test_solver.cpp:111-145)
    SolveConfig cfg;
    cfg.k = 2 * std::numbers::pi;
    CombinedOperator ref(mesh, cfg);
    ifgfb200::GpuCombinedOperator gpu(mesh, cfg);
    check("gamma", gpu.gamma() == ref.gamma(), gpu.gamma());

    const auto phi = random_density(mesh.size(), 31);
    check("apply parity", rel_l2(gpu.apply(phi), ref.apply(phi)) <= 1e-10, rel_l2(gpu.apply(phi), ref.apply(phi)));
    std::vector<cplx> s, d, sr, dr;
    gpu.layer_potentials(phi, s, d);
    ref.layer_potentials(phi, sr, dr);
    check("S parity", rel_l2(s, sr) <= 1e-10, rel_l2(s, sr));
    check("D parity", rel_l2(d, dr) <= 1e-10, rel_l2(d, dr));
    check("apply_direct parity", rel_l2(gpu.apply_direct(phi), ref.apply_direct(phi)) <= 1e-10,
          rel_l2(gpu.apply_direct(phi), ref.apply_direct(phi)));
    try {
        std::vector<cplx> wrong(5);
        (void)gpu.apply(wrong);
        check("size mismatch throws InvalidArgument", false, 0);
    } catch (const InvalidArgument&) {
        check("size mismatch throws InvalidArgument", true, 0);
    }

    // the reference's GMRES driving the GPU operator (solver.hpp:94-95)
    IncidentField inc;
    const auto ui = incident_trace(inc, mesh, cfg.k);
    std::vector<cplx> rhs(ui.size());
    for (std::size_t i = 0; i < ui.size(); ++i) rhs[i] = -ui[i];
    auto res_gpu = gmres_solve([&](std::span<const cplx> x) { return gpu.apply(x); }, rhs, 1e-6, 100, 0);
    auto res_ref = gmres_solve([&](std::span<const cplx> x) { return ref.apply(x); }, rhs, 1e-6, 100, 0);
    check("gmres iterations equal", res_gpu.iterations == res_ref.iterations, res_gpu.iterations);
    check("gmres solution", rel_l2(res_gpu.solution, res_ref.solution) <= 1e-8,
          rel_l2(res_gpu.solution, res_ref.solution));

    // solve() and far_field() through the header, against the reference's own
    SolveConfig scfg = cfg;
    scfg.tol = 1e-6;
    const auto sol_ref = solve(mesh, inc, scfg);
    const auto sol_gpu = gpu.solve(inc, scfg);
    check("solve iterations equal", sol_gpu.iterations == sol_ref.iterations && sol_gpu.converged, sol_gpu.iterations);
    check("solve density", rel_l2(sol_gpu.density, sol_ref.density) <= 1e-8, rel_l2(sol_gpu.density, sol_ref.density));
    const auto ff_ref = far_field(mesh, sol_ref.density, sol_ref.gamma, cfg.k, 9, 17);
    const auto ff_gpu = ifgfb200::gpu_far_field(mesh, sol_ref.density, sol_ref.gamma, cfg.k, 9, 17);
    check("far field", rel_l2(ff_gpu.values, ff_ref.values) <= 1e-12, rel_l2(ff_gpu.values, ff_ref.values));
    IncidentField pts;
    pts.kind = IncidentField::Kind::PointSources;
    pts.sources = {{0.1, 0.2, -0.1}};
    const auto ps_ref = solve(mesh, pts, scfg);
    const auto ps_gpu = gpu.solve(pts, scfg);
    check("point-source solve", ps_gpu.iterations == ps_ref.iterations &&
                                    rel_l2(ps_gpu.density, ps_ref.density) <= 1e-8,
          rel_l2(ps_gpu.density, ps_ref.density));

    // non-convergence: the reference's solve() throws ConvergenceFailure with the residual
    // history (solver.cpp:334-338); so must the GPU face
    SolveConfig tight = scfg;
    tight.tol = 1e-12;
    tight.max_iter = 3;
    std::vector<double> hist_ref, hist_gpu;
    try {
        (void)solve(mesh, inc, tight);
    } catch (const ConvergenceFailure& f) {
        hist_ref = f.residual_history;
    }
    try {
        (void)gpu.solve(inc, tight);
        check("non-convergence throws ConvergenceFailure", false, 0);
    } catch (const ConvergenceFailure& f) {
        hist_gpu = f.residual_history;
        bool same = hist_gpu.size() == hist_ref.size() && hist_ref.size() == 3;
        for (std::size_t i = 0; same && i < hist_ref.size(); ++i)
            same = std::abs(hist_gpu[i] - hist_ref[i]) <= 1e-10 * hist_ref[i];
        check("non-convergence throws ConvergenceFailure with the reference's history", same,
              double(hist_gpu.size()));
    }

    // SolveConfig::beta_cache_path (solver.cpp:64-74): the first operator writes the cache, the
    // second takes its tables from it, and the reference reads the same file
    {
        SolveConfig ccfg = cfg;
        ccfg.beta_cache_path = "/tmp/ifgf_b200_dropin_beta.bin";
        std::remove(ccfg.beta_cache_path.c_str());
        ifgfb200::GpuCombinedOperator g1(mesh, ccfg);
        ifgfb200::GpuCombinedOperator g2(mesh, ccfg);
        CombinedOperator r2(mesh, ccfg);
        check("beta cache written then reused", !g1.beta_cache_was_reused() && g2.beta_cache_was_reused() &&
                                                    r2.beta_cache_was_reused(), 0);
        check("apply with cached beta", rel_l2(g2.apply(phi), ref.apply(phi)) <= 1e-10,
              rel_l2(g2.apply(phi), ref.apply(phi)));
        std::remove(ccfg.beta_cache_path.c_str());
    }
    std::printf("%d failure(s)\n", failures);
    return failures == 0 ? 0 : 1;
}
