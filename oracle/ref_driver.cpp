// TEST INFRASTRUCTURE ONLY — never linked into or called from the product path.
//
// A thin extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libifgf_ref.so). It lets the
// Python tests, __graft_entry__.smoke() and bench.py's CPU legs drive the reference's own
// public API (geometry, CombinedOperator, ifgf_apply, level_d_fill, solve) and read back
// its plan objects, so the B200 path can be checked against the real thing.
//
// Reference entry points wrapped here (file:line under /root/reference/proj):
//   build_sphere / assemble_mesh          src/geometry.cpp:180-211, 121-178
//   CombinedOperator ctor/apply/...       src/solver.cpp:43-167 (include/ifgf/solver.hpp:50-84)
//   ifgf_apply / level_d_fill             src/ifgf.cpp:577-608, 312-391
//   rp_singular_apply                     src/rp.cpp:421-451
//   gmres_solve / solve                   src/solver.cpp:270-340
//   save_beta_cache                       src/rp.cpp:515-536
//   far_field / near_field / mie_far_field src/postprocess.cpp:83-205
//   rp_regular_apply                      src/rp.cpp:453-479
#include <chrono>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <numbers>
#include <random>
#include <string>
#include <vector>

#include "ifgf/geometry.hpp"
#include "ifgf/ifgf.hpp"
#include "ifgf/postprocess.hpp"
#include "ifgf/rp.hpp"
#include "ifgf/solver.hpp"

using namespace ifgf;

namespace {

thread_local std::string g_err;

struct RefOp {
    std::shared_ptr<SurfaceMesh> mesh;  // the operator borrows the mesh (solver.hpp:73)
    std::unique_ptr<CombinedOperator> op;
    DlStrategy strategy = DlStrategy::Hybrid;
};

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const InvalidArgument*>(&e)) return 1;
    if (dynamic_cast<const ParseError*>(&e)) return 2;
    if (dynamic_cast<const DegenerateGeometry*>(&e)) return 3;
    if (dynamic_cast<const ConvergenceFailure*>(&e)) return 4;
    if (dynamic_cast<const InternalError*>(&e)) return 5;
    return 6;
}

std::vector<cplx> to_cplx(const double* v, std::size_t n) {
    std::vector<cplx> out(n);
    for (std::size_t i = 0; i < n; ++i) out[i] = cplx(v[2 * i], v[2 * i + 1]);
    return out;
}
void from_cplx(const std::vector<cplx>& v, double* out) {
    for (std::size_t i = 0; i < v.size(); ++i) {
        out[2 * i] = v[i].real();
        out[2 * i + 1] = v[i].imag();
    }
}

DlStrategy strat(int s) {
    return s == 0 ? DlStrategy::W4 : (s == 1 ? DlStrategy::W2W3 : DlStrategy::Hybrid);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- geometry
void* ref_mesh_sphere(double radius, int splits, int nu, int nv) {
    try {
        return new std::shared_ptr<SurfaceMesh>(
            std::make_shared<SurfaceMesh>(build_sphere(radius, splits, nu, nv)));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// Prolate spheroid: the cube-sphere patch series scaled per axis, derivative series
// recomputed by assemble_mesh.
void* ref_mesh_spheroid(int splits, int nu, int nv, double ax, double ay, double az) {
    try {
        SurfaceMesh s = build_sphere(1.0, splits, nu, nv);
        std::vector<Patch> patches = s.patches;
        const double sc[3] = {ax, ay, az};
        for (auto& p : patches)
            for (int c = 0; c < 3; ++c) {
                for (auto& v : p.coeff[c]) v *= sc[c];
                p.coeff_u[c].clear();
                p.coeff_v[c].clear();
            }
        return new std::shared_ptr<SurfaceMesh>(
            std::make_shared<SurfaceMesh>(assemble_mesh(std::move(patches), Vec3{0, 0, 0})));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_mesh_free(void* m) { delete static_cast<std::shared_ptr<SurfaceMesh>*>(m); }

static SurfaceMesh& M(void* m) { return **static_cast<std::shared_ptr<SurfaceMesh>*>(m); }

long ref_mesh_size(void* m) { return long(M(m).size()); }
int ref_mesh_npatches(void* m) { return int(M(m).patches.size()); }
double ref_mesh_diameter(void* m) { return M(m).diameter(); }

void ref_mesh_nodes(void* m, double* pos, double* nrm, double* jac, double* w, double* pu,
                    double* pv, int* patch_of) {
    const SurfaceMesh& s = M(m);
    for (std::size_t i = 0; i < s.size(); ++i) {
        pos[3 * i] = s.pos[i].x;
        pos[3 * i + 1] = s.pos[i].y;
        pos[3 * i + 2] = s.pos[i].z;
        nrm[3 * i] = s.normal[i].x;
        nrm[3 * i + 1] = s.normal[i].y;
        nrm[3 * i + 2] = s.normal[i].z;
        jac[i] = s.jac[i];
        w[i] = s.weight[i];
        pu[i] = s.pu[i];
        pv[i] = s.pv[i];
        patch_of[i] = s.patch_of[i];
    }
}

// dims = {nu, nv, du, dv}
void ref_mesh_patch_dims(void* m, int q, int* dims, double* orient) {
    const Patch& p = M(m).patches[q];
    dims[0] = p.nu;
    dims[1] = p.nv;
    dims[2] = p.du;
    dims[3] = p.dv;
    *orient = p.orient;
}

// each output holds 3 * du * dv values: component-major, u index fastest
void ref_mesh_patch_coeffs(void* m, int q, double* coeff, double* cu, double* cv) {
    const Patch& p = M(m).patches[q];
    const std::size_t n = std::size_t(p.du) * p.dv;
    for (int c = 0; c < 3; ++c) {
        std::memcpy(coeff + c * n, p.coeff[c].data(), n * sizeof(double));
        std::memcpy(cu + c * n, p.coeff_u[c].data(), n * sizeof(double));
        std::memcpy(cv + c * n, p.coeff_v[c].data(), n * sizeof(double));
    }
}

// Seeded density exactly as the reference harness draws it (tools/main.cpp:252-254,
// tests/test_solver.cpp:13-19): cplx(u(rng), u(rng)) with GCC's argument order.
void ref_random_density(long n, unsigned long long seed, double* out) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1, 1);
    std::vector<cplx> a(n);
    for (auto& v : a) v = cplx(u(rng), u(rng));
    from_cplx(a, out);
}

// ---------------------------------------------------------------- operator
// strategy: 0 = W4, 1 = W2W3, 2 = Hybrid (default). gamma <= 0 selects max{3, A/lambda}.
void* ref_op_create(void* mesh, double k, double gamma, int strategy, int workers,
                    const char* beta_cache, int ps, int pang, int n_c0, int n_s0,
                    double finest_box_lambda, int n_beta, int cov_d) {
    try {
        SolveConfig cfg;
        cfg.k = k;
        cfg.gamma = gamma;
        cfg.dl_strategy = strat(strategy);
        cfg.workers = workers;
        if (beta_cache && *beta_cache) cfg.beta_cache_path = beta_cache;
        if (ps > 0) cfg.cone.ps = ps;
        if (pang > 0) cfg.cone.pang = pang;
        if (n_c0 > 0) cfg.cone.n_c0 = n_c0;
        if (n_s0 > 0) cfg.cone.n_s0 = n_s0;
        if (finest_box_lambda > 0) cfg.finest_box_lambda = finest_box_lambda;
        if (n_beta > 0) cfg.rp.n_beta = n_beta;
        if (cov_d > 0) cfg.rp.cov_d = cov_d;
        auto* r = new RefOp;
        r->mesh = *static_cast<std::shared_ptr<SurfaceMesh>*>(mesh);
        r->op = std::make_unique<CombinedOperator>(*r->mesh, cfg);
        // resolved strategy, as the ctor does (solver.cpp:55-62)
        r->strategy = cfg.dl_strategy;
        if (r->strategy == DlStrategy::Hybrid) {
            const double lambda = 2.0 * std::numbers::pi / k;
            bool any_sub = false;
            for (int d = 3; d <= r->op->tree().depth; ++d)
                if (r->op->tree().side(d) / lambda < 0.5 - 1e-12) any_sub = true;
            if (!any_sub) r->strategy = DlStrategy::W4;
        }
        return r;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_op_free(void* h) { delete static_cast<RefOp*>(h); }
static RefOp& R(void* h) { return *static_cast<RefOp*>(h); }

double ref_op_gamma(void* h) { return R(h).op->gamma(); }
double ref_op_setup_seconds(void* h) { return R(h).op->setup_seconds(); }
int ref_op_beta_cache_hit(void* h) { return R(h).op->beta_cache_was_reused() ? 1 : 0; }
int ref_op_strategy(void* h) {
    return R(h).strategy == DlStrategy::W4 ? 0 : (R(h).strategy == DlStrategy::W2W3 ? 1 : 2);
}

int ref_op_apply(void* h, const double* phi, double* out) {
    try {
        const auto n = R(h).mesh->size();
        from_cplx(R(h).op->apply(to_cplx(phi, n)), out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_op_layer_potentials(void* h, const double* phi, double* S, double* D) {
    try {
        const auto n = R(h).mesh->size();
        std::vector<cplx> s, d;
        R(h).op->layer_potentials(to_cplx(phi, n), s, d);
        from_cplx(s, S);
        from_cplx(d, D);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_op_apply_direct(void* h, const double* phi, double* out) {
    try {
        const auto n = R(h).mesh->size();
        from_cplx(R(h).op->apply_direct(to_cplx(phi, n)), out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// IFGF far part only, on quadrature-weighted sources a (original order). strategy < 0
// uses the operator's resolved strategy.
int ref_op_ifgf_apply(void* h, const double* a, int single, int dbl, int strategy, int workers,
                      double* S, double* D) {
    try {
        const auto n = R(h).mesh->size();
        IfgfRequest req;
        req.single_layer = single != 0;
        req.double_layer = dbl != 0;
        req.strategy = strategy < 0 ? R(h).strategy : strat(strategy);
        const auto o = ifgf_apply(R(h).op->plan(), to_cplx(a, n), req, workers);
        from_cplx(o.single, S);
        from_cplx(o.dbl, D);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// RP singular correction alone (accumulates into zeroed outputs), rp.cpp:421-451
int ref_op_rp_apply(void* h, const double* phi, double* S, double* D) {
    try {
        const auto n = R(h).mesh->size();
        std::vector<cplx> s(n), d(n);
        rp_singular_apply(*R(h).mesh, R(h).op->proximity(), R(h).op->precompute(),
                          to_cplx(phi, n), s, d, 0);
        from_cplx(s, S);
        from_cplx(d, D);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// level_d_fill with the given factor codes (1..4) on Morton-ordered sources; returns the
// number of complex values written (segments * npipes * P), or -1 on error. out may be null
// to query the size.
long ref_op_level_d_fill(void* h, const double* a_perm, const int* pipes, int npipes,
                         double* out) {
    try {
        const auto& plan = R(h).op->plan();
        const int D = plan.tree->depth;
        const std::size_t total = plan.level_segs[D - 1].segs.size() *
                                  std::size_t(plan.level_cones[D - 1].points_per_seg()) *
                                  std::size_t(npipes);
        if (!out) return long(total);
        std::vector<Factor> f(npipes);
        for (int i = 0; i < npipes; ++i) f[i] = Factor(pipes[i]);
        const auto data = level_d_fill(plan, to_cplx(a_perm, plan.pts.size()), f, 0);
        from_cplx(data.blocks, out);
        return long(data.blocks.size());
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

// ---------------------------------------------------------------- plan export
int ref_op_depth(void* h) { return R(h).op->tree().depth; }

void ref_op_tree_geom(void* h, double* root_min3, double* root_side) {
    const auto& t = R(h).op->tree();
    root_min3[0] = t.root_min.x;
    root_min3[1] = t.root_min.y;
    root_min3[2] = t.root_min.z;
    *root_side = t.root_side;
}

void ref_op_perm(void* h, std::uint32_t* perm) {
    const auto& p = R(h).op->tree().perm;
    std::memcpy(perm, p.data(), p.size() * sizeof(std::uint32_t));
}

void ref_op_leaf_of_point(void* h, std::int32_t* out) {
    const auto& p = R(h).op->tree().leaf_of_point();
    std::memcpy(out, p.data(), p.size() * sizeof(std::int32_t));
}

long ref_op_nboxes(void* h, int d) { return long(R(h).op->tree().levels[d - 1].size()); }

void ref_op_boxes(void* h, int d, std::uint64_t* key, std::int32_t* coords3, std::uint32_t* begin,
                  std::uint32_t* end, std::int32_t* parent, std::int32_t* children8) {
    const auto& v = R(h).op->tree().levels[d - 1];
    for (std::size_t b = 0; b < v.size(); ++b) {
        key[b] = v[b].key;
        for (int c = 0; c < 3; ++c) coords3[3 * b + c] = v[b].coords[c];
        begin[b] = v[b].begin;
        end[b] = v[b].end;
        parent[b] = v[b].parent;
        for (int c = 0; c < 8; ++c) children8[8 * b + c] = v[b].children[c];
    }
}

// which: 0 = neighbours, 1 = cousins. ptr has nboxes+1 entries; idx may be null (size query).
long ref_op_relation(void* h, int d, int which, std::int32_t* ptr, std::int32_t* idx) {
    const auto& rel = R(h).op->relations();
    const auto& lists = which == 0 ? rel.neighbors[d - 1] : rel.cousins[d - 1];
    long total = 0;
    for (std::size_t b = 0; b < lists.size(); ++b) {
        if (ptr) ptr[b] = std::int32_t(total);
        if (idx) std::memcpy(idx + total, lists[b].data(), lists[b].size() * sizeof(std::int32_t));
        total += long(lists[b].size());
    }
    if (ptr) ptr[lists.size()] = std::int32_t(total);
    return total;
}

// level cone parameters: {ns, nc, ps, pang}; returns relevant segment count
long ref_op_level_cones(void* h, int d, int* params, double* deltas3) {
    const auto& plan = R(h).op->plan();
    const auto& lc = plan.level_cones[d - 1];
    params[0] = lc.ns;
    params[1] = lc.nc;
    params[2] = lc.ps;
    params[3] = lc.pang;
    deltas3[0] = lc.ds;
    deltas3[1] = lc.dth;
    deltas3[2] = lc.dph;
    return long(plan.level_segs[d - 1].segs.size());
}

void ref_op_level_segs(void* h, int d, std::int32_t* box, std::int32_t* gamma) {
    const auto& s = R(h).op->plan().level_segs[d - 1].segs;
    for (std::size_t i = 0; i < s.size(); ++i) {
        box[i] = s[i].box;
        gamma[i] = s[i].gamma;
    }
}

long ref_op_npairs(void* h) { return long(R(h).op->proximity().pairs.size()); }
long ref_op_nfar(void* h) { return long(R(h).op->proximity().far_nodes.size()); }

void ref_op_pairs(void* h, std::uint32_t* target, std::int32_t* patch, double* ubar, double* vbar,
                  std::uint32_t* far_begin, std::uint32_t* far_end, std::uint32_t* target_pair_begin,
                  std::uint32_t* far_nodes) {
    const auto& p = R(h).op->proximity();
    for (std::size_t i = 0; i < p.pairs.size(); ++i) {
        target[i] = p.pairs[i].target;
        patch[i] = p.pairs[i].patch;
        ubar[i] = p.pairs[i].ubar;
        vbar[i] = p.pairs[i].vbar;
        far_begin[i] = p.pairs[i].far_begin;
        far_end[i] = p.pairs[i].far_end;
    }
    std::memcpy(target_pair_begin, p.target_pair_begin.data(),
                p.target_pair_begin.size() * sizeof(std::uint32_t));
    std::memcpy(far_nodes, p.far_nodes.data(), p.far_nodes.size() * sizeof(std::uint32_t));
}

void ref_op_delta(void* h, double* delta) {
    const auto& p = R(h).op->proximity();
    std::memcpy(delta, p.delta.data(), p.delta.size() * sizeof(double));
}

long ref_op_beta_size(void* h) { return long(R(h).op->precompute().beta_single.size()); }

void ref_op_beta(void* h, std::uint64_t* offset, double* bs, double* bd) {
    const auto& pc = R(h).op->precompute();
    for (std::size_t i = 0; i < pc.offset.size(); ++i) offset[i] = pc.offset[i];
    from_cplx(pc.beta_single, bs);
    from_cplx(pc.beta_dbl, bd);
}

unsigned long long ref_op_beta_fingerprint(void* h) { return R(h).op->precompute().fingerprint; }

int ref_op_save_beta_cache(void* h, const char* path) {
    try {
        save_beta_cache(path, R(h).op->precompute());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---------------------------------------------------------------- timing helpers
// Wall time of one CombinedOperator::apply (the reference's cmd_benchmark unit,
// tools/main.cpp:256-264).
double ref_op_time_apply(void* h, const double* phi, double* out) {
    const auto n = R(h).mesh->size();
    const auto in = to_cplx(phi, n);
    const auto t0 = std::chrono::steady_clock::now();
    auto o = R(h).op->apply(in);
    const double dt =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (out) from_cplx(o, out);
    return dt;
}

// ---------------------------------------------------------------- GMRES solve
// Plane-wave solve (solver.cpp:302-340). Returns iterations, or -rc on error.
int ref_solve(void* mesh, double k, double gamma, double theta, double phi, double tol,
              int max_iter, int restart, int workers, double* density_out, double* hist_out,
              int hist_cap) {
    try {
        SolveConfig cfg;
        cfg.k = k;
        cfg.gamma = gamma;
        cfg.tol = tol;
        cfg.max_iter = max_iter;
        cfg.restart = restart;
        cfg.workers = workers;
        IncidentField inc;
        inc.theta = theta;
        inc.phi = phi;
        const auto res = solve(M(mesh), inc, cfg);
        from_cplx(res.density, density_out);
        for (int i = 0; i < int(res.residual_history.size()) && i < hist_cap; ++i)
            hist_out[i] = res.residual_history[i];
        return res.iterations;
    } catch (const std::exception& e) {
        return -fail(e);
    }
}

// postprocess (postprocess.hpp:34-52)
int ref_far_field(void* mesh, const double* density, double gamma, double k, int n_phi, int n_theta,
                  double* dirs, double* values) {
    try {
        const auto phi = to_cplx(density, M(mesh).size());
        const FarFieldGrid g = far_field(M(mesh), phi, gamma, k, n_phi, n_theta, 0);
        for (std::size_t i = 0; i < g.directions.size(); ++i) {
            dirs[3 * i] = g.directions[i].x;
            dirs[3 * i + 1] = g.directions[i].y;
            dirs[3 * i + 2] = g.directions[i].z;
        }
        from_cplx(g.values, values);
        return 0;
    } catch (const std::exception& e) {
        return -fail(e);
    }
}

int ref_near_field(void* mesh, const double* density, double gamma, double k, double theta, double phi,
                   const double* points, long npts, double flag_distance, double* scattered, double* total,
                   unsigned char* flagged) {
    try {
        const auto dens = to_cplx(density, M(mesh).size());
        std::vector<Vec3> pts(npts);
        for (long i = 0; i < npts; ++i) pts[i] = {points[3 * i], points[3 * i + 1], points[3 * i + 2]};
        IncidentField inc;
        inc.theta = theta;
        inc.phi = phi;
        const NearFieldGrid g = near_field(M(mesh), dens, gamma, k, inc, pts, flag_distance, 0);
        from_cplx(g.scattered, scattered);
        from_cplx(g.total, total);
        for (long i = 0; i < npts; ++i) flagged[i] = g.flagged[i];
        return 0;
    } catch (const std::exception& e) {
        return -fail(e);
    }
}

int ref_mie_far_field(double radius, double k, const double* direction, const double* dirs, long n,
                      int extra, double* values) {
    try {
        std::vector<Vec3> d(n);
        for (long i = 0; i < n; ++i) d[i] = {dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]};
        from_cplx(mie_far_field(radius, k, {direction[0], direction[1], direction[2]}, d, extra), values);
        return 0;
    } catch (const std::exception& e) {
        return -fail(e);
    }
}

int ref_solve_sources(void* mesh, double k, double gamma, const double* src, long nsrc, double tol, int max_iter,
                      int restart, double* density_out, double* hist_out, int hist_cap) {
    try {
        SolveConfig cfg;
        cfg.k = k;
        cfg.gamma = gamma;
        cfg.tol = tol;
        cfg.max_iter = max_iter;
        cfg.restart = restart;
        IncidentField inc;
        inc.kind = IncidentField::Kind::PointSources;
        for (long j = 0; j < nsrc; ++j) inc.sources.push_back({src[3 * j], src[3 * j + 1], src[3 * j + 2]});
        const auto res = solve(M(mesh), inc, cfg);
        from_cplx(res.density, density_out);
        for (int i = 0; i < int(res.residual_history.size()) && i < hist_cap; ++i) hist_out[i] = res.residual_history[i];
        return res.iterations;
    } catch (const std::exception& e) {
        return -fail(e);
    }
}

int ref_rp_regular_apply(void* mesh, const double* density, const double* targets, long n, double k, double* S,
                         double* D) {
    try {
        const auto dens = to_cplx(density, M(mesh).size());
        std::vector<Vec3> t(n);
        for (long i = 0; i < n; ++i) t[i] = {targets[3 * i], targets[3 * i + 1], targets[3 * i + 2]};
        std::vector<cplx> s(n), d(n);
        rp_regular_apply(M(mesh), dens, t, k, s, d, 0);
        from_cplx(s, S);
        from_cplx(d, D);
        return 0;
    } catch (const std::exception& e) {
        return -fail(e);
    }
}

int ref_closest_point(void* mesh, int q, const double* x, double u0, double v0, double* out) {
    try {
        const auto c = closest_point(M(mesh).patches[q], {x[0], x[1], x[2]}, u0, v0);
        out[0] = c.u;
        out[1] = c.v;
        out[2] = c.dist;
        return 0;
    } catch (const std::exception& e) {
        return -fail(e);
    }
}

double ref_graded(int which, double alpha, double tau, int d) {
    try {
        switch (which) {
            case 0: return cov_w(tau, d);
            case 1: return cov_w_deriv(tau, d);
            case 2: return cov_xi(alpha, tau, d);
            default: return cov_xi_deriv(alpha, tau, d);
        }
    } catch (const std::exception& e) {
        fail(e);
        return std::numeric_limits<double>::quiet_NaN();
    }
}


// ---------------------------------------------------------------- plan without beta (cfg3/cfg4)
// The large configs cannot build the reference's beta tables here (101 GB at cfg3, 178 GB at
// cfg4, hours of CPU). BASELINE.md §3 / SURVEY.md §8(d) H5: the reference is then run as
// build_octree -> compute_relations -> plan_cones -> classify_targets (the ctor's own steps,
// solver.cpp:47-51, minus beta_precompute), ifgf_apply (ifgf.cpp:577-608) and a restatement
// of the level-D near-field loop (solver.cpp:100-144) that calls the reference's own green()
// and dlayer_kernel(). The RP term is checked on a sample of targets: the sample's pairs form
// a sub-ProximityMap whose beta tables the reference's beta_precompute builds and whose
// rp_singular_apply gives the sampled targets' RP contributions (rp.cpp:309-451).
struct RefPlan {
    std::shared_ptr<SurfaceMesh> mesh;
    SolveConfig cfg;
    double gamma = 0;
    DlStrategy strategy = DlStrategy::Hybrid;
    Octree tree;
    Relations rel;
    ConePlan plan;
    ProximityMap prox;
    double t_tree = 0, t_plan = 0, t_prox = 0;
};

static double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void* ref_plan_create(void* mesh, double k, double gamma, int workers, double* times3) {
    try {
        auto* r = new RefPlan;
        r->mesh = *static_cast<std::shared_ptr<SurfaceMesh>*>(mesh);
        r->cfg.k = k;
        r->cfg.gamma = gamma;
        r->cfg.workers = workers;
        const SurfaceMesh& m = *r->mesh;
        const double lambda = 2.0 * std::numbers::pi / k;
        r->gamma = gamma > 0 ? gamma : coupling_gamma(m.diameter(), lambda);
        double t0 = now_s();
        r->tree = build_octree(m.pos, k, r->cfg.finest_box_lambda);
        r->rel = compute_relations(r->tree);
        r->t_tree = now_s() - t0;
        t0 = now_s();
        r->plan = plan_cones(r->tree, r->rel, m.pos, m.normal, r->cfg.cone, workers);
        r->t_plan = now_s() - t0;
        t0 = now_s();
        r->prox = classify_targets(m, r->tree, r->rel, r->cfg.rp, workers);
        r->t_prox = now_s() - t0;
        bool any_sub = false;  // Hybrid resolution as the ctor (solver.cpp:55-62)
        for (int d = 3; d <= r->tree.depth; ++d)
            if (r->tree.side(d) / lambda < 0.5 - 1e-12) any_sub = true;
        r->strategy = any_sub ? DlStrategy::Hybrid : DlStrategy::W4;
        if (times3) {
            times3[0] = r->t_tree;
            times3[1] = r->t_plan;
            times3[2] = r->t_prox;
        }
        return r;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_plan_free(void* h) { delete static_cast<RefPlan*>(h); }
static RefPlan& RP(void* h) { return *static_cast<RefPlan*>(h); }
double ref_plan_gamma(void* h) { return RP(h).gamma; }
int ref_plan_depth(void* h) { return RP(h).tree.depth; }
long ref_plan_npairs(void* h) { return long(RP(h).prox.pairs.size()); }
long ref_plan_nfar(void* h) { return long(RP(h).prox.far_nodes.size()); }
long ref_plan_nsegs(void* h, int d) { return long(RP(h).plan.level_segs[d - 1].segs.size()); }

// Position-dependent sequence hash sum_i splitmix64(v_i + splitmix64(i)) (mod 2^64), the
// same as tests/golden/large_check.py:seq_hash (vectorisable on the checking side)
static std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    std::uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// the level's relevant (box, gamma) pairs in plan order: v_i = box << 32 | gamma
unsigned long long ref_plan_segment_hash(void* h, int d) {
    std::uint64_t x = 0, i = 0;
    for (const auto& s : RP(h).plan.level_segs[d - 1].segs)
        x += splitmix64(((std::uint64_t(std::uint32_t(s.box)) << 32) | std::uint32_t(s.gamma)) + splitmix64(i++));
    return x;
}

// the Morton permutation
unsigned long long ref_plan_perm_hash(void* h) {
    std::uint64_t x = 0, i = 0;
    for (std::uint32_t v : RP(h).tree.perm) x += splitmix64(std::uint64_t(v) + splitmix64(i++));
    return x;
}

// S, D = IFGF far part + near-field neighbour sum - singular far-node corrections (no RP),
// i.e. layer_potentials (solver.cpp:78-147) without its final rp_singular_apply. seconds2 gets
// the wall time of ifgf_apply and of the near loop.
int ref_plan_ifgf_near(void* h, const double* phi, double* S, double* D, double* seconds2) {
    try {
        const RefPlan& r = RP(h);
        const SurfaceMesh& m = *r.mesh;
        const std::size_t n = m.size();
        const auto dens = to_cplx(phi, n);
        double t0 = now_s();
        std::vector<cplx> a(n);
        for (std::size_t i = 0; i < n; ++i) a[i] = dens[i] * (m.jac[i] * m.weight[i]);
        IfgfRequest req;
        req.single_layer = true;
        req.double_layer = true;
        req.strategy = r.strategy;
        IfgfOutputs far = ifgf_apply(r.plan, a, req, r.cfg.workers);
        const double t_ifgf = now_s() - t0;
        t0 = now_s();
        const int D_ = r.tree.depth;
        const auto& leaves = r.tree.levels[D_ - 1];
        const auto& nbs = r.rel.neighbors[D_ - 1];
        const auto& lop = r.tree.leaf_of_point();
        const double k = r.cfg.k;
        const int w = resolve_workers(r.cfg.workers);
#pragma omp parallel for schedule(dynamic, 64) num_threads(w)
        for (std::int64_t t = 0; t < std::int64_t(n); ++t) {
            const std::uint32_t p0 = r.prox.target_pair_begin[t], p1 = r.prox.target_pair_begin[t + 1];
            const Vec3 x = m.pos[t];
            cplx s{}, d{};
            for (std::int32_t nb : nbs[lop[t]])
                for (std::uint32_t j = leaves[nb].begin; j < leaves[nb].end; ++j) {
                    const std::uint32_t src = r.tree.perm[j];
                    if (src == std::uint32_t(t)) continue;
                    bool singular = false;  // the target's pairs are patch-ascending
                    for (std::uint32_t pi = p0; pi < p1 && !singular; ++pi)
                        singular = r.prox.pairs[pi].patch == m.patch_of[src];
                    if (singular) continue;
                    s += green(x, m.pos[src], k) * a[src];
                    d += dlayer_kernel(x, m.pos[src], m.normal[src], k) * a[src];
                }
            for (std::uint32_t pi = p0; pi < p1; ++pi)
                for (std::uint32_t f = r.prox.pairs[pi].far_begin; f < r.prox.pairs[pi].far_end; ++f) {
                    const std::uint32_t src = r.prox.far_nodes[f];
                    s -= green(x, m.pos[src], k) * a[src];
                    d -= dlayer_kernel(x, m.pos[src], m.normal[src], k) * a[src];
                }
            const cplx fs = far.single[t] + s, fd = far.dbl[t] + d;
            S[2 * t] = fs.real();
            S[2 * t + 1] = fs.imag();
            D[2 * t] = fd.real();
            D[2 * t + 1] = fd.imag();
        }
        const double t_near = now_s() - t0;
        if (seconds2) {
            seconds2[0] = t_ifgf;
            seconds2[1] = t_near;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// RP singular correction of the given targets (ascending, original indices) through a
// sub-ProximityMap holding only their pairs: beta_precompute + rp_singular_apply of the
// reference. S/D receive ntarget values each; npairs_out the number of pairs used.
int ref_plan_rp_sample(void* h, const double* phi, const long* targets, long ntarget, double* S, double* D,
                       long* npairs_out, double* seconds) {
    try {
        const RefPlan& r = RP(h);
        const SurfaceMesh& m = *r.mesh;
        const std::size_t n = m.size();
        ProximityMap sub;
        sub.cfg = r.prox.cfg;
        sub.delta = r.prox.delta;
        sub.target_pair_begin.assign(n + 1, 0);
        std::vector<char> take(n, 0);
        for (long i = 0; i < ntarget; ++i) take[std::size_t(targets[i])] = 1;
        for (std::size_t t = 0; t < n; ++t) {
            sub.target_pair_begin[t] = std::uint32_t(sub.pairs.size());
            if (!take[t]) continue;
            for (std::uint32_t pi = r.prox.target_pair_begin[t]; pi < r.prox.target_pair_begin[t + 1]; ++pi) {
                SingularPair sp = r.prox.pairs[pi];
                sp.far_begin = sp.far_end = 0;  // far nodes are not used by the beta tables
                sub.pairs.push_back(sp);
            }
        }
        sub.target_pair_begin[n] = std::uint32_t(sub.pairs.size());
        const double t0 = now_s();
        const SingularPrecompute prec = beta_precompute(m, sub, r.cfg.k, r.cfg.workers);
        std::vector<cplx> s(n), d(n);
        rp_singular_apply(m, sub, prec, to_cplx(phi, n), s, d, r.cfg.workers);
        if (seconds) *seconds = now_s() - t0;
        for (long i = 0; i < ntarget; ++i) {
            const std::size_t t = std::size_t(targets[i]);
            S[2 * i] = s[t].real();
            S[2 * i + 1] = s[t].imag();
            D[2 * i] = d[t].real();
            D[2 * i + 1] = d[t].imag();
        }
        if (npairs_out) *npairs_out = long(sub.pairs.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
