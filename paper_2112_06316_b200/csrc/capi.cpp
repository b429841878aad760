// extern "C" boundary of the B200 CF-operator engine (declared in include/ifgf_b200.h).
// Every entry point catches C++ exceptions and converts them to the status codes of the
// reference's error taxonomy; messages are kept thread-local for ifgf_last_error().
#include <chrono>
#include <cstring>
#include <fstream>
#include <memory>
#include <random>
#include <string>

#include <nccl.h>

#include "../../include/ifgf_b200.h"
#include "engine.hpp"
#include "host/chebyshev.hpp"
#include <cuda_runtime.h>

#include <limits>

#include "fields_gpu.hpp"
#include "host/gmres.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace ifgfb200;

namespace ifgfb200 {
int worker_count(int requested) {
#ifdef _OPENMP
    if (requested > 0) return requested;
    return std::max(1, omp_get_max_threads());
#else
    (void)requested;
    return 1;
#endif
}
}  // namespace ifgfb200

struct ifgf_surface {
    std::shared_ptr<Surface> s;
};

struct ifgf_plan {
    std::shared_ptr<const Surface> surf;
    ifgf_config cfg{};
    double k = 0, gamma = 0;
    DlStrategy strategy = DlStrategy::Hybrid;
    BoxTree tree;
    BoxRelations rel;
    ConePlanHost cones;
    PairList pairs;
    double setup_seconds = 0;
    double t_tree = 0, t_cones = 0, t_pairs = 0;  // host setup phases (s)
};

struct ifgf_operator {
    double t_upload = 0, t_beta = 0;  // device setup phases (s)
    bool beta_cache_hit = false;      // tables loaded from cfg.beta_cache_path
    std::shared_ptr<ifgf_plan> plan;
    std::unique_ptr<Engine> eng;
};

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const EngineError& e) {
        g_error = e.what();
        return e.status;
    } catch (const std::bad_alloc& e) {
        g_error = std::string("out of memory: ") + e.what();
        return kInternalError;
    } catch (const std::exception& e) {
        g_error = e.what();
        return kInternalError;
    }
}

std::vector<cplx> as_cplx(const double* v, std::size_t n) {
    std::vector<cplx> out(n);
    std::memcpy(static_cast<void*>(out.data()), v, n * sizeof(cplx));
    return out;
}

void need(const void* p, const char* what) {
    if (!p) throw InvalidArgument(std::string(what) + ": null pointer");
}

std::shared_ptr<ifgf_plan> make_plan(std::shared_ptr<const Surface> s, const ifgf_config& c) {
    if (c.k <= 0) throw InvalidArgument("CombinedOperator: wavenumber must be positive");
    auto p = std::make_shared<ifgf_plan>();
    p->surf = s;
    p->cfg = c;
    p->k = c.k;
    const double lambda = 2.0 * kPi / c.k;
    if (c.gamma > 0) {
        p->gamma = c.gamma;
    } else {
        const double diam = s->extent();
        if (diam <= 0 || lambda <= 0) throw InvalidArgument("coupling_gamma: diameter and lambda must be positive");
        p->gamma = std::max(3.0, diam / lambda);
    }
    const auto t0 = std::chrono::steady_clock::now();
    auto lap = [t = std::chrono::steady_clock::now()]() mutable {
        const auto now = std::chrono::steady_clock::now();
        const double dt = std::chrono::duration<double>(now - t).count();
        t = now;
        return dt;
    };
    p->tree = build_boxtree(s->pos, c.k, c.finest_box_lambda);
    p->rel = build_relations(p->tree);
    p->t_tree = lap();
    std::vector<Vec3> pts(s->size());
    for (std::size_t t = 0; t < pts.size(); ++t) pts[t] = s->pos[p->tree.perm[t]];
    ConeParams cp;
    cp.n_c0 = c.n_c0;
    cp.n_s0 = c.n_s0;
    cp.ps = c.ps;
    cp.pang = c.pang;
    // segment decisions and closest-point searches batched on the GPU when one is there
    // (decisions equal to the host's bit for bit; the host redoes the flagged ones)
    int ndev = 0;
    const bool gpu = c.device >= 0 && cudaGetDeviceCount(&ndev) == cudaSuccess && c.device < ndev;
    if (!gpu) cudaGetLastError();  // clear a no-device error
    const int dev = c.device;
    const ConeDecider decider = [dev](const ConeDecisionJob& job, ConeLevel& L, std::vector<std::uint8_t>& marks,
                                      std::vector<std::int64_t>& fc, std::vector<std::int64_t>& fp) {
        gpu_cone_decisions(job, L, marks, fc, fp, dev);
    };
    if (c.part_world > 1) {  // per-rank plan: partition first (plan-free cost model), then prune
        if (c.part_rank < 0 || c.part_rank >= c.part_world) throw InvalidArgument("plan: bad part_rank / part_world");
        const auto bounds = partition_sources_light(p->tree, p->rel, c.part_world);
        const auto act = active_boxes(p->tree, bounds[c.part_rank], bounds[c.part_rank + 1]);
        p->cones = build_cone_plan(p->tree, p->rel, pts, cp, c.workers, gpu ? &decider : nullptr, &act);
        p->cones.rank = c.part_rank;
        p->cones.world = c.part_world;
        p->cones.bounds = bounds;
    } else {
        p->cones = build_cone_plan(p->tree, p->rel, pts, cp, c.workers, gpu ? &decider : nullptr);
    }
    p->t_cones = lap();
    RpParams rp;
    rp.delta_rel = c.delta_rel;
    rp.delta_abs = c.delta_abs;
    rp.n_beta = c.n_beta;
    rp.cov_d = c.cov_d;
    const ClosestPointBatch batch = [dev](const Surface& sf, const std::vector<ClosestPointRequest>& rq,
                                          std::vector<ClosestPoint>& out) { gpu_closest_points(sf, rq, out, dev); };
    std::vector<std::uint8_t> owned;  // per-rank plan: pairs of the owned targets only
    if (p->cones.world > 1) {
        owned.assign(s->size(), 0);
        for (std::uint32_t m = p->cones.bounds[p->cones.rank]; m < p->cones.bounds[p->cones.rank + 1]; ++m)
            owned[p->tree.perm[m]] = 1;
    }
    p->pairs = classify_pairs(*s, p->tree, p->rel, rp, c.workers, gpu ? &batch : nullptr,
                              owned.empty() ? nullptr : &owned);
    p->t_pairs = lap();
    p->strategy = c.strategy == 0 ? DlStrategy::W4 : (c.strategy == 1 ? DlStrategy::W2W3 : DlStrategy::Hybrid);
    if (p->strategy == DlStrategy::Hybrid) {  // solver.cpp:55-62
        bool any_sub = false;
        for (int d = 3; d <= p->tree.depth; ++d)
            if (p->tree.side(d) / lambda < 0.5 - 1e-12) any_sub = true;
        if (!any_sub) p->strategy = DlStrategy::W4;
    }
    p->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return p;
}

std::unique_ptr<Engine> make_engine(const ifgf_plan& p, int device) {
    OperatorSetup s;
    s.k = p.k;
    s.gamma = p.gamma;
    s.strategy = p.strategy;
    s.surf = p.surf.get();
    s.tree = &p.tree;
    s.rel = &p.rel;
    s.plan = &p.cones;
    s.pairs = &p.pairs;
    return std::make_unique<Engine>(s, device);
}

std::uint64_t fnv_bytes(const void* d, std::size_t n, std::uint64_t h) {
    const auto* b = static_cast<const unsigned char*>(d);
    for (std::size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 1099511628211ULL;
    }
    return h;
}

DlStrategy strategy_of(int s, DlStrategy dflt) {
    if (s < 0) return dflt;
    return s == 0 ? DlStrategy::W4 : (s == 1 ? DlStrategy::W2W3 : DlStrategy::Hybrid);
}

}  // namespace

extern "C" {

const char* ifgf_last_error(void) { return g_error.c_str(); }
int ifgf_version(void) { return 1; }

void ifgf_config_default(ifgf_config* c) {
    if (!c) return;
    c->k = 0;
    c->gamma = -1.0;
    c->strategy = 2;
    c->finest_box_lambda = 0.5;
    c->n_c0 = 2;
    c->n_s0 = 1;
    c->ps = 3;
    c->pang = 5;
    c->delta_rel = 1.0;
    c->delta_abs = -1.0;
    c->n_beta = 96;
    c->cov_d = 6;
    c->workers = 0;
    c->device = 0;
    c->part_rank = 0;
    c->part_world = 1;
    c->beta_cache_path = nullptr;
}

// ------------------------------------------------------------------ surfaces
int ifgf_surface_sphere(double radius, int splits, int nu, int nv, ifgf_surface** out) {
    return guarded([&] {
        need(out, "ifgf_surface_sphere");
        *out = new ifgf_surface{std::make_shared<Surface>(make_sphere(radius, splits, nu, nv))};
    });
}

int ifgf_surface_spheroid(int splits, int nu, int nv, double ax, double ay, double az, ifgf_surface** out) {
    return guarded([&] {
        need(out, "ifgf_surface_spheroid");
        *out = new ifgf_surface{std::make_shared<Surface>(make_spheroid(splits, nu, nv, ax, ay, az))};
    });
}

int ifgf_surface_from_series(int npatch, const int32_t* dims, const double* coeff, const double interior[3],
                             ifgf_surface** out) {
    return guarded([&] {
        need(out, "ifgf_surface_from_series");
        need(dims, "dims");
        need(coeff, "coeff");
        if (npatch < 1) throw InvalidArgument("surface: patch count must be positive");
        std::vector<Patch> ps(npatch);
        std::size_t off = 0;
        for (int q = 0; q < npatch; ++q) {
            Patch& p = ps[q];
            p.nu = dims[4 * q];
            p.nv = dims[4 * q + 1];
            p.du = dims[4 * q + 2];
            p.dv = dims[4 * q + 3];
            if (p.nu < 1 || p.nv < 1 || p.du < 1 || p.dv < 1) throw InvalidArgument("surface: nonpositive patch dimensions");
            const std::size_t m = std::size_t(p.du) * p.dv;
            for (int c = 0; c < 3; ++c) p.pos_c[c].assign(coeff + off + c * m, coeff + off + (c + 1) * m);
            off += 3 * m;
        }
        const Vec3 in = interior ? Vec3{interior[0], interior[1], interior[2]} : Vec3{0, 0, 0};
        *out = new ifgf_surface{std::make_shared<Surface>(assemble_surface(std::move(ps), in))};
    });
}

int ifgf_surface_import(int npatch, const int32_t* dims, const double* orient, const double* coeff,
                        const double* coeff_u, const double* coeff_v, const double interior[3], int64_t n,
                        const double* pos, const double* normal, const double* jac, const double* weight,
                        const double* pu, const double* pv, ifgf_surface** out) {
    return guarded([&] {
        need(out, "ifgf_surface_import");
        for (const void* p : {(const void*)dims, (const void*)orient, (const void*)coeff, (const void*)coeff_u,
                              (const void*)coeff_v, (const void*)pos, (const void*)normal, (const void*)jac,
                              (const void*)weight, (const void*)pu, (const void*)pv})
            need(p, "ifgf_surface_import");
        auto s = std::make_shared<Surface>();
        s->patches.resize(npatch);
        s->interior = interior ? Vec3{interior[0], interior[1], interior[2]} : Vec3{0, 0, 0};
        s->patch_start.assign(npatch + 1, 0);
        std::size_t off = 0;
        for (int q = 0; q < npatch; ++q) {
            Patch& p = s->patches[q];
            p.nu = dims[4 * q];
            p.nv = dims[4 * q + 1];
            p.du = dims[4 * q + 2];
            p.dv = dims[4 * q + 3];
            p.orient = orient[q];
            const std::size_t m = std::size_t(p.du) * p.dv;
            for (int c = 0; c < 3; ++c) {
                p.pos_c[c].assign(coeff + off + c * m, coeff + off + (c + 1) * m);
                p.du_c[c].assign(coeff_u + off + c * m, coeff_u + off + (c + 1) * m);
                p.dv_c[c].assign(coeff_v + off + c * m, coeff_v + off + (c + 1) * m);
            }
            off += 3 * m;
            s->patch_start[q + 1] = s->patch_start[q] + std::size_t(p.nu) * p.nv;
        }
        if (std::int64_t(s->patch_start.back()) != n) throw InvalidArgument("surface import: node count mismatch");
        s->pos.resize(n);
        s->nrm.resize(n);
        s->jac.assign(jac, jac + n);
        s->wt.assign(weight, weight + n);
        s->pu.assign(pu, pu + n);
        s->pv.assign(pv, pv + n);
        s->patch_of.resize(n);
        for (std::int64_t i = 0; i < n; ++i) {
            s->pos[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
            s->nrm[i] = {normal[3 * i], normal[3 * i + 1], normal[3 * i + 2]};
        }
        for (int q = 0; q < npatch; ++q)
            for (std::size_t l = s->patch_start[q]; l < s->patch_start[q + 1]; ++l) s->patch_of[l] = q;
        *out = new ifgf_surface{s};
    });
}

int64_t ifgf_surface_size(const ifgf_surface* s) { return s ? int64_t(s->s->size()) : -1; }
int ifgf_surface_npatches(const ifgf_surface* s) { return s ? int(s->s->patches.size()) : -1; }
double ifgf_surface_diameter(const ifgf_surface* s) { return s ? s->s->extent() : -1.0; }

int ifgf_surface_nodes(const ifgf_surface* sf, double* pos, double* normal, double* jac, double* weight,
                       double* pu, double* pv, int32_t* patch_of) {
    return guarded([&] {
        need(sf, "ifgf_surface_nodes");
        const Surface& s = *sf->s;
        for (std::size_t i = 0; i < s.size(); ++i) {
            if (pos) {
                pos[3 * i] = s.pos[i].x;
                pos[3 * i + 1] = s.pos[i].y;
                pos[3 * i + 2] = s.pos[i].z;
            }
            if (normal) {
                normal[3 * i] = s.nrm[i].x;
                normal[3 * i + 1] = s.nrm[i].y;
                normal[3 * i + 2] = s.nrm[i].z;
            }
            if (jac) jac[i] = s.jac[i];
            if (weight) weight[i] = s.wt[i];
            if (pu) pu[i] = s.pu[i];
            if (pv) pv[i] = s.pv[i];
            if (patch_of) patch_of[i] = s.patch_of[i];
        }
    });
}

int ifgf_surface_patch(const ifgf_surface* sf, int q, int32_t* dims4, double* orient, double* coeff,
                       double* coeff_u, double* coeff_v) {
    return guarded([&] {
        need(sf, "ifgf_surface_patch");
        if (q < 0 || q >= int(sf->s->patches.size())) throw InvalidArgument("surface: patch index out of range");
        const Patch& p = sf->s->patches[q];
        if (dims4) {
            dims4[0] = p.nu;
            dims4[1] = p.nv;
            dims4[2] = p.du;
            dims4[3] = p.dv;
        }
        if (orient) *orient = p.orient;
        const std::size_t m = std::size_t(p.du) * p.dv;
        for (int c = 0; c < 3; ++c) {
            if (coeff) std::memcpy(coeff + c * m, p.pos_c[c].data(), m * sizeof(double));
            if (coeff_u) std::memcpy(coeff_u + c * m, p.du_c[c].data(), m * sizeof(double));
            if (coeff_v) std::memcpy(coeff_v + c * m, p.dv_c[c].data(), m * sizeof(double));
        }
    });
}

void ifgf_surface_free(ifgf_surface* s) { delete s; }

int ifgf_random_density(int64_t n, uint64_t seed, double* out) {
    return guarded([&] {
        need(out, "ifgf_random_density");
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> u(-1, 1);
        for (int64_t i = 0; i < n; ++i) {
            // GCC evaluates cplx(u(rng), u(rng)) right to left: the first draw is the
            // imaginary part (SURVEY.md §0 finding 7); state it explicitly here
            const double im = u(rng);
            const double re = u(rng);
            out[2 * i] = re;
            out[2 * i + 1] = im;
        }
    });
}

// ------------------------------------------------------------------ plan
int ifgf_plan_create(const ifgf_surface* s, const ifgf_config* cfg, ifgf_plan** out) {
    return guarded([&] {
        need(s, "surface");
        need(cfg, "config");
        need(out, "out");
        auto p = make_plan(s->s, *cfg);
        *out = new ifgf_plan(std::move(*p));
    });
}

void ifgf_plan_free(ifgf_plan* p) { delete p; }
int ifgf_plan_depth(const ifgf_plan* p) { return p ? p->tree.depth : -1; }
double ifgf_plan_gamma(const ifgf_plan* p) { return p ? p->gamma : 0.0; }
int ifgf_plan_strategy(const ifgf_plan* p) { return p ? int(p->strategy) : -1; }
double ifgf_plan_setup_seconds(const ifgf_plan* p) { return p ? p->setup_seconds : 0.0; }

int ifgf_plan_perm(const ifgf_plan* p, uint32_t* perm) {
    return guarded([&] {
        need(p, "plan");
        std::memcpy(perm, p->tree.perm.data(), p->tree.perm.size() * sizeof(uint32_t));
    });
}

int ifgf_plan_tree_geom(const ifgf_plan* p, double root_min[3], double* root_side) {
    return guarded([&] {
        need(p, "plan");
        root_min[0] = p->tree.root_min.x;
        root_min[1] = p->tree.root_min.y;
        root_min[2] = p->tree.root_min.z;
        *root_side = p->tree.root_side;
    });
}

int64_t ifgf_plan_nboxes(const ifgf_plan* p, int level) {
    if (!p || level < 1 || level > p->tree.depth) return -1;
    return int64_t(p->tree.level[level - 1].size());
}

int ifgf_plan_boxes(const ifgf_plan* p, int level, uint64_t* key, int32_t* cell3, uint32_t* begin, uint32_t* end,
                    int32_t* parent, int32_t* child8) {
    return guarded([&] {
        need(p, "plan");
        if (level < 1 || level > p->tree.depth) throw InvalidArgument("plan: level out of range");
        const BoxLevel& B = p->tree.level[level - 1];
        for (std::size_t b = 0; b < B.size(); ++b) {
            if (key) key[b] = B.key[b];
            for (int c = 0; c < 3; ++c)
                if (cell3) cell3[3 * b + c] = B.cell[b][c];
            if (begin) begin[b] = B.begin[b];
            if (end) end[b] = B.end[b];
            if (parent) parent[b] = B.parent[b];
            for (int c = 0; c < 8; ++c)
                if (child8) child8[8 * b + c] = B.child[b][c];
        }
    });
}

int64_t ifgf_plan_relation(const ifgf_plan* p, int level, int which, int32_t* ptr, int32_t* idx) {
    if (!p || level < 1 || level > p->tree.depth) return -1;
    const Adjacency& a = which == 0 ? p->rel.nbr[level - 1] : p->rel.cousin[level - 1];
    if (ptr) std::memcpy(ptr, a.ptr.data(), a.ptr.size() * sizeof(int32_t));
    if (idx) std::memcpy(idx, a.idx.data(), a.idx.size() * sizeof(int32_t));
    return int64_t(a.idx.size());
}

int64_t ifgf_plan_level(const ifgf_plan* p, int level, int32_t* params4, double* deltas3, int32_t* seg_box,
                        int32_t* seg_gamma) {
    if (!p || level < 3 || level > p->tree.depth) return -1;
    const ConeLevel& L = p->cones.level[level - 1];
    if (params4) {
        params4[0] = L.ns;
        params4[1] = L.nc;
        params4[2] = L.ps;
        params4[3] = L.pang;
    }
    if (deltas3) {
        deltas3[0] = L.ds;
        deltas3[1] = L.dth;
        deltas3[2] = L.dph;
    }
    if (seg_box) std::memcpy(seg_box, L.seg_box.data(), L.seg_box.size() * sizeof(int32_t));
    if (seg_gamma) std::memcpy(seg_gamma, L.seg_gamma.data(), L.seg_gamma.size() * sizeof(int32_t));
    return int64_t(L.nseg());
}

uint64_t ifgf_plan_decision_hash(const ifgf_plan* p, int level) {
    if (!p || level < 3 || level > p->tree.depth) return 0;
    const ConeLevel& L = p->cones.level[level - 1];
    std::uint64_t h = 1469598103934665603ULL;
    auto mix = [&](const void* data, std::size_t n) {
        const auto* b = static_cast<const unsigned char*>(data);
        for (std::size_t i = 0; i < n; ++i) {
            h ^= b[i];
            h *= 1099511628211ULL;
        }
    };
    mix(L.cev_seg.data(), L.cev_seg.size() * sizeof(std::int32_t));
    mix(L.pev_seg.data(), L.pev_seg.size() * sizeof(std::int32_t));
    mix(L.pev_perm.data(), L.pev_perm.size() * sizeof(std::uint16_t));
    mix(L.pgrp_seg.data(), L.pgrp_seg.size() * sizeof(std::int32_t));
    return h;
}

int64_t ifgf_plan_evaluations(const ifgf_plan* p, int level, int which) {
    if (!p || level < 3 || level > p->tree.depth) return -1;
    const ConeLevel& L = p->cones.level[level - 1];
    return int64_t(which == 0 ? L.cev_seg.size() : L.pev_seg.size());
}

// {groups, evaluations, 8-row tensor-core tiles} of the parent-node evaluations into level
int ifgf_plan_tile_stats(const ifgf_plan* p, int level, int64_t* out3) {
    return guarded([&] {
        need(p, "plan");
        if (level < 4 || level > p->tree.depth) throw InvalidArgument("tile stats: level out of range");
        const ConeLevel& L = p->cones.level[level - 1];
        int64_t tiles = 0;
        for (std::size_t g = 0; g < L.pgrp_count.size(); ++g) tiles += (L.pgrp_count[g] + 7) / 8;
        out3[0] = int64_t(L.pgrp_seg.size());
        out3[1] = int64_t(L.pev_seg.size());
        out3[2] = tiles;
    });
}

int ifgf_plan_cousin_tile_stats(const ifgf_plan* p, int level, int items_of, int64_t* out3) {
    return guarded([&] {
        need(p, "plan");
        need(out3, "out");
        if (level < 3 || level > p->tree.depth || items_of < 1) throw InvalidArgument("cousin tile stats: bad level");
        const ConeLevel& L = p->cones.level[level - 1];
        const BoxLevel& B = p->tree.level[level - 1];
        int64_t evals = 0, groups = 0, tiles = 0;
        std::vector<std::int32_t> segs;
        for (std::size_t tb = 0; tb < B.size(); ++tb) {
            const int64_t n_t = B.end[tb] - B.begin[tb];
            const int ncz = int(L.cz.count(tb));
            for (int64_t q0 = 0; q0 < n_t; q0 += items_of)
                for (int j = 0; j < ncz; ++j) {
                    segs.clear();
                    for (int64_t q = q0; q < std::min(n_t, q0 + items_of); ++q)
                        segs.push_back(L.cev_seg[std::size_t(L.cev_begin[tb] + j * n_t + q)]);
                    std::sort(segs.begin(), segs.end());
                    for (std::size_t i = 0; i < segs.size();) {
                        std::size_t e = i;
                        while (e < segs.size() && segs[e] == segs[i]) ++e;
                        ++groups;
                        tiles += int64_t((e - i + 7) / 8);
                        evals += int64_t(e - i);
                        i = e;
                    }
                }
        }
        out3[0] = evals;
        out3[1] = groups;
        out3[2] = tiles;
    });
}

int64_t ifgf_plan_npairs(const ifgf_plan* p) { return p ? int64_t(p->pairs.size()) : -1; }
int64_t ifgf_plan_nfar(const ifgf_plan* p) { return p ? int64_t(p->pairs.far_nodes.size()) : -1; }

int ifgf_plan_pairs(const ifgf_plan* p, uint32_t* target, int32_t* patch, double* ubar, double* vbar,
                    uint32_t* far_begin, uint32_t* far_end, uint32_t* tpb, uint32_t* far_nodes) {
    return guarded([&] {
        need(p, "plan");
        const PairList& L = p->pairs;
        const std::size_t np = L.size();
        if (target) std::memcpy(target, L.target.data(), np * sizeof(uint32_t));
        if (patch) std::memcpy(patch, L.patch.data(), np * sizeof(int32_t));
        if (ubar) std::memcpy(ubar, L.ubar.data(), np * sizeof(double));
        if (vbar) std::memcpy(vbar, L.vbar.data(), np * sizeof(double));
        if (far_begin) std::memcpy(far_begin, L.far_begin.data(), np * sizeof(uint32_t));
        if (far_end) std::memcpy(far_end, L.far_end.data(), np * sizeof(uint32_t));
        if (tpb) std::memcpy(tpb, L.target_pair_begin.data(), L.target_pair_begin.size() * sizeof(uint32_t));
        if (far_nodes) std::memcpy(far_nodes, L.far_nodes.data(), L.far_nodes.size() * sizeof(uint32_t));
    });
}

uint64_t ifgf_plan_beta_fingerprint(const ifgf_plan* p) { return p ? beta_key(*p->surf, p->pairs, p->k) : 0; }

int ifgf_plan_diagnostics(const ifgf_plan* p, char* buf, size_t cap) {
    return guarded([&] {
        need(p, "plan");
        const std::string s = plan_diagnostics(p->tree, p->cones);
        if (buf && cap) {
            const std::size_t n = std::min(cap - 1, s.size());
            std::memcpy(buf, s.data(), n);
            buf[n] = 0;
        }
    });
}

static void plan_work(const ifgf_plan& p, double* w) {
    for (int i = 0; i < 16; ++i) w[i] = 0;
    const BoxTree& T = p.tree;
    const int D = T.depth;
    const Surface& S = *p.surf;
    auto npipes = [&](int d) {
        int n = 1;  // W1
        n += int(dl_pipes(T, d, p.strategy).size());
        return n;
    };
    const double P = double(p.cfg.ps) * p.cfg.pang * p.cfg.pang;
    constexpr double kTransform = 3900.0;  // block transform flops per block per pipe
    if (D >= 3) {
        const ConeLevel& L = p.cones.level[D - 1];
        const BoxLevel& B = T.level[D - 1];
        double inter = 0;
        for (std::size_t so = 0; so < L.nseg(); ++so) {
            const int b = L.seg_box[so];
            inter += P * double(B.end[b] - B.begin[b]);
        }
        w[0] = inter;
        w[5] = 47.0 * inter + kTransform * double(L.nseg()) * npipes(D);
        w[10] = 64.0 * double(S.size()) + 16.0 * P * double(L.nseg()) * npipes(D);
        for (int d = D; d >= 3; --d) {
            const ConeLevel& C = p.cones.level[d - 1];
            const double ev = double(C.cev_seg.size());
            const int pc = npipes(d);
            w[1] += ev;
            w[6] += ev * (26.0 + pc * 434.0 + 6.0 + 8.0 * pc);
            w[11] += 16.0 * P * double(C.nseg()) * pc + 4.0 * ev + 88.0 * double(S.size());
            if (d > 3) {
                const ConeLevel& PL = p.cones.level[d - 2];
                const double pev = double(C.pev_seg.size());
                const int pp = npipes(d - 1);
                const bool conv = dl_pipes(T, d, p.strategy).size() == 2 && dl_pipes(T, d - 1, p.strategy).size() == 1;
                w[2] += pev;
                w[7] += pev * (26.0 + pc * 434.0 + 27.0 + 8.0 * pp + (conv ? 19.0 : 0.0)) +
                        kTransform * double(PL.nseg()) * pp;
                w[12] += 16.0 * P * (double(C.nseg()) * pc + double(PL.nseg()) * pp) + 4.0 * pev;
            }
        }
    }
    // near field: evaluated neighbour pairs + far-node corrections (solver.cpp:100-144)
    const BoxLevel& leaves = T.level[D - 1];
    const Adjacency& nb = p.rel.nbr[D - 1];
    double pairs = 0;
#pragma omp parallel for reduction(+ : pairs) schedule(dynamic, 256)
    for (std::int64_t l = 0; l < std::int64_t(S.size()); ++l) {
        const int tb = T.leaf_of[l];
        const std::uint32_t p0 = p.pairs.target_pair_begin[l], p1 = p.pairs.target_pair_begin[l + 1];
        double cnt = 0;
        for (int j = nb.ptr[tb]; j < nb.ptr[tb + 1]; ++j) {
            const int b = nb.idx[j];
            for (std::uint32_t t = leaves.begin[b]; t < leaves.end[b]; ++t) {
                const std::uint32_t m = T.perm[t];
                if (m == std::uint32_t(l)) continue;
                bool sing = false;
                for (std::uint32_t q = p0; q < p1; ++q) sing |= (p.pairs.patch[q] == S.patch_of[m]);
                if (!sing) cnt += 1;
            }
        }
        for (std::uint32_t q = p0; q < p1; ++q) cnt += double(p.pairs.far_end[q] - p.pairs.far_begin[q]);
        pairs += cnt;
    }
    w[3] = pairs;
    w[8] = 47.0 * pairs;
    w[13] = 64.0 * double(S.size()) + 64.0 * double(S.size()) + 4.0 * double(p.pairs.far_nodes.size());
    double entries = 0;
    for (std::size_t i = 0; i < p.pairs.size(); ++i) {
        const Patch& q = S.patches[p.pairs.patch[i]];
        entries += double(q.nu) * q.nv;
    }
    w[4] = double(p.pairs.size());
    w[9] = 16.0 * entries;
    w[14] = 32.0 * entries + 8.0 * double(p.pairs.size());
    w[15] = w[5] + w[6] + w[7] + w[8] + w[9];
}

int ifgf_plan_work(const ifgf_plan* p, double* w) {
    return guarded([&] {
        need(p, "plan");
        need(w, "work");
        plan_work(*p, w);
    });
}

int ifgf_operator_work(const ifgf_operator* op, double* w) {
    return guarded([&] {
        need(op, "operator");
        need(w, "work");
        plan_work(*op->plan, w);
    });
}

// ------------------------------------------------------------------ operator
int ifgf_operator_create(const ifgf_surface* s, const ifgf_config* cfg, ifgf_operator** out) {
    return guarded([&] {
        need(s, "surface");
        need(cfg, "config");
        need(out, "out");
        auto op = std::make_unique<ifgf_operator>();
        op->plan = make_plan(s->s, *cfg);
        const auto t0 = std::chrono::steady_clock::now();
        op->eng = make_engine(*op->plan, cfg->device);
        const auto t1 = std::chrono::steady_clock::now();
        // the reference ctor's cache policy (solver.cpp:64-74): a matching cache is used,
        // otherwise the tables are computed and, with a path, written there
        const bool cached = cfg->beta_cache_path && *cfg->beta_cache_path &&
                            ifgf_operator_load_beta_cache(op.get(), cfg->beta_cache_path) == 1;
        if (!cached) {
            op->eng->compute_beta();
            if (cfg->beta_cache_path && *cfg->beta_cache_path) {
                const int rc = ifgf_operator_save_beta_cache(op.get(), cfg->beta_cache_path);
                if (rc) throw EngineError(rc, g_error);
            }
        }
        op->beta_cache_hit = cached;
        op->t_upload = std::chrono::duration<double>(t1 - t0).count();
        op->t_beta = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
        *out = op.release();
    });
}

int ifgf_operator_beta_cache_hit(const ifgf_operator* op) { return op && op->beta_cache_hit ? 1 : 0; }

int ifgf_operator_from_plan(ifgf_plan* p, int device, int compute_beta, ifgf_operator** out) {
    return guarded([&] {
        need(p, "plan");
        need(out, "out");
        auto op = std::make_unique<ifgf_operator>();
        // the operator shares the plan; the caller's handle stays valid and owns its copy
        op->plan = std::make_shared<ifgf_plan>(*p);
        op->eng = make_engine(*op->plan, device);
        if (compute_beta) op->eng->compute_beta();
        *out = op.release();
    });
}

int ifgf_operator_compute_beta(ifgf_operator* op) {
    return guarded([&] {
        need(op, "operator");
        const auto t = std::chrono::steady_clock::now();
        op->eng->compute_beta();
        op->t_beta = std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
    });
}

void ifgf_operator_free(ifgf_operator* op) { delete op; }
int64_t ifgf_operator_size(const ifgf_operator* op) { return op ? int64_t(op->eng->size()) : -1; }
double ifgf_operator_gamma(const ifgf_operator* op) { return op ? op->plan->gamma : 0.0; }

int ifgf_operator_apply(ifgf_operator* op, const double* phi, double* out) {
    return guarded([&] {
        need(op, "operator");
        need(phi, "phi");
        need(out, "out");
        op->eng->apply(reinterpret_cast<const cplx*>(phi), reinterpret_cast<cplx*>(out));
    });
}

int ifgf_operator_layer_potentials(ifgf_operator* op, const double* phi, double* S, double* D) {
    return guarded([&] {
        need(op, "operator");
        need(phi, "phi");
        need(S, "S");
        need(D, "D");
        std::vector<cplx> tmp(op->eng->size());
        op->eng->apply(reinterpret_cast<const cplx*>(phi), tmp.data(), reinterpret_cast<cplx*>(S),
                       reinterpret_cast<cplx*>(D));
    });
}

int ifgf_operator_apply_device(ifgf_operator* op, const void* phi_dev, void* out_dev) {
    return guarded([&] {
        need(op, "operator");
        need(phi_dev, "phi");
        need(out_dev, "out");
        op->eng->apply_device(phi_dev, out_dev);
    });
}

int ifgf_operator_apply_direct(ifgf_operator* op, const double* phi, double* out) {
    return guarded([&] {
        need(op, "operator");
        op->eng->apply_direct(reinterpret_cast<const cplx*>(phi), reinterpret_cast<cplx*>(out));
    });
}

int ifgf_operator_ifgf_apply(ifgf_operator* op, const double* a, int single, int dbl, int strategy, double* S,
                             double* D) {
    return guarded([&] {
        need(op, "operator");
        need(a, "a");
        op->eng->ifgf_apply(reinterpret_cast<const cplx*>(a), single != 0, dbl != 0,
                            strategy_of(strategy, op->plan->strategy), reinterpret_cast<cplx*>(S),
                            reinterpret_cast<cplx*>(D));
    });
}

int64_t ifgf_operator_level_d_fill(ifgf_operator* op, const double* a_perm, const int32_t* pipes, int npipes,
                                   double* out, int64_t capacity) {
    int64_t written = 0;
    const int rc = guarded([&] {
        need(op, "operator");
        need(pipes, "pipes");
        const ifgf_plan& p = *op->plan;
        const int D = p.tree.depth;
        if (D < 3) return;
        const ConeLevel& L = p.cones.level[D - 1];
        const int64_t total = int64_t(L.nseg()) * L.nodes_per_seg() * npipes;
        if (!out) {
            written = total;
            return;
        }
        if (capacity < total) throw InvalidArgument("level_d_fill: output too small");
        std::vector<int> pv(pipes, pipes + npipes);
        for (int f : pv)
            if (f < 1 || f > 4) throw InvalidArgument("level_d_fill: factor codes are 1..4");
        std::vector<cplx> blocks;
        op->eng->level_d_fill(reinterpret_cast<const cplx*>(a_perm), pv, blocks);
        std::memcpy(out, blocks.data(), blocks.size() * sizeof(cplx));
        written = int64_t(blocks.size());
    });
    return rc ? -rc : written;
}

int ifgf_operator_rp_apply(ifgf_operator* op, const double* phi, double* S, double* D) {
    return guarded([&] {
        need(op, "operator");
        op->eng->rp_apply(reinterpret_cast<const cplx*>(phi), reinterpret_cast<cplx*>(S),
                          reinterpret_cast<cplx*>(D));
    });
}

int64_t ifgf_operator_beta_entries(const ifgf_operator* op) {
    if (!op) return -1;
    int64_t total = 0;
    const ifgf_plan& p = *op->plan;
    for (std::size_t i = 0; i < p.pairs.size(); ++i) {
        const Patch& q = p.surf->patches[p.pairs.patch[i]];
        total += int64_t(q.nu) * q.nv;
    }
    return total;
}

int64_t ifgf_operator_npairs(const ifgf_operator* op) { return op ? int64_t(op->plan->pairs.size()) : -1; }

int ifgf_operator_set_beta(ifgf_operator* op, const uint64_t* offset, const double* bs, const double* bd) {
    return guarded([&] {
        need(op, "operator");
        std::vector<std::uint64_t> off(offset, offset + op->plan->pairs.size() + 1);
        op->eng->upload_beta(off, reinterpret_cast<const cplx*>(bs), reinterpret_cast<const cplx*>(bd));
    });
}

int ifgf_operator_get_beta(ifgf_operator* op, uint64_t* offset, double* bs, double* bd) {
    return guarded([&] {
        need(op, "operator");
        std::vector<std::uint64_t> off;
        std::vector<cplx> s, d;
        op->eng->download_beta(off, s, d);
        if (offset) std::memcpy(offset, off.data(), off.size() * sizeof(uint64_t));
        if (bs) std::memcpy(bs, s.data(), s.size() * sizeof(cplx));
        if (bd) std::memcpy(bd, d.data(), d.size() * sizeof(cplx));
    });
}

// "rpbeta v1" layout of rp.cpp:515-536
int ifgf_operator_save_beta_cache(ifgf_operator* op, const char* path) {
    return guarded([&] {
        need(op, "operator");
        need(path, "path");
        std::vector<std::uint64_t> off;
        std::vector<cplx> s, d;
        op->eng->download_beta(off, s, d);
        std::ofstream f(path, std::ios::binary);
        if (!f) throw InvalidArgument(std::string("save_beta_cache: cannot open ") + path);
        f << "rpbeta v1\n";
        auto put = [&](const void* p, std::size_t n) { f.write(static_cast<const char*>(p), std::streamsize(n)); };
        const ifgf_plan& p = *op->plan;
        const std::uint64_t fp = beta_key(*p.surf, p.pairs, p.k);
        const double k = p.k;
        const std::int32_t nb = p.pairs.cfg.n_beta, cd = p.pairs.cfg.cov_d;
        const std::uint64_t npairs = off.size() - 1, ntab = s.size();
        put(&fp, 8);
        put(&k, 8);
        put(&nb, 4);
        put(&cd, 4);
        put(&npairs, 8);
        put(&ntab, 8);
        put(off.data(), off.size() * 8);
        put(s.data(), ntab * sizeof(cplx));
        put(d.data(), ntab * sizeof(cplx));
        std::uint64_t chk = 14695981039346656037ULL;
        chk = fnv_bytes(off.data(), off.size() * 8, chk);
        chk = fnv_bytes(s.data(), ntab * sizeof(cplx), chk);
        chk = fnv_bytes(d.data(), ntab * sizeof(cplx), chk);
        put(&chk, 8);
    });
}

int ifgf_operator_load_beta_cache(ifgf_operator* op, const char* path) {
    int used = 0;
    const int rc = guarded([&] {
        need(op, "operator");
        need(path, "path");
        std::ifstream f(path, std::ios::binary);
        if (!f) return;
        std::string header;
        if (!std::getline(f, header) || header != "rpbeta v1") return;
        auto get = [&](void* p, std::size_t n) {
            f.read(static_cast<char*>(p), std::streamsize(n));
            return bool(f);
        };
        std::uint64_t fp = 0, npairs = 0, ntab = 0;
        double k = 0;
        std::int32_t nb = 0, cd = 0;
        if (!get(&fp, 8) || !get(&k, 8) || !get(&nb, 4) || !get(&cd, 4) || !get(&npairs, 8) || !get(&ntab, 8)) return;
        const ifgf_plan& p = *op->plan;
        if (fp != beta_key(*p.surf, p.pairs, p.k)) return;
        if (npairs != p.pairs.size() || ntab > (1ULL << 40)) return;
        std::vector<std::uint64_t> off(npairs + 1);
        std::vector<cplx> s(ntab), d(ntab);
        if (!get(off.data(), off.size() * 8) || !get(s.data(), ntab * sizeof(cplx)) || !get(d.data(), ntab * sizeof(cplx)))
            return;
        std::uint64_t want = 0;
        if (!get(&want, 8)) return;
        std::uint64_t chk = 14695981039346656037ULL;
        chk = fnv_bytes(off.data(), off.size() * 8, chk);
        chk = fnv_bytes(s.data(), ntab * sizeof(cplx), chk);
        chk = fnv_bytes(d.data(), ntab * sizeof(cplx), chk);
        if (chk != want) return;
        op->eng->upload_beta(off, s.data(), d.data());
        used = 1;
    });
    return rc ? -rc : used;
}

int ifgf_operator_upload_density(ifgf_operator* op, const double* phi) {
    return guarded([&] {
        need(op, "operator");
        op->eng->upload_density(reinterpret_cast<const cplx*>(phi));
    });
}

int ifgf_operator_time_applies(ifgf_operator* op, int iters, int flush_l2, double* ms) {
    return guarded([&] {
        need(op, "operator");
        need(ms, "ms");
        *ms = op->eng->time_device_applies(iters, flush_l2 != 0);
    });
}

int ifgf_operator_time_applies_each(ifgf_operator* op, int iters, int flush_l2, double* ms_each) {
    return guarded([&] {
        need(op, "operator");
        need(ms_each, "ms_each");
        const auto v = op->eng->time_device_applies_each(iters, flush_l2 != 0);
        for (std::size_t i = 0; i < v.size(); ++i) ms_each[i] = v[i];
    });
}

int ifgf_operator_time_phases(ifgf_operator* op, double* ms7) {
    return guarded([&] {
        need(op, "operator");
        need(ms7, "ms7");
        const PhaseTimes t = op->eng->time_phases();
        const double v[7] = {t.weights, t.leaf, t.cousin, t.parent, t.near, t.rp, t.total};
        std::memcpy(ms7, v, sizeof v);
    });
}

int ifgf_operator_kernels_per_apply(const ifgf_operator* op) { return op ? op->eng->kernels_per_apply() : -1; }
void* ifgf_operator_device_phi(ifgf_operator* op) { return op ? op->eng->device_phi() : nullptr; }
void* ifgf_operator_device_out(ifgf_operator* op) { return op ? op->eng->device_out() : nullptr; }

// {octree+relations, cone plan, proximity, HBM upload, GPU beta tables} seconds
int ifgf_operator_setup_times(const ifgf_operator* op, double* t5) {
    return guarded([&] {
        need(op, "operator");
        need(t5, "t5");
        const double v[5] = {op->plan->t_tree, op->plan->t_cones, op->plan->t_pairs, op->t_upload, op->t_beta};
        std::memcpy(t5, v, sizeof v);
    });
}

// ------------------------------------------------------------------ multi-GPU
int ifgf_nccl_unique_id(void* id128) {
    return guarded([&] {
        need(id128, "id");
        ncclUniqueId id;
        const ncclResult_t r = ncclGetUniqueId(&id);
        if (r != ncclSuccess) throw EngineError(kNcclError, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(id128, &id, sizeof id);
    });
}

int ifgf_operator_set_comm(ifgf_operator* op, int rank, int world, const void* id128) {
    return guarded([&] {
        need(op, "operator");
        need(id128, "id");
        op->eng->set_comm(rank, world, id128);
    });
}

int ifgf_operator_partition(const ifgf_operator* op, int parts, uint32_t* bounds) {
    return guarded([&] {
        need(op, "operator");
        need(bounds, "bounds");
        const auto b = op->eng->partition_bounds(parts);
        std::memcpy(bounds, b.data(), b.size() * sizeof(uint32_t));
    });
}

int ifgf_plan_partition(const ifgf_plan* p, int parts, uint32_t* bounds) {
    return guarded([&] {
        need(p, "plan");
        need(bounds, "bounds");
        const auto b = p->cones.world > 1 ? p->cones.bounds : partition_sources(p->tree, p->rel, p->cones, parts);
        if (p->cones.world > 1 && parts != p->cones.world)
            throw InvalidArgument("partition: a per-rank plan is partitioned " + std::to_string(p->cones.world) + " ways");
        std::memcpy(bounds, b.data(), b.size() * sizeof(uint32_t));
    });
}

int ifgf_operator_set_partition(ifgf_operator* op, uint32_t lo, uint32_t hi) {
    return guarded([&] {
        need(op, "operator");
        op->eng->set_partition(lo, hi);
    });
}

int ifgf_operator_finish_owned(ifgf_operator* op, const double* phi, const double* far_S, const double* far_D,
                               double* out) {
    return guarded([&] {
        need(op, "operator");
        for (const void* p : {(const void*)phi, (const void*)far_S, (const void*)far_D, (const void*)out})
            need(p, "finish_owned");
        op->eng->finish_owned(reinterpret_cast<const cplx*>(phi), reinterpret_cast<const cplx*>(far_S),
                              reinterpret_cast<const cplx*>(far_D), reinterpret_cast<cplx*>(out));
    });
}

// ------------------------------------------------------------------ GMRES
int ifgf_gmres_solve(ifgf_operator* op, const double* rhs, double tol, int max_iter, int restart, double* x,
                     double* history, int history_cap, int* iterations, int* converged) {
    return guarded([&] {
        need(op, "operator");
        need(rhs, "rhs");
        const std::size_t n = op->eng->size();
        const auto b = as_cplx(rhs, n);
        GmresOutcome r;
        try {
            r = op->eng->gmres(b.data(), tol, max_iter, restart);  // device-resident Krylov basis
        } catch (const ConvergenceFailure& e) {
            if (history)
                for (int i = 0; i < history_cap && i < int(e.history.size()); ++i) history[i] = e.history[i];
            if (iterations) *iterations = int(e.history.size());
            throw;
        }
        if (x) std::memcpy(x, r.x.data(), n * sizeof(cplx));
        if (history)
            for (int i = 0; i < history_cap && i < int(r.history.size()); ++i) history[i] = r.history[i];
        if (iterations) *iterations = r.iterations;
        if (converged) *converged = r.converged ? 1 : 0;
    });
}

namespace {
// incident_at (solver.cpp:25-35): plane wave along (cos t sin p, sin t sin p, cos p), or the
// sum of e^{ikr}/r over point sources when nsrc > 0
cplx incident_value(const Vec3& x, double k, const Vec3& dir, const double* src, int64_t nsrc) {
    if (nsrc <= 0) return std::polar(1.0, k * dot3(dir, x));
    cplx acc{};
    for (int64_t j = 0; j < nsrc; ++j) {
        const Vec3 y{src[3 * j], src[3 * j + 1], src[3 * j + 2]};
        const double r = len(x - y);
        if (r < 1e-12) throw InvalidArgument("incident_at: point source coincides with node");
        acc += std::polar(1.0 / r, k * r);
    }
    return acc;
}
Vec3 wave_direction(double theta, double phi) {
    return {std::cos(theta) * std::sin(phi), std::sin(theta) * std::sin(phi), std::cos(phi)};
}
}  // namespace

int ifgf_incident_trace(const ifgf_surface* s, double k, double theta, double phi, const double* src, int64_t nsrc,
                        double* out) {
    return guarded([&] {
        need(s, "surface");
        need(out, "out");
        if (nsrc > 0) need(src, "point sources");
        const Surface& S = *s->s;
        const Vec3 dir = wave_direction(theta, phi);
        for (std::size_t l = 0; l < S.size(); ++l) {
            const cplx u = incident_value(S.pos[l], k, dir, src, nsrc);
            out[2 * l] = u.real();
            out[2 * l + 1] = u.imag();
        }
    });
}

int ifgf_solve_incident(ifgf_operator* op, double theta, double phi, const double* src, int64_t nsrc, double tol,
                        int max_iter, int restart, double* density, double* history, int history_cap,
                        int* iterations, int* converged) {
    return guarded([&] {
        need(op, "operator");
        if (nsrc > 0) need(src, "point sources");
        const Surface& s = *op->plan->surf;
        const double k = op->plan->k;
        const Vec3 dir = wave_direction(theta, phi);
        std::vector<double> rhs(2 * s.size());  // -u^i on the nodes (solver.hpp:28-29)
        for (std::size_t l = 0; l < s.size(); ++l) {
            const cplx ui = incident_value(s.pos[l], k, dir, src, nsrc);
            rhs[2 * l] = -ui.real();
            rhs[2 * l + 1] = -ui.imag();
        }
        int it = 0, cv = 0;
        const int rc = ifgf_gmres_solve(op, rhs.data(), tol, max_iter, restart, density, history, history_cap, &it, &cv);
        if (iterations) *iterations = it;
        if (converged) *converged = cv;
        if (rc) throw EngineError(rc, g_error);
        if (!cv)
            throw ConvergenceFailure("solve: GMRES did not reach tolerance " + std::to_string(tol) + " in " +
                                         std::to_string(it) + " iterations",
                                     {});
    });
}

int ifgf_solve(ifgf_operator* op, double theta, double phi, double tol, int max_iter, int restart, double* density,
               double* history, int history_cap, int* iterations, int* converged) {
    return ifgf_solve_incident(op, theta, phi, nullptr, 0, tol, max_iter, restart, density, history, history_cap,
                               iterations, converged);
}

// ------------------------------------------------------------------ fields
int ifgf_far_field(const ifgf_surface* s, const double* density, double gamma, double k, int n_phi, int n_theta,
                   int device, double* dirs, double* values) {
    return guarded([&] {
        need(s, "surface");
        need(density, "density");
        need(values, "values");
        if (k <= 0) throw InvalidArgument("far_field: wavenumber must be positive");
        const Surface& S = *s->s;
        const auto phi = as_cplx(density, S.size());
        const FineQuad q = oversample_for_fields(S, phi.data(), k);
        const std::vector<Vec3> d = far_field_directions(n_phi, n_theta);
        gpu_far_field(q, d, k, gamma, device, reinterpret_cast<cplx*>(values));
        if (dirs)
            for (std::size_t i = 0; i < d.size(); ++i) {
                dirs[3 * i] = d[i].x;
                dirs[3 * i + 1] = d[i].y;
                dirs[3 * i + 2] = d[i].z;
            }
    });
}

int ifgf_near_field(const ifgf_surface* s, const double* density, double gamma, double k, double inc_theta,
                    double inc_phi, const double* src, int64_t nsrc, const double* points, int64_t npts,
                    double flag_distance, int device, double* scattered, double* total, uint8_t* flagged) {
    return guarded([&] {
        need(s, "surface");
        need(density, "density");
        if (npts > 0) {
            need(points, "points");
            need(scattered, "scattered");
            need(total, "total");
            need(flagged, "flagged");
        }
        if (nsrc > 0) need(src, "point sources");
        if (k <= 0) throw InvalidArgument("near_field: wavenumber must be positive");
        const Surface& S = *s->s;
        const auto phi = as_cplx(density, S.size());
        const FineQuad q = oversample_for_fields(S, phi.data(), k);
        std::vector<Vec3> pts(std::size_t(std::max<int64_t>(npts, 0)));
        for (std::size_t i = 0; i < pts.size(); ++i) pts[i] = {points[3 * i], points[3 * i + 1], points[3 * i + 2]};
        std::vector<double> dmin(pts.size()), gauss(pts.size());
        cplx* sc = reinterpret_cast<cplx*>(scattered);
        gpu_near_field(q, pts, k, gamma, device, sc, dmin.data(), gauss.data());
        // incident field (solver.cpp:25-35)
        const Vec3 dir{std::cos(inc_theta) * std::sin(inc_phi), std::sin(inc_theta) * std::sin(inc_phi),
                       std::cos(inc_phi)};
        for (std::size_t i = 0; i < pts.size(); ++i) {
            cplx inc{};
            if (nsrc > 0) {
                for (int64_t j = 0; j < nsrc; ++j) {
                    const Vec3 y{src[3 * j], src[3 * j + 1], src[3 * j + 2]};
                    const double r = len(pts[i] - y);
                    if (r < 1e-12) throw InvalidArgument("incident_at: point source coincides with node");
                    inc += std::polar(1.0 / r, k * r);
                }
            } else {
                inc = std::polar(1.0, k * dot3(dir, pts[i]));
            }
            const cplx t = sc[i] + inc;
            total[2 * i] = t.real();
            total[2 * i + 1] = t.imag();
            flagged[i] = (dmin[i] <= flag_distance || gauss[i] < -0.5) ? 1 : 0;
        }
    });
}

int ifgf_rp_regular_apply(const ifgf_surface* s, const double* density, const double* targets, int64_t ntargets,
                          double k, int device, double* S, double* D) {
    return guarded([&] {
        need(s, "surface");
        need(density, "density");
        if (ntargets > 0) {
            need(targets, "targets");
            need(S, "out_single");
            need(D, "out_dbl");
        }
        const Surface& sf = *s->s;
        // the nodal Fejer rule itself (rp.cpp:453-479): nodes, normals, J w, density
        FineQuad q;
        const auto phi = as_cplx(density, sf.size());
        for (std::size_t m = 0; m < sf.size(); ++m) {
            q.x.push_back(sf.pos[m].x);
            q.y.push_back(sf.pos[m].y);
            q.z.push_back(sf.pos[m].z);
            q.nx.push_back(sf.nrm[m].x);
            q.ny.push_back(sf.nrm[m].y);
            q.nz.push_back(sf.nrm[m].z);
            q.jw.push_back(sf.jac[m] * sf.wt[m]);
            q.density.push_back(phi[m]);
        }
        const std::size_t n = std::size_t(std::max<int64_t>(ntargets, 0));
        std::vector<Vec3> pts(n);
        for (std::size_t i = 0; i < n; ++i) pts[i] = {targets[3 * i], targets[3 * i + 1], targets[3 * i + 2]};
        std::vector<cplx> s_out(n), d_out(n);
        std::vector<double> dmin(n), gauss(n);
        gpu_layer_potentials_at(q, pts, k, device, s_out.data(), d_out.data(), dmin.data(), gauss.data());
        for (std::size_t i = 0; i < n; ++i)
            if (dmin[i] < 1e-14) throw InvalidArgument("rp_regular_apply: target coincides with a node");
        for (std::size_t i = 0; i < n; ++i) {  // accumulated into the outputs, like the reference
            S[2 * i] += s_out[i].real();
            S[2 * i + 1] += s_out[i].imag();
            D[2 * i] += d_out[i].real();
            D[2 * i + 1] += d_out[i].imag();
        }
    });
}

int ifgf_closest_point(const ifgf_surface* s, int q, const double* x, double u0, double v0, double* out) {
    return guarded([&] {
        need(s, "surface");
        need(x, "x");
        need(out, "out");
        if (q < 0 || q >= int(s->s->patches.size())) throw InvalidArgument("closest_point: patch index out of range");
        const ClosestPoint c = closest_point_on(s->s->patches[q], {x[0], x[1], x[2]}, u0, v0);
        out[0] = c.u;
        out[1] = c.v;
        out[2] = c.dist;
    });
}

double ifgf_graded(int which, double alpha, double tau, int d) {
    try {
        switch (which) {
            case 0: return grade_w(tau, d);
            case 1: return grade_w_deriv(tau, d);
            case 2: return grade_xi(alpha, tau, d);
            case 3: return grade_xi_deriv(alpha, tau, d);
            default: throw InvalidArgument("graded: which must be 0..3");
        }
    } catch (const std::exception& e) {
        g_error = e.what();
        return std::numeric_limits<double>::quiet_NaN();
    }
}

int ifgf_mie_far_field(double radius, double k, const double* direction, const double* dirs, int64_t n,
                       int extra_terms, double* values) {
    return guarded([&] {
        need(direction, "direction");
        if (n > 0) {
            need(dirs, "directions");
            need(values, "values");
        }
        std::vector<Vec3> d(std::size_t(std::max<int64_t>(n, 0)));
        for (std::size_t i = 0; i < d.size(); ++i) d[i] = {dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]};
        const auto v = mie_far_field(radius, k, {direction[0], direction[1], direction[2]}, d, extra_terms);
        if (!v.empty()) std::memcpy(values, v.data(), v.size() * sizeof(cplx));
    });
}

int ifgf_eps_metric(const double* ref, const double* apx, int64_t n, double* eps, int* skipped) {
    return guarded([&] {
        need(eps, "eps");
        if (n > 0) {
            need(ref, "reference");
            need(apx, "approximation");
        }
        *eps = eps_metric(reinterpret_cast<const cplx*>(ref), reinterpret_cast<const cplx*>(apx),
                          std::size_t(std::max<int64_t>(n, 0)), skipped);
    });
}

}  // extern "C"
