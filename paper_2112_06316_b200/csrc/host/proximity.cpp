#include "proximity.hpp"

#include "closest_point.hpp"

#include <algorithm>
#include <limits>

namespace ifgfb200 {

namespace {

std::uint64_t fnv(const void* data, std::size_t n, std::uint64_t h) {
    const auto* b = static_cast<const unsigned char*>(data);
    for (std::size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 1099511628211ULL;
    }
    return h;
}

}  // namespace

ClosestPoint closest_point_on(const Patch& p, const Vec3& x, double u0, double v0) {
    if (p.du > cp::kMaxExtent || p.dv > cp::kMaxExtent) throw InvalidArgument("closest point: series extent above 64");
    const cp::PatchSeries ps{p.pos_c[0].data(), p.pos_c[1].data(), p.pos_c[2].data(), p.du, p.dv};
    ClosestPoint out;
    cp::solve(ps, x.x, x.y, x.z, u0, v0, out.u, out.v, out.dist);
    return out;
}

double grade_w(double tau, int d) {
    if (tau < -1e-12 || tau > 2.0 * kPi + 1e-12) throw InvalidArgument("cov_w: tau outside [0, 2pi]");
    tau = std::clamp(tau, 0.0, 2.0 * kPi);
    auto nu = [&](double q) {
        const double a = (kPi - q) / kPi;
        const double b = (q - kPi) / kPi;
        return (1.0 / d - 0.5) * a * a * a + b / d + 0.5;
    };
    const double vd = std::pow(nu(tau), d);
    const double wd = std::pow(nu(2.0 * kPi - tau), d);
    return 2.0 * kPi * vd / (vd + wd);
}

double grade_w_deriv(double tau, int d) {
    tau = std::clamp(tau, 0.0, 2.0 * kPi);
    auto nu = [&](double q) {
        const double a = (kPi - q) / kPi;
        const double b = (q - kPi) / kPi;
        return (1.0 / d - 0.5) * a * a * a + b / d + 0.5;
    };
    auto nu_d = [&](double q) {
        const double a = (kPi - q) / kPi;
        return -3.0 * (1.0 / d - 0.5) * a * a / kPi + 1.0 / (d * kPi);
    };
    const double n1 = nu(tau), n2 = nu(2.0 * kPi - tau);
    const double p1 = std::pow(n1, d - 1), p2 = std::pow(n2, d - 1);
    const double f = p1 * n1, g = p2 * n2;
    const double fp = d * p1 * nu_d(tau);
    const double gp = -d * p2 * nu_d(2.0 * kPi - tau);
    return 2.0 * kPi * (fp * g - f * gp) / ((f + g) * (f + g));
}

double grade_xi(double alpha, double tau, int d) {
    if (tau < -1.0 - 1e-12 || tau > 1.0 + 1e-12) throw InvalidArgument("cov_xi: tau outside [-1, 1]");
    tau = std::clamp(tau, -1.0, 1.0);
    if (alpha >= 1.0) return 1.0 - (2.0 / kPi) * grade_w(kPi * std::abs(tau - 1.0) / 2.0, d);
    if (alpha <= -1.0) return -1.0 + (2.0 / kPi) * grade_w(kPi * std::abs(tau + 1.0) / 2.0, d);
    const double sg = tau > 0 ? 1.0 : (tau < 0 ? -1.0 : 0.0);
    return alpha + (sg - alpha) / kPi * grade_w(kPi * std::abs(tau), d);
}

double grade_xi_deriv(double alpha, double tau, int d) {
    tau = std::clamp(tau, -1.0, 1.0);
    if (alpha >= 1.0) return grade_w_deriv(kPi * (1.0 - tau) / 2.0, d);
    if (alpha <= -1.0) return grade_w_deriv(kPi * (tau + 1.0) / 2.0, d);
    if (tau == 0.0) return 0.0;
    const double sg = tau > 0 ? 1.0 : -1.0;
    return (sg - alpha) * sg * grade_w_deriv(kPi * std::abs(tau), d);
}

PairList classify_pairs(const Surface& s, const BoxTree& t, const BoxRelations& rel,
                        const RpParams& cfg, int workers, const ClosestPointBatch* batch,
                        const std::vector<std::uint8_t>* owned) {
    if (cfg.n_beta < 2 || cfg.cov_d < 2)
        throw InvalidArgument("classify_targets: n_beta >= 2 and cov_d >= 2 required");
    const std::size_t n = s.size();
    const std::size_t nq = s.patches.size();
    PairList out;
    out.cfg = cfg;
    const std::vector<double> spacing = s.spacing();
    out.delta.resize(nq);
    for (std::size_t q = 0; q < nq; ++q)
        out.delta[q] = cfg.delta_abs > 0 ? cfg.delta_abs : cfg.delta_rel * spacing[q];

    const int D = t.depth;
    const BoxLevel& leaves = t.level[D - 1];
    const Adjacency& nbr = rel.nbr[D - 1];
    std::vector<std::vector<std::int32_t>> box_patches(leaves.size());
    for (std::size_t b = 0; b < leaves.size(); ++b) {
        auto& v = box_patches[b];
        for (std::uint32_t i = leaves.begin[b]; i < leaves.end[b]; ++i) v.push_back(s.patch_of[t.perm[i]]);
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
    }

    struct Found {
        std::int32_t q;
        double u, v;
        std::vector<std::uint32_t> far;
    };
    std::vector<std::vector<Found>> per(n);
    const int w = worker_count(workers);
    // (1) per target: candidate patches of the neighbour leaves; the own patch is a pair at
    // the node's parameters, others need a closest-point search unless the nearest node is
    // already beyond delta + spacing
    std::vector<std::vector<ClosestPointRequest>> req(n);
#pragma omp parallel for schedule(dynamic, 64) num_threads(w)
    for (std::int64_t l = 0; l < std::int64_t(n); ++l) {
        if (owned && !(*owned)[l]) continue;  // another rank's target
        const std::int32_t tb = t.leaf_of[l];
        const auto nb0 = nbr.idx.begin() + nbr.ptr[tb], nb1 = nbr.idx.begin() + nbr.ptr[tb + 1];
        std::vector<std::int32_t> cand;
        for (auto it = nb0; it != nb1; ++it)
            cand.insert(cand.end(), box_patches[*it].begin(), box_patches[*it].end());
        std::sort(cand.begin(), cand.end());
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
        const Vec3 x = s.pos[l];
        for (std::int32_t q : cand) {
            if (q == s.patch_of[l]) {
                req[l].push_back({std::uint32_t(l), q, s.pu[l], s.pv[l], true});
                continue;
            }
            double best = std::numeric_limits<double>::max();
            std::size_t arg = s.patch_start[q];
            for (std::size_t m = s.patch_start[q]; m < s.patch_start[q + 1]; ++m) {
                const double d2 = len2(s.pos[m] - x);
                if (d2 < best) {
                    best = d2;
                    arg = m;
                }
            }
            if (std::sqrt(best) > out.delta[q] + spacing[q]) continue;
            req[l].push_back({std::uint32_t(l), q, s.pu[arg], s.pv[arg], false});
        }
    }
    // (2) the closest-point searches, batched (GPU when given, else host threads)
    std::vector<ClosestPointRequest> flat;
    std::vector<std::size_t> off(n + 1, 0);
    for (std::size_t l = 0; l < n; ++l) off[l + 1] = off[l] + req[l].size();
    flat.reserve(off[n]);
    for (std::size_t l = 0; l < n; ++l) {
        flat.insert(flat.end(), req[l].begin(), req[l].end());
        req[l].clear();
        req[l].shrink_to_fit();
    }
    std::vector<ClosestPoint> res(flat.size());
    if (batch) {
        (*batch)(s, flat, res);
    } else {
#pragma omp parallel for schedule(dynamic, 16) num_threads(w)
        for (std::int64_t i = 0; i < std::int64_t(flat.size()); ++i)
            if (!flat[i].own)
                res[i] = closest_point_on(s.patches[flat[i].q], s.pos[flat[i].target], flat[i].u0, flat[i].v0);
    }
    // (3) pairs within delta, with the far-node correction lists
#pragma omp parallel for schedule(dynamic, 64) num_threads(w)
    for (std::int64_t l = 0; l < std::int64_t(n); ++l) {
        const std::int32_t tb = t.leaf_of[l];
        const auto nb0 = nbr.idx.begin() + nbr.ptr[tb], nb1 = nbr.idx.begin() + nbr.ptr[tb + 1];
        for (std::size_t i = off[l]; i < off[l + 1]; ++i) {
            const ClosestPointRequest& r = flat[i];
            Found f;
            f.q = r.q;
            if (r.own) {
                f.u = r.u0;
                f.v = r.v0;
            } else {
                if (res[i].dist > out.delta[r.q]) continue;
                f.u = res[i].u;
                f.v = res[i].v;
            }
            for (std::size_t m = s.patch_start[r.q]; m < s.patch_start[r.q + 1]; ++m)
                if (!std::binary_search(nb0, nb1, t.leaf_of[m])) f.far.push_back(std::uint32_t(m));
            per[l].push_back(std::move(f));
        }
    }

    out.target_pair_begin.assign(n + 1, 0);
    for (std::size_t l = 0; l < n; ++l) {
        out.target_pair_begin[l] = std::uint32_t(out.target.size());
        for (Found& f : per[l]) {
            out.target.push_back(std::uint32_t(l));
            out.patch.push_back(f.q);
            out.ubar.push_back(f.u);
            out.vbar.push_back(f.v);
            if (out.far_nodes.size() + f.far.size() > std::size_t(0xffffffffu) ||
                out.target.size() >= std::size_t(0xffffffffu))
                throw InternalError("classify_targets: more than 2^32 far-node entries or pairs (32-bit offsets)");
            out.far_begin.push_back(std::uint32_t(out.far_nodes.size()));
            out.far_nodes.insert(out.far_nodes.end(), f.far.begin(), f.far.end());
            out.far_end.push_back(std::uint32_t(out.far_nodes.size()));
        }
        per[l].clear();
        per[l].shrink_to_fit();
    }
    out.target_pair_begin[n] = std::uint32_t(out.target.size());
    return out;
}

void graded_rules(const PairList& pl, std::size_t p0, std::size_t p1, const std::vector<double>& rx,
                  const std::vector<double>& rw, double* u, double* wu, double* v, double* wv,
                  int workers) {
    const int nb = int(rx.size());
    const int d = pl.cfg.cov_d;
    const int w = worker_count(workers);
#pragma omp parallel for schedule(static) num_threads(w)
    for (std::int64_t p = std::int64_t(p0); p < std::int64_t(p1); ++p) {
        const std::size_t o = std::size_t(p - std::int64_t(p0)) * nb;
        for (int i = 0; i < nb; ++i) {
            u[o + i] = grade_xi(pl.ubar[p], rx[i], d);
            wu[o + i] = grade_xi_deriv(pl.ubar[p], rx[i], d) * rw[i];
            v[o + i] = grade_xi(pl.vbar[p], rx[i], d);
            wv[o + i] = grade_xi_deriv(pl.vbar[p], rx[i], d) * rw[i];
        }
    }
}

void graded_rules(const PairList& pl, const std::uint32_t* idx, std::size_t count, const std::vector<double>& rx,
                  const std::vector<double>& rw, double* u, double* wu, double* v, double* wv, int workers) {
    const int nb = int(rx.size());
    const int d = pl.cfg.cov_d;
    const int w = worker_count(workers);
#pragma omp parallel for schedule(static) num_threads(w)
    for (std::int64_t i = 0; i < std::int64_t(count); ++i) {
        const std::size_t p = idx[i], o = std::size_t(i) * nb;
        for (int j = 0; j < nb; ++j) {
            u[o + j] = grade_xi(pl.ubar[p], rx[j], d);
            wu[o + j] = grade_xi_deriv(pl.ubar[p], rx[j], d) * rw[j];
            v[o + j] = grade_xi(pl.vbar[p], rx[j], d);
            wv[o + j] = grade_xi_deriv(pl.vbar[p], rx[j], d) * rw[j];
        }
    }
}

std::uint64_t beta_key(const Surface& s, const PairList& pl, double k) {
    std::uint64_t h = 14695981039346656037ULL;
    h = fnv(&k, sizeof k, h);
    h = fnv(&pl.cfg.n_beta, sizeof pl.cfg.n_beta, h);
    h = fnv(&pl.cfg.cov_d, sizeof pl.cfg.cov_d, h);
    for (double d : pl.delta) h = fnv(&d, sizeof d, h);
    for (const Patch& p : s.patches)
        for (int c = 0; c < 3; ++c) h = fnv(p.pos_c[c].data(), p.pos_c[c].size() * sizeof(double), h);
    for (std::size_t i = 0; i < pl.size(); ++i) {
        h = fnv(&pl.target[i], sizeof(std::uint32_t), h);
        h = fnv(&pl.patch[i], sizeof(std::int32_t), h);
        h = fnv(&pl.ubar[i], sizeof(double), h);
        h = fnv(&pl.vbar[i], sizeof(double), h);
    }
    return h;
}

}  // namespace ifgfb200
