#include "coneplan.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <atomic>
#include <exception>
#include <mutex>
#include <sstream>

#include "chebyshev.hpp"

namespace ifgfb200 {

namespace {

constexpr double kTwoPiC = 2.0 * kPi;
constexpr int kMaxOrder = 12;

struct Cone {
    double s, th, ph;
};

// kernels.cpp:34-48
inline Cone to_cone(const Vec3& x, const Vec3& c, double h) {
    const Vec3 v = x - c;
    const double r = len(v);
    if (r < 1e-300) throw InvalidArgument("cone coordinates: point at box center");
    Cone o;
    o.s = h / r;
    double ct = v.z / r;
    ct = std::min(1.0, std::max(-1.0, ct));
    o.th = std::acos(ct);
    double ph = std::atan2(v.y, v.x);
    if (ph < 0.0) ph += kTwoPiC;
    if (ph >= kTwoPiC) ph = 0.0;
    o.ph = ph;
    return o;
}

// kernels.cpp:27-32
inline Vec3 from_cone(double s, double th, double ph, const Vec3& c, double h) {
    if (s <= 0.0) throw InvalidArgument("cone point: s must be positive");
    const double r = h / s;
    const double st = std::sin(th), ct = std::cos(th);
    return c + Vec3{r * st * std::cos(ph), r * st * std::sin(ph), r * ct};
}

// LevelCones::segment_of (ifgf.cpp:161-176), returned as the gamma index of ifgf.hpp:34-36
inline int segment_gamma(const ConeLevel& L, const Cone& c) {
    if (c.s > kConeEtaC + 1e-12)
        throw InternalError("cone segment query with s > sqrt(3)/3: s=" + std::to_string(c.s));
    int g1 = int(std::floor(c.s / L.ds)) + 1;
    if (g1 > L.ns) g1 = L.ns;
    if (g1 < 1) g1 = 1;
    int g2, g3;
    if (c.th >= kPi) {
        g2 = L.nc;
        g3 = 2 * L.nc;
    } else {
        g2 = std::min(L.nc, int(std::floor(c.th / L.dth)) + 1);
        if (g2 < 1) g2 = 1;
        g3 = std::min(2 * L.nc, int(std::floor(c.ph / L.dph)) + 1);
        if (g3 < 1) g3 = 1;
    }
    return (g1 - 1) + L.ns * ((g2 - 1) + L.nc * (g3 - 1));
}

ConeLevel make_level(int d, double side, double lambda, const ConeParams& p) {
    ConeLevel L;
    L.d = d;
    const int m = cone_doublings(side, lambda);
    L.ns = p.n_s0 << m;
    L.nc = p.n_c0 << m;
    L.ps = p.ps;
    L.pang = p.pang;
    L.ds = kConeEtaC / L.ns;
    L.dth = kPi / L.nc;
    L.dph = kPi / L.nc;
    const auto xs = cheb::gauss_nodes(p.ps);
    const auto xa = cheb::gauss_nodes(p.pang);
    auto table = [](int cells, double width, const std::vector<double>& x) {
        std::vector<double> t(std::size_t(cells) * x.size());
        for (int g = 0; g < cells; ++g)
            for (std::size_t i = 0; i < x.size(); ++i)
                t[std::size_t(g) * x.size() + i] = g * width + (x[i] + 1.0) * 0.5 * width;
        return t;
    };
    L.s_nodes = table(L.ns, L.ds, xs);
    L.th_nodes = table(L.nc, L.dth, xa);
    L.ph_nodes = table(2 * L.nc, L.dph, xa);
    return L;
}

// Runs body(i) for i in [0, n) on the OpenMP team; the first exception is rethrown after
// the region (the reference's ParallelErrors, common.hpp:71-92).
template <class F>
void parallel_for(std::int64_t n, int workers, F&& body) {
    std::exception_ptr err;
    std::atomic<bool> failed{false};
    std::mutex mu;
#pragma omp parallel for schedule(dynamic, 4) num_threads(workers)
    for (std::int64_t i = 0; i < n; ++i) {
        if (failed.load(std::memory_order_relaxed)) continue;
        try {
            body(i);
        } catch (...) {
            std::lock_guard<std::mutex> g(mu);
            if (!failed) {
                err = std::current_exception();
                failed = true;
            }
        }
    }
    if (err) std::rethrow_exception(err);
}

inline void mark(std::vector<std::uint8_t>& m, std::size_t at) {
    __atomic_store_n(&m[at], std::uint8_t(1), __ATOMIC_RELAXED);
}

// per parent segment: stable order of its evaluations by child segment, and the groups
void group_parent_evaluations(ConeLevel& L, std::size_t pseg, int w, int P) {
    L.pev_perm.assign(L.pev_seg.size(), 0);
    std::vector<std::int32_t> ngroups(pseg + 1, 0);
    parallel_for(std::int64_t(pseg), w, [&](std::int64_t so) {
        const std::int64_t b = L.pev_begin[so], n = L.pev_begin[so + 1] - b;
        if (n > 65535) throw InternalError("cone plan: too many evaluations per parent segment");
        std::uint16_t* perm = L.pev_perm.data() + b;
        const std::int32_t* seg = L.pev_seg.data() + b;
        // stable bucketing by child segment: few distinct values per parent segment
        constexpr int kMaxU = 64;
        std::int32_t val[kMaxU];
        int cnt[kMaxU], u = 0;
        bool many = false;
        for (std::int64_t i = 0; i < n && !many; ++i) {
            int j = 0;
            while (j < u && val[j] != seg[i]) ++j;
            if (j == u) {
                if (u == kMaxU) {
                    many = true;
                    break;
                }
                val[u] = seg[i];
                cnt[u++] = 0;
            }
            ++cnt[j];
        }
        if (many) {
            for (std::int64_t i = 0; i < n; ++i) perm[i] = std::uint16_t(i);
            std::stable_sort(perm, perm + n, [&](std::uint16_t x, std::uint16_t y) { return seg[x] < seg[y]; });
            int g = 0;
            for (std::int64_t i = 0; i < n; ++i)
                if (i == 0 || seg[perm[i]] != seg[perm[i - 1]]) ++g;
            ngroups[so + 1] = g;
            return;
        }
        int order[kMaxU], start[kMaxU];
        for (int j = 0; j < u; ++j) order[j] = j;
        std::sort(order, order + u, [&](int x, int y) { return val[x] < val[y]; });
        int acc = 0;
        for (int r = 0; r < u; ++r) {
            start[order[r]] = acc;
            acc += cnt[order[r]];
        }
        for (std::int64_t i = 0; i < n; ++i) {
            int j = 0;
            while (val[j] != seg[i]) ++j;
            perm[start[j]++] = std::uint16_t(i);
        }
        ngroups[so + 1] = u;
    });
    L.pgrp_begin.assign(pseg + 1, 0);
    for (std::size_t so = 0; so < pseg; ++so) L.pgrp_begin[so + 1] = L.pgrp_begin[so] + ngroups[so + 1];
    const std::size_t ng = std::size_t(L.pgrp_begin[pseg]);
    L.pgrp_seg.assign(ng, 0);
    L.pgrp_start.assign(ng, 0);
    L.pgrp_count.assign(ng, 0);
    parallel_for(std::int64_t(pseg), w, [&](std::int64_t so) {
        const std::int64_t b = L.pev_begin[so], n = L.pev_begin[so + 1] - b;
        const std::uint16_t* perm = L.pev_perm.data() + b;
        const std::int32_t* seg = L.pev_seg.data() + b;
        std::int32_t g = L.pgrp_begin[so] - 1;
        for (std::int64_t i = 0; i < n; ++i) {
            if (i == 0 || seg[perm[i]] != seg[perm[i - 1]]) {
                ++g;
                L.pgrp_seg[g] = seg[perm[i]];
                L.pgrp_start[g] = std::uint16_t(i);
            }
            ++L.pgrp_count[g];
        }
    });
    // pack each local index e = node * nch + c as node | c << 8 for the device (P <= 255)
    if (P <= 255)
        parallel_for(std::int64_t(pseg), w, [&](std::int64_t so) {
            const std::int64_t b = L.pev_begin[so], n = L.pev_begin[so + 1] - b;
            const int nch = int(n / P);
            std::uint16_t* perm = L.pev_perm.data() + b;
            for (std::int64_t i = 0; i < n; ++i)
                perm[i] = std::uint16_t((perm[i] / nch) | ((perm[i] % nch) << 8));
        });
}

}  // namespace

int cone_doublings(double side, double lambda) {
    const double ratio = side / (0.3 * lambda);
    return std::max(0, int(std::floor(std::log2(ratio * (1.0 + 1e-9)))) + 1);
}

std::vector<int> dl_pipes(const BoxTree& t, int level, DlStrategy s) {
    switch (s) {
        case DlStrategy::W4:
            return {W4};
        case DlStrategy::W2W3:
            return {W2, W3};
        case DlStrategy::Hybrid: {
            const double lambda = 2.0 * kPi / t.k;
            if (t.side(level) / lambda < 0.5 - 1e-12) return {W2, W3};
            return {W4};
        }
    }
    return {W4};
}

ConePlanHost build_cone_plan(const BoxTree& t, const BoxRelations& rel,
                             const std::vector<Vec3>& pts, const ConeParams& p, int workers,
                             const ConeDecider* decider, const std::vector<std::vector<std::uint8_t>>* active) {
    if (p.ps < 1 || p.ps > kMaxOrder || p.pang < 1 || p.pang > kMaxOrder)
        throw InvalidArgument("plan_cones: interpolation orders must lie in [1,12]");
    if (p.n_s0 < 1 || p.n_c0 < 1) throw InvalidArgument("plan_cones: interval counts must be positive");
    const int w = worker_count(workers);
    ConePlanHost plan;
    plan.params = p;
    plan.k = t.k;
    const double lambda = 2.0 * kPi / t.k;
    const int D = t.depth;
    plan.level.resize(D);
    plan.child_ptr.resize(D);
    plan.child_idx.resize(D);
    for (int d = 1; d <= D; ++d) {
        const BoxLevel& B = t.level[d - 1];
        auto& cp = plan.child_ptr[d - 1];
        auto& ci = plan.child_idx[d - 1];
        cp.assign(B.size() + 1, 0);
        for (std::size_t b = 0; b < B.size(); ++b) {
            for (std::int32_t ch : B.child[b])
                if (ch >= 0 && (!active || d >= D || (*active)[d][ch])) ci.push_back(ch);
            cp[b + 1] = std::int32_t(ci.size());
        }
    }

    const bool timing = std::getenv("IFGF_PLAN_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto secs = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
    for (int d = 3; d <= D; ++d) {
        const auto T0 = now();
        ConeLevel& L = plan.level[d - 1];
        L = make_level(d, t.side(d), lambda, p);
        const BoxLevel& B = t.level[d - 1];
        const std::size_t nb = B.size();
        const std::size_t spb = std::size_t(L.segs_per_box());
        const double h = t.half_diag(d);
        std::vector<Vec3> ctr(nb);
        for (std::size_t b = 0; b < nb; ++b) ctr[b] = t.center(d, b);
        std::vector<std::uint8_t> marks(nb * spb, 0);

        // (1) cousin target points, evaluated in the frame of each cousin source box
        // cousin pairs evaluated by this plan (all, or those whose source box is active)
        if (!active) {
            L.cz = rel.cousin[d - 1];
        } else {
            const Adjacency& full = rel.cousin[d - 1];
            const auto& act = (*active)[d - 1];
            L.cz.ptr.assign(nb + 1, 0);
            L.cz.idx.clear();
            for (std::size_t b = 0; b < nb; ++b) {
                for (std::int32_t j = full.ptr[b]; j < full.ptr[b + 1]; ++j)
                    if (act[full.idx[j]]) L.cz.idx.push_back(full.idx[j]);
                L.cz.ptr[b + 1] = std::int32_t(L.cz.idx.size());
            }
        }
        const Adjacency& cz = L.cz;
        L.cev_begin.assign(nb + 1, 0);
        for (std::size_t b = 0; b < nb; ++b)
            L.cev_begin[b + 1] = L.cev_begin[b] + std::int64_t(cz.count(b)) * (B.end[b] - B.begin[b]);
        L.cev_seg.assign(std::size_t(L.cev_begin[nb]), 0);
        auto cev_decide = [&](std::int64_t tb, std::int64_t off) {  // evaluation off of box tb
            const std::int64_t n_t = B.end[tb] - B.begin[tb];
            const std::int32_t sb = cz.idx[cz.ptr[tb] + off / n_t];
            const int g = segment_gamma(L, to_cone(pts[B.begin[tb] + off % n_t], ctr[sb], h));
            L.cev_seg[L.cev_begin[tb] + off] = g;
            mark(marks, std::size_t(sb) * spb + g);
        };
        // (2) interpolation nodes of every relevant parent segment, in each child's frame
        const ConeLevel* PLp = d > 3 ? &plan.level[d - 2] : nullptr;
        const double ph = d > 3 ? t.half_diag(d - 1) : 0.0;
        const std::vector<std::int32_t>* cptr = d > 3 ? &plan.child_ptr[d - 2] : nullptr;
        const std::vector<std::int32_t>* cidx = d > 3 ? &plan.child_idx[d - 2] : nullptr;
        if (PLp) {
            const int P = PLp->nodes_per_seg();
            const std::size_t pseg = PLp->nseg();
            L.pev_begin.assign(pseg + 1, 0);
            for (std::size_t so = 0; so < pseg; ++so) {
                const std::int32_t pb = PLp->seg_box[so];
                L.pev_begin[so + 1] = L.pev_begin[so] + std::int64_t(P) * ((*cptr)[pb + 1] - (*cptr)[pb]);
            }
            L.pev_seg.assign(std::size_t(L.pev_begin[pseg]), 0);
        }
        auto pev_decide = [&](std::int64_t so, std::int64_t off) {  // evaluation off of parent segment so
            const ConeLevel& PL = *PLp;
            const std::int32_t pb = PL.seg_box[so];
            const int gam = PL.seg_gamma[so];
            const int g1 = gam % PL.ns, g2 = (gam / PL.ns) % PL.nc, g3 = gam / PL.ns / PL.nc;
            const int nch = (*cptr)[pb + 1] - (*cptr)[pb];
            const int node = int(off / nch), c = int(off % nch);
            const int is = node % PL.ps, it = (node / PL.ps) % PL.pang, ip = node / (PL.ps * PL.pang);
            const Vec3 x = from_cone(PL.s_nodes[std::size_t(g1) * PL.ps + is], PL.th_nodes[std::size_t(g2) * PL.pang + it],
                                     PL.ph_nodes[std::size_t(g3) * PL.pang + ip], t.center(d - 1, std::size_t(pb)), ph);
            const std::int32_t ch = (*cidx)[(*cptr)[pb] + c];
            const int g = segment_gamma(L, to_cone(x, ctr[ch], h));
            L.pev_seg[L.pev_begin[so] + off] = g;
            mark(marks, std::size_t(ch) * spb + g);
        };
        if (decider) {
            // batched decisions; the host redoes the ones the decider could not guarantee
            ConeDecisionJob job;
            job.L = &L;
            job.h = h;
            job.pts = &pts;
            job.ctr = &ctr;
            job.B = &B;
            job.cz = &cz;
            std::vector<Vec3> pctr;
            if (PLp) {
                job.PL = PLp;
                job.ph = ph;
                const BoxLevel& PB = t.level[d - 2];
                pctr.resize(PB.size());
                for (std::size_t b = 0; b < PB.size(); ++b) pctr[b] = t.center(d - 1, b);
                job.pctr = &pctr;
                job.cptr = cptr;
                job.cidx = cidx;
                for (double a : PLp->th_nodes) {
                    job.th_sin.push_back(std::sin(a));
                    job.th_cos.push_back(std::cos(a));
                }
                for (double a : PLp->ph_nodes) {
                    job.ph_sin.push_back(std::sin(a));
                    job.ph_cos.push_back(std::cos(a));
                }
            }
            std::vector<std::int64_t> fl_cev, fl_pev;
            (*decider)(job, L, marks, fl_cev, fl_pev);
            parallel_for(std::int64_t(fl_cev.size()), w, [&](std::int64_t i) {
                const std::int64_t at = fl_cev[i];
                const std::int64_t tb =
                    std::upper_bound(L.cev_begin.begin(), L.cev_begin.end(), at) - L.cev_begin.begin() - 1;
                cev_decide(tb, at - L.cev_begin[tb]);
            });
            parallel_for(std::int64_t(fl_pev.size()), w, [&](std::int64_t i) {
                const std::int64_t at = fl_pev[i];
                const std::int64_t so =
                    std::upper_bound(L.pev_begin.begin(), L.pev_begin.end(), at) - L.pev_begin.begin() - 1;
                pev_decide(so, at - L.pev_begin[so]);
            });
        } else {
            parallel_for(std::int64_t(nb), w, [&](std::int64_t tb) {
                const std::int64_t n = L.cev_begin[tb + 1] - L.cev_begin[tb];
                for (std::int64_t off = 0; off < n; ++off) cev_decide(tb, off);
            });
            if (PLp)
                parallel_for(std::int64_t(PLp->nseg()), w, [&](std::int64_t so) {  // x once per node
                    const ConeLevel& PL = *PLp;
                    const std::int32_t pb = PL.seg_box[so];
                    const int gam = PL.seg_gamma[so];
                    const int g1 = gam % PL.ns, g2 = (gam / PL.ns) % PL.nc, g3 = gam / PL.ns / PL.nc;
                    const Vec3 pc = t.center(d - 1, std::size_t(pb));
                    const int nch = (*cptr)[pb + 1] - (*cptr)[pb];
                    for (int ip = 0; ip < PL.pang; ++ip)
                        for (int it = 0; it < PL.pang; ++it)
                            for (int is = 0; is < PL.ps; ++is) {
                                const Vec3 x = from_cone(PL.s_nodes[std::size_t(g1) * PL.ps + is],
                                                         PL.th_nodes[std::size_t(g2) * PL.pang + it],
                                                         PL.ph_nodes[std::size_t(g3) * PL.pang + ip], pc, ph);
                                const int node = is + PL.ps * (it + PL.pang * ip);
                                std::int64_t at = L.pev_begin[so] + std::int64_t(node) * nch;
                                for (int c = 0; c < nch; ++c) {
                                    const std::int32_t ch = (*cidx)[(*cptr)[pb] + c];
                                    const int g = segment_gamma(L, to_cone(x, ctr[ch], h));
                                    L.pev_seg[at++] = g;
                                    mark(marks, std::size_t(ch) * spb + g);
                                }
                            }
                });
        }

        const auto T1 = now();
        // relevant segments in (box, gamma) order
        L.box_seg_begin.assign(nb + 1, 0);
        for (std::size_t b = 0; b < nb; ++b) {
            L.box_seg_begin[b] = std::int32_t(L.seg_box.size());
            const std::uint8_t* mb = marks.data() + b * spb;
            for (std::size_t g = 0; g < spb; ++g)
                if (mb[g]) {
                    L.seg_box.push_back(std::int32_t(b));
                    L.seg_gamma.push_back(std::int32_t(g));
                }
        }
        L.box_seg_begin[nb] = std::int32_t(L.seg_box.size());
        // gamma -> ordinal of (box, gamma) among the relevant segments: segments are in (box,
        // gamma) order, so the ordinal is the exclusive prefix count of the marks (a table
        // lookup; binary search per box when the candidate grid is too large for a table)
        std::vector<std::int32_t> ordtab;
        if (nb * spb <= (std::size_t(1) << 29)) {
            ordtab.assign(nb * spb, -1);
            std::int32_t o = 0;
            for (std::size_t i = 0; i < nb * spb; ++i)
                if (marks[i]) ordtab[i] = o++;
        }
        marks.clear();
        marks.shrink_to_fit();
        auto ordinal = [&](std::int32_t box, int g) {
            if (!ordtab.empty()) {
                const std::int32_t o = ordtab[std::size_t(box) * spb + std::size_t(g)];
                if (o < 0) throw InternalError("cone plan: unmarked segment");
                return o;
            }
            const auto b0 = L.seg_gamma.begin() + L.box_seg_begin[box];
            const auto b1 = L.seg_gamma.begin() + L.box_seg_begin[box + 1];
            const auto it = std::lower_bound(b0, b1, g);
            if (it == b1 || *it != g) throw InternalError("cone plan: unmarked segment");
            return std::int32_t(it - L.seg_gamma.begin());
        };
        parallel_for(std::int64_t(nb), w, [&](std::int64_t tb) {
            const std::uint32_t n_t = B.end[tb] - B.begin[tb];
            std::int64_t at = L.cev_begin[tb];
            for (std::int32_t j = cz.ptr[tb]; j < cz.ptr[tb + 1]; ++j) {
                const std::int32_t sb = cz.idx[j];
                for (std::uint32_t q = 0; q < n_t; ++q, ++at) L.cev_seg[at] = ordinal(sb, L.cev_seg[at]);
            }
        });
        if (d > 3) {
            const ConeLevel& PL = plan.level[d - 2];
            const auto& cptr = plan.child_ptr[d - 2];
            const auto& cidx = plan.child_idx[d - 2];
            const int P = PL.nodes_per_seg();
            parallel_for(std::int64_t(PL.nseg()), w, [&](std::int64_t so) {
                const std::int32_t pb = PL.seg_box[so];
                const int nch = cptr[pb + 1] - cptr[pb];
                std::int64_t at = L.pev_begin[so];
                for (int node = 0; node < P; ++node)
                    for (int c = 0; c < nch; ++c, ++at)
                        L.pev_seg[at] = ordinal(cidx[cptr[pb] + c], L.pev_seg[at]);
            });
            group_parent_evaluations(L, PL.nseg(), w, P);
        }
        if (timing)
            std::fprintf(stderr, "cone plan level %d: decisions %.3fs, segments/ordinals/groups %.3fs (cev %zu pev %zu)\n",
                         d, secs(T0, T1), secs(T1, now()), L.cev_seg.size(), L.pev_seg.size());
    }
    return plan;
}

void parent_templates(const BoxTree& t, const ConePlanHost& plan, int d, const std::vector<std::int32_t>& gammas,
                      int workers, uninit_vector<double>& entries, std::vector<std::int32_t>& gc) {
    const ConeLevel& PL = plan.level[d - 2];
    const ConeLevel& CL = plan.level[d - 1];
    const int P = PL.nodes_per_seg();
    const double hp = t.half_diag(d - 1), hc = t.half_diag(d), half = 0.5 * t.side(d);
    const double k = plan.k;
    constexpr int E = 6;  // doubles per entry (device_plan.cuh kTmplDoubles)
    entries.resize(gammas.size() * 8 * std::size_t(P) * E);  // every entry written below
    gc.assign(gammas.size() * 8 * std::size_t(P), -1);
    const Vec3 origin{0.0, 0.0, 0.0};
    parallel_for(std::int64_t(gammas.size()), worker_count(workers), [&](std::int64_t slot) {
        const int gam = gammas[slot];
        const int g1 = gam % PL.ns, g2 = (gam / PL.ns) % PL.nc, g3 = gam / PL.ns / PL.nc;
        for (int o = 0; o < 8; ++o) {
            const Vec3 off{(o & 1) ? half : -half, (o & 2) ? half : -half, (o & 4) ? half : -half};
            for (int ip = 0; ip < PL.pang; ++ip)
                for (int it = 0; it < PL.pang; ++it)
                    for (int is = 0; is < PL.ps; ++is) {
                        const int node = is + PL.ps * (it + PL.pang * ip);
                        const double s = PL.s_nodes[std::size_t(g1) * PL.ps + is];
                        const Vec3 x = from_cone(s, PL.th_nodes[std::size_t(g2) * PL.pang + it],
                                                 PL.ph_nodes[std::size_t(g3) * PL.pang + ip], origin, hp);
                        const Cone cc = to_cone(x, off, hc);
                        const int g = segment_gamma(CL, cc);
                        const int c1 = g % CL.ns, c2 = (g / CL.ns) % CL.nc, c3 = g / CL.ns / CL.nc;
                        const Vec3 v = x - off;
                        const double rc = len(v), rp = hp / s;
                        const Vec3 sv = off - 2.0 * x;  // stable r_c - r_p (ifgf.cpp:149-153)
                        const double dr = dot3(sv, off) / (rc + rp);
                        const std::size_t at = (std::size_t(slot) * 8 + o) * P + node;
                        double* e = entries.data() + at * E;
                        e[0] = 2.0 * cc.s / CL.ds - (2 * c1 + 1.0);
                        e[1] = 2.0 * (cc.th - (c2 + 0.5) * CL.dth) / CL.dth;
                        e[2] = 2.0 * (cc.ph - (c3 + 0.5) * CL.dph) / CL.dph;
                        e[3] = rp / rc * std::cos(k * dr);
                        e[4] = rp / rc * std::sin(k * dr);
                        e[5] = 1.0 / rc;
                        gc[at] = g;
                    }
        }
    });
}

std::vector<std::vector<std::uint8_t>> active_boxes(const BoxTree& t, std::uint32_t lo, std::uint32_t hi) {
    std::vector<std::vector<std::uint8_t>> a(t.depth);
    for (int d = 1; d <= t.depth; ++d) {
        const BoxLevel& B = t.level[d - 1];
        a[d - 1].resize(B.size());
        for (std::size_t b = 0; b < B.size(); ++b) a[d - 1][b] = (B.begin[b] < hi && B.end[b] > lo) ? 1 : 0;
    }
    return a;
}

std::vector<std::uint32_t> partition_sources_light(const BoxTree& t, const BoxRelations& rel, int parts) {
    if (parts < 1) throw InvalidArgument("partition: need at least one part");
    const std::size_t n = t.perm.size();
    const int D = t.depth;
    const BoxLevel& leaves = t.level[D - 1];
    const Adjacency& nbr = rel.nbr[D - 1];
    const Adjacency& cz = rel.cousin[D - 1];
    std::vector<double> cost(leaves.size(), 0.0);
    for (std::size_t b = 0; b < leaves.size(); ++b) {
        const double np = double(leaves.end[b] - leaves.begin[b]);
        double nn = 0, ce = 0;
        for (int j = nbr.ptr[b]; j < nbr.ptr[b + 1]; ++j) nn += leaves.end[nbr.idx[j]] - leaves.begin[nbr.idx[j]];
        for (int j = cz.ptr[b]; j < cz.ptr[b + 1]; ++j) ce += leaves.end[cz.idx[j]] - leaves.begin[cz.idx[j]];
        // near pairs, leaf fill over ~40 relevant segments x 75 nodes, cousin evaluations
        cost[b] = 47.0 * np * nn + 47.0 * 75.0 * 40.0 * np + 1358.0 * ce;
    }
    double total = 0;
    for (double c : cost) total += c;
    std::vector<std::uint32_t> out(parts + 1, 0);
    double acc = 0;
    int r = 1;
    for (std::size_t b = 0; b < leaves.size() && r < parts; ++b) {
        acc += cost[b];
        while (r < parts && acc >= total * r / parts) out[r++] = leaves.end[b];
    }
    for (; r < parts; ++r) out[r] = std::uint32_t(n);
    out[parts] = std::uint32_t(n);
    return out;
}

// cost-balanced leaf-aligned boundaries: per leaf box, near pairs + leaf-fill
// interactions + cousin evaluations (as source box) weighted by their flop counts
std::vector<std::uint32_t> partition_sources(const BoxTree& t, const BoxRelations& rel, const ConePlanHost& plan,
                                             int parts) {
    if (parts < 1) throw InvalidArgument("partition: need at least one part");
    const std::size_t n = t.perm.size();
    const int D = t.depth;
    const BoxLevel& leaves = t.level[D - 1];
    const std::size_t nb = leaves.size();
    std::vector<double> cost(nb, 0.0);
    const Adjacency& nbr = rel.nbr[D - 1];
    for (std::size_t b = 0; b < nb; ++b) {
        const double np = double(leaves.end[b] - leaves.begin[b]);
        double nn = 0;
        for (int j = nbr.ptr[b]; j < nbr.ptr[b + 1]; ++j) nn += leaves.end[nbr.idx[j]] - leaves.begin[nbr.idx[j]];
        cost[b] = 47.0 * np * nn;
        if (D >= 3) {
            const ConeLevel& CL = plan.level[D - 1];
            cost[b] += 47.0 * 75.0 * np * double(CL.box_seg_begin[b + 1] - CL.box_seg_begin[b]);
            const Adjacency& cz = rel.cousin[D - 1];
            double ce = 0;
            for (int j = cz.ptr[b]; j < cz.ptr[b + 1]; ++j) ce += leaves.end[cz.idx[j]] - leaves.begin[cz.idx[j]];
            cost[b] += 1358.0 * ce + 1400.0 * 75.0 * double(CL.box_seg_begin[b + 1] - CL.box_seg_begin[b]);
        }
    }
    double total = 0;
    for (double c : cost) total += c;
    std::vector<std::uint32_t> out(parts + 1, 0);
    double acc = 0;
    int r = 1;
    for (std::size_t b = 0; b < nb && r < parts; ++b) {
        acc += cost[b];
        while (r < parts && acc >= total * r / parts) out[r++] = leaves.end[b];
    }
    for (; r < parts; ++r) out[r] = std::uint32_t(n);
    out[parts] = std::uint32_t(n);
    return out;
}


std::string plan_diagnostics(const BoxTree& t, const ConePlanHost& plan) {
    std::ostringstream os;
    os << "levels " << t.depth << "\n";
    for (int d = 3; d <= t.depth; ++d) {
        const ConeLevel& L = plan.level[d - 1];
        os << "level " << d << ": boxes=" << t.level[d - 1].size() << " segments=" << L.nseg()
           << " interp_points=" << L.nseg() * std::size_t(L.nodes_per_seg()) << " ns=" << L.ns
           << " nc=" << L.nc << "\n";
    }
    return os.str();
}

}  // namespace ifgfb200
