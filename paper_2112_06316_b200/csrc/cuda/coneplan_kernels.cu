// Cone-segment decisions of the plan (host/coneplan.cpp build_cone_plan) batched on the GPU.
//
// A decision is segment_gamma(to_cone(x, c, h)) (ifgf.cpp:161-176, kernels.cpp:34-48). Every
// operation in it is IEEE-exact and reproduced here in the host's order (this file is
// compiled with --fmad=false), except acos and atan2, where CUDA's libm may differ from
// glibc's in the last ulps. Such a difference can only change a decision when the angle lies
// on (or within rounding of) a cell boundary, the theta = pi pole or the phi seam, so every
// evaluation within a conservative margin of one of those is FLAGGED and redone on the host
// with glibc; all other decisions are provably the host's. SURVEY.md Appendix D: exact ties
// (phi = pi/4) do occur, and they are exactly the flagged ones.
#include <vector>

#include "../fields_gpu.hpp"
#include "../host/coneplan.hpp"
#include "dev_common.cuh"
#include "kernels.cuh"

namespace ifgfb200 {
namespace {

constexpr double kTwoPiD = 2.0 * kPi;  // host/coneplan.cpp kTwoPiC
constexpr double kPiD = kPi;
constexpr double kAngleMargin = 1e-9;  // in cell units; CUDA vs glibc acos/atan2 differ by ~1e-16

struct GeoDev {
    int ns, nc;
    double ds, dth, dph, h, eta;
};

// gamma of the segment holding v (relative to the box centre); unsure: leave it to the host
__device__ __forceinline__ int decide(const GeoDev& L, double vx, double vy, double vz, bool& unsure) {
    const double r = sqrt(vx * vx + vy * vy + vz * vz);
    if (!(r >= 1e-300)) {  // the host throws ("point at box center")
        unsure = true;
        return 0;
    }
    const double s = L.h / r;
    if (s > L.eta) {  // the host throws (segment query with s > sqrt(3)/3)
        unsure = true;
        return 0;
    }
    double ct = vz / r;
    ct = fmin(1.0, fmax(-1.0, ct));
    const double th = acos(ct);
    const double phr = atan2(vy, vx);
    double ph = phr;
    if (ph < 0.0) ph += kTwoPiD;
    if (ph >= kTwoPiD) ph = 0.0;
    const double tt = th / L.dth, tp = ph / L.dph;
    if (fabs(tt - rint(tt)) < kAngleMargin || fabs(tp - rint(tp)) < kAngleMargin || kPiD - th < 1e-12 ||
        fabs(phr) < 1e-12 || kTwoPiD - ph < 1e-12)
        unsure = true;
    int g1 = int(floor(s / L.ds)) + 1;
    if (g1 > L.ns) g1 = L.ns;
    if (g1 < 1) g1 = 1;
    int g2, g3;
    if (th >= kPiD) {
        g2 = L.nc;
        g3 = 2 * L.nc;
    } else {
        g2 = min(L.nc, int(floor(th / L.dth)) + 1);
        if (g2 < 1) g2 = 1;
        g3 = min(2 * L.nc, int(floor(ph / L.dph)) + 1);
        if (g3 < 1) g3 = 1;
    }
    return (g1 - 1) + L.ns * ((g2 - 1) + L.nc * (g3 - 1));
}

__device__ __forceinline__ void flag(std::int64_t at, unsigned long long* cnt, std::int64_t* list, std::int64_t cap) {
    const unsigned long long i = atomicAdd(cnt, 1ull);
    if (std::int64_t(i) < cap) list[i] = at;
}

__global__ void cousin_decide_kernel(GeoDev L, std::int64_t n, int nb, const std::int64_t* __restrict__ cev_begin,
                                     const std::uint32_t* __restrict__ bbeg, const std::uint32_t* __restrict__ bend,
                                     const std::int32_t* __restrict__ czptr, const std::int32_t* __restrict__ czidx,
                                     const double* __restrict__ px, const double* __restrict__ py,
                                     const double* __restrict__ pz, const double* __restrict__ cx,
                                     const double* __restrict__ cy, const double* __restrict__ cz, int spb,
                                     std::int32_t* __restrict__ seg, std::uint8_t* __restrict__ marks,
                                     unsigned long long* nflag, std::int64_t* flags, std::int64_t cap) {
    const std::int64_t at = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
    if (at >= n) return;
    int lo = 0, hi = nb;  // last tb with cev_begin[tb] <= at
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (cev_begin[mid] <= at) lo = mid;
        else hi = mid;
    }
    const int tb = lo;
    const std::int64_t off = at - cev_begin[tb];
    const std::int64_t n_t = std::int64_t(bend[tb]) - bbeg[tb];
    const int sb = czidx[czptr[tb] + int(off / n_t)];
    const std::int64_t t = bbeg[tb] + off % n_t;
    bool unsure = false;
    const int g = decide(L, px[t] - cx[sb], py[t] - cy[sb], pz[t] - cz[sb], unsure);
    if (unsure) {
        flag(at, nflag, flags, cap);
        return;
    }
    seg[at] = g;
    marks[std::size_t(sb) * spb + g] = 1;
}

__global__ void parent_decide_kernel(GeoDev L, GeoDev PL, int ps, int pang, std::int64_t nsp,
                                     const std::int32_t* __restrict__ seg_box, const std::int32_t* __restrict__ seg_gamma,
                                     const double* __restrict__ s_nodes, const double* __restrict__ th_sin,
                                     const double* __restrict__ th_cos, const double* __restrict__ ph_sin,
                                     const double* __restrict__ ph_cos, const double* __restrict__ pcx,
                                     const double* __restrict__ pcy, const double* __restrict__ pcz,
                                     const std::int32_t* __restrict__ cptr, const std::int32_t* __restrict__ cidx,
                                     const double* __restrict__ cx, const double* __restrict__ cy,
                                     const double* __restrict__ cz, const std::int64_t* __restrict__ pev_begin,
                                     int spb, std::int32_t* __restrict__ seg, std::uint8_t* __restrict__ marks,
                                     unsigned long long* nflag, std::int64_t* flags, std::int64_t cap) {
    const std::int64_t idx = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
    const int P = ps * pang * pang;
    if (idx >= nsp * P) return;
    const std::int64_t so = idx / P;
    const int node = int(idx % P);
    const int pb = seg_box[so];
    const int gam = seg_gamma[so];
    const int g1 = gam % PL.ns, g2 = (gam / PL.ns) % PL.nc, g3 = gam / PL.ns / PL.nc;
    const int is = node % ps, it = (node / ps) % pang, ip = node / (ps * pang);
    // from_cone (kernels.cpp:27-32) with glibc sin/cos of the node tables
    const double r = PL.h / s_nodes[g1 * ps + is];
    const double st = th_sin[g2 * pang + it], ct = th_cos[g2 * pang + it];
    const double x = pcx[pb] + r * st * ph_cos[g3 * pang + ip];
    const double y = pcy[pb] + r * st * ph_sin[g3 * pang + ip];
    const double z = pcz[pb] + r * ct;
    const int c0 = cptr[pb], nch = cptr[pb + 1] - c0;
    const std::int64_t at0 = pev_begin[so] + std::int64_t(node) * nch;
    for (int c = 0; c < nch; ++c) {
        const int ch = cidx[c0 + c];
        bool unsure = false;
        const int g = decide(L, x - cx[ch], y - cy[ch], z - cz[ch], unsure);
        if (unsure) {
            flag(at0 + c, nflag, flags, cap);
            continue;
        }
        seg[at0 + c] = g;
        marks[std::size_t(ch) * spb + g] = 1;
    }
}

template <class T>
struct DBuf {
    T* p = nullptr;
    std::size_t n = 0;
    DBuf() = default;
    explicit DBuf(std::size_t count) : n(count) {
        IFGF_CUDA(cudaMalloc(&p, std::max<std::size_t>(count, 1) * sizeof(T)));
    }
    DBuf(const std::vector<T>& v) : DBuf(v.size()) {
        if (!v.empty()) IFGF_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    }
    ~DBuf() { cudaFree(p); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
};

void split(const std::vector<Vec3>& v, std::vector<double>& x, std::vector<double>& y, std::vector<double>& z) {
    x.resize(v.size());
    y.resize(v.size());
    z.resize(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) {
        x[i] = v[i].x;
        y[i] = v[i].y;
        z[i] = v[i].z;
    }
}

GeoDev geo_of(const ConeLevel& L, double h) {
    return {L.ns, L.nc, L.ds, L.dth, L.dph, h, kConeEtaC + 1e-12};
}

}  // namespace

void gpu_cone_decisions(const ConeDecisionJob& job, ConeLevel& L, std::vector<std::uint8_t>& marks,
                        std::vector<std::int64_t>& flagged_cev, std::vector<std::int64_t>& flagged_pev, int device) {
    IFGF_CUDA(cudaSetDevice(device));
    const int nb = int(job.B->size());
    const int spb = L.segs_per_box();
    const GeoDev G = geo_of(L, job.h);
    std::vector<double> hx, hy, hz;
    DBuf<std::uint8_t> d_marks(marks.size());
    IFGF_CUDA(cudaMemset(d_marks.p, 0, std::max<std::size_t>(marks.size(), 1)));
    DBuf<unsigned long long> d_cnt(1);
    split(*job.ctr, hx, hy, hz);
    DBuf<double> ccx(hx), ccy(hy), ccz(hz);
    auto run_flags = [&](std::int64_t n, auto&& launch, std::vector<std::int64_t>& flagged) {
        // flag capacity: a first pass with a bounded list; a full list on overflow (never in practice)
        for (std::int64_t cap = std::min<std::int64_t>(n, std::int64_t(1) << 22);; cap = n) {
            DBuf<std::int64_t> d_flags(std::size_t(std::max<std::int64_t>(cap, 1)));
            IFGF_CUDA(cudaMemset(d_cnt.p, 0, sizeof(unsigned long long)));
            launch(d_flags.p, cap);
            IFGF_CUDA(cudaGetLastError());
            unsigned long long cnt = 0;
            IFGF_CUDA(cudaMemcpy(&cnt, d_cnt.p, sizeof(cnt), cudaMemcpyDeviceToHost));
            if (std::int64_t(cnt) <= cap) {
                flagged.resize(cnt);
                if (cnt) IFGF_CUDA(cudaMemcpy(flagged.data(), d_flags.p, cnt * sizeof(std::int64_t), cudaMemcpyDeviceToHost));
                return;
            }
        }
    };
    // cousin evaluations
    {
        const std::int64_t n = L.cev_begin[nb];
        if (n > 0) {
            split(*job.pts, hx, hy, hz);
            DBuf<double> px(hx), py(hy), pz(hz);
            DBuf<std::int64_t> cb(L.cev_begin);
            DBuf<std::uint32_t> bb(job.B->begin), be(job.B->end);
            DBuf<std::int32_t> zp(job.cz->ptr), zi(job.cz->idx);
            DBuf<std::int32_t> seg{std::size_t(n)};
            run_flags(n, [&](std::int64_t* fl, std::int64_t cap) {
                cousin_decide_kernel<<<int((n + 255) / 256), 256>>>(G, n, nb, cb.p, bb.p, be.p, zp.p, zi.p, px.p, py.p,
                                                                    pz.p, ccx.p, ccy.p, ccz.p, spb, seg.p, d_marks.p,
                                                                    d_cnt.p, fl, cap);
            }, flagged_cev);
            IFGF_CUDA(cudaMemcpy(L.cev_seg.data(), seg.p, std::size_t(n) * sizeof(std::int32_t), cudaMemcpyDeviceToHost));
        }
    }
    // parent-node evaluations
    if (job.PL) {
        const ConeLevel& PL = *job.PL;
        const std::int64_t nsp = std::int64_t(PL.nseg());
        const std::int64_t n = L.pev_begin.empty() ? 0 : L.pev_begin.back();
        if (n > 0) {
            const GeoDev PG = geo_of(PL, job.ph);
            DBuf<std::int32_t> sbx(PL.seg_box), sgm(PL.seg_gamma);
            DBuf<double> sn(PL.s_nodes), ths(job.th_sin), thc(job.th_cos), phs(job.ph_sin), phc(job.ph_cos);
            split(*job.pctr, hx, hy, hz);
            DBuf<double> pcx(hx), pcy(hy), pcz(hz);
            DBuf<std::int32_t> cp(*job.cptr), ci(*job.cidx);
            DBuf<std::int64_t> pb(L.pev_begin);
            DBuf<std::int32_t> seg{std::size_t(n)};
            const std::int64_t items = nsp * PL.nodes_per_seg();
            run_flags(n, [&](std::int64_t* fl, std::int64_t cap) {
                parent_decide_kernel<<<int((items + 255) / 256), 256>>>(
                    G, PG, PL.ps, PL.pang, nsp, sbx.p, sgm.p, sn.p, ths.p, thc.p, phs.p, phc.p, pcx.p, pcy.p, pcz.p, cp.p,
                    ci.p, ccx.p, ccy.p, ccz.p, pb.p, spb, seg.p, d_marks.p, d_cnt.p, fl, cap);
            }, flagged_pev);
            IFGF_CUDA(cudaMemcpy(L.pev_seg.data(), seg.p, std::size_t(n) * sizeof(std::int32_t), cudaMemcpyDeviceToHost));
        }
    }
    if (!marks.empty())
        IFGF_CUDA(cudaMemcpy(marks.data(), d_marks.p, marks.size(), cudaMemcpyDeviceToHost));
}

}  // namespace ifgfb200
