// IFGF far-field kernels for sm_100a (complex fp64, FP64-pipe bound).
//
//  * leaf_fill   : level_d_fill (ifgf.cpp:312-391) — one CTA per leaf box, the box's sources
//                  staged in shared memory, one thread per (segment, interpolation node),
//                  followed by the separable 3x5x5 value->coefficient transform in shared
//                  memory (transform3, ifgf.cpp:92-130).
//  * cousin_eval : cousin_evaluate (ifgf.cpp:396-450) — one thread per target point, the
//                  cone segment taken from the host-decided ordinal list; the
//                  3-D Chebyshev series is evaluated as a nested basis contraction (replaces
//                  Clenshaw; equal to 1e-15).
//  * parent_fill : parent_fill (ifgf.cpp:452-568) — one thread per (parent segment, node),
//                  looping over the parent's children, re-centring ratio via the stable
//                  radius difference (ifgf.cpp:149-153), then the block transform.
#include <algorithm>

#include "dev_common.cuh"
#include <cstdlib>

#include "ifgf_device.cuh"
#include "kernels.cuh"

namespace ifgfb200 {
namespace {

using namespace dev;
using namespace ifgfdev;
constexpr int kLeafThreads = 384;
constexpr int kLeafTile = 256;
constexpr int kCousinThreads = 128;
constexpr int kCousinSlots = 2;
constexpr int kParentSlots = 2;
constexpr int kParentThreads = 320;

// ------------------------------------------------------------------ leaf fill
template <int NP>
__global__ void __launch_bounds__(kLeafThreads)
leaf_fill_kernel(LevelDev L, PointsDev P, const double2* __restrict__ a_p, double k, Pipes pp,
                 const double* __restrict__ Ms, const double* __restrict__ Ma,
                 double2* __restrict__ store) {
    extern __shared__ double smem[];
    const int b = blockIdx.x;
    const int s0 = L.box_seg_begin[b], s1 = L.box_seg_begin[b + 1];
    if (s0 == s1 || (L.active && !L.active[b])) return;
    const int ps = L.ps, pa = L.pang;
    const int NPTS = ps * pa * pa;
    const int G = max(1, int(blockDim.x) / NPTS);
    const int pb = int(L.beg[b]);
    const int nsrc = int(L.end[b]) - pb;
    const double cx = L.cx[b], cy = L.cy[b], cz = L.cz[b];
    const double h = L.h;

    double* sdx = smem;
    double* sdy = sdx + kLeafTile;
    double* sdz = sdy + kLeafTile;
    double* snx = sdz + kLeafTile;
    double* sny = snx + kLeafTile;
    double* snz = sny + kLeafTile;
    double* sar = snz + kLeafTile;
    double* sai = sar + kLeafTile;
    double2* v0 = reinterpret_cast<double2*>(sai + kLeafTile);
    double2* v1 = v0 + G * NP * NPTS;

    auto load_tile = [&](int t0, int tn) {
        for (int q = threadIdx.x; q < tn; q += blockDim.x) {
            const int t = pb + t0 + q;
            sdx[q] = P.x[t] - cx;
            sdy[q] = P.y[t] - cy;
            sdz[q] = P.z[t] - cz;
            snx[q] = P.nx[t];
            sny[q] = P.ny[t];
            snz[q] = P.nz[t];
            const double2 a = a_p[t];
            sar[q] = a.x;
            sai[q] = a.y;
        }
    };
    const bool one_tile = nsrc <= kLeafTile;
    if (one_tile) load_tile(0, nsrc);
    __syncthreads();

    for (int g0 = s0; g0 < s1; g0 += G) {
        const int gcount = min(G, s1 - g0);
        const int items = gcount * NPTS;
        for (int base = 0; base < items; base += blockDim.x) {
            const int item = base + threadIdx.x;
            const bool act = item < items;
            const int seg_l = act ? item / NPTS : 0;
            const int node = act ? item % NPTS : 0;
            double xh = 0, yh = 0, zh = 0, soh = 0, khos = 0;
            if (act) {
                const int gam = L.seg_gamma[g0 + seg_l];
                const int g1 = gam % L.ns, g2 = (gam / L.ns) % L.nc, g3 = gam / L.ns / L.nc;
                const int is = node % ps, it = (node / ps) % pa, ip = node / (ps * pa);
                const double s = L.s_nodes[g1 * ps + is];
                double sth, cth, sph, cph;
                sincos(L.th_nodes[g2 * pa + it], &sth, &cth);
                sincos(L.ph_nodes[g3 * pa + ip], &sph, &cph);
                xh = sth * cph;
                yh = sth * sph;
                zh = cth;
                soh = s / h;
                khos = k * h / s;
            }
            double2 acc[NP];
#pragma unroll
            for (int i = 0; i < NP; ++i) acc[i] = make_double2(0.0, 0.0);
            for (int t0 = 0; t0 < nsrc; t0 += kLeafTile) {
                const int tn = min(kLeafTile, nsrc - t0);
                if (!one_tile) {
                    __syncthreads();
                    load_tile(t0, tn);
                    __syncthreads();
                }
                if (!act) continue;
                for (int q = 0; q < tn; ++q) {
                    const double vx = fma(-sdx[q], soh, xh);
                    const double vy = fma(-sdy[q], soh, yh);
                    const double vz = fma(-sdz[q], soh, zh);
                    const double nv2 = fma(vx, vx, fma(vy, vy, vz * vz));
                    const double inv = rsqrt(nv2);
                    const double nv = nv2 * inv;
                    const double arg = khos * (nv2 - 1.0) * fast_rcp(nv + 1.0);
                    double sn, cs;
                    sincos_bounded(arg, &sn, &cs);
                    const double ar = sar[q], ai = sai[q];
                    const double2 pa_ = make_double2(fma(ar, cs, -ai * sn), fma(ar, sn, ai * cs));
                    const double dn = fma(vx, snx[q], fma(vy, sny[q], vz * snz[q]));
                    const double inv2 = inv * inv;
#pragma unroll
                    for (int i = 0; i < NP; ++i) {
                        switch (pp.f[i]) {
                            case 1:
                                cfma_r(acc[i], pa_, inv);
                                break;
                            case 2:
                                cfma_r(acc[i], pa_, dn * inv2 * inv);
                                break;
                            case 3:
                                cfma_r(acc[i], pa_, dn * inv2);
                                break;
                            default: {  // W4: (s/(h|v|) - i k) (v.n)/|v|^2
                                const double dn2 = dn * inv2;
                                cfma(acc[i], pa_, make_double2(soh * inv * dn2, -k * dn2));
                            }
                        }
                    }
                }
            }
            if (act) {
#pragma unroll
                for (int i = 0; i < NP; ++i) v0[(seg_l * NP + i) * NPTS + node] = acc[i];
            }
        }
        __syncthreads();
        block_transform(v0, v1, gcount * NP, ps, pa, Ms, Ma, store + std::size_t(g0) * NP * NPTS);
        __syncthreads();
    }
}

// ------------------------------------------------------------------ cousin evaluation
template <int NP, int PS, int PA>
__global__ void __launch_bounds__(kCousinThreads)
cousin_kernel(LevelDev L, PointsDev P, const double2* __restrict__ store, double k, Pipes pp,
              double2* __restrict__ Sp, double2* __restrict__ Dp) {
    extern __shared__ double2 cz_smem[];
    const int ps = L.ps, pa = L.pang;
    const int NPTS = ps * pa * pa;
    const int blk_elems = NP * NPTS;
    double2* wbuf = cz_smem + (threadIdx.x >> 5) * kCousinSlots * blk_elems;
    const int c = blockIdx.x;
    const int tb = L.chunk_box[c];
    const int tbeg = int(L.beg[tb]);
    const int n_t = int(L.end[tb]) - tbeg;
    const int q = L.chunk_q0[c] + threadIdx.x;
    const bool act = q < n_t;
    if (__all_sync(0xffffffffu, !act)) return;  // whole warp idle (no CTA-wide barriers here)
    const int t = act ? tbeg + q : tbeg;
    const double x = P.x[t], y = P.y[t], z = P.z[t];
    const double h = L.h;
    const int j0 = L.cz_ptr[tb], j1 = L.cz_ptr[tb + 1];
    const std::int64_t ev0 = L.cev_begin[tb] + q;
    double2 accS = make_double2(0.0, 0.0), accD = make_double2(0.0, 0.0);
    double ts[PS > 0 ? PS : kMaxOrd], tt[PA > 0 ? PA : kMaxOrd], tp[PA > 0 ? PA : kMaxOrd];
    for (int j = j0; j < j1; ++j) {
        const int sb = L.cz_idx[j];
        if (L.active && !L.active[sb]) continue;  // source box owned by another rank
        const int so = act ? L.cev_seg[ev0 + std::int64_t(j - j0) * n_t] : -1;
        const double vx = x - L.cx[sb], vy = y - L.cy[sb], vz = z - L.cz[sb];
        const double r2 = fma(vx, vx, fma(vy, vy, vz * vz));
        const double inv_r = rsqrt(r2);
        const double r = r2 * inv_r;
        double2 e1 = make_double2(0.0, 0.0);
        if (act) {
            const LocalCoords lc = local_coords(vx, vy, vz, inv_r, h, L.seg_gamma[so], L);
            basis3<PS, PA>(lc, ts, tt, tp, ps, pa);
            double sn, cs;
            sincos_bounded(k * r, &sn, &cs);
            const double f1 = kInv4PiD * inv_r;
            e1 = make_double2(cs * f1, sn * f1);  // e^{ikr}/(4 pi r)
        }
        with_staged_block<kCousinSlots>(so, store, blk_elems, wbuf, [&](const double2* blk) {
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                const double2 val = eval_series_sm<PS, PA>(blk + i * NPTS, ts, tt, tp, ps, pa);
                const double2 w = cmul(e1, val);
                switch (pp.f[i]) {
                    case 1:
                        accS = cadd(accS, w);
                        break;
                    case 2:
                        cfma_r(accD, w, inv_r);
                        break;
                    case 3:  // -ik e^{ikr}/(4 pi r) val
                        accD.x = fma(k, w.y, accD.x);
                        accD.y = fma(-k, w.x, accD.y);
                        break;
                    default:
                        accD = cadd(accD, w);
                }
            }
        });
    }
    if (!act) return;
    Sp[t] = cadd(Sp[t], accS);
    Dp[t] = cadd(Dp[t], accD);
}

// ------------------------------------------------------------------ parent fill
struct ChildMap {
    int w1, w2, w3, w4;
};

template <int NPP, int NPC, int PS, int PA>
__global__ void __launch_bounds__(kParentThreads, 2)
parent_kernel(LevelDev Lp, LevelDev Lc, const double2* __restrict__ cstore, double k, Pipes ppar,
              ChildMap cm, const double* __restrict__ Ms, const double* __restrict__ Ma,
              double2* __restrict__ pstore) {
    extern __shared__ double smem[];
    const int ps = Lp.ps, pa = Lp.pang;
    const int NPTS = ps * pa * pa;
    const int cps = Lc.ps, cpa = Lc.pang;
    const int CPTS = cps * cpa * cpa;
    const int cblk = NPC * CPTS;
    const int G = max(1, int(blockDim.x) / NPTS);
    const int g0 = blockIdx.x * G;
    if (g0 >= Lp.nseg) return;
    const int gcount = min(G, Lp.nseg - g0);
    const int items = gcount * NPTS;
    double2* v0 = reinterpret_cast<double2*>(smem);
    double2* v1 = v0 + G * NPP * NPTS;
    double2* wbuf = v1 + G * NPP * NPTS + (threadIdx.x >> 5) * kParentSlots * cblk;
    const double hp = Lp.h, hc = Lc.h;
    double ts[PS > 0 ? PS : kMaxOrd], tt[PA > 0 ? PA : kMaxOrd], tp[PA > 0 ? PA : kMaxOrd];

    for (int base = 0; base < items; base += blockDim.x) {
        const int item = base + threadIdx.x;
        const bool act = item < items;
        const int seg_l = act ? item / NPTS : 0, node = act ? item % NPTS : 0;
        const int so = g0 + seg_l;
        const int pb = Lp.seg_box[so];
        const int gam = Lp.seg_gamma[so];
        const int g1 = gam % Lp.ns, g2 = (gam / Lp.ns) % Lp.nc, g3 = gam / Lp.ns / Lp.nc;
        const int is = node % ps, it = (node / ps) % pa, ip = node / (ps * pa);
        const double s = Lp.s_nodes[g1 * ps + is];
        double sth, cth, sph, cph;
        sincos(Lp.th_nodes[g2 * pa + it], &sth, &cth);
        sincos(Lp.ph_nodes[g3 * pa + ip], &sph, &cph);
        const double rp = hp / s;
        const double pcx = Lp.cx[pb], pcy = Lp.cy[pb], pcz = Lp.cz[pb];
        const double x = pcx + rp * sth * cph;
        const double y = pcy + rp * sth * sph;
        const double z = pcz + rp * cth;
        const int c0 = Lp.ch_ptr[pb];
        const int nch = act ? Lp.ch_ptr[pb + 1] - c0 : 0;
        const int nch_warp = __reduce_max_sync(0xffffffffu, unsigned(nch));
        const std::int64_t ev = Lc.pev_begin[so] + std::int64_t(node) * nch;
        double2 acc[NPP];
#pragma unroll
        for (int i = 0; i < NPP; ++i) acc[i] = make_double2(0.0, 0.0);
        for (int c = 0; c < nch_warp; ++c) {
            const bool live = c < nch && (!Lc.active || Lc.active[Lp.ch_idx[c0 + c]]);
            const int ch = live ? Lp.ch_idx[c0 + c] : 0;
            const int cso = live ? Lc.pev_seg[ev + c] : -1;
            const double ccx = Lc.cx[ch], ccy = Lc.cy[ch], ccz = Lc.cz[ch];
            const double vx = x - ccx, vy = y - ccy, vz = z - ccz;
            const double rc2 = fma(vx, vx, fma(vy, vy, vz * vz));
            const double inv_rc = rsqrt(rc2);
            const double rc = rc2 * inv_rc;
            double sn = 0.0, cs = 0.0, q1 = 0.0;
            if (live) {
                const LocalCoords lc = local_coords(vx, vy, vz, inv_rc, hc, Lc.seg_gamma[cso], Lc);
                basis3<PS, PA>(lc, ts, tt, tp, cps, cpa);
                // stable r_c - r_p (ifgf.cpp:149-153)
                const double sx = ccx + pcx - 2.0 * x, sy = ccy + pcy - 2.0 * y, sz = ccz + pcz - 2.0 * z;
                const double dr = fma(sx, ccx - pcx, fma(sy, ccy - pcy, sz * (ccz - pcz))) / (rc + rp);
                sincos_bounded(k * dr, &sn, &cs);
                q1 = rp * inv_rc;
            }
            const double2 ratio1 = make_double2(cs * q1, sn * q1);
            with_staged_block<kParentSlots>(cso, cstore, cblk, wbuf, [&](const double2* blk) {
                double2 val[NPC];
#pragma unroll
                for (int i = 0; i < NPC; ++i) val[i] = eval_series_sm<PS, PA>(blk + i * CPTS, ts, tt, tp, cps, cpa);
#pragma unroll
                for (int i = 0; i < NPP; ++i) {
                    switch (ppar.f[i]) {
                        case 1:
                            cfma(acc[i], ratio1, val[cm.w1]);
                            break;
                        case 4:
                            if (cm.w4 >= 0) {
                                cfma(acc[i], ratio1, val[cm.w4]);
                            } else {  // child carries W2/W3: re-centre into W4
                                const double q2 = q1 * inv_rc;
                                cfma(acc[i], make_double2(cs * q2, sn * q2), val[cm.w2]);
                                const double2 r3 = cmul(ratio1, val[cm.w3]);
                                acc[i].x = fma(k, r3.y, acc[i].x);
                                acc[i].y = fma(-k, r3.x, acc[i].y);
                            }
                            break;
                        case 2: {
                            const double q3 = q1 * q1;
                            cfma(acc[i], make_double2(cs * q3, sn * q3), val[cm.w2]);
                            break;
                        }
                        default:  // W3
                            cfma(acc[i], ratio1, val[cm.w3]);
                    }
                }
            });
        }
        if (act) {
#pragma unroll
            for (int i = 0; i < NPP; ++i) v0[(seg_l * NPP + i) * NPTS + node] = acc[i];
        }
    }
    __syncthreads();
    block_transform(v0, v1, gcount * NPP, ps, pa, Ms, Ma, pstore + std::size_t(g0) * NPP * NPTS);
}

int div_up(long a, long b) { return int((a + b - 1) / b); }

}  // namespace

void launch_leaf_fill(const LevelDev& L, const PointsDev& P, const double2* a_p, double k,
                      const Pipes& pipes, const double* Ms, const double* Ma, double2* store,
                      cudaStream_t st) {
    if (L.nb == 0 || L.nseg == 0) return;
    if (launch_leaf_fill_ray(L, P, a_p, k, pipes, Ms, Ma, store, st)) return;
    const int NPTS = L.ps * L.pang * L.pang;
    const int G = std::max(1, kLeafThreads / NPTS);
    const std::size_t smem = 8 * kLeafTile * sizeof(double) + 2 * std::size_t(G) * pipes.n * NPTS * sizeof(double2);
    auto go = [&](auto kern) {
        IFGF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<L.nb, kLeafThreads, smem, st>>>(L, P, a_p, k, pipes, Ms, Ma, store);
    };
    switch (pipes.n) {
        case 1: go(leaf_fill_kernel<1>); break;
        case 2: go(leaf_fill_kernel<2>); break;
        default: go(leaf_fill_kernel<3>); break;
    }
    IFGF_CUDA(cudaGetLastError());
}

void launch_cousin_eval(const LevelDev& L, const PointsDev& P, const double2* store, double k,
                        const Pipes& pipes, double2* Sp, double2* Dp, cudaStream_t st) {
    if (L.nchunk == 0) return;
    static const bool tc_off = [] {
        const char* e = std::getenv("IFGF_COUSIN_TC");
        return e && e[0] == '0';
    }();
    if (!tc_off && launch_cousin_eval_tc(L, P, store, k, pipes, Sp, Dp, st)) return;
    const bool def = L.ps == 3 && L.pang == 5;
    const std::size_t smem = std::size_t(kCousinThreads / 32) * kCousinSlots * pipes.n * L.ps * L.pang * L.pang *
                             sizeof(double2);
    auto go = [&](auto kern) {
        IFGF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<L.nchunk, kCousinThreads, smem, st>>>(L, P, store, k, pipes, Sp, Dp);
    };
    if (def) {
        switch (pipes.n) {
            case 1: go(cousin_kernel<1, 3, 5>); break;
            case 2: go(cousin_kernel<2, 3, 5>); break;
            default: go(cousin_kernel<3, 3, 5>); break;
        }
    } else {
        switch (pipes.n) {
            case 1: go(cousin_kernel<1, 0, 0>); break;
            case 2: go(cousin_kernel<2, 0, 0>); break;
            default: go(cousin_kernel<3, 0, 0>); break;
        }
    }
    IFGF_CUDA(cudaGetLastError());
}

void launch_parent_fill(const LevelDev& Lp, const LevelDev& Lc, const double2* child_store,
                        double k, const Pipes& parent_pipes, const Pipes& child_pipes,
                        const double* Ms, const double* Ma, double2* parent_store, cudaStream_t st) {
    if (Lp.nseg == 0) return;
    ChildMap cm{-1, -1, -1, -1};
    for (int i = 0; i < child_pipes.n; ++i) {
        switch (child_pipes.f[i]) {
            case 1: cm.w1 = i; break;
            case 2: cm.w2 = i; break;
            case 3: cm.w3 = i; break;
            default: cm.w4 = i;
        }
    }
    for (int i = 0; i < parent_pipes.n; ++i) {
        const int f = parent_pipes.f[i];
        const bool ok = (f == 1 && cm.w1 >= 0) || (f == 4 && (cm.w4 >= 0 || (cm.w2 >= 0 && cm.w3 >= 0))) ||
                        (f == 2 && cm.w2 >= 0) || (f == 3 && cm.w3 >= 0);
        if (!ok) throw InternalError("parent pipeline without the child pipeline it needs");
    }
    const int NPTS = Lp.ps * Lp.pang * Lp.pang;
    const int G = std::max(1, kParentThreads / NPTS);
    const int CPTS = Lc.ps * Lc.pang * Lc.pang;
    const std::size_t smem = (2 * std::size_t(G) * parent_pipes.n * NPTS +
                              std::size_t(kParentThreads / 32) * kParentSlots * child_pipes.n * CPTS) *
                             sizeof(double2);
    const int grid = div_up(Lp.nseg, G);
    const bool def = Lp.ps == 3 && Lp.pang == 5 && Lc.ps == 3 && Lc.pang == 5;
    auto go = [&](auto kern) {
        IFGF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<grid, kParentThreads, smem, st>>>(Lp, Lc, child_store, k, parent_pipes, cm, Ms, Ma, parent_store);
    };
    if (launch_parent_fill_tc(Lp, Lc, child_store, k, parent_pipes, child_pipes, Ms, Ma, parent_store, st)) return;
    const int code = parent_pipes.n * 4 + child_pipes.n;
#define IFGF_PARENT_CASE(NPP, NPC)                                     \
    case NPP * 4 + NPC:                                                \
        if (def) go(parent_kernel<NPP, NPC, 3, 5>);                    \
        else go(parent_kernel<NPP, NPC, 0, 0>);                        \
        break;
    switch (code) {
        IFGF_PARENT_CASE(1, 1)
        IFGF_PARENT_CASE(1, 2)
        IFGF_PARENT_CASE(1, 3)
        IFGF_PARENT_CASE(2, 2)
        IFGF_PARENT_CASE(2, 3)
        IFGF_PARENT_CASE(3, 3)
        default:
            throw InternalError("unsupported parent/child pipe combination");
    }
#undef IFGF_PARENT_CASE
    IFGF_CUDA(cudaGetLastError());
}

}  // namespace ifgfb200
