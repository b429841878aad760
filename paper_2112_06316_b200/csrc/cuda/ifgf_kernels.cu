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
#include "kernels.cuh"

namespace ifgfb200 {
namespace {

using namespace dev;

constexpr int kMaxOrd = 12;
constexpr int kLeafThreads = 384;
constexpr int kLeafTile = 256;
constexpr int kCousinThreads = 128;
constexpr int kParentThreads = 320;

struct LocalCoords {
    double ls, lt, lp;
};

// Cone coordinates of v = x - centre (inv_r = 1/|v|) relative to the host-decided segment
// gamma, mapped to [-1,1]^3 (LevelCones::local_coords, ifgf.cpp:178-183).
__device__ __forceinline__ LocalCoords local_coords(double vx, double vy, double vz, double inv_r,
                                                    double h, int gamma, const LevelDev& L) {
    const double s = h * inv_r;
    double ct = vz * inv_r;
    ct = fmin(1.0, fmax(-1.0, ct));
    const double th = acos(ct);
    double ph = atan2(vy, vx);
    if (ph < 0.0) ph += kTwoPiD;
    const int g1 = gamma % L.ns;
    const int rest = gamma / L.ns;
    const int g2 = rest % L.nc;
    const int g3 = rest / L.nc;
    // the host decision is authoritative; keep phi on the decided side of the 0/2pi seam
    if (g3 == 0 && ph > kPiD) ph -= kTwoPiD;
    if (g3 == 2 * L.nc - 1 && ph < kPiD) ph += kTwoPiD;
    LocalCoords o;
    o.ls = fma(s, 2.0 * L.inv_ds, -(2 * g1 + 1.0));
    o.lt = fma(th, 2.0 * L.inv_dth, -(2 * g2 + 1.0));
    o.lp = fma(ph, 2.0 * L.inv_dph, -(2 * g3 + 1.0));
    return o;
}

// sum_{ip,it,is} c[is + ps*(it + pa*ip)] T_is(ls) T_it(lt) T_ip(lp)
template <int PS, int PA>
__device__ __forceinline__ double2 eval_series(const double2* __restrict__ c, const double* ts,
                                               const double* tt, const double* tp, int ps, int pa) {
    double2 acc = make_double2(0.0, 0.0);
    if constexpr (PS > 0) {
#pragma unroll
        for (int ip = 0; ip < PA; ++ip) {
            double2 a_t = make_double2(0.0, 0.0);
#pragma unroll
            for (int it = 0; it < PA; ++it) {
                const double2* line = c + PS * (it + PA * ip);
                double2 a_s = make_double2(0.0, 0.0);
#pragma unroll
                for (int is = 0; is < PS; ++is) cfma_r(a_s, ldg2(line + is), ts[is]);
                cfma_r(a_t, a_s, tt[it]);
            }
            cfma_r(acc, a_t, tp[ip]);
        }
    } else {
#pragma unroll 1
        for (int ip = 0; ip < pa; ++ip) {
            double2 a_t = make_double2(0.0, 0.0);
#pragma unroll 1
            for (int it = 0; it < pa; ++it) {
                const double2* line = c + ps * (it + pa * ip);
                double2 a_s = make_double2(0.0, 0.0);
#pragma unroll 1
                for (int is = 0; is < ps; ++is) cfma_r(a_s, ldg2(line + is), ts[is]);
                cfma_r(a_t, a_s, tt[it]);
            }
            cfma_r(acc, a_t, tp[ip]);
        }
    }
    return acc;
}

template <int PS, int PA>
__device__ __forceinline__ void basis3(const LocalCoords& lc, double* ts, double* tt, double* tp,
                                       int ps, int pa) {
    if constexpr (PS > 0) {
        cheb_row<PS>(lc.ls, ts);
        cheb_row<PA>(lc.lt, tt);
        cheb_row<PA>(lc.lp, tp);
    } else {
        ts[0] = tt[0] = tp[0] = 1.0;
        if (ps > 1) ts[1] = lc.ls;
        if (pa > 1) {
            tt[1] = lc.lt;
            tp[1] = lc.lp;
        }
        for (int i = 2; i < ps; ++i) ts[i] = 2.0 * lc.ls * ts[i - 1] - ts[i - 2];
        for (int i = 2; i < pa; ++i) {
            tt[i] = 2.0 * lc.lt * tt[i - 1] - tt[i - 2];
            tp[i] = 2.0 * lc.lp * tp[i - 1] - tp[i - 2];
        }
    }
}

// In-place separable value->coefficient transform of `nblk` blocks of P = ps*pa*pa values
// held in shared memory (v0), using v1 as scratch; the last pass writes to `dst`
// (global), block b going to dst + b*P. Called by the whole CTA.
__device__ void block_transform(double2* v0, double2* v1, int nblk, int ps, int pa,
                                const double* __restrict__ Ms, const double* __restrict__ Ma,
                                double2* __restrict__ dst) {
    const int P = ps * pa * pa;
    const int total = nblk * P;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {  // along s
        const int blk = e / P, node = e % P;
        const int is = node % ps, line = node / ps;
        const double2* src = v0 + blk * P + line * ps;
        double2 acc = make_double2(0.0, 0.0);
        for (int q = 0; q < ps; ++q) cfma_r(acc, src[q], Ms[is * ps + q]);
        v1[e] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < total; e += blockDim.x) {  // along theta
        const int blk = e / P, node = e % P;
        const int is = node % ps, it = (node / ps) % pa, ip = node / (ps * pa);
        const double2* src = v1 + blk * P + is + ps * pa * ip;
        double2 acc = make_double2(0.0, 0.0);
        for (int q = 0; q < pa; ++q) cfma_r(acc, src[ps * q], Ma[it * pa + q]);
        v0[e] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < total; e += blockDim.x) {  // along phi
        const int blk = e / P, node = e % P;
        const int is = node % ps, it = (node / ps) % pa, ip = node / (ps * pa);
        const double2* src = v0 + blk * P + is + ps * it;
        double2 acc = make_double2(0.0, 0.0);
        for (int q = 0; q < pa; ++q) cfma_r(acc, src[ps * pa * q], Ma[ip * pa + q]);
        dst[e] = acc;
    }
}

// ------------------------------------------------------------------ leaf fill
template <int NP>
__global__ void __launch_bounds__(kLeafThreads)
leaf_fill_kernel(LevelDev L, PointsDev P, const double2* __restrict__ a_p, double k, Pipes pp,
                 const double* __restrict__ Ms, const double* __restrict__ Ma,
                 double2* __restrict__ store) {
    extern __shared__ double smem[];
    const int b = blockIdx.x;
    const int s0 = L.box_seg_begin[b], s1 = L.box_seg_begin[b + 1];
    if (s0 == s1) return;
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
                    sincos(arg, &sn, &cs);
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
    const int c = blockIdx.x;
    const int tb = L.chunk_box[c];
    const int tbeg = int(L.beg[tb]);
    const int n_t = int(L.end[tb]) - tbeg;
    const int q = L.chunk_q0[c] + threadIdx.x;
    if (q >= n_t) return;
    const int t = tbeg + q;
    const double x = P.x[t], y = P.y[t], z = P.z[t];
    const int ps = L.ps, pa = L.pang;
    const int NPTS = ps * pa * pa;
    const double h = L.h;
    const int j0 = L.cz_ptr[tb], j1 = L.cz_ptr[tb + 1];
    const std::int64_t ev0 = L.cev_begin[tb] + q;
    double2 accS = make_double2(0.0, 0.0), accD = make_double2(0.0, 0.0);
    double ts[PS > 0 ? PS : kMaxOrd], tt[PA > 0 ? PA : kMaxOrd], tp[PA > 0 ? PA : kMaxOrd];
    for (int j = j0; j < j1; ++j) {
        const int sb = L.cz_idx[j];
        const int so = L.cev_seg[ev0 + std::int64_t(j - j0) * n_t];
        const double vx = x - L.cx[sb], vy = y - L.cy[sb], vz = z - L.cz[sb];
        const double r2 = fma(vx, vx, fma(vy, vy, vz * vz));
        const double inv_r = rsqrt(r2);
        const double r = r2 * inv_r;
        const LocalCoords lc = local_coords(vx, vy, vz, inv_r, h, L.seg_gamma[so], L);
        basis3<PS, PA>(lc, ts, tt, tp, ps, pa);
        double sn, cs;
        sincos(k * r, &sn, &cs);
        const double f1 = kInv4PiD * inv_r;
        const double2 e1 = make_double2(cs * f1, sn * f1);  // e^{ikr}/(4 pi r)
        const double2* blk = store + std::size_t(so) * NP * NPTS;
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const double2 val = eval_series<PS, PA>(blk + i * NPTS, ts, tt, tp, ps, pa);
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
    }
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
    const int G = max(1, int(blockDim.x) / NPTS);
    const int g0 = blockIdx.x * G;
    if (g0 >= Lp.nseg) return;
    const int gcount = min(G, Lp.nseg - g0);
    const int items = gcount * NPTS;
    double2* v0 = reinterpret_cast<double2*>(smem);
    double2* v1 = v0 + G * NPP * NPTS;
    const double hp = Lp.h, hc = Lc.h;
    double ts[PS > 0 ? PS : kMaxOrd], tt[PA > 0 ? PA : kMaxOrd], tp[PA > 0 ? PA : kMaxOrd];

    for (int base = 0; base < items; base += blockDim.x) {
        const int item = base + threadIdx.x;
        if (item >= items) continue;
        const int seg_l = item / NPTS, node = item % NPTS;
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
        const int c0 = Lp.ch_ptr[pb], nch = Lp.ch_ptr[pb + 1] - c0;
        const std::int64_t ev = Lc.pev_begin[so] + std::int64_t(node) * nch;
        double2 acc[NPP];
#pragma unroll
        for (int i = 0; i < NPP; ++i) acc[i] = make_double2(0.0, 0.0);
        for (int c = 0; c < nch; ++c) {
            const int ch = Lp.ch_idx[c0 + c];
            const int cso = Lc.pev_seg[ev + c];
            const double ccx = Lc.cx[ch], ccy = Lc.cy[ch], ccz = Lc.cz[ch];
            const double vx = x - ccx, vy = y - ccy, vz = z - ccz;
            const double rc2 = fma(vx, vx, fma(vy, vy, vz * vz));
            const double inv_rc = rsqrt(rc2);
            const double rc = rc2 * inv_rc;
            const LocalCoords lc = local_coords(vx, vy, vz, inv_rc, hc, Lc.seg_gamma[cso], Lc);
            basis3<PS, PA>(lc, ts, tt, tp, cps, cpa);
            // stable r_c - r_p (ifgf.cpp:149-153)
            const double sx = ccx + pcx - 2.0 * x, sy = ccy + pcy - 2.0 * y, sz = ccz + pcz - 2.0 * z;
            const double dr = fma(sx, ccx - pcx, fma(sy, ccy - pcy, sz * (ccz - pcz))) / (rc + rp);
            double sn, cs;
            sincos(k * dr, &sn, &cs);
            const double q1 = rp * inv_rc;
            const double2 ratio1 = make_double2(cs * q1, sn * q1);
            const double2* blk = cstore + std::size_t(cso) * NPC * CPTS;
            double2 val[NPC];
#pragma unroll
            for (int i = 0; i < NPC; ++i) val[i] = eval_series<PS, PA>(blk + i * CPTS, ts, tt, tp, cps, cpa);
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
        }
#pragma unroll
        for (int i = 0; i < NPP; ++i) v0[(seg_l * NPP + i) * NPTS + node] = acc[i];
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
    const bool def = L.ps == 3 && L.pang == 5;
    auto go = [&](auto kern) { kern<<<L.nchunk, kCousinThreads, 0, st>>>(L, P, store, k, pipes, Sp, Dp); };
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
    const std::size_t smem = 2 * std::size_t(G) * parent_pipes.n * NPTS * sizeof(double2);
    const int grid = div_up(Lp.nseg, G);
    const bool def = Lp.ps == 3 && Lp.pang == 5 && Lc.ps == 3 && Lc.pang == 5;
    auto go = [&](auto kern) {
        IFGF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<grid, kParentThreads, smem, st>>>(Lp, Lc, child_store, k, parent_pipes, cm, Ms, Ma, parent_store);
    };
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
