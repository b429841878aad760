// Device helpers shared by the IFGF kernels (cone coordinates, Chebyshev series
// evaluation, warp-cooperative block staging, separable block transform).
#pragma once

#include "dev_common.cuh"
#include "device_plan.cuh"

namespace ifgfb200 {
namespace ifgfdev {

using namespace dev;

constexpr int kMaxOrd = 12;

struct LocalCoords {
    double ls, lt, lp;
};

// Cone coordinates of v = x - centre (inv_r = 1/|v|) relative to the host-decided segment
// gamma, mapped to [-1,1]^3 (LevelCones::local_coords, ifgf.cpp:178-183).
__device__ __forceinline__ LocalCoords local_coords_lib(double vx, double vy, double vz, double inv_r,
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

// atan(t) for |t| <= 0.4225 (cells of at most pi/4: nc >= 4): t * P(t^2), degree-11
// least-squares fit (max abs error 6e-17 on the interval)
__device__ __forceinline__ double atan_small(double t) {
    const double u = t * t;
    double p = -0.01723604573229859;
    p = fma(p, u, 0.03744269623222812);
    p = fma(p, u, -0.05014437831961434);
    p = fma(p, u, 0.05842271768042808);
    p = fma(p, u, -0.06662315934685337);
    p = fma(p, u, 0.07691989116146059);
    p = fma(p, u, -0.09090893628137384);
    p = fma(p, u, 0.11111110633111605);
    p = fma(p, u, -0.14285714276966102);
    p = fma(p, u, 0.1999999999991704);
    p = fma(p, u, -0.33333333333333026);
    p = fma(p, u, 1.0);
    return t * p;
}

// host-decided cell of a segment, decoded once (and its centre directions when tabulated)
struct CellFrame {
    int g1, g2, g3;
    double ctc, stc, cpc, spc;
};
__device__ __forceinline__ CellFrame cell_frame(int gamma, const LevelDev& L) {
    CellFrame f;
    f.g1 = gamma % L.ns;
    const int rest = gamma / L.ns;
    f.g2 = rest % L.nc;
    f.g3 = rest / L.nc;
    if (L.thc_cos) {
        f.ctc = L.thc_cos[f.g2];
        f.stc = L.thc_sin[f.g2];
        f.cpc = L.phc_cos[f.g3];
        f.spc = L.phc_sin[f.g3];
    } else {
        f.ctc = f.stc = f.cpc = f.spc = 0.0;
    }
    return f;
}

// the same frame from a packed cell code (LevelDev::seg_code layout)
__device__ __forceinline__ CellFrame cell_frame_code(unsigned code, const LevelDev& L) {
    CellFrame f;
    f.g1 = int(code & 0xffu);
    f.g2 = int((code >> 8) & 0x7ffu);
    f.g3 = int(code >> 19);
    if (L.thc_cos) {
        f.ctc = L.thc_cos[f.g2];
        f.stc = L.thc_sin[f.g2];
        f.cpc = L.phc_cos[f.g3];
        f.spc = L.phc_sin[f.g3];
    } else {
        f.ctc = f.stc = f.cpc = f.spc = 0.0;
    }
    return f;
}

// local coordinates inside a decoded cell (see local_coords below)
__device__ __forceinline__ LocalCoords local_coords_in(double vx, double vy, double vz, double inv_r, double h,
                                                       const CellFrame& f, const LevelDev& L) {
    const int gamma = f.g1 + L.ns * (f.g2 + L.nc * f.g3);
    if (!L.thc_cos) return local_coords_lib(vx, vy, vz, inv_r, h, gamma, L);
    const double rho = sqrt_nonneg(fma(vx, vx, vy * vy));
    const double tn = fma(rho, f.ctc, -vz * f.stc), td = fma(vz, f.ctc, rho * f.stc);
    const double pn = fma(vy, f.cpc, -vx * f.spc), pd = fma(vx, f.cpc, vy * f.spc);
    const double inv = rcp_normal(td * pd);  // one division for both tangents (td, pd > 0 checked below)
    const double tt = tn * pd * inv, tp = pn * td * inv;
    if (!(fabs(tt) <= 0.4225 && fabs(tp) <= 0.4225 && td > 0.0 && pd > 0.0))
        return local_coords_lib(vx, vy, vz, inv_r, h, gamma, L);
    LocalCoords o;
    o.ls = fma(h * inv_r, 2.0 * L.inv_ds, -(2 * f.g1 + 1.0));
    o.lt = atan_small(tt) * (2.0 * L.inv_dth);
    o.lp = atan_small(tp) * (2.0 * L.inv_dph);
    return o;
}

// Same map without acos/atan2: the angles are taken relative to the centre of the
// host-decided cell, theta - theta_c = atan((rho cos th_c - vz sin th_c) / (vz cos th_c +
// rho sin th_c)) and likewise for phi (no 0/2pi seam at all), both inside +-pi/(2 nc).
// Falls back to local_coords_lib if a point lies unexpectedly far outside its cell.
__device__ __forceinline__ LocalCoords local_coords(double vx, double vy, double vz, double inv_r,
                                                    double h, int gamma, const LevelDev& L) {
    if (!L.thc_cos) return local_coords_lib(vx, vy, vz, inv_r, h, gamma, L);
    const int g1 = gamma % L.ns;
    const int rest = gamma / L.ns;
    const int g2 = rest % L.nc;
    const int g3 = rest / L.nc;
    const double rho = sqrt_nonneg(fma(vx, vx, vy * vy));
    const double ctc = L.thc_cos[g2], stc = L.thc_sin[g2];
    const double cpc = L.phc_cos[g3], spc = L.phc_sin[g3];
    const double tn = fma(rho, ctc, -vz * stc), td = fma(vz, ctc, rho * stc);
    const double pn = fma(vy, cpc, -vx * spc), pd = fma(vx, cpc, vy * spc);
    const double inv = rcp_normal(td * pd);  // one division for both tangents (td, pd > 0 checked below)
    const double tt = tn * pd * inv, tp = pn * td * inv;
    if (!(fabs(tt) <= 0.4225 && fabs(tp) <= 0.4225 && td > 0.0 && pd > 0.0))
        return local_coords_lib(vx, vy, vz, inv_r, h, gamma, L);
    LocalCoords o;
    o.ls = fma(h * inv_r, 2.0 * L.inv_ds, -(2 * g1 + 1.0));
    o.lt = atan_small(tt) * (2.0 * L.inv_dth);
    o.lp = atan_small(tp) * (2.0 * L.inv_dph);
    return o;
}

// local_coords for the segment with ordinal so, its cell decoded from the packed code
__device__ __forceinline__ LocalCoords local_coords_seg(double vx, double vy, double vz, double inv_r, double h,
                                                        int so, const LevelDev& L) {
    if (!L.thc_cos || !L.seg_code) return local_coords(vx, vy, vz, inv_r, h, L.seg_gamma[so], L);
    const unsigned code = L.seg_code[so];
    const int g1 = int(code & 0xffu), g2 = int((code >> 8) & 0x7ffu), g3 = int(code >> 19);
    const double rho = sqrt_nonneg(fma(vx, vx, vy * vy));
    const double ctc = L.thc_cos[g2], stc = L.thc_sin[g2];
    const double cpc = L.phc_cos[g3], spc = L.phc_sin[g3];
    const double tn = fma(rho, ctc, -vz * stc), td = fma(vz, ctc, rho * stc);
    const double pn = fma(vy, cpc, -vx * spc), pd = fma(vx, cpc, vy * spc);
    const double inv = rcp_normal(td * pd);  // one division for both tangents (td, pd > 0 checked below)
    const double tt = tn * pd * inv, tp = pn * td * inv;
    if (!(fabs(tt) <= 0.4225 && fabs(tp) <= 0.4225 && td > 0.0 && pd > 0.0))
        return local_coords_lib(vx, vy, vz, inv_r, h, L.seg_gamma[so], L);
    LocalCoords o;
    o.ls = fma(h * inv_r, 2.0 * L.inv_ds, -(2 * g1 + 1.0));
    o.lt = atan_small(tt) * (2.0 * L.inv_dth);
    o.lp = atan_small(tp) * (2.0 * L.inv_dph);
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

// Warp-cooperative staging of coefficient blocks. Every lane names the block it needs
// (seg < 0: none); the warp copies each distinct block once, coalesced, into its own
// shared-memory slots (SLOTS per round) and runs fn(block) on the lanes whose block is
// resident. Replaces 75*NP broadcast global loads per lane-evaluation by ~75*NP/32
// coalesced loads plus shared-memory reads. Must be called by all 32 lanes.
template <int SLOTS, class F>
__device__ __forceinline__ void with_staged_block(int seg, const double2* __restrict__ store,
                                                  int blk_elems, double2* wbuf, F&& fn) {
    constexpr unsigned kFull = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned peers = __match_any_sync(kFull, seg);
    const int leader = __ffs(peers) - 1;
    const unsigned leaders = __ballot_sync(kFull, lane == leader);
    const int nd = __popc(leaders);
    const int myslot = __popc(leaders & ((1u << leader) - 1u));
    unsigned rem = leaders;
    for (int r0 = 0; r0 < nd; r0 += SLOTS) {
        for (int i = 0; i < SLOTS && r0 + i < nd; ++i) {
            const int ln = __ffs(rem) - 1;
            rem &= rem - 1u;
            const int sg = __shfl_sync(kFull, seg, ln);
            if (sg >= 0) {
                const double2* src = store + std::size_t(sg) * blk_elems;
                double2* dst = wbuf + i * blk_elems;
                for (int e = lane; e < blk_elems; e += 32) dst[e] = __ldg(src + e);
            }
        }
        __syncwarp();
        if (seg >= 0 && myslot >= r0 && myslot < r0 + SLOTS) fn(wbuf + (myslot - r0) * blk_elems);
        __syncwarp();
    }
}

// eval_series on a block resident in shared memory
template <int PS, int PA>
__device__ __forceinline__ double2 eval_series_sm(const double2* c, const double* ts, const double* tt,
                                                  const double* tp, int ps, int pa) {
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
                for (int is = 0; is < PS; ++is) cfma_r(a_s, line[is], ts[is]);
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
                for (int is = 0; is < ps; ++is) cfma_r(a_s, line[is], ts[is]);
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
__device__ inline void block_transform(double2* v0, double2* v1, int nblk, int ps, int pa,
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

// the same transform with compile-time orders, CTA-wide and line by line: each thread
// transforms whole lines (PS or PA values in, as many out) with the matrices in registers;
// the same terms in the same order as the element-wise form, so identical results
template <int PS, int PA>
__device__ inline void block_transform_c(double2* v0, double2* v1, int nblk, const double* __restrict__ Ms,
                                         const double* __restrict__ Ma, double2* __restrict__ dst) {
    constexpr int P = PS * PA * PA;
    double ms[PS * PS], ma[PA * PA];
#pragma unroll
    for (int i = 0; i < PS * PS; ++i) ms[i] = __ldg(Ms + i);
#pragma unroll
    for (int i = 0; i < PA * PA; ++i) ma[i] = __ldg(Ma + i);
    for (int l = threadIdx.x; l < nblk * PA * PA; l += blockDim.x) {  // along s: line (it, ip)
        const int blk = l / (PA * PA), line = l - blk * (PA * PA);
        const double2* src = v0 + blk * P + line * PS;
        double2 in[PS];
#pragma unroll
        for (int q = 0; q < PS; ++q) in[q] = src[q];
#pragma unroll
        for (int is = 0; is < PS; ++is) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < PS; ++q) cfma_r(acc, in[q], ms[is * PS + q]);
            v1[blk * P + line * PS + is] = acc;
        }
    }
    __syncthreads();
    for (int l = threadIdx.x; l < nblk * PS * PA; l += blockDim.x) {  // along theta: line (is, ip)
        const int blk = l / (PS * PA), rem = l - blk * (PS * PA), is = rem % PS, ip = rem / PS;
        const double2* src = v1 + blk * P + is + PS * PA * ip;
        double2 in[PA];
#pragma unroll
        for (int q = 0; q < PA; ++q) in[q] = src[PS * q];
#pragma unroll
        for (int it = 0; it < PA; ++it) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < PA; ++q) cfma_r(acc, in[q], ma[it * PA + q]);
            v0[blk * P + is + PS * it + PS * PA * ip] = acc;
        }
    }
    __syncthreads();
    for (int l = threadIdx.x; l < nblk * PS * PA; l += blockDim.x) {  // along phi: line (is, it)
        const int blk = l / (PS * PA), rem = l - blk * (PS * PA);  // rem = is + PS it
        const double2* src = v0 + blk * P + rem;
        double2 in[PA];
#pragma unroll
        for (int q = 0; q < PA; ++q) in[q] = src[PS * PA * q];
#pragma unroll
        for (int ip = 0; ip < PA; ++ip) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < PA; ++q) cfma_r(acc, in[q], ma[ip * PA + q]);
            dst[blk * P + rem + PS * PA * ip] = acc;
        }
    }
}

}  // namespace ifgfdev
}  // namespace ifgfb200
