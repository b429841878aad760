// Cell-batched parent fill (ifgf.cpp:452-568) on the FP64 tensor cores.
//
// The position of a parent interpolation node in a child frame depends only on (parent cone
// cell, child octant, node) (host/coneplan.hpp parent_templates), and so does the child cone
// cell it falls in. All parent segments of ONE cone cell therefore interpolate their
// children's coefficient blocks with the SAME real matrix: row = node, column k = the 75
// products T_is(s) T_it(theta) T_ip(phi) of its local coordinates. A CTA takes up to
// kCbSegs (12) parent segments of one cell (an "item", built on the host) and, per child
// octant and per child-cell group of nodes, runs one small GEMM on mma.sync.m8n8k4.f64:
//
//   C (group nodes x [segment, child pipe, re/im]) = A (group nodes x 76) * B (76 x ...),
//
// A built once per octant in shared memory from the template entries, B = the children's
// coefficient blocks staged by cp.async into shared memory (double-buffered: the next
// group's blocks load while this group multiplies), 2x2 tiles of 8x8 per warp (4
// independent accumulator chains, one A and one B fragment load per two DMMAs). The
// epilogue multiplies each (node, child pipe) by its re-centring factor and adds into
// per-(segment, node, child pipe) accumulators in shared memory; each entry has one writer
// per group, and groups run in a fixed order, so results are bitwise reproducible.
// Evaluations whose host-decided child segment differs from the template's group (ties) are
// masked out of the GEMM and evaluated one by one (exceptions). Finally the child pipes are
// summed into the parent pipes and transform3 (ifgf.cpp:560-562) writes the blocks.
#include "ifgf_device.cuh"
#include "kernels.cuh"
#include "parent_common.cuh"
#include "tc_common.cuh"

namespace ifgfb200 {
namespace {

using namespace dev;
using namespace ifgfdev;
using namespace pfill;

constexpr int kW = 8;                  // warps per CTA
constexpr int kNP = 75, kK = 76;       // coefficients per pipe block; k padded to 19 steps of 4
constexpr int kKS = kK / 4;
constexpr int kMB = kCbSegs;
constexpr int kG = kCbMaxGrp;
constexpr int kCheb = 976;             // 75 rows x 13 basis values (+1: keeps B 16-byte aligned)

// staged block layout in shared memory: pipe stride SP, block stride SB (doubles), chosen
// so that an 8x4 B fragment load takes the minimum two wavefronts
template <int NPC>
struct Stage;
template <>
struct Stage<1> {
    static constexpr int SP = 150, SB = 152;
};
template <>
struct Stage<2> {
    static constexpr int SP = 150, SB = 312;
};
template <>
struct Stage<3> {
    static constexpr int SP = 152, SB = 456;
};

template <int NPC>
constexpr std::size_t cb_smem_bytes() {
    return std::size_t(kMB) * kNP * NPC * 16 + std::size_t(kNP) * kK * 8 + std::size_t(kNP) * NPC * 16 +
           std::size_t(kCheb) * 8 + 2 * std::size_t(kMB) * Stage<NPC>::SB * 8 + 2 * (kMB + 1) * 4 + kMB * kNP;
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    const unsigned s = unsigned(__cvta_generic_to_shared(sdst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <int COMBO>
__device__ __forceinline__ double2 child_factor(int p, double r1x, double r1y, double xf, double k) {
    using CB = Combo<COMBO>;
    const int f = CB::fac(p);
    if (f == MK) return make_double2(k * r1y, -k * r1x);  // -ik ratio1
    if (f == R1) return make_double2(r1x, r1y);
    return make_double2(r1x * xf, r1y * xf);              // RI (1/r_c) or RQ (r_p/r_c)
}

template <int COMBO>
__global__ void __launch_bounds__(32 * kW, 1)
parent_cb_kernel(LevelDev Lp, LevelDev Lc, const double2* __restrict__ cstore, double k,
                 const double* __restrict__ Ms, const double* __restrict__ Ma, double2* __restrict__ pstore) {
    using CB = Combo<COMBO>;
    constexpr int NPP = CB::npp, NPC = CB::npc;
    constexpr int SP = Stage<NPC>::SP, SB = Stage<NPC>::SB;
    constexpr int NCOL = 2 * NPC;  // B columns per staged block: (child pipe, re/im)
    extern __shared__ __align__(16) double smem[];
    double2* acc = reinterpret_cast<double2*>(smem);                    // [j][node][child pipe]
    double* A = smem + 2 * kMB * kNP * NPC;                              // [row][kK]
    double2* fac = reinterpret_cast<double2*>(A + kNP * kK);             // [row][child pipe]
    double* cheb = reinterpret_cast<double*>(fac + kNP * NPC);           // [row][13]
    double* Bs = cheb + kCheb;                                           // 2 x [kMB][SB]
    int* blist = reinterpret_cast<int*>(Bs + 2 * kMB * SB);              // 2 x (kMB + 1)
    unsigned char* mask = reinterpret_cast<unsigned char*>(blist + 2 * (kMB + 1));  // [j][node]
    __shared__ int segs_s[kMB];
    __shared__ unsigned char use_s[kMB * 8];
    __shared__ unsigned char nodes_s[kNP];
    __shared__ int steps_s[8 * kG];
    __shared__ int nsteps_s;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = lane >> 2, tig = lane & 3;
    const int item = blockIdx.x;
    const int slot = Lc.cb_item_slot[item];
    const std::int32_t* __restrict__ iseg = Lc.cb_item_seg + std::size_t(item) * kMB;

    if (tid < kMB) {
        int s = iseg[tid];
        if (s >= 0 && Lp.active && !Lp.active[Lp.seg_box[s]]) s = -1;  // no sources of this rank below
        segs_s[tid] = s;
    }
    for (int i = tid; i < kMB * kNP * NPC; i += 32 * kW) acc[i] = make_double2(0.0, 0.0);
    for (int i = tid; i < 2 * kMB * SB; i += 32 * kW) Bs[i] = 0.0;  // padding read as k = 75 stays 0
    __syncthreads();
    if (tid < kMB * 8) {
        const int j = tid >> 3, o = tid & 7;
        bool u = false;
        if (segs_s[j] >= 0) {
            const int ch = Lc.cb_child[(std::size_t(item) * kMB + j) * 8 + o];
            u = ch >= 0 && !(Lc.active && !Lc.active[ch]);
        }
        use_s[tid] = u ? 1 : 0;
    }
    __syncthreads();
    if (tid == 0) {
        int ns = 0;
        for (int o = 0; o < 8; ++o) {
            bool any = false;
            for (int j = 0; j < kMB; ++j) any = any || use_s[j * 8 + o];
            if (!any) continue;
            const int ng = Lc.cb_ngrp[slot * 8 + o];
            for (int g = 0; g < ng; ++g) steps_s[ns++] = (o << 8) | g;
        }
        nsteps_s = ns;
    }
    __syncthreads();
    const int nsteps = nsteps_s;

    // stage step s's child blocks into buffer buf (every warp derives the same list)
    auto stage = [&](int s, int buf) {
        const int o = steps_s[s] >> 8, g = steps_s[s] & 0xff;
        int cso = -1;
        if (lane < kMB && use_s[lane * 8 + o]) cso = Lc.cb_cso[((std::size_t(item) * kMB + lane) * 8 + o) * kG + g];
        const unsigned bal = __ballot_sync(0xffffffffu, cso >= 0);
        const int m = __popc(bal);
        if (warp == 0) {
            if (cso >= 0) blist[buf * (kMB + 1) + __popc(bal & ((1u << lane) - 1u))] = lane;
            if (lane == 0) blist[buf * (kMB + 1) + kMB] = m;
        }
        double* dstb = Bs + buf * kMB * SB;
        const int total = m * NPC * kNP;
        for (int c0 = warp * 32; c0 < total; c0 += 32 * kW) {  // warp-uniform trip count (shuffles)
            const int c = c0 + lane;
            const bool live = c < total;
            const int jj = live ? c / (NPC * kNP) : 0, rem = c - jj * (NPC * kNP);
            const int p = rem / kNP, kk = rem - p * kNP;
            // lane of the (jj + 1)-th listed segment
            unsigned rest = bal;
            for (int q = 0; q < jj; ++q) rest &= rest - 1u;
            const int cs = __shfl_sync(0xffffffffu, cso, __ffs(rest) - 1);
            if (live) cp_async16(dstb + jj * SB + p * SP + 2 * kk, cstore + std::size_t(cs) * NPC * kNP + p * kNP + kk);
        }
        cp_async_commit();
    };

    // this lane's three k columns of the A rows: (is, it, ip) of k = lane, lane + 32, lane + 64
    int kis[3], kit[3], kip[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const int kk = min(lane + 32 * q, kNP - 1);
        kis[q] = kk % 3;
        kit[q] = 3 + (kk / 3) % 5;
        kip[q] = 8 + kk / 15;
    }
    if (nsteps > 0) stage(0, 0);
    int o_cur = -1;
    for (int s = 0; s < nsteps; ++s) {
        const int o = steps_s[s] >> 8, g = steps_s[s] & 0xff, buf = s & 1;
        if (o != o_cur) {  // A rows, factors and exception mask of octant o
            if (o_cur >= 0) __syncthreads();  // the previous octant's multiplications read A
            o_cur = o;
            const std::size_t so8 = std::size_t(slot) * 8 + o;
            if (tid < kNP) {
                const int node = Lc.cb_nodes[so8 * kNP + tid];
                nodes_s[tid] = (unsigned char)node;
                const double* te = Lp.tmpl + (so8 * kNP + node) * kTmplDoubles;
                const double2 t0 = __ldg(reinterpret_cast<const double2*>(te));
                const double2 t1 = __ldg(reinterpret_cast<const double2*>(te) + 1);
                const double2 t2 = __ldg(reinterpret_cast<const double2*>(te) + 2);
                double* cr = cheb + tid * 13;
                cheb_row<3>(t0.x, cr);
                cheb_row<5>(t0.y, cr + 3);
                cheb_row<5>(t1.x, cr + 8);
                double xf = t2.y;  // 1/r_c
                if (CB::extra == RQ) {  // r_p/r_c = (h_p / s) (1/r_c), s of the cell's radial node
                    const int gam = Lp.seg_gamma[Lc.cb_item_seg[std::size_t(item) * kMB]];
                    xf *= Lp.h / Lp.s_nodes[(gam % Lp.ns) * 3 + node % 3];
                }
#pragma unroll
                for (int p = 0; p < NPC; ++p) fac[tid * NPC + p] = child_factor<COMBO>(p, t1.y, t2.x, xf, k);
            }
            for (int i = tid; i < kMB * kNP; i += 32 * kW) mask[i] = 0;
            __syncthreads();
            for (int row = warp; row < kNP; row += kW) {
                const double* cr = cheb + row * 13;
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const int kk = lane + 32 * q;
                    if (kk < kK) A[row * kK + kk] = kk < kNP ? cr[kis[q]] * cr[kit[q]] * cr[kip[q]] : 0.0;
                }
            }
            const std::int64_t e0 = Lc.cb_exc_begin[item], e1 = Lc.cb_exc_begin[item + 1];
            for (std::int64_t e = e0 + tid; e < e1; e += 32 * kW) {
                const unsigned key = Lc.cb_exc_key[e];
                if (int((key >> 8) & 0xffu) == o) mask[(key & 0xffu) * kNP + (key >> 16)] = 1;
            }
        }
        cp_async_wait_all();
        __syncthreads();
        if (s + 1 < nsteps) stage(s + 1, buf ^ 1);  // overlaps this step's multiplications

        const std::size_t so8 = std::size_t(slot) * 8 + o;
        const int gs = Lc.cb_gstart[so8 * (kG + 1) + g], ge = Lc.cb_gstart[so8 * (kG + 1) + g + 1];
        const int m = blist[buf * (kMB + 1) + kMB];
        const int* bl = blist + buf * (kMB + 1);
        const double* Bb = Bs + buf * kMB * SB;
        const int mt = (ge - gs + 7) >> 3, nt = (NCOL * m + 7) >> 3;
        const int mp = (mt + 1) >> 1, np = (nt + 1) >> 1;
        for (int u = warp; u < mp * np; u += kW) {
            const int mt0 = 2 * (u / np), nt0 = 2 * (u % np);
            const double* a0p = A + min(gs + mt0 * 8 + r, kNP - 1) * kK + tig;
            const double* a1p = A + min(gs + mt0 * 8 + 8 + r, kNP - 1) * kK + tig;
            auto bcol = [&](int col) {
                col = min(col, NCOL * kMB - 1);
                return Bb + (col / NCOL) * SB + ((col % NCOL) >> 1) * SP + (col & 1) + 2 * tig;
            };
            const double* b0p = bcol(nt0 * 8 + r);
            const double* b1p = bcol(nt0 * 8 + 8 + r);
            double d[2][2][2] = {};
            const bool m1 = mt0 + 1 < mt, n1 = nt0 + 1 < nt;  // warp-uniform: skip absent tiles
            if (m1 && n1) {
#pragma unroll
                for (int ks = 0; ks < kKS; ++ks) {
                    const double a0 = a0p[4 * ks], a1 = a1p[4 * ks];
                    const double b0 = b0p[8 * ks], b1 = b1p[8 * ks];
                    tc::dmma884(d[0][0][0], d[0][0][1], a0, b0);
                    tc::dmma884(d[0][1][0], d[0][1][1], a0, b1);
                    tc::dmma884(d[1][0][0], d[1][0][1], a1, b0);
                    tc::dmma884(d[1][1][0], d[1][1][1], a1, b1);
                }
            } else if (n1) {
#pragma unroll
                for (int ks = 0; ks < kKS; ++ks) {
                    const double a0 = a0p[4 * ks];
                    const double b0 = b0p[8 * ks], b1 = b1p[8 * ks];
                    tc::dmma884(d[0][0][0], d[0][0][1], a0, b0);
                    tc::dmma884(d[0][1][0], d[0][1][1], a0, b1);
                }
            } else if (m1) {
#pragma unroll
                for (int ks = 0; ks < kKS; ++ks) {
                    const double a0 = a0p[4 * ks], a1 = a1p[4 * ks];
                    const double b0 = b0p[8 * ks];
                    tc::dmma884(d[0][0][0], d[0][0][1], a0, b0);
                    tc::dmma884(d[1][0][0], d[1][0][1], a1, b0);
                }
            } else {
#pragma unroll
                for (int ks = 0; ks < kKS; ++ks) tc::dmma884(d[0][0][0], d[0][0][1], a0p[4 * ks], b0p[8 * ks]);
            }
#pragma unroll
            for (int im = 0; im < 2; ++im)
#pragma unroll
                for (int in = 0; in < 2; ++in) {
                    const int row = gs + (mt0 + im) * 8 + r;
                    const int c = (nt0 + in) * 8 + 2 * tig;
                    const int jj = c / NCOL, p = (c % NCOL) >> 1;
                    if (mt0 + im < mt && nt0 + in < nt && row < ge && jj < m) {
                        const int j = bl[jj], node = nodes_s[row];
                        if (!mask[j * kNP + node]) {
                            double2& a = acc[(j * kNP + node) * NPC + p];
                            a = cadd(a, cmul(fac[row * NPC + p], make_double2(d[im][in][0], d[im][in][1])));
                        }
                    }
                }
        }
        // no barrier here: the next step's top barrier orders its B / accumulator use after
        // this one, and an octant change waits before rebuilding A
    }
    __syncthreads();

    // exceptions: one thread, in list order (rare; each may share an accumulator with another)
    if (tid == 0) {
        const std::int64_t e0 = Lc.cb_exc_begin[item], e1 = Lc.cb_exc_begin[item + 1];
        const double hp = Lp.h, hc = Lc.h;
        for (std::int64_t e = e0; e < e1; ++e) {
            const unsigned key = Lc.cb_exc_key[e];
            const int j = int(key & 0xffu), o = int((key >> 8) & 0xffu), node = int(key >> 16);
            const int seg = segs_s[j];
            if (seg < 0 || !use_s[j * 8 + o]) continue;
            const int cso = Lc.cb_exc_cso[e];
            const int ch = Lc.cb_child[(std::size_t(item) * kMB + j) * 8 + o];
            const int pb = Lp.seg_box[seg], gam = Lp.seg_gamma[seg];
            const int g1 = gam % Lp.ns, g2 = (gam / Lp.ns) % Lp.nc, g3 = gam / Lp.ns / Lp.nc;
            const int is = node % 3, it = (node / 3) % 5, ip = node / 15;
            const double pcx = Lp.cx[pb], pcy = Lp.cy[pb], pcz = Lp.cz[pb];
            const double ccx = Lc.cx[ch], ccy = Lc.cy[ch], ccz = Lc.cz[ch];
            const double sv = Lp.s_nodes[g1 * 3 + is];
            const double rp = hp / sv;
            const double sth = Lp.th_sin[g2 * 5 + it], cth = Lp.th_cos[g2 * 5 + it];
            const double sph = Lp.ph_sin[g3 * 5 + ip], cph = Lp.ph_cos[g3 * 5 + ip];
            const double x = pcx + rp * sth * cph, y = pcy + rp * sth * sph, z = pcz + rp * cth;
            const double vx = x - ccx, vy = y - ccy, vz = z - ccz;
            const double rc2 = fma(vx, vx, fma(vy, vy, vz * vz));
            const double inv_rc = rsqrt(rc2);
            const double rc = rc2 * inv_rc;
            const CellFrame cf = Lc.seg_code ? cell_frame_code(Lc.seg_code[cso], Lc) : cell_frame(Lc.seg_gamma[cso], Lc);
            const LocalCoords lc = local_coords_in(vx, vy, vz, inv_rc, hc, cf, Lc);
            const double sx = ccx + pcx - 2.0 * x, sy = ccy + pcy - 2.0 * y, sz = ccz + pcz - 2.0 * z;
            const double dr = fma(sx, ccx - pcx, fma(sy, ccy - pcy, sz * (ccz - pcz))) / (rc + rp);
            double sn, cs;
            sincos_bounded(k * dr, &sn, &cs);
            const double q1 = rp * inv_rc;
            const double xf = CB::extra == RI ? inv_rc : q1;
            double ts[3], tt[5], tp[5];
            cheb_row<3>(lc.ls, ts);
            cheb_row<5>(lc.lt, tt);
            cheb_row<5>(lc.lp, tp);
            const double2* blk = cstore + std::size_t(cso) * NPC * kNP;
            for (int p = 0; p < NPC; ++p) {
                double2 v = make_double2(0.0, 0.0);
                for (int kk = 0; kk < kNP; ++kk) cfma_r(v, blk[p * kNP + kk], ts[kk % 3] * tt[(kk / 3) % 5] * tp[kk / 15]);
                double2& a = acc[(j * kNP + node) * NPC + p];
                a = cadd(a, cmul(child_factor<COMBO>(p, cs * q1, sn * q1, xf, k), v));
            }
        }
    }
    __syncthreads();

    // child pipes -> parent pipes, then values -> coefficients (transform3), warp per segment
    double2* v0 = reinterpret_cast<double2*>(Bs) + warp * 2 * NPP * kNP;
    double2* v1 = v0 + NPP * kNP;
    for (int j = warp; j < kMB; j += kW) {
        const int seg = segs_s[j];
        if (seg < 0) continue;
        for (int e = lane; e < NPP * kNP; e += 32) {
            const int node = e / NPP, pp = e % NPP;
            double2 a = make_double2(0.0, 0.0);
#pragma unroll
            for (int p = 0; p < NPC; ++p)
                if (CB::dst(p) == pp) a = cadd(a, acc[(j * kNP + node) * NPC + p]);
            v0[e] = a;
        }
        __syncwarp();
        double2* dst = pstore + std::size_t(seg) * NPP * kNP;
        for (int e = lane; e < NPP * kNP; e += 32) {
            const int blk = e / kNP, node = e % kNP;
            const int is = node % 3, line = node / 3;
            double2 a = make_double2(0.0, 0.0);
            for (int q = 0; q < 3; ++q) cfma_r(a, v0[(line * 3 + q) * NPP + blk], Ms[is * 3 + q]);
            v1[e] = a;
        }
        __syncwarp();
        for (int e = lane; e < NPP * kNP; e += 32) {
            const int blk = e / kNP, node = e % kNP;
            const int is = node % 3, it = (node / 3) % 5, ip = node / 15;
            const double2* src = v1 + blk * kNP + is + 15 * ip;
            double2 a = make_double2(0.0, 0.0);
            for (int q = 0; q < 5; ++q) cfma_r(a, src[3 * q], Ma[it * 5 + q]);
            v0[e] = a;
        }
        __syncwarp();
        for (int e = lane; e < NPP * kNP; e += 32) {
            const int blk = e / kNP, node = e % kNP;
            const int is = node % 3, it = (node / 3) % 5, ip = node / 15;
            const double2* src = v0 + blk * kNP + is + 3 * it;
            double2 a = make_double2(0.0, 0.0);
            for (int q = 0; q < 5; ++q) cfma_r(a, src[15 * q], Ma[ip * 5 + q]);
            dst[e] = a;
        }
        __syncwarp();
    }
}

}  // namespace

bool launch_parent_fill_cb(const LevelDev& Lp, const LevelDev& Lc, const double2* child_store, double k,
                           const Pipes& parent_pipes, const Pipes& child_pipes, const double* Ms, const double* Ma,
                           double2* parent_store, cudaStream_t st) {
    if (Lc.n_cbitem == 0 || !Lp.tmpl) return false;
    const int combo = combo_of(parent_pipes, child_pipes);
    if (combo < 0) return false;
    auto go = [&](auto kern, std::size_t smem) {
        IFGF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<Lc.n_cbitem, 32 * kW, smem, st>>>(Lp, Lc, child_store, k, Ms, Ma, parent_store);
    };
    switch (combo) {
        case 0: go(parent_cb_kernel<0>, cb_smem_bytes<Combo<0>::npc>()); break;
        case 1: go(parent_cb_kernel<1>, cb_smem_bytes<Combo<1>::npc>()); break;
        case 2: go(parent_cb_kernel<2>, cb_smem_bytes<Combo<2>::npc>()); break;
        case 3: go(parent_cb_kernel<3>, cb_smem_bytes<Combo<3>::npc>()); break;
        case 4: go(parent_cb_kernel<4>, cb_smem_bytes<Combo<4>::npc>()); break;
        default: go(parent_cb_kernel<5>, cb_smem_bytes<Combo<5>::npc>()); break;
    }
    IFGF_CUDA(cudaGetLastError());
    return true;
}

}  // namespace ifgfb200
