// Cell-batched parent fill (ifgf.cpp:452-568) as GEMMs on the FP64 tensor cores.
//
// The position of a parent interpolation node in a child frame depends only on (parent cone
// cell, child octant, node) (host/coneplan.hpp parent_templates), and so does the child cone
// cell it falls in. All parent segments of ONE cone cell therefore interpolate their
// children's coefficient blocks with the SAME real matrix. Per (cell, octant) a setup kernel
// tabulates, with the nodes in child-cell group order (rows [gs, ge) = group g):
//   A2[row][16]  T_is(s) T_it(theta) in tc_common.cuh's k-slot order (15 pairs + a zero pad),
//   phw[row][ip] T_ip(phi), geo[row] the re-centring data (ratio1, 1/r_c) of the template.
// A CTA takes an item of kCbSegs (16) parent segments of one cell (host-sorted by their
// child-octant pattern); warp w owns segments 4w..4w+3 for all octants and computes, per
// octant o and group g present among them,
//
//   V[node, (segment, child pipe)] += f[node, pipe] * sum_ip phw[row, ip]
//                                      * A2[row, :] B_ip[:, (segment, pipe)]
//
// with B_ip the 15 coefficients of phi index ip of each child block: the phi weight is folded
// into the A fragment (one multiply), so the 5 x 4 k-steps (mma.sync.m8n8k4.f64) accumulate
// straight into up to 5 x NPC register tiles whose 8 columns are the 4 segments x {re, im}:
// a lane's D fragment is one complex (row, segment) value, and there is no gather epilogue.
// The child blocks stream through a per-warp 3-stage cp.async ring (one chunk = one ip,
// two chunks ahead, across groups and octants). Warps never wait for each other: the
// accumulators V[segment][node][parent pipe] are warp-private (one writer, fixed order, so
// bitwise reproducible). Evaluations whose host-decided child segment differs from the
// template's group (ties) are masked out and evaluated one by one (exceptions); transform3
// (ifgf.cpp:560-562) finishes each segment.
#include <cstdio>

#include "ifgf_device.cuh"
#include "kernels.cuh"
#include "parent_common.cuh"
#include "tc_common.cuh"

namespace ifgfb200 {
namespace {

using namespace dev;
using namespace ifgfdev;
using namespace pfill;

constexpr int kW = kCbSegs / 4;  // warps per CTA (4 segments each)
constexpr int kNP = 75;          // nodes / coefficients per pipe block
constexpr int kRows = kCbRows;   // table rows (75 + zero padding)
#ifndef IFGF_CB_STAGES3
#define IFGF_CB_STAGES3 3
#endif
#ifndef IFGF_CB_MINB3
#define IFGF_CB_MINB3 2
#endif
// cp.async ring depth per warp (prefetch distance = stages - 1)
template <int NPC>
constexpr int cb_stages() { return NPC == 3 ? IFGF_CB_STAGES3 : 3; }
constexpr int kMaxUnits = kCbMaxUnits;

template <int NPC>
struct Ring {
    static constexpr int SS = NPC * 32 + 8;  // doubles per segment (pipes x 16 complex + pad):
                                              // 4 segments' fragment loads take 2 wavefronts
    static constexpr int STAGE = 4 * SS;
};

// per warp: accumulators [4][75][NPP] complex, ring, unit list, exception bits [8][4][75]
template <int NPC, int NPP>
struct WarpSmem {
    static constexpr int ACC = 4 * kNP * NPP * 2;                 // doubles
    static constexpr int RING = cb_stages<NPC>() * Ring<NPC>::STAGE;  // doubles
    static constexpr int UNITS = kMaxUnits * 5;                   // ints
    static constexpr int EXC = (8 * 4 * kNP + 31) / 32;           // words
    static constexpr std::size_t bytes = (std::size_t(ACC + RING) * 8 + std::size_t(UNITS + EXC) * 4 + 15) / 16 * 16;
};

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    const unsigned s = unsigned(__cvta_generic_to_shared(sdst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int COMBO>
__device__ __forceinline__ double2 child_factor(int p, double r1x, double r1y, double xf, double k) {
    using CB = Combo<COMBO>;
    const int f = CB::fac(p);
    if (f == MK) return make_double2(k * r1y, -k * r1x);  // -ik ratio1
    if (f == R1) return make_double2(r1x, r1y);
    return make_double2(r1x * xf, r1y * xf);              // RI (1/r_c) or RQ (r_p/r_c)
}

#ifdef IFGF_CB_STATS
__device__ unsigned long long g_cb_stats[4];
#endif

template <int COMBO>
__global__ void __launch_bounds__(32 * kW, Combo<COMBO>::npc == 3 ? IFGF_CB_MINB3 : 3)
parent_cb_kernel(LevelDev Lp, LevelDev Lc, const double2* __restrict__ cstore, double k,
                 const double* __restrict__ Ms, const double* __restrict__ Ma, double2* __restrict__ pstore) {
    using CB = Combo<COMBO>;
    constexpr int NPP = CB::npp, NPC = CB::npc;
    using WS = WarpSmem<NPC, NPP>;
    constexpr int SS = Ring<NPC>::SS, STAGE = Ring<NPC>::STAGE;
    constexpr int kMT = kCbMaxTiles3 > kCbMaxTiles ? kCbMaxTiles3 : kCbMaxTiles;  // 8-row tiles per unit (host-split)
    constexpr int kStages = cb_stages<NPC>();
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r = lane >> 2, tig = lane & 3;
    char* wbase = reinterpret_cast<char*>(smem) + std::size_t(warp) * WS::bytes;
    double2* acc = reinterpret_cast<double2*>(wbase);                       // [c][node][pp]
    double* ring = reinterpret_cast<double*>(wbase) + WS::ACC;               // [stage][STAGE]
    int* units = reinterpret_cast<int*>(ring + WS::RING);                    // [unit][5]
    unsigned* excb = reinterpret_cast<unsigned*>(units + WS::UNITS);         // [o][c][node] bits

    const int item = blockIdx.x;
    const int slot = Lc.cb_item_slot[item];
    const std::int32_t* __restrict__ iseg = Lc.cb_item_seg + std::size_t(item) * kCbSegs + 4 * warp;

    for (int i = lane; i < WS::RING; i += 32) ring[i] = 0.0;  // pad slots (coefficient "75") stay 0
    for (int i = lane; i < WS::ACC / 2; i += 32) acc[i] = make_double2(0.0, 0.0);
    for (int i = lane; i < WS::EXC; i += 32) excb[i] = 0u;

    // ---- unit list of this warp (host-built, engine.cu "cell-batched parent items")
    const int c_l = lane & 3;
    int seg_l = iseg[c_l];
    if (seg_l >= 0 && Lp.active && !Lp.active[Lp.seg_box[seg_l]]) seg_l = -1;
    const int ub = Lc.cb_unit_begin[item * kW + warp];
    const int nu = Lc.cb_unit_begin[item * kW + warp + 1] - ub;
    for (int i = lane; i < nu * 5; i += 32) units[i] = Lc.cb_unit[std::size_t(ub) * 5 + i];
    if (Lp.active || Lc.active) {  // multi-GPU: children without sources of this rank drop out
        __syncwarp();
        for (int i = lane; i < nu * 4; i += 32) {
            const int u = i >> 2, c = i & 3, o = units[u * 5] >> 24;
            const int seg = iseg[c];
            bool ok = seg >= 0 && !(Lp.active && !Lp.active[Lp.seg_box[seg]]);
            if (ok) {
                const int ch = Lc.cb_child[(std::size_t(item) * kCbSegs + 4 * warp + c) * 8 + o];
                ok = ch >= 0 && !(Lc.active && !Lc.active[ch]);
            }
            if (!ok) units[u * 5 + 1 + c] = -1;
        }
    }
#ifdef IFGF_CB_STATS
    if (lane == 0) {
        unsigned long long smt = 0;
        for (int ui = 0; ui < nu; ++ui) smt += (units[ui * 5] >> 8) & 0xff;
        atomicAdd(&g_cb_stats[0], (unsigned long long)nu);
        atomicAdd(&g_cb_stats[1], smt);
    }
#endif
    // exception bits of this warp's segments
    const std::int64_t e0 = Lc.cb_exc_begin[item], e1 = Lc.cb_exc_begin[item + 1];
    for (std::int64_t e = e0 + lane; e < e1; e += 32) {
        const unsigned key = Lc.cb_exc_key[e];
        const int c = int(key & 0xffu) - 4 * warp, o = int((key >> 8) & 0xffu), node = int(key >> 16);
        if (c >= 0 && c < 4) {
            const int bit = (o * 4 + c) * kNP + node;
            atomicOr(excb + (bit >> 5), 1u << (bit & 31));
        }
    }
    __syncwarp();

    // ---- chunk stream: chunk q = (unit q / 5, ip = q % 5). Lanes 0..29 copy 16 bytes of
    // coefficient e = lane % 15 for the (segment, pipe) pairs half, half + 2, ... (a lane-
    // constant plan: destination offsets fixed, source pointers set once per unit)
    int doff[2 * NPC], cpair[2 * NPC], sofs[2 * NPC];
    {
        const int e = lane % 15, half = lane / 15;
#pragma unroll
        for (int i = 0; i < 2 * NPC; ++i) {
            const int pr = half + 2 * i, c = pr / NPC, p = pr - (pr / NPC) * NPC;
            doff[i] = c * SS + p * 32 + 2 * e;
            cpair[i] = c < 4 ? c : 0;
            sofs[i] = p * kNP + e;
        }
    }
    const double2* sp[2 * NPC];
    unsigned sval = 0u;
    int iss_u = 0, iss_ip = 0, iss_st = 0;
    auto issue = [&]() {
        if (iss_u < nu) {
            if (iss_ip == 0) {  // a new unit: its segments' block pointers
                const int* U = units + iss_u * 5;
                sval = 0u;
#pragma unroll
                for (int i = 0; i < 2 * NPC; ++i) {
                    const int cso = U[1 + cpair[i]];
                    sp[i] = cstore + std::size_t(cso < 0 ? 0 : cso) * NPC * kNP + sofs[i];
                    if (cso >= 0 && lane < 30) sval |= 1u << i;
                }
            }
            double* dst = ring + iss_st * STAGE;
#pragma unroll
            for (int i = 0; i < 2 * NPC; ++i)
                if ((sval >> i) & 1u) cp_async16(dst + doff[i], sp[i] + 15 * iss_ip);
            if (++iss_ip == 5) {
                iss_ip = 0;
                ++iss_u;
            }
        }
        cp_async_commit();  // (empty groups keep the wait counts uniform)
        iss_st = iss_st == kStages - 1 ? 0 : iss_st + 1;
    };
#pragma unroll
    for (int i = 0; i < kStages - 1; ++i) issue();

    const double* __restrict__ tab0 = Lc.cb_tab + std::size_t(slot) * 8 * kCbTab;
    const int gam0 = CB::extra == RQ ? Lp.seg_gamma[Lc.cb_item_seg[std::size_t(item) * kCbSegs]] : 0;
    const double hp = Lp.h;
    int cst = 0;  // ring stage of the chunk being consumed
    for (int ui = 0; ui < nu; ++ui) {
        const int* U = units + ui * 5;
        const int u0 = U[0];
        const int row0 = u0 & 0xff, mtu = (u0 >> 8) & 0xff, ge = (u0 >> 16) & 0xff, o = u0 >> 24;
        const double* __restrict__ tab = tab0 + std::size_t(o) * kCbTab;
        auto run = [&]<int MT>() {
            double d[MT][NPC][2];
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int p = 0; p < NPC; ++p) d[i][p][0] = d[i][p][1] = 0.0;
            int arow[MT];
#pragma unroll
            for (int i = 0; i < MT; ++i) arow[i] = min(row0 + 8 * i + r, kRows - 1);
            double a[MT][4];  // A2 fragments of the unit's tiles (the same for every ip)
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) a[i][j] = __ldg(tab + arow[i] * 16 + 4 * j + tig);
            double wn[MT];  // phi weights of the next ip, loaded one chunk ahead
#pragma unroll
            for (int i = 0; i < MT; ++i) wn[i] = __ldg(tab + kCbTabP + arow[i] * 8);
            for (int ip = 0; ip < 5; ++ip) {
                double w[MT];
#pragma unroll
                for (int i = 0; i < MT; ++i) {
                    w[i] = wn[i];
                    wn[i] = __ldg(tab + kCbTabP + arow[i] * 8 + (ip < 4 ? ip + 1 : 4));
                }
                cp_async_wait<kStages - 2>();  // chunk q landed (later ones may still be in flight)
                __syncwarp();
                issue();  // chunk q + kStages - 1
                const double* bch = ring + cst * STAGE + (r >> 1) * SS + (r & 1);
                cst = cst == kStages - 1 ? 0 : cst + 1;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int ci = tig < 3 ? tig + 3 * j : (j < 3 ? j + 12 : 15);
                    double b[NPC];
#pragma unroll
                    for (int p = 0; p < NPC; ++p) b[p] = bch[p * 32 + 2 * ci];
#pragma unroll
                    for (int i = 0; i < MT; ++i) {
                        const double av = a[i][j] * w[i];
#pragma unroll
                        for (int p = 0; p < NPC; ++p) tc::dmma884(d[i][p][0], d[i][p][1], av, b[p]);
                    }
                }
                __syncwarp();  // this ring stage is refilled by the issue of chunk q + kStages
            }
            // epilogue: lane (r, tig) holds (re, im) of rows row0 + 8 i + r for segment tig;
            // the rows' table entries are loaded for all tiles first (one latency)
            if (U[1 + tig] >= 0) {
                double4 gq[MT];
#pragma unroll
                for (int i = 0; i < MT; ++i) {
                    const double2* gp = reinterpret_cast<const double2*>(tab + kCbTabG) + 2 * arow[i];
                    const double2 g0 = __ldg(gp), g1 = __ldg(gp + 1);
                    gq[i] = make_double4(g0.x, g0.y, g1.x, g1.y);
                }
#pragma unroll
                for (int i = 0; i < MT; ++i) {
                    const int row = row0 + 8 * i + r;
                    const int node = int(gq[i].w);
                    const int bit = (o * 4 + tig) * kNP + node;
                    if (row < ge && !((excb[bit >> 5] >> (bit & 31)) & 1u)) {
                        double xf = gq[i].z;
                        if (CB::extra == RQ) xf *= hp / Lp.s_nodes[(gam0 % Lp.ns) * 3 + node % 3];
                        double2 v[NPP];
#pragma unroll
                        for (int pp = 0; pp < NPP; ++pp) v[pp] = make_double2(0.0, 0.0);
#pragma unroll
                        for (int p = 0; p < NPC; ++p) {
                            const double2 t = cmul(child_factor<COMBO>(p, gq[i].x, gq[i].y, xf, k),
                                                   make_double2(d[i][p][0], d[i][p][1]));
                            v[CB::dst(p)] = cadd(v[CB::dst(p)], t);
                        }
#pragma unroll
                        for (int pp = 0; pp < NPP; ++pp) {
                            double2& av = acc[(tig * kNP + node) * NPP + pp];
                            av = cadd(av, v[pp]);
                        }
                    }
                }
            }
        };
        switch (mtu) {
            case 1: run.template operator()<1>(); break;
            case 2: run.template operator()<2>(); break;
            case 3: run.template operator()<3>(); break;
            case 4: run.template operator()<4>(); break;
            case 5: run.template operator()<5>(); break;
            case 6: run.template operator()<6>(); break;
            case 7: if constexpr (kMT >= 7) run.template operator()<7>(); break;
            default: if constexpr (kMT >= 8) run.template operator()<8>(); break;
        }
    }
    cp_async_wait<0>();
    __syncwarp();

    // exceptions of this warp's segments: lane 0, in list order (rare; each may share an
    // accumulator with another)
    if (lane == 0) {
        const double hc = Lc.h;
        for (std::int64_t e = e0; e < e1; ++e) {
            const unsigned key = Lc.cb_exc_key[e];
            const int c = int(key & 0xffu) - 4 * warp, o = int((key >> 8) & 0xffu), node = int(key >> 16);
            if (c < 0 || c >= 4) continue;
            const int seg = iseg[c];
            if (seg < 0 || (Lp.active && !Lp.active[Lp.seg_box[seg]])) continue;
            const int ch = Lc.cb_child[(std::size_t(item) * kCbSegs + 4 * warp + c) * 8 + o];
            if (ch < 0 || (Lc.active && !Lc.active[ch])) continue;
            const int cso = Lc.cb_exc_cso[e];
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
            double ts[3], tt[5], tpp[5];
            cheb_row<3>(lc.ls, ts);
            cheb_row<5>(lc.lt, tt);
            cheb_row<5>(lc.lp, tpp);
            const double2* blk = cstore + std::size_t(cso) * NPC * kNP;
            for (int p = 0; p < NPC; ++p) {
                double2 v = make_double2(0.0, 0.0);
                for (int kk = 0; kk < kNP; ++kk) cfma_r(v, blk[p * kNP + kk], ts[kk % 3] * tt[(kk / 3) % 5] * tpp[kk / 15]);
                double2& a = acc[(c * kNP + node) * NPP + CB::dst(p)];
                a = cadd(a, cmul(child_factor<COMBO>(p, cs * q1, sn * q1, xf, k), v));
            }
        }
    }
    __syncwarp();

    // values -> coefficients (transform3) per segment; scratch = the warp's ring
    for (int c = 0; c < 4; ++c) {
        const int seg = __shfl_sync(0xffffffffu, seg_l, c);
        if (seg < 0) continue;
        transform3_warp<NPP>(acc + c * kNP * NPP, reinterpret_cast<double2*>(ring),
                             pstore + std::size_t(seg) * NPP * kNP, Ms, Ma, lane);
    }
}

// per (slot, octant): A2 rows, phi weights and re-centring data in group order
__global__ void cb_table_kernel(const double* __restrict__ tmpl, const std::uint8_t* __restrict__ nodes,
                                double* __restrict__ tab) {
    const std::size_t so8 = blockIdx.x;
    const int row = threadIdx.x;
    double* T = tab + so8 * kCbTab;
    double a2[16], tp[5], g[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 16; ++i) a2[i] = 0.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) tp[i] = 0.0;
    if (row < kNP) {
        const int node = nodes[so8 * kNP + row];
        const double* te = tmpl + (so8 * kNP + node) * kTmplDoubles;
        double ts[3], tt[5];
        cheb_row<3>(te[0], ts);
        cheb_row<5>(te[1], tt);
        cheb_row<5>(te[2], tp);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int tg = 0; tg < 3; ++tg) a2[4 * j + tg] = ts[tg] * tt[j];
            a2[4 * j + 3] = j < 3 ? ts[j] * tt[4] : 0.0;
        }
        g[0] = te[3];
        g[1] = te[4];
        g[2] = te[5];
        g[3] = double(node);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) T[row * 16 + i] = a2[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) T[kCbTabP + row * 8 + i] = i < 5 ? tp[i] : 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) T[kCbTabG + row * 4 + i] = g[i];
}

}  // namespace

void launch_cb_tables(const double* tmpl, const std::uint8_t* nodes, std::int64_t nslot, double* tab, cudaStream_t st) {
    if (nslot == 0) return;
    cb_table_kernel<<<unsigned(nslot * 8), kRows, 0, st>>>(tmpl, nodes, tab);
    IFGF_CUDA(cudaGetLastError());
}

bool launch_parent_fill_cb(const LevelDev& Lp, const LevelDev& Lc, const double2* child_store, double k,
                           const Pipes& parent_pipes, const Pipes& child_pipes, const double* Ms, const double* Ma,
                           double2* parent_store, cudaStream_t st) {
    if (Lc.n_cbitem == 0 || !Lp.tmpl || !Lc.cb_tab) return false;
    const int combo = combo_of(parent_pipes, child_pipes);
    if (combo < 0) return false;
    auto go = [&](auto kern, std::size_t smem) {
        IFGF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<Lc.n_cbitem, 32 * kW, smem, st>>>(Lp, Lc, child_store, k, Ms, Ma, parent_store);
    };
    switch (combo) {
        case 0: go(parent_cb_kernel<0>, kW * WarpSmem<Combo<0>::npc, Combo<0>::npp>::bytes); break;
        case 1: go(parent_cb_kernel<1>, kW * WarpSmem<Combo<1>::npc, Combo<1>::npp>::bytes); break;
        case 2: go(parent_cb_kernel<2>, kW * WarpSmem<Combo<2>::npc, Combo<2>::npp>::bytes); break;
        case 3: go(parent_cb_kernel<3>, kW * WarpSmem<Combo<3>::npc, Combo<3>::npp>::bytes); break;
        case 4: go(parent_cb_kernel<4>, kW * WarpSmem<Combo<4>::npc, Combo<4>::npp>::bytes); break;
        default: go(parent_cb_kernel<5>, kW * WarpSmem<Combo<5>::npc, Combo<5>::npp>::bytes); break;
    }
    IFGF_CUDA(cudaGetLastError());
#ifdef IFGF_CB_STATS
    unsigned long long h[4] = {0, 0, 0, 0};
    IFGF_CUDA(cudaStreamSynchronize(st));
    IFGF_CUDA(cudaMemcpyFromSymbol(h, g_cb_stats, sizeof(h)));
    std::fprintf(stderr, "cb stats: items %d units %llu tiles %llu seg-octants %llu block-octants %llu\n", Lc.n_cbitem, h[0], h[1], h[2], h[3]);
    const unsigned long long z[4] = {0, 0, 0, 0};
    IFGF_CUDA(cudaMemcpyToSymbol(g_cb_stats, z, sizeof(z)));
#endif
    return true;
}

}  // namespace ifgfb200
