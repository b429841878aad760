// Parent fill (ifgf.cpp:452-568) on the FP64 tensor cores, for the default interpolation
// orders (ps = 3, pang = 5).
//
// One warp per parent segment (4 per CTA). The warp takes the host's child-segment groups
// of that segment in turn (all parent-node evaluations that land in one child cone
// segment, csrc/host/coneplan.cpp group_parent_evaluations):
//   1. the warp's lanes compute, for the group's evaluations, the child-frame local
//      coordinates and the re-centring factors (node directions from sin/cos tables);
//   2. tiles of 8 evaluations contract the child's 3x5x5 coefficient block with
//      mma.sync.m8n8k4.f64 (DMMA): A = T_s(s) T_t(theta) (rows = evaluations, k = the 15
//      (s, theta) index pairs in 4 steps of 4), B = coefficients whose 8 columns hold 4
//      (pipe, phi index) pairs x {re, im}, one accumulator per column group: a tile takes
//      4 x ceil(5 pipes / 4) DMMAs (16 for 3 pipes, 12 for 2, 8 for 1); B is loaded once
//      per group and reused by all its tiles;
//   3. the epilogue weights the accumulators by T_p(phi), gathers each pipe's phi terms
//      within the quad (shuffles), applies the re-centring factor and adds into the warp's private node
//      accumulators (no atomics).
// The separable block transform (warp-local) finishes the segment. Results equal the
// per-lane kernel to rounding (~1e-16); the evaluation order is fixed, so the output is
// bitwise reproducible run to run.
#include "ifgf_device.cuh"
#include "kernels.cuh"
#include "tc_common.cuh"
#include "parent_common.cuh"

namespace ifgfb200 {
namespace {

using namespace dev;
using namespace ifgfdev;

using namespace tc;
using namespace pfill;

constexpr int kWarps = 4;
#ifndef IFGF_PARENT_MINB
#define IFGF_PARENT_MINB 4
#endif
constexpr int kRow = kRowLen + 8;     // A slots, T(phi), per child pipe its factor (3 complex), node, pad (odd)
constexpr int kNode = kRowLen + 6;
constexpr int kGeoSz = 32 * kRow;      // one chunk of 32 evaluation rows per warp (even: the
                                       // accumulators behind it stay 16-byte aligned)

template <int COMBO>
__global__ void __launch_bounds__(32 * kWarps, IFGF_PARENT_MINB)
parent_tc_kernel(LevelDev Lp, LevelDev Lc, const double2* __restrict__ cstore, double k,
                 const double* __restrict__ Ms, const double* __restrict__ Ma,
                 double2* __restrict__ pstore) {
    using CB = Combo<COMBO>;
    constexpr int NPP = CB::npp, NPC = CB::npc;
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int merge = kParentMergeMax;  // accumulator blocks per warp (items may use fewer)
    double* geo = smem + warp * (kGeoSz + 2 * kNP * NPP * merge);  // per warp
    double2* acc = reinterpret_cast<double2*>(geo + kGeoSz);  // per item segment: 75 x NPP
    const int item = blockIdx.x * kWarps + warp;  // one warp per work item
    if (item >= Lc.n_pitem) return;
    const int* __restrict__ iseg = Lc.pitem_seg + item * kParentMergeMax;
    int segs[kParentMergeMax], tsl[kParentMergeMax], pcode[kParentMergeMax];
    const int pb = Lp.seg_box[iseg[0]];
    if (Lp.active && !Lp.active[pb]) return;  // no sources of this rank below
#pragma unroll
    for (int w = 0; w < kParentMergeMax; ++w) {
        segs[w] = iseg[w];
        const int gam = segs[w] >= 0 ? Lp.seg_gamma[segs[w]] : 0;
        tsl[w] = Lp.tmpl_slot && segs[w] >= 0 ? Lp.tmpl_slot[gam] : -1;
        pcode[w] = (gam % Lp.ns) | (((gam / Lp.ns) % Lp.nc) << 8) | ((gam / Lp.ns / Lp.nc) << 19);
    }
    for (int e = lane; e < kNP * NPP * merge; e += 32) acc[e] = make_double2(0.0, 0.0);
    const double hp = Lp.h, hc = Lc.h;
    const double pcx = Lp.cx[pb], pcy = Lp.cy[pb], pcz = Lp.cz[pb];

    const int r = lane >> 2, tig = lane & 3;
    using LY = Layout<NPC>;
    const int gb = Lc.pitem_grp[item], ge = Lc.pitem_grp[item + 1];
    // group records (host-packed: child segment, child box, start | count << 16 | child
    // octant << 24, cell) run two groups ahead and the first evaluation entries one group
    // ahead, so a group's template loads issue at its start without a dependent-load chain
    const int4* __restrict__ grec = Lc.pgrp_rec;
    const std::uint16_t* __restrict__ perm = Lc.pev_perm + Lc.pitem_ev[item];
    const int4 zero4 = make_int4(0, 0, 0, 0);
    int4 rec1 = gb < ge ? grec[gb] : zero4;
    int4 rec2 = gb + 1 < ge ? grec[gb + 1] : zero4;
    unsigned ent1 = (gb < ge && lane < ((rec1.z >> 16) & 0xff)) ? perm[(rec1.z & 0xffff) + lane] : 0u;
    for (int g = gb; g < ge; ++g) {
        const int4 rec = rec1;
        const unsigned ent_first = ent1;
        rec1 = rec2;
        if (g + 2 < ge) rec2 = grec[g + 2];
        ent1 = (g + 1 < ge && lane < ((rec1.z >> 16) & 0xff)) ? perm[(rec1.z & 0xffff) + lane] : 0u;
        const int cso = rec.x, ch = rec.y;
        const int start = rec.z & 0xffff, count = (rec.z >> 16) & 0xff, oct = (rec.z >> 24) & 7;
        if (Lc.active && !Lc.active[ch]) continue;  // child holds no sources of this rank
        // B fragments of the group's block, reused by all its tiles (tc_common.cuh)
        double bq[LY::NB];
        load_b<NPC>(cstore + std::size_t(cso) * NPC * kNP, lane, bq);
        for (int e0 = 0; e0 < count; e0 += 32) {  // chunks of 32 evaluations, one per lane
            const int cn = min(32, count - e0);
            if (lane < cn) {
                // entries are node | c << 8 | item segment << 11, bit 15: the template applies
                const unsigned ent = e0 == 0 ? ent_first : perm[start + e0 + lane];
                const int node = int(ent & 0xffu), ws = int((ent >> 11) & 1u);
                int tslot = tsl[0], code = pcode[0];
#pragma unroll
                for (int w = 1; w < kParentMergeMax; ++w)
                    if (ws == w) tslot = tsl[w], code = pcode[w];
                double ls, lt, lp, r1x, r1y, xf;
                if (ent & 0x8000u) {
                    // geometry template of (parent cell, child octant, node), host/coneplan.hpp
                    const std::size_t tent = (std::size_t(tslot) * 8 + oct) * kNP + node;
                    const double2* te = reinterpret_cast<const double2*>(Lp.tmpl + tent * kTmplDoubles);
                    const double2 t0 = __ldg(te), t1 = __ldg(te + 1), t2 = __ldg(te + 2);
                    ls = t0.x;
                    lt = t0.y;
                    lp = t1.x;
                    r1x = t1.y;
                    r1y = t2.x;
                    xf = t2.y;  // 1/r_c
                    if (CB::extra == RQ) xf *= hp / Lp.s_nodes[(code & 0xff) * kPS + node % kPS];  // r_p/r_c
                } else {
                    // child frame, loaded only on this (rare, non-template) path
                    const double ccx = Lc.cx[ch], ccy = Lc.cy[ch], ccz = Lc.cz[ch];
                    const CellFrame cf =
                        Lc.seg_code ? cell_frame_code(unsigned(rec.w), Lc) : cell_frame(rec.w, Lc);
                    const int is = node % kPS, it = (node / kPS) % kPA, ip = node / (kPS * kPA);
                    const int g1 = code & 0xff, g2 = (code >> 8) & 0x7ff, g3 = code >> 19;
                    const double s = Lp.s_nodes[g1 * kPS + is];
                    const double rp = hp / s;
                    const double sth = Lp.th_sin[g2 * kPA + it], cth = Lp.th_cos[g2 * kPA + it];
                    const double sph = Lp.ph_sin[g3 * kPA + ip], cph = Lp.ph_cos[g3 * kPA + ip];
                    const double x = pcx + rp * sth * cph, y = pcy + rp * sth * sph, z = pcz + rp * cth;
                    const double vx = x - ccx, vy = y - ccy, vz = z - ccz;
                    const double rc2 = fma(vx, vx, fma(vy, vy, vz * vz));
                    const double inv_rc = rsqrt_normal(rc2);
                    const double rc = rc2 * inv_rc;
                    const LocalCoords lc = local_coords_in(vx, vy, vz, inv_rc, hc, cf, Lc);
                    // stable r_c - r_p (ifgf.cpp:149-153)
                    const double sx = ccx + pcx - 2.0 * x, sy = ccy + pcy - 2.0 * y, sz = ccz + pcz - 2.0 * z;
                    const double dr = fma(sx, ccx - pcx, fma(sy, ccy - pcy, sz * (ccz - pcz))) / (rc + rp);
                    double sn, cs;
                    sincos_bounded(k * dr, &sn, &cs);
                    const double q1 = rp * inv_rc;
                    ls = lc.ls;
                    lt = lc.lt;
                    lp = lc.lp;
                    r1x = cs * q1;
                    r1y = sn * q1;
                    xf = CB::extra == RI ? inv_rc : q1;
                }
                double* row = geo + lane * kRow;
                fill_row(ls, lt, lp, row);
                // per child pipe: ratio1 times 1 (R1), -ik (MK) or the extra factor (RI, RQ)
#pragma unroll
                for (int pc = 0; pc < NPC; ++pc) {
                    double fx = r1x, fy = r1y;
                    if (CB::fac(pc) == MK) {
                        fx = k * r1y;
                        fy = -k * r1x;
                    } else if (CB::fac(pc) != R1) {
                        fx = r1x * xf;
                        fy = r1y * xf;
                    }
                    row[kRowLen + 2 * pc] = fx;
                    row[kRowLen + 2 * pc + 1] = fy;
                }
                row[kNode] = __longlong_as_double((long long)(node + kNP * ws));  // accumulator row of (segment, node), as integer bits
            }
            __syncwarp();
            // 2. 8-evaluation tensor-core tiles against the child block (issuing the next
            // tile's DMMAs before this tile's epilogue measured slower)
            auto mma = [&](int t0, double (&d)[LY::NQ][2]) {
                const bool valid = t0 + r < cn;
                tile_mma_row<NPC>(geo + (valid ? t0 + r : 0) * kRow, valid, tig, bq, d);
            };
            auto epilogue = [&](int t0, const double (&d)[LY::NQ][2]) {
                const bool valid = t0 + r < cn;
                const double* gp = geo + (valid ? t0 + r : 0) * kRow;
                const double2 val = tile_gather_row<NPC>(gp, lane, d);
                // lanes tig < NPC now hold (re, im) of child pipe tig for evaluation row r
                const int fp = tig < NPC ? tig : 0;
                double2 ctb = cmul(make_double2(gp[kRowLen + 2 * fp], gp[kRowLen + 2 * fp + 1]), val);
                if constexpr (COMBO == 0) {  // child W2, W3 -> parent W4: sum across the quad
                    const double ox = __shfl_down_sync(0xffffffffu, ctb.x, 1);
                    const double oy = __shfl_down_sync(0xffffffffu, ctb.y, 1);
                    if (tig == 1) ctb = make_double2(ctb.x + ox, ctb.y + oy);
                } else if constexpr (COMBO == 3) {
                    const double ox = __shfl_down_sync(0xffffffffu, ctb.x, 1);
                    const double oy = __shfl_down_sync(0xffffffffu, ctb.y, 1);
                    if (tig == 0) ctb = make_double2(ctb.x + ox, ctb.y + oy);
                }
                bool writer = valid && tig < NPC;
                if constexpr (COMBO == 0) writer = writer && tig != 2;
                if constexpr (COMBO == 3) writer = writer && tig == 0;
                if (writer) {
                    int dst = 0;
#pragma unroll
                    for (int pc = 0; pc < NPC; ++pc)
                        if (tig == pc) dst = CB::dst(pc);
                    double2& a = acc[int(__double_as_longlong(gp[kNode])) * NPP + dst];
                    a = cadd(a, ctb);
                }
            };
            for (int t0 = 0; t0 < cn; t0 += 8) {
                double d[LY::NQ][2];
                mma(t0, d);
                epilogue(t0, d);
            }
            __syncwarp();
        }
    }
    // values -> coefficients (transform3, ifgf.cpp:560-562), warp-local, per item segment
    for (int w = 0; w < kParentMergeMax; ++w) {
        if (segs[w] < 0) break;
        __syncwarp();
        transform3_warp<NPP>(acc + w * kNP * NPP, reinterpret_cast<double2*>(geo),
                             pstore + std::size_t(segs[w]) * NPP * kNP, Ms, Ma, lane);
    }
}

}  // namespace

bool launch_parent_fill_tc(const LevelDev& Lp, const LevelDev& Lc, const double2* child_store, double k,
                           const Pipes& parent_pipes, const Pipes& child_pipes, const double* Ms,
                           const double* Ma, double2* parent_store, cudaStream_t st) {
    const int combo = combo_of(parent_pipes, child_pipes);
    if (combo < 0 || Lp.ps != kPS || Lp.pang != kPA || Lc.ps != kPS || Lc.pang != kPA || !Lc.pitem_grp ||
        !Lp.th_sin)
        return false;
    // segments of cells shared across boxes: batched GEMMs (parent_cb.cu); the rest below
    launch_parent_fill_cb(Lp, Lc, child_store, k, parent_pipes, child_pipes, Ms, Ma, parent_store, st);
    if (Lc.n_pitem == 0) return true;
    const std::size_t smem =
        std::size_t(kWarps) * (kGeoSz + 2 * kNP * parent_pipes.n * kParentMergeMax) * sizeof(double);
    auto go = [&](auto kern) {
        IFGF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<(Lc.n_pitem + kWarps - 1) / kWarps, 32 * kWarps, smem, st>>>(Lp, Lc, child_store, k, Ms, Ma, parent_store);
    };
    switch (combo) {
        case 0: go(parent_tc_kernel<0>); break;
        case 1: go(parent_tc_kernel<1>); break;
        case 2: go(parent_tc_kernel<2>); break;
        case 3: go(parent_tc_kernel<3>); break;
        case 4: go(parent_tc_kernel<4>); break;
        default: go(parent_tc_kernel<5>); break;
    }
    IFGF_CUDA(cudaGetLastError());
    return true;
}

}  // namespace ifgfb200
