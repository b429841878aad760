// Cousin evaluation (ifgf.cpp:396-450) on the FP64 tensor cores, for the default
// interpolation orders (ps = 3, pang = 5).
//
// One warp per <= 32 targets of a box (independent warp items, 4 per CTA), one lane per
// target. Per cousin source box the warp
//   1. computes each lane's local coordinates in its host-decided segment (cev_seg) and
//      the centred factor e^{ikr}/(4 pi r) into warp shared memory;
//   2. forms groups of lanes that evaluate the same segment (ballot on the ordinal), lists
//      each group's lanes, loads the segment's B fragments once and runs 8-row DMMA tiles
//      over the group (tc_common.cuh: 16 DMMAs per tile for 3 pipes, 12 for 2);
//   3. applies the pipe factors (W1 -> S; W2 (1/r), W3 (-ik), W4 -> D; formed per row in
//      step 1), adds the D pipes of each evaluation (one shuffle) and accumulates into the
//      target's shared accumulators.
// Every target gets its cousins' contributions in cousin-list order: deterministic.
#include <cstdlib>

#include "ifgf_device.cuh"
#include "kernels.cuh"
#include "tc_common.cuh"

namespace ifgfb200 {
namespace {

using namespace dev;
using namespace ifgfdev;
using namespace tc;

constexpr int kThreads = 128, kWarps = kThreads / 32;
constexpr int kCG = kRowLen + 6;  // A slots, T(phi), the pipe factors (3 complex) (odd stride)

// CODE = f0 f1 f2 as decimal digits (factor codes of the pipes) for the common pipe sets, so the
// pipe logic folds at compile time; 0 = read them from pp
template <int NPC, int CODE, bool BPRE>
__global__ void __launch_bounds__(kThreads, 4)
cousin_tc_kernel(LevelDev L, PointsDev P, const double2* __restrict__ store, double k, Pipes pp,
                 double2* __restrict__ Sp, double2* __restrict__ Dp) {
    using LY = Layout<NPC>;
    auto fcode = [&](int i) -> int {
        if constexpr (CODE != 0) return i == 0 ? CODE / 100 : (i == 1 ? (CODE / 10) % 10 : CODE % 10);
        else return pp.f[i];
    };
    __shared__ double sgeo[kWarps][32 * kCG];
    __shared__ double2 sacc[kWarps][32][2];
    __shared__ int slist[kWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r = lane >> 2, tig = lane & 3;
    const int wc = blockIdx.x * kWarps + warp;  // one warp item = <= 32 targets of one box
    if (wc >= L.nwchunk) return;
    const int tb = L.wchunk_box[wc];
    const int tbeg = int(L.beg[tb]);
    const int n_t = int(L.end[tb]) - tbeg;
    const int q = L.wchunk_q0[wc] + lane;
    const bool act = q < n_t;
    const int t = act ? tbeg + q : tbeg;
    const double x = P.x[t], y = P.y[t], z = P.z[t];
    const double h = L.h;
    sacc[warp][lane][0] = sacc[warp][lane][1] = make_double2(0.0, 0.0);
    // S comes from the W1 lane alone; D from the first D-pipe lane plus, for (W2, W3), its
    // right neighbour (pipe lists keep W2, W3 adjacent)
    int s_lane = -1, d_lane = -1, n_d = 0;
#pragma unroll
    for (int i = 0; i < NPC; ++i) {
        if (fcode(i) == 1) s_lane = i;
        else if (n_d++ == 0) d_lane = i;
    }
    const int j0 = L.cz_ptr[tb], j1 = L.cz_ptr[tb + 1];
    const std::int64_t ev0 = L.cev_begin[tb] + q;
    double* mygeo = sgeo[warp] + lane * kCG;
    for (int j = j0; j < j1; ++j) {
        const int sb = L.cz_idx[j];
        if (L.active && !L.active[sb]) continue;  // source box owned by another rank
        const int so = act ? L.cev_seg[ev0 + std::int64_t(j - j0) * n_t] : -1;
        // BPRE: the first group's B fragments (the first active lane's segment) are loaded
        // before the geometry step, so their latency hides behind it
        unsigned pending = __ballot_sync(0xffffffffu, act);
        double bq0[LY::NB];
        if constexpr (BPRE) {
            if (pending) {
                const int seg0 = __shfl_sync(0xffffffffu, so, __ffs(pending) - 1);
                load_b<NPC>(store + std::size_t(seg0) * NPC * kNP, lane, bq0);
            }
        }
        if (act) {
            const double vx = x - L.cx[sb], vy = y - L.cy[sb], vz = z - L.cz[sb];
            const double r2 = fma(vx, vx, fma(vy, vy, vz * vz));
            const double inv_r = rsqrt_normal(r2);
            const LocalCoords lc = local_coords_seg(vx, vy, vz, inv_r, h, so, L);
            double sn, cs;
            sincos_bounded(k * (r2 * inv_r), &sn, &cs);
            const double f1 = kInv4PiD * inv_r;
            const double2 e1 = make_double2(cs * f1, sn * f1);  // e^{ikr}/(4 pi r)
            fill_row(lc.ls, lc.lt, lc.lp, mygeo);
            // per pipe: W1 -> S and W4 -> D take e1, W2 -> D e1/r, W3 -> D -ik e1
#pragma unroll
            for (int p = 0; p < NPC; ++p) {
                double2 f = e1;
                if (fcode(p) == 2) f = cscale(e1, inv_r);
                if (fcode(p) == 3) f = make_double2(k * e1.y, -k * e1.x);
                mygeo[kRowLen + 2 * p] = f.x;
                mygeo[kRowLen + 2 * p + 1] = f.y;
            }
        }
        __syncwarp();
        bool first = true;
        while (pending) {
            const int seg = __shfl_sync(0xffffffffu, so, __ffs(pending) - 1);
            const unsigned gmask = __ballot_sync(0xffffffffu, act && so == seg);
            pending &= ~gmask;
            if ((gmask >> lane) & 1u) slist[warp][__popc(gmask & ((1u << lane) - 1u))] = lane;
            __syncwarp();
            const int count = __popc(gmask);
            double bq[LY::NB];
            if (BPRE && first) {
#pragma unroll
                for (int i = 0; i < LY::NB; ++i) bq[i] = bq0[i];
            } else {
                load_b<NPC>(store + std::size_t(seg) * NPC * kNP, lane, bq);
            }
            first = false;
            for (int t0 = 0; t0 < count; t0 += 8) {
                const bool valid = t0 + r < count;
                const int src = valid ? slist[warp][t0 + r] : 0;
                const double* gp = sgeo[warp] + src * kCG;
                double d[LY::NQ][2];
                tile_mma_row<NPC>(gp, valid, tig, bq, d);
                const double2 val = tile_gather_row<NPC>(gp, lane, d);
                const int fp = tig < NPC ? tig : 0;
                double2 w = cmul(make_double2(gp[kRowLen + 2 * fp], gp[kRowLen + 2 * fp + 1]), val);
                if (n_d == 2) {  // (W2, W3): the second D pipe joins the first
                    const double ox = __shfl_down_sync(0xffffffffu, w.x, 1);
                    const double oy = __shfl_down_sync(0xffffffffu, w.y, 1);
                    if (tig == d_lane) w = make_double2(w.x + ox, w.y + oy);
                }
                if (valid && tig == s_lane) sacc[warp][src][0] = cadd(sacc[warp][src][0], w);
                if (valid && tig == d_lane) sacc[warp][src][1] = cadd(sacc[warp][src][1], w);
            }
            __syncwarp();
        }
    }
    __syncwarp();
    if (!act) return;
    Sp[t] = cadd(Sp[t], sacc[warp][lane][0]);
    Dp[t] = cadd(Dp[t], sacc[warp][lane][1]);
}

}  // namespace

bool launch_cousin_eval_tc(const LevelDev& L, const PointsDev& P, const double2* store, double k, const Pipes& pipes,
                           double2* Sp, double2* Dp, cudaStream_t st) {
    if (L.ps != kPS || L.pang != kPA || pipes.n < 1 || pipes.n > 3) return false;
    if (pipes.n == 3 && pipes.f[1] == 1) return false;  // D pipes must be adjacent (epilogue shuffle)
    if (L.nwchunk == 0) return true;
    const int grid = (L.nwchunk + kWarps - 1) / kWarps;
    const int code = pipes.f[0] * 100 + (pipes.n > 1 ? pipes.f[1] * 10 : 0) + (pipes.n > 2 ? pipes.f[2] : 0);
    // IFGF_COUSIN_BPRE=1: the first group's coefficients are loaded before the geometry step.
    // Off by default: measured slower (cfg3 cousins 105 -> 117 ms, cfg2 4.87 -> 5.45 ms; the 24
    // extra live registers across the geometry step cost more than the hidden latency)
    static const bool bpre = [] {
        const char* e = std::getenv("IFGF_COUSIN_BPRE");
        return e && e[0] == '1';
    }();
    auto go = [&](auto kpre, auto kplain) {
        if (bpre) kpre<<<grid, kThreads, 0, st>>>(L, P, store, k, pipes, Sp, Dp);
        else kplain<<<grid, kThreads, 0, st>>>(L, P, store, k, pipes, Sp, Dp);
    };
    switch (code) {
        case 123: go(cousin_tc_kernel<3, 123, true>, cousin_tc_kernel<3, 123, false>); break;
        case 140: go(cousin_tc_kernel<2, 140, true>, cousin_tc_kernel<2, 140, false>); break;
        case 100: go(cousin_tc_kernel<1, 100, true>, cousin_tc_kernel<1, 100, false>); break;
        default:
            switch (pipes.n) {
                case 1: go(cousin_tc_kernel<1, 0, true>, cousin_tc_kernel<1, 0, false>); break;
                case 2: go(cousin_tc_kernel<2, 0, true>, cousin_tc_kernel<2, 0, false>); break;
                default: go(cousin_tc_kernel<3, 0, true>, cousin_tc_kernel<3, 0, false>); break;
            }
    }
    IFGF_CUDA(cudaGetLastError());
    return true;
}

}  // namespace ifgfb200
