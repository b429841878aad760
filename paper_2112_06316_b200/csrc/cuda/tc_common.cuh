// FP64 tensor-core (mma.sync.m8n8k4.f64, DMMA) evaluation of 3x5x5 Chebyshev blocks, shared
// by the parent fill (parent_tc.cu) and the cousin evaluation (cousin_tc.cu).
//
// A warp evaluates tiles of 8 evaluations of ONE coefficient block (NPC pipes x 75 complex
// coefficients, ifgf.cpp:71-89 eval3 with ps = 3, pang = 5):
//   A (8 x 4 per step) = T_is(s) T_it(theta) of the tile's rows, k running over the 15
//     (is, it) pairs in 4 steps of 4: slot (j, tig) = (tig, j) for tig < 3 and (j, 4) for
//     tig = 3, slot (3, 3) padding;
//   B (4 x 8 per step) = coefficients; the 8 columns are 4 (pipe, phi index) pairs x
//     {re, im}, one accumulator per column group q: 3 pipes -> pairs (c, q) for c < 3 and
//     (q, 4) for c = 3 (15 pairs, 4 groups, 16 DMMAs per tile); fewer pipes -> IPG = 4/NPC
//     phi indices per group (12 DMMAs for 2 pipes, 8 for 1);
//   gather: T_ip(phi) weights, then each pipe's phi terms are collected within the quad, so
//     lanes (r, tig < NPC) end up with (re, im) of pipe tig for row r.
// B is loaded once per block into registers and reused by every tile of that block.
#pragma once

#include "dev_common.cuh"

namespace ifgfb200 {
namespace tc {

constexpr int kPS = 3, kPA = 5, kNP = 75;
constexpr int kKS = kPA - 1;  // DMMA k-steps over the 15 (s, theta) pairs (4 x 4 slots)
static_assert(kPS == 3 && kPA == 5, "the k-slot map assumes 3 x 5 (s, theta) pairs");

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int NPC>
struct Layout {
    static constexpr int IPG = 4 / NPC;
    static constexpr int NQ = NPC == 3 ? 4 : (kPA + IPG - 1) / IPG;
    static constexpr int NB = kKS * NQ;  // B registers per lane
    // (pipe, phi index) of column pair c in group q; false for padding
    __device__ static bool pair_of(int q, int c, int& pipe, int& ip) {
        if constexpr (NPC == 3) {
            if (c < 3) {
                pipe = c;
                ip = q;
                return true;
            }
            pipe = q;
            ip = kPA - 1;
            return q < 3;
        } else {
            const int sub = c / NPC;
            pipe = c % NPC;
            ip = IPG * q + sub;
            return sub < IPG && ip < kPA;
        }
    }
};

// B fragments of one block (pipe-major, 75 complex per pipe, node = is + 3 (it + 5 ip))
template <int NPC>
__device__ __forceinline__ void load_b(const double2* __restrict__ block, int lane, double* bq) {
    using LY = Layout<NPC>;
    const int tig = lane & 3, ncol = lane >> 2, bc = ncol >> 1, reim = ncol & 1;
    const bool lo = tig < kPS;
    const double* blk = reinterpret_cast<const double*>(block) + reim;
#pragma unroll
    for (int q = 0; q < LY::NQ; ++q) {
        int pipe, ip;
        const bool live = LY::pair_of(q, bc, pipe, ip);
#pragma unroll
        for (int j = 0; j < kKS; ++j) {
            const int is = lo ? tig : j, it = lo ? j : kPA - 1;
            bq[q * kKS + j] = (live && (lo || j < kPS)) ? __ldg(blk + 2 * (pipe * kNP + is + kPS * (it + kPA * ip)))
                                                         : 0.0;
        }
    }
}

// one tile: row r = lane >> 2 has local coordinates (ls, lt) (valid = false: zero row)
template <int NPC>
__device__ __forceinline__ void tile_mma(double ls, double lt, bool valid, int tig, const double* bq,
                                         double (&d)[Layout<NPC>::NQ][2]) {
    using LY = Layout<NPC>;
    double ts[kPS], tt[kPA];
    dev::cheb_row<kPS>(ls, ts);
    dev::cheb_row<kPA>(lt, tt);
    const bool lo = tig < kPS;
    // lane-constant operand choice: T_tig(s) for the first three k columns, T_4(theta) for
    // the fourth
    double tsel = tig == 0 ? ts[0] : (tig == 1 ? ts[1] : ts[2]);
    double t4 = tt[kPA - 1];
    if (!valid) tsel = t4 = 0.0;
#pragma unroll
    for (int q = 0; q < LY::NQ; ++q) d[q][0] = d[q][1] = 0.0;
#pragma unroll
    for (int j = 0; j < kKS; ++j) {
        const double x = lo ? tsel : (j < kPS ? ts[j] : 0.0);
        const double y = lo ? tt[j] : t4;
        const double a = x * y;
#pragma unroll
        for (int q = 0; q < LY::NQ; ++q) dmma884(d[q][0], d[q][1], a, bq[q * kKS + j]);
    }
}

// T(phi) weights and the per-pipe gather within the quad: lanes tig < NPC return (re, im)
// of pipe tig for row r (other lanes: unspecified)
template <int NPC>
__device__ __forceinline__ double2 tile_gather(double lp, int lane, const double (&d)[Layout<NPC>::NQ][2]) {
    using LY = Layout<NPC>;
    const int tig = lane & 3;
    double tq[kPA];
    dev::cheb_row<kPA>(lp, tq);
    double2 val = make_double2(0.0, 0.0);
    if constexpr (NPC == 3) {
#pragma unroll
        for (int q = 0; q < LY::NQ; ++q) {
            val.x = fma(tq[q], d[q][0], val.x);
            val.y = fma(tq[q], d[q][1], val.y);
        }
        // phi index 4 of pipe q sits in lane 3 of the quad, group q
        const int src = (lane & ~3) | 3;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const double ex = __shfl_sync(0xffffffffu, d[q][0], src);
            const double ey = __shfl_sync(0xffffffffu, d[q][1], src);
            if (tig == q) {
                val.x = fma(tq[kPA - 1], ex, val.x);
                val.y = fma(tq[kPA - 1], ey, val.y);
            }
        }
    } else {
        const int sub = tig / NPC;
#pragma unroll
        for (int q = 0; q < LY::NQ; ++q) {
            double w = 0.0;
#pragma unroll
            for (int s = 0; s < LY::IPG; ++s)
                if (LY::IPG * q + s < kPA && sub == s) w = tq[LY::IPG * q + s];
            val.x = fma(w, d[q][0], val.x);
            val.y = fma(w, d[q][1], val.y);
        }
#pragma unroll
        for (int off = NPC; off < NPC * LY::IPG; off <<= 1) {
            val.x += __shfl_down_sync(0xffffffffu, val.x, off);
            val.y += __shfl_down_sync(0xffffffffu, val.y, off);
        }
    }
    return val;
}

// ---- precomputed evaluation rows: the geometry step of an evaluation writes, once, its
// A operands in k-slot order and its T(phi) row, so the tiles only load them.
constexpr int kRowA = 16;           // A slots: (j, tig) at 4 j + tig
constexpr int kRowTq = kRowA;       // T_0..T_4(phi)
constexpr int kRowLen = kRowA + kPA;

__device__ __forceinline__ void fill_row(double ls, double lt, double lp, double* row) {
    double ts[kPS], tt[kPA], tq[kPA];
    dev::cheb_row<kPS>(ls, ts);
    dev::cheb_row<kPA>(lt, tt);
    dev::cheb_row<kPA>(lp, tq);
#pragma unroll
    for (int j = 0; j < kKS; ++j) {
#pragma unroll
        for (int tg = 0; tg < kPS; ++tg) row[4 * j + tg] = ts[tg] * tt[j];  // (is, it) = (tg, j)
        row[4 * j + 3] = j < kPS ? ts[j] * tt[kPA - 1] : 0.0;              // (j, 4), (3, 3) padding
    }
#pragma unroll
    for (int p = 0; p < kPA; ++p) row[kRowTq + p] = tq[p];
}

// tile from precomputed rows (row = this lane's row r, valid = false: zero row)
template <int NPC>
__device__ __forceinline__ void tile_mma_row(const double* row, bool valid, int tig, const double* bq,
                                             double (&d)[Layout<NPC>::NQ][2]) {
    using LY = Layout<NPC>;
#pragma unroll
    for (int q = 0; q < LY::NQ; ++q) d[q][0] = d[q][1] = 0.0;
#pragma unroll
    for (int j = 0; j < kKS; ++j) {
        const double a = valid ? row[4 * j + tig] : 0.0;
#pragma unroll
        for (int q = 0; q < LY::NQ; ++q) dmma884(d[q][0], d[q][1], a, bq[q * kKS + j]);
    }
}

template <int NPC>
__device__ __forceinline__ double2 tile_gather_row(const double* row, int lane, const double (&d)[Layout<NPC>::NQ][2]) {
    using LY = Layout<NPC>;
    const int tig = lane & 3;
    const double* tq = row + kRowTq;
    double2 val = make_double2(0.0, 0.0);
    if constexpr (NPC == 3) {
#pragma unroll
        for (int q = 0; q < LY::NQ; ++q) {
            const double w = tq[q];
            val.x = fma(w, d[q][0], val.x);
            val.y = fma(w, d[q][1], val.y);
        }
        const double w4 = tq[kPA - 1];
        const int src = (lane & ~3) | 3;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const double ex = __shfl_sync(0xffffffffu, d[q][0], src);
            const double ey = __shfl_sync(0xffffffffu, d[q][1], src);
            if (tig == q) {
                val.x = fma(w4, ex, val.x);
                val.y = fma(w4, ey, val.y);
            }
        }
    } else {
        const int sub = tig / NPC;
#pragma unroll
        for (int q = 0; q < LY::NQ; ++q) {
            const int ip = LY::IPG * q + sub;
            const double w = ip < kPA ? tq[ip < kPA ? ip : 0] : 0.0;
            val.x = fma(w, d[q][0], val.x);
            val.y = fma(w, d[q][1], val.y);
        }
#pragma unroll
        for (int off = NPC; off < NPC * LY::IPG; off <<= 1) {
            val.x += __shfl_down_sync(0xffffffffu, val.x, off);
            val.y += __shfl_down_sync(0xffffffffu, val.y, off);
        }
    }
    return val;
}

}  // namespace tc
}  // namespace ifgfb200
