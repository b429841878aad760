// Child -> parent pipe combinations of the parent fill (ifgf.cpp:525-555), shared by the
// tensor-core parent kernels (parent_tc.cu: one warp per parent segment; parent_cb.cu:
// parent segments of one cone cell batched into small GEMMs).
#pragma once

#include <initializer_list>

#include "dev_common.cuh"
#include "kernels.cuh"

namespace ifgfb200 {
namespace pfill {

// Child->parent pipe combinations of the strategies (ifgf.cpp:525-555). Each child pipe
// feeds one parent pipe with one factor: R1 = ratio1, RI = ratio1/r_c (W2 -> W4),
// MK = -ik ratio1 (W3 -> W4), RQ = ratio1 r_p/r_c (W2 -> W2).
enum Fac { R1 = 0, RI = 1, MK = 2, RQ = 3 };
template <int C>
struct Combo;
template <>
struct Combo<0> {  // (W1,W4) <- (W1,W2,W3): Hybrid, sub-half-wavelength child
    static constexpr int npp = 2, npc = 3, extra = RI;
    __device__ static constexpr int dst(int i) { return i == 0 ? 0 : 1; }
    __device__ static constexpr int fac(int i) { return i == 0 ? R1 : (i == 1 ? RI : MK); }
};
template <>
struct Combo<1> {  // (W1,W4) <- (W1,W4)
    static constexpr int npp = 2, npc = 2, extra = R1;
    __device__ static constexpr int dst(int i) { return i; }
    __device__ static constexpr int fac(int) { return R1; }
};
template <>
struct Combo<2> {  // (W1) <- (W1), or (W4) <- (W4)
    static constexpr int npp = 1, npc = 1, extra = R1;
    __device__ static constexpr int dst(int) { return 0; }
    __device__ static constexpr int fac(int) { return R1; }
};
template <>
struct Combo<3> {  // (W4) <- (W2,W3)
    static constexpr int npp = 1, npc = 2, extra = RI;
    __device__ static constexpr int dst(int) { return 0; }
    __device__ static constexpr int fac(int i) { return i == 0 ? RI : MK; }
};
template <>
struct Combo<4> {  // (W1,W2,W3) <- (W1,W2,W3)
    static constexpr int npp = 3, npc = 3, extra = RQ;
    __device__ static constexpr int dst(int i) { return i; }
    __device__ static constexpr int fac(int i) { return i == 1 ? RQ : R1; }
};
template <>
struct Combo<5> {  // (W2,W3) <- (W2,W3)
    static constexpr int npp = 2, npc = 2, extra = RQ;
    __device__ static constexpr int dst(int i) { return i; }
    __device__ static constexpr int fac(int i) { return i == 0 ? RQ : R1; }
};

inline int combo_of(const Pipes& pp, const Pipes& pc) {
    auto is = [](const Pipes& p, std::initializer_list<int> f) {
        if (p.n != int(f.size())) return false;
        int i = 0;
        for (int x : f)
            if (p.f[i++] != x) return false;
        return true;
    };
    if (is(pp, {1, 4}) && is(pc, {1, 2, 3})) return 0;
    if (is(pp, {1, 4}) && is(pc, {1, 4})) return 1;
    if ((is(pp, {1}) && is(pc, {1})) || (is(pp, {4}) && is(pc, {4}))) return 2;
    if (is(pp, {4}) && is(pc, {2, 3})) return 3;
    if (is(pp, {1, 2, 3}) && is(pc, {1, 2, 3})) return 4;
    if (is(pp, {2, 3}) && is(pc, {2, 3})) return 5;
    return -1;
}


// values -> coefficients of one parent segment (transform3, ifgf.cpp:560-562) by one warp:
// v0 holds the node values node-major ([node][NPP], node = is + 3 (it + 5 ip)); v1 is a
// scratch of NPP x 75; dst receives the pipe-major coefficient block. Each lane transforms
// whole lines with the 3x3 (s) and 5x5 (theta, phi) matrices held in registers, adding the
// terms in the same order as the element-wise form (bitwise the same results). v0 is
// overwritten (pipe-major after the second pass).
template <int NPP>
__device__ __forceinline__ void transform3_warp(double2* v0, double2* v1, double2* __restrict__ dst,
                                                const double* __restrict__ Ms, const double* __restrict__ Ma,
                                                int lane) {
    constexpr int kNP = 75;
    double ms[9], ma[25];
#pragma unroll
    for (int i = 0; i < 9; ++i) ms[i] = __ldg(Ms + i);
#pragma unroll
    for (int i = 0; i < 25; ++i) ma[i] = __ldg(Ma + i);
    // s: line = (it, ip) of pipe pp
    for (int l = lane; l < 25 * NPP; l += 32) {
        const int pp = l / 25, line = l - pp * 25;
        double2 in[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) in[q] = v0[(line * 3 + q) * NPP + pp];
#pragma unroll
        for (int is = 0; is < 3; ++is) {
            double2 a = make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < 3; ++q) dev::cfma_r(a, in[q], ms[is * 3 + q]);
            v1[pp * kNP + is + 3 * line] = a;
        }
    }
    __syncwarp();
    // theta: line = (is, ip) of pipe pp
    for (int l = lane; l < 15 * NPP; l += 32) {
        const int pp = l / 15, rem = l - pp * 15, is = rem % 3, ip = rem / 3;
        const double2* src = v1 + pp * kNP + is + 15 * ip;
        double2 in[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) in[q] = src[3 * q];
#pragma unroll
        for (int it = 0; it < 5; ++it) {
            double2 a = make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < 5; ++q) dev::cfma_r(a, in[q], ma[it * 5 + q]);
            v0[pp * kNP + is + 3 * it + 15 * ip] = a;
        }
    }
    __syncwarp();
    // phi: line = (is, it) of pipe pp
    for (int l = lane; l < 15 * NPP; l += 32) {
        const int pp = l / 15, rem = l - pp * 15;  // rem = is + 3 it
        const double2* src = v0 + pp * kNP + rem;
        double2 in[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) in[q] = src[15 * q];
#pragma unroll
        for (int ip = 0; ip < 5; ++ip) {
            double2 a = make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < 5; ++q) dev::cfma_r(a, in[q], ma[ip * 5 + q]);
            dst[pp * kNP + rem + 15 * ip] = a;
        }
    }
    __syncwarp();
}

}  // namespace pfill
}  // namespace ifgfb200
