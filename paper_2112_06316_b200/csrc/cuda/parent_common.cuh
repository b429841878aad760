// Child -> parent pipe combinations of the parent fill (ifgf.cpp:525-555), shared by the
// tensor-core parent kernels (parent_tc.cu: one warp per parent segment; parent_cb.cu:
// parent segments of one cone cell batched into small GEMMs).
#pragma once

#include <initializer_list>

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


}  // namespace pfill
}  // namespace ifgfb200
