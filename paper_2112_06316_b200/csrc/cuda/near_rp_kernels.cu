// Near-field, RP singular correction, combine and direct-sum kernels for sm_100a.
//
//  * weights      : a_m = phi_m J_m w_m gathered into Morton order (solver.cpp:87-88,
//                   ifgf.cpp:586-587)
//  * near_field   : level-D neighbour sum minus singular-patch exclusions and far-node
//                   corrections (solver.cpp:100-144); one thread per target, sources of the
//                   <=27 neighbour leaves read by the whole warp in lock step (broadcast).
//  * density_coeffs + rp_combine : per-patch 2-D Chebyshev coefficients of phi
//                   (rp.cpp:400-417) and the per-(target, patch) beta dot products
//                   (rp.cpp:421-451), one warp per target with coalesced beta streaming,
//                   fused with 1/2 phi + D - i gamma S (solver.cpp:152-156) and the
//                   Morton un-permute (ifgf.cpp:603-606).
//  * direct       : layer_potential_direct's regular part (rp.cpp:481-513), O(N^2).
#include <cstdlib>
#include <string>

#include "dev_common.cuh"
#include "kernels.cuh"

namespace ifgfb200 {
namespace {

using namespace dev;

constexpr int kNearThreads = 128;
constexpr int kMaxSing = 8;

__global__ void weights_kernel(int n, const std::uint32_t* __restrict__ perm,
                               const double2* __restrict__ phi, const double* __restrict__ jw_p,
                               double2* __restrict__ a_p) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    a_p[t] = cscale(phi[perm[t]], jw_p[t]);
}

__global__ void unpermute1_kernel(int n, const std::uint32_t* __restrict__ perm, const double2* __restrict__ in_m,
                                  double2* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    out[perm[t]] = in_m[t];
}

__global__ void unpermute_kernel(int n, const std::uint32_t* __restrict__ perm,
                                 const double2* __restrict__ Sp, const double2* __restrict__ Dp,
                                 double2* __restrict__ S, double2* __restrict__ D) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const std::uint32_t l = perm[t];
    S[l] = Sp[t];
    D[l] = Dp[t];
}

// G a and dG/dnu_y a for one pair, accumulated with sign sg
__device__ __forceinline__ void pair_kernels(double x, double y, double z, double yx, double yy,
                                             double yz, double nx, double ny, double nz, double2 a,
                                             double k, double sg, double2& accS, double2& accD) {
    const double dx = x - yx, dy = y - yy, dz = z - yz;
    const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
    const double inv = rsqrt_normal(r2);
    const double r = r2 * inv;
    double sn, cs;
    sincos_bounded(k * r, &sn, &cs);
    const double g = kInv4PiD * inv;
    const double2 ga = cmul(make_double2(cs * g, sn * g), a);  // G a = e^{ikr} a / (4 pi r)
    accS.x = fma(sg, ga.x, accS.x);
    accS.y = fma(sg, ga.y, accS.y);
    // dG/dnu_y a = (1 - ikr) G a <x - y, nu> / r^2
    const double dn = fma(dx, nx, fma(dy, ny, dz * nz));
    const double kr = k * r;
    const double f = sg * dn * (inv * inv);
    accD.x = fma(fma(kr, ga.y, ga.x), f, accD.x);
    accD.y = fma(fma(-kr, ga.x, ga.y), f, accD.y);
}

__global__ void __launch_bounds__(kNearThreads, 8)
near_kernel(NearDev N, PointsDev P, const double2* __restrict__ a_p, double k,
            double2* __restrict__ Sp, double2* __restrict__ Dp) {
    const int c = blockIdx.x;
    const int tb = N.chunk_box[c];
    if (N.leaf_active && !N.leaf_active[tb]) return;  // targets owned by another rank
    const int tbeg = int(N.beg[tb]);
    const int n_t = int(N.end[tb]) - tbeg;
    const int q = N.chunk_q0[c] + threadIdx.x;
    const bool act = q < n_t;
    if (__all_sync(0xffffffffu, !act)) return;  // whole warp past the box's targets (no barriers here)
    const int t = act ? tbeg + q : tbeg;
    const std::uint32_t l = N.perm[t];
    const double x = P.x[t], y = P.y[t], z = P.z[t];
    const int p0 = int(N.tpb[l]), p1 = int(N.tpb[l + 1]);
    const int nsing = p1 - p0;
    int sing[kMaxSing];
#pragma unroll
    for (int i = 0; i < kMaxSing; ++i) sing[i] = (i < nsing) ? N.pair_patch[p0 + i] : -1;
    double2 accS = make_double2(0.0, 0.0), accD = make_double2(0.0, 0.0);
    for (int j = N.nb_ptr[tb]; j < N.nb_ptr[tb + 1]; ++j) {
        const int nb = N.nb_idx[j];
        const int u1 = int(N.end[nb]);
        for (int u = int(N.beg[nb]); u < u1; ++u) {
            if (!act || u == t) continue;
            const int pq = N.patch_p[u];
            bool skip = false;
#pragma unroll
            for (int i = 0; i < kMaxSing; ++i) skip |= (sing[i] == pq);
            if (nsing > kMaxSing)
                for (int i = kMaxSing; i < nsing; ++i) skip |= (N.pair_patch[p0 + i] == pq);
            if (skip) continue;
            pair_kernels(x, y, z, P.x[u], P.y[u], P.z[u], P.nx[u], P.ny[u], P.nz[u], a_p[u], k, 1.0,
                         accS, accD);
        }
    }
    if (!act) return;
    // far-node corrections of the singular patches (solver.cpp:131-139)
    for (int p = p0; p < p1; ++p)
        for (std::uint32_t f = N.far_begin[p]; f < N.far_end[p]; ++f) {
            const int u = int(N.far_pos[f]);
            pair_kernels(x, y, z, P.x[u], P.y[u], P.z[u], P.nx[u], P.ny[u], P.nz[u], a_p[u], k, -1.0,
                         accS, accD);
        }
    Sp[t] = cadd(Sp[t], accS);
    Dp[t] = cadd(Dp[t], accD);
}

// Warp per target, lanes over sources: each warp screens its target's neighbourhood 32
// candidates at a time (self and singular-patch exclusions, solver.cpp:117-124), appends the
// valid sources to a per-warp queue (ballot) and evaluates full 32-lane batches of pairs, so
// excluded pairs cost no lane time; the far-node corrections (solver.cpp:131-139) run
// lane-parallel, and a fixed shuffle tree sums the lanes (deterministic).
// MODE 1 / 2 run the same screening once at setup and count / write the compacted sources
// per target (the near lists below), in exactly the order the batches would take them.
constexpr int kNearWarps = 4;
template <int MODE>
__global__ void __launch_bounds__(32 * kNearWarps, 8)
near_warp_kernel(NearDev N, PointsDev P, const double2* __restrict__ a_p, double k, double2* __restrict__ Sp,
                 double2* __restrict__ Dp, std::int32_t* __restrict__ out) {
    __shared__ int queue[kNearWarps][64];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int t = blockIdx.x * kNearWarps + w;  // Morton target
    if (t >= N.n) return;
    const int tb = N.leaf_of_m[t];
    if (N.leaf_active && !N.leaf_active[tb]) {  // target owned by another rank
        if (MODE == 1 && lane == 0) out[t] = 0;
        return;
    }
    const std::uint32_t l = N.perm[t];
    const double x = P.x[t], y = P.y[t], z = P.z[t];
    const int p0 = int(N.tpb[l]), p1 = int(N.tpb[l + 1]);
    const int nsing = p1 - p0;
    int sing[kMaxSing];
#pragma unroll
    for (int i = 0; i < kMaxSing; ++i) sing[i] = (i < nsing) ? N.pair_patch[p0 + i] : -1;
    int* q = queue[w];
    int qn = 0;
    std::int64_t written = MODE == 2 ? N.list_off[t] : 0;
    double2 accS = make_double2(0.0, 0.0), accD = make_double2(0.0, 0.0);
    for (int j = N.nb_ptr[tb]; j < N.nb_ptr[tb + 1]; ++j) {
        const int nb = N.nb_idx[j];
        const int u1 = int(N.end[nb]);
        for (int ub = int(N.beg[nb]); ub < u1; ub += 32) {
            const int u = ub + lane;
            bool ok = u < u1 && u != t;
            if (ok) {
                const int pq = N.patch_p[u];
#pragma unroll
                for (int i = 0; i < kMaxSing; ++i) ok &= (sing[i] != pq);
                if (nsing > kMaxSing)
                    for (int i = kMaxSing; i < nsing; ++i) ok &= (N.pair_patch[p0 + i] != pq);
            }
            const unsigned m = __ballot_sync(0xffffffffu, ok);
            if (ok) q[qn + __popc(m & ((1u << lane) - 1u))] = u;
            qn += __popc(m);
            __syncwarp();
            if (qn >= 32) {
                const int v = q[lane];
                if constexpr (MODE == 0)
                    pair_kernels(x, y, z, P.x[v], P.y[v], P.z[v], P.nx[v], P.ny[v], P.nz[v], a_p[v], k, 1.0, accS, accD);
                if constexpr (MODE == 2) N.list_src[written + lane] = v;
                written += 32;
                __syncwarp();
                if (lane < qn - 32) q[lane] = q[lane + 32];
                qn -= 32;
                __syncwarp();
            }
        }
    }
    if constexpr (MODE == 1) {
        if (lane == 0) out[t] = int(written) + qn;
        return;
    }
    if (lane < qn) {
        const int v = q[lane];
        if constexpr (MODE == 0)
            pair_kernels(x, y, z, P.x[v], P.y[v], P.z[v], P.nx[v], P.ny[v], P.nz[v], a_p[v], k, 1.0, accS, accD);
        if constexpr (MODE == 2) N.list_src[written + lane] = v;
    }
    if constexpr (MODE == 0) {
        for (int p = p0; p < p1; ++p)
            for (std::uint32_t f = N.far_begin[p] + lane; f < N.far_end[p]; f += 32) {
                const int u = int(N.far_pos[f]);
                pair_kernels(x, y, z, P.x[u], P.y[u], P.z[u], P.nx[u], P.ny[u], P.nz[u], a_p[u], k, -1.0, accS, accD);
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            accS.x += __shfl_xor_sync(0xffffffffu, accS.x, o);
            accS.y += __shfl_xor_sync(0xffffffffu, accS.y, o);
            accD.x += __shfl_xor_sync(0xffffffffu, accD.x, o);
            accD.y += __shfl_xor_sync(0xffffffffu, accD.y, o);
        }
        if (lane == 0) {
            Sp[t] = cadd(Sp[t], accS);
            Dp[t] = cadd(Dp[t], accD);
        }
    }
}

// pair_kernels with the source's geometry from its packed 48-byte row
__device__ __forceinline__ void near_pair(const double2* __restrict__ geo, int v, double x, double y, double z,
                                          const double2* __restrict__ a_p, double k, double sg, double2& accS,
                                          double2& accD) {
    const double2 g0 = __ldg(geo + 3 * v), g1 = __ldg(geo + 3 * v + 1), g2 = __ldg(geo + 3 * v + 2);
    pair_kernels(x, y, z, g0.x, g0.y, g1.x, g1.y, g2.x, g2.y, a_p[v], k, sg, accS, accD);
}

// Warp per target over its precomputed near list (the compacted sources of near_warp_kernel,
// built once at setup): lane i takes list entries i, i + 32, ..., the same sources in the same
// order as the screening kernel, so the sums are bitwise equal to it without the per-apply
// screening (ballots, patch tests, queue traffic).
#ifndef IFGF_NEAR_UNROLL
#define IFGF_NEAR_UNROLL 2
#endif
#ifndef IFGF_NEAR_MINB
#define IFGF_NEAR_MINB 8
#endif
constexpr int kNearUnroll = IFGF_NEAR_UNROLL;
__global__ void __launch_bounds__(32 * kNearWarps, IFGF_NEAR_MINB)
near_list_kernel(NearDev N, PointsDev P, const double2* __restrict__ a_p, double k, double2* __restrict__ Sp,
                 double2* __restrict__ Dp) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int t = blockIdx.x * kNearWarps + w;  // Morton target
    if (t >= N.n) return;
    if (N.leaf_active && !N.leaf_active[N.leaf_of_m[t]]) return;
    const std::uint32_t l = N.perm[t];
    const double x = P.x[t], y = P.y[t], z = P.z[t];
    double2 accS = make_double2(0.0, 0.0), accD = make_double2(0.0, 0.0);
    const std::int64_t e = N.list_off[t + 1];
#pragma unroll kNearUnroll
    for (std::int64_t i = N.list_off[t] + lane; i < e; i += 32) {
        const int v = N.list_src[i];
        near_pair(N.geo, v, x, y, z, a_p, k, 1.0, accS, accD);
    }
    const int p0 = int(N.tpb[l]), p1 = int(N.tpb[l + 1]);
    for (int p = p0; p < p1; ++p)
        for (std::uint32_t f = N.far_begin[p] + lane; f < N.far_end[p]; f += 32) {
            const int u = int(N.far_pos[f]);
            near_pair(N.geo, u, x, y, z, a_p, k, -1.0, accS, accD);
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        accS.x += __shfl_xor_sync(0xffffffffu, accS.x, o);
        accS.y += __shfl_xor_sync(0xffffffffu, accS.y, o);
        accD.x += __shfl_xor_sync(0xffffffffu, accD.x, o);
        accD.y += __shfl_xor_sync(0xffffffffu, accD.y, o);
    }
    if (lane == 0) {
        Sp[t] = cadd(Sp[t], accS);
        Dp[t] = cadd(Dp[t], accD);
    }
}

// TARGET PAIRS: consecutive Morton targets t0, t0 + 1 of one leaf share their neighbourhood
// and, almost always, their singular patches, so one union list serves both: entry = source |
// m << 30 with bit 0 of m set when the pair (t0, source) is evaluated and bit 1 for t0 + 1 (the
// screening of near_warp_kernel applied to each). The evaluation kernel loads each source row
// once for both targets: half the gathers and half the list bytes of the single-target lists.
// Item w: t0 = pitem[w] & 0x7fffffff, bit 31 set when t0 is a leaf's last, unpaired target.
// MODE 1 counts, MODE 2 writes the lists (in neighbourhood order).
template <int MODE>
__global__ void __launch_bounds__(32 * kNearWarps, 8)
near_pair_screen_kernel(NearDev N, std::int32_t* __restrict__ counts) {
    __shared__ unsigned queue[kNearWarps][64];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int item = blockIdx.x * kNearWarps + w;
    if (item >= N.npitem) return;
    const std::uint32_t pi = std::uint32_t(N.pitem[item]);
    const int t0 = int(pi & 0x7fffffffu);
    const bool two = !(pi >> 31);
    const int tb = N.leaf_of_m[t0];
    if (N.leaf_active && !N.leaf_active[tb]) {
        if (MODE == 1 && lane == 0) counts[item] = 0;
        return;
    }
    int sing0[kMaxSing], sing1[kMaxSing];
    const std::uint32_t l0 = N.perm[t0];
    const int a0 = int(N.tpb[l0]), n0 = int(N.tpb[l0 + 1]) - a0;
    int a1 = 0, n1 = 0;
    if (two) {
        const std::uint32_t l1 = N.perm[t0 + 1];
        a1 = int(N.tpb[l1]);
        n1 = int(N.tpb[l1 + 1]) - a1;
    }
#pragma unroll
    for (int i = 0; i < kMaxSing; ++i) {
        sing0[i] = i < n0 ? N.pair_patch[a0 + i] : -1;
        sing1[i] = i < n1 ? N.pair_patch[a1 + i] : -1;
    }
    unsigned* q = queue[w];
    int qn = 0;
    std::int64_t written = MODE == 2 ? N.plist_off[item] : 0;
    for (int j = N.nb_ptr[tb]; j < N.nb_ptr[tb + 1]; ++j) {
        const int nb = N.nb_idx[j];
        const int u1 = int(N.end[nb]);
        for (int ub = int(N.beg[nb]); ub < u1; ub += 32) {
            const int u = ub + lane;
            unsigned m = 0;
            if (u < u1) {
                const int pq = N.patch_p[u];
                bool ok0 = u != t0, ok1 = two && u != t0 + 1;
#pragma unroll
                for (int i = 0; i < kMaxSing; ++i) {
                    ok0 &= (sing0[i] != pq);
                    ok1 &= (sing1[i] != pq);
                }
                for (int i = kMaxSing; i < n0; ++i) ok0 &= (N.pair_patch[a0 + i] != pq);
                for (int i = kMaxSing; i < n1; ++i) ok1 &= (N.pair_patch[a1 + i] != pq);
                m = (ok0 ? 1u : 0u) | (ok1 ? 2u : 0u);
            }
            const unsigned b = __ballot_sync(0xffffffffu, m != 0);
            if (m) q[qn + __popc(b & ((1u << lane) - 1u))] = std::uint32_t(u) | (m << 30);
            qn += __popc(b);
            __syncwarp();
            if (qn >= 32) {
                if constexpr (MODE == 2) N.plist_src[written + lane] = q[lane];
                written += 32;
                __syncwarp();
                if (lane < qn - 32) q[lane] = q[lane + 32];
                qn -= 32;
                __syncwarp();
            }
        }
    }
    if constexpr (MODE == 1) {
        if (lane == 0) counts[item] = int(written) + qn;
    } else {
        if (lane < qn) N.plist_src[written + lane] = q[lane];
    }
}

// one target's far-node corrections (solver.cpp:131-139), lane-parallel
__device__ __forceinline__ void near_far_nodes(const NearDev& N, int t, double x, double y, double z,
                                               const double2* __restrict__ a_p, double k, double2& accS,
                                               double2& accD) {
    const std::uint32_t l = N.perm[t];
    const int p0 = int(N.tpb[l]), p1 = int(N.tpb[l + 1]);
    const int lane = threadIdx.x & 31;
    for (int p = p0; p < p1; ++p)
        for (std::uint32_t f = N.far_begin[p] + lane; f < N.far_end[p]; f += 32) {
            const int u = int(N.far_pos[f]);
            near_pair(N.geo, u, x, y, z, a_p, k, -1.0, accS, accD);
        }
}

__device__ __forceinline__ void warp_sum4(double2& a, double2& b) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
        a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
        b.x += __shfl_xor_sync(0xffffffffu, b.x, o);
        b.y += __shfl_xor_sync(0xffffffffu, b.y, o);
    }
}

// warp per target pair over its union list: one source row, up to two pairs
// 8 CTAs (32 warps) per SM at 64 registers (a few spills) and 3 list entries in flight per
// lane measured best (cfg2 near 2.46 -> 2.21 ms; 6 CTAs at 78 registers, unroll 2: 2.46 ms;
// 10 CTAs: 2.63 ms)
#ifndef IFGF_NEAR_PAIR_MINB
#define IFGF_NEAR_PAIR_MINB 8
#endif
#ifndef IFGF_NEAR_PAIR_UNROLL
#define IFGF_NEAR_PAIR_UNROLL 3
#endif
constexpr int kNearPairUnroll = IFGF_NEAR_PAIR_UNROLL;
__global__ void __launch_bounds__(32 * kNearWarps, IFGF_NEAR_PAIR_MINB)
near_pair_kernel(NearDev N, PointsDev P, const double2* __restrict__ a_p, double k, double2* __restrict__ Sp,
                 double2* __restrict__ Dp) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int item = blockIdx.x * kNearWarps + w;
    if (item >= N.npitem) return;
    const std::uint32_t pi = std::uint32_t(N.pitem[item]);
    const int t0 = int(pi & 0x7fffffffu);
    const bool two = !(pi >> 31);
    if (N.leaf_active && !N.leaf_active[N.leaf_of_m[t0]]) return;
    const int t1 = two ? t0 + 1 : t0;
    const double x0 = P.x[t0], y0 = P.y[t0], z0 = P.z[t0];
    const double x1 = P.x[t1], y1 = P.y[t1], z1 = P.z[t1];
    double2 s0 = make_double2(0.0, 0.0), d0 = s0, s1 = s0, d1 = s0;
    const std::int64_t e = N.plist_off[item + 1];
#pragma unroll kNearPairUnroll
    for (std::int64_t i = N.plist_off[item] + lane; i < e; i += 32) {
        const std::uint32_t ent = N.plist_src[i];
        const int v = int(ent & 0x3fffffffu);
        const double2 g0 = __ldg(N.geo + 3 * v), g1 = __ldg(N.geo + 3 * v + 1), g2 = __ldg(N.geo + 3 * v + 2);
        const double2 a = a_p[v];
        if (ent & (1u << 30)) pair_kernels(x0, y0, z0, g0.x, g0.y, g1.x, g1.y, g2.x, g2.y, a, k, 1.0, s0, d0);
        if (ent & (2u << 30)) pair_kernels(x1, y1, z1, g0.x, g0.y, g1.x, g1.y, g2.x, g2.y, a, k, 1.0, s1, d1);
    }
    near_far_nodes(N, t0, x0, y0, z0, a_p, k, s0, d0);
    warp_sum4(s0, d0);
    if (lane == 0) {
        Sp[t0] = cadd(Sp[t0], s0);
        Dp[t0] = cadd(Dp[t0], d0);
    }
    if (two) {
        near_far_nodes(N, t1, x1, y1, z1, a_p, k, s1, d1);
        warp_sum4(s1, d1);
        if (lane == 0) {
            Sp[t1] = cadd(Sp[t1], s1);
            Dp[t1] = cadd(Dp[t1], d1);
        }
    }
}

// Warp per target over its neighbourhood's PATCH RUNS (no per-pair lists): a run whose patch
// is singular for the target is dropped whole (warp-uniform), the target itself is cut out
// of its run, and lane i takes entries i, i + 32, ... of the remaining sequence — the same
// sources in the same order as the near lists / the screening kernel, so the sums are
// bitwise equal to theirs, without the lists' 4 bytes per pair in HBM (cfg3: 27 GB) and with
// consecutive (coalesced) source rows. Runs are taken 32 at a time: lanes load a window of
// runs, a warp scan gives their offsets, and each lane walks its entries with a cursor.
__global__ void __launch_bounds__(32 * kNearWarps, IFGF_NEAR_MINB)
near_run_kernel(NearDev N, PointsDev P, const double2* __restrict__ a_p, double k, double2* __restrict__ Sp,
                double2* __restrict__ Dp) {
    __shared__ int rs_s[kNearWarps][33], rb_s[kNearWarps][33], re_s[kNearWarps][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int t = blockIdx.x * kNearWarps + w;  // Morton target
    if (t >= N.n) return;
    const int tb = N.leaf_of_m[t];
    if (N.leaf_active && !N.leaf_active[tb]) return;
    const std::uint32_t l = N.perm[t];
    const double x = P.x[t], y = P.y[t], z = P.z[t];
    const int p0 = int(N.tpb[l]), p1 = int(N.tpb[l + 1]);
    const int nsing = p1 - p0;
    int sing[kMaxSing];
#pragma unroll
    for (int i = 0; i < kMaxSing; ++i) sing[i] = (i < nsing) ? N.pair_patch[p0 + i] : -1;
    double2 accS = make_double2(0.0, 0.0), accD = make_double2(0.0, 0.0);
    const int r0 = N.run_ptr[tb], r1 = N.run_ptr[tb + 1];
    int phase = 0;  // (entries before this window) mod 32
    for (int wr = r0; wr < r1; wr += 32) {
        const int r = wr + lane;
        int st = 0, len = 0;
        bool self = false;
        if (r < r1) {
            st = N.run_start[r];
            len = N.run_len[r];
            const int pq = N.run_patch[r];
            bool ok = true;
#pragma unroll
            for (int i = 0; i < kMaxSing; ++i) ok &= (sing[i] != pq);
            if (nsing > kMaxSing)
                for (int i = kMaxSing; i < nsing; ++i) ok &= (N.pair_patch[p0 + i] != pq);
            if (!ok) {
                len = 0;
            } else if (t >= st && t < st + len) {
                self = true;
                len -= 1;
            }
        }
        int inc = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        const int tot = __shfl_sync(0xffffffffu, inc, 31);
        const unsigned selfm = __ballot_sync(0xffffffffu, self);
        rs_s[w][lane] = st;
        rb_s[w][lane] = inc - len;
        re_s[w][lane] = inc;
        if (lane == 0) re_s[w][32] = 0x7fffffff;  // cursor sentinel
        __syncwarp();
        int cur = 0, cst = rs_s[w][0], cb = rb_s[w][0], ce = re_s[w][0];
        bool cself = selfm & 1u;
#pragma unroll 2
        for (int e = (lane - phase) & 31; e < tot; e += 32) {
            while (ce <= e) {  // advance to the run holding entry e (skips emptied runs)
                ++cur;
                cst = rs_s[w][cur];
                cb = rb_s[w][cur];
                ce = re_s[w][cur];
                cself = (selfm >> cur) & 1u;
            }
            int v = cst + (e - cb);
            if (cself && v >= t) ++v;  // the target itself is not in the sequence
            near_pair(N.geo, v, x, y, z, a_p, k, 1.0, accS, accD);
        }
        phase = (phase + tot) & 31;
        __syncwarp();
    }
    for (int p = p0; p < p1; ++p)
        for (std::uint32_t f = N.far_begin[p] + lane; f < N.far_end[p]; f += 32) {
            const int u = int(N.far_pos[f]);
            near_pair(N.geo, u, x, y, z, a_p, k, -1.0, accS, accD);
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        accS.x += __shfl_xor_sync(0xffffffffu, accS.x, o);
        accS.y += __shfl_xor_sync(0xffffffffu, accS.y, o);
        accD.x += __shfl_xor_sync(0xffffffffu, accD.x, o);
        accD.y += __shfl_xor_sync(0xffffffffu, accD.y, o);
    }
    if (lane == 0) {
        Sp[t] = cadd(Sp[t], accS);
        Dp[t] = cadd(Dp[t], accD);
    }
}

// one CTA per patch: a^q = Mv (Mu phi_q) along u then v (chebyshev.cpp:43-61)
__global__ void density_coeffs_kernel(RpDev R, const double2* __restrict__ phi,
                                      double2* __restrict__ coeffs) {
    extern __shared__ double2 tmp[];
    const int q = blockIdx.x;
    const int nu = R.patch_nu[q], nv = R.patch_nv[q];
    const std::int64_t st = R.patch_start[q];
    const double* Mu = R.mats + R.mat_off[2 * q];
    const double* Mv = R.mats + R.mat_off[2 * q + 1];
    const int nn = nu * nv;
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
        const int i = e % nu, j = e / nu;
        double2 acc = make_double2(0.0, 0.0);
        for (int kk = 0; kk < nu; ++kk) cfma_r(acc, phi[st + kk + std::int64_t(nu) * j], Mu[i * nu + kk]);
        tmp[e] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
        const int i = e % nu, j = e / nu;
        double2 acc = make_double2(0.0, 0.0);
        for (int kk = 0; kk < nv; ++kk) cfma_r(acc, tmp[i + nu * kk], Mv[j * nv + kk]);
        coeffs[st + e] = acc;
    }
}

// one singular pair's beta rows against its patch's coefficients, lanes strided; 16 x 16
// patches (every bench config) take a fixed, unrolled stream (more loads in flight)
__device__ __forceinline__ void rp_pair_stream(const double2* __restrict__ a, const double2* __restrict__ bs,
                                               const double2* __restrict__ bd, int nn, int lane, double2& as,
                                               double2& ad) {
    if (nn == 256) {
#pragma unroll
        for (int i = lane; i < 256; i += 32) {
            const double2 ai = a[i];
            cfma(as, ai, __ldcs(bs + i));
            cfma(ad, ai, __ldcs(bd + i));
        }
    } else {
        for (int i = lane; i < nn; i += 32) {
            const double2 ai = a[i];
            cfma(as, ai, __ldcs(bs + i));
            cfma(ad, ai, __ldcs(bd + i));
        }
    }
}

__global__ void rp_combine_kernel(RpDev R, const double2* __restrict__ coeffs,
                                  const double2* __restrict__ phi, const double2* __restrict__ Sp,
                                  const double2* __restrict__ Dp, double gamma,
                                  double2* __restrict__ out, double2* __restrict__ S,
                                  double2* __restrict__ D) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= R.n) return;
    const int l = warp;
    const std::uint32_t tm = R.pos[l];
    if (tm < R.own_lo || tm >= R.own_hi) return;  // target owned by another rank
    double2 as = make_double2(0.0, 0.0), ad = make_double2(0.0, 0.0);
    for (std::uint32_t p = R.tpb[l]; p < R.tpb[l + 1]; ++p) {
        const int q = R.pair_patch[p];
        const int nn = R.patch_nu[q] * R.patch_nv[q];
        const double2* a = coeffs + R.patch_start[q];
        const double2* bs = R.beta_s + R.beta_off[p];
        const double2* bd = R.beta_d + R.beta_off[p];
        rp_pair_stream(a, bs, bd, nn, lane, as, ad);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        as.x += __shfl_xor_sync(0xffffffffu, as.x, o);
        as.y += __shfl_xor_sync(0xffffffffu, as.y, o);
        ad.x += __shfl_xor_sync(0xffffffffu, ad.x, o);
        ad.y += __shfl_xor_sync(0xffffffffu, ad.y, o);
    }
    if (lane != 0) return;
    const int t = int(R.pos[l]);
    const double2 s = cadd(Sp[t], as);
    const double2 d = cadd(Dp[t], ad);
    const double2 f = phi[l];
    const double2 o = make_double2(0.5 * f.x + d.x + gamma * s.y, 0.5 * f.y + d.y - gamma * s.x);
    if (R.out_m) R.out_m[t] = o;
    else out[l] = o;
    if (S) S[l] = s;
    if (D) D[l] = d;
}

// RP correction alone, accumulated into the Morton-order near-field buffers (Sn, Dn): the
// same warp-per-target beta streaming as rp_combine_kernel, for the side stream of the
// concurrent apply
__global__ void rp_accum_kernel(RpDev R, const double2* __restrict__ coeffs, double2* __restrict__ Sn,
                                double2* __restrict__ Dn) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= R.n) return;
    const int l = warp;
    const std::uint32_t tm = R.pos[l];
    if (tm < R.own_lo || tm >= R.own_hi) return;  // target owned by another rank
    double2 as = make_double2(0.0, 0.0), ad = make_double2(0.0, 0.0);
    for (std::uint32_t p = R.tpb[l]; p < R.tpb[l + 1]; ++p) {
        const int q = R.pair_patch[p];
        const int nn = R.patch_nu[q] * R.patch_nv[q];
        const double2* a = coeffs + R.patch_start[q];
        const double2* bs = R.beta_s + R.beta_off[p];
        const double2* bd = R.beta_d + R.beta_off[p];
        rp_pair_stream(a, bs, bd, nn, lane, as, ad);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        as.x += __shfl_xor_sync(0xffffffffu, as.x, o);
        as.y += __shfl_xor_sync(0xffffffffu, as.y, o);
        ad.x += __shfl_xor_sync(0xffffffffu, ad.x, o);
        ad.y += __shfl_xor_sync(0xffffffffu, ad.y, o);
    }
    if (lane != 0) return;
    Sn[tm] = cadd(Sn[tm], as);
    Dn[tm] = cadd(Dn[tm], ad);
}

// out = 1/2 phi + D - i gamma S with S = far + (near + RP), per original target
// (solver.cpp:152-156, ifgf.cpp:603-606 un-permute)
__global__ void combine_kernel(RpDev R, const double2* __restrict__ phi, const double2* __restrict__ Sp,
                               const double2* __restrict__ Dp, const double2* __restrict__ Sn,
                               const double2* __restrict__ Dn, double gamma, double2* __restrict__ out,
                               double2* __restrict__ S, double2* __restrict__ D) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= R.n) return;
    const std::uint32_t t = R.pos[l];
    if (t < R.own_lo || t >= R.own_hi) return;
    const double2 s = cadd(Sp[t], Sn[t]);
    const double2 d = cadd(Dp[t], Dn[t]);
    const double2 f = phi[l];
    const double2 o = make_double2(0.5 * f.x + d.x + gamma * s.y, 0.5 * f.y + d.y - gamma * s.x);
    if (R.out_m) R.out_m[t] = o;
    else out[l] = o;
    if (S) S[l] = s;
    if (D) D[l] = d;
}

constexpr int kDirectThreads = 256;

__global__ void __launch_bounds__(kDirectThreads)
direct_kernel(DirectDev Dd, const double2* __restrict__ phi, double k, double2* __restrict__ S,
              double2* __restrict__ D) {
    __shared__ double sx[kDirectThreads], sy[kDirectThreads], sz[kDirectThreads];
    __shared__ double snx[kDirectThreads], sny[kDirectThreads], snz[kDirectThreads];
    __shared__ double2 sa[kDirectThreads];
    __shared__ int spq[kDirectThreads];
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    const bool act = l < Dd.n;
    double x = 0, y = 0, z = 0;
    int sing[kMaxSing];
    int p0 = 0, nsing = 0;
    if (act) {
        x = Dd.x[l];
        y = Dd.y[l];
        z = Dd.z[l];
        p0 = int(Dd.tpb[l]);
        nsing = int(Dd.tpb[l + 1]) - p0;
    }
#pragma unroll
    for (int i = 0; i < kMaxSing; ++i) sing[i] = (i < nsing) ? Dd.pair_patch[p0 + i] : -1;
    double2 accS = make_double2(0.0, 0.0), accD = make_double2(0.0, 0.0);
    for (int m0 = 0; m0 < Dd.n; m0 += kDirectThreads) {
        __syncthreads();
        const int m = m0 + threadIdx.x;
        if (m < Dd.n) {
            sx[threadIdx.x] = Dd.x[m];
            sy[threadIdx.x] = Dd.y[m];
            sz[threadIdx.x] = Dd.z[m];
            snx[threadIdx.x] = Dd.nx[m];
            sny[threadIdx.x] = Dd.ny[m];
            snz[threadIdx.x] = Dd.nz[m];
            sa[threadIdx.x] = cscale(phi[m], Dd.jw[m]);
            spq[threadIdx.x] = Dd.patch_of[m];
        }
        __syncthreads();
        if (!act) continue;
        const int cnt = min(kDirectThreads, Dd.n - m0);
        for (int j = 0; j < cnt; ++j) {
            if (m0 + j == l) continue;
            const int pq = spq[j];
            bool skip = false;
#pragma unroll
            for (int i = 0; i < kMaxSing; ++i) skip |= (sing[i] == pq);
            if (nsing > kMaxSing)
                for (int i = kMaxSing; i < nsing; ++i) skip |= (Dd.pair_patch[p0 + i] == pq);
            if (skip) continue;
            pair_kernels(x, y, z, sx[j], sy[j], sz[j], snx[j], sny[j], snz[j], sa[j], k, 1.0, accS, accD);
        }
    }
    if (!act) return;
    S[l] = accS;
    D[l] = accD;
}

}  // namespace

void launch_weights(int n, const std::uint32_t* perm, const double2* phi, const double* jw_p,
                    double2* a_p, cudaStream_t st) {
    if (n == 0) return;
    weights_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, perm, phi, jw_p, a_p);
    IFGF_CUDA(cudaGetLastError());
}

void launch_unpermute(int n, const std::uint32_t* perm, const double2* Sp, const double2* Dp,
                      double2* S, double2* D, cudaStream_t st) {
    if (n == 0) return;
    unpermute_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, perm, Sp, Dp, S, D);
    IFGF_CUDA(cudaGetLastError());
}

void launch_unpermute1(int n, const std::uint32_t* perm, const double2* in_m, double2* out, cudaStream_t st) {
    if (n == 0) return;
    unpermute1_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, perm, in_m, out);
    IFGF_CUDA(cudaGetLastError());
}

void launch_near_field(const NearDev& N, const PointsDev& P, const double2* a_p, double k,
                       double2* Sp, double2* Dp, cudaStream_t st) {
    if (N.nchunk == 0) return;
    static const bool per_thread = [] {
        const char* e = std::getenv("IFGF_NEAR");
        return e && std::string(e) == "thread";
    }();
    const int grid = (N.n + kNearWarps - 1) / kNearWarps;
    if (per_thread || !N.leaf_of_m)
        near_kernel<<<N.nchunk, kNearThreads, 0, st>>>(N, P, a_p, k, Sp, Dp);
    else if (N.plist_off)
        near_pair_kernel<<<(N.npitem + kNearWarps - 1) / kNearWarps, 32 * kNearWarps, 0, st>>>(N, P, a_p, k, Sp, Dp);
    else if (N.list_off)
        near_list_kernel<<<grid, 32 * kNearWarps, 0, st>>>(N, P, a_p, k, Sp, Dp);
    else if (N.run_ptr)
        near_run_kernel<<<grid, 32 * kNearWarps, 0, st>>>(N, P, a_p, k, Sp, Dp);
    else
        near_warp_kernel<0><<<grid, 32 * kNearWarps, 0, st>>>(N, P, a_p, k, Sp, Dp, nullptr);
    IFGF_CUDA(cudaGetLastError());
}

void launch_near_list_count(const NearDev& N, const PointsDev& P, std::int32_t* counts, cudaStream_t st) {
    if (N.n == 0 || !N.leaf_of_m) return;
    near_warp_kernel<1><<<(N.n + kNearWarps - 1) / kNearWarps, 32 * kNearWarps, 0, st>>>(N, P, nullptr, 0.0, nullptr,
                                                                                         nullptr, counts);
    IFGF_CUDA(cudaGetLastError());
}

void launch_near_pair_lists(const NearDev& N, std::int32_t* counts, cudaStream_t st) {
    if (N.npitem == 0 || !N.leaf_of_m) return;
    const int grid = (N.npitem + kNearWarps - 1) / kNearWarps;
    if (counts)
        near_pair_screen_kernel<1><<<grid, 32 * kNearWarps, 0, st>>>(N, counts);
    else
        near_pair_screen_kernel<2><<<grid, 32 * kNearWarps, 0, st>>>(N, nullptr);
    IFGF_CUDA(cudaGetLastError());
}

void launch_near_list_fill(const NearDev& N, const PointsDev& P, cudaStream_t st) {
    if (N.n == 0 || !N.leaf_of_m || !N.list_off) return;
    near_warp_kernel<2><<<(N.n + kNearWarps - 1) / kNearWarps, 32 * kNearWarps, 0, st>>>(N, P, nullptr, 0.0, nullptr,
                                                                                         nullptr, nullptr);
    IFGF_CUDA(cudaGetLastError());
}

void launch_density_coeffs(const RpDev& R, const double2* phi, double2* coeffs, cudaStream_t st) {
    if (R.npatch == 0) return;
    const int threads = R.max_nn >= 256 ? 256 : ((R.max_nn + 31) / 32) * 32;
    density_coeffs_kernel<<<R.npatch, threads, std::size_t(R.max_nn) * sizeof(double2), st>>>(R, phi, coeffs);
    IFGF_CUDA(cudaGetLastError());
}

void launch_rp_combine(const RpDev& R, const double2* coeffs, const double2* phi,
                       const double2* Sp, const double2* Dp, double gamma, double2* out,
                       double2* S, double2* D, cudaStream_t st) {
    if (R.n == 0) return;
    const int threads = 256;
    const long warps = R.n;
    const int grid = int((warps * 32 + threads - 1) / threads);
    rp_combine_kernel<<<grid, threads, 0, st>>>(R, coeffs, phi, Sp, Dp, gamma, out, S, D);
    IFGF_CUDA(cudaGetLastError());
}

void launch_rp_accum(const RpDev& R, const double2* coeffs, double2* Sn, double2* Dn, cudaStream_t st) {
    if (R.n == 0) return;
    const int threads = 256;
    rp_accum_kernel<<<int((long(R.n) * 32 + threads - 1) / threads), threads, 0, st>>>(R, coeffs, Sn, Dn);
    IFGF_CUDA(cudaGetLastError());
}

void launch_combine(const RpDev& R, const double2* phi, const double2* Sp, const double2* Dp, const double2* Sn,
                    const double2* Dn, double gamma, double2* out, double2* S, double2* D, cudaStream_t st) {
    if (R.n == 0) return;
    combine_kernel<<<(R.n + 255) / 256, 256, 0, st>>>(R, phi, Sp, Dp, Sn, Dn, gamma, out, S, D);
    IFGF_CUDA(cudaGetLastError());
}

void launch_direct(const DirectDev& Dd, const double2* phi, double k, double2* S, double2* D,
                   cudaStream_t st) {
    if (Dd.n == 0) return;
    direct_kernel<<<(Dd.n + kDirectThreads - 1) / kDirectThreads, kDirectThreads, 0, st>>>(Dd, phi, k, S, D);
    IFGF_CUDA(cudaGetLastError());
}

}  // namespace ifgfb200
