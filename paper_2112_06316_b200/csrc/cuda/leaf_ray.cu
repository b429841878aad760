// Level-D fill (ifgf.cpp:312-391) with one thread per interpolation RAY: the ps = 3 radial
// nodes of a segment share the direction x^ = (sin th cos ph, sin th sin ph, cos th), so per
// (ray, source) the projections x^.dy and x^.n are formed once and each radial node needs
//   |v|^2 = 1 + sigma (sigma |dy|^2 - 2 x^.dy),   sigma = s/h
//   arg = k h/s (|v| - 1) with |v| - 1 = fma(|v|^2, 1/|v|, -1) (one rounding; the
//         reference's (|v|^2-1)/(|v|+1) has the same ~1e-16 absolute error)
//   v.n = x^.n - sigma dy.n
// Sources are staged in shared memory with |dy|^2 and dy.n precomputed; a CTA works on an
// item of up to 10 segments of at most two boxes. The 3x5x5
// value->coefficient transform runs in shared memory before the store, as in the per-node
// kernel. Equal to the reference to rounding (the reference forms |v|^2-1 from |v|^2).
#include "ifgf_device.cuh"
#include "kernels.cuh"

namespace ifgfb200 {
namespace {

using namespace dev;
using namespace ifgfdev;

constexpr int kThreads = 256;
constexpr int kTile = 256;
constexpr int kPS = 3;

// pipe sets carried by the leaf store: F0..F2 factor codes (0 = absent)
template <int F0, int F1, int F2>
struct PipeSet {
    static constexpr int n = (F0 ? 1 : 0) + (F1 ? 1 : 0) + (F2 ? 1 : 0);
    __device__ static constexpr int f(int i) { return i == 0 ? F0 : (i == 1 ? F1 : F2); }
};

// One CTA per work item: up to G = kThreads / NRAY consecutive segments of at most two leaf
// boxes (host: Engine leaf items), one thread per ray. Items pack the last segments of a box
// with the first of the next one, so a box's segment count need not be a multiple of G to
// keep the threads busy. A box with more than kTile sources gets items of its own and
// streams its sources through the tile in several passes.
template <class PSET>
__global__ void __launch_bounds__(kThreads, 2)
leaf_ray_kernel(LevelDev L, PointsDev P, const double2* __restrict__ a_p, double k,
                const double* __restrict__ Ms, const double* __restrict__ Ma, double2* __restrict__ store) {
    constexpr int NP = PSET::n;
    extern __shared__ double smem[];
    const int item = blockIdx.x;
    const int s0 = L.litem_seg0[item], ns = L.litem_nseg[item], split = L.litem_split[item];
    const int b0 = L.litem_box0[item], b1 = L.litem_box1[item];  // b1 < 0: one box
    const int pa = L.pang;
    const int NRAY = pa * pa;
    const int NPTS = kPS * NRAY;
    const int G = max(1, int(blockDim.x) / NRAY);
    const double h = L.h, inv_h = 1.0 / L.h;
    // staged sources (10 doubles each) of b0 at smem[0, 10 kTile), of b1 at smem[10 kTile, 20 kTile)
    double2* v0 = reinterpret_cast<double2*>(smem + 20 * kTile);
    double2* v1 = v0 + G * NP * NPTS;

    auto load_tile = [&](double* R, int box, int t0, int tn) {
        const int pb = int(L.beg[box]);
        const double cx = L.cx[box], cy = L.cy[box], cz = L.cz[box];
        for (int q = threadIdx.x; q < tn; q += blockDim.x) {
            const int t = pb + t0 + q;
            const double dx = P.x[t] - cx, dy = P.y[t] - cy, dz = P.z[t] - cz;
            const double nx = P.nx[t], ny = P.ny[t], nz = P.nz[t];
            // one 80-byte row per source (5 x 16-byte loads in the loop)
            double* row = R + 10 * q;
            row[0] = dx;
            row[1] = dy;
            row[2] = dz;
            row[3] = fma(dx, dx, fma(dy, dy, dz * dz));
            row[4] = nx;
            row[5] = ny;
            row[6] = nz;
            row[7] = fma(dx, nx, fma(dy, ny, dz * nz));
            const double2 a = a_p[t];
            row[8] = a.x;
            row[9] = a.y;
        }
    };
    const int n0 = int(L.end[b0]) - int(L.beg[b0]);
    const int n1 = b1 >= 0 ? int(L.end[b1]) - int(L.beg[b1]) : 0;
    const bool one_tile = n0 <= kTile;  // two-box items have both boxes within one tile
    if (one_tile) load_tile(smem, b0, 0, n0);
    if (b1 >= 0) load_tile(smem + 10 * kTile, b1, 0, n1);
    __syncthreads();

    const int tix = threadIdx.x;
    const bool in = tix < ns * NRAY;
    const int seg_l = in ? tix / NRAY : 0;
    const int ray = in ? tix % NRAY : 0;  // it + pa * ip
    const int rg = seg_l < split ? 0 : 1;
    const int box = rg ? b1 : b0;
    const bool act = in && !(L.active && !L.active[box]);
    const double* R = smem + rg * 10 * kTile;
    double xh = 0, yh = 0, zh = 0;
    double sig[kPS], khos[kPS];
    if (act) {
        const int gam = L.seg_gamma[s0 + seg_l];
        const int g1 = gam % L.ns, g2 = (gam / L.ns) % L.nc, g3 = gam / L.ns / L.nc;
        const int it = ray % pa, ip = ray / pa;
        const double sth = L.th_sin[g2 * pa + it], cth = L.th_cos[g2 * pa + it];
        const double sph = L.ph_sin[g3 * pa + ip], cph = L.ph_cos[g3 * pa + ip];
        xh = sth * cph;
        yh = sth * sph;
        zh = cth;
#pragma unroll
        for (int is = 0; is < kPS; ++is) {
            const double s = L.s_nodes[g1 * kPS + is];
            sig[is] = s * inv_h;
            khos[is] = k * h / s;
        }
    } else {
#pragma unroll
        for (int is = 0; is < kPS; ++is) sig[is] = 0.5, khos[is] = 0.0;
    }
    double2 acc[kPS][NP];
#pragma unroll
    for (int is = 0; is < kPS; ++is)
#pragma unroll
        for (int i = 0; i < NP; ++i) acc[is][i] = make_double2(0.0, 0.0);
    const int nsrc = one_tile ? (rg ? n1 : n0) : n0;
    for (int t0 = 0; t0 < nsrc; t0 += kTile) {
        const int tn = min(kTile, nsrc - t0);
        if (!one_tile) {  // one box for the whole CTA: the barriers are uniform
            __syncthreads();
            load_tile(smem, b0, t0, tn);
            __syncthreads();
        }
        if (!act) continue;
        const double2* rows = reinterpret_cast<const double2*>(R);
        for (int q = 0; q < tn; ++q) {
            const double2 s0 = rows[5 * q], s1 = rows[5 * q + 1], s2 = rows[5 * q + 2], s3 = rows[5 * q + 3],
                          s4 = rows[5 * q + 4];  // (dx, dy) (dz, |d|^2) (nx, ny) (nz, d.n) (a)
            const double xd = fma(xh, s0.x, fma(yh, s0.y, zh * s1.x));
            const double xn = fma(xh, s2.x, fma(yh, s2.y, zh * s3.x));
            const double d2 = s1.y, dn0 = s3.y;
            const double ar = s4.x, ai = s4.y;
#pragma unroll
            for (int is = 0; is < kPS; ++is) {
                const double sg = sig[is];
                const double w = fma(sg, d2, -2.0 * xd);   // (|v|^2 - 1) / sigma
                const double nv2 = fma(sg, w, 1.0);
                const double inv = rsqrt_normal(nv2);
                const double arg = khos[is] * fma(nv2, inv, -1.0);  // kh/s (|v| - 1)
                double sn, cs;
                sincos_tab(arg, &sn, &cs);  // (cfg2 leaf 4.70 -> 4.15 ms against sincos_bounded)
                const double2 pa_ = make_double2(fma(ar, cs, -ai * sn), fma(ar, sn, ai * cs));
                const double dn = fma(-sg, dn0, xn);      // v.n
                const double inv2 = inv * inv;
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    switch (PSET::f(i)) {
                        case 1:
                            cfma_r(acc[is][i], pa_, inv);
                            break;
                        case 2:
                            cfma_r(acc[is][i], pa_, dn * inv2 * inv);
                            break;
                        case 3:
                            cfma_r(acc[is][i], pa_, dn * inv2);
                            break;
                        default: {  // W4: (s/(h|v|) - i k) (v.n)/|v|^2
                            const double dn2 = dn * inv2;
                            cfma(acc[is][i], pa_, make_double2(sg * inv * dn2, -k * dn2));
                        }
                    }
                }
            }
        }
    }
    if (in) {
#pragma unroll
        for (int is = 0; is < kPS; ++is)
#pragma unroll
            for (int i = 0; i < NP; ++i) v0[(seg_l * NP + i) * NPTS + is + kPS * ray] = acc[is][i];
    }
    __syncthreads();
    if (pa == 5)
        block_transform_c<kPS, 5>(v0, v1, ns * NP, Ms, Ma, store + std::size_t(s0) * NP * NPTS);
    else
        block_transform(v0, v1, ns * NP, kPS, pa, Ms, Ma, store + std::size_t(s0) * NP * NPTS);
}

}  // namespace

int leaf_item_segments(int pang) { return std::max(1, kThreads / (pang * pang)); }
int leaf_item_tile() { return kTile; }

bool launch_leaf_fill_ray(const LevelDev& L, const PointsDev& P, const double2* a_p, double k, const Pipes& pipes,
                          const double* Ms, const double* Ma, double2* store, cudaStream_t st) {
    if (L.ps != kPS || !L.th_sin || !L.litem_seg0) return false;
    if (L.nb == 0 || L.nseg == 0 || L.n_litem == 0) return true;
    const int NRAY = L.pang * L.pang;
    const int G = std::max(1, kThreads / NRAY);
    const std::size_t smem = 20 * kTile * sizeof(double) + 2 * std::size_t(G) * pipes.n * kPS * NRAY * sizeof(double2);
    auto go = [&](auto kern) {
        IFGF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<L.n_litem, kThreads, smem, st>>>(L, P, a_p, k, Ms, Ma, store);
    };
    const int code = pipes.f[0] * 100 + (pipes.n > 1 ? pipes.f[1] * 10 : 0) + (pipes.n > 2 ? pipes.f[2] : 0);
    switch (code) {
        case 123: go(leaf_ray_kernel<PipeSet<1, 2, 3>>); break;
        case 140: go(leaf_ray_kernel<PipeSet<1, 4, 0>>); break;
        case 100: go(leaf_ray_kernel<PipeSet<1, 0, 0>>); break;
        case 400: go(leaf_ray_kernel<PipeSet<4, 0, 0>>); break;
        case 230: go(leaf_ray_kernel<PipeSet<2, 3, 0>>); break;
        case 200: go(leaf_ray_kernel<PipeSet<2, 0, 0>>); break;
        case 300: go(leaf_ray_kernel<PipeSet<3, 0, 0>>); break;
        default: return false;  // other orderings: the per-node kernel
    }
    IFGF_CUDA(cudaGetLastError());
    return true;
}

}  // namespace ifgfb200
