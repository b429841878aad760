// Level-D fill (ifgf.cpp:312-391) with one thread per interpolation RAY: the ps = 3 radial
// nodes of a segment share the direction x^ = (sin th cos ph, sin th sin ph, cos th), so per
// (ray, source) the projections x^.dy and x^.n are formed once and each radial node needs
//   |v|^2 = 1 + sigma (sigma |dy|^2 - 2 x^.dy),   sigma = s/h
//   arg = k h/s (|v| - 1) with |v| - 1 = fma(|v|^2, 1/|v|, -1) (one rounding; the
//         reference's (|v|^2-1)/(|v|+1) has the same ~1e-16 absolute error)
//   v.n = x^.n - sigma dy.n
// Sources are staged in shared memory with |dy|^2 and dy.n precomputed. The 3x5x5
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

template <class PSET>
__global__ void __launch_bounds__(kThreads, 2)
leaf_ray_kernel(LevelDev L, PointsDev P, const double2* __restrict__ a_p, double k,
                const double* __restrict__ Ms, const double* __restrict__ Ma, double2* __restrict__ store) {
    constexpr int NP = PSET::n;
    extern __shared__ double smem[];
    const int b = blockIdx.x;
    const int s0 = L.box_seg_begin[b], s1 = L.box_seg_begin[b + 1];
    if (s0 == s1 || (L.active && !L.active[b])) return;
    const int pa = L.pang;
    const int NRAY = pa * pa;
    const int NPTS = kPS * NRAY;
    const int G = max(1, int(blockDim.x) / NRAY);
    const int pb = int(L.beg[b]);
    const int nsrc = int(L.end[b]) - pb;
    const double cx = L.cx[b], cy = L.cy[b], cz = L.cz[b];
    const double h = L.h, inv_h = 1.0 / L.h;

    double* sdx = smem;
    double* sdy = sdx + kTile;
    double* sdz = sdy + kTile;
    double* sd2 = sdz + kTile;
    double* snx = sd2 + kTile;
    double* sny = snx + kTile;
    double* snz = sny + kTile;
    double* sdn = snz + kTile;
    double* sar = sdn + kTile;
    double* sai = sar + kTile;
    double2* v0 = reinterpret_cast<double2*>(sai + kTile);
    double2* v1 = v0 + G * NP * NPTS;

    auto load_tile = [&](int t0, int tn) {
        for (int q = threadIdx.x; q < tn; q += blockDim.x) {
            const int t = pb + t0 + q;
            const double dx = P.x[t] - cx, dy = P.y[t] - cy, dz = P.z[t] - cz;
            const double nx = P.nx[t], ny = P.ny[t], nz = P.nz[t];
            sdx[q] = dx;
            sdy[q] = dy;
            sdz[q] = dz;
            sd2[q] = fma(dx, dx, fma(dy, dy, dz * dz));
            snx[q] = nx;
            sny[q] = ny;
            snz[q] = nz;
            sdn[q] = fma(dx, nx, fma(dy, ny, dz * nz));
            const double2 a = a_p[t];
            sar[q] = a.x;
            sai[q] = a.y;
        }
    };
    const bool one_tile = nsrc <= kTile;
    if (one_tile) load_tile(0, nsrc);
    __syncthreads();

    for (int g0 = s0; g0 < s1; g0 += G) {
        const int gcount = min(G, s1 - g0);
        const int items = gcount * NRAY;
        for (int base = 0; base < items; base += blockDim.x) {
            const int item = base + threadIdx.x;
            const bool act = item < items;
            const int seg_l = act ? item / NRAY : 0;
            const int ray = act ? item % NRAY : 0;  // it + pa * ip
            double xh = 0, yh = 0, zh = 0;
            double sig[kPS], khos[kPS];
            if (act) {
                const int gam = L.seg_gamma[g0 + seg_l];
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
            for (int t0 = 0; t0 < nsrc; t0 += kTile) {
                const int tn = min(kTile, nsrc - t0);
                if (!one_tile) {
                    __syncthreads();
                    load_tile(t0, tn);
                    __syncthreads();
                }
                if (!act) continue;
                for (int q = 0; q < tn; ++q) {
                    const double xd = fma(xh, sdx[q], fma(yh, sdy[q], zh * sdz[q]));
                    const double xn = fma(xh, snx[q], fma(yh, sny[q], zh * snz[q]));
                    const double d2 = sd2[q], dn0 = sdn[q];
                    const double ar = sar[q], ai = sai[q];
#pragma unroll
                    for (int is = 0; is < kPS; ++is) {
                        const double sg = sig[is];
                        const double w = fma(sg, d2, -2.0 * xd);   // (|v|^2 - 1) / sigma
                        const double nv2 = fma(sg, w, 1.0);
                        const double inv = rsqrt(nv2);
                        const double arg = khos[is] * fma(nv2, inv, -1.0);  // kh/s (|v| - 1)
                        double sn, cs;
                        sincos_bounded(arg, &sn, &cs);
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
            if (act) {
#pragma unroll
                for (int is = 0; is < kPS; ++is)
#pragma unroll
                    for (int i = 0; i < NP; ++i) v0[(seg_l * NP + i) * NPTS + is + kPS * ray] = acc[is][i];
            }
        }
        __syncthreads();
        block_transform(v0, v1, gcount * NP, kPS, pa, Ms, Ma, store + std::size_t(g0) * NP * NPTS);
        __syncthreads();
    }
}

}  // namespace

bool launch_leaf_fill_ray(const LevelDev& L, const PointsDev& P, const double2* a_p, double k, const Pipes& pipes,
                          const double* Ms, const double* Ma, double2* store, cudaStream_t st) {
    if (L.ps != kPS || !L.th_sin) return false;
    if (L.nb == 0 || L.nseg == 0) return true;
    const int NRAY = L.pang * L.pang;
    const int G = std::max(1, kThreads / NRAY);
    const std::size_t smem = 10 * kTile * sizeof(double) + 2 * std::size_t(G) * pipes.n * kPS * NRAY * sizeof(double2);
    auto go = [&](auto kern) {
        IFGF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<L.nb, kThreads, smem, st>>>(L, P, a_p, k, Ms, Ma, store);
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
