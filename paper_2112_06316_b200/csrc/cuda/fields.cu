// Far- and near-field evaluation of the solved density (reference postprocess.cpp:83-139)
// as dense GPU sums over the oversampled surface quadrature (host/fields.cpp): one thread
// per direction / evaluation point, quadrature nodes staged through shared memory in tiles
// read by the whole CTA.
//   far : u_inf(xhat) = 1/(4 pi) sum_m (-i k <xhat, nu_m> - i gamma) e^{-ik xhat.y_m} phi_m w_m
//   near: u_s(x) = sum_m (dG/dnu_y - i gamma G)(x, y_m) phi_m w_m, plus the total field, the
//         closest-node distance and the static double layer of unit density (interior flag)
#include <vector>

#include "../fields_gpu.hpp"
#include "dev_common.cuh"
#include "kernels.cuh"

namespace ifgfb200 {
namespace {

using namespace dev;

constexpr int kT = 256;

struct QuadDev {
    int n = 0;
    const double *x, *y, *z, *nx, *ny, *nz, *jw;
    const double2* a;  // density * jw
};

__global__ void __launch_bounds__(kT) far_field_kernel(QuadDev Q, int nd, const double* __restrict__ dx,
                                                       const double* __restrict__ dy, const double* __restrict__ dz,
                                                       double k, double gamma, double2* __restrict__ out) {
    __shared__ double sx[kT], sy[kT], sz[kT], snx[kT], sny[kT], snz[kT];
    __shared__ double2 sa[kT];
    const int g = blockIdx.x * kT + threadIdx.x;
    const bool act = g < nd;
    const double ex = act ? dx[g] : 0.0, ey = act ? dy[g] : 0.0, ez = act ? dz[g] : 0.0;
    double2 acc = make_double2(0.0, 0.0);
    for (int m0 = 0; m0 < Q.n; m0 += kT) {
        const int tn = min(kT, Q.n - m0);
        __syncthreads();
        if (threadIdx.x < tn) {
            const int m = m0 + threadIdx.x;
            sx[threadIdx.x] = Q.x[m];
            sy[threadIdx.x] = Q.y[m];
            sz[threadIdx.x] = Q.z[m];
            snx[threadIdx.x] = Q.nx[m];
            sny[threadIdx.x] = Q.ny[m];
            snz[threadIdx.x] = Q.nz[m];
            sa[threadIdx.x] = Q.a[m];
        }
        __syncthreads();
        for (int m = 0; m < tn; ++m) {
            const double xy = fma(ex, sx[m], fma(ey, sy[m], ez * sz[m]));
            const double xn = fma(ex, snx[m], fma(ey, sny[m], ez * snz[m]));
            double sn, cs;
            sincos_bounded(-k * xy, &sn, &cs);
            // (0, -k xn - gamma) * e^{-ik xhat.y} * a
            const double2 t = cmul(make_double2(cs, sn), sa[m]);
            const double f = -k * xn - gamma;
            acc.x = fma(-f, t.y, acc.x);
            acc.y = fma(f, t.x, acc.y);
        }
    }
    if (act) out[g] = make_double2(acc.x * kInv4PiD, acc.y * kInv4PiD);
}

__global__ void __launch_bounds__(kT) near_field_kernel(QuadDev Q, int np, const double* __restrict__ px,
                                                        const double* __restrict__ py,
                                                        const double* __restrict__ pz, double k,
                                                        double2* __restrict__ S_out, double2* __restrict__ D_out,
                                                        double* __restrict__ dmin_out, double* __restrict__ gauss_out) {
    __shared__ double sx[kT], sy[kT], sz[kT], snx[kT], sny[kT], snz[kT], sw[kT];
    __shared__ double2 sa[kT];
    const int t = blockIdx.x * kT + threadIdx.x;
    const bool act = t < np;
    const double x = act ? px[t] : 0.0, y = act ? py[t] : 0.0, z = act ? pz[t] : 0.0;
    double2 accs = make_double2(0.0, 0.0), accd = make_double2(0.0, 0.0);
    double dmin = 1.7976931348623157e308, gauss = 0.0;
    for (int m0 = 0; m0 < Q.n; m0 += kT) {
        const int tn = min(kT, Q.n - m0);
        __syncthreads();
        if (threadIdx.x < tn) {
            const int m = m0 + threadIdx.x;
            sx[threadIdx.x] = Q.x[m];
            sy[threadIdx.x] = Q.y[m];
            sz[threadIdx.x] = Q.z[m];
            snx[threadIdx.x] = Q.nx[m];
            sny[threadIdx.x] = Q.ny[m];
            snz[threadIdx.x] = Q.nz[m];
            sw[threadIdx.x] = Q.jw[m];
            sa[threadIdx.x] = Q.a[m];
        }
        __syncthreads();
        for (int m = 0; m < tn; ++m) {
            const double ddx = x - sx[m], ddy = y - sy[m], ddz = z - sz[m];
            const double r2 = fma(ddx, ddx, fma(ddy, ddy, ddz * ddz));
            const double r = sqrt(r2);
            dmin = fmin(dmin, r);
            if (r < 1e-14) continue;
            const double inv = 1.0 / r;
            double sn, cs;
            sincos_bounded(k * r, &sn, &cs);
            const double2 a = sa[m];
            const double g = kInv4PiD * inv;
            const double2 ga = cmul(make_double2(cs * g, sn * g), a);  // G a
            accs = cadd(accs, ga);
            const double dn = fma(ddx, snx[m], fma(ddy, sny[m], ddz * snz[m]));
            const double f = dn * kInv4PiD * inv * inv * inv;
            const double kr = k * r;
            // e^{ikr} (1 - ikr) dn/(4 pi r^3)
            const double2 e = make_double2(fma(kr, sn, cs) * f, fma(-kr, cs, sn) * f);
            accd = cadd(accd, cmul(e, a));
            gauss = fma(f, sw[m], gauss);
        }
    }
    if (!act) return;
    S_out[t] = accs;
    D_out[t] = accd;
    dmin_out[t] = dmin;
    gauss_out[t] = gauss;
}

template <class T>
struct Buf {
    T* p = nullptr;
    explicit Buf(std::size_t n) { IFGF_CUDA(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T))); }
    ~Buf() { cudaFree(p); }
    Buf(const Buf&) = delete;
    void put(const T* h, std::size_t n) {
        if (n) IFGF_CUDA(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice));
    }
    void get(T* h, std::size_t n) const {
        if (n) IFGF_CUDA(cudaMemcpy(h, p, n * sizeof(T), cudaMemcpyDeviceToHost));
    }
};

struct QuadBufs {
    Buf<double> x, y, z, nx, ny, nz, jw;
    Buf<double2> a;
    QuadDev dev;
    explicit QuadBufs(const FineQuad& q)
        : x(q.size()), y(q.size()), z(q.size()), nx(q.size()), ny(q.size()), nz(q.size()), jw(q.size()),
          a(q.size()) {
        const std::size_t n = q.size();
        x.put(q.x.data(), n);
        y.put(q.y.data(), n);
        z.put(q.z.data(), n);
        nx.put(q.nx.data(), n);
        ny.put(q.ny.data(), n);
        nz.put(q.nz.data(), n);
        jw.put(q.jw.data(), n);
        std::vector<double2> aw(n);
        for (std::size_t m = 0; m < n; ++m) {
            const cplx v = q.density[m] * q.jw[m];
            aw[m] = make_double2(v.real(), v.imag());
        }
        a.put(aw.data(), n);
        dev = {int(n), x.p, y.p, z.p, nx.p, ny.p, nz.p, jw.p, a.p};
    }
};

}  // namespace

void gpu_far_field(const FineQuad& q, const std::vector<Vec3>& dirs, double k, double gamma, int device, cplx* out) {
    IFGF_CUDA(cudaSetDevice(device));
    if (q.size() > std::size_t(0x7fffffff) || dirs.size() > std::size_t(0x7fffffff))
        throw InvalidArgument("far_field: too many nodes or directions");
    QuadBufs Q(q);
    const std::size_t nd = dirs.size();
    std::vector<double> hx(nd), hy(nd), hz(nd);
    for (std::size_t i = 0; i < nd; ++i) {
        hx[i] = dirs[i].x;
        hy[i] = dirs[i].y;
        hz[i] = dirs[i].z;
    }
    Buf<double> dx(nd), dy(nd), dz(nd);
    Buf<double2> o(nd);
    dx.put(hx.data(), nd);
    dy.put(hy.data(), nd);
    dz.put(hz.data(), nd);
    if (nd) far_field_kernel<<<int((nd + kT - 1) / kT), kT>>>(Q.dev, int(nd), dx.p, dy.p, dz.p, k, gamma, o.p);
    IFGF_CUDA(cudaGetLastError());
    IFGF_CUDA(cudaDeviceSynchronize());
    o.get(reinterpret_cast<double2*>(out), nd);
}

void gpu_layer_potentials_at(const FineQuad& q, const std::vector<Vec3>& pts, double k, int device, cplx* S, cplx* D,
                             double* dmin, double* gauss) {
    IFGF_CUDA(cudaSetDevice(device));
    if (q.size() > std::size_t(0x7fffffff) || pts.size() > std::size_t(0x7fffffff))
        throw InvalidArgument("layer potentials: too many nodes or points");
    QuadBufs Q(q);
    const std::size_t np = pts.size();
    std::vector<double> hx(np), hy(np), hz(np);
    for (std::size_t i = 0; i < np; ++i) {
        hx[i] = pts[i].x;
        hy[i] = pts[i].y;
        hz[i] = pts[i].z;
    }
    Buf<double> px(np), py(np), pz(np), dm(np), ga(np);
    Buf<double2> s_out(np), d_out(np);
    px.put(hx.data(), np);
    py.put(hy.data(), np);
    pz.put(hz.data(), np);
    if (np)
        near_field_kernel<<<int((np + kT - 1) / kT), kT>>>(Q.dev, int(np), px.p, py.p, pz.p, k, s_out.p, d_out.p, dm.p,
                                                            ga.p);
    IFGF_CUDA(cudaGetLastError());
    IFGF_CUDA(cudaDeviceSynchronize());
    s_out.get(reinterpret_cast<double2*>(S), np);
    d_out.get(reinterpret_cast<double2*>(D), np);
    dm.get(dmin, np);
    ga.get(gauss, np);
}

void gpu_near_field(const FineQuad& q, const std::vector<Vec3>& pts, double k, double gamma, int device,
                    cplx* scattered, double* dmin, double* gauss) {
    std::vector<cplx> S(pts.size()), D(pts.size());
    gpu_layer_potentials_at(q, pts, k, device, S.data(), D.data(), dmin, gauss);
    for (std::size_t i = 0; i < pts.size(); ++i) scattered[i] = D[i] - cplx(0.0, gamma) * S[i];  // D - i gamma S
}

}  // namespace ifgfb200
