// RP beta tables on the GPU (the setup step ranked first in SURVEY.md §8(f)):
//
//   beta^{S,D}_{n,m} = sum_{i,j} K(x, y(u_i, v_j)) J(u_i, v_j) w_i w_j T_n(u_i) T_m(v_j)
//
// over the graded Fejér rule around (ubar, vbar) (rp.cpp:309-395), K = G or dG/dnu_y,
// zeroed within max(1e-14, 1e-8 spacing) of the target. One CTA per (target, patch) pair;
// the patch geometry on the graded grid is produced by two small separable contractions in
// shared memory, a slab of JV v-nodes at a time, and the two tables are accumulated by the
// same (n, m) thread across slabs. FP64 throughout; results agree with the reference
// tables to ~1e-15 relative (different contraction order).
#include "dev_common.cuh"
#include "kernels.cuh"

namespace ifgfb200 {
namespace {

using namespace dev;

constexpr int kBetaThreads = 256;
constexpr int kJV = 8;

__device__ double d_grade_w(double tau, int d) {
    tau = fmin(fmax(tau, 0.0), 2.0 * kPiD);
    auto nu = [&](double q) {
        const double a = (kPiD - q) / kPiD;
        const double b = (q - kPiD) / kPiD;
        return (1.0 / d - 0.5) * a * a * a + b / d + 0.5;
    };
    const double vd = pow(nu(tau), double(d));
    const double wd = pow(nu(2.0 * kPiD - tau), double(d));
    return 2.0 * kPiD * vd / (vd + wd);
}

__device__ double d_grade_w_deriv(double tau, int d) {
    tau = fmin(fmax(tau, 0.0), 2.0 * kPiD);
    auto nu = [&](double q) {
        const double a = (kPiD - q) / kPiD;
        const double b = (q - kPiD) / kPiD;
        return (1.0 / d - 0.5) * a * a * a + b / d + 0.5;
    };
    auto nu_d = [&](double q) {
        const double a = (kPiD - q) / kPiD;
        return -3.0 * (1.0 / d - 0.5) * a * a / kPiD + 1.0 / (d * kPiD);
    };
    const double n1 = nu(tau), n2 = nu(2.0 * kPiD - tau);
    const double p1 = pow(n1, double(d - 1)), p2 = pow(n2, double(d - 1));
    const double f = p1 * n1, g = p2 * n2;
    const double fp = d * p1 * nu_d(tau);
    const double gp = -d * p2 * nu_d(2.0 * kPiD - tau);
    return 2.0 * kPiD * (fp * g - f * gp) / ((f + g) * (f + g));
}

__device__ double d_grade_xi(double alpha, double tau, int d) {
    tau = fmin(fmax(tau, -1.0), 1.0);
    if (alpha >= 1.0) return 1.0 - (2.0 / kPiD) * d_grade_w(kPiD * fabs(tau - 1.0) / 2.0, d);
    if (alpha <= -1.0) return -1.0 + (2.0 / kPiD) * d_grade_w(kPiD * fabs(tau + 1.0) / 2.0, d);
    const double sg = tau > 0 ? 1.0 : (tau < 0 ? -1.0 : 0.0);
    return alpha + (sg - alpha) / kPiD * d_grade_w(kPiD * fabs(tau), d);
}

__device__ double d_grade_xi_deriv(double alpha, double tau, int d) {
    tau = fmin(fmax(tau, -1.0), 1.0);
    if (alpha >= 1.0) return d_grade_w_deriv(kPiD * (1.0 - tau) / 2.0, d);
    if (alpha <= -1.0) return d_grade_w_deriv(kPiD * (tau + 1.0) / 2.0, d);
    if (tau == 0.0) return 0.0;
    const double sg = tau > 0 ? 1.0 : -1.0;
    return (sg - alpha) * sg * d_grade_w_deriv(kPiD * fabs(tau), d);
}

__global__ void __launch_bounds__(kBetaThreads)
beta_kernel(BetaDev B, int TT, int max_du, int max_nunv, double2* __restrict__ bs_out,
            double2* __restrict__ bd_out) {
    extern __shared__ double sm[];
    const int p = blockIdx.x;
    const int nb = B.n_beta;
    const int q = B.patch[p];
    const int nu = B.nu[q], nv = B.nv[q], du = B.du[q], dv = B.dv[q];
    const int nn = nu * nv;
    const double orient = B.orient[q];
    const double cutoff = B.cutoff[q];
    const std::uint32_t tg = B.target[p];
    const double X = B.tx[tg], Y = B.ty[tg], Z = B.tz[tg];
    const double k = B.k;
    const double* ser = B.series + B.series_off[q];  // 9 series of du*dv

    double* us = sm;
    double* vs = us + nb;
    double* wu = vs + nb;
    double* wv = wu + nb;
    double* Tu = wv + nb;               // nb x TT
    double* Tv = Tu + nb * TT;          // nb x TT
    double* P2 = Tv + nb * TT;          // 9 x max_du x kJV
    double2* fS = reinterpret_cast<double2*>(P2 + 9 * max_du * kJV);  // nb x kJV
    double2* fD = fS + nb * kJV;
    double2* rS = fD + nb * kJV;        // kJV x nu
    double2* rD = rS + kJV * max_nunv;  // (sized generously)
    double2* aS = rD + kJV * max_nunv;  // nn
    double2* aD = aS + max_nunv;

    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        const double x = B.rule_x[i], w = B.rule_w[i];
        us[i] = d_grade_xi(B.ubar[p], x, B.cov_d);
        wu[i] = d_grade_xi_deriv(B.ubar[p], x, B.cov_d) * w;
        vs[i] = d_grade_xi(B.vbar[p], x, B.cov_d);
        wv[i] = d_grade_xi_deriv(B.vbar[p], x, B.cov_d) * w;
    }
    __syncthreads();
    const int tmax = max(max(du, nu), max(dv, nv));
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        const double u = fmin(fmax(us[i], -1.0), 1.0), v = fmin(fmax(vs[i], -1.0), 1.0);
        double* tu = Tu + i * TT;
        double* tv = Tv + i * TT;
        tu[0] = 1.0;
        tv[0] = 1.0;
        if (tmax > 1) {
            tu[1] = u;
            tv[1] = v;
        }
        for (int c = 2; c < tmax; ++c) {
            tu[c] = 2.0 * u * tu[c - 1] - tu[c - 2];
            tv[c] = 2.0 * v * tv[c - 1] - tv[c - 2];
        }
    }
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
        aS[e] = make_double2(0.0, 0.0);
        aD[e] = make_double2(0.0, 0.0);
    }
    __syncthreads();

    for (int j0 = 0; j0 < nb; j0 += kJV) {
        const int jn = min(kJV, nb - j0);
        // P2[s][i][jj] = sum_j series_s[i + du j] T_j(v_{j0+jj})
        for (int e = threadIdx.x; e < 9 * du * jn; e += blockDim.x) {
            const int jj = e % jn, rest = e / jn, i = rest % du, s = rest / du;
            const double* c = ser + std::size_t(s) * du * dv + i;
            const double* tv = Tv + (j0 + jj) * TT;
            double acc = 0.0;
            for (int j = 0; j < dv; ++j) acc = fma(c[std::size_t(du) * j], tv[j], acc);
            P2[(s * max_du + i) * kJV + jj] = acc;
        }
        __syncthreads();
        // geometry + kernels at the slab's nodes
        for (int e = threadIdx.x; e < nb * jn; e += blockDim.x) {
            const int iu = e % nb, jj = e / nb;
            const double* tu = Tu + iu * TT;
            double g[9];
#pragma unroll
            for (int s = 0; s < 9; ++s) {
                const double* col = P2 + (s * max_du) * kJV + jj;
                double acc = 0.0;
                for (int i = 0; i < du; ++i) acc = fma(col[i * kJV], tu[i], acc);
                g[s] = acc;
            }
            // g: pos xyz, d/du xyz, d/dv xyz
            const double crx = g[4] * g[8] - g[5] * g[7];
            const double cry = g[5] * g[6] - g[3] * g[8];
            const double crz = g[3] * g[7] - g[4] * g[6];
            const double jac = sqrt(crx * crx + cry * cry + crz * crz);
            double2 ks = make_double2(0.0, 0.0), kd = make_double2(0.0, 0.0);
            const double dx = X - g[0], dy = Y - g[1], dz = Z - g[2];
            const double r = sqrt(dx * dx + dy * dy + dz * dz);
            if (r >= cutoff) {
                const double sc = jac > 0 ? orient / jac : 0.0;
                const double nx = crx * sc, ny = cry * sc, nz = crz * sc;
                double sn, cs;
                sincos(k * r, &sn, &cs);
                const double inv = 1.0 / r;
                const double gg = kInv4PiD * inv;
                ks = make_double2(cs * gg, sn * gg);
                const double dn = dx * nx + dy * ny + dz * nz;
                const double kr = k * r;
                const double f = dn * kInv4PiD * inv * inv * inv;
                kd = make_double2((cs + kr * sn) * f, (sn - kr * cs) * f);
            }
            const double f = jac * wu[iu] * wv[j0 + jj];
            fS[jj * nb + iu] = cscale(ks, f);
            fD[jj * nb + iu] = cscale(kd, f);
        }
        __syncthreads();
        // rows[jj][n] = sum_iu f(iu, jj) T_n(u_iu)
        for (int e = threadIdx.x; e < 2 * jn * nu; e += blockDim.x) {
            const int n = e % nu, rest = e / nu, jj = rest % jn, tab = rest / jn;
            const double2* f = (tab == 0 ? fS : fD) + jj * nb;
            double2 acc = make_double2(0.0, 0.0);
            for (int iu = 0; iu < nb; ++iu) cfma_r(acc, f[iu], Tu[iu * TT + n]);
            (tab == 0 ? rS : rD)[jj * max_nunv + n] = acc;
        }
        __syncthreads();
        // beta[n + nu m] += sum_jj rows[jj][n] T_m(v_jj)
        for (int e = threadIdx.x; e < nn; e += blockDim.x) {
            const int n = e % nu, m = e / nu;
            double2 s = aS[e], d = aD[e];
            for (int jj = 0; jj < jn; ++jj) {
                const double t = Tv[(j0 + jj) * TT + m];
                cfma_r(s, rS[jj * max_nunv + n], t);
                cfma_r(d, rD[jj * max_nunv + n], t);
            }
            aS[e] = s;
            aD[e] = d;
        }
        __syncthreads();
    }
    const std::uint64_t off = B.offset[p];
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
        bs_out[off + e] = aS[e];
        bd_out[off + e] = aD[e];
    }
}

}  // namespace

void launch_beta(const BetaDev& B, double2* bs, double2* bd, int max_dudv, int max_nunv,
                 cudaStream_t st) {
    if (B.npairs == 0) return;
    const int TT = max_dudv;  // basis length covers max(du, dv, nu, nv)
    const int nb = B.n_beta;
    const std::size_t smem = sizeof(double) * (4 * nb + 2 * nb * TT + 9 * TT * kJV) +
                             sizeof(double2) * (2 * nb * kJV + 2 * kJV * max_nunv + 2 * max_nunv);
    IFGF_CUDA(cudaFuncSetAttribute(beta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    // pairs in launches of at most 2^20 CTAs
    const int chunk = 1 << 20;
    for (int p0 = 0; p0 < B.npairs; p0 += chunk) {
        BetaDev Bc = B;
        const int cnt = std::min(chunk, B.npairs - p0);
        Bc.target += p0;
        Bc.patch += p0;
        Bc.ubar += p0;
        Bc.vbar += p0;
        Bc.offset += p0;
        Bc.npairs = cnt;
        beta_kernel<<<cnt, kBetaThreads, smem, st>>>(Bc, TT, TT, max_nunv, bs, bd);
        IFGF_CUDA(cudaGetLastError());
    }
}

}  // namespace ifgfb200
