// Chebyshev-Gauss utilities used by the host setup (geometry series, cone node tables,
// Fejér weights, block transform matrices). Each routine restates the reference routine
// named in its comment with the same floating-point evaluation order, because geometry
// and cone nodes feed discrete decisions that must match the reference bit for bit.
#pragma once

#include <vector>

#include "core.hpp"

namespace ifgfb200::cheb {

// x_k = cos((2k+1) pi / (2n)), k = 0..n-1 (chebyshev.cpp:77-83)
std::vector<double> gauss_nodes(int n);
// T_0..T_{n-1}(x) by the three-term recurrence (chebyshev.cpp:85-89)
void basis(int n, double x, double* out);
// a_i = (alpha_i/n) sum_k u(x_k) T_i(x_k), alpha_0 = 1, alpha_i = 2 (chebyshev.cpp:28-40)
std::vector<double> coeffs_1d(const double* samples, int n);
std::vector<cplx> coeffs_1d(const cplx* samples, int n);
// tensor transform, u fastest: along u per row, then along v per column (chebyshev.cpp:43-61)
std::vector<double> coeffs_2d(const double* samples, int nu, int nv);
std::vector<cplx> coeffs_2d(const cplx* samples, int nu, int nv);
// clamped Clenshaw, |x| may exceed 1 by 1e-12 (chebyshev.cpp:12-25, 63-74)
double eval_2d(const double* coeffs, int nu, int nv, double u, double v);
// derivative series along u / v (chebyshev.cpp:119-153)
std::vector<double> deriv_u(const std::vector<double>& c, int nu, int nv);
std::vector<double> deriv_v(const std::vector<double>& c, int nu, int nv);
// Fejér's first rule on gauss_nodes(J) (chebyshev.cpp:155-167)
void fejer(int J, std::vector<double>& nodes, std::vector<double>& weights);
// dense n x n transform, a = M u (chebyshev.cpp:169-179)
std::vector<double> transform(int n);

}  // namespace ifgfb200::cheb
