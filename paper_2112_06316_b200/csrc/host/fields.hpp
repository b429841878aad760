// Field evaluation after the solve (reference postprocess.hpp/.cpp):
// the oversampled surface quadrature the field sums run over, the analytic sound-soft
// sphere (Mie) far field used to validate a solve, and the eps error metric. The dense
// direction x quadrature-node sums themselves run on the GPU (cuda/fields.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "core.hpp"
#include "surface.hpp"

namespace ifgfb200 {

// Per patch a Fejér rule of order m = min(24, max(nu, nv, 8 + ceil(0.75 k diam))) with the
// density carried by its per-patch Chebyshev expansion (postprocess.cpp:20-58).
struct FineQuad {
    std::vector<double> x, y, z, nx, ny, nz, jw;
    std::vector<cplx> density;  // density at the fine nodes
    std::size_t size() const { return x.size(); }
};
FineQuad oversample_for_fields(const Surface& s, const cplx* density, double k);

// far-field directions, polar index fastest: phi_m = m pi/(n_phi-1), theta_n = n 2pi/(n_theta-1)
// (postprocess.cpp:62-81)
std::vector<Vec3> far_field_directions(int n_phi, int n_theta);

// u_inf of a sound-soft sphere of radius R for a plane wave along `direction`
// (partial-wave series sum_l (2l+1) i/k j_l(kR)/h_l(kR) P_l(cos angle), truncated at
// L = ceil(kR + 6 (kR)^(1/3) + 20) + extra_terms; postprocess.cpp:176-205)
std::vector<cplx> mie_far_field(double radius, double k, const Vec3& direction, const std::vector<Vec3>& dirs,
                                int extra_terms);

// max_i | |ref_i| - |apx_i| | / |ref_i| over nonzero references (postprocess.cpp:209-226)
double eps_metric(const cplx* ref, const cplx* apx, std::size_t n, int* skipped);

}  // namespace ifgfb200
