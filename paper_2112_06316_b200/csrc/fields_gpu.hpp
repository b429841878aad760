// GPU field sums over an oversampled surface quadrature (cuda/fields.cu); plain C++
// interface for the C-ABI layer.
#pragma once

#include <vector>

#include "host/fields.hpp"

namespace ifgfb200 {

// far-field pattern values at `dirs` (postprocess.cpp:83-104)
void gpu_far_field(const FineQuad& q, const std::vector<Vec3>& dirs, double k, double gamma, int device, cplx* out);
// scattered field, closest-node distance and unit-density static double layer at `pts`
// (postprocess.cpp:106-139; the caller adds the incident field and sets the flags)
void gpu_near_field(const FineQuad& q, const std::vector<Vec3>& pts, double k, double gamma, int device,
                    cplx* scattered, double* dmin, double* gauss);

}  // namespace ifgfb200
