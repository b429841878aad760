// GPU helpers called from the host setup / C-ABI layer, plain C++ interface: field sums
// over an oversampled surface quadrature (cuda/fields.cu) and the batched closest-point
// searches of the pair classification (cuda/proximity_kernels.cu).
#pragma once

#include <vector>

#include "host/coneplan.hpp"
#include "host/fields.hpp"
#include "host/proximity.hpp"

namespace ifgfb200 {

// far-field pattern values at `dirs` (postprocess.cpp:83-104)
void gpu_far_field(const FineQuad& q, const std::vector<Vec3>& dirs, double k, double gamma, int device, cplx* out);
// scattered field, closest-node distance and unit-density static double layer at `pts`
// (postprocess.cpp:106-139; the caller adds the incident field and sets the flags)
void gpu_near_field(const FineQuad& q, const std::vector<Vec3>& pts, double k, double gamma, int device,
                    cplx* scattered, double* dmin, double* gauss);
// S and D of the quadrature's density at `pts` (zero contribution from nodes within 1e-14),
// with the closest-node distance and the unit-density static double layer
void gpu_layer_potentials_at(const FineQuad& q, const std::vector<Vec3>& pts, double k, int device, cplx* S, cplx* D,
                             double* dmin, double* gauss);
// closest_point_on for every non-own request, bit for bit (ClosestPointBatch)
// segment decisions of one plan level (ConeDecider); uncertain ones are flagged for the host
void gpu_cone_decisions(const ConeDecisionJob& job, ConeLevel& L, std::vector<std::uint8_t>& marks,
                        std::vector<std::int64_t>& flagged_cev, std::vector<std::int64_t>& flagged_pev, int device);
void gpu_closest_points(const Surface& s, const std::vector<ClosestPointRequest>& req, std::vector<ClosestPoint>& res,
                        int device);

}  // namespace ifgfb200
