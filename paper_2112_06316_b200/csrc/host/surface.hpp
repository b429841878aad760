// Surface description consumed by the operator: logical-quadrilateral patches with
// Chebyshev position series plus flat per-node arrays (node l = patch_start[q] + i + nu*j),
// the layout of /root/reference/proj/include/ifgf/geometry.hpp:16-57. The mesh is an input
// of the hot path; the generators here exist so the benchmark and tests can produce the
// BASELINE geometries without the reference.
#pragma once

#include <array>
#include <vector>

#include "core.hpp"

namespace ifgfb200 {

struct Patch {
    int nu = 0, nv = 0;  // nodes per direction
    int du = 0, dv = 0;  // series extents
    std::array<std::vector<double>, 3> pos_c;  // position series, u fastest
    std::array<std::vector<double>, 3> du_c;   // d/du series
    std::array<std::vector<double>, 3> dv_c;   // d/dv series
    double orient = 1.0;
};

struct Surface {
    std::vector<Patch> patches;
    Vec3 interior;
    std::vector<Vec3> pos, nrm;
    std::vector<double> jac, wt, pu, pv;
    std::vector<int> patch_of;
    std::vector<std::size_t> patch_start;  // Q+1

    std::size_t size() const { return pos.size(); }
    std::size_t node(int q, int i, int j) const {
        return patch_start[q] + std::size_t(i) + std::size_t(patches[q].nu) * j;
    }
    std::vector<double> spacing() const;  // per patch max adjacent-node distance (geometry.cpp:93-107)
    double extent() const;                // max bounding-box side (geometry.cpp:109-119)
};

Vec3 patch_point(const Patch& p, double u, double v);  // geometry.cpp:71-75
// tangents, unit normal, Jacobian (geometry.cpp:77-91)
void patch_tangent_frame(const Patch& p, double u, double v, Vec3& tu, Vec3& tv, Vec3& n,
                         double& jac);

// finalise derivative series, orientation and node arrays (geometry.cpp:121-178)
Surface assemble_surface(std::vector<Patch> patches, const Vec3& interior);
// 6·4^splits cube-sphere patches fitted to 1e-12 (geometry.cpp:180-211); nu, nv > 48 is
// accepted here (the fit degree starts at max(nu, nv)) where the reference crashes.
Surface make_sphere(double radius, int splits, int nu, int nv);
// cube-sphere with position series scaled by (ax, ay, az): the BASELINE spheroid (cfg4)
Surface make_spheroid(int splits, int nu, int nv, double ax, double ay, double az);

}  // namespace ifgfb200
