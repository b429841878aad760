// Singular / near-singular (target, patch) pairs for the RP correction and the near-field
// exclusion lists. Restates classify_targets (/root/reference/proj/src/rp.cpp:194-289) and
// its golden-section closest_point (rp.cpp:22-43, 122-137) with identical decisions; the
// pair set, (ubar, vbar) and the far-node correction lists feed the hot path.
#pragma once

#include <cstdint>
#include <functional>
#include <vector>

#include "boxtree.hpp"
#include "surface.hpp"

namespace ifgfb200 {

struct RpParams {
    double delta_rel = 1.0;
    double delta_abs = -1.0;
    int n_beta = 96;
    int cov_d = 6;
};

struct PairList {
    RpParams cfg;
    std::vector<double> delta;                   // per patch
    std::vector<std::uint32_t> target;           // per pair (original node index)
    std::vector<std::int32_t> patch;
    std::vector<double> ubar, vbar;
    std::vector<std::uint32_t> far_begin, far_end;
    std::vector<std::uint32_t> target_pair_begin;  // N + 1
    std::vector<std::uint32_t> far_nodes;          // original node indices
    std::size_t size() const { return target.size(); }
};

struct ClosestPoint {
    double u = 0, v = 0, dist = 0;
};
ClosestPoint closest_point_on(const Patch& p, const Vec3& x, double u0, double v0);

// one closest-point search of classify_pairs: target node, patch, start parameters (the
// nearest node's); `own` pairs (the target's own patch) need no search
struct ClosestPointRequest {
    std::uint32_t target;
    std::int32_t q;
    double u0, v0;
    bool own;
};
// batched solver for the non-own requests (the GPU one: cuda/proximity_kernels.cu); must
// return closest_point_on's results bit for bit
using ClosestPointBatch = std::function<void(const Surface&, const std::vector<ClosestPointRequest>&,
                                             std::vector<ClosestPoint>&)>;

// owned (per original node, optional): only those targets get pairs (per-rank plans)
PairList classify_pairs(const Surface& s, const BoxTree& t, const BoxRelations& rel,
                        const RpParams& cfg, int workers, const ClosestPointBatch* batch = nullptr,
                        const std::vector<std::uint8_t>* owned = nullptr);

// graded change of variables (rp.cpp:139-192)
double grade_w(double tau, int d);
double grade_w_deriv(double tau, int d);
double grade_xi(double alpha, double tau, int d);
double grade_xi_deriv(double alpha, double tau, int d);

// graded Fejér nodes/weights of pairs [p0, p1) (rp.cpp:345-351): out arrays are
// (p1-p0) x n_beta, pair-major; computed with glibc pow exactly as the reference does
void graded_rules(const PairList& pl, std::size_t p0, std::size_t p1, const std::vector<double>& rx,
                  const std::vector<double>& rw, double* u, double* wu, double* v, double* wv,
                  int workers);
// the same for the pairs idx[0 .. count) (output row i = pair idx[i])
void graded_rules(const PairList& pl, const std::uint32_t* idx, std::size_t count, const std::vector<double>& rx,
                  const std::vector<double>& rw, double* u, double* wu, double* v, double* wv, int workers);

// FNV-1a fingerprint of everything the beta tables depend on (rp.cpp:291-307), so beta
// caches written here and by the reference are interchangeable.
std::uint64_t beta_key(const Surface& s, const PairList& pl, double k);

}  // namespace ifgfb200
