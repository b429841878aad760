// Cone-segment plan of the IFGF far field, precompiled into device work lists.
//
// The reference decides, during every apply, which cone segment each cousin target point
// and each parent interpolation node falls into (ifgf.cpp:161-176 via cartesian_to_cone,
// kernels.cpp:34-48). Those decisions hinge on the last ulp of glibc acos/atan2 (3,168
// exact ties at cfg1), so they are taken ONCE here, on the host, with
// the reference's own expressions, and shipped to HBM as per-evaluation segment ordinals.
// The B200 kernels then only recompute the continuous local coordinates. The relevance
// marking is the reference's plan_cones (ifgf.cpp:209-296); the cone geometry is
// make_level_cones / doublings_for_side (ifgf.cpp:18-55).
#pragma once

#include <cstdint>
#include <functional>
#include <vector>

#include "boxtree.hpp"

namespace ifgfb200 {

struct ConeParams {
    int n_c0 = 2, n_s0 = 1, ps = 3, pang = 5;  // ifgf.hpp:12-17 defaults
};

enum Factor : int { W1 = 1, W2 = 2, W3 = 3, W4 = 4 };
enum class DlStrategy : int { W4 = 0, W2W3 = 1, Hybrid = 2 };

struct ConeLevel {
    int d = 0;
    int ns = 0, nc = 0, ps = 0, pang = 0;
    double ds = 0, dth = 0, dph = 0;
    std::vector<double> s_nodes, th_nodes, ph_nodes;  // ns*ps, nc*pang, 2nc*pang

    std::vector<std::int32_t> seg_box, seg_gamma;  // relevant segments, (box, gamma) order
    std::vector<std::int32_t> box_seg_begin;       // nboxes + 1
    // cousin lists the plan evaluates (BoxRelations::cousin, restricted to source boxes with
    // owned sources in a per-rank plan)
    Adjacency cz;

    // cousin evaluations, target-box major: for box tb, cousin j (ascending cousin list),
    // point t of tb -> segment ordinal of the cousin box at this level
    std::vector<std::int64_t> cev_begin;  // nboxes + 1
    std::vector<std::int32_t> cev_seg;
    // parent-node evaluations of level d-1 segments into this level's segments:
    // parent segment so, node (is + ps*(it + pang*ip)), child slot c -> child segment ordinal
    std::vector<std::int64_t> pev_begin;  // nseg(d-1) + 1 (empty at d = 3)
    std::vector<std::int32_t> pev_seg;
    // the same evaluations grouped by child segment, per parent segment (FP64 tensor-core
    // tiles need 8 evaluations of one coefficient block): pev_perm lists local indices
    // (node * nch + c) in group order; group g of parent segment so covers
    // [pgrp_start[g], pgrp_start[g] + pgrp_count[g]) of that list and uses pgrp_seg[g];
    // when nodes_per_seg <= 255 the entries are packed as node | c << 8
    std::vector<std::uint16_t> pev_perm;
    std::vector<std::int32_t> pgrp_begin;  // nseg(d-1) + 1
    std::vector<std::int32_t> pgrp_seg;
    std::vector<std::uint16_t> pgrp_start, pgrp_count;

    int segs_per_box() const { return ns * nc * 2 * nc; }
    int nodes_per_seg() const { return ps * pang * pang; }
    std::size_t nseg() const { return seg_box.size(); }
};

struct ConePlanHost {
    ConeParams params;
    double k = 0;
    std::vector<ConeLevel> level;  // level[d-1], valid for 3 <= d <= depth
    // per leaf/coarse level: children lists compacted in slot order (nch <= 8)
    std::vector<std::vector<std::int32_t>> child_ptr, child_idx;  // [d-1] over boxes of level d
    // per-rank plan (multi-GPU): only boxes holding sources of the Morton range
    // [bounds[rank], bounds[rank + 1]) carry segments; world == 1: the full plan
    int rank = 0, world = 1;
    std::vector<std::uint32_t> bounds;
};

int cone_doublings(double side, double lambda);  // ifgf.cpp:18-25
std::vector<int> dl_pipes(const BoxTree& t, int level, DlStrategy s);  // ifgf.cpp:193-207

// Segment decisions of one level, for a batched (GPU) decider: every cousin evaluation
// (cev, target-box major as ConeLevel::cev_seg) and every parent-node evaluation (pev) gets
// the gamma of the segment it falls into, and marks[box * segs_per_box + gamma] is set.
// A decider may leave decisions it cannot guarantee to equal glibc's acos/atan2 to the host:
// it lists them in flagged_cev / flagged_pev (their gamma and marks are then ignored).
struct ConeDecisionJob {
    const ConeLevel* L = nullptr;        // this level (ns, nc, ds, dth, dph)
    double h = 0;                        // half diagonal of this level's boxes
    const std::vector<Vec3>* pts = nullptr;   // Morton-ordered points
    const std::vector<Vec3>* ctr = nullptr;   // box centres of this level
    const BoxLevel* B = nullptr;
    const Adjacency* cz = nullptr;             // cousin lists
    // parent part (level d - 1), absent at d = 3
    const ConeLevel* PL = nullptr;
    double ph = 0;                              // parent half diagonal
    const std::vector<Vec3>* pctr = nullptr;    // parent centres (level d - 1)
    const std::vector<std::int32_t>* cptr = nullptr;  // children of parent boxes (compacted)
    const std::vector<std::int32_t>* cidx = nullptr;
    std::vector<double> th_sin, th_cos, ph_sin, ph_cos;  // glibc sin/cos of the parent node tables
};
using ConeDecider = std::function<void(const ConeDecisionJob& job, ConeLevel& L, std::vector<std::uint8_t>& marks,
                                       std::vector<std::int64_t>& flagged_cev, std::vector<std::int64_t>& flagged_pev)>;

// active: per level [d-1], per box, 1 if the box holds sources this plan covers (null = all)
ConePlanHost build_cone_plan(const BoxTree& t, const BoxRelations& rel,
                             const std::vector<Vec3>& pts_morton, const ConeParams& p,
                             int workers, const ConeDecider* decider = nullptr,
                             const std::vector<std::vector<std::uint8_t>>* active = nullptr);

// leaf-aligned Morton boundaries from a plan-free cost model (points, neighbour and cousin
// point counts per leaf), for building per-rank plans before any cone plan exists
std::vector<std::uint32_t> partition_sources_light(const BoxTree& t, const BoxRelations& rel, int parts);
// per level, per box: 1 if the box holds sources of the Morton range [lo, hi)
std::vector<std::vector<std::uint8_t>> active_boxes(const BoxTree& t, std::uint32_t lo, std::uint32_t hi);

// Parent-fill geometry templates (device data, not decisions). The position of a parent
// interpolation node relative to a child box depends only on the parent cone cell, the
// node and the child's octant (box centres are exact grid points up to one rounding), so
// per (parent cell gamma_p, octant, node) the child cell the node falls in and its
// continuous data are tabulated once per level: entry = {ls, lt, lp, re/im of
// (r_p/r_c) e^{ik(r_c - r_p)}, 1/r_c} (6 doubles; r_p/r_c = (h_p/s) (1/r_c) is formed on the
// device where needed) and gc = child cell. The
// per-box decisions stay the host's (pev ordinals); a device evaluation uses an entry only
// when gc equals its host-decided child cell. d = child level (parent level d - 1).
void parent_templates(const BoxTree& t, const ConePlanHost& plan, int d, const std::vector<std::int32_t>& gammas,
                      int workers, uninit_vector<double>& entries, std::vector<std::int32_t>& gc);

// Cost-balanced, leaf-aligned Morton boundaries (parts + 1) of the multi-GPU source/target
// ownership: per leaf box, near pairs, leaf-fill interactions and cousin
// and parent evaluations weighted by their flops
std::vector<std::uint32_t> partition_sources(const BoxTree& t, const BoxRelations& rel, const ConePlanHost& plan,
                                             int parts);

// textual per-level counts, the reference's ConePlan::diagnostics (ifgf.cpp:298-310)
std::string plan_diagnostics(const BoxTree& t, const ConePlanHost& plan);

}  // namespace ifgfb200
