// POD views of the HBM-resident plan, passed by value to the kernels.
#pragma once

#include <cstdint>

namespace ifgfb200 {

// Morton-ordered source/target points (structure of arrays)
struct PointsDev {
    const double *x, *y, *z;
    const double *nx, *ny, *nz;
};

constexpr int kParentMergeMax = 2;  // parent segments per warp item (IFGF_PARENT_MERGE <= this; 3 measured slower)
constexpr int kTmplDoubles = 6;      // parent template entry: ls, lt, lp, ratio1 (re, im), 1/r_c
constexpr int kCbSegs = 16;         // parent segments per cell-batched parent item (parent_cb.cu: 4 per warp)
constexpr int kCbRows = 80;         // rows of a cell-batched (slot, octant) table (75 nodes + padding)
constexpr int kCbTabP = kCbRows * 16;            // table: A2 [80][16], then phi weights [80][8],
constexpr int kCbTabG = kCbTabP + kCbRows * 8;   // then re-centring data [80][4] (ratio1, 1/r_c)
constexpr int kCbTab = kCbTabG + kCbRows * 4;    // doubles per (slot, octant)
constexpr int kCbMaxGrp = 8;        // child-cell groups per (parent cell, octant) in a batched item
#ifndef IFGF_CB_MT3
#define IFGF_CB_MT3 6
#endif
// 8-row tiles per unit of the cell-batched kernel (a larger child-cell group is split in two
// units): IFGF_CB_MT3 where the children carry 3 pipes, 5 otherwise
constexpr int kCbMaxTiles3 = IFGF_CB_MT3, kCbMaxTiles = 5;
constexpr int kCbMaxUnits = 8 * (kCbMaxGrp + 1);  // per warp: per octant its groups, one of which may split

struct LevelDev {
    int d = 0;
    int nb = 0;      // boxes at this level
    int nseg = 0;    // relevant segments
    int ns = 0, nc = 0, ps = 0, pang = 0;
    double ds = 0, dth = 0, dph = 0;
    double inv_ds = 0, inv_dth = 0, inv_dph = 0;
    double h = 0;    // half diagonal of this level's boxes
    const double *cx = nullptr, *cy = nullptr, *cz = nullptr;  // box centres
    const std::uint32_t *beg = nullptr, *end = nullptr;       // Morton spans
    const std::int32_t *cz_ptr = nullptr, *cz_idx = nullptr;  // cousin lists
    const std::int64_t* cev_begin = nullptr;                  // per target box
    const std::int32_t* cev_seg = nullptr;                    // per cousin evaluation
    const std::int32_t *seg_box = nullptr, *seg_gamma = nullptr, *box_seg_begin = nullptr;
    // per segment: (g1, g2, g3) of its cell packed as g1 | g2 << 8 | g3 << 19 (no integer
    // division on the device); null when the grid is too large to pack
    const std::uint32_t* seg_code = nullptr;
    const std::int64_t* pev_begin = nullptr;  // per parent (level d-1) segment
    const std::int32_t* pev_seg = nullptr;    // per parent-node evaluation into this level
    const std::uint16_t* pev_perm = nullptr;  // evaluations grouped by child segment
    const std::int32_t *pgrp_begin = nullptr, *pgrp_seg = nullptr;
    const std::uint16_t *pgrp_start = nullptr, *pgrp_count = nullptr;
    // tensor-core parent kernel work (engine.cu "parent work items"): per item up to
    // kParentMergeMax parent segments of one box (-1: none), its merged groups
    // [pitem_grp[i], pitem_grp[i + 1]) of pgrp_rec = {child segment, child box, start |
    // count << 16 | child octant << 24, cell of the child segment (seg_code layout when
    // seg_code is set, else gamma)} and its evaluations from pev_perm + pitem_ev[i] (node |
    // child slot << 8 | item-local segment << 11 | template bit << 15)
    const int4* pgrp_rec = nullptr;
    const std::int32_t *pitem_seg = nullptr, *pitem_grp = nullptr;
    const std::int64_t* pitem_ev = nullptr;
    int n_pitem = 0;
    int pitem_merge = 1;  // segments per item (the kernel always reserves kParentMergeMax blocks)
    // cell-batched parent work (parent_cb.cu, engine.cu "cell-batched parent items"): item i
    // = up to kCbSegs parent segments of ONE parent cone cell (template slot cb_item_slot[i],
    // segments cb_item_seg[i * kCbSegs + j], -1: none). Per (slot, octant): the 75 nodes in
    // child-cell group order (cb_nodes), group starts (cb_gstart, kCbMaxGrp + 1 entries) and
    // count (host only). Per (item, j, octant): child box (cb_child). Per (item, warp) the
    // host lists the warp's UNITS (cb_unit_begin, 5 ints each in cb_unit): first table row |
    // tiles << 8 | group end row << 16 | octant << 24, then the child segment of each of the
    // warp's 4 parent segments in that (octant, child-cell group) (-1: none). Evaluations
    // whose host-decided child segment differs from the template's group (ties) are
    // exceptions: key j | octant << 8 | node << 16, cso.
    int n_cbitem = 0;
    const std::int32_t *cb_item_slot = nullptr, *cb_item_seg = nullptr;
    const std::uint8_t* cb_nodes = nullptr;
    const std::int32_t *cb_child = nullptr, *cb_unit_begin = nullptr, *cb_unit = nullptr;
    const std::int64_t* cb_exc_begin = nullptr;
    const std::uint32_t* cb_exc_key = nullptr;
    const std::int32_t* cb_exc_cso = nullptr;
    const double* cb_tab = nullptr;  // per (slot, octant): kCbTab doubles (parent_cb.cu cb_table_kernel)
    const std::int32_t *ch_ptr = nullptr, *ch_idx = nullptr;  // children (level d+1) of this level's boxes
    const double *s_nodes = nullptr, *th_nodes = nullptr, *ph_nodes = nullptr;
    // sin/cos of the angular node tables (interpolation-node directions)
    const double *th_sin = nullptr, *th_cos = nullptr, *ph_sin = nullptr, *ph_cos = nullptr;
    // cos/sin of the theta- and phi-cell centres (nc and 2nc entries); null when cells are
    // wider than pi/4 (nc < 4), where local_coords uses acos/atan2
    const double *thc_cos = nullptr, *thc_sin = nullptr, *phc_cos = nullptr, *phc_sin = nullptr;
    // parent-fill geometry templates for this level's children (host/coneplan.hpp
    // parent_templates): slot per cone cell (-1: none) and kTmplDoubles per (slot, octant, node)
    // entry; which evaluations may use them is marked in the child level's pev_perm
    const std::int32_t* tmpl_slot = nullptr;
    const double* tmpl = nullptr;
    // multi-GPU source ownership: box has sources in this rank's Morton range (null = all)
    const std::uint8_t* active = nullptr;
    const std::int32_t *chunk_box = nullptr, *chunk_q0 = nullptr;  // cousin work chunks
    int nchunk = 0;
    const std::int32_t *wchunk_box = nullptr, *wchunk_q0 = nullptr;  // 32-target warp items
    int nwchunk = 0;
    // leaf-fill work items (leaf level): consecutive segments [seg0, seg0 + nseg) of box0
    // (the first `split`) and box1 (the rest; -1: none)
    const std::int32_t *litem_seg0 = nullptr, *litem_nseg = nullptr, *litem_split = nullptr;
    const std::int32_t *litem_box0 = nullptr, *litem_box1 = nullptr;
    int n_litem = 0;
    int max_pts = 0;  // largest box
};

// factor codes carried by one level's coefficient store (W1..W4 = 1..4)
struct Pipes {
    int n = 0;
    int f[3] = {0, 0, 0};
};

}  // namespace ifgfb200
