// Uniform-depth Morton box hierarchy over the surface nodes, plus the neighbour and
// cousin relations. Restates /root/reference/proj/src/octree.cpp:37-186 (build_octree,
// compute_relations) with the same decisions (bounding cube, depth rule, floor cells,
// stable (key, index) sort), stored level-wise as structure-of-arrays so the arrays can be
// uploaded to HBM unchanged.
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "core.hpp"

namespace ifgfb200 {

struct BoxLevel {
    std::vector<std::uint64_t> key;           // Morton key at this level, ascending
    std::vector<std::array<std::int32_t, 3>> cell;
    std::vector<std::uint32_t> begin, end;    // span into the Morton permutation
    std::vector<std::int32_t> parent;         // index into level d-1
    std::vector<std::array<std::int32_t, 8>> child;  // slot = key & 7, -1 if absent
    std::size_t size() const { return key.size(); }
};

struct BoxTree {
    int depth = 0;
    Vec3 root_min;
    double root_side = 0;
    double k = 0;
    std::vector<std::uint32_t> perm;      // Morton position -> original node
    std::vector<std::int32_t> leaf_of;    // original node -> leaf box
    std::vector<BoxLevel> level;          // level[d-1]

    double side(int d) const { return root_side / double(1u << (d - 1)); }
    Vec3 center(int d, std::size_t b) const {
        const double H = side(d);
        const auto& c = level[d - 1].cell[b];
        return root_min + Vec3{(c[0] + 0.5) * H, (c[1] + 0.5) * H, (c[2] + 0.5) * H};
    }
    double half_diag(int d) const { return kHalfDiag * side(d); }
    int find(int d, std::uint64_t key) const;
};

std::uint64_t morton_key(std::uint32_t x, std::uint32_t y, std::uint32_t z);

BoxTree build_boxtree(const std::vector<Vec3>& pts, double k, double finest_box_lambda);

// CSR adjacency per level; each list ascending.
struct Adjacency {
    std::vector<std::int32_t> ptr, idx;
    std::size_t count(std::size_t b) const { return std::size_t(ptr[b + 1] - ptr[b]); }
};
struct BoxRelations {
    std::vector<Adjacency> nbr, cousin;  // [d-1]
};
BoxRelations build_relations(const BoxTree& t);

}  // namespace ifgfb200
