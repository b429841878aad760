// Launchers of the sm_100a kernels (one translation unit per kernel family).
#pragma once

#include <cuda_runtime.h>

#include "device_plan.cuh"

namespace ifgfb200 {

// index of each factor in a pipe set, -1 if absent
struct PipeIndex {
    int w1 = -1, w2 = -1, w3 = -1, w4 = -1;
};

// ---- IFGF far field (ifgf_kernels.cu) ----
// level-D fill + block transform (ifgf.cpp:312-391), one CTA per leaf box
void launch_leaf_fill(const LevelDev& L, const PointsDev& P, const double2* a_p, double k,
                      const Pipes& pipes, const double* Ms, const double* Ma, double2* store,
                      cudaStream_t st);
// cousin interpolation into the targets (ifgf.cpp:396-450), one CTA per target chunk
void launch_cousin_eval(const LevelDev& L, const PointsDev& P, const double2* store, double k,
                        const Pipes& pipes, double2* Sp, double2* Dp, cudaStream_t st);
// child -> parent re-centred interpolation + block transform (ifgf.cpp:452-568)
void launch_parent_fill(const LevelDev& Lp, const LevelDev& Lc, const double2* child_store,
                        double k, const Pipes& parent_pipes, const Pipes& child_pipes,
                        const double* Ms, const double* Ma, double2* parent_store, cudaStream_t st);

// ray-blocked level-D fill (leaf_ray.cu) for ps = 3; false if not applicable
// tensor-core cousin evaluation (cousin_tc.cu); false when the orders are not (3, 5)
bool launch_cousin_eval_tc(const LevelDev& L, const PointsDev& P, const double2* store, double k, const Pipes& pipes,
                           double2* Sp, double2* Dp, cudaStream_t st);
// leaf-fill work items: segments per item for an angular order, sources per staged tile
int leaf_item_segments(int pang);
int leaf_item_tile();
bool launch_leaf_fill_ray(const LevelDev& L, const PointsDev& P, const double2* a_p, double k, const Pipes& pipes,
                          const double* Ms, const double* Ma, double2* store, cudaStream_t st);
// FP64 tensor-core parent fill (parent_tc.cu) for ps = 3, pang = 5; false if not applicable
// cell-batched items of the level (Lc.n_cbitem), false when there are none
bool launch_parent_fill_cb(const LevelDev& Lp, const LevelDev& Lc, const double2* child_store, double k,
                           const Pipes& parent_pipes, const Pipes& child_pipes, const double* Ms, const double* Ma,
                           double2* parent_store, cudaStream_t st);
// per (slot, octant) tables of the cell-batched parent fill from the geometry templates
void launch_cb_tables(const double* tmpl, const std::uint8_t* nodes, std::int64_t nslot, double* tab, cudaStream_t st);
bool launch_parent_fill_tc(const LevelDev& Lp, const LevelDev& Lc, const double2* child_store, double k,
                           const Pipes& parent_pipes, const Pipes& child_pipes, const double* Ms,
                           const double* Ma, double2* parent_store, cudaStream_t st);

// ---- near field, RP, combine, direct (near_rp_kernels.cu) ----
struct NearDev {
    int n = 0;       // points
    int nleaf = 0;
    const std::uint32_t* perm = nullptr;      // Morton -> original
    const std::uint32_t* beg = nullptr;       // leaf spans
    const std::uint32_t* end = nullptr;
    const std::int32_t *nb_ptr = nullptr, *nb_idx = nullptr;  // leaf neighbours
    const std::int32_t* patch_p = nullptr;    // patch of each Morton point
    const std::uint32_t* tpb = nullptr;       // pairs per ORIGINAL target (CSR, N+1)
    const std::int32_t* pair_patch = nullptr;
    const std::uint32_t *far_begin = nullptr, *far_end = nullptr;
    const std::uint32_t* far_pos = nullptr;   // far nodes as Morton positions
    const std::int32_t *chunk_box = nullptr, *chunk_q0 = nullptr;
    int nchunk = 0;
    const std::uint8_t* leaf_active = nullptr;  // owned target leaves (null = all)
    const std::int32_t* leaf_of_m = nullptr;    // leaf box of each Morton point (warp kernel)
    // near lists (null: screen the neighbourhood every apply): the compacted sources of each
    // Morton target, [list_off[t], list_off[t + 1]) of list_src (Morton indices)
    const std::int64_t* list_off = nullptr;
    const double2* geo = nullptr;  // (x, y), (z, nx), (ny, nz) per Morton point
    std::int32_t* list_src = nullptr;
    // patch runs of each leaf's neighbourhood (near_run_kernel): the neighbour leaves' Morton
    // spans in neighbour order, split where the patch changes (within a leaf the points are in
    // original, i.e. patch-major, order), CSR per leaf
    const std::int32_t* run_ptr = nullptr;
    const std::int32_t *run_start = nullptr, *run_len = nullptr, *run_patch = nullptr;
    // target-pair lists (near_pair_kernel): item w = targets pitem[w] (& 0x7fffffff) and the
    // next one (bit 31: unpaired), union list [plist_off[w], plist_off[w + 1]) of plist_src =
    // source | m << 30 (m bit 0: pair with the first target, bit 1: with the second)
    const std::int32_t* pitem = nullptr;
    int npitem = 0;
    const std::int64_t* plist_off = nullptr;
    std::uint32_t* plist_src = nullptr;
};
void launch_weights(int n, const std::uint32_t* perm, const double2* phi, const double* jw_p,
                    double2* a_p, cudaStream_t st);
// S[perm[t]] = Sp[t], D[perm[t]] = Dp[t]
void launch_unpermute(int n, const std::uint32_t* perm, const double2* Sp, const double2* Dp,
                      double2* S, double2* D, cudaStream_t st);
void launch_near_field(const NearDev& N, const PointsDev& P, const double2* a_p, double k,
                       double2* Sp, double2* Dp, cudaStream_t st);
// near lists: per-target source counts (N.n entries), then the lists at N.list_off
void launch_near_list_count(const NearDev& N, const PointsDev& P, std::int32_t* counts, cudaStream_t st);
void launch_near_list_fill(const NearDev& N, const PointsDev& P, cudaStream_t st);
// target-pair lists: counts per item (counts != null), else the lists at N.plist_off
void launch_near_pair_lists(const NearDev& N, std::int32_t* counts, cudaStream_t st);

struct RpDev {
    int n = 0, npatch = 0;
    const std::int32_t* patch_nu = nullptr;
    const std::int32_t* patch_nv = nullptr;
    const std::int64_t* patch_start = nullptr;   // node start (== coefficient start)
    const std::int32_t* mat_off = nullptr;       // per patch: offsets of (Mu, Mv) in mats
    const double* mats = nullptr;
    const std::uint32_t* tpb = nullptr;          // pairs per original target
    const std::int32_t* pair_patch = nullptr;
    const std::uint64_t* beta_off = nullptr;     // per pair
    const double2 *beta_s = nullptr, *beta_d = nullptr;
    const std::uint32_t* pos = nullptr;          // original -> Morton
    int max_nn = 0;
    std::uint32_t own_lo = 0, own_hi = 0xffffffffu;  // owned Morton target range
    double2* out_m = nullptr;                     // if set: out written in Morton order
};
// out[perm[t]] = out_m[t]
void launch_unpermute1(int n, const std::uint32_t* perm, const double2* in_m, double2* out, cudaStream_t st);
void launch_density_coeffs(const RpDev& R, const double2* phi, double2* coeffs, cudaStream_t st);

// concurrent-apply split of rp_combine: RP accumulated into the near buffers (Morton order),
// then the combine of far (Sp, Dp) + near/RP (Sn, Dn)
void launch_rp_accum(const RpDev& R, const double2* coeffs, double2* Sn, double2* Dn, cudaStream_t st);
void launch_combine(const RpDev& R, const double2* phi, const double2* Sp, const double2* Dp, const double2* Sn,
                    const double2* Dn, double gamma, double2* out, double2* S, double2* D, cudaStream_t st);

// multi-GPU exchange layouts (exchange_kernels.cu): each rank's Morton range padded to C
void launch_pack_ranges(const double2* Sp, const double2* Dp, const std::uint32_t* bounds, int world,
                        std::int64_t C, double2* send, cudaStream_t st);  // send[r][S|D][C]
void launch_unpack_owned(const double2* recv, std::int64_t lo, std::int64_t cnt, std::int64_t C, double2* Sp,
                         double2* Dp, cudaStream_t st);
void launch_copy_pad(const double2* src, std::int64_t cnt, std::int64_t C, double2* dst, cudaStream_t st);
// out[perm[t]] = recv[r(t) C + t - bounds[r(t)]]
void launch_unpermute_padded(std::int64_t n, const std::uint32_t* perm, const std::uint32_t* bounds, int world,
                             std::int64_t C, const double2* recv, double2* out, cudaStream_t st);
// out[i] = in[perm[lo + i]], i < cnt (original-order vector -> owned Morton segment)
void launch_gather_local(const std::uint32_t* perm, std::int64_t lo, std::int64_t cnt, const double2* in,
                         double2* out, cudaStream_t st);
void launch_csqrt_re(double2* h, cudaStream_t st);  // h = (sqrt(re h), 0)

// device-resident GMRES vector kernels (gmres_kernels.cu); reductions deterministic
int gmres_reduce_blocks();
// dst = sum conj(a) b (as_norm: dst = (sqrt(re), 0)); partial holds gmres_reduce_blocks() entries
void launch_cdot(std::int64_t n, const double2* a, const double2* b, double2* partial, double2* dst, bool as_norm,
                 cudaStream_t st);
void launch_caxpy_dev(std::int64_t n, const double2* h, double2* w, const double2* v, cudaStream_t st);  // w -= h v
void launch_cscale_inv(std::int64_t n, const double2* h, const double2* w, double2* v, cudaStream_t st);  // v = w/h
void launch_csub(std::int64_t n, const double2* b, const double2* ax, double2* r, cudaStream_t st);      // r = b - ax
void launch_cupdate(std::int64_t n, int m, const double2* y, const double2* V, std::int64_t ld, double2* x,
                    cudaStream_t st);  // x += sum y_i V_i
// out[l] = 1/2 phi + (D_far+near+rp) - i gamma (S_far+near+rp); S/D written when non-null
void launch_rp_combine(const RpDev& R, const double2* coeffs, const double2* phi,
                       const double2* Sp, const double2* Dp, double gamma, double2* out,
                       double2* S, double2* D, cudaStream_t st);

// non-accelerated: every non-singular pair directly (rp.cpp:481-513), original order
struct DirectDev {
    int n = 0;
    const double *x, *y, *z, *nx, *ny, *nz, *jw;
    const std::int32_t* patch_of;
    const std::uint32_t* tpb;
    const std::int32_t* pair_patch;
};
void launch_direct(const DirectDev& Dd, const double2* phi, double k, double2* S, double2* D,
                   cudaStream_t st);

// ---- beta tables (beta_kernel.cu) ----
struct BetaDev {
    int npairs = 0, n_beta = 0, cov_d = 0;
    double k = 0;
    const std::uint32_t* target = nullptr;
    const std::int32_t* patch = nullptr;
    const double *ubar = nullptr, *vbar = nullptr;
    const std::uint64_t* offset = nullptr;
    const double *tx = nullptr, *ty = nullptr, *tz = nullptr;   // target positions (original order)
    // per patch: dims and series (pos, d/du, d/dv; 3 comps each, du*dv, u fastest)
    const std::int32_t *nu = nullptr, *nv = nullptr, *du = nullptr, *dv = nullptr;
    const double* orient = nullptr;
    const std::int64_t* series_off = nullptr;  // start of the 9 series of a patch
    const double* series = nullptr;
    const double* cutoff = nullptr;            // per patch: max(1e-14, 1e-8 spacing)
    // graded nodes/weights of the current batch (host-computed, glibc pow): batch x n_beta
    const double *grid_u = nullptr, *grid_wu = nullptr, *grid_v = nullptr, *grid_wv = nullptr;
    // pairs to compute, by position (all pairs, or the owned ones of a target-sharded operator)
    const std::uint32_t* pidx = nullptr;
};
std::size_t beta_smem_bytes(int nb, int TT, int max_dv, int max_nu, int max_nunv);
// pairs B.pidx[p_base .. p_base + count) of the batch whose graded rules are in B.grid_*
void launch_beta_batch(const BetaDev& B, int p_base, int count, double2* bs, double2* bd, int TT,
                       int max_dv, int max_nu, int max_nunv, cudaStream_t st);

}  // namespace ifgfb200
