/*
 * ifgf_b200.h — C-ABI of the B200-native combined-field operator apply.
 *
 * Drop-in boundary for the hot path of the IFGF/RP-accelerated CFIE solver
 * (arXiv 2112.06316; reference C++ at /root/reference/proj). Every entry point is plain C:
 * pointers, sizes and status codes, no C++ or CUDA types. Complex vectors are interleaved
 * (re, im) doubles of length 2*N in the ORIGINAL node order l = patch_start[q] + i + nu*j
 * (geometry.hpp:38-50). Status codes map 1:1 onto the reference's exception taxonomy
 * (common.hpp:40-66): 0 ok, 1 InvalidArgument, 2 ParseError, 3 DegenerateGeometry,
 * 4 ConvergenceFailure, 5 InternalError, 6 CUDA failure. ifgf_last_error() returns the
 * thread-local message of the last failure.
 *
 * Reference interfaces replaced (file:line under /root/reference/proj):
 *   ifgf_surface_*          SurfaceMesh, build_sphere, assemble_mesh   geometry.hpp:36-73
 *   ifgf_plan_create        CombinedOperator ctor, host part: build_octree, compute_relations,
 *                           plan_cones, classify_targets, Hybrid resolution
 *                                                                      solver.cpp:43-62
 *   ifgf_operator_create    CombinedOperator ctor incl. beta_precompute solver.hpp:52, rp.cpp:309-395
 *   ifgf_operator_apply     CombinedOperator::apply                    solver.hpp:54, solver.cpp:149-157
 *   ifgf_operator_layer_potentials  CombinedOperator::layer_potentials solver.hpp:56-57
 *   ifgf_operator_apply_direct      CombinedOperator::apply_direct     solver.hpp:59
 *   ifgf_operator_ifgf_apply        ifgf_apply / propagate_and_evaluate ifgf.hpp:106-115
 *   ifgf_operator_level_d_fill      level_d_fill                       ifgf.hpp:92-93
 *   ifgf_operator_rp_apply          rp_singular_apply                  rp.hpp:74-76
 *   ifgf_operator_save/load_beta_cache  save_beta_cache/load_beta_cache rp.hpp:91-94
 *   ifgf_gmres_solve        gmres_solve(std::function apply, ...)      solver.hpp:94-95
 *   ifgf_solve              solve(mesh, incident, cfg)                 solver.hpp:111-112
 *   ifgf_plan_diagnostics   ConePlan::diagnostics                      ifgf.hpp:74
 *   ifgf_far_field          far_field (+ FarFieldGrid::make)           postprocess.hpp:34-37
 *   ifgf_near_field         near_field                                 postprocess.hpp:39-41
 *   ifgf_mie_far_field      mie_far_field                              postprocess.hpp:44-45
 *   ifgf_rp_regular_apply   rp_regular_apply                           rp.hpp:78-82
 *   ifgf_closest_point      closest_point                              rp.hpp:49-51
 *   ifgf_graded             cov_w / cov_w_deriv / cov_xi / cov_xi_deriv rp.hpp:53-57
 *   ifgf_eps_metric         eps_far / eps_near                         postprocess.hpp:49-52
 */
#ifndef IFGF_B200_H
#define IFGF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ifgf_surface ifgf_surface;
typedef struct ifgf_plan ifgf_plan;
typedef struct ifgf_operator ifgf_operator;

/* SolveConfig + ConeConfig + RpConfig (solver.hpp:32-45, ifgf.hpp:12-17, rp.hpp:14-19) */
typedef struct {
    double k;                 /* wavenumber, > 0 */
    double gamma;             /* coupling; <= 0 selects max{3, diameter/lambda} */
    int32_t strategy;         /* 0 = W4, 1 = W2W3, 2 = Hybrid (default) */
    double finest_box_lambda; /* 0.5 */
    int32_t n_c0, n_s0, ps, pang;   /* 2, 1, 3, 5 */
    double delta_rel, delta_abs;    /* 1.0, -1.0 */
    int32_t n_beta, cov_d;          /* 96, 6 */
    int32_t workers;          /* host setup threads, <= 0: all */
    int32_t device;           /* CUDA device ordinal */
    int32_t part_rank, part_world;  /* per-rank plan of a multi-GPU run (0, 1: the full plan):
                                       only boxes with sources of rank part_rank's Morton range */
    const char* beta_cache_path; /* SolveConfig::beta_cache_path: NULL/"" none; else the
                                    "rpbeta v1" cache is loaded when it matches, otherwise
                                    the tables are computed and saved there (solver.cpp:64-74) */
} ifgf_config;

const char* ifgf_last_error(void);
void ifgf_config_default(ifgf_config* cfg);
int ifgf_version(void);

/* ---- surfaces ---- */
int ifgf_surface_sphere(double radius, int splits, int nu, int nv, ifgf_surface** out);
int ifgf_surface_spheroid(int splits, int nu, int nv, double ax, double ay, double az,
                          ifgf_surface** out);
/* Patches from position series: dims = {nu, nv, du, dv} per patch; coeff = concatenated
 * 3*du*dv per patch (component-major, u fastest). Assembled like assemble_mesh. */
int ifgf_surface_from_series(int npatch, const int32_t* dims, const double* coeff,
                             const double interior[3], ifgf_surface** out);
/* Exact import of an already assembled mesh (no re-evaluation): series (position, d/du,
 * d/dv, each 3*du*dv per patch), orientation and the flat node arrays (pos/normal 3N). */
int ifgf_surface_import(int npatch, const int32_t* dims, const double* orient,
                        const double* coeff, const double* coeff_u, const double* coeff_v,
                        const double interior[3], int64_t n, const double* pos,
                        const double* normal, const double* jac, const double* weight,
                        const double* pu, const double* pv, ifgf_surface** out);
int64_t ifgf_surface_size(const ifgf_surface* s);
int ifgf_surface_npatches(const ifgf_surface* s);
double ifgf_surface_diameter(const ifgf_surface* s);
/* any pointer may be NULL */
int ifgf_surface_nodes(const ifgf_surface* s, double* pos, double* normal, double* jac,
                       double* weight, double* pu, double* pv, int32_t* patch_of);
int ifgf_surface_patch(const ifgf_surface* s, int q, int32_t* dims4, double* orient,
                       double* coeff, double* coeff_u, double* coeff_v);
void ifgf_surface_free(ifgf_surface* s);
/* density U(-1,1) + i U(-1,1) from std::mt19937_64(seed), drawn as the reference harness
 * draws it (tools/main.cpp:252-254) */
int ifgf_random_density(int64_t n, uint64_t seed, double* out);

/* ---- host plan (CPU only: octree, relations, cone plan, proximity) ---- */
int ifgf_plan_create(const ifgf_surface* s, const ifgf_config* cfg, ifgf_plan** out);
void ifgf_plan_free(ifgf_plan* p);
int ifgf_plan_depth(const ifgf_plan* p);
double ifgf_plan_gamma(const ifgf_plan* p);
int ifgf_plan_strategy(const ifgf_plan* p);       /* resolved (solver.cpp:55-62) */
double ifgf_plan_setup_seconds(const ifgf_plan* p);
int ifgf_plan_perm(const ifgf_plan* p, uint32_t* perm);
int ifgf_plan_tree_geom(const ifgf_plan* p, double root_min[3], double* root_side);
int64_t ifgf_plan_nboxes(const ifgf_plan* p, int level);
int ifgf_plan_boxes(const ifgf_plan* p, int level, uint64_t* key, int32_t* cell3,
                    uint32_t* begin, uint32_t* end, int32_t* parent, int32_t* child8);
/* which: 0 neighbours, 1 cousins; ptr may be NULL for a size query */
int64_t ifgf_plan_relation(const ifgf_plan* p, int level, int which, int32_t* ptr, int32_t* idx);
/* params4 = {ns, nc, ps, pang}; returns segment count; box/gamma may be NULL */
int64_t ifgf_plan_level(const ifgf_plan* p, int level, int32_t* params4, double* deltas3,
                        int32_t* seg_box, int32_t* seg_gamma);
/* number of cousin / parent-node evaluations planned at a level */
int64_t ifgf_plan_evaluations(const ifgf_plan* p, int level, int which);
/* cousin DMMA tile statistics of a level for warp items of `items_of` targets:
 * out3 = (evaluations, segment groups, 8-row tiles) (kernel design diagnostics) */
int ifgf_plan_cousin_tile_stats(const ifgf_plan* p, int level, int items_of, int64_t* out3);
int64_t ifgf_plan_npairs(const ifgf_plan* p);
/* {groups, evaluations, 8-row tensor-core tiles} of the parent-node evaluations into level */
int ifgf_plan_tile_stats(const ifgf_plan* p, int level, int64_t* out3);
int64_t ifgf_plan_nfar(const ifgf_plan* p);
int ifgf_plan_pairs(const ifgf_plan* p, uint32_t* target, int32_t* patch, double* ubar,
                    double* vbar, uint32_t* far_begin, uint32_t* far_end,
                    uint32_t* target_pair_begin, uint32_t* far_nodes);
uint64_t ifgf_plan_beta_fingerprint(const ifgf_plan* p);
int ifgf_plan_diagnostics(const ifgf_plan* p, char* buf, size_t cap);
/* algorithmic work of one apply, 16 doubles:
 * [0] leaf interactions  [1] cousin evaluations  [2] parent evaluations
 * [3] near pairs (evaluated + corrections)  [4] RP pairs
 * [5..9]  flops of leaf, cousin, parent, near, RP (SURVEY.md §8(d) counting)
 * [10..14] algorithmic HBM bytes of leaf, cousin, parent, near, RP  [15] total flops */
/* FNV-1a hash of a level's per-evaluation segment ordinals (cousin and parent) and the
 * grouped parent permutation: compares plans built with and without the GPU decider */
uint64_t ifgf_plan_decision_hash(const ifgf_plan* p, int level);
int ifgf_plan_work(const ifgf_plan* p, double* work16);
int ifgf_operator_work(const ifgf_operator* op, double* work16);

/* ---- device operator ---- */
/* host setup + HBM upload + beta tables on the GPU */
int ifgf_operator_create(const ifgf_surface* s, const ifgf_config* cfg, ifgf_operator** out);
/* from an existing plan (the plan is shared, not copied); compute_beta = 0 leaves the
 * tables to ifgf_operator_set_beta / ifgf_operator_load_beta_cache */
int ifgf_operator_from_plan(ifgf_plan* p, int device, int compute_beta, ifgf_operator** out);
void ifgf_operator_free(ifgf_operator* op);
int64_t ifgf_operator_size(const ifgf_operator* op);
/* setup phases in seconds: {octree+relations, cone plan, proximity, HBM upload, GPU beta} */
int ifgf_operator_setup_times(const ifgf_operator* op, double* t5);
double ifgf_operator_gamma(const ifgf_operator* op);
int ifgf_operator_apply(ifgf_operator* op, const double* phi, double* out);
int ifgf_operator_layer_potentials(ifgf_operator* op, const double* phi, double* S, double* D);
int ifgf_operator_apply_device(ifgf_operator* op, const void* phi_dev, void* out_dev);
int ifgf_operator_apply_direct(ifgf_operator* op, const double* phi, double* out);
/* a = quadrature-weighted sources; strategy < 0: the operator's resolved strategy */
int ifgf_operator_ifgf_apply(ifgf_operator* op, const double* a, int single, int dbl,
                             int strategy, double* S, double* D);
/* returns number of complex values written (or needed, when out == NULL); -status on error */
int64_t ifgf_operator_level_d_fill(ifgf_operator* op, const double* a_perm, const int32_t* pipes,
                                   int npipes, double* out, int64_t capacity);
int ifgf_operator_rp_apply(ifgf_operator* op, const double* phi, double* S, double* D);
int64_t ifgf_operator_beta_entries(const ifgf_operator* op);
int64_t ifgf_operator_npairs(const ifgf_operator* op);
int ifgf_operator_set_beta(ifgf_operator* op, const uint64_t* offset, const double* bs,
                           const double* bd);
int ifgf_operator_get_beta(ifgf_operator* op, uint64_t* offset, double* bs, double* bd);
/* "rpbeta v1" cache, interchangeable with the reference's (rp.cpp:515-570);
 * load returns 1 when the cache was used, 0 when absent/mismatched */
int ifgf_operator_save_beta_cache(ifgf_operator* op, const char* path);
int ifgf_operator_load_beta_cache(ifgf_operator* op, const char* path);
/* 1 when ifgf_operator_create took the tables from cfg->beta_cache_path
 * (CombinedOperator::beta_cache_was_reused, solver.hpp:70) */
int ifgf_operator_beta_cache_hit(const ifgf_operator* op);
/* benchmark helpers: phi resident in HBM, CUDA-graph replays timed with CUDA events */
int ifgf_operator_upload_density(ifgf_operator* op, const double* phi);
int ifgf_operator_time_applies(ifgf_operator* op, int iters, int flush_l2, double* ms_per_apply);
/* ms for {weights, leaf, cousin, parent, near, rp, total} of one instrumented apply */
/* device time of each of iters graph applies (ms_each: iters entries) */
int ifgf_operator_time_applies_each(ifgf_operator* op, int iters, int flush_l2, double* ms_each);
int ifgf_operator_time_phases(ifgf_operator* op, double* ms7);
int ifgf_operator_kernels_per_apply(const ifgf_operator* op);
void* ifgf_operator_device_phi(ifgf_operator* op);
void* ifgf_operator_device_out(ifgf_operator* op);

/* ---- multi-GPU (one process per GPU, NCCL over NVLink) ----
 * Each operator owns the sources and targets of a leaf-aligned Morton range: the far
 * field is computed from owned sources for ALL targets and reduced to the target owners
 * (grouped ncclReduce), near field + RP run target-owned, the owners broadcast their
 * outputs. Every rank passes the full phi and receives the full out. */
int ifgf_nccl_unique_id(void* id128);
/* collective over the world; computes the cost-balanced partition and takes part `rank` */
int ifgf_operator_set_comm(ifgf_operator* op, int rank, int world, const void* id128);
/* cost-balanced, leaf-aligned Morton boundaries: parts + 1 values (host only) */
int ifgf_operator_partition(const ifgf_operator* op, int parts, uint32_t* bounds);
int ifgf_plan_partition(const ifgf_plan* p, int parts, uint32_t* bounds);
/* own [lo, hi) without a communicator (single-GPU emulation of one rank) */
/* (re)compute the beta tables on the GPU: all pairs, or — after set_partition / set_comm — only
 * the pairs whose target this operator owns (target-sharded tables) */
int ifgf_operator_compute_beta(ifgf_operator* op);
int ifgf_operator_set_partition(ifgf_operator* op, uint32_t lo, uint32_t hi);
/* near field + RP + combine for the owned targets given the full far field S, D
 * (original order, e.g. the sum of every rank's ifgf_operator_ifgf_apply); out is zero
 * outside the owned targets */
int ifgf_operator_finish_owned(ifgf_operator* op, const double* phi, const double* far_S,
                               const double* far_D, double* out);

/* ---- GMRES (solver.cpp:169-340 semantics: MGS, Givens, optional restart) ---- */
int ifgf_gmres_solve(ifgf_operator* op, const double* rhs, double tol, int max_iter,
                     int restart, double* x, double* history, int history_cap,
                     int* iterations, int* converged);
/* plane wave along (cos t sin p, sin t sin p, cos p) (solver.hpp:23-25), rhs = -u^i */
int ifgf_solve(ifgf_operator* op, double theta, double phi, double tol, int max_iter,
               int restart, double* density, double* history, int history_cap,
               int* iterations, int* converged);
/* solve(mesh, incident, cfg) for either IncidentField kind (solver.hpp:17-26): point sources
 * src (3*nsrc) when nsrc > 0, else the plane wave (theta, phi) */
int ifgf_solve_incident(ifgf_operator* op, double theta, double phi, const double* src, int64_t nsrc,
                        double tol, int max_iter, int restart, double* density, double* history,
                        int history_cap, int* iterations, int* converged);
/* incident_trace (solver.hpp:28-30): u^i at the nodes, 2*N doubles */
int ifgf_incident_trace(const ifgf_surface* s, double k, double theta, double phi,
                        const double* src, int64_t nsrc, double* out);

/* closest point on patch q to x (3) from (u0, v0): alternating golden-section sweeps
 * (rp.hpp:49-51); out = (u, v, dist), bit-identical to the reference */
int ifgf_closest_point(const ifgf_surface* s, int q, const double* x, double u0, double v0, double* out);
/* graded change of variables around alpha (rp.hpp:53-57): which = 0 w, 1 w', 2 xi, 3 xi' */
double ifgf_graded(int which, double alpha, double tau, int d);

/* ---- fields after the solve (postprocess.cpp). The dense sums run on
 * GPU `device` over the oversampled per-patch Fejér quadrature of the density. ---- */
/* far-field pattern on the (n_phi x n_theta) grid, polar index fastest (postprocess.cpp:62-104):
 * dirs (3*n_phi*n_theta, may be NULL) and values (2*n_phi*n_theta) */
int ifgf_far_field(const ifgf_surface* s, const double* density, double gamma, double k, int n_phi,
                   int n_theta, int device, double* dirs, double* values);
/* scattered / total field at npts points (3*npts) for plane-wave incidence (theta, phi) or,
 * when nsrc > 0, point sources src (3*nsrc, solver.cpp:25-35); flagged[i] = 1 within
 * flag_distance of the quadrature or inside the scatterer (postprocess.cpp:106-139) */
int ifgf_near_field(const ifgf_surface* s, const double* density, double gamma, double k,
                    double inc_theta, double inc_phi, const double* src, int64_t nsrc,
                    const double* points, int64_t npts, double flag_distance, int device,
                    double* scattered, double* total, uint8_t* flagged);
/* regular Fejér-rule S and D of the density at off-surface targets (3*n), ADDED into S / D
 * (2*n each); a target within 1e-14 of a node is InvalidArgument (rp.cpp:453-479) */
int ifgf_rp_regular_apply(const ifgf_surface* s, const double* density, const double* targets,
                          int64_t ntargets, double k, int device, double* S, double* D);
/* sound-soft sphere far field for a plane wave along direction (3) at n directions (3*n) */
int ifgf_mie_far_field(double radius, double k, const double* direction, const double* dirs,
                       int64_t n, int extra_terms, double* values);
/* max | |ref| - |apx| | / |ref| over nonzero ref (complex interleaved, length 2n) */
int ifgf_eps_metric(const double* ref, const double* apx, int64_t n, double* eps, int* skipped);

#ifdef __cplusplus
}
#endif
#endif /* IFGF_B200_H */
