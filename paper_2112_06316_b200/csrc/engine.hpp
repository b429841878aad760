// The B200 CF-operator engine: owns the HBM-resident plan (Morton-ordered sources, box
// levels, cone work lists, near-field and RP lists, beta tables) and runs the per-apply
// kernel sequence on one stream, captured once into a CUDA graph.
//
//   out = 1/2 phi + D[phi] - i gamma S[phi]          (solver.cpp:149-157)
//
// Plain C++ interface (no CUDA types) so the host setup code and the C-ABI can include it.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "host/boxtree.hpp"
#include "host/gmres.hpp"
#include "host/coneplan.hpp"
#include "host/proximity.hpp"
#include "host/surface.hpp"

namespace ifgfb200 {

struct OperatorSetup {
    double k = 0, gamma = 0;
    DlStrategy strategy = DlStrategy::Hybrid;  // resolved (solver.cpp:55-62)
    const Surface* surf = nullptr;
    const BoxTree* tree = nullptr;
    const BoxRelations* rel = nullptr;
    const ConePlanHost* plan = nullptr;
    const PairList* pairs = nullptr;
};

// Per-phase device times of the last timed apply (ms), CUDA events on the engine stream.
struct PhaseTimes {
    double weights = 0, leaf = 0, cousin = 0, parent = 0, near = 0, rp = 0, total = 0;
};

class Engine {
  public:
    Engine(const OperatorSetup& s, int device);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    std::size_t size() const;
    int device() const;

    // beta tables: computed on the GPU from the pair list (graded Fejér rule), or uploaded
    void compute_beta();
    void upload_beta(const std::vector<std::uint64_t>& offset, const cplx* bs, const cplx* bd);
    void download_beta(std::vector<std::uint64_t>& offset, std::vector<cplx>& bs, std::vector<cplx>& bd);

    // host buffers in original node order; S/D optional
    void apply(const cplx* phi, cplx* out, cplx* S = nullptr, cplx* D = nullptr);
    // device pointers (complex interleaved), stream-ordered on the engine stream then synced
    void apply_device(const void* phi_dev, void* out_dev, void* S_dev = nullptr, void* D_dev = nullptr);
    // only the far field on quadrature-weighted sources a (original order)
    void ifgf_apply(const cplx* a, bool single, bool dbl, DlStrategy strategy, cplx* S, cplx* D);
    // level-D Chebyshev blocks on Morton-ordered sources (seg-major, pipe, 75 coefficients)
    void level_d_fill(const cplx* a_perm, const std::vector<int>& pipes, std::vector<cplx>& out);
    // non-accelerated operator: singular pairs via beta, everything else direct (rp.cpp:481-513)
    void apply_direct(const cplx* phi, cplx* out);
    // RP correction alone (rp.cpp:421-451), outputs overwritten
    void rp_apply(const cplx* phi, cplx* S, cplx* D);

    // restarted MGS-GMRES on the device (solver.cpp:177-300 semantics): Krylov basis in HBM,
    // operator applies from the captured graph, only Hessenberg columns cross to the host.
    // rhs in original node order. Under a communicator every rank runs the same iteration
    // on replicated vectors (the applies are collective, the reductions deterministic).
    GmresOutcome gmres(const cplx* rhs, double tol, int max_iter, int restart);

    // ---- multi-GPU: each engine owns the sources and targets of a
    // leaf-aligned Morton range; the far field is computed from owned sources for all
    // targets and reduced to the target owners, near field + RP run target-owned.
    // cost-balanced boundaries (parts + 1 Morton indices)
    std::vector<std::uint32_t> partition_bounds(int parts) const;
    void set_partition(std::uint32_t lo, std::uint32_t hi);
    // NCCL communicator from a 128-byte ncclUniqueId; sets the partition of `rank`
    void set_comm(int rank, int world, const void* unique_id);
    // near field + RP + combine for the owned targets only, given the full far field
    // (original order); out is zero outside the owned targets
    void finish_owned(const cplx* phi, const cplx* far_S, const cplx* far_D, cplx* out);

    // benchmark helpers: graph replays with device-resident phi (no host copies)
    void upload_density(const cplx* phi);
    double time_device_applies(int iters, bool flush_l2);   // mean ms per apply
    std::vector<double> time_device_applies_each(int iters, bool flush_l2);  // ms of each apply
    PhaseTimes time_phases();                               // one instrumented apply
    int kernels_per_apply() const;
    std::string describe() const;
    void* device_phi();
    void* device_out();
    void sync();

    struct Impl;

  private:
    std::unique_ptr<Impl> d_;
};

}  // namespace ifgfb200
