// Engine: uploads the host plan into HBM once and runs the per-apply kernel sequence
//
//   weights -> leaf_fill(D) -> [cousin_eval(d) -> parent_fill(d -> d-1)]_{d=D..4}
//   -> cousin_eval(3) -> near_field -> density_coeffs -> rp_combine
//
// on one stream, captured into a CUDA graph after the first eager apply (ifgf_apply,
// ifgf.cpp:577-608; layer_potentials + apply, solver.cpp:78-157). Only two IFGF levels of
// coefficient blocks are live at a time (ifgf.cpp:589-597), in two ping-pong buffers.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <array>
#include <atomic>
#include <type_traits>
#include <cstdlib>
#include <string>
#include <cstring>
#include <mutex>
#include <sstream>

#include "../engine.hpp"
#include "../host/chebyshev.hpp"
#include "dev_common.cuh"
#include "kernels.cuh"

namespace ifgfb200 {

#define IFGF_NCCL(call)                                                                     \
    do {                                                                                     \
        ncclResult_t r_ = (call);                                                            \
        if (r_ != ncclSuccess)                                                               \
            throw ::ifgfb200::EngineError(::ifgfb200::kNcclError,                            \
                                          std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)

namespace {

constexpr int kChunk = 128;  // targets per CTA in the cousin / near-field work lists

// Host -> HBM uploads through pinned staging buffers: the host threads copy chunk i into one
// pinned buffer while the copy engine moves chunk i - 1 from the other (a synchronous
// pageable cudaMemcpy per array ran at ~4 GB/s: 15 s of cfg3's setup). Inside an
// UploadBatch the copies are left in flight and the batch waits once at its end; outside
// one every upload waits for its own copies.
class Uploader {
  public:
    static Uploader& get() {
        thread_local Uploader u;
        int dev = 0;
        IFGF_CUDA(cudaGetDevice(&dev));
        if (u.dev_ != dev) u.init(dev);
        return u;
    }
    void copy(void* dst, const void* src, std::size_t bytes) {
        if (bytes < (std::size_t(1) << 20)) {  // small: not worth the staging
            IFGF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st_));
            if (!batch_) IFGF_CUDA(cudaStreamSynchronize(st_));
            return;
        }
        for (std::size_t off = 0; off < bytes; off += kChunk) {
            const std::size_t len = std::min(kChunk, bytes - off);
            IFGF_CUDA(cudaEventSynchronize(ev_[cur_]));  // this buffer's previous copy is done
            char* pin = pin_[cur_];
            const char* s = static_cast<const char*>(src) + off;
            const std::int64_t parts = std::int64_t((len + (std::size_t(4) << 20) - 1) >> 22);
#pragma omp parallel for schedule(static) num_threads(16)
            for (std::int64_t q = 0; q < parts; ++q) {
                const std::size_t a = std::size_t(q) << 22, n = std::min(std::size_t(4) << 20, len - a);
                std::memcpy(pin + a, s + a, n);
            }
            IFGF_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, pin, len, cudaMemcpyHostToDevice, st_));
            IFGF_CUDA(cudaEventRecord(ev_[cur_], st_));
            cur_ ^= 1;
        }
        if (!batch_) IFGF_CUDA(cudaStreamSynchronize(st_));
    }
    void begin_batch() { ++batch_; }
    cudaError_t end_batch() noexcept {  // called from a destructor: reports, never throws
        return --batch_ == 0 ? cudaStreamSynchronize(st_) : cudaSuccess;
    }
    ~Uploader() { release(); }

  private:
    static constexpr std::size_t kChunk = std::size_t(64) << 20;
    void release() {
        for (int i = 0; i < 2; ++i) {
            if (pin_[i]) cudaFreeHost(pin_[i]);
            if (ev_[i]) cudaEventDestroy(ev_[i]);
            pin_[i] = nullptr;
            ev_[i] = nullptr;
        }
        if (st_) cudaStreamDestroy(st_);
        st_ = nullptr;
        cur_ = 0;
    }
    void init(int dev) {
        release();
        dev_ = dev;
        IFGF_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            IFGF_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&pin_[i]), kChunk, cudaHostAllocDefault));
            IFGF_CUDA(cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming));
        }
    }
    int dev_ = -1, cur_ = 0, batch_ = 0;
    cudaStream_t st_ = nullptr;
    char* pin_[2] = {nullptr, nullptr};
    cudaEvent_t ev_[2] = {nullptr, nullptr};
};

struct UploadBatch {
    Uploader& u;
    UploadBatch() : u(Uploader::get()) { u.begin_batch(); }
    ~UploadBatch() { (void)u.end_batch(); }  // the engine's final cudaDeviceSynchronize reports errors
};

class DevBuf {
  public:
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), bytes_(o.bytes_) {
        o.p_ = nullptr;
        o.bytes_ = 0;
    }
    ~DevBuf() {
        if (p_) cudaFree(p_);
    }
    void alloc(std::size_t bytes) {
        if (p_) cudaFree(p_);
        p_ = nullptr;
        bytes_ = bytes;
        if (bytes) IFGF_CUDA(cudaMalloc(&p_, bytes));
    }
    template <class T, class A>
    void upload(const std::vector<T, A>& v) {
        alloc(v.size() * sizeof(T));
        if (!v.empty()) Uploader::get().copy(p_, v.data(), v.size() * sizeof(T));
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p_);
    }
    std::size_t bytes() const { return bytes_; }

  private:
    void* p_ = nullptr;
    std::size_t bytes_ = 0;
};

struct LevelBufs {
    DevBuf cx, cy, cz, beg, end, cz_ptr, cz_idx, cev_begin, cev_seg, seg_box, seg_gamma,
        box_seg_begin, pev_begin, pev_seg, pev_perm, pgrp_begin, pgrp_seg, pgrp_start, pgrp_count, ch_ptr, ch_idx, s_nodes, th_nodes, ph_nodes, th_sin, th_cos, ph_sin, ph_cos, thc_cos, thc_sin, phc_cos, phc_sin,
        chunk_box, chunk_q0, wchunk_box, wchunk_q0, tmpl_slot, tmpl, seg_code, litem_seg0,
        litem_nseg, litem_split, litem_box0, litem_box1, pgrp_rec, pitem_seg, pitem_grp, pitem_ev;
    DevBuf cb_item_slot, cb_item_seg, cb_nodes, cb_child, cb_unit_begin, cb_unit, cb_exc_begin, cb_exc_key,
        cb_exc_cso, cb_tab;
};

Pipes make_pipes(const std::vector<int>& f) {
    Pipes p;
    p.n = int(f.size());
    for (int i = 0; i < p.n && i < 3; ++i) p.f[i] = f[i];
    return p;
}

}  // namespace

struct Engine::Impl {
    int dev = 0;
    cudaStream_t st = nullptr;
    cudaStream_t st2 = nullptr;            // side stream: near field + RP, concurrent with the IFGF
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // cousin stream: cousin(d) beside parent(d); ev_store[d] = level d's store ready (on st),
    // ev_cousin[d] = cousin(d) done reading it (on st3)
    cudaStream_t st3 = nullptr;
    std::vector<cudaEvent_t> ev_store, ev_cousin;
    std::mutex mu;
    std::size_t n = 0;
    int depth = 0;
    double k = 0, gamma = 0;
    DlStrategy strategy = DlStrategy::Hybrid;
    int ps = 3, pang = 5;
    const Surface* surf = nullptr;
    const PairList* pairs = nullptr;
    const BoxTree* tree = nullptr;
    const BoxRelations* rel = nullptr;
    const ConePlanHost* cones = nullptr;

    // points (Morton order)
    DevBuf px, py, pz, pnx, pny, pnz, jw_p, ones_p, perm, pos, patch_p, identity;
    DevBuf pgeo;  // (x, y), (z, nx), (ny, nz) per Morton point: one 48-byte row per near-pair source
    // original order copies for the direct sum and beta
    DevBuf ox, oy, oz, onx, ony, onz, ojw, opatch;
    std::vector<LevelBufs> lb;   // [d-1]
    std::vector<LevelDev> L;     // [d-1]
    DevBuf Ms, Ma;
    DevBuf storeA, storeB;
    std::size_t store_elems = 0;
    std::size_t capA = 0, capB = 0;  // complex entries of the two stores
    // The IFGF stores alternate: level d lives in storeA when D - d is even (the leaf level,
    // then every second level), else in storeB. Each is sized for ITS levels' segments x
    // pipes of the request (cfg3: 11.5 + 8.5 GB instead of 2 x 13 GB for 3 pipes everywhere);
    // a request with more pipes (another strategy) grows them, dropping the captured graph.
    void ensure_stores(bool single, bool dbl, DlStrategy s, int leaf_pipes = -1) {
        std::size_t a = 1, b = 1;
        for (int d = 3; d <= depth; ++d) {
            const int np = (d == depth && leaf_pipes > 0) ? leaf_pipes : int(pipes_at(d, single, dbl, s).size());
            const std::size_t need = std::size_t(L[d - 1].nseg) * std::size_t(L[d - 1].ps * L[d - 1].pang * L[d - 1].pang) * np;
            ((depth - d) % 2 == 0 ? a : b) = std::max((depth - d) % 2 == 0 ? a : b, need);
        }
        if (a > capA) {
            storeA.alloc(a * sizeof(double2));
            capA = a;
            drop_graph();
        }
        if (b > capB) {
            storeB.alloc(b * sizeof(double2));
            capB = b;
            drop_graph();
        }
        store_elems = std::max(capA, capB);
    }
    // near field
    DevBuf nb_ptr, nb_idx, leaf_of_m, tpb, pair_patch, far_begin, far_end, far_pos, near_chunk_box, near_chunk_q0;
    DevBuf near_off, near_src;  // near lists (ensure_near_lists)
    DevBuf near_pitem;          // target-pair items of the pair lists
    DevBuf run_ptr, run_start, run_len, run_patch;  // neighbourhood patch runs (near_run_kernel)
    bool near_lists_done = false;
    NearDev near;
    // rp
    DevBuf patch_nu, patch_nv, patch_start, mat_off, mats, beta_off, beta_s, beta_d, coeffs;
    RpDev rp;
    std::size_t beta_entries = 0;
    bool beta_ready = false;
    bool beta_sharded = false;              // tables hold only the owned targets' pairs
    std::vector<std::uint64_t> beta_off_full;  // per pair offsets of the full tables (host)

    // storage for the pairs in `pairs_idx` (all pairs when empty list means full), offsets
    // compacted; non-stored pairs get offset 0 and are never read (their targets are not owned)
    void alloc_beta(const std::vector<std::uint32_t>* owned) {
        std::vector<std::uint64_t> off;
        std::size_t entries;
        if (!owned) {
            off = beta_off_full;
            entries = beta_off_full.back();
        } else {
            off.assign(beta_off_full.size(), 0);
            std::uint64_t acc = 0;
            for (std::uint32_t p : *owned) {
                off[p] = acc;
                acc += beta_off_full[p + 1] - beta_off_full[p];
            }
            entries = acc;
        }
        beta_off.upload(off);
        beta_s.alloc(std::max<std::size_t>(entries, 1) * sizeof(double2));
        beta_d.alloc(std::max<std::size_t>(entries, 1) * sizeof(double2));
        rp.beta_off = beta_off.as<std::uint64_t>();
        rp.beta_s = beta_s.as<double2>();
        rp.beta_d = beta_d.as<double2>();
        beta_sharded = owned != nullptr;
        beta_stale = false;
        beta_lo = own_lo;
        beta_hi = own_hi;
        drop_graph();
    }
    std::uint32_t beta_lo = 0, beta_hi = 0;  // owned range the sharded tables were built for
    // beta inputs
    DevBuf b_target, b_ubar, b_vbar, b_du, b_dv, b_orient, b_series_off, b_series, b_cutoff,
        b_gu, b_gwu, b_gv, b_gwv;
    std::vector<double> rule_x, rule_w;
    int max_dudv = 1, max_nunv = 1, max_dv = 1, max_nu = 1;
    // work vectors
    DevBuf d_phi, d_out, d_S, d_D, a_p, Sp, Dp, Sn, Dn, scratch, flush;
    PointsDev P;
    DirectDev direct;
    // graph of the full apply on (d_phi -> d_out, d_S, d_D)
    cudaGraphExec_t graph = nullptr;
    bool eager_done = false;
    int kernels = 0;

    std::vector<int> pipes_at(int d, bool single, bool dbl, DlStrategy s) const {
        std::vector<int> p;
        if (single) p.push_back(W1);
        if (dbl) {
            const auto x = dl_pipes(*tree, d, s);
            p.insert(p.end(), x.begin(), x.end());
        }
        return p;
    }

    // the IFGF far field on a_p (Morton) into Sp/Dp (accumulated)
    // after_leaf (optional) is issued right after the leaf-fill launch: side-stream work then
    // queues behind the leaf's CTAs and fills the room they leave
    template <class F = void (*)()>
    int run_ifgf(bool single, bool dbl, DlStrategy s, cudaEvent_t* ev = nullptr, F after_leaf = nullptr) {
        int launches = 0;
        if (depth < 3 || (!single && !dbl)) {
            if constexpr (!std::is_same_v<F, void (*)()>) after_leaf();
            return 0;
        }
        double2* cur = storeA.as<double2>();
        double2* nxt = storeB.as<double2>();
        auto pipes_d = make_pipes(pipes_at(depth, single, dbl, s));
        launch_leaf_fill(L[depth - 1], P, a_p.as<double2>(), k, pipes_d, Ms.as<double>(),
                         Ma.as<double>(), cur, st);
        ++launches;
        if constexpr (!std::is_same_v<F, void (*)()>) after_leaf();
        if (ev) IFGF_CUDA(cudaEventRecord(ev[0], st));
        // cousin(d) on st3 beside parent(d) on st (both only read level d's store); parent(d)
        // overwrites level d+1's store, so it waits for cousin(d+1); the cousins stay in level
        // order on one stream, so every target's sums are added in the same order as serially
        const char* cenv = std::getenv("IFGF_COUSIN_STREAM");
        const bool two = !ev && !(cenv && cenv[0] == '0') && st3;
        for (int d = depth; d >= 3; --d) {
            const Pipes pc = make_pipes(pipes_at(d, single, dbl, s));
            if (two) {
                IFGF_CUDA(cudaEventRecord(ev_store[d], st));
                IFGF_CUDA(cudaStreamWaitEvent(st3, ev_store[d], 0));
                launch_cousin_eval(L[d - 1], P, cur, k, pc, Sp.as<double2>(), Dp.as<double2>(), st3);
                IFGF_CUDA(cudaEventRecord(ev_cousin[d], st3));
                if (d < depth) IFGF_CUDA(cudaStreamWaitEvent(st, ev_cousin[d + 1], 0));
            } else {
                launch_cousin_eval(L[d - 1], P, cur, k, pc, Sp.as<double2>(), Dp.as<double2>(), st);
            }
            ++launches;
            if (d > 3) {
                const Pipes pp = make_pipes(pipes_at(d - 1, single, dbl, s));
                launch_parent_fill(L[d - 2], L[d - 1], cur, k, pp, pc, Ms.as<double>(),
                                   Ma.as<double>(), nxt, st);
                ++launches;
                std::swap(cur, nxt);
            }
        }
        if (two) IFGF_CUDA(cudaStreamWaitEvent(st, ev_cousin[3], 0));  // join before Sp/Dp are read
        return launches;
    }

    // full operator on d_phi -> out, S, D (device pointers). The near field and the RP
    // correction do not depend on the far field: they run on the side stream st2 into
    // (Sn, Dn) while the IFGF fills (Sp, Dp) on st; a combine kernel joins both.
    // local_out (sharded GMRES): the owned outputs stay in out_m[own_lo, own_hi) (Morton
    // order), no gather
    int run_apply(const double2* phi, double2* out, double2* S, double2* D, bool local_out = false) {
        ensure_near_lists();
        int launches = 0;
        const std::size_t vb = n * sizeof(double2);
        IFGF_CUDA(cudaMemsetAsync(Sp.as<void>(), 0, vb, st));
        IFGF_CUDA(cudaMemsetAsync(Dp.as<void>(), 0, vb, st));
        IFGF_CUDA(cudaMemsetAsync(Sn.as<void>(), 0, vb, st));
        IFGF_CUDA(cudaMemsetAsync(Dn.as<void>(), 0, vb, st));
        launch_weights(int(n), perm.as<std::uint32_t>(), phi, jw_p.as<double>(), a_p.as<double2>(), st);
        ++launches;
        // IFGF_SIDE_STREAM: 0 (default) = everything on st; 1 = near field and RP on the side
        // stream; rp = only the (HBM-bound) RP on the side stream. Measured: cfg3 456.7 ms
        // serial against 462.4 (1) and 461.9 (rp): every kernel fills the GPU on its own and
        // the concurrent ones slow each other; cfg2 20.48 / 20.40 / 20.44 ms
        static const int side_mode = [] {
            const char* e = std::getenv("IFGF_SIDE_STREAM");
            if (e && e[0] == '1') return 1;
            if (e && std::string(e) == "rp") return 2;
            return 0;
        }();
        const bool one_stream = side_mode == 0;
        cudaStream_t side = one_stream ? st : st2;
        cudaStream_t near_st = side_mode == 1 ? side : st;
        if (!one_stream) {
            IFGF_CUDA(cudaEventRecord(ev_fork, st));
            IFGF_CUDA(cudaStreamWaitEvent(st2, ev_fork, 0));
        }
        auto side_work = [&] {
            launch_near_field(near, P, a_p.as<double2>(), k, Sn.as<double2>(), Dn.as<double2>(), near_st);
            launch_density_coeffs(rp, phi, coeffs.as<double2>(), side);
            launch_rp_accum(rp, coeffs.as<double2>(), Sn.as<double2>(), Dn.as<double2>(), side);
            IFGF_CUDA(cudaEventRecord(ev_join, side));
        };
        // measured (cfg2): side work issued before the leaf fill is fastest with the warp-per-
        // target near kernel; IFGF_SIDE_ORDER=after_leaf queues it behind the leaf instead
        static const bool side_first = [] {
            const char* e = std::getenv("IFGF_SIDE_ORDER");
            return !(e && std::string(e) == "after_leaf");
        }();
        launches += 3;
        if (side_first || one_stream) {
            side_work();
            launches += run_ifgf(true, true, strategy);
        } else {
            launches += run_ifgf(true, true, strategy, nullptr, side_work);
        }
        if (collective()) launches += reduce_far_to_owners();  // far-field partials -> target owners
        IFGF_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
        RpDev r = rp;
        if (collective()) {  // owned targets in Morton order, then exchanged
            r.out_m = out_m.as<double2>();
            S = D = nullptr;
        }
        launch_combine(r, phi, Sp.as<double2>(), Dp.as<double2>(), Sn.as<double2>(), Dn.as<double2>(), gamma, out, S,
                       D, st);
        ++launches;
        if (collective() && !local_out) launches += gather_out_from_owners(out);
        return launches;
    }

    bool beta_stale = false;
    void ensure_beta() {
        if (beta_stale)
            throw InternalError("beta tables are target-sharded for another Morton range: compute_beta again");
        if (!beta_ready) throw InternalError("beta tables not computed");
    }

    // Near lists: the screening of every target's neighbourhood (self and singular-patch
    // exclusions) runs once, on the device, and its compacted sources are kept in HBM (4 bytes
    // per near pair) so the per-apply near kernel only evaluates pairs. Built at the first
    // eager apply after construction or a partition change (never under graph capture);
    // skipped when the lists would not leave the reserve below free in HBM, or with
    // IFGF_NEAR_LISTS=0.
    void ensure_near_lists() {
        if (near_lists_done) return;
        cudaStreamCaptureStatus cs;
        IFGF_CUDA(cudaStreamIsCapturing(st, &cs));
        if (cs != cudaStreamCaptureStatusNone) throw InternalError("near lists requested under graph capture");
        near_lists_done = true;
        near.list_off = nullptr;
        near.list_src = nullptr;
        near.plist_off = nullptr;
        near.plist_src = nullptr;
        near_off.alloc(0);
        near_src.alloc(0);
        // target-pair lists unless another near kernel is requested (IFGF_NEAR=lists |
        // runs | screen | thread); where they do not fit, the patch-run kernel (no per-pair
        // data) takes over
        const char* env = std::getenv("IFGF_NEAR");
        if ((env && std::string(env) != "lists" && std::string(env) != "pairs") || !near.leaf_of_m || near.n == 0) return;
        // keep a reserve for the solver's Krylov basis and work vectors (GMRES at restart 50
        // needs 51 x 16 N bytes): IFGF_NEAR_LISTS_RESERVE_GB, default max(6 GB, 51 x 16 N)
        const char* renv = std::getenv("IFGF_NEAR_LISTS_RESERVE_GB");
        const std::size_t reserve = renv ? std::size_t(std::atof(renv) * 1e9)
                                         : std::max<std::size_t>(std::size_t(6e9), 51 * 16 * n);
        if (!(env && std::string(env) == "lists") && near.npitem > 0) {
            DevBuf cnt;
            cnt.alloc(std::size_t(near.npitem) * sizeof(std::int32_t));
            launch_near_pair_lists(near, cnt.as<std::int32_t>(), st);
            std::vector<std::int32_t> c(near.npitem);
            IFGF_CUDA(cudaMemcpyAsync(c.data(), cnt.as<void>(), c.size() * sizeof(std::int32_t), cudaMemcpyDeviceToHost, st));
            IFGF_CUDA(cudaStreamSynchronize(st));
            std::vector<std::int64_t> off(std::size_t(near.npitem) + 1, 0);
            for (int t = 0; t < near.npitem; ++t) off[t + 1] = off[t] + c[t];
            const std::size_t bytes = std::size_t(off.back()) * sizeof(std::uint32_t) + off.size() * sizeof(std::int64_t);
            std::size_t free_b = 0, total_b = 0;
            IFGF_CUDA(cudaMemGetInfo(&free_b, &total_b));
            if (std::getenv("IFGF_SETUP_DEBUG"))
                std::fprintf(stderr, "near pair lists: %.2f GB (%lld entries), free %.2f GB\n", bytes / 1e9,
                             (long long)off.back(), free_b / 1e9);
            if (bytes + reserve > free_b) return;
            near_off.upload(off);
            near_src.alloc(std::max<std::size_t>(std::size_t(off.back()), 1) * sizeof(std::uint32_t));
            near.plist_off = near_off.as<std::int64_t>();
            near.plist_src = near_src.as<std::uint32_t>();
            launch_near_pair_lists(near, nullptr, st);
            IFGF_CUDA(cudaStreamSynchronize(st));
            return;
        }
        DevBuf cnt;
        cnt.alloc(std::size_t(near.n) * sizeof(std::int32_t));
        launch_near_list_count(near, P, cnt.as<std::int32_t>(), st);
        std::vector<std::int32_t> c(near.n);
        IFGF_CUDA(cudaMemcpyAsync(c.data(), cnt.as<void>(), c.size() * sizeof(std::int32_t), cudaMemcpyDeviceToHost, st));
        IFGF_CUDA(cudaStreamSynchronize(st));
        std::vector<std::int64_t> off(std::size_t(near.n) + 1, 0);
        for (int t = 0; t < near.n; ++t) off[t + 1] = off[t] + c[t];
        const std::size_t bytes = std::size_t(off.back()) * sizeof(std::int32_t) + off.size() * sizeof(std::int64_t);
        std::size_t free_b = 0, total_b = 0;
        IFGF_CUDA(cudaMemGetInfo(&free_b, &total_b));
        if (std::getenv("IFGF_SETUP_DEBUG"))
            std::fprintf(stderr, "near lists: %.2f GB, free %.2f GB\n", bytes / 1e9, free_b / 1e9);
        if (bytes + reserve > free_b) return;
        near_off.upload(off);
        near_src.alloc(std::max<std::size_t>(std::size_t(off.back()), 1) * sizeof(std::int32_t));
        near.list_off = near_off.as<std::int64_t>();
        near.list_src = near_src.as<std::int32_t>();
        launch_near_list_fill(near, P, st);
        IFGF_CUDA(cudaStreamSynchronize(st));
    }

    // ---- multi-GPU: source ownership by Morton ranges of leaf boxes
    std::uint32_t own_lo = 0, own_hi = 0;
    bool partitioned = false;
    std::vector<DevBuf> active;  // per level, uint8 per box
    int rank = 0, world = 1;
    std::vector<std::uint32_t> bounds;  // world + 1 Morton boundaries
    ncclComm_t comm = nullptr;
    DevBuf out_m;

    void drop_graph() {
        if (graph) cudaGraphExecDestroy(graph);
        graph = nullptr;
        eager_done = false;
    }

    // Morton range [lo, hi) of sources (and targets) owned by this engine; leaf-box aligned
    void set_partition(std::uint32_t lo, std::uint32_t hi) {
        if (lo > hi || hi > n) throw InvalidArgument("partition: bad Morton range");
        // a per-rank plan holds only its own range's boxes: no other range is valid for it
        if (cones->world > 1 && (lo != cones->bounds[cones->rank] || hi != cones->bounds[cones->rank + 1]))
            throw InvalidArgument("partition: a per-rank plan only serves its own Morton range");
        // target-sharded tables hold only the pairs of the range they were built for
        if (beta_sharded && beta_ready && (lo != beta_lo || hi != beta_hi)) {
            beta_ready = false;
            beta_stale = true;
        }
        own_lo = lo;
        own_hi = hi;
        partitioned = !(lo == 0 && hi == n);
        near_lists_done = false;  // rebuilt for the owned targets at the next eager apply
        const bool all = lo == 0 && hi == n;
        active.resize(depth);
        for (int d = 3; d <= depth; ++d) {
            const BoxLevel& B = tree->level[d - 1];
            std::vector<std::uint8_t> a(B.size());
            for (std::size_t b = 0; b < B.size(); ++b) a[b] = (B.begin[b] < hi && B.end[b] > lo) ? 1 : 0;
            active[d - 1].upload(a);
            L[d - 1].active = all ? nullptr : active[d - 1].as<std::uint8_t>();
        }
        const BoxLevel& leaves = tree->level[depth - 1];
        for (std::size_t b = 0; b < leaves.size(); ++b)
            if ((leaves.begin[b] < lo && leaves.end[b] > lo) || (leaves.begin[b] < hi && leaves.end[b] > hi))
                throw InvalidArgument("partition: range splits a leaf box");
        if (depth < 3) {  // leaf activity for the near field
            std::vector<std::uint8_t> a(leaves.size());
            for (std::size_t b = 0; b < leaves.size(); ++b) a[b] = (leaves.begin[b] < hi && leaves.end[b] > lo) ? 1 : 0;
            active.resize(depth);
            active[depth - 1].upload(a);
        }
        near.leaf_active = all ? nullptr : active[depth - 1].as<std::uint8_t>();
        rp.own_lo = all ? 0u : lo;
        rp.own_hi = all ? 0xffffffffu : hi;
        drop_graph();
    }

    std::vector<std::uint32_t> partition(int parts) const {
        if (cones->world > 1) {  // a per-rank plan carries its partition
            if (parts != cones->world) throw InvalidArgument("partition: the plan is per rank of a different world");
            return cones->bounds;
        }
        return partition_sources(*tree, *rel, *cones, parts);
    }

    // The per-apply exchange: ONE ncclReduceScatter of the far-field
    // partials (S and D of every rank's range, padded to the longest range C) delivers each
    // owner the sums over ranks of its targets, then ONE ncclAllGather of the owned outputs.
    bool collective() const { return comm != nullptr; }
    std::int64_t chunk = 0;  // C: the longest owned range
    DevBuf ex_send, ex_recv, ag_send, ag_recv, d_bounds;

    void alloc_exchange() {
        chunk = 0;
        for (int r = 0; r < world; ++r) chunk = std::max<std::int64_t>(chunk, bounds[r + 1] - bounds[r]);
        const std::size_t C = std::size_t(std::max<std::int64_t>(chunk, 1));
        ex_send.alloc(std::size_t(world) * 2 * C * sizeof(double2));
        ex_recv.alloc(2 * C * sizeof(double2));
        ag_send.alloc(C * sizeof(double2));
        ag_recv.alloc(std::size_t(world) * C * sizeof(double2));
        d_bounds.upload(bounds);
    }

    int reduce_far_to_owners() {
        const std::uint32_t* bd = d_bounds.as<std::uint32_t>();
        launch_pack_ranges(Sp.as<double2>(), Dp.as<double2>(), bd, world, chunk, ex_send.as<double2>(), st);
        IFGF_NCCL(ncclReduceScatter(ex_send.as<double>(), ex_recv.as<double>(), std::size_t(4 * chunk), ncclFloat64,
                                    ncclSum, comm, st));
        launch_unpack_owned(ex_recv.as<double2>(), own_lo, std::int64_t(own_hi - own_lo), chunk, Sp.as<double2>(),
                            Dp.as<double2>(), st);
        return 2;
    }

    // this rank's owned Morton segment `seg` (own_hi - own_lo entries) -> every rank's
    // original-order full vector `out`
    int allgather_to_original(const double2* seg, double2* out) {
        launch_copy_pad(seg, std::int64_t(own_hi - own_lo), chunk, ag_send.as<double2>(), st);
        IFGF_NCCL(ncclAllGather(ag_send.as<double>(), ag_recv.as<double>(), std::size_t(2 * chunk), ncclFloat64, comm,
                                st));
        launch_unpermute_padded(std::int64_t(n), perm.as<std::uint32_t>(), d_bounds.as<std::uint32_t>(), world, chunk,
                                ag_recv.as<double2>(), out, st);
        return 2;
    }
    int gather_out_from_owners(double2* out) { return allgather_to_original(out_m.as<double2>() + own_lo, out); }

    bool nccl_graph_failed = false;
    void apply_graph() {
        // under a communicator the NCCL calls are captured with the kernels (one graph launch
        // per apply on every rank); IFGF_NCCL_GRAPH=0 runs them eagerly
        static const bool nccl_graph = [] {
            const char* e = std::getenv("IFGF_NCCL_GRAPH");
            return !(e && e[0] == '0');
        }();
        if (collective() && (!nccl_graph || nccl_graph_failed)) {
            kernels = run_apply(d_phi.as<double2>(), d_out.as<double2>(), d_S.as<double2>(), d_D.as<double2>());
            eager_done = true;
            return;
        }
        if (!eager_done) {
            kernels = run_apply(d_phi.as<double2>(), d_out.as<double2>(), d_S.as<double2>(),
                                d_D.as<double2>());
            IFGF_CUDA(cudaStreamSynchronize(st));
            eager_done = true;
            cudaGraph_t g;
            IFGF_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            try {
                run_apply(d_phi.as<double2>(), d_out.as<double2>(), d_S.as<double2>(), d_D.as<double2>());
            } catch (...) {
                cudaStreamEndCapture(st, &g);
                if (g) cudaGraphDestroy(g);
                cudaGetLastError();
                if (!collective()) throw;
                nccl_graph_failed = true;  // this NCCL cannot be captured: eager from now on
                return;
            }
            IFGF_CUDA(cudaStreamEndCapture(st, &g));
            IFGF_CUDA(cudaGraphInstantiate(&graph, g, 0));
            IFGF_CUDA(cudaGraphDestroy(g));
            return;
        }
        IFGF_CUDA(cudaGraphLaunch(graph, st));
    }
};

Engine::Engine(const OperatorSetup& s, int device) : d_(std::make_unique<Impl>()) {
    Impl& e = *d_;
    e.dev = device;
    IFGF_CUDA(cudaSetDevice(device));
    UploadBatch batch;  // plan uploads stay in flight until the end of the constructor
    // IFGF_SETUP_DEBUG: host wall time of each setup phase (uploads are asynchronous)
    const bool phase_dbg = std::getenv("IFGF_SETUP_DEBUG") != nullptr;
    auto phase_t0 = std::chrono::steady_clock::now();
    std::string phase_name = "start";
    auto phase_mark = [&](const char* next) {
        const auto t = std::chrono::steady_clock::now();
        if (phase_dbg)
            std::fprintf(stderr, "engine setup %-20s %.3f s\n", phase_name.c_str(),
                         std::chrono::duration<double>(t - phase_t0).count());
        phase_t0 = t;
        phase_name = next;
    };
    IFGF_CUDA(cudaStreamCreateWithFlags(&e.st, cudaStreamNonBlocking));
    IFGF_CUDA(cudaStreamCreateWithFlags(&e.st2, cudaStreamNonBlocking));
    IFGF_CUDA(cudaEventCreateWithFlags(&e.ev_fork, cudaEventDisableTiming));
    IFGF_CUDA(cudaEventCreateWithFlags(&e.ev_join, cudaEventDisableTiming));
    IFGF_CUDA(cudaStreamCreateWithFlags(&e.st3, cudaStreamNonBlocking));
    e.ev_store.assign(64, nullptr);
    e.ev_cousin.assign(64, nullptr);
    for (int d = 0; d < 64; ++d) {
        IFGF_CUDA(cudaEventCreateWithFlags(&e.ev_store[d], cudaEventDisableTiming));
        IFGF_CUDA(cudaEventCreateWithFlags(&e.ev_cousin[d], cudaEventDisableTiming));
    }
    const Surface& S = *s.surf;
    const BoxTree& T = *s.tree;
    const BoxRelations& R = *s.rel;
    const ConePlanHost& C = *s.plan;
    const PairList& PL = *s.pairs;
    e.surf = s.surf;
    e.pairs = s.pairs;
    e.tree = s.tree;
    e.rel = s.rel;
    e.cones = s.plan;
    e.n = S.size();
    e.depth = T.depth;
    e.k = s.k;
    e.gamma = s.gamma;
    e.strategy = s.strategy;
    e.ps = C.params.ps;
    e.pang = C.params.pang;
    const std::size_t n = e.n;

    phase_mark("points");
    // ---- points in Morton order
    {
        std::vector<double> x(n), y(n), z(n), nx(n), ny(n), nz(n), jw(n), one(n, 1.0);
        std::vector<std::uint32_t> pos(n), ident(n);
        std::vector<std::int32_t> pp(n);
        for (std::size_t t = 0; t < n; ++t) {
            const std::uint32_t l = T.perm[t];
            x[t] = S.pos[l].x;
            y[t] = S.pos[l].y;
            z[t] = S.pos[l].z;
            nx[t] = S.nrm[l].x;
            ny[t] = S.nrm[l].y;
            nz[t] = S.nrm[l].z;
            jw[t] = S.jac[l] * S.wt[l];
            pos[l] = std::uint32_t(t);
            pp[t] = S.patch_of[l];
            ident[t] = std::uint32_t(t);
        }
        {
            std::vector<double> g(6 * n);
            for (std::size_t t = 0; t < n; ++t) {
                g[6 * t] = x[t];
                g[6 * t + 1] = y[t];
                g[6 * t + 2] = z[t];
                g[6 * t + 3] = nx[t];
                g[6 * t + 4] = ny[t];
                g[6 * t + 5] = nz[t];
            }
            e.pgeo.upload(g);
        }
        e.px.upload(x);
        e.py.upload(y);
        e.pz.upload(z);
        e.pnx.upload(nx);
        e.pny.upload(ny);
        e.pnz.upload(nz);
        e.jw_p.upload(jw);
        e.ones_p.upload(one);
        e.perm.upload(T.perm);
        e.pos.upload(pos);
        e.patch_p.upload(pp);
        e.identity.upload(ident);
        e.P = {e.px.as<double>(), e.py.as<double>(), e.pz.as<double>(),
               e.pnx.as<double>(), e.pny.as<double>(), e.pnz.as<double>()};
        for (std::size_t l = 0; l < n; ++l) {
            x[l] = S.pos[l].x;
            y[l] = S.pos[l].y;
            z[l] = S.pos[l].z;
            nx[l] = S.nrm[l].x;
            ny[l] = S.nrm[l].y;
            nz[l] = S.nrm[l].z;
            jw[l] = S.jac[l] * S.wt[l];
        }
        e.ox.upload(x);
        e.oy.upload(y);
        e.oz.upload(z);
        e.onx.upload(nx);
        e.ony.upload(ny);
        e.onz.upload(nz);
        e.ojw.upload(jw);
        e.opatch.upload(S.patch_of);
    }

    phase_mark("levels");
    // ---- IFGF levels
    e.lb.resize(T.depth);
    e.L.resize(T.depth);
    std::size_t store = 0;
    for (int d = 3; d <= T.depth; ++d) {
        const BoxLevel& B = T.level[d - 1];
        const ConeLevel& CL = C.level[d - 1];
        LevelBufs& b = e.lb[d - 1];
        LevelDev& L = e.L[d - 1];
        const std::size_t nb = B.size();
        std::vector<double> cx(nb), cy(nb), cz(nb);
        int max_pts = 0;
        for (std::size_t i = 0; i < nb; ++i) {
            const Vec3 c = T.center(d, i);
            cx[i] = c.x;
            cy[i] = c.y;
            cz[i] = c.z;
            max_pts = std::max(max_pts, int(B.end[i] - B.begin[i]));
        }
        std::vector<std::int32_t> chunk_box, chunk_q0;
        for (std::size_t i = 0; i < nb; ++i)
            if (CL.cz.count(i) > 0)
                for (std::uint32_t q = 0; q < B.end[i] - B.begin[i]; q += kChunk) {
                    chunk_box.push_back(std::int32_t(i));
                    chunk_q0.push_back(std::int32_t(q));
                }
        std::vector<std::int32_t> wchunk_box, wchunk_q0;  // one warp per 32 targets
        for (std::size_t i = 0; i < nb; ++i)
            if (CL.cz.count(i) > 0)
                for (std::uint32_t q = 0; q < B.end[i] - B.begin[i]; q += 32) {
                    wchunk_box.push_back(std::int32_t(i));
                    wchunk_q0.push_back(std::int32_t(q));
                }
        b.wchunk_box.upload(wchunk_box);
        b.wchunk_q0.upload(wchunk_q0);
        L.wchunk_box = b.wchunk_box.as<std::int32_t>();
        L.wchunk_q0 = b.wchunk_q0.as<std::int32_t>();
        L.nwchunk = int(wchunk_box.size());
        if (d == T.depth) {  // leaf-fill items: <= G consecutive segments of at most two boxes
            const int G = leaf_item_segments(CL.pang), tile = leaf_item_tile();
            std::vector<std::int32_t> i_s0, i_n, i_split, i_b0, i_b1;
            int cs0 = 0, cn = 0, cb0 = -1, cb1 = -1, csplit = 0;
            auto flush = [&] {
                if (cn == 0) return;
                i_s0.push_back(cs0);
                i_n.push_back(cn);
                i_split.push_back(cb1 < 0 ? cn : csplit);
                i_b0.push_back(cb0);
                i_b1.push_back(cb1);
                cn = 0;
                cb0 = cb1 = -1;
            };
            for (std::size_t bx = 0; bx < nb; ++bx) {
                int s = CL.box_seg_begin[bx];
                int S = CL.box_seg_begin[bx + 1] - s;
                if (S == 0) continue;
                const bool big = int(B.end[bx] - B.begin[bx]) > tile;
                if (big) flush();  // a box streaming its sources in tiles gets items of its own
                while (S > 0) {
                    if (cn > 0 && cb0 != int(bx) && cb1 < 0 && !big) {  // second box of the item
                        cb1 = int(bx);
                        csplit = cn;
                    } else if (cn > 0 && cb0 != int(bx) && cb1 != int(bx)) {
                        flush();
                    }
                    if (cn == 0) {
                        cs0 = s;
                        cb0 = int(bx);
                    }
                    const int take = std::min(G - cn, S);
                    cn += take;
                    s += take;
                    S -= take;
                    if (cn == G || big) flush();
                }
            }
            flush();
            b.litem_seg0.upload(i_s0);
            b.litem_nseg.upload(i_n);
            b.litem_split.upload(i_split);
            b.litem_box0.upload(i_b0);
            b.litem_box1.upload(i_b1);
            L.litem_seg0 = b.litem_seg0.as<std::int32_t>();
            L.litem_nseg = b.litem_nseg.as<std::int32_t>();
            L.litem_split = b.litem_split.as<std::int32_t>();
            L.litem_box0 = b.litem_box0.as<std::int32_t>();
            L.litem_box1 = b.litem_box1.as<std::int32_t>();
            L.n_litem = int(i_s0.size());
        }
        b.cx.upload(cx);
        b.cy.upload(cy);
        b.cz.upload(cz);
        b.beg.upload(B.begin);
        b.end.upload(B.end);
        b.cz_ptr.upload(CL.cz.ptr);  // the plan's cousin lists (pruned in a per-rank plan)
        b.cz_idx.upload(CL.cz.idx);
        b.cev_begin.upload(CL.cev_begin);
        b.cev_seg.upload(CL.cev_seg);
        b.seg_box.upload(CL.seg_box);
        b.seg_gamma.upload(CL.seg_gamma);
        if (CL.ns <= 256 && CL.nc <= 2048 && 2 * CL.nc <= 8192) {  // packed cells (no device division)
            std::vector<std::uint32_t> code(CL.seg_gamma.size());
            for (std::size_t i = 0; i < code.size(); ++i) {
                const int g = CL.seg_gamma[i];
                const int g1 = g % CL.ns, rest = g / CL.ns, g2 = rest % CL.nc, g3 = rest / CL.nc;
                code[i] = std::uint32_t(g1) | (std::uint32_t(g2) << 8) | (std::uint32_t(g3) << 19);
            }
            b.seg_code.upload(code);
            L.seg_code = b.seg_code.as<std::uint32_t>();
        }
        b.box_seg_begin.upload(CL.box_seg_begin);
        b.pev_begin.upload(CL.pev_begin);
        // per-evaluation child ordinals are only read by the generic-order parent kernel;
        // the tensor-core kernel (ps = 3, pang = 5) works from the grouped permutation
        if (!(CL.ps == 3 && CL.pang == 5)) b.pev_seg.upload(CL.pev_seg);
        b.pev_perm.upload(CL.pev_perm);
        b.pgrp_begin.upload(CL.pgrp_begin);
        b.pgrp_seg.upload(CL.pgrp_seg);
        b.pgrp_start.upload(CL.pgrp_start);
        b.pgrp_count.upload(CL.pgrp_count);
        b.ch_ptr.upload(C.child_ptr[d - 1]);
        b.ch_idx.upload(C.child_idx[d - 1]);
        b.s_nodes.upload(CL.s_nodes);
        b.th_nodes.upload(CL.th_nodes);
        b.ph_nodes.upload(CL.ph_nodes);
        {
            std::vector<double> ts(CL.th_nodes.size()), tc(CL.th_nodes.size()), ps_(CL.ph_nodes.size()), pc_(CL.ph_nodes.size());
            for (std::size_t i = 0; i < ts.size(); ++i) { ts[i] = std::sin(CL.th_nodes[i]); tc[i] = std::cos(CL.th_nodes[i]); }
            for (std::size_t i = 0; i < ps_.size(); ++i) { ps_[i] = std::sin(CL.ph_nodes[i]); pc_[i] = std::cos(CL.ph_nodes[i]); }
            b.th_sin.upload(ts);
            b.th_cos.upload(tc);
            b.ph_sin.upload(ps_);
            b.ph_cos.upload(pc_);
            if (CL.nc >= 4) {  // cell centres for the acos/atan2-free local coordinates
                std::vector<double> a(CL.nc), bb(CL.nc), c(2 * CL.nc), d(2 * CL.nc);
                for (int g = 0; g < CL.nc; ++g) {
                    a[g] = std::cos((g + 0.5) * CL.dth);
                    bb[g] = std::sin((g + 0.5) * CL.dth);
                }
                for (int g = 0; g < 2 * CL.nc; ++g) {
                    c[g] = std::cos((g + 0.5) * CL.dph);
                    d[g] = std::sin((g + 0.5) * CL.dph);
                }
                b.thc_cos.upload(a);
                b.thc_sin.upload(bb);
                b.phc_cos.upload(c);
                b.phc_sin.upload(d);
            }
        }
        b.chunk_box.upload(chunk_box);
        b.chunk_q0.upload(chunk_q0);
        L.d = d;
        L.nb = int(nb);
        L.nseg = int(CL.nseg());
        L.ns = CL.ns;
        L.nc = CL.nc;
        L.ps = CL.ps;
        L.pang = CL.pang;
        L.ds = CL.ds;
        L.dth = CL.dth;
        L.dph = CL.dph;
        L.inv_ds = 1.0 / CL.ds;
        L.inv_dth = 1.0 / CL.dth;
        L.inv_dph = 1.0 / CL.dph;
        L.h = T.half_diag(d);
        L.cx = b.cx.as<double>();
        L.cy = b.cy.as<double>();
        L.cz = b.cz.as<double>();
        L.beg = b.beg.as<std::uint32_t>();
        L.end = b.end.as<std::uint32_t>();
        L.cz_ptr = b.cz_ptr.as<std::int32_t>();
        L.cz_idx = b.cz_idx.as<std::int32_t>();
        L.cev_begin = b.cev_begin.as<std::int64_t>();
        L.cev_seg = b.cev_seg.as<std::int32_t>();
        L.seg_box = b.seg_box.as<std::int32_t>();
        L.seg_gamma = b.seg_gamma.as<std::int32_t>();
        L.box_seg_begin = b.box_seg_begin.as<std::int32_t>();
        L.pev_begin = b.pev_begin.as<std::int64_t>();
        L.pev_seg = b.pev_seg.as<std::int32_t>();
        L.pev_perm = b.pev_perm.as<std::uint16_t>();
        L.pgrp_begin = b.pgrp_begin.as<std::int32_t>();
        L.pgrp_seg = b.pgrp_seg.as<std::int32_t>();
        L.pgrp_start = b.pgrp_start.as<std::uint16_t>();
        L.pgrp_count = b.pgrp_count.as<std::uint16_t>();
        L.ch_ptr = b.ch_ptr.as<std::int32_t>();
        L.ch_idx = b.ch_idx.as<std::int32_t>();
        L.s_nodes = b.s_nodes.as<double>();
        L.th_nodes = b.th_nodes.as<double>();
        L.ph_nodes = b.ph_nodes.as<double>();
        L.th_sin = b.th_sin.as<double>();
        L.th_cos = b.th_cos.as<double>();
        L.ph_sin = b.ph_sin.as<double>();
        L.ph_cos = b.ph_cos.as<double>();
        L.thc_cos = CL.nc >= 4 ? b.thc_cos.as<double>() : nullptr;
        L.thc_sin = CL.nc >= 4 ? b.thc_sin.as<double>() : nullptr;
        L.phc_cos = CL.nc >= 4 ? b.phc_cos.as<double>() : nullptr;
        L.phc_sin = CL.nc >= 4 ? b.phc_sin.as<double>() : nullptr;
        L.chunk_box = b.chunk_box.as<std::int32_t>();
        L.chunk_q0 = b.chunk_q0.as<std::int32_t>();
        L.nchunk = int(chunk_box.size());
        L.max_pts = max_pts;
        store = std::max(store, CL.nseg() * std::size_t(CL.nodes_per_seg()) * 3);
    }
    (void)store;
    e.ensure_stores(true, true, e.strategy);
    e.Ms.upload(cheb::transform(e.ps));
    e.Ma.upload(cheb::transform(e.pang));

    phase_mark("templates");
    // ---- parent-fill geometry templates on every level whose table is at most 8 GiB and has
    // no more entries than the level has evaluations (measured: templates on every level beat
    // building them only where each entry serves >= 8 evaluations, cfg2 8.97 -> 8.69 ms,
    // cfg3 271 -> 260 ms of parent fill); IFGF_PARENT_TEMPLATES=0 turns them off, =force
    // builds them on every level (tests)
    std::vector<std::vector<std::int32_t>> tmpl_slot_h(T.depth + 1), tmpl_gc_h(T.depth + 1);
    {
        const char* env = std::getenv("IFGF_PARENT_TEMPLATES");
        const bool enabled = !(env && std::string(env) == "0");
        const bool force = env && std::string(env) == "force";
        for (int d = 4; enabled && d <= T.depth; ++d) {
            const ConeLevel& PL = C.level[d - 2];
            const ConeLevel& CL = C.level[d - 1];
            if (PL.ps != 3 || PL.pang != 5 || CL.ps != 3 || CL.pang != 5) continue;
            std::vector<std::int32_t> slot(PL.segs_per_box(), -1), gammas;
            for (std::int32_t g : PL.seg_gamma)
                if (slot[g] < 0) {
                    slot[g] = std::int32_t(gammas.size());
                    gammas.push_back(g);
                }
            const std::size_t entries = gammas.size() * 8 * std::size_t(PL.nodes_per_seg());
            if (std::getenv("IFGF_SETUP_DEBUG"))
                std::fprintf(stderr, "templates level %d: entries %zu evaluations %zu (%.2f GB)\n", d, entries,
                             CL.pev_perm.size(), entries * 8 * kTmplDoubles / 1e9);
            if (!force && (entries > CL.pev_perm.size() || entries * 8 * kTmplDoubles > (std::size_t(8) << 30))) continue;
            uninit_vector<double> tab;
            std::vector<std::int32_t> gc;
            parent_templates(T, C, d, gammas, 0, tab, gc);
            LevelBufs& b = e.lb[d - 2];
            b.tmpl_slot.upload(slot);
            b.tmpl.upload(tab);
            LevelDev& L = e.L[d - 2];
            L.tmpl_slot = b.tmpl_slot.as<std::int32_t>();
            L.tmpl = b.tmpl.as<double>();
            tmpl_slot_h[d] = std::move(slot);
            tmpl_gc_h[d] = std::move(gc);
        }
    }

    phase_mark("cell-batched items");
    // ---- cell-batched parent items (parent_cb.cu): on levels with templates whose parent cone
    // cells are each shared by >= min_avg parent segments on average (default 400: cfg3's two
    // finest parent levels), the segments of one cell are batched (kCbSegs per CTA, sorted by
    // child-octant pattern) into GEMMs against their children's blocks; the per-segment kernel
    // below takes the remaining segments. IFGF_PARENT_CB=0 disables, =force batches every
    // template level, IFGF_PARENT_CB_MINAVG sets the threshold. cfg3: parent 251 -> 231 ms;
    // on levels with fewer segments per cell the per-segment kernel is faster (cfg2 level 5,
    // 396 per cell: break-even; level 4, 45 per cell: 30% slower).
    std::vector<std::vector<std::uint8_t>> cb_seg_h(T.depth + 1);
    {
        const char* env = std::getenv("IFGF_PARENT_CB");
        const bool enabled = !(env && env[0] == '0');
        const bool force = env && std::string(env) == "force";
        const bool dbg = std::getenv("IFGF_SETUP_DEBUG") != nullptr;
        // tests: also route every n-th evaluation through the exception path (same segment)
        const char* xenv = std::getenv("IFGF_PARENT_CB_EXC_EVERY");
        const int exc_every = xenv ? std::max(0, std::atoi(xenv)) : 0;
        // levels batch when their template cells hold >= min_avg segments on average
        const char* menv = std::getenv("IFGF_PARENT_CB_MINAVG");
        const std::size_t min_avg = menv ? std::size_t(std::max(1, std::atoi(menv))) : 400;
        for (int d = 4; enabled && d <= T.depth; ++d) {
            const std::vector<std::int32_t>& slot = tmpl_slot_h[d];
            const std::vector<std::int32_t>& gcs = tmpl_gc_h[d];
            if (slot.empty() || gcs.empty()) continue;
            const ConeLevel& PL = C.level[d - 2];
            const ConeLevel& CL = C.level[d - 1];
            constexpr int P = 75;
            const int nslot = int(gcs.size() / (8 * P));
            // per (slot, octant): nodes in child-cell order, group starts and cells
            std::vector<std::uint8_t> nodes(std::size_t(nslot) * 8 * P), gstart(std::size_t(nslot) * 8 * (kCbMaxGrp + 1), P),
                ngrp(std::size_t(nslot) * 8, 0), bad(nslot, 0), gpos(std::size_t(nslot) * 8 * P);
            std::vector<std::int32_t> ggc(std::size_t(nslot) * 8 * kCbMaxGrp, -1);
#pragma omp parallel for schedule(static)
            for (int sl = 0; sl < nslot; ++sl)
                for (int o = 0; o < 8; ++o) {
                    const std::size_t so8 = std::size_t(sl) * 8 + o;
                    std::array<std::pair<int, int>, P> v;
                    for (int nd = 0; nd < P; ++nd) v[nd] = {gcs[so8 * P + nd], nd};
                    std::stable_sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
                    int ng = 0;
                    for (int i = 0; i < P; ++i) {
                        if (i == 0 || v[i].first != v[i - 1].first) {
                            if (ng == kCbMaxGrp) {
                                bad[sl] = 1;
                                break;
                            }
                            gstart[so8 * (kCbMaxGrp + 1) + ng] = std::uint8_t(i);
                            ggc[so8 * kCbMaxGrp + ng] = v[i].first;
                            ++ng;
                        }
                        nodes[so8 * P + i] = std::uint8_t(v[i].second);
                        gpos[so8 * P + v[i].second] = std::uint8_t(ng - 1);  // group of node
                    }
                    ngrp[so8] = std::uint8_t(ng);
                    gstart[so8 * (kCbMaxGrp + 1) + ng] = P;
                }
            const auto& cptr = C.child_ptr[d - 2];
            const auto& cidx = C.child_idx[d - 2];
            // child-octant pattern of each parent box: an item's warps take 4 segments each, so
            // segments with the same pattern are kept together (no idle GEMM columns)
            std::vector<std::uint8_t> omask(PL.box_seg_begin.size() - 1, 0);
#pragma omp parallel for schedule(static)
            for (std::int64_t pb = 0; pb < std::int64_t(omask.size()); ++pb) {
                const Vec3 pc = T.center(d - 1, std::size_t(pb));
                std::uint8_t m = 0;
                for (int c = cptr[pb]; c < cptr[pb + 1]; ++c) {
                    const Vec3 cc = T.center(d, std::size_t(cidx[c]));
                    m |= std::uint8_t(1u << ((cc.x > pc.x ? 1 : 0) | (cc.y > pc.y ? 2 : 0) | (cc.z > pc.z ? 4 : 0)));
                }
                omask[pb] = m;
            }
            std::vector<std::vector<std::int32_t>> by_slot(nslot);
            for (std::size_t so = 0; so < PL.nseg(); ++so) {
                const int sl = slot[PL.seg_gamma[so]];
                if (sl >= 0 && !bad[sl]) by_slot[sl].push_back(std::int32_t(so));
            }
#pragma omp parallel for schedule(dynamic, 64)
            for (int sl = 0; sl < nslot; ++sl)
                std::stable_sort(by_slot[sl].begin(), by_slot[sl].end(), [&](std::int32_t a, std::int32_t b) {
                    return omask[PL.seg_box[a]] < omask[PL.seg_box[b]];
                });
            std::size_t cnt = 0, used = 0;
            for (const auto& v : by_slot) {
                cnt += v.size();
                used += v.empty() ? 0 : 1;
            }
            if (!force && cnt < min_avg * used) continue;  // cells too rarely shared at this level
            std::vector<std::int32_t> item_slot, item_seg;
            for (int sl = 0; sl < nslot; ++sl)
                for (std::size_t a = 0; a < by_slot[sl].size(); a += kCbSegs) {
                    item_slot.push_back(sl);
                    for (int j = 0; j < kCbSegs; ++j)
                        item_seg.push_back(a + j < by_slot[sl].size() ? by_slot[sl][a + j] : -1);
                }
            const std::int64_t n_item = std::int64_t(item_slot.size());
            std::vector<std::int32_t> child(std::size_t(n_item) * kCbSegs * 8, -1);
            std::vector<std::vector<std::pair<std::uint32_t, std::int32_t>>> exc(n_item);
            // unit lists (parent_cb.cu): per (item, warp of 4 segments), per octant with a child
            // and per child-cell group met by one of the 4, the rows [gs, ge) in at most
            // max_tiles 8-row tiles per unit (a larger group: two units) and the 4 child segments
            constexpr int kW = kCbSegs / 4;
            const int max_tiles = e.pipes_at(d, true, true, e.strategy).size() == 3 ? kCbMaxTiles3 : kCbMaxTiles;
            std::vector<std::vector<std::int32_t>> ulist(static_cast<std::size_t>(n_item) * kW);
            int too_long = 0;
            auto ordinal = [&](int ch, int gam) {
                const auto b0 = CL.seg_gamma.begin() + CL.box_seg_begin[ch];
                const auto b1 = CL.seg_gamma.begin() + CL.box_seg_begin[ch + 1];
                const auto it = std::lower_bound(b0, b1, gam);
                return (it == b1 || *it != gam) ? -1 : std::int32_t(it - CL.seg_gamma.begin());
            };
#pragma omp parallel for schedule(dynamic, 256)
            for (std::int64_t it = 0; it < n_item; ++it) {
                const int sl = item_slot[it];
                // child segment of (item segment, octant, child-cell group), -1: none
                std::int32_t cso[kCbSegs][8][kCbMaxGrp];
                std::fill(&cso[0][0][0], &cso[0][0][0] + kCbSegs * 8 * kCbMaxGrp, -1);
                for (int j = 0; j < kCbSegs; ++j) {
                    const int so = item_seg[it * kCbSegs + j];
                    if (so < 0) continue;
                    const int pb = PL.seg_box[so];
                    const int nch = cptr[pb + 1] - cptr[pb];
                    const Vec3 pc = T.center(d - 1, std::size_t(pb));
                    for (int c = 0; c < nch; ++c) {
                        const int ch = cidx[cptr[pb] + c];
                        const Vec3 cc = T.center(d, std::size_t(ch));
                        const int o = (cc.x > pc.x ? 1 : 0) | (cc.y > pc.y ? 2 : 0) | (cc.z > pc.z ? 4 : 0);
                        const std::size_t so8 = std::size_t(sl) * 8 + o;
                        child[(std::size_t(it) * kCbSegs + j) * 8 + o] = ch;
                        std::int32_t* cg = cso[j][o];
                        for (int g = 0; g < ngrp[so8]; ++g) cg[g] = ordinal(ch, ggc[so8 * kCbMaxGrp + g]);
                        for (int nd = 0; nd < P; ++nd) {
                            const std::int32_t host = CL.pev_seg[CL.pev_begin[so] + std::int64_t(nd) * nch + c];
                            if (host != cg[gpos[so8 * P + nd]] || (exc_every > 0 && (nd + j + o) % exc_every == 0))
                                exc[it].push_back({std::uint32_t(j) | (std::uint32_t(o) << 8) | (std::uint32_t(nd) << 16), host});
                        }
                    }
                }
                for (int w = 0; w < kW; ++w) {
                    std::vector<std::int32_t>& U = ulist[std::size_t(it) * kW + w];
                    for (int o = 0; o < 8; ++o) {
                        const std::size_t so8 = std::size_t(sl) * 8 + o;
                        for (int g = 0; g < ngrp[so8]; ++g) {
                            std::int32_t c4[4];
                            bool any = false;
                            for (int c = 0; c < 4; ++c) {
                                c4[c] = cso[4 * w + c][o][g];  // -1 without a child in this octant
                                any = any || c4[c] >= 0;
                            }
                            if (!any) continue;
                            const int gs = gstart[so8 * (kCbMaxGrp + 1) + g], ge = gstart[so8 * (kCbMaxGrp + 1) + g + 1];
                            const int mt = (ge - gs + 7) >> 3;
                            const int nh = mt > max_tiles ? 2 : 1;
                            for (int h = 0; h < nh; ++h) {
                                const int t0 = h == 0 ? 0 : (mt + 1) / 2, t1 = nh == 1 ? mt : (h == 0 ? (mt + 1) / 2 : mt);
                                U.push_back((gs + 8 * t0) | ((t1 - t0) << 8) | (ge << 16) | (o << 24));
                                U.insert(U.end(), c4, c4 + 4);
                            }
                        }
                    }
                    if (U.size() > std::size_t(kCbMaxUnits) * 5) {
#pragma omp atomic write
                        too_long = 1;
                    }
                }
            }
            if (too_long) throw std::logic_error("cell-batched unit list too long");
            std::vector<std::int32_t> unit_begin(ulist.size() + 1, 0);
            for (std::size_t i = 0; i < ulist.size(); ++i) {
                const std::size_t nxt = std::size_t(unit_begin[i]) + ulist[i].size() / 5;
                if (nxt > std::size_t(std::numeric_limits<std::int32_t>::max())) throw std::logic_error("cell-batched unit count overflow");
                unit_begin[i + 1] = std::int32_t(nxt);
            }
            std::vector<std::int32_t> unit(std::size_t(unit_begin.back()) * 5);
#pragma omp parallel for schedule(static)
            for (std::int64_t i = 0; i < std::int64_t(ulist.size()); ++i)
                std::copy(ulist[i].begin(), ulist[i].end(), unit.begin() + std::size_t(unit_begin[i]) * 5);
            ulist.clear();
            ulist.shrink_to_fit();
            std::vector<std::int64_t> exc_begin(n_item + 1, 0);
            for (std::int64_t it = 0; it < n_item; ++it) exc_begin[it + 1] = exc_begin[it] + std::int64_t(exc[it].size());
            std::vector<std::uint32_t> exc_key(static_cast<std::size_t>(exc_begin[n_item]));
            std::vector<std::int32_t> exc_cso(exc_key.size());
            for (std::int64_t it = 0; it < n_item; ++it)
                for (std::size_t x = 0; x < exc[it].size(); ++x) {
                    exc_key[std::size_t(exc_begin[it]) + x] = exc[it][x].first;
                    exc_cso[std::size_t(exc_begin[it]) + x] = exc[it][x].second;
                }
            std::vector<std::uint8_t>& done = cb_seg_h[d];
            done.assign(PL.nseg(), 0);
            for (std::int32_t so : item_seg)
                if (so >= 0) done[so] = 1;
            if (dbg) {
                double sg = 0, st = 0, nso = 0;
                for (int sl = 0; sl < nslot; ++sl)
                    for (int o = 0; o < 8; ++o) {
                        const std::size_t so8 = std::size_t(sl) * 8 + o;
                        if (by_slot[sl].empty()) continue;
                        nso += 1;
                        sg += ngrp[so8];
                        for (int g = 0; g < ngrp[so8]; ++g)
                            st += (gstart[so8 * (kCbMaxGrp + 1) + g + 1] - gstart[so8 * (kCbMaxGrp + 1) + g] + 7) / 8;
                    }
                std::fprintf(stderr, "cell-batched parent level %d: %zu of %zu segments in %lld items, %zu cells, %zu exceptions; "
                             "per (cell, octant): %.2f child cells, %.2f 8-row tiles\n",
                             d - 1, cnt, PL.nseg(), (long long)n_item, used, exc_key.size(), sg / std::max(1.0, nso), st / std::max(1.0, nso));
            }
            LevelBufs& b = e.lb[d - 1];
            b.cb_item_slot.upload(item_slot);
            b.cb_item_seg.upload(item_seg);
            b.cb_nodes.upload(nodes);
            b.cb_child.upload(child);
            b.cb_unit_begin.upload(unit_begin);
            b.cb_unit.upload(unit);
            b.cb_exc_begin.upload(exc_begin);
            b.cb_exc_key.upload(exc_key);
            b.cb_exc_cso.upload(exc_cso);
            LevelDev& L = e.L[d - 1];
            L.n_cbitem = int(n_item);
            L.cb_item_slot = b.cb_item_slot.as<std::int32_t>();
            L.cb_item_seg = b.cb_item_seg.as<std::int32_t>();
            L.cb_nodes = b.cb_nodes.as<std::uint8_t>();
            L.cb_child = b.cb_child.as<std::int32_t>();
            L.cb_unit_begin = b.cb_unit_begin.as<std::int32_t>();
            L.cb_unit = b.cb_unit.as<std::int32_t>();
            L.cb_exc_begin = b.cb_exc_begin.as<std::int64_t>();
            L.cb_exc_key = b.cb_exc_key.as<std::uint32_t>();
            L.cb_exc_cso = b.cb_exc_cso.as<std::int32_t>();
            // (slot, octant) tables from the level's geometry templates (device-side)
            b.cb_tab.alloc(std::size_t(nslot) * 8 * kCbTab * sizeof(double));
            IFGF_CUDA(cudaDeviceSynchronize());  // the template and node uploads are in flight
            launch_cb_tables(e.L[d - 2].tmpl, L.cb_nodes, nslot, b.cb_tab.as<double>(), 0);
            L.cb_tab = b.cb_tab.as<double>();
        }
    }

    phase_mark("parent items");
    // ---- parent work items (tensor-core parent kernel): up to `merge` relevant segments of one
    // parent box per warp (IFGF_PARENT_MERGE, default 2), with their child-segment groups merged
    // so that evaluations of the item's segments that land in the same child segment share
    // DMMA tiles. One 16-byte record per merged group {child segment, child box, start |
    // count << 16 | child octant << 24, packed cell} and per evaluation its node | child slot
    // << 8 | item-local segment << 11 | template bit << 15, so the kernel's loads do not chain
    // through pev_perm -> ch_idx / seg_gamma -> cell tables -> template cells. Within a merged
    // group the evaluations keep their segments' group order, so every node accumulator sees
    // the same additions in the same order as with one segment per warp.
    {
        const char* menv = std::getenv("IFGF_PARENT_MERGE");
        const int merge = std::clamp(menv ? std::atoi(menv) : 2, 1, kParentMergeMax);
        for (int d = 4; d <= T.depth; ++d) {
            const ConeLevel& PL = C.level[d - 2];
            const ConeLevel& CL = C.level[d - 1];
            if (PL.ps != 3 || PL.pang != 5 || CL.ps != 3 || CL.pang != 5 || CL.pgrp_begin.empty()) continue;
            const auto& cptr = C.child_ptr[d - 2];
            const auto& cidx = C.child_idx[d - 2];
            const std::vector<std::int32_t>& slot = tmpl_slot_h[d];
            const std::vector<std::int32_t>& gc = tmpl_gc_h[d];
            const bool packed = e.L[d - 1].seg_code != nullptr;
            auto cell_of = [&](int gam, const ConeLevel& L) {
                if (!packed) return gam;
                const int g1 = gam % L.ns, rest = gam / L.ns;
                return int(std::uint32_t(g1) | (std::uint32_t(rest % L.nc) << 8) | (std::uint32_t(rest / L.nc) << 19));
            };
            // items: consecutive relevant segments of one parent box (those not cell-batched)
            const std::vector<std::uint8_t>& cbd = cb_seg_h[d];
            std::vector<std::int32_t> item_seg, rest;
            for (std::size_t pb = 0; pb + 1 < PL.box_seg_begin.size(); ++pb) {
                rest.clear();
                for (int s = PL.box_seg_begin[pb]; s < PL.box_seg_begin[pb + 1]; ++s)
                    if (cbd.empty() || !cbd[s]) rest.push_back(s);
                for (std::size_t s0 = 0; s0 < rest.size(); s0 += merge)
                    for (int w = 0; w < kParentMergeMax; ++w)
                        item_seg.push_back(w < merge && s0 + w < rest.size() ? rest[s0 + w] : -1);
            }
            const std::int64_t n_item = std::int64_t(item_seg.size()) / kParentMergeMax;
            // an item's groups: (child segment, item-local segment, group), ordered by child
            // segment, then segment (stable)
            auto item_groups = [&](std::int64_t it, std::vector<std::array<int, 3>>& v) {
                v.clear();
                for (int w = 0; w < kParentMergeMax; ++w) {
                    const int so = item_seg[it * kParentMergeMax + w];
                    if (so < 0) continue;
                    for (int g = CL.pgrp_begin[so]; g < CL.pgrp_begin[so + 1]; ++g) v.push_back({CL.pgrp_seg[g], w, g});
                }
                std::stable_sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a[0] < b[0]; });
            };
            std::vector<std::int64_t> ig(n_item + 1, 0), ie(n_item + 1, 0);
#pragma omp parallel
            {
                std::vector<std::array<int, 3>> v;
#pragma omp for schedule(dynamic, 256)
                for (std::int64_t it = 0; it < n_item; ++it) {
                    item_groups(it, v);
                    std::int64_t ng = 0, nev = 0;
                    for (std::size_t x = 0; x < v.size(); ++x) {
                        if (x == 0 || v[x][0] != v[x - 1][0]) ++ng;
                        nev += CL.pgrp_count[v[x][2]];
                    }
                    ig[it + 1] = ng;
                    ie[it + 1] = nev;
                }
            }
            for (std::int64_t it = 0; it < n_item; ++it) {
                ig[it + 1] += ig[it];
                ie[it + 1] += ie[it];
            }
            uninit_vector<int4> rec(static_cast<std::size_t>(ig[n_item]));  // every entry written below
            uninit_vector<std::uint16_t> perm(static_cast<std::size_t>(ie[n_item]));
            std::atomic<bool> too_big{false};
#pragma omp parallel
            {
                std::vector<std::array<int, 3>> v;
#pragma omp for schedule(dynamic, 256)
                for (std::int64_t it = 0; it < n_item; ++it) {
                    item_groups(it, v);
                    const int pb = PL.seg_box[item_seg[it * kParentMergeMax]];
                    const Vec3 pc = T.center(d - 1, std::size_t(pb));
                    std::int64_t gi = ig[it];
                    int at = 0;  // item-local evaluation index
                    for (std::size_t x = 0; x < v.size();) {
                        const int cso = v[x][0];
                        const int start = at;
                        const int c = (CL.pev_perm[CL.pev_begin[item_seg[it * kParentMergeMax + v[x][1]]] +
                                                   CL.pgrp_start[v[x][2]]] >> 8) & 7;
                        const int ch = cidx[cptr[pb] + c];
                        const int cgam = CL.seg_gamma[cso];
                        const Vec3 cc = T.center(d, std::size_t(ch));
                        const int oct = (cc.x > pc.x ? 1 : 0) | (cc.y > pc.y ? 2 : 0) | (cc.z > pc.z ? 4 : 0);
                        for (; x < v.size() && v[x][0] == cso; ++x) {
                            const int w = v[x][1], g = v[x][2];
                            const int so = item_seg[it * kParentMergeMax + w];
                            const std::int64_t ev0 = CL.pev_begin[so];
                            const int tslot = slot.empty() ? -1 : slot[PL.seg_gamma[so]];
                            const std::size_t tbase = (std::size_t(std::max(tslot, 0)) * 8 + oct) * 75;
                            for (int i = CL.pgrp_start[g]; i < CL.pgrp_start[g] + CL.pgrp_count[g]; ++i) {
                                std::uint16_t ent = std::uint16_t((CL.pev_perm[ev0 + i] & 0x7ffu) | (w << 11));  // w < 2
                                if (tslot >= 0 && gc[tbase + (ent & 0xff)] == cgam) ent = std::uint16_t(ent | 0x8000u);
                                perm[std::size_t(ie[it] + at++)] = ent;
                            }
                        }
                        const int count = at - start;
                        if (count > 255 || at > 65535) too_big = true;
                        rec[std::size_t(gi++)] = make_int4(cso, ch, start | (count << 16) | (oct << 24), cell_of(cgam, CL));
                    }
                }
            }
            if (too_big) throw InternalError("parent items: more than 255 evaluations in one merged group");
            // bounds the kernel relies on (no device-side checks)
            for (std::int64_t it = 0; it < n_item; ++it)
                for (std::int64_t g = ig[it]; g < ig[it + 1]; ++g) {
                    const int4 r4 = rec[std::size_t(g)];
                    const int st0 = r4.z & 0xffff, cnt = (r4.z >> 16) & 0xff;
                    if (r4.x < 0 || std::size_t(r4.x) >= CL.nseg() || r4.y < 0 ||
                        std::size_t(r4.y) >= T.level[d - 1].size() || cnt < 1 || ie[it] + st0 + cnt > ie[it + 1])
                        throw InternalError("parent items: inconsistent group record");
                }
            std::vector<std::int32_t> igr(ig.begin(), ig.end());
            LevelBufs& b = e.lb[d - 1];
            b.pgrp_rec.upload(rec);
            b.pev_perm.upload(perm);
            b.pitem_seg.upload(item_seg);
            b.pitem_grp.upload(igr);
            b.pitem_ev.upload(ie);
            LevelDev& L = e.L[d - 1];
            L.pgrp_rec = b.pgrp_rec.as<int4>();
            L.pev_perm = b.pev_perm.as<std::uint16_t>();
            L.pitem_seg = b.pitem_seg.as<std::int32_t>();
            L.pitem_grp = b.pitem_grp.as<std::int32_t>();
            L.pitem_ev = b.pitem_ev.as<std::int64_t>();
            L.n_pitem = int(n_item);
            L.pitem_merge = merge;
            if (ig[n_item] > std::int64_t(INT32_MAX)) throw InternalError("parent items: too many groups");
        }
    }

    phase_mark("near field");
    // ---- near field
    {
        const int D = T.depth;
        const BoxLevel& B = T.level[D - 1];
        std::vector<std::int32_t> chunk_box, chunk_q0;
        for (std::size_t i = 0; i < B.size(); ++i)
            for (std::uint32_t q = 0; q < B.end[i] - B.begin[i]; q += kChunk) {
                chunk_box.push_back(std::int32_t(i));
                chunk_q0.push_back(std::int32_t(q));
            }
        std::vector<std::uint32_t> fpos(PL.far_nodes.size());
        std::vector<std::uint32_t> inv(n);
        for (std::size_t t = 0; t < n; ++t) inv[T.perm[t]] = std::uint32_t(t);
        for (std::size_t i = 0; i < fpos.size(); ++i) fpos[i] = inv[PL.far_nodes[i]];
        if (D < 3) {
            // leaf-level spans still needed for the near field
            e.lb[D - 1].beg.upload(B.begin);
            e.lb[D - 1].end.upload(B.end);
        }
        {
            std::vector<std::int32_t> lom(n, 0);
            for (std::size_t b = 0; b < B.size(); ++b)
                for (std::uint32_t t = B.begin[b]; t < B.end[b]; ++t) lom[t] = std::int32_t(b);
            e.leaf_of_m.upload(lom);
        }
        e.nb_ptr.upload(R.nbr[D - 1].ptr);
        e.nb_idx.upload(R.nbr[D - 1].idx);
        e.tpb.upload(PL.target_pair_begin);
        e.pair_patch.upload(PL.patch);
        e.far_begin.upload(PL.far_begin);
        e.far_end.upload(PL.far_end);
        e.far_pos.upload(fpos);
        e.near_chunk_box.upload(chunk_box);
        e.near_chunk_q0.upload(chunk_q0);
        {
            // target pairs of every leaf (near pair lists): (b, b + 1), (b + 2, b + 3), ...,
            // an odd leaf's last target alone (bit 31)
            std::vector<std::int32_t> pit;
            pit.reserve(n / 2 + B.size());
            for (std::size_t b = 0; b < B.size(); ++b)
                for (std::uint32_t t = B.begin[b]; t < B.end[b]; t += 2)
                    pit.push_back(std::int32_t(t | (t + 1 < B.end[b] ? 0u : 0x80000000u)));
            e.near_pitem.upload(pit);
            e.near.npitem = int(pit.size());
        }
        // patch runs of every leaf's neighbourhood (near_run_kernel: used when the near lists
        // do not fit, or with IFGF_NEAR=runs; cfg2 2.77 vs 2.45 ms with lists, cfg3 45 vs
        // 40 ms, 61 ms screening every apply)
        const char* nenv = std::getenv("IFGF_NEAR");
        if (!nenv || std::string(nenv) == "runs") {
            std::vector<std::int32_t> rptr(B.size() + 1, 0), rst, rln, rpa;
            for (std::size_t b = 0; b < B.size(); ++b) {
                rptr[b] = std::int32_t(rst.size());
                for (int j = R.nbr[D - 1].ptr[b]; j < R.nbr[D - 1].ptr[b + 1]; ++j) {
                    const int nb = R.nbr[D - 1].idx[j];
                    for (std::uint32_t u = B.begin[nb]; u < B.end[nb];) {
                        const std::int32_t pq = S.patch_of[T.perm[u]];
                        std::uint32_t v = u + 1;
                        while (v < B.end[nb] && S.patch_of[T.perm[v]] == pq) ++v;
                        rst.push_back(std::int32_t(u));
                        rln.push_back(std::int32_t(v - u));
                        rpa.push_back(pq);
                        u = v;
                    }
                }
            }
            rptr[B.size()] = std::int32_t(rst.size());
            e.run_ptr.upload(rptr);
            e.run_start.upload(rst);
            e.run_len.upload(rln);
            e.run_patch.upload(rpa);
            if (std::getenv("IFGF_SETUP_DEBUG"))
                std::fprintf(stderr, "near runs: %zu over %zu leaves (%.1f per neighbourhood)\n", rst.size(), B.size(),
                             double(rst.size()) / double(std::max<std::size_t>(B.size(), 1)));
        }
        NearDev& N = e.near;
        N.n = int(n);
        N.nleaf = int(B.size());
        N.perm = e.perm.as<std::uint32_t>();
        N.beg = e.lb[D - 1].beg.as<std::uint32_t>();
        N.end = e.lb[D - 1].end.as<std::uint32_t>();
        N.nb_ptr = e.nb_ptr.as<std::int32_t>();
        N.nb_idx = e.nb_idx.as<std::int32_t>();
        N.patch_p = e.patch_p.as<std::int32_t>();
        N.leaf_of_m = e.leaf_of_m.as<std::int32_t>();
        N.geo = e.pgeo.as<double2>();
        N.tpb = e.tpb.as<std::uint32_t>();
        N.pair_patch = e.pair_patch.as<std::int32_t>();
        N.far_begin = e.far_begin.as<std::uint32_t>();
        N.far_end = e.far_end.as<std::uint32_t>();
        N.far_pos = e.far_pos.as<std::uint32_t>();
        N.chunk_box = e.near_chunk_box.as<std::int32_t>();
        N.run_ptr = e.run_ptr.as<std::int32_t>();
        N.run_start = e.run_start.as<std::int32_t>();
        N.run_len = e.run_len.as<std::int32_t>();
        N.run_patch = e.run_patch.as<std::int32_t>();
        N.chunk_q0 = e.near_chunk_q0.as<std::int32_t>();
        N.pitem = e.near_pitem.as<std::int32_t>();
        N.nchunk = int(chunk_box.size());
    }

    phase_mark("rp");
    // ---- RP: patch transforms, pair lists; beta offsets
    {
        const std::size_t nq = S.patches.size();
        std::vector<std::int32_t> nu(nq), nv(nq), du(nq), dv(nq), mat_off(2 * nq);
        std::vector<std::int64_t> start(nq + 1), soff(nq + 1);
        std::vector<double> mats, orient(nq), series, cutoff(nq);
        std::vector<std::pair<int, std::int32_t>> cache;  // n -> offset
        auto mat_for = [&](int m) {
            for (auto& c : cache)
                if (c.first == m) return c.second;
            const auto M = cheb::transform(m);
            const std::int32_t off = std::int32_t(mats.size());
            mats.insert(mats.end(), M.begin(), M.end());
            cache.push_back({m, off});
            return off;
        };
        const std::vector<double> spacing = S.spacing();
        int max_nn = 1;
        for (std::size_t q = 0; q < nq; ++q) {
            const Patch& p = S.patches[q];
            nu[q] = p.nu;
            nv[q] = p.nv;
            du[q] = p.du;
            dv[q] = p.dv;
            orient[q] = p.orient;
            start[q] = std::int64_t(S.patch_start[q]);
            mat_off[2 * q] = mat_for(p.nu);
            mat_off[2 * q + 1] = mat_for(p.nv);
            max_nn = std::max(max_nn, p.nu * p.nv);
            e.max_dudv = std::max({e.max_dudv, p.du, p.dv, p.nu, p.nv});
            e.max_dv = std::max(e.max_dv, p.dv);
            e.max_nu = std::max(e.max_nu, p.nu);
            soff[q] = std::int64_t(series.size());
            for (const auto* set : {&p.pos_c, &p.du_c, &p.dv_c})
                for (int c = 0; c < 3; ++c) series.insert(series.end(), (*set)[c].begin(), (*set)[c].end());
            cutoff[q] = std::max(1e-14, 1e-8 * spacing[q]);
        }
        start[nq] = std::int64_t(S.patch_start[nq]);
        e.max_nunv = max_nn;
        e.patch_nu.upload(nu);
        e.patch_nv.upload(nv);
        e.patch_start.upload(start);
        e.mat_off.upload(mat_off);
        e.mats.upload(mats);
        std::vector<std::uint64_t> boff(PL.size() + 1, 0);
        for (std::size_t i = 0; i < PL.size(); ++i) {
            const Patch& p = S.patches[PL.patch[i]];
            boff[i + 1] = boff[i] + std::uint64_t(p.nu) * p.nv;
        }
        e.beta_entries = boff.back();  // full tables; storage comes with compute/upload_beta
        e.beta_off_full = std::move(boff);
        e.coeffs.alloc(std::max<std::size_t>(n, 1) * sizeof(double2));
        RpDev& rp = e.rp;
        rp.n = int(n);
        rp.npatch = int(nq);
        rp.patch_nu = e.patch_nu.as<std::int32_t>();
        rp.patch_nv = e.patch_nv.as<std::int32_t>();
        rp.patch_start = e.patch_start.as<std::int64_t>();
        rp.mat_off = e.mat_off.as<std::int32_t>();
        rp.mats = e.mats.as<double>();
        rp.tpb = e.tpb.as<std::uint32_t>();
        rp.pair_patch = e.pair_patch.as<std::int32_t>();
        // rp.beta_off / beta_s / beta_d are set when the tables are allocated (alloc_beta)
        rp.pos = e.pos.as<std::uint32_t>();
        rp.max_nn = max_nn;
        // beta inputs
        e.b_target.upload(PL.target);
        e.b_ubar.upload(PL.ubar);
        e.b_vbar.upload(PL.vbar);
        e.b_du.upload(du);
        e.b_dv.upload(dv);
        e.b_orient.upload(orient);
        e.b_series_off.upload(soff);
        e.b_series.upload(series);
        e.b_cutoff.upload(cutoff);
        cheb::fejer(PL.cfg.n_beta, e.rule_x, e.rule_w);
    }

    phase_mark("work vectors");
    // ---- direct-sum view and work vectors
    e.direct = {int(n), e.ox.as<double>(), e.oy.as<double>(), e.oz.as<double>(), e.onx.as<double>(),
                e.ony.as<double>(), e.onz.as<double>(), e.ojw.as<double>(), e.opatch.as<std::int32_t>(),
                e.tpb.as<std::uint32_t>(), e.pair_patch.as<std::int32_t>()};
    const std::size_t vb = std::max<std::size_t>(n, 1) * sizeof(double2);
    for (DevBuf* b : {&e.d_phi, &e.d_out, &e.d_S, &e.d_D, &e.a_p, &e.Sp, &e.Dp, &e.Sn, &e.Dn, &e.scratch, &e.out_m})
        b->alloc(vb);
    e.own_lo = 0;
    e.own_hi = std::uint32_t(n);
    e.bounds = {0u, std::uint32_t(n)};
    phase_mark("device sync");
    IFGF_CUDA(cudaDeviceSynchronize());
    phase_mark("end");
}

Engine::~Engine() {
    if (d_) {
        cudaSetDevice(d_->dev);
        if (d_->graph) cudaGraphExecDestroy(d_->graph);
        if (d_->comm) ncclCommDestroy(d_->comm);
        if (d_->ev_fork) cudaEventDestroy(d_->ev_fork);
        if (d_->ev_join) cudaEventDestroy(d_->ev_join);
        for (auto x : d_->ev_store)
            if (x) cudaEventDestroy(x);
        for (auto x : d_->ev_cousin)
            if (x) cudaEventDestroy(x);
        if (d_->st3) cudaStreamDestroy(d_->st3);
        if (d_->st2) cudaStreamDestroy(d_->st2);
        if (d_->st) cudaStreamDestroy(d_->st);
    }
}

std::size_t Engine::size() const { return d_->n; }
int Engine::device() const { return d_->dev; }

void Engine::compute_beta() {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    IFGF_CUDA(cudaSetDevice(e.dev));
    BetaDev B;
    B.npairs = int(e.pairs->size());
    B.n_beta = e.pairs->cfg.n_beta;
    B.cov_d = e.pairs->cfg.cov_d;
    B.k = e.k;
    B.target = e.b_target.as<std::uint32_t>();
    B.patch = e.pair_patch.as<std::int32_t>();
    B.ubar = e.b_ubar.as<double>();
    B.vbar = e.b_vbar.as<double>();
    B.tx = e.ox.as<double>();
    B.ty = e.oy.as<double>();
    B.tz = e.oz.as<double>();
    B.nu = e.patch_nu.as<std::int32_t>();
    B.nv = e.patch_nv.as<std::int32_t>();
    B.du = e.b_du.as<std::int32_t>();
    B.dv = e.b_dv.as<std::int32_t>();
    B.orient = e.b_orient.as<double>();
    B.series_off = e.b_series_off.as<std::int64_t>();
    B.series = e.b_series.as<double>();
    B.cutoff = e.b_cutoff.as<double>();
    // the pairs to compute: all, or (under a partition) those whose target this engine owns
    const bool shard = e.partitioned;
    std::vector<std::uint32_t> idx;
    {
        std::vector<std::uint32_t> pos(e.n);
        for (std::size_t t = 0; t < e.n; ++t) pos[e.tree->perm[t]] = std::uint32_t(t);
        for (std::size_t p = 0; p < e.pairs->size(); ++p) {
            const std::uint32_t m = pos[e.pairs->target[p]];
            if (!shard || (m >= e.own_lo && m < e.own_hi)) idx.push_back(std::uint32_t(p));
        }
    }
    e.alloc_beta(shard ? &idx : nullptr);
    B.offset = e.beta_off.as<std::uint64_t>();
    DevBuf d_idx;
    d_idx.upload(idx);
    B.pidx = d_idx.as<std::uint32_t>();
    // graded rules on the host (glibc pow, bit-identical to the reference), in batches
    const std::size_t np = idx.size();
    const int nb = B.n_beta;
    const std::size_t batch = std::min<std::size_t>(std::max<std::size_t>(np, 1), std::size_t(1) << 17);
    std::vector<double> hu(batch * nb), hwu(batch * nb), hv(batch * nb), hwv(batch * nb);
    for (DevBuf* b : {&e.b_gu, &e.b_gwu, &e.b_gv, &e.b_gwv}) b->alloc(std::max<std::size_t>(batch * nb, 1) * sizeof(double));
    B.grid_u = e.b_gu.as<double>();
    B.grid_wu = e.b_gwu.as<double>();
    B.grid_v = e.b_gv.as<double>();
    B.grid_wv = e.b_gwv.as<double>();
    for (std::size_t p0 = 0; p0 < np; p0 += batch) {
        const std::size_t cnt = std::min(batch, np - p0);
        graded_rules(*e.pairs, idx.data() + p0, cnt, e.rule_x, e.rule_w, hu.data(), hwu.data(), hv.data(), hwv.data(),
                     0);
        IFGF_CUDA(cudaStreamSynchronize(e.st));  // previous batch done with the device buffers
        const std::size_t bytes = cnt * nb * sizeof(double);
        IFGF_CUDA(cudaMemcpyAsync(e.b_gu.as<void>(), hu.data(), bytes, cudaMemcpyHostToDevice, e.st));
        IFGF_CUDA(cudaMemcpyAsync(e.b_gwu.as<void>(), hwu.data(), bytes, cudaMemcpyHostToDevice, e.st));
        IFGF_CUDA(cudaMemcpyAsync(e.b_gv.as<void>(), hv.data(), bytes, cudaMemcpyHostToDevice, e.st));
        IFGF_CUDA(cudaMemcpyAsync(e.b_gwv.as<void>(), hwv.data(), bytes, cudaMemcpyHostToDevice, e.st));
        launch_beta_batch(B, int(p0), int(cnt), e.beta_s.as<double2>(), e.beta_d.as<double2>(), e.max_dudv,
                          e.max_dv, e.max_nu, e.max_nunv, e.st);
    }
    IFGF_CUDA(cudaStreamSynchronize(e.st));
    for (DevBuf* b : {&e.b_gu, &e.b_gwu, &e.b_gv, &e.b_gwv}) b->alloc(0);
    e.beta_ready = true;
}

void Engine::upload_beta(const std::vector<std::uint64_t>& offset, const cplx* bs, const cplx* bd) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    IFGF_CUDA(cudaSetDevice(e.dev));
    if (offset.size() != e.pairs->size() + 1 || offset.back() != e.beta_entries)
        throw InvalidArgument("upload_beta: table layout does not match the pair list");
    e.alloc_beta(nullptr);
    IFGF_CUDA(cudaMemcpy(e.beta_s.as<void>(), bs, e.beta_entries * sizeof(double2), cudaMemcpyHostToDevice));
    IFGF_CUDA(cudaMemcpy(e.beta_d.as<void>(), bd, e.beta_entries * sizeof(double2), cudaMemcpyHostToDevice));
    e.beta_ready = true;
}

void Engine::download_beta(std::vector<std::uint64_t>& offset, std::vector<cplx>& bs,
                           std::vector<cplx>& bd) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    e.ensure_beta();
    if (e.beta_sharded) throw InvalidArgument("beta tables are target-sharded under a partition (no full tables here)");
    IFGF_CUDA(cudaSetDevice(e.dev));
    offset.resize(e.pairs->size() + 1);
    IFGF_CUDA(cudaMemcpy(offset.data(), e.beta_off.as<void>(), offset.size() * 8, cudaMemcpyDeviceToHost));
    bs.resize(e.beta_entries);
    bd.resize(e.beta_entries);
    IFGF_CUDA(cudaMemcpy(bs.data(), e.beta_s.as<void>(), e.beta_entries * sizeof(double2), cudaMemcpyDeviceToHost));
    IFGF_CUDA(cudaMemcpy(bd.data(), e.beta_d.as<void>(), e.beta_entries * sizeof(double2), cudaMemcpyDeviceToHost));
}

void Engine::apply(const cplx* phi, cplx* out, cplx* S, cplx* D) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    e.ensure_beta();
    if (e.collective() && (S || D))
        throw InvalidArgument("layer_potentials: S and D are target-distributed under a communicator");
    IFGF_CUDA(cudaSetDevice(e.dev));
    const std::size_t bytes = e.n * sizeof(double2);
    IFGF_CUDA(cudaMemcpyAsync(e.d_phi.as<void>(), phi, bytes, cudaMemcpyHostToDevice, e.st));
    e.apply_graph();
    IFGF_CUDA(cudaMemcpyAsync(out, e.d_out.as<void>(), bytes, cudaMemcpyDeviceToHost, e.st));
    if (S) IFGF_CUDA(cudaMemcpyAsync(S, e.d_S.as<void>(), bytes, cudaMemcpyDeviceToHost, e.st));
    if (D) IFGF_CUDA(cudaMemcpyAsync(D, e.d_D.as<void>(), bytes, cudaMemcpyDeviceToHost, e.st));
    IFGF_CUDA(cudaStreamSynchronize(e.st));
}

void Engine::apply_device(const void* phi, void* out, void* S, void* D) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    e.ensure_beta();
    IFGF_CUDA(cudaSetDevice(e.dev));
    e.run_apply(static_cast<const double2*>(phi), static_cast<double2*>(out), static_cast<double2*>(S),
                static_cast<double2*>(D));
    IFGF_CUDA(cudaStreamSynchronize(e.st));
}

// Restarted MGS-GMRES with Givens rotations (solver.cpp:177-300), vectors in HBM. Each
// Arnoldi step: V_j -> d_phi (device copy), one graph apply -> d_out = w, MGS against
// V_0..V_j with the coefficients kept on the device, |w|, then ONE copy of the column
// H[0..j+1] to the host for the rotations and the residual estimate.
//
// Under a communicator the solve is SHARDED by the operator's Morton ranges (SURVEY.md
// §8(e), north_star "GMRES vector segments"): each rank keeps only its owned segment of
// b, x, r and the Krylov basis (Morton order, (m+1) x n_owned), the apply all-gathers the
// segment into the full density and returns only the owned outputs, and every inner product
// and norm is a local partial sum followed by one ncclAllReduce of 2 doubles (modified
// Gram-Schmidt keeps the reference's orthogonalisation order, so the iteration counts and
// residual histories are the reference's). The Hessenberg column and the rotations are the
// same on every rank.
GmresOutcome Engine::gmres(const cplx* rhs, double tol, int max_iter, int restart) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    e.ensure_beta();
    if (tol <= 0) throw InvalidArgument("gmres_solve: tolerance must be positive");
    if (max_iter < 0) throw InvalidArgument("gmres_solve: max_iter must be >= 0");
    IFGF_CUDA(cudaSetDevice(e.dev));
    const bool shard = e.collective();
    const std::int64_t lo = shard ? std::int64_t(e.own_lo) : 0;
    const std::int64_t n = shard ? std::int64_t(e.own_hi - e.own_lo) : std::int64_t(e.n);  // local length
    const std::size_t vb = std::size_t(n) * sizeof(double2);
    const std::size_t vfull = e.n * sizeof(double2);
    const int m_max = restart > 0 ? std::min(restart, std::max(max_iter, 1)) : std::max(max_iter, 1);
    DevBuf b, x, r, V, H, partial, yv;
    b.alloc(std::max<std::size_t>(vb, 16));
    x.alloc(std::max<std::size_t>(vb, 16));
    r.alloc(std::max<std::size_t>(vb, 16));
    V.alloc(std::max<std::size_t>(std::size_t(m_max + 1) * vb, 16));
    H.alloc(std::size_t(m_max + 2) * sizeof(double2));
    partial.alloc(std::size_t(gmres_reduce_blocks()) * sizeof(double2));
    yv.alloc(std::size_t(m_max + 1) * sizeof(double2));
    cudaStream_t st = e.st;
    if (shard) {  // the owned Morton segment of rhs
        IFGF_CUDA(cudaMemcpyAsync(e.scratch.as<void>(), rhs, vfull, cudaMemcpyHostToDevice, st));
        launch_gather_local(e.perm.as<std::uint32_t>(), lo, n, e.scratch.as<double2>(), b.as<double2>(), st);
    } else {
        IFGF_CUDA(cudaMemcpyAsync(b.as<void>(), rhs, vb, cudaMemcpyHostToDevice, st));
    }
    IFGF_CUDA(cudaMemsetAsync(x.as<void>(), 0, std::max<std::size_t>(vb, 16), st));
    auto Vi = [&](int i) { return V.as<double2>() + std::size_t(i) * std::size_t(n); };
    auto read_h = [&](int cnt, std::vector<cplx>& dst) {
        dst.resize(cnt);
        IFGF_CUDA(cudaMemcpyAsync(dst.data(), H.as<void>(), cnt * sizeof(double2), cudaMemcpyDeviceToHost, st));
        IFGF_CUDA(cudaStreamSynchronize(st));
    };
    // the operator output of `in`: d_out (full) or, sharded, the owned segment of out_m
    double2* w_out = shard ? e.out_m.as<double2>() + lo : e.d_out.as<double2>();
    auto apply_to = [&](const double2* in) {
        if (shard) {  // segments -> full density on every rank, owned outputs only
            e.allgather_to_original(in, e.d_phi.as<double2>());
            e.run_apply(e.d_phi.as<double2>(), e.d_out.as<double2>(), nullptr, nullptr, true);
        } else {
            IFGF_CUDA(cudaMemcpyAsync(e.d_phi.as<void>(), in, vb, cudaMemcpyDeviceToDevice, st));
            e.apply_graph();
        }
    };
    // dst = <a, b> (as_norm: ||a||) over the whole distributed vector
    auto dot = [&](const double2* a, const double2* bb, double2* dst, bool as_norm) {
        if (!shard) {
            launch_cdot(n, a, bb, partial.as<double2>(), dst, as_norm, st);
            return;
        }
        launch_cdot(n, a, bb, partial.as<double2>(), dst, false, st);
        IFGF_NCCL(ncclAllReduce(dst, dst, 2, ncclFloat64, ncclSum, e.comm, st));
        if (as_norm) launch_csqrt_re(dst, st);
    };
    std::vector<cplx> hcol;
    dot(b.as<double2>(), b.as<double2>(), H.as<double2>(), true);
    read_h(1, hcol);
    const double bnorm = hcol[0].real();
    GmresOutcome total;
    if (bnorm == 0.0) {
        total.x.assign(e.n, cplx{});
        total.converged = true;
        return total;
    }
    bool x_nonzero = false;
    // one Arnoldi cycle of length m from the current x; returns converged
    auto cycle = [&](int m, GmresOutcome& res) {
        if (x_nonzero) {
            apply_to(x.as<double2>());
            launch_csub(n, b.as<double2>(), w_out, r.as<double2>(), st);
        } else if (n > 0) {
            IFGF_CUDA(cudaMemcpyAsync(r.as<void>(), b.as<void>(), vb, cudaMemcpyDeviceToDevice, st));
        }
        dot(r.as<double2>(), r.as<double2>(), H.as<double2>(), true);
        read_h(1, hcol);
        const double beta = hcol[0].real();
        if (beta / bnorm <= tol) return true;
        launch_cscale_inv(n, H.as<double2>(), r.as<double2>(), Vi(0), st);  // V_0 = r / beta
        std::vector<std::vector<cplx>> Hh;
        std::vector<cplx> cs(m), sn(m), gv(m + 1, cplx{});
        gv[0] = beta;
        for (int j = 0; j < m; ++j) {
            apply_to(Vi(j));
            double2* w = w_out;
            for (int i = 0; i <= j; ++i) {
                double2* hi = H.as<double2>() + i;
                dot(Vi(i), w, hi, false);
                launch_caxpy_dev(n, hi, w, Vi(i), st);
            }
            dot(w, w, H.as<double2>() + j + 1, true);
            read_h(j + 2, hcol);
            Hh.push_back(hcol);
            std::vector<cplx>& Hj = Hh.back();
            const double hn = Hj[j + 1].real();
            ++res.iterations;
            for (int i = 0; i < j; ++i) {
                const cplx t = std::conj(cs[i]) * Hj[i] + std::conj(sn[i]) * Hj[i + 1];
                Hj[i + 1] = -sn[i] * Hj[i] + cs[i] * Hj[i + 1];
                Hj[i] = t;
            }
            const double den = std::sqrt(std::norm(Hj[j]) + hn * hn);
            if (den < 1e-300) {
                res.history.push_back(std::abs(gv[j]) / bnorm);
                throw ConvergenceFailure("gmres: Arnoldi breakdown", res.history);
            }
            cs[j] = Hj[j] / den;
            sn[j] = cplx(hn / den, 0.0);
            Hj[j] = std::conj(cs[j]) * Hj[j] + std::conj(sn[j]) * hn;
            Hj[j + 1] = 0.0;
            gv[j + 1] = -sn[j] * gv[j];
            gv[j] = std::conj(cs[j]) * gv[j];
            const double rel = std::abs(gv[j + 1]) / bnorm;
            res.history.push_back(rel);
            if (rel <= tol || j == m - 1 || hn < 1e-14) {
                std::vector<cplx> y(j + 1);
                for (int i = j; i >= 0; --i) {
                    cplx acc = gv[i];
                    for (int t = i + 1; t <= j; ++t) acc -= Hh[t][i] * y[t];
                    y[i] = acc / Hh[i][i];
                }
                IFGF_CUDA(cudaMemcpyAsync(yv.as<void>(), y.data(), y.size() * sizeof(double2),
                                          cudaMemcpyHostToDevice, st));
                launch_cupdate(n, j + 1, yv.as<double2>(), V.as<double2>(), n, x.as<double2>(), st);
                x_nonzero = true;
                return rel <= tol;
            }
            launch_cscale_inv(n, H.as<double2>() + j + 1, w, Vi(j + 1), st);  // V_{j+1} = w / hn
        }
        return false;
    };
    try {
        if (restart <= 0) {
            GmresOutcome part;
            total.converged = cycle(std::max(max_iter, 0), part);
            total.iterations = part.iterations;
            total.history = std::move(part.history);
        } else {
            while (total.iterations < max_iter) {
                const int len = std::min(restart, max_iter - total.iterations);
                GmresOutcome part;
                const bool ok = cycle(len, part);
                total.iterations += part.iterations;
                total.history.insert(total.history.end(), part.history.begin(), part.history.end());
                if (ok) {
                    total.converged = true;
                    break;
                }
            }
        }
    } catch (const ConvergenceFailure& f) {
        std::vector<double> h = total.history;
        h.insert(h.end(), f.history.begin(), f.history.end());
        throw ConvergenceFailure(f.what(), h);
    }
    total.x.resize(e.n);
    if (shard) {  // every rank returns the full solution (original order)
        e.allgather_to_original(x.as<double2>(), e.scratch.as<double2>());
        IFGF_CUDA(cudaMemcpyAsync(total.x.data(), e.scratch.as<void>(), vfull, cudaMemcpyDeviceToHost, st));
    } else {
        IFGF_CUDA(cudaMemcpyAsync(total.x.data(), x.as<void>(), vb, cudaMemcpyDeviceToHost, st));
    }
    IFGF_CUDA(cudaStreamSynchronize(st));
    return total;
}

void Engine::ifgf_apply(const cplx* a, bool single, bool dbl, DlStrategy s, cplx* S, cplx* D) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    IFGF_CUDA(cudaSetDevice(e.dev));
    const std::size_t bytes = e.n * sizeof(double2);
    IFGF_CUDA(cudaMemcpyAsync(e.d_phi.as<void>(), a, bytes, cudaMemcpyHostToDevice, e.st));
    IFGF_CUDA(cudaMemsetAsync(e.Sp.as<void>(), 0, bytes, e.st));
    IFGF_CUDA(cudaMemsetAsync(e.Dp.as<void>(), 0, bytes, e.st));
    launch_weights(int(e.n), e.perm.as<std::uint32_t>(), e.d_phi.as<double2>(), e.ones_p.as<double>(),
                   e.a_p.as<double2>(), e.st);
    e.ensure_stores(single, dbl, s);
    e.run_ifgf(single, dbl, s);
    launch_unpermute(int(e.n), e.perm.as<std::uint32_t>(), e.Sp.as<double2>(), e.Dp.as<double2>(),
                     e.d_S.as<double2>(), e.d_D.as<double2>(), e.st);
    IFGF_CUDA(cudaMemcpyAsync(S, e.d_S.as<void>(), bytes, cudaMemcpyDeviceToHost, e.st));
    IFGF_CUDA(cudaMemcpyAsync(D, e.d_D.as<void>(), bytes, cudaMemcpyDeviceToHost, e.st));
    IFGF_CUDA(cudaStreamSynchronize(e.st));
}

void Engine::level_d_fill(const cplx* a_perm, const std::vector<int>& pipes, std::vector<cplx>& out) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    IFGF_CUDA(cudaSetDevice(e.dev));
    out.clear();
    if (e.depth < 3) return;
    if (pipes.empty() || pipes.size() > 3) throw InvalidArgument("level_d_fill: 1..3 pipelines");
    const LevelDev& L = e.L[e.depth - 1];
    const std::size_t total = std::size_t(L.nseg) * (L.ps * L.pang * L.pang) * pipes.size();
    e.ensure_stores(true, true, e.strategy, int(pipes.size()));
    IFGF_CUDA(cudaMemcpyAsync(e.a_p.as<void>(), a_perm, e.n * sizeof(double2), cudaMemcpyHostToDevice, e.st));
    launch_leaf_fill(L, e.P, e.a_p.as<double2>(), e.k, make_pipes(pipes), e.Ms.as<double>(),
                     e.Ma.as<double>(), e.storeA.as<double2>(), e.st);
    out.resize(total);
    IFGF_CUDA(cudaMemcpyAsync(out.data(), e.storeA.as<void>(), total * sizeof(double2), cudaMemcpyDeviceToHost, e.st));
    IFGF_CUDA(cudaStreamSynchronize(e.st));
}

void Engine::apply_direct(const cplx* phi, cplx* out) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    e.ensure_beta();
    IFGF_CUDA(cudaSetDevice(e.dev));
    const std::size_t bytes = e.n * sizeof(double2);
    IFGF_CUDA(cudaMemcpyAsync(e.d_phi.as<void>(), phi, bytes, cudaMemcpyHostToDevice, e.st));
    launch_direct(e.direct, e.d_phi.as<double2>(), e.k, e.Sp.as<double2>(), e.Dp.as<double2>(), e.st);
    RpDev rp = e.rp;
    rp.pos = e.identity.as<std::uint32_t>();  // Sp/Dp are in original order here
    launch_density_coeffs(rp, e.d_phi.as<double2>(), e.coeffs.as<double2>(), e.st);
    launch_rp_combine(rp, e.coeffs.as<double2>(), e.d_phi.as<double2>(), e.Sp.as<double2>(),
                      e.Dp.as<double2>(), e.gamma, e.scratch.as<double2>(), nullptr, nullptr, e.st);
    IFGF_CUDA(cudaMemcpyAsync(out, e.scratch.as<void>(), bytes, cudaMemcpyDeviceToHost, e.st));
    IFGF_CUDA(cudaStreamSynchronize(e.st));
}

void Engine::rp_apply(const cplx* phi, cplx* S, cplx* D) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    e.ensure_beta();
    IFGF_CUDA(cudaSetDevice(e.dev));
    const std::size_t bytes = e.n * sizeof(double2);
    IFGF_CUDA(cudaMemcpyAsync(e.d_phi.as<void>(), phi, bytes, cudaMemcpyHostToDevice, e.st));
    IFGF_CUDA(cudaMemsetAsync(e.Sp.as<void>(), 0, bytes, e.st));
    IFGF_CUDA(cudaMemsetAsync(e.Dp.as<void>(), 0, bytes, e.st));
    launch_density_coeffs(e.rp, e.d_phi.as<double2>(), e.coeffs.as<double2>(), e.st);
    launch_rp_combine(e.rp, e.coeffs.as<double2>(), e.d_phi.as<double2>(), e.Sp.as<double2>(),
                      e.Dp.as<double2>(), 0.0, e.scratch.as<double2>(), e.d_S.as<double2>(),
                      e.d_D.as<double2>(), e.st);
    IFGF_CUDA(cudaMemcpyAsync(S, e.d_S.as<void>(), bytes, cudaMemcpyDeviceToHost, e.st));
    IFGF_CUDA(cudaMemcpyAsync(D, e.d_D.as<void>(), bytes, cudaMemcpyDeviceToHost, e.st));
    IFGF_CUDA(cudaStreamSynchronize(e.st));
}

void Engine::upload_density(const cplx* phi) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    IFGF_CUDA(cudaSetDevice(e.dev));
    IFGF_CUDA(cudaMemcpy(e.d_phi.as<void>(), phi, e.n * sizeof(double2), cudaMemcpyHostToDevice));
}

double Engine::time_device_applies(int iters, bool flush_l2) {
    const std::vector<double> each = time_device_applies_each(iters, flush_l2);
    double total = 0;
    for (double t : each) total += t;
    return each.empty() ? 0.0 : total / double(each.size());
}

std::vector<double> Engine::time_device_applies_each(int iters, bool flush_l2) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    e.ensure_beta();
    IFGF_CUDA(cudaSetDevice(e.dev));
    const std::size_t flush_bytes = std::size_t(256) << 20;  // 2x the 126 MB L2
    if (flush_l2 && e.flush.bytes() < flush_bytes) e.flush.alloc(flush_bytes);
    e.apply_graph();  // eager run + capture on first use
    IFGF_CUDA(cudaStreamSynchronize(e.st));
    cudaEvent_t a, b;
    IFGF_CUDA(cudaEventCreate(&a));
    IFGF_CUDA(cudaEventCreate(&b));
    std::vector<double> each;
    for (int i = 0; i < iters; ++i) {
        if (flush_l2) IFGF_CUDA(cudaMemsetAsync(e.flush.as<void>(), i & 0xff, flush_bytes, e.st));
        IFGF_CUDA(cudaEventRecord(a, e.st));
        e.apply_graph();
        IFGF_CUDA(cudaEventRecord(b, e.st));
        IFGF_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        IFGF_CUDA(cudaEventElapsedTime(&ms, a, b));
        each.push_back(double(ms));
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return each;
}

PhaseTimes Engine::time_phases() {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    e.ensure_beta();
    IFGF_CUDA(cudaSetDevice(e.dev));
    PhaseTimes pt;
    if (!e.eager_done) e.apply_graph();
    IFGF_CUDA(cudaStreamSynchronize(e.st));
    // events: start, weights, leaf, then per level (cousin, parent), near, rp
    std::vector<cudaEvent_t> ev(4 + 2 * e.depth + 4);
    for (auto& x : ev) IFGF_CUDA(cudaEventCreate(&x));
    int ie = 0;
    auto rec = [&] { IFGF_CUDA(cudaEventRecord(ev[ie++], e.st)); };
    auto el = [&](int i0, int i1) {
        float ms = 0.f;
        IFGF_CUDA(cudaEventElapsedTime(&ms, ev[i0], ev[i1]));
        return double(ms);
    };
    const double2* phi = e.d_phi.as<double2>();
    rec();  // 0
    IFGF_CUDA(cudaMemsetAsync(e.Sp.as<void>(), 0, e.n * sizeof(double2), e.st));
    IFGF_CUDA(cudaMemsetAsync(e.Dp.as<void>(), 0, e.n * sizeof(double2), e.st));
    launch_weights(int(e.n), e.perm.as<std::uint32_t>(), phi, e.jw_p.as<double>(), e.a_p.as<double2>(), e.st);
    rec();  // 1
    std::vector<std::pair<int, int>> cousin_ev, parent_ev;
    if (e.depth >= 3) {
        double2* cur = e.storeA.as<double2>();
        double2* nxt = e.storeB.as<double2>();
        launch_leaf_fill(e.L[e.depth - 1], e.P, e.a_p.as<double2>(), e.k,
                         make_pipes(e.pipes_at(e.depth, true, true, e.strategy)), e.Ms.as<double>(),
                         e.Ma.as<double>(), cur, e.st);
        rec();  // 2
        for (int d = e.depth; d >= 3; --d) {
            const Pipes pc = make_pipes(e.pipes_at(d, true, true, e.strategy));
            const int c0 = ie - 1;
            launch_cousin_eval(e.L[d - 1], e.P, cur, e.k, pc, e.Sp.as<double2>(), e.Dp.as<double2>(), e.st);
            rec();
            cousin_ev.push_back({c0, ie - 1});
            if (d > 3) {
                const Pipes pp = make_pipes(e.pipes_at(d - 1, true, true, e.strategy));
                const int p0 = ie - 1;
                launch_parent_fill(e.L[d - 2], e.L[d - 1], cur, e.k, pp, pc, e.Ms.as<double>(),
                                   e.Ma.as<double>(), nxt, e.st);
                rec();
                parent_ev.push_back({p0, ie - 1});
                std::swap(cur, nxt);
            }
        }
    } else {
        rec();
    }
    const int n0 = ie - 1;
    e.ensure_near_lists();
    launch_near_field(e.near, e.P, e.a_p.as<double2>(), e.k, e.Sp.as<double2>(), e.Dp.as<double2>(), e.st);
    rec();
    const int r0 = ie - 1;
    launch_density_coeffs(e.rp, phi, e.coeffs.as<double2>(), e.st);
    launch_rp_combine(e.rp, e.coeffs.as<double2>(), phi, e.Sp.as<double2>(), e.Dp.as<double2>(), e.gamma,
                      e.d_out.as<double2>(), e.d_S.as<double2>(), e.d_D.as<double2>(), e.st);
    rec();
    IFGF_CUDA(cudaEventSynchronize(ev[ie - 1]));
    pt.weights = el(0, 1);
    pt.leaf = el(1, 2);
    for (auto& c : cousin_ev) pt.cousin += el(c.first, c.second);
    for (auto& p : parent_ev) pt.parent += el(p.first, p.second);
    pt.near = el(n0, n0 + 1);
    pt.rp = el(r0, r0 + 1);
    pt.total = el(0, ie - 1);
    for (auto& x : ev) cudaEventDestroy(x);
    return pt;
}

int Engine::kernels_per_apply() const {
    const Impl& e = *d_;
    if (e.kernels > 0) return e.kernels;  // counted by the last run_apply
    // weights + leaf + cousin per level + parent per level > 3 + near + coeffs + rp + combine
    // (+ the output un-permute under a communicator)
    const int ifgf = e.depth < 3 ? 0 : 1 + (e.depth - 2) + (e.depth - 3);
    return 1 + ifgf + 3 + 1 + (e.collective() ? 4 : 0);
}

std::string Engine::describe() const {
    const Impl& e = *d_;
    std::ostringstream os;
    os << "N=" << e.n << " depth=" << e.depth << " store_elems=" << e.store_elems
       << " beta_entries=" << e.beta_entries << " pairs=" << e.pairs->size();
    return os.str();
}

std::vector<std::uint32_t> Engine::partition_bounds(int parts) const {
    if (parts < 1) throw InvalidArgument("partition: need at least one part");
    return d_->partition(parts);
}

void Engine::set_partition(std::uint32_t lo, std::uint32_t hi) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    IFGF_CUDA(cudaSetDevice(e.dev));
    e.set_partition(lo, hi);
}

void Engine::set_comm(int rank, int world, const void* unique_id) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    if (world < 1 || rank < 0 || rank >= world) throw InvalidArgument("set_comm: bad rank/world");
    IFGF_CUDA(cudaSetDevice(e.dev));
    if (e.comm) {
        ncclCommDestroy(e.comm);
        e.comm = nullptr;
    }
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof id);
    IFGF_NCCL(ncclCommInitRank(&e.comm, world, id, rank));
    e.rank = rank;
    e.world = world;
    e.bounds = e.partition(world);
    e.set_partition(e.bounds[rank], e.bounds[rank + 1]);
    e.alloc_exchange();
}

void Engine::finish_owned(const cplx* phi, const cplx* far_S, const cplx* far_D, cplx* out) {
    Impl& e = *d_;
    std::lock_guard<std::mutex> g(e.mu);
    e.ensure_beta();
    IFGF_CUDA(cudaSetDevice(e.dev));
    const std::size_t bytes = e.n * sizeof(double2);
    IFGF_CUDA(cudaMemcpyAsync(e.d_phi.as<void>(), phi, bytes, cudaMemcpyHostToDevice, e.st));
    IFGF_CUDA(cudaMemcpyAsync(e.d_S.as<void>(), far_S, bytes, cudaMemcpyHostToDevice, e.st));
    IFGF_CUDA(cudaMemcpyAsync(e.d_D.as<void>(), far_D, bytes, cudaMemcpyHostToDevice, e.st));
    // far field into Morton order, weighted sources, then the target-owned stages
    launch_weights(int(e.n), e.perm.as<std::uint32_t>(), e.d_S.as<double2>(), e.ones_p.as<double>(),
                   e.Sp.as<double2>(), e.st);
    launch_weights(int(e.n), e.perm.as<std::uint32_t>(), e.d_D.as<double2>(), e.ones_p.as<double>(),
                   e.Dp.as<double2>(), e.st);
    launch_weights(int(e.n), e.perm.as<std::uint32_t>(), e.d_phi.as<double2>(), e.jw_p.as<double>(),
                   e.a_p.as<double2>(), e.st);
    e.ensure_near_lists();
    launch_near_field(e.near, e.P, e.a_p.as<double2>(), e.k, e.Sp.as<double2>(), e.Dp.as<double2>(), e.st);
    launch_density_coeffs(e.rp, e.d_phi.as<double2>(), e.coeffs.as<double2>(), e.st);
    IFGF_CUDA(cudaMemsetAsync(e.scratch.as<void>(), 0, bytes, e.st));
    launch_rp_combine(e.rp, e.coeffs.as<double2>(), e.d_phi.as<double2>(), e.Sp.as<double2>(), e.Dp.as<double2>(),
                      e.gamma, e.scratch.as<double2>(), nullptr, nullptr, e.st);
    IFGF_CUDA(cudaMemcpyAsync(out, e.scratch.as<void>(), bytes, cudaMemcpyDeviceToHost, e.st));
    IFGF_CUDA(cudaStreamSynchronize(e.st));
}

void* Engine::device_phi() { return d_->d_phi.as<void>(); }
void* Engine::device_out() { return d_->d_out.as<void>(); }
void Engine::sync() {
    IFGF_CUDA(cudaSetDevice(d_->dev));
    IFGF_CUDA(cudaStreamSynchronize(d_->st));
}

}  // namespace ifgfb200
