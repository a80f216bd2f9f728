// context.cu -- host runtime of libmpm_b200.so: device context, buffer ownership, step
// orchestration (CUDA graph per step), error attribution and the C ABI (include/mpm_capi.h).
//
// The context is the device-side Stepper (stepper.hpp:49-70): it owns the particle state
// (double-buffered SoA), the node-block grid, the sort / segment tables, the P2G partial tiles
// and the adjoint workspace, all on one CUDA stream. Calls are synchronous at return.

#include "../../include/mpm_capi.h"
#include "common.cuh"
#include "constit.cuh"
#include "kernels_adj.cuh"
#include "kernels_fwd.cuh"
#include "kernels_sort.cuh"
#include "kernels_dist.cuh"

#include <dlfcn.h>
#include <nccl.h> // types only: the functions are resolved at run time (dyn::api)
#include <type_traits>
#include "kernels_util.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

using namespace mpmgpu;

#ifndef G2P_ABL
#define G2P_ABL 0 // timing-ablation builds only (tools/p2g_ablate.py)
#endif
#ifndef P2G_ABL
#define P2G_ABL 0 // timing-ablation builds only (tools/p2g_ablate.py)
#endif
#if P2G_ABL == 16
__global__ void k_spin_abl(long long cycles) // idle the SMs (no memory traffic) in front of P2G
{
    pdl_wait();
    pdl_trigger();
    const long long t0 = clock64();
    while (clock64() - t0 < cycles)
        __nanosleep(1000);
}
#endif
#ifndef P2G_WIDE
#define P2G_WIDE false
#endif

namespace {

struct ApiError : std::runtime_error {
    int code;
    int64_t particle, step;
    ApiError(int c, const std::string& m, int64_t p = -1, int64_t s = -1)
        : std::runtime_error(m), code(c), particle(p), step(s)
    {
    }
};

// NCCL is resolved at run time, on the first decomposed call, so the library carries no load-time
// dependency on a particular libnccl: a process that loads it before torch (which needs its own
// bundled, newer libnccl.so.2) keeps working, and single-GPU use never touches NCCL. An already
// loaded libnccl.so.2 (torch's) is preferred; otherwise the loader's search path decides.
namespace dyn {
struct Api {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    std::string error;
};
inline const Api& api()
{
    static const Api a = [] {
        Api r;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h)
            h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            const char* e = dlerror();
            r.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return r;
        }
        auto sym = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp && r.error.empty())
                r.error = std::string("libnccl.so.2 lacks ") + name;
        };
        sym(r.GetUniqueId, "ncclGetUniqueId");
        sym(r.CommInitRank, "ncclCommInitRank");
        sym(r.CommDestroy, "ncclCommDestroy");
        sym(r.GetErrorString, "ncclGetErrorString");
        sym(r.GroupStart, "ncclGroupStart");
        sym(r.GroupEnd, "ncclGroupEnd");
        sym(r.Send, "ncclSend");
        sym(r.Recv, "ncclRecv");
        sym(r.AllReduce, "ncclAllReduce");
        sym(r.AllGather, "ncclAllGather");
        return r;
    }();
    if (!a.error.empty())
        throw ApiError(MPM_ERR_USAGE, "dist: " + a.error);
    return a;
}
inline ncclResult_t ncclGetUniqueId(ncclUniqueId* id) { return api().GetUniqueId(id); }
inline ncclResult_t ncclCommInitRank(ncclComm_t* c, int n, ncclUniqueId id, int r) { return api().CommInitRank(c, n, id, r); }
inline ncclResult_t ncclCommDestroy(ncclComm_t c) { return api().CommDestroy(c); }
inline const char* ncclGetErrorString(ncclResult_t e) { return api().GetErrorString(e); }
inline ncclResult_t ncclGroupStart() { return api().GroupStart(); }
inline ncclResult_t ncclGroupEnd() { return api().GroupEnd(); }
inline ncclResult_t ncclSend(const void* b, size_t n, ncclDataType_t t, int p, ncclComm_t c, cudaStream_t s)
{
    return api().Send(b, n, t, p, c, s);
}
inline ncclResult_t ncclRecv(void* b, size_t n, ncclDataType_t t, int p, ncclComm_t c, cudaStream_t s)
{
    return api().Recv(b, n, t, p, c, s);
}
inline ncclResult_t ncclAllReduce(const void* a, void* b, size_t n, ncclDataType_t t, ncclRedOp_t o, ncclComm_t c,
                                  cudaStream_t s)
{
    return api().AllReduce(a, b, n, t, o, c, s);
}
inline ncclResult_t ncclAllGather(const void* a, void* b, size_t n, ncclDataType_t t, ncclComm_t c, cudaStream_t s)
{
    return api().AllGather(a, b, n, t, c, s);
}
} // namespace dyn

#define NCK(call)                                                                                  \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess)                                                                     \
            throw ApiError(MPM_ERR_CUDA, std::string("NCCL error: ") + dyn::ncclGetErrorString(r_) + " at " \
                                             + __FILE__ + ":" + std::to_string(__LINE__));         \
    } while (0)

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            throw ApiError(MPM_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " \
                                             + __FILE__ + ":" + std::to_string(__LINE__));         \
    } while (0)

struct LocalHub;

struct ProfEvent {
    const char* name;
    cudaEvent_t a, b;
};

// ----------------------------------------------------------------------------------------
struct CtxBase {
    virtual ~CtxBase() = default;
    virtual void upload(const mpm_state_view* s) = 0;
    virtual void download(mpm_state_view* s) = 0;
    virtual uint64_t digest() = 0;
    virtual double max_speed() = 0;
    virtual void advance(int64_t n, uint32_t flags) = 0;
    virtual double advance_timed(int64_t n, uint32_t flags) = 0;
    virtual void phase_p2g() = 0;
    virtual void phase_mom() = 0;
    virtual void phase_corr() = 0;
    virtual void phase_g2p() = 0;
    virtual void phase_constit() = 0;
    virtual void grid_download(mpm_grid_view* g) = 0;
    virtual void grid_upload(const mpm_grid_view* g) = 0;
    virtual void step_vjp(const mpm_state_view* s, const mpm_cot_view* co, mpm_cot_view* ci, mpm_param_grads* pg) = 0;
    virtual void backprop(const mpm_state_view* s0, int64_t total, int nseg, const mpm_seeder_desc* sd,
                          mpm_cot_view* c0, mpm_param_grads* pg, mpm_backprop_result* res) = 0;
    virtual void grid_stats(int64_t* an, int64_t* ob, int64_t* anb) = 0;
    virtual void upload_ids(const mpm_state_view* s, const int64_t* ids) = 0;
    virtual void download_local(mpm_state_view* s, int64_t* ids) = 0;
    virtual void slab_set(int lo, int hi, int64_t mig_cap) = 0;
    virtual void step_p2g_local() = 0;
    virtual void step_grid_interior() = 0;
    virtual void snapshot_begin(int slot) = 0;
    virtual void snapshot_fetch(int slot, mpm_state_view* s) = 0;
    virtual void init_scene_dev(const mpm_region* rg, int nreg, double mass, double volume, double rho0,
                                int64_t* n_out) = 0;
    virtual void slab_vjp_begin(const mpm_cot_view* co) = 0;
    virtual void slab_vjp_interior() = 0;
    virtual void slab_vjp_scatter() = 0;
    virtual void halo_cot(int plane_lo, int n_planes, void* dev_buf, int mode) = 0;
    virtual void slab_vjp_finish(mpm_cot_view* ci, mpm_param_grads* pg) = 0;
    virtual void halo(int plane_lo, int n_planes, void* dev_buf, int mode) = 0;
    virtual void step_finish_local(uint32_t flags) = 0;
    virtual void step_finish_async(uint32_t flags, long long* dev_report) = 0;
    virtual void step_commit(int64_t n_lo, int64_t n_hi, int any_failed) = 0;
    virtual void migrate_export(void* lo, int* lo_pid, void* hi, int* hi_pid, int64_t cap, int64_t* n_lo, int64_t* n_hi) = 0;
    virtual void migrate_import(const void* recs, const int* pids, int64_t k) = 0;
    virtual int rec_size() const = 0;
    virtual int64_t local_count() const = 0;
    virtual void set_stream(void* s) = 0;
    virtual void migrate_counts(int64_t* lo, int64_t* hi) const = 0;
    // library-owned slab decomposition (kernels_dist.cuh)
    virtual void dist_attach(int rank, int nranks, int lo, int hi, int64_t mig_cap, const void* nccl_id) = 0;
    virtual void dist_advance(int64_t n, uint32_t flags, double* ms) = 0;
    virtual int dist_device() const = 0;
    virtual void dist_enqueue_local(std::vector<CtxBase*>& all, int64_t n, uint32_t flags) = 0;
    virtual void dist_finish() = 0;
    virtual void dist_backprop_nccl(int64_t total, int nseg, const mpm_seeder_desc* sd, int64_t id_space,
                                    mpm_cot_view* c0, int64_t* c0_ids, mpm_param_grads* pg, mpm_backprop_result* res) = 0;
    virtual void dist_backprop_local(LocalHub* hub, int64_t total, int nseg, const mpm_seeder_desc* sd,
                                     int64_t id_space, mpm_cot_view* c0, int64_t* c0_ids, mpm_param_grads* pg,
                                     mpm_backprop_result* res) = 0;

    // profiling
    bool prof = false;
    std::vector<ProfEvent> events;
    std::vector<std::pair<std::string, std::pair<double, int64_t>>> prof_acc;
    int64_t launches = 0;
};

// ---- transports of the library-owned decomposition --------------------------------------------
// An exchange is a list of (send, recv, bytes, peer) pairs; every rank lists its pairs with a peer
// in the same order as the peer lists its pairs with it. begin() puts the transfers on the
// timeline of `stream` (sends read after the work enqueued so far), end() orders the work enqueued
// after it behind the receives. NCCL: grouped ncclSend / ncclRecv on a communication stream,
// ordered by events (capturable in a CUDA graph). Same-process ranks (one host thread per rank):
// a rendezvous publishes the send buffers, then device copies from the peers' buffers, ordered by
// events; nothing waits for the device on the host.
struct XItem {
    const void* send;
    void* recv;
    size_t bytes;
    int peer;
};
struct DistTransport {
    virtual ~DistTransport() = default;
    virtual void begin(cudaStream_t s, const std::vector<XItem>& items) = 0;
    virtual void end(cudaStream_t s) = 0;
    // recv[nranks * bytes] <- every rank's send[bytes], rank order
    virtual void allgather(cudaStream_t s, const void* send, void* recv, size_t bytes) = 0;
};

struct NcclX : DistTransport {
    ncclComm_t comm;
    cudaStream_t cs;
    cudaEvent_t ea, eb;
    NcclX(ncclComm_t c, cudaStream_t s, cudaEvent_t a, cudaEvent_t b) : comm(c), cs(s), ea(a), eb(b) {}
    void begin(cudaStream_t s, const std::vector<XItem>& items) override
    {
        CK(cudaEventRecord(ea, s));
        CK(cudaStreamWaitEvent(cs, ea, 0));
        NCK(dyn::ncclGroupStart());
        for (const XItem& it : items) {
            NCK(dyn::ncclSend(it.send, it.bytes, ncclUint8, it.peer, comm, cs));
            NCK(dyn::ncclRecv(it.recv, it.bytes, ncclUint8, it.peer, comm, cs));
        }
        NCK(dyn::ncclGroupEnd());
        CK(cudaEventRecord(eb, cs));
    }
    void end(cudaStream_t s) override { CK(cudaStreamWaitEvent(s, eb, 0)); }
    void allgather(cudaStream_t s, const void* send, void* recv, size_t bytes) override
    {
        CK(cudaEventRecord(ea, s));
        CK(cudaStreamWaitEvent(cs, ea, 0));
        NCK(dyn::ncclAllGather(send, recv, bytes, ncclUint8, comm, cs));
        CK(cudaEventRecord(eb, cs));
        CK(cudaStreamWaitEvent(s, eb, 0));
    }
};

struct LocalHub {
    int R;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    long long gen = 0;
    std::vector<std::vector<XItem>> items;
    std::vector<const void*> gsend;
    std::vector<cudaEvent_t> ready, done;
    std::vector<std::string> err; // a rank that failed on the host side releases the others
    bool failed = false;
    explicit LocalHub(int r) : R(r), items(r), gsend(r), ready(r), done(r), err(r)
    {
        for (int k = 0; k < R; ++k) {
            CK(cudaEventCreateWithFlags(&ready[k], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
        }
    }
    ~LocalHub()
    {
        for (int k = 0; k < R; ++k) {
            cudaEventDestroy(ready[k]);
            cudaEventDestroy(done[k]);
        }
    }
    void barrier()
    {
        std::unique_lock<std::mutex> lk(m);
        if (failed)
            throw ApiError(MPM_ERR_CUDA, "dist: another same-process rank failed");
        const long long g = gen;
        if (++arrived == R) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g || failed; });
            if (failed)
                throw ApiError(MPM_ERR_CUDA, "dist: another same-process rank failed");
        }
    }
    void fail()
    {
        std::lock_guard<std::mutex> lk(m);
        failed = true;
        cv.notify_all();
    }
};

struct LocalX : DistTransport {
    LocalHub* hub;
    int rank;
    LocalX(LocalHub* h, int r) : hub(h), rank(r) {}
    void settle(cudaStream_t s)
    {
        CK(cudaEventRecord(hub->done[rank], s));
        hub->barrier();
        for (int p = 0; p < hub->R; ++p) // peers' copies out of this rank's buffers come first
            if (p != rank)
                CK(cudaStreamWaitEvent(s, hub->done[p], 0));
        hub->barrier(); // every rank has queued its waits before the events are recorded again
    }
    void begin(cudaStream_t s, const std::vector<XItem>& items) override
    {
        hub->items[rank] = items;
        CK(cudaEventRecord(hub->ready[rank], s));
        hub->barrier();
        std::vector<int> seen(hub->R, 0);
        for (const XItem& it : items) {
            const int p = it.peer;
            int j = seen[p]++, k = -1;
            for (size_t q = 0; q < hub->items[p].size(); ++q)
                if (hub->items[p][q].peer == rank && j-- == 0) {
                    k = int(q);
                    break;
                }
            if (k < 0 || hub->items[p][k].bytes != it.bytes)
                throw ApiError(MPM_ERR_CUDA, "dist: mismatched same-process exchange");
            CK(cudaStreamWaitEvent(s, hub->ready[p], 0));
            CK(cudaMemcpyAsync(it.recv, hub->items[p][k].send, it.bytes, cudaMemcpyDeviceToDevice, s));
        }
        settle(s);
    }
    void end(cudaStream_t) override {}
    void allgather(cudaStream_t s, const void* send, void* recv, size_t bytes) override
    {
        hub->gsend[rank] = send;
        CK(cudaEventRecord(hub->ready[rank], s));
        hub->barrier();
        for (int p = 0; p < hub->R; ++p) {
            CK(cudaStreamWaitEvent(s, hub->ready[p], 0));
            CK(cudaMemcpyAsync(static_cast<char*>(recv) + size_t(p) * bytes, hub->gsend[p], bytes,
                               cudaMemcpyDeviceToDevice, s));
        }
        settle(s);
    }
};

template <class T> T* dalloc(size_t n)
{
    T* p = nullptr;
    if (n == 0)
        n = 1;
    CK(cudaMalloc(&p, n * sizeof(T)));
    return p;
}

template <class T, int D> struct Ctx : CtxBase {
    using C = Cfg<D>;
    DevScene<T, D> sc{};
    mpm_scene_desc desc{};
    cudaStream_t stream{};
    cudaStream_t own_stream{}; // stream may be a caller's (mpm_ctx_set_stream)
    // 3-D P2G: 2 warp-specialized (default), 1 pipe3, 0 lanes3 (experimental). MEASURED C4 (same
    // box, bench): f64 ws 0.410-0.414 ms vs pipe3 0.472 ms
    int p2g_impl = 2, p2g_lanes_per_sm = 1;
    int device = 0;
    int64_t cap = 0, n = 0;
    int64_t step = 0;
    double time = 0;
    bool has_aff = false, has_F = false;
    std::vector<void*> allocs;

    PBuf<T, D> buf[2]{};
    int cur = 0;
    int *keys = nullptr, *keys_sorted = nullptr, *perm = nullptr, *iota = nullptr;
    // K1 incremental sort (kernels_sort.cuh). The context's own sort arrays alternate with the
    // buffer parity (sorted keys and block ranges of step t are read while step t+1 writes the
    // other pair); the replay tape's sort sets are distinct arrays anyway.
    int *ks_own[2] = {}, *bs_own[2] = {}, *be_own[2] = {};
    bool own_set = true;
    IncSort inc{};
    // the order a particle buffer is stored in: base of the buffer the last G2P wrote and the
    // sort arrays of that step. Valid until the buffer's content changes any other way.
    struct IncSrc {
        const T* base;
        const int *ks, *bs, *be;
    } inc_src{};
    bool inc_enabled = !(std::getenv("MPM_SORT") && std::string(std::getenv("MPM_SORT")) == "cub");
    void inc_invalidate() { inc_src = IncSrc{}; }
    bool last_sort_full = true;
    // the stored order is a previous sort's (decomposed steps always sort incrementally: their
    // particle count is on the device, which the radix sort cannot take)
    bool inc_source_ok() const
    {
        return (inc_enabled || dist.on) && (!slab || dist.on) && inc_src.base == buf[cur].base && inc_src.ks;
    }
    void* cub_tmp = nullptr;
    size_t cub_bytes = 0;
    int *bstart = nullptr, *bend = nullptr, *lstart = nullptr, *occ = nullptr, *act = nullptr, *counts = nullptr; // counts[0]=n_occ, [1]=n_act
    unsigned char* nflag = nullptr;
    int* wq = nullptr; // [WQ_INTS]: occupancy-bucket histogram and cursors, work-counter pairs (kernels_util.cuh)
    int *d_nb = nullptr, *d_nnb = nullptr;
    T* partials = nullptr;
    GBuf<T, D> G{};
    DevStatus* st = nullptr;
    DevStatus* st_host = nullptr;
    Stage<T, D> stage{};
    T* stage_host = nullptr;
    size_t stage_elems = 0;
    unsigned long long* d_red = nullptr;
    bool keys_valid = false;
    bool grid_touched_all = false;
    int nsm = 148;
    int p2g_ctas_per_sm = 1;
    // occupied blocks listed heaviest first and taken through work counters (MPM_OCC_ORDER=index:
    // the plain compaction, for A/B)
    bool occ_lpt = !(std::getenv("MPM_OCC_ORDER") && std::getenv("MPM_OCC_ORDER")[0] == 'i');
    // 2-D P2G: the column-march kernel k_p2g (several CTAs' worth of warps per block) by default;
    // the staged variant (48 threads per block) is kept for A/B with MPM_P2G2D=staged. Measured
    // (C3, 102k particles): 25.7 vs 58.5 us; C2 (250k): 32 vs 72 us.
    bool p2g2d_generic = !(std::getenv("MPM_P2G2D") && std::getenv("MPM_P2G2D")[0] == 's');
    AdjWork<T, D> aw{};
    // slab decomposition (multi-GPU)
    bool slab = false;
    // library-owned decomposition (mpm_dist_*): device-resident counts, NCCL or same-process peers
    struct Dist {
        bool on = false;
        int rank = 0, nranks = 1, lo_peer = -1, hi_peer = -1;
        ncclComm_t comm = nullptr;
        cudaStream_t comm_stream = nullptr;
        cudaEvent_t ev_a = nullptr, ev_b = nullptr;
        int64_t halo_elems = 0;            // 2 node planes x NF values
        T* halo_send[2] = {nullptr, nullptr}; // [0] toward the lower neighbour, [1] the upper
        T* halo_recv[2] = {nullptr, nullptr};
        long long* cnt_send = nullptr;     // [2]
        long long* cnt_recv = nullptr;     // [2]
        T* recs_recv[2] = {nullptr, nullptr};
        int* pid_recv[2] = {nullptr, nullptr};
        int* d_n = nullptr;
        int* d_nlive = nullptr;
        int* abort_red = nullptr;          // [2]: [0] published (NCCL: reduced in place), [1] local max
        cudaGraphExec_t graph[2][2] = {}; // [guard][cur]
        int64_t graph_launches = 0;
        IncSrc graph_inc[2][2] = {};
    } dist;
    MigBuf<T> mig{};
    int64_t n_dead = 0;  // vacated slots (pid < 0) left in storage by the last G2P
    int* d_cells = nullptr;
    int mig_cnt[2] = {0, 0};

    IncSrc captured_inc_src{};
    cudaGraphExec_t graphs[2][2][2] = {}; // [guard][stores grad v][cur]
    IncSrc graph_inc[2][2][2] = {};       // the stored-order record a replay of each graph leaves
    int64_t graph_n[2][2][2] = {};        // particle count each forward graph was captured with
    // slab phases: P2G phase [cur] (valid for slab_g1_n[cur] particles), finish phase [guard][cur]
    cudaGraphExec_t slab_g1[2] = {nullptr, nullptr};
    int64_t slab_g1_n[2] = {-1, -1};
    int64_t slab_g1_launches = 0, slab_g2_launches = 0;
    cudaGraphExec_t slab_g2[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    bool status_dirty = true; // host step changed (upload): push it to the device counter
    bool has_state = false;   // a state was uploaded or seeded (it may hold no particles)
    void drop_slab_graphs()
    {
        for (auto& e : slab_g1)
            if (e) {
                cudaGraphExecDestroy(e);
                e = nullptr;
            }
        for (auto& g : slab_g2)
            for (auto& e : g)
                if (e) {
                    cudaGraphExecDestroy(e);
                    e = nullptr;
                }
        slab_g1_n[0] = slab_g1_n[1] = -1;
    }
    // capture f() on the stream into `out` (launch counter, buffer parity and key state restored)
    template <class F> int64_t capture(cudaGraphExec_t& out, F&& f)
    {
        const int cur0 = cur;
        const bool kv0 = keys_valid;
        const int64_t l0 = launches;
        const IncSrc inc0 = inc_src;
        const bool own0 = own_set;
        int* const ptr0[3] = {keys_sorted, bstart, bend};
        auto restore = [&] {
            launches = l0;
            cur = cur0;
            keys_valid = kv0;
            inc_src = inc0;
            own_set = own0;
            keys_sorted = ptr0[0];
            bstart = ptr0[1];
            bend = ptr0[2];
        };
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
        try {
            f();
        } catch (...) { // leave the stream out of capture mode and the context state as it was
            cudaStreamEndCapture(stream, &g);
            if (g)
                cudaGraphDestroy(g);
            (void)cudaGetLastError();
            restore();
            throw;
        }
        CK(cudaStreamEndCapture(stream, &g));
        captured_inc_src = inc_src; // what replaying the graph leaves behind
        struct GraphGuard {
            cudaGraph_t g;
            ~GraphGuard() { cudaGraphDestroy(g); }
        } guard_g{g};
        // an existing executable graph of the same phase (the slab P2G phase after the particle
        // count changed) is updated in place: same topology, new launch dimensions. A topology or
        // node-type change (cub's tile count moving a memset's size, say) falls back to instantiation.
        bool updated = false;
        if (out) {
            cudaGraphExecUpdateResultInfo info{};
            updated = cudaGraphExecUpdate(out, g, &info) == cudaSuccess;
            if (!updated) {
                (void)cudaGetLastError(); // cudaErrorGraphExecUpdateFailure is not sticky
                CK(cudaGraphExecDestroy(out));
                out = nullptr;
            }
        }
        if (!updated) {
            const cudaError_t ie = cudaGraphInstantiate(&out, g, 0);
            if (ie != cudaSuccess) {
                out = nullptr;
                restore();
                CK(ie);
            }
        }
        const int64_t k = launches - l0;
        restore();
        return k;
    }

    template <class X> X* alloc(size_t k)
    {
        X* p = dalloc<X>(k);
        allocs.push_back(p);
        return p;
    }

    Ctx(const mpm_scene_desc* d, int64_t max_particles, int dev)
    {
        desc = *d;
        device = dev;
        CK(cudaSetDevice(dev));
        cudaDeviceProp prop{};
        CK(cudaGetDeviceProperties(&prop, dev));
        if (prop.major < 10)
            throw ApiError(MPM_ERR_CUDA, "libmpm_b200 requires an sm_100 (Blackwell) device; found " + std::string(prop.name));
        nsm = prop.multiProcessorCount;
        CK(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking));
        stream = own_stream;
        build_scene(d);
        cap = std::max<int64_t>(max_particles, 1); // an empty state still gets valid (1-slot) buffers
        has_aff = d->scheme == MPM_SCHEME_APIC;
        has_F = d->track_def_grad != 0;
        for (int b = 0; b < 2; ++b)
            alloc_pbuf(buf[b]);
        keys = alloc<int>(cap);
        for (int k = 0; k < 2; ++k) {
            ks_own[k] = alloc<int>(cap);
            bs_own[k] = alloc<int>(sc.nb_total);
            be_own[k] = alloc<int>(sc.nb_total);
        }
        keys_sorted = ks_own[0];
        inc.cnt_in = alloc<int>(sc.nb_total);
        inc.cnt_out = alloc<int>(sc.nb_total);
        inc.in_off = alloc<int>(sc.nb_total);
        inc.xlist = alloc<int>(cap);
        inc.inbuf = alloc<int>(cap);
        inc.nx = alloc<int>(1);
        inc.nlive = alloc<int>(1);
        inc.part = alloc<int>(3 * ((sc.nb_total + 255) / 256));
        inc.hist = alloc<int>(OCC_NBUCKET);
        inc.bcur = alloc<int>(OCC_NBUCKET);
        CK(cudaMemsetAsync(inc.hist, 0, sizeof(int) * OCC_NBUCKET, stream));
        CK(cudaMemsetAsync(inc.bcur, 0, sizeof(int) * OCC_NBUCKET, stream));
        CK(cudaMemsetAsync(inc.cnt_in, 0, sizeof(int) * sc.nb_total, stream));
        CK(cudaMemsetAsync(inc.cnt_out, 0, sizeof(int) * sc.nb_total, stream));
        CK(cudaMemsetAsync(inc.nx, 0, sizeof(int), stream));
        perm = alloc<int>(cap);
        iota = alloc<int>(cap);
        k_iota<<<unsigned((cap + 255) / 256), 256, 0, stream>>>(iota, int(cap));
        CK(cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, keys, keys_sorted, iota, perm, int(cap), 0, 32, stream));
        cub_tmp = alloc<unsigned char>(cub_bytes);
        bstart = bs_own[0];
        bend = be_own[0];
        lstart = alloc<int>((size_t)sc.nb_total * (C::B + 1));
        occ = alloc<int>(sc.nb_total);
        act = alloc<int>(sc.nnb_total);
        counts = alloc<int>(4);
        CK(cudaMemsetAsync(counts, 0, sizeof(int) * 4, stream));
        wq = alloc<int>(WQ_INTS);
        CK(cudaMemsetAsync(wq, 0, sizeof(int) * WQ_INTS, stream));
        nflag = alloc<unsigned char>(sc.nnb_total);
        d_nb = alloc<int>(D);
        d_nnb = alloc<int>(D);
        d_cells = alloc<int>(D);
        CK(cudaMemcpyAsync(d_cells, sc.cells, sizeof(int) * D, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(d_nb, sc.nb, sizeof(int) * D, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(d_nnb, sc.nnb, sizeof(int) * D, cudaMemcpyHostToDevice, stream));
        partials = alloc<T>((size_t)sc.nb_total * C::NF * C::TN);
        const size_t nodes = (size_t)sc.nnb_total * C::NB;
        G.m = alloc<T>(nodes);
        for (int a = 0; a < D; ++a) {
            G.p[a] = alloc<T>(nodes);
            G.f[a] = alloc<T>(nodes);
            G.v[a] = alloc<T>(nodes);
            G.vold[a] = alloc<T>(nodes);
        }
        zero_grid();
        st = alloc<DevStatus>(1);
        CK(cudaMallocHost(&st_host, sizeof(DevStatus)));
        reset_status();
        stage_elems = 0;
        for (int f = 0; f < S_NFIELDS; ++f)
            stage_elems += (size_t)cap * stage_comps<D>(f);
        T* sbase = alloc<T>(stage_elems);
        size_t off = 0;
        for (int f = 0; f < S_NFIELDS; ++f) {
            stage.f[f] = sbase + off;
            off += (size_t)cap * stage_comps<D>(f);
        }
        CK(cudaMallocHost(&stage_host, stage_elems * sizeof(T)));
        d_red = alloc<unsigned long long>(2);
        aw.init(*this);
        set_smem_attrs();
        CK(cudaStreamSynchronize(stream));
    }

    ~Ctx() override
    {
        for (auto& g : graphs)
            for (auto& h : g)
                for (auto& e : h)
                    if (e)
                        cudaGraphExecDestroy(e);
        drop_slab_graphs();
        for (auto& g : dist.graph)
            for (auto& e : g)
                if (e)
                    cudaGraphExecDestroy(e);
        if (dist.comm)
            dyn::ncclCommDestroy(dist.comm);
        if (dist.comm_stream)
            cudaStreamDestroy(dist.comm_stream);
        if (dist.ev_a)
            cudaEventDestroy(dist.ev_a);
        if (dist.ev_b)
            cudaEventDestroy(dist.ev_b);
        for (void* p : bp_pool_mem)
            cudaFree(p);
        tape_free();
        for (auto& e : events) {
            cudaEventDestroy(e.a);
            cudaEventDestroy(e.b);
        }
        aw.free_all();
        if (ids_scratch)
            cudaFree(ids_scratch);
        for (void* p : allocs)
            cudaFree(p);
        if (st_host)
            cudaFreeHost(st_host);
        if (stage_host)
            cudaFreeHost(stage_host);
        for (auto& q : snaps) {
            if (q.host)
                cudaFreeHost(q.host);
            if (q.gathered)
                cudaEventDestroy(q.gathered);
            if (q.ready)
                cudaEventDestroy(q.ready);
        }
        if (copy_stream)
            cudaStreamDestroy(copy_stream);
        if (own_stream)
            cudaStreamDestroy(own_stream);
    }

    void build_scene(const mpm_scene_desc* d)
    {
        if (d->dh <= 0 || d->dt <= 0)
            throw ApiError(MPM_ERR_VALIDATION, "config: grid spacing and time step must be positive");
        sc.dh = T(d->dh);
        sc.inv_dh = T(1) / sc.dh;
        sc.dt = T(d->dt);
        sc.alpha = d->scheme == MPM_SCHEME_FLIP ? T(1) : (d->scheme == MPM_SCHEME_BLEND ? T(d->alpha_flip) : T(0));
        for (int a = 0; a < D; ++a) {
            if (d->cells[a] < 5)
                throw ApiError(MPM_ERR_VALIDATION, "config: need at least 5 cells per axis");
            sc.cells[a] = d->cells[a];
            sc.origin[a] = T(d->origin[a]);
            sc.gravity[a] = T(d->gravity[a]);
            sc.nb[a] = (d->cells[a] - 1 + C::B - 1) / C::B;
            sc.nnb[a] = (d->cells[a] + 1 + C::B - 1) / C::B;
        }
        sc.slab_lo = 0;
        sc.slab_hi = d->cells[0];
        sc.band_lo = sc.band_hi = -(1 << 28); // no neighbours
        sc.nb_total = 1;
        sc.nnb_total = 1;
        for (int a = 0; a < D; ++a) {
            sc.nb_total *= sc.nb[a];
            sc.nnb_total *= sc.nnb[a];
        }
        if ((int64_t)sc.nb_total << C::LOGNB >= (int64_t(1) << 31) - 1)
            throw ApiError(MPM_ERR_VALIDATION, "grid too large for 32-bit cell keys");
        sc.scheme = d->scheme;
        sc.apic = d->scheme == MPM_SCHEME_APIC;
        sc.tpic = d->scheme == MPM_SCHEME_TPIC;
        sc.track_F = d->track_def_grad;
        sc.material = d->material;
        sc.rho0 = T(d->rho0);
        sc.visc = T(d->viscosity);
        sc.c = T(d->sound_speed);
        sc.rate_form = d->rate_form;
        sc.K = T(d->K);
        sc.G = T(d->G);
        sc.q_phi = T(d->q_phi);
        sc.k_phi = T(d->k_phi);
        sc.q_psi = T(d->q_psi);
        sc.tau_P = T(d->tau_P);
        sc.alpha_P = T(d->alpha_P);
        sc.sigma_t = T(d->sigma_t);
        sc.band = d->band_layers;
        int off = 0;
        for (int w = 0; w < 2 * D; ++w) {
            sc.wall_kind[w] = d->wall_kind[w];
            sc.n_fric[w] = d->n_friction[w];
            sc.fric_off[w] = off;
            if (d->wall_kind[w] == MPM_WALL_COULOMB && d->n_friction[w] < 1)
                throw ApiError(MPM_ERR_VALIDATION, "scene: coulomb wall needs at least one segment");
            for (int k = 0; k < d->n_friction[w]; ++k) {
                if (off >= MAX_FRIC)
                    throw ApiError(MPM_ERR_VALIDATION, "too many Coulomb friction segments (max 64 total)");
                sc.fric[off++] = T(d->friction[w][k]);
            }
        }
        if (d->n_obstacles > MAX_OBST)
            throw ApiError(MPM_ERR_VALIDATION, "too many obstacles (max 16)");
        sc.n_obst = d->n_obstacles;
        for (int o = 0; o < d->n_obstacles; ++o)
            for (int k = 0; k < 2 * D; ++k)
                sc.obst[o][k] = T(d->obstacles[o * 2 * D + k]);
        sc.mass_eps = T(d->mass_epsilon);
        // constitutive scene constants, evaluated by the device with the expressions they replace
        DevScene<T, D>* ds = nullptr;
        CK(cudaMalloc(&ds, sizeof(sc)));
        CK(cudaMemcpyAsync(ds, &sc, sizeof(sc), cudaMemcpyHostToDevice, stream));
        k_scene_consts<T, D><<<1, 1, 0, stream>>>(ds);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&sc, ds, sizeof(sc), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        CK(cudaFree(ds));
    }

    void alloc_pbuf(PBuf<T, D>& P)
    {
        using L = PLay<D>;
        const long long S = (cap + 63) / 64 * 64; // 512-byte aligned field stride
        const int nf = has_F ? L::END : (has_aff ? L::F : L::AFF);
        P.base = alloc<T>((size_t)S * nf);
        P.S = S;
        auto f = [&](int k) { return P.base + (size_t)k * S; };
        for (int a = 0; a < D; ++a) {
            P.x[a] = f(L::X + a);
            P.v[a] = f(L::V + a);
        }
        P.m = f(L::M);
        P.V = f(L::VOL);
        P.rho = f(L::RHO);
        P.eps = f(L::EPS);
        P.szz = D == 2 ? f(L::SZZ) : nullptr;
        for (int s = 0; s < C::NS; ++s)
            P.sig[s] = f(L::SIG + s);
        for (int k = 0; k < D * D; ++k) {
            P.gv[k] = f(L::GV + k);
            P.aff[k] = has_aff ? f(L::AFF + k) : nullptr;
            P.F[k] = has_F ? f(L::F + k) : nullptr;
        }
        P.pid = alloc<int>(cap);
    }

    void zero_grid()
    {
        const size_t nodes = (size_t)sc.nnb_total * C::NB;
        CK(cudaMemsetAsync(G.m, 0, nodes * sizeof(T), stream));
        for (int a = 0; a < D; ++a) {
            CK(cudaMemsetAsync(G.p[a], 0, nodes * sizeof(T), stream));
            CK(cudaMemsetAsync(G.f[a], 0, nodes * sizeof(T), stream));
            CK(cudaMemsetAsync(G.v[a], 0, nodes * sizeof(T), stream));
            CK(cudaMemsetAsync(G.vold[a], 0, nodes * sizeof(T), stream));
        }
    }

    void reset_status()
    {
        k_reset_status<<<1, 1, 0, stream>>>(st, (long long)step); // no pageable host copy per step
        CK(cudaGetLastError());
    }

    // ---- kernel launch helpers ------------------------------------------------------------
    size_t g2p_smem(bool trackf) const
    {
        return trackf ? G2PStage<T, D, true>::SMEM : G2PStage<T, D, false>::SMEM;
    }

    void set_smem_attrs()
    {
        size_t sm = g2p_smem(true);
        auto set = [&](auto kern) { CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm))); };
        set(k_g2p<T, D, P_CONSTIT, false, false>);
#if G2P_ABL
        set(k_g2p<T, D, P_CONSTIT, false, false, G2P_ABL>);
        set(k_g2p<T, D, P_CONSTIT | P_GUARD, false, false, G2P_ABL>);
#endif
        set(k_g2p<T, D, P_CONSTIT | P_GUARD, false, false>);
        set(k_g2p<T, D, P_CONSTIT | P_NOGV, false, false>);
        set(k_g2p<T, D, P_CONSTIT | P_GUARD | P_NOGV, false, false>);
        set(k_g2p<T, D, P_CONSTIT, true, false>);
        set(k_g2p<T, D, P_CONSTIT | P_GUARD, true, false>);
        set(k_g2p<T, D, P_CONSTIT, false, true>);
        set(k_g2p<T, D, P_CONSTIT | P_GUARD, false, true>);
        set(k_g2p<T, D, P_CONSTIT, true, true>);
        set(k_g2p<T, D, P_CONSTIT | P_GUARD, true, true>);
        set(k_g2p<T, D, 0, false, false>);
        set(k_g2p<T, D, 0, true, false>);
        set(k_g2p<T, D, 0, false, true>);
        set(k_g2p<T, D, 0, true, true>);
        if constexpr (D == 3) {
            CK(cudaFuncSetAttribute(k_p2g_pipe3<T, P2G_WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(Pipe3Cfg<T, P2G_WIDE>::SMEM)));
#if P2G_ABL
            CK(cudaFuncSetAttribute(k_p2g_pipe3<T, P2G_WIDE, P2G_ABL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(Pipe3Cfg<T, P2G_WIDE>::SMEM)));
#endif
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p2g_ctas_per_sm, k_p2g_pipe3<T, P2G_WIDE>,
                                                             Pipe3Cfg<T, P2G_WIDE>::THREADS, Pipe3Cfg<T, P2G_WIDE>::SMEM));
            CK(cudaFuncSetAttribute(k_p2g_lanes3<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(Lane3Cfg<T>::SMEM)));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p2g_lanes_per_sm, k_p2g_lanes3<T>, Lane3Cfg<T>::THREADS,
                                                             Lane3Cfg<T>::SMEM));
            if (p2g_lanes_per_sm < 1)
                p2g_lanes_per_sm = 1;
            CK(cudaFuncSetAttribute(k_p2g_ws<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(WsCfg<T>::SMEM)));
#if P2G_ABL == 64
            CK(cudaFuncSetAttribute(k_p2g_ws<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(WsCfg<T>::SMEM)));
#endif
            if (const char* e = std::getenv("MPM_P2G_IMPL")) // A/B measurement only
                p2g_impl = std::string(e) == "lanes3" ? 0 : std::string(e) == "pipe3" ? 1 : 2;
        } else {
            CK(cudaFuncSetAttribute(k_p2g<T, D, false, D == 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(p2g2_smem<T>())));
            CK(cudaFuncSetAttribute(k_p2g_staged<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(StageCfg<T, D>::SMEM)));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p2g_ctas_per_sm, k_p2g_staged<T, D>, StageCfg<T, D>::THREADS,
                                                             StageCfg<T, D>::SMEM));
        }
        if (p2g_ctas_per_sm < 1)
            p2g_ctas_per_sm = 1;
        aw.set_attrs(*this);
    }

    template <class F> void launch(const char* name, F&& f)
    {
        ++launches;
        if (prof) {
            ProfEvent e{name, nullptr, nullptr};
            CK(cudaEventCreate(&e.a));
            CK(cudaEventCreate(&e.b));
            CK(cudaEventRecord(e.a, stream));
            f();
            CK(cudaEventRecord(e.b, stream));
            events.push_back(e);
        } else {
            f();
        }
        CK(cudaGetLastError());
    }

    // programmatic dependent launch of the step's kernels (common.cuh pdl_wait), MPM_PDL=1. It lets
    // a kernel be scheduled while its predecessor drains. MEASURED (graph-replayed steps, on vs off):
    // C4 898 vs 883 us, C3 45.7 vs 43.5 us, C2 48.6 vs 50.1 us -- no gain, so it is off by default.
    bool use_pdl = std::getenv("MPM_PDL") && std::getenv("MPM_PDL")[0] == '1';
    template <class... KArgs> struct PdlLaunch {
        void (*k)(KArgs...);
        dim3 g, b;
        size_t smem;
        cudaStream_t s;
        bool on;
        template <class... A> void operator()(A&&... a) const
        {
            if (!on) {
                k<<<g, b, smem, s>>>(std::forward<A>(a)...);
                return;
            }
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = g;
            cfg.blockDim = b;
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaLaunchAttribute at{};
            at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at.val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = &at;
            cfg.numAttrs = 1;
            CK(cudaLaunchKernelEx(&cfg, k, std::forward<A>(a)...));
        }
    };
    template <class... KArgs> PdlLaunch<KArgs...> pdl(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem)
    {
        return {k, g, b, smem, stream, use_pdl};
    }

    // a kernel's work-counter pair when the occupied-block list is heaviest-first (3-D), else
    // nullptr: the static CTA stride. MEASURED (C4 f64): G2P 0.410 -> 0.352 ms, step 1.102 -> 1.030 ms;
    // in 2-D (C2/C3: small blocks, latency-bound steps) the extra list pass cost 5-7 us per step.
    int* wq_ptr(int pair) const { return (occ_lpt && D == 3) ? wq + pair : nullptr; }

    unsigned grid_for(int64_t k, int tpb) const { return k > 0 ? unsigned((k + tpb - 1) / tpb) : 1u; } // n may be 0 on a slab
    unsigned persistent(int per_sm) const { return unsigned(nsm * per_sm); }

    // ---- sort + segment tables ---------------------------------------------------------------
    void sort_and_segment()
    {
        if (own_set) { // the pair the previous step did not write (host-orchestrated slab steps: pair 0)
            const int k = (slab && !dist.on) ? 0 : cur;
            keys_sorted = ks_own[k];
            bstart = bs_own[k];
            bend = be_own[k];
        }
        if (!keys_valid) {
            launch("k_keys", [&] { k_keys<T, D><<<grid_for(n, 256), 256, 0, stream>>>(sc, buf[cur], int(n), keys, st); });
            keys_valid = true;
        }
        // K1: the stored order is the previous step's sort -> rebuild it incrementally
        const bool inc_ok = inc_source_ok() && (n > 0 || dist.on) && inc_src.ks != keys_sorted &&
                            inc_src.bs != bstart && inc_src.be != bend;
        last_sort_full = !inc_ok;
        if (inc_ok) {
            const IncSrc o = inc_src;
            IncSort is = inc;
            is.d_n = dist.on ? dist.d_n : nullptr; // decomposed steps: the count lives on the device
            is.nflag = nflag;
            is.nnb_total = sc.nnb_total;
            is.nb = d_nb;
            is.nnb = d_nnb;
            is.act = act;
            is.counts = counts;
            const int64_t nthr = dist.on ? cap : n;
            launch("k_sort_classify", [&] {
                pdl(k_inc_classify<D>, grid_for((nthr + 3) / 4, 256), 256, 0)(keys, o.ks, int(n), sc.nb_total, is);
            });
            const bool lpt = occ_lpt && D == 3;
            const unsigned nbc = unsigned((sc.nb_total + 255) / 256);
            launch("k_sort_count", [&] {
                pdl(k_inc_count<D>, nbc, 256, 0)(sc.nb_total, o.bs, o.be, is, bend);
            });
            launch("k_sort_offsets", [&] {
                if (lpt)
                    pdl(k_inc_offsets<D, true>, nbc, 256, 0)(sc.nb_total, is, bstart, bend, occ, counts);
                else
                    pdl(k_inc_offsets<D, false>, nbc, 256, 0)(sc.nb_total, is, bstart, bend, occ, counts);
            });
            launch("k_sort_place", [&] { pdl(k_inc_place<D>, nsm, 256, 0)(keys, is, nsm * 256); });
            launch("k_sort_block", [&] {
                pdl(k_inc_block<D>, persistent(8), INC_THREADS, 0)(keys, o.ks, o.bs, o.be, is, bstart, bend,
                                                                          occ, counts, perm, keys_sorted, lstart);
            });
        } else {
            // radix-sort only the bits a valid key can have (C4: 24 bits -> 3 onesweep passes). An
            // out-of-domain particle's sentinel key aliases in those bits, but such a step is aborted.
            int end_bit = 1;
            const int64_t need = (int64_t(sc.nb_total) << C::LOGNB) + (slab ? 2 : 0); // dead keys sort last
            while ((int64_t(1) << end_bit) < need)
                ++end_bit;
            size_t bytes = cub_bytes;
            CK(cub::DeviceRadixSort::SortPairs(cub_tmp, bytes, keys, keys_sorted, iota, perm, int(n), 0, end_bit, stream));
            CK(cudaMemsetAsync(bstart, 0xff, sizeof(int) * sc.nb_total, stream));
            CK(cudaMemsetAsync(bend, 0xff, sizeof(int) * sc.nb_total, stream));
            CK(cudaMemsetAsync(lstart, 0xff, sizeof(int) * sc.nb_total * (C::B + 1), stream));
            CK(cudaMemsetAsync(counts, 0, sizeof(int) * 4, stream));
            CK(cudaMemsetAsync(nflag, 0, sc.nnb_total, stream));
            launch("k_seg", [&] { k_seg4<D><<<grid_for((n + 3) / 4, 256), 256, 0, stream>>>(keys_sorted, int(n), sc.nb_total, bstart, bend, lstart); });
            if (occ_lpt && D == 3) { // heaviest blocks first (kernels_util.cuh)
                CK(cudaMemsetAsync(wq, 0, sizeof(int) * WQ_CTR, stream));
                launch("k_occ", [&] { k_occ_hist<<<grid_for(sc.nb_total, 256), 256, 0, stream>>>(bstart, bend, sc.nb_total, wq); });
                launch("k_occ", [&] { k_occ_scatter<<<grid_for(sc.nb_total, 256), 256, 0, stream>>>(bstart, bend, sc.nb_total, wq, occ, counts); });
            } else {
                launch("k_compact", [&] { k_compact_pos<<<grid_for(sc.nb_total, 256), 256, 0, stream>>>(bstart, sc.nb_total, occ, counts); });
            }
        }
        if (!inc_ok) { // (the incremental sort's kernels mark and list the node blocks themselves)
            launch("k_mark_nodes", [&] { k_mark_nodes<D><<<grid_for(sc.nb_total, 128), 128, 0, stream>>>(occ, counts, d_nb, d_nnb, nflag); });
            launch("k_compact", [&] { k_compact_flag<<<grid_for(sc.nnb_total, 256), 256, 0, stream>>>(nflag, sc.nnb_total, act, counts + 1); });
        }
    }

    void p2g_kernel()
    {
        if (sc.apic || sc.tpic) {
            const int tpb = D == 2 ? 160 : 256;
            launch("k_p2g", [&] {
                pdl(k_p2g<T, D, true>, persistent(8), tpb, 0)(sc, buf[cur], perm, keys_sorted, bstart, bend, occ,
                                                                     counts, partials, st);
            });
        } else {
            if constexpr (D == 3) {
                if (p2g_impl == 2) {
                    using S = WsCfg<T>;
#if P2G_ABL == 64
                    launch("k_p2g_abl", [&] {
                        pdl(k_p2g_ws<T, true>, unsigned(nsm), S::THREADS, S::SMEM)(sc, buf[cur], perm, keys_sorted, bstart,
                                                                                   bend, lstart, occ, counts, partials,
                                                                                   st, wq_ptr(WQ_P2G));
                    });
#endif
                    launch("k_p2g", [&] {
                        pdl(k_p2g_ws<T>, unsigned(nsm), S::THREADS, S::SMEM)(sc, buf[cur], perm, keys_sorted, bstart,
                                                                             bend, lstart, occ, counts, partials, st,
                                                                             wq_ptr(WQ_P2G));
                    });
                } else if (p2g_impl == 1) {
                    using S = Pipe3Cfg<T, P2G_WIDE>;
#if P2G_ABL == 16
                    launch("k_p2g_abl", [&] { pdl(k_spin_abl, nsm, 32, 0)(600000); });
#elif P2G_ABL
                    launch("k_p2g_abl", [&] {
                        pdl(k_p2g_pipe3<T, P2G_WIDE, P2G_ABL>, unsigned(nsm * p2g_ctas_per_sm), S::THREADS, S::SMEM)(
                            sc, buf[cur], perm, keys_sorted, bstart, bend, lstart, occ, counts, partials, st, wq_ptr(WQ_P2G));
                    });
#endif
                    launch("k_p2g", [&] {
                        pdl(k_p2g_pipe3<T, P2G_WIDE>, unsigned(nsm * p2g_ctas_per_sm), S::THREADS, S::SMEM)(
                            sc, buf[cur], perm, keys_sorted, bstart, bend, lstart, occ, counts, partials, st, wq_ptr(WQ_P2G));
                    });
                } else {
                    using S = Lane3Cfg<T>;
                    launch("k_p2g", [&] {
                        pdl(k_p2g_lanes3<T>, unsigned(nsm * p2g_lanes_per_sm), S::THREADS, S::SMEM)(
                            sc, buf[cur], perm, keys_sorted, bstart, bend, lstart, occ, counts, partials, st);
                    });
                }
            } else if (p2g2d_generic) {
                launch("k_p2g", [&] {
                    if constexpr (D == 2)
                        pdl(k_p2g<T, D, false, true>, persistent(2), 160, p2g2_smem<T>())(
                            sc, buf[cur], perm, keys_sorted, bstart, bend, occ, counts, partials, st);
                    else
                        pdl(k_p2g<T, D, false>, persistent(8), 160, 0)(sc, buf[cur], perm, keys_sorted, bstart,
                                                                              bend, occ, counts, partials, st);
                });
            } else {
                using S = StageCfg<T, D>;
                launch("k_p2g", [&] {
                    pdl(k_p2g_staged<T, D>, unsigned(nsm * p2g_ctas_per_sm), S::THREADS, S::SMEM)(
                        sc, buf[cur], perm, keys_sorted, bstart, bend, occ, counts, partials, st);
                });
            }
        }
    }

    template <int MODE> void grid_kernel()
    {
        launch("k_grid", [&] {
            pdl(k_grid<T, D, MODE>, persistent(4), C::NB, 0)(sc, G, partials, bstart, act, counts + 1, st);
        });
    }

    template <int FL> void g2p_kernel_fl()
    {
        auto& Pin = buf[cur];
        auto& Pout = buf[cur ^ 1];
        const size_t sm = g2p_smem(has_F);
        const unsigned gr = persistent(D == 2 ? 8 : 4);
        if constexpr ((FL & P_NOGV) != 0) { // requested only without affine / F state
            if (has_aff || has_F)
                throw ApiError(MPM_ERR_USAGE, "internal: P_NOGV with affine or F state");
            launch("k_g2p", [&] { pdl(k_g2p<T, D, FL, false, false>, gr, 256, sm)(sc, Pin, Pout, G, perm, bstart, bend, occ, counts, keys, st, mig, wq_ptr(WQ_G2P)); });
        } else if (has_aff && has_F)
            launch("k_g2p", [&] { pdl(k_g2p<T, D, FL, true, true>, gr, 256, sm)(sc, Pin, Pout, G, perm, bstart, bend, occ, counts, keys, st, mig, wq_ptr(WQ_G2P)); });
        else if (has_aff)
            launch("k_g2p", [&] { pdl(k_g2p<T, D, FL, true, false>, gr, 256, sm)(sc, Pin, Pout, G, perm, bstart, bend, occ, counts, keys, st, mig, wq_ptr(WQ_G2P)); });
        else if (has_F)
            launch("k_g2p", [&] { pdl(k_g2p<T, D, FL, false, true>, gr, 256, sm)(sc, Pin, Pout, G, perm, bstart, bend, occ, counts, keys, st, mig, wq_ptr(WQ_G2P)); });
        else {
#if G2P_ABL
            launch("k_g2p_abl", [&] { pdl(k_g2p<T, D, FL, false, false, G2P_ABL>, gr, 256, sm)(sc, Pin, Pout, G, perm, bstart, bend, occ, counts, keys, st, mig, wq_ptr(WQ_G2P)); });
#endif
            launch("k_g2p", [&] { pdl(k_g2p<T, D, FL, false, false>, gr, 256, sm)(sc, Pin, Pout, G, perm, bstart, bend, occ, counts, keys, st, mig, wq_ptr(WQ_G2P)); });
        }
        inc_src = (slab && !dist.on) ? IncSrc{} : IncSrc{Pout.base, keys_sorted, bstart, bend};
        cur ^= 1;
        keys_valid = true;
    }

    // grad v is dead state between the steps of one advance() call unless the scheme reads it
    // (APIC's B lives in its own field; TPIC's affine matrix is grad v) or F is tracked
    bool gv_skippable() const { return !has_aff && !has_F && !sc.tpic; }

    void step_once(bool guard, bool store = false, bool gv = true)
    {
        sort_and_segment();
        p2g_kernel();
        if (store)
            grid_kernel<G_SUM | G_MOM | G_CORR | G_STORE>();
        else
            grid_kernel<G_SUM | G_MOM | G_CORR>();
        const bool nogv = !gv && gv_skippable();
        if (guard)
            nogv ? g2p_kernel_fl<P_CONSTIT | P_GUARD | P_NOGV>() : g2p_kernel_fl<P_CONSTIT | P_GUARD>();
        else
            nogv ? g2p_kernel_fl<P_CONSTIT | P_NOGV>() : g2p_kernel_fl<P_CONSTIT>();
        launch("k_step_end", [&] { pdl(k_step_end, 1, 1, 0)(st); });
    }

    // ---- status ------------------------------------------------------------------------------
    void fetch_status()
    {
        CK(cudaMemcpyAsync(st_host, st, sizeof(DevStatus), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
    }

    // raise the reference's exception for whatever the device flagged
    void check_status(int64_t step_before)
    {
        fetch_status();
        DevStatus s = *st_host;
        step = s.step;
        time = double(T(step) * sc.dt);
        if (!s.abort)
            return;
        reset_status();
        inc_invalidate();
        if (s.den_flag)
            throw ApiError(MPM_ERR_NUMERICAL, "update: 1 + tr(dd) <= 0, time step too large for the compression rate",
                           s.den_pid, s.step + 1);
        if (s.nan_flag) {
            step = s.step + 1; // the step completed, then the guard fired (stepper.hpp:106-109)
            time = double(T(step) * sc.dt);
            throw ApiError(MPM_ERR_NUMERICAL, "run: non-finite particle field detected at step " + std::to_string(step),
                           -1, step);
        }
        if (s.ood_flag) {
            // keys of step s.step+1's output -> the state after that step is complete; the
            // next P2G is where the reference throws (bspline.hpp:86-91)
            throw ApiError(MPM_ERR_OUT_OF_DOMAIN,
                           "particle " + std::to_string(s.ood_pid) + " outside valid grid interior", s.ood_pid,
                           s.step + 1);
        }
        if (s.far_flag)
            throw ApiError(MPM_ERR_NUMERICAL, "P2G: a particle block exceeds the staging capacity (extreme compression)",
                           -1, s.step + 1);
        if (s.mig_over)
            throw ApiError(MPM_ERR_CUDA, "slab migration buffer overflow (raise mig_cap)", -1, s.step + 1);
        if (s.pad2)
            throw ApiError(MPM_ERR_NUMERICAL, "slab: another rank aborted step " + std::to_string(s.step + 1), -1,
                           s.step + 1);
        throw ApiError(MPM_ERR_NUMERICAL, "device step aborted", -1, s.step);
    }

    // ---- API ----------------------------------------------------------------------------------
    void upload(const mpm_state_view* s) override { upload_ids(s, nullptr); }

    void upload_ids(const mpm_state_view* s, const int64_t* ids) override
    {
        inc_invalidate();
        if (s->n < 0 || s->n > cap) // an empty state is valid (the reference steps it; a slab may be empty)
            throw ApiError(MPM_ERR_USAGE, "state size " + std::to_string(s->n) + " outside [1, " + std::to_string(cap) + "]");
        if (s->n > 0 && (!s->x || !s->v || !s->mass || !s->volume || !s->rho || !s->sigma))
            throw ApiError(MPM_ERR_USAGE, "state view missing required fields");
        if (has_aff && !s->affine)
            throw ApiError(MPM_ERR_USAGE, "APIC scheme needs the affine field");
        const int64_t n_prev = n;
        n = s->n;
        const void* src[S_NFIELDS] = {s->x, s->v, s->mass, s->volume, s->rho, s->eps_eq, D == 2 ? s->sigma_zz : nullptr,
                                      s->sigma, s->grad_v, s->affine, s->def_grad};
        for (int f = 0; f < S_NFIELDS; ++f) {
            size_t bytes = (size_t)n * stage_comps<D>(f) * sizeof(T);
            if (src[f])
                CK(cudaMemcpyAsync(stage.f[f], src[f], bytes, cudaMemcpyHostToDevice, stream));
            else if (f == S_EPS || f == S_GV || f == S_SZZ)
                CK(cudaMemsetAsync(stage.f[f], 0, bytes, stream));
            else if (f == S_F && has_F)
                throw ApiError(MPM_ERR_USAGE, "track_def_grad needs the def_grad field");
        }
        long long* d_ids = nullptr;
        if (ids) {
            d_ids = reinterpret_cast<long long*>(aw_ids_scratch(n));
            CK(cudaMemcpyAsync(d_ids, ids, n * sizeof(long long), cudaMemcpyHostToDevice, stream));
        }
        // symmetric stress contract (packed storage): reject genuinely non-symmetric input before
        // the particle buffers change, checked on the device copy (no host pass over the state)
        if (n > 0) {
            int* d_bad = reinterpret_cast<int*>(d_red); // scratch; the digest / max-speed reductions reset it
            const int big = 0x7fffffff;
            CK(cudaMemcpyAsync(d_bad, &big, sizeof(int), cudaMemcpyHostToDevice, stream));
            launch("k_check_sym", [&] {
                k_check_sym<T, D><<<grid_for(n, 256), 256, 0, stream>>>(stage.f[S_SIG], int(n), d_bad);
            });
            int bad = big;
            CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            if (bad != big) {
                n = n_prev;
                throw ApiError(MPM_ERR_VALIDATION, "stress of particle " + std::to_string(bad) + " is not symmetric", bad);
            }
        }
        launch("k_upload", [&] {
            k_upload<T, D><<<grid_for(n, 256), 256, 0, stream>>>(stage, buf[cur], int(n), D == 2 && s->sigma_zz != nullptr,
                                                                 has_aff, has_F, d_ids);
        });
        n_dead = 0;
        status_dirty = true;
        has_state = true;
        step = s->step;
        time = s->time;
        keys_valid = false;
        reset_status();
        CK(cudaStreamSynchronize(stream));
    }

    void download(mpm_state_view* s) override
    {
        if (slab)
            throw ApiError(MPM_ERR_USAGE, "slab mode: use mpm_state_download_local");
        if (!has_state)
            throw ApiError(MPM_ERR_USAGE, "no state uploaded");
        launch("k_download", [&] { k_download<T, D><<<grid_for(n, 256), 256, 0, stream>>>(stage, buf[cur], int(n), has_aff, has_F); });
        void* dst[S_NFIELDS] = {s->x, s->v, s->mass, s->volume, s->rho, s->eps_eq, D == 2 ? s->sigma_zz : nullptr,
                                s->sigma, s->grad_v, has_aff ? s->affine : nullptr, has_F ? s->def_grad : nullptr};
        for (int f = 0; f < S_NFIELDS; ++f)
            if (dst[f])
                CK(cudaMemcpyAsync(dst[f], stage.f[f], (size_t)n * stage_comps<D>(f) * sizeof(T),
                                   cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        s->n = n;
        s->step = step;
        s->time = time;
    }

    // ---- asynchronous snapshots (run's snapshot policy, stepper.hpp:112-117) -----
    struct Snap {
        Stage<T, D> dev{};
        T* dbase = nullptr;
        T* host = nullptr;
        cudaEvent_t gathered{}, ready{};
        int64_t n = 0, step = 0;
        double time = 0;
        bool pending = false;
    };
    Snap snaps[2];
    cudaStream_t copy_stream{};
    void snapshot_begin(int slot) override
    {
        if (slot < 0 || slot > 1)
            throw ApiError(MPM_ERR_USAGE, "snapshot slot must be 0 or 1");
        if (slab || !has_state)
            throw ApiError(MPM_ERR_USAGE, "snapshot: no single-context state");
        Snap& q = snaps[slot];
        if (!q.dbase) {
            q.dbase = alloc<T>(stage_elems);
            size_t off = 0;
            for (int f = 0; f < S_NFIELDS; ++f) {
                q.dev.f[f] = q.dbase + off;
                off += (size_t)cap * stage_comps<D>(f);
            }
            CK(cudaMallocHost(&q.host, stage_elems * sizeof(T)));
            CK(cudaEventCreateWithFlags(&q.gathered, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&q.ready, cudaEventDisableTiming));
            if (!copy_stream)
                CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
        }
        if (q.pending) // the previous snapshot in this slot must have left the staging buffer
            CK(cudaEventSynchronize(q.ready));
        // id-order gather on the compute stream (reads the current buffer before a later step
        // overwrites it), the D2H copy on the copy stream, overlapping the following steps
        launch("k_download", [&] { k_download<T, D><<<grid_for(n, 256), 256, 0, stream>>>(q.dev, buf[cur], int(n), has_aff, has_F); });
        CK(cudaEventRecord(q.gathered, stream));
        CK(cudaStreamWaitEvent(copy_stream, q.gathered, 0));
        size_t off = 0;
        for (int f = 0; f < S_NFIELDS; ++f) {
            const size_t len = (size_t)n * stage_comps<D>(f);
            CK(cudaMemcpyAsync(q.host + off, q.dev.f[f], len * sizeof(T), cudaMemcpyDeviceToHost, copy_stream));
            off += (size_t)cap * stage_comps<D>(f);
        }
        CK(cudaEventRecord(q.ready, copy_stream));
        q.n = n;
        q.step = step;
        q.time = time;
        q.pending = true;
    }
    void snapshot_fetch(int slot, mpm_state_view* s) override
    {
        if (slot < 0 || slot > 1 || !snaps[slot].pending)
            throw ApiError(MPM_ERR_USAGE, "snapshot_fetch: no snapshot in that slot");
        Snap& q = snaps[slot];
        CK(cudaEventSynchronize(q.ready));
        void* dst[S_NFIELDS] = {s->x, s->v, s->mass, s->volume, s->rho, s->eps_eq, D == 2 ? s->sigma_zz : nullptr,
                                s->sigma, s->grad_v, has_aff ? s->affine : nullptr, has_F ? s->def_grad : nullptr};
        size_t off = 0;
        for (int f = 0; f < S_NFIELDS; ++f) {
            const size_t len = (size_t)q.n * stage_comps<D>(f);
            if (dst[f])
                std::memcpy(dst[f], q.host + off, len * sizeof(T));
            off += (size_t)cap * stage_comps<D>(f);
        }
        s->n = q.n;
        s->step = q.step;
        s->time = q.time;
        q.pending = false;
    }

    uint64_t digest() override
    {
        CK(cudaMemsetAsync(d_red, 0, sizeof(unsigned long long), stream));
        launch("k_digest", [&] { k_digest<T, D><<<grid_for(n, 256), 256, 0, stream>>>(buf[cur], int(n), has_aff, d_red); });
        unsigned long long h = 0;
        CK(cudaMemcpyAsync(&h, d_red, sizeof(h), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        return h ^ (uint64_t)step * 0x9e3779b97f4a7c15ull;
    }

    double max_speed() override
    {
        CK(cudaMemsetAsync(d_red + 1, 0, sizeof(unsigned long long), stream));
        launch("k_max_speed", [&] { k_max_speed<T, D><<<grid_for(n, 256), 256, 0, stream>>>(buf[cur], int(n), d_red + 1); });
        unsigned long long h = 0;
        CK(cudaMemcpyAsync(&h, d_red + 1, sizeof(h), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        double v;
        std::memcpy(&v, &h, sizeof(v));
        return v;
    }

    void advance(int64_t nsteps, uint32_t flags) override
    {
        if (!has_state)
            throw ApiError(MPM_ERR_USAGE, "no state uploaded");
        if (nsteps <= 0)
            return;
        const int64_t step0 = step;
        advance_enqueue(nsteps, flags);
        check_status(step0);
    }

    void advance_enqueue(int64_t nsteps, uint32_t flags)
    {
        if (slab)
            throw ApiError(MPM_ERR_USAGE, "slab mode: step with mpm_step_p2g_local / mpm_halo / mpm_step_finish_local");
        if (!has_state)
            throw ApiError(MPM_ERR_USAGE, "no state uploaded");
        if (nsteps <= 0)
            return;
        const bool guard = flags & MPM_ADV_NAN_GUARD;
        const bool store = flags & MPM_ADV_STORE_GRID;
        reset_status();
        // only the call's last step stores grad v (the state a download, snapshot or the next
        // call sees); the steps before it skip the dead 9-value write when gv_skippable()
        if (prof || store) {
            for (int64_t k = 0; k < nsteps; ++k)
                step_once(guard, store, k == nsteps - 1);
        } else {
            // first step runs eagerly (computes keys if needed); the rest replay a captured graph
            step_once(guard, false, nsteps == 1);
            for (int64_t k = 1; k < nsteps; ++k) {
                const int gv = k == nsteps - 1 ? 1 : 0;
                cudaGraphExec_t& ge = graphs[guard][gv][cur];
                // a graph bakes in the particle count it was captured with (sort sizes, grids):
                // recapture after an upload / init_scene changed n
                if (!ge || graph_n[guard][gv][cur] != n) { // (updated in place when only sizes moved)
                    graph_launches = capture(ge, [&] { step_once(guard, false, gv); });
                    graph_n[guard][gv][cur] = n;
                    graph_inc[guard][gv][cur] = captured_inc_src;
                }
                CK(cudaGraphLaunch(graphs[guard][gv][cur], stream));
                launches += graph_launches;
                inc_src = graph_inc[guard][gv][cur];
                keys_sorted = ks_own[cur]; // the pair the replayed step wrote (own set: advance)
                bstart = bs_own[cur];
                bend = be_own[cur];
                cur ^= 1;
            }
        }
    }
    int64_t graph_launches = 0;

    double advance_timed(int64_t nsteps, uint32_t flags) override
    {
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        CK(cudaEventRecord(a, stream));
        advance_enqueue(nsteps, flags);
        CK(cudaEventRecord(b, stream));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        check_status(step);
        return ms;
    }

    // ---- phase functions (per-phase parity with the reference free functions) ---------------
    void phase_p2g() override
    {
        reset_status();
        sort_and_segment();
        p2g_kernel();
        zero_grid(); // Grid::reset (state.hpp:154-161)
        grid_kernel<G_SUM | G_STORE>();
        grid_touched_all = false;
        check_status(step);
    }
    void activate_all_node_blocks()
    {
        // phases applied to an uploaded grid act on every node (contact.hpp:83-96)
        CK(cudaMemsetAsync(nflag, 1, sc.nnb_total, stream));
        CK(cudaMemsetAsync(counts + 1, 0, sizeof(int), stream));
        launch("k_compact", [&] { k_compact_flag<<<grid_for(sc.nnb_total, 256), 256, 0, stream>>>(nflag, sc.nnb_total, act, counts + 1); });
    }
    void phase_mom() override
    {
        reset_status();
        if (grid_touched_all)
            activate_all_node_blocks();
        grid_kernel<G_MOM | G_STORE>();
        check_status(step);
    }
    void phase_corr() override
    {
        reset_status();
        if (grid_touched_all)
            activate_all_node_blocks();
        grid_kernel<G_CORR | G_STORE>();
        check_status(step);
    }
    void phase_g2p() override
    {
        reset_status();
        sort_and_segment();
        g2p_kernel_fl<0>();
        fetch_status();
        if (st_host->abort && st_host->ood_flag == 2 && !st_host->den_flag && !st_host->nan_flag) {
            // g2p itself does not check the domain (transfer.hpp:92-121): the next p2g throws
            reset_status();
            keys_valid = false;
            return;
        }
        check_status(step);
    }
    void phase_constit() override
    {
        reset_status();
        launch("k_constitutive", [&] {
            if (has_F)
                k_constitutive<T, D, true><<<grid_for(n, 256), 256, 0, stream>>>(sc, buf[cur], int(n), st);
            else
                k_constitutive<T, D, false><<<grid_for(n, 256), 256, 0, stream>>>(sc, buf[cur], int(n), st);
        });
        fetch_status();
        if (st_host->den_flag) {
            int p = st_host->den_pid;
            reset_status();
            throw ApiError(MPM_ERR_NUMERICAL, "update: 1 + tr(dd) <= 0, time step too large for the compression rate", p);
        }
    }

    // dense (row-major node index) <-> node-block layout
    void grid_download(mpm_grid_view* g) override
    {
        const int64_t nn = num_nodes();
        std::vector<T> blk((size_t)sc.nnb_total * C::NB);
        // only node blocks active in the last grid phase hold current values (the rest is stale)
        std::vector<unsigned char> active(sc.nnb_total);
        CK(cudaMemcpyAsync(active.data(), nflag, sc.nnb_total, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        auto pull = [&](T* dptr, void* dst, int comps, int comp) {
            if (!dst)
                return;
            CK(cudaMemcpyAsync(blk.data(), dptr, blk.size() * sizeof(T), cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            T* out = static_cast<T*>(dst);
            for (int64_t i = 0; i < nn; ++i) {
                const size_t b = block_index(i);
                out[i * comps + comp] = active[b / C::NB] ? blk[b] : T(0);
            }
        };
        pull(G.m, g->mass, 1, 0);
        for (int a = 0; a < D; ++a) {
            pull(G.p[a], g->momentum, D, a);
            pull(G.vold[a], g->v_old, D, a);
            pull(G.v[a], g->v, D, a);
            pull(G.f[a], g->force, D, a);
        }
        g->num_nodes = nn;
    }
    void grid_upload(const mpm_grid_view* g) override
    {
        const int64_t nn = num_nodes();
        std::vector<T> blk((size_t)sc.nnb_total * C::NB);
        auto push = [&](T* dptr, const void* srcp, int comps, int comp) {
            std::fill(blk.begin(), blk.end(), T(0));
            if (srcp) {
                const T* in = static_cast<const T*>(srcp);
                for (int64_t i = 0; i < nn; ++i)
                    blk[block_index(i)] = in[i * comps + comp];
            }
            CK(cudaMemcpyAsync(dptr, blk.data(), blk.size() * sizeof(T), cudaMemcpyHostToDevice, stream));
            CK(cudaStreamSynchronize(stream));
        };
        push(G.m, g->mass, 1, 0);
        for (int a = 0; a < D; ++a) {
            push(G.p[a], g->momentum, D, a);
            push(G.vold[a], g->v_old, D, a);
            push(G.v[a], g->v, D, a);
            push(G.f[a], g->force, D, a);
        }
        grid_touched_all = true;
        activate_all_node_blocks();
        CK(cudaStreamSynchronize(stream));
    }
    int64_t num_nodes() const
    {
        int64_t r = 1;
        for (int a = 0; a < D; ++a)
            r *= sc.cells[a] + 1;
        return r;
    }
    size_t block_index(int64_t flat) const
    {
        int idx[D];
        for (int a = D - 1; a >= 0; --a) {
            idx[a] = int(flat % (sc.cells[a] + 1));
            flat /= (sc.cells[a] + 1);
        }
        size_t q = 0, loc = 0;
        for (int a = 0; a < D; ++a) {
            q = q * sc.nnb[a] + (idx[a] >> C::LOGB);
            loc = (loc << C::LOGB) | (idx[a] & (C::B - 1));
        }
        return q * C::NB + loc;
    }

    void grid_stats(int64_t* an, int64_t* ob, int64_t* anb) override
    {
        fetch_status();
        int cnt[4];
        CK(cudaMemcpyAsync(cnt, counts, sizeof(cnt), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        if (an)
            *an = int64_t(st_host->active_nodes);
        if (ob)
            *ob = cnt[0];
        if (anb)
            *anb = cnt[1];
    }

    // ---- slab decomposition (multi-GPU) --------------------------------------------
    int64_t local_count() const override { return n - n_dead; }
    void set_stream(void* s) override { stream = s ? static_cast<cudaStream_t>(s) : own_stream; }
    void migrate_counts(int64_t* lo, int64_t* hi) const override
    {
        *lo = mig_cnt[0];
        *hi = mig_cnt[1];
    }
    // ---- library-owned slab decomposition (kernels_dist.cuh) -----------------------
    // One decomposed step, all on the device (no host synchronisation):
    //   A  sort (incremental, device count) + P2G + band-only grid sum; pack both halo bands
    //   X1 halo exchange with the x-neighbours (NCCL on the communication stream, or device copies)
    //   B  interior grid pass while the bands travel; fixed-order import of the neighbours' bands
    //      (lower rank's partial first); band grid update; G2P (exports leavers); publish the
    //      export counts and the abort flag
    //   X2 migration messages (count + fixed-capacity records) and the abort max-reduction
    //   C  a peer's abort becomes this rank's; append the received migrants (particle-id order)
    int dist_device() const override { return device; }
    void dist_attach(int rank, int nranks, int lo, int hi, int64_t mig_cap, const void* nccl_id) override
    {
        if (nranks < 1 || rank < 0 || rank >= nranks)
            throw ApiError(MPM_ERR_USAGE, "dist: rank outside [0, nranks)");
        if (dist.on)
            throw ApiError(MPM_ERR_USAGE, "dist: context already attached");
        if (mig_cap < 1)
            throw ApiError(MPM_ERR_USAGE, "dist: migration capacity must be positive");
        slab_set(lo, hi, mig_cap);
        dist.on = true;
        dist.rank = rank;
        dist.nranks = nranks;
        dist.lo_peer = rank > 0 ? rank - 1 : -1;
        dist.hi_peer = rank + 1 < nranks ? rank + 1 : -1;
        int64_t plane = 1;
        for (int a = 1; a < D; ++a)
            plane *= sc.cells[a] + 1;
        dist.halo_elems = 2 * plane * C::NF;
        for (int k = 0; k < 2; ++k) {
            dist.halo_send[k] = alloc<T>(dist.halo_elems);
            dist.halo_recv[k] = alloc<T>(dist.halo_elems);
            dist.recs_recv[k] = alloc<T>((size_t)mig.cap * mig.rec);
            dist.pid_recv[k] = alloc<int>(mig.cap);
        }
        dist.cnt_send = alloc<long long>(2);
        dist.cnt_recv = alloc<long long>(2);
        dist.d_n = alloc<int>(1);
        dist.d_nlive = inc.nlive;
        dist.abort_red = alloc<int>(2);
        CK(cudaMemsetAsync(dist.abort_red, 0, 2 * sizeof(int), stream));
        CK(cudaMemsetAsync(dist.cnt_send, 0, 2 * sizeof(long long), stream));
        CK(cudaMemsetAsync(dist.cnt_recv, 0, 2 * sizeof(long long), stream));
        CK(cudaEventCreateWithFlags(&dist.ev_a, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&dist.ev_b, cudaEventDisableTiming));
        if (nccl_id) {
            CK(cudaStreamCreateWithFlags(&dist.comm_stream, cudaStreamNonBlocking));
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            CK(cudaSetDevice(device));
            NCK(dyn::ncclCommInitRank(&dist.comm, nranks, id, rank));
        }
        CK(cudaStreamSynchronize(stream));
    }
    void dist_step_begin()
    {
        const int ni = int(n);
        CK(cudaMemcpyAsync(dist.d_n, &ni, sizeof(int), cudaMemcpyHostToDevice, stream));
    }
    void dist_phase_a()
    {
        launch("k_dist", [&] { k_dist_step_begin<<<1, 1, 0, stream>>>(st); });
        sort_and_segment();
        if (last_sort_full) { // the radix sort path: the live count from the block tables
            CK(cudaMemsetAsync(dist.d_nlive, 0, sizeof(int), stream));
            launch("k_dist", [&] { k_dist_nlive<<<grid_for(sc.nb_total, 256), 256, 0, stream>>>(bend, sc.nb_total, dist.d_nlive); });
        }
        p2g_kernel();
        if (!dist_has_peers()) // one rank: the fused grid pass of the plain step
            return;
        grid_kernel<G_BANDONLY | G_SUM | G_NOGRAV | G_STORE>();
        if (dist.lo_peer >= 0)
            halo(sc.slab_lo, 2, dist.halo_send[0], 0);
        if (dist.hi_peer >= 0)
            halo(sc.slab_hi, 2, dist.halo_send[1], 0);
    }
    bool dist_has_peers() const { return dist.lo_peer >= 0 || dist.hi_peer >= 0; }
    bool dist_store = false; // keep m, p, f in the grid (a replay step whose grid goes to the tape)
    void dist_grid_interior()
    {
        if (dist_has_peers()) {
            if (dist_store)
                grid_kernel<G_INTERIOR | G_SUM | G_MOM | G_CORR | G_STORE>();
            else
                step_grid_interior();
        } else if (dist_store) {
            grid_kernel<G_SUM | G_MOM | G_CORR | G_STORE>();
        } else {
            grid_kernel<G_SUM | G_MOM | G_CORR>();
        }
    }
    void dist_phase_b(bool guard)
    {
        // (the interior pass ran while the bands were in flight)
        if (dist.lo_peer >= 0) // the lower rank's partial first: received + own
            halo(sc.slab_lo, 2, dist.halo_recv[0], 1);
        if (dist.hi_peer >= 0) // own (lower) + received
            halo(sc.slab_hi, 2, dist.halo_recv[1], 2);
        if (dist_has_peers()) {
            finish_phase(guard);
        } else {
            if (guard)
                g2p_kernel_fl<P_CONSTIT | P_GUARD>();
            else
                g2p_kernel_fl<P_CONSTIT>();
            launch("k_step_end", [&] { k_step_end<<<1, 1, 0, stream>>>(st); });
        }
        if (dist.nranks > 1)
            launch("k_dist", [&] {
                k_dist_publish<<<1, 1, 0, stream>>>(st, dist.cnt_send, dist.cnt_send + 1, dist.abort_red, mig.cap);
            });
    }
    void dist_phase_c(const int* reduced)
    {
        if (dist.nranks > 1)
            launch("k_dist", [&] { k_dist_merge_abort<<<1, 1, 0, stream>>>(st, reduced); });
        launch("k_dist", [&] {
            k_dist_import<T, D><<<grid_for(2 * int64_t(mig.cap), 256), 256, 0, stream>>>(
                sc, buf[cur], dist.d_nlive, dist.d_n, dist.cnt_recv, dist.recs_recv[0], dist.pid_recv[0],
                dist.cnt_recv + 1, dist.recs_recv[1], dist.pid_recv[1], mig.cap, mig.rec, has_aff, has_F, keys,
                const_cast<int*>(keys_sorted), int(cap), st);
        });
    }
    // NCCL: both exchanges of a step on the communication stream, ordered by events
    void dist_exchange_halo_nccl()
    {
        const size_t hb = sizeof(T) * dist.halo_elems;
        CK(cudaEventRecord(dist.ev_a, stream));
        CK(cudaStreamWaitEvent(dist.comm_stream, dist.ev_a, 0));
        NCK(dyn::ncclGroupStart());
        if (dist.lo_peer >= 0) {
            NCK(dyn::ncclSend(dist.halo_send[0], hb, ncclUint8, dist.lo_peer, dist.comm, dist.comm_stream));
            NCK(dyn::ncclRecv(dist.halo_recv[0], hb, ncclUint8, dist.lo_peer, dist.comm, dist.comm_stream));
        }
        if (dist.hi_peer >= 0) {
            NCK(dyn::ncclSend(dist.halo_send[1], hb, ncclUint8, dist.hi_peer, dist.comm, dist.comm_stream));
            NCK(dyn::ncclRecv(dist.halo_recv[1], hb, ncclUint8, dist.hi_peer, dist.comm, dist.comm_stream));
        }
        NCK(dyn::ncclGroupEnd());
        CK(cudaEventRecord(dist.ev_b, dist.comm_stream));
    }
    void dist_exchange_mig_nccl()
    {
        const size_t rb = sizeof(T) * size_t(mig.rec) * mig.cap, pb = sizeof(int) * size_t(mig.cap);
        CK(cudaEventRecord(dist.ev_a, stream));
        CK(cudaStreamWaitEvent(dist.comm_stream, dist.ev_a, 0));
        NCK(dyn::ncclGroupStart());
        for (int side = 0; side < 2; ++side) {
            const int peer = side == 0 ? dist.lo_peer : dist.hi_peer;
            if (peer < 0)
                continue;
            NCK(dyn::ncclSend(dist.cnt_send + side, sizeof(long long), ncclUint8, peer, dist.comm, dist.comm_stream));
            NCK(dyn::ncclSend(side == 0 ? mig.lo : mig.hi, rb, ncclUint8, peer, dist.comm, dist.comm_stream));
            NCK(dyn::ncclSend(side == 0 ? mig.lo_pid : mig.hi_pid, pb, ncclUint8, peer, dist.comm, dist.comm_stream));
            NCK(dyn::ncclRecv(dist.cnt_recv + side, sizeof(long long), ncclUint8, peer, dist.comm, dist.comm_stream));
            NCK(dyn::ncclRecv(dist.recs_recv[side], rb, ncclUint8, peer, dist.comm, dist.comm_stream));
            NCK(dyn::ncclRecv(dist.pid_recv[side], pb, ncclUint8, peer, dist.comm, dist.comm_stream));
        }
        NCK(dyn::ncclGroupEnd());
        if (dist.nranks > 1) // (a collective of its own, after the point-to-point group)
            NCK(dyn::ncclAllReduce(dist.abort_red, dist.abort_red, 1, ncclInt32, ncclMax, dist.comm, dist.comm_stream));
        CK(cudaEventRecord(dist.ev_b, dist.comm_stream));
        CK(cudaStreamWaitEvent(stream, dist.ev_b, 0));
    }
    void dist_step_nccl(bool guard)
    {
        dist_phase_a();
        if (dist.nranks > 1)
            dist_exchange_halo_nccl();
        dist_grid_interior(); // overlaps the band exchange
        if (dist.nranks > 1)
            CK(cudaStreamWaitEvent(stream, dist.ev_b, 0));
        dist_phase_b(guard);
        if (dist.nranks > 1)
            dist_exchange_mig_nccl();
        dist_phase_c(dist.abort_red);
    }
    // same-process ranks (tests, or several GPUs driven by one host thread): the same phases in
    // lock-step, exchanges as device copies ordered by events; all[r] is rank r
    void dist_enqueue_local(std::vector<CtxBase*>& all, int64_t nsteps, uint32_t flags) override
    {
        const int R = int(all.size());
        if (R > DIST_MAX_LOCAL)
            throw ApiError(MPM_ERR_USAGE, "dist: too many same-process ranks");
        std::vector<Ctx*> cs(R);
        for (int r = 0; r < R; ++r) {
            cs[r] = dynamic_cast<Ctx*>(all[r]);
            if (!cs[r] || !cs[r]->dist.on || cs[r]->dist.comm || cs[r]->dist.rank != r || cs[r]->dist.nranks != R)
                throw ApiError(MPM_ERR_USAGE, "dist: contexts must be attached as same-process ranks 0..R-1 of one scene type");
            if (!cs[r]->has_state)
                throw ApiError(MPM_ERR_USAGE, "no state uploaded");
        }
        const bool guard = flags & MPM_ADV_NAN_GUARD;
        AbortPtrs ap{};
        ap.R = R;
        for (int r = 0; r < R; ++r)
            ap.p[r] = cs[r]->dist.abort_red;
        for (Ctx* c : cs) {
            c->reset_status();
            c->dist_step_begin();
        }
        auto wait_on = [](Ctx* c, Ctx* peer) { CK(cudaStreamWaitEvent(c->stream, peer->dist.ev_a, 0)); };
        for (int64_t k = 0; k < nsteps; ++k) {
            for (Ctx* c : cs) {
                c->dist_phase_a();
                CK(cudaEventRecord(c->dist.ev_a, c->stream));
            }
            for (int r = 0; r < R; ++r) {
                Ctx* c = cs[r];
                const size_t hb = sizeof(T) * c->dist.halo_elems;
                for (int side = 0; side < 2; ++side) {
                    const int pr = side == 0 ? c->dist.lo_peer : c->dist.hi_peer;
                    if (pr < 0)
                        continue;
                    wait_on(c, cs[pr]);
                    CK(cudaMemcpyAsync(c->dist.halo_recv[side], cs[pr]->dist.halo_send[1 - side], hb,
                                       cudaMemcpyDeviceToDevice, c->stream));
                }
            }
            for (Ctx* c : cs) {
                c->dist_grid_interior();
                c->dist_phase_b(guard);
                CK(cudaEventRecord(c->dist.ev_a, c->stream));
            }
            for (int r = 0; r < R; ++r) {
                Ctx* c = cs[r];
                const size_t rb = sizeof(T) * size_t(c->mig.rec) * c->mig.cap, pb = sizeof(int) * size_t(c->mig.cap);
                for (int q = 0; q < R; ++q)
                    if (q != r)
                        wait_on(c, cs[q]);
                for (int side = 0; side < 2; ++side) {
                    const int pr = side == 0 ? c->dist.lo_peer : c->dist.hi_peer;
                    if (pr < 0)
                        continue;
                    Ctx* p = cs[pr];
                    CK(cudaMemcpyAsync(c->dist.cnt_recv + side, p->dist.cnt_send + (1 - side), sizeof(long long),
                                       cudaMemcpyDeviceToDevice, c->stream));
                    CK(cudaMemcpyAsync(c->dist.recs_recv[side], side == 0 ? p->mig.hi : p->mig.lo, rb,
                                       cudaMemcpyDeviceToDevice, c->stream));
                    CK(cudaMemcpyAsync(c->dist.pid_recv[side], side == 0 ? p->mig.hi_pid : p->mig.lo_pid, pb,
                                       cudaMemcpyDeviceToDevice, c->stream));
                }
                c->launch("k_dist", [&] { k_dist_abort_max<<<1, 1, 0, c->stream>>>(ap, c->dist.abort_red + 1); });
                CK(cudaEventRecord(c->dist.ev_b, c->stream));
            }
            for (Ctx* c : cs) { // every rank has read its peers' messages before they are rewritten
                for (Ctx* q : cs)
                    if (q != c)
                        CK(cudaStreamWaitEvent(c->stream, q->dist.ev_b, 0));
                c->dist_phase_c(c->dist.abort_red + 1);
            }
        }
    }
    void dist_finish() override { dist_finish_call(); }
    // ---- decomposed backprop_trajectory on the library-owned path (checkpoint.hpp:72-143) --------
    // Every rank runs the same sequence with its own particles: a forward sweep with per-rank HBM
    // checkpoints at segment starts (and rank-local digests), then per segment (reversed) a replay
    // into per-rank slots recording each step's migration (export lists with the vacated slots,
    // import layout), a digest check (any rank's mismatch fails every rank), and per step: the
    // device seeder on global particle ids, the return of migrants' cotangent rows to their step-t
    // owner, and the decomposed step_vjp (adjoint.hpp:328-525) with its two halo exchanges. Loss and
    // ParamGrads are per-rank device sums, gathered and added in rank order at the end.
    struct DistTape {
        int64_t n_before = 0, n_after = 0; // counts of S^j and S^{j+1}
        long long* ex_cnt = nullptr; // [2] exports toward lo / hi during the step
        int* ex_pid[2] = {nullptr, nullptr};
        int* ex_slot[2] = {nullptr, nullptr};
        int* nlive = nullptr;         // the step's G2P output count
        long long* im_cnt = nullptr;  // [2] imports from lo / hi
    };
    std::vector<DistTape> dtape;
    T* cot_xbuf[4] = {nullptr, nullptr, nullptr, nullptr}; // cotangent-row messages: send lo / hi, recv lo / hi
    int* dist_sop = nullptr;   // slot of a global particle id
    int64_t dist_sop_n = 0;
    int* abort_all = nullptr;  // [nranks]
    double* dist_gather = nullptr;

    std::vector<XItem> halo_items(size_t bytes)
    {
        std::vector<XItem> v;
        if (dist.lo_peer >= 0)
            v.push_back({dist.halo_send[0], dist.halo_recv[0], bytes, dist.lo_peer});
        if (dist.hi_peer >= 0)
            v.push_back({dist.halo_send[1], dist.halo_recv[1], bytes, dist.hi_peer});
        return v;
    }
    std::vector<XItem> mig_items()
    {
        const size_t rb = sizeof(T) * size_t(mig.rec) * mig.cap, pb = sizeof(int) * size_t(mig.cap);
        std::vector<XItem> v;
        for (int side = 0; side < 2; ++side) {
            const int peer = side == 0 ? dist.lo_peer : dist.hi_peer;
            if (peer < 0)
                continue;
            v.push_back({dist.cnt_send + side, dist.cnt_recv + side, sizeof(long long), peer});
            v.push_back({side == 0 ? mig.lo : mig.hi, dist.recs_recv[side], rb, peer});
            v.push_back({side == 0 ? mig.lo_pid : mig.hi_pid, dist.pid_recv[side], pb, peer});
        }
        return v;
    }
    void dist_abort_reduce(DistTransport& X)
    {
        X.allgather(stream, dist.abort_red, abort_all, sizeof(int));
        AbortPtrs ap{};
        ap.R = dist.nranks;
        for (int r = 0; r < dist.nranks; ++r)
            ap.p[r] = abort_all + r;
        launch("k_dist", [&] { k_dist_abort_max<<<1, 1, 0, stream>>>(ap, dist.abort_red + 1); });
    }
    // one decomposed forward step over any transport (eager)
    void dist_step_x(DistTransport& X, bool guard)
    {
        dist_phase_a();
        if (dist_has_peers())
            X.begin(stream, halo_items(sizeof(T) * dist.halo_elems));
        dist_grid_interior();
        if (dist_has_peers())
            X.end(stream);
        dist_phase_b(guard);
        if (dist.nranks > 1) {
            X.begin(stream, mig_items());
            X.end(stream);
            dist_abort_reduce(X);
        }
        dist_phase_c(dist.abort_red + 1);
    }
    // the decomposed step_vjp of the state in buf[cur] (host n valid): cot[bo] -> cot[bi]
    void dist_vjp_x(DistTransport& X, int bo, int bi)
    {
        sort_and_segment();
        p2g_kernel();
        if (!dist_has_peers()) {
            grid_kernel<G_SUM | G_MOM | G_CORR | G_STORE>();
            aw.vjp_reverse(*this, bo, bi);
            return;
        }
        grid_kernel<G_BANDONLY | G_SUM | G_NOGRAV | G_STORE>();
        if (dist.lo_peer >= 0)
            halo(sc.slab_lo, 2, dist.halo_send[0], 0);
        if (dist.hi_peer >= 0)
            halo(sc.slab_hi, 2, dist.halo_send[1], 0);
        X.begin(stream, halo_items(sizeof(T) * dist.halo_elems));
        grid_kernel<G_INTERIOR | G_SUM | G_MOM | G_CORR | G_STORE>();
        X.end(stream);
        if (dist.lo_peer >= 0)
            halo(sc.slab_lo, 2, dist.halo_recv[0], 1);
        if (dist.hi_peer >= 0)
            halo(sc.slab_hi, 2, dist.halo_recv[1], 2);
        grid_kernel<G_BANDONLY | G_GRAV | G_ZEROV | G_MOM | G_CORR | G_STORE>();
        dist_vjp_reverse_x(X, bo, bi);
    }
    // the reverse part of the decomposed step_vjp, on the step's sort and full forward grid (from
    // the replay's tape, or just recomputed by dist_vjp_x)
    void dist_vjp_reverse_x(DistTransport& X, int bo, int bi)
    {
        if (!dist_has_peers()) {
            aw.vjp_reverse(*this, bo, bi);
            return;
        }
        aw.k5(*this, bo, bi);
        launch("k_adj_grid", [&] {
            k_adj_grid<T, D, ADJ_BAND_SUM><<<persistent(4), C::NB, 0, stream>>>(sc, G, aw.gc, aw.partials, bstart, act,
                                                                               counts + 1, aw.fr_block, st);
        });
        const HaloFields<T> H = aw.cot_halo_fields();
        int64_t plane = 1;
        for (int a = 1; a < D; ++a)
            plane *= sc.cells[a] + 1;
        if (dist.lo_peer >= 0)
            halo_fields(H, sc.slab_lo, 2, dist.halo_send[0], 0);
        if (dist.hi_peer >= 0)
            halo_fields(H, sc.slab_hi, 2, dist.halo_send[1], 0);
        X.begin(stream, halo_items(sizeof(T) * 2 * plane * 2 * D));
        X.end(stream);
        if (dist.lo_peer >= 0)
            halo_fields(H, sc.slab_lo, 2, dist.halo_recv[0], 1);
        if (dist.hi_peer >= 0)
            halo_fields(H, sc.slab_hi, 2, dist.halo_recv[1], 2);
        launch("k_adj_grid", [&] {
            k_adj_grid<T, D, ADJ_INTERIOR><<<persistent(4), C::NB, 0, stream>>>(sc, G, aw.gc, aw.partials, bstart, act,
                                                                               counts + 1, aw.fr_block, st);
        });
        launch("k_adj_grid", [&] {
            k_adj_grid<T, D, ADJ_BAND_LOAD><<<persistent(4), C::NB, 0, stream>>>(sc, G, aw.gc, aw.partials, bstart, act,
                                                                                counts + 1, aw.fr_block, st);
        });
        aw.k7(*this, bi);
    }
    int cot_values() const { return 2 * D + 2 + (D == 2 ? 1 : 0) + 2 * D * D + (has_aff ? D * D : 0); }
    // migrants' cotangent rows back to their step-t owners (kernels_dist.cuh)
    void dist_cot_return(DistTransport& X, const DistTape& tp, int cb)
    {
        if (!dist_has_peers())
            return;
        const int nv = cot_values();
        const size_t bytes = sizeof(T) * size_t(nv) * mig.cap;
        const unsigned g = grid_for(mig.cap, 256);
        const int gz = aw.gvz[cb] ? 1 : 0;
        std::vector<XItem> items;
        for (int side = 0; side < 2; ++side) {
            const int peer = side == 0 ? dist.lo_peer : dist.hi_peer;
            if (peer < 0)
                continue;
            launch("k_cot_pack", [&] {
                k_cot_pack<T, D><<<g, 256, 0, stream>>>(aw.cot[cb], tp.nlive, tp.im_cnt, tp.im_cnt + side, side,
                                                        cot_xbuf[side], gz, has_aff);
            });
            items.push_back({cot_xbuf[side], cot_xbuf[2 + side], bytes, peer});
        }
        X.begin(stream, items);
        X.end(stream);
        for (int side = 0; side < 2; ++side) {
            const int peer = side == 0 ? dist.lo_peer : dist.hi_peer;
            if (peer < 0)
                continue;
            launch("k_cot_unpack", [&] {
                k_cot_unpack<T, D><<<g, 256, 0, stream>>>(aw.cot[cb], tp.ex_cnt + side, tp.ex_pid[side], tp.ex_slot[side],
                                                          cot_xbuf[2 + side], gz, has_aff);
            });
        }
    }
    void dist_bp_alloc(int64_t Lmax, int64_t id_space)
    {
        while (int64_t(dtape.size()) < Lmax) {
            DistTape t;
            t.ex_cnt = alloc<long long>(2);
            t.im_cnt = alloc<long long>(2);
            t.nlive = alloc<int>(1);
            for (int s2 = 0; s2 < 2; ++s2) {
                t.ex_pid[s2] = alloc<int>(mig.cap);
                t.ex_slot[s2] = alloc<int>(mig.cap);
            }
            dtape.push_back(t);
        }
        if (!cot_xbuf[0])
            for (auto& b : cot_xbuf)
                b = alloc<T>(size_t(cot_values()) * mig.cap);
        if (id_space > dist_sop_n) {
            dist_sop = alloc<int>(id_space);
            dist_sop_n = id_space;
        }
        if (!abort_all) {
            abort_all = alloc<int>(dist.nranks);
            dist_gather = alloc<double>(size_t(dist.nranks) * (PG_SLOTS + 1));
        }
    }
    void dist_backprop(DistTransport& X, int64_t total, int nseg, const mpm_seeder_desc* sd, int64_t id_space,
                       mpm_cot_view* c0, int64_t* c0_ids, mpm_param_grads* pg, mpm_backprop_result* res)
    {
        if (!dist.on)
            throw ApiError(MPM_ERR_USAGE, "dist: context not attached");
        if (!has_state)
            throw ApiError(MPM_ERR_USAGE, "no state uploaded");
        if (total < 1 || nseg < 1 || int64_t(nseg) > total)
            throw ApiError(MPM_ERR_VALIDATION, "checkpoint plan: n_segments must lie in [1, N_t]");
        if (sd && sd->kind != MPM_SEEDER_LAGRANGIAN_LS && sd->n_obs > 0)
            throw ApiError(MPM_ERR_USAGE, "dist backprop: the Lagrangian least-squares seeder only");
        std::vector<int64_t> bnd(nseg + 1, 0);
        {
            const int64_t base = total / nseg, rem = total % nseg;
            for (int k = 0; k < nseg; ++k)
                bnd[k + 1] = bnd[k] + base + (k < rem ? 1 : 0);
        }
        int64_t Lmax = 0;
        for (int k = 0; k < nseg; ++k)
            Lmax = std::max(Lmax, bnd[k + 1] - bnd[k]);
        aw.ensure(*this);
        dist_bp_alloc(Lmax, std::max<int64_t>(id_space, 1));
        const bool seeding = sd && sd->n_obs > 0;
        const int64_t nsel = seeding ? (sd->sel ? sd->n_sel : id_space) : 0;
        struct Owned {
            std::vector<void*> v;
            ~Owned()
            {
                for (void* p : v)
                    cudaFree(p);
            }
        } owned;
        long long* d_sel = nullptr;
        T* d_tgt = nullptr;
        T* d_lblk = nullptr;
        if (seeding) {
            if (sd->sel) {
                CK(cudaMalloc(&d_sel, nsel * sizeof(long long)));
                owned.v.push_back(d_sel);
                for (int64_t l = 0; l < nsel; ++l)
                    if (sd->sel[l] < 0 || sd->sel[l] >= id_space)
                        throw ApiError(MPM_ERR_VALIDATION, "seeder: particle id out of range");
                h2d_raw(d_sel, sd->sel, nsel * sizeof(long long));
            }
            CK(cudaMalloc(&d_tgt, (size_t)sd->n_obs * nsel * D * sizeof(T)));
            owned.v.push_back(d_tgt);
            h2d_raw(d_tgt, sd->target, (size_t)sd->n_obs * nsel * D * sizeof(T));
            CK(cudaMalloc(&d_lblk, sizeof(T) * std::max<int64_t>(1, grid_for(nsel, 256))));
            owned.v.push_back(d_lblk);
        }
        auto obs_index = [&](int64_t t) {
            if (!seeding)
                return -1;
            for (int k = 0; k < sd->n_obs; ++k)
                if (sd->obs_steps[k] == t)
                    return k;
            return -1;
        };
        auto seed = [&](const PBuf<T, D>& P, int64_t nP, int k, int cb, int do_cot) {
            CK(cudaMemsetAsync(dist_sop, 0xff, sizeof(int) * dist_sop_n, stream));
            launch("k_slot_of_pid", [&] { k_slot_of_pid<T, D><<<grid_for(nP, 256), 256, 0, stream>>>(P, int(nP), dist_sop); });
            const int sb = int(grid_for(nsel, 256));
            launch("k_seed", [&] {
                k_seed_lagrangian<T, D><<<sb, 256, 0, stream>>>(P, int(nP), dist_sop, d_sel, nsel,
                                                                d_tgt + (size_t)k * nsel * D, sd->field, aw.cot[cb],
                                                                do_cot, d_lblk);
            });
            launch("k_seed", [&] { k_seed_sum<T><<<1, 1024, 0, stream>>>(d_lblk, sb, aw.loss_acc); });
        };
        const PBuf<T, D> own0 = buf[0], own1 = buf[1];
        const int cur0 = cur;
        const int64_t step0 = step;
        struct Ev {
            cudaEvent_t e{};
            Ev() { CK(cudaEventCreate(&e)); }
            ~Ev() { cudaEventDestroy(e); }
        } ev0, ev1;
        std::vector<int64_t> ckn(nseg);
        std::vector<uint64_t> bhash(nseg + 1);
        int cb = 0;
        const SortSet own_ss0 = sort_set();
        try {
            std::vector<PBuf<T, D>> ckpt(nseg), replay(Lmax + 1);
            for (int k = 0; k < nseg; ++k)
                ckpt[k] = pool_buf(size_t(k));
            for (int64_t j = 0; j <= Lmax; ++j)
                replay[j] = pool_buf(size_t(nseg + j));
            // the replay tape (the step's sort arrays and forward grid kept, as backprop_run does): the
            // VJP then skips its forward replay; slots sized from S0's active node blocks (+25 %),
            // a step that outgrows its slot falls back to the recompute
            const SortSet own_ss = sort_set();
            bool use_tape = false;
            {
                keys_valid = false;
                inc_invalidate();
                sort_and_segment();
                keys_valid = false;
                int n_act_now = 0;
                d2h_raw(&n_act_now, counts + 1, sizeof(int));
                const char* cap_env = std::getenv("MPM_TAPE_CAP"); // test hook: force slot overflows
                const int64_t grid_cap = cap_env ? std::max<int64_t>(1, std::atoll(cap_env))
                                                 : std::min<int64_t>(sc.nnb_total, (int64_t(n_act_now) * 5 / 4 + 255) / 256 * 256);
                use_tape = tape_enabled && tape_reserve(Lmax, grid_cap);
                if (use_tape)
                    CK(cudaMemsetAsync(tape_over, 0, sizeof(int) * Lmax, stream));
            }
            CK(cudaMemsetAsync(aw.loss_acc, 0, sizeof(double), stream));
            aw.pg_reset(*this, nullptr);
            reset_status();
            CK(cudaEventRecord(ev0.e, stream));
            // the steps of segment k run in the replay slots (state j in replay[j]), each step's
            // migration recorded for the reverse sweep; `fwd_seed`: evaluate the loss at observed
            // steps (the forward sweep's run of the last segment)
            std::vector<int> over(Lmax, 1);
            auto run_in_slots = [&](int k, bool fwd_seed) {
                const int64_t b0 = bnd[k], len = bnd[k + 1] - b0;
                n = ckn[k]; // (pbuf_copy moves n rows)
                pbuf_copy(replay[0], ckpt[k]);
                if (use_tape)
                    CK(cudaMemsetAsync(tape_over, 0, sizeof(int) * len, stream));
                for (int64_t j = 0; j < len; ++j) {
                    DistTape& tp = dtape[size_t(j)];
                    tp.n_before = n;
                    buf[0] = replay[j];
                    buf[1] = replay[j + 1];
                    cur = 0;
                    keys_valid = false;
                    inc_invalidate();
                    dist_step_begin();
                    if (use_tape) {
                        use_sort_set(tape[j].ss);
                        dist_store = true;
                    }
                    dist_step_x(X, false);
                    if (use_tape) {
                        tape_grid<true>(int(j));
                        dist_store = false;
                        use_sort_set(own_ss);
                    }
                    CK(cudaMemcpyAsync(tp.nlive, dist.d_nlive, sizeof(int), cudaMemcpyDeviceToDevice, stream));
                    CK(cudaMemcpyAsync(tp.im_cnt, dist.cnt_recv, 2 * sizeof(long long), cudaMemcpyDeviceToDevice, stream));
                    launch("k_dist", [&] { k_dist_export_counts<<<1, 1, 0, stream>>>(st, tp.ex_cnt, mig.cap); });
                    for (int s2 = 0; s2 < 2; ++s2) {
                        CK(cudaMemcpyAsync(tp.ex_pid[s2], s2 ? mig.hi_pid : mig.lo_pid, sizeof(int) * mig.cap,
                                           cudaMemcpyDeviceToDevice, stream));
                        CK(cudaMemcpyAsync(tp.ex_slot[s2], s2 ? mig.hi_slot : mig.lo_slot, sizeof(int) * mig.cap,
                                           cudaMemcpyDeviceToDevice, stream));
                    }
                    if (dist.nranks == 1) // no imports: the recorded counts are zero
                        CK(cudaMemsetAsync(tp.im_cnt, 0, 2 * sizeof(long long), stream));
                    dist_sync_count();
                    tp.n_after = n;
                    if (fwd_seed && obs_index(b0 + j + 1) >= 0)
                        seed(buf[cur], n, obs_index(b0 + j + 1), 0, 0);
                }
                if (use_tape)
                    d2h_raw(over.data(), tape_over, sizeof(int) * len);
            };
            // forward sweep; the last segment runs directly in the replay slots: its states are the
            // ones a replay would recompute bit for bit, so the reverse sweep starts without
            // replaying it (with one segment: 1 forward pass + 1 VJP per step)
            if (obs_index(0) >= 0)
                seed(buf[cur], n, obs_index(0), 0, 0);
            for (int k = 0; k < nseg; ++k) {
                pbuf_copy(ckpt[k], buf[cur]);
                ckn[k] = n;
                if (k >= 1)
                    bhash[k] = digest_of(buf[cur]);
                if (k == nseg - 1) {
                    run_in_slots(k, true);
                    break;
                }
                dist_step_begin();
                for (int64_t t = bnd[k]; t < bnd[k + 1]; ++t) {
                    dist_step_x(X, false);
                    if (obs_index(t + 1) >= 0) {
                        dist_sync_count();
                        seed(buf[cur], n, obs_index(t + 1), 0, 0);
                    }
                }
                dist_sync_count();
            }
            check_status(step0);
            double loss_local = 0;
            d2h_raw(&loss_local, aw.loss_acc, sizeof(double));
            // reverse sweep
            n = dtape[size_t(bnd[nseg] - bnd[nseg - 1] - 1)].n_after; // S^N: the last slot
            aw.cot_zero(*this, 0);
            int64_t peak = 0;
            for (int k = nseg - 1; k >= 0; --k) {
                const int64_t b0 = bnd[k], b1 = bnd[k + 1], len = b1 - b0;
                const bool kept = k == nseg - 1;
                if (!kept) // replay into the slots, recording every step's migration
                    run_in_slots(k, false);
                peak = std::max(peak, len + 1);
                // digest check of a replayed segment; any rank's mismatch fails every rank
                int bad = !kept && digest_of(replay[len]) != bhash[k + 1] ? 1 : 0;
                h2d_raw(dist.abort_red, &bad, sizeof(int));
                if (dist.nranks > 1)
                    dist_abort_reduce(X);
                else
                    CK(cudaMemcpyAsync(dist.abort_red + 1, dist.abort_red, sizeof(int), cudaMemcpyDeviceToDevice, stream));
                int any = 0;
                d2h_raw(&any, dist.abort_red + 1, sizeof(int));
                if (any)
                    throw ApiError(MPM_ERR_CHECKPOINT, "checkpoint mismatch: recomputed segment end differs from the "
                                                       "recorded state at step " + std::to_string(step0 + b1));
                for (int64_t t = b1; t > b0; --t) {
                    const int64_t j = t - b0 - 1;
                    const DistTape& tp = dtape[size_t(j)];
                    if (obs_index(t) >= 0) // cotangent of S^t, storage order of replay[j + 1]
                        seed(replay[j + 1], tp.n_after, obs_index(t), cb, 1);
                    dist_cot_return(X, tp, cb);
                    buf[0] = replay[j];
                    buf[1] = replay[j + 1];
                    cur = 0;
                    n = tp.n_before;
                    keys_valid = false;
                    inc_invalidate();
                    if (use_tape && !over[size_t(j)]) { // the replay's sort and grid
                        use_sort_set(tape[size_t(j)].ss);
                        tape_grid<false>(int(j));
                        dist_vjp_reverse_x(X, cb, cb ^ 1);
                        use_sort_set(own_ss);
                    } else {
                        dist_vjp_x(X, cb, cb ^ 1);
                    }
                    cb ^= 1;
                }
                check_status(step);
            }
            n = ckn[0];
            if (obs_index(0) >= 0)
                seed(ckpt[0], n, obs_index(0), cb, 1);
            CK(cudaEventRecord(ev1.e, stream));
            // rank-ordered sums of the loss and the ParamGrads
            double mine[PG_SLOTS + 1];
            d2h_raw(mine, aw.pg_acc, sizeof(double) * PG_SLOTS);
            mine[PG_SLOTS] = loss_local;
            h2d_raw(dist_gather, mine, sizeof(mine));
            std::vector<double> all(size_t(dist.nranks) * (PG_SLOTS + 1));
            if (dist.nranks > 1) {
                double* gbuf = nullptr;
                CK(cudaMalloc(&gbuf, sizeof(double) * all.size()));
                owned.v.push_back(gbuf);
                X.allgather(stream, dist_gather, gbuf, sizeof(double) * (PG_SLOTS + 1));
                d2h_raw(all.data(), gbuf, sizeof(double) * all.size());
            } else {
                std::memcpy(all.data(), mine, sizeof(mine));
            }
            double tot[PG_SLOTS + 1] = {0};
            for (int r = 0; r < dist.nranks; ++r)
                for (int q = 0; q <= PG_SLOTS; ++q)
                    tot[q] += all[size_t(r) * (PG_SLOTS + 1) + q];
            h2d_raw(aw.pg_acc, tot, sizeof(double) * PG_SLOTS);
            aw.pg_download(*this, pg);
            float dev_ms = 0;
            CK(cudaEventElapsedTime(&dev_ms, ev0.e, ev1.e));
            // this rank's cotangent of S^0 (storage order of the checkpoint) and the particle ids
            buf[0] = ckpt[0];
            cur = 0;
            aw.cot_download(*this, c0, cb);
            std::vector<int> pids(std::max<int64_t>(n, 1));
            d2h_raw(pids.data(), ckpt[0].pid, sizeof(int) * n);
            for (int64_t i = 0; i < n; ++i)
                c0_ids[i] = pids[i];
            c0->n = n;
            if (res) {
                res->loss = tot[PG_SLOTS];
                res->checkpoints_stored = nseg;
                res->peak_replay_states = peak;
                res->device_ms = dev_ms;
            }
            buf[0] = own0;
            buf[1] = own1;
            cur = cur0;
            n = ckn[0];
            pbuf_copy(buf[cur], ckpt[0]);
            step = step0;
            keys_valid = false;
            inc_invalidate();
            CK(cudaStreamSynchronize(stream));
        } catch (...) {
            buf[0] = own0;
            buf[1] = own1;
            cur = cur0;
            keys_valid = false;
            dist_store = false;
            use_sort_set(own_ss0);
            inc_invalidate();
            cudaStreamSynchronize(stream);
            throw;
        }
    }
    void dist_backprop_nccl(int64_t total, int nseg, const mpm_seeder_desc* sd, int64_t id_space, mpm_cot_view* c0,
                            int64_t* c0_ids, mpm_param_grads* pg, mpm_backprop_result* res) override
    {
        if (!dist.comm)
            throw ApiError(MPM_ERR_USAGE, "dist: context not attached to an NCCL communicator");
        NcclX X(dist.comm, dist.comm_stream, dist.ev_a, dist.ev_b);
        dist_backprop(X, total, nseg, sd, id_space, c0, c0_ids, pg, res);
    }
    void dist_backprop_local(LocalHub* hub, int64_t total, int nseg, const mpm_seeder_desc* sd, int64_t id_space,
                             mpm_cot_view* c0, int64_t* c0_ids, mpm_param_grads* pg, mpm_backprop_result* res) override
    {
        CK(cudaSetDevice(device));
        LocalX X(hub, dist.rank);
        dist_backprop(X, total, nseg, sd, id_space, c0, c0_ids, pg, res);
    }
    void dist_sync_count()
    {
        int dn = 0;
        CK(cudaMemcpyAsync(&dn, dist.d_n, sizeof(int), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        n = dn;
    }

    // n decomposed steps on an NCCL rank; graph-replayed after the first (its radix sort and the
    // count upload run eagerly), no host synchronisation until the status check at the end
    void dist_advance(int64_t nsteps, uint32_t flags, double* ms) override
    {
        if (!dist.on || !dist.comm)
            throw ApiError(MPM_ERR_USAGE, "dist: context not attached to an NCCL communicator");
        if (!has_state)
            throw ApiError(MPM_ERR_USAGE, "no state uploaded");
        const bool guard = flags & MPM_ADV_NAN_GUARD;
        reset_status();
        dist_step_begin();
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (ms) {
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(cudaEventRecord(e0, stream));
        }
        // NCCL calls inside a captured graph are supported, but untested here beyond one rank (this
        // pool gives one GPU per call): with peers the steps are enqueued eagerly unless
        // MPM_DIST_GRAPH=1 (the host runs ahead asynchronously, so C4-sized steps stay GPU-bound);
        // MPM_DIST_GRAPH=0 forces the eager path on one rank too (tests compare the two)
        const char* dg = std::getenv("MPM_DIST_GRAPH");
        const bool graph_ok = dg ? dg[0] == '1' : dist.nranks == 1;
        for (int64_t k = 0; k < nsteps; ++k) {
            const bool eager = prof || !inc_source_ok() || !graph_ok;
            if (eager) {
                dist_step_nccl(guard);
                continue;
            }
            cudaGraphExec_t& ge = dist.graph[guard][cur];
            if (!ge) {
                dist.graph_launches = capture(ge, [&] { dist_step_nccl(guard); });
                dist.graph_inc[guard][cur] = captured_inc_src;
            }
            CK(cudaGraphLaunch(ge, stream));
            launches += dist.graph_launches;
            inc_src = dist.graph_inc[guard][cur];
            keys_sorted = ks_own[cur];
            bstart = bs_own[cur];
            bend = be_own[cur];
            cur ^= 1;
            keys_valid = true;
        }
        if (ms) {
            CK(cudaEventRecord(e1, stream));
            CK(cudaEventSynchronize(e1));
            float t = 0;
            CK(cudaEventElapsedTime(&t, e0, e1));
            *ms = t;
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
        }
        dist_finish_call();
    }
    // after a call: the device count and status come back once
    void dist_finish_call()
    {
        int dn = 0;
        CK(cudaMemcpyAsync(&dn, dist.d_n, sizeof(int), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        n = dn;
        n_dead = 0; // vacated slots are dropped by the next sort; download_local skips them (pid < 0)
        check_status(step);
    }

    void* ids_scratch = nullptr;
    size_t ids_scratch_bytes = 0;
    void* aw_ids_scratch(int64_t k)
    {
        const size_t b = size_t(k) * sizeof(long long);
        if (b > ids_scratch_bytes) {
            if (ids_scratch)
                cudaFree(ids_scratch);
            CK(cudaMalloc(&ids_scratch, b));
            ids_scratch_bytes = b;
        }
        return ids_scratch;
    }
    int rec_size() const override { return 2 * D + 5 + C::NS + D * D + (has_aff ? D * D : 0) + (has_F ? D * D : 0); }
    void slab_set(int lo, int hi, int64_t mig_cap) override
    {
        inc_invalidate();
        if (own_set) { // slab phases are graph-replayed with eager kernels between them: one fixed pair
            keys_sorted = ks_own[0];
            bstart = bs_own[0];
            bend = be_own[0];
        }
        if (lo < 0 || hi <= lo || lo % C::B || (hi % C::B && hi < sc.cells[0]))
            throw ApiError(MPM_ERR_USAGE, "slab bounds must be block-aligned (multiples of " + std::to_string(C::B) + ")");
        sc.slab_lo = lo;
        sc.slab_hi = hi;
        sc.band_lo = lo > 0 ? lo : -(1 << 28);
        sc.band_hi = hi < sc.cells[0] ? hi : -(1 << 28);
        slab = true;
        if (!mig.on || mig.cap < mig_cap) {
            mig.on = 1;
            mig.cap = int(mig_cap);
            mig.rec = rec_size();
            mig.lo = alloc<T>((size_t)mig_cap * mig.rec);
            mig.hi = alloc<T>((size_t)mig_cap * mig.rec);
            mig.lo_pid = alloc<int>(mig_cap);
            mig.hi_pid = alloc<int>(mig_cap);
            mig.lo_slot = alloc<int>(mig_cap);
            mig.hi_slot = alloc<int>(mig_cap);
        }
        for (auto& g : graphs)
            for (auto& h : g)
                for (auto& e : h)
                    if (e) {
                        cudaGraphExecDestroy(e);
                        e = nullptr;
                    }
        drop_slab_graphs();
        keys_valid = false;
    }
    void p2g_phase()
    {
        launch("k_reset", [&] { k_reset_flags<<<1, 1, 0, stream>>>(st); });
        sort_and_segment();
        p2g_kernel();
        // halo-band nodes only: their partial sums (without g m) go to the neighbours; an abort
        // here is reported by step_finish_local
        grid_kernel<G_BANDONLY | G_SUM | G_NOGRAV | G_STORE>();
    }
    // every node off the halo bands: the fused sum + g m + momentum + corrections, enqueued while
    // the bands travel (the transport overlaps it)
    void step_grid_interior() override { grid_kernel<G_INTERIOR | G_SUM | G_MOM | G_CORR>(); }
    // init_scene (scene.hpp:55-116) on the device: count per cell, exclusive scan, write in order
    void init_scene_dev(const mpm_region* rg, int nreg, double mass, double volume, double rho0,
                        int64_t* n_out) override
    {
        inc_invalidate();
        if (nreg < 1 || !rg)
            throw ApiError(MPM_ERR_VALIDATION, "scene: no geometry regions");
        SeedBox bx{};
        bx.ncell = 1;
        for (int a = 0; a < D; ++a) { // union bounding box, as the host seeding restricts its visit
            double lo = 1e300, hi = -1e300;
            for (int r = 0; r < nreg; ++r) {
                const mpm_region& g = rg[r];
                const double l = g.shape == 0 ? g.lo[a] : (a < 2 ? g.center[a] - g.radius : g.zmin);
                const double h = g.shape == 0 ? g.hi[a] : (a < 2 ? g.center[a] + g.radius : g.zmax);
                lo = std::min(lo, l);
                hi = std::max(hi, h);
            }
            const double o = desc.origin[a], dh = desc.dh;
            bx.lo[a] = std::max(0, int(std::floor((lo - o) / dh)) - 1);
            const int hc = std::min(desc.cells[a], int(std::ceil((hi - o) / dh)) + 1);
            bx.ext[a] = std::max(0, hc - bx.lo[a]);
            bx.ncell *= bx.ext[a];
        }
        if (bx.ncell <= 0)
            throw ApiError(MPM_ERR_VALIDATION, "scene: geometry produced no particles");
        mpm_region* d_rg = nullptr;
        int *counts_d = nullptr, *offs = nullptr;
        void* tmp = nullptr;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&d_rg), sizeof(mpm_region) * nreg, stream));
        CK(cudaMallocAsync(reinterpret_cast<void**>(&counts_d), sizeof(int) * bx.ncell, stream));
        CK(cudaMallocAsync(reinterpret_cast<void**>(&offs), sizeof(int) * bx.ncell, stream));
        CK(cudaMemcpyAsync(d_rg, rg, sizeof(mpm_region) * nreg, cudaMemcpyHostToDevice, stream));
        launch("k_seed", [&] {
            k_seed_count<T, D><<<grid_for(bx.ncell, 256), 256, 0, stream>>>(sc, bx, d_rg, nreg, counts_d);
        });
        size_t bytes = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, counts_d, offs, int(bx.ncell), stream));
        CK(cudaMallocAsync(&tmp, bytes, stream));
        CK(cub::DeviceScan::ExclusiveSum(tmp, bytes, counts_d, offs, int(bx.ncell), stream));
        int last[2] = {0, 0};
        CK(cudaMemcpyAsync(&last[0], offs + bx.ncell - 1, sizeof(int), cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(&last[1], counts_d + bx.ncell - 1, sizeof(int), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        const int64_t total = int64_t(last[0]) + last[1];
        *n_out = total;
        auto release = [&] {
            cudaFreeAsync(tmp, stream);
            cudaFreeAsync(offs, stream);
            cudaFreeAsync(counts_d, stream);
            cudaFreeAsync(d_rg, stream);
        };
        if (total < 1 || total > cap) {
            release();
            throw ApiError(total < 1 ? MPM_ERR_VALIDATION : MPM_ERR_USAGE,
                           total < 1 ? "scene: geometry produced no particles"
                                     : "init_scene: " + std::to_string(total) + " particles exceed the context capacity " +
                                           std::to_string(cap));
        }
        launch("k_seed", [&] {
            k_seed_write<T, D><<<grid_for(bx.ncell, 256), 256, 0, stream>>>(sc, bx, d_rg, nreg, offs, buf[cur], T(mass),
                                                                           T(volume), T(rho0), has_aff, has_F);
        });
        release();
        CK(cudaStreamSynchronize(stream));
        n = total;
        n_dead = 0;
        keys_valid = false;
        status_dirty = true;
        has_state = true;
        step = 0;
        time = 0.0;
    }

    // step_vjp over a slab (same exchange points as the forward step, plus the node cotangents)
    void slab_vjp_begin(const mpm_cot_view* co) override
    {
        if (!slab)
            throw ApiError(MPM_ERR_USAGE, "mpm_slab_vjp_begin needs mpm_slab_set first");
        aw.slab_vjp_begin(*this, co);
    }
    void slab_vjp_interior() override { aw.slab_vjp_interior(*this); }
    void slab_vjp_scatter() override { aw.slab_vjp_scatter(*this); }
    void halo_cot(int plane_lo, int n_planes, void* dev_buf, int mode) override
    {
        halo_fields(aw.cot_halo_fields(), plane_lo, n_planes, dev_buf, mode);
    }
    void slab_vjp_finish(mpm_cot_view* ci, mpm_param_grads* pg) override { aw.slab_vjp_finish(*this, ci, pg); }
    void step_p2g_local() override
    {
        if (status_dirty) {
            reset_status();
            status_dirty = false;
        }
        if (!keys_valid || prof) { // keys need computing (after upload / import): eager
            p2g_phase();
            return;
        }
        // replay a graph of the phase; recapture when the particle count changed (migration)
        if (!slab_g1[cur] || slab_g1_n[cur] != n) {
            slab_g1_launches = capture(slab_g1[cur], [&] { p2g_phase(); });
            slab_g1_n[cur] = n;
        }
        CK(cudaGraphLaunch(slab_g1[cur], stream));
        launches += slab_g1_launches;
    }
    void halo(int plane_lo, int n_planes, void* dev_buf, int mode) override
    {
        HaloFields<T> H{};
        H.nf = 1 + 2 * D;
        H.f[0] = G.m;
        for (int a = 0; a < D; ++a) {
            H.f[1 + a] = G.p[a];
            H.f[1 + D + a] = G.f[a];
        }
        halo_fields(H, plane_lo, n_planes, dev_buf, mode);
    }
    void halo_fields(const HaloFields<T>& H, int plane_lo, int n_planes, void* dev_buf, int mode)
    {
        int64_t per = n_planes;
        for (int a = 1; a < D; ++a)
            per *= sc.cells[a] + 1;
        launch("k_halo", [&] {
            k_halo<T, D><<<grid_for(per, 256), 256, 0, stream>>>(H, nflag, d_nnb, d_cells, plane_lo, n_planes,
                                                                 static_cast<T*>(dev_buf), mode);
        }); // stream-ordered: the caller's transport runs on the same stream (mpm_ctx_set_stream)
    }
    void finish_phase(bool guard)
    {
        grid_kernel<G_BANDONLY | G_GRAV | G_ZEROV | G_MOM | G_CORR | G_STORE>();
        if (guard)
            g2p_kernel_fl<P_CONSTIT | P_GUARD>();
        else
            g2p_kernel_fl<P_CONSTIT>();
        launch("k_step_end", [&] { k_step_end<<<1, 1, 0, stream>>>(st); });
    }
    void step_finish_local(uint32_t flags) override
    {
        const bool guard = flags & MPM_ADV_NAN_GUARD;
        if (prof) {
            finish_phase(guard);
        } else {
            cudaGraphExec_t& ge = slab_g2[guard][cur];
            if (!ge)
                slab_g2_launches = capture(ge, [&] { finish_phase(guard); });
            CK(cudaGraphLaunch(ge, stream));
            launches += slab_g2_launches;
            cur ^= 1;
            keys_valid = true;
        }
        fetch_status();
        mig_cnt[0] = st_host->mig_lo;
        mig_cnt[1] = st_host->mig_hi;
        const int64_t before = n;
        n = n - n_dead;          // the previous G2P's vacated slots sorted to the end and are gone
        n_dead = mig_cnt[0] + mig_cnt[1];
        (void)before;
        if (st_host->mig_over)
            throw ApiError(MPM_ERR_CUDA, "slab migration buffer overflow (raise mig_cap)");
        check_status(step);
    }
    // finish without a host synchronisation: the (failed, n_lo, n_hi) report lands in device memory
    // behind G2P so the caller's collective can gather it on the same stream; step_commit does the
    // host bookkeeping once the caller has the gathered reports
    void step_finish_async(uint32_t flags, long long* dev_report) override
    {
        const bool guard = flags & MPM_ADV_NAN_GUARD;
        if (prof) {
            finish_phase(guard);
        } else {
            cudaGraphExec_t& ge = slab_g2[guard][cur];
            if (!ge)
                slab_g2_launches = capture(ge, [&] { finish_phase(guard); });
            CK(cudaGraphLaunch(ge, stream));
            launches += slab_g2_launches;
            cur ^= 1;
            keys_valid = true;
        }
        launch("k_report", [&] { k_report<<<1, 1, 0, stream>>>(st, dev_report); });
    }
    void step_commit(int64_t n_lo, int64_t n_hi, int any_failed) override
    {
        mig_cnt[0] = int(n_lo);
        mig_cnt[1] = int(n_hi);
        n = n - n_dead;
        n_dead = n_lo + n_hi;
        if (any_failed) { // raise this rank's own error, if it has one
            fetch_status();
            if (st_host->mig_over)
                throw ApiError(MPM_ERR_CUDA, "slab migration buffer overflow (raise mig_cap)");
            check_status(step);
            return;
        }
        step += 1; // k_step_end advanced the device counter
        time = double(T(step) * sc.dt);
    }
    void migrate_export(void* lo, int* lo_pid, void* hi, int* hi_pid, int64_t cap, int64_t* n_lo, int64_t* n_hi) override
    {
        if (mig_cnt[0] > cap || mig_cnt[1] > cap)
            throw ApiError(MPM_ERR_USAGE, "migration export: destination capacity too small");
        const size_t rb = sizeof(T) * mig.rec;
        if (mig_cnt[0] && lo) {
            CK(cudaMemcpyAsync(lo, mig.lo, mig_cnt[0] * rb, cudaMemcpyDeviceToDevice, stream));
            CK(cudaMemcpyAsync(lo_pid, mig.lo_pid, mig_cnt[0] * sizeof(int), cudaMemcpyDeviceToDevice, stream));
        }
        if (mig_cnt[1] && hi) {
            CK(cudaMemcpyAsync(hi, mig.hi, mig_cnt[1] * rb, cudaMemcpyDeviceToDevice, stream));
            CK(cudaMemcpyAsync(hi_pid, mig.hi_pid, mig_cnt[1] * sizeof(int), cudaMemcpyDeviceToDevice, stream));
        }
        *n_lo = mig_cnt[0];
        *n_hi = mig_cnt[1];
    }
    void migrate_import(const void* recs, const int* pids, int64_t k) override
    {
        inc_invalidate();
        if (k <= 0)
            return;
        if (n + k > cap)
            throw ApiError(MPM_ERR_USAGE, "migration import exceeds the context capacity");
        // deterministic append order: by particle id
        int* keys_in = static_cast<int*>(aw_ids_scratch(4 * k)); // 4k ints: pid copy, sorted, order
        int* sorted = keys_in + k;
        int* order = keys_in + 2 * k;
        CK(cudaMemcpyAsync(keys_in, pids, k * sizeof(int), cudaMemcpyDeviceToDevice, stream));
        size_t bytes = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys_in, sorted, iota, order, int(k), 0, 31, stream));
        void* tmp = nullptr;
        CK(cudaMallocAsync(&tmp, bytes, stream));
        CK(cub::DeviceRadixSort::SortPairs(tmp, bytes, keys_in, sorted, iota, order, int(k), 0, 31, stream));
        launch("k_mig_unpack", [&] {
            k_mig_unpack<T, D><<<grid_for(k, 256), 256, 0, stream>>>(buf[cur], int(n), int(k), static_cast<const T*>(recs),
                                                                     pids, order, mig.rec, has_aff, has_F);
        });
        CK(cudaFreeAsync(tmp, stream));
        n += k;
        keys_valid = false;
    }
    void download_local(mpm_state_view* s, int64_t* ids) override
    {
        // compact download of the alive slots in storage order, with their global ids
        int* idx = static_cast<int*>(aw_ids_scratch(2 * n + 2)); // n slot indices + count (2n ints fit)
        int* d_num = idx + n;
        size_t bytes = 0;
        CK(cub::DeviceSelect::If(nullptr, bytes, iota, idx, d_num, int(n), AliveSlot{buf[cur].pid}, stream));
        void* tmp = nullptr;
        CK(cudaMallocAsync(&tmp, bytes > 0 ? bytes : 1, stream));
        CK(cub::DeviceSelect::If(tmp, bytes, iota, idx, d_num, int(n), AliveSlot{buf[cur].pid}, stream));
        CK(cudaFreeAsync(tmp, stream));
        int k = 0;
        CK(cudaMemcpyAsync(&k, d_num, sizeof(int), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        if (k > cap)
            throw ApiError(MPM_ERR_CUDA, "download_local: count exceeds capacity");
        long long* dids = nullptr;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&dids), sizeof(long long) * (k > 0 ? k : 1), stream));
        launch("k_download", [&] {
            k_download_compact<T, D><<<grid_for(k, 256), 256, 0, stream>>>(stage, buf[cur], idx, k, has_aff, has_F, dids);
        });
        void* dst[S_NFIELDS] = {s->x, s->v, s->mass, s->volume, s->rho, s->eps_eq, D == 2 ? s->sigma_zz : nullptr,
                                s->sigma, s->grad_v, has_aff ? s->affine : nullptr, has_F ? s->def_grad : nullptr};
        for (int f = 0; f < S_NFIELDS; ++f)
            if (dst[f] && k)
                CK(cudaMemcpyAsync(dst[f], stage.f[f], (size_t)k * stage_comps<D>(f) * sizeof(T), cudaMemcpyDeviceToHost,
                                   stream));
        if (k)
            CK(cudaMemcpyAsync(ids, dids, sizeof(long long) * k, cudaMemcpyDeviceToHost, stream));
        CK(cudaFreeAsync(dids, stream));
        CK(cudaStreamSynchronize(stream));
        s->n = k;
        s->step = step;
        s->time = time;
    }

    // ---- small transfer helpers (used by the adjoint workspace) ---------------------------------
    void copy_async(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind)
    {
        CK(cudaMemcpyAsync(dst, src, bytes, kind, stream));
    }
    void sync() { CK(cudaStreamSynchronize(stream)); }
    void h2d(T* dst, const T* src, int64_t k) { CK(cudaMemcpyAsync(dst, src, k * sizeof(T), cudaMemcpyHostToDevice, stream)); CK(cudaStreamSynchronize(stream)); }
    void d2h(T* dst, const T* src, int64_t k) { CK(cudaMemcpyAsync(dst, src, k * sizeof(T), cudaMemcpyDeviceToHost, stream)); CK(cudaStreamSynchronize(stream)); }
    void zero(T* dst, int64_t k) { if (dst) CK(cudaMemsetAsync(dst, 0, k * sizeof(T), stream)); }
    void h2d_raw(void* dst, const void* src, size_t b) { CK(cudaMemcpyAsync(dst, src, b, cudaMemcpyHostToDevice, stream)); CK(cudaStreamSynchronize(stream)); }
    void d2h_raw(void* dst, const void* src, size_t b) { CK(cudaMemcpyAsync(dst, src, b, cudaMemcpyDeviceToHost, stream)); CK(cudaStreamSynchronize(stream)); }

    // every device array of a particle buffer, for slot copies
    std::vector<std::pair<void*, size_t>> pbuf_arrays(const PBuf<T, D>& P)
    {
        std::vector<std::pair<void*, size_t>> v;
        for (int a = 0; a < D; ++a) {
            v.push_back({P.x[a], sizeof(T)});
            v.push_back({P.v[a], sizeof(T)});
        }
        v.push_back({P.m, sizeof(T)});
        v.push_back({P.V, sizeof(T)});
        v.push_back({P.rho, sizeof(T)});
        v.push_back({P.eps, sizeof(T)});
        if (D == 2)
            v.push_back({P.szz, sizeof(T)});
        for (int q = 0; q < C::NS; ++q)
            v.push_back({P.sig[q], sizeof(T)});
        for (int k = 0; k < D * D; ++k) {
            v.push_back({P.gv[k], sizeof(T)});
            if (has_aff)
                v.push_back({P.aff[k], sizeof(T)});
            if (has_F)
                v.push_back({P.F[k], sizeof(T)});
        }
        v.push_back({P.pid, sizeof(int)});
        return v;
    }
    void pbuf_copy(const PBuf<T, D>& dst, const PBuf<T, D>& src)
    {
        if (dst.base == inc_src.base)
            inc_invalidate();
        auto d = pbuf_arrays(dst), s = pbuf_arrays(src);
        for (size_t i = 0; i < d.size(); ++i)
            CK(cudaMemcpyAsync(d[i].first, s[i].first, n * s[i].second, cudaMemcpyDeviceToDevice, stream));
    }
    // backprop's checkpoint / replay particle buffers, kept across calls (allocation of several
    // GB per call dominated a short backprop); released with the context
    std::vector<PBuf<T, D>> bp_pool;
    std::vector<void*> bp_pool_mem;

    // ---- replay tape (backprop): per segment-replay step, the sort arrays (pointer-swapped in,
    // no copies) and the active grid blocks, so that step_vjp skips its forward replay
    // (sort + P2G + grid); a step whose grid outgrew its slot falls back to the replay
    struct SortSet {
        int *keys_sorted, *perm, *bstart, *bend, *lstart, *occ, *act, *counts;
        unsigned char* nflag;
    };
    SortSet sort_set() const { return {keys_sorted, perm, bstart, bend, lstart, occ, act, counts, nflag}; }
    void use_sort_set(const SortSet& s)
    {
        keys_sorted = s.keys_sorted;
        perm = s.perm;
        bstart = s.bstart;
        bend = s.bend;
        lstart = s.lstart;
        occ = s.occ;
        act = s.act;
        counts = s.counts;
        nflag = s.nflag;
        own_set = s.keys_sorted == ks_own[0] || s.keys_sorted == ks_own[1];
    }
    struct TapeSlot {
        SortSet ss{};
        T* grid = nullptr;
    };
    std::vector<TapeSlot> tape;
    bool tape_enabled = !(std::getenv("MPM_TAPE") && std::getenv("MPM_TAPE")[0] == '0');
    std::vector<void*> tape_mem;
    int64_t tape_grid_cap = 0; // node blocks per slot
    int* tape_over = nullptr;  // [slots] overflow flags
    void tape_free()
    {
        for (void* p : tape_mem)
            cudaFree(p);
        tape_mem.clear();
        tape.clear();
        tape_over = nullptr;
        tape_grid_cap = 0;
    }
    size_t tape_slot_bytes(int64_t grid_cap) const
    {
        return sizeof(int) * (2 * size_t(cap) + size_t(sc.nb_total) * (3 + C::B + 1) + size_t(sc.nnb_total) + 4) +
               size_t(sc.nnb_total) + sizeof(T) * size_t(grid_cap) * C::NB * (1 + 4 * D);
    }
    // slots for `L` replay steps with `grid_cap` node blocks each; false when HBM is short
    bool tape_reserve(int64_t L, int64_t grid_cap)
    {
        if (int64_t(tape.size()) >= L && tape_grid_cap >= grid_cap)
            return true;
        tape_free();
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        if (double(tape_slot_bytes(grid_cap)) * double(L) > 0.5 * double(fr))
            return false;
        auto al = [&](auto*& p, size_t k) {
            CK(cudaMalloc(reinterpret_cast<void**>(&p), (k ? k : 1) * sizeof(*p)));
            tape_mem.push_back(p);
        };
        tape.resize(L);
        for (auto& t : tape) {
            al(t.ss.keys_sorted, cap);
            al(t.ss.perm, cap);
            al(t.ss.bstart, sc.nb_total);
            al(t.ss.bend, sc.nb_total);
            al(t.ss.lstart, (size_t)sc.nb_total * (C::B + 1));
            al(t.ss.occ, sc.nb_total);
            al(t.ss.act, sc.nnb_total);
            al(t.ss.counts, 4);
            al(t.ss.nflag, sc.nnb_total);
            al(t.grid, (size_t)grid_cap * C::NB * (1 + 4 * D));
        }
        al(tape_over, L);
        tape_grid_cap = grid_cap;
        return true;
    }
    template <bool SAVE> void tape_grid(int j)
    {
        const int64_t per = tape_grid_cap * C::NB * (1 + 4 * D);
        const unsigned blocks = unsigned(std::min<int64_t>((per + 255) / 256, int64_t(nsm) * 16));
        launch(SAVE ? "k_tape_save" : "k_tape_load", [&] {
            k_grid_tape<T, D, SAVE><<<std::max(1u, blocks), 256, 0, stream>>>(G, act, counts + 1, tape[j].grid,
                                                                             int(tape_grid_cap), tape_over + j);
        });
    }
    PBuf<T, D> pool_buf(size_t k)
    {
        while (bp_pool.size() <= k)
            bp_pool.push_back(pbuf_alloc(bp_pool_mem));
        return bp_pool[k];
    }
    PBuf<T, D> pbuf_alloc(std::vector<void*>& owned)
    {
        PBuf<T, D> P{};
        const size_t before = allocs.size();
        alloc_pbuf(P);
        for (size_t i = before; i < allocs.size(); ++i)
            owned.push_back(allocs[i]);
        allocs.resize(before); // owned by the caller
        return P;
    }
    uint64_t digest_of(const PBuf<T, D>& P)
    {
        CK(cudaMemsetAsync(d_red, 0, sizeof(unsigned long long), stream));
        launch("k_digest", [&] { k_digest<T, D><<<grid_for(n, 256), 256, 0, stream>>>(P, int(n), has_aff, d_red); });
        unsigned long long h = 0;
        CK(cudaMemcpyAsync(&h, d_red, sizeof(h), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        return h;
    }

    // ---- adjoint (kernels_adj.cuh) -------------------------------------------------------------
    // backprop_trajectory (checkpoint.hpp:72-143): forward sweep keeping segment-start states in
    // HBM slots (+ a device digest at every boundary), then per segment (reversed): replay into
    // L+1 slots, digest check against the sweep (checkpoint.hpp:124-126), seed + step_vjp per step.
    void backprop_run(AdjWork<T, D>& aw, const mpm_state_view* s0, int64_t total, int nseg, const mpm_seeder_desc* sd,
                      mpm_cot_view* c0, mpm_param_grads* pg, mpm_backprop_result* res)
    {
        if (total < 1)
            throw ApiError(MPM_ERR_VALIDATION, "checkpoint plan: need at least one step");
        if (nseg < 1 || int64_t(nseg) > total)
            throw ApiError(MPM_ERR_VALIDATION, "checkpoint plan: n_segments must lie in [1, N_t]");
        std::vector<int64_t> bnd(nseg + 1, 0);
        {
            const int64_t base = total / nseg, rem = total % nseg;
            int64_t at = 0;
            for (int k = 0; k < nseg; ++k) {
                at += base + (k < rem ? 1 : 0);
                bnd[k + 1] = at;
            }
        }
        int64_t Lmax = 0;
        for (int k = 0; k < nseg; ++k)
            Lmax = std::max(Lmax, bnd[k + 1] - bnd[k]);
        upload(s0);
        aw.ensure(*this);
        const int64_t step0 = step;
        const PBuf<T, D> own0 = buf[0], own1 = buf[1];
        const int cur0 = cur;
        // seeder tables on the device
        const bool eul = sd && sd->kind == MPM_SEEDER_EULERIAN_LS && sd->n_obs > 0;
        const bool seeding = (sd && sd->kind == MPM_SEEDER_LAGRANGIAN_LS && sd->n_obs > 0) || eul;
        const int64_t nsel = seeding ? (eul ? sd->n_regions : (sd->sel ? sd->n_sel : n)) : 0;
        struct Owned { // seeder tables: released on every exit path (validation throws included)
            std::vector<void*> v;
            void push_back(void* p) { v.push_back(p); }
            ~Owned()
            {
                for (void* p : v)
                    cudaFree(p);
            }
        } owned;
        long long* d_sel = nullptr;
        T* d_tgt = nullptr;
        T *d_cen = nullptr, *d_half = nullptr, *d_epart = nullptr, *d_g = nullptr;
        unsigned char* d_mask = nullptr;
        const int eblocks = int(grid_for(n, 256));
        if (eul) {
            if (sd->n_regions < 1 || sd->n_regions > EUL_MAXREG || !sd->centers || !sd->half)
                throw ApiError(MPM_ERR_VALIDATION, "seeder: Eulerian needs 1.." + std::to_string(EUL_MAXREG) +
                                                       " regions with centers and half sizes");
            auto dev = [&](auto*& p, size_t bytes, const void* src) {
                CK(cudaMalloc(reinterpret_cast<void**>(&p), bytes));
                owned.push_back(p);
                if (src)
                    h2d_raw(p, src, bytes);
            };
            dev(d_cen, (size_t)nsel * D * sizeof(T), sd->centers);
            dev(d_half, (size_t)nsel * D * sizeof(T), sd->half);
            if (sd->mask)
                dev(d_mask, (size_t)sd->n_obs * nsel, sd->mask);
            dev(d_epart, (size_t)eblocks * nsel * (D + 1) * sizeof(T), nullptr);
            dev(d_g, (size_t)nsel * D * sizeof(T), nullptr);
        }
        T* d_lblk = nullptr; // per-block loss partials of the Lagrangian seeder
        if (seeding && !eul) {
            CK(cudaMalloc(&d_lblk, sizeof(T) * std::max<int64_t>(1, grid_for(nsel, 256))));
            owned.push_back(d_lblk);
        }
        if (seeding) {
            if (sd->sel && !eul) {
                CK(cudaMalloc(&d_sel, nsel * sizeof(long long)));
                owned.push_back(d_sel);
                std::vector<long long> hs(sd->sel, sd->sel + nsel);
                for (long long p : hs)
                    if (p < 0 || p >= n)
                        throw ApiError(MPM_ERR_VALIDATION, "seeder: particle index out of range");
                h2d_raw(d_sel, hs.data(), nsel * sizeof(long long));
            }
            CK(cudaMalloc(&d_tgt, (size_t)sd->n_obs * nsel * D * sizeof(T)));
            owned.push_back(d_tgt);
            h2d_raw(d_tgt, sd->target, (size_t)sd->n_obs * nsel * D * sizeof(T));
        }
        auto obs_index = [&](int64_t t) {
            if (!seeding)
                return -1;
            for (int k = 0; k < sd->n_obs; ++k)
                if (sd->obs_steps[k] == t)
                    return k;
            return -1;
        };
        auto seed = [&](const PBuf<T, D>& P, int k, int cb, int do_cot) {
            if (eul) {
                launch("k_seed", [&] {
                    k_eul_partial<T, D><<<eblocks, 256, 0, stream>>>(P, int(n), d_cen, d_half, int(nsel), sd->field,
                                                                     d_epart);
                });
                launch("k_seed", [&] {
                    k_eul_final<T, D><<<1, EUL_MAXREG, 0, stream>>>(d_epart, eblocks, int(nsel),
                                                                    d_tgt + (size_t)k * nsel * D,
                                                                    d_mask ? d_mask + (size_t)k * nsel : nullptr,
                                                                    d_g, aw.loss_acc);
                });
                if (do_cot)
                    launch("k_seed", [&] {
                        k_eul_seed<T, D><<<eblocks, 256, 0, stream>>>(P, int(n), d_cen, d_half, int(nsel), d_g,
                                                                      sd->field, aw.cot[cb]);
                    });
                return;
            }
            launch("k_slot_of_pid", [&] { k_slot_of_pid<T, D><<<grid_for(n, 256), 256, 0, stream>>>(P, int(n), aw.slot_of_pid); });
            const int sb = int(grid_for(nsel, 256));
            launch("k_seed", [&] {
                k_seed_lagrangian<T, D><<<sb, 256, 0, stream>>>(P, int(n), aw.slot_of_pid, d_sel, nsel,
                                                                d_tgt + (size_t)k * nsel * D, sd->field, aw.cot[cb],
                                                                do_cot, d_lblk);
            });
            launch("k_seed", [&] { k_seed_sum<T><<<1, 1024, 0, stream>>>(d_lblk, sb, aw.loss_acc); });
        };
        const SortSet own_ss = sort_set();
        try {
            std::vector<PBuf<T, D>> ckpt(nseg), replay(Lmax + 1);
            for (int k = 0; k < nseg; ++k) // checkpoint and replay slots persist across calls
                ckpt[k] = pool_buf(size_t(k));
            for (int64_t j = 0; j <= Lmax; ++j)
                replay[j] = pool_buf(size_t(nseg + j));
            std::vector<uint64_t> bhash(nseg + 1);
            CK(cudaMemsetAsync(aw.loss_acc, 0, sizeof(double), stream));
            struct Ev { // released on every exit path
                cudaEvent_t e{};
                Ev() { CK(cudaEventCreate(&e)); }
                ~Ev() { cudaEventDestroy(e); }
            } ev0, ev1;
            CK(cudaEventRecord(ev0.e, stream));
            // replay tape, sized by the active node blocks of the latest forward step (+25 %)
            bool use_tape = false;
            auto reserve_tape = [&](bool fresh) {
                if (fresh) { // no step of this trajectory ran yet: size from S0's own active blocks
                    keys_valid = false;
                    sort_and_segment();
                    keys_valid = false;
                }
                int n_act_now = 0;
                d2h_raw(&n_act_now, counts + 1, sizeof(int));
                const char* cap_env = std::getenv("MPM_TAPE_CAP"); // test hook: force slot overflows
                const int64_t grid_cap =
                    cap_env ? std::max<int64_t>(1, std::atoll(cap_env))
                            : std::min<int64_t>(sc.nnb_total, (int64_t(n_act_now) * 5 / 4 + 255) / 256 * 256);
                use_tape = tape_enabled && n > 0 && tape_reserve(Lmax, grid_cap);
                if (use_tape)
                    CK(cudaMemsetAsync(tape_over, 0, sizeof(int) * Lmax, stream));
            };
            // one step of a segment kept in the replay slots: S^j -> S^{j+1}, with its tape entry
            auto slot_step = [&](int64_t j) {
                buf[0] = replay[j];
                buf[1] = replay[j + 1];
                cur = 0;
                keys_valid = false;
                if (use_tape) {
                    use_sort_set(tape[j].ss);
                    step_once(false, true);
                    tape_grid<true>(int(j));
                    use_sort_set(own_ss);
                } else {
                    step_once(false);
                }
            };
            // forward sweep. The last segment runs directly in the replay slots (and fills the
            // tape): its states are the ones a replay would recompute bit for bit, so the reverse
            // sweep starts without replaying it. With one segment (a plan whose L_max + 1 replay
            // slots fit in HBM) nothing is replayed at all.
            const bool last_kept = tape_enabled && n > 0;
            reset_status();
            if (obs_index(0) >= 0)
                seed(buf[cur], obs_index(0), 0, 0);
            for (int k = 0; k < nseg; ++k) {
                pbuf_copy(ckpt[k], buf[cur]);
                if (k >= 1) // digests only where a replayed segment ends (S^0 is never checked)
                    bhash[k] = digest_of(buf[cur]);
                if (k == nseg - 1 && last_kept) {
                    reserve_tape(bnd[k] == 0);
                    pbuf_copy(replay[0], buf[cur]);
                    for (int64_t t = bnd[k]; t < bnd[k + 1]; ++t) {
                        slot_step(t - bnd[k]);
                        if (obs_index(t + 1) >= 0)
                            seed(buf[cur], obs_index(t + 1), 0, 0);
                    }
                    continue;
                }
                for (int64_t t = bnd[k]; t < bnd[k + 1]; ++t) {
                    step_once(false);
                    if (obs_index(t + 1) >= 0)
                        seed(buf[cur], obs_index(t + 1), 0, 0);
                }
            }
            if (!last_kept)
                bhash[nseg] = digest_of(buf[cur]);
            check_status(step0);
            double loss = 0;
            d2h_raw(&loss, aw.loss_acc, sizeof(double));
            if (!last_kept)
                reserve_tape(false);
            std::vector<int> over(Lmax, 1);
            // backward sweep
            aw.cot_zero(*this, 0);
            aw.pg_reset(*this, pg);
            int cb = 0;
            int64_t peak = 0;
            for (int k = nseg - 1; k >= 0; --k) {
                const int64_t b0 = bnd[k], b1 = bnd[k + 1], len = b1 - b0;
                const bool kept = k == nseg - 1 && last_kept;
                if (!kept) {
                    pbuf_copy(replay[0], ckpt[k]);
                    for (int64_t j = 0; j < len; ++j)
                        slot_step(j);
                }
                peak = std::max(peak, len + 1);
                if (!kept && digest_of(replay[len]) != bhash[k + 1])
                    throw ApiError(MPM_ERR_CHECKPOINT,
                                   "checkpoint mismatch: recomputed segment end differs from the recorded state at step "
                                       + std::to_string(step0 + b1));
                if (use_tape) { // the digest read synchronised the stream
                    d2h_raw(over.data(), tape_over, sizeof(int) * len);
                    CK(cudaMemsetAsync(tape_over, 0, sizeof(int) * len, stream));
                }
                for (int64_t t = b1; t > b0; --t) {
                    if (obs_index(t) >= 0)
                        seed(replay[t - b0], obs_index(t), cb, 1);
                    const int64_t j = t - b0 - 1;
                    buf[0] = replay[j];
                    buf[1] = replay[j + 1];
                    cur = 0;
                    keys_valid = false;
                    if (use_tape && !over[j]) { // the step's sort and grid from the replay
                        use_sort_set(tape[j].ss);
                        tape_grid<false>(int(j));
                        aw.vjp_reverse(*this, cb, cb ^ 1);
                    } else {
                        use_sort_set(own_ss);
                        aw.vjp_enqueue(*this, cb, cb ^ 1);
                    }
                    cb ^= 1;
                }
                use_sort_set(own_ss);
                check_status(step);
            }
            if (obs_index(0) >= 0)
                seed(ckpt[0], obs_index(0), cb, 1);
            CK(cudaEventRecord(ev1.e, stream));
            CK(cudaStreamSynchronize(stream));
            float dev_ms = 0;
            CK(cudaEventElapsedTime(&dev_ms, ev0.e, ev1.e));
            aw.cot_download(*this, c0, cb);
            aw.pg_download(*this, pg);
            if (res) {
                res->loss = loss;
                res->checkpoints_stored = nseg;
                res->peak_replay_states = peak;
                res->device_ms = dev_ms;
            }
            // restore the context's own buffers holding S0
            buf[0] = own0;
            buf[1] = own1;
            cur = cur0;
            pbuf_copy(buf[cur], ckpt[0]);
            step = step0;
            keys_valid = false;
            CK(cudaStreamSynchronize(stream));
        } catch (...) {
            use_sort_set(own_ss);
            buf[0] = own0;
            buf[1] = own1;
            cur = cur0;
            keys_valid = false;
            cudaStreamSynchronize(stream);
            throw;
        }
    }

    void step_vjp(const mpm_state_view* s, const mpm_cot_view* co, mpm_cot_view* ci, mpm_param_grads* pg) override
    {
        aw.step_vjp_api(*this, s, co, ci, pg);
    }
    void backprop(const mpm_state_view* s0, int64_t total, int nseg, const mpm_seeder_desc* sd, mpm_cot_view* c0,
                  mpm_param_grads* pg, mpm_backprop_result* res) override
    {
        aw.backprop_api(*this, s0, total, nseg, sd, c0, pg, res);
    }
};

} // namespace

// ---------------------------------------------------------------------------------------------
struct mpm_ctx {
    std::unique_ptr<CtxBase> impl;
    int code = 0;
    int64_t particle = -1, step = -1;
    std::string msg;
};

template <class F> static int guarded(mpm_ctx* c, F&& f)
{
    if (c) {
        c->code = 0;
        c->particle = -1;
        c->step = -1;
        c->msg.clear();
    }
    try {
        f();
        return MPM_OK;
    } catch (const ApiError& e) {
        if (c) {
            c->code = e.code;
            c->particle = e.particle;
            c->step = e.step;
            c->msg = e.what();
        }
        return e.code;
    } catch (const std::exception& e) {
        if (c) {
            c->code = MPM_ERR_USAGE;
            c->msg = e.what();
        }
        return MPM_ERR_USAGE;
    }
}

extern "C" {

int mpm_version(void) { return MPM_CAPI_VERSION; }

int mpm_device_name(char* buf, size_t len)
{
    cudaDeviceProp p{};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&p, dev) != cudaSuccess)
        return MPM_ERR_CUDA;
    std::snprintf(buf, len, "%s (sm_%d%d, %d SMs)", p.name, p.major, p.minor, p.multiProcessorCount);
    return MPM_OK;
}

int mpm_ctx_create(const mpm_scene_desc* d, int64_t max_particles, int device, mpm_ctx** out)
{
    if (!d || !out || max_particles < 0)
        return MPM_ERR_USAGE;
    *out = nullptr;
    static thread_local mpm_ctx scratch;
    return guarded(&scratch, [&] {
        std::unique_ptr<mpm_ctx> c(new mpm_ctx);
        if (d->dim == 2 && d->dtype == MPM_F64)
            c->impl.reset(new Ctx<double, 2>(d, max_particles, device));
        else if (d->dim == 3 && d->dtype == MPM_F64)
            c->impl.reset(new Ctx<double, 3>(d, max_particles, device));
        else if (d->dim == 2 && d->dtype == MPM_F32)
            c->impl.reset(new Ctx<float, 2>(d, max_particles, device));
        else if (d->dim == 3 && d->dtype == MPM_F32)
            c->impl.reset(new Ctx<float, 3>(d, max_particles, device));
        else
            throw ApiError(MPM_ERR_USAGE, "dim must be 2 or 3 and dtype MPM_F32 or MPM_F64");
        *out = c.release();
    });
}

void mpm_ctx_destroy(mpm_ctx* c) { delete c; }

int mpm_last_error(const mpm_ctx* c, int* code, int64_t* particle, int64_t* step, char* msg, size_t len)
{
    if (!c)
        return MPM_ERR_USAGE;
    if (code)
        *code = c->code;
    if (particle)
        *particle = c->particle;
    if (step)
        *step = c->step;
    if (msg && len) {
        std::strncpy(msg, c->msg.c_str(), len - 1);
        msg[len - 1] = 0;
    }
    return MPM_OK;
}

#define MPM_CALL(c, body)                                                                          \
    do {                                                                                           \
        if (!(c))                                                                                  \
            return MPM_ERR_USAGE;                                                                  \
        return guarded(c, [&] { body; });                                                          \
    } while (0)

int mpm_state_upload(mpm_ctx* c, const mpm_state_view* s) { MPM_CALL(c, c->impl->upload(s)); }
int mpm_state_download(mpm_ctx* c, mpm_state_view* s) { MPM_CALL(c, c->impl->download(s)); }
int mpm_state_digest(mpm_ctx* c, uint64_t* out) { MPM_CALL(c, *out = c->impl->digest()); }
int mpm_max_speed(mpm_ctx* c, double* v) { MPM_CALL(c, *v = c->impl->max_speed()); }
int mpm_advance(mpm_ctx* c, int64_t n, uint32_t flags) { MPM_CALL(c, c->impl->advance(n, flags)); }
int mpm_advance_timed(mpm_ctx* c, int64_t n, uint32_t flags, double* ms)
{
    MPM_CALL(c, {
        double t = c->impl->advance_timed(n, flags);
        if (ms)
            *ms = t;
    });
}
int mpm_p2g(mpm_ctx* c) { MPM_CALL(c, c->impl->phase_p2g()); }
int mpm_grid_momentum_update(mpm_ctx* c) { MPM_CALL(c, c->impl->phase_mom()); }
int mpm_grid_corrections(mpm_ctx* c) { MPM_CALL(c, c->impl->phase_corr()); }
int mpm_g2p(mpm_ctx* c) { MPM_CALL(c, c->impl->phase_g2p()); }
int mpm_constitutive(mpm_ctx* c) { MPM_CALL(c, c->impl->phase_constit()); }
int mpm_grid_download(mpm_ctx* c, mpm_grid_view* g) { MPM_CALL(c, c->impl->grid_download(g)); }
int mpm_grid_upload(mpm_ctx* c, const mpm_grid_view* g) { MPM_CALL(c, c->impl->grid_upload(g)); }
int mpm_step_vjp(mpm_ctx* c, const mpm_state_view* s, const mpm_cot_view* co, mpm_cot_view* ci, mpm_param_grads* pg)
{
    MPM_CALL(c, c->impl->step_vjp(s, co, ci, pg));
}
int mpm_backprop(mpm_ctx* c, const mpm_state_view* s0, int64_t total, int nseg, const mpm_seeder_desc* sd,
                 mpm_cot_view* c0, mpm_param_grads* pg, mpm_backprop_result* res)
{
    MPM_CALL(c, c->impl->backprop(s0, total, nseg, sd, c0, pg, res));
}

int mpm_state_upload_ids(mpm_ctx* c, const mpm_state_view* s, const int64_t* ids) { MPM_CALL(c, c->impl->upload_ids(s, ids)); }
int mpm_state_download_local(mpm_ctx* c, mpm_state_view* s, int64_t* ids) { MPM_CALL(c, c->impl->download_local(s, ids)); }
int mpm_slab_set(mpm_ctx* c, int cell_lo, int cell_hi, int64_t mig_cap) { MPM_CALL(c, c->impl->slab_set(cell_lo, cell_hi, mig_cap)); }
int mpm_step_p2g_local(mpm_ctx* c) { MPM_CALL(c, c->impl->step_p2g_local()); }
int mpm_step_grid_interior(mpm_ctx* c) { MPM_CALL(c, c->impl->step_grid_interior()); }
int mpm_snapshot_begin(mpm_ctx* c, int slot) { MPM_CALL(c, c->impl->snapshot_begin(slot)); }
int mpm_snapshot_fetch(mpm_ctx* c, int slot, mpm_state_view* s) { MPM_CALL(c, c->impl->snapshot_fetch(slot, s)); }
int mpm_init_scene(mpm_ctx* c, const mpm_region* regions, int n_regions, double mass, double volume, double rho0,
                   int64_t* n_out)
{
    MPM_CALL(c, c->impl->init_scene_dev(regions, n_regions, mass, volume, rho0, n_out));
}
int mpm_slab_vjp_begin(mpm_ctx* c, const mpm_cot_view* cot_out) { MPM_CALL(c, c->impl->slab_vjp_begin(cot_out)); }
int mpm_slab_vjp_interior(mpm_ctx* c) { MPM_CALL(c, c->impl->slab_vjp_interior()); }
int mpm_slab_vjp_scatter(mpm_ctx* c) { MPM_CALL(c, c->impl->slab_vjp_scatter()); }
int mpm_halo_cot(mpm_ctx* c, int plane_lo, int n_planes, void* dev_buf, int mode)
{
    MPM_CALL(c, c->impl->halo_cot(plane_lo, n_planes, dev_buf, mode));
}
int mpm_slab_vjp_finish(mpm_ctx* c, mpm_cot_view* cot_in, mpm_param_grads* pg)
{
    MPM_CALL(c, c->impl->slab_vjp_finish(cot_in, pg));
}
int mpm_halo(mpm_ctx* c, int plane_lo, int n_planes, void* dev_buf, int mode) { MPM_CALL(c, c->impl->halo(plane_lo, n_planes, dev_buf, mode)); }
int mpm_step_finish_local(mpm_ctx* c, uint32_t flags) { MPM_CALL(c, c->impl->step_finish_local(flags)); }
int mpm_step_finish_async(mpm_ctx* c, uint32_t flags, int64_t* dev_report)
{
    MPM_CALL(c, c->impl->step_finish_async(flags, reinterpret_cast<long long*>(dev_report)));
}
int mpm_step_commit(mpm_ctx* c, int64_t n_lo, int64_t n_hi, int any_failed)
{
    MPM_CALL(c, c->impl->step_commit(n_lo, n_hi, any_failed));
}
int mpm_migrate_export(mpm_ctx* c, void* lo, int* lo_pid, void* hi, int* hi_pid, int64_t cap, int64_t* n_lo, int64_t* n_hi)
{
    MPM_CALL(c, c->impl->migrate_export(lo, lo_pid, hi, hi_pid, cap, n_lo, n_hi));
}
int mpm_migrate_import(mpm_ctx* c, const void* recs, const int* pids, int64_t k) { MPM_CALL(c, c->impl->migrate_import(recs, pids, k)); }
int mpm_particle_record_size(const mpm_ctx* c) { return c ? c->impl->rec_size() : -1; }
int64_t mpm_local_count(const mpm_ctx* c) { return c ? c->impl->local_count() : -1; }
int mpm_ctx_set_stream(mpm_ctx* c, void* stream) { MPM_CALL(c, c->impl->set_stream(stream)); }
int mpm_migrate_counts(const mpm_ctx* c, int64_t* n_lo, int64_t* n_hi)
{
    if (!c || !n_lo || !n_hi)
        return MPM_ERR_USAGE;
    c->impl->migrate_counts(n_lo, n_hi);
    return MPM_OK;
}

int mpm_profile_enable(mpm_ctx* c, int enable) { MPM_CALL(c, c->impl->prof = enable != 0); }

int mpm_profile_reset(mpm_ctx* c)
{
    MPM_CALL(c, {
        for (auto& e : c->impl->events) {
            cudaEventDestroy(e.a);
            cudaEventDestroy(e.b);
        }
        c->impl->events.clear();
        c->impl->prof_acc.clear();
    });
}

int mpm_profile_query(mpm_ctx* c, const char* name, double* ms, int64_t* launches)
{
    MPM_CALL(c, {
        double tot = 0;
        int64_t k = 0;
        for (auto& e : c->impl->events) {
            if (name && *name && !std::strstr(e.name, name))
                continue;
            float t = 0;
            CK(cudaEventSynchronize(e.b));
            CK(cudaEventElapsedTime(&t, e.a, e.b));
            tot += t;
            ++k;
        }
        if (ms)
            *ms = tot;
        if (launches)
            *launches = k;
    });
}

int64_t mpm_launch_count(const mpm_ctx* c) { return c ? c->impl->launches : -1; }

int mpm_dist_unique_id(void* id_out)
{
    if (!id_out)
        return MPM_ERR_USAGE;
    ncclUniqueId id;
    if (dyn::ncclGetUniqueId(&id) != ncclSuccess)
        return MPM_ERR_CUDA;
    std::memcpy(id_out, &id, sizeof(id));
    return MPM_OK;
}
int mpm_dist_attach_nccl(mpm_ctx* c, int rank, int nranks, const void* nccl_id, int cell_lo, int cell_hi,
                         int64_t mig_cap)
{
    if (!nccl_id)
        return MPM_ERR_USAGE;
    MPM_CALL(c, c->impl->dist_attach(rank, nranks, cell_lo, cell_hi, mig_cap, nccl_id));
}
int mpm_dist_attach_local(mpm_ctx* const* ctxs, int nranks, const int* bounds, int64_t mig_cap)
{
    if (!ctxs || nranks < 1 || !bounds)
        return MPM_ERR_USAGE;
    for (int r = 0; r < nranks; ++r) {
        const int rc = guarded(ctxs[r], [&] {
            if (!ctxs[r])
                throw ApiError(MPM_ERR_USAGE, "null context");
            ctxs[r]->impl->dist_attach(r, nranks, bounds[r], bounds[r + 1], mig_cap, nullptr);
        });
        if (rc)
            return rc;
    }
    return MPM_OK;
}
int mpm_dist_advance(mpm_ctx* c, int64_t n_steps, uint32_t flags, double* device_ms)
{
    MPM_CALL(c, c->impl->dist_advance(n_steps, flags, device_ms));
}
int mpm_dist_advance_local(mpm_ctx* const* ctxs, int nranks, int64_t n_steps, uint32_t flags)
{
    if (!ctxs || nranks < 1)
        return MPM_ERR_USAGE;
    std::vector<CtxBase*> all(nranks);
    for (int r = 0; r < nranks; ++r) {
        if (!ctxs[r])
            return MPM_ERR_USAGE;
        all[r] = ctxs[r]->impl.get();
    }
    int rc = guarded(ctxs[0], [&] { all[0]->dist_enqueue_local(all, n_steps, flags); });
    if (rc)
        return rc;
    for (int r = 0; r < nranks; ++r) { // every rank's status once, after the call
        const int e = guarded(ctxs[r], [&] { all[r]->dist_finish(); });
        if (e && !rc)
            rc = e;
    }
    return rc;
}

int mpm_dist_backprop(mpm_ctx* c, int64_t total, int nseg, const mpm_seeder_desc* sd, int64_t id_space,
                      mpm_cot_view* c0, int64_t* c0_ids, mpm_param_grads* pg, mpm_backprop_result* res)
{
    MPM_CALL(c, c->impl->dist_backprop_nccl(total, nseg, sd, id_space, c0, c0_ids, pg, res));
}
int mpm_dist_backprop_local(mpm_ctx* const* ctxs, int nranks, int64_t total, int nseg, const mpm_seeder_desc* sd,
                            int64_t id_space, mpm_cot_view* c0s, int64_t* const* c0_ids, mpm_param_grads* pg,
                            mpm_backprop_result* res)
{
    if (!ctxs || nranks < 1 || !c0s || !c0_ids || !pg)
        return MPM_ERR_USAGE;
    for (int r = 0; r < nranks; ++r)
        if (!ctxs[r])
            return MPM_ERR_USAGE;
    std::unique_ptr<LocalHub> hub;
    int rc = guarded(ctxs[0], [&] { hub = std::make_unique<LocalHub>(nranks); });
    if (rc)
        return rc;
    // ranks other than 0 write their (identical, rank-ordered) ParamGrads into scratch copies
    std::vector<std::vector<std::vector<double>>> fr(nranks, std::vector<std::vector<double>>(6));
    std::vector<mpm_param_grads> pgs(nranks, *pg);
    for (int r = 1; r < nranks; ++r)
        for (int w = 0; w < 6; ++w)
            if (pg->wall_friction[w]) {
                fr[r][w].assign(MAX_FRIC, 0.0);
                pgs[r].wall_friction[w] = fr[r][w].data();
            }
    std::vector<mpm_backprop_result> rs(nranks);
    std::vector<int> codes(nranks, 0);
    std::vector<std::thread> th;
    for (int r = 0; r < nranks; ++r)
        th.emplace_back([&, r] {
            codes[r] = guarded(ctxs[r], [&] {
                try {
                    ctxs[r]->impl->dist_backprop_local(hub.get(), total, nseg, sd, id_space, &c0s[r], c0_ids[r],
                                                       r == 0 ? pg : &pgs[r], &rs[r]);
                } catch (...) {
                    hub->fail();
                    throw;
                }
            });
        });
    for (auto& t : th)
        t.join();
    if (res)
        *res = rs[0];
    for (int r = 0; r < nranks; ++r)
        if (codes[r])
            return codes[r];
    return MPM_OK;
}

int mpm_grid_stats(mpm_ctx* c, int64_t* an, int64_t* ob, int64_t* anb) { MPM_CALL(c, c->impl->grid_stats(an, ob, anb)); }

} // extern "C"
