// mpm_gpu.hpp -- C++ drop-in layer over the C ABI (include/mpm_capi.h) for callers of the reference
// solver API (/root/reference/proj/include/mpm, namespace mpm).
//
// It takes the reference's own types (Scene, SimState, StateCotangent, ParamGrads, Grid,
// CheckpointPlan) and passes their std::vector<Eigen::Matrix> storage to the ABI without copying
// (vectors [n][d], matrices column-major: exactly the ABI's host layout). Errors come back as the
// reference's exception types (common.hpp:22-36).
//
//   mpm::gpu::Stepper<T,dim>          stepper.hpp:49-70   (Stepper::grid is a host mirror)
//   mpm::gpu::run                     stepper.hpp:91-122
//   mpm::gpu::constitutive_update     stepper.hpp:15-43
//   mpm::gpu::step_vjp                adjoint.hpp:328-525
//   mpm::gpu::backprop_trajectory     checkpoint.hpp:72-143 (built-in device seeder, or any
//                                     duck-typed Seeder through a host-orchestrated sweep)
//
// include/mpm_gpu/mpm/stepper.hpp re-exports these under the reference's own names, so a caller
// that includes "mpm/stepper.hpp" with include/mpm_gpu first on the include path runs on the GPU
// unchanged. This header must not include the reference's mpm/stepper.hpp.
#pragma once

#include "../mpm_capi.h"

#include <mpm/constitutive.hpp>
#include <mpm/contact.hpp>
#include <mpm/scene.hpp>
#include <mpm/transfer.hpp>

#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

namespace mpm {
namespace gpu {

template <class T> constexpr int dtype_of() { return std::is_same_v<T, double> ? MPM_F64 : MPM_F32; }

[[noreturn]] inline void rethrow(mpm_ctx* c, int rc)
{
    int code = rc;
    int64_t particle = -1, step = -1;
    char msg[1024] = {0};
    if (c)
        mpm_last_error(c, &code, &particle, &step, msg, sizeof(msg));
    std::string m = msg[0] ? msg : ("libmpm_b200 status " + std::to_string(rc));
    switch (rc) {
    case MPM_ERR_VALIDATION:
        throw ValidationError(m);
    case MPM_ERR_OUT_OF_DOMAIN:
        throw OutOfDomainError(particle, m);
    case MPM_ERR_NUMERICAL:
    case MPM_ERR_CHECKPOINT:
        throw NumericalError(m);
    default:
        throw std::runtime_error(m);
    }
}

// Scene<T,dim> -> mpm_scene_desc (owns the friction / obstacle arrays it points to)
template <class T, int dim> struct SceneDesc {
    mpm_scene_desc d{};
    std::vector<std::vector<double>> fr;
    std::vector<double> ob;

    explicit SceneDesc(const Scene<T, dim>& s)
    {
        const auto& c = s.config;
        d.dim = dim;
        d.dtype = dtype_of<T>();
        d.dh = double(c.dh);
        for (int a = 0; a < dim; ++a) {
            d.cells[a] = c.cells[a];
            d.origin[a] = double(c.origin[a]);
            d.gravity[a] = double(c.gravity[a]);
        }
        d.dt = double(c.dt);
        d.scheme = int(c.scheme.kind);
        d.alpha_flip = double(c.scheme.alpha_flip);
        d.track_def_grad = c.track_def_grad ? 1 : 0;
        if (std::holds_alternative<FluidParams<T>>(s.material)) {
            const auto& f = std::get<FluidParams<T>>(s.material);
            d.material = MPM_MAT_FLUID;
            d.rho0 = double(f.rho0);
            d.viscosity = double(f.viscosity);
            d.sound_speed = double(f.sound_speed);
            d.rate_form = f.rate_form ? 1 : 0;
        } else {
            const auto& p = std::get<DruckerPragerParams<T>>(s.material);
            d.material = MPM_MAT_DRUCKER_PRAGER;
            d.rho0 = double(p.rho0);
            d.K = double(p.K);
            d.nu = double(p.nu);
            d.G = double(p.G);
            d.phi = double(p.phi);
            d.psi = double(p.psi);
            d.cohesion = double(p.cohesion);
            d.sigma_t = double(p.sigma_t);
            d.q_phi = double(p.q_phi);
            d.k_phi = double(p.k_phi);
            d.q_psi = double(p.q_psi);
            d.tau_P = double(p.tau_P);
            d.alpha_P = double(p.alpha_P);
        }
        d.band_layers = s.boundary.band_layers;
        fr.resize(2 * dim);
        for (int w = 0; w < 2 * dim; ++w) {
            d.wall_kind[w] = int(s.boundary.walls[w].kind);
            for (T mu : s.boundary.walls[w].friction)
                fr[w].push_back(double(mu));
            d.n_friction[w] = int(fr[w].size());
            d.friction[w] = fr[w].empty() ? nullptr : fr[w].data();
        }
        for (const auto& o : s.obstacles) {
            for (int a = 0; a < dim; ++a)
                ob.push_back(double(o.lo[a]));
            for (int a = 0; a < dim; ++a)
                ob.push_back(double(o.hi[a]));
        }
        d.n_obstacles = int(s.obstacles.size());
        d.obstacles = ob.empty() ? nullptr : ob.data();
        d.mass_epsilon = double(s.mass_epsilon);
    }
};

template <class V> void* ptr_or_null(V& v) { return v.empty() ? nullptr : static_cast<void*>(v.data()); }
template <class V> const void* cptr_or_null(const V& v)
{
    return v.empty() ? nullptr : static_cast<const void*>(v.data());
}

// SimState<T,dim> <-> mpm_state_view: the reference's vectors are passed as they are
template <class T, int dim> mpm_state_view state_view(SimState<T, dim>& s)
{
    auto& p = s.particles;
    mpm_state_view v{};
    v.n = p.size();
    v.x = ptr_or_null(p.x);
    v.v = ptr_or_null(p.v);
    v.mass = ptr_or_null(p.mass);
    v.volume = ptr_or_null(p.volume);
    v.rho = ptr_or_null(p.rho);
    v.eps_eq = ptr_or_null(p.eps_eq);
    v.sigma_zz = dim == 2 ? ptr_or_null(p.sigma_zz) : nullptr;
    v.sigma = ptr_or_null(p.sigma);
    v.grad_v = ptr_or_null(p.grad_v);
    v.affine = ptr_or_null(p.affine);
    v.def_grad = ptr_or_null(p.def_grad);
    v.step = s.step;
    v.time = double(s.time);
    return v;
}

// StateCotangent<T,dim> (adjoint.hpp:10-72) -> mpm_cot_view (generic: adjoint.hpp is optional here)
template <class Cot> mpm_cot_view cot_view(Cot& c)
{
    mpm_cot_view v{};
    v.n = Index(c.x.size());
    v.x = ptr_or_null(c.x);
    v.v = ptr_or_null(c.v);
    v.rho = ptr_or_null(c.rho);
    v.volume = ptr_or_null(c.volume);
    v.eps_eq = ptr_or_null(c.eps_eq);
    v.sigma_zz = ptr_or_null(c.sigma_zz);
    v.sigma = ptr_or_null(c.sigma);
    v.grad_v = ptr_or_null(c.grad_v);
    v.affine = ptr_or_null(c.affine);
    return v;
}

template <class T, int dim> mpm_grid_view grid_view(Grid<T, dim>& g)
{
    mpm_grid_view v{};
    v.num_nodes = Index(g.num_nodes());
    v.mass = ptr_or_null(g.mass);
    v.momentum = ptr_or_null(g.momentum);
    v.v_old = ptr_or_null(g.v_old);
    v.v = ptr_or_null(g.v);
    v.force = ptr_or_null(g.force);
    return v;
}

// one device context per scene (RAII)
template <class T, int dim> class Context {
public:
    Context(const Scene<T, dim>& s, Index max_particles, int device = 0)
        : desc_(s)
    {
        int rc = mpm_ctx_create(&desc_.d, max_particles, device, &h_);
        if (rc)
            rethrow(nullptr, rc);
        cap_ = max_particles;
    }
    ~Context()
    {
        if (h_)
            mpm_ctx_destroy(h_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

    Index capacity() const { return cap_; }
    mpm_ctx* handle() { return h_; }
    void check(int rc)
    {
        if (rc)
            rethrow(h_, rc);
    }
    void upload(SimState<T, dim>& s)
    {
        auto v = state_view(s);
        check(mpm_state_upload(h_, &v));
    }
    void download(SimState<T, dim>& s)
    {
        auto v = state_view(s);
        check(mpm_state_download(h_, &v));
        s.step = v.step;
        s.time = T(v.time);
    }
    void advance(Index n, bool nan_guard, bool store_grid = false)
    {
        check(mpm_advance(h_, n, (nan_guard ? MPM_ADV_NAN_GUARD : 0u) | (store_grid ? MPM_ADV_STORE_GRID : 0u)));
    }
    void grid_download(Grid<T, dim>& g)
    {
        auto v = grid_view(g);
        check(mpm_grid_download(h_, &v));
    }

private:
    SceneDesc<T, dim> desc_;
    mpm_ctx* h_ = nullptr;
    Index cap_ = 0;
};

// ---- forward ---------------------------------------------------------------------------
template <class T, int dim> struct Stepper {
    const Scene<T, dim>* scene;
    Grid<T, dim> grid; // host mirror (the device grid is derived data, state.hpp:89-90)

    explicit Stepper(const Scene<T, dim>& s)
        : scene(&s)
    {
        grid.configure(s.config.cells, s.config.dh, s.config.origin);
    }

    void advance(SimState<T, dim>& state)
    {
        ensure(state.particles.size());
        ctx_->upload(state);
        ctx_->advance(1, false, true);
        ctx_->download(state);
    }
    // refresh the host mirror of the step's grid (Stepper::grid in the reference)
    Grid<T, dim>& fetch_grid()
    {
        if (ctx_)
            ctx_->grid_download(grid);
        return grid;
    }

private:
    std::unique_ptr<Context<T, dim>> ctx_;
    void ensure(Index n)
    {
        if (!ctx_ || ctx_->capacity() < n)
            ctx_ = std::make_unique<Context<T, dim>>(*scene, n);
    }
};

template <class T, int dim> struct RunResult {
    std::vector<SimState<T, dim>> snapshots;
    double seconds_per_1000_steps = 0;
};

template <class T, int dim> T max_particle_speed(const SimState<T, dim>& state)
{
    T vmax = T(0);
    for (const auto& v : state.particles.v)
        vmax = std::max(vmax, v.norm());
    return vmax;
}

// run (stepper.hpp:91-122): CFL refusal, NaN guard every step, snapshots at the stride, the
// observer after every step (which forces a per-step download of state and grid). Steps between
// snapshots run as one device call.
template <class T, int dim>
RunResult<T, dim> run(const Scene<T, dim>& scene, SimState<T, dim> state, Index num_steps, Index stride,
                      bool force = false,
                      const std::type_identity_t<std::function<void(const SimState<T, dim>&, const Grid<T, dim>&)>>&
                          observer = {})
{
    T courant = cfl_report(scene.config, scene.material, gpu::max_particle_speed(state));
    if (courant > T(1) && !force)
        throw ValidationError("run: Courant number " + std::to_string(double(courant))
                              + " > 1; refusing to start (use force to override)");
    RunResult<T, dim> result;
    result.snapshots.push_back(state);
    if (num_steps <= 0)
        return result;
    Context<T, dim> ctx(scene, state.particles.size());
    ctx.upload(state);
    Grid<T, dim> grid;
    grid.configure(scene.config.cells, scene.config.dh, scene.config.origin);
    const Index step0 = state.step;
    auto t0 = std::chrono::steady_clock::now();
    Index done = 0;
    while (done < num_steps) {
        Index chunk = num_steps - done;
        if (observer)
            chunk = 1;
        else if (stride > 0) {
            const Index r = (step0 + done) % stride;
            chunk = std::min(chunk, stride - r);
        }
        ctx.advance(chunk, true, bool(observer));
        done += chunk;
        const Index cur = step0 + done;
        const bool snap = stride > 0 && cur % stride == 0 && cur != num_steps; // stepper.hpp:112
        if (observer || snap)
            ctx.download(state);
        if (observer) {
            ctx.grid_download(grid);
            observer(state, grid);
        }
        if (snap)
            result.snapshots.push_back(state);
    }
    auto t1 = std::chrono::steady_clock::now();
    ctx.download(state);
    result.snapshots.push_back(state);
    result.seconds_per_1000_steps = std::chrono::duration<double>(t1 - t0).count() / double(num_steps) * 1000.0;
    return result;
}

// constitutive_update (stepper.hpp:15-43) on the device
template <class T, int dim> void constitutive_update(ParticleSoA<T, dim>& prt, const Material<T>& material, T dt)
{
    Scene<T, dim> s;
    s.config.dh = T(1);
    for (int a = 0; a < dim; ++a)
        s.config.cells[a] = 8;
    s.config.dt = dt;
    s.config.track_def_grad = !prt.def_grad.empty();
    s.config.scheme.kind = prt.affine.empty() ? SchemeKind::pic : SchemeKind::apic;
    s.material = material;
    SimState<T, dim> st;
    st.particles = prt;
    // positions are irrelevant to the constitutive phase; keep them in-domain for upload checks
    for (auto& x : st.particles.x)
        for (int a = 0; a < dim; ++a)
            x[a] = T(4);
    Context<T, dim> ctx(s, prt.size());
    ctx.upload(st);
    ctx.check(mpm_constitutive(ctx.handle()));
    ctx.download(st);
    for (Index p = 0; p < prt.size(); ++p) {
        prt.sigma[p] = st.particles.sigma[p];
        prt.rho[p] = st.particles.rho[p];
        prt.volume[p] = st.particles.volume[p];
        prt.eps_eq[p] = st.particles.eps_eq[p];
        if (dim == 2)
            prt.sigma_zz[p] = st.particles.sigma_zz[p];
        if (!prt.def_grad.empty())
            prt.def_grad[p] = st.particles.def_grad[p];
    }
}

// ---- multi-GPU: the library-owned slab decomposition (mpm_dist_*) -------------
// The decomposed Stepper::advance (stepper.hpp:59-69) for a C++ caller: rank r owns the particles
// whose base cell along x, floor((x - o) / dh - 1/2) (bspline.hpp:79-91), lies in
// [bounds[r], bounds[r + 1]) -- bounds are multiples of the particle-block edge (16 cells in 2-D,
// 8 in 3-D). The library does the halo exchange, the migration and the error reduction on the
// device; a call of advance(n) has no host synchronisation inside.
template <class T, int dim>
std::vector<std::vector<Index>> slab_partition(const Scene<T, dim>& scene, const SimState<T, dim>& s,
                                               const std::vector<int>& bounds)
{
    const int R = int(bounds.size()) - 1;
    std::vector<std::vector<Index>> out(R);
    for (Index i = 0; i < s.particles.size(); ++i) {
        const double u = double((s.particles.x[i][0] - scene.config.origin[0]) / scene.config.dh);
        const int b = int(std::floor(u - 0.5));
        int r = 0;
        while (r + 1 < R && b >= bounds[r + 1])
            ++r;
        out[r].push_back(i);
    }
    return out;
}

template <class T, int dim> SimState<T, dim> take_rows(const SimState<T, dim>& s, const std::vector<Index>& ids)
{
    SimState<T, dim> o;
    const auto& p = s.particles;
    auto& q = o.particles;
    q.resize(Index(ids.size()), !p.affine.empty(), !p.def_grad.empty());
    for (std::size_t k = 0; k < ids.size(); ++k) {
        const Index i = ids[k];
        q.x[k] = p.x[i];
        q.v[k] = p.v[i];
        q.mass[k] = p.mass[i];
        q.volume[k] = p.volume[i];
        q.rho[k] = p.rho[i];
        q.eps_eq[k] = p.eps_eq[i];
        if (dim == 2)
            q.sigma_zz[k] = p.sigma_zz[i];
        q.sigma[k] = p.sigma[i];
        q.grad_v[k] = p.grad_v[i];
        if (!p.affine.empty())
            q.affine[k] = p.affine[i];
        if (!p.def_grad.empty())
            q.def_grad[k] = p.def_grad[i];
    }
    o.step = s.step;
    o.time = s.time;
    return o;
}

template <class T, int dim> void put_rows(SimState<T, dim>& s, const SimState<T, dim>& sub, const std::vector<Index>& ids)
{
    auto& p = s.particles;
    const auto& q = sub.particles;
    for (std::size_t k = 0; k < ids.size(); ++k) {
        const Index i = ids[k];
        p.x[i] = q.x[k];
        p.v[i] = q.v[k];
        p.mass[i] = q.mass[k];
        p.volume[i] = q.volume[k];
        p.rho[i] = q.rho[k];
        p.eps_eq[i] = q.eps_eq[k];
        if (dim == 2)
            p.sigma_zz[i] = q.sigma_zz[k];
        p.sigma[i] = q.sigma[k];
        p.grad_v[i] = q.grad_v[k];
        if (!p.affine.empty())
            p.affine[i] = q.affine[k];
        if (!p.def_grad.empty())
            p.def_grad[i] = q.def_grad[k];
    }
    s.step = sub.step;
    s.time = sub.time;
}

// one rank's context: upload of its subset (with global ids) and the compact download
template <class T, int dim> class SlabContext : public Context<T, dim> {
public:
    SlabContext(const Scene<T, dim>& s, Index capacity, int device)
        : Context<T, dim>(s, capacity, device)
    {
    }
    void upload_subset(SimState<T, dim>& sub, const std::vector<Index>& ids)
    {
        auto v = state_view(sub);
        std::vector<int64_t> id64(ids.begin(), ids.end());
        this->check(mpm_state_upload_ids(this->handle(), &v, id64.data()));
    }
    // this rank's live particles and their global ids
    SimState<T, dim> download_subset(std::vector<Index>& ids, bool with_affine, bool with_def_grad)
    {
        const Index k = Index(mpm_local_count(this->handle()));
        SimState<T, dim> sub;
        sub.particles.resize(k, with_affine, with_def_grad);
        auto v = state_view(sub);
        std::vector<int64_t> id64(std::max<Index>(k, 1));
        this->check(mpm_state_download_local(this->handle(), &v, id64.data()));
        auto& q = sub.particles; // keep the first v.n rows
        const std::size_t m = std::size_t(v.n);
        q.x.resize(m);
        q.v.resize(m);
        q.mass.resize(m);
        q.volume.resize(m);
        q.rho.resize(m);
        q.eps_eq.resize(m);
        q.sigma_zz.resize(dim == 2 ? m : 0);
        q.sigma.resize(m);
        q.grad_v.resize(m);
        q.affine.resize(with_affine ? m : 0);
        q.def_grad.resize(with_def_grad ? m : 0);
        ids.assign(id64.begin(), id64.begin() + v.n);
        sub.step = v.step;
        sub.time = T(v.time);
        return sub;
    }
};

inline Index slab_capacity(Index n_local, Index n_total, int R, Index mig_cap)
{
    return std::max<Index>(1024, Index(1.25 * double(n_local)) + n_total / (4 * R) + 2 * mig_cap);
}

// all ranks in this process (R contexts, e.g. R slabs on one GPU): the library steps them in
// lock-step with device-copy exchanges (mpm_dist_attach_local / mpm_dist_advance_local)
template <class T, int dim> class SlabGroup {
public:
    SlabGroup(const Scene<T, dim>& scene, const SimState<T, dim>& state, std::vector<int> bounds, Index mig_cap = 0,
              int device = 0)
        : bounds_(std::move(bounds)), template_(state)
    {
        const int R = int(bounds_.size()) - 1;
        const Index n = state.particles.size();
        mig_cap_ = mig_cap > 0 ? mig_cap : std::max<Index>(256, n / (64 * R));
        const auto parts = slab_partition(scene, state, bounds_);
        for (int r = 0; r < R; ++r) {
            ctxs_.push_back(std::make_unique<SlabContext<T, dim>>(
                scene, slab_capacity(Index(parts[r].size()), n, R, mig_cap_), device));
            SimState<T, dim> sub = take_rows(state, parts[r]);
            ctxs_.back()->upload_subset(sub, parts[r]);
            handles_.push_back(ctxs_.back()->handle());
        }
        int rc = mpm_dist_attach_local(handles_.data(), R, bounds_.data(), mig_cap_);
        if (rc)
            ctxs_[0]->check(rc);
    }
    void advance(Index n, bool nan_guard = false)
    {
        const int rc = mpm_dist_advance_local(handles_.data(), int(handles_.size()), n,
                                              nan_guard ? MPM_ADV_NAN_GUARD : 0u);
        if (!rc)
            return;
        for (auto& c : ctxs_) { // the failing rank's own error first, then the peer report
            int code = 0;
            char msg[512];
            mpm_last_error(c->handle(), &code, nullptr, nullptr, msg, sizeof(msg));
            if (code && !std::strstr(msg, "another rank"))
                c->check(code);
        }
        ctxs_[0]->check(rc);
    }
    // the global state in particle-index order
    SimState<T, dim> gather()
    {
        SimState<T, dim> out = template_;
        const bool aff = !template_.particles.affine.empty(), F = !template_.particles.def_grad.empty();
        for (auto& c : ctxs_) {
            std::vector<Index> ids;
            SimState<T, dim> sub = c->download_subset(ids, aff, F);
            put_rows(out, sub, ids);
        }
        return out;
    }
    int ranks() const { return int(ctxs_.size()); }

private:
    std::vector<int> bounds_;
    SimState<T, dim> template_;
    Index mig_cap_ = 0;
    std::vector<std::unique_ptr<SlabContext<T, dim>>> ctxs_;
    std::vector<mpm_ctx*> handles_;
};

// this process's rank of an NCCL-connected decomposition (one process per GPU)
template <class T, int dim> class SlabRank {
public:
    using Id = std::array<unsigned char, MPM_DIST_ID_BYTES>;
    static Id unique_id()
    {
        Id id{};
        const int rc = mpm_dist_unique_id(id.data());
        if (rc)
            rethrow(nullptr, rc);
        return id;
    }
    SlabRank(const Scene<T, dim>& scene, SimState<T, dim> local, const std::vector<Index>& ids, int rank, int nranks,
             const Id& id, int cell_lo, int cell_hi, Index n_total, Index mig_cap = 0, int device = 0)
        : aff_(!local.particles.affine.empty()), F_(!local.particles.def_grad.empty())
    {
        mig_cap = mig_cap > 0 ? mig_cap : std::max<Index>(1024, n_total / (256 * nranks));
        ctx_ = std::make_unique<SlabContext<T, dim>>(
            scene, slab_capacity(local.particles.size(), n_total, nranks, mig_cap), device);
        ctx_->upload_subset(local, ids);
        ctx_->check(mpm_dist_attach_nccl(ctx_->handle(), rank, nranks, id.data(), cell_lo, cell_hi, mig_cap));
    }
    // n steps; returns their device time (ms)
    double advance(Index n, bool nan_guard = false)
    {
        double ms = 0;
        ctx_->check(mpm_dist_advance(ctx_->handle(), n, nan_guard ? MPM_ADV_NAN_GUARD : 0u, &ms));
        return ms;
    }
    SimState<T, dim> download(std::vector<Index>& ids) { return ctx_->download_subset(ids, aff_, F_); }

private:
    bool aff_, F_;
    std::unique_ptr<SlabContext<T, dim>> ctx_;
};

} // namespace gpu
} // namespace mpm
