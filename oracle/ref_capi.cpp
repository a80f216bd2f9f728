// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Wraps the UNMODIFIED reference (/root/reference/proj/include/mpm, compiled against the
// Eigen-API shim) behind the stateless oracle ABI (mpm_oracle.h, prefix ref_). Every entry
// point converts the plain host views into the reference's own types, calls the reference
// function named in the comment, and converts back. No arithmetic of the method lives here.
// Built by oracle/Makefile into oracle/_ref/libmpm_ref.so.

#include "mpm_oracle.h"

#include <mpm/checkpoint.hpp>
#include <mpm/scene.hpp>
#include <mpm/stepper.hpp>

#include <cstring>
#include <string>

namespace {

thread_local int64_t g_err_particle = -1;
thread_local std::string g_err_msg;

template <class T, int dim>
mpm::Scene<T, dim> make_scene(const mpm_scene_desc* d)
{
    using namespace mpm;
    Scene<T, dim> s;
    s.config.dh = T(d->dh);
    for (int a = 0; a < dim; ++a) {
        s.config.cells[a] = d->cells[a];
        s.config.origin[a] = T(d->origin[a]);
        s.config.gravity[a] = T(d->gravity[a]);
    }
    s.config.dt = T(d->dt);
    s.config.scheme.kind = static_cast<SchemeKind>(d->scheme);
    s.config.scheme.alpha_flip = T(d->alpha_flip);
    s.config.track_def_grad = d->track_def_grad != 0;
    if (d->material == MPM_MAT_FLUID) {
        FluidParams<T> f;
        f.rho0 = T(d->rho0);
        f.viscosity = T(d->viscosity);
        f.sound_speed = T(d->sound_speed);
        f.rate_form = d->rate_form != 0;
        s.material = f;
    } else {
        DruckerPragerParams<T> p;
        p.rho0 = T(d->rho0);
        p.K = T(d->K);
        p.nu = T(d->nu);
        p.G = T(d->G);
        p.phi = T(d->phi);
        p.psi = T(d->psi);
        p.cohesion = T(d->cohesion);
        p.sigma_t = T(d->sigma_t);
        p.q_phi = T(d->q_phi);
        p.k_phi = T(d->k_phi);
        p.q_psi = T(d->q_psi);
        p.tau_P = T(d->tau_P);
        p.alpha_P = T(d->alpha_P);
        s.material = p;
    }
    s.boundary.band_layers = d->band_layers;
    for (int w = 0; w < 2 * dim; ++w) {
        s.boundary.walls[w].kind = static_cast<WallKind>(d->wall_kind[w]);
        s.boundary.walls[w].friction.clear();
        for (int k = 0; k < d->n_friction[w]; ++k)
            s.boundary.walls[w].friction.push_back(T(d->friction[w][k]));
    }
    for (int o = 0; o < d->n_obstacles; ++o) {
        Obstacle<T, dim> ob;
        for (int a = 0; a < dim; ++a) {
            ob.lo[a] = T(d->obstacles[o * 2 * dim + a]);
            ob.hi[a] = T(d->obstacles[o * 2 * dim + dim + a]);
        }
        s.obstacles.push_back(ob);
    }
    s.mass_epsilon = T(d->mass_epsilon);
    return s;
}

template <class T, int dim>
void add_regions(mpm::Scene<T, dim>& s, const orc_region* r, int nreg)
{
    using namespace mpm;
    for (int i = 0; i < nreg; ++i) {
        GeometryRegion<T, dim> g;
        g.shape = r[i].shape == 0 ? RegionShape::box : RegionShape::cylinder;
        for (int a = 0; a < dim; ++a) {
            g.lo[a] = T(r[i].lo[a]);
            g.hi[a] = T(r[i].hi[a]);
            g.center[a] = T(r[i].center[a]);
            g.velocity.value[a] = T(r[i].value[a]);
        }
        g.radius = T(r[i].radius);
        g.zmin = T(r[i].zmin);
        g.zmax = T(r[i].zmax);
        g.velocity.kind = static_cast<VelExprKind>(r[i].vel_kind);
        g.velocity.alpha = T(r[i].alpha);
        g.velocity.h0 = T(r[i].h0);
        g.velocity.amplitude = T(r[i].amplitude);
        g.velocity.perturbation = T(r[i].perturbation);
        g.velocity.frequency = T(r[i].frequency);
        s.geometry.push_back(g);
    }
}

template <class E>
void copy_in(std::vector<E>& dst, const void* src, int64_t n)
{
    if (!src) {
        dst.clear();
        return;
    }
    dst.resize(static_cast<std::size_t>(n));
    std::memcpy(static_cast<void*>(dst.data()), src, sizeof(E) * static_cast<std::size_t>(n));
}

template <class E>
void copy_out(const std::vector<E>& src, void* dst)
{
    if (dst && !src.empty())
        std::memcpy(dst, static_cast<const void*>(src.data()), sizeof(E) * src.size());
}

template <class T, int dim>
mpm::SimState<T, dim> state_in(const mpm_state_view* v)
{
    mpm::SimState<T, dim> s;
    auto& p = s.particles;
    copy_in(p.x, v->x, v->n);
    copy_in(p.v, v->v, v->n);
    copy_in(p.mass, v->mass, v->n);
    copy_in(p.volume, v->volume, v->n);
    copy_in(p.rho, v->rho, v->n);
    copy_in(p.eps_eq, v->eps_eq, v->n);
    if (dim == 2)
        copy_in(p.sigma_zz, v->sigma_zz, v->n);
    if (dim == 2 && p.sigma_zz.empty())
        p.sigma_zz.assign(static_cast<std::size_t>(v->n), T(0));
    copy_in(p.sigma, v->sigma, v->n);
    copy_in(p.grad_v, v->grad_v, v->n);
    copy_in(p.affine, v->affine, v->n);
    copy_in(p.def_grad, v->def_grad, v->n);
    s.step = v->step;
    s.time = T(v->time);
    return s;
}

template <class T, int dim>
void state_out(const mpm::SimState<T, dim>& s, mpm_state_view* v)
{
    const auto& p = s.particles;
    v->n = p.size();
    copy_out(p.x, v->x);
    copy_out(p.v, v->v);
    copy_out(p.mass, v->mass);
    copy_out(p.volume, v->volume);
    copy_out(p.rho, v->rho);
    copy_out(p.eps_eq, v->eps_eq);
    copy_out(p.sigma_zz, v->sigma_zz);
    copy_out(p.sigma, v->sigma);
    copy_out(p.grad_v, v->grad_v);
    copy_out(p.affine, v->affine);
    copy_out(p.def_grad, v->def_grad);
    v->step = s.step;
    v->time = double(s.time);
}

template <class T, int dim>
mpm::StateCotangent<T, dim> cot_in_view(const mpm_cot_view* c, const mpm::ParticleSoA<T, dim>& prt)
{
    auto k = mpm::StateCotangent<T, dim>::zeros_like(prt);
    auto get = [&](auto& dst, const void* src) {
        if (src && !dst.empty())
            std::memcpy(static_cast<void*>(dst.data()), src, sizeof(dst[0]) * dst.size());
    };
    get(k.x, c->x);
    get(k.v, c->v);
    get(k.rho, c->rho);
    get(k.volume, c->volume);
    get(k.eps_eq, c->eps_eq);
    get(k.sigma_zz, c->sigma_zz);
    get(k.sigma, c->sigma);
    get(k.grad_v, c->grad_v);
    get(k.affine, c->affine);
    return k;
}

template <class T, int dim>
void cot_out_view(const mpm::StateCotangent<T, dim>& k, mpm_cot_view* c)
{
    copy_out(k.x, c->x);
    copy_out(k.v, c->v);
    copy_out(k.rho, c->rho);
    copy_out(k.volume, c->volume);
    copy_out(k.eps_eq, c->eps_eq);
    copy_out(k.sigma_zz, c->sigma_zz);
    copy_out(k.sigma, c->sigma);
    copy_out(k.grad_v, c->grad_v);
    copy_out(k.affine, c->affine);
}

template <class T, int dim>
mpm::Grid<T, dim> grid_in(const mpm::Scene<T, dim>& sc, const mpm_grid_view* g)
{
    mpm::Grid<T, dim> grid;
    grid.configure(sc.config.cells, sc.config.dh, sc.config.origin);
    auto n = static_cast<int64_t>(grid.num_nodes());
    copy_in(grid.mass, g->mass, n);
    copy_in(grid.momentum, g->momentum, n);
    copy_in(grid.v_old, g->v_old, n);
    copy_in(grid.v, g->v, n);
    copy_in(grid.force, g->force, n);
    return grid;
}

template <class T, int dim>
void grid_out(const mpm::Grid<T, dim>& grid, mpm_grid_view* g)
{
    g->num_nodes = static_cast<int64_t>(grid.num_nodes());
    copy_out(grid.mass, g->mass);
    copy_out(grid.momentum, g->momentum);
    copy_out(grid.v_old, g->v_old);
    copy_out(grid.v, g->v);
    copy_out(grid.force, g->force);
}

template <class F>
int guarded(F&& f)
{
    g_err_particle = -1;
    g_err_msg.clear();
    try {
        return f();
    } catch (const mpm::OutOfDomainError& e) {
        g_err_particle = e.particle;
        g_err_msg = e.what();
        return MPM_ERR_OUT_OF_DOMAIN;
    } catch (const mpm::NumericalError& e) {
        g_err_msg = e.what();
        return std::string(e.what()).find("checkpoint mismatch") != std::string::npos ? MPM_ERR_CHECKPOINT
                                                                                     : MPM_ERR_NUMERICAL;
    } catch (const mpm::ValidationError& e) {
        g_err_msg = e.what();
        return MPM_ERR_VALIDATION;
    } catch (const std::exception& e) {
        g_err_msg = e.what();
        return MPM_ERR_USAGE;
    }
}

// dispatch on (dtype, dim)
template <template <class, int> class Op, class... A>
auto dispatch(const mpm_scene_desc* d, A&&... a)
{
    if (d->dtype == MPM_F64) {
        if (d->dim == 2)
            return Op<double, 2>::run(d, a...);
        return Op<double, 3>::run(d, a...);
    }
    if (d->dim == 2)
        return Op<float, 2>::run(d, a...);
    return Op<float, 3>::run(d, a...);
}

template <class T, int dim>
struct InitCount {
    static int64_t run(const mpm_scene_desc* d, const orc_region* r, int nreg)
    {
        auto sc = make_scene<T, dim>(d);
        add_regions(sc, r, nreg);
        try {
            return mpm::init_scene(sc).particles.size();
        } catch (...) {
            return -1;
        }
    }
};

template <class T, int dim>
struct Init {
    static int run(const mpm_scene_desc* d, const orc_region* r, int nreg, mpm_state_view* out, double* meps)
    {
        return guarded([&] {
            auto sc = make_scene<T, dim>(d);
            add_regions(sc, r, nreg);
            auto s = mpm::init_scene(sc);
            state_out(s, out);
            if (meps)
                *meps = double(sc.mass_epsilon);
            return MPM_OK;
        });
    }
};

template <class T, int dim>
struct Advance {
    static int run(const mpm_scene_desc* d, mpm_state_view* v, int64_t n, int nan_guard)
    {
        return guarded([&] {
            auto sc = make_scene<T, dim>(d);
            auto s = state_in<T, dim>(v);
            mpm::Stepper<T, dim> stepper(sc);
            int rc = MPM_OK;
            try {
                for (int64_t i = 0; i < n; ++i) {
                    stepper.advance(s);
                    if (nan_guard && !s.particles.all_finite())
                        throw mpm::NumericalError("run: non-finite particle field detected at step "
                                                  + std::to_string(s.step));
                }
            } catch (...) {
                state_out(s, v);
                throw;
            }
            state_out(s, v);
            return rc;
        });
    }
};

template <class T, int dim>
struct P2G {
    static int run(const mpm_scene_desc* d, const mpm_state_view* v, mpm_grid_view* g)
    {
        return guarded([&] {
            auto sc = make_scene<T, dim>(d);
            auto s = state_in<T, dim>(v);
            mpm::Grid<T, dim> grid;
            grid.configure(sc.config.cells, sc.config.dh, sc.config.origin);
            mpm::p2g(s.particles, sc.config.scheme, sc.config.gravity, grid);
            grid_out(grid, g);
            return MPM_OK;
        });
    }
};

template <class T, int dim>
struct GridUpdate {
    static int run(const mpm_scene_desc* d, mpm_grid_view* g)
    {
        return guarded([&] {
            auto sc = make_scene<T, dim>(d);
            auto grid = grid_in(sc, g);
            mpm::grid_momentum_update(grid, sc.config.dt, sc.mass_epsilon);
            grid_out(grid, g);
            return MPM_OK;
        });
    }
};

template <class T, int dim>
struct GridCorr {
    static int run(const mpm_scene_desc* d, mpm_grid_view* g)
    {
        return guarded([&] {
            auto sc = make_scene<T, dim>(d);
            auto grid = grid_in(sc, g);
            mpm::apply_grid_corrections(grid, sc.boundary, sc.obstacles);
            grid_out(grid, g);
            return MPM_OK;
        });
    }
};

template <class T, int dim>
struct G2P {
    static int run(const mpm_scene_desc* d, const mpm_grid_view* g, mpm_state_view* v)
    {
        return guarded([&] {
            auto sc = make_scene<T, dim>(d);
            auto grid = grid_in(sc, g);
            auto s = state_in<T, dim>(v);
            mpm::g2p(grid, sc.config.scheme, sc.config.dt, s.particles);
            state_out(s, v);
            return MPM_OK;
        });
    }
};

template <class T, int dim>
struct Constit {
    static int run(const mpm_scene_desc* d, mpm_state_view* v)
    {
        return guarded([&] {
            auto sc = make_scene<T, dim>(d);
            auto s = state_in<T, dim>(v);
            mpm::constitutive_update(s.particles, sc.material, sc.config.dt);
            state_out(s, v);
            return MPM_OK;
        });
    }
};

template <class T, int dim>
mpm::ParamGrads<T, dim> pg_in(const mpm::Scene<T, dim>& sc, const mpm_param_grads* pg)
{
    auto g = mpm::ParamGrads<T, dim>::zeros_like(sc.boundary);
    g.sound_speed = T(pg->sound_speed);
    g.viscosity = T(pg->viscosity);
    for (int w = 0; w < 2 * dim; ++w)
        for (std::size_t k = 0; k < g.wall_friction[w].size(); ++k)
            g.wall_friction[w][k] = pg->wall_friction[w] ? T(pg->wall_friction[w][k]) : T(0);
    return g;
}

template <class T, int dim>
void pg_out(const mpm::ParamGrads<T, dim>& g, mpm_param_grads* pg)
{
    pg->sound_speed = double(g.sound_speed);
    pg->viscosity = double(g.viscosity);
    for (int w = 0; w < 2 * dim; ++w)
        for (std::size_t k = 0; k < g.wall_friction[w].size(); ++k)
            if (pg->wall_friction[w])
                pg->wall_friction[w][k] = double(g.wall_friction[w][k]);
}

template <class T, int dim>
struct Vjp {
    static int run(const mpm_scene_desc* d, const mpm_state_view* v, const mpm_cot_view* co,
                   mpm_cot_view* ci, mpm_param_grads* pg)
    {
        return guarded([&] {
            auto sc = make_scene<T, dim>(d);
            auto s = state_in<T, dim>(v);
            auto cout_ = cot_in_view<T, dim>(co, s.particles);
            mpm::StateCotangent<T, dim> cin;
            auto g = pg_in(sc, pg);
            mpm::AdjointWorkspace<T, dim> ws;
            ws.configure(sc);
            mpm::step_vjp(sc, s, cout_, cin, g, ws);
            cot_out_view(cin, ci);
            pg_out(g, pg);
            return MPM_OK;
        });
    }
};

// Built-in Lagrangian least-squares seeder in the reference's duck-typed Seeder protocol
// (checkpoint.hpp:63-66).
template <class T, int dim>
struct LagrangianSeeder {
    const mpm_seeder_desc* sd;
    int64_t n;
    int find(mpm::Index step) const
    {
        if (!sd || sd->kind != MPM_SEEDER_LAGRANGIAN_LS)
            return -1;
        for (int k = 0; k < sd->n_obs; ++k)
            if (sd->obs_steps[k] == step)
                return k;
        return -1;
    }
    int64_t nsel() const { return sd->sel ? sd->n_sel : n; }
    int64_t pid(int64_t l) const { return sd->sel ? sd->sel[l] : l; }
    const T* target(int k, int64_t l) const
    {
        return static_cast<const T*>(sd->target) + (static_cast<int64_t>(k) * nsel() + l) * dim;
    }
    bool observes(mpm::Index step) const { return find(step) >= 0; }
    T loss_at(mpm::Index step, const mpm::SimState<T, dim>& s) const
    {
        int k = find(step);
        T L = T(0);
        const auto& z = sd->field == 0 ? s.particles.x : s.particles.v;
        for (int64_t l = 0; l < nsel(); ++l) {
            const T* t = target(k, l);
            for (int a = 0; a < dim; ++a) {
                T r = z[pid(l)][a] - t[a];
                L += r * r;
            }
        }
        return L;
    }
    void seed(mpm::Index step, const mpm::SimState<T, dim>& s, mpm::StateCotangent<T, dim>& c) const
    {
        int k = find(step);
        const auto& z = sd->field == 0 ? s.particles.x : s.particles.v;
        auto& zc = sd->field == 0 ? c.x : c.v;
        for (int64_t l = 0; l < nsel(); ++l) {
            const T* t = target(k, l);
            for (int a = 0; a < dim; ++a)
                zc[pid(l)][a] += T(2) * (z[pid(l)][a] - t[a]);
        }
    }
};

template <class T, int dim>
struct Backprop {
    static int run(const mpm_scene_desc* d, const mpm_state_view* v, int64_t total, int nseg,
                   const mpm_seeder_desc* sd, mpm_cot_view* c0, mpm_param_grads* pg, mpm_backprop_result* res)
    {
        return guarded([&] {
            auto sc = make_scene<T, dim>(d);
            auto s = state_in<T, dim>(v);
            auto plan = mpm::CheckpointPlan::make(total, nseg);
            LagrangianSeeder<T, dim> seeder{sd, v->n};
            auto r = mpm::backprop_trajectory(sc, s, plan, seeder);
            cot_out_view(r.initial_state_cot, c0);
            auto g = pg_in(sc, pg);
            g.sound_speed += r.param_grads.sound_speed;
            g.viscosity += r.param_grads.viscosity;
            for (int w = 0; w < 2 * dim; ++w)
                for (std::size_t k = 0; k < g.wall_friction[w].size(); ++k)
                    g.wall_friction[w][k] += r.param_grads.wall_friction[w][k];
            pg_out(g, pg);
            if (res) {
                res->loss = double(r.loss);
                res->checkpoints_stored = r.checkpoints_stored;
                res->peak_replay_states = r.peak_replay_states;
            }
            return MPM_OK;
        });
    }
};

template <class T, int dim>
struct Hash {
    static uint64_t run(const mpm_scene_desc*, const mpm_state_view* v) { return state_in<T, dim>(v).hash(); }
};

template <class T, int dim>
struct RunTimer {
    static double run(const mpm_scene_desc* d, mpm_state_view* v, int64_t n)
    {
        double secs = -1.0;
        guarded([&] {
            auto sc = make_scene<T, dim>(d);
            auto s = state_in<T, dim>(v);
            auto r = mpm::run(sc, s, n, 0, /*force=*/true);
            secs = r.seconds_per_1000_steps;
            state_out(r.snapshots.back(), v);
            return MPM_OK;
        });
        return secs;
    }
};

} // namespace

extern "C" {

int ref_last_error(int64_t* particle, char* msg, size_t len)
{
    if (particle)
        *particle = g_err_particle;
    if (msg && len) {
        std::strncpy(msg, g_err_msg.c_str(), len - 1);
        msg[len - 1] = 0;
    }
    return 0;
}

int ref_dp_make(mpm_scene_desc* d, double rho0, double K, double nu, double phi, double psi, double cohesion,
                double sigma_t)
{
    return guarded([&] {
        auto p = mpm::DruckerPragerParams<double>::make(rho0, K, nu, phi, psi, cohesion, sigma_t);
        d->material = MPM_MAT_DRUCKER_PRAGER;
        d->rho0 = p.rho0;
        d->K = p.K;
        d->nu = p.nu;
        d->G = p.G;
        d->phi = p.phi;
        d->psi = p.psi;
        d->cohesion = p.cohesion;
        d->sigma_t = p.sigma_t;
        d->q_phi = p.q_phi;
        d->k_phi = p.k_phi;
        d->q_psi = p.q_psi;
        d->tau_P = p.tau_P;
        d->alpha_P = p.alpha_P;
        return MPM_OK;
    });
}

int64_t ref_init_scene_count(const mpm_scene_desc* d, const orc_region* r, int nreg)
{
    return dispatch<InitCount>(d, r, nreg);
}
int ref_init_scene(const mpm_scene_desc* d, const orc_region* r, int nreg, mpm_state_view* out, double* meps)
{
    return dispatch<Init>(d, r, nreg, out, meps);
}
int ref_advance(const mpm_scene_desc* d, mpm_state_view* s, int64_t n, int nan_guard)
{
    return dispatch<Advance>(d, s, n, nan_guard);
}
int ref_p2g(const mpm_scene_desc* d, const mpm_state_view* s, mpm_grid_view* g) { return dispatch<P2G>(d, s, g); }
int ref_grid_momentum_update(const mpm_scene_desc* d, mpm_grid_view* g) { return dispatch<GridUpdate>(d, g); }
int ref_grid_corrections(const mpm_scene_desc* d, mpm_grid_view* g) { return dispatch<GridCorr>(d, g); }
int ref_g2p(const mpm_scene_desc* d, const mpm_grid_view* g, mpm_state_view* s) { return dispatch<G2P>(d, g, s); }
int ref_constitutive(const mpm_scene_desc* d, mpm_state_view* s) { return dispatch<Constit>(d, s); }
int ref_step_vjp(const mpm_scene_desc* d, const mpm_state_view* s, const mpm_cot_view* co, mpm_cot_view* ci,
                 mpm_param_grads* pg)
{
    return dispatch<Vjp>(d, s, co, ci, pg);
}
int ref_backprop(const mpm_scene_desc* d, const mpm_state_view* s0, int64_t total, int nseg,
                 const mpm_seeder_desc* sd, mpm_cot_view* c0, mpm_param_grads* pg, mpm_backprop_result* res)
{
    return dispatch<Backprop>(d, s0, total, nseg, sd, c0, pg, res);
}
uint64_t ref_state_hash(const mpm_scene_desc* d, const mpm_state_view* s) { return dispatch<Hash>(d, s); }
double ref_run_seconds_per_1000(const mpm_scene_desc* d, mpm_state_view* s, int64_t n)
{
    return dispatch<RunTimer>(d, s, n);
}

} // extern "C"
