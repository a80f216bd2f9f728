// mpm_gpu_adjoint.hpp -- C++ drop-in for step_vjp (adjoint.hpp:328-525) and backprop_trajectory
// (checkpoint.hpp:72-143) over the C ABI. Uses the reference's own StateCotangent, ParamGrads,
// AdjointWorkspace, CheckpointPlan and BackpropResult types.
#pragma once

#include "mpm_gpu.hpp"

#include <mpm/checkpoint.hpp>

#include <memory>
#include <vector>

namespace mpm {
namespace gpu {

template <class T, int dim> mpm_param_grads pg_view(ParamGrads<T, dim>& g, std::vector<double> (&tmp)[6])
{
    mpm_param_grads v{};
    v.sound_speed = double(g.sound_speed);
    v.viscosity = double(g.viscosity);
    for (int w = 0; w < 2 * dim; ++w) {
        tmp[w].assign(g.wall_friction[w].begin(), g.wall_friction[w].end());
        v.wall_friction[w] = tmp[w].empty() ? nullptr : tmp[w].data();
    }
    return v;
}
template <class T, int dim> void pg_back(ParamGrads<T, dim>& g, const mpm_param_grads& v, std::vector<double> (&tmp)[6])
{
    g.sound_speed = T(v.sound_speed);
    g.viscosity = T(v.viscosity);
    for (int w = 0; w < 2 * dim; ++w)
        for (std::size_t k = 0; k < tmp[w].size(); ++k)
            g.wall_friction[w][k] = T(tmp[w][k]);
}

namespace detail {
// The scene's content as bytes (scalars + friction + obstacles): the key of the cached context.
template <class T, int dim> std::vector<unsigned char> scene_key(const SceneDesc<T, dim>& sd)
{
    mpm_scene_desc d = sd.d;
    for (auto& f : d.friction)
        f = nullptr;
    d.obstacles = nullptr;
    std::vector<unsigned char> k(reinterpret_cast<const unsigned char*>(&d),
                                 reinterpret_cast<const unsigned char*>(&d) + sizeof(d));
    auto put = [&](const double* p, std::size_t n) {
        k.insert(k.end(), reinterpret_cast<const unsigned char*>(p), reinterpret_cast<const unsigned char*>(p + n));
    };
    for (int w = 0; w < 2 * dim; ++w)
        put(sd.fr[w].data(), sd.fr[w].size());
    put(sd.ob.data(), sd.ob.size());
    return k;
}

// step_vjp's device context. The reference's AdjointWorkspace (adjoint.hpp:298-322) is its
// scratch; its layout is fixed by the reference headers, so the device context lives beside it,
// one per host thread, reused while the scene is the same and the particle count fits.
template <class T, int dim> Context<T, dim>& vjp_context(const Scene<T, dim>& scene, Index n)
{
    struct Cache {
        std::unique_ptr<Context<T, dim>> ctx;
        std::vector<unsigned char> key;
    };
    thread_local Cache c;
    SceneDesc<T, dim> sd(scene);
    std::vector<unsigned char> key = scene_key(sd);
    if (!c.ctx || c.key != key || c.ctx->capacity() < n) {
        c.ctx.reset();
        c.ctx = std::make_unique<Context<T, dim>>(scene, std::max<Index>(n, 1));
        c.key = std::move(key);
    }
    return *c.ctx;
}

template <class T, int dim>
void step_vjp_on(Context<T, dim>& ctx, const SimState<T, dim>& input, const StateCotangent<T, dim>& cot_out,
                 StateCotangent<T, dim>& cot_in, ParamGrads<T, dim>& pg)
{
    SimState<T, dim> s = input;
    auto sv = state_view(s);
    StateCotangent<T, dim> co = cot_out;
    cot_in = StateCotangent<T, dim>::zeros_like(input.particles);
    auto cov = cot_view(co);
    auto civ = cot_view(cot_in);
    std::vector<double> tmp[6];
    auto pv = pg_view(pg, tmp);
    ctx.check(mpm_step_vjp(ctx.handle(), &sv, &cov, &civ, &pv));
    pg_back(pg, pv, tmp);
}
} // namespace detail

// step_vjp: cot_in is overwritten, pg accumulated (adjoint.hpp:371, :145, :172). The device
// context is cached per thread (detail::vjp_context): no allocation per call in a reverse loop.
template <class T, int dim>
void step_vjp(const Scene<T, dim>& scene, const SimState<T, dim>& input, const StateCotangent<T, dim>& cot_out,
              StateCotangent<T, dim>& cot_in, ParamGrads<T, dim>& pg, AdjointWorkspace<T, dim>& ws)
{
    (void)ws;
    detail::step_vjp_on(detail::vjp_context(scene, input.particles.size()), input, cot_out, cot_in, pg);
}

// backprop_trajectory with any duck-typed Seeder (observes / loss_at / seed, checkpoint.hpp:63-66):
// the forward sweep, segment replays (with the digest check) and every step_vjp run on the
// device; the Seeder is called on host copies of the observed states only.
template <class T, int dim, class Seeder>
BackpropResult<T, dim> backprop_trajectory(const Scene<T, dim>& scene, const SimState<T, dim>& initial,
                                           const CheckpointPlan& plan, Seeder&& seeder)
{
    const int nseg = plan.n_segments;
    BackpropResult<T, dim> result;
    Context<T, dim> ctx(scene, initial.particles.size());
    auto digest = [&]() {
        uint64_t d = 0;
        ctx.check(mpm_state_digest(ctx.handle(), &d));
        return d;
    };
    std::vector<SimState<T, dim>> checkpoints;
    std::vector<uint64_t> bhash(static_cast<std::size_t>(nseg) + 1);
    SimState<T, dim> s = initial;
    ctx.upload(s);
    if (seeder.observes(0))
        result.loss += seeder.loss_at(0, s);
    for (int k = 0; k < nseg; ++k) {
        ctx.download(s);
        checkpoints.push_back(s);
        bhash[k] = digest();
        for (Index t = plan.boundaries[k]; t < plan.boundaries[k + 1]; ++t) {
            ctx.advance(1, false);
            if (seeder.observes(t + 1)) {
                ctx.download(s);
                result.loss += seeder.loss_at(t + 1, s);
            }
        }
    }
    bhash[nseg] = digest();
    result.checkpoints_stored = nseg;
    StateCotangent<T, dim> cot = StateCotangent<T, dim>::zeros_like(initial.particles), cot_prev = cot;
    result.param_grads = ParamGrads<T, dim>::zeros_like(scene.boundary);
    AdjointWorkspace<T, dim> ws;
    std::vector<SimState<T, dim>> replay;
    for (int k = nseg - 1; k >= 0; --k) {
        const Index b0 = plan.boundaries[k], b1 = plan.boundaries[k + 1];
        replay.assign(1, checkpoints[k]);
        SimState<T, dim> r = checkpoints[k];
        ctx.upload(r);
        for (Index t = b0; t < b1; ++t) {
            ctx.advance(1, false);
            ctx.download(r);
            replay.push_back(r);
        }
        if (digest() != bhash[k + 1])
            throw NumericalError("checkpoint mismatch: recomputed segment end differs from the recorded state at step "
                                 + std::to_string(b1));
        result.peak_replay_states = std::max(result.peak_replay_states, Index(replay.size()));
        for (Index t = b1; t > b0; --t) {
            if (seeder.observes(t))
                seeder.seed(t, replay[t - b0], cot);
            (void)ws;
            detail::step_vjp_on(ctx, replay[t - b0 - 1], cot, cot_prev, result.param_grads); // trajectory's context
            std::swap(cot, cot_prev);
        }
    }
    if (seeder.observes(0))
        seeder.seed(0, initial, cot);
    result.initial_state_cot = std::move(cot);
    return result;
}

} // namespace gpu
} // namespace mpm
