// The C++ drop-in layer against the reference in one translation unit: the reference's
// Stepper / step_vjp / backprop_trajectory run on the CPU, mpm::gpu's on the B200, on the same
// reference-typed inputs. Built by tests/cpp/Makefile, run by tests/test_dropin_cpp.py (gpu).
#include <mpm/checkpoint.hpp>
#include <mpm/stepper.hpp>
#include <mpm_gpu/mpm_gpu_adjoint.hpp>

#include "helpers.hpp"

#include <doctest.h>

using namespace mpm;

namespace {

template <class V> double rel(const std::vector<V>& a, const std::vector<V>& b)
{
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        num = std::max(num, double((a[i] - b[i]).template lpNorm<Eigen::Infinity>()));
        den = std::max(den, double(b[i].template lpNorm<Eigen::Infinity>()));
    }
    return num / std::max(den, 1e-300);
}
double rels(const std::vector<double>& a, const std::vector<double>& b)
{
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        num = std::max(num, std::abs(a[i] - b[i]));
        den = std::max(den, std::abs(b[i]));
    }
    return num / std::max(den, 1e-300);
}

Scene<double, 2> dp_scene()
{
    Scene<double, 2> s;
    s.config.dh = 0.05;
    s.config.cells = {20, 20};
    s.config.dt = 1e-5;
    s.config.gravity = Vec<double, 2>(0, -9.8);
    s.config.scheme.kind = SchemeKind::flip;
    s.material = DruckerPragerParams<double>::make(2650.0, 0.7e6, 0.3, 19.8 * M_PI / 180.0, 0.0, 0.0, 0.0);
    s.boundary.walls[2].kind = WallKind::coulomb;
    s.boundary.walls[2].friction = {0.1, 0.4, 0.2};
    GeometryRegion<double, 2> r;
    r.lo = Vec<double, 2>(0.1, 0.1);
    r.hi = Vec<double, 2>(0.5, 0.35);
    r.velocity.kind = VelExprKind::constant;
    r.velocity.value = Vec<double, 2>(1.5, 0.0);
    s.geometry.push_back(r);
    return s;
}

struct FinalXSeeder {
    Index N;
    std::vector<Vec<double, 2>> target;
    bool observes(Index t) const { return t == N; }
    double loss_at(Index, const SimState<double, 2>& s) const
    {
        double L = 0;
        for (std::size_t p = 0; p < target.size(); ++p)
            L += (s.particles.x[p] - target[p]).squaredNorm();
        return L;
    }
    void seed(Index, const SimState<double, 2>& s, StateCotangent<double, 2>& c) const
    {
        for (std::size_t p = 0; p < target.size(); ++p)
            c.x[p] += 2.0 * (s.particles.x[p] - target[p]);
    }
};

} // namespace

TEST_CASE("gpu::Stepper matches the reference Stepper on a D-P column with a Coulomb floor")
{
    auto scene = dp_scene();
    auto state = init_scene(scene);
    auto ref = state;
    Stepper<double, 2> cpu(scene);
    gpu::Stepper<double, 2> dev(scene);
    for (int k = 0; k < 20; ++k) {
        cpu.advance(ref);
        dev.advance(state);
    }
    CHECK(state.step == 20);
    CHECK(rel(state.particles.x, ref.particles.x) < 1e-12);
    CHECK(rel(state.particles.v, ref.particles.v) < 1e-9);
    CHECK(rel(state.particles.sigma, ref.particles.sigma) < 1e-9);
    CHECK(rels(state.particles.rho, ref.particles.rho) < 1e-12);
}

TEST_CASE("gpu::run keeps the reference run() contract")
{
    auto scene = testing::small_fluid_scene(SchemeKind::flip);
    scene.config.gravity = Vec<double, 2>(0, -9.8);
    auto state = init_scene(scene);
    auto r_cpu = run(scene, state, 9, 3);
    auto r_gpu = gpu::run(scene, state, 9, 3);
    REQUIRE(r_gpu.snapshots.size() == r_cpu.snapshots.size());
    for (std::size_t k = 0; k < r_cpu.snapshots.size(); ++k) {
        CHECK(r_gpu.snapshots[k].step == r_cpu.snapshots[k].step);
        CHECK(rel(r_gpu.snapshots[k].particles.v, r_cpu.snapshots[k].particles.v) < 1e-10);
    }
}

TEST_CASE("gpu::step_vjp matches the reference step_vjp (fluid, flip)")
{
    auto scene = testing::small_fluid_scene(SchemeKind::flip);
    scene.config.gravity = Vec<double, 2>(0, -9.8);
    auto state = init_scene(scene);
    Stepper<double, 2> cpu(scene);
    for (int k = 0; k < 5; ++k)
        cpu.advance(state);
    auto cot = StateCotangent<double, 2>::zeros_like(state.particles);
    auto gen = testing::rng(3);
    std::normal_distribution<double> nd;
    for (auto& x : cot.x)
        x = Vec<double, 2>(nd(gen), nd(gen));
    for (auto& v : cot.v)
        v = Vec<double, 2>(nd(gen), nd(gen));
    for (auto& r : cot.rho)
        r = nd(gen);
    StateCotangent<double, 2> ci_cpu, ci_gpu;
    auto pg_cpu = ParamGrads<double, 2>::zeros_like(scene.boundary), pg_gpu = pg_cpu;
    AdjointWorkspace<double, 2> ws;
    ws.configure(scene);
    step_vjp(scene, state, cot, ci_cpu, pg_cpu, ws);
    gpu::step_vjp(scene, state, cot, ci_gpu, pg_gpu, ws);
    CHECK(rel(ci_gpu.x, ci_cpu.x) < 1e-10);
    CHECK(rel(ci_gpu.v, ci_cpu.v) < 1e-10);
    CHECK(rels(ci_gpu.rho, ci_cpu.rho) < 1e-10);
    CHECK(std::abs(pg_gpu.sound_speed - pg_cpu.sound_speed) <= 1e-10 * std::abs(pg_cpu.sound_speed));
}

TEST_CASE("gpu::backprop_trajectory with a duck-typed Seeder matches the reference")
{
    auto scene = testing::small_fluid_scene(SchemeKind::flip);
    scene.config.gravity = Vec<double, 2>(0, -9.8);
    auto state = init_scene(scene);
    auto fin = state;
    Stepper<double, 2> cpu(scene);
    for (int k = 0; k < 8; ++k)
        cpu.advance(fin);
    FinalXSeeder seeder{8, {}};
    for (const auto& x : fin.particles.x)
        seeder.target.push_back(x + Vec<double, 2>(0.01, -0.01));
    auto plan = CheckpointPlan::make(8, 3);
    auto r_cpu = backprop_trajectory(scene, state, plan, seeder);
    auto r_gpu = gpu::backprop_trajectory(scene, state, plan, seeder);
    CHECK(std::abs(r_gpu.loss - r_cpu.loss) <= 1e-10 * r_cpu.loss);
    CHECK(r_gpu.peak_replay_states == r_cpu.peak_replay_states);
    CHECK(rel(r_gpu.initial_state_cot.v, r_cpu.initial_state_cot.v) < 1e-8);
    CHECK(rel(r_gpu.initial_state_cot.x, r_cpu.initial_state_cot.x) < 1e-8);
}

TEST_CASE("gpu::SlabGroup (library-owned slab decomposition, 1-3 ranks on one GPU) matches gpu::Stepper")
{
    Scene<double, 2> scene = dp_scene();
    scene.config.cells = {64, 20};
    scene.geometry[0].lo = Vec<double, 2>(0.6, 0.1); // spans the slab bound at x = 16 cells
    scene.geometry[0].hi = Vec<double, 2>(1.0, 0.35);
    SimState<double, 2> state = init_scene(scene);
    SimState<double, 2> ref = state;
    gpu::Stepper<double, 2> stepper(scene);
    const int N = 30;
    for (int k = 0; k < N; ++k)
        stepper.advance(ref);
    for (int R = 1; R <= 3; ++R) {
        std::vector<int> bounds;
        for (int r = 0; r <= R; ++r)
            bounds.push_back(r == R ? 64 : 16 * ((4 * r) / R));
        gpu::SlabGroup<double, 2> group(scene, state, bounds);
        group.advance(1);
        group.advance(N - 1, true);
        SimState<double, 2> got = group.gather();
        CHECK(got.step == N);
        CHECK(rel(got.particles.x, ref.particles.x) < 1e-12);
        CHECK(rel(got.particles.v, ref.particles.v) < 1e-9);
        CHECK(rel(got.particles.sigma, ref.particles.sigma) < 1e-9);
        if (R == 1) { // one slab: the same operations in the same order as the plain step
            CHECK(rel(got.particles.x, ref.particles.x) == 0.0);
            CHECK(rel(got.particles.sigma, ref.particles.sigma) == 0.0);
        }
    }
}

TEST_CASE("gpu::SlabRank: a 1-rank NCCL communicator owned by the library")
{
    Scene<double, 2> scene = dp_scene();
    SimState<double, 2> state = init_scene(scene);
    SimState<double, 2> ref = state;
    gpu::Stepper<double, 2> stepper(scene);
    for (int k = 0; k < 12; ++k)
        stepper.advance(ref);
    std::vector<Index> ids(state.particles.size());
    for (std::size_t i = 0; i < ids.size(); ++i)
        ids[i] = Index(i);
    gpu::SlabRank<double, 2> rank(scene, state, ids, 0, 1, gpu::SlabRank<double, 2>::unique_id(), 0,
                                  scene.config.cells[0], state.particles.size());
    CHECK(rank.advance(12) > 0.0);
    std::vector<Index> got_ids;
    SimState<double, 2> sub = rank.download(got_ids);
    SimState<double, 2> got = state;
    gpu::put_rows(got, sub, got_ids);
    CHECK(got.step == 12);
    CHECK(rel(got.particles.x, ref.particles.x) == 0.0);
    CHECK(rel(got.particles.sigma, ref.particles.sigma) == 0.0);
}
