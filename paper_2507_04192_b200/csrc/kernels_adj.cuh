// kernels_adj.cuh -- reverse-mode adjoint of the step (adjoint.hpp) -- placeholder.
#pragma once

#include "common.cuh"

#include <stdexcept>

namespace mpmgpu {

template <class T, int D> struct AdjWork {
    template <class Ctx> void init(Ctx&) {}
    void free_all() {}
    template <class Ctx> void set_attrs(Ctx&) {}
    template <class Ctx>
    void step_vjp_api(Ctx&, const mpm_state_view*, const mpm_cot_view*, mpm_cot_view*, mpm_param_grads*)
    {
        throw std::runtime_error("step_vjp: adjoint kernels not built yet");
    }
    template <class Ctx>
    void backprop_api(Ctx&, const mpm_state_view*, int64_t, int, const mpm_seeder_desc*, mpm_cot_view*,
                      mpm_param_grads*, mpm_backprop_result*)
    {
        throw std::runtime_error("backprop: adjoint kernels not built yet");
    }
};

} // namespace mpmgpu
