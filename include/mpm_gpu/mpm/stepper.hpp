// mpm/stepper.hpp -- GPU drop-in for the reference header of the same name
// (/root/reference/proj/include/mpm/stepper.hpp). Put include/mpm_gpu/ BEFORE the reference's
// include directory and every `#include "mpm/stepper.hpp"` resolves here: Stepper, run,
// RunResult, max_particle_speed and constitutive_update keep their names and signatures but run
// on the B200 through libmpm_b200.so. The headers this one replaces includes (constitutive,
// contact, scene, transfer) are the reference's own. Nothing of the reference file is copied.
#pragma once

#include "../mpm_gpu.hpp"

namespace mpm {

template <class T, int dim> using Stepper = gpu::Stepper<T, dim>;
template <class T, int dim> using RunResult = gpu::RunResult<T, dim>;
using gpu::constitutive_update;
using gpu::max_particle_speed;
using gpu::run;

} // namespace mpm
