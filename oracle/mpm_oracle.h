/*
 * mpm_oracle.h -- TEST INFRASTRUCTURE ONLY. Never linked into the product.
 *
 * Two CPU implementations of the reference MPM step, behind one stateless C ABI, used
 * only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference:
 *
 *   orc_*  oracle/mpm_oracle.cpp  -> oracle/_build/liboracle.so
 *          An independent restatement of the reference algorithm (plain C++, no Eigen),
 *          each function citing the reference file:line it follows. Pinned against the
 *          reference's own known-answer tests (tests/test_oracle_*.py) and against ref_*.
 *   ref_*  oracle/ref_capi.cpp    -> oracle/_ref/libmpm_ref.so
 *          The reference itself: /root/reference/proj/include/mpm compiled UNMODIFIED
 *          against the Eigen-API shim (oracle/shim/), wrapped in this ABI.
 *
 * Types (scene / state / cotangent / grid views) are those of the product ABI
 * (include/mpm_capi.h), so a test can feed the same host arrays to all three.
 * Return codes follow MPM_OK / MPM_ERR_*; *_last_error() gives the offending particle.
 */
#ifndef MPM_ORACLE_H
#define MPM_ORACLE_H

#include "../include/mpm_capi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* GeometryRegion (config.hpp:132-184) + VelocityExpr (config.hpp:90-130), init-only.
 * shape: 0 box, 1 cylinder; vel_kind: 0 constant, 1 linear_in_y, 2 parabolic_sine. */
typedef struct orc_region {
    int shape;
    double lo[3], hi[3], center[3];
    double radius, zmin, zmax;
    int vel_kind;
    double value[3];
    double alpha, h0, amplitude, perturbation, frequency;
} orc_region;

#define MPM_ORACLE_DECLARE(P)                                                                        \
    int P##_last_error(int64_t* particle, char* msg, size_t len);                                    \
    /* DruckerPragerParams::make (material.hpp:64-83): fills K..alpha_P and rho0 of desc */          \
    int P##_dp_make(mpm_scene_desc* d, double rho0, double K, double nu, double phi, double psi,     \
                    double cohesion, double sigma_t);                                                \
    /* init_scene (scene.hpp:55-116): count, then fill (arrays sized by the count) */                \
    int64_t P##_init_scene_count(const mpm_scene_desc* d, const orc_region* r, int nreg);            \
    int P##_init_scene(const mpm_scene_desc* d, const orc_region* r, int nreg, mpm_state_view* out,  \
                       double* mass_epsilon);                                                        \
    /* n x Stepper::advance (stepper.hpp:59-69), optional run() NaN guard */                       \
    int P##_advance(const mpm_scene_desc* d, mpm_state_view* s, int64_t n, int nan_guard);           \
    int P##_p2g(const mpm_scene_desc* d, const mpm_state_view* s, mpm_grid_view* g);                 \
    int P##_grid_momentum_update(const mpm_scene_desc* d, mpm_grid_view* g);                         \
    int P##_grid_corrections(const mpm_scene_desc* d, mpm_grid_view* g);                             \
    int P##_g2p(const mpm_scene_desc* d, const mpm_grid_view* g, mpm_state_view* s);                 \
    int P##_constitutive(const mpm_scene_desc* d, mpm_state_view* s);                                \
    int P##_step_vjp(const mpm_scene_desc* d, const mpm_state_view* s, const mpm_cot_view* cot_out,  \
                     mpm_cot_view* cot_in, mpm_param_grads* pg);                                     \
    int P##_backprop(const mpm_scene_desc* d, const mpm_state_view* s0, int64_t total_steps,         \
                     int n_segments, const mpm_seeder_desc* seeder, mpm_cot_view* cot0,              \
                     mpm_param_grads* pg, mpm_backprop_result* res);                                 \
    /* SimState::hash (state.hpp:71-86) */                                                         \
    uint64_t P##_state_hash(const mpm_scene_desc* d, const mpm_state_view* s);                       \
    /* run(...).seconds_per_1000_steps (stepper.hpp:91-122), state advanced in place */             \
    double P##_run_seconds_per_1000(const mpm_scene_desc* d, mpm_state_view* s, int64_t n);

MPM_ORACLE_DECLARE(orc)
MPM_ORACLE_DECLARE(ref)

#ifdef __cplusplus
}
#endif

#endif /* MPM_ORACLE_H */
