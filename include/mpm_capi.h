/*
 * mpm_capi.h -- C ABI of the B200-native MPM one-step operator Phi = G2P o U o P2G and
 * its reverse-mode adjoint (libmpm_b200.so).
 *
 * The reference (/root/reference/proj, "arxiv/paper_2507_04192") is a header-only C++20
 * template library in namespace mpm with no ABI (proj/CMakeLists.txt:13-15 builds a static
 * lib holding only src/hash.cpp). Each entry point below is the plain-pointer form of one
 * reference API; the C++ drop-in layer (include/mpm_gpu/) converts the reference's own
 * Scene/SimState/StateCotangent/ParamGrads/Grid types into these views, so existing callers
 * compile unchanged. The reference interface each call replaces is cited beside it.
 *
 * Conventions
 *  - Scalars in views are T = float (MPM_F32) or double (MPM_F64), chosen at ctx creation.
 *  - Host arrays use the reference's in-memory layout (std::vector<Eigen::Matrix>):
 *      vectors   T[n][dim]
 *      matrices  T[n][dim*dim], each matrix COLUMN-MAJOR (Eigen default)
 *    so a std::vector<Vec<T,dim>>::data() / std::vector<Mat<T,dim>>::data() can be passed
 *    directly (state.hpp:17-63, adjoint.hpp:10-72).
 *  - Particles are addressed by their index in the host arrays (the reference's particle
 *    id). The device keeps its own cell-sorted order and maps back at this boundary.
 *  - Every call is synchronous at return (reference semantics); the context owns a CUDA
 *    stream and all device buffers. One context per host thread.
 *  - Errors: int status (below) + mpm_last_error(). The C++ layer rethrows the reference
 *    exception types (common.hpp:22-36): 2 -> ValidationError, 3 -> NumericalError,
 *    4 -> OutOfDomainError{particle}, 5 -> NumericalError("checkpoint mismatch ...").
 *  - There is NO CPU fallback: without a usable sm_100 device, mpm_ctx_create fails with
 *    MPM_ERR_CUDA.
 */
#ifndef MPM_CAPI_H
#define MPM_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPM_CAPI_VERSION 1

/* dtype tags */
enum { MPM_F32 = 0, MPM_F64 = 1 };

/* status codes (common.hpp:22-36 exit-code convention, extended) */
enum {
    MPM_OK = 0,
    MPM_ERR_USAGE = 1,         /* bad arguments to this ABI */
    MPM_ERR_VALIDATION = 2,    /* ValidationError */
    MPM_ERR_NUMERICAL = 3,     /* NumericalError */
    MPM_ERR_OUT_OF_DOMAIN = 4, /* OutOfDomainError{particle} */
    MPM_ERR_CHECKPOINT = 5,    /* checkpoint replay mismatch (checkpoint.hpp:124-126) */
    MPM_ERR_CUDA = 6           /* device / CUDA / NCCL failure */
};

/* config.hpp:13 SchemeKind, same order */
enum { MPM_SCHEME_PIC = 0, MPM_SCHEME_FLIP = 1, MPM_SCHEME_BLEND = 2, MPM_SCHEME_APIC = 3, MPM_SCHEME_TPIC = 4 };
/* config.hpp:34 WallKind, same order */
enum { MPM_WALL_SLIP = 0, MPM_WALL_NO_SLIP = 1, MPM_WALL_FIXED = 2, MPM_WALL_COULOMB = 3 };
/* material.hpp:106-107 Material variant index */
enum { MPM_MAT_FLUID = 0, MPM_MAT_DRUCKER_PRAGER = 1 };

/* Scene<T,dim> (scene.hpp:9-16) minus the init-only geometry. All reals are passed as
 * double and converted to T once (exact when the caller's Scene<T> holds T values). */
typedef struct mpm_scene_desc {
    int dim;             /* 2 or 3 */
    int dtype;           /* MPM_F32 / MPM_F64 */
    double dh;           /* SimConfig::dh */
    int cells[3];        /* SimConfig::cells */
    double origin[3];    /* SimConfig::origin */
    double dt;           /* SimConfig::dt */
    double gravity[3];   /* SimConfig::gravity */
    int scheme;          /* TransferScheme::kind */
    double alpha_flip;   /* TransferScheme::alpha_flip */
    int track_def_grad;  /* SimConfig::track_def_grad */
    int material;        /* MPM_MAT_* */
    /* FluidParams (material.hpp:13-29) */
    double rho0, viscosity, sound_speed;
    int rate_form;
    /* DruckerPragerParams (material.hpp:52-95), derived constants passed as stored */
    double K, nu, G, phi, psi, cohesion, sigma_t, q_phi, k_phi, q_psi, tau_P, alpha_P;
    /* BoundarySpec (config.hpp:45-57) */
    int band_layers;
    int wall_kind[6];           /* w = 2*axis + side */
    int n_friction[6];          /* Coulomb segments per wall */
    const double* friction[6];  /* n_friction[w] coefficients */
    /* Obstacles (config.hpp:61-88): n_obstacles * (lo[dim], hi[dim]) */
    int n_obstacles;
    const double* obstacles;
    double mass_epsilon;        /* Scene::mass_epsilon (set by init_scene) */
} mpm_scene_desc;

/* SimState<T,dim> (state.hpp:17-87) as host arrays; NULL = field absent. */
typedef struct mpm_state_view {
    int64_t n;
    void* x;        /* [n][dim] */
    void* v;        /* [n][dim] */
    void* mass;     /* [n] */
    void* volume;   /* [n] */
    void* rho;      /* [n] */
    void* eps_eq;   /* [n] */
    void* sigma_zz; /* [n] (2-D only) */
    void* sigma;    /* [n][dim*dim] col-major, symmetric */
    void* grad_v;   /* [n][dim*dim] col-major */
    void* affine;   /* [n][dim*dim] col-major, APIC only */
    void* def_grad; /* [n][dim*dim] col-major, track_def_grad only */
    int64_t step;
    double time;
} mpm_state_view;

/* StateCotangent<T,dim> (adjoint.hpp:10-72); sigma/grad_v/affine are full matrices. */
typedef struct mpm_cot_view {
    int64_t n;
    void* x;        /* [n][dim] */
    void* v;        /* [n][dim] */
    void* rho;      /* [n] */
    void* volume;   /* [n] */
    void* eps_eq;   /* [n] (discarded on input, zero on output) */
    void* sigma_zz; /* [n] (2-D) */
    void* sigma;    /* [n][dim*dim] */
    void* grad_v;   /* [n][dim*dim] */
    void* affine;   /* [n][dim*dim] (APIC) */
} mpm_cot_view;

/* ParamGrads<T,dim> (adjoint.hpp:77-90); ACCUMULATED into (+=) like the reference. */
typedef struct mpm_param_grads {
    double sound_speed;
    double viscosity;
    double* wall_friction[6]; /* n_friction[w] entries each (may be NULL if 0) */
} mpm_param_grads;

/* Grid<T,dim> (state.hpp:91-173), dense, row-major node index (last axis fastest). */
typedef struct mpm_grid_view {
    int64_t num_nodes;
    void* mass;     /* [nodes] */
    void* momentum; /* [nodes][dim] */
    void* v_old;    /* [nodes][dim] */
    void* v;        /* [nodes][dim] */
    void* force;    /* [nodes][dim] */
} mpm_grid_view;

/* Built-in loss seeders for backprop_trajectory (checkpoint.hpp:63-66 Seeder protocol):
 * masked Lagrangian least squares (SPEC.md observe_lagrangian + loss):
 *   L = sum_{k<n_obs} sum_{l<n_sel} || z_{sel[l]}(obs_steps[k]) - target[k][l] ||^2,
 * z = x (field 0) or v (field 1); sel = NULL means all particles in id order.
 * masked Eulerian least squares (SPEC.md observe_eulerian, PAPER §3.2 "average over all particles
 * within this region"): monitor regions are closed boxes |x - center| <= half per axis,
 *   Q_l(t) = mean of z over the particles inside region l at step t,
 *   L = sum_k sum_l m[k][l] || Q_l(obs_steps[k]) - target[k][l] ||^2,
 * an empty region has m = 0 (no term, no gradient); mask = NULL means all 1. The membership is
 * piecewise constant in x, so only the z cotangent is seeded: 2 m (Q_l - target) / |P_l| per member. */
enum { MPM_SEEDER_NONE = 0, MPM_SEEDER_LAGRANGIAN_LS = 1, MPM_SEEDER_EULERIAN_LS = 2 };
typedef struct mpm_seeder_desc {
    int kind;
    int field;               /* 0 = x, 1 = v */
    int n_obs;               /* number of observed steps */
    const int64_t* obs_steps;
    int64_t n_sel;
    const int64_t* sel;      /* particle ids, or NULL = all */
    const void* target;      /* T[n_obs][n_sel][dim] (Lagrangian) or T[n_obs][n_regions][dim] (Eulerian) */
    /* Eulerian only */
    int64_t n_regions;
    const void* centers;     /* T[n_regions][dim] */
    const void* half;        /* T[n_regions][dim] */
    const unsigned char* mask; /* [n_obs][n_regions] or NULL */
} mpm_seeder_desc;

/* BackpropResult (checkpoint.hpp:53-61) counters */
typedef struct mpm_backprop_result {
    double loss;
    int64_t checkpoints_stored;
    int64_t peak_replay_states;
    double device_ms; /* device time of the sweep (forward sweep, segment replays, VJPs; CUDA events on
                         the context stream), excluding the S0 upload and the cotangent download */
} mpm_backprop_result;

/* advance flags */
enum {
    MPM_ADV_NAN_GUARD = 1u, /* run(): abort on non-finite state (stepper.hpp:106-109) */
    MPM_ADV_STORE_GRID = 2u /* also keep the step's full grid (mass, momentum, force) so that
                               mpm_grid_download returns Stepper::grid as the reference has it */
};

typedef struct mpm_ctx mpm_ctx;

/* ---- context ---------------------------------------------------------------------- */
/* Stepper<T,dim>::Stepper(const Scene&) (stepper.hpp:53-57): validates the scene and
 * allocates device state, grid blocks, sort and workspace buffers for up to max_particles. */
int mpm_ctx_create(const mpm_scene_desc* scene, int64_t max_particles, int device, mpm_ctx** out);
void mpm_ctx_destroy(mpm_ctx* ctx);
/* last error: code, offending particle id (-1), step (-1), message */
int mpm_last_error(const mpm_ctx* ctx, int* code, int64_t* particle, int64_t* step, char* msg, size_t msg_len);
int mpm_version(void);
/* human-readable device name for logs */
int mpm_device_name(char* buf, size_t len);

/* ---- state transfer ------------------------------------------------------------------ */
int mpm_state_upload(mpm_ctx* ctx, const mpm_state_view* s);
int mpm_state_download(mpm_ctx* ctx, mpm_state_view* s);
/* order-independent 64-bit digest of the device state (replaces SimState::hash at the
 * checkpoint replay check, state.hpp:71-86 / checkpoint.hpp:124) */
int mpm_state_digest(mpm_ctx* ctx, uint64_t* out);
/* max_particle_speed (stepper.hpp:78-85) */
int mpm_max_speed(mpm_ctx* ctx, double* vmax);

/* ---- forward ------------------------------------------------------------------------ */
/* n x Stepper::advance (stepper.hpp:59-69); MPM_ADV_NAN_GUARD adds run()'s all_finite
 * check after every step (stepper.hpp:106-109). */
int mpm_advance(mpm_ctx* ctx, int64_t n_steps, uint32_t flags);
/* mpm_advance with CUDA events recorded on the context stream around the n steps:
 * *device_ms = device time of the steps (bench / instrumentation) */
int mpm_advance_timed(mpm_ctx* ctx, int64_t n_steps, uint32_t flags, double* device_ms);
/* phase functions (each backs one reference free function, for per-phase parity):
 * p2g (transfer.hpp:37-69), grid_momentum_update (transfer.hpp:75-84),
 * apply_grid_corrections (contact.hpp:228-245), g2p (transfer.hpp:92-121),
 * constitutive_update (stepper.hpp:15-43). */
int mpm_p2g(mpm_ctx* ctx);
int mpm_grid_momentum_update(mpm_ctx* ctx);
int mpm_grid_corrections(mpm_ctx* ctx);
int mpm_g2p(mpm_ctx* ctx);
int mpm_constitutive(mpm_ctx* ctx);
/* Stepper::grid (stepper.hpp:51) as a dense host grid, and the reverse for tests that
 * drive the phase functions on a prescribed grid (test_contact.cpp, test_transfer.cpp). */
int mpm_grid_download(mpm_ctx* ctx, mpm_grid_view* g);
int mpm_grid_upload(mpm_ctx* ctx, const mpm_grid_view* g);

/* ---- adjoint ------------------------------------------------------------------------ */
/* step_vjp (adjoint.hpp:328-525): cot_in is OVERWRITTEN, pg is ACCUMULATED. */
int mpm_step_vjp(mpm_ctx* ctx, const mpm_state_view* state_in, const mpm_cot_view* cot_out,
                 mpm_cot_view* cot_in, mpm_param_grads* pg);
/* backprop_trajectory (checkpoint.hpp:72-143) with CheckpointPlan::make(total_steps,
 * n_segments) (checkpoint.hpp:15-34) and a built-in device seeder. */
int mpm_backprop(mpm_ctx* ctx, const mpm_state_view* initial, int64_t total_steps, int n_segments,
                 const mpm_seeder_desc* seeder, mpm_cot_view* initial_state_cot,
                 mpm_param_grads* pg, mpm_backprop_result* result);

/* ---- device scene seeding ------------------------------------------- */
/* GeometryRegion + VelocityExpr (config.hpp:99-184) */
typedef struct mpm_region {
    int shape;                               /* 0 box, 1 cylinder */
    double lo[3], hi[3];                     /* box: lo <= x < hi */
    double center[3], radius, zmin, zmax;    /* cylinder: |xy - center| < radius, zmin <= z < zmax */
    int vel_kind;                            /* 0 constant, 1 linear_in_y, 2 parabolic_sine */
    double value[3], alpha, h0, amplitude, perturbation, frequency;
    double min_y;                            /* the region's lowest y (velocity profile origin) */
} mpm_region;
/* init_scene (scene.hpp:55-116) on the device, into the context's state: 2^d sub-cell lattice at
 * +-dh/4 in every cell of the regions' bounding box (cells row-major, axis 0 slowest, corners in
 * bit order), the first containing region owns a point; mass / volume / rho0 as init_scene sets
 * them (passed in so the host formula stays the single source). Same particles, order and bits as
 * the host seeding, except parabolic_sine (device sin). *n_out = particles seeded; fails with
 * MPM_ERR_USAGE and *n_out = the count when it exceeds the context capacity. */
int mpm_init_scene(mpm_ctx* ctx, const mpm_region* regions, int n_regions, double mass, double volume, double rho0,
                   int64_t* n_out);

/* Asynchronous snapshots (run's snapshot policy, stepper.hpp:112-117): mpm_snapshot_begin gathers
 * the current state in id order on the context stream and copies it to library-owned pinned host
 * memory on a second stream, overlapping the steps that follow; mpm_snapshot_fetch (slot 0 or 1)
 * waits for that copy and fills `s` (reference layout). A slot holds one snapshot at a time. */
int mpm_snapshot_begin(mpm_ctx* ctx, int slot);
int mpm_snapshot_fetch(mpm_ctx* ctx, int slot, mpm_state_view* s);

/* ---- slab decomposition across GPUs ------------------------------------ */
/* One context per GPU, global coordinates; the context owns the particles whose base cell along
 * x lies in [cell_lo, cell_hi) (multiples of the block edge, 16 in 2-D / 8 in 3-D). A step is
 *   mpm_step_p2g_local (P2G + partial sums of the 2 node planes shared with each x-neighbour)
 *   -> mpm_halo export, start the neighbour send/recv -> mpm_step_grid_interior (all other
 *   nodes, overlapping the transfer) -> wait, mpm_halo import -> mpm_step_finish_local (band
 *   nodes, G2P) -> migration (mpm_migrate_export / mpm_migrate_import) of particles that left
 *   the slab.
 * The transport between GPUs (NCCL over NVLink via torch.distributed, or device copies in the
 * single-process mode) belongs to the caller (paper_2507_04192_b200/distributed.py). */
int mpm_slab_set(mpm_ctx* ctx, int cell_lo, int cell_hi, int64_t mig_cap);
/* enqueue all further work of ctx on `stream` (a cudaStream_t; NULL = the context's own). The
 * slab entry points below only enqueue (no host synchronisation) except mpm_step_finish_local,
 * so a transport on the same stream (NCCL via torch) is ordered with them. */
int mpm_ctx_set_stream(mpm_ctx* ctx, void* stream);
/* upload a rank-local subset: s holds n particles, ids their global particle ids */
int mpm_state_upload_ids(mpm_ctx* ctx, const mpm_state_view* s, const int64_t* ids);
/* compact download of the alive local particles in storage order (s sized >= mpm_local_count)
 * + their global ids */
int mpm_state_download_local(mpm_ctx* ctx, mpm_state_view* s, int64_t* ids);
int64_t mpm_local_count(const mpm_ctx* ctx);
int mpm_step_p2g_local(mpm_ctx* ctx);
int mpm_step_grid_interior(mpm_ctx* ctx);
/* node planes [plane_lo, plane_lo + n_planes) x all other nodes, (1 + 2 dim) scalars each:
 * mode 0 export into dev_buf; 1 import as received + own; 2 import as own + received */
int mpm_halo(mpm_ctx* ctx, int plane_lo, int n_planes, void* dev_buf, int mode);
int mpm_step_finish_local(mpm_ctx* ctx, uint32_t flags);
/* the same without a host synchronisation: enqueues the finish and writes (failed, n_lo, n_hi) as
 * int64 into device memory `dev_report` on the context stream, for the caller's collective; then
 * mpm_step_commit with the counts and whether any rank failed (raises this rank's own error) */
int mpm_step_finish_async(mpm_ctx* ctx, uint32_t flags, int64_t* dev_report);
int mpm_step_commit(mpm_ctx* ctx, int64_t n_lo, int64_t n_hi, int any_failed);
/* step_vjp over a slab (adjoint.hpp:328-525 decomposed). The state (this rank's particles at step t,
 * uploaded with mpm_state_upload in the same order as cot_out) and per step:
 *   mpm_slab_vjp_begin (forward replay: P2G + band sums) -> mpm_halo export/exchange/import ->
 *   mpm_slab_vjp_interior -> mpm_slab_vjp_scatter (band finish, G2P transpose and its scatter,
 *   band sums of the node v / v_old cotangents) -> mpm_halo_cot export/exchange/import (2 dim
 *   values per node) -> mpm_slab_vjp_finish (grid VJP, P2G transpose; cot_in overwritten, pg =
 *   this rank's partial ParamGrads, which the caller sums over the ranks). */
int mpm_slab_vjp_begin(mpm_ctx* ctx, const mpm_cot_view* cot_out);
int mpm_slab_vjp_interior(mpm_ctx* ctx);
int mpm_slab_vjp_scatter(mpm_ctx* ctx);
int mpm_halo_cot(mpm_ctx* ctx, int plane_lo, int n_planes, void* dev_buf, int mode);
int mpm_slab_vjp_finish(mpm_ctx* ctx, mpm_cot_view* cot_in, mpm_param_grads* pg);

/* particles that left the slab during the last step, toward -x (lo) and +x (hi) */
int mpm_particle_record_size(const mpm_ctx* ctx);
/* host-side counts of the last mpm_step_finish_local (known after it returns) */
int mpm_migrate_counts(const mpm_ctx* ctx, int64_t* n_lo, int64_t* n_hi);
int mpm_migrate_export(mpm_ctx* ctx, void* lo, int* lo_pid, void* hi, int* hi_pid, int64_t cap, int64_t* n_lo,
                       int64_t* n_hi);
int mpm_migrate_import(mpm_ctx* ctx, const void* recs, const int* pids, int64_t n);

/* ---- library-owned slab decomposition ---------------------------------- */
/* The decomposed step of Stepper::advance (stepper.hpp:59-69) run entirely inside the library:
 * one context per rank, rank r owning base cells [cell_lo, cell_hi) along x. Each step is
 * sort + P2G + band sums -> halo exchange of the 2 shared node planes (overlapping the interior
 * grid pass) -> fixed-order band import -> band update + G2P -> migration messages (count + up to
 * mig_cap records per neighbour, fixed size) + a device max-reduction of the abort flag -> import.
 * Particle counts stay on the device; there is no host synchronisation inside mpm_dist_advance,
 * whose status (this rank's error, or "another rank aborted") is checked once at its end.
 * Per-rank state goes in and out with mpm_state_upload_ids / mpm_state_download_local.
 *
 * NCCL ranks (one process per GPU): rank 0 makes an id with mpm_dist_unique_id, every rank
 * receives it (any side channel) and calls mpm_dist_attach_nccl; the library then owns an
 * ncclComm_t (ncclSend / ncclRecv to the x-neighbours, ncclAllReduce of the abort flag, on its
 * own communication stream ordered by events against the context stream). */
#define MPM_DIST_ID_BYTES 128
int mpm_dist_unique_id(void* id_out);
int mpm_dist_attach_nccl(mpm_ctx* ctx, int rank, int nranks, const void* nccl_id, int cell_lo, int cell_hi,
                         int64_t mig_cap);
/* n decomposed steps (MPM_ADV_NAN_GUARD as mpm_advance); *device_ms (may be NULL) = CUDA-event
 * time of the steps on the context stream */
int mpm_dist_advance(mpm_ctx* ctx, int64_t n_steps, uint32_t flags, double* device_ms);
/* Same-process ranks (several contexts driven by one host thread, e.g. R slabs on one GPU): ctxs[r]
 * is rank r of bounds[r]..bounds[r+1]; exchanges are device copies ordered by events. */
int mpm_dist_attach_local(mpm_ctx* const* ctxs, int nranks, const int* bounds, int64_t mig_cap);
int mpm_dist_advance_local(mpm_ctx* const* ctxs, int nranks, int64_t n_steps, uint32_t flags);
/* backprop_trajectory (checkpoint.hpp:72-143) over the decomposition, device-resident: per-rank
 * HBM checkpoints and replay slots, rank-local digests (a mismatch on any rank fails all), the
 * Lagrangian least-squares seeder on global particle ids in [0, id_space), the cotangent rows of
 * migrants returned to their step-t owner, the decomposed step_vjp with two halo exchanges.
 * Out: this rank's cotangent of S^0 (c0, storage order, c0->n rows; size the view with
 * mpm_local_count) with the rows' global ids, and the rank-ordered sums of the loss and the
 * ParamGrads (every rank gets the same). */
int mpm_dist_backprop(mpm_ctx* ctx, int64_t total_steps, int n_segments, const mpm_seeder_desc* seeder,
                      int64_t id_space, mpm_cot_view* c0, int64_t* c0_ids, mpm_param_grads* pg,
                      mpm_backprop_result* res);
/* the same for same-process ranks (one host thread per rank inside the call): c0s[r] / c0_ids[r]
 * per rank, pg / res once */
int mpm_dist_backprop_local(mpm_ctx* const* ctxs, int nranks, int64_t total_steps, int n_segments,
                            const mpm_seeder_desc* seeder, int64_t id_space, mpm_cot_view* c0s,
                            int64_t* const* c0_ids, mpm_param_grads* pg, mpm_backprop_result* res);

/* ---- instrumentation (bench / tests) --------------------------------------------------- */
/* enable per-kernel CUDA-event timing on the context stream */
int mpm_profile_enable(mpm_ctx* ctx, int enable);
/* total device time (ms) and launch count of kernels whose name contains `name` since the
 * last reset; name = "" sums all kernels of this library */
int mpm_profile_query(mpm_ctx* ctx, const char* name, double* ms, int64_t* launches);
int mpm_profile_reset(mpm_ctx* ctx);
/* number of this library's kernels launched on the context so far */
int64_t mpm_launch_count(const mpm_ctx* ctx);
/* number of active grid nodes (m > mass_epsilon) of the last P2G, and occupied blocks */
int mpm_grid_stats(mpm_ctx* ctx, int64_t* active_nodes, int64_t* occupied_blocks, int64_t* active_node_blocks);

#ifdef __cplusplus
}
#endif

#endif /* MPM_CAPI_H */
