// common.cuh -- device-side scene block, HBM layouts and stencil math for the B200 MPM path.
//
// Layout decisions:
//  * particles: structure-of-arrays, one array per scalar component, kept in cell-sorted
//    order (block of base cell, then base cell, stable) -- re-established every step by a
//    stable radix sort of 32-bit cell keys; the reference's particle id travels in `pid`.
//    sigma is stored packed-symmetric (3 in 2-D, 6 in 3-D), grad_v / affine / F full.
//  * grid: dense table of B^d node blocks (B = 16 in 2-D, 8 in 3-D) over the whole domain;
//    only blocks adjacent to occupied particle blocks are touched in a step.
//  * P2G partials: one (B+2)^d node tile per occupied particle block (its particles' full
//    stencil support), combined per node in a fixed order -> deterministic, atomic-free.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mpmgpu {

constexpr int MAX_OBST = 16;
constexpr int MAX_FRIC = 64;

template <int D> struct Cfg {
    static constexpr int B = D == 2 ? 16 : 8;              // cells per block edge
    static constexpr int LOGB = D == 2 ? 4 : 3;
    static constexpr int NB = D == 2 ? 256 : 512;          // cells (= nodes) per block
    static constexpr int LOGNB = D == 2 ? 8 : 9;
    static constexpr int TE = B + 2;                       // tile edge (nodes)
    static constexpr int TN = D == 2 ? TE * TE : TE * TE * TE; // tile nodes
    static constexpr int NOFF = D == 2 ? 9 : 27;           // stencil nodes
    static constexpr int NS = D == 2 ? 3 : 6;              // packed symmetric stress
    static constexpr int NF = 1 + 2 * D;                   // P2G fields: m, p[D], f[D]
    static constexpr int NCOL = D == 2 ? TE : TE * TE;     // node columns of a tile
    static constexpr int SEGS = D == 2 ? 8 : 2;            // march segments (B % SEGS == 0, >= 2 levels each)
};

// occupied-block list buckets and work counters (the list kernels are in kernels_util.cuh)
constexpr int OCC_NBUCKET = 64;
constexpr int WQ_HIST = 0, WQ_CUR = OCC_NBUCKET, WQ_CTR = 2 * OCC_NBUCKET; // scratch layout
constexpr int WQ_P2G = WQ_CTR, WQ_G2P = WQ_CTR + 2, WQ_K5A = WQ_CTR + 4, WQ_K5B = WQ_CTR + 6, WQ_K7 = WQ_CTR + 8;
constexpr int WQ_INTS = WQ_CTR + 16; // one counter pair per kernel

__device__ __forceinline__ int occ_bucket(int cnt) // cnt >= 1
{
    const int L = 31 - __clz(cnt);
    const int half = L > 0 ? (cnt >> (L - 1)) & 1 : 0;
    return min(2 * L + half, OCC_NBUCKET - 1);
}

// A CTA's exit from a work-counter loop: the last CTA out resets the pair (next item, CTAs done)
// for the next launch. Every CTA must call it exactly once, after its final fetch.
// wq == nullptr: the plain static stride (blockIdx.x, + gridDim.x, ...), no counter.
__device__ __forceinline__ int wq_first(int* wq) { return wq ? atomicAdd(wq, 1) : int(blockIdx.x); }
__device__ __forceinline__ int wq_next(int* wq, int w) { return wq ? atomicAdd(wq, 1) : w + int(gridDim.x); }
__device__ __forceinline__ void wq_finish(int* pair)
{
    if (pair && threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(pair + 1, 1) == int(gridDim.x) - 1) {
            atomicExch(pair, 0);
            atomicExch(pair + 1, 0);
        }
    }
}

// index of node (tile level z, node column col) inside a P2G partial tile: z fastest, so that
// k_grid's threads (node-block-local index, z fastest) read consecutive addresses
template <int D> __host__ __device__ __forceinline__ int ptile(int z, int col) { return col * Cfg<D>::TE + z; }

// packed symmetric index (i,j) -> slot; 2-D: 00 11 01, 3-D: 00 11 22 01 02 12
template <int D> __host__ __device__ constexpr int sym_idx(int i, int j)
{
    if (i > j) {
        int t = i;
        i = j;
        j = t;
    }
    if (i == j)
        return i;
    if (D == 2)
        return 2;
    return i == 0 ? (j == 1 ? 3 : 4) : 5;
}

// Device copy of Scene<T,dim> (scene.hpp) + derived block geometry; passed by value.
template <class T, int D> struct DevScene {
    T dh, inv_dh, dt, alpha;
    T origin[D], gravity[D];
    int cells[D];
    int scheme; // MPM_SCHEME_*
    int apic, tpic, track_F, material;
    T rho0, visc, c;
    int rate_form;
    T K, G, q_phi, k_phi, q_psi, tau_P, alpha_P, sigma_t;
    int band;
    int wall_kind[2 * D];
    int n_fric[2 * D];
    int fric_off[2 * D];
    T fric[MAX_FRIC];
    int n_obst;
    T obst[MAX_OBST][2 * D];
    T mass_eps;
    // blocks
    int nb[D];    // particle blocks per axis (base cells 0..cells-2)
    int nnb[D];   // node blocks per axis (nodes 0..cells)
    int nb_total, nnb_total;
    // slab decomposition: this context owns particles whose base cell along x lies in
    // [slab_lo, slab_hi); the whole domain otherwise. Walls and Coulomb segments stay global.
    int slab_lo, slab_hi;
    // halo bands: node x-planes [band_lo, band_lo + 2) and [band_hi, band_hi + 2) are shared with
    // the x-neighbours (far outside the grid when there is no neighbour)
    int band_lo, band_hi;
    // scene constants of the constitutive updates, evaluated once on the device with the exact
    // expressions of constitutive.hpp (k_scene_consts) so results are bit-identical
    T dp_lam;      // K - 2G/3
    T dp_dlam_den; // G + K q_phi q_psi
    T dp_deps_fac; // sqrt(1/3 + 2/9 q_psi^2)
    T dp_apex;     // k_phi / q_phi
    T dp_deps_t;   // sqrt(2) / 3
    T fl_k;        // visc / dt (rate form) or visc
};

// particle buffer field order inside one strided allocation (field k at base + k * S)
template <int D> struct PLay {
    static constexpr int X = 0, V = D, M = 2 * D, VOL = 2 * D + 1, RHO = 2 * D + 2, EPS = 2 * D + 3,
                         SZZ = 2 * D + 4, SIG = 2 * D + 4 + (D == 2 ? 1 : 0), GV = SIG + Cfg<D>::NS,
                         AFF = GV + D * D, F = AFF + D * D, END = F + D * D;
};

// particle buffer: SoA pointers (one array per component). The hot kernels address field k as
// base + k * S (PLay order) so that they need two kernel parameters instead of ~40 pointers.
template <class T, int D> struct PBuf {
    T* base;
    long long S;
    T* x[D];
    T* v[D];
    T* m;
    T* V;
    T* rho;
    T* eps;
    T* szz;                  // 2-D only
    T* sig[Cfg<D>::NS];
    T* gv[D * D];            // row-major (i,j) -> i*D+j
    T* aff[D * D];           // APIC only
    T* F[D * D];             // track_def_grad only
    int* pid;
};

// grid node-block storage: component arrays over nnb_total * NB nodes
template <class T, int D> struct GBuf {
    T* m;
    T* p[D];
    T* f[D];
    T* v[D];
    T* vold[D];
};

// device status / error flags (one per context)
struct DevStatus {
    int abort;
    int den_flag;
    int nan_flag;
    int ood_flag;
    int den_pid;
    int ood_pid;
    int far_flag;
    int ood_counted;      // the completed step whose output left the domain was counted
    long long step;       // absolute step index of the state currently in the buffers
    long long err_step;   // step during which a den/nan error occurred
    unsigned long long active_nodes;
    int mig_lo, mig_hi; // particles that left the slab this step, toward -x / +x
    int mig_over;       // export buffer overflow
    int pad2;
};

__global__ void k_reset_status(DevStatus* st, long long step)
{
    DevStatus s{};
    s.den_pid = 0x7fffffff;
    s.ood_pid = 0x7fffffff;
    s.step = step;
    s.err_step = -1;
    *st = s;
}

// per-step reset that keeps the device-maintained step counter (capturable in a graph)
__global__ void k_reset_flags(DevStatus* st)
{
    DevStatus s{};
    s.den_pid = 0x7fffffff;
    s.ood_pid = 0x7fffffff;
    s.step = st->step;
    s.err_step = -1;
    *st = s;
}

constexpr int KEY_OOD = 0x7fffffff;  // out of the domain (error)
constexpr int KEY_DEAD = 0x7ffffffe; // slot vacated by a migrated particle (sorts last, ignored)

// ---- small math ------------------------------------------------------------------------
template <class T> __device__ __forceinline__ T dfloor(T x);
template <> __device__ __forceinline__ double dfloor<double>(double x) { return floor(x); }
template <> __device__ __forceinline__ float dfloor<float>(float x) { return floorf(x); }
template <class T> __device__ __forceinline__ T dsqrt(T x);
template <> __device__ __forceinline__ double dsqrt<double>(double x) { return sqrt(x); }
template <> __device__ __forceinline__ float dsqrt<float>(float x) { return sqrtf(x); }

template <class T> __device__ __forceinline__ bool finite_(T x) { return isfinite(x); }

// Programmatic dependent launch (the step's kernels are launched with it, context.cu launch_pdl):
// a kernel may be scheduled while its predecessor drains; it waits here before touching any of
// the predecessor's outputs, and lets its own successor be scheduled. Both are no-ops for a
// kernel launched the ordinary way.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// quadratic B-spline weights along one axis (bspline.hpp:76-108): base = floor(u - 1/2),
// fx = u - base in [1/2, 3/2); returns false when out of the valid interior.
template <class T> struct Axis {
    int base;
    T w[3], dw[3];
};

template <class T> __device__ __forceinline__ bool axis_stencil(T x, T origin, T inv_dh, int cells, Axis<T>& s)
{
    T u = (x - origin) * inv_dh;
    T fl = dfloor<T>(u - T(0.5));
    if (!(fl >= T(0)) || fl + T(2) > T(cells))
        return false;
    int b = int(fl);
    s.base = b;
    T fx = u - T(b);
    T h0 = T(1.5) - fx, h1 = fx - T(1), h2 = fx - T(0.5);
    s.w[0] = T(0.5) * h0 * h0;
    s.w[1] = T(0.75) - h1 * h1;
    s.w[2] = T(0.5) * h2 * h2;
    s.dw[0] = -h0 * inv_dh;
    s.dw[1] = -T(2) * h1 * inv_dh;
    s.dw[2] = h2 * inv_dh;
    return true;
}

// cell key: particle block id (row-major over nb) << LOGNB | local cell, where the local cell
// is "level-major": the last axis (the P2G march axis) slowest, the others row-major. A base
// level of a block is therefore one contiguous run of the sorted order.
template <int D> __host__ __device__ __forceinline__ int local_cell(const int* b)
{
    using C = Cfg<D>;
    int loc = b[D - 1] & (C::B - 1);
    for (int a = 0; a < D - 1; ++a)
        loc = (loc << C::LOGB) | (b[a] & (C::B - 1));
    return loc;
}

template <class T, int D> __device__ __forceinline__ bool cell_key(const DevScene<T, D>& sc, const T* x, int& key)
{
    using C = Cfg<D>;
    int blk = 0, b[D];
    for (int a = 0; a < D; ++a) {
        T u = (x[a] - sc.origin[a]) * sc.inv_dh;
        T fl = dfloor<T>(u - T(0.5));
        if (!(fl >= T(0)) || fl + T(2) > T(sc.cells[a]))
            return false;
        b[a] = int(fl);
        blk = blk * sc.nb[a] + (b[a] >> C::LOGB);
    }
    key = (blk << C::LOGNB) | local_cell<D>(b);
    return true;
}

template <int D> __host__ __device__ __forceinline__ void block_coords(int blk, const int* nb, int* q)
{
    for (int a = D - 1; a >= 0; --a) {
        q[a] = blk % nb[a];
        blk /= nb[a];
    }
}

} // namespace mpmgpu
