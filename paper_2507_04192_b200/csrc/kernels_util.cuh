// kernels_util.cuh -- boundary conversion and bookkeeping kernels.
//
// Host views use the reference's layout (std::vector<Eigen::Matrix>: vectors [n][d],
// matrices [n][d*d] column-major). Upload places particle id p at storage slot p; download
// scatters every slot back to its id, so the device's sorted order never leaks out.
#pragma once

#include "common.cuh"

namespace mpmgpu {

// staging layout (elements of T): per field a contiguous [n][comps] block
enum StageField { S_X, S_V, S_M, S_VOL, S_RHO, S_EPS, S_SZZ, S_SIG, S_GV, S_AFF, S_F, S_NFIELDS };

template <int D> __host__ __device__ constexpr int stage_comps(int f)
{
    return (f == S_X || f == S_V) ? D : (f >= S_SIG ? D * D : 1);
}

template <class T, int D> struct Stage {
    T* f[S_NFIELDS];
};

template <class T, int D>
__global__ void k_upload(Stage<T, D> S, PBuf<T, D> P, int n, int has_szz, int has_aff, int has_F,
                         const long long* __restrict__ ids)
{
    using C = Cfg<D>;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        P.x[a][i] = S.f[S_X][i * D + a];
        P.v[a][i] = S.f[S_V][i * D + a];
    }
    P.m[i] = S.f[S_M][i];
    P.V[i] = S.f[S_VOL][i];
    P.rho[i] = S.f[S_RHO][i];
    P.eps[i] = S.f[S_EPS][i];
    if (D == 2)
        P.szz[i] = has_szz ? S.f[S_SZZ][i] : T(0);
    // column-major (r, c) at c*D + r; packed symmetric keeps the upper triangle (r <= c)
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = r; c < D; ++c)
            P.sig[sym_idx<D>(r, c)][i] = S.f[S_SIG][i * D * D + c * D + r];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) {
            P.gv[r * D + c][i] = S.f[S_GV][i * D * D + c * D + r];
            if (has_aff)
                P.aff[r * D + c][i] = S.f[S_AFF][i * D * D + c * D + r];
            if (has_F)
                P.F[r * D + c][i] = S.f[S_F][i * D * D + c * D + r];
        }
    P.pid[i] = ids ? int(ids[i]) : i;
    (void)C::NS;
}

// the packed-symmetric stress contract, checked on the staged upload (lowest offending index)
template <class T, int D>
__global__ void k_check_sym(const T* __restrict__ sig, int n, int* __restrict__ bad)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    bool ok = true;
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = r + 1; c < D; ++c) {
            const T a = sig[i * D * D + c * D + r], b = sig[i * D * D + r * D + c];
            const T scale = fmax(fabs(a), fabs(b));
            ok = ok && !(fabs(a - b) > T(1e-5) * scale); // NaN passes here, as on the host
        }
    if (!ok)
        atomicMin(bad, i);
}

// append migrated particles (records sorted by pid beforehand) at storage [base, base + n)
template <class T, int D>
__global__ void k_mig_unpack(PBuf<T, D> P, int base, int n, const T* __restrict__ recs, const int* __restrict__ pids,
                             const int* __restrict__ order, int rec, int has_aff, int has_F)
{
    using C = Cfg<D>;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n)
        return;
    const int r = order[j];
    const T* in = recs + (size_t)r * rec;
    const int i = base + j;
    int q = 0;
#pragma unroll
    for (int a = 0; a < D; ++a)
        P.x[a][i] = in[q++];
#pragma unroll
    for (int a = 0; a < D; ++a)
        P.v[a][i] = in[q++];
    P.m[i] = in[q++];
    P.V[i] = in[q++];
    P.rho[i] = in[q++];
    P.eps[i] = in[q++];
    const T szz = in[q++];
    if (D == 2)
        P.szz[i] = szz;
#pragma unroll
    for (int s = 0; s < C::NS; ++s)
        P.sig[s][i] = in[q++];
#pragma unroll
    for (int k = 0; k < D * D; ++k)
        P.gv[k][i] = in[q++];
    if (has_aff)
        for (int k = 0; k < D * D; ++k)
            P.aff[k][i] = in[q++];
    if (has_F)
        for (int k = 0; k < D * D; ++k)
            P.F[k][i] = in[q++];
    P.pid[i] = pids[r];
}

// halo planes of a set of node fields: node x-planes [p0, p0 + np) x all (y[, z]) nodes, nf values
// per node (forward: m, p, f; adjoint: the v and v_old cotangents). Export writes zeros for
// inactive node blocks; import adds into active blocks only, in a fixed order (received + own, or
// own + received) so both owners of a band agree bitwise.
template <class T> struct HaloFields {
    T* f[7];
    int nf;
};

template <class T, int D>
__global__ void k_halo(HaloFields<T> H, const unsigned char* __restrict__ nflag, const int* __restrict__ nnb,
                       const int* __restrict__ cells, int p0, int np, T* __restrict__ buf, int mode)
{
    using C = Cfg<D>;
    long long per = 1;
    for (int a = 1; a < D; ++a)
        per *= cells[a] + 1;
    const long long total = per * np;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total)
        return;
    int n[D];
    n[0] = p0 + int(t / per);
    long long rem = t % per;
    for (int a = D - 1; a >= 1; --a) {
        n[a] = int(rem % (cells[a] + 1));
        rem /= cells[a] + 1;
    }
    int q = 0, loc = 0;
    bool ok = n[0] >= 0 && n[0] <= cells[0];
    for (int a = 0; a < D; ++a) {
        q = q * nnb[a] + (n[a] >> C::LOGB);
        loc = (loc << C::LOGB) | (n[a] & (C::B - 1));
    }
    ok = ok && nflag[q];
    const size_t gi = (size_t)q * C::NB + loc;
    T* b = buf + (size_t)t * H.nf;
    if (mode == 0) {
        for (int f = 0; f < H.nf; ++f)
            b[f] = ok ? H.f[f][gi] : T(0);
    } else if (ok) {
        for (int f = 0; f < H.nf; ++f)
            H.f[f][gi] = mode == 1 ? b[f] + H.f[f][gi] : H.f[f][gi] + b[f];
    }
}

template <class T, int D>
__global__ void k_download(Stage<T, D> S, PBuf<T, D> P, int n, int has_aff, int has_F)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const int p = P.pid[i];
    if (p < 0)
        return; // vacated slot
#pragma unroll
    for (int a = 0; a < D; ++a) {
        S.f[S_X][p * D + a] = P.x[a][i];
        S.f[S_V][p * D + a] = P.v[a][i];
    }
    S.f[S_M][p] = P.m[i];
    S.f[S_VOL][p] = P.V[i];
    S.f[S_RHO][p] = P.rho[i];
    S.f[S_EPS][p] = P.eps[i];
    if (D == 2)
        S.f[S_SZZ][p] = P.szz[i];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) {
            S.f[S_SIG][p * D * D + c * D + r] = P.sig[sym_idx<D>(r, c)][i];
            S.f[S_GV][p * D * D + c * D + r] = P.gv[r * D + c][i];
            if (has_aff)
                S.f[S_AFF][p * D * D + c * D + r] = P.aff[r * D + c][i];
            if (has_F)
                S.f[S_F][p * D * D + c * D + r] = P.F[r * D + c][i];
        }
}

// ---- device scene seeding (init_scene, scene.hpp:55-116) ------------------------------------
// exact IEEE ops (no FMA contraction) so the lattice matches the host seeding bit for bit
template <class T> __device__ __forceinline__ T radd(T a, T b);
template <class T> __device__ __forceinline__ T rmul(T a, T b);
template <> __device__ __forceinline__ double radd<double>(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ float radd<float>(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double rmul<double>(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ float rmul<float>(float a, float b) { return __fmul_rn(a, b); }

struct SeedBox {
    int lo[3], ext[3];
    long long ncell;
};

template <class T, int D>
__device__ __forceinline__ void seed_points(const DevScene<T, D>& sc, const SeedBox& bx, long long c, T (*p)[D])
{
    int ci[D];
    long long r = c;
    for (int a = D - 1; a >= 0; --a) {
        ci[a] = bx.lo[a] + int(r % bx.ext[a]);
        r /= bx.ext[a];
    }
    const T quarter = sc.dh / T(4); // exact
#pragma unroll
    for (int k = 0; k < (1 << D); ++k)
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const T center = radd<T>(sc.origin[a], rmul<T>(radd<T>(T(ci[a]), T(0.5)), sc.dh));
            p[k][a] = ((k >> a) & 1) ? radd<T>(center, quarter) : radd<T>(center, -quarter);
        }
}

template <class T, int D> __device__ __forceinline__ int seed_owner(const mpm_region* rg, int nreg, const T* p)
{
    for (int r = 0; r < nreg; ++r) {
        const mpm_region& g = rg[r];
        bool ok = true;
        if (g.shape == 0) {
            for (int a = 0; a < D; ++a)
                ok = ok && p[a] >= T(g.lo[a]) && p[a] < T(g.hi[a]);
        } else {
            if (D == 3)
                ok = p[2] >= T(g.zmin) && p[2] < T(g.zmax);
            const T dx = radd<T>(p[0], -T(g.center[0])), dy = radd<T>(p[1], -T(g.center[1]));
            const T rr = rmul<T>(T(g.radius), T(g.radius));
            ok = ok && radd<T>(rmul<T>(dx, dx), rmul<T>(dy, dy)) < rr;
        }
        if (ok)
            return r;
    }
    return -1;
}

template <class T, int D>
__global__ void k_seed_count(DevScene<T, D> sc, SeedBox bx, const mpm_region* __restrict__ rg, int nreg,
                             int* __restrict__ counts)
{
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= bx.ncell)
        return;
    T p[1 << D][D];
    seed_points<T, D>(sc, bx, c, p);
    int k = 0;
#pragma unroll
    for (int q = 0; q < (1 << D); ++q)
        k += seed_owner<T, D>(rg, nreg, p[q]) >= 0;
    counts[c] = k;
}

template <class T, int D>
__global__ void k_seed_write(DevScene<T, D> sc, SeedBox bx, const mpm_region* __restrict__ rg, int nreg,
                             const int* __restrict__ offs, PBuf<T, D> P, T mass, T volume, T rho0, int has_aff,
                             int has_F)
{
    using C = Cfg<D>;
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= bx.ncell)
        return;
    T p[1 << D][D];
    seed_points<T, D>(sc, bx, c, p);
    int i = offs[c];
    for (int q = 0; q < (1 << D); ++q) {
        const int r = seed_owner<T, D>(rg, nreg, p[q]);
        if (r < 0)
            continue;
        const mpm_region& g = rg[r];
        T v[D];
        for (int a = 0; a < D; ++a)
            v[a] = T(0);
        const T yr = radd<T>(p[q][1], -T(g.min_y));
        if (g.vel_kind == 0) { // VelocityExpr::evaluate (config.hpp:109-129)
            for (int a = 0; a < D; ++a)
                v[a] = T(g.value[a]);
        } else if (g.vel_kind == 1) {
            v[0] = rmul<T>(T(g.alpha), radd<T>(T(g.h0), -yr));
        } else {
            const T yn = yr / T(g.h0);
            const T arg = rmul<T>(rmul<T>(T(g.frequency), T(3.14159265358979323846)), yn);
            v[0] = radd<T>(rmul<T>(T(g.amplitude), radd<T>(T(1), -rmul<T>(yn, yn))),
                           rmul<T>(T(g.perturbation), T(sin(double(arg)))));
        }
        for (int a = 0; a < D; ++a) {
            P.x[a][i] = p[q][a];
            P.v[a][i] = v[a];
        }
        P.m[i] = mass;
        P.V[i] = volume;
        P.rho[i] = rho0;
        P.eps[i] = T(0);
        if (D == 2)
            P.szz[i] = T(0);
        for (int s2 = 0; s2 < C::NS; ++s2)
            P.sig[s2][i] = T(0);
        for (int k = 0; k < D * D; ++k) {
            P.gv[k][i] = T(0);
            if (has_aff)
                P.aff[k][i] = T(0);
            if (has_F)
                P.F[k][i] = (k % (D + 1) == 0) ? T(1) : T(0);
        }
        P.pid[i] = i;
        ++i;
    }
}

// slab step report for the caller's collective: (failed, left toward -x, left toward +x)
__global__ void k_report(const DevStatus* st, long long* out)
{
    out[0] = st->abort ? 1 : 0;
    out[1] = st->mig_lo;
    out[2] = st->mig_hi;
}

// compact download for a slab: slot list idx[0..k) (storage order), ids alongside
template <class T, int D>
__global__ void k_download_compact(Stage<T, D> S, PBuf<T, D> P, const int* __restrict__ idx, int k, int has_aff,
                                   int has_F, long long* __restrict__ ids)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k)
        return;
    const int i = idx[j];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        S.f[S_X][j * D + a] = P.x[a][i];
        S.f[S_V][j * D + a] = P.v[a][i];
    }
    S.f[S_M][j] = P.m[i];
    S.f[S_VOL][j] = P.V[i];
    S.f[S_RHO][j] = P.rho[i];
    S.f[S_EPS][j] = P.eps[i];
    if (D == 2)
        S.f[S_SZZ][j] = P.szz[i];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) {
            S.f[S_SIG][j * D * D + c * D + r] = P.sig[sym_idx<D>(r, c)][i];
            S.f[S_GV][j * D * D + c * D + r] = P.gv[r * D + c][i];
            if (has_aff)
                S.f[S_AFF][j * D * D + c * D + r] = P.aff[r * D + c][i];
            if (has_F)
                S.f[S_F][j * D * D + c * D + r] = P.F[r * D + c][i];
        }
    ids[j] = P.pid[i];
}

struct AliveSlot {
    const int* pid;
    __device__ __forceinline__ bool operator()(int i) const { return pid[i] >= 0; }
};

// ---- occupied-block list, heaviest blocks first, taken through a work counter ----------------
// The list order is free: every listed block's outputs depend only on the block, not on which
// CTA runs it or when. So it is chosen for load balance. Blocks are bucketed by particle count
// (two buckets per octave) and listed heaviest bucket first; the persistent kernels take blocks
// from the list through an atomic counter (longest-processing-time first), so a launch's tail is
// made of light blocks instead of whichever blocks a static CTA stride happened to leave last.
__global__ void k_occ_hist(const int* __restrict__ bstart, const int* __restrict__ bend, int n, int* __restrict__ wq)
{
    __shared__ int h[OCC_NBUCKET];
    for (int t = threadIdx.x; t < OCC_NBUCKET; t += blockDim.x)
        h[t] = 0;
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && bstart[i] >= 0)
        atomicAdd(&h[occ_bucket(bend[i] - bstart[i])], 1);
    __syncthreads();
    for (int t = threadIdx.x; t < OCC_NBUCKET; t += blockDim.x)
        if (h[t])
            atomicAdd(&wq[WQ_HIST + t], h[t]);
}

__global__ void k_occ_scatter(const int* __restrict__ bstart, const int* __restrict__ bend, int n, int* __restrict__ wq,
                              int* __restrict__ list, int* __restrict__ count)
{
    __shared__ int off[OCC_NBUCKET];
    if (threadIdx.x == 0) {
        int s = 0;
        for (int b = OCC_NBUCKET - 1; b >= 0; --b) {
            off[b] = s;
            s += wq[WQ_HIST + b];
        }
        if (blockIdx.x == 0)
            *count = s;
    }
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && bstart[i] >= 0) {
        const int b = occ_bucket(bend[i] - bstart[i]);
        list[off[b] + atomicAdd(&wq[WQ_CUR + b], 1)] = i;
    }
}

// unordered compaction of a dense predicate (list order does not affect results: every
// listed block is processed independently)
__global__ void k_compact_pos(const int* __restrict__ dense, int n, int* __restrict__ list, int* __restrict__ count)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool p = i < n && dense[i] >= 0;
    unsigned m = __ballot_sync(0xffffffffu, p);
    int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0 && m)
        base = atomicAdd(count, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (p)
        list[base + __popc(m & ((1u << lane) - 1))] = i;
}

__global__ void k_compact_flag(const unsigned char* __restrict__ dense, int n, int* __restrict__ list,
                               int* __restrict__ count)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool p = i < n && dense[i] != 0;
    unsigned m = __ballot_sync(0xffffffffu, p);
    int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0 && m)
        base = atomicAdd(count, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (p)
        list[base + __popc(m & ((1u << lane) - 1))] = i;
}

// ---- digest: order-independent 64-bit sum of per-particle content hashes -------------
__device__ __forceinline__ unsigned long long mix64(unsigned long long z)
{
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
template <class T> __device__ __forceinline__ unsigned long long bits_of(T x);
template <> __device__ __forceinline__ unsigned long long bits_of<double>(double x)
{
    return (unsigned long long)__double_as_longlong(x);
}
template <> __device__ __forceinline__ unsigned long long bits_of<float>(float x)
{
    return (unsigned long long)(unsigned)__float_as_uint(x);
}

template <class T, int D>
__global__ void k_digest(PBuf<T, D> P, int n, int has_aff, unsigned long long* out)
{
    using C = Cfg<D>;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long h = 0;
    if (i < n && P.pid[i] >= 0) {
        h = mix64((unsigned long long)P.pid[i]);
#pragma unroll
        for (int a = 0; a < D; ++a) {
            h = mix64(h ^ bits_of(P.x[a][i]));
            h = mix64(h ^ bits_of(P.v[a][i]));
        }
        h = mix64(h ^ bits_of(P.V[i]));
        h = mix64(h ^ bits_of(P.rho[i]));
        h = mix64(h ^ bits_of(P.eps[i]));
        if (D == 2)
            h = mix64(h ^ bits_of(P.szz[i]));
#pragma unroll
        for (int s = 0; s < C::NS; ++s)
            h = mix64(h ^ bits_of(P.sig[s][i]));
#pragma unroll
        for (int k = 0; k < D * D; ++k) {
            h = mix64(h ^ bits_of(P.gv[k][i]));
            if (has_aff)
                h = mix64(h ^ bits_of(P.aff[k][i]));
        }
    }
    for (int o = 16; o > 0; o >>= 1)
        h += __shfl_down_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0)
        atomicAdd(out, h);
}

// max |v| (stepper.hpp:78-85) as the bit pattern of a non-negative double
template <class T, int D>
__global__ void k_max_speed(PBuf<T, D> P, int n, unsigned long long* out)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    double s = 0;
    if (i < n && P.pid[i] >= 0) {
        T q = T(0);
#pragma unroll
        for (int a = 0; a < D; ++a)
            q += P.v[a][i] * P.v[a][i];
        s = (double)dsqrt<T>(q);
        if (!(s >= 0))
            s = __longlong_as_double(0x7ff0000000000000ll); // NaN -> +inf
    }
    for (int o = 16; o > 0; o >>= 1)
        s = fmax(s, __shfl_down_sync(0xffffffffu, s, o));
    if ((threadIdx.x & 31) == 0)
        atomicMax(out, (unsigned long long)__double_as_longlong(s));
}

} // namespace mpmgpu
