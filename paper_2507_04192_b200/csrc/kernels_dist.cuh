// kernels_dist.cuh -- device side of the library-owned slab decomposition.
//
// A decomposed step keeps every count on the device, so no host synchronisation is needed inside
// an advance() call:
//   * the particle count of a rank lives in `d_n`; the sort (kernels_sort.cuh) leaves the number
//     of particles it placed in `d_nlive` (vacated slots of exported particles are simply not
//     placed), G2P writes that many, and the import below appends the neighbours' migrants;
//   * migration messages have a fixed capacity (count + cap records per neighbour per step), so the
//     transport's sizes never depend on device data;
//   * the abort flag of every rank is max-reduced on the device once per step; a rank whose peer
//     failed skips its remaining steps exactly as if it had failed itself, and the host looks at
//     the status once, after the call (errors are checked lazily, one call behind the device).
#pragma once

#include "common.cuh"
#include "kernels_adj.cuh"
#include "kernels_fwd.cuh"

namespace mpmgpu {

// begin a decomposed step: the export counters restart (the abort state is sticky)
__global__ void k_dist_step_begin(DevStatus* st)
{
    st->mig_lo = 0;
    st->mig_hi = 0;
}

// publish this step's exports (G2P counted them) into the outgoing message headers, and the local
// abort flag into the reduction buffer
__global__ void k_dist_publish(const DevStatus* st, long long* cnt_lo, long long* cnt_hi, int* abort_red, int cap)
{
    *cnt_lo = st->mig_lo < cap ? st->mig_lo : cap;
    *cnt_hi = st->mig_hi < cap ? st->mig_hi : cap;
    *abort_red = st->abort;
}

// after the max-reduction: a peer's failure stops this rank too (pad2 = 1 records "peer")
__global__ void k_dist_merge_abort(DevStatus* st, const int* abort_red)
{
    if (*abort_red && !st->abort) {
        st->abort = 1;
        st->pad2 = 1;
    }
}

// same-process ranks: the max of every rank's published abort flag
constexpr int DIST_MAX_LOCAL = 64;
struct AbortPtrs {
    const int* p[DIST_MAX_LOCAL];
    int R;
};
__global__ void k_dist_abort_max(AbortPtrs a, int* out)
{
    int m = 0;
    for (int r = 0; r < a.R; ++r)
        m = max(m, *a.p[r]);
    *out = m;
}

// n_live after a full (radix) sort: the end of the last occupied block (blocks are contiguous)
__global__ void k_dist_nlive(const int* __restrict__ bend, int nb_total, int* __restrict__ nlive)
{
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nb_total && bend[b] > 0)
        atomicMax(nlive, bend[b]);
}

// append the migrants received from the lower (lo) and upper (hi) neighbour at d_nlive: lo's
// records first, then hi's, each in particle-id order (a rank by comparison inside the message:
// the sender's export order comes from atomics), so the storage order -- and with it the next sort
// and every sum -- is deterministic. Imported slots get an invalid previous key (-1): the
// incremental sort treats them as arrivals. New count -> d_n.
template <class T, int D>
__global__ void k_dist_import(DevScene<T, D> sc, PBuf<T, D> P, const int* __restrict__ d_nlive, int* __restrict__ d_n,
                              const long long* __restrict__ cnt_lo, const T* __restrict__ recs_lo,
                              const int* __restrict__ pid_lo, const long long* __restrict__ cnt_hi,
                              const T* __restrict__ recs_hi, const int* __restrict__ pid_hi, int cap, int rec,
                              int has_aff, int has_F, int* __restrict__ keys, int* __restrict__ okeys, int capacity,
                              DevStatus* st)
{
    using C = Cfg<D>;
    const int klo = int(*cnt_lo), khi = int(*cnt_hi), base = *d_nlive;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j == 0) {
        if (base + klo + khi > capacity) {
            st->mig_over = 1;
            st->abort = 1;
        } else {
            *d_n = base + klo + khi;
        }
    }
    if (j >= klo + khi || base + klo + khi > capacity)
        return;
    const bool from_lo = j < klo;
    const int r = from_lo ? j : j - klo, k = from_lo ? klo : khi;
    const int* pids = from_lo ? pid_lo : pid_hi;
    const int me = pids[r];
    int rank = 0;
    for (int l = 0; l < k; ++l)
        rank += pids[l] < me;
    const int i = base + (from_lo ? 0 : klo) + rank;
    const T* in = (from_lo ? recs_lo : recs_hi) + (size_t)r * rec;
    int q = 0;
    T x[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        x[a] = in[q++];
        P.x[a][i] = x[a];
    }
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
    for (int k2 = 0; k2 < D * D; ++k2)
        P.gv[k2][i] = in[q++];
    if (has_aff)
        for (int k2 = 0; k2 < D * D; ++k2)
            P.aff[k2][i] = in[q++];
    if (has_F)
        for (int k2 = 0; k2 < D * D; ++k2)
            P.F[k2][i] = in[q++];
    P.pid[i] = me;
    int key;
    if (!cell_key<T, D>(sc, x, key)) {
        key = KEY_OOD;
        atomicMin(&st->ood_pid, me);
        st->ood_flag = 2;
        st->abort = 1;
    }
    keys[i] = key;
    okeys[i] = -1;
}

// ---- decomposed adjoint: the cotangent rows of migrants go back to their step-t owner ----------
// A particle exported by rank r during step t sits, at t+1, on the neighbour (appended after the
// neighbour's G2P output in particle-id order). The VJP of step t runs on r, which holds the particle
// in S^t; it needs the particle's cotangent of S^{t+1}, i.e. the neighbour's row. The neighbour packs
// the rows of its imports from r (fixed capacity, count in front) and r writes them into the slots
// its G2P vacated (export list sorted by particle id = the neighbour's import order).
template <class T, int D> __device__ __forceinline__ int cot_row_values(int has_aff) { return 2 * D + 2 + (D == 2 ? 1 : 0) + 2 * D * D + (has_aff ? D * D : 0); }

template <class T, int D>
__device__ __forceinline__ void cot_row_io(CBuf<T, D>& c, int i, T* row, bool load, int gv_zero, int has_aff)
{
    int q = 0;
    auto io = [&](T* a) {
        if (load)
            row[q] = a ? a[i] : T(0);
        else if (a)
            a[i] = row[q];
        ++q;
    };
#pragma unroll
    for (int a = 0; a < D; ++a)
        io(c.x[a]);
#pragma unroll
    for (int a = 0; a < D; ++a)
        io(c.v[a]);
    io(c.rho);
    io(c.V);
    if (D == 2)
        io(c.szz);
#pragma unroll
    for (int k = 0; k < D * D; ++k)
        io(c.sig[k]);
#pragma unroll
    for (int k = 0; k < D * D; ++k)
        io(gv_zero ? nullptr : c.gv[k]);
    if (has_aff)
        for (int k = 0; k < D * D; ++k)
            io(c.aff[k]);
}

// rows [base + off, base + off + k) of cot -> out (k = *cnt, base = *nlive); off = 0 for the imports
// from the lower neighbour, *cnt_lo for those from the upper one
template <class T, int D>
__global__ void k_cot_pack(CBuf<T, D> c, const int* __restrict__ nlive, const long long* __restrict__ cnt_lo,
                           const long long* __restrict__ cnt, int upper, T* __restrict__ out, int gv_zero, int has_aff)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = int(*cnt);
    if (j >= k)
        return;
    const int i = *nlive + (upper ? int(*cnt_lo) : 0) + j;
    const int nv = cot_row_values<T, D>(has_aff);
    cot_row_io<T, D>(c, i, out + (size_t)j * nv, true, gv_zero, has_aff);
}

// in (rows in particle-id order of this rank's exports to one side) -> cot at the vacated slots
template <class T, int D>
__global__ void k_cot_unpack(CBuf<T, D> c, const long long* __restrict__ ex_cnt, const int* __restrict__ ex_pid,
                             const int* __restrict__ ex_slot, const T* __restrict__ in, int gv_zero, int has_aff)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = int(*ex_cnt);
    if (e >= k)
        return;
    const int me = ex_pid[e];
    int rank = 0;
    for (int l = 0; l < k; ++l)
        rank += ex_pid[l] < me;
    const int nv = cot_row_values<T, D>(has_aff);
    T row[2 * D + 3 + 3 * D * D];
    const T* r = in + (size_t)rank * nv;
    for (int q = 0; q < nv; ++q)
        row[q] = r[q];
    cot_row_io<T, D>(c, ex_slot[e], row, false, gv_zero, has_aff);
}

// the export counts of the step just taken (G2P's counters; capped like the messages)
__global__ void k_dist_export_counts(const DevStatus* st, long long* cnt, int cap)
{
    cnt[0] = st->mig_lo < cap ? st->mig_lo : cap;
    cnt[1] = st->mig_hi < cap ? st->mig_hi : cap;
}

} // namespace mpmgpu
