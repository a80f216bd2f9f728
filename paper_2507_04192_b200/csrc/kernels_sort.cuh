// kernels_sort.cuh -- K1: the per-step cell sort kept incrementally (north_star (1)).
//
// The particle state is stored in the order of the previous step's sort (G2P writes slot i with
// the particle the sort put at position i), and CFL < 1 moves a particle by less than a cell per
// step. So the previous sorted keys `okeys` (non-decreasing, in storage order) and the new keys
// `keys` (same storage order) differ only at the few particles that changed cell. The required
// result is the stable sort of `keys` over the storage index -- exactly what the radix sort of
// (key, index) pairs returns (SPEC.md:149,155 canonical order; transfer.hpp:43 particle-index
// order inside a cell) -- and it is rebuilt here block by block:
//
//   k_inc_classify  thread per particle: a particle whose block changed is a cross-block mover;
//                   per-block in / out counts, mover list (order irrelevant: sorted later)
//   k_inc_scan      one CTA over the dense block table: new count = old range - out + in,
//                   exclusive scans -> bstart / bend, in-mover offsets, the occupied-block list
//                   (heaviest first for the 3-D work-counter kernels)
//   k_inc_place     movers into their destination block's bucket (atomic slot, order fixed later)
//   k_inc_block     CTA per occupied block: its members in storage order are
//                     [in-movers below the old range] [stayers of the old range] [in-movers above]
//                   (the old range is contiguous in storage and in-movers come from other
//                   blocks, so this concatenation is ordered by storage index); a stable
//                   counting sort by local cell (histogram, scan, per-warp match ranks) writes
//                   perm / keys_sorted / the level starts.
//
// Bitwise the same perm and keys_sorted as the radix sort for every input (tests compare the
// states after many steps); there is no capacity limit, only a slower path when a block
// receives more than one CTA's worth of movers in one step. The first sort after an upload (or a
// migration import) has no previous order and uses the full radix sort.
#pragma once

#include "common.cuh"

namespace mpmgpu {

constexpr int INC_THREADS = 256; // k_inc_block CTA size
constexpr int INC_WARPS = INC_THREADS / 32;

// scratch of the incremental sort, owned by the context (self-cleaning: every counter the
// kernels raise is returned to zero by a later kernel of the same sort)
struct IncSort {
    int* cnt_in;  // [nb_total] movers arriving per block (zeroed by k_inc_block)
    int* cnt_out; // [nb_total] movers leaving per block; reused as the bucket cursor (zeroed by k_inc_scan / k_inc_block)
    int* in_off;  // [nb_total] bucket offset of a block's in-movers
    int* xlist;   // [cap] mover storage indices; then the buckets sorted by index
    int* inbuf;   // [cap] mover buckets (unordered within a bucket)
    int* nx;      // [1] mover count (zeroed by k_inc_block)
};

template <int D>
__global__ void __launch_bounds__(256) k_inc_classify(const int* __restrict__ keys, const int* __restrict__ okeys, int n,
                                                      int nb_total, IncSort S)
{
    using C = Cfg<D>;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool mover = false, valid = false;
    if (i < n) {
        const int b = keys[i] >> C::LOGNB, ob = okeys[i] >> C::LOGNB;
        if (b != ob) {
            mover = true;
            valid = b < nb_total; // out-of-domain / dead keys join no block (the step aborts)
            if (valid)
                atomicAdd(&S.cnt_in[b], 1);
            if (ob < nb_total)
                atomicAdd(&S.cnt_out[ob], 1);
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, mover && valid);
    if (m) {
        const int lane = threadIdx.x & 31;
        int base = 0;
        if (lane == 0)
            base = atomicAdd(S.nx, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (mover && valid)
            S.xlist[base + __popc(m & ((1u << lane) - 1))] = i;
    }
}

// exclusive scan of three ints over a 1024-thread CTA (warp shuffles + one smem round)
__device__ __forceinline__ void cta_scan3(int& a, int& b, int& c, int (*ws)[3], int* tot)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int xa = a, xb = b, xc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int ya = __shfl_up_sync(0xffffffffu, xa, o), yb = __shfl_up_sync(0xffffffffu, xb, o),
                  yc = __shfl_up_sync(0xffffffffu, xc, o);
        if (lane >= o) {
            xa += ya;
            xb += yb;
            xc += yc;
        }
    }
    if (lane == 31) {
        ws[w][0] = xa;
        ws[w][1] = xb;
        ws[w][2] = xc;
    }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        int va = lane < nw ? ws[lane][0] : 0, vb = lane < nw ? ws[lane][1] : 0, vc = lane < nw ? ws[lane][2] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int ya = __shfl_up_sync(0xffffffffu, va, o), yb = __shfl_up_sync(0xffffffffu, vb, o),
                      yc = __shfl_up_sync(0xffffffffu, vc, o);
            if (lane >= o) {
                va += ya;
                vb += yb;
                vc += yc;
            }
        }
        if (lane < nw) {
            ws[lane][0] = va;
            ws[lane][1] = vb;
            ws[lane][2] = vc;
        }
        if (lane == 31) {
            tot[0] = va;
            tot[1] = vb;
            tot[2] = vc;
        }
    }
    __syncthreads();
    const int pa = w > 0 ? ws[w - 1][0] : 0, pb = w > 0 ? ws[w - 1][1] : 0, pc = w > 0 ? ws[w - 1][2] : 0;
    a = pa + xa - a;
    b = pb + xb - b;
    c = pc + xc - c;
}

// one CTA of 1024 threads over the dense block table (ITEMS consecutive blocks per thread)
template <int D, bool LPT>
__global__ void __launch_bounds__(1024) k_inc_scan(int nb_total, const int* __restrict__ obstart,
                                                   const int* __restrict__ obend, IncSort S, int* __restrict__ bstart,
                                                   int* __restrict__ bend, int* __restrict__ occ, int* __restrict__ counts)
{
    constexpr int ITEMS = 8;
    __shared__ int ws[32][3];
    __shared__ int tot[3];
    __shared__ int carry[3];
    __shared__ int hist[OCC_NBUCKET], bcur[OCC_NBUCKET];
    if (threadIdx.x < 3)
        carry[threadIdx.x] = 0;
    if (threadIdx.x < OCC_NBUCKET) {
        hist[threadIdx.x] = 0;
        bcur[threadIdx.x] = 0;
    }
    __syncthreads();
    for (int base = 0; base < nb_total; base += 1024 * ITEMS) {
        const int b0 = base + threadIdx.x * ITEMS;
        int cnt[ITEMS], cin[ITEMS];
        int sa = 0, sb = 0, sc = 0;
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const int b = b0 + j;
            cnt[j] = cin[j] = 0;
            if (b < nb_total) {
                const int os = obstart[b];
                const int old = os >= 0 ? obend[b] - os : 0;
                cin[j] = S.cnt_in[b];
                cnt[j] = old - S.cnt_out[b] + cin[j];
                S.cnt_out[b] = 0; // becomes k_inc_place's bucket cursor
            }
            sa += cnt[j];
            sb += cin[j];
            sc += cnt[j] > 0;
        }
        cta_scan3(sa, sb, sc, ws, tot);
        sa += carry[0];
        sb += carry[1];
        sc += carry[2];
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const int b = b0 + j;
            if (b < nb_total) {
                bstart[b] = cnt[j] > 0 ? sa : -1;
                bend[b] = cnt[j] > 0 ? sa + cnt[j] : -1;
                S.in_off[b] = sb;
                if (cnt[j] > 0) {
                    if (LPT)
                        atomicAdd(&hist[occ_bucket(cnt[j])], 1);
                    else
                        occ[sc] = b;
                    ++sc;
                }
            }
            sa += cnt[j];
            sb += cin[j];
        }
        __syncthreads();
        if (threadIdx.x < 3)
            carry[threadIdx.x] += tot[threadIdx.x];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        counts[0] = carry[2];
    if (LPT) { // heaviest bucket first (the order k_occ_hist / k_occ_scatter give)
        if (threadIdx.x == 0) {
            int s = 0;
            for (int k = OCC_NBUCKET - 1; k >= 0; --k) {
                const int h = hist[k];
                hist[k] = s;
                s += h;
            }
        }
        __syncthreads();
        for (int b = threadIdx.x; b < nb_total; b += blockDim.x) {
            const int s = bstart[b];
            if (s >= 0) {
                const int k = occ_bucket(bend[b] - s);
                occ[hist[k] + atomicAdd(&bcur[k], 1)] = b;
            }
        }
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_inc_place(const int* __restrict__ keys, IncSort S, int grid_threads)
{
    using C = Cfg<D>;
    const int nx = *S.nx;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nx; j += grid_threads) {
        const int i = S.xlist[j];
        const int b = keys[i] >> C::LOGNB;
        S.inbuf[S.in_off[b] + atomicAdd(&S.cnt_out[b], 1)] = i;
    }
}

// CTA per occupied block (static stride over the list); see the file comment
template <int D>
__global__ void __launch_bounds__(INC_THREADS) k_inc_block(const int* __restrict__ keys, const int* __restrict__ obstart,
                                                           const int* __restrict__ obend, IncSort S,
                                                           const int* __restrict__ bstart, const int* __restrict__ bend,
                                                           const int* __restrict__ occ, const int* __restrict__ counts,
                                                           int* __restrict__ perm, int* __restrict__ keys_sorted,
                                                           int* __restrict__ lstart)
{
    using C = Cfg<D>;
    constexpr int NB = C::NB;
    constexpr int LVLBITS = (D - 1) * C::LOGB;
    __shared__ int wcnt[INC_WARPS][NB];
    __shared__ int cur[NB];
    __shared__ int sin_[INC_THREADS];
    __shared__ int s_nlo;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1;
    for (int k = tid; k < INC_WARPS * NB; k += INC_THREADS)
        (&wcnt[0][0])[k] = 0;
    if (blockIdx.x == 0 && tid == 0)
        *S.nx = 0; // k_inc_place has finished reading it
    const int n_occ = counts[0];
    for (int w = blockIdx.x; w < n_occ; w += gridDim.x) {
        const int b = occ[w];
        const int start = bstart[b], cnt = bend[b] - start;
        const int os = obstart[b], oe = os >= 0 ? obend[b] : os;
        const int kin = S.cnt_in[b], ioff = S.in_off[b];
        int* insorted = S.xlist + ioff; // the bucket sorted by storage index
        // ---- in-movers by storage index (ranks by comparison: buckets are small)
        __syncthreads(); // previous block's readers of sin_ / insorted are done
        if (kin <= INC_THREADS) {
            if (tid < kin)
                sin_[tid] = S.inbuf[ioff + tid];
            __syncthreads();
            if (tid < kin) {
                const int me = sin_[tid];
                int r = 0;
                for (int l = 0; l < kin; ++l)
                    r += sin_[l] < me;
                insorted[r] = me;
            }
        } else { // a block receiving more than a CTA's worth of movers in one step (rare)
            for (int j = tid; j < kin; j += INC_THREADS) {
                const int me = S.inbuf[ioff + j];
                int r = 0;
                for (int l = 0; l < kin; ++l)
                    r += S.inbuf[ioff + l] < me;
                insorted[r] = me;
            }
        }
        __syncthreads();
        if (tid == 0) {
            int lo = 0, hi = kin; // first in-mover at or above the old range
            if (os >= 0)
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (insorted[mid] < os)
                        lo = mid + 1;
                    else
                        hi = mid;
                }
            else
                lo = kin;
            s_nlo = lo;
            S.cnt_in[b] = 0;
            S.cnt_out[b] = 0;
        }
        for (int c = tid; c < NB; c += INC_THREADS)
            cur[c] = 0;
        __syncthreads();
        const int nlo = s_nlo, nrange = os >= 0 ? oe - os : 0, total = kin + nrange;
        // member v of the concatenation -> (storage index, local cell) or invalid (an out-mover)
        auto member = [&](int v, int& idx, int& loc) -> bool {
            if (v >= total)
                return false;
            if (v < nlo)
                idx = insorted[v];
            else if (v < nlo + nrange)
                idx = os + (v - nlo);
            else
                idx = insorted[v - nrange];
            const int k = keys[idx];
            loc = k & (NB - 1);
            return (k >> C::LOGNB) == b;
        };
        // ---- pass 1: cell histogram
        for (int v0 = 0; v0 < total; v0 += INC_THREADS) {
            int idx, loc;
            if (member(v0 + tid, idx, loc))
                atomicAdd(&cur[loc], 1);
        }
        __syncthreads();
        // exclusive scan of the NB cell counts (NB / INC_THREADS consecutive cells per thread)
        {
            constexpr int PER = NB / INC_THREADS;
            int v[PER], s = 0;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                v[j] = cur[tid * PER + j];
                s += v[j];
            }
            int incl = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o)
                    incl += y;
            }
            if (lane == 31)
                sin_[warp] = incl; // sin_ is free again (insorted lives in global memory)
            __syncthreads();
            int pre = 0;
            for (int k = 0; k < warp; ++k)
                pre += sin_[k];
            int e = pre + incl - s;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                cur[tid * PER + j] = e;
                e += v[j];
            }
        }
        __syncthreads();
        // level starts (a level is a contiguous run of the local-cell order); an empty level
        // gets the next level's start, which the readers' suffix minimum treats the same way
        for (int z = tid; z < C::B; z += INC_THREADS)
            lstart[b * (C::B + 1) + z] = start + cur[z << LVLBITS];
        __syncthreads();
        // ---- pass 2: stable placement, rank = cell start + earlier members of the same cell
        for (int v0 = 0; v0 < total; v0 += INC_THREADS) {
            int idx = 0, loc = 0;
            const bool ok = member(v0 + tid, idx, loc);
            const unsigned peers = __match_any_sync(0xffffffffu, ok ? loc : NB + lane);
            const bool leader = ok && (peers & lt) == 0;
            if (leader)
                wcnt[warp][loc] = __popc(peers);
            __syncthreads();
            if (ok) {
                int pre = cur[loc] + __popc(peers & lt);
                for (int k = 0; k < warp; ++k)
                    pre += wcnt[k][loc];
                perm[start + pre] = idx;
                keys_sorted[start + pre] = (b << C::LOGNB) | loc;
            }
            __syncthreads();
            if (leader) {
                atomicAdd(&cur[loc], __popc(peers));
                wcnt[warp][loc] = 0;
            }
        }
        (void)cnt;
    }
}

} // namespace mpmgpu
