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
//   k_inc_count     thread per block of the dense table: new count = old range - out + in;
//                   per-CTA sums, the occupancy-bucket histogram
//   k_inc_offsets   thread per block: exclusive scans (CTA prefix from the per-CTA sums) ->
//                   bstart / bend, in-mover offsets, the occupied-block list (heaviest first
//                   for the 3-D work-counter kernels)
//   k_inc_place     movers into their destination block's bucket (atomic slot, order fixed later)
//   k_inc_block     CTA per occupied block. U = old-range particles whose key did not change
//                   (already in order), C = changed members (cell changed inside the block, or
//                   arrived from another block), X = old-range positions not in U. C and X are
//                   small and sorted in shared memory; then every member's rank is a merge:
//                     u at old-range position r:  r - |X below r| + |C below (key_u, idx_u)|
//                     c at rank q inside C:       q + |U below (key_c, idx_c)|
//                   (the old range is sorted by (old key, index), so |U below| is a binary
//                   search minus |X below|). No barrier per element; a block whose C or X
//                   overflows shared memory falls back to a stable counting sort by local cell
//                   (histogram, scan, per-warp match ranks) in the same kernel.
//
// Bitwise the same perm and keys_sorted as the radix sort for every input (tests compare the
// states after many steps); there is no capacity limit, only a slower path when a block
// receives more than one CTA's worth of movers in one step. The first sort after an upload (or a
// migration import) has no previous order and uses the full radix sort.
#pragma once

#include "common.cuh"

namespace mpmgpu {

constexpr int INC_THREADS = 256; // k_inc_block CTA size
#ifndef INC_UNR
#define INC_UNR 4 // old-range keys in flight per thread in k_inc_block (MEASURED C4: 8 is slower, 21.0 vs 18.9 us)
#endif
constexpr int INC_WARPS = INC_THREADS / 32;

// scratch of the incremental sort, owned by the context (self-cleaning: every counter the
// kernels raise is returned to zero by a later kernel of the same sort)
struct IncSort {
    int* cnt_in;  // [nb_total] movers arriving per block (zeroed by k_inc_block)
    int* cnt_out; // [nb_total] movers leaving per block; reused as the bucket cursor (zeroed by k_inc_count / k_inc_block)
    int* in_off;  // [nb_total] bucket offset of a block's in-movers
    int* xlist;   // [cap] mover storage indices; then the buckets sorted by index
    int* inbuf;   // [cap] mover buckets (unordered within a bucket)
    int* nx;      // [1] mover count (zeroed by k_inc_block)
    int* part;    // [3 * ceil(nb_total / 256)] per-CTA sums of k_inc_count
    int* hist;    // [OCC_NBUCKET] occupancy buckets (zeroed by k_inc_block)
    int* bcur;    // [OCC_NBUCKET] bucket cursors (zeroed by k_inc_block)
    int* nlive;   // [1] particles the sort placed (= the count G2P writes)
    const int* d_n; // device particle count (decomposed steps) or nullptr (the host's n)
    // the step's active-node bookkeeping, folded into the sort's kernels (fewer graph nodes per
    // step: the 2-D scenes are launch-latency bound)
    unsigned char* nflag; // [nnb_total] node blocks touched (zeroed by k_inc_classify, set by k_inc_offsets)
    int nnb_total;
    const int* nb;        // [D] particle blocks per axis (device)
    const int* nnb;       // [D] node blocks per axis (device)
    int* act;             // active node-block list (k_inc_place)
    int* counts;          // [4] counts[0] occupied blocks, counts[1] active node blocks
};

// 4 particles per thread (two 16-byte loads per thread keep enough bytes in flight)
template <int D>
__global__ void __launch_bounds__(256) k_inc_classify(const int* __restrict__ keys, const int* __restrict__ okeys, int n,
                                                      int nb_total, IncSort S)
{
    pdl_wait();
    pdl_trigger();
    using C = Cfg<D>;
    if (S.d_n)
        n = *S.d_n;
    { // zero this step's node-block flags (16 bytes per thread) and the list counters
        const int t = blockIdx.x * blockDim.x + threadIdx.x;
        const int nq = (S.nnb_total + 15) / 16;
        for (int q = t; q < nq; q += gridDim.x * blockDim.x) {
            if (16 * q + 16 <= S.nnb_total)
                reinterpret_cast<uint4*>(S.nflag)[q] = make_uint4(0, 0, 0, 0);
            else
                for (int c = 16 * q; c < S.nnb_total; ++c)
                    S.nflag[c] = 0;
        }
        if (t == 0)
            S.counts[1] = 0;
    }
    const int i0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    int k[4], o[4];
    if (i0 + 3 < n) {
        const int4 a = *reinterpret_cast<const int4*>(keys + i0), b = *reinterpret_cast<const int4*>(okeys + i0);
        k[0] = a.x, k[1] = a.y, k[2] = a.z, k[3] = a.w;
        o[0] = b.x, o[1] = b.y, o[2] = b.z, o[3] = b.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            k[j] = i0 + j < n ? keys[i0 + j] : 0;
            o[j] = i0 + j < n ? okeys[i0 + j] : 0;
        }
    }
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int b = k[j] >> C::LOGNB, ob = o[j] >> C::LOGNB;
        const bool mover = i0 + j < n && b != ob;
        // out-of-domain / dead keys join no block (the step aborts / the slot was vacated); an
        // imported particle has no previous block (old key -1)
        const bool valid = mover && unsigned(b) < unsigned(nb_total);
        if (valid)
            atomicAdd(&S.cnt_in[b], 1);
        if (mover && unsigned(ob) < unsigned(nb_total))
            atomicAdd(&S.cnt_out[ob], 1);
        const unsigned m = __ballot_sync(0xffffffffu, valid);
        if (m) {
            int base = 0;
            if (lane == 0)
                base = atomicAdd(S.nx, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (valid)
                S.xlist[base + __popc(m & ((1u << lane) - 1))] = i0 + j;
        }
    }
}

// per-block counts of the new order: cnt = |old range| - out + in (parked in the new bend table,
// which k_inc_offsets overwrites), per-CTA sums and the occupancy-bucket histogram
template <int D>
__global__ void __launch_bounds__(256) k_inc_count(int nb_total, const int* __restrict__ obstart,
                                                   const int* __restrict__ obend, IncSort S, int* __restrict__ bend)
{
    pdl_wait();
    pdl_trigger();
    __shared__ int ws[8][3];
    const int b = blockIdx.x * 256 + threadIdx.x;
    int cnt = 0, cin = 0;
    if (b < nb_total) {
        const int os = obstart[b];
        const int old = os >= 0 ? obend[b] - os : 0;
        cin = S.cnt_in[b];
        cnt = old - S.cnt_out[b] + cin;
        S.cnt_out[b] = 0; // becomes k_inc_place's bucket cursor
        bend[b] = cnt;    // scratch: the count (k_inc_offsets writes the real bend)
        if (cnt > 0)
            atomicAdd(&S.hist[occ_bucket(cnt)], 1);
    }
    int a = cnt, c = cin, o = cnt > 0;
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, k);
        c += __shfl_down_sync(0xffffffffu, c, k);
        o += __shfl_down_sync(0xffffffffu, o, k);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        ws[w][0] = a;
        ws[w][1] = c;
        ws[w][2] = o;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        int t = 0;
        for (int k = 0; k < 8; ++k)
            t += ws[k][threadIdx.x];
        S.part[blockIdx.x * 3 + threadIdx.x] = t;
    }
}

// exclusive scans of (count, in-movers, occupied) -> bstart / bend / in_off / occupied list
template <int D, bool LPT>
__global__ void __launch_bounds__(256) k_inc_offsets(int nb_total, IncSort S, int* __restrict__ bstart,
                                                     int* __restrict__ bend, int* __restrict__ occ,
                                                     int* __restrict__ counts)
{
    pdl_wait();
    pdl_trigger();
    __shared__ int ws[8][3];
    __shared__ int pre[3];
    __shared__ int boff[OCC_NBUCKET];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nblk = gridDim.x;
    if (w == 0) { // this CTA's prefix: the sums of the CTAs before it
        int a = 0, c = 0, o = 0;
        for (int k = lane; k < int(blockIdx.x); k += 32) {
            a += S.part[k * 3];
            c += S.part[k * 3 + 1];
            o += S.part[k * 3 + 2];
        }
#pragma unroll
        for (int k = 16; k > 0; k >>= 1) {
            a += __shfl_down_sync(0xffffffffu, a, k);
            c += __shfl_down_sync(0xffffffffu, c, k);
            o += __shfl_down_sync(0xffffffffu, o, k);
        }
        if (lane == 0) {
            pre[0] = a;
            pre[1] = c;
            pre[2] = o;
            if (blockIdx.x == nblk - 1) {
                counts[0] = o + S.part[blockIdx.x * 3 + 2];
                *S.nlive = a + S.part[blockIdx.x * 3];
            }
        }
    } else if (LPT && w == 1) { // bucket offsets, heaviest bucket first
        int h0 = S.hist[2 * lane], h1 = S.hist[2 * lane + 1];
        // descending order: offset of bucket k = sum of buckets > k
        int tot = h0 + h1, incl = tot;
#pragma unroll
        for (int k = 1; k < 32; k <<= 1) { // suffix sum over lanes
            const int y = __shfl_down_sync(0xffffffffu, incl, k);
            if (lane + k < 32)
                incl += y;
        }
        const int above = incl - tot; // buckets of higher lanes
        boff[2 * lane + 1] = above;
        boff[2 * lane] = above + h1;
    }
    const int b = blockIdx.x * 256 + threadIdx.x;
    int cnt = 0, cin = 0;
    if (b < nb_total) {
        cnt = bend[b];
        cin = S.cnt_in[b];
    }
    int a = cnt, c = cin, o = cnt > 0;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
        const int ya = __shfl_up_sync(0xffffffffu, a, k), yc = __shfl_up_sync(0xffffffffu, c, k),
                  yo = __shfl_up_sync(0xffffffffu, o, k);
        if (lane >= k) {
            a += ya;
            c += yc;
            o += yo;
        }
    }
    if (lane == 31) {
        ws[w][0] = a;
        ws[w][1] = c;
        ws[w][2] = o;
    }
    __syncthreads();
    int pa = pre[0], pc = pre[1], po = pre[2];
    for (int k = 0; k < w; ++k) {
        pa += ws[k][0];
        pc += ws[k][1];
        po += ws[k][2];
    }
    if (b < nb_total) {
        const int start = pa + a - cnt;
        bstart[b] = cnt > 0 ? start : -1;
        bend[b] = cnt > 0 ? start + cnt : -1;
        S.in_off[b] = pc + c - cin;
        if (cnt > 0) {
            if (LPT) {
                const int k = occ_bucket(cnt);
                occ[boff[k] + atomicAdd(&S.bcur[k], 1)] = b;
            } else {
                occ[po + o - 1] = b;
            }
            // node blocks touched by block b: b + s, s in {0,1}^D (k_mark_nodes)
            int q[D], rem = b;
#pragma unroll
            for (int a = D - 1; a >= 0; --a) {
                q[a] = rem % S.nb[a];
                rem /= S.nb[a];
            }
#pragma unroll
            for (int sft = 0; sft < (1 << D); ++sft) {
                int id = 0;
                bool ok = true;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    const int c2 = q[a] + ((sft >> (D - 1 - a)) & 1);
                    ok &= c2 < S.nnb[a];
                    id = id * S.nnb[a] + c2;
                }
                if (ok)
                    S.nflag[id] = 1;
            }
        }
    }
}

// movers into their buckets, and the active node-block list (k_compact_flag's compaction)
template <int D>
__global__ void __launch_bounds__(256) k_inc_place(const int* __restrict__ keys, IncSort S, int grid_threads)
{
    pdl_wait();
    pdl_trigger();
    using C = Cfg<D>;
    const int nx = *S.nx;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nx; j += grid_threads) {
        const int i = S.xlist[j];
        const int b = keys[i] >> C::LOGNB;
        S.inbuf[S.in_off[b] + atomicAdd(&S.cnt_out[b], 1)] = i;
    }
    const int lane = threadIdx.x & 31;
    for (int q0 = blockIdx.x * blockDim.x; q0 < S.nnb_total; q0 += grid_threads) {
        const int q = q0 + threadIdx.x;
        const bool p = q < S.nnb_total && S.nflag[q] != 0;
        const unsigned m = __ballot_sync(0xffffffffu, p);
        int base = 0;
        if (lane == 0 && m)
            base = atomicAdd(S.counts + 1, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (p)
            S.act[base + __popc(m & ((1u << lane) - 1))] = q;
    }
}

constexpr int INC_XCAP = 512, INC_CCAP = 512; // merge path: changed members / excluded positions per block

// shared memory of k_inc_block: the merge path's sorted lists, or the fallback's counters
template <int D> union IncSmem {
    struct {
        int xu[INC_XCAP], xs[INC_XCAP];            // excluded old-range positions: unsorted, sorted
        int cu_i[INC_CCAP], cu_k[INC_CCAP];        // changed members (storage index, key): unsorted
        int cs_i[INC_CCAP], cs_k[INC_CCAP];        // ... sorted by (key, index)
    } m;
    struct {
        int wcnt[INC_WARPS][Cfg<D>::NB];
        int cur[Cfg<D>::NB];
        int sin_[INC_THREADS];
    } f;
};

// CTA per occupied block (static stride over the list); see the file comment
template <int D>
__global__ void __launch_bounds__(INC_THREADS) k_inc_block(const int* __restrict__ keys, const int* __restrict__ okeys,
                                                           const int* __restrict__ obstart,
                                                           const int* __restrict__ obend, IncSort S,
                                                           const int* __restrict__ bstart, const int* __restrict__ bend,
                                                           const int* __restrict__ occ, const int* __restrict__ counts,
                                                           int* __restrict__ perm, int* __restrict__ keys_sorted,
                                                           int* __restrict__ lstart)
{
    pdl_wait();
    pdl_trigger();
    using C = Cfg<D>;
    constexpr int NB = C::NB;
    constexpr int LVLBITS = (D - 1) * C::LOGB;
    __shared__ IncSmem<D> sm;
    __shared__ int s_nx, s_nc, s_nlo;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1;
    if (blockIdx.x == 0 && tid == 0)
        *S.nx = 0; // k_inc_place has finished reading it
    if (blockIdx.x == 0 && tid < OCC_NBUCKET) {
        S.hist[tid] = 0;
        S.bcur[tid] = 0;
    }
    const int n_occ = counts[0];
    for (int w = blockIdx.x; w < n_occ; w += gridDim.x) {
        const int b = occ[w];
        const int start = bstart[b], cnt = bend[b] - start;
        const int os = obstart[b];
        const int nrange = os >= 0 ? obend[b] - os : 0;
        const int kin = S.cnt_in[b], ioff = S.in_off[b];
        __syncthreads(); // the previous block's readers of the shared lists are done
        if (tid == 0) {
            s_nx = 0;
            s_nc = 0;
        }
        __syncthreads();
        // ---- collect C (in-movers, cell changes inside the block) and X (old positions not in U)
        for (int j = tid; j < kin; j += INC_THREADS) {
            const int idx = S.inbuf[ioff + j];
            const int q = atomicAdd(&s_nc, 1);
            if (q < INC_CCAP) {
                sm.m.cu_i[q] = idx;
                sm.m.cu_k[q] = keys[idx];
            }
        }
        for (int r0 = 0; r0 < nrange; r0 += INC_UNR * INC_THREADS) {
            int kk[INC_UNR], oo[INC_UNR];
#pragma unroll
            for (int j = 0; j < INC_UNR; ++j) { // independent loads in flight per thread
                const int r = r0 + j * INC_THREADS + tid;
                kk[j] = r < nrange ? keys[os + r] : 0;
                oo[j] = r < nrange ? okeys[os + r] : 0;
            }
#pragma unroll
            for (int j = 0; j < INC_UNR; ++j) {
                const int r = r0 + j * INC_THREADS + tid;
                const int k = kk[j];
                const bool ex = r < nrange && k != oo[j];
                const bool ch = ex && (k >> C::LOGNB) == b;
                const unsigned mx = __ballot_sync(0xffffffffu, ex), mc = __ballot_sync(0xffffffffu, ch);
                if ((mx | mc) == 0)
                    continue;
                int bx = 0, bc = 0;
                if (lane == 0) {
                    if (mx)
                        bx = atomicAdd(&s_nx, __popc(mx));
                    if (mc)
                        bc = atomicAdd(&s_nc, __popc(mc));
                }
                bx = __shfl_sync(0xffffffffu, bx, 0);
                bc = __shfl_sync(0xffffffffu, bc, 0);
                if (ex) {
                    const int q = bx + __popc(mx & lt);
                    if (q < INC_XCAP)
                        sm.m.xu[q] = r;
                }
                if (ch) {
                    const int q = bc + __popc(mc & lt);
                    if (q < INC_CCAP) {
                        sm.m.cu_i[q] = os + r;
                        sm.m.cu_k[q] = k;
                    }
                }
            }
        }
        __syncthreads();
        const int nx = s_nx, nc = s_nc;
        if (nx <= INC_XCAP && nc <= INC_CCAP) {
            // ---- merge path: sort X and C in shared memory (ranks by comparison; both small)
            for (int j = tid; j < nx; j += INC_THREADS) {
                const int v = sm.m.xu[j];
                int rk = 0;
                for (int l = 0; l < nx; ++l)
                    rk += sm.m.xu[l] < v;
                sm.m.xs[rk] = v;
            }
            for (int j = tid; j < nc; j += INC_THREADS) {
                const int ki = sm.m.cu_k[j], ii = sm.m.cu_i[j];
                int rk = 0;
                for (int l = 0; l < nc; ++l) {
                    const int kl = sm.m.cu_k[l];
                    rk += kl < ki || (kl == ki && sm.m.cu_i[l] < ii);
                }
                sm.m.cs_k[rk] = ki;
                sm.m.cs_i[rk] = ii;
            }
            __syncthreads();
            auto x_below = [&](int r) { // |X < r|
                int lo = 0, hi = nx;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (sm.m.xs[mid] < r)
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                return lo;
            };
            // U: rank = r - |X below r| + |C below (key, index)|
            for (int r0 = 0; r0 < nrange; r0 += 4 * INC_THREADS) {
              int kk[4], oo[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                  const int r = r0 + j * INC_THREADS + tid;
                  kk[j] = r < nrange ? keys[os + r] : 0;
                  oo[j] = r < nrange ? okeys[os + r] : 1;
              }
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int r = r0 + j * INC_THREADS + tid;
                const int k = kk[j];
                if (r >= nrange || k != oo[j])
                    continue;
                const int idx = os + r;
                if (nx == 0 && nc == 0) { // block without changes: the old order as is
                    perm[start + r] = idx;
                    keys_sorted[start + r] = k;
                    continue;
                }
                int lo = 0, hi = nc;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    const int km = sm.m.cs_k[mid];
                    if (km < k || (km == k && sm.m.cs_i[mid] < idx))
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                const int pos = r - x_below(r) + lo;
                perm[start + pos] = idx;
                keys_sorted[start + pos] = k;
              }
            }
            // C: rank = q + |U below (key, index)|; the old range is strictly increasing in
            // (old key, index), so |range below| is a binary search and |U below| = that - |X below|
            for (int q = tid; q < nc; q += INC_THREADS) {
                const int k = sm.m.cs_k[q], idx = sm.m.cs_i[q];
                int lo = 0, hi = nrange;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    const int km = okeys[os + mid];
                    if (km < k || (km == k && os + mid < idx))
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                const int pos = q + lo - x_below(lo);
                perm[start + pos] = idx;
                keys_sorted[start + pos] = k;
            }
            __syncthreads(); // this block's keys_sorted complete (block-scope visibility)
            // level starts: first position of each level; an empty level gets the next level's
            // start, which the readers' suffix minimum treats the same way
            for (int z = tid; z < C::B; z += INC_THREADS) {
                const int key0 = (b << C::LOGNB) | (z << LVLBITS);
                int lo = 0, hi = cnt;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (keys_sorted[start + mid] < key0)
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                lstart[b * (C::B + 1) + z] = start + lo;
            }
        } else {
            // ---- fallback: stable counting sort by local cell over the members in storage order
            // [in-movers below the old range][U and in-block changes of the range][in-movers above]
            int* insorted = S.xlist + ioff; // the bucket sorted by storage index
            if (kin <= INC_THREADS) {
                if (tid < kin)
                    sm.f.sin_[tid] = S.inbuf[ioff + tid];
                __syncthreads();
                if (tid < kin) {
                    const int me = sm.f.sin_[tid];
                    int r = 0;
                    for (int l = 0; l < kin; ++l)
                        r += sm.f.sin_[l] < me;
                    insorted[r] = me;
                }
            } else {
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
            }
            for (int k = tid; k < INC_WARPS * NB; k += INC_THREADS)
                (&sm.f.wcnt[0][0])[k] = 0;
            for (int c = tid; c < NB; c += INC_THREADS)
                sm.f.cur[c] = 0;
            __syncthreads();
            const int nlo = s_nlo, total = kin + nrange;
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
            for (int v0 = 0; v0 < total; v0 += INC_THREADS) { // cell histogram
                int idx, loc;
                if (member(v0 + tid, idx, loc))
                    atomicAdd(&sm.f.cur[loc], 1);
            }
            __syncthreads();
            {
                constexpr int PER = NB / INC_THREADS;
                int v[PER], sum = 0;
#pragma unroll
                for (int j = 0; j < PER; ++j) {
                    v[j] = sm.f.cur[tid * PER + j];
                    sum += v[j];
                }
                int incl = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o)
                        incl += y;
                }
                __syncthreads();
                if (lane == 31)
                    sm.f.sin_[warp] = incl;
                __syncthreads();
                int pre = 0;
                for (int k = 0; k < warp; ++k)
                    pre += sm.f.sin_[k];
                int e = pre + incl - sum;
#pragma unroll
                for (int j = 0; j < PER; ++j) {
                    sm.f.cur[tid * PER + j] = e;
                    e += v[j];
                }
            }
            __syncthreads();
            for (int z = tid; z < C::B; z += INC_THREADS)
                lstart[b * (C::B + 1) + z] = start + sm.f.cur[z << LVLBITS];
            __syncthreads();
            for (int v0 = 0; v0 < total; v0 += INC_THREADS) { // stable placement by match ranks
                int idx = 0, loc = 0;
                const bool ok = member(v0 + tid, idx, loc);
                const unsigned peers = __match_any_sync(0xffffffffu, ok ? loc : NB + lane);
                const bool leader = ok && (peers & lt) == 0;
                if (leader)
                    sm.f.wcnt[warp][loc] = __popc(peers);
                __syncthreads();
                if (ok) {
                    int pre = sm.f.cur[loc] + __popc(peers & lt);
                    for (int k = 0; k < warp; ++k)
                        pre += sm.f.wcnt[k][loc];
                    perm[start + pre] = idx;
                    keys_sorted[start + pre] = (b << C::LOGNB) | loc;
                }
                __syncthreads();
                if (leader) {
                    atomicAdd(&sm.f.cur[loc], __popc(peers));
                    sm.f.wcnt[warp][loc] = 0;
                }
                __syncwarp();
            }
        }
        if (tid == 0) {
            S.cnt_in[b] = 0;
            S.cnt_out[b] = 0;
        }
        (void)cnt;
    }
}

} // namespace mpmgpu
