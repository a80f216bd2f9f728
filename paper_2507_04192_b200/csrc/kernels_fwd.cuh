// kernels_fwd.cuh -- forward step Phi = G2P o U o P2G on B200 (sm_100a).
//
// Per step:
//   sort      stable radix sort of 32-bit cell keys (block << LOGNB | local cell) -> perm
//   k_seg     dense per-block segment [bstart, bend) of the sorted order
//   k_p2g     CTA per occupied particle block: node-column march (deterministic gather,
//             no atomics) of the block's particles into its (B+2)^d partial tile
//   k_grid    CTA per active node block: sum <= 2^d partial tiles in fixed order, momentum
//             update, wall / obstacle / Coulomb corrections (transfer.hpp:75-84,
//             contact.hpp:228-245)
//   k_g2p     CTA per occupied particle block: node tile in smem, gather + v/x/grad v update
//             (transfer.hpp:92-121) fused with the constitutive update (stepper.hpp:15-43),
//             writes the new state in sorted order and the next step's cell keys
#pragma once

#include <cstdio>

#include "common.cuh"
#include "constit.cuh"

namespace mpmgpu {

// ---------------------------------------------------------------------------------------
// keys / segments
template <class T, int D>
__global__ void k_keys(DevScene<T, D> sc, PBuf<T, D> P, int n, int* keys, DevStatus* st)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    if (P.pid[i] < 0) { // vacated slot (migrated away)
        keys[i] = KEY_DEAD;
        return;
    }
    T x[D];
#pragma unroll
    for (int a = 0; a < D; ++a)
        x[a] = P.x[a][i];
    int key;
    if (!cell_key<T, D>(sc, x, key)) {
        key = KEY_OOD;
        atomicMin(&st->ood_pid, P.pid[i]);
        st->ood_flag = 1;
        st->abort = 1;
    }
    keys[i] = key;
}

__global__ void k_iota(int* a, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n)
        a[i] = i;
}

// dense segment table: bstart[b] / bend[b] for every particle block present in sorted keys,
// plus the first sorted index of every non-empty base level (lstart[b][z], others untouched;
// the reader fills gaps with a suffix minimum)
template <int D>
__global__ void k_seg(const int* keys, int n, int nb_total, int* bstart, int* bend, int* lstart)
{
    using C = Cfg<D>;
    constexpr int LVLBITS = (D - 1) * C::LOGB;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const int k = keys[i];
    int b = k >> C::LOGNB;
    if (b >= nb_total)
        return;
    const int kp = i > 0 ? keys[i - 1] : -1;
    int bp = i > 0 ? (kp >> C::LOGNB) : -1;
    int bn = i + 1 < n ? (keys[i + 1] >> C::LOGNB) : -1;
    if (b != bp)
        bstart[b] = i;
    if (b != bn)
        bend[b] = i + 1;
    const int z = (k & (C::NB - 1)) >> LVLBITS;
    if (b != bp || z != ((kp & (C::NB - 1)) >> LVLBITS))
        lstart[b * (C::B + 1) + z] = i;
}

// k_seg over 4 sorted keys per thread (one 16-byte load; the neighbours across threads come by
// shuffle): the same tables, 4x fewer threads and loads
template <int D>
__global__ void k_seg4(const int* __restrict__ keys, int n, int nb_total, int* __restrict__ bstart,
                       int* __restrict__ bend, int* __restrict__ lstart)
{
    using C = Cfg<D>;
    constexpr int LVLBITS = (D - 1) * C::LOGB;
    const int i0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    int k[6]; // keys i0 - 1 .. i0 + 4; -1 where out of range
    if (i0 + 3 < n) {
        const int4 v = *reinterpret_cast<const int4*>(keys + i0);
        k[1] = v.x;
        k[2] = v.y;
        k[3] = v.z;
        k[4] = v.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            k[1 + j] = i0 + j < n ? keys[i0 + j] : -1;
    }
    const int lane = threadIdx.x & 31;
    k[0] = __shfl_up_sync(0xffffffffu, k[4], 1);
    k[5] = __shfl_down_sync(0xffffffffu, k[1], 1);
    if (lane == 0)
        k[0] = (i0 > 0 && i0 - 1 < n) ? keys[i0 - 1] : -1;
    if (lane == 31)
        k[5] = i0 + 4 < n ? keys[i0 + 4] : -1;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int i = i0 + j;
        const int kk = k[j + 1];
        const int b = kk >> C::LOGNB;
        if (i >= n || b >= nb_total)
            continue;
        const int kp = k[j];
        const int bp = kp >> C::LOGNB; // -1 for i == 0
        const int bn = k[j + 2] >> C::LOGNB;
        if (b != bp)
            bstart[b] = i;
        if (b != bn)
            bend[b] = i + 1;
        const int z = (kk & (C::NB - 1)) >> LVLBITS;
        if (b != bp || z != ((kp & (C::NB - 1)) >> LVLBITS))
            lstart[b * (C::B + 1) + z] = i;
    }
}

// node blocks touched by occupied particle block Q: Q + s, s in {0,1}^D
template <int D>
__global__ void k_mark_nodes(const int* occ, const int* n_occ, const int* nb, const int* nnb, unsigned char* nflag)
{
    int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= *n_occ)
        return;
    int q[D];
    block_coords<D>(occ[w], nb, q);
#pragma unroll
    for (int s = 0; s < (1 << D); ++s) {
        int id = 0;
        bool ok = true;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            int c = q[a] + ((s >> (D - 1 - a)) & 1);
            ok &= c < nnb[a];
            id = id * nnb[a] + c;
        }
        if (ok)
            nflag[id] = 1;
    }
}

// ---------------------------------------------------------------------------------------
// P2G: node-column march.
//
// Thread (column, segment) owns the node column `col` of the block tile (all axes but the
// last) and a range of base levels along the last axis. Walking base levels upward it
// gathers, from the 3^(d-1) base cells around its column, every particle's contributions to
// the three nodes above it, in a rolling 3-node register window. A node is final (for this
// segment) once the march passes it and is written once -- no atomics, no smem tile, fixed
// summation order (level, then base cell in canonical offset order, then sorted particle
// order). The two nodes a segment shares with the next one are added after a barrier.
template <class T, int D> struct P2GContrib {
    T acc[3][Cfg<D>::NF];
};

template <class T, int D>
__device__ __forceinline__ void axis_weights(T x, T origin, T inv_dh, T* w, T* dw)
{
    T u = (x - origin) * inv_dh;
    T fl = dfloor<T>(u - T(0.5));
    T fx = u - fl;
    T h0 = T(1.5) - fx, h1 = fx - T(1), h2 = fx - T(0.5);
    w[0] = T(0.5) * h0 * h0;
    w[1] = T(0.75) - h1 * h1;
    w[2] = T(0.5) * h2 * h2;
    dw[0] = -h0 * inv_dh;
    dw[1] = -T(2) * h1 * inv_dh;
    dw[2] = h2 * inv_dh;
}

// APIC / TPIC velocity augmentation matrix A (transfer.hpp:14-32), row-major D x D
template <class T, int D>
__device__ __forceinline__ void affine_matrix(const DevScene<T, D>& sc, const PBuf<T, D>& P, int src, const T* x,
                                              const T (&w)[D][3], const int* base, T* A)
{
    if (sc.tpic) {
#pragma unroll
        for (int k = 0; k < D * D; ++k)
            A[k] = __ldg(P.gv[k] + src);
        return;
    }
    // D = sum_o phi r r^T, canonical order, then A = B D^-1
    T Dm[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j)
            Dm[i][j] = T(0);
    for (int k = 0; k < Cfg<D>::NOFF; ++k) {
        int o[D];
        int kk = k;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
            o[a] = kk % 3;
            kk /= 3;
        }
        T phi = T(1), r[D];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            phi *= w[a][o[a]];
            r[a] = (sc.origin[a] + T(base[a] + o[a]) * sc.dh) - x[a];
        }
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j)
                Dm[i][j] += phi * r[i] * r[j];
    }
    T inv[D][D];
    if constexpr (D == 2) {
        T det = Dm[0][0] * Dm[1][1] - Dm[0][1] * Dm[1][0];
        T id = T(1) / det;
        inv[0][0] = Dm[1][1] * id;
        inv[0][1] = -Dm[0][1] * id;
        inv[1][0] = -Dm[1][0] * id;
        inv[1][1] = Dm[0][0] * id;
    } else {
        T c00 = Dm[1][1] * Dm[2][2] - Dm[1][2] * Dm[2][1];
        T c01 = Dm[1][2] * Dm[2][0] - Dm[1][0] * Dm[2][2];
        T c02 = Dm[1][0] * Dm[2][1] - Dm[1][1] * Dm[2][0];
        T det = Dm[0][0] * c00 + Dm[0][1] * c01 + Dm[0][2] * c02;
        T id = T(1) / det;
        inv[0][0] = c00 * id;
        inv[1][0] = c01 * id;
        inv[2][0] = c02 * id;
        inv[0][1] = (Dm[0][2] * Dm[2][1] - Dm[0][1] * Dm[2][2]) * id;
        inv[1][1] = (Dm[0][0] * Dm[2][2] - Dm[0][2] * Dm[2][0]) * id;
        inv[2][1] = (Dm[0][1] * Dm[2][0] - Dm[0][0] * Dm[2][1]) * id;
        inv[0][2] = (Dm[0][1] * Dm[1][2] - Dm[0][2] * Dm[1][1]) * id;
        inv[1][2] = (Dm[0][2] * Dm[1][0] - Dm[0][0] * Dm[1][2]) * id;
        inv[2][2] = (Dm[0][0] * Dm[1][1] - Dm[0][1] * Dm[1][0]) * id;
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            T s = T(0);
#pragma unroll
            for (int k = 0; k < D; ++k)
                s += __ldg(P.aff[i * D + k] + src) * inv[k][j];
            A[i * D + j] = s;
        }
}

// STAGED (2-D PIC / FLIP / blend): a block of up to P2G2_CAP particles is first gathered through
// the permutation into shared memory by all threads at once (independent loads, several in
// flight per thread), so the column march below reads shared memory instead of issuing a
// dependent global load chain per visited particle (the 2-D steps are latency-bound: C2 / C3
// have 100-1000 occupied blocks, under one wave). Larger blocks read global memory as before.
// The arithmetic is the same expression in the same order: results are bit-identical.
constexpr int P2G2_CAP = 1280;
template <class T> constexpr size_t p2g2_smem() { return sizeof(T) * 9 * P2G2_CAP + sizeof(int) * P2G2_CAP; }

template <class T, int D, bool AFF, bool STAGED = false>
__global__ void __launch_bounds__(256) k_p2g(DevScene<T, D> sc, PBuf<T, D> P, const int* __restrict__ perm,
                                             const int* __restrict__ keys, const int* __restrict__ bstart,
                                             const int* __restrict__ bend, const int* __restrict__ occ,
                                             const int* __restrict__ n_occ, T* __restrict__ partials,
                                             const DevStatus* st)
{
    pdl_wait();
    pdl_trigger();
    using C = Cfg<D>;
    constexpr int B = C::B, TE = C::TE, NF = C::NF;
    static_assert(!STAGED || (D == 2 && !AFF), "staged P2G: 2-D without affine transfer");
    __shared__ int cst[C::NB + 1];
    extern __shared__ unsigned char p2g2_raw[];
    T* rec = reinterpret_cast<T*>(p2g2_raw);                                   // [9][CAP]: x v m V sigma
    int* lc = reinterpret_cast<int*>(p2g2_raw + sizeof(T) * 9 * P2G2_CAP);    // [CAP] local cell
    if (st->abort)
        return;
    const int nocc = *n_occ;
    const int tid = threadIdx.x;
    const int col = tid % C::NCOL, seg = tid / C::NCOL;
    // column coordinates (all axes but the last)
    int cn[D - 1 > 0 ? D - 1 : 1];
    {
        int cc = col;
#pragma unroll
        for (int a = D - 2; a >= 0; --a) {
            cn[a] = cc % TE;
            cc /= TE;
        }
    }
    const int zb = seg * B / C::SEGS, ze = (seg + 1) * B / C::SEGS;
    const bool active = seg < C::SEGS;

    for (int w = blockIdx.x; w < nocc; w += gridDim.x) {
        const int Q = occ[w];
        const int s0 = bstart[Q], s1 = bend[Q], len = s1 - s0;
        int qc[D];
        block_coords<D>(Q, sc.nb, qc);
        const bool staged = STAGED && len <= P2G2_CAP;
        if (staged) { // gather the block through the permutation: 4 particles in flight per thread
            for (int r0 = 0; r0 < len; r0 += 4 * int(blockDim.x)) {
                int src[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int r = r0 + j * int(blockDim.x) + tid;
                    src[j] = r < len ? __ldg(perm + s0 + r) : 0;
                    if (r < len)
                        lc[r] = __ldg(keys + s0 + r) & (C::NB - 1);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int r = r0 + j * int(blockDim.x) + tid;
                    if (r >= len)
                        continue;
                    const int q = src[j];
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        rec[a * P2G2_CAP + r] = __ldg(P.x[a] + q);
                        rec[(D + a) * P2G2_CAP + r] = __ldg(P.v[a] + q);
                    }
                    rec[2 * D * P2G2_CAP + r] = __ldg(P.m + q);
                    rec[(2 * D + 1) * P2G2_CAP + r] = __ldg(P.V + q);
#pragma unroll
                    for (int q2 = 0; q2 < C::NS; ++q2)
                        rec[(2 * D + 2 + q2) * P2G2_CAP + r] = __ldg(P.sig[q2] + q);
                }
            }
            __syncthreads();
        }
        // cell ranges: cst[c] = first index (segment-relative) with local cell >= c
        for (int c = tid; c <= C::NB; c += blockDim.x) {
            int lo = 0, hi = len;
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if ((staged ? lc[mid] : (keys[s0 + mid] & (C::NB - 1))) < c)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            cst[c] = lo;
        }
        __syncthreads();
        T* part = partials + (size_t)Q * NF * C::TN;
        T ov[2][NF];
        if (active) {
            T acc[3][NF];
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int f = 0; f < NF; ++f)
                    acc[k][f] = T(0);
            for (int z = zb; z < ze; ++z) {
#pragma unroll
                for (int oo = 0; oo < C::NOFF / 3; ++oo) { // offsets on the non-march axes
                    int o[D - 1 > 0 ? D - 1 : 1];
                    int bcell = 0;
                    bool ok = true;
                    {
                        int kk = oo;
#pragma unroll
                        for (int a = D - 2; a >= 0; --a) {
                            o[a] = kk % 3;
                            kk /= 3;
                        }
#pragma unroll
                        for (int a = 0; a < D - 1; ++a) {
                            int bc = cn[a] - o[a];
                            ok &= bc >= 0 && bc < B;
                            bcell = (bcell << C::LOGB) | (bc & (B - 1));
                        }
                    }
                    if (!ok)
                        continue;
                    bcell |= z << ((D - 1) * C::LOGB); // level-major local cell (common.cuh)
                    const int kb = cst[bcell], ke = cst[bcell + 1];
                    for (int k = kb; k < ke; ++k) {
                        int src = 0;
                        T x[D], v[D], m, V, sig[C::NS];
                        if (staged) {
#pragma unroll
                            for (int a = 0; a < D; ++a) {
                                x[a] = rec[a * P2G2_CAP + k];
                                v[a] = rec[(D + a) * P2G2_CAP + k];
                            }
                            m = rec[2 * D * P2G2_CAP + k];
                            V = rec[(2 * D + 1) * P2G2_CAP + k];
#pragma unroll
                            for (int q2 = 0; q2 < C::NS; ++q2)
                                sig[q2] = rec[(2 * D + 2 + q2) * P2G2_CAP + k];
                        } else {
                            src = __ldg(perm + s0 + k);
#pragma unroll
                            for (int a = 0; a < D; ++a) {
                                x[a] = __ldg(P.x[a] + src);
                                v[a] = __ldg(P.v[a] + src);
                            }
                            m = __ldg(P.m + src);
                            V = __ldg(P.V + src);
#pragma unroll
                            for (int q2 = 0; q2 < C::NS; ++q2)
                                sig[q2] = __ldg(P.sig[q2] + src);
                        }
                        (void)src;
                        T w[D][3], dw[D][3];
#pragma unroll
                        for (int a = 0; a < D; ++a)
                            axis_weights<T, D>(x[a], sc.origin[a], sc.inv_dh, w[a], dw[a]);
                        T A[D * D];
                        int base[D];
                        if constexpr (AFF) {
#pragma unroll
                            for (int a = 0; a < D - 1; ++a)
                                base[a] = qc[a] * B + cn[a] - o[a];
                            base[D - 1] = qc[D - 1] * B + z;
                            affine_matrix<T, D>(sc, P, src, x, w, base, A);
                        }
                        // product of the non-march weights / derivative factors
                        T wp = T(1);
#pragma unroll
                        for (int a = 0; a < D - 1; ++a)
                            wp *= w[a][o[a]];
#pragma unroll
                        for (int o2 = 0; o2 < 3; ++o2) {
                            const T phi = wp * w[D - 1][o2];
                            T gw[D];
#pragma unroll
                            for (int a = 0; a < D; ++a) {
                                T r = (a == D - 1) ? dw[a][o2] : dw[a][o[a]];
#pragma unroll
                                for (int b = 0; b < D; ++b)
                                    if (b != a)
                                        r *= (b == D - 1) ? w[b][o2] : w[b][o[b]];
                                gw[a] = r;
                            }
                            T vel[D];
#pragma unroll
                            for (int a = 0; a < D; ++a)
                                vel[a] = v[a];
                            if constexpr (AFF) {
                                T r[D];
#pragma unroll
                                for (int a = 0; a < D; ++a) {
                                    int idx = a == D - 1 ? base[a] + o2 : base[a] + o[a];
                                    r[a] = (sc.origin[a] + T(idx) * sc.dh) - x[a];
                                }
#pragma unroll
                                for (int a = 0; a < D; ++a) {
                                    T s = T(0);
#pragma unroll
                                    for (int b = 0; b < D; ++b)
                                        s += A[a * D + b] * r[b];
                                    vel[a] += s;
                                }
                            }
                            const T mphi = m * phi;
                            acc[o2][0] += mphi;
#pragma unroll
                            for (int a = 0; a < D; ++a) {
                                T sg = T(0);
#pragma unroll
                                for (int b = 0; b < D; ++b)
                                    sg += sig[sym_idx<D>(a, b)] * gw[b];
                                acc[o2][1 + a] += mphi * vel[a];
                                acc[o2][1 + D + a] = acc[o2][1 + D + a] - V * sg; // gravity: + g m_i per node (k_grid)
                            }
                        }
                    }
                }
                // node z of this column is final for this segment
                const int idx = ptile<D>(z, col);
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    part[f * C::TN + idx] = acc[0][f];
                    acc[0][f] = acc[1][f];
                    acc[1][f] = acc[2][f];
                    acc[2][f] = T(0);
                }
            }
            if (seg == C::SEGS - 1) { // top of the tile: nodes B and B+1
#pragma unroll
                for (int k = 0; k < 2; ++k)
#pragma unroll
                    for (int f = 0; f < NF; ++f)
                        part[f * C::TN + ptile<D>(ze + k, col)] = acc[k][f];
            } else {
#pragma unroll
                for (int k = 0; k < 2; ++k)
#pragma unroll
                    for (int f = 0; f < NF; ++f)
                        ov[k][f] = acc[k][f];
            }
        }
        __syncthreads(); // next segment's own sums for the shared nodes are written
        if (active && seg < C::SEGS - 1) {
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    T* p = part + f * C::TN + ptile<D>(ze + k, col);
                    *p = *p + ov[k][f];
                }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// P2G, staged (PIC / FLIP / blend).
//
// One CTA per occupied particle block, base levels (last axis) processed in order. Each level's
// particles -- one contiguous run of the level-major sorted order -- are staged by the whole CTA
// into shared memory as P2G records { w[d][3], dw[d][3], m, m v, V sigma } (weights computed
// once per particle). Thread (base column bc, offset oo on the first d-1 axes) owns the 3
// nodes (bc + oo, z .. z+2) in a rolling register window and visits only the particles of its
// own base column; the 3^(d-1) lanes of one base column are adjacent, so every record read is
// a shared-memory broadcast and no lane is idle. After each level the window's finished node
// is written to an exclusive (node column, source offset) slot; NCOL threads then sum the
// 3^(d-1) slots of each node column in fixed order into the block's partial tile. No atomics;
// per-node order = (source offset, level, chunk, sorted particle order): deterministic.
template <class T, int D> struct StageCfg {
    static constexpr int NSRC = D == 2 ? 3 : 9;              // offsets on the non-march axes
    static constexpr int NBC = Cfg<D>::NB / Cfg<D>::B;        // base columns per block
    static constexpr int THREADS = NBC * NSRC;                // 48 (2-D), 576 (3-D)
    static constexpr int NREC = 6 * D + 1 + D + Cfg<D>::NS;   // w, dw, m, mv, Vsig
    static constexpr int CAP = D == 2 ? 128 : (sizeof(T) == 8 ? 256 : 512);
    static constexpr size_t SMEM_REC = sizeof(T) * NREC * CAP;
    static constexpr size_t SMEM_SLOT = sizeof(T) * Cfg<D>::NCOL * NSRC * Cfg<D>::NF;
    static constexpr size_t SMEM = SMEM_REC + SMEM_SLOT;
};

template <class T, int D>
__global__ void __launch_bounds__(StageCfg<T, D>::THREADS, 1)
    k_p2g_staged(DevScene<T, D> sc, PBuf<T, D> P, const int* __restrict__ perm, const int* __restrict__ keys,
                 const int* __restrict__ bstart, const int* __restrict__ bend, const int* __restrict__ occ,
                 const int* __restrict__ n_occ, T* __restrict__ partials, const DevStatus* st)
{
    pdl_wait();
    pdl_trigger();
    using C = Cfg<D>;
    using S = StageCfg<T, D>;
    constexpr int B = C::B, TE = C::TE, NF = C::NF, CAP = S::CAP, NSRC = S::NSRC, NBC = S::NBC;
    constexpr int LVLBITS = (D - 1) * C::LOGB;
    // record field offsets (in units of CAP)
    constexpr int RW = 0, RDW = 3 * D, RM = 6 * D, RMV = 6 * D + 1, RVS = 7 * D + 1;
    extern __shared__ unsigned char smem_raw[];
    T* rec = reinterpret_cast<T*>(smem_raw);                            // [NREC][CAP]
    T* slots = reinterpret_cast<T*>(smem_raw + S::SMEM_REC);            // [NCOL][NSRC][NF]
    __shared__ int lvl[B + 1];
    __shared__ int cst[NBC + 1];
    if (st->abort)
        return;
    const int nocc = *n_occ;
    const int tid = threadIdx.x;
    const int bc = tid / NSRC, oo = tid % NSRC;
    int o[D - 1], bcc[D - 1], ncol = 0;
    {
        int kk = oo, rem = bc;
#pragma unroll
        for (int a = D - 2; a >= 0; --a) {
            o[a] = kk % 3;
            kk /= 3;
            bcc[a] = rem & (B - 1);
            rem >>= C::LOGB;
        }
#pragma unroll
        for (int a = 0; a < D - 1; ++a)
            ncol = ncol * TE + bcc[a] + o[a];
    }

    for (int w = blockIdx.x; w < nocc; w += gridDim.x) {
        const int Q = occ[w];
        const int s0 = bstart[Q], s1 = bend[Q], len = s1 - s0;
        __syncthreads();
        for (int z = tid; z <= B; z += blockDim.x) { // first index with level >= z
            int lo = 0, hi = len;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (((keys[s0 + mid] & (C::NB - 1)) >> LVLBITS) < z)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            lvl[z] = lo;
        }
        T* part = partials + (size_t)Q * NF * C::TN;
        T acc[3][NF];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int f = 0; f < NF; ++f)
                acc[k][f] = T(0);

        // after base level z (z < B) or at the tail (z = B, B+1): publish node level z
        auto emit_and_reduce = [&](int z) {
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                slots[(ncol * NSRC + oo) * NF + f] = acc[0][f];
                acc[0][f] = acc[1][f];
                acc[1][f] = acc[2][f];
                acc[2][f] = T(0);
            }
            __syncthreads();
            for (int c = tid; c < C::NCOL; c += blockDim.x) {
                int nc[D - 1];
                {
                    int rem = c;
#pragma unroll
                    for (int a = D - 2; a >= 0; --a) {
                        nc[a] = rem % TE;
                        rem /= TE;
                    }
                }
                T sum[NF];
#pragma unroll
                for (int f = 0; f < NF; ++f)
                    sum[f] = T(0);
#pragma unroll
                for (int q = 0; q < NSRC; ++q) {
                    bool ok = true;
                    int kk = q;
#pragma unroll
                    for (int a = D - 2; a >= 0; --a) {
                        const int bcq = nc[a] - kk % 3;
                        kk /= 3;
                        ok &= bcq >= 0 && bcq < B;
                    }
                    if (ok)
#pragma unroll
                        for (int f = 0; f < NF; ++f)
                            sum[f] += slots[(c * NSRC + q) * NF + f];
                }
#pragma unroll
                for (int f = 0; f < NF; ++f)
                    part[f * C::TN + ptile<D>(z, c)] = sum[f];
            }
        };

        for (int z = 0; z < B; ++z) {
            __syncthreads(); // lvl ready / previous reduce done
            const int l0 = lvl[z], nl = lvl[z + 1] - l0;
            for (int ch = 0; ch * CAP < nl || ch == 0; ++ch) {
                const int b0 = l0 + ch * CAP, cl = max(0, min(CAP, nl - ch * CAP));
                if (ch > 0)
                    __syncthreads(); // previous chunk consumed
                for (int c = tid; c <= NBC; c += blockDim.x) {
                    int lo = 0, hi = cl;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if ((keys[s0 + b0 + mid] & ((1 << LVLBITS) - 1)) < c)
                            lo = mid + 1;
                        else
                            hi = mid;
                    }
                    cst[c] = c == NBC ? cl : lo;
                }
                for (int r = tid; r < cl; r += blockDim.x) {
                    const int src = __ldg(perm + s0 + b0 + r);
                    const T m = __ldg(P.m + src), V = __ldg(P.V + src);
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        const T u = (__ldg(P.x[a] + src) - sc.origin[a]) * sc.inv_dh;
                        const T fx = u - dfloor<T>(u - T(0.5));
                        const T h0 = T(1.5) - fx, h1 = fx - T(1), h2 = fx - T(0.5);
                        rec[(RW + 3 * a + 0) * CAP + r] = T(0.5) * h0 * h0;
                        rec[(RW + 3 * a + 1) * CAP + r] = T(0.75) - h1 * h1;
                        rec[(RW + 3 * a + 2) * CAP + r] = T(0.5) * h2 * h2;
                        rec[(RDW + 3 * a + 0) * CAP + r] = -h0 * sc.inv_dh;
                        rec[(RDW + 3 * a + 1) * CAP + r] = -T(2) * h1 * sc.inv_dh;
                        rec[(RDW + 3 * a + 2) * CAP + r] = h2 * sc.inv_dh;
                        rec[(RMV + a) * CAP + r] = m * __ldg(P.v[a] + src);
                    }
                    rec[RM * CAP + r] = m;
#pragma unroll
                    for (int q = 0; q < C::NS; ++q)
                        rec[(RVS + q) * CAP + r] = V * __ldg(P.sig[q] + src);
                }
                __syncthreads();
                const int kb = cst[bc], ke = cst[bc + 1];
                for (int k = kb; k < ke; ++k) {
                    // weights of the first d-1 axes at this thread's offsets
                    T wn[D - 1], dwn[D - 1];
#pragma unroll
                    for (int a = 0; a < D - 1; ++a) {
                        wn[a] = rec[(RW + 3 * a + o[a]) * CAP + k];
                        dwn[a] = rec[(RDW + 3 * a + o[a]) * CAP + k];
                    }
                    T pw = T(1), pdw[D - 1];
#pragma unroll
                    for (int a = 0; a < D - 1; ++a)
                        pw *= wn[a];
#pragma unroll
                    for (int a = 0; a < D - 1; ++a) {
                        T r = dwn[a];
#pragma unroll
                        for (int b2 = 0; b2 < D - 1; ++b2)
                            if (b2 != a)
                                r *= wn[b2];
                        pdw[a] = r;
                    }
                    T wz[3], dwz[3], mv[D], vs[C::NS];
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        wz[q] = rec[(RW + 3 * (D - 1) + q) * CAP + k];
                        dwz[q] = rec[(RDW + 3 * (D - 1) + q) * CAP + k];
                    }
                    const T m = rec[RM * CAP + k];
#pragma unroll
                    for (int a = 0; a < D; ++a)
                        mv[a] = rec[(RMV + a) * CAP + k];
#pragma unroll
                    for (int q = 0; q < C::NS; ++q)
                        vs[q] = rec[(RVS + q) * CAP + k];
                    // V sigma grad(phi) = wz * u + dwz * t  (grad phi = (pdw wz, pw dwz))
                    T u[D], t[D];
#pragma unroll
                    for (int r = 0; r < D; ++r) {
                        T sacc = T(0);
#pragma unroll
                        for (int a = 0; a < D - 1; ++a)
                            sacc += vs[sym_idx<D>(r, a)] * pdw[a];
                        u[r] = sacc;
                        t[r] = vs[sym_idx<D>(r, D - 1)] * pw;
                    }
                    const T mpw = m * pw;
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        const T phi = pw * wz[q];
                        acc[q][0] += mpw * wz[q];
#pragma unroll
                        for (int a = 0; a < D; ++a) {
                            acc[q][1 + a] += phi * mv[a];
                            acc[q][1 + D + a] = acc[q][1 + D + a] - wz[q] * u[a] - dwz[q] * t[a]; // two FMAs
                        }
                    }
                }
            }
            __syncthreads(); // all records of this level consumed before the slots are reused
            emit_and_reduce(z);
        }
        __syncthreads();
        emit_and_reduce(B);
        __syncthreads();
        emit_and_reduce(B + 1);
    }
}

// quadratic B-spline weight and derivative of stencil offset o (bspline.hpp:94-108)
template <class T> __device__ __forceinline__ void quad_w(T fx, int o, T inv_dh, T& w, T& dw)
{
    if (o == 0) {
        const T h = T(1.5) - fx;
        w = T(0.5) * h * h;
        dw = -h * inv_dh;
    } else if (o == 1) {
        const T h = fx - T(1);
        w = T(0.75) - h * h;
        dw = -T(2) * h * inv_dh;
    } else {
        const T h = fx - T(0.5);
        w = T(0.5) * h * h;
        dw = h * inv_dh;
    }
}

// 3-D P2G, asynchronous pipeline (PIC / FLIP / blend). Thread = (base column, x-offset o0),
// looping the 3 y-offsets: 63 accumulators (3 node columns x a rolling 3-node window along z);
// the 3 lanes of a column read its particle records as shared-memory broadcasts. The staging
// is software-pipelined with cp.async (LDGSTS): work items are
// (base level, chunk <= CAP particles); item j+2's perm/keys and item j+1's particle fields
// are in flight while item j is marched, so the dependent gathers through the sort
// permutation never stall the CTA. Raw fields are staged (x, v, m, V, sigma); fractional
// offsets, m v and V sigma are formed per visit. One CTA per SM, full register file.
#ifndef P2G_SPLIT
#define P2G_SPLIT 1 // f64: the narrow mapping's 7 node fields split over two thread groups
#endif
// SPLIT (f64 only; bit-identical sums): 12 warps of <= 45 accumulators instead of 6 warps of 63.
// MEASURED C4: f64 k_p2g 0.517-0.523 -> 0.508 ms; f32 0.262 -> 0.318 ms (so f32 stays narrow).
// 3-D slot buffer layout: value (node column c < 100, source lane q < 9, field f < 7) at
// c + 107 q + 999 f. Strides from an exhaustive search over a bank model of the emit's writes
// (lanes = (base column, x offset)) and the sums' reads (lanes = consecutive (c, f) tasks):
// ~1.3x / ~1.0x the ideal wavefronts instead of 1.5x / 1.6x for the dense [c][q][f] layout
// (ncu at C4 f64: the dense layout's slot traffic was 32% of the kernel's shared wavefronts,
// half of it bank conflicts).
#ifndef SLOT3_DENSE
#define SLOT3_DENSE 0
#endif
__host__ __device__ constexpr int slot3(int c, int q, int f) { return SLOT3_DENSE ? (c * 9 + q) * 7 + f : c + 107 * q + 999 * f; }
constexpr int SLOT3_SIZE = 99 + 107 * 8 + 999 * 6 + 1;
static_assert(Cfg<3>::NCOL == 100 && Cfg<3>::NF == 7, "slot3 strides assume B = 8");

template <class T, bool WIDE = true, int NGR = 2> struct Pipe3Cfg {
    // NG thread groups of 192 lanes split the 7 node fields (m, p[3], f[3]); f64 only
    static constexpr int NG = (!WIDE && P2G_SPLIT && sizeof(T) == 8) ? NGR : 1;
    static constexpr bool SPLIT = NG > 1;
    static constexpr int LANES = WIDE ? 576 : 192 * NG;
    static constexpr int NBC = 64, THREADS = LANES, NSRC = 9, NRAW = 14, MAXIT = 64;
    static constexpr int CAP = 640;
    static constexpr size_t SMEM_RAW = sizeof(T) * 2 * NRAW * CAP;
    static constexpr size_t SMEM_PK = sizeof(int) * 3 * 2 * CAP;
    static constexpr size_t SMEM_SLOT = sizeof(T) * SLOT3_SIZE;
    static constexpr size_t SMEM = SMEM_RAW + SMEM_PK + SMEM_SLOT;
    // field range [fb(g), fb(g + 1)) of group g in the order m, p0..2, f0..2.
    // NG 2: {m, p, f_x} {f_y, f_z}; NG 3: {m, p} {f_x, f_y} {f_z} (FP64 work per lane-particle
    // ~73 / 85 / 58 instead of ~106 / 85). MEASURED C4 f64: NG 3 (18 warps) 0.98 ms against NG 2's
    // 0.49 ms -- ptxas caps it at 96 registers with 120 B of spills -- so NG 2 is the default.
    static constexpr int fb(int g) { return NG == 1 ? (g ? 7 : 0) : NG == 2 ? (g == 0 ? 0 : g == 1 ? 5 : 7) : (g == 0 ? 0 : g == 1 ? 4 : g == 2 ? 6 : 7); }
    static constexpr int NA = NG == 1 ? 7 : NG == 2 ? 5 : 4; // accumulated fields per thread (largest group)
};

// one staged particle's contributions to this lane's 3 x NO1 x 3 nodes, fields [FB, FE) only.
// The arithmetic per field is the same expression whatever the grouping (bit-identical sums).
template <int FB, int FE, int NO1, int NA, class T>
__device__ __forceinline__ void p2g_visit(T (&acc)[NO1][3][NA], T wx, T dwx, const T (&wy)[NO1], const T (&dwy)[NO1],
                                          const T (&wz)[3], const T (&dwz)[3], const T* __restrict__ R, int k, int CAP)
{
    constexpr int RV = 3, RM = 6, RS = 8;
    constexpr bool HM = FB == 0, HP = FB < 4 && FE > 1, HF = FE > 4;
#pragma unroll
    for (int o1 = 0; o1 < NO1; ++o1) {
        const T pw = wx * wy[o1];
        if constexpr (HM || HP) {
            T m = T(0), mv[3];
            if constexpr (HM)
                m = R[RM * CAP + k];
#pragma unroll
            for (int a = 0; a < 3; ++a)
                mv[a] = R[(RV + a) * CAP + k];
            const T mpw = m * pw;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const T phi = pw * wz[q];
                if constexpr (HM)
                    acc[o1][q][0] += mpw * wz[q];
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    if (1 + a >= FB && 1 + a < FE)
                        acc[o1][q][1 + a - FB] += phi * mv[a];
            }
        }
        if constexpr (HF) {
            // grad phi = (dwx wy wz, wx dwy wz, wx wy dwz): V sigma grad phi = wz u + dwz t
            const T p1 = dwx * wy[o1], p2 = wx * dwy[o1];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                if (4 + r >= FB && 4 + r < FE) {
                    const T u = R[(RS + sym_idx<3>(r, 0)) * CAP + k] * p1 + R[(RS + sym_idx<3>(r, 1)) * CAP + k] * p2;
                    const T t = R[(RS + sym_idx<3>(r, 2)) * CAP + k] * pw;
#pragma unroll
                    for (int q = 0; q < 3; ++q)
                        acc[o1][q][4 + r - FB] = acc[o1][q][4 + r - FB] - wz[q] * u - dwz[q] * t; // two FMAs
                }
            }
        }
    }
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
template <class T> __device__ __forceinline__ void cp_async_t(T* smem, const T* gmem)
{
    if constexpr (sizeof(T) == 8)
        cp_async8(smem, gmem);
    else
        cp_async4(smem, gmem);
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ABL != 0: timing ablation only (1 skip reduce, 2 skip convert, 4 skip march, 32 phase clocks:
// thread 0 of CTAs 0..3 prints cycles per phase, with a barrier after the march), launched in
// front of the real kernel by ablation builds (-DP2G_ABL=...), never on its own
template <class T, bool WIDE, int ABL = 0, int NGR = 2>
__global__ void __launch_bounds__(Pipe3Cfg<T, WIDE, NGR>::THREADS, 1)
    k_p2g_pipe3(DevScene<T, 3> sc, PBuf<T, 3> P, const int* __restrict__ perm, const int* __restrict__ keys,
                const int* __restrict__ bstart, const int* __restrict__ bend, const int* __restrict__ lstart,
                const int* __restrict__ occ, const int* __restrict__ n_occ, T* __restrict__ partials, DevStatus* st,
                int* __restrict__ wq)
{
    pdl_wait();
    pdl_trigger();
    using C = Cfg<3>;
    using S = Pipe3Cfg<T, WIDE, NGR>;
    constexpr int B = C::B, TE = C::TE, NF = C::NF, CAP = S::CAP, NBC = S::NBC, NSRC = S::NSRC, NRAW = S::NRAW;
    constexpr int NO1 = WIDE ? 1 : 3; // y-offsets handled per thread
    // NG > 1: the node fields are split over NG groups of 192 lanes (S::fb): e.g. NG 2 gives
    // 12 warps with <= 45 accumulators each instead of 6 warps with 63
    constexpr int NG = S::NG;
    constexpr int NA = S::NA; // accumulated fields per thread
    // raw field rows: x0..2, v0..2, m, V, sig0..5
    constexpr int RX = 0, RV = 3, RM = 6, RVOL = 7, RS = 8;
    extern __shared__ unsigned char smem_raw[];
    T* raw = reinterpret_cast<T*>(smem_raw);                                   // [2][NRAW][CAP]
    int* pk = reinterpret_cast<int*>(smem_raw + S::SMEM_RAW);                  // [3][2][CAP] (perm, col)
    T* slots = reinterpret_cast<T*>(smem_raw + S::SMEM_RAW + S::SMEM_PK);      // [NCOL][NSRC][NF]
    __shared__ int it_start[S::MAXIT], it_len[S::MAXIT], it_lvl[S::MAXIT], it_last[S::MAXIT];
    __shared__ int nit_s, ccount[2][NBC]; // per-item column counts, double-buffered
    __shared__ int w_s;                   // next list entry (work counter, kernels_util.cuh)
    const int nocc = st->abort ? 0 : *n_occ; // every CTA still passes wq_finish
    if (threadIdx.x == 0)
        w_s = wq_first(wq);
    const int tid = threadIdx.x;
    const int grp = NG > 1 ? tid / 192 : 0; // warp-uniform
    const int lt = tid - 192 * grp;
    const int gfb = S::fb(grp), gfn = S::fb(grp + 1) - gfb; // this group's fields
    const int bc = WIDE ? lt / 9 : lt / 3;
    const int o0 = WIDE ? (lt % 9) / 3 : lt % 3;
    const int o1t = WIDE ? lt % 3 : 0; // WIDE: this thread's y-offset
    const bool mid = o0 == 1;
    const T xoff = o0 == 0 ? T(1.5) : (o0 == 1 ? T(1) : T(0.5)); // h = fx - xoff (bspline.hpp:94-99)
    const int bc0 = bc >> C::LOGB, bc1 = bc & (B - 1);
    // raw rows x0..2 v0..2 m V sigma0..5 = PLay fields 0..7 and SIG..SIG+5 of the strided buffer
    // (one base pointer and a stride instead of 14 pointers reloaded from the parameter bank)
    using PL = PLay<3>;
    static_assert(PL::M == RM && PL::VOL == RVOL && PL::SIG == RS + 2 && RS + 6 == NRAW, "raw row map");
    const long long SI = P.S;
    constexpr bool CLK = (ABL & 32) != 0;
    // staged record r lives at column rsw(r) of its field row: an XOR swizzle inside each group of
    // 16 (a bank-width of doubles), so the march's lanes -- different node columns, whose records
    // sit a column count apart (8 at a uniform 8 per column: C4's lattice) -- hit different banks
    // instead of 4-6-way conflicting. A permutation of [0, CAP) since CAP % 16 == 0.
    static_assert(CAP % 16 == 0, "swizzle groups");
    auto rsw = [](int r) { return r ^ ((r >> 4) & 15); };
    long long ck[16] = {}, t0 = 0;
    auto mark = [&](int ph) {
        if constexpr (CLK) {
            const long long t = clock64();
            ck[ph] += t - t0;
            t0 = t;
        }
    };
    if constexpr (CLK)
        t0 = clock64();

    for (;;) {
        __syncthreads(); // w_s published; the previous block's shared-memory readers are done
        const int w = w_s;
        if (w >= nocc)
            break;
        if constexpr (CLK)
            ck[7] += 1;
        const int Q = occ[w];
        const int s0 = bstart[Q], s1 = bend[Q];
        int qc[3];
        block_coords<3>(Q, sc.nb, qc);
        if (tid == 0) { // level starts (suffix minimum) -> work items
            int lv[B + 1];
            int nxt = s1;
            lv[B] = s1 - s0;
            for (int z = B - 1; z >= 0; --z) {
                const int v = lstart[Q * (B + 1) + z];
                nxt = (v >= s0 && v < s1) ? v : nxt;
                lv[z] = nxt - s0;
            }
            int k = 0;
            for (int z = 0; z < B; ++z) {
                const int nl = lv[z + 1] - lv[z];
                const int nch = nl > 0 ? (nl + CAP - 1) / CAP : 1;
                for (int c = 0; c < nch; ++c) {
                    if (k < S::MAXIT) {
                        it_start[k] = lv[z] + c * CAP;
                        it_len[k] = min(CAP, nl - c * CAP);
                        it_lvl[k] = z;
                        it_last[k] = c == nch - 1;
                    }
                    ++k;
                }
            }
            if (k > S::MAXIT) { // pathological compression: refuse loudly
                st->far_flag = 1;
                st->abort = 1;
                k = 0;
            }
            nit_s = k;
        }
        __syncthreads();
        const int nit = nit_s;
        if (tid == 0) // every thread read w_s before the barrier above
            w_s = wq_next(wq, w);
        mark(8);
        auto issue_pk = [&](int j) {
            int* dp = pk + (j % 3) * 2 * CAP;
            const int b = s0 + it_start[j];
            for (int r = tid; r < it_len[j]; r += blockDim.x) {
                cp_async4(dp + r, perm + b + r);
                cp_async4(dp + CAP + r, keys + b + r);
            }
        };
        auto issue_fields = [&](int j) {
            const int* pp = pk + (j % 3) * 2 * CAP;
            T* rb = raw + (j & 1) * NRAW * CAP;
            const int len = it_len[j];
            for (int r = tid; r < len; r += blockDim.x) {
                const T* q = P.base + pp[r];
#pragma unroll
                for (int f = 0; f < NRAW; ++f)
                    cp_async_t<T>(rb + f * CAP + rsw(r), q + (f < RS ? f : f + 2) * SI);
            }
        };
        if (tid < NBC) {
            ccount[0][tid] = 0;
            ccount[1][tid] = 0;
        }
        if (nit > 0)
            issue_pk(0);
        if (nit > 1)
            issue_pk(1);
        cp_async_commit();
        cp_async_wait_all();
        __syncthreads();
        if (nit > 0)
            issue_fields(0);
        cp_async_commit();
        mark(0);

        T* part = partials + (size_t)Q * NF * C::TN;
        T acc[NO1][3][NA];
#pragma unroll
        for (int a = 0; a < NO1; ++a)
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int f = 0; f < NA; ++f)
                    acc[a][k][f] = T(0);

        auto emit_and_reduce = [&](int z) {
#pragma unroll
            for (int i1 = 0; i1 < NO1; ++i1) {
                const int o1 = WIDE ? o1t : i1;
                const int ncol = (bc0 + o0) * TE + bc1 + o1;
#pragma unroll
                for (int f = 0; f < NA; ++f) {
                    if (f < gfn)
                        slots[slot3(ncol, o0 * 3 + o1, gfb + f)] = acc[i1][0][f];
                    acc[i1][0][f] = acc[i1][1][f];
                    acc[i1][1][f] = acc[i1][2][f];
                    acc[i1][2][f] = T(0);
                }
            }
            mark(11);
            __syncthreads(); // slots complete
            mark(12);
            // one (node column, field) per task: 700 short fixed-order sums over all threads
            for (int t = tid; t < ((ABL & 1) ? 0 : C::NCOL * NF); t += blockDim.x) {
                const int c = t / NF, f = t - c * NF;
                const int n0 = c / TE, n1 = c - n0 * TE;
                T sum = T(0);
#pragma unroll
                for (int q = 0; q < NSRC; ++q) {
                    const int b0 = n0 - q / 3, b1 = n1 - q % 3;
                    if (b0 >= 0 && b0 < B && b1 >= 0 && b1 < B)
                        sum += slots[slot3(c, q, f)];
                }
                part[f * C::TN + ptile<3>(z, c)] = sum;
            }
            // no closing barrier: the next emit's slot writes follow the next item's top barrier
            // (or the explicit one between the two final emits)
        };

        for (int j = 0; j < nit; ++j) {
            cp_async_wait_all();
            __syncthreads(); // fields(j) and pk(j+1) have landed for every thread
            mark(1);
            if (j + 2 < nit)
                issue_pk(j + 2);
            // fields(j+1) are issued one row per march iteration below, so the LDGSTS traffic
            // overlaps the FP64 march instead of stalling every warp at once (MEASURED C4 f64: the
            // up-front issue took 17% of the kernel's cycles); the commit follows the march
            const int nrow1 = j + 1 < nit ? it_len[j + 1] : 0;
            int prow = tid;
            const int* pp1 = pk + ((j + 1) % 3) * 2 * CAP;
            T* rb1 = raw + ((j + 1) & 1) * NRAW * CAP;
            auto issue_row = [&]() {
                const T* q = P.base + pp1[prow];
#pragma unroll
                for (int f = 0; f < NRAW; ++f)
                    cp_async_t<T>(rb1 + f * CAP + rsw(prow), q + (f < RS ? f : f + 2) * SI);
                prow += blockDim.x;
            };
            mark(9);
            // item j: convert each staged particle once (x -> fractional offset, v -> m v,
            // sigma -> V sigma) and count its column (records are column-sorted inside a level)
            const int len = it_len[j];
            const int* col = pk + (j % 3) * 2 * CAP + CAP;
            int* cnt = ccount[j & 1];
            if (tid < NBC) // the other buffer was last read before this item's top barrier
                ccount[(j + 1) & 1][tid] = 0;
            {
                T* Rw = raw + (j & 1) * NRAW * CAP;
                for (int r0 = tid; r0 < len; r0 += blockDim.x) {
                    atomicAdd(&cnt[col[r0] & (NBC - 1)], 1);
                    if (ABL & 2)
                        continue;
                    const int r = rsw(r0);
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const T u = (Rw[(RX + a) * CAP + r] - sc.origin[a]) * sc.inv_dh;
                        Rw[(RX + a) * CAP + r] = u - dfloor<T>(u - T(0.5));
                    }
                    const T m = Rw[RM * CAP + r], V = Rw[RVOL * CAP + r];
#pragma unroll
                    for (int a = 0; a < 3; ++a)
                        Rw[(RV + a) * CAP + r] *= m;
#pragma unroll
                    for (int q = 0; q < 6; ++q)
                        Rw[(RS + q) * CAP + r] *= V;
                }
            }
            mark(10);
            __syncthreads(); // converted records and the counts are complete
            mark(2);
            // every warp scans the 64 column counts itself (no extra barrier): lane l holds the
            // exclusive prefix of columns 2l and 2l+1
            int kb, ke;
            {
                const int lane = tid & 31;
                const int c0 = cnt[2 * lane], c1 = cnt[2 * lane + 1];
                int v = c0 + c1;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, v, d);
                    if (lane >= d)
                        v += t;
                }
                const int excl = v - c0 - c1;
                const int src = bc >> 1;
                const int e = __shfl_sync(0xffffffffu, excl, src);
                const int a0 = __shfl_sync(0xffffffffu, c0, src);
                const int a1 = __shfl_sync(0xffffffffu, c1, src);
                kb = (bc & 1) ? e + a0 : e;
                ke = kb + ((bc & 1) ? a1 : a0);
            }
            const T* R = raw + (j & 1) * NRAW * CAP;
            for (int k0 = kb; k0 < ((ABL & 4) ? kb : ke); ++k0) {
                const int k = rsw(k0);
                T f[3];
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    f[a] = R[(RX + a) * CAP + k];
                T wx, dwx, wy[NO1], dwy[NO1], wz[3], dwz[3];
                { // this lane's x offset o0 (lanes differ): branch-free quadratic B-spline
                    const T h = f[0] - xoff;
                    const T hh = h * h;
                    wx = mid ? T(0.75) - hh : T(0.5) * hh;
                    dwx = (mid ? -T(2) * h : h) * sc.inv_dh;
                }
#pragma unroll
                for (int i1 = 0; i1 < NO1; ++i1)
                    quad_w<T>(f[1], WIDE ? o1t : i1, sc.inv_dh, wy[i1], dwy[i1]);
#pragma unroll
                for (int q = 0; q < 3; ++q)
                    quad_w<T>(f[2], q, sc.inv_dh, wz[q], dwz[q]);
                if (grp == 0)
                    p2g_visit<S::fb(0), S::fb(1)>(acc, wx, dwx, wy, dwy, wz, dwz, R, k, CAP);
                else if constexpr (NG > 1) {
                    if (NG == 2 || grp == 1)
                        p2g_visit<S::fb(1), S::fb(2)>(acc, wx, dwx, wy, dwy, wz, dwz, R, k, CAP);
                    else if constexpr (NG > 2)
                        p2g_visit<S::fb(2), S::fb(3)>(acc, wx, dwx, wy, dwy, wz, dwz, R, k, CAP);
                }
                if (prow < nrow1)
                    issue_row();
            }
            while (prow < nrow1)
                issue_row();
            cp_async_commit();
            if constexpr (CLK) {
                mark(3);
                __syncthreads();
                mark(4);
                ck[6] += 1;
            }
            if (it_last[j]) // slots were last read before the previous emit's closing barrier
                emit_and_reduce(it_lvl[j]);
            mark(5);
        }
        cp_async_wait_all();
        __syncthreads();
        emit_and_reduce(B);
        __syncthreads(); // slots reused by the next emit right away
        emit_and_reduce(B + 1);
        mark(0);
    }
    if constexpr (CLK)
        if (threadIdx.x == 0 && blockIdx.x < 4)
            printf("p2g-clk cta %d blocks %lld items %lld setup+tail %lld wait %lld convert %lld march0 %lld "
                   "march-imbalance %lld emit %lld\n",
                   blockIdx.x, ck[7], ck[6], ck[0], ck[1], ck[2], ck[3], ck[4], ck[5]);
    if constexpr (CLK)
        if (threadIdx.x == 0 && blockIdx.x < 4)
            printf("p2g-clk2 cta %d blocksetup %lld issue %lld convloop %lld slotwrite %lld slotbar %lld\n", blockIdx.x,
                   ck[8], ck[9], ck[10], ck[11], ck[12]);
    wq_finish(wq);
}

// ---- 3-D P2G, warp-specialized (PIC / FLIP / blend) ---------------------------------------
// The same per-particle arithmetic, node fields, partial tiles and fixed combine order as
// k_p2g_pipe3 (bit-identical output), with the work split by role instead of by phase:
//   producer warps (f64: 2, f32: 4): pull occupied blocks from the work counter, build their
//     (level, chunk) item lists, gather each item's particle fields through the sort permutation
//     with cp.async into one of two record buffers, convert them (fractional offset, m v, V sigma),
//     count the node columns and publish the item on an mbarrier (full/empty pair per buffer);
//   consumer warps (the pipe3 lane mapping, 6 warps): wait for an item, march it (FP64), release
//     the buffer, and emit finished node planes: slot writes, then the fixed-order 9-source sums
//     into the block's partial tile, between two named barriers of the consumers only.
// No CTA-wide barrier after the setup. Variants kept for A/B (macros): WS_NG=2 splits the 7 node
// fields over two consumer groups (12 warps at 152 registers: setmaxnreg moves 128 x 72 registers
// from a 4-warp producer warpgroup; the register file is split over the 4 SM sub-partitions,
// 16384 each, warps round-robin, so 3 x 152 + 56 = 512 per lane slot); WS_PRED=1 has the
// producers do the plane sums (two slot buffers).
// MEASURED (C4 f64): pipe3 0.47 ms with the FP64 pipe 37% busy, the march ~60% of its cycles;
// this kernel 0.41 ms, FP64 45%, shared wavefronts 34% of peak. Tried and slower (same-box A/B,
// phase clocks in tools/p2g_clocks.py): the sums on the producers (PRED, 0.402 vs 0.388 ms), on
// a separate reducer warp (0.415), on the lighter consumer group only (0.45); releasing the record
// buffer after the sums (0.417 vs 0.406: the producers' gather burst then slows the march as much
// as it sped up the sums -- the LSU/MIO traffic of the gathers is paid by whichever phase it
// overlaps); unconditional slot loads in the sums (0.414).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b)
{
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(b)) : "memory");
}
// a protocol bug must not hang the GPU: after 2^26 polls (seconds even when a poll returns at
// once; legitimate waits are microseconds, and the margin covers time-slicing with other
// contexts) the kernel reports the barrier and traps, which surfaces as a launch failure
#ifndef MBAR_ASM_LOOP
#define MBAR_ASM_LOOP 0
#endif
#ifndef WS_SLEEP_NS
#define WS_SLEEP_NS 128
#endif
// SLEEP: back off between polls (a waiting producer warp shares its sub-partition's issue slots
// with three consumer warps)
template <bool SLEEP = false> __device__ __forceinline__ void mbar_wait(unsigned long long* b, int parity)
{
    if (MBAR_ASM_LOOP) {
        asm volatile("{\n .reg .pred P1;\n"
                     "WAIT_%=:\n"
                     " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                     " @!P1 bra WAIT_%=;\n"
                     "}\n" ::"r"(smem_u32(b)),
                     "r"(parity)
                     : "memory");
        return;
    }
    const unsigned a = smem_u32(b);
    unsigned ok = 0, spins = 0;
    for (;;) {
        asm volatile("{\n .reg .pred P1;\n"
                     " mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, P1;\n"
                     "}\n"
                     : "=r"(ok)
                     : "r"(a), "r"(parity)
                     : "memory");
        if (ok)
            return;
        if (SLEEP && WS_SLEEP_NS > 0)
            __nanosleep(WS_SLEEP_NS);
        if (++spins == (1u << 26)) {
            printf("mbarrier wait timed out: block %d thread %d barrier smem+%u parity %d\n", blockIdx.x, threadIdx.x,
                   a, parity);
            __trap();
        }
    }
}
__device__ __forceinline__ void named_bar(int id, int count)
{
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

#ifndef WS_REALLOC
#define WS_REALLOC 1
#endif
#ifndef WS_PRED
#define WS_PRED 0
#endif
#ifndef WS_CAP
#define WS_CAP 576 // records per item (a multiple of 16: the swizzle groups). MEASURED C4 f64 P2G: 640 0.378 ms, 576 0.347, 512 0.347, 448 0.435, 384 0.451 (a C4 level holds 512 particles: below that every level splits), 256 0.392
#endif
#ifndef WS_PREFETCH_REC
#define WS_PREFETCH_REC 0 // next record in registers during the march: MEASURED f64 0.390 vs 0.380 ms, f32 equal
#endif
#ifndef WS_PROD_REGS
#define WS_PROD_REGS 56
#endif
#ifndef WS_LB
#define WS_LB 0
#endif
#ifndef WS_PREFETCH_LATE
#define WS_PREFETCH_LATE 0
#endif
// Shape (A/B on one box, C4): f64 one field group (6 consumer warps, 63 accumulators, ~200
// registers) + 2 producer warps 0.378 ms; two field groups (12 consumer warps at 152 registers via
// setmaxnreg) + 4 producer warps 0.406 ms; one group + 4 producer warps 0.531 ms (320 threads cap
// the consumers at 168 registers: spills). f32: one group + 4 producer warps 0.268 ms, + 2: 0.285.
#ifndef WS_NG
#define WS_NG 1
#endif
#ifndef WS_PROD1
#define WS_PROD1 0 // 0: 64 (f64) / 128 (f32)
#endif
template <class T> struct WsCfg {
    using P3 = Pipe3Cfg<T, false, WS_NG>;
    static constexpr int NG = P3::NG, NA = P3::NA;
    static constexpr int CONS = 192 * NG;  // consumer threads (f64: 12 warps, f32: 6)
    static constexpr int PROD = NG == 1 ? (WS_PROD1 ? WS_PROD1 : sizeof(T) == 8 ? 64 : 128) : 128; // producer threads
    static constexpr int THREADS = CONS + PROD;
    static constexpr bool REALLOC = WS_REALLOC && CONS % 128 == 0;
    static constexpr int WPS = (THREADS / 32 + 3) / 4; // warps per SM sub-partition
    static constexpr int BASE_REGS = (512 / WPS) / 8 * 8 > 255 ? 255 : (512 / WPS) / 8 * 8, PROD_REGS = WS_PROD_REGS, CONS_REGS = 152;
    static_assert(!REALLOC || CONS * (CONS_REGS - BASE_REGS) <= PROD * (BASE_REGS - PROD_REGS), "register pool");
    static_assert(!REALLOC || (WPS == 4 && 3 * CONS_REGS + PROD_REGS <= 512), "sub-partition register file");
    // PRED: the producers sum the finished node planes (two slot buffers, so CAP 512: f64
    // 2 x 14 x 512 x 8 + 2 x 55600 B = 226 KB); otherwise the consumers do, between two named
    // barriers of their own, from one slot buffer. MEASURED C4 f64: consumers 0.388 ms, producers
    // 0.402 ms (their sums' shared-memory traffic slows the overlapping march by ~25%).
    static constexpr bool PRED = WS_PRED;
    static constexpr int NBC = 64, NSRC = 9, NRAW = 14, MAXIT = 64, CAP = PRED ? 512 : WS_CAP, NSLOT = PRED ? 2 : 1;
    static constexpr int SLOT = SLOT3_SIZE; // values per slot buffer
    static constexpr size_t SMEM_RAW = sizeof(T) * 2 * NRAW * CAP;
    static constexpr size_t SMEM = SMEM_RAW + sizeof(T) * NSLOT * SLOT;
};

// CLK: timing build only (tools/p2g_clocks.py): thread 0 of each role in CTAs 0..3 prints cycles per phase
template <class T, bool CLK = false>
__global__ void
#if WS_LB
__launch_bounds__(WsCfg<T>::THREADS, 1)
#else
__maxnreg__(WsCfg<T>::BASE_REGS)
#endif
    k_p2g_ws(DevScene<T, 3> sc, PBuf<T, 3> P, const int* __restrict__ perm, const int* __restrict__ keys,
             const int* __restrict__ bstart, const int* __restrict__ bend, const int* __restrict__ lstart,
             const int* __restrict__ occ, const int* __restrict__ n_occ, T* __restrict__ partials, DevStatus* st,
             int* __restrict__ wq)
{
    pdl_wait();
    pdl_trigger();
    using C = Cfg<3>;
    using S = WsCfg<T>;
    constexpr int B = C::B, TE = C::TE, NF = C::NF, CAP = S::CAP, NBC = S::NBC, NSRC = S::NSRC, NRAW = S::NRAW;
    constexpr int NO1 = 3, NG = S::NG, NA = S::NA, CONS = S::CONS;
    constexpr int RX = 0, RV = 3, RM = 6, RVOL = 7, RS = 8;
    extern __shared__ unsigned char smem_raw[];
    T* raw = reinterpret_cast<T*>(smem_raw);                      // [2][NRAW][CAP]
    T* slots = reinterpret_cast<T*>(smem_raw + S::SMEM_RAW);      // [2][NCOL][NSRC][NF]
    __shared__ int cnt_s[2][NBC];                                 // per-item column counts
    __shared__ int4 desc_s[2];                                    // (Q, level, flags, -): 1 level done, 2 block done, 4 end
    __shared__ int2 em_s[2];                                      // slot buffer: (Q, node plane)
    __shared__ __align__(8) unsigned long long bar_full[2], bar_empty[2], sl_full[2], sl_empty[2];
    __shared__ int it_start[S::MAXIT], it_len[S::MAXIT], it_lvl[S::MAXIT], it_last[S::MAXIT]; // producers only
    __shared__ int blk_s[4];                                      // producers only: w, Q, s0, nit
    const int tid = threadIdx.x;
    const int nocc = st->abort ? 0 : *n_occ;
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar_full[i], S::PROD);
            mbar_init(&bar_empty[i], CONS / 32);
            mbar_init(&sl_full[i], CONS / 32);
            mbar_init(&sl_empty[i], S::PROD);
        }
    }
    __syncthreads();
    // staged record r at column rsw(r) of its field row (bank swizzle, as in k_p2g_pipe3)
    auto rsw = [](int r) { return r ^ ((r >> 4) & 15); };
    using PL = PLay<3>;
    static_assert(PL::M == RM && PL::VOL == RVOL && PL::SIG == RS + 2 && RS + 6 == NRAW, "raw row map");
    long long ck[6] = {}, t0 = 0;
    auto mark = [&](int ph) {
        if constexpr (CLK) {
            const long long t = clock64();
            ck[ph] += t - t0;
            t0 = t;
        }
    };
    if constexpr (CLK)
        t0 = clock64();

    if (tid >= CONS) { // ================= producer warpgroup =================
        if constexpr (S::REALLOC) // registers to the consumers
            asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(S::PROD_REGS));
        const int pt = tid - CONS;
        const long long SI = P.S;
        // the plane sums of slot buffer (e & 1): one (node column, field) per task, fixed order
        // over the 9 source lanes; emits are reduced in the consumers' order
        int nred = 0;
        auto reduce_one = [&]() {
            const int sb = nred & 1;
            mbar_wait(&sl_full[sb], (nred >> 1) & 1);
            const int2 em = em_s[sb];
            const T* sl = slots + sb * S::SLOT;
            T* part = partials + (size_t)em.x * NF * C::TN;
            constexpr int NT = C::NCOL * NF, UR = 2;
            for (int t0 = pt; t0 < NT; t0 += UR * S::PROD) {
                T sum[UR];
#pragma unroll
                for (int x = 0; x < UR; ++x) {
                    const int t = t0 + x * S::PROD;
                    const int c = t / NF, f = t - c * NF;
                    const int n0 = c / TE, n1 = c - n0 * TE;
                    sum[x] = T(0);
#pragma unroll
                    for (int q = 0; q < NSRC; ++q) {
                        const int b0 = n0 - q / 3, b1 = n1 - q % 3;
                        if (t < NT && b0 >= 0 && b0 < B && b1 >= 0 && b1 < B)
                            sum[x] += sl[slot3(c, q, f)];
                    }
                }
#pragma unroll
                for (int x = 0; x < UR; ++x) {
                    const int t = t0 + x * S::PROD;
                    if (t < NT) {
                        const int c = t / NF, f = t - c * NF;
                        part[f * C::TN + ptile<3>(em.y, c)] = sum[x];
                    }
                }
            }
            mbar_arrive(&sl_empty[sb]);
            ++nred;
        };
        int em_prev2 = 0, em_prev1 = 0; // node planes the consumers emit after items j-2, j-1
        int w = 0;
        if (pt == 0)
            w = wq_first(wq);
        int j = 0; // items published so far (both buffers)
        for (;;) {
            if (pt == 0) {
                blk_s[0] = w;
                if (w < nocc) { // level starts (suffix minimum) -> work items, as k_p2g_pipe3
                    const int Q = occ[w];
                    const int s0 = bstart[Q], s1 = bend[Q];
                    int lv[B + 1];
                    int nxt = s1;
                    lv[B] = s1 - s0;
                    for (int z = B - 1; z >= 0; --z) {
                        const int v = lstart[Q * (B + 1) + z];
                        nxt = (v >= s0 && v < s1) ? v : nxt;
                        lv[z] = nxt - s0;
                    }
                    int k = 0;
                    for (int z = 0; z < B; ++z) {
                        const int nl = lv[z + 1] - lv[z];
                        const int nch = nl > 0 ? (nl + CAP - 1) / CAP : 1;
                        for (int c = 0; c < nch; ++c) {
                            if (k < S::MAXIT) {
                                it_start[k] = lv[z] + c * CAP;
                                it_len[k] = min(CAP, nl - c * CAP);
                                it_lvl[k] = z;
                                it_last[k] = c == nch - 1;
                            }
                            ++k;
                        }
                    }
                    if (k > S::MAXIT) { // pathological compression: refuse loudly
                        st->far_flag = 1;
                        st->abort = 1;
                        k = S::MAXIT;
                    }
                    blk_s[1] = Q;
                    blk_s[2] = s0;
                    blk_s[3] = k;
                    w = wq_next(wq, w);
                }
            }
            named_bar(2, S::PROD);
            mark(0);
            const bool done = blk_s[0] >= nocc;
            const int Q = blk_s[1], s0 = blk_s[2], nit = done ? 1 : blk_s[3];
            for (int i = 0; i < nit; ++i, ++j) {
                const int b = j & 1, u = j >> 1;
                // this item's permutation and keys are loaded before the buffer is free
                constexpr int RPT = (CAP + S::PROD - 1) / S::PROD; // rows per producer thread
                const int len = done ? 0 : it_len[i], base = s0 + (done ? 0 : it_start[i]);
                int pr[RPT], kr[RPT];
                if (WS_PREFETCH_LATE && u > 0)
                    mbar_wait<true>(&bar_empty[b], (u - 1) & 1);
#pragma unroll
                for (int e = 0; e < RPT; ++e) {
                    const int r = pt + e * S::PROD;
                    pr[e] = r < len ? perm[base + r] : 0;
                    kr[e] = r < len ? keys[base + r] : 0;
                }
                if (!WS_PREFETCH_LATE && u > 0) // the consumers are done with this buffer's previous item (j - 2)
                    mbar_wait<true>(&bar_empty[b], (u - 1) & 1);
                mark(1);
                if (done) { // end marker; then the planes of the last two items
                    if (pt == 0)
                        desc_s[b] = make_int4(-1, 0, 4, 0);
                    mbar_arrive(&bar_full[b]);
                    if constexpr (S::PRED)
                        for (int e = 0; e < em_prev2 + em_prev1; ++e)
                            reduce_one();
                    break;
                }
                if (pt < NBC)
                    cnt_s[b][pt] = 0;
                named_bar(2, S::PROD); // counts zeroed before any producer adds to them
                T* rb = raw + b * NRAW * CAP;
#pragma unroll
                for (int e = 0; e < RPT; ++e) {
                    const int r = pt + e * S::PROD;
                    if (r < len) {
                        const T* q = P.base + pr[e];
                        const int rs = rsw(r);
#pragma unroll
                        for (int f = 0; f < NRAW; ++f)
                            cp_async_t<T>(rb + f * CAP + rs, q + (f < RS ? f : f + 2) * SI);
                        atomicAdd(&cnt_s[b][kr[e] & (NBC - 1)], 1);
                    }
                }
                cp_async_commit();
                mark(2);
                if constexpr (S::PRED)
                    for (int e = 0; e < em_prev2; ++e) // while the copies land: item j-2's node planes
                        reduce_one();
                cp_async_wait_all(); // this thread's rows have landed; it converts only those
                mark(3);
                for (int r0 = pt; r0 < len; r0 += S::PROD) {
                    const int r = rsw(r0);
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const T uu = (rb[(RX + a) * CAP + r] - sc.origin[a]) * sc.inv_dh;
                        rb[(RX + a) * CAP + r] = uu - dfloor<T>(uu - T(0.5));
                    }
                    const T m = rb[RM * CAP + r], V = rb[RVOL * CAP + r];
#pragma unroll
                    for (int a = 0; a < 3; ++a)
                        rb[(RV + a) * CAP + r] *= m;
#pragma unroll
                    for (int q = 0; q < 6; ++q)
                        rb[(RS + q) * CAP + r] *= V;
                }
                if (pt == 0)
                    desc_s[b] = make_int4(Q, it_lvl[i], (it_last[i] ? 1 : 0) | (i == nit - 1 ? 2 : 0), 0);
                mbar_arrive(&bar_full[b]); // release: records, counts and descriptor
                em_prev2 = em_prev1;
                em_prev1 = (it_last[i] ? 1 : 0) + (i == nit - 1 ? 2 : 0);
                mark(4);
            }
            if (done)
                break;
            named_bar(2, S::PROD); // every producer has read it_* / blk_s before they are rewritten
        }
        if constexpr (CLK)
            if (pt == 0 && blockIdx.x < 4)
                printf("ws-prod cta %d blocklist %lld wait_empty %lld issue %lld landed %lld convert %lld\n", blockIdx.x,
                       ck[0], ck[1], ck[2], ck[3], ck[4]);
        if (wq && pt == 0) { // the work counter pair resets after the last CTA (wq_finish)
            __threadfence();
            if (atomicAdd(wq + 1, 1) == int(gridDim.x) - 1) {
                atomicExch(wq, 0);
                atomicExch(wq + 1, 0);
            }
        }
        return;
    }

    // ================= consumers (k_p2g_pipe3's narrow lane mapping) =================
    if constexpr (S::REALLOC)
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(S::CONS_REGS));
    const int grp = NG > 1 ? tid / 192 : 0; // warp-uniform
    const int lt = tid - 192 * grp;
    const int gfb = S::P3::fb(grp), gfn = S::P3::fb(grp + 1) - gfb;
    const int bc = lt / 3, o0 = lt % 3;
    const bool mid = o0 == 1;
    const T xoff = o0 == 0 ? T(1.5) : (o0 == 1 ? T(1) : T(0.5)); // h = fx - xoff (bspline.hpp:94-99)
    const int bc0 = bc >> C::LOGB, bc1 = bc & (B - 1);
    const int lane = tid & 31;
    T acc[NO1][3][NA];
#pragma unroll
    for (int a = 0; a < NO1; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int f = 0; f < NA; ++f)
                acc[a][k][f] = T(0);
    int ne = 0; // slot buffers filled so far
    // node plane z of block Q is final in acc[.][0]: write it to a slot buffer and roll the window;
    // the 9-source sums follow (PRED: by the producers, here: by the consumers)
    auto emit = [&](int z, int Q) {
        const int sb = S::NSLOT == 2 ? ne & 1 : 0, u = ne >> 1;
        if constexpr (S::PRED) {
            if (u > 0) // the producers have summed this buffer's previous plane
                mbar_wait(&sl_empty[sb], (u - 1) & 1);
        } else {
            named_bar(1, CONS); // the previous sums are done reading the slots
        }
        T* sl = slots + sb * S::SLOT;
#pragma unroll
        for (int o1 = 0; o1 < NO1; ++o1) {
            const int ncol = (bc0 + o0) * TE + bc1 + o1;
#pragma unroll
            for (int f = 0; f < NA; ++f) {
                if (f < gfn)
                    sl[slot3(ncol, o0 * 3 + o1, gfb + f)] = acc[o1][0][f];
                acc[o1][0][f] = acc[o1][1][f];
                acc[o1][1][f] = acc[o1][2][f];
                acc[o1][2][f] = T(0);
            }
        }
        if constexpr (S::PRED) {
            if (tid == 0)
                em_s[sb] = make_int2(Q, z);
            __syncwarp();
            if (lane == 0)
                mbar_arrive(&sl_full[sb]);
        } else {
            named_bar(1, CONS); // slots complete
            T* part = partials + (size_t)Q * NF * C::TN;
            for (int t = tid; t < C::NCOL * NF; t += CONS) {
                const int c = t / NF, f = t - c * NF;
                const int n0 = c / TE, n1 = c - n0 * TE;
                T sum = T(0);
#pragma unroll
                for (int q = 0; q < NSRC; ++q) {
                    const int b0 = n0 - q / 3, b1 = n1 - q % 3;
                    if (b0 >= 0 && b0 < B && b1 >= 0 && b1 < B)
                        sum += sl[slot3(c, q, f)];
                }
                part[f * C::TN + ptile<3>(z, c)] = sum;
            }
        }
        ++ne;
    };
    for (int j = 0;; ++j) {
        const int b = j & 1;
        mark(5);
        mbar_wait(&bar_full[b], (j >> 1) & 1);
        mark(0);
        const int4 d = desc_s[b];
        if (d.z & 4)
            break;
        int kb, ke; // this column's records (lane l of each warp scans columns 2l, 2l+1)
        {
            const int* cnt = cnt_s[b];
            const int c0 = cnt[2 * lane], c1 = cnt[2 * lane + 1];
            int v = c0 + c1;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, v, dd);
                if (lane >= dd)
                    v += t;
            }
            const int excl = v - c0 - c1;
            const int src = bc >> 1;
            const int e = __shfl_sync(0xffffffffu, excl, src);
            const int a0 = __shfl_sync(0xffffffffu, c0, src);
            const int a1 = __shfl_sync(0xffffffffu, c1, src);
            kb = (bc & 1) ? e + a0 : e;
            ke = kb + ((bc & 1) ? a1 : a0);
        }
        const T* R = raw + b * NRAW * CAP;
#if WS_PREFETCH_REC
        // the next record is loaded into registers while this one is marched (the visit reads its
        // fields from the register copy: same values, same expressions)
        T nx[NRAW];
        auto load_rec = [&](int kk) {
            const int k = rsw(kk);
#pragma unroll
            for (int f = 0; f < NRAW; ++f)
                if (f != RVOL) // folded into sigma by the producers
                    nx[f] = R[f * CAP + k];
        };
        if (kb < ke)
            load_rec(kb);
#endif
        for (int k0 = kb; k0 < ke; ++k0) {
#if WS_PREFETCH_REC
            T cr[NRAW];
#pragma unroll
            for (int f = 0; f < NRAW; ++f)
                cr[f] = f != RVOL ? nx[f] : T(0);
            if (k0 + 1 < ke)
                load_rec(k0 + 1);
            const T* RR = cr;
            constexpr int CAPR = 1;
            const int k = 0;
#else
            const T* RR = R;
            constexpr int CAPR = CAP;
            const int k = rsw(k0);
#endif
            T f[3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
                f[a] = RR[(RX + a) * CAPR + k];
            T wx, dwx, wy[NO1], dwy[NO1], wz[3], dwz[3];
            {
                const T h = f[0] - xoff;
                const T hh = h * h;
                wx = mid ? T(0.75) - hh : T(0.5) * hh;
                dwx = (mid ? -T(2) * h : h) * sc.inv_dh;
            }
#pragma unroll
            for (int i1 = 0; i1 < NO1; ++i1)
                quad_w<T>(f[1], i1, sc.inv_dh, wy[i1], dwy[i1]);
#pragma unroll
            for (int q = 0; q < 3; ++q)
                quad_w<T>(f[2], q, sc.inv_dh, wz[q], dwz[q]);
            if (grp == 0)
                p2g_visit<S::P3::fb(0), S::P3::fb(1)>(acc, wx, dwx, wy, dwy, wz, dwz, RR, k, CAPR);
            else if constexpr (NG > 1)
                p2g_visit<S::P3::fb(1), S::P3::fb(2)>(acc, wx, dwx, wy, dwy, wz, dwz, RR, k, CAPR);
        }
        __syncwarp();
        if (lane == 0)
            mbar_arrive(&bar_empty[b]); // this warp is done with the buffer
        mark(1);
        if (d.z & 1)
            emit(d.y, d.x);
        if (d.z & 2) {
            emit(B, d.x);
            emit(B + 1, d.x);
        }
        mark(2);
    }
    if constexpr (CLK)
        if (tid == 0 && blockIdx.x < 4)
            printf("ws-cons cta %d wait_full %lld march %lld emit %lld\n", blockIdx.x, ck[0], ck[1], ck[2]);
}

// 3-D P2G, lane-per-stencil-offset (PIC / FLIP / blend). A warp owns 4 particle columns of
// the block; lane (i, j, k) < 27 owns the stencil offset (i, j, k) and accumulates the column's
// contributions to node (x + i, y + j, z + k) for the current base level z in 7 registers per
// column. After a level, lanes k = 0 hold the column's finished node-plane z; the window rolls by
// one lane (__shfl_down). Each staged particle is converted once per level into its weights,
// m v and V sigma (shared memory, read by broadcast LDS.128), so a lane-particle costs ~20 FP64
// instructions. 16 warps per SM with 7 x 4 accumulators each (vs 6 warps holding 63 in
// k_p2g_pipe3) hide the FP64 latency. Same partial tiles and fixed combine order as pipe3.
// MEASURED (C4 f64, ncu): 0.88-0.91 ms vs pipe3's 0.58 ms -- shared-memory bound: 16 broadcast
// LDS.64 per lane-particle cost ~2 wavefronts each (154M wavefronts, L1 74% busy). Kept for A/B
// (MPM_P2G_IMPL=lanes3); a node per lane is too little reuse of each particle read.
template <class T> struct Lane3Cfg {
    static constexpr int THREADS = 512, WARPS = THREADS / 32, NBC = 64, CPW = NBC / WARPS;
    static constexpr int CAP = 384, NRAW = 14, ND = 28, NSRC = 9, MAXIT = 64;
    static constexpr size_t SMEM_RAW = sizeof(T) * NRAW * CAP;
    static constexpr size_t SMEM_DER = sizeof(T) * ND * CAP;
    static constexpr size_t SMEM_PK = sizeof(int) * 3 * 2 * CAP;
    static constexpr size_t SMEM_SLOT = sizeof(T) * Cfg<3>::NCOL * NSRC * Cfg<3>::NF;
    static constexpr size_t SMEM = SMEM_RAW + SMEM_DER + SMEM_PK + SMEM_SLOT;
};

template <class T>
__global__ void __launch_bounds__(Lane3Cfg<T>::THREADS, 1)
    k_p2g_lanes3(DevScene<T, 3> sc, PBuf<T, 3> P, const int* __restrict__ perm, const int* __restrict__ keys,
                 const int* __restrict__ bstart, const int* __restrict__ bend, const int* __restrict__ lstart,
                 const int* __restrict__ occ, const int* __restrict__ n_occ, T* __restrict__ partials, DevStatus* st)
{
    pdl_wait();
    pdl_trigger();
    using C = Cfg<3>;
    using S = Lane3Cfg<T>;
    using PL = PLay<3>;
    constexpr int B = C::B, TE = C::TE, NF = C::NF, CAP = S::CAP, NBC = S::NBC, NSRC = S::NSRC, NRAW = S::NRAW,
                  ND = S::ND, CPW = S::CPW, NT = S::THREADS;
    // derived record per particle (ND doubles): (w, dw) pairs x0..2 | y0..2 | z0..2, m, m v, V sigma
    constexpr int DX = 0, DY = 6, DZ = 12, DM = 18, DS = 22;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* raw = reinterpret_cast<T*>(smem_raw);                                           // [NRAW][CAP]
    T* der = reinterpret_cast<T*>(smem_raw + S::SMEM_RAW);                             // [CAP][ND]
    int* pk = reinterpret_cast<int*>(smem_raw + S::SMEM_RAW + S::SMEM_DER);            // [3][2][CAP]
    T* slots = reinterpret_cast<T*>(smem_raw + S::SMEM_RAW + S::SMEM_DER + S::SMEM_PK); // [NCOL][NSRC][NF]
    __shared__ int it_start[S::MAXIT], it_len[S::MAXIT], it_lvl[S::MAXIT], it_last[S::MAXIT];
    __shared__ int nit_s, ccount[NBC], cst[NBC + 1];
    if (st->abort)
        return;
    const int nocc = *n_occ;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool act = lane < 27;
    const int li = lane / 9, lj = (lane / 3) % 3, lk = lane % 3; // this lane's stencil offset
    const long long SI = P.S;

    for (int w = blockIdx.x; w < nocc; w += gridDim.x) {
        const int Q = occ[w];
        const int s0 = bstart[Q], s1 = bend[Q];
        __syncthreads();
        if (tid == 0) { // level starts (suffix minimum) -> work items of <= CAP particles
            int lv[B + 1];
            int nxt = s1;
            lv[B] = s1 - s0;
            for (int z = B - 1; z >= 0; --z) {
                const int v = lstart[Q * (B + 1) + z];
                nxt = (v >= s0 && v < s1) ? v : nxt;
                lv[z] = nxt - s0;
            }
            int k = 0;
            for (int z = 0; z < B; ++z) {
                const int nl = lv[z + 1] - lv[z];
                const int nch = nl > 0 ? (nl + CAP - 1) / CAP : 1;
                for (int c = 0; c < nch; ++c) {
                    if (k < S::MAXIT) {
                        it_start[k] = lv[z] + c * CAP;
                        it_len[k] = min(CAP, nl - c * CAP);
                        it_lvl[k] = z;
                        it_last[k] = c == nch - 1;
                    }
                    ++k;
                }
            }
            if (k > S::MAXIT) { // pathological compression: refuse loudly
                st->far_flag = 1;
                st->abort = 1;
                k = 0;
            }
            nit_s = k;
        }
        if (tid < NBC)
            ccount[tid] = 0;
        __syncthreads();
        const int nit = nit_s;
        auto issue_pk = [&](int j) {
            int* dp = pk + (j % 3) * 2 * CAP;
            const int b = s0 + it_start[j];
            for (int r = tid; r < it_len[j]; r += NT) {
                cp_async4(dp + r, perm + b + r);
                cp_async4(dp + CAP + r, keys + b + r);
            }
        };
        // raw rows: x0..2 v0..2 m V sigma0..5 (PLay fields 0..7 and SIG..SIG+5; rho, eps skipped)
        constexpr int RX = 0, RV = 3, RM = 6, RVOL = 7, RS = 8;
        static_assert(PL::M == RM && PL::VOL == RVOL && PL::SIG == RS + 2 && RS + 6 == NRAW, "raw row map");
        auto issue_raw = [&](int j) {
            const int* pp = pk + (j % 3) * 2 * CAP;
            for (int r = tid; r < it_len[j]; r += NT) {
                const T* q = P.base + pp[r];
#pragma unroll
                for (int f = 0; f < NRAW; ++f)
                    cp_async_t<T>(raw + f * CAP + r, q + (f < RS ? f : f + 2) * SI);
            }
        };
        if (nit > 0)
            issue_pk(0);
        if (nit > 1)
            issue_pk(1);
        cp_async_commit();
        cp_async_wait_all();
        __syncthreads();
        if (nit > 0)
            issue_raw(0);
        cp_async_commit();

        T* part = partials + (size_t)Q * NF * C::TN;
        T acc[CPW][NF];
#pragma unroll
        for (int c = 0; c < CPW; ++c)
#pragma unroll
            for (int f = 0; f < NF; ++f)
                acc[c][f] = T(0);

        // lanes k = 0 publish node plane z of their columns, the window rolls, columns are combined
        auto emit = [&](int z) {
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const int bc = warp + c * S::WARPS;
                const int ncol = ((bc >> 3) + li) * TE + (bc & 7) + lj;
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    if (act && lk == 0)
                        slots[(ncol * NSRC + li * 3 + lj) * NF + f] = acc[c][f];
                    const T nx = __shfl_down_sync(0xffffffffu, acc[c][f], 1);
                    acc[c][f] = (lk < 2 && act) ? nx : T(0);
                }
            }
            __syncthreads();
            for (int t = tid; t < C::NCOL * NF; t += NT) {
                const int cidx = t / NF, f = t - cidx * NF;
                const int n0 = cidx / TE, n1 = cidx - n0 * TE;
                T sum = T(0);
#pragma unroll
                for (int q = 0; q < NSRC; ++q) {
                    const int b0 = n0 - q / 3, b1 = n1 - q % 3;
                    if (b0 >= 0 && b0 < B && b1 >= 0 && b1 < B)
                        sum += slots[(cidx * NSRC + q) * NF + f];
                }
                part[f * C::TN + ptile<3>(z, cidx)] = sum;
            }
            __syncthreads();
        };

        for (int j = 0; j < nit; ++j) {
            cp_async_wait_all();
            __syncthreads(); // raw(j), pk(j + 1) landed for every thread
            const int len = it_len[j];
            const int* col = pk + (j % 3) * 2 * CAP + CAP;
            // convert each staged particle once: weights (bspline.hpp:94-108), m v, V sigma
            for (int r = tid; r < len; r += NT) {
                atomicAdd(&ccount[col[r] & (NBC - 1)], 1);
                T* d = der + r * ND;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const T u = (raw[(RX + a) * CAP + r] - sc.origin[a]) * sc.inv_dh;
                    const T fx = u - dfloor<T>(u - T(0.5));
                    const T h0 = T(1.5) - fx, h1 = fx - T(1), h2 = fx - T(0.5);
                    d[a * 6 + 0] = T(0.5) * h0 * h0;
                    d[a * 6 + 1] = -h0 * sc.inv_dh;
                    d[a * 6 + 2] = T(0.75) - h1 * h1;
                    d[a * 6 + 3] = -T(2) * h1 * sc.inv_dh;
                    d[a * 6 + 4] = T(0.5) * h2 * h2;
                    d[a * 6 + 5] = h2 * sc.inv_dh;
                }
                const T m = raw[RM * CAP + r], V = raw[RVOL * CAP + r];
                d[DM] = m;
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    d[DM + 1 + a] = m * raw[(RV + a) * CAP + r];
#pragma unroll
                for (int q = 0; q < 6; ++q)
                    d[DS + q] = V * raw[(RS + q) * CAP + r];
            }
            __syncthreads(); // derived ready, raw free, counts complete
            if (j + 1 < nit)
                issue_raw(j + 1);
            if (j + 2 < nit)
                issue_pk(j + 2);
            cp_async_commit();
            if (tid < 32) {
                const int c0 = ccount[2 * tid], c1 = ccount[2 * tid + 1];
                int v = c0 + c1;
#pragma unroll
                for (int dd = 1; dd < 32; dd <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, v, dd);
                    if (tid >= dd)
                        v += t;
                }
                const int excl = v - c0 - c1;
                cst[2 * tid] = excl;
                cst[2 * tid + 1] = excl + c0;
                if (tid == 31)
                    cst[NBC] = v;
                ccount[2 * tid] = 0;
                ccount[2 * tid + 1] = 0;
            }
            __syncthreads();
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const int bc = warp + c * S::WARPS;
                const int kb = cst[bc], ke = cst[bc + 1];
                for (int k = kb; k < ke; ++k) {
                    const T* d = der + k * ND;
                    // broadcast reads: (w, dw) of this lane's x, y, z offsets; m, m v; V sigma
                    const T wx = d[DX + 2 * li], dwx = d[DX + 2 * li + 1];
                    const T wy = d[DY + 2 * lj], dwy = d[DY + 2 * lj + 1];
                    const T wz = d[DZ + 2 * lk], dwz = d[DZ + 2 * lk + 1];
                    const T m = d[DM], mv0 = d[DM + 1], mv1 = d[DM + 2], mv2 = d[DM + 3];
                    const T s00 = d[DS + 0], s11 = d[DS + 1], s22 = d[DS + 2], s01 = d[DS + 3], s02 = d[DS + 4],
                            s12 = d[DS + 5];
                    const T wxy = wx * wy;
                    const T wgt = wxy * wz;
                    const T g0 = (dwx * wy) * wz, g1 = (wx * dwy) * wz, g2 = wxy * dwz; // grad phi
                    acc[c][0] += m * wgt;
                    acc[c][1] += mv0 * wgt;
                    acc[c][2] += mv1 * wgt;
                    acc[c][3] += mv2 * wgt;
                    // f -= V sigma grad phi (transfer.hpp:55-62); gravity is added per node in k_grid
                    acc[c][4] = acc[c][4] - s00 * g0 - s01 * g1 - s02 * g2;
                    acc[c][5] = acc[c][5] - s01 * g0 - s11 * g1 - s12 * g2;
                    acc[c][6] = acc[c][6] - s02 * g0 - s12 * g1 - s22 * g2;
                }
            }
            if (it_last[j]) {
                __syncthreads();
                emit(it_lvl[j]);
            }
        }
        cp_async_wait_all();
        __syncthreads();
        emit(B);
        emit(B + 1);
    }
}

// ---------------------------------------------------------------------------------------
// grid update: combine partial tiles, momentum update, boundary/contact corrections.
// G_NOGRAV: sum without the g m_i term (slab halo sums first); G_GRAV: add g m_i to a stored
// grid; G_ZEROV: massless nodes of a stored grid get v = v_old = 0 (as after a fresh sum)
// G_BANDONLY / G_INTERIOR: only the halo-band nodes / only the others (slab decomposition)
enum GridMode {
    G_SUM = 1, G_MOM = 2, G_CORR = 4, G_STORE = 8, G_NOGRAV = 16, G_GRAV = 32, G_ZEROV = 64, G_BANDONLY = 128,
    G_INTERIOR = 256
};
template <class T, int D> __device__ __forceinline__ bool in_band(const DevScene<T, D>& sc, int x)
{
    return (unsigned)(x - sc.band_lo) < 2u || (unsigned)(x - sc.band_hi) < 2u;
}

// collect_node_corrections + apply_node_correction (contact.hpp:141-224), fixed order
template <class T, int D>
__device__ __forceinline__ void node_corrections(const DevScene<T, D>& sc, const int* n, T* v)
{
    // plain walls in wall order (slip zeroes the axis component, no-slip/fixed zero v)
#pragma unroll
    for (int w = 0; w < 2 * D; ++w) {
        const int kind = sc.wall_kind[w];
        if (kind == 3)
            continue;
        const int a = w / 2;
        const bool in = (w % 2 == 0) ? n[a] < sc.band : n[a] > sc.cells[a] - sc.band;
        if (!in)
            continue;
        if (kind == 0)
            v[a] = T(0);
        else {
#pragma unroll
            for (int b = 0; b < D; ++b)
                v[b] = T(0);
        }
    }
    if (sc.n_obst > 0) {
        T xp[D];
#pragma unroll
        for (int a = 0; a < D; ++a)
            xp[a] = sc.origin[a] + T(n[a]) * sc.dh;
        for (int ob = 0; ob < sc.n_obst; ++ob) {
            bool inside = true;
#pragma unroll
            for (int a = 0; a < D; ++a)
                inside &= !(xp[a] < sc.obst[ob][a] || xp[a] > sc.obst[ob][D + a]);
            if (!inside)
                continue;
            int best_a = 0, best_s = 0;
            T best = T(0);
            bool first = true;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                T dlo = xp[a] - sc.obst[ob][a];
                T dhi = sc.obst[ob][D + a] - xp[a];
                if (first || dlo < best) {
                    best = dlo;
                    best_a = a;
                    best_s = 0;
                    first = false;
                }
                if (dhi < best) {
                    best = dhi;
                    best_a = a;
                    best_s = 1;
                }
            }
            const T nrm = best_s == 0 ? T(-1) : T(1);
            const T vn = v[best_a] * nrm; // v . n with a unit axis normal
            if (vn < T(0)) {
#pragma unroll
                for (int a = 0; a < D; ++a)
                    v[a] = v[a] - vn * (a == best_a ? nrm : T(0));
            }
        }
    }
    // Coulomb walls (contact.hpp:40-51, 336-351)
#pragma unroll
    for (int w = 0; w < 2 * D; ++w) {
        if (sc.wall_kind[w] != 3)
            continue;
        const int a = w / 2;
        const bool in = (w % 2 == 0) ? n[a] < sc.band : n[a] > sc.cells[a] - sc.band;
        if (!in)
            continue;
        const int seg_axis = a == 0 ? 1 : 0;
        const T coord = sc.origin[seg_axis] + T(n[seg_axis]) * sc.dh;
        const int ns = sc.n_fric[w];
        const T len = (T(sc.cells[seg_axis]) * sc.dh) / T(ns);
        int k = int(ceil(double((coord - sc.origin[seg_axis]) / len))) - 1;
        k = k < 0 ? 0 : (k > ns - 1 ? ns - 1 : k);
        const T mu = sc.fric[sc.fric_off[w] + k];
        const T nrm = (w % 2 == 0) ? T(-1) : T(1);
        T vn = T(0);
#pragma unroll
        for (int b = 0; b < D; ++b)
            vn += v[b] * (b == a ? nrm : T(0));
        if (vn <= T(0))
            continue;
        T t[D], t2 = T(0);
#pragma unroll
        for (int b = 0; b < D; ++b) {
            t[b] = v[b] - vn * (b == a ? nrm : T(0));
            t2 += t[b] * t[b];
        }
        const T tn = dsqrt<T>(t2);
        if (tn <= mu * vn) {
#pragma unroll
            for (int b = 0; b < D; ++b)
                v[b] = T(0);
        } else {
            const T s = mu * vn / tn;
#pragma unroll
            for (int b = 0; b < D; ++b)
                v[b] = t[b] - s * t[b];
        }
    }
}

template <class T, int D, int MODE>
__global__ void __launch_bounds__(Cfg<D>::NB) k_grid(DevScene<T, D> sc, GBuf<T, D> G, const T* __restrict__ partials,
                                                     const int* __restrict__ bstart, const int* __restrict__ act,
                                                     const int* __restrict__ n_act, DevStatus* st)
{
    pdl_wait();
    pdl_trigger();
    using C = Cfg<D>;
    if (st->abort)
        return;
    const int nact = *n_act;
    const int tid = threadIdx.x;
    int lc[D];
    {
        int t = tid;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
            lc[a] = t & (C::B - 1);
            t >>= C::LOGB;
        }
    }
    unsigned long long nact_nodes = 0;
    // the (up to 2^D) source tiles of the current node block, resolved once per CTA: the per-node
    // loop then issues its tile loads without a dependent bstart load per source
    __shared__ const T* s_part[1 << D];
    for (int w = blockIdx.x; w < nact; w += gridDim.x) {
        const int q = act[w];
        int qc[D], n[D];
        block_coords<D>(q, sc.nnb, qc);
        if constexpr ((MODE & G_BANDONLY) != 0) { // whole node blocks off the bands: nothing to do
            const int x0 = qc[0] * C::B;
            if (!((sc.band_lo + 1 >= x0 && sc.band_lo < x0 + C::B) || (sc.band_hi + 1 >= x0 && sc.band_hi < x0 + C::B)))
                continue;
        }
        if (MODE & G_SUM) {
            __syncthreads(); // the previous node block's readers are done
            if (tid < (1 << D)) {
                int Qid = 0;
                bool ok = true;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    const int Qa = qc[a] - ((tid >> (D - 1 - a)) & 1);
                    ok &= Qa >= 0 && Qa < sc.nb[a];
                    Qid = Qid * sc.nb[a] + Qa;
                }
                s_part[tid] = ok && bstart[Qid] >= 0 ? partials + (size_t)Qid * C::NF * C::TN : nullptr;
            }
            __syncthreads();
        }
        bool inside = true;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            n[a] = qc[a] * C::B + lc[a];
            inside &= n[a] <= sc.cells[a];
        }
        if constexpr ((MODE & G_BANDONLY) != 0) {
            if (!in_band<T, D>(sc, n[0]))
                continue;
        }
        if constexpr ((MODE & G_INTERIOR) != 0) {
            if (in_band<T, D>(sc, n[0]))
                continue;
        }
        const size_t gi = (size_t)q * C::NB + tid;
        T m = T(0), p[D], f[D], v[D], vold[D];
#pragma unroll
        for (int a = 0; a < D; ++a)
            p[a] = f[a] = v[a] = vold[a] = T(0);
        if (MODE & G_SUM) {
            // fixed order over source blocks Q = q - s, s lexicographic in {0,1}^D
#pragma unroll
            for (int s = 0; s < (1 << D); ++s) {
                const T* base = s_part[s];
                bool ok = base != nullptr;
                // tile index: last axis slowest, columns row-major over the other axes
                int colx = 0, z = 0;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    const int sa = (s >> (D - 1 - a)) & 1;
                    const int t = lc[a] + sa * C::B; // n[a] - (qc[a] - sa) B
                    ok &= t < C::TE;
                    if (a == D - 1)
                        z = t;
                    else
                        colx = colx * C::TE + t;
                }
                if (!ok)
                    continue;
                const T* part = base + ptile<D>(z, colx);
                m += part[0];
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    p[a] += part[(1 + a) * C::TN];
                    f[a] += part[(1 + D + a) * C::TN];
                }
            }
            // sum_p phi m g = g m_i (transfer.hpp:62, gravity term factored out of the scatter)
            if (!(MODE & G_NOGRAV)) {
#pragma unroll
                for (int a = 0; a < D; ++a)
                    f[a] += sc.gravity[a] * m;
            }
        } else {
            m = G.m[gi];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                p[a] = G.p[a][gi];
                f[a] = G.f[a][gi];
                v[a] = G.v[a][gi];
                vold[a] = G.vold[a][gi];
            }
            if (MODE & G_GRAV) {
#pragma unroll
                for (int a = 0; a < D; ++a)
                    f[a] += sc.gravity[a] * m;
            }
        }
        if (MODE & G_MOM) {
            if (m > sc.mass_eps) {
                const T s = sc.dt / m;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    vold[a] = p[a] / m;
                    v[a] = vold[a] + s * f[a];
                }
                nact_nodes += inside;
            } else if (MODE & (G_SUM | G_ZEROV)) {
#pragma unroll
                for (int a = 0; a < D; ++a)
                    v[a] = vold[a] = T(0);
            }
        }
        if ((MODE & G_CORR) && inside)
            node_corrections<T, D>(sc, n, v);
        if (!inside) {
            m = T(0);
#pragma unroll
            for (int a = 0; a < D; ++a)
                p[a] = f[a] = v[a] = vold[a] = T(0);
        }
        if (MODE & G_STORE) {
            G.m[gi] = m;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                G.p[a][gi] = p[a];
                G.f[a][gi] = f[a];
            }
        }
#pragma unroll
        for (int a = 0; a < D; ++a) {
            G.v[a][gi] = v[a];
            G.vold[a][gi] = vold[a];
        }
    }
    if (MODE & G_MOM) {
        // warp-aggregated count of active nodes (diagnostic only)
        for (int o = 16; o > 0; o >>= 1)
            nact_nodes += __shfl_down_sync(0xffffffffu, nact_nodes, o);
        if ((tid & 31) == 0 && nact_nodes)
            atomicAdd(&st->active_nodes, nact_nodes);
    }
}

// ---------------------------------------------------------------------------------------
// G2P (+ constitutive): CTA per occupied particle block, node tile (v, v_old) in smem.
// P_NOGV: grad v is not stored (a step inside an advance() call whose scheme never reads the
// stored grad v -- FLIP / PIC / blend without F tracking; the call's last step stores it)
enum G2PFlags { P_CONSTIT = 1, P_GUARD = 2, P_NOGV = 4 };

// migration export buffers (slab mode): one record of `rec` scalars + the pid per mover
template <class T> struct MigBuf {
    int on, cap, rec;
    T* lo;
    T* hi;
    int* lo_pid;
    int* hi_pid;
    int* lo_slot; // the vacated output slot of each export (the decomposed adjoint returns
    int* hi_slot; // the particle's cotangent row there)
};

// per-thread staging of a particle's G2P inputs (x, v, m, V, rho, eps, [szz], sigma, [F]).
// Tried: the node tile through cp.async with zero fill (all loads in flight, v - v_old formed after
// the wait): MEASURED C4 f64 0.342 -> 0.345 ms, f32 0.201 -> 0.196; not kept.
template <class T, int D, bool TRACKF> struct G2PStage {
    static constexpr int NSF = 2 * D + 4 + (D == 2 ? 1 : 0) + Cfg<D>::NS + (TRACKF ? D * D : 0);
    static constexpr int THREADS = 256;
    static constexpr size_t TILE = sizeof(T) * 2 * D * Cfg<D>::TN;
    static constexpr size_t SMEM = TILE + sizeof(T) * 2 * NSF * THREADS + sizeof(int) * 2 * THREADS; // tile + 2 slots (+ pid)
};

// ABL != 0: timing ablation only (1 skip the node-tile load, 2 skip the constitutive update,
// 4 skip the gather arithmetic, 8 none), launched in front of the real kernel by -DG2P_ABL builds
template <class T, int D, int FLAGS, bool APIC, bool TRACKF, int ABL = 0>
__global__ void __launch_bounds__(256, 2) k_g2p(DevScene<T, D> sc, PBuf<T, D> Pin, PBuf<T, D> Pout,
                                             GBuf<T, D> G, const int* __restrict__ perm,
                                             const int* __restrict__ bstart, const int* __restrict__ bend,
                                             const int* __restrict__ occ, const int* __restrict__ n_occ,
                                             int* __restrict__ keys_out, DevStatus* st, MigBuf<T> MG,
                                             int* __restrict__ wq)
{
    pdl_wait();
    pdl_trigger();
    using C = Cfg<D>;
    using SG = G2PStage<T, D, TRACKF>;
    constexpr int TE = C::TE, TN = C::TN, NSF = SG::NSF, NT = SG::THREADS;
    extern __shared__ unsigned char smem_raw[];
    T* tile = reinterpret_cast<T*>(smem_raw); // [2D][TN]: v[0..D), v - vold[0..D) (formed once per node)
    T* stg = tile + 2 * D * TN;               // [2][NSF][NT]: this thread's column only
    int* stg_pid = reinterpret_cast<int*>(stg + 2 * NSF * NT); // [2][NT]
    __shared__ int w_s; // next list entry (work counter, kernels_util.cuh)
    const int nocc = st->abort ? 0 : *n_occ; // every CTA still passes wq_finish
    if (threadIdx.x == 0)
        w_s = wq_first(wq);
    const T alpha = sc.alpha;
    const int tid = threadIdx.x;
    // cp.async of particle `src`'s inputs into slot `slot` (each thread its own column: no barrier)
    using PL = PLay<D>;
    const long long SI = Pin.S, SO = Pout.S;
    auto issue = [&](int slot, int src) {
        T* b = stg + slot * NSF * NT + tid;
        const T* q = Pin.base + src; // field k at q + k * SI (PLay order: x v m V rho eps [szz] sigma)
#pragma unroll
        for (int f = 0; f < PL::SIG + C::NS; ++f)
            cp_async_t<T>(b + f * NT, q + f * SI);
        if constexpr (TRACKF) {
#pragma unroll
            for (int k = 0; k < D * D; ++k)
                cp_async_t<T>(b + (PL::SIG + C::NS + k) * NT, q + (PL::F + k) * SI);
        }
        cp_async4(stg_pid + slot * NT + tid, Pin.pid + src); // its id too: no exposed load before the stores
    };
    static_assert(PL::SIG + C::NS + (TRACKF ? D * D : 0) == NSF, "staging mirrors the PLay field order");
    for (;;) {
        cp_async_wait_all();
        __syncthreads(); // w_s published; the previous block's tile readers are done
        const int w = w_s;
        if (w >= nocc)
            break;
        const int Q = occ[w];
        const int s0 = bstart[Q], s1 = bend[Q];
        int qc[D];
        block_coords<D>(Q, sc.nb, qc);
        // first particle of this thread in flight while the node tile loads
        int i0 = s0 + tid;
        int src_a = i0 < s1 ? perm[i0] : -1;                    // particle i0
        int src_b = i0 + NT < s1 ? perm[i0 + NT] : -1;          // particle i0 + NT (prefetched index)
        if (src_a >= 0)
            issue(0, src_a);
        cp_async_commit();
        for (int t = threadIdx.x; t < TN; t += blockDim.x) {
            int tl[D], rem = t, nid = 0, loc = 0;
            bool ok = true;
#pragma unroll
            for (int a = D - 1; a >= 0; --a) {
                tl[a] = rem % TE;
                rem /= TE;
            }
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const int nn = qc[a] * C::B + tl[a];
                const int qb = nn >> C::LOGB;
                ok &= qb < sc.nnb[a];
                nid = nid * sc.nnb[a] + qb;
                loc = (loc << C::LOGB) | (nn & (C::B - 1));
            }
            const size_t gi = (size_t)nid * C::NB + loc;
            if (ABL & 1)
                ok = false;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const T vn = ok ? G.v[a][gi] : T(0), vo = ok ? G.vold[a][gi] : T(0);
                tile[a * TN + t] = vn;
                tile[(D + a) * TN + t] = vn - vo;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) // every thread read w_s before the barrier above
            w_s = wq_next(wq, w);
        int slot = 0;
        for (int i = i0; i < s1; i += NT) {
            // keep the next particle's fields and the one after's index in flight
            src_a = src_b;
            src_b = i + 2 * NT < s1 ? perm[i + 2 * NT] : -1;
            if (src_a >= 0)
                issue(slot ^ 1, src_a);
            cp_async_commit();
            asm volatile("cp.async.wait_group 1;\n" ::: "memory"); // this thread's slot `slot` landed
            const T* sb = stg + slot * NSF * NT + tid;
            const int pid = stg_pid[slot * NT + tid];
            slot ^= 1;
            T x[D], v[D];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                x[a] = sb[a * NT];
                v[a] = sb[(D + a) * NT];
            }
            T w[D][3], dw[D][3];
            int tb[D];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                axis_weights<T, D>(x[a], sc.origin[a], sc.inv_dh, w[a], dw[a]);
                const int b = int(dfloor<T>((x[a] - sc.origin[a]) * sc.inv_dh - T(0.5)));
                tb[a] = b - qc[a] * C::B;
            }
            T vpic[D], vinc[D], L[D * D], Bm[D * D];
#pragma unroll
            for (int a = 0; a < D; ++a)
                vpic[a] = vinc[a] = T(0);
#pragma unroll
            for (int k = 0; k < D * D; ++k)
                L[k] = Bm[k] = T(0);
            if constexpr (!APIC && !(ABL & 4)) {
                // tensor-product factorisation along the last axis: for each outer offset,
                // A = sum w_z v, Bz = sum dw_z v, Cd = sum w_z (v - v_old); then
                // v_pic += w_o A, v_inc += w_o Cd, grad v[:, a<d-1] += dw_o A, grad v[:, d-1] += w_o Bz
#pragma unroll
                for (int oo = 0; oo < C::NOFF / 3; ++oo) {
                    int o[D - 1 > 0 ? D - 1 : 1];
                    int kk = oo, t0 = 0;
#pragma unroll
                    for (int a = D - 2; a >= 0; --a) {
                        o[a] = kk % 3;
                        kk /= 3;
                    }
#pragma unroll
                    for (int a = 0; a < D - 1; ++a)
                        t0 = t0 * TE + tb[a] + o[a];
                    t0 = t0 * TE + tb[D - 1];
                    T A[D], Bz[D], Cd[D];
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        const T* va = tile + a * TN + t0;
                        const T* voa = tile + (D + a) * TN + t0;
                        const T v0 = va[0], v1 = va[1], v2 = va[2];
                        A[a] = w[D - 1][0] * v0 + w[D - 1][1] * v1 + w[D - 1][2] * v2;
                        Bz[a] = dw[D - 1][0] * v0 + dw[D - 1][1] * v1 + dw[D - 1][2] * v2;
                        Cd[a] = w[D - 1][0] * voa[0] + w[D - 1][1] * voa[1] + w[D - 1][2] * voa[2]; // voa: v - vold
                    }
                    T wo = T(1), po[D - 1 > 0 ? D - 1 : 1];
#pragma unroll
                    for (int a = 0; a < D - 1; ++a)
                        wo *= w[a][o[a]];
#pragma unroll
                    for (int a = 0; a < D - 1; ++a) {
                        T r = dw[a][o[a]];
#pragma unroll
                        for (int b = 0; b < D - 1; ++b)
                            if (b != a)
                                r *= w[b][o[b]];
                        po[a] = r;
                    }
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        vpic[a] += wo * A[a];
                        vinc[a] += wo * Cd[a];
#pragma unroll
                        for (int b = 0; b < D - 1; ++b)
                            L[a * D + b] += po[b] * A[a];
                        L[a * D + D - 1] += wo * Bz[a];
                    }
                }
            } else if constexpr (APIC) {
#pragma unroll
            for (int k = 0; k < C::NOFF; ++k) {
                int o[D];
                int kk = k, ti = 0;
#pragma unroll
                for (int a = D - 1; a >= 0; --a) {
                    o[a] = kk % 3;
                    kk /= 3;
                }
#pragma unroll
                for (int a = 0; a < D; ++a)
                    ti = ti * TE + tb[a] + o[a];
                T phi = T(1);
#pragma unroll
                for (int a = 0; a < D; ++a)
                    phi *= w[a][o[a]];
                T gw[D];
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    T r = dw[a][o[a]];
#pragma unroll
                    for (int b = 0; b < D; ++b)
                        if (b != a)
                            r *= w[b][o[b]];
                    gw[a] = r;
                }
                T nv[D];
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    nv[a] = tile[a * TN + ti];
                    const T ndv = tile[(D + a) * TN + ti]; // v - vold
                    vpic[a] += phi * nv[a];
                    vinc[a] += phi * ndv;
                }
#pragma unroll
                for (int a = 0; a < D; ++a)
#pragma unroll
                    for (int b = 0; b < D; ++b)
                        L[a * D + b] += nv[a] * gw[b];
                T r[D];
#pragma unroll
                for (int a = 0; a < D; ++a)
                    r[a] = (sc.origin[a] + T(qc[a] * C::B + tb[a] + o[a]) * sc.dh) - x[a];
#pragma unroll
                for (int a = 0; a < D; ++a)
#pragma unroll
                    for (int b = 0; b < D; ++b)
                        Bm[a * D + b] += phi * nv[a] * r[b];
            }
            }
            T xn[D], vn[D];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                vn[a] = alpha * (v[a] + vinc[a]) + (T(1) - alpha) * vpic[a];
                xn[a] = x[a] + sc.dt * vpic[a];
            }
            constexpr int FM = 2 * D, FS = 2 * D + 4 + (D == 2 ? 1 : 0);
            T m = sb[FM * NT], V = sb[(FM + 1) * NT], rho = sb[(FM + 2) * NT], eps = sb[(FM + 3) * NT];
            T szz = D == 2 ? sb[(FM + 4) * NT] : T(0);
            T sig[C::NS];
#pragma unroll
            for (int s = 0; s < C::NS; ++s)
                sig[s] = sb[(FS + s) * NT];
            T Fm[D * D];
            if constexpr (TRACKF) {
#pragma unroll
                for (int k = 0; k < D * D; ++k)
                    Fm[k] = sb[(FS + C::NS + k) * NT];
            }
            bool ok_den = true;
            if ((FLAGS & P_CONSTIT) && !(ABL & 2)) {
                ok_den = constitutive_particle<T, D>(sc, sig, szz, rho, V, eps, L);
                if constexpr (TRACKF) { // F <- (I + L dt) F (stepper.hpp:39-42)
                    T Fn[D * D];
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int b = 0; b < D; ++b) {
                            T s = T(0);
#pragma unroll
                            for (int k = 0; k < D; ++k)
                                s += ((a == k ? T(1) : T(0)) + L[a * D + k] * sc.dt) * Fm[k * D + b];
                            Fn[a * D + b] = s;
                        }
#pragma unroll
                    for (int k = 0; k < D * D; ++k)
                        Fm[k] = Fn[k];
                }
            }
            // write the new state at sorted slot i (field k at o + k * SO)
            T* o = Pout.base + i;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                o[(PL::X + a) * SO] = xn[a];
                o[(PL::V + a) * SO] = vn[a];
            }
            o[PL::M * SO] = m;
            o[PL::VOL * SO] = V;
            o[PL::RHO * SO] = rho;
            o[PL::EPS * SO] = eps;
            if (D == 2)
                o[PL::SZZ * SO] = szz;
#pragma unroll
            for (int s = 0; s < C::NS; ++s)
                o[(PL::SIG + s) * SO] = sig[s];
            if constexpr (!(FLAGS & P_NOGV)) {
#pragma unroll
                for (int k = 0; k < D * D; ++k)
                    o[(PL::GV + k) * SO] = L[k];
            }
            if constexpr (APIC) {
#pragma unroll
                for (int k = 0; k < D * D; ++k)
                    o[(PL::AFF + k) * SO] = Bm[k];
            }
            if constexpr (TRACKF) {
#pragma unroll
                for (int k = 0; k < D * D; ++k)
                    o[(PL::F + k) * SO] = Fm[k];
            }
            Pout.pid[i] = pid;
            if (!ok_den) {
                atomicMin(&st->den_pid, pid);
                st->den_flag = 1;
                st->abort = 1;
            }
            if (FLAGS & P_GUARD) { // ParticleSoA::all_finite (state.hpp:48-62)
                bool fin = finite_(V) && finite_(rho) && finite_(eps) && finite_(szz);
#pragma unroll
                for (int a = 0; a < D; ++a)
                    fin &= finite_(xn[a]) && finite_(vn[a]);
#pragma unroll
                for (int s = 0; s < C::NS; ++s)
                    fin &= finite_(sig[s]);
#pragma unroll
                for (int k = 0; k < D * D; ++k)
                    fin &= finite_(L[k]) && (!APIC || finite_(Bm[k]));
                if (!fin) {
                    st->nan_flag = 1;
                    st->abort = 1;
                }
            }
            int key;
            if (!cell_key<T, D>(sc, xn, key)) {
                key = KEY_OOD;
                atomicMin(&st->ood_pid, pid);
                st->ood_flag = 2;
                st->abort = 1;
            } else if (MG.on) {
                const int bx = int(dfloor<T>((xn[0] - sc.origin[0]) * sc.inv_dh - T(0.5)));
                if (bx < sc.slab_lo || bx >= sc.slab_hi) { // leaves the slab: export, vacate the slot
                    const int side = bx < sc.slab_lo ? 0 : 1;
                    const int k = atomicAdd(side ? &st->mig_hi : &st->mig_lo, 1);
                    if (k < MG.cap) {
                        T* rec = (side ? MG.hi : MG.lo) + (size_t)k * MG.rec;
                        int q = 0;
#pragma unroll
                        for (int a = 0; a < D; ++a)
                            rec[q++] = xn[a];
#pragma unroll
                        for (int a = 0; a < D; ++a)
                            rec[q++] = vn[a];
                        rec[q++] = m;
                        rec[q++] = V;
                        rec[q++] = rho;
                        rec[q++] = eps;
                        rec[q++] = szz;
#pragma unroll
                        for (int s2 = 0; s2 < C::NS; ++s2)
                            rec[q++] = sig[s2];
#pragma unroll
                        for (int k2 = 0; k2 < D * D; ++k2)
                            rec[q++] = L[k2];
                        if constexpr (APIC) {
#pragma unroll
                            for (int k2 = 0; k2 < D * D; ++k2)
                                rec[q++] = Bm[k2];
                        }
                        if constexpr (TRACKF) {
#pragma unroll
                            for (int k2 = 0; k2 < D * D; ++k2)
                                rec[q++] = Fm[k2];
                        }
                        (side ? MG.hi_pid : MG.lo_pid)[k] = pid;
                        (side ? MG.hi_slot : MG.lo_slot)[k] = i;
                    } else {
                        st->mig_over = 1;
                        st->abort = 1;
                    }
                    Pout.pid[i] = -1;
                    key = KEY_DEAD;
                }
            }
            keys_out[i] = key;
        }
    }
    wq_finish(wq);
}

// constitutive-only phase (constitutive_update on the stored grad_v), in place
template <class T, int D, bool TRACKF>
__global__ void k_constitutive(DevScene<T, D> sc, PBuf<T, D> P, int n, DevStatus* st)
{
    using C = Cfg<D>;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || st->abort)
        return;
    T L[D * D], sig[C::NS];
#pragma unroll
    for (int k = 0; k < D * D; ++k)
        L[k] = P.gv[k][i];
#pragma unroll
    for (int s = 0; s < C::NS; ++s)
        sig[s] = P.sig[s][i];
    T szz = D == 2 ? P.szz[i] : T(0), rho = P.rho[i], V = P.V[i], eps = P.eps[i];
    if (!constitutive_particle<T, D>(sc, sig, szz, rho, V, eps, L)) {
        atomicMin(&st->den_pid, P.pid[i]);
        st->den_flag = 1;
        return;
    }
#pragma unroll
    for (int s = 0; s < C::NS; ++s)
        P.sig[s][i] = sig[s];
    if (D == 2)
        P.szz[i] = szz;
    P.rho[i] = rho;
    P.V[i] = V;
    P.eps[i] = eps;
    if constexpr (TRACKF) {
        T Fm[D * D], Fn[D * D];
#pragma unroll
        for (int k = 0; k < D * D; ++k)
            Fm[k] = P.F[k][i];
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = 0; b < D; ++b) {
                T s = T(0);
#pragma unroll
                for (int k = 0; k < D; ++k)
                    s += ((a == k ? T(1) : T(0)) + L[a * D + k] * sc.dt) * Fm[k * D + b];
                Fn[a * D + b] = s;
            }
#pragma unroll
        for (int k = 0; k < D * D; ++k)
            P.F[k][i] = Fn[k];
    }
}

// step counter: a step whose only failure is that its OUTPUT left the domain (detected while
// forming the next step's keys) did complete -- the reference throws in the next step's P2G
__global__ void k_step_end(DevStatus* st)
{
    pdl_wait();
    pdl_trigger();
    if (!st->abort) {
        st->step += 1;
    } else if (st->ood_flag == 2 && !st->den_flag && !st->nan_flag && !st->ood_counted) {
        st->step += 1;
        st->ood_counted = 1;
    }
}

} // namespace mpmgpu
