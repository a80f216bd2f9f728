// kernels_adj.cuh -- reverse-mode adjoint of the step (adjoint.hpp:328-525) and the segmented
// checkpoint driver (checkpoint.hpp:72-143) on B200.
//
// Cotangents are stored in particle-id order (pid-indexed), so the per-step cell re-sort of the
// forward state never has to be inverted: step t's cotangent and step t-1's state meet through
// pid. step_vjp = forward replay (sort, P2G, grid with stored m/p/f) then
//   K5a k_adj_g2pT_gather  per particle: G2P gather of grad v (forward), constitutive VJP
//                          (fluid_vjp adjoint.hpp:153-184 / dp_vjp :188-293), the gather half of
//                          the G2P transpose (x cotangent, :429-434); writes per-particle scatter
//                          records in sorted order
//   K5b k_adj_scatter      G2P transpose scatter (:427-428, 436) of gv_cot / gvold_cot into
//                          per-block partial tiles: the deterministic node-column march of P2G
//   K6  k_adj_grid         per node: fixed-order partial sum, correction-chain VJP replayed
//                          from v_tilde (:441-460, node_correction_vjp :114-150), momentum
//                          update transpose (:462-477)
//   K7  k_adj_p2gT         per particle: P2G transpose gather (:479-524)
// Parameter gradients (c, mu, friction segments) are reduced per block and then over blocks
// in a fixed order: adjoints are bit-reproducible run to run.
#pragma once

#include "common.cuh"
#include "constit.cuh"
#include "kernels_fwd.cuh"
#include "kernels_util.cuh"

#include <stdexcept>
#include <vector>

namespace mpmgpu {

constexpr int PG_SLOTS = 2 + MAX_FRIC; // c, mu, friction[fric_off[w] + k]

// pid-indexed cotangent arrays (StateCotangent, adjoint.hpp:10-72); matrices full, row-major
template <class T, int D> struct CBuf {
    T* x[D];
    T* v[D];
    T* rho;
    T* V;
    T* eps;
    T* szz;
    T* sig[D * D];
    T* gv[D * D];
    T* aff[D * D];
};

// per-particle scatter records of the G2P transpose, sorted-slot order
template <class T, int D> struct SBuf {
    T* a[D];       // pic_cot + inc_cot
    T* inc[D];     // inc_cot
    T* L[D * D];   // grad v_new cotangent
    T* Bc[D * D];  // APIC: affine cotangent (cot_out.affine)
};

// cotangent grid (node blocks): gv_cot / gvold_cot sums are transient; these are the outputs of K6
template <class T, int D> struct GCBuf {
    T* gm;
    T* gmom[D];
    T* gf[D];
};

// ---- device VJP math ----------------------------------------------------------------------
// detail::fluid_vjp (adjoint.hpp:152-184); L row-major; sc_ (sigma cotangent) full row-major
template <class T, int D>
__device__ __forceinline__ void fluid_vjp_dev(const DevScene<T, D>& sc, T rho, T V, const T* L, const T* sgc, T rho_c,
                                              T V_c, T* gvn_c, T& rho_in_c, T& V_in_c, T& c_acc, T& mu_acc)
{
    T dd[D][D];
    T trd = T(0);
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j)
            dd[i][j] = T(0.5) * (L[i * D + j] + L[j * D + i]) * sc.dt;
#pragma unroll
    for (int i = 0; i < D; ++i)
        trd += dd[i][i];
    const T den = T(1) + trd;
    const T rho_new = rho / den;
    const T c = sc.c;
    const T k = sc.fl_k;
    T trs = T(0);
#pragma unroll
    for (int i = 0; i < D; ++i)
        trs += sgc[i * D + i];
    const T p_c = -trs;
    T mu_sum = T(0);
    const T vis = -(T(2) / T(3)) * trd;
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
        for (int i = 0; i < D; ++i)
            mu_sum += sgc[i * D + j] * (vis * (i == j ? T(1) : T(0)) + T(2) * dd[i][j]);
    mu_acc += mu_sum * (sc.rate_form ? T(1) / sc.dt : T(1));
    T trd_c = -(T(2) / T(3)) * k * trs;
    T dd_c[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j)
            dd_c[i][j] = T(2) * k * sgc[i * D + j];
    c_acc += T(2) * c * (rho_new - sc.rho0) * p_c;
    const T rho_new_c = rho_c + c * c * p_c;
    rho_in_c += rho_new_c / den;
    T den_c = -(rho / (den * den)) * rho_new_c;
    V_in_c += den * V_c;
    den_c += V * V_c;
    trd_c += den_c;
#pragma unroll
    for (int i = 0; i < D; ++i)
        dd_c[i][i] += trd_c;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j)
            gvn_c[i * D + j] += sc.dt * T(0.5) * (dd_c[i][j] + dd_c[j][i]);
}

// detail::dp_vjp (adjoint.hpp:186-293). S: input stress (3x3 embedding); sgc: sigma cotangent
// (D x D full, row-major). Outputs accumulate into gvn_c (D x D), sig_in_c (D x D), szz_in_c.
template <class T, int D>
__device__ __forceinline__ void dp_vjp_dev(const DevScene<T, D>& sc, const T (&S)[3][3], const T* L, const T* sgc,
                                           T szz_c, T rho_c, T V_c, T rho_in, T V_in, T* gvn_c, T* sig_in_c,
                                           T& szz_in_c, T& rho_in_c, T& V_in_c)
{
    DpTrial<T, D> t;
    dp_trial<T, D>(sc, S, L, t);
    T oc[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            oc[i][j] = (i < D && j < D) ? sgc[i * D + j] : T(0);
    if (D == 2)
        oc[2][2] += szz_c;
    T tc[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            tc[i][j] = T(0);
    auto assemble = [&](const T (&dc)[3][3], T sm_c) {
        T trdc = T(0);
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                tc[i][j] += dc[i][j];
#pragma unroll
        for (int i = 0; i < 3; ++i)
            trdc += dc[i][i];
        const T sm_total = sm_c - trdc;
#pragma unroll
        for (int i = 0; i < 3; ++i)
            tc[i][i] += sm_total / T(3);
    };
    auto contract_dev = [&]() { // (out_cot .* dev).sum(), column-major order
        T s = T(0);
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int i = 0; i < 3; ++i)
                s += oc[i][j] * t.dev[i][j];
        return s;
    };
    if (t.zone == 1) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                tc[i][j] = oc[i][j];
    } else if (t.zone == 2) {
        const T denom = sc.dp_dlam_den;
        const T dlam = t.fs / denom;
        const T sm_new = t.sm - sc.K * sc.q_psi * dlam;
        const T tau_new = sc.k_phi - sc.q_phi * sm_new;
        if (!(t.tau <= T(0) || tau_new < T(0))) {
            const bool capped = sm_new > sc.sigma_t;
            const T ratio = tau_new / t.tau;
            T dc[3][3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    dc[i][j] = ratio * oc[i][j];
            const T ratio_c = contract_dev();
            T sm_new_c = capped ? T(0) : (oc[0][0] + oc[1][1] + oc[2][2]);
            const T tau_new_c = ratio_c / t.tau;
            T tau_c = -ratio_c * tau_new / (t.tau * t.tau);
            sm_new_c += -sc.q_phi * tau_new_c;
            T sm_c = sm_new_c;
            const T dlam_c = -sc.K * sc.q_psi * sm_new_c;
            const T fs_c = dlam_c / denom;
            tau_c += fs_c;
            sm_c += sc.q_phi * fs_c;
            if (t.tau > T(0))
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        dc[i][j] += (tau_c / (T(2) * t.tau)) * t.dev[i][j];
            assemble(dc, sm_c);
        }
    } else {
        if (t.tau > sc.tau_P) {
            const T ratio = sc.tau_P / t.tau;
            T dc[3][3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    dc[i][j] = ratio * oc[i][j];
            const T ratio_c = contract_dev();
            const T tau_c = -ratio_c * sc.tau_P / (t.tau * t.tau);
            if (t.tau > T(0))
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        dc[i][j] += (tau_c / (T(2) * t.tau)) * t.dev[i][j];
            assemble(dc, T(0));
        } else {
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    tc[i][j] = oc[i][j];
            const T sm_c = -(oc[0][0] + oc[1][1] + oc[2][2]);
#pragma unroll
            for (int i = 0; i < 3; ++i)
                tc[i][i] += sm_c / T(3);
        }
    }
    // trial = sR + 2G dd + (K - 2G/3) tr(dd) I
    const T lam = sc.dp_lam;
    const T ttr = tc[0][0] + tc[1][1] + tc[2][2];
    T dd_c[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            dd_c[i][j] = T(2) * sc.G * tc[i][j] + (i == j ? lam * ttr : T(0));
    const T den = T(1) + t.trd;
    const T den_c = V_in * V_c - (rho_in / (den * den)) * rho_c;
    V_in_c += den * V_c;
    rho_in_c += rho_c / den;
#pragma unroll
    for (int i = 0; i < 3; ++i)
        dd_c[i][i] += den_c;
    // sR = S + S dw^T + dw S^T
    T S_c[3][3], dw_c[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            T a1 = T(0), a2 = T(0), b1 = T(0), b2 = T(0);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                a1 += tc[i][k] * t.dw[k][j];
                a2 += t.dw[k][i] * tc[k][j];
                b1 += tc[k][i] * S[k][j];
                b2 += tc[i][k] * S[k][j];
            }
            S_c[i][j] = tc[i][j] + a1 + a2;
            dw_c[i][j] = b1 + b2;
        }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            gvn_c[i * D + j] += sc.dt * (T(0.5) * (dd_c[i][j] + dd_c[j][i]) + T(0.5) * (dw_c[i][j] - dw_c[j][i]));
            sig_in_c[i * D + j] += S_c[i][j];
        }
    if (D == 2)
        szz_in_c += S_c[2][2];
}

// fixed-order CTA reduction of per-thread values -> out[slot] (deterministic)
template <class T, int NT>
__device__ __forceinline__ T block_sum_fixed(T v, T* scratch)
{
    scratch[threadIdx.x] = v;
    __syncthreads();
#pragma unroll
    for (int s = NT / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s)
            scratch[threadIdx.x] = scratch[threadIdx.x] + scratch[threadIdx.x + s];
        __syncthreads();
    }
    T r = scratch[0];
    __syncthreads();
    return r;
}

// ---- tensor-product stencil moments ----------------------------------------------------------
// For one node field f of a tile (last axis fastest, t0 = the particle's stencil corner):
//   phi  = sum_o  w0 w1 (w2) f                        (PHI)
//   g[a] = sum_o  d(phi)/dx_a f                       (grad of the shape function)
//   h    = sum_o  d2(phi)/dx_a dx_b f                 (HES; stencil_hessian, adjoint.hpp:95-110)
// evaluated axis by axis (last-axis sums, then the middle axis, then the first). All 1 + D +
// D(D+1)/2 moments of a field cost ~150 FP64 ops in 3-D instead of 27 x (weight products +
// contraction); the per-node weight products are never formed. The second-derivative weights are
// (1, -2, 1) / dh^2 on every axis (bspline.hpp:43-108), applied as adds and one scale at the end.
template <class T, int D> struct Mom {
    T phi;
    T g[D];
    T h[D][D];
};
template <class T, int D, bool PHI, bool HES>
__device__ __forceinline__ void stencil_moments(const T* __restrict__ f, int t0, const T (&w)[D][3],
                                                const T (&dw)[D][3], T idh2, Mom<T, D>& m)
{
    constexpr int TE = Cfg<D>::TE;
    if constexpr (D == 3) {
        T phi = T(0), g0 = T(0), g1 = T(0), g2 = T(0);
        T h00 = T(0), h11 = T(0), h22 = T(0), h01 = T(0), h02 = T(0), h12 = T(0);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            T ww = T(0), dww = T(0), wdw = T(0), ddw = T(0), wdd = T(0), dwdw = T(0);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const T* p = f + t0 + (i * TE + j) * TE;
                const T f0 = p[0], f1 = p[1], f2 = p[2];
                const T zw = w[2][0] * f0 + w[2][1] * f1 + w[2][2] * f2;
                const T zdw = dw[2][0] * f0 + dw[2][1] * f1 + dw[2][2] * f2;
                ww += w[1][j] * zw;
                dww += dw[1][j] * zw;
                wdw += w[1][j] * zdw;
                if constexpr (HES) {
                    const T zdd = (f0 + f2) - T(2) * f1;
                    ddw += (j == 1 ? T(-2) : T(1)) * zw;
                    wdd += w[1][j] * zdd;
                    dwdw += dw[1][j] * zdw;
                }
            }
            if constexpr (PHI)
                phi += w[0][i] * ww;
            g0 += dw[0][i] * ww;
            g1 += w[0][i] * dww;
            g2 += w[0][i] * wdw;
            if constexpr (HES) {
                h00 += (i == 1 ? T(-2) : T(1)) * ww;
                h11 += w[0][i] * ddw;
                h22 += w[0][i] * wdd;
                h01 += dw[0][i] * dww;
                h02 += dw[0][i] * wdw;
                h12 += w[0][i] * dwdw;
            }
        }
        m.phi = phi;
        m.g[0] = g0;
        m.g[1] = g1;
        m.g[2] = g2;
        if constexpr (HES) {
            m.h[0][0] = h00 * idh2;
            m.h[1][1] = h11 * idh2;
            m.h[2][2] = h22 * idh2;
            m.h[0][1] = m.h[1][0] = h01;
            m.h[0][2] = m.h[2][0] = h02;
            m.h[1][2] = m.h[2][1] = h12;
        }
    } else {
        T phi = T(0), g0 = T(0), g1 = T(0), h00 = T(0), h11 = T(0), h01 = T(0);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const T* p = f + t0 + i * TE;
            const T f0 = p[0], f1 = p[1], f2 = p[2];
            const T zw = w[1][0] * f0 + w[1][1] * f1 + w[1][2] * f2;
            const T zdw = dw[1][0] * f0 + dw[1][1] * f1 + dw[1][2] * f2;
            if constexpr (PHI)
                phi += w[0][i] * zw;
            g0 += dw[0][i] * zw;
            g1 += w[0][i] * zdw;
            if constexpr (HES) {
                const T zdd = (f0 + f2) - T(2) * f1;
                h00 += (i == 1 ? T(-2) : T(1)) * zw;
                h11 += w[0][i] * zdd;
                h01 += dw[0][i] * zdw;
            }
        }
        m.phi = phi;
        m.g[0] = g0;
        m.g[1] = g1;
        if constexpr (HES) {
            m.h[0][0] = h00 * idh2;
            m.h[1][1] = h11 * idh2;
            m.h[0][1] = m.h[1][0] = h01;
        }
    }
}

// ---- K5a: G2P-transpose gather + constitutive VJP ------------------------------------------
template <int D> struct K5aStage { // staged rows per thread (K5a, below)
    static constexpr int CSIG = 0, CRHO = D * D, CV = CRHO + 1, RHO = CV + 1, VOL = RHO + 1, SIG = VOL + 1,
                         SZZ = SIG + Cfg<D>::NS, CSZZ = SZZ + 1, N = CSZZ + 1;
    static constexpr int NX = 3 * D; // + 2 slots of (x, co.v, co.x) of the next round's particle
    template <class T> static constexpr size_t smem() { return sizeof(T) * (2 * D * Cfg<D>::TN + (N + 2 * NX) * 256); }
};
// Cotangents live in state-storage order: co (cot at t+1) is indexed by the sorted slot i (the
// storage order of S^{t+1}, which the forward G2P wrote in this step's sort order) and ci (cot at
// t) by src = perm[i] (the storage slot of S^t). Both are streamed, not gathered through ids.
// GVZ: co.grad_v is known zero (FLIP/PIC chains and seeded losses) and ci.grad_v is left to the
// caller's zero flag unless TPIC accumulates into it in K7.
#ifndef K5A_MINB
#define K5A_MINB 1 // MEASURED C4: 2 CTAs per SM (128 registers, 312 B of spills) 0.873 ms vs 0.837
#endif
template <class T, int D, bool APIC>
__global__ void __launch_bounds__(256, K5A_MINB) k_adj_g2pT_gather(DevScene<T, D> sc, PBuf<T, D> Pin, GBuf<T, D> G,
                                                         const int* __restrict__ perm, const int* __restrict__ bstart,
                                                         const int* __restrict__ bend, const int* __restrict__ occ,
                                                         const int* __restrict__ n_occ, CBuf<T, D> co, CBuf<T, D> ci,
                                                         SBuf<T, D> S, T* __restrict__ pg_block, DevStatus* st,
                                                         int co_gv_zero, int ci_gv_write, int* __restrict__ wq)
{
    using C = Cfg<D>;
    constexpr int TE = C::TE, TN = C::TN;
    extern __shared__ unsigned char smem_raw[];
    T* tile = reinterpret_cast<T*>(smem_raw); // [2D][TN]: v, v - v_old
    // the constitutive-transpose inputs of the thread's particle (co.sigma, co.rho, co.V, rho, V,
    // sigma[, szz]) are fetched with cp.async at the top of the iteration into this thread's column
    // and read after the stencil moments, so their latency overlaps the moments without holding
    // registers (K5a runs one CTA per SM at ~216 registers)
    using KS = K5aStage<D>;
    T* kst = tile + 2 * D * TN + threadIdx.x; // [KS::N][256]
    __shared__ T red[256];
    __shared__ int w_s; // next list entry (work counter, common.cuh)
    const int nocc = st->abort ? 0 : *n_occ; // every CTA still passes wq_finish
    if (threadIdx.x == 0)
        w_s = wq_first(wq);
    const T alpha = sc.alpha;
    // x, co.v and co.x of the thread's next particle: cp.async one round ahead into slot (slot ^ 1)
    auto issue_x = [&](int slot, int src, int i) {
        T* b = kst + (KS::N + slot * KS::NX) * 256;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            cp_async_t<T>(b + a * 256, Pin.x[a] + src);
            cp_async_t<T>(b + (D + a) * 256, co.v[a] + i);
            cp_async_t<T>(b + (2 * D + a) * 256, co.x[a] + i);
        }
    };
    for (;;) {
        cp_async_wait_all();
        __syncthreads(); // w_s published; the previous block's shared-memory readers are done
        const int w = w_s;
        if (w >= nocc)
            break;
        const int Q = occ[w];
        const int s0 = bstart[Q], s1 = bend[Q];
        // the first two rounds' permutation entries in flight during the tile load
        const int i0 = s0 + int(threadIdx.x);
        int src_a = i0 < s1 ? perm[i0] : 0, src_b = i0 + int(blockDim.x) < s1 ? perm[i0 + blockDim.x] : 0;
        int qc[D];
        block_coords<D>(Q, sc.nb, qc);
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
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const T vn = ok ? G.v[a][gi] : T(0), vo = ok ? G.vold[a][gi] : T(0);
                tile[a * TN + t] = vn;
                tile[(D + a) * TN + t] = vn - vo;
            }
        }
        if (i0 < s1)
            issue_x(0, src_a, i0);
        cp_async_commit();
        __syncthreads();
        if (threadIdx.x == 0) // every thread read w_s before the barrier above
            w_s = wq_next(wq, w);
        T c_acc = T(0), mu_acc = T(0);
        int xslot = 0;
        const T idh2 = sc.inv_dh * sc.inv_dh;
        // process the segment in rounds so every thread reaches the block reductions; the next
        // round's permutation entry is loaded one round ahead (the first one before the tile load)
        for (int base = s0; base < s1; base += blockDim.x) {
            const int i = base + threadIdx.x;
            const int src_cur = src_a;
            src_a = src_b;
            src_b = i + 2 * int(blockDim.x) < s1 ? perm[i + 2 * blockDim.x] : 0;
            if (i + int(blockDim.x) < s1)
                issue_x(xslot ^ 1, src_a, i + blockDim.x);
            cp_async_commit();
            const T* xs = kst + (KS::N + xslot * KS::NX) * 256;
            xslot ^= 1;
            if (i < s1) {
                const int src = src_cur;
                {
#pragma unroll
                    for (int k = 0; k < D * D; ++k)
                        cp_async_t<T>(kst + (KS::CSIG + k) * 256, co.sig[k] + i);
                    cp_async_t<T>(kst + KS::CRHO * 256, co.rho + i);
                    cp_async_t<T>(kst + KS::CV * 256, co.V + i);
                    cp_async_t<T>(kst + KS::RHO * 256, Pin.rho + src);
                    cp_async_t<T>(kst + KS::VOL * 256, Pin.V + src);
                    if (sc.material != 0) {
#pragma unroll
                        for (int q = 0; q < Cfg<D>::NS; ++q)
                            cp_async_t<T>(kst + (KS::SIG + q) * 256, Pin.sig[q] + src);
                        if constexpr (D == 2)
                            cp_async_t<T>(kst + KS::SZZ * 256, Pin.szz + src);
                    }
                    if constexpr (D == 2)
                        cp_async_t<T>(kst + KS::CSZZ * 256, co.szz + i);
                    cp_async_commit();
                }
                // pending: this particle's x group, the next one's, and the group above
                asm volatile("cp.async.wait_group 2;\n" ::: "memory");
                T x[D];
#pragma unroll
                for (int a = 0; a < D; ++a)
                    x[a] = xs[a * 256];
                T w[D][3], dw[D][3];
                int tb[D];
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    const T u = (x[a] - sc.origin[a]) * sc.inv_dh;
                    const T fl = dfloor<T>(u - T(0.5));
                    const T fx = u - fl;
                    const T h0 = T(1.5) - fx, h1 = fx - T(1), h2 = fx - T(0.5);
                    w[a][0] = T(0.5) * h0 * h0;
                    w[a][1] = T(0.75) - h1 * h1;
                    w[a][2] = T(0.5) * h2 * h2;
                    dw[a][0] = -h0 * sc.inv_dh;
                    dw[a][1] = -T(2) * h1 * sc.inv_dh;
                    dw[a][2] = h2 * sc.inv_dh;
                    tb[a] = int(fl) - qc[a] * C::B;
                }
                // co.* at the sorted slot i, ci.* at the storage slot src (see the kernel comment)
                T vc[D], xc[D], pic[D], inc[D], xp[D];
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    vc[a] = xs[(D + a) * 256];
                    xc[a] = xs[(2 * D + a) * 256];
                    pic[a] = (T(1) - alpha) * vc[a] + sc.dt * xc[a];
                    inc[a] = alpha * vc[a];
                    xp[a] = T(0);
                }
                T L[D * D];
                T HM[D][D][D]; // HM[c][a][b] = sum_o H_ab(o) v_c(o)   (non-APIC)
                int t0 = 0;
#pragma unroll
                for (int a = 0; a < D; ++a)
                    t0 = t0 * TE + tb[a];
                if constexpr (!APIC) {
                    // forward gather grad v_new = sum v (x) grad phi (transfer.hpp:111) and every
                    // stencil sum of the G2P transpose, as moments of the v and v - v_old fields:
                    //   sum_o grad phi (pic.v + inc.(v - v_old)) = sum_c pic_c G1[c] + inc_c Gd[c]
                    //   sum_o H (L^T v)                          = sum_bc L_cb HM[c][:, b]
#pragma unroll
                    for (int c = 0; c < D; ++c) {
                        Mom<T, D> m;
                        stencil_moments<T, D, false, true>(tile + c * TN, t0, w, dw, idh2, m);
#pragma unroll
                        for (int a = 0; a < D; ++a) {
                            L[c * D + a] = m.g[a];
                            xp[a] += pic[c] * m.g[a];
#pragma unroll
                            for (int b = 0; b < D; ++b)
                                HM[c][a][b] = m.h[a][b];
                        }
                        Mom<T, D> md;
                        stencil_moments<T, D, false, false>(tile + (D + c) * TN, t0, w, dw, idh2, md);
#pragma unroll
                        for (int a = 0; a < D; ++a)
                            xp[a] += inc[c] * md.g[a];
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < D * D; ++k)
                        L[k] = T(0);
                    for (int k = 0; k < C::NOFF; ++k) {
                        int o[D], kk = k, ti = 0;
#pragma unroll
                        for (int a = D - 1; a >= 0; --a) {
                            o[a] = kk % 3;
                            kk /= 3;
                        }
#pragma unroll
                        for (int a = 0; a < D; ++a)
                            ti = ti * TE + tb[a] + o[a];
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
#pragma unroll
                        for (int a = 0; a < D; ++a) {
                            const T nv = tile[a * TN + ti];
#pragma unroll
                            for (int b = 0; b < D; ++b)
                                L[a * D + b] += nv * gw[b];
                        }
                    }
                }
                // (1) constitutive transpose (adjoint.hpp:374-400)
                cp_async_wait_all(); // the staged inputs above
                T sgc[D * D], gvn_c[D * D], sig_in_c[D * D];
#pragma unroll
                for (int k = 0; k < D * D; ++k) {
                    sgc[k] = kst[(KS::CSIG + k) * 256];
                    gvn_c[k] = T(0);
                    sig_in_c[k] = T(0);
                }
                T rho_in_c = T(0), V_in_c = T(0), szz_in_c = T(0);
                const T rho = kst[KS::RHO * 256], V = kst[KS::VOL * 256];
                const T co_rho = kst[KS::CRHO * 256], co_V = kst[KS::CV * 256];
                if (sc.material == 0) {
                    fluid_vjp_dev<T, D>(sc, rho, V, L, sgc, co_rho, co_V, gvn_c, rho_in_c, V_in_c, c_acc, mu_acc);
                } else {
                    T Sm[3][3];
#pragma unroll
                    for (int a = 0; a < 3; ++a)
#pragma unroll
                        for (int b = 0; b < 3; ++b)
                            Sm[a][b] = (a < D && b < D) ? kst[(KS::SIG + sym_idx<D>(a, b)) * 256] : T(0);
                    if constexpr (D == 2)
                        Sm[2][2] = kst[KS::SZZ * 256];
                    dp_vjp_dev<T, D>(sc, Sm, L, sgc, D == 2 ? kst[KS::CSZZ * 256] : T(0), co_rho, co_V, rho, V,
                                     gvn_c, sig_in_c, szz_in_c, rho_in_c, V_in_c);
                }
                // cot_out.grad_v joins (adjoint.hpp:398-400)
                if (!co_gv_zero)
#pragma unroll
                    for (int k = 0; k < D * D; ++k)
                        gvn_c[k] += co.gv[k][i];
                // (2) G2P transpose, gather half (adjoint.hpp:405-439)
                T Bc[D * D];
                if constexpr (APIC) {
#pragma unroll
                    for (int k = 0; k < D * D; ++k)
                        Bc[k] = co.aff[k][i];
                }
                if constexpr (!APIC) {
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int b = 0; b < D; ++b)
#pragma unroll
                            for (int c = 0; c < D; ++c)
                                xp[a] += gvn_c[c * D + b] * HM[c][a][b];
                } else {
                for (int k = 0; k < C::NOFF; ++k) {
                    int o[D], kk = k, ti = 0;
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
                    // Hessian of phi (stencil_hessian adjoint.hpp:95-110)
                    T H[D][D];
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int b = a; b < D; ++b) {
                            T r = a == b ? (o[a] == 1 ? -T(2) * idh2 : idh2) : dw[a][o[a]] * dw[b][o[b]];
#pragma unroll
                            for (int c = 0; c < D; ++c)
                                if (c != a && c != b)
                                    r *= w[c][o[c]];
                            H[a][b] = r;
                            H[b][a] = r;
                        }
                    T wv[D], dv[D];
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        wv[a] = tile[a * TN + ti];
                        dv[a] = tile[(D + a) * TN + ti]; // v - v_old
                    }
                    T s1 = T(0), s2 = T(0);
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        s1 += pic[a] * wv[a];
                        s2 += inc[a] * dv[a];
                    }
                    T LTw[D];
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        T s = T(0);
#pragma unroll
                        for (int b = 0; b < D; ++b)
                            s += gvn_c[b * D + a] * wv[b];
                        LTw[a] = s;
                    }
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        T hs = T(0);
#pragma unroll
                        for (int b = 0; b < D; ++b)
                            hs += H[a][b] * LTw[b];
                        xp[a] += gw[a] * (s1 + s2);
                        xp[a] += hs;
                    }
                    T r[D];
#pragma unroll
                    for (int a = 0; a < D; ++a)
                        r[a] = (sc.origin[a] + T(qc[a] * C::B + tb[a] + o[a]) * sc.dh) - x[a];
                    T Bcr[D], BcTw[D], wBr = T(0);
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        T s = T(0), s2b = T(0);
#pragma unroll
                        for (int b = 0; b < D; ++b) {
                            s += Bc[a * D + b] * r[b];
                            s2b += Bc[b * D + a] * wv[b];
                        }
                        Bcr[a] = s;
                        BcTw[a] = s2b;
                    }
#pragma unroll
                    for (int a = 0; a < D; ++a)
                        wBr += wv[a] * Bcr[a];
#pragma unroll
                    for (int a = 0; a < D; ++a)
                        xp[a] += gw[a] * wBr - phi * BcTw[a];
                }
                }
                // write cot_in at the storage slot (overwrites: this kernel is the first writer;
                // the eps cotangent is discarded, adjoint.hpp:399-400, and never stored)
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    ci.v[a][src] = alpha * vc[a];
                    ci.x[a][src] = xc[a] + xp[a];
                }
                ci.rho[src] = rho_in_c;
                ci.V[src] = V_in_c;
                if (D == 2)
                    ci.szz[src] = szz_in_c;
#pragma unroll
                for (int k = 0; k < D * D; ++k) {
                    ci.sig[k][src] = sig_in_c[k];
                    if (ci_gv_write)
                        ci.gv[k][src] = T(0);
                    if constexpr (APIC)
                        ci.aff[k][src] = T(0);
                }
                // scatter records (sorted slot i)
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    S.a[a][i] = pic[a] + inc[a];
                    S.inc[a][i] = inc[a];
                }
#pragma unroll
                for (int k = 0; k < D * D; ++k) {
                    S.L[k][i] = gvn_c[k];
                    if constexpr (APIC)
                        S.Bc[k][i] = Bc[k];
                }
            }
        }
        // per-block c / mu partials (fixed-order tree) -> pg_block[Q][0..1]
        if (sc.material == 0) {
            const T cs = block_sum_fixed<T, 256>(c_acc, red);
            const T ms = block_sum_fixed<T, 256>(mu_acc, red);
            if (threadIdx.x == 0) {
                pg_block[(size_t)Q * 2 + 0] = cs;
                pg_block[(size_t)Q * 2 + 1] = ms;
            }
        }
    }
    wq_finish(wq);
}

// ---- K5b: G2P-transpose scatter (node-column march over the sorted records) ----------------
// Contributions per node (adjoint.hpp:427-436): gv_cot += phi a + L grad(phi) (+ APIC phi Bc r),
// gvold_cot -= phi inc. 2D fields per node, deterministic order as in k_p2g.
template <class T, int D, bool APIC>
__global__ void __launch_bounds__(256) k_adj_scatter(DevScene<T, D> sc, PBuf<T, D> Pin, SBuf<T, D> S,
                                                     const int* __restrict__ perm, const int* __restrict__ keys,
                                                     const int* __restrict__ bstart, const int* __restrict__ bend,
                                                     const int* __restrict__ occ, const int* __restrict__ n_occ,
                                                     T* __restrict__ partials, const DevStatus* st)
{
    using C = Cfg<D>;
    constexpr int B = C::B, TE = C::TE, NF = 2 * D;
    constexpr int LVLBITS = (D - 1) * C::LOGB;
    __shared__ int cst[C::NB + 1];
    if (st->abort)
        return;
    const int nocc = *n_occ;
    const int tid = threadIdx.x;
    const int col = tid % C::NCOL, seg = tid / C::NCOL;
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
    for (int wq = blockIdx.x; wq < nocc; wq += gridDim.x) {
        const int Q = occ[wq];
        const int s0 = bstart[Q], s1 = bend[Q], len = s1 - s0;
        int qc[D];
        block_coords<D>(Q, sc.nb, qc);
        for (int c = tid; c <= C::NB; c += blockDim.x) {
            int lo = 0, hi = len;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if ((keys[s0 + mid] & (C::NB - 1)) < c)
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
                for (int oo = 0; oo < C::NOFF / 3; ++oo) {
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
                            const int bc = cn[a] - o[a];
                            ok &= bc >= 0 && bc < B;
                            bcell = (bcell << C::LOGB) | (bc & (B - 1));
                        }
                    }
                    if (!ok)
                        continue;
                    bcell |= z << LVLBITS;
                    const int kb = cst[bcell], ke = cst[bcell + 1];
                    for (int k = kb; k < ke; ++k) {
                        const int i = s0 + k;
                        const int src = __ldg(perm + i);
                        T x[D], wgt[D][3], dwt[D][3];
#pragma unroll
                        for (int a = 0; a < D; ++a) {
                            x[a] = __ldg(Pin.x[a] + src);
                            const T u = (x[a] - sc.origin[a]) * sc.inv_dh;
                            const T fx = u - dfloor<T>(u - T(0.5));
                            const T h0 = T(1.5) - fx, h1 = fx - T(1), h2 = fx - T(0.5);
                            wgt[a][0] = T(0.5) * h0 * h0;
                            wgt[a][1] = T(0.75) - h1 * h1;
                            wgt[a][2] = T(0.5) * h2 * h2;
                            dwt[a][0] = -h0 * sc.inv_dh;
                            dwt[a][1] = -T(2) * h1 * sc.inv_dh;
                            dwt[a][2] = h2 * sc.inv_dh;
                        }
                        T av[D], iv[D], L[D * D];
#pragma unroll
                        for (int a = 0; a < D; ++a) {
                            av[a] = S.a[a][i];
                            iv[a] = S.inc[a][i];
                        }
#pragma unroll
                        for (int q = 0; q < D * D; ++q)
                            L[q] = S.L[q][i];
#pragma unroll
                        for (int o2 = 0; o2 < 3; ++o2) {
                            T phi = wgt[D - 1][o2];
#pragma unroll
                            for (int a = 0; a < D - 1; ++a)
                                phi *= wgt[a][o[a]];
                            T gw[D];
#pragma unroll
                            for (int a = 0; a < D; ++a) {
                                T r = (a == D - 1) ? dwt[a][o2] : dwt[a][o[a]];
#pragma unroll
                                for (int b = 0; b < D; ++b)
                                    if (b != a)
                                        r *= (b == D - 1) ? wgt[b][o2] : wgt[b][o[b]];
                                gw[a] = r;
                            }
                            T add[D];
#pragma unroll
                            for (int a = 0; a < D; ++a) {
                                T s = T(0);
#pragma unroll
                                for (int b = 0; b < D; ++b)
                                    s += L[a * D + b] * gw[b];
                                add[a] = phi * av[a] + s;
                            }
                            if constexpr (APIC) {
                                T r[D];
#pragma unroll
                                for (int a = 0; a < D; ++a) {
                                    const int idx = a == D - 1 ? qc[a] * B + z + o2 : qc[a] * B + cn[a];
                                    r[a] = (sc.origin[a] + T(idx) * sc.dh) - x[a];
                                }
#pragma unroll
                                for (int a = 0; a < D; ++a) {
                                    T s = T(0);
#pragma unroll
                                    for (int b = 0; b < D; ++b)
                                        s += S.Bc[a * D + b][i] * r[b];
                                    add[a] += phi * s;
                                }
                            }
#pragma unroll
                            for (int a = 0; a < D; ++a) {
                                acc[o2][a] += add[a];
                                acc[o2][D + a] -= phi * iv[a];
                            }
                        }
                    }
                }
                const int idx = z * C::NCOL + col;
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    part[f * C::TN + idx] = acc[0][f];
                    acc[0][f] = acc[1][f];
                    acc[1][f] = acc[2][f];
                    acc[2][f] = T(0);
                }
            }
            if (seg == C::SEGS - 1) {
#pragma unroll
                for (int k = 0; k < 2; ++k)
#pragma unroll
                    for (int f = 0; f < NF; ++f)
                        part[f * C::TN + (ze + k) * C::NCOL + col] = acc[k][f];
            } else {
#pragma unroll
                for (int k = 0; k < 2; ++k)
#pragma unroll
                    for (int f = 0; f < NF; ++f)
                        ov[k][f] = acc[k][f];
            }
        }
        __syncthreads();
        if (active && seg < C::SEGS - 1) {
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    T* p = part + f * C::TN + (ze + k) * C::NCOL + col;
                    *p = *p + ov[k][f];
                }
        }
        __syncthreads();
    }
}

// ---- K5b, 3-D PIC / FLIP / blend: the same pipelined column march as the forward P2G ----------
// (k_p2g_pipe3). Staged per particle: fx (through the sort permutation), the scatter record
// a = pic_cot + inc_cot, inc_cot and L = grad-v cotangent (sorted slot order). Thread = (base
// column, x-offset), 3 y-offsets x a rolling 3-node z window x 6 fields. Per node
// (adjoint.hpp:427-436): gv_cot += phi a + L grad(phi) = wz u + dwz t with u = pw a + L[:,0] p1 +
// L[:,1] p2, t = L[:,2] pw; gvold_cot -= phi inc. Fixed-order slot reduction into the partial tiles.
// SPLIT (f64, A/B only): the 6 node fields over two thread groups, (gv_x, gv_y) and
// (gv_z, gvold_xyz), as the forward P2G's split: 12 warps with <= 36 accumulators. MEASURED C4:
// 0.54 -> 0.67 ms (slower, unlike the forward P2G), so it is off by default.
#ifndef ADJ_SPLIT
#define ADJ_SPLIT 0
#endif
template <class T> struct AdjScatterCfg {
    static constexpr bool SPLIT = ADJ_SPLIT && sizeof(T) == 8;
    static constexpr int THREADS = SPLIT ? 384 : 192, NBC = 64, NSRC = 9, NRAW = 18, MAXIT = 64, CAP = 512, NF = 6;
    static constexpr int NA = SPLIT ? 4 : NF; // accumulated fields per thread
    static constexpr size_t SMEM_RAW = sizeof(T) * 2 * NRAW * CAP;
    static constexpr size_t SMEM_PK = sizeof(int) * 3 * 2 * CAP;
    static constexpr size_t SMEM_SLOT = sizeof(T) * Cfg<3>::NCOL * NSRC * NF;
    static constexpr size_t SMEM = SMEM_RAW + SMEM_PK + SMEM_SLOT;
};

template <class T>
__global__ void __launch_bounds__(AdjScatterCfg<T>::THREADS, 1)
    k_adj_scatter_pipe3(DevScene<T, 3> sc, PBuf<T, 3> P, SBuf<T, 3> Sb, const int* __restrict__ perm,
                        const int* __restrict__ keys, const int* __restrict__ bstart, const int* __restrict__ bend,
                        const int* __restrict__ lstart, const int* __restrict__ occ, const int* __restrict__ n_occ,
                        T* __restrict__ partials, const DevStatus* st, int* __restrict__ wq)
{
    using C = Cfg<3>;
    using S = AdjScatterCfg<T>;
    constexpr int B = C::B, TE = C::TE, NF = S::NF, CAP = S::CAP, NBC = S::NBC, NSRC = S::NSRC, NRAW = S::NRAW;
    constexpr int RX = 0, RA = 3, RI = 6, RL = 9; // raw rows: fx, a, inc, L (row-major a*3+b)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* raw = reinterpret_cast<T*>(smem_raw);                              // [2][NRAW][CAP]
    int* pk = reinterpret_cast<int*>(smem_raw + S::SMEM_RAW);             // [3][2][CAP] (perm, key)
    T* slots = reinterpret_cast<T*>(smem_raw + S::SMEM_RAW + S::SMEM_PK); // [NCOL][NSRC][NF]
    __shared__ int it_start[S::MAXIT], it_len[S::MAXIT], it_lvl[S::MAXIT], it_last[S::MAXIT];
    __shared__ int nit_s, ccount[2][NBC];
    __shared__ int w_s; // next list entry (work counter, common.cuh)
    const int nocc = st->abort ? 0 : *n_occ; // every CTA still passes wq_finish
    if (threadIdx.x == 0)
        w_s = wq_first(wq);
    const int tid = threadIdx.x;
    constexpr bool SPLIT = S::SPLIT;
    constexpr int NA = S::NA;
    const int grp = SPLIT ? tid / 192 : 0; // warp-uniform
    const int lt = SPLIT ? tid - 192 * grp : tid;
    const int f0 = SPLIT && grp ? 2 : 0;   // first slot field of this thread's group
    const int bc = lt / 3, o0 = lt % 3;
    const bool mid = o0 == 1;
    const T xoff = o0 == 0 ? T(1.5) : (o0 == 1 ? T(1) : T(0.5));
    const int bc0 = bc >> C::LOGB, bc1 = bc & (B - 1);
    const long long SI = P.S;

    for (;;) {
        __syncthreads(); // w_s published; the previous block's shared-memory readers are done
        const int w = w_s;
        if (w >= nocc)
            break;
        const int Q = occ[w];
        const int s0 = bstart[Q], s1 = bend[Q];
        if (tid == 0) { // level starts -> work items (as k_p2g_pipe3)
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
            nit_s = k > S::MAXIT ? -1 : k;
        }
        __syncthreads();
        int nit = nit_s;
        if (tid == 0) // every thread read w_s before the barrier above
            w_s = wq_next(wq, w);
        if (nit < 0) // the forward refused this block already (far_flag); nothing consistent to do
            nit = 0;
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
            const int b = s0 + it_start[j];
            for (int r = tid; r < it_len[j]; r += blockDim.x) {
                const T* q = P.base + pp[r];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    cp_async_t<T>(rb + (RX + a) * CAP + r, q + a * SI); // x (PLay field 0..2)
                    cp_async_t<T>(rb + (RA + a) * CAP + r, Sb.a[a] + b + r);
                    cp_async_t<T>(rb + (RI + a) * CAP + r, Sb.inc[a] + b + r);
                }
#pragma unroll
                for (int k = 0; k < 9; ++k)
                    cp_async_t<T>(rb + (RL + k) * CAP + r, Sb.L[k] + b + r);
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

        T* part = partials + (size_t)Q * NF * C::TN;
        T acc[3][3][NA];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int f = 0; f < NA; ++f)
                    acc[a][k][f] = T(0);

        auto emit_and_reduce = [&](int z) {
#pragma unroll
            for (int o1 = 0; o1 < 3; ++o1) {
                const int ncol = (bc0 + o0) * TE + bc1 + o1;
#pragma unroll
                for (int f = 0; f < NA; ++f) {
                    if (!SPLIT || grp == 1 || f < 2)
                        slots[(ncol * NSRC + o0 * 3 + o1) * NF + f0 + f] = acc[o1][0][f];
                    acc[o1][0][f] = acc[o1][1][f];
                    acc[o1][1][f] = acc[o1][2][f];
                    acc[o1][2][f] = T(0);
                }
            }
            __syncthreads(); // slots complete
            for (int t = tid; t < C::NCOL * NF; t += blockDim.x) {
                const int c = t / NF, f = t - c * NF;
                const int n0 = c / TE, n1 = c - n0 * TE;
                T sum = T(0);
#pragma unroll
                for (int q = 0; q < NSRC; ++q) {
                    const int b0 = n0 - q / 3, b1 = n1 - q % 3;
                    if (b0 >= 0 && b0 < B && b1 >= 0 && b1 < B)
                        sum += slots[(c * NSRC + q) * NF + f];
                }
                part[f * C::TN + z * C::NCOL + c] = sum; // the adjoint partial-tile layout (k_adj_grid)
            }
        };

        for (int j = 0; j < nit; ++j) {
            cp_async_wait_all();
            __syncthreads();
            if (j + 1 < nit)
                issue_fields(j + 1);
            if (j + 2 < nit)
                issue_pk(j + 2);
            cp_async_commit();
            const int len = it_len[j];
            const int* col = pk + (j % 3) * 2 * CAP + CAP;
            int* cnt = ccount[j & 1];
            if (tid < NBC)
                ccount[(j + 1) & 1][tid] = 0;
            {
                T* Rw = raw + (j & 1) * NRAW * CAP;
                for (int r = tid; r < len; r += blockDim.x) {
                    atomicAdd(&cnt[col[r] & (NBC - 1)], 1);
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const T u = (Rw[(RX + a) * CAP + r] - sc.origin[a]) * sc.inv_dh;
                        Rw[(RX + a) * CAP + r] = u - dfloor<T>(u - T(0.5));
                    }
                }
            }
            __syncthreads();
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
            for (int k = kb; k < ke; ++k) {
                const T fx = R[(RX + 0) * CAP + k], fy = R[(RX + 1) * CAP + k], fz = R[(RX + 2) * CAP + k];
                T wx, dwx, wy[3], dwy[3], wz[3], dwz[3];
                {
                    const T h = fx - xoff;
                    const T hh = h * h;
                    wx = mid ? T(0.75) - hh : T(0.5) * hh;
                    dwx = (mid ? -T(2) * h : h) * sc.inv_dh;
                }
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    quad_w<T>(fy, q, sc.inv_dh, wy[q], dwy[q]);
                    quad_w<T>(fz, q, sc.inv_dh, wz[q], dwz[q]);
                }
                T av[3], iv[3], L[9];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    av[a] = R[(RA + a) * CAP + k];
                    iv[a] = R[(RI + a) * CAP + k];
                }
#pragma unroll
                for (int q = 0; q < 9; ++q)
                    L[q] = R[(RL + q) * CAP + k];
                if constexpr (SPLIT) {
#pragma unroll
                    for (int o1 = 0; o1 < 3; ++o1) {
                        const T pw = wx * wy[o1], p1 = dwx * wy[o1], p2 = wx * dwy[o1];
                        if (grp == 0) { // gv_x, gv_y
#pragma unroll
                            for (int a = 0; a < 2; ++a) {
                                const T u = pw * av[a] + L[a * 3 + 0] * p1 + L[a * 3 + 1] * p2;
                                const T t = L[a * 3 + 2] * pw;
#pragma unroll
                                for (int q = 0; q < 3; ++q)
                                    acc[o1][q][a] = acc[o1][q][a] + wz[q] * u + dwz[q] * t;
                            }
                        } else { // gv_z, gvold_xyz
                            const T u = pw * av[2] + L[6] * p1 + L[7] * p2;
                            const T t = L[8] * pw;
                            T ui[3];
#pragma unroll
                            for (int a = 0; a < 3; ++a)
                                ui[a] = pw * iv[a];
#pragma unroll
                            for (int q = 0; q < 3; ++q) {
                                acc[o1][q][0] = acc[o1][q][0] + wz[q] * u + dwz[q] * t;
#pragma unroll
                                for (int a = 0; a < 3; ++a)
                                    acc[o1][q][1 + a] = acc[o1][q][1 + a] - wz[q] * ui[a];
                            }
                        }
                    }
                } else {
#pragma unroll
                for (int o1 = 0; o1 < 3; ++o1) {
                    // grad phi = (p1 wz, p2 wz, pw dwz) with pw = wx wy, p1 = dwx wy, p2 = wx dwy
                    const T pw = wx * wy[o1], p1 = dwx * wy[o1], p2 = wx * dwy[o1];
                    T u[3], t[3], ui[3];
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        u[a] = pw * av[a] + L[a * 3 + 0] * p1 + L[a * 3 + 1] * p2;
                        t[a] = L[a * 3 + 2] * pw;
                        ui[a] = pw * iv[a];
                    }
#pragma unroll
                    for (int q = 0; q < 3; ++q)
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            acc[o1][q][a] = acc[o1][q][a] + wz[q] * u[a] + dwz[q] * t[a];
                            acc[o1][q][3 + a] = acc[o1][q][3 + a] - wz[q] * ui[a];
                        }
                }
                }
            }
            if (it_last[j])
                emit_and_reduce(it_lvl[j]);
        }
        cp_async_wait_all();
        __syncthreads();
        emit_and_reduce(B);
        __syncthreads();
        emit_and_reduce(B + 1);
    }
    wq_finish(wq);
}

// ---- K5b, warp-specialized (3-D PIC / FLIP / blend): k_adj_scatter_pipe3's arithmetic, tiles
// and fixed sum order (bit-identical), with k_p2g_ws's split by role: 2 producer warps pull the
// blocks, gather fx through the permutation and copy the (sorted-order) scatter records a, inc, L
// with cp.async into one of two record buffers, convert fx, count the columns and publish the item
// on an mbarrier; the 6 consumer warps (up to 255 registers: 8 warps, 2 per SM sub-partition) only
// march and emit node planes (slots + fixed-order sums between named barriers of their own).
template <class T> struct AdjScatterWsCfg {
    static constexpr int CONS = 192, PROD = 64, THREADS = CONS + PROD;
    static constexpr int NBC = 64, NSRC = 9, NRAW = 18, MAXIT = 64, CAP = 512, NF = 6;
    static constexpr size_t SMEM_RAW = sizeof(T) * 2 * NRAW * CAP;
    static constexpr size_t SMEM = SMEM_RAW + sizeof(T) * Cfg<3>::NCOL * NSRC * NF;
};

template <class T>
__global__ void __launch_bounds__(AdjScatterWsCfg<T>::THREADS, 1)
    k_adj_scatter_ws(DevScene<T, 3> sc, PBuf<T, 3> P, SBuf<T, 3> Sb, const int* __restrict__ perm,
                     const int* __restrict__ keys, const int* __restrict__ bstart, const int* __restrict__ bend,
                     const int* __restrict__ lstart, const int* __restrict__ occ, const int* __restrict__ n_occ,
                     T* __restrict__ partials, const DevStatus* st, int* __restrict__ wq)
{
    using C = Cfg<3>;
    using S = AdjScatterWsCfg<T>;
    constexpr int B = C::B, TE = C::TE, NF = S::NF, CAP = S::CAP, NBC = S::NBC, NSRC = S::NSRC, NRAW = S::NRAW;
    constexpr int CONS = S::CONS;
    constexpr int RX = 0, RA = 3, RI = 6, RL = 9; // raw rows: fx, a, inc, L (row-major a*3+b)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* raw = reinterpret_cast<T*>(smem_raw);                 // [2][NRAW][CAP]
    T* slots = reinterpret_cast<T*>(smem_raw + S::SMEM_RAW); // [NCOL][NSRC][NF]
    __shared__ int cnt_s[2][NBC];
    __shared__ int4 desc_s[2]; // (Q, level, flags: 1 level done, 2 block done, 4 end, -)
    __shared__ __align__(8) unsigned long long bar_full[2], bar_empty[2];
    __shared__ int it_start[S::MAXIT], it_len[S::MAXIT], it_lvl[S::MAXIT], it_last[S::MAXIT]; // producers only
    __shared__ int blk_s[4];                                                                   // w, Q, s0, nit
    const int tid = threadIdx.x;
    const int nocc = st->abort ? 0 : *n_occ;
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar_full[i], S::PROD);
            mbar_init(&bar_empty[i], CONS / 32);
        }
    }
    __syncthreads();

    if (tid >= CONS) { // ================= producer warps =================
        const int pt = tid - CONS;
        const long long SI = P.S;
        int w = 0;
        if (pt == 0)
            w = wq_first(wq);
        int j = 0;
        for (;;) {
            if (pt == 0) {
                blk_s[0] = w;
                if (w < nocc) { // level starts -> work items (as k_adj_scatter_pipe3)
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
                    blk_s[1] = Q;
                    blk_s[2] = s0;
                    blk_s[3] = k > S::MAXIT ? 0 : k; // the forward refused this block already (far_flag)
                    w = wq_next(wq, w);
                }
            }
            named_bar(2, S::PROD);
            const bool done = blk_s[0] >= nocc;
            const int Q = blk_s[1], s0 = blk_s[2], nit = done ? 1 : blk_s[3];
            for (int i = 0; i < nit; ++i, ++j) {
                const int b = j & 1, u = j >> 1;
                constexpr int RPT = CAP / S::PROD;
                const int len = done ? 0 : it_len[i], base = s0 + (done ? 0 : it_start[i]);
                int pr[RPT], kr[RPT];
#pragma unroll
                for (int e = 0; e < RPT; ++e) {
                    const int r = pt + e * S::PROD;
                    pr[e] = r < len ? perm[base + r] : 0;
                    kr[e] = r < len ? keys[base + r] : 0;
                }
                if (u > 0)
                    mbar_wait<true>(&bar_empty[b], (u - 1) & 1);
                if (done) {
                    if (pt == 0)
                        desc_s[b] = make_int4(-1, 0, 4, 0);
                    mbar_arrive(&bar_full[b]);
                    break;
                }
                cnt_s[b][pt] = 0; // PROD == NBC
                named_bar(2, S::PROD);
                T* rb = raw + b * NRAW * CAP;
#pragma unroll
                for (int e = 0; e < RPT; ++e) {
                    const int r = pt + e * S::PROD;
                    if (r < len) {
                        const T* q = P.base + pr[e];
                        const int g = base + r;
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            cp_async_t<T>(rb + (RX + a) * CAP + r, q + a * SI); // x (PLay field 0..2)
                            cp_async_t<T>(rb + (RA + a) * CAP + r, Sb.a[a] + g);
                            cp_async_t<T>(rb + (RI + a) * CAP + r, Sb.inc[a] + g);
                        }
#pragma unroll
                        for (int k = 0; k < 9; ++k)
                            cp_async_t<T>(rb + (RL + k) * CAP + r, Sb.L[k] + g);
                        atomicAdd(&cnt_s[b][kr[e] & (NBC - 1)], 1);
                    }
                }
                cp_async_commit();
                cp_async_wait_all();
                for (int r = pt; r < len; r += S::PROD) {
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const T uu = (rb[(RX + a) * CAP + r] - sc.origin[a]) * sc.inv_dh;
                        rb[(RX + a) * CAP + r] = uu - dfloor<T>(uu - T(0.5));
                    }
                }
                if (pt == 0)
                    desc_s[b] = make_int4(Q, it_lvl[i], (it_last[i] ? 1 : 0) | (i == nit - 1 ? 2 : 0), 0);
                mbar_arrive(&bar_full[b]);
            }
            if (done)
                break;
            named_bar(2, S::PROD);
        }
        if (wq && pt == 0) { // wq_finish
            __threadfence();
            if (atomicAdd(wq + 1, 1) == int(gridDim.x) - 1) {
                atomicExch(wq, 0);
                atomicExch(wq + 1, 0);
            }
        }
        return;
    }

    // ================= consumers (k_adj_scatter_pipe3's lane mapping) =================
    const int bc = tid / 3, o0 = tid % 3;
    const bool mid = o0 == 1;
    const T xoff = o0 == 0 ? T(1.5) : (o0 == 1 ? T(1) : T(0.5));
    const int bc0 = bc >> C::LOGB, bc1 = bc & (B - 1);
    const int lane = tid & 31;
    T acc[3][3][NF];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int f = 0; f < NF; ++f)
                acc[a][k][f] = T(0);
    auto emit = [&](int z, int Q) {
        named_bar(1, CONS); // the previous sums are done reading the slots
#pragma unroll
        for (int o1 = 0; o1 < 3; ++o1) {
            const int ncol = (bc0 + o0) * TE + bc1 + o1;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                slots[(ncol * NSRC + o0 * 3 + o1) * NF + f] = acc[o1][0][f];
                acc[o1][0][f] = acc[o1][1][f];
                acc[o1][1][f] = acc[o1][2][f];
                acc[o1][2][f] = T(0);
            }
        }
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
                    sum += slots[(c * NSRC + q) * NF + f];
            }
            part[f * C::TN + z * C::NCOL + c] = sum; // the adjoint partial-tile layout (k_adj_grid)
        }
    };
    for (int j = 0;; ++j) {
        const int b = j & 1;
        mbar_wait(&bar_full[b], (j >> 1) & 1);
        const int4 d = desc_s[b];
        if (d.z & 4)
            break;
        int kb, ke;
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
        for (int k = kb; k < ke; ++k) {
            const T fx = R[(RX + 0) * CAP + k], fy = R[(RX + 1) * CAP + k], fz = R[(RX + 2) * CAP + k];
            T wx, dwx, wy[3], dwy[3], wz[3], dwz[3];
            {
                const T h = fx - xoff;
                const T hh = h * h;
                wx = mid ? T(0.75) - hh : T(0.5) * hh;
                dwx = (mid ? -T(2) * h : h) * sc.inv_dh;
            }
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                quad_w<T>(fy, q, sc.inv_dh, wy[q], dwy[q]);
                quad_w<T>(fz, q, sc.inv_dh, wz[q], dwz[q]);
            }
            T av[3], iv[3], L[9];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                av[a] = R[(RA + a) * CAP + k];
                iv[a] = R[(RI + a) * CAP + k];
            }
#pragma unroll
            for (int q = 0; q < 9; ++q)
                L[q] = R[(RL + q) * CAP + k];
#pragma unroll
            for (int o1 = 0; o1 < 3; ++o1) {
                // grad phi = (p1 wz, p2 wz, pw dwz) with pw = wx wy, p1 = dwx wy, p2 = wx dwy
                const T pw = wx * wy[o1], p1 = dwx * wy[o1], p2 = wx * dwy[o1];
                T u[3], t[3], ui[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    u[a] = pw * av[a] + L[a * 3 + 0] * p1 + L[a * 3 + 1] * p2;
                    t[a] = L[a * 3 + 2] * pw;
                    ui[a] = pw * iv[a];
                }
#pragma unroll
                for (int q = 0; q < 3; ++q)
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        acc[o1][q][a] = acc[o1][q][a] + wz[q] * u[a] + dwz[q] * t[a];
                        acc[o1][q][3 + a] = acc[o1][q][3 + a] - wz[q] * ui[a];
                    }
            }
        }
        __syncwarp();
        if (lane == 0)
            mbar_arrive(&bar_empty[b]);
        if (d.z & 1)
            emit(d.y, d.x);
        if (d.z & 2) {
            emit(B, d.x);
            emit(B + 1, d.x);
        }
    }
}

// ---- K6: per node: sum partials, correction-chain VJP, momentum-update transpose ------------
// a node's friction-gradient terms: at most one segment per Coulomb wall it lies in the band of
template <class T, int D> struct FricAcc {
    int n = 0;
    int k[2 * D];
    T v[2 * D];
    __device__ __forceinline__ void add(int slot, T x)
    {
        for (int i = 0; i < n; ++i)
            if (k[i] == slot) {
                v[i] += x;
                return;
            }
        k[n] = slot;
        v[n] = x;
        ++n;
    }
    __device__ __forceinline__ T get(int slot) const
    {
        T r = T(0);
        for (int i = 0; i < n; ++i)
            if (k[i] == slot)
                r = v[i];
        return r;
    }
};
template <class T, int D>
__device__ __forceinline__ void corr_vjp_chain(const DevScene<T, D>& sc, const int* n, const T* vtilde, T* cot,
                                               FricAcc<T, D>& fr_acc)
{
    // forward replay of the chain (contact.hpp:141-224): record inputs of each correction
    constexpr int MAXC = 2 * D + MAX_OBST + 2 * D;
    struct Rec {
        int kind; // 0 slip, 1 zero, 2 obstacle, 3 coulomb
        int axis;
        T nrm;    // normal sign along `axis` (obstacle / coulomb normals are axis-aligned)
        T mu;
        int fidx;
        T vin[D];
    };
    Rec rec[MAXC];
    int nc = 0;
    T v[D];
#pragma unroll
    for (int a = 0; a < D; ++a)
        v[a] = vtilde[a];
    for (int w = 0; w < 2 * D; ++w) {
        const int kind = sc.wall_kind[w];
        if (kind == 3)
            continue;
        const int a = w / 2;
        const bool in = (w % 2 == 0) ? n[a] < sc.band : n[a] > sc.cells[a] - sc.band;
        if (!in)
            continue;
        Rec& r = rec[nc++];
        r.kind = kind == 0 ? 0 : 1;
        r.axis = a;
#pragma unroll
        for (int b = 0; b < D; ++b)
            r.vin[b] = v[b];
        if (kind == 0)
            v[a] = T(0);
        else
#pragma unroll
            for (int b = 0; b < D; ++b)
                v[b] = T(0);
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
                const T dlo = xp[a] - sc.obst[ob][a];
                const T dhi = sc.obst[ob][D + a] - xp[a];
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
            Rec& r = rec[nc++];
            r.kind = 2;
            r.axis = best_a;
            r.nrm = best_s == 0 ? T(-1) : T(1);
#pragma unroll
            for (int b = 0; b < D; ++b)
                r.vin[b] = v[b];
            const T vn = v[best_a] * r.nrm;
            if (vn < T(0))
#pragma unroll
                for (int b = 0; b < D; ++b)
                    v[b] = v[b] - vn * (b == best_a ? r.nrm : T(0));
        }
    }
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
        Rec& r = rec[nc++];
        r.kind = 3;
        r.axis = a;
        r.nrm = (w % 2 == 0) ? T(-1) : T(1);
        r.mu = sc.fric[sc.fric_off[w] + k];
        r.fidx = sc.fric_off[w] + k;
#pragma unroll
        for (int b = 0; b < D; ++b)
            r.vin[b] = v[b];
        T vn = v[a] * r.nrm;
        if (vn <= T(0))
            continue;
        T t[D], t2 = T(0);
#pragma unroll
        for (int b = 0; b < D; ++b) {
            t[b] = v[b] - vn * (b == a ? r.nrm : T(0));
            t2 += t[b] * t[b];
        }
        const T tn = dsqrt<T>(t2);
        if (tn <= r.mu * vn) {
#pragma unroll
            for (int b = 0; b < D; ++b)
                v[b] = T(0);
        } else {
            const T s = r.mu * vn / tn;
#pragma unroll
            for (int b = 0; b < D; ++b)
                v[b] = t[b] - s * t[b];
        }
    }
    // reverse (node_correction_vjp, adjoint.hpp:114-150)
    for (int q = nc - 1; q >= 0; --q) {
        const Rec& r = rec[q];
        if (r.kind == 0) {
            cot[r.axis] = T(0);
        } else if (r.kind == 1) {
#pragma unroll
            for (int b = 0; b < D; ++b)
                cot[b] = T(0);
        } else if (r.kind == 2) {
            const T vn = r.vin[r.axis] * r.nrm;
            if (vn < T(0)) {
                const T ncd = r.nrm * cot[r.axis];
                cot[r.axis] = cot[r.axis] - r.nrm * ncd;
            }
        } else {
            T vn = T(0);
#pragma unroll
            for (int b = 0; b < D; ++b)
                vn += r.vin[b] * (b == r.axis ? r.nrm : T(0));
            if (vn <= T(0))
                continue;
            T t[D], t2 = T(0);
#pragma unroll
            for (int b = 0; b < D; ++b) {
                t[b] = r.vin[b] - vn * (b == r.axis ? r.nrm : T(0));
                t2 += t[b] * t[b];
            }
            const T tn = dsqrt<T>(t2);
            if (tn <= r.mu * vn) {
#pragma unroll
                for (int b = 0; b < D; ++b)
                    cot[b] = T(0);
                continue;
            }
            const T s = T(1) - r.mu * vn / tn;
            T that[D], tc = T(0), ncd = T(0), thc = T(0);
#pragma unroll
            for (int b = 0; b < D; ++b) {
                that[b] = t[b] / tn;
                tc += t[b] * cot[b];
                ncd += (b == r.axis ? r.nrm : T(0)) * cot[b];
                thc += that[b] * cot[b];
            }
            T out[D];
#pragma unroll
            for (int b = 0; b < D; ++b) {
                const T nb = b == r.axis ? r.nrm : T(0);
                out[b] = s * (cot[b] - nb * ncd) + tc * (-(r.mu / tn) * nb + (r.mu * vn / (tn * tn)) * that[b]);
            }
            fr_acc.add(r.fidx, -vn * thc);
#pragma unroll
            for (int b = 0; b < D; ++b)
                cot[b] = out[b];
        }
    }
}

// MODE (slab decomposition): ADJ_FULL every node; ADJ_BAND_SUM halo-band nodes only, partial
// sums of the v / v_old cotangents parked in GC.gmom / GC.gf for the exchange; ADJ_INTERIOR the
// other nodes; ADJ_BAND_LOAD band nodes from the exchanged sums. Friction gradients count only
// nodes this rank owns (x in [slab_lo, slab_hi)), so a band node is not counted twice.
enum AdjGridMode { ADJ_FULL = 0, ADJ_BAND_SUM = 1, ADJ_INTERIOR = 2, ADJ_BAND_LOAD = 3 };

template <class T, int D, int MODE = ADJ_FULL>
__global__ void __launch_bounds__(Cfg<D>::NB) k_adj_grid(DevScene<T, D> sc, GBuf<T, D> G, GCBuf<T, D> GC,
                                                         const T* __restrict__ partials, const int* __restrict__ bstart,
                                                         const int* __restrict__ act, const int* __restrict__ n_act,
                                                         T* __restrict__ fr_block, const DevStatus* st)
{
    using C = Cfg<D>;
    constexpr int NF = 2 * D;
    static_assert(MAX_FRIC <= 64, "segment slots are tracked in a 64-bit mask");
    __shared__ T red[C::NB];
    __shared__ unsigned long long fr_mask;
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
    int nfr = 0;
    for (int w = 0; w < 2 * D; ++w)
        nfr += sc.n_fric[w];
    for (int wq = blockIdx.x; wq < nact; wq += gridDim.x) {
        const int q = act[wq];
        int qc[D], n[D];
        block_coords<D>(q, sc.nnb, qc);
        if constexpr (MODE == ADJ_BAND_SUM || MODE == ADJ_BAND_LOAD) { // block-uniform skip
            const int x0 = qc[0] * C::B;
            if (!((sc.band_lo + 1 >= x0 && sc.band_lo < x0 + C::B) || (sc.band_hi + 1 >= x0 && sc.band_hi < x0 + C::B)))
                continue;
        }
        bool inside = true;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            n[a] = qc[a] * C::B + lc[a];
            inside &= n[a] <= sc.cells[a];
        }
        const bool band = in_band<T, D>(sc, n[0]);
        const bool mine = MODE == ADJ_FULL || ((MODE == ADJ_INTERIOR) ? !band : band);
        const bool owned = n[0] >= sc.slab_lo && (n[0] < sc.slab_hi || sc.slab_hi >= sc.cells[0]);
        if constexpr (MODE == ADJ_BAND_SUM) { // no block reductions in this mode: per-thread skip
            if (!mine)
                continue;
        }
        const size_t gi = (size_t)q * C::NB + tid;
        T gv[D], gvo[D];
#pragma unroll
        for (int a = 0; a < D; ++a)
            gv[a] = gvo[a] = T(0);
        if constexpr (MODE == ADJ_BAND_LOAD) {
            if (mine) {
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    gv[a] = GC.gmom[a][gi];
                    gvo[a] = GC.gf[a][gi];
                }
            }
        }
        // every source's bstart entry loaded up front (independent loads in flight together)
        int bsrc[1 << D];
#pragma unroll
        for (int s = 0; s < (1 << D); ++s) {
            int Qid = 0;
            bool okb = MODE != ADJ_BAND_LOAD && mine;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const int Qa = qc[a] - ((s >> (D - 1 - a)) & 1);
                okb &= Qa >= 0 && Qa < sc.nb[a];
                Qid = Qid * sc.nb[a] + Qa;
            }
            bsrc[s] = okb ? bstart[Qid] : -1;
        }
#pragma unroll
        for (int s = 0; s < (MODE == ADJ_BAND_LOAD ? 0 : (1 << D)); ++s) {
            if (!mine)
                break;
            int Qid = 0, colx = 0, z = 0;
            bool ok = true;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const int sa = (s >> (D - 1 - a)) & 1;
                const int Qa = qc[a] - sa;
                const int t = n[a] - Qa * C::B;
                ok &= Qa >= 0 && Qa < sc.nb[a] && t < C::TE;
                Qid = Qid * sc.nb[a] + Qa;
                if (a == D - 1)
                    z = t;
                else
                    colx = colx * C::TE + t;
            }
            if (!ok || bsrc[s] < 0)
                continue;
            const T* part = partials + (size_t)Qid * NF * C::TN + z * C::NCOL + colx;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                gv[a] += part[a * C::TN];
                gvo[a] += part[(D + a) * C::TN];
            }
        }
        if constexpr (MODE == ADJ_BAND_SUM) { // park the partial sums for the halo exchange
#pragma unroll
            for (int a = 0; a < D; ++a) {
                GC.gmom[a][gi] = gv[a];
                GC.gf[a][gi] = gvo[a];
            }
            continue;
        }
        const T m = G.m[gi];
        FricAcc<T, D> fr_acc;
        T gm = T(0), gmom[D], gf[D];
#pragma unroll
        for (int a = 0; a < D; ++a)
            gmom[a] = gf[a] = T(0);
        if (mine && inside && m > sc.mass_eps) {
            T p[D], f[D], vt[D];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                p[a] = G.p[a][gi];
                f[a] = G.f[a][gi];
            }
            // v_tilde = v_old + (dt/m) f, recomputed with the forward's arithmetic (k_grid)
            const T sdt = sc.dt / m;
#pragma unroll
            for (int a = 0; a < D; ++a)
                vt[a] = p[a] / m + sdt * f[a];
            corr_vjp_chain<T, D>(sc, n, vt, gv, fr_acc);
            T uc[D];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                uc[a] = gvo[a] + gv[a];
                gf[a] = (sc.dt / m) * gv[a];
                gmom[a] = uc[a] / m;
            }
            T pu = T(0), fv = T(0);
#pragma unroll
            for (int a = 0; a < D; ++a) {
                pu += p[a] * uc[a];
                fv += f[a] * gv[a];
            }
            gm = -(pu) / (m * m) - sc.dt * (fv) / (m * m);
        }
        if (mine) {
            GC.gm[gi] = gm;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                GC.gmom[a][gi] = gmom[a];
                GC.gf[a][gi] = gf[a];
            }
        }
        if (!owned)
            fr_acc.n = 0;
        // friction gradient partials per node block: a fixed-order tree per segment slot the block
        // touched (a block meets at most a few of a wall's segments); untouched slots are zero.
        // The band pass adds to the interior pass's value of the same block.
        if (nfr > 0) {
            __syncthreads(); // the previous block's readers of fr_mask are done
            if (tid == 0)
                fr_mask = 0ull;
            __syncthreads();
            for (int i = 0; i < fr_acc.n; ++i)
                atomicOr(&fr_mask, 1ull << fr_acc.k[i]);
            __syncthreads();
            const unsigned long long mask = fr_mask;
            if constexpr (MODE != ADJ_BAND_LOAD) {
                if (tid < nfr && !((mask >> tid) & 1ull))
                    fr_block[(size_t)q * MAX_FRIC + tid] = T(0);
            }
            for (unsigned long long rest = mask; rest; rest &= rest - 1) {
                const int k = __ffsll((long long)rest) - 1;
                const T s = block_sum_fixed<T, C::NB>(fr_acc.get(k), red);
                if (tid == 0) {
                    if constexpr (MODE == ADJ_BAND_LOAD)
                        fr_block[(size_t)q * MAX_FRIC + k] += s;
                    else
                        fr_block[(size_t)q * MAX_FRIC + k] = s;
                }
            }
        }
    }
}

// ---- K7: P2G transpose gather (adjoint.hpp:479-524) -----------------------------------------
template <class T, int D, bool AFF>
__global__ void __launch_bounds__(256) k_adj_p2gT(DevScene<T, D> sc, PBuf<T, D> Pin, GCBuf<T, D> GC,
                                                  const int* __restrict__ perm, const int* __restrict__ bstart,
                                                  const int* __restrict__ bend, const int* __restrict__ occ,
                                                  const int* __restrict__ n_occ, CBuf<T, D> ci, const DevStatus* st, int* __restrict__ wq)
{
    using C = Cfg<D>;
    constexpr int TE = C::TE, TN = C::TN; // tile fields: 1 + 2 D
    extern __shared__ unsigned char smem_raw[];
    T* tile = reinterpret_cast<T*>(smem_raw); // [NF][TN]: gm, gmom[D], gf[D]
    // x and v of the thread's next particle: cp.async one iteration ahead into slot (slot ^ 1)
    constexpr int NT = 256;
    T* xst = tile + (1 + 2 * D) * TN + threadIdx.x; // [2][2D][NT]
    auto issue_x = [&](int slot, int src) {
#pragma unroll
        for (int a = 0; a < D; ++a) {
            cp_async_t<T>(xst + (slot * 2 * D + a) * NT, Pin.x[a] + src);
            cp_async_t<T>(xst + (slot * 2 * D + D + a) * NT, Pin.v[a] + src);
        }
    };
    __shared__ int w_s; // next list entry (work counter, common.cuh)
    const int nocc = st->abort ? 0 : *n_occ; // every CTA still passes wq_finish
    if (threadIdx.x == 0)
        w_s = wq_first(wq);
    for (;;) {
        cp_async_wait_all();
        __syncthreads(); // w_s published; the previous block's shared-memory readers are done
        const int w = w_s;
        if (w >= nocc)
            break;
        const int Q = occ[w];
        const int s0 = bstart[Q], s1 = bend[Q];
        // the first two particles' permutation entries in flight during the tile load
        const int i0 = s0 + int(threadIdx.x);
        int src_a = i0 < s1 ? perm[i0] : 0, src_b = i0 + NT < s1 ? perm[i0 + NT] : 0;
        int qc[D];
        block_coords<D>(Q, sc.nb, qc);
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
            tile[t] = ok ? GC.gm[gi] : T(0);
#pragma unroll
            for (int a = 0; a < D; ++a) {
                tile[(1 + a) * TN + t] = ok ? GC.gmom[a][gi] : T(0);
                tile[(1 + D + a) * TN + t] = ok ? GC.gf[a][gi] : T(0);
            }
        }
        if (i0 < s1)
            issue_x(0, src_a);
        cp_async_commit();
        __syncthreads();
        if (threadIdx.x == 0) // every thread read w_s before the barrier above
            w_s = wq_next(wq, w);
        int xslot = 0;
        for (int i = i0; i < s1; i += NT) {
            const int src = src_a; // perm[i]
            src_a = src_b;
            src_b = i + 2 * NT < s1 ? perm[i + 2 * NT] : 0;
            if (i + NT < s1)
                issue_x(xslot ^ 1, src_a);
            cp_async_commit();
            asm volatile("cp.async.wait_group 1;\n" ::: "memory"); // this particle's x, v landed
            const T* xs = xst + xslot * 2 * D * NT;
            xslot ^= 1;
            T x[D], v[D], sig[D][D];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                x[a] = xs[a * NT];
                v[a] = xs[(D + a) * NT];
            }
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
                for (int b = 0; b < D; ++b)
                    sig[a][b] = Pin.sig[sym_idx<D>(a, b)][src];
            const T mass = Pin.m[src], vol = Pin.V[src];
            // cot_in as K5a left it, read up front so that its latency overlaps the gather
            T ox[D], ov[D], oV, osg[D * D];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                ox[a] = ci.x[a][src];
                ov[a] = ci.v[a][src];
            }
            oV = ci.V[src];
#pragma unroll
            for (int k = 0; k < D * D; ++k)
                osg[k] = ci.sig[k][src];
            T w[D][3], dw[D][3];
            int tb[D], base[D];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const T u = (x[a] - sc.origin[a]) * sc.inv_dh;
                const T fl = dfloor<T>(u - T(0.5));
                const T fx = u - fl;
                const T h0 = T(1.5) - fx, h1 = fx - T(1), h2 = fx - T(0.5);
                w[a][0] = T(0.5) * h0 * h0;
                w[a][1] = T(0.75) - h1 * h1;
                w[a][2] = T(0.5) * h2 * h2;
                dw[a][0] = -h0 * sc.inv_dh;
                dw[a][1] = -T(2) * h1 * sc.inv_dh;
                dw[a][2] = h2 * sc.inv_dh;
                base[a] = int(fl);
                tb[a] = base[a] - qc[a] * C::B;
            }
            T A[D * D], Dinv[D * D];
            if constexpr (AFF) {
                if (sc.tpic) {
#pragma unroll
                    for (int k = 0; k < D * D; ++k)
                        A[k] = Pin.gv[k][src];
                } else {
                    // D = sum phi r r^T (canonical order), Dinv, A = B Dinv (adjoint.hpp:346-362)
                    T Dm[D][D];
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int b = 0; b < D; ++b)
                            Dm[a][b] = T(0);
                    for (int k = 0; k < C::NOFF; ++k) {
                        int o[D], kk = k;
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
                        for (int a = 0; a < D; ++a)
#pragma unroll
                            for (int b = 0; b < D; ++b)
                                Dm[a][b] += phi * r[a] * r[b];
                    }
                    if constexpr (D == 2) {
                        const T det = Dm[0][0] * Dm[1][1] - Dm[0][1] * Dm[1][0];
                        const T id = T(1) / det;
                        Dinv[0] = Dm[1][1] * id;
                        Dinv[1] = -Dm[0][1] * id;
                        Dinv[2] = -Dm[1][0] * id;
                        Dinv[3] = Dm[0][0] * id;
                    } else {
                        const T c00 = Dm[1][1] * Dm[2][2] - Dm[1][2] * Dm[2][1];
                        const T c01 = Dm[1][2] * Dm[2][0] - Dm[1][0] * Dm[2][2];
                        const T c02 = Dm[1][0] * Dm[2][1] - Dm[1][1] * Dm[2][0];
                        const T det = Dm[0][0] * c00 + Dm[0][1] * c01 + Dm[0][2] * c02;
                        const T id = T(1) / det;
                        Dinv[0] = c00 * id;
                        Dinv[3] = c01 * id;
                        Dinv[6] = c02 * id;
                        Dinv[1] = (Dm[0][2] * Dm[2][1] - Dm[0][1] * Dm[2][2]) * id;
                        Dinv[4] = (Dm[0][0] * Dm[2][2] - Dm[0][2] * Dm[2][0]) * id;
                        Dinv[7] = (Dm[0][1] * Dm[2][0] - Dm[0][0] * Dm[2][1]) * id;
                        Dinv[2] = (Dm[0][1] * Dm[1][2] - Dm[0][2] * Dm[1][1]) * id;
                        Dinv[5] = (Dm[0][2] * Dm[1][0] - Dm[0][0] * Dm[1][2]) * id;
                        Dinv[8] = (Dm[0][0] * Dm[1][1] - Dm[0][1] * Dm[1][0]) * id;
                    }
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int b = 0; b < D; ++b) {
                            T s = T(0);
#pragma unroll
                            for (int k = 0; k < D; ++k)
                                s += Pin.aff[a * D + k][src] * Dinv[k * D + b];
                            A[a * D + b] = s;
                        }
                }
            }
            T vcot[D], xpc[D], sigc[D * D], Vc = T(0), Ac[D * D];
#pragma unroll
            for (int a = 0; a < D; ++a)
                vcot[a] = xpc[a] = T(0);
#pragma unroll
            for (int k = 0; k < D * D; ++k)
                sigc[k] = Ac[k] = T(0);
            if constexpr (!AFF) {
                // every stencil sum of the P2G transpose as moments of the node cotangent fields:
                //   v:     m sum phi gmom
                //   sigma: -V sum gf (x) grad phi;  V: -sum (sigma grad phi).gf
                //   x:     m sum grad phi (gm + v.gmom + g.gf) - V sum H (sigma gf)
                int t0 = 0;
#pragma unroll
                for (int a = 0; a < D; ++a)
                    t0 = t0 * TE + tb[a];
                const T idh2 = sc.inv_dh * sc.inv_dh;
                {
                    Mom<T, D> m;
                    stencil_moments<T, D, false, false>(tile, t0, w, dw, idh2, m);
#pragma unroll
                    for (int a = 0; a < D; ++a)
                        xpc[a] += mass * m.g[a];
                }
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    Mom<T, D> m;
                    stencil_moments<T, D, true, false>(tile + (1 + c) * TN, t0, w, dw, idh2, m);
                    vcot[c] = mass * m.phi;
#pragma unroll
                    for (int a = 0; a < D; ++a)
                        xpc[a] += (mass * v[c]) * m.g[a];
                }
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    Mom<T, D> m;
                    stencil_moments<T, D, false, true>(tile + (1 + D + c) * TN, t0, w, dw, idh2, m);
#pragma unroll
                    for (int b = 0; b < D; ++b) {
                        sigc[c * D + b] = -vol * m.g[b];
                        Vc -= sig[c][b] * m.g[b];
                    }
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        T hs = T(0);
#pragma unroll
                        for (int b = 0; b < D; ++b)
                            hs += sig[b][c] * m.h[a][b];
                        xpc[a] += (mass * sc.gravity[c]) * m.g[a] - vol * hs;
                    }
                }
            } else {
            for (int k = 0; k < C::NOFF; ++k) {
                int o[D], kk = k, ti = 0;
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
                T H[D][D];
#pragma unroll
                for (int a = 0; a < D; ++a)
#pragma unroll
                    for (int b = a; b < D; ++b) {
                        T r = a == b ? (o[a] == 1 ? -T(2) * sc.inv_dh * sc.inv_dh : sc.inv_dh * sc.inv_dh)
                                     : dw[a][o[a]] * dw[b][o[b]];
#pragma unroll
                        for (int c = 0; c < D; ++c)
                            if (c != a && c != b)
                                r *= w[c][o[c]];
                        H[a][b] = r;
                        H[b][a] = r;
                    }
                const T gmc = tile[ti];
                T mc[D], fc[D];
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    mc[a] = tile[(1 + a) * TN + ti];
                    fc[a] = tile[(1 + D + a) * TN + ti];
                }
#pragma unroll
                for (int a = 0; a < D; ++a)
                    vcot[a] += mass * phi * mc[a];
                T vel[D];
#pragma unroll
                for (int a = 0; a < D; ++a)
                    vel[a] = v[a];
                if constexpr (AFF) {
                    T r[D];
#pragma unroll
                    for (int a = 0; a < D; ++a)
                        r[a] = (sc.origin[a] + T(base[a] + o[a]) * sc.dh) - x[a];
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        T s = T(0), sT = T(0);
#pragma unroll
                        for (int b = 0; b < D; ++b) {
                            s += A[a * D + b] * r[b];
                            sT += A[b * D + a] * mc[b];
                        }
                        vel[a] += s;
                        xpc[a] -= mass * phi * sT;
#pragma unroll
                        for (int b = 0; b < D; ++b)
                            Ac[a * D + b] += mass * phi * mc[a] * r[b];
                    }
                }
#pragma unroll
                for (int a = 0; a < D; ++a)
#pragma unroll
                    for (int b = 0; b < D; ++b)
                        sigc[a * D + b] += -vol * fc[a] * gw[b];
                T sg[D], sf[D];
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    T s1 = T(0), s2 = T(0);
#pragma unroll
                    for (int b = 0; b < D; ++b) {
                        s1 += sig[a][b] * gw[b];
                        s2 += sig[a][b] * fc[b];
                    }
                    sg[a] = s1;
                    sf[a] = s2;
                }
                T sgf = T(0), gdf = T(0), mdv = T(0);
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    sgf += sg[a] * fc[a];
                    gdf += sc.gravity[a] * fc[a];
                    mdv += mc[a] * vel[a];
                }
                Vc += -sgf;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    T hs = T(0);
#pragma unroll
                    for (int b = 0; b < D; ++b)
                        hs += H[a][b] * sf[b];
                    xpc[a] += mass * gmc * gw[a];
                    xpc[a] += mass * mdv * gw[a];
                    xpc[a] += mass * gdf * gw[a];
                    xpc[a] += -vol * hs;
                }
            }
            }
#pragma unroll
            for (int a = 0; a < D; ++a) {
                ci.v[a][src] = ov[a] + vcot[a];
                ci.x[a][src] = ox[a] + xpc[a];
            }
            ci.V[src] = oV + Vc;
#pragma unroll
            for (int k = 0; k < D * D; ++k)
                ci.sig[k][src] = osg[k] + sigc[k];
            if constexpr (AFF) {
                if (sc.tpic) {
#pragma unroll
                    for (int k = 0; k < D * D; ++k)
                        ci.gv[k][src] += Ac[k];
                } else {
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int b = 0; b < D; ++b) {
                            T s = T(0);
#pragma unroll
                            for (int k = 0; k < D; ++k)
                                s += Ac[a * D + k] * Dinv[k * D + b];
                            ci.aff[a * D + b][src] += s;
                        }
                }
            }
        }
    }
    wq_finish(wq);
}

// ---- parameter-gradient reductions (fixed order over dense block ids) ------------------------
// pg_acc[0] += sum_Q c[Q], pg_acc[1] += sum_Q mu[Q] over occupied particle blocks;
// pg_acc[2 + k] += sum_q fr[q][k] over active node blocks. One CTA, fixed chunking.
template <class T>
__global__ void __launch_bounds__(1024) k_pg_reduce(const T* __restrict__ pg_block, const int* __restrict__ bstart,
                                                    int nb_total, const T* __restrict__ fr_block,
                                                    const unsigned char* __restrict__ nflag, int nnb_total, int nfr,
                                                    int fluid, double* pg_acc)
{
    __shared__ T red[1024];
    const int nslot = 2 + nfr;
    for (int s = 0; s < nslot; ++s) {
        T acc = T(0);
        if (s < 2) {
            if (!fluid)
                continue;
            const int per = (nb_total + 1023) / 1024;
            for (int j = 0; j < per; ++j) {
                const int b = threadIdx.x * per + j;
                if (b < nb_total && bstart[b] >= 0)
                    acc += pg_block[(size_t)b * 2 + s];
            }
        } else {
            const int per = (nnb_total + 1023) / 1024;
            for (int j = 0; j < per; ++j) {
                const int q = threadIdx.x * per + j;
                if (q < nnb_total && nflag[q])
                    acc += fr_block[(size_t)q * MAX_FRIC + (s - 2)];
            }
        }
        const T tot = block_sum_fixed<T, 1024>(acc, red);
        if (threadIdx.x == 0)
            pg_acc[s] += double(tot);
    }
}

// ---- Lagrangian least-squares seeder (SPEC observe_lagrangian + loss) -------------------------
// loss += sum ||z - target||^2, cot.z[slot of pid] += 2 (z - target), z = x or v. Grid-wide: one
// selection entry per thread, per-block sums (fixed tree), then k_seed_sum adds the blocks in order.
template <class T, int D>
__global__ void __launch_bounds__(256) k_seed_lagrangian(PBuf<T, D> P, int n, const int* __restrict__ slot_of_pid,
                                                         const long long* __restrict__ sel, long long nsel,
                                                         const T* __restrict__ target, int field, CBuf<T, D> cot,
                                                         int do_cot, T* __restrict__ block_loss)
{
    __shared__ T red[256];
    T acc = T(0);
    const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (l < nsel) {
        const int pid = sel ? int(sel[l]) : int(l);
        const int s = slot_of_pid[pid]; // -1: not on this rank (slab decomposition)
#pragma unroll
        for (int a = 0; a < D; ++a) {
            if (s < 0)
                break;
            const T z = field == 0 ? P.x[a][s] : P.v[a][s];
            const T r = z - target[l * D + a];
            acc += r * r;
            if (do_cot) {
                T* zc = field == 0 ? cot.x[a] : cot.v[a];
                zc[s] += T(2) * r; // cot in the storage order of P
            }
        }
    }
    const T tot = block_sum_fixed<T, 256>(acc, red);
    if (threadIdx.x == 0)
        block_loss[blockIdx.x] = tot;
}
template <class T>
__global__ void __launch_bounds__(1024) k_seed_sum(const T* __restrict__ block_loss, int nb, double* loss_acc)
{
    __shared__ T red[1024];
    T acc = T(0);
    const int per = (nb + 1023) / 1024;
    for (int j = 0; j < per; ++j) { // contiguous ranges per thread, then a fixed tree
        const int b = threadIdx.x * per + j;
        if (b < nb)
            acc += block_loss[b];
    }
    const T tot = block_sum_fixed<T, 1024>(acc, red);
    if (threadIdx.x == 0)
        *loss_acc += double(tot);
}

// ---- Eulerian monitor regions (SPEC observe_eulerian): per-block sums of (z, 1) over the
// particles inside each region, in storage order (warp shuffles, then warps in order)
constexpr int EUL_MAXREG = 64;
template <class T, int D>
__global__ void __launch_bounds__(256) k_eul_partial(PBuf<T, D> P, int n, const T* __restrict__ centers,
                                                     const T* __restrict__ half, int nreg, int field,
                                                     T* __restrict__ partials)
{
    __shared__ T wsum[8][D + 1];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool live = i < n && P.pid[i] >= 0;
    T x[D], z[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        x[a] = live ? P.x[a][i] : T(0);
        z[a] = live ? (field == 0 ? P.x[a][i] : P.v[a][i]) : T(0);
    }
    for (int l = 0; l < nreg; ++l) {
        bool in = live;
#pragma unroll
        for (int a = 0; a < D; ++a)
            in = in && fabs(x[a] - centers[l * D + a]) <= half[l * D + a];
        T v[D + 1];
#pragma unroll
        for (int a = 0; a < D; ++a)
            v[a] = in ? z[a] : T(0);
        v[D] = in ? T(1) : T(0);
#pragma unroll
        for (int c = 0; c <= D; ++c)
            for (int o = 16; o > 0; o >>= 1)
                v[c] += __shfl_down_sync(0xffffffffu, v[c], o);
        __syncthreads();
        if (lane == 0)
#pragma unroll
            for (int c = 0; c <= D; ++c)
                wsum[wid][c] = v[c];
        __syncthreads();
        if (threadIdx.x <= D) {
            T s = T(0);
            for (int w = 0; w < int(blockDim.x / 32); ++w)
                s += wsum[w][threadIdx.x];
            partials[((size_t)blockIdx.x * nreg + l) * (D + 1) + threadIdx.x] = s;
        }
    }
}

// block sums in block order -> Q_l; loss += sum_l m ||Q_l - target||^2; g_l = 2 m (Q_l - target)/|P_l|
template <class T, int D>
__global__ void k_eul_final(const T* __restrict__ partials, int nblocks, int nreg, const T* __restrict__ target,
                            const unsigned char* __restrict__ mask, T* __restrict__ g, double* loss_acc)
{
    __shared__ T term[EUL_MAXREG];
    const int l = threadIdx.x;
    if (l < nreg) {
        T s[D + 1];
#pragma unroll
        for (int c = 0; c <= D; ++c)
            s[c] = T(0);
        for (int b = 0; b < nblocks; ++b)
#pragma unroll
            for (int c = 0; c <= D; ++c)
                s[c] += partials[((size_t)b * nreg + l) * (D + 1) + c];
        const bool on = s[D] > T(0) && (!mask || mask[l]);
        T t = T(0);
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const T r = on ? s[a] / s[D] - target[l * D + a] : T(0);
            t += r * r;
            g[l * D + a] = on ? T(2) * r / s[D] : T(0);
        }
        term[l] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        T L = T(0);
        for (int k = 0; k < nreg; ++k)
            L += term[k];
        *loss_acc += double(L);
    }
}

// cot.z[i] += g_l (storage order) for every region containing the particle (region order)
template <class T, int D>
__global__ void k_eul_seed(PBuf<T, D> P, int n, const T* __restrict__ centers, const T* __restrict__ half, int nreg,
                           const T* __restrict__ g, int field, CBuf<T, D> cot)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || P.pid[i] < 0)
        return;
    T x[D];
#pragma unroll
    for (int a = 0; a < D; ++a)
        x[a] = P.x[a][i];
    for (int l = 0; l < nreg; ++l) {
        bool in = true;
#pragma unroll
        for (int a = 0; a < D; ++a)
            in = in && fabs(x[a] - centers[l * D + a]) <= half[l * D + a];
        if (in)
#pragma unroll
            for (int a = 0; a < D; ++a) {
                T* zc = field == 0 ? cot.x[a] : cot.v[a];
                zc[i] += g[l * D + a];
            }
    }
}

// cotangent views (reference layout, id order: vectors [n][d], matrices [n][d*d] column-major)
// <-> id-indexed SoA cotangents, through the context's device staging buffer
enum CotField { CF_X = 1, CF_V = 2, CF_RHO = 4, CF_VOL = 8, CF_EPS = 16, CF_SZZ = 32, CF_SIG = 64, CF_GV = 128,
                CF_AFF = 256 };
template <class T, int D>
__global__ void k_cot_in(Stage<T, D> S, CBuf<T, D> k, int n, int mask, int has_aff, const int* __restrict__ perm)
{
    // host row j pairs with the uploaded state's storage slot j; with perm the cotangent is placed
    // at the sorted slot i (perm[i] = j), the storage order of the step's output state
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const int j = perm ? perm[i] : i;
    auto get = [&](int f, int bit, size_t idx) { return (mask & bit) ? S.f[f][idx] : T(0); };
#pragma unroll
    for (int a = 0; a < D; ++a) {
        k.x[a][i] = get(S_X, CF_X, (size_t)j * D + a);
        k.v[a][i] = get(S_V, CF_V, (size_t)j * D + a);
    }
    k.rho[i] = get(S_RHO, CF_RHO, j);
    k.V[i] = get(S_VOL, CF_VOL, j);
    if (D == 2)
        k.szz[i] = get(S_SZZ, CF_SZZ, j);
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int q = 0; q < D; ++q) {
            const size_t m = (size_t)j * D * D + q * D + r; // column-major (r, q)
            k.sig[r * D + q][i] = get(S_SIG, CF_SIG, m);
            if (mask & CF_GV)
                k.gv[r * D + q][i] = S.f[S_GV][m];
            if (has_aff)
                k.aff[r * D + q][i] = get(S_AFF, CF_AFF, m);
        }
}
template <class T, int D>
__global__ void k_cot_out(Stage<T, D> S, CBuf<T, D> k, int n, int has_aff, int gv_zero)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        S.f[S_X][(size_t)i * D + a] = k.x[a][i];
        S.f[S_V][(size_t)i * D + a] = k.v[a][i];
    }
    S.f[S_RHO][i] = k.rho[i];
    S.f[S_VOL][i] = k.V[i];
    S.f[S_EPS][i] = T(0); // the eps cotangent is discarded (adjoint.hpp:399-400)
    if (D == 2)
        S.f[S_SZZ][i] = k.szz[i];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int q = 0; q < D; ++q) {
            const size_t m = (size_t)i * D * D + q * D + r;
            S.f[S_SIG][m] = k.sig[r * D + q][i];
            S.f[S_GV][m] = gv_zero ? T(0) : k.gv[r * D + q][i];
            if (has_aff)
                S.f[S_AFF][m] = k.aff[r * D + q][i];
        }
}

template <class T, int D> __global__ void k_slot_of_pid(PBuf<T, D> P, int n, int* slot_of_pid)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && P.pid[i] >= 0) // vacated slots (exported particles) carry pid -1
        slot_of_pid[P.pid[i]] = i;
}

// ---- replay tape: a step's forward grid kept from the segment replay --------------------------
// field f of the dense grid: m, p[D], f[D], v[D], v_old[D]
template <class T, int D> __device__ __forceinline__ T* grid_field(const GBuf<T, D>& G, int f)
{
    if (f == 0)
        return G.m;
    if (f <= D)
        return G.p[f - 1];
    if (f <= 2 * D)
        return G.f[f - 1 - D];
    if (f <= 3 * D)
        return G.v[f - 1 - 2 * D];
    return G.vold[f - 1 - 3 * D];
}
// SAVE: active node blocks of G -> dst[w][field][node]; LOAD: the reverse. A step whose active
// block count exceeds the slot capacity is flagged (the VJP then recomputes its grid).
template <class T, int D, bool SAVE>
__global__ void __launch_bounds__(256) k_grid_tape(GBuf<T, D> G, const int* __restrict__ act,
                                                   const int* __restrict__ n_act, T* __restrict__ tape, int cap_blocks,
                                                   int* overflow)
{
    using C = Cfg<D>;
    constexpr int NFLD = 1 + 4 * D;
    const int na = *n_act;
    if (na > cap_blocks) {
        if (SAVE && blockIdx.x == 0 && threadIdx.x == 0)
            *overflow = 1;
        return;
    }
    const long long total = (long long)na * NFLD * C::NB;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int loc = int(e % C::NB);
        const long long r = e / C::NB;
        const int f = int(r % NFLD), w = int(r / NFLD);
        T* g = grid_field<T, D>(G, f) + (size_t)act[w] * C::NB + loc;
        if (SAVE)
            tape[e] = *g;
        else
            *g = tape[e];
    }
}

// ---------------------------------------------------------------------------------------------
// Adjoint workspace + drivers (host side, templated on the context type)
template <class T, int D> struct AdjWork {
    using C = Cfg<D>;
    CBuf<T, D> cot[2]{};
    SBuf<T, D> sb{};
    GCBuf<T, D> gc{};
    T* partials = nullptr;  // 2D fields per tile node
    T* pg_block = nullptr;  // [nb_total][2]
    T* fr_block = nullptr;  // [nnb_total][MAX_FRIC]
    double* pg_acc = nullptr;
    double* loss_acc = nullptr;
    int* slot_of_pid = nullptr;
    bool gvz[2] = {true, true}; // cot[b].grad_v is known zero (not stored)
    // 3-D K5b: the warp-specialized march (default) or k_adj_scatter_pipe3 (MPM_K5B=pipe3, A/B)
    bool k5b_ws = !(std::getenv("MPM_K5B") && std::getenv("MPM_K5B")[0] == 'p');
    std::vector<void*> allocs;
    bool ready = false;
    int64_t cap = 0;

    template <class X> X* al(size_t k)
    {
        X* p = nullptr;
        if (cudaMalloc(&p, (k ? k : 1) * sizeof(X)) != cudaSuccess)
            throw std::runtime_error("adjoint workspace: cudaMalloc failed (out of device memory)");
        allocs.push_back(p);
        return p;
    }

    template <class Ctx> void init(Ctx&) {}

    template <class Ctx> void ensure(Ctx& c)
    {
        if (ready)
            return;
        cap = c.cap;
        for (int b = 0; b < 2; ++b) {
            auto& k = cot[b];
            for (int a = 0; a < D; ++a) {
                k.x[a] = al<T>(cap);
                k.v[a] = al<T>(cap);
            }
            k.rho = al<T>(cap);
            k.V = al<T>(cap);
            k.eps = nullptr; // discarded cotangent (adjoint.hpp:399-400): never stored
            k.szz = D == 2 ? al<T>(cap) : nullptr;
            for (int q = 0; q < D * D; ++q) {
                k.sig[q] = al<T>(cap);
                k.gv[q] = al<T>(cap);
                k.aff[q] = c.has_aff ? al<T>(cap) : nullptr;
            }
        }
        for (int a = 0; a < D; ++a) {
            sb.a[a] = al<T>(cap);
            sb.inc[a] = al<T>(cap);
        }
        for (int q = 0; q < D * D; ++q) {
            sb.L[q] = al<T>(cap);
            sb.Bc[q] = c.has_aff ? al<T>(cap) : nullptr;
        }
        const size_t nodes = (size_t)c.sc.nnb_total * C::NB;
        gc.gm = al<T>(nodes);
        for (int a = 0; a < D; ++a) {
            gc.gmom[a] = al<T>(nodes);
            gc.gf[a] = al<T>(nodes);
        }
        partials = al<T>((size_t)c.sc.nb_total * 2 * D * C::TN);
        pg_block = al<T>((size_t)c.sc.nb_total * 2);
        fr_block = al<T>((size_t)c.sc.nnb_total * MAX_FRIC);
        pg_acc = al<double>(PG_SLOTS);
        loss_acc = al<double>(1);
        slot_of_pid = al<int>(cap);
        ready = true;
        set_attrs(c);
    }

    void free_all()
    {
        for (void* p : allocs)
            cudaFree(p);
        allocs.clear();
        ready = false;
    }

    template <class Ctx> void set_attrs(Ctx& c)
    {
        if (!ready)
            return;
        const int sm5 = int(K5aStage<D>::template smem<T>()), sm7 = int(sizeof(T) * ((1 + 2 * D) * C::TN + 2 * 2 * D * 256));
        cudaFuncSetAttribute(k_adj_g2pT_gather<T, D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm5);
        cudaFuncSetAttribute(k_adj_g2pT_gather<T, D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm5);
        cudaFuncSetAttribute(k_adj_p2gT<T, D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm7);
        cudaFuncSetAttribute(k_adj_p2gT<T, D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm7);
        if constexpr (D == 3) {
            cudaFuncSetAttribute(k_adj_scatter_pipe3<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(AdjScatterCfg<T>::SMEM));
            cudaFuncSetAttribute(k_adj_scatter_ws<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(AdjScatterWsCfg<T>::SMEM));
        }
        (void)c;
    }

    // upload / download a host cotangent view (reference layout, id order) <-> cot[b]
    // perm: place row j at the sorted slot i with perm[i] = j (cot_out of a step whose replay has
    // sorted the input state); nullptr: storage order of the uploaded state
    template <class Ctx> void cot_upload(Ctx& c, const mpm_cot_view* v, int b, const int* perm)
    {
        const int64_t n = c.n;
        if (n == 0)
            return;
        const void* src[S_NFIELDS] = {v->x, v->v, nullptr, v->volume, v->rho, nullptr, D == 2 ? v->sigma_zz : nullptr,
                                      v->sigma, v->grad_v, c.has_aff ? v->affine : nullptr, nullptr};
        const int bit[S_NFIELDS] = {CF_X, CF_V, 0, CF_VOL, CF_RHO, 0, CF_SZZ, CF_SIG, CF_GV, CF_AFF, 0};
        int mask = 0;
        for (int f = 0; f < S_NFIELDS; ++f)
            if (src[f]) {
                c.copy_async(c.stage.f[f], src[f], (size_t)n * stage_comps<D>(f) * sizeof(T),
                             cudaMemcpyHostToDevice);
                mask |= bit[f];
            }
        c.launch("k_cot_in", [&] {
            k_cot_in<T, D><<<c.grid_for(n, 256), 256, 0, c.stream>>>(c.stage, cot[b], int(n), mask, c.has_aff,
                                                                     perm);
        });
        gvz[b] = !(mask & CF_GV);
        c.sync(); // the staging buffer is reused by the next transfer
    }
    template <class Ctx> void cot_zero(Ctx& c, int b)
    {
        auto& k = cot[b];
        const int64_t n = c.n;
        for (int a = 0; a < D; ++a) {
            c.zero(k.x[a], n);
            c.zero(k.v[a], n);
        }
        c.zero(k.rho, n);
        c.zero(k.V, n);
        if (D == 2)
            c.zero(k.szz, n);
        for (int q = 0; q < D * D; ++q) {
            c.zero(k.sig[q], n);
            if (c.has_aff)
                c.zero(k.aff[q], n);
        }
        gvz[b] = true;
    }

    template <class Ctx> void cot_download(Ctx& c, mpm_cot_view* v, int b)
    {
        const int64_t n = c.n;
        if (n == 0)
            return;
        c.launch("k_cot_out", [&] {
            k_cot_out<T, D><<<c.grid_for(n, 256), 256, 0, c.stream>>>(c.stage, cot[b], int(n), c.has_aff, gvz[b]);
        });
        void* dst[S_NFIELDS] = {v->x, v->v, nullptr, v->volume, v->rho, v->eps_eq, D == 2 ? v->sigma_zz : nullptr,
                                v->sigma, v->grad_v, c.has_aff ? v->affine : nullptr, nullptr};
        for (int f = 0; f < S_NFIELDS; ++f)
            if (dst[f])
                c.copy_async(dst[f], c.stage.f[f], (size_t)n * stage_comps<D>(f) * sizeof(T),
                             cudaMemcpyDeviceToHost);
        c.sync();
    }

    // one reverse step on the state currently in c.buf[c.cur]: cot[bo] (out, storage order of the
    // step's output state = this replay's sort order) -> cot[bi] (in, storage order of the input)
    template <class Ctx> void vjp_enqueue(Ctx& c, int bo, int bi)
    {
        ensure(c);
        vjp_replay(c);
        vjp_reverse(c, bo, bi);
    }
    // forward replay with the full grid stored (m, p, f, v, v_old)
    template <class Ctx> void vjp_replay(Ctx& c)
    {
        c.sort_and_segment();
        c.p2g_kernel();
        c.template grid_kernel<G_SUM | G_MOM | G_CORR | G_STORE>();
    }
    template <class Ctx> void vjp_reverse(Ctx& c, int bo, int bi)
    {
        k5(c, bo, bi);
        c.launch("k_adj_grid", [&] {
            k_adj_grid<T, D><<<c.persistent(4), C::NB, 0, c.stream>>>(c.sc, c.G, gc, partials, c.bstart, c.act,
                                                                      c.counts + 1, fr_block, c.st);
        });
        k7(c, bi);
    }

    // ---- slab decomposition of step_vjp (SURVEY §8e adjoint row): the forward replay and the
    // node-cotangent sum each exchange the 2 halo planes with the x-neighbours
    template <class Ctx> void slab_vjp_begin(Ctx& c, const mpm_cot_view* co)
    {
        ensure(c);
        pg_reset(c, nullptr); // this rank's partial; the caller sums the ranks
        c.reset_status();
        c.sort_and_segment();
        cot_upload(c, co, 0, c.perm);
        c.p2g_kernel();
        c.template grid_kernel<G_BANDONLY | G_SUM | G_NOGRAV | G_STORE>();
    }
    template <class Ctx> void slab_vjp_interior(Ctx& c)
    {
        c.template grid_kernel<G_INTERIOR | G_SUM | G_MOM | G_CORR | G_STORE>();
    }
    template <class Ctx> void slab_vjp_scatter(Ctx& c)
    {
        c.template grid_kernel<G_BANDONLY | G_GRAV | G_ZEROV | G_MOM | G_CORR | G_STORE>();
        k5(c, 0, 1);
        c.launch("k_adj_grid", [&] {
            k_adj_grid<T, D, ADJ_BAND_SUM><<<c.persistent(4), C::NB, 0, c.stream>>>(
                c.sc, c.G, gc, partials, c.bstart, c.act, c.counts + 1, fr_block, c.st);
        });
    }
    HaloFields<T> cot_halo_fields() const
    {
        HaloFields<T> H{};
        H.nf = 2 * D;
        for (int a = 0; a < D; ++a) {
            H.f[a] = gc.gmom[a]; // v cotangent partial sums (parked)
            H.f[D + a] = gc.gf[a]; // v_old cotangent partial sums (parked)
        }
        return H;
    }
    template <class Ctx> void slab_vjp_finish(Ctx& c, mpm_cot_view* ci, mpm_param_grads* pg)
    {
        c.launch("k_adj_grid", [&] {
            k_adj_grid<T, D, ADJ_INTERIOR><<<c.persistent(4), C::NB, 0, c.stream>>>(
                c.sc, c.G, gc, partials, c.bstart, c.act, c.counts + 1, fr_block, c.st);
        });
        c.launch("k_adj_grid", [&] {
            k_adj_grid<T, D, ADJ_BAND_LOAD><<<c.persistent(4), C::NB, 0, c.stream>>>(
                c.sc, c.G, gc, partials, c.bstart, c.act, c.counts + 1, fr_block, c.st);
        });
        k7(c, 1);
        c.check_status(c.step);
        cot_download(c, ci, 1);
        pg_download(c, pg);
    }

    // K5a gather + constitutive VJP, K5b scatter of the v / v_old cotangents into partial tiles
    template <class Ctx> void k5(Ctx& c, int bo, int bi)
    {
        auto& Pin = c.buf[c.cur];
        const unsigned gr = c.persistent(4);
        const size_t sm5 = K5aStage<D>::template smem<T>();
        const int gvw = c.sc.tpic ? 1 : 0; // only TPIC accumulates a grad_v cotangent (K7)
        gvz[bi] = !gvw;
        if (c.has_aff)
            c.launch("k_adj_g2pT_gather", [&] {
                k_adj_g2pT_gather<T, D, true><<<gr, 256, sm5, c.stream>>>(c.sc, Pin, c.G, c.perm, c.bstart, c.bend,
                                                                           c.occ, c.counts, cot[bo], cot[bi], sb,
                                                                           pg_block, c.st, gvz[bo], gvw, c.wq_ptr(WQ_K5A));
            });
        else
            c.launch("k_adj_g2pT_gather", [&] {
                k_adj_g2pT_gather<T, D, false><<<gr, 256, sm5, c.stream>>>(c.sc, Pin, c.G, c.perm, c.bstart, c.bend,
                                                                            c.occ, c.counts, cot[bo], cot[bi], sb,
                                                                            pg_block, c.st, gvz[bo], gvw, c.wq_ptr(WQ_K5A));
            });
        const int tpb = D == 2 ? 160 : 256;
        if constexpr (D == 3) {
            if (!c.has_aff && k5b_ws) { // warp-specialized column march (as the forward P2G)
                using SW = AdjScatterWsCfg<T>;
                c.launch("k_adj_scatter", [&] {
                    k_adj_scatter_ws<T><<<c.nsm, SW::THREADS, SW::SMEM, c.stream>>>(
                        c.sc, Pin, sb, c.perm, c.keys_sorted, c.bstart, c.bend, c.lstart, c.occ, c.counts, partials,
                        c.st, c.wq_ptr(WQ_K5B));
                });
                return;
            }
            if (!c.has_aff) { // pipelined column march (as the forward P2G)
                using SC = AdjScatterCfg<T>;
                c.launch("k_adj_scatter", [&] {
                    k_adj_scatter_pipe3<T><<<c.persistent(1), SC::THREADS, SC::SMEM, c.stream>>>(
                        c.sc, Pin, sb, c.perm, c.keys_sorted, c.bstart, c.bend, c.lstart, c.occ, c.counts, partials,
                        c.st, c.wq_ptr(WQ_K5B));
                });
                return;
            }
        }
        if (c.has_aff)
            c.launch("k_adj_scatter", [&] {
                k_adj_scatter<T, D, true><<<c.persistent(8), tpb, 0, c.stream>>>(c.sc, Pin, sb, c.perm, c.keys_sorted,
                                                                                 c.bstart, c.bend, c.occ, c.counts,
                                                                                 partials, c.st);
            });
        else
            c.launch("k_adj_scatter", [&] {
                k_adj_scatter<T, D, false><<<c.persistent(8), tpb, 0, c.stream>>>(c.sc, Pin, sb, c.perm, c.keys_sorted,
                                                                                  c.bstart, c.bend, c.occ, c.counts,
                                                                                  partials, c.st);
            });
    }

    // K7 P2G-transpose gather into the particle cotangents, then the fixed-order ParamGrads reduce
    template <class Ctx> void k7(Ctx& c, int bi)
    {
        auto& Pin = c.buf[c.cur];
        const unsigned gr = c.persistent(4);
        const size_t sm7 = sizeof(T) * ((1 + 2 * D) * C::TN + 2 * 2 * D * 256); // tile + 2 slots of (x, v)
        const bool aff = c.has_aff || c.sc.tpic;
        if (aff)
            c.launch("k_adj_p2gT", [&] {
                k_adj_p2gT<T, D, true><<<gr, 256, sm7, c.stream>>>(c.sc, Pin, gc, c.perm, c.bstart, c.bend, c.occ,
                                                                   c.counts, cot[bi], c.st, c.wq_ptr(WQ_K7));
            });
        else
            c.launch("k_adj_p2gT", [&] {
                k_adj_p2gT<T, D, false><<<gr, 256, sm7, c.stream>>>(c.sc, Pin, gc, c.perm, c.bstart, c.bend, c.occ,
                                                                    c.counts, cot[bi], c.st, c.wq_ptr(WQ_K7));
            });
        int nfr = 0;
        for (int w = 0; w < 2 * D; ++w)
            nfr += c.sc.n_fric[w];
        c.launch("k_pg_reduce", [&] {
            k_pg_reduce<T><<<1, 1024, 0, c.stream>>>(pg_block, c.bstart, c.sc.nb_total, fr_block, c.nflag,
                                                     c.sc.nnb_total, nfr, c.sc.material == 0, pg_acc);
        });
    }

    template <class Ctx> void pg_reset(Ctx& c, const mpm_param_grads* pg)
    {
        double h[PG_SLOTS] = {0};
        h[0] = pg ? pg->sound_speed : 0.0;
        h[1] = pg ? pg->viscosity : 0.0;
        for (int w = 0; w < 2 * D; ++w)
            if (c.sc.wall_kind[w] == 3 && pg && pg->wall_friction[w])
                for (int k = 0; k < c.sc.n_fric[w]; ++k)
                    h[2 + c.sc.fric_off[w] + k] = pg->wall_friction[w][k];
        c.h2d_raw(pg_acc, h, sizeof(h));
    }

    template <class Ctx> void pg_download(Ctx& c, mpm_param_grads* pg)
    {
        double h[PG_SLOTS];
        c.d2h_raw(h, pg_acc, sizeof(h));
        pg->sound_speed = h[0];
        pg->viscosity = h[1];
        for (int w = 0; w < 2 * D; ++w)
            if (c.sc.wall_kind[w] == 3 && pg->wall_friction[w])
                for (int k = 0; k < c.sc.n_fric[w]; ++k)
                    pg->wall_friction[w][k] = h[2 + c.sc.fric_off[w] + k];
    }

    template <class Ctx>
    void step_vjp_api(Ctx& c, const mpm_state_view* s, const mpm_cot_view* co, mpm_cot_view* ci, mpm_param_grads* pg)
    {
        c.upload(s);
        ensure(c);
        pg_reset(c, pg);
        c.reset_status();
        vjp_replay(c);
        cot_upload(c, co, 0, c.perm);
        vjp_reverse(c, 0, 1);
        c.check_status(c.step);
        cot_download(c, ci, 1);
        pg_download(c, pg);
    }

    template <class Ctx>
    void backprop_api(Ctx& c, const mpm_state_view* s0, int64_t total, int nseg, const mpm_seeder_desc* sd,
                      mpm_cot_view* c0, mpm_param_grads* pg, mpm_backprop_result* res)
    {
        c.backprop_run(*this, s0, total, nseg, sd, c0, pg, res);
    }
};

} // namespace mpmgpu
