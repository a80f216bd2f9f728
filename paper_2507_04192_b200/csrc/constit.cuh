// constit.cuh -- constitutive updates fused into the G2P epilogue (registers only).
//
// fluid_stress_update  constitutive.hpp:32-50
// dp_stress_update     constitutive.hpp:101-164 (2-D runs on the plane-strain 3x3 embedding)
// constitutive_update  stepper.hpp:15-43 (volume / density / eps / F bookkeeping)
#pragma once

#include "common.cuh"

namespace mpmgpu {

template <class T, int D> __global__ void k_scene_consts(DevScene<T, D>* s)
{
    s->dp_lam = s->K - T(2) * s->G / T(3);
    s->dp_dlam_den = s->G + s->K * s->q_phi * s->q_psi;
    s->dp_deps_fac = dsqrt<T>(T(1) / T(3) + T(2) / T(9) * s->q_psi * s->q_psi);
    s->dp_apex = s->q_phi > T(0) ? s->k_phi / s->q_phi : T(0);
    s->dp_deps_t = dsqrt<T>(T(2)) / T(3);
    s->fl_k = s->rate_form ? s->visc / s->dt : s->visc;
}

template <class T> struct M3 {
    T a[3][3];
};

// D-P trial state and zone (constitutive.hpp:62-83, 113-124); shared with the adjoint
template <class T, int D> struct DpTrial {
    T dd[3][3], dw[3][3], S[3][3], sR[3][3], trial[3][3], dev[3][3];
    T trd, sm, tau, fs, ft, h;
    int zone; // 1 elastic, 2 shear, 3 tensile
};

// S: full 3x3 input stress (2-D: szz in (2,2)); L: velocity gradient (D x D, row-major)
template <class T, int D>
__device__ __forceinline__ void dp_trial(const DevScene<T, D>& sc, const T (&S)[3][3], const T* L, DpTrial<T, D>& t)
{
    T Lf[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            Lf[i][j] = (i < D && j < D) ? L[i * D + j] : T(0);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            t.S[i][j] = S[i][j];
            t.dd[i][j] = T(0.5) * (Lf[i][j] + Lf[j][i]) * sc.dt;
            t.dw[i][j] = T(0.5) * (Lf[i][j] - Lf[j][i]) * sc.dt;
        }
    // sR = S + S dw^T + dw S^T  (constitutive.hpp:117)
    // X = S dw^T, so that (dw S^T)_ij = X_ji: each product sum is formed once (same operands and
    // order as the two sums it replaces, so bit-identical)
    T X[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            T a = T(0);
#pragma unroll
            for (int k = 0; k < 3; ++k)
                a += S[i][k] * t.dw[j][k];
            X[i][j] = a;
        }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            t.sR[i][j] = S[i][j] + X[i][j] + X[j][i];
    t.trd = t.dd[0][0] + t.dd[1][1] + t.dd[2][2];
    const T lam = sc.dp_lam;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            t.trial[i][j] = t.sR[i][j] + T(2) * sc.G * t.dd[i][j] + (i == j ? lam * t.trd : T(0));
    t.sm = (t.trial[0][0] + t.trial[1][1] + t.trial[2][2]) / T(3);
    T f2 = T(0);
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            t.dev[i][j] = t.trial[i][j] - (i == j ? t.sm : T(0));
            f2 += t.dev[i][j] * t.dev[i][j];
        }
    t.tau = dsqrt<T>(T(0.5) * f2);
    t.fs = t.tau - sc.k_phi + sc.q_phi * t.sm;
    t.ft = t.sm - sc.sigma_t;
    t.h = t.tau - sc.tau_P - sc.alpha_P * (t.sm - sc.sigma_t);
    if (t.fs <= T(0) && t.ft < T(0))
        t.zone = 1;
    else if (t.ft < T(0))
        t.zone = 2;
    else
        t.zone = t.h > T(0) ? 2 : 3;
}

// returns den = 1 + tr(dd); writes the new stress (3x3) and delta eps
template <class T, int D>
__device__ __forceinline__ T dp_update(const DevScene<T, D>& sc, const T (&S)[3][3], const T* L, T (&out)[3][3], T& deps)
{
    DpTrial<T, D> t;
    dp_trial<T, D>(sc, S, L, t);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            out[i][j] = t.trial[i][j];
    deps = T(0);
    if (t.zone == 2) {
        T dlam = t.fs / sc.dp_dlam_den;
        deps = dlam * sc.dp_deps_fac;
        T sm_new = t.sm - sc.K * sc.q_psi * dlam;
        T tau_new = sc.k_phi - sc.q_phi * sm_new;
        if (t.tau <= T(0) || tau_new < T(0)) {
            sm_new = sc.q_phi > T(0) ? sc.dp_apex : sm_new;
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    out[i][j] = i == j ? sm_new : T(0);
        } else {
            T ratio = tau_new / t.tau;
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    out[i][j] = ratio * t.dev[i][j] + (i == j ? sm_new : T(0));
        }
        if (sm_new > sc.sigma_t) {
#pragma unroll
            for (int i = 0; i < 3; ++i)
                out[i][i] += sc.sigma_t - sm_new;
        }
    } else if (t.zone == 3) {
        T dlam_t = t.ft / sc.K;
        deps = sc.dp_deps_t * dlam_t;
#pragma unroll
        for (int i = 0; i < 3; ++i)
            out[i][i] = t.trial[i][i] + (sc.sigma_t - t.sm);
        if (t.tau > sc.tau_P) {
            T ratio = sc.tau_P / t.tau;
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    out[i][j] = ratio * t.dev[i][j] + (i == j ? sc.sigma_t : T(0));
        }
    }
    return T(1) + t.trd;
}

// Constitutive step on one particle's registers. sig: packed symmetric (in/out); L: new
// velocity gradient. Returns false on catastrophic compression (1 + tr(dd) <= 0).
template <class T, int D>
__device__ __forceinline__ bool constitutive_particle(const DevScene<T, D>& sc, T* sig, T& szz, T& rho, T& V,
                                                      T& eps, const T* L)
{
    using C = Cfg<D>;
    if (sc.material == 0) { // fluid (constitutive.hpp:32-50, stepper.hpp:18-25)
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
        T den = T(1) + trd;
        if (!(den > T(0)))
            return false;
        T rho_new = rho / den;
        T pres = sc.c * sc.c * (rho_new - sc.rho0);
        T k = sc.fl_k;
        T vis = (T(2) / T(3)) * k * trd, k2 = T(2) * k;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = i; j < D; ++j) {
                T I = i == j ? T(1) : T(0);
                sig[sym_idx<D>(i, j)] = (I * -pres - I * vis) + k2 * dd[i][j];
            }
        rho = rho_new;
        V *= den;
        return true;
    }
    // Drucker-Prager (stepper.hpp:27-37)
    T S[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            S[i][j] = (i < D && j < D) ? sig[sym_idx<D>(i, j)] : T(0);
    if (D == 2)
        S[2][2] = szz;
    T out[3][3], deps;
    T den = dp_update<T, D>(sc, S, L, out, deps);
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i; j < D; ++j)
            sig[sym_idx<D>(i, j)] = out[i][j];
    if (D == 2)
        szz = out[2][2];
    eps += deps;
    if (!(den > T(0)))
        return false;
    rho /= den;
    V *= den;
    (void)C::NS;
    return true;
}

} // namespace mpmgpu
