// mpm_oracle.cpp -- TEST INFRASTRUCTURE ONLY. Never linked into the product.
//
// An independent CPU restatement of the reference MPM step (/root/reference/proj, the
// C++ re-implementation of arXiv 2507.04192 "JAX-MPM") and of its reverse-mode adjoint,
// written without Eigen on plain fixed-size arrays. Every function cites the reference
// file:line it restates. Serial, particle-index order, like the reference. It is the
// checker for the CUDA path (tests/, __graft_entry__.smoke(), bench.py cpu_baseline); it is
// pinned by tests/test_oracle_golden.py against the reference's own known-answer tests and
// by tests/test_oracle_vs_ref.py against the reference compiled unmodified (oracle/_ref).
//
// ABI: mpm_oracle.h, prefix orc_. Built by oracle/Makefile -> oracle/_build/liboracle.so.

#include "mpm_oracle.h"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

// ---------------------------------------------------------------------------------------
// errors (common.hpp:22-36)
struct Err : std::runtime_error {
    int code;
    int64_t particle;
    Err(int c, const std::string& m, int64_t p = -1)
        : std::runtime_error(m), code(c), particle(p)
    {
    }
};

thread_local int64_t g_particle = -1;
thread_local std::string g_msg;

// ---------------------------------------------------------------------------------------
// small fixed-size linear algebra. Matrices are row-major a[i][j].
template <class T, int D> struct Vec {
    T a[D];
    T& operator[](int i) { return a[i]; }
    const T& operator[](int i) const { return a[i]; }
};
template <class T, int D> struct Mat {
    T a[D][D];
};

template <class T, int D> Vec<T, D> vzero()
{
    Vec<T, D> v;
    for (int i = 0; i < D; ++i)
        v.a[i] = T(0);
    return v;
}
template <class T, int D> Mat<T, D> mzero()
{
    Mat<T, D> m;
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j)
            m.a[i][j] = T(0);
    return m;
}
template <class T, int D> Mat<T, D> ident()
{
    Mat<T, D> m = mzero<T, D>();
    for (int i = 0; i < D; ++i)
        m.a[i][i] = T(1);
    return m;
}
template <class T, int D> T dotv(const Vec<T, D>& x, const Vec<T, D>& y)
{
    T s = T(0);
    for (int i = 0; i < D; ++i)
        s += x.a[i] * y.a[i];
    return s;
}
template <class T, int D> T normv(const Vec<T, D>& x) { return std::sqrt(dotv(x, x)); }
template <class T, int D> Vec<T, D> matvec(const Mat<T, D>& m, const Vec<T, D>& x)
{
    Vec<T, D> r;
    for (int i = 0; i < D; ++i) {
        T s = T(0);
        for (int k = 0; k < D; ++k)
            s += m.a[i][k] * x.a[k];
        r.a[i] = s;
    }
    return r;
}
template <class T, int D> Mat<T, D> matmul(const Mat<T, D>& x, const Mat<T, D>& y)
{
    Mat<T, D> r;
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
            T s = T(0);
            for (int k = 0; k < D; ++k)
                s += x.a[i][k] * y.a[k][j];
            r.a[i][j] = s;
        }
    return r;
}
template <class T, int D> Mat<T, D> transp(const Mat<T, D>& x)
{
    Mat<T, D> r;
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j)
            r.a[i][j] = x.a[j][i];
    return r;
}
template <class T, int D> T trace(const Mat<T, D>& x)
{
    T s = T(0);
    for (int i = 0; i < D; ++i)
        s += x.a[i][i];
    return s;
}
// Frobenius reductions run in Eigen's storage order (column-major): the reference's
// Jaumann-rotated stress is only symmetric up to rounding, so the order is observable.
template <class T, int D> T fro2(const Mat<T, D>& x)
{
    T s = T(0);
    for (int j = 0; j < D; ++j)
        for (int i = 0; i < D; ++i)
            s += x.a[i][j] * x.a[i][j];
    return s;
}
template <class T, int D> T contract(const Mat<T, D>& x, const Mat<T, D>& y) // sum_ij x_ij y_ij
{
    T s = T(0);
    for (int j = 0; j < D; ++j)
        for (int i = 0; i < D; ++i)
            s += x.a[i][j] * y.a[i][j];
    return s;
}
template <class T, int D> Mat<T, D> inverse(const Mat<T, D>& m)
{
    Mat<T, D> r;
    if constexpr (D == 2) {
        T det = m.a[0][0] * m.a[1][1] - m.a[0][1] * m.a[1][0];
        T inv = T(1) / det;
        r.a[0][0] = m.a[1][1] * inv;
        r.a[0][1] = -m.a[0][1] * inv;
        r.a[1][0] = -m.a[1][0] * inv;
        r.a[1][1] = m.a[0][0] * inv;
    } else {
        T c00 = m.a[1][1] * m.a[2][2] - m.a[1][2] * m.a[2][1];
        T c01 = m.a[1][2] * m.a[2][0] - m.a[1][0] * m.a[2][2];
        T c02 = m.a[1][0] * m.a[2][1] - m.a[1][1] * m.a[2][0];
        T det = m.a[0][0] * c00 + m.a[0][1] * c01 + m.a[0][2] * c02;
        T inv = T(1) / det;
        r.a[0][0] = c00 * inv;
        r.a[1][0] = c01 * inv;
        r.a[2][0] = c02 * inv;
        r.a[0][1] = (m.a[0][2] * m.a[2][1] - m.a[0][1] * m.a[2][2]) * inv;
        r.a[1][1] = (m.a[0][0] * m.a[2][2] - m.a[0][2] * m.a[2][0]) * inv;
        r.a[2][1] = (m.a[0][1] * m.a[2][0] - m.a[0][0] * m.a[2][1]) * inv;
        r.a[0][2] = (m.a[0][1] * m.a[1][2] - m.a[0][2] * m.a[1][1]) * inv;
        r.a[1][2] = (m.a[0][2] * m.a[1][0] - m.a[0][0] * m.a[1][2]) * inv;
        r.a[2][2] = (m.a[0][0] * m.a[1][1] - m.a[0][1] * m.a[1][0]) * inv;
    }
    return r;
}

// ---------------------------------------------------------------------------------------
// scene (scene.hpp:9-16 + config.hpp + material.hpp), decoded from the ABI descriptor
template <class T, int D> struct Scene {
    T dh, dt, alpha;
    int cells[D];
    T origin[D], gravity[D];
    int scheme;
    bool track_F;
    int material;
    T rho0, visc, c;
    bool rate_form;
    T K, G, q_phi, k_phi, q_psi, tau_P, alpha_P, sigma_t;
    int band;
    int wall_kind[2 * D];
    std::vector<T> friction[2 * D];
    std::vector<std::array<T, 2 * D>> obstacles;
    T mass_eps;

    bool apic() const { return scheme == MPM_SCHEME_APIC; }
    bool tpic() const { return scheme == MPM_SCHEME_TPIC; }
    // TransferScheme::flip_fraction (config.hpp:22-29)
    T flip_fraction() const
    {
        return scheme == MPM_SCHEME_FLIP ? T(1) : scheme == MPM_SCHEME_BLEND ? alpha : T(0);
    }
    int nodes(int a) const { return cells[a] + 1; }
    int64_t num_nodes() const
    {
        int64_t n = 1;
        for (int a = 0; a < D; ++a)
            n *= nodes(a);
        return n;
    }
    // Grid::node_index (state.hpp:127-133): row-major, last axis fastest
    int64_t node_index(const int* idx) const
    {
        int64_t r = 0;
        for (int a = 0; a < D; ++a)
            r = r * nodes(a) + idx[a];
        return r;
    }
    // Grid::node_multi_index (state.hpp:135-144)
    void node_multi(int64_t f, int* idx) const
    {
        for (int a = D - 1; a >= 0; --a) {
            idx[a] = int(f % nodes(a));
            f /= nodes(a);
        }
    }
    // Grid::node_position (state.hpp:146-152)
    Vec<T, D> node_pos(const int* idx) const
    {
        Vec<T, D> p;
        for (int a = 0; a < D; ++a)
            p.a[a] = origin[a] + T(idx[a]) * dh;
        return p;
    }
};

template <class T, int D> Scene<T, D> decode(const mpm_scene_desc* d)
{
    Scene<T, D> s;
    s.dh = T(d->dh);
    s.dt = T(d->dt);
    s.alpha = T(d->alpha_flip);
    for (int a = 0; a < D; ++a) {
        s.cells[a] = d->cells[a];
        s.origin[a] = T(d->origin[a]);
        s.gravity[a] = T(d->gravity[a]);
    }
    s.scheme = d->scheme;
    s.track_F = d->track_def_grad != 0;
    s.material = d->material;
    s.rho0 = T(d->rho0);
    s.visc = T(d->viscosity);
    s.c = T(d->sound_speed);
    s.rate_form = d->rate_form != 0;
    s.K = T(d->K);
    s.G = T(d->G);
    s.q_phi = T(d->q_phi);
    s.k_phi = T(d->k_phi);
    s.q_psi = T(d->q_psi);
    s.tau_P = T(d->tau_P);
    s.alpha_P = T(d->alpha_P);
    s.sigma_t = T(d->sigma_t);
    s.band = d->band_layers;
    for (int w = 0; w < 2 * D; ++w) {
        s.wall_kind[w] = d->wall_kind[w];
        for (int k = 0; k < d->n_friction[w]; ++k)
            s.friction[w].push_back(T(d->friction[w][k]));
    }
    for (int o = 0; o < d->n_obstacles; ++o) {
        std::array<T, 2 * D> b;
        for (int i = 0; i < 2 * D; ++i)
            b[i] = T(d->obstacles[o * 2 * D + i]);
        s.obstacles.push_back(b);
    }
    s.mass_eps = T(d->mass_epsilon);
    return s;
}

// ---------------------------------------------------------------------------------------
// particle state (state.hpp:17-87) in the restatement's own layout
template <class T, int D> struct State {
    int64_t n = 0;
    std::vector<Vec<T, D>> x, v;
    std::vector<T> m, V, rho, eps, szz;
    std::vector<Mat<T, D>> sig, gv, B, F;
    bool has_B = false, has_F = false;
    int64_t step = 0;
    double time = 0;
};

template <class T, int D> void load_vec(std::vector<Vec<T, D>>& dst, const void* src, int64_t n)
{
    dst.assign(n, vzero<T, D>());
    if (!src)
        return;
    const T* p = static_cast<const T*>(src);
    for (int64_t i = 0; i < n; ++i)
        for (int a = 0; a < D; ++a)
            dst[i].a[a] = p[i * D + a];
}
template <class T> void load_sc(std::vector<T>& dst, const void* src, int64_t n)
{
    dst.assign(n, T(0));
    if (src)
        std::memcpy(dst.data(), src, sizeof(T) * n);
}
// matrices arrive column-major per particle (Eigen layout)
template <class T, int D> void load_mat(std::vector<Mat<T, D>>& dst, const void* src, int64_t n)
{
    dst.assign(n, mzero<T, D>());
    if (!src)
        return;
    const T* p = static_cast<const T*>(src);
    for (int64_t i = 0; i < n; ++i)
        for (int r = 0; r < D; ++r)
            for (int c = 0; c < D; ++c)
                dst[i].a[r][c] = p[i * D * D + c * D + r];
}
template <class T, int D> void store_vec(const std::vector<Vec<T, D>>& s, void* dst)
{
    if (!dst)
        return;
    T* p = static_cast<T*>(dst);
    for (size_t i = 0; i < s.size(); ++i)
        for (int a = 0; a < D; ++a)
            p[i * D + a] = s[i].a[a];
}
template <class T> void store_sc(const std::vector<T>& s, void* dst)
{
    if (dst && !s.empty())
        std::memcpy(dst, s.data(), sizeof(T) * s.size());
}
template <class T, int D> void store_mat(const std::vector<Mat<T, D>>& s, void* dst)
{
    if (!dst)
        return;
    T* p = static_cast<T*>(dst);
    for (size_t i = 0; i < s.size(); ++i)
        for (int r = 0; r < D; ++r)
            for (int c = 0; c < D; ++c)
                p[i * D * D + c * D + r] = s[i].a[r][c];
}

template <class T, int D> State<T, D> load_state(const mpm_state_view* v)
{
    State<T, D> s;
    s.n = v->n;
    load_vec(s.x, v->x, s.n);
    load_vec(s.v, v->v, s.n);
    load_sc(s.m, v->mass, s.n);
    load_sc(s.V, v->volume, s.n);
    load_sc(s.rho, v->rho, s.n);
    load_sc(s.eps, v->eps_eq, s.n);
    load_sc(s.szz, D == 2 ? v->sigma_zz : nullptr, s.n);
    load_mat(s.sig, v->sigma, s.n);
    load_mat(s.gv, v->grad_v, s.n);
    s.has_B = v->affine != nullptr;
    load_mat(s.B, v->affine, s.n);
    s.has_F = v->def_grad != nullptr;
    load_mat(s.F, v->def_grad, s.n);
    s.step = v->step;
    s.time = v->time;
    return s;
}
template <class T, int D> void store_state(const State<T, D>& s, mpm_state_view* v)
{
    v->n = s.n;
    store_vec(s.x, v->x);
    store_vec(s.v, v->v);
    store_sc(s.m, v->mass);
    store_sc(s.V, v->volume);
    store_sc(s.rho, v->rho);
    store_sc(s.eps, v->eps_eq);
    if (D == 2)
        store_sc(s.szz, v->sigma_zz);
    store_mat(s.sig, v->sigma);
    store_mat(s.gv, v->grad_v);
    if (s.has_B)
        store_mat(s.B, v->affine);
    if (s.has_F)
        store_mat(s.F, v->def_grad);
    v->step = s.step;
    v->time = s.time;
}

// ---------------------------------------------------------------------------------------
// dense grid (state.hpp:172-254)
template <class T, int D> struct Grid {
    std::vector<T> m;
    std::vector<Vec<T, D>> p, vold, v, f;
    void reset(int64_t n)
    {
        m.assign(n, T(0));
        p.assign(n, vzero<T, D>());
        vold.assign(n, vzero<T, D>());
        v.assign(n, vzero<T, D>());
        f.assign(n, vzero<T, D>());
    }
};
template <class T, int D> Grid<T, D> load_grid(const Scene<T, D>& sc, const mpm_grid_view* g)
{
    Grid<T, D> r;
    int64_t n = sc.num_nodes();
    load_sc(r.m, g->mass, n);
    load_vec(r.p, g->momentum, n);
    load_vec(r.vold, g->v_old, n);
    load_vec(r.v, g->v, n);
    load_vec(r.f, g->force, n);
    return r;
}
template <class T, int D> void store_grid(const Scene<T, D>& sc, const Grid<T, D>& r, mpm_grid_view* g)
{
    g->num_nodes = sc.num_nodes();
    store_sc(r.m, g->mass);
    store_vec(r.p, g->momentum);
    store_vec(r.vold, g->v_old);
    store_vec(r.v, g->v);
    store_vec(r.f, g->force);
}

// ---------------------------------------------------------------------------------------
// quadratic B-spline stencil: shape_and_grad (bspline.hpp:76-108)
template <class T, int D> struct Stencil {
    int base[D];
    T w[D][3], dw[D][3], ddw[D][3];
};

template <class T, int D> Stencil<T, D> stencil(const Scene<T, D>& sc, const Vec<T, D>& x, int64_t particle)
{
    Stencil<T, D> st;
    T inv_dh = T(1) / sc.dh;
    for (int a = 0; a < D; ++a) {
        T u = (x.a[a] - sc.origin[a]) * inv_dh;
        T fl = std::floor(u - T(0.5));
        // bspline.hpp:86-91; a non-finite coordinate is out of domain (the reference's
        // int cast of NaN/inf is undefined; on x86 it yields INT_MIN < 0 -> throws)
        if (!(fl >= T(0)) || fl + T(2) > T(sc.cells[a]))
            throw Err(MPM_ERR_OUT_OF_DOMAIN,
                      "particle " + std::to_string(particle) + " outside valid grid interior on axis "
                          + std::to_string(a) + " (coordinate " + std::to_string(double(x.a[a])) + ")",
                      particle);
        int b = int(fl);
        st.base[a] = b;
        T fx = u - T(b);
        T h0 = T(1.5) - fx, h1 = fx - T(1), h2 = fx - T(0.5);
        st.w[a][0] = T(0.5) * h0 * h0;
        st.w[a][1] = T(0.75) - h1 * h1;
        st.w[a][2] = T(0.5) * h2 * h2;
        st.dw[a][0] = -h0 * inv_dh;
        st.dw[a][1] = -T(2) * h1 * inv_dh;
        st.dw[a][2] = h2 * inv_dh;
        st.ddw[a][0] = inv_dh * inv_dh;
        st.ddw[a][1] = -T(2) * inv_dh * inv_dh;
        st.ddw[a][2] = inv_dh * inv_dh;
    }
    return st;
}

// canonical offset order: row-major over {0,1,2}^D (bspline.hpp:110-127)
template <int D> void offset_of(int k, int* o)
{
    for (int a = D - 1; a >= 0; --a) {
        o[a] = k % 3;
        k /= 3;
    }
}
template <int D> constexpr int n_off() { return D == 2 ? 9 : 27; }

// Stencil::weight / Stencil::grad (bspline.hpp:50-70)
template <class T, int D> T weight(const Stencil<T, D>& st, const int* o)
{
    T r = T(1);
    for (int a = 0; a < D; ++a)
        r *= st.w[a][o[a]];
    return r;
}
template <class T, int D> Vec<T, D> grad(const Stencil<T, D>& st, const int* o)
{
    Vec<T, D> g;
    for (int a = 0; a < D; ++a) {
        T r = st.dw[a][o[a]];
        for (int b = 0; b < D; ++b)
            if (b != a)
                r *= st.w[b][o[b]];
        g.a[a] = r;
    }
    return g;
}
// detail::stencil_hessian (adjoint.hpp:95-110)
template <class T, int D> Mat<T, D> hessian(const Stencil<T, D>& st, const int* o)
{
    Mat<T, D> H;
    for (int a = 0; a < D; ++a)
        for (int b = a; b < D; ++b) {
            T r = a == b ? st.ddw[a][o[a]] : st.dw[a][o[a]] * st.dw[b][o[b]];
            for (int c = 0; c < D; ++c)
                if (c != a && c != b)
                    r *= st.w[c][o[c]];
            H.a[a][b] = r;
            H.a[b][a] = r;
        }
    return H;
}

template <class T, int D> Vec<T, D> node_rel(const Scene<T, D>& sc, const Stencil<T, D>& st, const int* o,
                                             const Vec<T, D>& xp, int* idx)
{
    for (int a = 0; a < D; ++a)
        idx[a] = st.base[a] + o[a];
    Vec<T, D> r = sc.node_pos(idx);
    for (int a = 0; a < D; ++a)
        r.a[a] -= xp.a[a];
    return r;
}

// APIC moment matrix D = sum phi r r^T recomputed from the stencil (transfer.hpp:23-31)
template <class T, int D> Mat<T, D> apic_D(const Scene<T, D>& sc, const Stencil<T, D>& st, const Vec<T, D>& xp)
{
    Mat<T, D> Dm = mzero<T, D>();
    for (int k = 0; k < n_off<D>(); ++k) {
        int o[D], idx[D];
        offset_of<D>(k, o);
        Vec<T, D> r = node_rel(sc, st, o, xp, idx);
        T w = weight(st, o);
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j)
                Dm.a[i][j] += w * r.a[i] * r.a[j];
    }
    return Dm;
}

// ---------------------------------------------------------------------------------------
// P2G (transfer.hpp:37-69): reset, then particles in index order, offsets canonical.
template <class T, int D> void p2g(const Scene<T, D>& sc, const State<T, D>& s, Grid<T, D>& g)
{
    g.reset(sc.num_nodes());
    for (int64_t p = 0; p < s.n; ++p) {
        Stencil<T, D> st = stencil(sc, s.x[p], p);
        // p2g_affine_matrix (transfer.hpp:14-32)
        Mat<T, D> A = mzero<T, D>();
        bool affine = sc.apic() || sc.tpic();
        if (sc.tpic())
            A = s.gv[p];
        else if (sc.apic())
            A = matmul(s.B[p], inverse(apic_D(sc, st, s.x[p])));
        T m = s.m[p], V = s.V[p];
        for (int k = 0; k < n_off<D>(); ++k) {
            int o[D], idx[D];
            offset_of<D>(k, o);
            Vec<T, D> r = node_rel(sc, st, o, s.x[p], idx);
            int64_t ni = sc.node_index(idx);
            T phi = weight(st, o);
            Vec<T, D> gw = grad(st, o);
            g.m[ni] += m * phi;
            Vec<T, D> vel = s.v[p];
            if (affine) {
                Vec<T, D> Ar = matvec(A, r);
                for (int a = 0; a < D; ++a)
                    vel.a[a] += Ar.a[a];
            }
            T mphi = m * phi;
            Vec<T, D> sg = matvec(s.sig[p], gw);
            for (int a = 0; a < D; ++a) {
                g.p[ni].a[a] += mphi * vel.a[a];
                g.f[ni].a[a] += -(V * sg.a[a]) + phi * m * sc.gravity[a];
            }
        }
    }
}

// grid_momentum_update (transfer.hpp:75-84)
template <class T, int D> void momentum_update(const Scene<T, D>& sc, Grid<T, D>& g)
{
    for (int64_t i = 0; i < (int64_t)g.m.size(); ++i) {
        if (g.m[i] > sc.mass_eps) {
            for (int a = 0; a < D; ++a)
                g.vold[i].a[a] = g.p[i].a[a] / g.m[i];
            T s = sc.dt / g.m[i];
            for (int a = 0; a < D; ++a)
                g.v[i].a[a] = g.vold[i].a[a] + s * g.f[i].a[a];
        }
    }
}

// ---------------------------------------------------------------------------------------
// contact / boundary corrections (contact.hpp)
enum CorrKind { C_SLIP, C_ZERO, C_OBST, C_COUL };
template <class T, int D> struct Corr {
    int kind;
    int axis;
    Vec<T, D> n;
    T mu;
    int wall, seg;
};

// node_in_wall_band (contact.hpp:17-24)
template <class T, int D> bool in_band(const Scene<T, D>& sc, const int* idx, int w)
{
    int a = w / 2;
    return w % 2 == 0 ? idx[a] < sc.band : idx[a] > sc.cells[a] - sc.band;
}
// coulomb_segment_index (contact.hpp:68-74)
template <class T> int segment_index(T coord, T lo, T extent, int n)
{
    T len = extent / T(n);
    int k = int(std::ceil(double((coord - lo) / len))) - 1;
    return std::clamp(k, 0, n - 1);
}
// collect_node_corrections (contact.hpp:141-186): walls, obstacles, Coulomb walls
template <class T, int D> void collect(const Scene<T, D>& sc, const int* idx, std::vector<Corr<T, D>>& out)
{
    out.clear();
    for (int w = 0; w < 2 * D; ++w) {
        if (sc.wall_kind[w] == MPM_WALL_COULOMB || !in_band(sc, idx, w))
            continue;
        Corr<T, D> c{};
        c.kind = sc.wall_kind[w] == MPM_WALL_SLIP ? C_SLIP : C_ZERO;
        c.axis = w / 2;
        out.push_back(c);
    }
    Vec<T, D> xp = sc.node_pos(idx);
    for (const auto& ob : sc.obstacles) {
        // Obstacle::contains (config.hpp:65-71)
        bool inside = true;
        for (int a = 0; a < D; ++a)
            if (xp.a[a] < ob[a] || xp.a[a] > ob[D + a])
                inside = false;
        if (!inside)
            continue;
        // Obstacle::outward_normal (config.hpp:73-87): nearest face, strict <
        int best_a = 0, best_s = 0;
        T best = std::numeric_limits<T>::max();
        for (int a = 0; a < D; ++a) {
            T dlo = xp.a[a] - ob[a];
            T dhi = ob[D + a] - xp.a[a];
            if (dlo < best) {
                best = dlo;
                best_a = a;
                best_s = 0;
            }
            if (dhi < best) {
                best = dhi;
                best_a = a;
                best_s = 1;
            }
        }
        Corr<T, D> c{};
        c.kind = C_OBST;
        c.n = vzero<T, D>();
        c.n.a[best_a] = best_s == 0 ? T(-1) : T(1);
        out.push_back(c);
    }
    for (int w = 0; w < 2 * D; ++w) {
        if (sc.wall_kind[w] != MPM_WALL_COULOMB || !in_band(sc, idx, w))
            continue;
        int seg_axis = w / 2 == 0 ? 1 : 0;
        int k = segment_index(xp.a[seg_axis], sc.origin[seg_axis], T(sc.cells[seg_axis]) * sc.dh,
                              int(sc.friction[w].size()));
        Corr<T, D> c{};
        c.kind = C_COUL;
        c.n = vzero<T, D>();
        c.n.a[w / 2] = w % 2 == 0 ? T(-1) : T(1); // wall_contact_normal (contact.hpp:28-34)
        c.mu = sc.friction[w][k];
        c.wall = w;
        c.seg = k;
        out.push_back(c);
    }
}
// apply_node_correction (contact.hpp:188-224)
template <class T, int D> Vec<T, D> apply_corr(const Corr<T, D>& c, const Vec<T, D>& v)
{
    switch (c.kind) {
    case C_SLIP: {
        Vec<T, D> r = v;
        r.a[c.axis] = T(0);
        return r;
    }
    case C_ZERO:
        return vzero<T, D>();
    case C_OBST: {
        T vn = dotv(v, c.n);
        if (vn < T(0)) {
            Vec<T, D> r;
            for (int a = 0; a < D; ++a)
                r.a[a] = v.a[a] - vn * c.n.a[a];
            return r;
        }
        return v;
    }
    default: {
        T vn = dotv(v, c.n);
        if (vn <= T(0))
            return v;
        Vec<T, D> t;
        for (int a = 0; a < D; ++a)
            t.a[a] = v.a[a] - vn * c.n.a[a];
        T tn = normv(t);
        if (tn <= c.mu * vn)
            return vzero<T, D>();
        T s = c.mu * vn / tn;
        Vec<T, D> r;
        for (int a = 0; a < D; ++a)
            r.a[a] = t.a[a] - s * t.a[a];
        return r;
    }
    }
}
// apply_grid_corrections (contact.hpp:228-245): every node, fixed order
template <class T, int D> void corrections(const Scene<T, D>& sc, Grid<T, D>& g)
{
    std::vector<Corr<T, D>> list;
    for (int64_t i = 0; i < sc.num_nodes(); ++i) {
        int idx[D];
        sc.node_multi(i, idx);
        collect(sc, idx, list);
        for (const auto& c : list)
            g.v[i] = apply_corr(c, g.v[i]);
    }
}

// ---------------------------------------------------------------------------------------
// G2P (transfer.hpp:92-121)
template <class T, int D> void g2p(const Scene<T, D>& sc, const Grid<T, D>& g, State<T, D>& s)
{
    T alpha = sc.flip_fraction();
    for (int64_t p = 0; p < s.n; ++p) {
        Stencil<T, D> st = stencil(sc, s.x[p], p);
        Vec<T, D> vpic = vzero<T, D>(), vinc = vzero<T, D>();
        Mat<T, D> L = mzero<T, D>(), B = mzero<T, D>();
        for (int k = 0; k < n_off<D>(); ++k) {
            int o[D], idx[D];
            offset_of<D>(k, o);
            Vec<T, D> r = node_rel(sc, st, o, s.x[p], idx);
            int64_t ni = sc.node_index(idx);
            T phi = weight(st, o);
            Vec<T, D> gw = grad(st, o);
            for (int a = 0; a < D; ++a) {
                vpic.a[a] += phi * g.v[ni].a[a];
                vinc.a[a] += phi * (g.v[ni].a[a] - g.vold[ni].a[a]);
                for (int b = 0; b < D; ++b)
                    L.a[a][b] += g.v[ni].a[a] * gw.a[b];
            }
            if (sc.apic())
                for (int a = 0; a < D; ++a)
                    for (int b = 0; b < D; ++b)
                        B.a[a][b] += phi * g.v[ni].a[a] * r.a[b];
        }
        for (int a = 0; a < D; ++a) {
            s.v[p].a[a] = alpha * (s.v[p].a[a] + vinc.a[a]) + (T(1) - alpha) * vpic.a[a];
            s.x[p].a[a] += sc.dt * vpic.a[a];
        }
        s.gv[p] = L;
        if (sc.apic())
            s.B[p] = B;
    }
}

// ---------------------------------------------------------------------------------------
// constitutive (constitutive.hpp)
template <class T> using M3 = Mat<T, 3>;

template <class T, int D> M3<T> embed(const Mat<T, D>& m)
{
    M3<T> r = mzero<T, 3>();
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j)
            r.a[i][j] = m.a[i][j];
    return r;
}
template <class T, int D> Mat<T, D> corner(const M3<T>& m)
{
    Mat<T, D> r;
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j)
            r.a[i][j] = m.a[i][j];
    return r;
}

// dp_trial_invariants (constitutive.hpp:72-83) + dp_classify (:62-70)
template <class T> struct Trial {
    T sm, tau, fs, ft, h;
    int zone; // 1 elastic, 2 shear, 3 tensile
};
template <class T, int D> Trial<T> trial_inv(const Scene<T, D>& sc, const M3<T>& tr)
{
    Trial<T> t;
    t.sm = trace(tr) / T(3);
    M3<T> dev = tr;
    for (int i = 0; i < 3; ++i)
        dev.a[i][i] -= t.sm;
    t.tau = std::sqrt(T(0.5) * fro2(dev));
    t.fs = t.tau - sc.k_phi + sc.q_phi * t.sm;
    t.ft = t.sm - sc.sigma_t;
    t.h = t.tau - sc.tau_P - sc.alpha_P * (t.sm - sc.sigma_t);
    if (t.fs <= T(0) && t.ft < T(0))
        t.zone = 1;
    else if (t.ft < T(0))
        t.zone = 2;
    else
        t.zone = t.h > T(0) ? 2 : 3;
    return t;
}

// shared forward intermediates of dp_stress_update (constitutive.hpp:101-124)
template <class T, int D> struct DpFwd {
    M3<T> dd, dw, sR, trial, dev;
    T trd;
    Trial<T> tr;
};
template <class T, int D> DpFwd<T, D> dp_forward(const Scene<T, D>& sc, const Mat<T, D>& sig, T szz,
                                                 const Mat<T, D>& gv)
{
    DpFwd<T, D> f;
    M3<T> S = embed<T, D>(sig), L = embed<T, D>(gv);
    if (D == 2)
        S.a[2][2] = szz;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            f.dd.a[i][j] = T(0.5) * (L.a[i][j] + L.a[j][i]) * sc.dt;
            f.dw.a[i][j] = T(0.5) * (L.a[i][j] - L.a[j][i]) * sc.dt;
        }
    // sR = S + S dw^T + dw S^T (constitutive.hpp:117)
    M3<T> a = matmul(S, transp(f.dw)), b = matmul(f.dw, transp(S));
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            f.sR.a[i][j] = S.a[i][j] + a.a[i][j] + b.a[i][j];
    f.trd = trace(f.dd);
    T lam = sc.K - T(2) * sc.G / T(3);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            f.trial.a[i][j] = f.sR.a[i][j] + T(2) * sc.G * f.dd.a[i][j] + (i == j ? lam * f.trd : T(0));
    f.tr = trial_inv(sc, f.trial);
    f.dev = f.trial;
    for (int i = 0; i < 3; ++i)
        f.dev.a[i][i] -= f.tr.sm;
    return f;
}

// dp_stress_update (constitutive.hpp:101-164); returns den
template <class T, int D> T dp_update(const Scene<T, D>& sc, Mat<T, D>& sig, T& szz, const Mat<T, D>& gv, T& deps,
                                      int& zone)
{
    DpFwd<T, D> f = dp_forward(sc, sig, szz, gv);
    const Trial<T>& tr = f.tr;
    M3<T> result = f.trial;
    deps = T(0);
    zone = tr.zone;
    if (tr.zone == 2) {
        T dlam = tr.fs / (sc.G + sc.K * sc.q_phi * sc.q_psi);
        deps = dlam * std::sqrt(T(1) / T(3) + T(2) / T(9) * sc.q_psi * sc.q_psi);
        T sm_new = tr.sm - sc.K * sc.q_psi * dlam;
        T tau_new = sc.k_phi - sc.q_phi * sm_new;
        if (tr.tau <= T(0) || tau_new < T(0)) {
            sm_new = sc.q_phi > T(0) ? sc.k_phi / sc.q_phi : sm_new;
            result = mzero<T, 3>();
            for (int i = 0; i < 3; ++i)
                result.a[i][i] = sm_new;
        } else {
            T ratio = tau_new / tr.tau;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j)
                    result.a[i][j] = ratio * f.dev.a[i][j] + (i == j ? sm_new : T(0));
        }
        if (sm_new > sc.sigma_t)
            for (int i = 0; i < 3; ++i)
                result.a[i][i] += sc.sigma_t - sm_new;
    } else if (tr.zone == 3) {
        T dlam_t = tr.ft / sc.K;
        deps = std::sqrt(T(2)) / T(3) * dlam_t;
        for (int i = 0; i < 3; ++i)
            result.a[i][i] = f.trial.a[i][i] + (sc.sigma_t - tr.sm);
        if (tr.tau > sc.tau_P) {
            T ratio = sc.tau_P / tr.tau;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j)
                    result.a[i][j] = ratio * f.dev.a[i][j] + (i == j ? sc.sigma_t : T(0));
        }
    }
    sig = corner<T, D>(result);
    if (D == 2)
        szz = result.a[2][2];
    T den = T(1) + f.trd;
    if (!(den > T(0)))
        throw Err(MPM_ERR_NUMERICAL, "dp update: 1 + tr(dd) <= 0, time step too large for the compression rate");
    return den;
}

// constitutive_update (stepper.hpp:15-43)
template <class T, int D> void constitutive(const Scene<T, D>& sc, State<T, D>& s)
{
    if (sc.material == MPM_MAT_FLUID) {
        for (int64_t p = 0; p < s.n; ++p) {
            // fluid_stress_update (constitutive.hpp:32-50)
            Mat<T, D> dd;
            for (int i = 0; i < D; ++i)
                for (int j = 0; j < D; ++j)
                    dd.a[i][j] = T(0.5) * (s.gv[p].a[i][j] + s.gv[p].a[j][i]) * sc.dt;
            T trd = trace(dd);
            T den = T(1) + trd;
            if (!(den > T(0)))
                throw Err(MPM_ERR_NUMERICAL,
                          "fluid update: 1 + tr(dd) <= 0, time step too large for the compression rate");
            T rho = s.rho[p] / den;
            T pres = sc.c * sc.c * (rho - sc.rho0);
            T k = sc.rate_form ? sc.visc / sc.dt : sc.visc;
            // sigma = -p I - (2/3) k tr(dd) I + 2 k dd, coefficient-wise in the reference's
            // expression order (signed zeros included)
            T vis = (T(2) / T(3)) * k * trd, k2 = T(2) * k;
            for (int i = 0; i < D; ++i)
                for (int j = 0; j < D; ++j) {
                    T I = i == j ? T(1) : T(0);
                    s.sig[p].a[i][j] = (I * -pres - I * vis) + k2 * dd.a[i][j];
                }
            s.rho[p] = rho;
            s.V[p] *= den;
        }
    } else {
        for (int64_t p = 0; p < s.n; ++p) {
            T szz = D == 2 ? s.szz[p] : T(0);
            T deps;
            int zone;
            T den = dp_update(sc, s.sig[p], szz, s.gv[p], deps, zone);
            if (D == 2)
                s.szz[p] = szz;
            s.eps[p] += deps;
            s.rho[p] /= den;
            s.V[p] *= den;
        }
    }
    if (s.has_F)
        for (int64_t p = 0; p < s.n; ++p) {
            Mat<T, D> A = ident<T, D>();
            for (int i = 0; i < D; ++i)
                for (int j = 0; j < D; ++j)
                    A.a[i][j] += s.gv[p].a[i][j] * sc.dt;
            s.F[p] = matmul(A, s.F[p]);
        }
}

// Stepper::advance (stepper.hpp:59-69)
template <class T, int D> void advance(const Scene<T, D>& sc, State<T, D>& s)
{
    Grid<T, D> g;
    p2g(sc, s, g);
    momentum_update(sc, g);
    corrections(sc, g);
    g2p(sc, g, s);
    constitutive(sc, s);
    s.step += 1;
    s.time = double(T(s.step) * sc.dt);
}

// ParticleSoA::all_finite (state.hpp:48-62)
template <class T, int D> bool all_finite(const State<T, D>& s)
{
    auto fv = [](const auto& vec) {
        for (const auto& e : vec)
            for (int a = 0; a < D; ++a)
                if (!std::isfinite(e.a[a]))
                    return false;
        return true;
    };
    auto fs = [](const std::vector<T>& vec) {
        for (T e : vec)
            if (!std::isfinite(e))
                return false;
        return true;
    };
    auto fm = [](const std::vector<Mat<T, D>>& vec) {
        for (const auto& e : vec)
            for (int a = 0; a < D; ++a)
                for (int b = 0; b < D; ++b)
                    if (!std::isfinite(e.a[a][b]))
                        return false;
        return true;
    };
    return fv(s.x) && fv(s.v) && fs(s.V) && fs(s.rho) && fs(s.eps) && (D == 3 || fs(s.szz)) && fm(s.sig)
        && fm(s.gv) && (!s.has_B || fm(s.B));
}

// ---------------------------------------------------------------------------------------
// adjoint (adjoint.hpp)
template <class T, int D> struct Cot {
    std::vector<Vec<T, D>> x, v;
    std::vector<T> rho, V, eps, szz;
    std::vector<Mat<T, D>> sig, gv, B;
    void zeros(int64_t n, bool has_B)
    {
        x.assign(n, vzero<T, D>());
        v.assign(n, vzero<T, D>());
        rho.assign(n, T(0));
        V.assign(n, T(0));
        eps.assign(n, T(0));
        szz.assign(D == 2 ? n : 0, T(0));
        sig.assign(n, mzero<T, D>());
        gv.assign(n, mzero<T, D>());
        B.assign(has_B ? n : 0, mzero<T, D>());
    }
};
template <class T, int D> Cot<T, D> load_cot(const mpm_cot_view* c, int64_t n, bool has_B)
{
    Cot<T, D> k;
    load_vec(k.x, c->x, n);
    load_vec(k.v, c->v, n);
    load_sc(k.rho, c->rho, n);
    load_sc(k.V, c->volume, n);
    load_sc(k.eps, c->eps_eq, n);
    if (D == 2)
        load_sc(k.szz, c->sigma_zz, n);
    load_mat(k.sig, c->sigma, n);
    load_mat(k.gv, c->grad_v, n);
    if (has_B)
        load_mat(k.B, c->affine, n);
    return k;
}
template <class T, int D> void store_cot(const Cot<T, D>& k, mpm_cot_view* c)
{
    store_vec(k.x, c->x);
    store_vec(k.v, c->v);
    store_sc(k.rho, c->rho);
    store_sc(k.V, c->volume);
    store_sc(k.eps, c->eps_eq);
    if (D == 2)
        store_sc(k.szz, c->sigma_zz);
    store_mat(k.sig, c->sigma);
    store_mat(k.gv, c->grad_v);
    if (!k.B.empty())
        store_mat(k.B, c->affine);
}

template <class T, int D> struct PG {
    T c = T(0), mu = T(0);
    std::vector<T> fr[2 * D];
};

// detail::node_correction_vjp (adjoint.hpp:112-150)
template <class T, int D> Vec<T, D> corr_vjp(const Corr<T, D>& c, const Vec<T, D>& vin, const Vec<T, D>& cot,
                                             PG<T, D>& pg)
{
    switch (c.kind) {
    case C_SLIP: {
        Vec<T, D> r = cot;
        r.a[c.axis] = T(0);
        return r;
    }
    case C_ZERO:
        return vzero<T, D>();
    case C_OBST: {
        if (dotv(vin, c.n) < T(0)) {
            T nc = dotv(c.n, cot);
            Vec<T, D> r;
            for (int a = 0; a < D; ++a)
                r.a[a] = cot.a[a] - c.n.a[a] * nc;
            return r;
        }
        return cot;
    }
    default: {
        T vn = dotv(vin, c.n);
        if (vn <= T(0))
            return cot;
        Vec<T, D> t;
        for (int a = 0; a < D; ++a)
            t.a[a] = vin.a[a] - vn * c.n.a[a];
        T tn = normv(t);
        if (tn <= c.mu * vn)
            return vzero<T, D>();
        T s = T(1) - c.mu * vn / tn;
        Vec<T, D> that;
        for (int a = 0; a < D; ++a)
            that.a[a] = t.a[a] / tn;
        T tc = dotv(t, cot);
        T nc = dotv(c.n, cot);
        Vec<T, D> r;
        for (int a = 0; a < D; ++a)
            r.a[a] = s * (cot.a[a] - c.n.a[a] * nc)
                + tc * (-(c.mu / tn) * c.n.a[a] + (c.mu * vn / (tn * tn)) * that.a[a]);
        pg.fr[c.wall][c.seg] += -vn * dotv(that, cot);
        return r;
    }
    }
}

// detail::fluid_vjp (adjoint.hpp:152-184)
template <class T, int D> void fluid_vjp(const Scene<T, D>& sc, T rho, T V, const Mat<T, D>& gvn, const Mat<T, D>& sc_,
                                         T rho_c, T V_c, Mat<T, D>& gvn_c, T& rho_in_c, T& V_in_c, PG<T, D>& pg)
{
    Mat<T, D> dd;
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j)
            dd.a[i][j] = T(0.5) * (gvn.a[i][j] + gvn.a[j][i]) * sc.dt;
    T trd = trace(dd);
    T den = T(1) + trd;
    T rho_new = rho / den;
    T c = sc.c;
    T k = sc.rate_form ? sc.visc / sc.dt : sc.visc;
    T p_c = -trace(sc_);
    T mu_acc = T(0); // (sigma_cot .* (-(2/3) trd I + 2 dd)).sum(), column-major like Eigen
    T vis = -(T(2) / T(3)) * trd;
    for (int j = 0; j < D; ++j)
        for (int i = 0; i < D; ++i) {
            T I = i == j ? T(1) : T(0);
            mu_acc += sc_.a[i][j] * (vis * I + T(2) * dd.a[i][j]);
        }
    pg.mu += mu_acc * (sc.rate_form ? T(1) / sc.dt : T(1));
    T trd_c = -(T(2) / T(3)) * k * trace(sc_);
    Mat<T, D> dd_c;
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j)
            dd_c.a[i][j] = T(2) * k * sc_.a[i][j];
    pg.c += T(2) * c * (rho_new - sc.rho0) * p_c;
    T rho_new_c = rho_c + c * c * p_c;
    rho_in_c += rho_new_c / den;
    T den_c = -(rho / (den * den)) * rho_new_c;
    V_in_c += den * V_c;
    den_c += V * V_c;
    trd_c += den_c;
    for (int i = 0; i < D; ++i)
        dd_c.a[i][i] += trd_c;
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j)
            gvn_c.a[i][j] += sc.dt * T(0.5) * (dd_c.a[i][j] + dd_c.a[j][i]);
}

// detail::dp_vjp (adjoint.hpp:186-293)
template <class T, int D> void dp_vjp(const Scene<T, D>& sc, const Mat<T, D>& sig_in, T szz_in, const Mat<T, D>& gvn,
                                      const Mat<T, D>& sig_c, T szz_c, T rho_c, T V_c, T rho_in, T V_in,
                                      Mat<T, D>& gvn_c, Mat<T, D>& sig_in_c, T& szz_in_c, T& rho_in_c, T& V_in_c)
{
    DpFwd<T, D> f = dp_forward(sc, sig_in, szz_in, gvn);
    const Trial<T>& tr = f.tr;
    M3<T> out_c = embed<T, D>(sig_c);
    if (D == 2)
        out_c.a[2][2] += szz_c;
    M3<T> trial_c = mzero<T, 3>();
    auto assemble = [&](const M3<T>& dev_c, T sm_c) {
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                trial_c.a[i][j] += dev_c.a[i][j];
        T sm_total = sm_c - trace(dev_c);
        for (int i = 0; i < 3; ++i)
            trial_c.a[i][i] += sm_total / T(3);
    };
    if (tr.zone == 1) {
        trial_c = out_c;
    } else if (tr.zone == 2) {
        T denom = sc.G + sc.K * sc.q_phi * sc.q_psi;
        T dlam = tr.fs / denom;
        T sm_new = tr.sm - sc.K * sc.q_psi * dlam;
        T tau_new = sc.k_phi - sc.q_phi * sm_new;
        if (tr.tau <= T(0) || tau_new < T(0)) {
            // apex: constant output
        } else {
            bool capped = sm_new > sc.sigma_t;
            T ratio = tau_new / tr.tau;
            M3<T> dev_c;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j)
                    dev_c.a[i][j] = ratio * out_c.a[i][j];
            T ratio_c = contract(out_c, f.dev);
            T sm_new_c = capped ? T(0) : trace(out_c);
            T tau_new_c = ratio_c / tr.tau;
            T tau_c = -ratio_c * tau_new / (tr.tau * tr.tau);
            sm_new_c += -sc.q_phi * tau_new_c;
            T sm_c = sm_new_c;
            T dlam_c = -sc.K * sc.q_psi * sm_new_c;
            T fs_c = dlam_c / denom;
            tau_c += fs_c;
            sm_c += sc.q_phi * fs_c;
            if (tr.tau > T(0))
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j)
                        dev_c.a[i][j] += (tau_c / (T(2) * tr.tau)) * f.dev.a[i][j];
            assemble(dev_c, sm_c);
        }
    } else {
        if (tr.tau > sc.tau_P) {
            T ratio = sc.tau_P / tr.tau;
            M3<T> dev_c;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j)
                    dev_c.a[i][j] = ratio * out_c.a[i][j];
            T ratio_c = contract(out_c, f.dev);
            T tau_c = -ratio_c * sc.tau_P / (tr.tau * tr.tau);
            if (tr.tau > T(0))
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j)
                        dev_c.a[i][j] += (tau_c / (T(2) * tr.tau)) * f.dev.a[i][j];
            assemble(dev_c, T(0));
        } else {
            trial_c = out_c;
            T sm_c = -trace(out_c);
            for (int i = 0; i < 3; ++i)
                trial_c.a[i][i] += sm_c / T(3);
        }
    }
    // trial = sR + 2G dd + (K - 2G/3) tr(dd) I  (adjoint.hpp:273-275)
    M3<T> sR_c = trial_c;
    T lam = sc.K - T(2) * sc.G / T(3);
    T tc = trace(trial_c);
    M3<T> dd_c;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            dd_c.a[i][j] = T(2) * sc.G * trial_c.a[i][j] + (i == j ? lam * tc : T(0));
    // V' = den V, rho' = rho / den (adjoint.hpp:277-282)
    T den = T(1) + f.trd;
    T den_c = V_in * V_c - (rho_in / (den * den)) * rho_c;
    V_in_c += den * V_c;
    rho_in_c += rho_c / den;
    for (int i = 0; i < 3; ++i)
        dd_c.a[i][i] += den_c;
    // sR = S + S dw^T + dw S^T (adjoint.hpp:284-286)
    M3<T> S = embed<T, D>(sig_in);
    if (D == 2)
        S.a[2][2] = szz_in;
    M3<T> a1 = matmul(sR_c, f.dw), a2 = matmul(transp(f.dw), sR_c);
    M3<T> S_c;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            S_c.a[i][j] = sR_c.a[i][j] + a1.a[i][j] + a2.a[i][j];
    M3<T> b1 = matmul(transp(sR_c), S), b2 = matmul(sR_c, S);
    M3<T> dw_c;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            dw_c.a[i][j] = b1.a[i][j] + b2.a[i][j];
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
            gvn_c.a[i][j] += sc.dt
                * (T(0.5) * (dd_c.a[i][j] + dd_c.a[j][i]) + T(0.5) * (dw_c.a[i][j] - dw_c.a[j][i]));
            sig_in_c.a[i][j] += S_c.a[i][j];
        }
    if (D == 2)
        szz_in_c += S_c.a[2][2];
}

// step_vjp (adjoint.hpp:328-525)
template <class T, int D> void step_vjp(const Scene<T, D>& sc, const State<T, D>& s, const Cot<T, D>& co, Cot<T, D>& ci,
                                        PG<T, D>& pg)
{
    const T dt = sc.dt;
    const T alpha = sc.flip_fraction();
    const bool apic = sc.apic(), tpic = sc.tpic();
    const int64_t n = s.n;
    // forward replay (adjoint.hpp:341-368)
    std::vector<Stencil<T, D>> st(n);
    for (int64_t p = 0; p < n; ++p)
        st[p] = stencil(sc, s.x[p], p);
    std::vector<Mat<T, D>> A(apic ? n : 0), Dinv(apic ? n : 0);
    if (apic)
        for (int64_t p = 0; p < n; ++p) {
            Dinv[p] = inverse(apic_D(sc, st[p], s.x[p]));
            A[p] = matmul(s.B[p], Dinv[p]);
        }
    Grid<T, D> g;
    p2g(sc, s, g);
    momentum_update(sc, g);
    std::vector<Vec<T, D>> vtilde = g.v;
    corrections(sc, g);
    State<T, D> out = s;
    g2p(sc, g, out);

    // reverse sweep
    ci.zeros(n, s.has_B);
    std::vector<Mat<T, D>> gvn_c(n, mzero<T, D>());
    // (1) constitutive transpose (adjoint.hpp:374-400)
    if (sc.material == MPM_MAT_FLUID) {
        for (int64_t p = 0; p < n; ++p)
            fluid_vjp(sc, s.rho[p], s.V[p], out.gv[p], co.sig[p], co.rho[p], co.V[p], gvn_c[p], ci.rho[p], ci.V[p], pg);
    } else {
        for (int64_t p = 0; p < n; ++p) {
            T szz_in = D == 2 ? s.szz[p] : T(0);
            T szz_c = D == 2 ? co.szz[p] : T(0);
            T szz_in_c = T(0);
            dp_vjp(sc, s.sig[p], szz_in, out.gv[p], co.sig[p], szz_c, co.rho[p], co.V[p], s.rho[p], s.V[p], gvn_c[p],
                   ci.sig[p], szz_in_c, ci.rho[p], ci.V[p]);
            if (D == 2)
                ci.szz[p] = szz_in_c;
        }
    }
    for (int64_t p = 0; p < n; ++p)
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j)
                gvn_c[p].a[i][j] += co.gv[p].a[i][j];

    // (2) G2P transpose (adjoint.hpp:402-439)
    int64_t nn = sc.num_nodes();
    std::vector<Vec<T, D>> gv_c(nn, vzero<T, D>()), gvold_c(nn, vzero<T, D>());
    for (int64_t p = 0; p < n; ++p) {
        const Mat<T, D>& Lc = gvn_c[p];
        Vec<T, D> pic_c, inc_c, xp_c = vzero<T, D>();
        for (int a = 0; a < D; ++a) {
            ci.v[p].a[a] += alpha * co.v[p].a[a];
            ci.x[p].a[a] += co.x[p].a[a];
            pic_c.a[a] = (T(1) - alpha) * co.v[p].a[a] + dt * co.x[p].a[a];
            inc_c.a[a] = alpha * co.v[p].a[a];
        }
        Mat<T, D> Bc = apic ? co.B[p] : mzero<T, D>();
        for (int k = 0; k < n_off<D>(); ++k) {
            int o[D], idx[D];
            offset_of<D>(k, o);
            Vec<T, D> r = node_rel(sc, st[p], o, s.x[p], idx);
            int64_t ni = sc.node_index(idx);
            T phi = weight(st[p], o);
            Vec<T, D> gw = grad(st[p], o);
            Mat<T, D> H = hessian(st[p], o);
            const Vec<T, D>& w = g.v[ni];
            const Vec<T, D>& u = g.vold[ni];
            Vec<T, D> Lgw = matvec(Lc, gw);
            Vec<T, D> add;
            for (int a = 0; a < D; ++a) {
                add.a[a] = phi * (pic_c.a[a] + inc_c.a[a]) + Lgw.a[a];
                gvold_c[ni].a[a] -= phi * inc_c.a[a];
            }
            T s1 = dotv(pic_c, w);
            Vec<T, D> wu;
            for (int a = 0; a < D; ++a)
                wu.a[a] = w.a[a] - u.a[a];
            T s2 = dotv(inc_c, wu);
            Vec<T, D> LTw = matvec(transp(Lc), w);
            Vec<T, D> HLTw = matvec(H, LTw);
            for (int a = 0; a < D; ++a) {
                xp_c.a[a] += gw.a[a] * (s1 + s2);
                xp_c.a[a] += HLTw.a[a];
            }
            if (apic) {
                Vec<T, D> Bcr = matvec(Bc, r);
                T wBr = dotv(w, Bcr);
                Vec<T, D> BcTw = matvec(transp(Bc), w);
                for (int a = 0; a < D; ++a) {
                    add.a[a] += phi * Bcr.a[a];
                    xp_c.a[a] += gw.a[a] * wBr - phi * BcTw.a[a];
                }
            }
            for (int a = 0; a < D; ++a)
                gv_c[ni].a[a] += add.a[a];
        }
        for (int a = 0; a < D; ++a)
            ci.x[p].a[a] += xp_c.a[a];
    }

    // (3) correction transpose (adjoint.hpp:441-460)
    std::vector<Corr<T, D>> list;
    std::vector<Vec<T, D>> chain;
    for (int64_t i = 0; i < nn; ++i) {
        if (g.m[i] <= sc.mass_eps) {
            gv_c[i] = vzero<T, D>();
            gvold_c[i] = vzero<T, D>();
            continue;
        }
        int idx[D];
        sc.node_multi(i, idx);
        collect(sc, idx, list);
        if (list.empty())
            continue;
        chain.resize(list.size() + 1);
        chain[0] = vtilde[i];
        for (size_t k = 0; k < list.size(); ++k)
            chain[k + 1] = apply_corr(list[k], chain[k]);
        Vec<T, D> cot = gv_c[i];
        for (size_t k = list.size(); k-- > 0;)
            cot = corr_vjp(list[k], chain[k], cot, pg);
        gv_c[i] = cot;
    }

    // (4) momentum update transpose (adjoint.hpp:462-477)
    std::vector<T> gm_c(nn, T(0));
    std::vector<Vec<T, D>> gmom_c(nn, vzero<T, D>()), gf_c(nn, vzero<T, D>());
    for (int64_t i = 0; i < nn; ++i) {
        T mass = g.m[i];
        if (mass <= sc.mass_eps)
            continue;
        Vec<T, D> vt_c = gv_c[i], u_c;
        for (int a = 0; a < D; ++a) {
            u_c.a[a] = gvold_c[i].a[a] + vt_c.a[a];
            gf_c[i].a[a] = (dt / mass) * vt_c.a[a];
            gmom_c[i].a[a] = u_c.a[a] / mass;
        }
        gm_c[i] = -(dotv(g.p[i], u_c)) / (mass * mass) - dt * (dotv(g.f[i], vt_c)) / (mass * mass);
    }

    // (5) P2G transpose (adjoint.hpp:479-524)
    for (int64_t p = 0; p < n; ++p) {
        T mass = s.m[p], vol = s.V[p];
        const Mat<T, D>& sig = s.sig[p];
        Mat<T, D> Ap = mzero<T, D>();
        if (apic)
            Ap = A[p];
        else if (tpic)
            Ap = s.gv[p];
        bool affine = apic || tpic;
        Mat<T, D> A_c = mzero<T, D>();
        Vec<T, D> xp_c = vzero<T, D>();
        for (int k = 0; k < n_off<D>(); ++k) {
            int o[D], idx[D];
            offset_of<D>(k, o);
            Vec<T, D> r = node_rel(sc, st[p], o, s.x[p], idx);
            int64_t ni = sc.node_index(idx);
            T phi = weight(st[p], o);
            Vec<T, D> gw = grad(st[p], o);
            Mat<T, D> H = hessian(st[p], o);
            const Vec<T, D>& mc = gmom_c[ni];
            const Vec<T, D>& fc = gf_c[ni];
            for (int a = 0; a < D; ++a)
                ci.v[p].a[a] += mass * phi * mc.a[a];
            Vec<T, D> vel = s.v[p];
            if (affine) {
                Vec<T, D> Ar = matvec(Ap, r);
                Vec<T, D> ATm = matvec(transp(Ap), mc);
                for (int a = 0; a < D; ++a) {
                    vel.a[a] += Ar.a[a];
                    xp_c.a[a] -= mass * phi * ATm.a[a];
                    for (int b = 0; b < D; ++b)
                        A_c.a[a][b] += mass * phi * mc.a[a] * r.a[b];
                }
            }
            for (int a = 0; a < D; ++a)
                for (int b = 0; b < D; ++b)
                    ci.sig[p].a[a][b] += -vol * fc.a[a] * gw.a[b];
            Vec<T, D> sg = matvec(sig, gw);
            ci.V[p] += -dotv(sg, fc);
            Vec<T, D> sfc = matvec(sig, fc);
            Vec<T, D> Hs = matvec(H, sfc);
            T gdf = T(0);
            for (int a = 0; a < D; ++a)
                gdf += sc.gravity[a] * fc.a[a];
            T mdv = dotv(mc, vel);
            for (int a = 0; a < D; ++a) {
                xp_c.a[a] += mass * gm_c[ni] * gw.a[a];
                xp_c.a[a] += mass * mdv * gw.a[a];
                xp_c.a[a] += mass * gdf * gw.a[a];
                xp_c.a[a] += -vol * Hs.a[a];
            }
        }
        for (int a = 0; a < D; ++a)
            ci.x[p].a[a] += xp_c.a[a];
        if (apic)
            ci.B[p] = matmul(A_c, Dinv[p]);
        else if (tpic)
            for (int a = 0; a < D; ++a)
                for (int b = 0; b < D; ++b)
                    ci.gv[p].a[a][b] += A_c.a[a][b];
    }
}

// ---------------------------------------------------------------------------------------
// FNV-1a state hash (common.hpp:40-57, hash.cpp:5-13, state.hpp:71-86). Hashes the
// reference's in-memory layout (vectors AoS, matrices column-major).
inline uint64_t fnv(const void* data, size_t n, uint64_t h)
{
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}
template <class T, int D> uint64_t hash_state(const mpm_state_view* v)
{
    uint64_t h = 0xcbf29ce484222325ull;
    int64_t n = v->n;
    auto hs = [&](const void* p, size_t elems) {
        if (p && elems)
            h = fnv(p, elems * sizeof(T), h);
    };
    if (n > 0) {
        hs(v->x, n * D);
        hs(v->v, n * D);
        hs(v->volume, n);
        hs(v->rho, n);
        hs(v->eps_eq, n);
        if (D == 2)
            hs(v->sigma_zz, n);
        hs(v->sigma, n * D * D);
        hs(v->grad_v, n * D * D);
        hs(v->affine, n * D * D);
    }
    h = fnv(&v->step, sizeof(int64_t), h);
    return h;
}

// ---------------------------------------------------------------------------------------
// init_scene (scene.hpp:55-116) restated, with the validation subset the seeding relies on
template <class T, int D> struct Region {
    int shape;
    T lo[D], hi[D], center[D], radius, zmin, zmax;
    int vk;
    T value[D], alpha, h0, amp, pert, freq;
};
template <class T, int D> bool contains(const Region<T, D>& r, const Vec<T, D>& p)
{
    if (r.shape == 0) {
        for (int a = 0; a < D; ++a)
            if (p.a[a] < r.lo[a] || p.a[a] >= r.hi[a])
                return false;
        return true;
    }
    if constexpr (D == 3) {
        if (p.a[2] < r.zmin || p.a[2] >= r.zmax)
            return false;
    }
    T dx = p.a[0] - r.center[0], dy = p.a[1] - r.center[1];
    return dx * dx + dy * dy < r.radius * r.radius;
}
template <class T, int D> Vec<T, D> vel_eval(const Region<T, D>& r, T y)
{
    Vec<T, D> v = vzero<T, D>();
    switch (r.vk) {
    case 0:
        for (int a = 0; a < D; ++a)
            v.a[a] = r.value[a];
        return v;
    case 1:
        v.a[0] = r.alpha * (r.h0 - y);
        return v;
    case 2: {
        T yn = y / r.h0;
        v.a[0] = r.amp * (T(1) - yn * yn) + r.pert * std::sin(r.freq * T(3.141592653589793238462643383279502884L) * yn);
        return v;
    }
    default:
        throw Err(MPM_ERR_VALIDATION, "oracle: mlp velocity fields are not restated");
    }
}
template <class T, int D> std::vector<Region<T, D>> decode_regions(const orc_region* r, int nreg)
{
    std::vector<Region<T, D>> out;
    for (int i = 0; i < nreg; ++i) {
        Region<T, D> g{};
        g.shape = r[i].shape;
        for (int a = 0; a < D; ++a) {
            g.lo[a] = T(r[i].lo[a]);
            g.hi[a] = T(r[i].hi[a]);
            g.center[a] = T(r[i].center[a]);
            g.value[a] = T(r[i].value[a]);
        }
        g.radius = T(r[i].radius);
        g.zmin = T(r[i].zmin);
        g.zmax = T(r[i].zmax);
        g.vk = r[i].vel_kind;
        g.alpha = T(r[i].alpha);
        g.h0 = T(r[i].h0);
        g.amp = T(r[i].amplitude);
        g.pert = T(r[i].perturbation);
        g.freq = T(r[i].frequency);
        out.push_back(g);
    }
    return out;
}
template <class T, int D> State<T, D> init_scene(const Scene<T, D>& sc, const std::vector<Region<T, D>>& regs,
                                                 T& mass_eps)
{
    if (regs.empty())
        throw Err(MPM_ERR_VALIDATION, "scene: no geometry regions");
    T rho0 = sc.rho0;
    T cell_vol = std::pow(sc.dh, T(D));
    T mp = rho0 * cell_vol / T(1 << D);
    std::vector<Vec<T, D>> pos;
    std::vector<int> owner;
    int ci[3] = {0, 0, 0};
    int total = 1;
    for (int a = 0; a < D; ++a)
        total *= sc.cells[a];
    for (int lin = 0; lin < total; ++lin) {
        int rem = lin;
        for (int a = D - 1; a >= 0; --a) {
            ci[a] = rem % sc.cells[a];
            rem /= sc.cells[a];
        }
        Vec<T, D> center;
        for (int a = 0; a < D; ++a)
            center.a[a] = sc.origin[a] + (T(ci[a]) + T(0.5)) * sc.dh;
        for (int corner = 0; corner < (1 << D); ++corner) {
            Vec<T, D> p = center;
            for (int a = 0; a < D; ++a)
                p.a[a] += ((corner >> a) & 1) ? sc.dh / T(4) : -sc.dh / T(4);
            for (size_t r = 0; r < regs.size(); ++r)
                if (contains(regs[r], p)) {
                    pos.push_back(p);
                    owner.push_back(int(r));
                    break;
                }
        }
    }
    if (pos.empty())
        throw Err(MPM_ERR_VALIDATION, "scene: geometry produced no particles");
    State<T, D> s;
    s.n = int64_t(pos.size());
    s.x = pos;
    s.v.assign(s.n, vzero<T, D>());
    s.m.assign(s.n, mp);
    s.V.assign(s.n, mp / rho0);
    s.rho.assign(s.n, rho0);
    s.eps.assign(s.n, T(0));
    s.szz.assign(s.n, T(0));
    s.sig.assign(s.n, mzero<T, D>());
    s.gv.assign(s.n, mzero<T, D>());
    s.has_B = sc.apic();
    s.B.assign(s.n, mzero<T, D>());
    s.has_F = sc.track_F;
    s.F.assign(s.n, ident<T, D>());
    for (int64_t p = 0; p < s.n; ++p) {
        const Region<T, D>& r = regs[owner[p]];
        T miny = r.shape == 0 ? r.lo[1] : r.center[1] - r.radius;
        s.v[p] = vel_eval(r, pos[p].a[1] - miny);
    }
    mass_eps = T(1e-12) * mp;
    return s;
}

template <class F> int guarded(F&& f)
{
    g_particle = -1;
    g_msg.clear();
    try {
        return f();
    } catch (const Err& e) {
        g_particle = e.particle;
        g_msg = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return MPM_ERR_USAGE;
    }
}

template <template <class, int> class Op, class... A> auto dispatch(const mpm_scene_desc* d, A&&... a)
{
    if (d->dtype == MPM_F64)
        return d->dim == 2 ? Op<double, 2>::run(d, a...) : Op<double, 3>::run(d, a...);
    return d->dim == 2 ? Op<float, 2>::run(d, a...) : Op<float, 3>::run(d, a...);
}

template <class T, int D> struct OpInitCount {
    static int64_t run(const mpm_scene_desc* d, const orc_region* r, int nreg)
    {
        try {
            T me;
            return init_scene(decode<T, D>(d), decode_regions<T, D>(r, nreg), me).n;
        } catch (...) {
            return -1;
        }
    }
};
template <class T, int D> struct OpInit {
    static int run(const mpm_scene_desc* d, const orc_region* r, int nreg, mpm_state_view* out, double* meps)
    {
        return guarded([&] {
            T me;
            State<T, D> s = init_scene(decode<T, D>(d), decode_regions<T, D>(r, nreg), me);
            store_state(s, out);
            if (meps)
                *meps = double(me);
            return MPM_OK;
        });
    }
};
template <class T, int D> struct OpAdvance {
    static int run(const mpm_scene_desc* d, mpm_state_view* v, int64_t n, int guard)
    {
        State<T, D> s = load_state<T, D>(v);
        Scene<T, D> sc = decode<T, D>(d);
        int rc = guarded([&] {
            for (int64_t i = 0; i < n; ++i) {
                advance(sc, s);
                if (guard && !all_finite(s))
                    throw Err(MPM_ERR_NUMERICAL, "run: non-finite particle field detected at step " + std::to_string(s.step));
            }
            return MPM_OK;
        });
        store_state(s, v);
        return rc;
    }
};
template <class T, int D> struct OpP2G {
    static int run(const mpm_scene_desc* d, const mpm_state_view* v, mpm_grid_view* gv)
    {
        return guarded([&] {
            Scene<T, D> sc = decode<T, D>(d);
            Grid<T, D> g;
            p2g(sc, load_state<T, D>(v), g);
            store_grid(sc, g, gv);
            return MPM_OK;
        });
    }
};
template <class T, int D> struct OpMom {
    static int run(const mpm_scene_desc* d, mpm_grid_view* gv)
    {
        return guarded([&] {
            Scene<T, D> sc = decode<T, D>(d);
            Grid<T, D> g = load_grid(sc, gv);
            momentum_update(sc, g);
            store_grid(sc, g, gv);
            return MPM_OK;
        });
    }
};
template <class T, int D> struct OpCorr {
    static int run(const mpm_scene_desc* d, mpm_grid_view* gv)
    {
        return guarded([&] {
            Scene<T, D> sc = decode<T, D>(d);
            Grid<T, D> g = load_grid(sc, gv);
            corrections(sc, g);
            store_grid(sc, g, gv);
            return MPM_OK;
        });
    }
};
template <class T, int D> struct OpG2P {
    static int run(const mpm_scene_desc* d, const mpm_grid_view* gv, mpm_state_view* v)
    {
        return guarded([&] {
            Scene<T, D> sc = decode<T, D>(d);
            Grid<T, D> g = load_grid(sc, gv);
            State<T, D> s = load_state<T, D>(v);
            g2p(sc, g, s);
            store_state(s, v);
            return MPM_OK;
        });
    }
};
template <class T, int D> struct OpConst {
    static int run(const mpm_scene_desc* d, mpm_state_view* v)
    {
        return guarded([&] {
            Scene<T, D> sc = decode<T, D>(d);
            State<T, D> s = load_state<T, D>(v);
            constitutive(sc, s);
            store_state(s, v);
            return MPM_OK;
        });
    }
};
template <class T, int D> PG<T, D> load_pg(const Scene<T, D>& sc, const mpm_param_grads* pg)
{
    PG<T, D> g;
    g.c = T(pg->sound_speed);
    g.mu = T(pg->viscosity);
    for (int w = 0; w < 2 * D; ++w) {
        g.fr[w].assign(sc.friction[w].size(), T(0));
        if (pg->wall_friction[w])
            for (size_t k = 0; k < g.fr[w].size(); ++k)
                g.fr[w][k] = T(pg->wall_friction[w][k]);
    }
    return g;
}
template <class T, int D> void store_pg(const PG<T, D>& g, mpm_param_grads* pg)
{
    pg->sound_speed = double(g.c);
    pg->viscosity = double(g.mu);
    for (int w = 0; w < 2 * D; ++w)
        if (pg->wall_friction[w])
            for (size_t k = 0; k < g.fr[w].size(); ++k)
                pg->wall_friction[w][k] = double(g.fr[w][k]);
}
template <class T, int D> struct OpVjp {
    static int run(const mpm_scene_desc* d, const mpm_state_view* v, const mpm_cot_view* co, mpm_cot_view* ci,
                   mpm_param_grads* pgv)
    {
        return guarded([&] {
            Scene<T, D> sc = decode<T, D>(d);
            State<T, D> s = load_state<T, D>(v);
            Cot<T, D> cout_ = load_cot<T, D>(co, s.n, s.has_B);
            Cot<T, D> cin;
            PG<T, D> pg = load_pg(sc, pgv);
            step_vjp(sc, s, cout_, cin, pg);
            store_cot(cin, ci);
            store_pg(pg, pgv);
            return MPM_OK;
        });
    }
};
// CheckpointPlan::make (checkpoint.hpp:15-34) + backprop_trajectory (checkpoint.hpp:72-143)
template <class T, int D> struct OpBackprop {
    static int run(const mpm_scene_desc* d, const mpm_state_view* v, int64_t total, int nseg,
                   const mpm_seeder_desc* sd, mpm_cot_view* c0, mpm_param_grads* pgv, mpm_backprop_result* res)
    {
        return guarded([&] {
            if (total < 1)
                throw Err(MPM_ERR_VALIDATION, "checkpoint plan: need at least one step");
            if (nseg < 1 || int64_t(nseg) > total)
                throw Err(MPM_ERR_VALIDATION, "checkpoint plan: n_segments must lie in [1, N_t]");
            std::vector<int64_t> bnd(nseg + 1, 0);
            int64_t base = total / nseg, rem = total % nseg, at = 0;
            for (int k = 0; k < nseg; ++k) {
                at += base + (k < rem ? 1 : 0);
                bnd[k + 1] = at;
            }
            Scene<T, D> sc = decode<T, D>(d);
            State<T, D> s0 = load_state<T, D>(v);
            int64_t n = s0.n;
            // built-in least-squares seeders (checkpoint.hpp:63-66 protocol): Lagrangian, and the
            // Eulerian monitor regions of SPEC.md observe_eulerian / PAPER §3.2 (the reference
            // specifies but does not implement the inverse module; restated from the SPEC formula)
            const bool eul = sd && sd->kind == MPM_SEEDER_EULERIAN_LS;
            auto find = [&](int64_t step) {
                if (!sd || (sd->kind != MPM_SEEDER_LAGRANGIAN_LS && !eul))
                    return -1;
                for (int k = 0; k < sd->n_obs; ++k)
                    if (sd->obs_steps[k] == step)
                        return k;
                return -1;
            };
            int64_t nsel = eul ? sd->n_regions : (sd && sd->sel ? sd->n_sel : n);
            auto pid = [&](int64_t l) { return sd && sd->sel ? sd->sel[l] : l; };
            auto tgt = [&](int k, int64_t l) { return static_cast<const T*>(sd->target) + (int64_t(k) * nsel + l) * D; };
            // Eulerian: Q_l = mean z over particles p with |x_p - c_l| <= h_l (every axis), in index order
            auto inside = [&](const State<T, D>& s, int64_t p, int64_t l) {
                const T* c = static_cast<const T*>(sd->centers) + l * D;
                const T* h = static_cast<const T*>(sd->half) + l * D;
                for (int a = 0; a < D; ++a)
                    if (!(std::fabs(s.x[p].a[a] - c[a]) <= h[a]))
                        return false;
                return true;
            };
            auto region = [&](int k, const State<T, D>& s, int64_t l, T* r) { // r = m (Q - target); count
                const auto& z = sd->field == 0 ? s.x : s.v;
                T sum[D] = {}, cnt = T(0);
                for (int64_t p = 0; p < s.n; ++p)
                    if (inside(s, p, l)) {
                        for (int a = 0; a < D; ++a)
                            sum[a] += z[p].a[a];
                        cnt += T(1);
                    }
                const bool on = cnt > T(0) && (!sd->mask || sd->mask[int64_t(k) * nsel + l]);
                for (int a = 0; a < D; ++a)
                    r[a] = on ? sum[a] / cnt - tgt(k, l)[a] : T(0);
                return on ? cnt : T(0);
            };
            auto loss_at = [&](int64_t step, const State<T, D>& s) {
                int k = find(step);
                T L = T(0);
                if (eul) {
                    for (int64_t l = 0; l < nsel; ++l) {
                        T r[D];
                        region(k, s, l, r);
                        for (int a = 0; a < D; ++a)
                            L += r[a] * r[a];
                    }
                    return L;
                }
                const auto& z = sd->field == 0 ? s.x : s.v;
                for (int64_t l = 0; l < nsel; ++l)
                    for (int a = 0; a < D; ++a) {
                        T r = z[pid(l)].a[a] - tgt(k, l)[a];
                        L += r * r;
                    }
                return L;
            };
            auto seed = [&](int64_t step, const State<T, D>& s, Cot<T, D>& c) {
                int k = find(step);
                const auto& z = sd->field == 0 ? s.x : s.v;
                auto& zc = sd->field == 0 ? c.x : c.v;
                if (eul) { // d/dz_p of m ||Q - target||^2 = 2 m (Q - target) / |P| for every member p
                    for (int64_t l = 0; l < nsel; ++l) {
                        T r[D];
                        const T cnt = region(k, s, l, r);
                        if (cnt > T(0))
                            for (int64_t p = 0; p < s.n; ++p)
                                if (inside(s, p, l))
                                    for (int a = 0; a < D; ++a)
                                        zc[p].a[a] += T(2) * r[a] / cnt;
                    }
                    return;
                }
                for (int64_t l = 0; l < nsel; ++l)
                    for (int a = 0; a < D; ++a)
                        zc[pid(l)].a[a] += T(2) * (z[pid(l)].a[a] - tgt(k, l)[a]);
            };
            T loss = T(0);
            std::vector<State<T, D>> ckpt;
            {
                State<T, D> s = s0;
                if (find(0) >= 0)
                    loss += loss_at(0, s);
                for (int k = 0; k < nseg; ++k) {
                    ckpt.push_back(s);
                    for (int64_t t = bnd[k]; t < bnd[k + 1]; ++t) {
                        advance(sc, s);
                        if (find(t + 1) >= 0)
                            loss += loss_at(t + 1, s);
                    }
                }
            }
            Cot<T, D> cot, cprev;
            cot.zeros(n, s0.has_B);
            PG<T, D> pg = load_pg(sc, pgv);
            PG<T, D> acc;
            for (int w = 0; w < 2 * D; ++w)
                acc.fr[w].assign(sc.friction[w].size(), T(0));
            int64_t peak = 0;
            std::vector<State<T, D>> replay;
            for (int k = nseg - 1; k >= 0; --k) {
                replay.clear();
                replay.push_back(ckpt[k]);
                State<T, D> s = ckpt[k];
                for (int64_t t = bnd[k]; t < bnd[k + 1]; ++t) {
                    advance(sc, s);
                    replay.push_back(s);
                }
                peak = std::max<int64_t>(peak, int64_t(replay.size()));
                for (int64_t t = bnd[k + 1]; t > bnd[k]; --t) {
                    if (find(t) >= 0)
                        seed(t, replay[t - bnd[k]], cot);
                    step_vjp(sc, replay[t - bnd[k] - 1], cot, cprev, acc);
                    std::swap(cot, cprev);
                }
            }
            if (find(0) >= 0)
                seed(0, s0, cot);
            store_cot(cot, c0);
            pg.c += acc.c;
            pg.mu += acc.mu;
            for (int w = 0; w < 2 * D; ++w)
                for (size_t k = 0; k < pg.fr[w].size(); ++k)
                    pg.fr[w][k] += acc.fr[w][k];
            store_pg(pg, pgv);
            if (res) {
                res->loss = double(loss);
                res->checkpoints_stored = nseg;
                res->peak_replay_states = peak;
            }
            return MPM_OK;
        });
    }
};
template <class T, int D> struct OpHash {
    static uint64_t run(const mpm_scene_desc*, const mpm_state_view* v) { return hash_state<T, D>(v); }
};
template <class T, int D> struct OpTimer {
    static double run(const mpm_scene_desc* d, mpm_state_view* v, int64_t n)
    {
        Scene<T, D> sc = decode<T, D>(d);
        State<T, D> s = load_state<T, D>(v);
        double secs = -1;
        guarded([&] {
            auto t0 = std::chrono::steady_clock::now();
            for (int64_t i = 0; i < n; ++i)
                advance(sc, s);
            auto t1 = std::chrono::steady_clock::now();
            secs = std::chrono::duration<double>(t1 - t0).count() / double(n) * 1000.0;
            return MPM_OK;
        });
        store_state(s, v);
        return secs;
    }
};

} // namespace orc

using namespace orc;

extern "C" {

int orc_last_error(int64_t* particle, char* msg, size_t len)
{
    if (particle)
        *particle = g_particle;
    if (msg && len) {
        std::strncpy(msg, g_msg.c_str(), len - 1);
        msg[len - 1] = 0;
    }
    return 0;
}

// DruckerPragerParams::make + dp_derived_params (material.hpp:37-84)
int orc_dp_make(mpm_scene_desc* d, double rho0, double K, double nu, double phi, double psi, double cohesion,
                double sigma_t)
{
    double s3 = std::sqrt(3.0);
    d->material = MPM_MAT_DRUCKER_PRAGER;
    d->rho0 = rho0;
    d->K = K;
    d->nu = nu;
    d->G = 3.0 * K * (1.0 - 2.0 * nu) / (2.0 * (1.0 + nu));
    d->phi = phi;
    d->psi = psi;
    d->cohesion = cohesion;
    d->sigma_t = sigma_t;
    d->q_phi = 6.0 * std::sin(phi) / (s3 * (3.0 + std::sin(phi)));
    d->k_phi = 6.0 * cohesion * std::cos(phi) / (s3 * (3.0 + std::sin(phi)));
    d->q_psi = 6.0 * std::sin(psi) / (s3 * (3.0 + std::sin(psi)));
    d->tau_P = d->k_phi - d->q_phi * sigma_t;
    d->alpha_P = std::sqrt(1.0 + d->q_phi * d->q_phi) - d->q_phi;
    // validate (material.hpp:86-104)
    if (!(rho0 > 0) || !(K > 0) || !(nu >= 0 && nu < 0.5) || !(d->G > 0) || !(phi >= 0 && phi < 1.5707963267948966)
        || !(psi >= 0 && psi <= phi) || cohesion < 0 || sigma_t < 0
        || (d->q_phi > 0 && sigma_t > d->k_phi / d->q_phi)) {
        g_msg = "drucker_prager: invalid parameters";
        return MPM_ERR_VALIDATION;
    }
    return MPM_OK;
}

int64_t orc_init_scene_count(const mpm_scene_desc* d, const orc_region* r, int nreg)
{
    return dispatch<OpInitCount>(d, r, nreg);
}
int orc_init_scene(const mpm_scene_desc* d, const orc_region* r, int nreg, mpm_state_view* out, double* meps)
{
    return dispatch<OpInit>(d, r, nreg, out, meps);
}
int orc_advance(const mpm_scene_desc* d, mpm_state_view* s, int64_t n, int guard)
{
    return dispatch<OpAdvance>(d, s, n, guard);
}
int orc_p2g(const mpm_scene_desc* d, const mpm_state_view* s, mpm_grid_view* g) { return dispatch<OpP2G>(d, s, g); }
int orc_grid_momentum_update(const mpm_scene_desc* d, mpm_grid_view* g) { return dispatch<OpMom>(d, g); }
int orc_grid_corrections(const mpm_scene_desc* d, mpm_grid_view* g) { return dispatch<OpCorr>(d, g); }
int orc_g2p(const mpm_scene_desc* d, const mpm_grid_view* g, mpm_state_view* s) { return dispatch<OpG2P>(d, g, s); }
int orc_constitutive(const mpm_scene_desc* d, mpm_state_view* s) { return dispatch<OpConst>(d, s); }
int orc_step_vjp(const mpm_scene_desc* d, const mpm_state_view* s, const mpm_cot_view* co, mpm_cot_view* ci,
                 mpm_param_grads* pg)
{
    return dispatch<OpVjp>(d, s, co, ci, pg);
}
int orc_backprop(const mpm_scene_desc* d, const mpm_state_view* s0, int64_t total, int nseg,
                 const mpm_seeder_desc* sd, mpm_cot_view* c0, mpm_param_grads* pg, mpm_backprop_result* res)
{
    return dispatch<OpBackprop>(d, s0, total, nseg, sd, c0, pg, res);
}
uint64_t orc_state_hash(const mpm_scene_desc* d, const mpm_state_view* s) { return dispatch<OpHash>(d, s); }
double orc_run_seconds_per_1000(const mpm_scene_desc* d, mpm_state_view* s, int64_t n)
{
    return dispatch<OpTimer>(d, s, n);
}

} // extern "C"
