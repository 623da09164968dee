// k_material.cuh — state-dependent coefficients and zone radiation on the
// per-step path:
//   * k_star_tables: StarTables (wall.cpp:89-138) of one layer for every
//     nonlinear wall — the node set at node j and the half set at the
//     midpoint j+1/2, from the load-bearing material (hyg_material.cuh) or the
//     analytic functor; strict (DF steps: a box violation is a domain error
//     at the lowest wall, first node then first half node, wall.cpp:99-126)
//     or clamped (starting steps).  One thread per cell, two evaluations per
//     cell like the reference (n node + n-1 half evaluations per wall).
//   * k_implicit_table_pass: implicit_wall_pass (wall.cpp:433-513) of the
//     nonlinear walls inside the building fixed point, Thomas elimination as
//     solve_tridiagonal (tridiag.hpp:11-23), one thread per wall.
//   * k_radiation: radiation_fluxes (building.cpp:88-105) — per wall face the
//     long-wave flux of its zone's radiation links from a temperature layer.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hyg_material.cuh"
#include "k_step.cuh"

namespace hyg {

struct StarArgs {
    int n_walls, n;
    const double* u;            // the layer the coefficients are frozen at
    const double* v;
    const int* wall_kind;       // [n_walls] kCoeff*
    double p[4];                // analytic functor
    double T_i, P_vi;           // ScalingContext
    const mat::Set* ref;        // [n_walls] reference sets of material walls
    int strict;
    double* node;               // [6][cells]
    double* half;               // [3][cells]
    int64_t cells;
    int64_t layer;              // layer of (u, v)
    unsigned long long* fail_key;
    unsigned long long* dom_key;   // (wall << 32) | order, order = j (node) or n + j (half)
    int64_t own0, own1;
    int exact;                  // 1: the parity evaluation (CrMath, IEEE divisions); 0: evaluate_fast
};

__device__ __forceinline__ bool star_at(const StarArgs& a, int wk, int w, double u, double v, mat::Set& s) {
    if (wk == kCoeffAnalyticD) {
        s = mat::Set{1.0, analytic_kM(a.p, v), 1.0, 1.0, 1.0, 1.0};
        return true;
    }
    return mat::star(u, v, a.T_i, a.P_vi, a.ref[w], a.strict != 0, s, a.exact != 0);
}

__device__ __forceinline__ void star_fail(const StarArgs& a, int w, unsigned order) {
    atomicMin(a.dom_key, (static_cast<unsigned long long>(w) << 32) | order);
    atomicMin(a.fail_key, (static_cast<unsigned long long>(a.layer + 1) << 32) | static_cast<unsigned>(w));
}

__global__ void __launch_bounds__(128) k_star_tables(const StarArgs a) {
    const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= a.cells) return;
    if (a.strict && frozen_before(a.fail_key, a.layer)) return;
    const int w = static_cast<int>(c / a.n), j = static_cast<int>(c - static_cast<int64_t>(w) * a.n);
    const int wk = a.wall_kind[w];
    if (wk == kCoeffConstant) return;
    const bool own = c >= a.own0 && c < a.own1;
    const double uc = a.u[c], vc = a.v[c];
    mat::Set s;
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    const mat::Set bad{nan, nan, nan, nan, nan, nan};   // clamped evaluation of a NaN state
    bool ok = star_at(a, wk, w, uc, vc, s);
    if (!ok && a.strict && own) star_fail(a, w, static_cast<unsigned>(j));
    if (!ok) s = bad;
    {
        a.node[kSc_M * a.cells + c] = s.c_M;
        a.node[kSk_M * a.cells + c] = s.k_M;
        a.node[kSc_TT * a.cells + c] = s.c_TT;
        a.node[kSk_TT * a.cells + c] = s.k_TT;
        a.node[kSc_TM * a.cells + c] = s.c_TM;
        a.node[kSk_TM * a.cells + c] = s.k_TM;
    }
    if (j + 1 < a.n) {
        const double um = 0.5 * (uc + a.u[c + 1]), vm = 0.5 * (vc + a.v[c + 1]);
        ok = star_at(a, wk, w, um, vm, s);
        if (!ok && a.strict && own) star_fail(a, w, static_cast<unsigned>(a.n + j));
        if (!ok) s = bad;
        a.half[kHk_M * a.cells + c] = s.k_M;
        a.half[kHk_TT * a.cells + c] = s.k_TT;
        a.half[kHk_TM * a.cells + c] = s.k_TM;
    }
}

// implicit_wall_pass (wall.cpp:433-513) for one nonlinear wall: tables built
// (clamped) from the current iterate out[1]/out[3]; base layer n = in[1]/in[3].
// Scratch node-major [5][n][n_walls].  Writes the new iterate, max |change|
// into *diff and layer n into out[0]/out[2], like k_implicit_unit_pass.
__global__ void k_implicit_table_pass(const StepArgs a, double* scr, unsigned long long* diff) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= a.n_walls || a.wall_kind[w] == kCoeffConstant) return;
    const int n = a.n, B = a.n_walls;
    const double dx = a.dx, dt = a.dt;
    const Groups p = a.groups[w];
    const int64_t o = static_cast<int64_t>(w) * n;
    const double *uc = a.in[1] + o, *vc = a.in[3] + o;
    const size_t nb = static_cast<size_t>(n) * B;
    double *LO = scr, *DI = scr + nb, *UP = scr + 2 * nb, *XV = scr + 3 * nb, *XU = scr + 4 * nb;
    auto at = [&](double* base, int i) -> double& { return base[static_cast<size_t>(i) * B + w]; };
    const StarTab& s = a.star;
    const FaceVals F[2] = {resolve(a, w, 0), resolve(a, w, 1)};
    const double r = p.Fo_M * dt / (dx * dx);
    const double rb = p.Fo_TT * dt / (dx * dx);
    const double rg = p.Fo_TM * p.gamma * dt / (dx * dx);
    auto thomas = [&](double* X) {                     // solve_tridiagonal tridiag.hpp:11-23
        for (int i = 1; i < n; ++i) {
            const double m = at(LO, i) / at(DI, i - 1);
            at(DI, i) -= m * at(UP, i - 1);
            at(X, i) -= m * at(X, i - 1);
        }
        at(X, n - 1) /= at(DI, n - 1);
        for (int i = n - 1; i-- > 0;) at(X, i) = (at(X, i) - at(UP, i) * at(X, i + 1)) / at(DI, i);
    };
    // moisture system (wall.cpp:456-476)
    for (int j = 1; j + 1 < n; ++j) {
        const double kp = s.hf(kHk_M, o + j), km = s.hf(kHk_M, o + j - 1);
        at(LO, j) = -r * km;
        at(DI, j) = s.nd(kSc_M, o + j) + r * (kp + km);
        at(UP, j) = -r * kp;
        at(XV, j) = s.nd(kSc_M, o + j) * vc[j];
    }
    for (int k = 0; k < 2; ++k) {
        const int jb = k == 0 ? 0 : n - 1;
        const FaceVals& b = F[k];
        const int64_t hb = o + (jb == 0 ? 0 : n - 2);
        const double km_b = s.nd(kSk_M, o + jb), kp_b = s.hf(kHk_M, hb);
        at(DI, jb) = s.nd(kSc_M, o + jb) + r * (kp_b + km_b) + 2.0 * r * dx * b.Bi_M;
        const double off = -r * (kp_b + km_b);
        if (jb == 0) at(UP, 0) = off; else at(LO, n - 1) = off;
        at(XV, jb) = s.nd(kSc_M, o + jb) * vc[jb] + 2.0 * r * dx * (b.Bi_M * b.v_inf + b.g_inf);
    }
    thomas(XV);
    // energy system with the new moisture layer as data (wall.cpp:481-510)
    for (int j = 1; j + 1 < n; ++j) {
        const double ktp = s.hf(kHk_TT, o + j), ktm = s.hf(kHk_TT, o + j - 1);
        const double kmp = s.hf(kHk_TM, o + j), kmm = s.hf(kHk_TM, o + j - 1);
        at(LO, j) = -rb * ktm;
        at(DI, j) = s.nd(kSc_TT, o + j) + rb * (ktp + ktm);
        at(UP, j) = -rb * ktp;
        at(XU, j) = s.nd(kSc_TT, o + j) * uc[j] - p.gamma * s.nd(kSc_TM, o + j) * (at(XV, j) - vc[j]) +
                    rg * (kmp * (at(XV, j + 1) - at(XV, j)) - kmm * (at(XV, j) - at(XV, j - 1)));
    }
    for (int k = 0; k < 2; ++k) {
        const int jb = k == 0 ? 0 : n - 1, jn = k == 0 ? 1 : n - 2;
        const FaceVals& b = F[k];
        const int64_t hb = o + (jb == 0 ? 0 : n - 2);
        const double kt_b = s.nd(kSk_TT, o + jb), kTM_b = s.nd(kSk_TM, o + jb);
        const double ctt = s.nd(kSc_TT, o + jb), ctm = s.nd(kSc_TM, o + jb);
        at(DI, jb) = ctt + rb * (s.hf(kHk_TT, hb) + kt_b) + 2.0 * rb * dx * b.Bi_TT;
        const double off = -rb * (s.hf(kHk_TT, hb) + kt_b);
        if (jb == 0) at(UP, 0) = off; else at(LO, n - 1) = off;
        at(XU, jb) = ctt * uc[jb] - p.gamma * ctm * (at(XV, jb) - vc[jb]) +
                     rg * (s.hf(kHk_TM, hb) + kTM_b) * (at(XV, jn) - at(XV, jb)) +
                     2.0 * rb * dx * (b.Bi_TT * b.u_inf - b.Bi_TM * (at(XV, jb) - b.v_inf) + b.q_inf);
    }
    thomas(XU);
    double* uout = a.out[1] + o;
    double* vout = a.out[3] + o;
    double d = 0.0, mx = 0.0;
    bool finite = true;
    for (int i = 0; i < n; ++i) {
        const double nu = at(XU, i), nv = at(XV, i);
        d = fmax(d, fabs(nu - uout[i]));     // building.cpp:231-234
        d = fmax(d, fabs(nv - vout[i]));
        uout[i] = nu;
        vout[i] = nv;
        a.out[0][o + i] = uc[i];
        a.out[2][o + i] = vc[i];
        mx = fmax(mx, fmax(fabs(nu), fabs(nv)));
        finite = finite && isfinite(nu) && isfinite(nv);
    }
    const bool own = o >= a.own0 && o + n <= a.own1;
    if (own) atomic_max_nonneg(diff, d);
    if (own && (!(mx <= a.norm) || !finite)) {
        const unsigned long long key =
            (static_cast<unsigned long long>(a.layer + 1) << 32) | static_cast<unsigned>(w);
        atomicMin(a.fail_key, key);
    }
}

// ---- radiation ------------------------------------------------------------------
// For every wall face (target 2*w+face): the groups (one per zone link of
// that face, in zone / link order) and their terms (radiation links whose
// receiver is the linked wall, in link order): emitter and receiver surface
// cells as zone_surface_u resolves them for that zone (-1: the wall has no
// link to the zone, surface 0), coef = view_factor * emissivity * sigma.
struct RadArgs {
    int n_targets;
    const int* tgt_off;        // [n_targets + 1] -> groups
    const int* grp_off;        // [n_groups + 1] -> terms
    const double* grp_num;     // BuildingWall::thickness
    const double* grp_den;     // T_i * BuildingWall::k_TT0
    const int64_t* t_e;
    const int64_t* t_r;
    const double* t_coef;
    double T_i;
    const double* u;           // wall temperature layer
    double* q;                 // [n_targets]
};

__global__ void k_radiation(const RadArgs a) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.n_targets) return;
    double q = 0.0;
    for (int g = a.tgt_off[t]; g < a.tgt_off[t + 1]; ++g) {
        double q_rw = 0.0;                          // radiative_flux zone.cpp:55-67
        for (int i = a.grp_off[g]; i < a.grp_off[g + 1]; ++i) {
            const double Te = (a.t_e[i] >= 0 ? a.u[a.t_e[i]] : 0.0) * a.T_i;
            const double Tr = (a.t_r[i] >= 0 ? a.u[a.t_r[i]] : 0.0) * a.T_i;
            q_rw += a.t_coef[i] * (Te * Te * Te * Te - Tr * Tr * Tr * Tr);
        }
        if (q_rw != 0.0) q += a.grp_num[g] * q_rw / a.grp_den[g];
    }
    a.q[t] = q;
}

}  // namespace hyg

namespace hyg {

// ---- fused material step --------------------------------------------------------
// One DF step of a building whose walls are (partly) material walls, StarTables
// and rows in one launch: a 256-thread CTA owns 255 consecutive cells; thread t
// evaluates the node set of cell base+t (t < 255) and the half set between
// cells base+t-1 and base+t (the 256 half nodes its 255 cells need), both into
// shared memory — two evaluations per lane as in the reference, balanced
// across warps — then runs the literal rows of df_step_nonlinear (material
// walls) or the increment rows (constant walls) for its cell.  A strict
// evaluation outside the box raises the domain key; the step's outputs go to
// the scratch layer and the host discards them (the failing step never ran).
// Blocks >= wall_blocks advance the zones (k_building_step).
constexpr int kMatThreads = 256, kMatCells = 255;

// df_step_nonlinear rows (wall.cpp:213-259) from the CTA's shared tables:
// node f at nS[f*256 + t], half (j-1)+1/2 at hS[f*256 + t], j+1/2 at hS[f*256 + t+1]
// p: the wall's groups, loaded by the caller before the StarTables evaluation.
// !EXACT (the default): reciprocals (frcp, 3 FMAs) instead of the divisions,
// <= 1 ulp per quotient (cfg5 1.78e10 -> 1.90e10); a zero denominator gives
// NaN where the division gave inf, both trip the guard.  EXACT
// (HYG_TUNE_MATERIAL_EXACT): the reference's statements with IEEE divisions
// (and, the library being built with -fmad=false, no contraction).
template <bool EXACT>
__device__ __forceinline__ void material_cell(const StepArgs& a, const NodeIn& x, int w, int j, const Groups& p,
                                              const double* nS, const double* hS, int t, double& un, double& vn) {
    const int n = a.n;
    const double dx = a.dx, dt = a.dt;
    const double idx2 = EXACT ? 0.0 : frcp(dx * dx);
    const double ad = EXACT ? p.Fo_M * dt / (dx * dx) : p.Fo_M * dt * idx2;
    const double b_ = EXACT ? p.Fo_TT * dt / (dx * dx) : p.Fo_TT * dt * idx2;
    const double g_ = EXACT ? p.Fo_TM * p.gamma * dt / (dx * dx) : p.Fo_TM * p.gamma * dt * idx2;
    const double ratio = p.Fo_TT != 0.0 ? (EXACT ? p.Fo_TM * p.gamma / p.Fo_TT : p.Fo_TM * p.gamma * frcp(p.Fo_TT)) : 0.0;
#define MAT_DIV(x, y) (EXACT ? (x) / (y) : (x) * frcp(y))
    auto nd = [&](int f) { return nS[f * kMatThreads + t]; };
    auto hl = [&](int f) { return hS[f * kMatThreads + t]; };       // (j-1)+1/2
    auto hr = [&](int f) { return hS[f * kMatThreads + t + 1]; };   // j+1/2
    if (j > 0 && j < n - 1) {
        const double kp = hr(kHk_M), km = hl(kHk_M), cm = nd(kSc_M);
        vn = MAT_DIV((cm - ad * (kp + km)) * x.vp + 2.0 * ad * (kp * x.vr + km * x.vl), cm + ad * (kp + km));
        const double ktp = hr(kHk_TT), ktm = hl(kHk_TT), kmp = hr(kHk_TM), kmm = hl(kHk_TM);
        const double ctt = nd(kSc_TT), ctm = nd(kSc_TM);
        un = MAT_DIV((ctt - b_ * (ktp + ktm)) * x.up - p.gamma * ctm * (vn - x.vp) +
                         2.0 * b_ * (ktp * x.ur + ktm * x.ul) + 2.0 * g_ * (kmp * x.vr + kmm * x.vl) -
                         g_ * (kmp + kmm) * (vn + x.vp),
                     ctt + b_ * (ktp + ktm));
        return;
    }
    const int k = j == 0 ? 0 : 1;
    const double vcn = j == 0 ? x.vr : x.vl, ucn = j == 0 ? x.ur : x.ul;
    const FaceVals b = resolve(a, w, k);
    auto hb = [&](int f) { return j == 0 ? hr(f) : hl(f); };         // half_front / half_back
    const double km_b = nd(kSk_M), kp_b = hb(kHk_M), cm = nd(kSc_M);
    const double cpl = 2.0 * ad * dx * b.Bi_M;
    vn = ((cm - ad * (kp_b + km_b) - cpl) * x.vp + 2.0 * ad * (kp_b + km_b) * vcn +
          4.0 * ad * dx * (b.Bi_M * b.v_inf + b.g_inf)) /
         (cm + ad * (kp_b + km_b) + cpl);
    const double kt_b = nd(kSk_TT), kTM_b = nd(kSk_TM);
    const double ktp_b = hb(kHk_TT), kmp_b = hb(kHk_TM);
    const double ctt = nd(kSc_TT), ctm = nd(kSc_TM);
    const double vbar = 0.5 * (vn + x.vp);
    const double vg = vcn - (2.0 * dx / km_b) * (b.Bi_M * (vbar - b.v_inf) - b.g_inf);
    const double cplu = 2.0 * b_ * dx * b.Bi_TT;
    un = ((ctt - b_ * (ktp_b + kt_b) - cplu) * x.up - p.gamma * ctm * (vn - x.vp) +
          2.0 * b_ * (ktp_b + kt_b) * ucn + 2.0 * b_ * ratio * kTM_b * (vcn - vg) -
          4.0 * b_ * dx * (b.Bi_TM * (vbar - b.v_inf) - b.q_inf) + 2.0 * cplu * b.u_inf +
          2.0 * g_ * (kmp_b * vcn + kTM_b * vg) - g_ * (kmp_b + kTM_b) * (vn + x.vp)) /
         (ctt + b_ * (ktp_b + kt_b) + cplu);
}
#undef MAT_DIV

template <bool EXACT>
__global__ void __launch_bounds__(kMatThreads, 4) k_material_step(const StepArgs a, const StarArgs s,
                                                              const ZoneArgs z, int wall_blocks) {
    if (static_cast<int>(blockIdx.x) >= wall_blocks) {              // zones (step_explicit :179-183)
        const int zi = (static_cast<int>(blockIdx.x) - wall_blocks) * blockDim.x + threadIdx.x;
        if (zi < z.n_zones && !frozen_before(z.fail_key, z.layer)) zone_update(z, zi);
        return;
    }
    __shared__ double nS[6 * kMatThreads];
    __shared__ double hS[3 * kMatThreads];
    const int t = threadIdx.x;
    const int64_t total = static_cast<int64_t>(a.n_walls) * a.n;
    const int64_t c = static_cast<int64_t>(blockIdx.x) * kMatCells + t;
    const bool out_cell = t < kMatCells && c < total;
    // loads first (they overlap the evaluations)
    int w = 0, j = 0;
    NodeIn x{};
    if (c < total) {
        w = static_cast<int>(c / a.n);
        j = static_cast<int>(c - static_cast<int64_t>(w) * a.n);
    }
    if (out_cell) x = load_node(a, w, j);
    const Groups gp = a.groups[out_cell ? w : 0];                    // in flight during the evaluations
    const bool frozen = frozen_before(a.fail_key, a.layer);
    const int wk = c < total ? a.wall_kind[w] : kCoeffConstant;
    const bool own = c >= a.own0 && c < a.own1;
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    if (!frozen && wk != kCoeffConstant) {
        mat::Set m;
        if (out_cell) {                                              // node j
            if (!star_at(s, wk, w, x.uc, x.vc, m)) {
                if (own) star_fail(s, w, static_cast<unsigned>(j));
                m = mat::Set{nan, nan, nan, nan, nan, nan};
            }
            nS[kSc_M * kMatThreads + t] = m.c_M;
            nS[kSk_M * kMatThreads + t] = m.k_M;
            nS[kSc_TT * kMatThreads + t] = m.c_TT;
            nS[kSk_TT * kMatThreads + t] = m.k_TT;
            nS[kSc_TM * kMatThreads + t] = m.c_TM;
            nS[kSk_TM * kMatThreads + t] = m.k_TM;
        }
        if (j > 0) {                                                 // half (j-1)+1/2
            const double ul = a.in[1][c - 1], vl = a.in[3][c - 1];
            const double uh = out_cell ? x.uc : a.in[1][c], vh = out_cell ? x.vc : a.in[3][c];
            if (!star_at(s, wk, w, 0.5 * (ul + uh), 0.5 * (vl + vh), m)) {
                if (own) star_fail(s, w, static_cast<unsigned>(a.n + j - 1));
                m.k_M = m.k_TT = m.k_TM = nan;
            }
            hS[kHk_M * kMatThreads + t] = m.k_M;
            hS[kHk_TT * kMatThreads + t] = m.k_TT;
            hS[kHk_TM * kMatThreads + t] = m.k_TM;
        }
    }
    __syncthreads();
    if (!out_cell || frozen) return;
    double un, vn;
    if (wk == kCoeffConstant) coupled_node(a, w, j, x, un, vn);
    else material_cell<EXACT>(a, x, w, j, gp, nS, hS, t, un, vn);
    a.out[1][c] = un;
    a.out[3][c] = vn;
    if (own && (!(fabs(un) <= a.norm) || !(fabs(vn) <= a.norm))) {
        const unsigned long long key =
            (static_cast<unsigned long long>(a.layer + 1) << 32) | static_cast<unsigned>(w);
        atomicMin(a.fail_key, key);
    }
}

}  // namespace hyg
