// k_step.cuh — one-step kernels: the general DF step (any grid size, zone
// faces, analytic coefficient functor), the explicit and implicit starting
// steps, the zone air balance and small utility kernels.
//
// These are the paths the fused K1 kernel does not cover: walls whose faces
// read zone states every step (step_explicit, building.cpp:152-187), grids
// that do not tile onto lanes, state-dependent coefficients.  One thread per
// (wall, node); layers stream through HBM/L2, so these kernels are
// memory-bound (48 B/node-update for the four read + two written layers).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hyg_coef.cuh"
#include "k_coupled.cuh"

namespace hyg {

enum : int { kCoeffConstant = 0, kCoeffAnalyticD = 1, kCoeffMaterial = 2 };

// Frozen starred coefficients of one layer (StarTables wall.cpp:89-138), SoA
// over cells: node sets at node j, half sets at the midpoint j+1/2 (stored at
// the cell of node j).  Built by k_star_tables (k_material.cuh).
enum : int { kSc_M = 0, kSk_M = 1, kSc_TT = 2, kSk_TT = 3, kSc_TM = 4, kSk_TM = 5 };   // node[6]
enum : int { kHk_M = 0, kHk_TT = 1, kHk_TM = 2 };                                    // half[3]
struct StarTab {
    const double* node;     // [6][cells]
    const double* half;     // [3][cells]
    int64_t cells;
    __device__ __forceinline__ double nd(int f, int64_t c) const { return node[f * cells + c]; }
    __device__ __forceinline__ double hf(int f, int64_t c) const { return half[f * cells + c]; }
};

struct Attach { int kind, index; };   // 0 exterior(channel), 1 zone

struct StepArgs {
    int n_walls, n;
    double dx, dt;
    const Groups* groups;
    const Biot* biot;           // [2*w+k]
    const Attach* attach;       // [2*w+k]
    int n_channels;
    const Ambient* amb;         // ambient row of this step [n_channels]
    const double* zu;           // zone states of layer n (nullable)
    const double* zv;
    int coeff_kind;
    double p[4];
    const double* in[4];        // up, uc, vp, vc
    double* out[4];             // new prev (= old curr), new curr
    int64_t layer;              // index of layer n
    double norm;
    unsigned long long* fail_key;
    int64_t own0, own1;         // cells whose guard/residual count (a shard owns a range)
    const WallCoef* coef;       // constant walls: per-wall rows for this dt (k_coupled_coef)
    const int* wall_kind;       // [n_walls] kCoeff* of each wall (per-wall CoefficientModel)
    StarTab star;               // nonlinear walls: tables of this layer (node == nullptr: none)
    const double* q_rad;        // [2*n_walls] zone radiation flux per face (nullable)
    const unsigned long long* dom_key;   // domain-error key of the material kernels
};

// A failure raised by an EARLIER step (key layer <= this step's input layer)
// freezes the march; failures raised within the step itself do not, so every
// failing wall of the step reports and atomicMin keeps the lowest index
// (check_bounded walks walls in order, building.cpp:282-300).
__device__ __forceinline__ bool frozen_before(const unsigned long long* key, int64_t layer) {
    const unsigned long long k = *key;
    return k != ~0ull && static_cast<int64_t>(k >> 32) <= layer;
}

// d(v) functor of HYG_COEFF_ANALYTIC_D: k_M* = 1 + p0 v + p1 exp(-p2 (v - p3)^2)
__device__ __forceinline__ double analytic_kM(const double* p, double v) {
    const double d = v - p[3];
    return 1.0 + p[0] * v + p[1] * exp(-p[2] * d * d);
}

struct FaceVals { double Bi_M, Bi_TT, Bi_TM, u_inf, v_inf, g_inf, q_inf; };

__device__ __forceinline__ FaceVals resolve(const StepArgs& a, int w, int k) {
    // resolve_face (building.cpp:107-126), no radiation
    const Biot b = a.biot[2 * w + k];
    const Attach at = a.attach[2 * w + k];
    const double q_rad = a.q_rad ? a.q_rad[2 * w + k] : 0.0;   // radiation_fluxes building.cpp:88-105
    FaceVals f{b.Bi_M, b.Bi_TT, b.Bi_TM, 1.0, 1.0, 0.0, 0.0};
    if (at.kind == 0) {
        const Ambient am = a.amb[at.index];
        f.u_inf = am.u;
        f.v_inf = am.v;
        f.g_inf = am.g;
        f.q_inf = am.q + q_rad;
    } else {
        f.u_inf = a.zu[at.index];
        f.v_inf = a.zv[at.index];
        f.q_inf = q_rad;
    }
    return f;
}

// The node's inputs, loaded before anything else so a warp's loads are all in
// flight together (the per-step path is memory-latency-bound).  At a face
// the missing neighbour is the mirrored interior one.
struct NodeIn { double vp, up, vc, uc, vl, vr, ul, ur; };

__device__ __forceinline__ NodeIn load_node(const StepArgs& a, int w, int j) {
    const int n = a.n;
    const size_t o = static_cast<size_t>(w) * n;
    const int jl = j == 0 ? 1 : j - 1, jr = j == n - 1 ? n - 2 : j + 1;
    NodeIn x;
    x.vp = a.in[2][o + j];
    x.up = a.in[0][o + j];
    x.vc = a.in[3][o + j];
    x.uc = a.in[1][o + j];
    x.vl = a.in[3][o + jl];
    x.vr = a.in[3][o + jr];
    x.ul = a.in[1][o + jl];
    x.ur = a.in[1][o + jr];
    return x;
}

// df_step_coupled (wall.cpp:144-194), one node per thread, in the increment
// form of hyg_coef.cuh with the per-wall coefficients of this dt (a.coef):
// the same arithmetic as K1, so fused and per-step marches agree, and no
// divisions per node (the per-step path stays HBM-bound, 48 B/update).
__device__ __forceinline__ void coupled_node(const StepArgs& a, int w, int j, const NodeIn& x, double& un,
                                             double& vn) {
    const int n = a.n;
    const double d = fma(-2.0, x.vp, x.vl + x.vr);
    const double du = fma(-2.0, x.up, x.ul + x.ur);
    if (j > 0 && j < n - 1) {
        const RowCoef& c = a.coef[w].in;
        vn = fma(c.b, d, x.vp);
        un = fma(c.c_sv, d, fma(c.c_su, du, x.up));
        return;
    }
    const RowCoef& c = a.coef[w].face[j == 0 ? 0 : 1];
    const FaceVals b = resolve(a, w, j == 0 ? 0 : 1);
    const double t = b.v_inf - x.vp, tu = b.u_inf - x.up;
    vn = fma(c.e, t, fma(c.b, d, fma(c.e_g, b.g_inf, x.vp)));
    un = fma(c.c_tv, t, fma(c.c_sv, d, fma(c.c_tu, tu, fma(c.c_su, du, fma(c.c_q, b.q_inf, fma(c.c_g, b.g_inf, x.up))))));
}

// df_step_nonlinear (wall.cpp:196-264) for the analytic functor (k_M* = d(v),
// the other five starred coefficients 1), one node per thread, literal form.
// StarTables (wall.cpp:89-138): node values at j, half-node values at the
// midpoint state average.
__device__ __forceinline__ void analytic_node(const StepArgs& a, int w, int j, const NodeIn& x, double& un,
                                              double& vn) {
    const int n = a.n;
    const double dx = a.dx, dt = a.dt;
    const Groups p = a.groups[w];
    const double ad = p.Fo_M * dt / (dx * dx);
    const double b_ = p.Fo_TT * dt / (dx * dx);
    const double g_ = p.Fo_TM * p.gamma * dt / (dx * dx);
    const double ratio = p.Fo_TT != 0.0 ? p.Fo_TM * p.gamma / p.Fo_TT : 0.0;
    const double cm = 1.0, ctt = 1.0, ctm = 1.0;
    if (j > 0 && j < n - 1) {
        const double kp = analytic_kM(a.p, 0.5 * (x.vc + x.vr));
        const double km = analytic_kM(a.p, 0.5 * (x.vl + x.vc));
        vn = ((cm - ad * (kp + km)) * x.vp + 2.0 * ad * (kp * x.vr + km * x.vl)) / (cm + ad * (kp + km));
        const double ktp = 1.0, ktm = 1.0, kmp = 1.0, kmm = 1.0;
        un = ((ctt - b_ * (ktp + ktm)) * x.up - p.gamma * ctm * (vn - x.vp) +
              2.0 * b_ * (ktp * x.ur + ktm * x.ul) + 2.0 * g_ * (kmp * x.vr + kmm * x.vl) -
              g_ * (kmp + kmm) * (vn + x.vp)) /
             (ctt + b_ * (ktp + ktm));
        return;
    }
    const int k = j == 0 ? 0 : 1;
    const double vcn = j == 0 ? x.vr : x.vl, ucn = j == 0 ? x.ur : x.ul;   // vc[jn], uc[jn]
    const FaceVals b = resolve(a, w, k);
    const double km_b = analytic_kM(a.p, x.vc);                        // ghost side: node value
    const double kp_b = analytic_kM(a.p, j == 0 ? 0.5 * (x.vc + vcn) : 0.5 * (vcn + x.vc));
    const double cpl = 2.0 * ad * dx * b.Bi_M;
    vn = ((cm - ad * (kp_b + km_b) - cpl) * x.vp + 2.0 * ad * (kp_b + km_b) * vcn +
          4.0 * ad * dx * (b.Bi_M * b.v_inf + b.g_inf)) /
         (cm + ad * (kp_b + km_b) + cpl);
    const double kt_b = 1.0, kTM_b = 1.0, ktp_b = 1.0, kmp_b = 1.0;
    const double vbar = 0.5 * (vn + x.vp);
    const double vg = vcn - (2.0 * dx / km_b) * (b.Bi_M * (vbar - b.v_inf) - b.g_inf);
    const double cplu = 2.0 * b_ * dx * b.Bi_TT;
    un = ((ctt - b_ * (ktp_b + kt_b) - cplu) * x.up - p.gamma * ctm * (vn - x.vp) +
          2.0 * b_ * (ktp_b + kt_b) * ucn + 2.0 * b_ * ratio * kTM_b * (vcn - vg) -
          4.0 * b_ * dx * (b.Bi_TM * (vbar - b.v_inf) - b.q_inf) + 2.0 * cplu * b.u_inf +
          2.0 * g_ * (kmp_b * vcn + kTM_b * vg) - g_ * (kmp_b + kTM_b) * (vn + x.vp)) /
         (ctt + b_ * (ktp_b + kt_b) + cplu);
}

// One DF step of NPT nodes per thread (cells base + k * stride); guard per
// node (exact check_bounded semantics).  Every state load of all NPT nodes is
// issued before the stop flag is read and before any arithmetic, so a thread
// keeps 4·NPT DRAM loads in flight (the per-step path is bound by bytes in
// flight, profiles/r01_cfg3_cfg0_cfg4_ncu_summary.md).
template <int NPT, int KIND>
__device__ __forceinline__ void wall_nodes_step(const StepArgs& a, int64_t base, int stride) {
    const int64_t total = static_cast<int64_t>(a.n_walls) * a.n;
    const bool narrow = total <= 0xffffffffll;       // 32-bit cell -> (wall, node)
    NodeIn x[NPT];
    int w[NPT], j[NPT];
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int64_t cell = base + static_cast<int64_t>(k) * stride;
        w[k] = -1;
        if (cell < total) {
            if (narrow) {
                const unsigned c32 = static_cast<unsigned>(cell), n32 = static_cast<unsigned>(a.n);
                w[k] = static_cast<int>(c32 / n32);
                j[k] = static_cast<int>(c32 - static_cast<unsigned>(w[k]) * n32);
            } else {
                w[k] = static_cast<int>(cell / a.n);
                j[k] = static_cast<int>(cell - static_cast<int64_t>(w[k]) * a.n);
            }
            x[k] = load_node(a, w[k], j[k]);
        }
    }
    if (frozen_before(a.fail_key, a.layer)) return;    // an earlier step failed: freeze
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        if (w[k] < 0) continue;
        const int64_t cell = base + static_cast<int64_t>(k) * stride;
        double un, vn;
        // (material walls step in k_material_step, k_material.cuh)
        if (KIND == kCoeffConstant) coupled_node(a, w[k], j[k], x[k], un, vn);
        else analytic_node(a, w[k], j[k], x[k], un, vn);
        // only the new layer is written; the host rotates layer pointers
        // (prev <- curr) instead of copying: 32 B read + 16 B written per update
        a.out[1][cell] = un;
        a.out[3][cell] = vn;
        if (cell >= a.own0 && cell < a.own1 && (!(fabs(un) <= a.norm) || !(fabs(vn) <= a.norm))) {
            const unsigned long long key =
                (static_cast<unsigned long long>(a.layer + 1) << 32) | static_cast<unsigned>(w[k]);
            atomicMin(a.fail_key, key);
        }
    }
}

constexpr int kStepThreads = 256;
// nodes per thread of the per-step kernels: two for the lean constant rows,
// one for the d(v) rows (two would spill at the 64-register budget)
__host__ __device__ constexpr int step_npt(int kind) { return kind == kCoeffConstant ? 2 : 1; }
__host__ __device__ constexpr int step_cells(int kind) { return kStepThreads * step_npt(kind); }

template <int KIND>
__global__ void __launch_bounds__(kStepThreads, KIND == kCoeffConstant ? 4 : 3) k_df_step_general(const StepArgs a) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * step_cells(KIND) + threadIdx.x;
    wall_nodes_step<step_npt(KIND), KIND>(a, base, kStepThreads);
}

// ---- zones -----------------------------------------------------------------
struct ZoneDev {
    double kappa_a_tt1, g_v, q_v1, q_v2, sign;
    int sources;
    int wall_begin, wall_end;     // range in the link arrays
    int inz_begin, inz_end;
};
struct ZoneLinkDev { int wall, face; double Bi_M, Bi_TT, Bi_TM, theta_T, theta_M; };
struct InzLinkDev { int peer; double g_inz, q_inz1, q_inz2; };

struct ZoneArgs {
    int n_zones, n;
    double dt;
    const ZoneDev* zones;
    const ZoneLinkDev* links;
    const InzLinkDev* inz;
    const double* src;       // this step: [n_sources][3] (g_o, q_o, q_h) then outdoor u, v
    int n_sources;
    const double* uc;        // wall layer n (surface samples)
    const double* vc;
    const double* zu_in;
    const double* zv_in;
    double* zu_out;
    double* zv_out;
    int64_t layer;
    double norm;
    unsigned long long* fail_key;
    int own0, own1;             // zones whose guard counts
};

// zone_step_explicit (zone.cpp:69-74) of zone_rhs (zone.cpp:26-53) with the
// layer-n samples gathered as in building.cpp:128-140,162-164.
__device__ __forceinline__ void zone_update(const ZoneArgs& a, int z) {
    const ZoneDev d = a.zones[z];
    const double u_a = a.zu_in[z], v_a = a.zv_in[z];
    const double* s = a.src + 3 * d.sources;
    const double u_inf = a.src[3 * a.n_sources + 0], v_inf = a.src[3 * a.n_sources + 1];
    double du = s[1] + s[2] + d.q_v1 * (u_inf * v_inf - u_a * v_a) + d.q_v2 * (u_inf - u_a);
    double dv = s[0] + d.g_v * (v_inf - v_a);
    for (int i = d.inz_begin; i < d.inz_end; ++i) {
        const InzLinkDev l = a.inz[i];
        const double pu = a.zu_in[l.peer], pv = a.zv_in[l.peer];
        du += l.q_inz1 * (pu * pv - u_a * v_a) + l.q_inz2 * (pu - u_a);
        dv += l.g_inz * (pv - v_a);
    }
    for (int i = d.wall_begin; i < d.wall_end; ++i) {
        const ZoneLinkDev l = a.links[i];
        const size_t idx = static_cast<size_t>(l.wall) * a.n + (l.face == 0 ? 0 : a.n - 1);
        const double us = a.uc[idx], vs = a.vc[idx];
        du += l.Bi_TT * l.theta_T * (us - u_a) + l.Bi_TM * l.theta_T * (vs - v_a);
        dv += d.sign * l.Bi_M * l.theta_M * (v_a - vs);
    }
    const double nu = u_a + a.dt * (du / (1.0 + d.kappa_a_tt1));
    const double nv = v_a + a.dt * dv;
    a.zu_out[z] = nu;
    a.zv_out[z] = nv;
    if (z >= a.own0 && z < a.own1 &&
        (!isfinite(nu) || !isfinite(nv) || fabs(nu) > a.norm || fabs(nv) > a.norm)) {
        // zone failures rank after every wall of the same layer (building.cpp:288-299)
        const unsigned long long key = (static_cast<unsigned long long>(a.layer + 1) << 32) | 0xffffffffu;
        atomicMin(a.fail_key, key);
    }
}

__global__ void k_zone_step(const ZoneArgs a) {
    const int z = blockIdx.x * blockDim.x + threadIdx.x;
    if (z >= a.n_zones) return;
    if (frozen_before(a.fail_key, a.layer)) return;
    zone_update(a, z);
}

// One building step (step_explicit, building.cpp:152-187) in one launch: the
// first wall_blocks blocks advance the wall nodes with layer-n zone values,
// the remaining blocks advance the zones with layer-n surface samples.  Both
// halves read layer n only and write disjoint buffers.
template <int KIND>
__global__ void __launch_bounds__(kStepThreads, KIND == kCoeffConstant ? 4 : 3) k_building_step(const StepArgs a, const ZoneArgs z,
                                                                  int wall_blocks) {
    if (static_cast<int>(blockIdx.x) < wall_blocks) {
        const int64_t base = static_cast<int64_t>(blockIdx.x) * step_cells(KIND) + threadIdx.x;
        wall_nodes_step<step_npt(KIND), KIND>(a, base, kStepThreads);
    } else {
        const int zi = (static_cast<int>(blockIdx.x) - wall_blocks) * blockDim.x + threadIdx.x;
        if (zi < z.n_zones && !frozen_before(z.fail_key, z.layer)) zone_update(z, zi);
    }
}

// ---- starting steps --------------------------------------------------------
// euler_explicit_step (wall.cpp:266-317), one node per thread.  Coefficients
// are clamped (strict=false): material walls read the layer's tables (built
// clamped by k_star_tables), the analytic functor (no box) is evaluated
// inline, constant walls use the unit set.
__global__ void k_explicit_boot(const StepArgs a) {
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t total = static_cast<int64_t>(a.n_walls) * a.n;
    if (tid >= total) return;
    const int n = a.n;
    const int w = static_cast<int>(tid / n), j = static_cast<int>(tid % n);
    const Groups p = a.groups[w];
    const double dx = a.dx, dt = a.dt;
    const size_t o = static_cast<size_t>(w) * n;
    const double *uc = a.in[1] + o, *vc = a.in[3] + o;
    const int wk = a.wall_kind ? a.wall_kind[w] : a.coeff_kind;
    const bool tab = a.star.node != nullptr && wk != kCoeffConstant;
    const bool an = !tab && wk == kCoeffAnalyticD;
    auto NS = [&](int f, int i) -> double {            // StarTables::at_node(i)
        if (tab) return a.star.nd(f, static_cast<int64_t>(o) + i);
        return (an && f == kSk_M) ? analytic_kM(a.p, vc[i]) : 1.0;
    };
    auto HS = [&](int f, int i) -> double {            // StarTables::at_half(i), i+1/2
        if (tab) return a.star.hf(f, static_cast<int64_t>(o) + i);
        return (an && f == kHk_M) ? analytic_kM(a.p, 0.5 * (vc[i] + vc[i + 1])) : 1.0;
    };
    // ghost values from layer-n boundary states (wall.cpp:276-288)
    auto ghosts = [&](int k, double& vg, double& ug) {
        const int jb = k == 0 ? 0 : n - 1, jn = k == 0 ? 1 : n - 2;
        const FaceVals b = resolve(a, w, k);
        const double nkM = NS(kSk_M, jb), nkTM = NS(kSk_TM, jb), nkTT = NS(kSk_TT, jb);
        vg = vc[jn] - (2.0 * dx / nkM) * (b.Bi_M * (vc[jb] - b.v_inf) - b.g_inf);
        ug = uc[jn] + (p.Fo_TM * p.gamma * nkTM) / (p.Fo_TT * nkTT) * (vc[jn] - vg) -
             (2.0 * dx / nkTT) * (b.Bi_TT * (uc[jb] - b.u_inf) + b.Bi_TM * (vc[jb] - b.v_inf) - b.q_inf);
    };
    double vL, vR, uL, uR;
    if (j == 0) ghosts(0, vL, uL); else { vL = vc[j - 1]; uL = uc[j - 1]; }
    if (j == n - 1) ghosts(1, vR, uR); else { vR = vc[j + 1]; uR = uc[j + 1]; }
    const double rdt = dt / (dx * dx);
    // ghost-side half-node coefficients collapse onto the boundary node (wall.cpp:297-303)
    const double km = j == 0 ? NS(kSk_M, 0) : HS(kHk_M, j - 1);
    const double kp = j == n - 1 ? NS(kSk_M, n - 1) : HS(kHk_M, j);
    const double ktm = j == 0 ? NS(kSk_TT, 0) : HS(kHk_TT, j - 1);
    const double ktp = j == n - 1 ? NS(kSk_TT, n - 1) : HS(kHk_TT, j);
    const double kmm = j == 0 ? NS(kSk_TM, 0) : HS(kHk_TM, j - 1);
    const double kmp = j == n - 1 ? NS(kSk_TM, n - 1) : HS(kHk_TM, j);
    const double cM = NS(kSc_M, j), cTM = NS(kSc_TM, j), cTT = NS(kSc_TT, j);
    const double div_v = kp * (vR - vc[j]) - km * (vc[j] - vL);
    const double vn = vc[j] + rdt * p.Fo_M * div_v / cM;
    const double div_u = ktp * (uR - uc[j]) - ktm * (uc[j] - uL);
    const double div_vm = kmp * (vR - vc[j]) - kmm * (vc[j] - vL);
    const double un = uc[j] + (rdt * (p.Fo_TT * div_u + p.Fo_TM * p.gamma * div_vm) -
                               p.gamma * cTM * (vn - vc[j])) / cTT;
    a.out[0][tid] = uc[j];
    a.out[2][tid] = vc[j];
    a.out[1][tid] = un;
    a.out[3][tid] = vn;
    if (tid >= a.own0 && tid < a.own1 && (!(fabs(un) <= a.norm) || !(fabs(vn) <= a.norm))) {
        const unsigned long long key =
            (static_cast<unsigned long long>(a.layer + 1) << 32) | static_cast<unsigned>(w);
        atomicMin(a.fail_key, key);
    }
}

// implicit_wall_pass_unit (wall.cpp:398-429) with the factorisation of
// cached_factors (wall.cpp:360-395) and FactoredTridiag (wall.cpp:322-346):
// one pass of the whole-building fixed point step_implicit
// (building.cpp:189-268) for constant-coefficient walls.  Faces read the zone
// iterate snapshot (a.zu/a.zv) and forcing at t^{n+1}.  One thread per wall;
// scratch is node-major [n][n_walls] (coalesced).  out[1]/out[3] hold the
// wall iterate (initialised to layer n by the host before pass 1); the pass
// overwrites it and accumulates max |new - old| into *diff (non-negative
// doubles order like their bit patterns).  out[0]/out[2] receive layer n.
// The reference folds residuals with std::max(diff, |x|) (building.cpp:232-243),
// which drops NaN; fmax does the same and NaN never reaches the atomic.
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* p, double x) {
    if (!(x >= 0.0)) return;
    atomicMax(p, static_cast<unsigned long long>(__double_as_longlong(x)));
}

__global__ void k_implicit_unit_pass(const StepArgs a, double* scr, unsigned long long* diff) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= a.n_walls) return;
    if (a.wall_kind && a.wall_kind[w] != kCoeffConstant) return;   // k_implicit_table_pass
    const int n = a.n, B = a.n_walls;
    const double dx = a.dx, dt = a.dt;
    const Groups p = a.groups[w];
    const size_t o = static_cast<size_t>(w) * n;
    const double *uc = a.in[1] + o, *vc = a.in[3] + o;
    double* M = scr;
    double* INV = scr + static_cast<size_t>(n) * B;
    double* XV = scr + 2 * static_cast<size_t>(n) * B;
    double* XU = scr + 3 * static_cast<size_t>(n) * B;
    auto at = [&](double* base, int i) -> double& { return base[static_cast<size_t>(i) * B + w]; };
    const FaceVals L = resolve(a, w, 0), R = resolve(a, w, 1);
    const double r = p.Fo_M * dt / (dx * dx);
    const double rb = p.Fo_TT * dt / (dx * dx);
    const double rg = p.Fo_TM * p.gamma * dt / (dx * dx);
    auto lo_ = [&](int i, double rr) { return i == 0 ? 0.0 : (i == n - 1 ? -2.0 * rr : -rr); };
    auto up_ = [&](int i, double rr) { return i == 0 ? -2.0 * rr : (i == n - 1 ? 0.0 : -rr); };
    auto di_ = [&](int i, double rr, double b0, double b1) {
        return i == 0 ? 1.0 + 2.0 * rr + 2.0 * rr * dx * b0
                      : (i == n - 1 ? 1.0 + 2.0 * rr + 2.0 * rr * dx * b1 : 1.0 + 2.0 * rr);
    };
    auto factor = [&](double rr, double b0, double b1) {
        double dp = di_(0, rr, b0, b1);
        at(M, 0) = 0.0;
        at(INV, 0) = 1.0 / dp;
        for (int i = 1; i < n; ++i) {
            const double m = lo_(i, rr) * at(INV, i - 1);
            at(M, i) = m;
            dp = di_(i, rr, b0, b1) - m * up_(i - 1, rr);
            at(INV, i) = 1.0 / dp;
        }
    };
    auto solve = [&](double* X, double rr) {
        for (int i = 1; i < n; ++i) at(X, i) -= at(M, i) * at(X, i - 1);
        at(X, n - 1) *= at(INV, n - 1);
        for (int i = n - 1; i-- > 0;) at(X, i) = (at(X, i) - up_(i, rr) * at(X, i + 1)) * at(INV, i);
    };
    // moisture (wall.cpp:409-413)
    factor(r, L.Bi_M, R.Bi_M);
    for (int i = 0; i < n; ++i) at(XV, i) = vc[i];
    at(XV, 0) += 2.0 * r * dx * (L.Bi_M * L.v_inf + L.g_inf);
    at(XV, n - 1) += 2.0 * r * dx * (R.Bi_M * R.v_inf + R.g_inf);
    solve(XV, r);
    // energy right-hand side with the new moisture layer (wall.cpp:415-427)
    for (int j = 1; j + 1 < n; ++j)
        at(XU, j) = uc[j] - p.gamma * (at(XV, j) - vc[j]) +
                    rg * (at(XV, j + 1) - 2.0 * at(XV, j) + at(XV, j - 1));
    at(XU, 0) = uc[0] - p.gamma * (at(XV, 0) - vc[0]) + 2.0 * rg * (at(XV, 1) - at(XV, 0)) +
                2.0 * rb * dx * (L.Bi_TT * L.u_inf - L.Bi_TM * (at(XV, 0) - L.v_inf) + L.q_inf);
    at(XU, n - 1) = uc[n - 1] - p.gamma * (at(XV, n - 1) - vc[n - 1]) +
                    2.0 * rg * (at(XV, n - 2) - at(XV, n - 1)) +
                    2.0 * rb * dx * (R.Bi_TT * R.u_inf - R.Bi_TM * (at(XV, n - 1) - R.v_inf) + R.q_inf);
    factor(rb, L.Bi_TT, R.Bi_TT);
    solve(XU, rb);
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
    const bool own = static_cast<int64_t>(w) * n >= a.own0 && static_cast<int64_t>(w + 1) * n <= a.own1;
    if (own) atomic_max_nonneg(diff, d);
    if (own && (!(mx <= a.norm) || !finite)) {
        const unsigned long long key =
            (static_cast<unsigned long long>(a.layer + 1) << 32) | static_cast<unsigned>(w);
        atomicMin(a.fail_key, key);
    }
}

// zone_step_implicit (zone.cpp:76-115) inside the building fixed point:
// samples from the current wall iterate, peers from the zone snapshot.
struct ZoneImplicitArgs {
    int n_zones, n;
    double dt;
    const ZoneDev* zones;
    const ZoneLinkDev* links;
    const InzLinkDev* inz;
    const double* src;          // row at t^{n+1}: [n_sources][3] then outdoor u, v
    int n_sources;
    const double* wu;           // wall iterate [n_walls][n]
    const double* wv;
    const double* zu_n;         // zone state at layer n
    const double* zv_n;
    const double* zu_s;         // zone iterate snapshot (peers)
    const double* zv_s;
    double* zu_out;
    double* zv_out;
    int64_t layer;
    double norm;
    unsigned long long* diff;
    unsigned long long* fail_key;
    int own0, own1;             // zones whose residual/guard count
};

__global__ void k_zone_implicit(const ZoneImplicitArgs a) {
    const int z = blockIdx.x * blockDim.x + threadIdx.x;
    if (z >= a.n_zones) return;
    const ZoneDev d = a.zones[z];
    const double* s = a.src + 3 * d.sources;
    const double u_inf = a.src[3 * a.n_sources + 0], v_inf = a.src[3 * a.n_sources + 1];
    double sum_gz = 0.0, sum_gz_v = 0.0;
    for (int i = d.inz_begin; i < d.inz_end; ++i) {
        sum_gz += a.inz[i].g_inz;
        sum_gz_v += a.inz[i].g_inz * a.zv_s[a.inz[i].peer];
    }
    double S_M = 0.0, W_M = 0.0;
    for (int i = d.wall_begin; i < d.wall_end; ++i) {
        const ZoneLinkDev l = a.links[i];
        const size_t idx = static_cast<size_t>(l.wall) * a.n + (l.face == 0 ? 0 : a.n - 1);
        S_M += l.Bi_M * l.theta_M;
        W_M += l.Bi_M * l.theta_M * a.wv[idx];
    }
    const double dt = a.dt;
    const double v_den = 1.0 + dt * (d.g_v + sum_gz - d.sign * S_M);
    const double v_num = a.zv_n[z] + dt * (s[0] + d.g_v * v_inf + sum_gz_v - d.sign * W_M);
    const double v1 = v_num / v_den;
    double u_coef = (1.0 + d.kappa_a_tt1) + dt * (d.q_v1 * v1 + d.q_v2);
    double u_rhs = (1.0 + d.kappa_a_tt1) * a.zu_n[z] +
                   dt * (s[1] + s[2] + d.q_v1 * u_inf * v_inf + d.q_v2 * u_inf);
    for (int i = d.inz_begin; i < d.inz_end; ++i) {
        const InzLinkDev l = a.inz[i];
        const double pu = a.zu_s[l.peer], pv = a.zv_s[l.peer];
        u_coef += dt * (l.q_inz1 * v1 + l.q_inz2);
        u_rhs += dt * (l.q_inz1 * pu * pv + l.q_inz2 * pu);
    }
    for (int i = d.wall_begin; i < d.wall_end; ++i) {
        const ZoneLinkDev l = a.links[i];
        const size_t idx = static_cast<size_t>(l.wall) * a.n + (l.face == 0 ? 0 : a.n - 1);
        u_coef += dt * l.Bi_TT * l.theta_T;
        u_rhs += dt * (l.Bi_TT * l.theta_T * a.wu[idx] + l.Bi_TM * l.theta_T * (a.wv[idx] - v1));
    }
    const double u1 = u_rhs / u_coef;
    const double dd = fmax(fabs(u1 - a.zu_s[z]), fabs(v1 - a.zv_s[z]));   // building.cpp:240-243
    const bool own = z >= a.own0 && z < a.own1;
    if (own) atomic_max_nonneg(a.diff, dd);
    a.zu_out[z] = u1;
    a.zv_out[z] = v1;
    if (own && (!isfinite(u1) || !isfinite(v1) || fabs(u1) > a.norm || fabs(v1) > a.norm)) {
        const unsigned long long key = (static_cast<unsigned long long>(a.layer + 1) << 32) | 0xffffffffu;
        atomicMin(a.fail_key, key);
    }
}

// ---- utilities ---------------------------------------------------------------
__global__ void k_coupled_coef(int n_walls, double dx, double dt, const Groups* g, const Biot* b,
                               WallCoef* c) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w < n_walls) coupled_coef(g[w], dx, dt, b[2 * w], b[2 * w + 1], c[w]);
}

// fp64 state <-> fp32 deviations from the uniform state 1
__global__ void k_to_dev32(int64_t count, const double* in, float* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < count) out[i] = static_cast<float>(in[i] - 1.0);
}
__global__ void k_from_dev32(int64_t count, const float* in, double* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < count) out[i] = 1.0 + static_cast<double>(in[i]);
}

}  // namespace hyg
