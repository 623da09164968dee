// k_nonlinear.cuh — K2: nonlinear DF march for walls with the analytic
// coefficient functor k_M* = d(v) (HYG_COEFF_ANALYTIC_D), one CTA per wall,
// the four layers in shared memory, all steps of a segment in one launch.
//
// Replaces: df_step_nonlinear (/root/reference/proj/src/wall.cpp:196-264) with
// StarTables (wall.cpp:89-138) for the d(v) functor, called per step from
// run()/step_explicit; guard as check_bounded (building.cpp:282-300).
//
// configs[0] is one wall of 101 nodes marched 1e5 steps: the work per step is
// ~100 node-updates, so the step is latency-bound (one dependency chain:
// neighbours -> half-node d(v) (exp) -> reciprocal -> v -> u).  One CTA per
// wall with a thread per node keeps one node's chain + one barrier per step;
// batches of such walls run one CTA each.
//
// Rows are the reference's, rewritten in increment form around the layer
// n-1 value (exact in real arithmetic; a uniform state at ambient values is
// a fixed point bit for bit, cf. hyg_coef.cuh):
//   v (wall.cpp:213-217):  vn = vp + 2a (kp (vR - vp) + km (vL - vp)) / (c_M + a (kp + km))
//   u (wall.cpp:231-240):  with k_TT = k_TM = c_TT = c_TM = 1,
//       un = up + (2b (uR + uL - 2 up) + 2g (vR + vL - vn - vp) - gamma (vn - vp)) / (1 + 2b)
//   face rows (wall.cpp:218-229, 241-259) likewise, with the ghost-side
//   coefficient k_M at the boundary node and vg from vbar = (vn + vp)/2.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "hyg_coef.cuh"
#include "hyg_fastmath.cuh"
#include "k_coupled.cuh"

namespace hyg {

struct NonlinearSegArgs {
    int n_walls, n, nsteps, n_channels;
    int64_t layer0;
    int seg_index;
    double dx, dt;
    double p[4];                 // d(v) = 1 + p0 v + p1 exp(-p2 (v - p3)^2)
    const Groups* groups;
    const Biot* biot;            // [2*w + face]
    const int* chan;             // [2*w + face]
    const Ambient* table;        // [nsteps][n_channels]
    const double* in[4];
    double* out[4];
    const int* stop;
    int* suspect;
};

__device__ __forceinline__ double d_of(const double* p, double v, const double* tab) {
    const double e = v - p[3];
    return 1.0 + p[0] * v + p[1] * fexp(-p[2] * e * e, tab);
}

// Stage the 2^(j/64) table of fexp into shared memory (call before a barrier).
__device__ __forceinline__ void stage_exp_table(double* s_tab, int tid, int nthreads) {
    for (int i = tid; i < 64; i += nthreads) s_tab[i] = kExp2Tab64[i];
}

// fexp_addend's table (exp_tab_biased) in shared memory, kExpRep copies (entry j of copy c
// at j * kExpRep + c, lane l reading copy l & (kExpRep - 1)).  One copy: neighbouring
// lanes hold neighbouring states and mostly read the same or adjacent entries, so bank
// replication buys nothing (16 copies of the round-1 table were within 1 % of one on K3w),
// while a single copy lets the compiler address the table as an immediate offset from the
// masked index — an LEA and a mask fewer per exp (4 copies: cfg4 3.53e11, one: 3.55e11;
// cfg0 4.16e8 -> 4.21e8)
constexpr int kExpRep = 1;
constexpr int kExpTab = 256;
__device__ __forceinline__ void stage_exp_table_rep(double* s_tab, int tid, int nthreads) {
    for (int i = tid; i < kExpTab * kExpRep; i += nthreads) s_tab[i] = exp_tab_biased(i / kExpRep);
}

constexpr int kNlChunk = 64;   // forcing rows staged per chunk

// Per-wall scalars of the d(v) rows (wall.cpp:199-204).
struct AnalyticRow { double a, b, g, gamma, ratio, dx, inv_u; };

__device__ __forceinline__ AnalyticRow analytic_row(const Groups& g, double dx, double dt) {
    AnalyticRow r;
    r.a = g.Fo_M * dt / (dx * dx);
    r.b = g.Fo_TT * dt / (dx * dx);
    r.g = g.Fo_TM * g.gamma * dt / (dx * dx);
    r.gamma = g.gamma;
    r.ratio = g.Fo_TT != 0.0 ? g.Fo_TM * g.gamma / g.Fo_TT : 0.0;
    r.dx = dx;
    r.inv_u = 1.0 / (1.0 + 2.0 * r.b);
    return r;
}

// Interior node (wall.cpp:213-217, 231-240) with half-node coefficients km, kp.
__device__ __forceinline__ void analytic_interior(const AnalyticRow& r, double vp, double up, double vL,
                                                  double vR, double uL, double uR, double km, double kp,
                                                  double& vn, double& un) {
    vn = vp + 2.0 * r.a * (kp * (vR - vp) + km * (vL - vp)) * frcp(1.0 + r.a * (kp + km));
    un = up + (2.0 * r.b * (uR + uL - 2.0 * up) + 2.0 * r.g * (vR + vL - vn - vp) - r.gamma * (vn - vp)) *
                  r.inv_u;
}

// Face node (wall.cpp:218-229, 241-259): jn = interior neighbour, km_b = node
// value d(v_face) (ghost side), kp_b = half-node value next to the face.
__device__ __forceinline__ void analytic_face(const AnalyticRow& r, const Biot& fb, const Ambient& am,
                                              double vp, double up, double vcn, double ucn, double km_b,
                                              double kp_b, double& vn, double& un) {
    const double S = kp_b + km_b;
    const double cpl = 2.0 * r.a * r.dx * fb.Bi_M;
    vn = vp + (2.0 * r.a * S * (vcn - vp) + 2.0 * cpl * (am.v - vp) + 4.0 * r.a * r.dx * am.g) *
                  frcp(1.0 + r.a * S + cpl);
    const double vbar = 0.5 * (vn + vp);
    const double vg = vcn - (2.0 * r.dx * frcp(km_b)) * (fb.Bi_M * (vbar - am.v) - am.g);
    const double cplu = 2.0 * r.b * r.dx * fb.Bi_TT;
    un = up + (4.0 * r.b * (ucn - up) + 2.0 * cplu * (am.u - up) - r.gamma * (vn - vp) +
               2.0 * r.b * r.ratio * (vcn - vg) - 4.0 * r.b * r.dx * (fb.Bi_TM * (vbar - am.v) - am.q) +
               2.0 * r.g * (vcn + vg) - 2.0 * r.g * (vn + vp)) *
                  frcp(1.0 + 2.0 * r.b + cplu);
}

// One CTA per wall: IT threads stride over the interior nodes 1..n-2 and one
// extra warp takes the two face nodes (lanes 0 and 1), so no warp mixes the
// interior and face rows.  For configs[0] (n = 101) IT = 128: one interior
// node per thread; a step costs one node's chain plus a block barrier.
template <int MAXN, int IT>
__global__ void __launch_bounds__(IT + 32) k_df_analytic_walls(const NonlinearSegArgs A) {
    constexpr int THREADS = IT + 32;
    __shared__ double s_lay[4][MAXN];            // up, uc, vp, vc (roles rotate)
    __shared__ Ambient s_amb[kNlChunk][2];       // [step][face]
    __shared__ double s_tab[64];
    if (launch_stopped(A.stop)) return;
    const int w = blockIdx.x, tid = threadIdx.x, n = A.n;
    const size_t o = static_cast<size_t>(w) * n;
    stage_exp_table(s_tab, tid, THREADS);
    for (int j = tid; j < n; j += THREADS) {
        s_lay[0][j] = A.in[0][o + j];
        s_lay[1][j] = A.in[1][o + j];
        s_lay[2][j] = A.in[2][o + j];
        s_lay[3][j] = A.in[3][o + j];
    }
    const Groups g = A.groups[w];
    const double dx = A.dx, dt = A.dt;
    const AnalyticRow rc = analytic_row(g, dx, dt);
    const bool face_warp = tid >= IT;
    const int flane = tid - IT;                  // 0: x*=0 face, 1: x*=1 face
    const Biot fb = A.biot[2 * w + (flane == 1 ? 1 : 0)];
    const int chl = A.chan[2 * w], chr = A.chan[2 * w + 1];
    double p[4] = {A.p[0], A.p[1], A.p[2], A.p[3]};
    unsigned acc = 0;
    int P = 0;    // roles: u_prev = s_lay[P], u_curr = s_lay[1-P], v_prev = s_lay[2+P], v_curr = s_lay[3-P]

    for (int c0 = 0; c0 < A.nsteps; c0 += kNlChunk) {
        const int clen = min(kNlChunk, A.nsteps - c0);
        __syncthreads();
        for (int i = tid; i < 2 * clen; i += THREADS) {
            const int s = i >> 1, f = i & 1;
            s_amb[s][f] = A.table[static_cast<size_t>(c0 + s) * A.n_channels + (f ? chr : chl)];
        }
        __syncthreads();
        // one step with compile-time layer roles (PP): the 2-step unroll keeps
        // every shared address a constant offset (no per-step address math)
        auto step = [&](int s, auto PPc) {
            constexpr int PP = decltype(PPc)::value;
            double* up = s_lay[PP];
            const double* uc = s_lay[1 - PP];
            double* vp = s_lay[2 + PP];
            const double* vc = s_lay[3 - PP];
            if (!face_warp) {
                for (int j = 1 + tid; j < n - 1; j += IT) {
                    const double vpj = vp[j], upj = up[j], vcj = vc[j];
                    const double vL = vc[j - 1], vR = vc[j + 1];
                    double vn, un;
                    analytic_interior(rc, vpj, upj, vL, vR, uc[j - 1], uc[j + 1],
                                      d_of(p, 0.5 * (vL + vcj), s_tab), d_of(p, 0.5 * (vcj + vR), s_tab), vn, un);
                    acc |= static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn));
                    vp[j] = vn;     // layer n-1 slot becomes layer n+1
                    up[j] = un;
                }
            } else if (flane < 2) {
                const bool left = flane == 0;
                const int j = left ? 0 : n - 1;
                const int jn = left ? 1 : n - 2;
                const double vcj = vc[j], vcn = vc[jn];
                double vn, un;
                analytic_face(rc, fb, s_amb[s][flane], vp[j], up[j], vcn, uc[jn], d_of(p, vcj, s_tab),
                              d_of(p, 0.5 * (vcj + vcn), s_tab), vn, un);
                acc |= static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn));
                vp[j] = vn;
                up[j] = un;
            }
            __syncthreads();
        };
        int s = 0;
        if (P == 0) {
            for (; s + 1 < clen; s += 2) {
                step(s, std::integral_constant<int, 0>{});
                step(s + 1, std::integral_constant<int, 1>{});
            }
            if (s < clen) { step(s, std::integral_constant<int, 0>{}); P = 1; }
        } else {
            for (; s + 1 < clen; s += 2) {
                step(s, std::integral_constant<int, 1>{});
                step(s + 1, std::integral_constant<int, 0>{});
            }
            if (s < clen) { step(s, std::integral_constant<int, 1>{}); P = 0; }
        }
    }
    // fast guard verdict (bit 30 of the high word: |x| >= 2 or not finite)
    const unsigned any = __reduce_or_sync(0xffffffffu, acc);
    if ((any & 0x40000000u) && (tid % 32) == 0) atomicCAS(A.suspect, 0, A.seg_index + 1);
    const double* up = s_lay[P];
    const double* uc = s_lay[1 - P];
    const double* vp = s_lay[2 + P];
    const double* vc = s_lay[3 - P];
    for (int j = tid; j < n; j += THREADS) {
        A.out[0][o + j] = up[j];
        A.out[1][o + j] = uc[j];
        A.out[2][o + j] = vp[j];
        A.out[3][o + j] = vc[j];
    }
}

}  // namespace hyg
