// hyg_coef.cuh — per-wall DF coefficients for the constant-coefficient coupled
// step, derived once per (wall, dt) from the reference's update formulas.
//
// Reference: df_step_coupled, /root/reference/proj/src/wall.cpp:144-194.
//   interior v  (wall.cpp:159-160)  vn = ((1-lam) vp + lam (vc[j+1]+vc[j-1])) / (1+lam)
//   boundary v  (wall.cpp:162-169)  closed-form Robin row, cpl = lam dx Bi_M
//   interior u  (wall.cpp:171-176)  uses the new layer vn
//   boundary u  (wall.cpp:177-189)  ghost vg from vbar = (vn + vp)/2
// with lam = 2 Fo_M dt/dx^2, mu = 2 Fo_TT dt/dx^2, beta = 2 Fo_TM gamma dt/dx^2.
//
// Every row is rewritten exactly (in real arithmetic) in increment form
// around the layer n-1 value, with d = sv - 2 vp, du = su - 2 up,
// sv = vL + vR, su = uL + uR:
//   interior:  vn = vp + b d                      un = up + c_su du + c_sv d
//   face:      vn = vp + b d + e (v_inf - vp) [+ e_g g]
//              un = up + c_su du + c_tu (u_inf - up) + c_sv d + c_tv (v_inf - vp)
//                   [+ c_q q + c_g g]
// (at a face the missing neighbour is the mirrored interior one, sv = 2 vc[jn]).
// A uniform state at the ambient values is then a fixed point bit for bit:
// the folded coefficients carry no rounding bias that could pump the slow
// mean mode (a form a vp + b sv with a + 2b != 1 by one ulp drifts ~1e-16 per
// step, 1e-11 after 1e5 steps).  The interior node costs 7 FP64 instructions
// (2 adds, 5 FMA) against 9 plus two divisions in the reference form.
#pragma once

#ifndef HYG_HD
#ifdef __CUDACC__
#define HYG_HD __host__ __device__ __forceinline__
#else
#define HYG_HD inline
#endif
#endif

namespace hyg {
#ifdef __CUDACC__
// The stop flag of a launch sequence (an earlier launch — or another CTA of
// this launch — tripped the guard).  Read once per CTA by thread 0 and decided
// for the whole block through a barrier, so every warp of the CTA agrees
// (a per-thread read could let some warps leave while others wait on a
// barrier: undefined behaviour).
__device__ __forceinline__ bool launch_stopped(const int* stop) {
    return __syncthreads_or(threadIdx.x == 0 ? *const_cast<const volatile int*>(stop) : 0) != 0;
}
#endif

struct Groups { double Fo_M, Fo_TT, Fo_TM, gamma; };
struct Biot { double Bi_M, Bi_TT, Bi_TM; };

// One row in increment form.  Interior rows have e = c_tu = c_tv = e_g = c_q = c_g = 0.
struct RowCoef {
    double b, e, e_g;              // v: d, (v_inf - vp), g_inf
    double c_su, c_tu, c_sv, c_tv;  // u: du, (u_inf - up), d, (v_inf - vp)
    double c_q, c_g;                // u: q_inf, g_inf
};

struct WallCoef {
    RowCoef in;          // interior rows
    RowCoef face[2];     // [0]: node 0 (x*=0), [1]: node n-1 (x*=1)
};

// k_ring_split.cuh stages rows as arrays of doubles in this order
static_assert(sizeof(RowCoef) == 9 * sizeof(double) && sizeof(WallCoef) == 27 * sizeof(double), "row layout");

HYG_HD void coupled_face(const Groups& p, double dx, double lam, double mu, double beta,
                         double ratio, const Biot& f, RowCoef& c) {
    const double g = p.gamma;
    // v row, wall.cpp:165-168:  vn Dv = (1-lam-cpl) vp + 2 lam vc[jn] + 2 lam dx (Bi_M v_inf + g_inf)
    //                                 = Dv vp + lam d + 2 cpl (v_inf - vp) + 2 lam dx g_inf
    const double cpl = lam * dx * f.Bi_M;
    const double dv = 1.0 / (1.0 + lam + cpl);
    c.b = lam * dv;
    c.e = 2.0 * cpl * dv;
    c.e_g = 2.0 * lam * dx * dv;
    // u row, wall.cpp:178-188.  With rho = mu*ratio (= beta when Fo_TT != 0):
    //   mu ratio (vc - vg) + beta (vc + vg) = 2 beta vc - 2 dx (beta - rho) (Bi_M (vbar - v_inf) - g_inf)
    //   vbar - v_inf = (vn - vp)/2 - (v_inf - vp)
    // so  un Du = Du up + mu du + 2 cplu (u_inf - up) + beta d - K' (vn - vp)
    //             + (2 mu dx Bi_TM + 2 dx (beta - rho) Bi_M) (v_inf - vp) + 2 mu dx q_inf + 2 dx (beta - rho) g_inf
    // with K' = gamma + beta + mu dx Bi_TM + dx (beta - rho) Bi_M, and vn - vp from the v row.
    const double rho = mu * ratio;
    const double cplu = mu * dx * f.Bi_TT;
    const double du = 1.0 / (1.0 + mu + cplu);
    const double k = (g + beta + mu * dx * f.Bi_TM + dx * (beta - rho) * f.Bi_M) * du;
    c.c_su = mu * du;
    c.c_tu = 2.0 * cplu * du;
    c.c_sv = beta * du - k * c.b;
    c.c_tv = (2.0 * mu * dx * f.Bi_TM + 2.0 * dx * (beta - rho) * f.Bi_M) * du - k * c.e;
    c.c_q = 2.0 * mu * dx * du;
    c.c_g = 2.0 * dx * (beta - rho) * du - k * c.e_g;
}

HYG_HD void coupled_coef(const Groups& p, double dx, double dt, const Biot& left,
                         const Biot& right, WallCoef& w) {
    const double r = dt / (dx * dx);
    const double lam = 2.0 * p.Fo_M * r;               // wall.cpp:148
    const double mu = 2.0 * p.Fo_TT * r;               // wall.cpp:149
    const double beta = 2.0 * p.Fo_TM * p.gamma * r;   // wall.cpp:150
    const double ratio = p.Fo_TT != 0.0 ? p.Fo_TM * p.gamma / p.Fo_TT : 0.0;  // wall.cpp:151
    const double g = p.gamma;
    // interior, wall.cpp:160,172-175:
    //   vn (1+lam) = (1+lam) vp + lam d
    //   un (1+mu)  = (1+mu) up + mu du + beta d - (gamma+beta)(vn - vp),  vn - vp = b d
    w.in.b = lam / (1.0 + lam);
    w.in.c_su = mu / (1.0 + mu);
    w.in.c_sv = (beta - (g + beta) * w.in.b) / (1.0 + mu);
    w.in.e = w.in.e_g = w.in.c_tu = w.in.c_tv = w.in.c_q = w.in.c_g = 0.0;
    coupled_face(p, dx, lam, mu, beta, ratio, left, w.face[0]);
    coupled_face(p, dx, lam, mu, beta, ratio, right, w.face[1]);
}

}  // namespace hyg
