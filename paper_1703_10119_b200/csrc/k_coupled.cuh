// k_coupled.cuh — K1: batched constant-coefficient coupled Dufort–Frankel
// march, many steps fused per launch, whole wall profile in registers.
//
// Replaces: df_step_coupled (/root/reference/proj/src/wall.cpp:144-194) called
// per wall per step from step_explicit (building.cpp:166-177) inside run()
// (building.cpp:325-337), plus the divergence guard check_bounded
// (building.cpp:282-300) / max_abs_field (wall.cpp:579-587).
//
// Mapping: one wall = LPW consecutive lanes (a "wall group" inside a warp),
// NPT consecutive nodes per lane held in registers (N = LPW*NPT).  Four
// layers (u_prev,u_curr,v_prev,v_curr) live in registers for the whole
// segment; neighbour values across lanes come from __shfl; the layer rotation
// of wall.cpp:80-83 is a register renaming (the step is unrolled by two).
// The last lane of a group stores its nodes in REVERSED order, so that both
// face nodes (node 0 in lane 0, node N-1 in lane LPW-1) sit in register 0:
// only register 0 runs the (more expensive) face-capable row, with per-lane
// coefficients that are the interior ones everywhere else.
// Rows use the increment form of hyg_coef.cuh (7 FP64 instructions per
// interior node-update, 12 for register 0).
//
// Forcing is a per-layer ambient table staged through shared memory in chunks.
//
// Divergence guard: the reference checks |field| <= divergence_norm and
// finiteness after every step.  Here every new value's high word is OR-ed
// into a per-lane accumulator (one LOP3 per node-update, ALU pipe).  Bit 30
// of an IEEE double's high word is set iff |x| >= 2 or x is not finite
// (for fp32 deviations w = x - 1: |w| >= 2), so a clear bit proves every
// value of the segment passed any norm >= 2 (>= 3 for fp32 deviations).  A
// set bit makes the host re-run the segment with EXACT=true, which performs
// the reference's comparison per step and records the first failing layer.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hyg_coef.cuh"

namespace hyg {

struct Ambient { double u, v, g, q; };

template <typename Real>
struct CoupledSegArgs {
    int n_walls;
    int n_channels;
    int nsteps;
    int64_t layer0;              // absolute index of layer "curr" at segment start
    int seg_index;               // position of this launch in its batch (fast-guard flag)
    double divergence_norm;      // exact mode only
    const WallCoef* coef;        // [n_walls], derived for this segment's dt
    const int* chan;             // [n_walls*2] exterior channel per face
    const Ambient* table;        // [nsteps][n_channels], row s = layer layer0+s
    const Real* in[4];           // up, uc, vp, vc   [n_walls][N]
    Real* out[4];
    const int* stop;             // non-zero: skip (an earlier segment flagged)
    int* suspect;                // fast guard fired: seg_index + 1 of the first such launch
    unsigned long long* fail_key;  // exact mode: min((layer<<32) | wall)
};

template <typename Real> struct HiWord;
template <> struct HiWord<double> {
    static __device__ __forceinline__ unsigned get(double x) {
        return static_cast<unsigned>(__double2hiint(x));
    }
};
template <> struct HiWord<float> {
    static __device__ __forceinline__ unsigned get(float x) { return __float_as_uint(x); }
};

template <typename Real> struct InRow { Real b, c_su, c_sv; };
template <typename Real> struct FaceRow { Real b, e, c_su, c_tu, c_sv, c_tv; };

// Per-step scalars of register 0 (ambient of this lane's face).
template <typename Real> struct StepAmb { Real u_inf, v_inf, ev, eu; };

// One fused DF step for this lane's NPT nodes.  P holds layer n-1 on entry
// and layer n+1 on exit; C holds layer n.
template <typename Real, int LPW, int NPT, bool FLUX, bool EXACT, bool EDGE_FIRST = false>
__device__ __forceinline__ void coupled_step(Real (&vP)[NPT], Real (&vC)[NPT], Real (&uP)[NPT],
                                             Real (&uC)[NPT], const InRow<Real>& ci,
                                             const FaceRow<Real>& c0, const StepAmb<Real>& am,
                                             bool mirror0, bool rev, unsigned& acc, bool& bad,
                                             Real norm) {
    constexpr unsigned FULL = 0xffffffffu;
    // neighbour exchange inside the wall group (see header: last lane reversed)
    const Real vs = rev ? vC[NPT - 1] : vC[0];
    const Real us = rev ? uC[NPT - 1] : uC[0];
    const Real vup = __shfl_up_sync(FULL, vC[NPT - 1], 1, LPW);
    const Real uup = __shfl_up_sync(FULL, uC[NPT - 1], 1, LPW);
    const Real vdn = __shfl_down_sync(FULL, vs, 1, LPW);
    const Real udn = __shfl_down_sync(FULL, us, 1, LPW);
    // outer neighbour of register 0: mirrored node 1 at a face (wall.cpp:162-169)
    const Real vx0 = mirror0 ? vC[1] : vup;
    const Real ux0 = mirror0 ? uC[1] : uup;
    const Real vx1 = rev ? vup : vdn;
    const Real ux1 = rev ? uup : udn;
#pragma unroll
    for (int jj = 0; jj < NPT; ++jj) {
        // EDGE_FIRST: registers 0 and NPT-1 (the ones the next step shuffles) first
        const int j = !EDGE_FIRST ? jj : (jj == 0 ? 0 : (jj == 1 ? NPT - 1 : jj - 1));
        const Real sv = (j == 0 ? vx0 : vC[j - 1]) + (j == NPT - 1 ? vx1 : vC[j + 1]);
        const Real su = (j == 0 ? ux0 : uC[j - 1]) + (j == NPT - 1 ? ux1 : uC[j + 1]);
        const Real d = fma(Real(-2), vP[j], sv);
        const Real du = fma(Real(-2), uP[j], su);
        Real vn, un;
        if (j == 0) {
            const Real t = am.v_inf - vP[j];
            const Real tu = am.u_inf - uP[j];
            vn = fma(c0.e, t, fma(c0.b, d, FLUX ? vP[j] + am.ev : vP[j]));
            un = fma(c0.c_tv, t, fma(c0.c_sv, d, fma(c0.c_tu, tu, fma(c0.c_su, du, FLUX ? uP[j] + am.eu : uP[j]))));
        } else {
            vn = fma(ci.b, d, vP[j]);
            un = fma(ci.c_sv, d, fma(ci.c_su, du, uP[j]));
        }
        if (EXACT) {
            // max_abs_field semantics: fail on |x| > norm or non-finite
            constexpr Real OFF = sizeof(Real) == 4 ? Real(1) : Real(0);   // fp32 holds x - 1
            bad |= !(fabs(un + OFF) <= norm) || !(fabs(vn + OFF) <= norm);
        } else {
            acc |= HiWord<Real>::get(un) | HiWord<Real>::get(vn);
        }
        vP[j] = vn;
        uP[j] = un;
    }
}

// MINB > 0 caps registers (launch_bounds min blocks per SM) for occupancy experiments.
template <typename Real, int LPW, int NPT, int WARPS, int CHUNK, bool FLUX, bool EXACT, int MINB = 0,
          int UNROLL = 2, bool EDGE_FIRST = false>
__global__ void __launch_bounds__(WARPS * 32, MINB)
k_df_coupled(const CoupledSegArgs<Real> a) {
    constexpr bool DEV = sizeof(Real) == 4;   // fp32 state = deviations from 1
    constexpr int WALLS_PER_CTA = WARPS * 32 / LPW;
    constexpr int N = LPW * NPT;
    extern __shared__ Ambient s_tab[];   // [CHUNK][n_channels]

    if (launch_stopped(a.stop)) return;
    const int tid = threadIdx.x;
    const int sub = tid % LPW;
    const int wall = blockIdx.x * WALLS_PER_CTA + tid / LPW;
    const bool active = wall < a.n_walls;
    const int w = active ? wall : a.n_walls - 1;
    const bool first = sub == 0, rev = sub == LPW - 1;
    const bool mirror0 = first || rev;

    const WallCoef& wc = a.coef[w];
    const InRow<Real> ci{Real(wc.in.b), Real(wc.in.c_su), Real(wc.in.c_sv)};
    FaceRow<Real> c0{ci.b, Real(0), ci.c_su, Real(0), ci.c_sv, Real(0)};
    double e_g = 0.0, c_q = 0.0, c_g = 0.0;
    int ch = a.chan[2 * w + 0];
    if (mirror0) {
        const RowCoef& f = wc.face[first ? 0 : 1];
        c0 = FaceRow<Real>{Real(f.b), Real(f.e), Real(f.c_su), Real(f.c_tu), Real(f.c_sv), Real(f.c_tv)};
        e_g = f.e_g;
        c_q = f.c_q;
        c_g = f.c_g;
        ch = a.chan[2 * w + (first ? 0 : 1)];
    }

    Real up[NPT], uc[NPT], vp[NPT], vc[NPT];
    const size_t base = static_cast<size_t>(w) * N + sub * NPT;
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        const size_t i = base + (rev ? NPT - 1 - j : j);
        up[j] = a.in[0][i];
        uc[j] = a.in[1][i];
        vp[j] = a.in[2][i];
        vc[j] = a.in[3][i];
    }

    unsigned acc = 0;
    bool bad = false;
    const Real norm = Real(a.divergence_norm);
    const int nch = a.n_channels;
    const unsigned gmask = (LPW == 32 ? 0xffffffffu : ((1u << LPW) - 1u)) << (tid % 32 / LPW * LPW);
    auto group_bad = [&](bool b) { return (__ballot_sync(0xffffffffu, b) & gmask) != 0u; };
    auto amb = [&](int s) {
        const Ambient x = s_tab[s * nch + ch];
        StepAmb<Real> r;
        r.u_inf = Real(DEV ? x.u - 1.0 : x.u);
        r.v_inf = Real(DEV ? x.v - 1.0 : x.v);
        if (FLUX) {   // fp64 flux terms, rounded once into the row
            r.ev = Real(e_g * x.g);
            r.eu = Real(fma(c_q, x.q, c_g * x.g));
        } else {
            r.ev = r.eu = Real(0);
        }
        return r;
    };
    auto swap_layers = [&]() {
#pragma unroll
        for (int j = 0; j < NPT; ++j) {
            Real t = vp[j]; vp[j] = vc[j]; vc[j] = t;
            t = up[j]; up[j] = uc[j]; uc[j] = t;
        }
    };
    int failed_at = -1;      // exact mode: steps completed when the guard failed
    // Exact mode: a wall group that fails stores the failing layer pair at once
    // and is then frozen, but keeps stepping in lockstep — the other wall group
    // of the warp still needs its lanes in every full-mask shuffle and ballot.
    auto store = [&](const Real (&u0)[NPT], const Real (&u1)[NPT], const Real (&v0)[NPT],
                     const Real (&v1)[NPT]) {
        if (!active) return;
#pragma unroll
        for (int j = 0; j < NPT; ++j) {
            const size_t i = base + (rev ? NPT - 1 - j : j);
            a.out[0][i] = u0[j];
            a.out[1][i] = u1[j];
            a.out[2][i] = v0[j];
            a.out[3][i] = v1[j];
        }
    };

    for (int c0s = 0; c0s < a.nsteps; c0s += CHUNK) {
        const int clen = min(CHUNK, a.nsteps - c0s);
        __syncthreads();
        for (int i = tid; i < clen * nch; i += WARPS * 32) s_tab[i] = a.table[(size_t)c0s * nch + i];
        __syncthreads();
        int s = 0;
        // an even number of steps per iteration: the layer rotation is a
        // register renaming (UNROLL > 2 shortens the per-iteration drain)
        auto pair = [&](int s2) {
            coupled_step<Real, LPW, NPT, FLUX, EXACT, EDGE_FIRST>(vp, vc, up, uc, ci, c0, amb(s2), mirror0, rev,
                                                                  acc, bad, norm);
            if (EXACT && group_bad(bad) && failed_at < 0) {   // ballot first: every lane votes
                failed_at = c0s + s2 + 1;
                store(uc, up, vc, vp);   // after this step curr lives in the P registers
            }
            coupled_step<Real, LPW, NPT, FLUX, EXACT, EDGE_FIRST>(vc, vp, uc, up, ci, c0, amb(s2 + 1), mirror0,
                                                                  rev, acc, bad, norm);
            if (EXACT && group_bad(bad) && failed_at < 0) {
                failed_at = c0s + s2 + 2;
                store(up, uc, vp, vc);
            }
        };
        for (; s + UNROLL - 1 < clen; s += UNROLL) {
#pragma unroll
            for (int q = 0; q < UNROLL; q += 2) pair(s + q);
        }
        for (; s + 1 < clen; s += 2) pair(s);
        if (s < clen) {   // odd tail (last chunk only)
            coupled_step<Real, LPW, NPT, FLUX, EXACT>(vp, vc, up, uc, ci, c0, amb(s), mirror0, rev, acc,
                                                      bad, norm);
            swap_layers();
            if (EXACT && group_bad(bad) && failed_at < 0) {   // ballot first: every lane votes
                failed_at = c0s + s + 1;
                store(up, uc, vp, vc);
            }
        }
    }
    if (EXACT && failed_at >= 0 && active && first) {
        const unsigned long long key =
            (static_cast<unsigned long long>(a.layer0 + failed_at) << 32) |
            static_cast<unsigned>(wall);
        atomicMin(a.fail_key, key);
    }
    if (!EXACT) {
        // fast guard verdict for the segment (bit 30: |x| >= 2 or non-finite)
        const unsigned any = __reduce_or_sync(0xffffffffu, active ? acc : 0u);
        if ((any & 0x40000000u) && (tid % 32) == 0) atomicCAS(a.suspect, 0, a.seg_index + 1);
    }
    if (failed_at < 0) store(up, uc, vp, vc);
}

}  // namespace hyg
