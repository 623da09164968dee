// k_dv_warp.cuh — register-resident nonlinear DF marches for the analytic
// d(v) functor (HYG_COEFF_ANALYTIC_D): a warp owns a whole wall (configs[0]
// and batches of short walls, K2w) or a window of one long wall that it
// advances NPT steps per launch (configs[4], K3w).
//
// Replaces: df_step_nonlinear (/root/reference/proj/src/wall.cpp:196-264) with
// StarTables (wall.cpp:89-138) for the d(v) functor, called per step from
// run()/step_explicit (building.cpp:166-177, 325-337); guard as check_bounded
// (building.cpp:282-300).
//
// Layout (as K1, k_coupled.cuh): lane l holds NPT consecutive nodes of the
// four layers in registers; neighbours across lanes come from shuffles, so a
// step needs no shared memory and no barrier.  The last live lane holds its
// M nodes in REVERSED order, so both faces sit in register 0 (lane 0 and the
// last lane) and only register 0 carries the face row.  In register order a
// node's successor is register j+1, or for the last register the next lane's
// first node (shuffle down) — for the reversed lane the previous lane's last
// node (shuffle up).  The rows are symmetric in their two neighbours, so the
// reversed lane runs the same code.
//
// Per step and lane: the half-node coefficients h_j = d((v_j + v_succ(j))/2)
// once each (h of the previous lane's last half node by one shuffle), then the
// rows of wall.cpp:213-217 / 231-240 in increment form around layer n-1 (a
// uniform state at ambient values is a fixed point bit for bit):
//   v:  vn = vp + 2a (kp (vR - vp) + km (vL - vp)) / (1 + a (kp + km))
//   u:  un = up + B (uL + uR - 2 up) + G (vL + vR - (vn + vp)) - Gm (vn - vp)
//       with B = 2b/(1+2b), G = 2g/(1+2b), Gm = gamma/(1+2b), evaluated as
//       up + B (uL + uR - 2 up) + G ((vL - vp) + (vR - vp)) - (G + Gm) inc
//       where inc is the v row's increment (vn = vp + inc)
// and the face rows of wall.cpp:218-229, 241-259 (analytic_face) in register
// 0 of the face lanes, with the ghost-side coefficient d(v_face) (node value).
// Cost: 33 FP64 instructions per interior node-update (15 of them the half
// node: fexp is 10 + the clamp; frcp 3 FMAs), against ~55 in the shared-memory kernels.
//
// K3w temporal blocking: a window of W = 32 NPT nodes, S = NPT steps per
// launch.  An artificial window edge (not a real face) contaminates one node
// per step, so after S steps exactly lane 0 and lane 31 are stale: a middle
// window owns lanes 1..30 (T = 30 NPT nodes).  The first window starts at the
// left face (owns lanes 0..30), the last ends at the right face.  Traffic per
// launch: 32 W + 32 T bytes for T S updates (8.3 B/update at NPT = 8; NPT = 12
// or 16 would halve it but exceed 255 registers).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "k_nonlinear.cuh"

namespace hyg {

// One launch of the long-wall march (K3w): A.steps <= NPT steps over all nodes.
struct TiledArgs {
    int64_t n;                 // nodes of the wall
    int steps;                 // <= NPT
    int n_channels, chl, chr;
    int seg_index;
    double dx, dt;
    double p[4];
    Groups groups;
    Biot bl, br;
    const Ambient* table;      // [steps][n_channels] rows of this launch
    const double* in[4];
    double* out[4];
    const int* stop;
    int* suspect;
    int64_t t_begin, t_end;    // interior windows of this launch: [t_begin, t_end) within [1, rface(n))
};

// d(v) = 1 + p0 v + p1 exp(-p2 (v - p3)^2) at a half node, from the SUM of its
// two node values (midpoint = sum/2 is exact; e and p0 v round as the
// reference's midpoint form).  For a node value pass 2 v.
// The exponent -p2 (m - p3)^2 is -(e e) with e = sqrt(p2) (m - p3) from one
// FMA (p2 >= 0 on this path, hyg_create), one DMUL fewer than (-p2 e) e.
// Every coefficient is returned SCALED by a2 = 2 Fo_M dt/dx^2 (the rows use
// 2a k only): hp0 = a2 p0/2, p1 = a2 p1, one = a2 — the same two FMAs.
struct DvParams { double hp0, hsq, nsqp3, p1, np2, p3, one; };

__device__ __forceinline__ DvParams dv_params(const double* p, double a2) {
    const double sq = sqrt(p[2]);
    return DvParams{a2 * (0.5 * p[0]), 0.5 * sq, -p[3] * sq, a2 * p[1], -p[2], p[3], a2};
}

__device__ __forceinline__ double d_half(const DvParams& q, double sum, const double* tab) {
    const double e = fma(q.hsq, sum, q.nsqp3);
    const double E = fexp_addend<kExpRep>(-(e * e), tab);
    return fma(q.p1, E, fma(q.hp0, sum, q.one));
}

// The same with the exponent as (-p2 e) e, e = m - p3: one DMUL more, but
// measured 5 % faster in the latency-bound single-wall march (K2s), where
// the compiler's schedule of the three exps per lane differs.
__device__ __forceinline__ double d_half_lat(const DvParams& q, double sum, const double* tab) {
    const double e = fma(0.5, sum, -q.p3);
    const double E = fexp_addend<kExpRep>((q.np2 * e) * e, tab);
    return fma(q.p1, E, fma(q.hp0, sum, q.one));
}

// Interior-row constants of one wall (wall.cpp:199-204).
struct DvRow { double a, a2, B, G, Gp; };

__device__ __forceinline__ DvRow dv_row(const AnalyticRow& r) {
    return DvRow{r.a, 2.0 * r.a, 2.0 * r.b * r.inv_u, 2.0 * r.g * r.inv_u, (2.0 * r.g + r.gamma) * r.inv_u};
}

__device__ __forceinline__ void dv_interior(const DvRow& r, double vp, double up, double vL, double vR,
                                            double uL, double uR, double km, double kp, double& vn,
                                            double& un, bool rev = false) {
    // Every node rounds the same whatever lane holds it, so every window of K3w
    // (and the sharded run) computes it bit for bit alike.  The sums dl + dr and
    // kp + km commute; the numerator k_left d_left + k_right d_right is ONE
    // product and one FMA in the geometric order — the right-hand product rounded
    // first, the left-hand one inside the FMA — so a lane whose registers hold
    // its nodes reversed (rev: its "L" arguments are the geometric right) swaps
    // the operands by selects; where rev is a compile-time false (K3w's interior
    // windows, the one-node-per-lane kernels) they fold away.  The u row reuses
    // the v row's differences and its increment inc ~ vn - vp: (vL + vR) - (vn + vp)
    // = dl + dr - inc, so G w - Gm (vn - vp) = G (dl + dr) - (G + Gm) inc (every
    // term vanishes exactly at a uniform state)
    // km, kp arrive scaled by 2a (dv_params): num = 2a (km dl + kp dr) and
    // 1 + a (kp + km) = 1 + (kp' + km')/2
    const double dl = vL - vp, dr = vR - vp;
    const double ka = rev ? kp : km, da = rev ? dr : dl, kb = rev ? km : kp, db = rev ? dl : dr;
    const double num = fma(ka, da, __dmul_rn(kb, db));
    const double den = fma(0.5, kp + km, 1.0);
    const double inc = __dmul_rn(num, frcp2(den));
    vn = __dadd_rn(vp, inc);
    const double du = fma(-2.0, up, uL + uR);
    un = fma(-r.Gp, inc, fma(r.G, dl + dr, fma(r.B, du, up)));
}

// Face row (wall.cpp:218-229, 241-259; analytic_face) with the per-lane
// constants folded once: the u row's denominator is a per-wall constant.
struct DvFace { double a, a2, cpl1, cpl2, ag4, dx2, BiM, b4, cplu2, gamma, b2r, b4dx, BiTM, g2, inv_fu, dx2a; };

__device__ __forceinline__ DvFace dv_face_consts(const AnalyticRow& r, const Biot& fb) {
    DvFace f;
    const double cpl = 2.0 * r.a * r.dx * fb.Bi_M;
    const double cplu = 2.0 * r.b * r.dx * fb.Bi_TT;
    f.a = r.a;
    f.a2 = 2.0 * r.a;
    f.cpl1 = 1.0 + cpl;
    f.cpl2 = 2.0 * cpl;
    f.ag4 = 4.0 * r.a * r.dx;
    f.dx2 = 2.0 * r.dx;
    f.BiM = fb.Bi_M;
    f.b4 = 4.0 * r.b;
    f.cplu2 = 2.0 * cplu;
    f.gamma = r.gamma;
    f.b2r = 2.0 * r.b * r.ratio;
    f.b4dx = 4.0 * r.b * r.dx;
    f.BiTM = fb.Bi_TM;
    f.g2 = 2.0 * r.g;
    f.inv_fu = 1.0 / (1.0 + 2.0 * r.b + cplu);
    f.dx2a = 2.0 * r.dx * (2.0 * r.a);   // 2 dx / k = 2 dx 2a / k' for a scaled k'
    return f;
}

// vcn, ucn: the interior neighbour; km_b = d(v_face) (ghost side), kp_b = the
// half node next to the face.
__device__ __forceinline__ void dv_face(const DvFace& f, const Ambient& am, double vp, double up, double vcn,
                                        double ucn, double km_b, double kp_b, double& vn, double& un) {
    // km_b, kp_b scaled by 2a (dv_params): 2a S = S', a S = S'/2
    const double S = kp_b + km_b;
    const double rk = frcp(km_b);                      // off the v row's chain
    // explicit FMA chains (the library is built with -fmad=false)
    vn = fma(fma(f.ag4, am.g, fma(f.cpl2, am.v - vp, S * (vcn - vp))), frcp(fma(0.5, S, f.cpl1)), vp);
    const double vbar = 0.5 * (vn + vp);
    const double vg = fma(-(f.dx2a * rk), fma(f.BiM, vbar - am.v, -am.g), vcn);
    double t = f.b4 * (ucn - up);
    t = fma(f.cplu2, am.u - up, t);
    t = fma(-f.gamma, vn - vp, t);
    t = fma(f.b2r, vcn - vg, t);
    t = fma(-f.b4dx, fma(f.BiTM, vbar - am.v, -am.q), t);
    t = fma(f.g2, vcn + vg, t);
    t = fma(-f.g2, vn + vp, t);
    un = fma(t, f.inv_fu, up);
}

struct DvLane {
    bool rev;       // registers hold nodes in reversed order (last live lane / lane 31)
    bool mirror0;   // register 0's outer neighbour is the mirrored inner one
    bool face;      // register 0 is a real face (FACES steps only)
};

// One DF step of this lane's NPT nodes: P holds layer n-1 on entry and n+1 on
// exit, C holds layer n.  M = live registers of the reversed lane.  FACES: the
// warp holds a real face (uniform per warp): register 0 also runs the face row.
template <int NPT, int M, bool FACES>
__device__ __forceinline__ void dv_step(double (&vP)[NPT], const double (&vC)[NPT], double (&uP)[NPT],
                                        const double (&uC)[NPT], const DvLane& L, const DvRow& r,
                                        const DvFace& fc, const DvParams& q, const double* tab,
                                        const Ambient& am, unsigned& acc) {
    constexpr unsigned FULL = 0xffffffffu;
    const double vs = L.rev ? vC[M - 1] : vC[0];       // this lane's lowest node
    const double us = L.rev ? uC[M - 1] : uC[0];
    const double vup = __shfl_up_sync(FULL, vC[NPT - 1], 1);
    const double uup = __shfl_up_sync(FULL, uC[NPT - 1], 1);
    const double vdn = __shfl_down_sync(FULL, vs, 1);
    const double udn = __shfl_down_sync(FULL, us, 1);
    double vN[NPT], uN[NPT];                           // register-order successors
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        if (M < NPT && j == M - 1) {
            vN[j] = L.rev ? vup : vC[j + 1];
            uN[j] = L.rev ? uup : uC[j + 1];
        } else if (j == NPT - 1) {
            vN[j] = (M == NPT && L.rev) ? vup : vdn;
            uN[j] = (M == NPT && L.rev) ? uup : udn;
        } else {
            vN[j] = vC[j + 1];
            uN[j] = uC[j + 1];
        }
    }
    const double hl = d_half(q, vC[NPT - 1] + vN[NPT - 1], tab);
    double hprev = __shfl_up_sync(FULL, hl, 1);        // half node left of register 0
    const double dnode = FACES ? d_half(q, vC[0] + vC[0], tab) : 0.0;   // ghost side: node value
    const double vx0 = L.mirror0 ? vN[0] : vup;
    const double ux0 = L.mirror0 ? uN[0] : uup;
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        const double hj = j == NPT - 1 ? hl : d_half(q, vC[j] + vN[j], tab);
        double vn, un;
        dv_interior(r, vP[j], uP[j], j == 0 ? vx0 : vC[j - 1], vN[j], j == 0 ? ux0 : uC[j - 1], uN[j], hprev, hj,
                    vn, un, L.rev);
        if (FACES && j == 0) {
            double vf, uf;
            dv_face(fc, am, vP[0], uP[0], vN[0], uN[0], dnode, hj, vf, uf);
            vn = L.face ? vf : vn;
            un = L.face ? uf : un;
        }
        const unsigned g = static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn));
        if (j < M) acc |= g;
        else acc |= L.rev ? 0u : g;                    // dead registers of the reversed lane
        vP[j] = vn;
        uP[j] = un;
        hprev = hj;
    }
}

constexpr int kDvWarps = 4;     // walls (K2w) or windows (K3w) per CTA
// K3w: 3 CTAs (12 warps) per SM — caps registers at 168 (uncapped the
// compiler takes 222 and only 8 warps fit; 4 CTAs at 128 registers spill: 3.07e11 vs 3.17e11)
constexpr int kK3MinB = 3;

// K2w: one warp per wall, n <= 32 NPT, all steps of a segment in one launch.
// The host picks NPT = the smallest power of two >= n/32 and M = n - Lr NPT
// (Lr = (n-1)/NPT, the reversed lane).
template <int NPT, int M>
__global__ void __launch_bounds__(kDvWarps * 32) k_dv_walls(const NonlinearSegArgs A) {
    __shared__ double s_tab_rep[kExpTab * kExpRep];
    const double* s_tab = s_tab_rep + (threadIdx.x & (kExpRep - 1));   // this lane's copy
    __shared__ Ambient s_amb[kDvWarps][kNlChunk][2];   // [warp][step][face]
    if (launch_stopped(A.stop)) return;
    stage_exp_table_rep(s_tab_rep, threadIdx.x, blockDim.x);
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int w = blockIdx.x * kDvWarps + warp;
    if (w >= A.n_walls) return;                        // whole warp
    const int n = A.n;
    const int Lr = (n - 1) / NPT;
    const bool live = lane <= Lr;
    DvLane L;
    L.rev = lane == Lr;
    L.face = lane == 0 || L.rev;
    L.mirror0 = L.face;
    const size_t o = static_cast<size_t>(w) * n;
    double up[NPT], uc[NPT], vp[NPT], vc[NPT];
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        const bool ok = live && (!L.rev || j < M);
        const size_t i = o + (L.rev ? n - 1 - j : lane * NPT + j);
        up[j] = ok ? A.in[0][i] : 1.0;
        uc[j] = ok ? A.in[1][i] : 1.0;
        vp[j] = ok ? A.in[2][i] : 1.0;
        vc[j] = ok ? A.in[3][i] : 1.0;
    }
    const AnalyticRow rc = analytic_row(A.groups[w], A.dx, A.dt);
    const DvRow r = dv_row(rc);
    const DvParams q = dv_params(A.p, 2.0 * rc.a);
    const int f = L.rev ? 1 : 0;
    const DvFace fc = dv_face_consts(rc, A.biot[2 * w + f]);
    const int chl = A.chan[2 * w], chr = A.chan[2 * w + 1];
    unsigned acc = 0;
    for (int c0 = 0; c0 < A.nsteps; c0 += kNlChunk) {
        const int clen = min(kNlChunk, A.nsteps - c0);
        __syncwarp();
        for (int i = lane; i < 2 * clen; i += 32)
            s_amb[warp][i >> 1][i & 1] = A.table[static_cast<size_t>(c0 + (i >> 1)) * A.n_channels + ((i & 1) ? chr : chl)];
        __syncwarp();
        int s = 0;
        for (; s + 1 < clen; s += 2) {
            dv_step<NPT, M, true>(vp, vc, up, uc, L, r, fc, q, s_tab, s_amb[warp][s][f], acc);
            dv_step<NPT, M, true>(vc, vp, uc, up, L, r, fc, q, s_tab, s_amb[warp][s + 1][f], acc);
        }
        if (s < clen) {   // odd tail (last chunk only): rotate by copies
            dv_step<NPT, M, true>(vp, vc, up, uc, L, r, fc, q, s_tab, s_amb[warp][s][f], acc);
#pragma unroll
            for (int j = 0; j < NPT; ++j) {
                double t = vp[j]; vp[j] = vc[j]; vc[j] = t;
                t = up[j]; up[j] = uc[j]; uc[j] = t;
            }
        }
    }
    // fast guard verdict (bit 30 of the high word: |x| >= 2 or not finite)
    const unsigned any = __reduce_or_sync(0xffffffffu, live ? acc : 0u);
    if ((any & 0x40000000u) && lane == 0) atomicCAS(A.suspect, 0, A.seg_index + 1);
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        if (!live || (L.rev && j >= M)) continue;
        const size_t i = o + (L.rev ? n - 1 - j : lane * NPT + j);
        A.out[0][i] = up[j];
        A.out[1][i] = uc[j];
        A.out[2][i] = vp[j];
        A.out[3][i] = vc[j];
    }
}

// K2s: one wall split over NW warps, one node per lane, for walls too few to
// fill the GPU (configs[0]: a single 101-node wall).  The march is then bound
// by the per-step dependency chain of one warp's in-order instruction stream;
// splitting the wall over NW warps (one per scheduler) cuts that stream NW
// ways.  Neighbours inside a warp come from shuffles, across warps through
// shared memory (double-buffered by step parity) behind one barrier per step.
// Each lane evaluates both of its half nodes (the shared one is computed
// twice, bit for bit alike: the sum commutes), so no second exchange is
// needed.  Only the warps holding a face run the face row (warp-uniform).
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_dv_wall_split(const NonlinearSegArgs A) {
    constexpr bool FACE_ALL = NW <= 4;                 // every warp runs the face code: no branch
    __shared__ double s_tab_rep[kExpTab * kExpRep];
    const double* s_tab = s_tab_rep + (threadIdx.x & (kExpRep - 1));   // this lane's copy
    __shared__ Ambient s_amb[kNlChunk][2];
    __shared__ double s_x[2][NW][4];                  // [parity][warp] {v, u} of lanes 0 and 31
    if (launch_stopped(A.stop)) return;
    stage_exp_table_rep(s_tab_rep, threadIdx.x, blockDim.x);
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int w = blockIdx.x, n = A.n, j = tid;
    const bool live = j < n;
    const bool lf = j == 0, rf = j == n - 1;
    const bool face_warp = warp == 0 || warp == (n - 1) / 32;
    const size_t o = static_cast<size_t>(w) * n + j;
    double up = live ? A.in[0][o] : 1.0, uc = live ? A.in[1][o] : 1.0;
    double vp = live ? A.in[2][o] : 1.0, vc = live ? A.in[3][o] : 1.0;
    const AnalyticRow rc = analytic_row(A.groups[w], A.dx, A.dt);
    const DvRow r = dv_row(rc);
    const DvParams q = dv_params(A.p, 2.0 * rc.a);
    const DvFace fc = dv_face_consts(rc, A.biot[2 * w + (rf ? 1 : 0)]);
    const int chl = A.chan[2 * w], chr = A.chan[2 * w + 1];
    constexpr unsigned FULL = 0xffffffffu;
    unsigned acc = 0;
    for (int c0 = 0; c0 < A.nsteps; c0 += kNlChunk) {
        const int clen = min(kNlChunk, A.nsteps - c0);
        __syncthreads();
        for (int i = tid; i < 2 * clen; i += NW * 32)
            s_amb[i >> 1][i & 1] = A.table[static_cast<size_t>(c0 + (i >> 1)) * A.n_channels + ((i & 1) ? chr : chl)];
        for (int s = 0; s < clen; ++s) {
            const int b = s & 1;
            if (lane == 0) { s_x[b][warp][0] = vc; s_x[b][warp][1] = uc; }
            if (lane == 31) { s_x[b][warp][2] = vc; s_x[b][warp][3] = uc; }
            __syncthreads();
            double vL = __shfl_up_sync(FULL, vc, 1), uL = __shfl_up_sync(FULL, uc, 1);
            double vR = __shfl_down_sync(FULL, vc, 1), uR = __shfl_down_sync(FULL, uc, 1);
            if (lane == 0 && warp > 0) { vL = s_x[b][warp - 1][2]; uL = s_x[b][warp - 1][3]; }
            if (lane == 31 && warp < NW - 1) { vR = s_x[b][warp + 1][0]; uR = s_x[b][warp + 1][1]; }
            const double hL = d_half_lat(q, vL + vc, s_tab);
            const double hR = d_half_lat(q, vc + vR, s_tab);
            double vn, un;
            dv_interior(r, vp, up, vL, vR, uL, uR, hL, hR, vn, un);
            if (FACE_ALL || face_warp) {
                // branch-free inside the warp: the face chain runs beside the
                // interior one, not after it.  Ghost side d(v_face); the row
                // needs the interior neighbour only.
                const double dnode = d_half_lat(q, vc + vc, s_tab);
                double vf, uf;
                dv_face(fc, s_amb[s][rf ? 1 : 0], vp, up, rf ? vL : vR, rf ? uL : uR, dnode, rf ? hL : hR, vf, uf);
                vn = (lf || rf) ? vf : vn;
                un = (lf || rf) ? uf : un;
            }
#ifdef DV_SKIP_U   // timing experiment only: the u chain left out of the step
            un = up;
#endif
            acc |= live ? (static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn))) : 0u;
            up = uc;
            vp = vc;
            uc = un;
            vc = vn;
        }
    }
    const unsigned any = __reduce_or_sync(FULL, acc);
    if ((any & 0x40000000u) && lane == 0) atomicCAS(A.suspect, 0, A.seg_index + 1);
    if (live) {
        A.out[0][o] = up;
        A.out[1][o] = uc;
        A.out[2][o] = vp;
        A.out[3][o] = vc;
    }
}

// K2h: K2s with redundant halos instead of a barrier per step.  Warp k holds
// the 32 consecutive nodes g = k (32 - 2H) - H + lane and owns lanes
// H .. 31-H; an artificial warp edge corrupts one lane per step, so the owned
// lanes stay exact for H steps between exchanges (the faces read only their
// interior neighbour, so lanes outside [0, n) never reach a live node).  Every
// H steps the owned lanes publish both layers to shared memory and every lane
// reloads its node behind one barrier.  Each lane evaluates its right half
// node only and takes the left one from the previous lane by a shuffle (K2s
// evaluates both: its lane 0 has no in-warp predecessor).  Per node the
// arithmetic is K2s's, so the two are bitwise equal.
template <int NW, int H>
__global__ void __launch_bounds__(NW * 32) k_dv_wall_halo(const NonlinearSegArgs A) {
    constexpr int T = 32 - 2 * H;                      // owned nodes per warp
    __shared__ double s_tab_rep[kExpTab * kExpRep];
    const double* s_tab = s_tab_rep + (threadIdx.x & (kExpRep - 1));   // this lane's copy
    __shared__ Ambient s_amb[kNlChunk][2];
    __shared__ double s_st[4][NW * T];                 // {u_prev, u_curr, v_prev, v_curr} by node
    if (launch_stopped(A.stop)) return;
    stage_exp_table_rep(s_tab_rep, threadIdx.x, blockDim.x);
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int w = blockIdx.x, n = A.n, j = warp * T - H + lane;
    const bool live = j >= 0 && j < n;
    const bool own = live && lane >= H && lane < 32 - H;
    const bool lf = j == 0, rf = j == n - 1;
    const size_t base = static_cast<size_t>(w) * n;
    double up = live ? A.in[0][base + j] : 1.0, uc = live ? A.in[1][base + j] : 1.0;
    double vp = live ? A.in[2][base + j] : 1.0, vc = live ? A.in[3][base + j] : 1.0;
    const AnalyticRow rc = analytic_row(A.groups[w], A.dx, A.dt);
    const DvRow r = dv_row(rc);
    const DvParams q = dv_params(A.p, 2.0 * rc.a);
    const DvFace fc = dv_face_consts(rc, A.biot[2 * w + (rf ? 1 : 0)]);
    const int chl = A.chan[2 * w], chr = A.chan[2 * w + 1];
    constexpr unsigned FULL = 0xffffffffu;
    unsigned acc = 0;
    int since = 0;
    for (int c0 = 0; c0 < A.nsteps; c0 += kNlChunk) {
        const int clen = min(kNlChunk, A.nsteps - c0);
        __syncthreads();
        for (int i = tid; i < 2 * clen; i += NW * 32)
            s_amb[i >> 1][i & 1] = A.table[static_cast<size_t>(c0 + (i >> 1)) * A.n_channels + ((i & 1) ? chr : chl)];
        __syncthreads();
        for (int s = 0; s < clen; ++s) {
            if (since == H) {                          // halo refresh (block-uniform)
                if (own) { s_st[0][j] = up; s_st[1][j] = uc; s_st[2][j] = vp; s_st[3][j] = vc; }
                __syncthreads();
                if (live) { up = s_st[0][j]; uc = s_st[1][j]; vp = s_st[2][j]; vc = s_st[3][j]; }
                __syncthreads();                       // the next refresh overwrites s_st
                since = 0;
            }
            const double vL = __shfl_up_sync(FULL, vc, 1), uL = __shfl_up_sync(FULL, uc, 1);
            const double vR = __shfl_down_sync(FULL, vc, 1), uR = __shfl_down_sync(FULL, uc, 1);
            // the left half node is the previous lane's right one (the sum
            // commutes: bit for bit the local evaluation); lane 0 is a halo lane
#ifdef DV_HALO_SQRT   // timing experiment only (tools/dv_time_probe.py)
            const double hR = d_half(q, vc + vR, s_tab);
#else
            const double hR = d_half_lat(q, vc + vR, s_tab);
#endif
            const double hL = __shfl_up_sync(FULL, hR, 1);
            double vn, un;
            dv_interior(r, vp, up, vL, vR, uL, uR, hL, hR, vn, un);
            {
#ifdef DV_HALO_SQRT
                const double dnode = d_half(q, vc + vc, s_tab);
#else
                const double dnode = d_half_lat(q, vc + vc, s_tab);
#endif
                double vf, uf;
                dv_face(fc, s_amb[s][rf ? 1 : 0], vp, up, rf ? vL : vR, rf ? uL : uR, dnode, rf ? hL : hR, vf, uf);
                vn = (lf || rf) ? vf : vn;
                un = (lf || rf) ? uf : un;
            }
            acc |= own ? (static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn))) : 0u;
            up = uc;
            vp = vc;
            uc = un;
            vc = vn;
            ++since;
        }
    }
    const unsigned any = __reduce_or_sync(FULL, acc);
    if ((any & 0x40000000u) && lane == 0) atomicCAS(A.suspect, 0, A.seg_index + 1);
    if (own) {
        A.out[0][base + j] = up;
        A.out[1][base + j] = uc;
        A.out[2][base + j] = vp;
        A.out[3][base + j] = vc;
    }
}

// K3w window geometry (n >= 32 NPT): window t starts at min(t T, n - W) and
// owns [t == 0 ? 0 : t T + NPT, min(t T + 31 NPT, n)).  Window 0 holds the
// left face, windows t >= rface(n) end at the right face (at most three).
template <int NPT>
struct DvTiles {
    static constexpr int W = 32 * NPT, T = W - 2 * NPT;
    static __host__ __device__ int64_t count(int64_t n) { return (n - NPT + T - 1) / T; }
    static __host__ __device__ int64_t rface(int64_t n) { return (n - W + T - 1) / T; }
};

// K3w: one warp per window, A.steps <= NPT steps per launch.  FACES = false:
// the interior windows 1 .. rface-1 (no face code, fewer registers); FACES =
// true: one CTA for window 0 and the right-face windows.
template <int NPT, bool FACES>
__global__ void __launch_bounds__(kDvWarps * 32) k_dv_tiled(const TiledArgs A) {
    using G = DvTiles<NPT>;
    constexpr int W = G::W, T = G::T;
    __shared__ double s_tab_rep[kExpTab * kExpRep];
    const double* s_tab = s_tab_rep + (threadIdx.x & (kExpRep - 1));   // this lane's copy
    if (launch_stopped(A.stop)) return;
    stage_exp_table_rep(s_tab_rep, threadIdx.x, blockDim.x);
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t n = A.n;
    const int64_t tr = G::rface(n);
    int64_t t;
    if (FACES) {
        t = warp == 0 ? 0 : tr + warp - 1;
        if (warp > 0 && (t <= 0 || t >= G::count(n))) return;
    } else {
        t = static_cast<int64_t>(blockIdx.x) * kDvWarps + warp;
        if (t == 0 || t >= tr) return;
    }
    const int64_t own0 = t == 0 ? 0 : t * T + NPT;
    const int64_t own1 = min(t * T + 31 * NPT, n);
    const int64_t g0 = min(t * T, n - W);
    const bool lf = FACES && g0 == 0, rf = FACES && g0 + W == n;
    DvLane L;
    L.rev = lane == 31;
    L.mirror0 = (lane == 0 && lf) || L.rev;
    L.face = (lane == 0 && lf) || (L.rev && rf);
    const bool guard = (lane != 0 || lf) && (lane != 31 || rf);   // stale lanes stay out
    double up[NPT], uc[NPT], vp[NPT], vc[NPT];
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        const int64_t i = g0 + (L.rev ? W - 1 - j : lane * NPT + j);
        up[j] = A.in[0][i];
        uc[j] = A.in[1][i];
        vp[j] = A.in[2][i];
        vc[j] = A.in[3][i];
    }
    const AnalyticRow rc = analytic_row(A.groups, A.dx, A.dt);
    const DvRow r = dv_row(rc);
    const DvParams q = dv_params(A.p, 2.0 * rc.a);
    const DvFace fc = dv_face_consts(rc, L.rev ? A.br : A.bl);
    const int ch = L.rev ? A.chr : A.chl;
    unsigned acc = 0;
    auto amb = [&](int k) { return FACES ? A.table[static_cast<size_t>(k) * A.n_channels + ch] : Ambient{}; };
    int k = 0;
    for (; k + 1 < A.steps; k += 2) {
        dv_step<NPT, NPT, FACES>(vp, vc, up, uc, L, r, fc, q, s_tab, amb(k), acc);
        dv_step<NPT, NPT, FACES>(vc, vp, uc, up, L, r, fc, q, s_tab, amb(k + 1), acc);
    }
    if (k < A.steps) {
        dv_step<NPT, NPT, FACES>(vp, vc, up, uc, L, r, fc, q, s_tab, amb(k), acc);
#pragma unroll
        for (int j = 0; j < NPT; ++j) {
            double x = vp[j]; vp[j] = vc[j]; vc[j] = x;
            x = up[j]; up[j] = uc[j]; uc[j] = x;
        }
    }
    const unsigned any = __reduce_or_sync(0xffffffffu, guard ? acc : 0u);
    if ((any & 0x40000000u) && lane == 0) atomicCAS(A.suspect, 0, A.seg_index + 1);
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        const int64_t i = g0 + (L.rev ? W - 1 - j : lane * NPT + j);
        if (i < own0 || i >= own1) continue;
        A.out[0][i] = up[j];
        A.out[1][i] = uc[j];
        A.out[2][i] = vp[j];
        A.out[3][i] = vc[j];
    }
}

__device__ __forceinline__ void dv_cp_async8(double* smem, const double* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void dv_cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void dv_cp_async_wait() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// K3w interior windows, persistent: each warp marches windows t, t + stride, ...
// (stride = all warps of the grid) and prefetches its next window into its own
// shared-memory buffer with cp.async while it computes the current one, so
// the window loads leave the critical path.  Buffer layout per field: lane
// block l of NPT nodes, node j of the block at l NPT + (j ^ (l mod NPT)) (XOR
// swizzle: the per-register reads of a warp spread over the banks).
template <int NPT, int MINB = 0>
__global__ void __launch_bounds__(kDvWarps * 32, MINB) k_dv_tiled_stream(const TiledArgs A) {
    using G = DvTiles<NPT>;
    constexpr int W = G::W, T = G::T;
    static_assert((NPT & (NPT - 1)) == 0, "NPT must be a power of two");
    __shared__ double s_tab_rep[kExpTab * kExpRep];
    const double* s_tab = s_tab_rep + (threadIdx.x & (kExpRep - 1));   // this lane's copy
    __shared__ __align__(16) double s_buf[kDvWarps][4][W];
    if (launch_stopped(A.stop)) return;
    stage_exp_table_rep(s_tab_rep, threadIdx.x, blockDim.x);
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t tr = A.t_end;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kDvWarps;
    int64_t t = A.t_begin + static_cast<int64_t>(blockIdx.x) * kDvWarps + warp;
    if (t >= tr) return;
    double(*buf)[W] = s_buf[warp];
    auto swz = [](int i) { return (i & ~(NPT - 1)) | ((i ^ (i / NPT)) & (NPT - 1)); };
    auto prefetch = [&](int64_t tt) {
        const int64_t g0 = tt * T;
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int k = 0; k < W / 32; ++k) {
                const int i = lane + 32 * k;
                dv_cp_async8(&buf[f][swz(i)], A.in[f] + g0 + i);
            }
        dv_cp_async_commit();
    };
    prefetch(t);
    const AnalyticRow rc = analytic_row(A.groups, A.dx, A.dt);
    const DvRow r = dv_row(rc);
    const DvParams q = dv_params(A.p, 2.0 * rc.a);
    const DvFace fc{};
    DvLane L;
    L.rev = false;        // no reversed lane here (lanes 0 and 31 are the stale ones): the selects of
    L.mirror0 = false;    // dv_step / dv_interior fold away; the artificial window edges are the
    L.face = false;       // shuffles' own-value results in lanes 0 and 31
    const bool store = lane != 0 && lane != 31;      // the stale lanes stay out of the guard and the output
    unsigned acc = 0;
    for (; t < tr; t += stride) {
        double up[NPT], uc[NPT], vp[NPT], vc[NPT];
        dv_cp_async_wait();
        __syncwarp();
#pragma unroll
        for (int j = 0; j < NPT; ++j) {
            const int i = swz(L.rev ? W - 1 - j : lane * NPT + j);
            up[j] = buf[0][i];
            uc[j] = buf[1][i];
            vp[j] = buf[2][i];
            vc[j] = buf[3][i];
        }
        __syncwarp();
        if (t + stride < tr) prefetch(t + stride);
        int k = 0;
        for (; k + 1 < A.steps; k += 2) {
            dv_step<NPT, NPT, false>(vp, vc, up, uc, L, r, fc, q, s_tab, Ambient{}, acc);
            dv_step<NPT, NPT, false>(vc, vp, uc, up, L, r, fc, q, s_tab, Ambient{}, acc);
        }
        if (k < A.steps) {
            dv_step<NPT, NPT, false>(vp, vc, up, uc, L, r, fc, q, s_tab, Ambient{}, acc);
#pragma unroll
            for (int j = 0; j < NPT; ++j) {
                double x = vp[j]; vp[j] = vc[j]; vc[j] = x;
                x = up[j]; up[j] = uc[j]; uc[j] = x;
            }
        }
        if (store) {   // lanes 1..30: NPT consecutive owned nodes, 16-byte stores
            const int64_t i0 = t * T + lane * NPT;
#pragma unroll
            for (int j = 0; j < NPT; j += 2) {
                reinterpret_cast<double2*>(A.out[0] + i0)[j / 2] = make_double2(up[j], up[j + 1]);
                reinterpret_cast<double2*>(A.out[1] + i0)[j / 2] = make_double2(uc[j], uc[j + 1]);
                reinterpret_cast<double2*>(A.out[2] + i0)[j / 2] = make_double2(vp[j], vp[j + 1]);
                reinterpret_cast<double2*>(A.out[3] + i0)[j / 2] = make_double2(vc[j], vc[j + 1]);
            }
        }
    }
    const unsigned any = __reduce_or_sync(0xffffffffu, store ? acc : 0u);
    if ((any & 0x40000000u) && lane == 0) atomicCAS(A.suspect, 0, A.seg_index + 1);
}


// ---- K3w with TMA-staged windows ------------------------------------------------------
// The four layers of a window arrive as 2-D tiles on the TMA engine (UTMALDG):
// each state array is described to the hardware as rows of NPT = 8 nodes (64 B),
// a window is a box of 32 rows (W = 256 nodes, 2 KB), and the 64-byte swizzle
// mode stores 16-byte chunk c of row r at chunk c ^ ((r / 2) mod 4).  Lane l owns
// row l, so its four 16-byte reads hit eight distinct bank groups per quarter
// warp in register order — no per-lane copies (64 LDGSTS per window in
// k_dv_tiled_stream), no swizzled address arithmetic, no select network.  One
// elected lane issues the four copies of the warp's NEXT window on the warp's
// mbarrier while the current window is marched in registers.
struct TiledMaps { CUtensorMap m[4]; };   // the launch's input layers (up, uc, vp, vc)

__device__ __forceinline__ unsigned dv_smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void dv_mbar_init(void* mb, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(dv_smem_u32(mb)), "r"(count));
}
__device__ __forceinline__ void dv_mbar_expect_tx(void* mb, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(dv_smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void dv_mbar_wait(void* mb, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n DV_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra DV_WAIT_%=;\n}\n" ::"r"(dv_smem_u32(mb)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void dv_tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, void* mb) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            dv_smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(dv_smem_u32(mb))
        : "memory");
}

template <int NPT, int MINB = 0>
__global__ void __launch_bounds__(kDvWarps * 32, MINB) k_dv_tiled_tma(const TiledArgs A,
                                                                      const __grid_constant__ TiledMaps M) {
    using G = DvTiles<NPT>;
    constexpr int W = G::W, T = G::T;
    static_assert(NPT == 8, "a row of the tensor maps is NPT = 8 nodes (64-byte swizzle)");
    __shared__ double s_tab_rep[kExpTab * kExpRep];
    const double* s_tab = s_tab_rep + (threadIdx.x & (kExpRep - 1));   // this lane's copy
    __shared__ __align__(1024) double s_buf[kDvWarps][4][W];           // 2 KB tiles, swizzle period 512 B
    __shared__ __align__(8) unsigned long long s_mbar[kDvWarps];
    if (launch_stopped(A.stop)) return;
    stage_exp_table_rep(s_tab_rep, threadIdx.x, blockDim.x);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (lane == 0) {
        dv_mbar_init(&s_mbar[warp], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int64_t tr = A.t_end;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kDvWarps;
    int64_t t = A.t_begin + static_cast<int64_t>(blockIdx.x) * kDvWarps + warp;
    if (t >= tr) return;
    double(*buf)[W] = s_buf[warp];
    void* mbar = &s_mbar[warp];
    auto prefetch = [&](int64_t tt) {
        if (lane == 0) {
            dv_mbar_expect_tx(mbar, 4u * W * sizeof(double));
            const int row = static_cast<int>(tt * (T / NPT));          // window start tt T = row tt T / 8
#pragma unroll
            for (int f = 0; f < 4; ++f) dv_tma_load_2d(buf[f], &M.m[f], 0, row, mbar);
        }
    };
    prefetch(t);
    const AnalyticRow rc = analytic_row(A.groups, A.dx, A.dt);
    const DvRow r = dv_row(rc);
    const DvParams q = dv_params(A.p, 2.0 * rc.a);
    const DvFace fc{};
    DvLane L;
    L.rev = false;        // no reversed lane here (lanes 0 and 31 are the stale ones): the selects of
    L.mirror0 = false;    // dv_step / dv_interior fold away; the artificial window edges are the
    L.face = false;       // shuffles' own-value results in lanes 0 and 31
    const bool store = lane != 0 && lane != 31;      // the stale lanes stay out of the guard and the output
    const int sw = (lane >> 1) & 3;                  // this row's chunk swizzle
    unsigned acc = 0;
    for (int it = 0; t < tr; t += stride, ++it) {
        double up[NPT], uc[NPT], vp[NPT], vc[NPT];
        dv_mbar_wait(mbar, it & 1);
        auto rd = [&](int f, double (&x)[NPT]) {
            double tv[NPT];
#pragma unroll
            for (int c = 0; c < NPT / 2; ++c) {
                const double2 v = *reinterpret_cast<const double2*>(&buf[f][lane * NPT + 2 * (c ^ sw)]);
                tv[2 * c] = v.x;
                tv[2 * c + 1] = v.y;
            }
#pragma unroll
            for (int j = 0; j < NPT; ++j) x[j] = L.rev ? tv[NPT - 1 - j] : tv[j];
        };
        rd(0, up);
        rd(1, uc);
        rd(2, vp);
        rd(3, vc);
        __syncwarp();                                // the tiles are free for the next window
        if (t + stride < tr) prefetch(t + stride);
        int k = 0;
        for (; k + 1 < A.steps; k += 2) {
            dv_step<NPT, NPT, false>(vp, vc, up, uc, L, r, fc, q, s_tab, Ambient{}, acc);
            dv_step<NPT, NPT, false>(vc, vp, uc, up, L, r, fc, q, s_tab, Ambient{}, acc);
        }
        if (k < A.steps) {
            dv_step<NPT, NPT, false>(vp, vc, up, uc, L, r, fc, q, s_tab, Ambient{}, acc);
#pragma unroll
            for (int j = 0; j < NPT; ++j) {
                double x = vp[j]; vp[j] = vc[j]; vc[j] = x;
                x = up[j]; up[j] = uc[j]; uc[j] = x;
            }
        }
        if (store) {   // lanes 1..30: NPT consecutive owned nodes, 16-byte stores
            const int64_t i0 = t * T + lane * NPT;
#pragma unroll
            for (int j = 0; j < NPT; j += 2) {
                reinterpret_cast<double2*>(A.out[0] + i0)[j / 2] = make_double2(up[j], up[j + 1]);
                reinterpret_cast<double2*>(A.out[1] + i0)[j / 2] = make_double2(uc[j], uc[j + 1]);
                reinterpret_cast<double2*>(A.out[2] + i0)[j / 2] = make_double2(vp[j], vp[j + 1]);
                reinterpret_cast<double2*>(A.out[3] + i0)[j / 2] = make_double2(vc[j], vc[j + 1]);
            }
        }
    }
    const unsigned any = __reduce_or_sync(0xffffffffu, store ? acc : 0u);
    if ((any & 0x40000000u) && lane == 0) atomicCAS(A.suspect, 0, A.seg_index + 1);
}

}  // namespace hyg
