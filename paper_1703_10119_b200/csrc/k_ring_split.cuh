// k_ring_split.cuh — K6: the zone-ring building march split along its
// dependency cone (configs[3]: 8,192 zones x 6 constant walls x 128 nodes).
//
// Replaces S consecutive step_explicit calls (building.cpp:152-187) exactly as
// K4 / K4r do — same increment-form rows (hyg_coef.cuh), same zone arithmetic
// (zone_rhs / zone_step_explicit, zone.cpp:26-74) in the same order — but
// without a barrier per step on the walls' path.  A wall meets its zone only
// through its face-1 node, and after k DF steps that node depends on the last
// k + 1 nodes of the wall alone (plus the zone air of layers 0 .. k-1).  So:
//
//   phase 1, k_ring_cone: for every zone the air ODE together with the last
//     S + 1 nodes of each of its walls (the "cone": the cut end goes stale one
//     node per step and never reaches the face node within S steps) is marched
//     S steps — one thread per wall cone, one per zone, a CTA of LB
//     consecutive zones whose outer S on each side are halo copies (the zone
//     cone grows one zone per step along the ring).  It records the layer-k
//     air of every owned zone, k = 0 .. S-1, in `series` ([zone][S][2]) and
//     writes the zone air of layer S.  ~4 % of the walls' node-updates.
//   phase 2, k_ring_walls: every wall is marched S steps in registers in K1's
//     layout (k_coupled.cuh: 16 lanes x NPT nodes, two walls per warp,
//     neighbours by shuffles, both faces in register 0), its face-1 ambient
//     read from `series`.  No shared surfaces, no barrier in the step loop,
//     no halo walls: 64 B per node per S steps of HBM traffic (8 B per update
//     at S = 8) and K1's 7 FP64 instructions per update.
//
// The face-1 node is computed twice (cone thread and owning lane) with the
// same instruction sequence on the same inputs, so both phases hold the same
// bits and the result equals K4r's and the per-step path's bit for bit.
// Guard: K1's fast guard (bit 30 of the high word) over walls (phase 2) and
// owned zones (phase 1); a set bit stops the following launches and the host
// replays from the flagged launch's untouched input with K4 (exact guard).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "k_ring_reg.cuh"

namespace hyg {

#ifndef HYG_RING_CONE_THREADS
#define HYG_RING_CONE_THREADS 544
#endif
constexpr int kRingConeThreads = HYG_RING_CONE_THREADS;
constexpr int kRingWallWarps = 4;        // k_ring_walls: warps per CTA (two walls each)

template <int S>
struct RingConeShape {
    static constexpr int kP = S + 1;                 // nodes kept per wall cone
    static constexpr int kPS = (kP + 1) & ~1;        // loaded (even: 16-byte loads)
    __host__ __device__ static int cone_warps(int LB, int W) { return ((LB - 2) * W + 31) / 32; }
    __host__ __device__ static int zone_warps(int LB) { return (LB + 31) / 32; }
    __host__ __device__ static int threads(int LB, int W) { return 32 * (cone_warps(LB, W) + zone_warps(LB)); }
    // doubles: surfaces [parity][field][W][LB], zone air [parity][field][LB], forcing rows [S][rw]
    __host__ __device__ static size_t smem_doubles(int LB, int W, int rw) {
        return static_cast<size_t>(4) * W * LB + 4 * LB + static_cast<size_t>(S) * rw;
    }
};

// ---- phase 1 ---------------------------------------------------------------------------
template <int S, int NL = kRingMaxLinks, int NP = kRingMaxPeers>
__global__ void __launch_bounds__(kRingConeThreads, 1) k_ring_cone(const RingArgs a, double* __restrict__ series,
                                                                  const int LB) {
    using Sh = RingConeShape<S>;
    constexpr int P = Sh::kP, PS = Sh::kPS;
    extern __shared__ double smem[];
    if (launch_stopped(a.stop)) return;
    const int W = a.W, Z = a.n_zones, N = a.n;
    const int OB = LB - 2 * S;                          // owned zones per CTA
    const int z0 = blockIdx.x * OB, nown = min(OB, Z - z0), L = nown + 2 * S;
    const int rw = RingShape<8, S>::row_width(a.n_channels, a.n_sources);
    const int oSF = 0, oAR = oSF + 4 * W * LB, oRW = oAR + 4 * LB;
    auto sf_ix = [&](int par, int f, int slot) { return oSF + (par * 2 + f) * W * LB + slot; };
    auto ar_ix = [&](int par, int f, int i) { return oAR + (par * 2 + f) * LB + i; };
    const int tid = threadIdx.x, nthr = blockDim.x;
    for (int i = tid; i < a.steps * rw; i += nthr) {    // forcing rows of this launch
        const int k = i / rw, r = i - k * rw;
        smem[oRW + i] = r < 4 * a.n_channels
                            ? (reinterpret_cast<const double*>(a.table + static_cast<size_t>(k) * a.n_channels))[r]
                            : a.src[static_cast<size_t>(k) * (3 * a.n_sources + 2) + (r - 4 * a.n_channels)];
    }
    auto gz = [&](int i) {                              // global zone of local zone i (ring wrap)
        int g = (z0 - S + i) % Z;
        return g < 0 ? g + Z : g;
    };
    const int warp = tid / 32, lane = tid % 32;
    const int cone_w = Sh::cone_warps(LB, W);
    unsigned acc = 0;
    int cur = 0;
    if (warp < cone_w) {
        // wall cone: global nodes N-P .. N-1 of wall wi of local zone li; the cut
        // end (p = 0) mirrors itself
        const int li0 = 1 + tid / W, wi = tid - (li0 - 1) * W;
        const bool live = li0 <= L - 2;
        const int li = live ? li0 : 1;
        const int w = gz(li) * W + wi;
        const WallCoef& wc = a.coef[w];
        const double cb = wc.in.b, csu = wc.in.c_su, csv = wc.in.c_sv;
        const RowCoef c = wc.face[1];
        double up[P], uc[P], vp[P], vc[P];
        {
            const size_t g0 = static_cast<size_t>(w) * N + (N - PS);
            auto rd = [&](int f, double (&x)[P]) {
                double t[PS];
#pragma unroll
                for (int q = 0; q < PS / 2; ++q) {
                    const double2 v = *reinterpret_cast<const double2*>(a.in[f] + g0 + 2 * q);
                    t[2 * q] = v.x;
                    t[2 * q + 1] = v.y;
                }
#pragma unroll
                for (int p = 0; p < P; ++p) x[p] = t[PS - P + p];
            };
            rd(0, up);
            rd(1, uc);
            rd(2, vp);
            rd(3, vc);
        }
        const int slot = wi * LB + li;
        if (live) {
            smem[sf_ix(0, 0, slot)] = uc[P - 1];
            smem[sf_ix(0, 1, slot)] = vc[P - 1];
        }
        __syncthreads();                                // layer-0 surfaces, air and rows published
        auto step = [&](double (&vP)[P], double (&vC)[P], double (&uP)[P], double (&uC)[P]) {
            const double u_a = smem[ar_ix(cur, 0, li)], v_a = smem[ar_ix(cur, 1, li)];
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const double vl = p == 0 ? vC[0] : vC[p - 1], ul = p == 0 ? uC[0] : uC[p - 1];
                const double vr = p == P - 1 ? vC[P - 2] : vC[p + 1], ur = p == P - 1 ? uC[P - 2] : uC[p + 1];
                const double d = fma(-2.0, vP[p], vl + vr);
                const double du = fma(-2.0, uP[p], ul + ur);
                double vn, un;
                if (p < P - 1) {
                    vn = fma(cb, d, vP[p]);
                    un = fma(csv, d, fma(csu, du, uP[p]));
                } else {
                    const double t = v_a - vP[p], tu = u_a - uP[p];
                    vn = fma(c.e, t, fma(c.b, d, fma(c.e_g, 0.0, vP[p])));
                    un = fma(c.c_tv, t, fma(c.c_sv, d, fma(c.c_tu, tu, fma(c.c_su, du, fma(c.c_q, 0.0,
                                                                                        fma(c.c_g, 0.0, uP[p]))))));
                }
                vP[p] = vn;
                uP[p] = un;
            }
            if (live) {
                smem[sf_ix(cur ^ 1, 0, slot)] = uP[P - 1];
                smem[sf_ix(cur ^ 1, 1, slot)] = vP[P - 1];
            }
            __syncthreads();
            cur ^= 1;
        };
        int k = 0;
        for (; k + 1 < a.steps; k += 2) {
            step(vp, vc, up, uc);
            step(vc, vp, uc, up);
        }
        if (k < a.steps) step(vp, vc, up, uc);
    } else {
        // zone thread i: zone_step_explicit (zone.cpp:69-74) of local zone i (1 .. L-2
        // live; 0 and L-1 contribute their layer-0 air only); parameter block as K4r's
        const int i = tid - 32 * cone_w;
        const bool valid = i < L;
        const bool live = i >= 1 && i < L - 1;
        const bool owned = i >= S && i < S + nown;
        const int zg = gz(valid ? i : 0);
        const double* zp = a.zparams + static_cast<size_t>(zg) * kRingZP;
        int nlink = 0, npeer = 0, sidx = 0;
        if (live) {
            nlink = static_cast<int>(zp[4]);
            npeer = static_cast<int>(zp[5]);
            sidx = static_cast<int>(zp[6]);
        }
        int ls[NL], pidx[NP];
        const double c0 = zp[0], gv = zp[1], qv1 = zp[2], qv2 = zp[3];
        double lT[NL], lM[NL], lD[NL], pg[NP], pq1[NP], pq2[NP];
        const int iv = valid ? i : 0;
#pragma unroll
        for (int q = 0; q < NL; ++q) {
            const int wi = q < nlink ? static_cast<int>(zp[8 + 4 * q]) : 0;
            ls[q] = wi * LB + iv;
            lT[q] = zp[9 + 4 * q];
            lM[q] = zp[10 + 4 * q];
            lD[q] = zp[11 + 4 * q];
        }
        const int zprev = gz(iv >= 1 ? iv - 1 : 0);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const int pz = q < npeer ? static_cast<int>(zp[40 + 4 * q]) : -1;
            pidx[q] = live ? (zprev == pz ? iv - 1 : iv + 1) : 0;   // the adjacent copy
            pg[q] = zp[41 + 4 * q];
            pq1[q] = zp[42 + 4 * q];
            pq2[q] = zp[43 + 4 * q];
        }
        if (valid) {
            smem[ar_ix(0, 0, i)] = a.zu_in[zg];
            smem[ar_ix(0, 1, i)] = a.zv_in[zg];
        }
        double* ser = series + static_cast<size_t>(zg) * S * 2;
        __syncthreads();
        for (int k = 0; k < a.steps; ++k) {
            if (live) {
                const double u_a = smem[ar_ix(cur, 0, i)], v_a = smem[ar_ix(cur, 1, i)];
                if (owned) *reinterpret_cast<double2*>(ser + 2 * k) = make_double2(u_a, v_a);   // layer-k air for phase 2
                const int srow = oRW + k * rw + 4 * a.n_channels;
                const int sz = srow + 3 * sidx;
                const double u_inf = smem[srow + 3 * a.n_sources + 0], v_inf = smem[srow + 3 * a.n_sources + 1];
                double du = smem[sz + 1] + smem[sz + 2] + qv1 * (u_inf * v_inf - u_a * v_a) + qv2 * (u_inf - u_a);
                double dv = smem[sz + 0] + gv * (v_inf - v_a);
                // branch-free over the maximum link/peer counts: unused slots carry zero
                // coefficients (their terms add +0), the additions keep the per-step order
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    const double pu = smem[ar_ix(cur, 0, pidx[q])], pv = smem[ar_ix(cur, 1, pidx[q])];
                    du += pq1[q] * (pu * pv - u_a * v_a) + pq2[q] * (pu - u_a);
                    dv += pg[q] * (pv - v_a);
                }
#pragma unroll
                for (int q = 0; q < NL; ++q) {
                    const double us = smem[sf_ix(cur, 0, ls[q])], vs = smem[sf_ix(cur, 1, ls[q])];
                    du += lT[q] * (us - u_a) + lM[q] * (vs - v_a);
                    dv += lD[q] * (v_a - vs);
                }
                const double nu = u_a + a.dt * (du / c0);
                const double nv = v_a + a.dt * dv;
                smem[ar_ix(cur ^ 1, 0, i)] = nu;
                smem[ar_ix(cur ^ 1, 1, i)] = nv;
                if (owned) acc |= static_cast<unsigned>(__double2hiint(nu)) | static_cast<unsigned>(__double2hiint(nv));
            }
            __syncthreads();
            cur ^= 1;
        }
        if (owned) {
            a.zu_out[zg] = smem[ar_ix(cur, 0, i)];
            a.zv_out[zg] = smem[ar_ix(cur, 1, i)];
        }
    }
    if (__syncthreads_or((acc & 0x40000000u) != 0u) && tid == 0) atomicCAS(a.stop, 0, a.seg_index + 1);
}

// ---- phase 2 ---------------------------------------------------------------------------
template <int NPT, int S>
__global__ void __launch_bounds__(32 * kRingWallWarps, 4) k_ring_walls(const RingArgs a,
                                                                      const double* __restrict__ series) {
    constexpr int N = 16 * NPT;
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ double smem[];                    // forcing rows [S][4 nch], air [warps][2 walls][S][2]
    if (launch_stopped(a.stop)) return;
    const int W = a.W, n_walls = a.n_zones * W;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int rwc = 4 * a.n_channels;
    for (int i = tid; i < a.steps * rwc; i += blockDim.x)
        smem[i] = reinterpret_cast<const double*>(a.table)[i];
    const int wl = (blockIdx.x * kRingWallWarps + warp) * 2 + lane / 16, sub = lane % 16;
    const bool live = wl < n_walls;
    const int w = live ? wl : 0;
    double* s_air = smem + S * rwc + (warp * 2 + lane / 16) * 2 * S;
    for (int i = sub; i < 2 * a.steps; i += 16) s_air[i] = series[static_cast<size_t>(w / W) * S * 2 + i];
    const bool first = sub == 0, rev = sub == 15, mirror0 = first || rev;
    const WallCoef& wc = a.coef[w];
    const double cb = wc.in.b, csu = wc.in.c_su, csv = wc.in.c_sv;
    // register 0's row: a face row in the face lanes, else the interior row,
    // whose face terms are 0 (hyg_coef.cuh)
    const RowCoef& c = first ? wc.face[0] : (rev ? wc.face[1] : wc.in);
    const double fe = c.e, fb = c.b, feg = c.e_g, fctv = c.c_tv, fcsv = c.c_sv, fctu = c.c_tu, fcsu = c.c_su,
                 fcq = c.c_q, fcg = c.c_g;
    const int ch = a.attach[2 * w].index;
    double up[NPT], uc[NPT], vp[NPT], vc[NPT];
    const size_t g0 = static_cast<size_t>(w) * N + sub * NPT;
    auto rd = [&](int f, double (&x)[NPT]) {
        double t[NPT];
#pragma unroll
        for (int q = 0; q < NPT / 2; ++q) {
            const double2 v = __ldcs(reinterpret_cast<const double2*>(a.in[f] + g0 + 2 * q));
            t[2 * q] = v.x;
            t[2 * q + 1] = v.y;
        }
#pragma unroll
        for (int q = 0; q < NPT; ++q) x[q] = rev ? t[NPT - 1 - q] : t[q];
    };
    rd(0, up);
    rd(1, uc);
    rd(2, vp);
    rd(3, vc);
    __syncthreads();                                    // rows and air staged
    unsigned acc = 0;
    auto step = [&](double (&vP)[NPT], double (&vC)[NPT], double (&uP)[NPT], double (&uC)[NPT], int k) {
        // face inputs of register 0, branch-free (wall.cpp:162-169, 177-189):
        // x = 0 the exterior channel, x = 1 the zone's layer-k air (phase 1)
        const int am = k * rwc + 4 * ch;
        const double ru = smem[am + 0], rv = smem[am + 1], rg = smem[am + 2], rq = smem[am + 3] + 0.0;
        const double au = s_air[2 * k], av = s_air[2 * k + 1];
        const double u_inf = first ? ru : au, v_inf = first ? rv : av;
        const double g_inf = first ? rg : 0.0, q_inf = first ? rq : 0.0;
        const double vs = rev ? vC[NPT - 1] : vC[0], us = rev ? uC[NPT - 1] : uC[0];
        const double vup = __shfl_up_sync(FULL, vC[NPT - 1], 1, 16);
        const double uup = __shfl_up_sync(FULL, uC[NPT - 1], 1, 16);
        const double vdn = __shfl_down_sync(FULL, vs, 1, 16);
        const double udn = __shfl_down_sync(FULL, us, 1, 16);
        const double vx0 = mirror0 ? vC[1] : vup, ux0 = mirror0 ? uC[1] : uup;
        const double vx1 = rev ? vup : vdn, ux1 = rev ? uup : udn;
#pragma unroll
        for (int q = 0; q < NPT; ++q) {
            const double vl = q == 0 ? vx0 : vC[q - 1], ul = q == 0 ? ux0 : uC[q - 1];
            const double vr = q == NPT - 1 ? vx1 : vC[q + 1], ur = q == NPT - 1 ? ux1 : uC[q + 1];
            const double d = fma(-2.0, vP[q], vl + vr);
            const double du = fma(-2.0, uP[q], ul + ur);
            double vn, un;
            if (q == 0) {
                const double t = v_inf - vP[0], tu = u_inf - uP[0];
                vn = fma(fe, t, fma(fb, d, fma(feg, g_inf, vP[0])));
                un = fma(fctv, t, fma(fcsv, d, fma(fctu, tu, fma(fcsu, du, fma(fcq, q_inf, fma(fcg, g_inf, uP[0]))))));
            } else {
                vn = fma(cb, d, vP[q]);
                un = fma(csv, d, fma(csu, du, uP[q]));
            }
            acc |= static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn));
            vP[q] = vn;
            uP[q] = un;
        }
    };
    int k = 0;
    for (; k + 1 < a.steps; k += 2) {
        step(vp, vc, up, uc, k);
        step(vc, vp, uc, up, k + 1);
    }
    if (k < a.steps) {
        step(vp, vc, up, uc, k);
#pragma unroll
        for (int q = 0; q < NPT; ++q) {
            double x = vp[q]; vp[q] = vc[q]; vc[q] = x;
            x = up[q]; up[q] = uc[q]; uc[q] = x;
        }
    }
    if (live) {
        auto wr = [&](int f, const double (&x)[NPT]) {
#pragma unroll
            for (int q = 0; q < NPT / 2; ++q) {
                const double2 v = rev ? make_double2(x[NPT - 1 - 2 * q], x[NPT - 2 - 2 * q]) : make_double2(x[2 * q], x[2 * q + 1]);
                __stcs(reinterpret_cast<double2*>(a.out[f] + g0 + 2 * q), v);
            }
        };
        wr(0, up);
        wr(1, uc);
        wr(2, vp);
        wr(3, vc);
    } else {
        acc = 0;
    }
    if (__syncthreads_or((acc & 0x40000000u) != 0u) && tid == 0) atomicCAS(a.stop, 0, a.seg_index + 1);
}

}  // namespace hyg
