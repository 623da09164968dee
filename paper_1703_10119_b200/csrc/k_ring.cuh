// k_ring.cuh — K4: temporally blocked building steps for zones in a ring
// (configs[3]: 8,192 zones x 6 constant walls x 128 nodes).
//
// Replaces S consecutive step_explicit calls (building.cpp:152-187: every wall
// advanced with layer-n zone air, every zone advanced with layer-n surface
// samples) for buildings whose walls each touch one zone on face 1 (face 0
// exterior) and whose zones exchange air only with their ring neighbours.
// The per-step path streams 48 B per node-update through HBM; here a CTA
// keeps B zones and their walls in shared memory for S steps:
//
//   * owned zones [z0, z0+B): all W walls, all n nodes, both layers of both
//     fields (in-place DF: the new layer overwrites layer n-1);
//   * halo zones at distance d = 1..S-1 on each side: only the last S+1
//     nodes of each wall (the zone-face side).  A cut wall is wrong from its
//     cut inward, one node per step, so its face node stays exact for S steps;
//     the zone air at distance d is exact through step S-d, which is all the
//     owned zones consume (the zone cone grows one zone per step);
//   * the zones at distance S only contribute their layer-0 air.
//
// HBM per launch: owned walls read + written once (64 B per node), halo
// walls read once (32 B per halo node): (64 B W n B + 32 B H) / (W n B S)
// ~ 8.5 B per update at W = 6, n = 128, B = 7, S = 8, against 48 B.
// Every owned value is exactly the value of the per-step march (same
// increment-form rows, coupled_node); a guard failure in a launch stops the
// following launches and the host replays from that launch's input with the
// exact per-step path (k_building_step).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "k_step.cuh"

namespace hyg {

struct RingArgs {
    int n_zones, W, n;             // zones, walls per zone, nodes per wall
    int B;                         // owned zones per CTA
    int steps;                     // steps of this launch (<= S)
    double norm;
    const Biot* biot;              // [2*w+k]
    const Attach* attach;
    const WallCoef* coef;          // per-wall rows for this dt (k_coupled_coef)
    const Ambient* table;          // rows of this launch: [steps][n_channels]
    int n_channels;
    const double* src;             // rows of this launch: [steps][n_sources*3 + 2]
    int n_sources;
    double dt;
    const ZoneDev* zones;
    const ZoneLinkDev* links;
    const InzLinkDev* inz;
    const double* in[4];           // up, uc, vp, vc (layer k-1, k)
    double* out[4];
    const double* zu_in;
    const double* zv_in;
    double* zu_out;
    double* zv_out;
    int* stop;                     // first failing launch + 1 (0: none)
    int seg_index;
};

template <int NPT, int S>
struct RingShape {
    static constexpr int kLanes = 16;              // threads per owned wall
    static constexpr int kPad = NPT + 1;           // padded segment (bank-conflict free)
    static constexpr int kP = S + 1;               // nodes kept per halo wall
    static constexpr int kHaloZones = 2 * (S - 1);
    static constexpr int kLocalZones = 2 * S;      // + B
    __host__ __device__ static int wall_stride() { return kLanes * kPad; }       // n = 16 NPT
    __host__ __device__ static int owned_walls(int B, int W) { return B * W; }
    __host__ __device__ static int halo_walls(int W) { return kHaloZones * W; }
    __host__ __device__ static size_t smem_bytes(int B, int W) {
        const size_t own = static_cast<size_t>(owned_walls(B, W)) * wall_stride();
        const size_t halo = static_cast<size_t>(halo_walls(W)) * kP;
        const size_t zones = static_cast<size_t>(B + kLocalZones);
        return sizeof(double) * (4 * own + 4 * halo + 4 * zones);
    }
    __host__ __device__ static int threads(int B, int W) {
        const int own = owned_walls(B, W) * kLanes;
        const int halo = (halo_walls(W) + 31) / 32 * 32;
        return own + halo + 32;   // + one zone warp (B + 2S <= 32)
    }
};

// padded position of node j inside an owned wall
template <int NPT>
__device__ __forceinline__ int ring_pos(int j) { return (j / NPT) * (NPT + 1) + (j % NPT); }

template <int NPT, int S>
__global__ void __launch_bounds__(896, 1) k_ring_tiled(const RingArgs a) {
    using Sh = RingShape<NPT, S>;
    extern __shared__ double smem[];
    if (*a.stop) return;                          // an earlier launch tripped the guard
    const int n = a.n, W = a.W, B = a.B, Z = a.n_zones;
    const int ow = Sh::owned_walls(B, W), hw = Sh::halo_walls(W);
    const int ws = Sh::wall_stride();
    const int z0 = blockIdx.x * B;
    const int nown = min(B, Z - z0);              // owned zones of this CTA (the last may own fewer)
    const int L = nown + Sh::kLocalZones;         // local zones: i = 0 .. L-1, global z0 - S + i
    constexpr int P = Sh::kP;
    // layout: owned [field u,v][slot 0,1][ow * ws], halo [field][slot][hw * P], zones [field][slot][L]
    double* OWN = smem;
    double* HAL = OWN + 4 * static_cast<size_t>(ow) * ws;
    double* ZN = HAL + 4 * static_cast<size_t>(hw) * P;
    auto own_at = [&](int f, int slot, int wl, int j) -> double& {
        return OWN[(static_cast<size_t>(f * 2 + slot) * ow + wl) * ws + ring_pos<NPT>(j)];
    };
    auto hal_at = [&](int f, int slot, int hl, int p) -> double& {
        return HAL[(static_cast<size_t>(f * 2 + slot) * hw + hl) * P + p];
    };
    auto zn_at = [&](int f, int slot, int i) -> double& { return ZN[(f * 2 + slot) * L + i]; };

    auto gzone = [&](int i) { return ((z0 - S + i) % Z + Z) % Z; };
    const int tid = threadIdx.x, nthr = blockDim.x;

    // ---- load: slot 0 = layer k-1 (prev), slot 1 = layer k (curr) --------------------
    for (int i = tid; i < ow * n; i += nthr) {
        const int wl = i / n, j = i - wl * n;
        if (wl >= nown * W) continue;
        const size_t g = (static_cast<size_t>(z0) * W + wl) * n + j;
        own_at(0, 0, wl, j) = a.in[0][g];
        own_at(0, 1, wl, j) = a.in[1][g];
        own_at(1, 0, wl, j) = a.in[2][g];
        own_at(1, 1, wl, j) = a.in[3][g];
    }
    for (int i = tid; i < hw * P; i += nthr) {
        const int hl = i / P, p = i - hl * P;
        const int hz = hl / W, wi = hl - hz * W;             // halo zone 0..2(S-1)-1
        const int li = hz < S - 1 ? 1 + hz : S + nown + (hz - (S - 1));   // its local zone index
        const size_t g = (static_cast<size_t>(gzone(li)) * W + wi) * n + (n - P + p);
        hal_at(0, 0, hl, p) = a.in[0][g];
        hal_at(0, 1, hl, p) = a.in[1][g];
        hal_at(1, 0, hl, p) = a.in[2][g];
        hal_at(1, 1, hl, p) = a.in[3][g];
    }
    for (int i = tid; i < L; i += nthr) {
        zn_at(0, 1, i) = a.zu_in[gzone(i)];
        zn_at(1, 1, i) = a.zv_in[gzone(i)];
    }
    __syncthreads();

    // ---- roles -------------------------------------------------------------------------
    const int own_thr = ow * Sh::kLanes;
    const int halo_thr = (hw + 31) / 32 * 32;
    bool bad = false;
    int cur = 1;                                   // slot holding layer k
    for (int k = 0; k < a.steps; ++k) {
        const int prv = cur ^ 1;
        const Ambient* amb = a.table + static_cast<size_t>(k) * a.n_channels;
        if (tid < own_thr) {
            // owned wall wl, nodes [s*NPT, s*NPT + NPT)
            const int wl = tid / Sh::kLanes, s = tid - wl * Sh::kLanes;
            if (wl < nown * W) {
                const int w = z0 * W + wl;
                const int li = S + wl / W;         // local zone of the wall (face 1)
                const double cb = a.coef[w].in.b, csu = a.coef[w].in.c_su, csv = a.coef[w].in.c_sv;
                const int j0 = s * NPT;
                double ul = own_at(0, cur, wl, j0 == 0 ? 1 : j0 - 1);
                double vl = own_at(1, cur, wl, j0 == 0 ? 1 : j0 - 1);
                double uc = own_at(0, cur, wl, j0), vc = own_at(1, cur, wl, j0);
#pragma unroll
                for (int q = 0; q < NPT; ++q) {
                    const int j = j0 + q;
                    const int jr = j == n - 1 ? n - 2 : j + 1;
                    const double ur = own_at(0, cur, wl, jr), vr = own_at(1, cur, wl, jr);
                    const double up = own_at(0, prv, wl, j), vp = own_at(1, prv, wl, j);
                    const double d = fma(-2.0, vp, vl + vr);
                    const double du = fma(-2.0, up, ul + ur);
                    double vn, un;
                    if (j > 0 && j < n - 1) {
                        vn = fma(cb, d, vp);
                        un = fma(csv, d, fma(csu, du, up));
                    } else {
                        // faces: x=0 exterior channel, x=1 the zone's layer-k air
                        const int f = j == 0 ? 0 : 1;
                        const RowCoef c = a.coef[w].face[f];
                        double u_inf, v_inf, g_inf = 0.0, q_inf = 0.0;
                        if (f == 0) {
                            const Ambient am = amb[a.attach[2 * w].index];
                            u_inf = am.u;
                            v_inf = am.v;
                            g_inf = am.g;
                            q_inf = am.q + 0.0;
                        } else {
                            u_inf = zn_at(0, cur, li);
                            v_inf = zn_at(1, cur, li);
                        }
                        const double t = v_inf - vp, tu = u_inf - up;
                        vn = fma(c.e, t, fma(c.b, d, fma(c.e_g, g_inf, vp)));
                        un = fma(c.c_tv, t, fma(c.c_sv, d, fma(c.c_tu, tu, fma(c.c_su, du, fma(c.c_q, q_inf,
                                                                                          fma(c.c_g, g_inf, up))))));
                    }
                    own_at(0, prv, wl, j) = un;    // layer k+1 overwrites layer k-1
                    own_at(1, prv, wl, j) = vn;
                    bad = bad || !(fabs(un) <= a.norm) || !(fabs(vn) <= a.norm);
                    ul = uc;
                    vl = vc;
                    uc = ur;
                    vc = vr;
                }
            }
        } else if (tid < own_thr + halo_thr) {
            const int hl = tid - own_thr;
            if (hl < hw) {
                // halo wall: global nodes n-P .. n-1; the cut end (p = 0) has no
                // left neighbour — its error moves inward one node per step and
                // never reaches the face node within S steps
                const int hz = hl / W, wi = hl - hz * W;
                const int li = hz < S - 1 ? 1 + hz : S + nown + (hz - (S - 1));
                const int w = gzone(li) * W + wi;
                const double cb = a.coef[w].in.b, csu = a.coef[w].in.c_su, csv = a.coef[w].in.c_sv;
                double ul = hal_at(0, cur, hl, 0), vl = hal_at(1, cur, hl, 0);
                double uc = ul, vc = vl;
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const int pr = p == P - 1 ? P - 2 : p + 1;
                    const double ur = hal_at(0, cur, hl, pr), vr = hal_at(1, cur, hl, pr);
                    const double up = hal_at(0, prv, hl, p), vp = hal_at(1, prv, hl, p);
                    const double d = fma(-2.0, vp, vl + vr);
                    const double du = fma(-2.0, up, ul + ur);
                    double vn, un;
                    if (p < P - 1) {
                        vn = fma(cb, d, vp);
                        un = fma(csv, d, fma(csu, du, up));
                    } else {
                        const RowCoef c = a.coef[w].face[1];
                        const double t = zn_at(1, cur, li) - vp, tu = zn_at(0, cur, li) - up;
                        vn = fma(c.e, t, fma(c.b, d, fma(c.e_g, 0.0, vp)));
                        un = fma(c.c_tv, t, fma(c.c_sv, d, fma(c.c_tu, tu, fma(c.c_su, du, fma(c.c_q, 0.0,
                                                                                          fma(c.c_g, 0.0, up))))));
                    }
                    hal_at(0, prv, hl, p) = un;
                    hal_at(1, prv, hl, p) = vn;
                    ul = uc;
                    vl = vc;
                    uc = ur;
                    vc = vr;
                }
            }
        } else {
            // zone warp: zone_step_explicit (zone.cpp:69-74) of every local zone
            // that has a layer-k state and samples (i = 1 .. L-2)
            const int i = tid - own_thr - halo_thr;
            if (i >= 1 && i < L - 1) {
                const int z = gzone(i);
                const ZoneDev d = a.zones[z];
                const double u_a = zn_at(0, cur, i), v_a = zn_at(1, cur, i);
                const double* srow = a.src + static_cast<size_t>(k) * (3 * a.n_sources + 2);
                const double* sz = srow + 3 * d.sources;
                const double u_inf = srow[3 * a.n_sources + 0], v_inf = srow[3 * a.n_sources + 1];
                double du = sz[1] + sz[2] + d.q_v1 * (u_inf * v_inf - u_a * v_a) + d.q_v2 * (u_inf - u_a);
                double dv = sz[0] + d.g_v * (v_inf - v_a);
                for (int q = d.inz_begin; q < d.inz_end; ++q) {
                    const InzLinkDev l = a.inz[q];
                    const int pi = gzone(i - 1) == l.peer ? i - 1 : i + 1;   // the adjacent copy
                    const double pu = zn_at(0, cur, pi), pv = zn_at(1, cur, pi);
                    du += l.q_inz1 * (pu * pv - u_a * v_a) + l.q_inz2 * (pu - u_a);
                    dv += l.g_inz * (pv - v_a);
                }
                const bool owned = i >= S && i < S + nown;
                const int hz = i < S ? i - 1 : (S - 1) + (i - S - nown);
                for (int q = d.wall_begin; q < d.wall_end; ++q) {
                    const ZoneLinkDev l = a.links[q];
                    const int wi = l.wall - z * W;
                    const double us = owned ? own_at(0, cur, (i - S) * W + wi, n - 1)
                                            : hal_at(0, cur, hz * W + wi, P - 1);
                    const double vs = owned ? own_at(1, cur, (i - S) * W + wi, n - 1)
                                            : hal_at(1, cur, hz * W + wi, P - 1);
                    du += l.Bi_TT * l.theta_T * (us - u_a) + l.Bi_TM * l.theta_T * (vs - v_a);
                    dv += d.sign * l.Bi_M * l.theta_M * (v_a - vs);
                }
                const double nu = u_a + a.dt * (du / (1.0 + d.kappa_a_tt1));
                const double nv = v_a + a.dt * dv;
                zn_at(0, cur ^ 1, i) = nu;
                zn_at(1, cur ^ 1, i) = nv;
                if (owned) bad = bad || !isfinite(nu) || !isfinite(nv) || fabs(nu) > a.norm || fabs(nv) > a.norm;
            }
        }
        __syncthreads();
        cur ^= 1;
    }

    // ---- guard + store: out = (layer k+S-1, layer k+S) ------------------------------------
    if (__syncthreads_or(bad)) {
        if (tid == 0) atomicCAS(a.stop, 0, a.seg_index + 1);
        return;
    }
    const int prv = cur ^ 1;
    for (int i = tid; i < nown * W * n; i += nthr) {
        const int wl = i / n, j = i - wl * n;
        const size_t g = (static_cast<size_t>(z0) * W + wl) * n + j;
        a.out[0][g] = own_at(0, prv, wl, j);
        a.out[1][g] = own_at(0, cur, wl, j);
        a.out[2][g] = own_at(1, prv, wl, j);
        a.out[3][g] = own_at(1, cur, wl, j);
    }
    for (int i = tid; i < nown; i += nthr) {
        a.zu_out[z0 + i] = zn_at(0, cur, S + i);
        a.zv_out[z0 + i] = zn_at(1, cur, S + i);
    }
}

}  // namespace hyg
