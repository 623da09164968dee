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
    const double* zparams;         // K4r: per-zone parameter blocks [n_zones][kRingZP]
    const double* in[4];           // up, uc, vp, vc (layer k-1, k)
    double* out[4];
    const double* zu_in;
    const double* zv_in;
    double* zu_out;
    double* zv_out;
    int* stop;                     // first failing launch + 1 (0: none)
    int seg_index;
    int dbg_skip;                  // timing experiments only (K5: 1 skip halo copies); 0 in the library
};

// Per local zone, staged in shared memory before the step loop (the zone
// warp's inputs, folded exactly as zone_update multiplies them):
//   [0] 1 + kappa_a_tt1, [1] g_v, [2] q_v1, [3] q_v2, [4] #links, [5] #peers,
//   [6] source index, links [8 + 4q] = (wall in zone, Bi_TT theta_T,
//   Bi_TM theta_T, sign Bi_M theta_M), peers [40 + 4q] = (local index,
//   g_inz, q_inz1, q_inz2)
constexpr int kRingMaxLinks = 8, kRingMaxPeers = 4, kRingZP = 56;
constexpr int kRingFace = 9;        // face row: e, b, e_g, c_tv, c_sv, c_tu, c_su, c_q, c_g

template <int NPT, int S>
struct RingShape {
    static constexpr int kLanes = 16;              // threads per owned wall (n = 16 NPT)
    static constexpr int kP = S + 1;               // nodes kept per halo wall
    static constexpr int kHaloZones = 2 * (S - 1);
    static constexpr int kLocalZones = 2 * S;      // + B
    __host__ __device__ static int owned_walls(int B, int W) { return B * W; }
    __host__ __device__ static int halo_walls(int W) { return kHaloZones * W; }
    __host__ __device__ static int row_width(int nch, int nsrc) { return 4 * nch + 3 * nsrc + 2; }
    __host__ __device__ static size_t smem_bytes(int B, int W, int nch, int nsrc) {
        const size_t n = 16 * NPT;
        const size_t own = static_cast<size_t>(owned_walls(B, W)) * n;
        const size_t halo = static_cast<size_t>(halo_walls(W)) * kP;
        const size_t zones = static_cast<size_t>(B + kLocalZones);
        return sizeof(double) * (4 * own + 4 * halo + 4 * zones + zones * kRingZP +
                                 static_cast<size_t>(owned_walls(B, W)) * 2 * kRingFace +
                                 static_cast<size_t>(S) * row_width(nch, nsrc));
    }
    // roles are whole warps (bar.sync from two call sites inside one warp is unsafe)
    __host__ __device__ static int own_threads(int B, int W) { return (owned_walls(B, W) * kLanes + 31) / 32 * 32; }
    __host__ __device__ static int halo_threads(int W) { return (halo_walls(W) + 31) / 32 * 32; }
    __host__ __device__ static int threads(int B, int W) {
        return own_threads(B, W) + halo_threads(W) + 32;   // + one zone warp (B + 2S <= 32)
    }
};

// Ampere-style asynchronous global -> shared copies: every thread issues all
// of its copies before one wait, so the load phase keeps the whole tile in
// flight instead of one register round trip per element.
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// position of node j inside an owned wall: segments of NPT nodes, the node
// index XOR-swizzled per segment so the 16 lanes of a wall (one segment each)
// hit 16 distinct bank pairs
template <int NPT>
__device__ __forceinline__ int ring_pos(int j) {
    const int s = j / NPT, q = j % NPT;
    return s * NPT + (q ^ ((s / (16 / NPT)) & (NPT - 1)));
}

template <int NPT, int S>
__global__ void __launch_bounds__(896, 1) k_ring_tiled(const RingArgs a) {
    using Sh = RingShape<NPT, S>;
    extern __shared__ double smem[];
    if (launch_stopped(a.stop)) return;                          // an earlier launch tripped the guard
    const int n = a.n, W = a.W, B = a.B, Z = a.n_zones;
    const int ow = Sh::owned_walls(B, W), hw = Sh::halo_walls(W);
    const int z0 = blockIdx.x * B;
    const int nown = min(B, Z - z0);              // owned zones of this CTA (the last may own fewer)
    const int L = nown + Sh::kLocalZones;         // local zones: i = 0 .. L-1, global z0 - S + i
    const int LB = B + Sh::kLocalZones;           // allocated local zones
    const int rw = Sh::row_width(a.n_channels, a.n_sources);
    constexpr int P = Sh::kP;
    // layout: owned [field u,v][slot 0,1][ow * n], halo [field][slot][hw * P],
    // zones [field][slot][LB], zone params [LB][kRingZP], face rows [ow][2][9], rows [S][rw]
    // every access is smem[integer offset] (shared-space loads/stores, never generic)
    const int oOWN = 0;
    const int oHAL = oOWN + 4 * ow * n;
    const int oZN = oHAL + 4 * hw * P;
    const int oZP = oZN + 4 * LB;
    const int oFC = oZP + LB * kRingZP;
    const int oRW = oFC + ow * 2 * kRingFace;
    auto own_ix = [&](int f, int slot, int wl, int j) { return oOWN + ((f * 2 + slot) * ow + wl) * n + ring_pos<NPT>(j); };
    auto hal_ix = [&](int f, int slot, int hl, int p) { return oHAL + ((f * 2 + slot) * hw + hl) * P + p; };
    auto zn_ix = [&](int f, int slot, int i) { return oZN + (f * 2 + slot) * LB + i; };

    auto gzone = [&](int i) { return ((z0 - S + i) % Z + Z) % Z; };
    const int tid = threadIdx.x, nthr = blockDim.x;

    // ---- load: slot 0 = layer k-1 (prev), slot 1 = layer k (curr) --------------------
    for (int i = tid; i < nown * W * n; i += nthr) {
        const int wl = i / n, j = i - wl * n;
        const size_t g = (static_cast<size_t>(z0) * W + wl) * n + j;
        cp_async8(&smem[own_ix(0, 0, wl, j)], a.in[0] + g);
        cp_async8(&smem[own_ix(0, 1, wl, j)], a.in[1] + g);
        cp_async8(&smem[own_ix(1, 0, wl, j)], a.in[2] + g);
        cp_async8(&smem[own_ix(1, 1, wl, j)], a.in[3] + g);
    }
    for (int i = tid; i < hw * P; i += nthr) {
        const int hl = i / P, p = i - hl * P;
        const int hz = hl / W, wi = hl - hz * W;             // halo zone 0..2(S-1)-1
        const int li = hz < S - 1 ? 1 + hz : S + nown + (hz - (S - 1));   // its local zone index
        const size_t g = (static_cast<size_t>(gzone(li)) * W + wi) * n + (n - P + p);
        cp_async8(&smem[hal_ix(0, 0, hl, p)], a.in[0] + g);
        cp_async8(&smem[hal_ix(0, 1, hl, p)], a.in[1] + g);
        cp_async8(&smem[hal_ix(1, 0, hl, p)], a.in[2] + g);
        cp_async8(&smem[hal_ix(1, 1, hl, p)], a.in[3] + g);
    }
    for (int i = tid; i < nown * W * 2; i += nthr) {         // face rows of the owned walls
        const int wl = i / 2, f = i - wl * 2;
        const RowCoef c = a.coef[z0 * W + wl].face[f];
        const int d = oFC + i * kRingFace;
        smem[d + 0] = c.e; smem[d + 1] = c.b; smem[d + 2] = c.e_g; smem[d + 3] = c.c_tv; smem[d + 4] = c.c_sv;
        smem[d + 5] = c.c_tu; smem[d + 6] = c.c_su; smem[d + 7] = c.c_q; smem[d + 8] = c.c_g;
    }
    for (int i = tid; i < a.steps * rw; i += nthr) {         // forcing rows of this launch
        const int k = i / rw, r = i - k * rw;
        smem[oRW + i] = r < 4 * a.n_channels
                    ? reinterpret_cast<const double*>(a.table + static_cast<size_t>(k) * a.n_channels)[r]
                    : a.src[static_cast<size_t>(k) * (3 * a.n_sources + 2) + (r - 4 * a.n_channels)];
    }
    for (int i = tid; i < L; i += nthr) {
        const int z = gzone(i);
        smem[zn_ix(0, 1, i)] = a.zu_in[z];
        smem[zn_ix(1, 1, i)] = a.zv_in[z];
        const ZoneDev d = a.zones[z];
        double* zp = &smem[oZP + i * kRingZP];
        zp[0] = 1.0 + d.kappa_a_tt1;
        zp[1] = d.g_v;
        zp[2] = d.q_v1;
        zp[3] = d.q_v2;
        zp[4] = d.wall_end - d.wall_begin;
        zp[5] = d.inz_end - d.inz_begin;
        zp[6] = d.sources;
        for (int q = 0; q < d.wall_end - d.wall_begin; ++q) {
            const ZoneLinkDev l = a.links[d.wall_begin + q];
            zp[8 + 4 * q] = l.wall - z * W;
            zp[9 + 4 * q] = l.Bi_TT * l.theta_T;
            zp[10 + 4 * q] = l.Bi_TM * l.theta_T;
            zp[11 + 4 * q] = d.sign * l.Bi_M * l.theta_M;
        }
        for (int q = 0; q < d.inz_end - d.inz_begin; ++q) {
            const InzLinkDev l = a.inz[d.inz_begin + q];
            const int pi = i >= 1 && gzone(i - 1) == l.peer ? i - 1 : i + 1;   // the adjacent copy
            zp[40 + 4 * q] = pi;
            zp[41 + 4 * q] = l.g_inz;
            zp[42 + 4 * q] = l.q_inz1;
            zp[43 + 4 * q] = l.q_inz2;
        }
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- roles -------------------------------------------------------------------------
    const int own_thr = Sh::own_threads(B, W);
    const int halo_thr = Sh::halo_threads(W);
    bool bad = false;
    int cur = 1;                                   // slot holding layer k
    if (tid < own_thr) {
        // owned wall wl, nodes [s*NPT, s*NPT + NPT)
        const int wl = tid / Sh::kLanes, s = tid - wl * Sh::kLanes;
        const bool live = wl < nown * W;            // (the rounding lanes of the last warp idle)
        const int w = z0 * W + (live ? wl : 0);
        const int li = S + wl / W;                 // local zone of the wall (face 1)
        const double cb = a.coef[w].in.b, csu = a.coef[w].in.c_su, csv = a.coef[w].in.c_sv;
        const int ch = a.attach[2 * w].index;
        const int j0 = s * NPT;
        // this wall's four shared rows and the swizzled offsets of the thread's nodes
        const int U0 = oOWN + (0 * ow + wl) * n, U1 = oOWN + (1 * ow + wl) * n;
        const int V0 = oOWN + (2 * ow + wl) * n, V1 = oOWN + (3 * ow + wl) * n;
        const int g = (s / (16 / NPT)) & (NPT - 1);
        const int base = s * NPT;
        const int left = j0 == 0 ? ring_pos<NPT>(1) : ring_pos<NPT>(j0 - 1);
        const int right = j0 + NPT - 1 == n - 1 ? ring_pos<NPT>(n - 2) : ring_pos<NPT>(j0 + NPT);
        const int fc0 = oFC + (wl * 2 + 0) * kRingFace, fc1 = fc0 + kRingFace;
        for (int k = 0; k < a.steps; ++k) {
            if (live) {
                const int uc_ = cur ? U1 : U0, vc_ = cur ? V1 : V0;
                const int up_ = cur ? U0 : U1, vp_ = cur ? V0 : V1;
                double ul = smem[uc_ + left], vl = smem[vc_ + left];
                double uc = smem[uc_ + base + (0 ^ g)], vc = smem[vc_ + base + (0 ^ g)];
#pragma unroll
                for (int q = 0; q < NPT; ++q) {
                    const int j = j0 + q;
                    const int pq = base + (q ^ g);
                    const int pr = q == NPT - 1 ? right : base + ((q + 1) ^ g);
                    const double ur = smem[uc_ + pr], vr = smem[vc_ + pr];
                    const double up = smem[up_ + pq], vp = smem[vp_ + pq];
                    const double d = fma(-2.0, vp, vl + vr);
                    const double du = fma(-2.0, up, ul + ur);
                    double vn, un;
                    if (j > 0 && j < n - 1) {
                        vn = fma(cb, d, vp);
                        un = fma(csv, d, fma(csu, du, up));
                    } else {
                        // faces (coupled_node): x=0 the exterior channel, x=1 the zone's layer-k air
                        const int c = j == 0 ? fc0 : fc1;
                        double u_inf, v_inf, g_inf = 0.0, q_inf = 0.0;
                        if (j == 0) {
                            const int am = oRW + k * rw + 4 * ch;
                            u_inf = smem[am + 0];
                            v_inf = smem[am + 1];
                            g_inf = smem[am + 2];
                            q_inf = smem[am + 3] + 0.0;
                        } else {
                            u_inf = smem[zn_ix(0, cur, li)];
                            v_inf = smem[zn_ix(1, cur, li)];
                        }
                        const double t = v_inf - vp, tu = u_inf - up;
                        vn = fma(smem[c + 0], t, fma(smem[c + 1], d, fma(smem[c + 2], g_inf, vp)));
                        un = fma(smem[c + 3], t, fma(smem[c + 4], d, fma(smem[c + 5], tu, fma(smem[c + 6], du,
                                 fma(smem[c + 7], q_inf, fma(smem[c + 8], g_inf, up))))));
                    }
                    smem[up_ + pq] = un;            // layer k+1 overwrites layer k-1
                    smem[vp_ + pq] = vn;
                    bad = bad || !(fabs(un) <= a.norm) || !(fabs(vn) <= a.norm);
                    ul = uc;
                    vl = vc;
                    uc = ur;
                    vc = vr;
                }
            }
            __syncthreads();
            cur ^= 1;
        }
    } else if (tid < own_thr + halo_thr) {
        // halo wall: global nodes n-P .. n-1; the cut end (p = 0) has no left
        // neighbour — its error moves inward one node per step and never
        // reaches the face node within S steps
        const int hl = tid - own_thr;
        const bool live = hl < hw;
        const int hz = (live ? hl : 0) / W, wi = (live ? hl : 0) - hz * W;
        const int li = hz < S - 1 ? 1 + hz : S + nown + (hz - (S - 1));
        const int w = gzone(li) * W + wi;
        const double cb = a.coef[w].in.b, csu = a.coef[w].in.c_su, csv = a.coef[w].in.c_sv;
        const RowCoef c = a.coef[w].face[1];
        for (int k = 0; k < a.steps; ++k) {
            const int prv = cur ^ 1;
            if (live) {
                const int hu = hal_ix(0, cur, hl, 0), hv = hal_ix(1, cur, hl, 0);
                const int hpu = hal_ix(0, prv, hl, 0), hpv = hal_ix(1, prv, hl, 0);
                double ul = smem[hu], vl = smem[hv];
                double uc = ul, vc = vl;
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const int pr = p == P - 1 ? P - 2 : p + 1;
                    const double ur = smem[hu + pr], vr = smem[hv + pr];
                    const double up = smem[hpu + p], vp = smem[hpv + p];
                    const double d = fma(-2.0, vp, vl + vr);
                    const double du = fma(-2.0, up, ul + ur);
                    double vn, un;
                    if (p < P - 1) {
                        vn = fma(cb, d, vp);
                        un = fma(csv, d, fma(csu, du, up));
                    } else {
                        const double t = smem[zn_ix(1, cur, li)] - vp, tu = smem[zn_ix(0, cur, li)] - up;
                        vn = fma(c.e, t, fma(c.b, d, fma(c.e_g, 0.0, vp)));
                        un = fma(c.c_tv, t, fma(c.c_sv, d, fma(c.c_tu, tu, fma(c.c_su, du, fma(c.c_q, 0.0,
                                                                                          fma(c.c_g, 0.0, up))))));
                    }
                    smem[hpu + p] = un;
                    smem[hpv + p] = vn;
                    ul = uc;
                    vl = vc;
                    uc = ur;
                    vc = vr;
                }
            }
            __syncthreads();
            cur ^= 1;
        }
    } else {
        // zone warp: zone_step_explicit (zone.cpp:69-74) of every local zone
        // with a layer-k state and samples (i = 1 .. L-2), from staged params
        const int i = tid - own_thr - halo_thr;
        const bool live = i >= 1 && i < L - 1;
        const int zp = oZP + (live ? i : 0) * kRingZP;
        const bool owned = i >= S && i < S + nown;
        const int hz = i < S ? i - 1 : (S - 1) + (i - S - nown);
        for (int k = 0; k < a.steps; ++k) {
            if (live) {
                const double u_a = smem[zn_ix(0, cur, i)], v_a = smem[zn_ix(1, cur, i)];
                const int srow = oRW + k * rw + 4 * a.n_channels;
                const int sz = srow + 3 * static_cast<int>(smem[zp + 6]);
                const double u_inf = smem[srow + 3 * a.n_sources + 0], v_inf = smem[srow + 3 * a.n_sources + 1];
                double du = smem[sz + 1] + smem[sz + 2] + smem[zp + 2] * (u_inf * v_inf - u_a * v_a) +
                            smem[zp + 3] * (u_inf - u_a);
                double dv = smem[sz + 0] + smem[zp + 1] * (v_inf - v_a);
                const int npeer = static_cast<int>(smem[zp + 5]), nlink = static_cast<int>(smem[zp + 4]);
                for (int q = 0; q < npeer; ++q) {
                    const int pi = static_cast<int>(smem[zp + 40 + 4 * q]);
                    const double pu = smem[zn_ix(0, cur, pi)], pv = smem[zn_ix(1, cur, pi)];
                    du += smem[zp + 42 + 4 * q] * (pu * pv - u_a * v_a) + smem[zp + 43 + 4 * q] * (pu - u_a);
                    dv += smem[zp + 41 + 4 * q] * (pv - v_a);
                }
                for (int q = 0; q < nlink; ++q) {
                    const int wi = static_cast<int>(smem[zp + 8 + 4 * q]);
                    const int iu = owned ? own_ix(0, cur, (i - S) * W + wi, n - 1) : hal_ix(0, cur, hz * W + wi, P - 1);
                    const int iv = owned ? own_ix(1, cur, (i - S) * W + wi, n - 1) : hal_ix(1, cur, hz * W + wi, P - 1);
                    const double us = smem[iu], vs = smem[iv];
                    du += smem[zp + 9 + 4 * q] * (us - u_a) + smem[zp + 10 + 4 * q] * (vs - v_a);
                    dv += smem[zp + 11 + 4 * q] * (v_a - vs);
                }
                const double nu = u_a + a.dt * (du / smem[zp + 0]);
                const double nv = v_a + a.dt * dv;
                smem[zn_ix(0, cur ^ 1, i)] = nu;
                smem[zn_ix(1, cur ^ 1, i)] = nv;
                if (owned) bad = bad || !isfinite(nu) || !isfinite(nv) || fabs(nu) > a.norm || fabs(nv) > a.norm;
            }
            __syncthreads();
            cur ^= 1;
        }
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
        a.out[0][g] = smem[own_ix(0, prv, wl, j)];
        a.out[1][g] = smem[own_ix(0, cur, wl, j)];
        a.out[2][g] = smem[own_ix(1, prv, wl, j)];
        a.out[3][g] = smem[own_ix(1, cur, wl, j)];
    }
    for (int i = tid; i < nown; i += nthr) {
        a.zu_out[z0 + i] = smem[zn_ix(0, cur, S + i)];
        a.zv_out[z0 + i] = smem[zn_ix(1, cur, S + i)];
    }
}

}  // namespace hyg
