// k_ring_reg.cuh — K4r: the zone-ring temporal blocking of K4 (k_ring.cuh)
// with the owned walls in registers and a persistent, prefetching CTA
// (configs[3]: 8,192 zones x 6 constant walls x 128 nodes).
//
// Replaces S consecutive step_explicit calls (building.cpp:152-187) exactly as
// K4 does — same decomposition, same rows, same zone arithmetic — but:
//   * owned walls: K1's layout (k_coupled.cuh): 16 lanes x NPT nodes per wall,
//     two walls per warp, the four layers in registers, neighbours by shuffles,
//     the last lane reversed so both faces sit in register 0 (face 0: the
//     exterior channel, face 1: the wall's zone air of the current layer);
//   * halo walls (the last S+1 nodes of the walls of the S-1 zones on each
//     side, cut end stale one node per step) and the zone air ODEs: one thread
//     per halo wall (its S+1 nodes in registers) and one per local zone;
//   * one barrier per step: surface samples and zone air go through two small
//     shared arrays double-buffered by step parity;
//   * persistent: a CTA walks the zone blocks blockIdx.x, +gridDim.x, ... and
//     while it marches one block in registers, the next block's owned walls
//     arrive in a shared staging buffer by four 1-D bulk copies (TMA engine,
//     one contiguous range per field, completion on an mbarrier), its halo
//     walls, zone parameter blocks and zone air by cp.async (the load leaves
//     the step loop's critical path); results leave through per-warp scratch
//     and TMA bulk stores.  Staging reads and scratch writes start each lane
//     at a rotated 16-byte pair, so quarter warps hit distinct banks.
//     (Staging the row coefficients with the prefetch instead of loading them
//     per block measured slower: 2.68e11 vs 3.14e11.)
// Guard: K1's fast guard (bit 30 of the high word: |x| >= 2 or not finite) over
// the owned walls and zones; a set bit stops the following launches and the
// host replays from the flagged launch with K4, whose exact guard reports the
// reference's first failing layer.  Used for divergence_norm >= 2 only.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "k_ring.cuh"

// timing experiments only (tools/ring_step_probe.py): skip the arithmetic of
// roles (1 halo, 2 zone, 4 owned), the owned walls' outputs (8), their bulk
// loads (16), the other prefetches (32); 0 in the library
#ifndef RING_VSTORE
#define RING_VSTORE 0
#endif
#ifndef RING_SKIP
#define RING_SKIP 0
#endif
// timing experiments only: per-phase clock64 stamps of CTA 0 (owned warp 0,
// the zone warp) into g_ring_prof[block iteration][event]; 0 in the library
#ifndef RING_PROF
#define RING_PROF 0
#endif
#if RING_PROF
__device__ unsigned long long g_ring_prof[32 * 16];
#define RPROF(e) do { if (blockIdx.x == 0 && tid == 0 && it < 32) g_ring_prof[it * 16 + (e)] = clock64(); } while (0)
#define ZPROF(e) do { if (blockIdx.x == 0 && tid == 32 * (own_w + halo_w) && it < 32) g_ring_prof[it * 16 + 10 + (e)] = clock64(); } while (0)
#else
#define RPROF(e) do { } while (0)
#define ZPROF(e) do { } while (0)
#endif

namespace hyg {

// K4r CTA size cap: 16 warps (12 owned + 3 halo + 1 zone at B = 4, W = 6, S = 8),
// 128 registers per thread (ptxas sizes registers for whole 4-warp groups)
#ifndef HYG_RING_REG_THREADS
#define HYG_RING_REG_THREADS 512
#endif
constexpr int kRingRegThreads = HYG_RING_REG_THREADS;

template <int NPT, int S>
struct RingRegShape {
    static constexpr int kP = S + 1;                           // nodes kept per halo wall
    static constexpr int kPS = (kP + 1) & ~1;                   // their staging slot (even: 16-byte copies)
    static constexpr int kHaloZones = 2 * (S - 1);
    // shared stride of a zone's parameter block: odd, so the zone warp's lanes
    // (one zone each) read distinct banks (56 put every lane on two banks)
    static constexpr int kZPS = kRingZP + 1;
    __host__ __device__ static int own_warps(int B, int W) { return (B * W + 1) / 2; }
    __host__ __device__ static int halo_walls(int W) { return kHaloZones * W; }
    __host__ __device__ static int halo_warps(int W) { return (halo_walls(W) + 31) / 32; }
    __host__ __device__ static int threads(int B, int W) { return 32 * (own_warps(B, W) + halo_warps(W) + 1); }
    __host__ __device__ static int local_zones(int B) { return B + 2 * S; }
    // doubles: staging of the owned walls (one bulk copy per field) and of the
    // halo walls, of the zone parameters and zone air (double-buffered by block
    // parity), the per-step surfaces [2][2][B W + halo] and zone air
    // [2][2][local], forcing rows, the mbarrier of the owned-wall copies, and
    // per owned warp an output scratch [2 fields][2 walls][n] for its bulk stores
    __host__ __device__ static size_t smem_doubles(int B, int W, int n, int rw) {
        const size_t LB = local_zones(B);
        return static_cast<size_t>(4) * B * W * n + static_cast<size_t>(4) * halo_walls(W) * kPS +
               2 * LB * kZPS + 4 * LB + 4 * static_cast<size_t>(B * W + halo_walls(W)) + 4 * LB +
               ((static_cast<size_t>(S) * rw + 1) & ~static_cast<size_t>(1)) + 2 +
               static_cast<size_t>(own_warps(B, W)) * 2 * 2 * n;
    }
};

// 1-D bulk copies (TMA engine) and their mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(void* mb, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(void* mb, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(void* mb, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n RING_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra RING_WAIT_%=;\n}\n" ::"r"(smem_u32(mb)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, void* mb) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(mb))
                 : "memory");
}

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void cp_async16(double* smem_dst, const double* gsrc) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc));
}

// NL, NP: link and peer slots walked per zone (compile-time, branch-free; the
// host picks the smallest instantiation that covers every zone)
template <int NPT, int S, int NL = kRingMaxLinks, int NP = kRingMaxPeers>
__global__ void __launch_bounds__(kRingRegThreads, 1) k_ring_reg(const RingArgs a) {
    using Sh = RingRegShape<NPT, S>;
    constexpr int P = Sh::kP, PS = Sh::kPS, N = 16 * NPT;
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ double smem[];
    if (launch_stopped(a.stop)) return;
    const int W = a.W, B = a.B, Z = a.n_zones;
    const int OW = B * W, HW = Sh::halo_walls(W), LB = Sh::local_zones(B);
    const int rw = RingShape<NPT, S>::row_width(a.n_channels, a.n_sources);
    // shared layout (integer offsets; every access a shared-space access)
    const int oSO = 0;                                  // staging owned [4][OW][N] (linear: bulk copies)
    const int oSH = oSO + 4 * OW * N;                   // staging halo [4][HW][PS] (last PS nodes)
    constexpr int ZPS = Sh::kZPS;
    const int oZS = oSH + 4 * HW * PS;                  // staged zone parameters [2][LB][ZPS]
    const int oZA = oZS + 2 * LB * ZPS;                 // staged zone air [2][2][LB]
    const int oSF = oZA + 4 * LB;                       // surfaces [parity][field][OW + HW]
    const int oAR = oSF + 4 * (OW + HW);                // zone air [parity][field][LB]
    const int oRW = oAR + 4 * LB;                       // forcing rows [S][rw]
    const int oMB = oRW + ((S * rw + 1) & ~1);          // mbarrier of the owned-wall bulk copies (16-byte aligned)
    const int oOUT = oMB + 2;                           // output scratch [own warps][2][2 N] (16-byte aligned)
    void* mbar = &smem[oMB];
    auto so_ix = [&](int f, int i) { return oSO + f * OW * N + i; };
    // surfaces: slot of owned wall (zone z, wall q) = q B + z, of halo wall
    // (halo zone h, wall q) = OW + q HZ + h: the zone warp's lanes (one zone
    // each) read consecutive slots
    constexpr int HZ = Sh::kHaloZones;
    auto sf_ix = [&](int par, int f, int i) { return oSF + (par * 2 + f) * (OW + HW) + i; };
    auto own_slot = [&](int wl) { const int z = wl / W; return (wl - z * W) * B + z; };
    auto halo_slot = [&](int hl) { const int h = hl / W; return OW + (hl - h * W) * HZ + h; };
    auto ar_ix = [&](int par, int f, int i) { return oAR + (par * 2 + f) * LB + i; };
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int nblk = (Z + B - 1) / B;

    for (int i = tid; i < a.steps * rw; i += nthr) {    // forcing rows of this launch (all blocks), asynchronous
        const int k = i / rw, r = i - k * rw;
        cp_async8(&smem[oRW + i],
                  r < 4 * a.n_channels
                      ? reinterpret_cast<const double*>(a.table + static_cast<size_t>(k) * a.n_channels) + r
                      : a.src + static_cast<size_t>(k) * (3 * a.n_sources + 2) + (r - 4 * a.n_channels));
    }
    // global zone of local zone i; rings with Z >= B + 3 S wrap by one add (no division)
    const bool wide = Z >= B + 3 * S;
    auto gz = [&](int z0, int i) {
        int g = z0 - S + i;
        if (wide) {
            g += g < 0 ? Z : 0;
            return g >= Z ? g - Z : g;
        }
        return (g % Z + Z) % Z;
    };
    auto halo_local = [&](int hz, int nown) { return hz < S - 1 ? 1 + hz : S + nown + (hz - (S - 1)); };
    // prefetch of block b (zone parameters and air into parity par)
    auto prefetch = [&](int b, int par) {
        const int z0 = b * B, nown = min(B, Z - z0), L = nown + 2 * S;
        if (tid == 0) {   // the owned walls of the block: one contiguous range per field
            const unsigned bytes = (RING_SKIP & 16) ? 0u : static_cast<unsigned>(nown * W * N * sizeof(double));
            mbar_expect_tx(mbar, 4 * bytes);
#pragma unroll
            for (int f = 0; f < 4 * !(RING_SKIP & 16); ++f)
                bulk_g2s(&smem[so_ix(f, 0)], a.in[f] + static_cast<size_t>(z0) * W * N, bytes, mbar);
        }
        if (RING_SKIP & 32) {
            asm volatile("cp.async.commit_group;\n" ::);
            return;
        }
        for (int i = tid; i < HW * (PS / 2); i += nthr) {   // the last PS nodes, 16-byte pieces
            const int hl = i / (PS / 2), c = i - hl * (PS / 2);
            const int hz = hl / W, wi = hl - hz * W;
            const size_t g = (static_cast<size_t>(gz(z0, halo_local(hz, nown))) * W + wi) * N + (N - PS) + 2 * c;
#pragma unroll
            for (int f = 0; f < 4; ++f) cp_async16(&smem[oSH + (f * HW + hl) * PS + 2 * c], a.in[f] + g);
        }
        for (int i = tid; i < L * kRingZP; i += nthr) {
            const int li = i / kRingZP, c = i - li * kRingZP;
            cp_async8(&smem[oZS + (par * LB + li) * ZPS + c], a.zparams + static_cast<size_t>(gz(z0, li)) * kRingZP + c);
        }
        for (int i = tid; i < 2 * L; i += nthr) {
            const int f = i / L, li = i - f * L;
            cp_async8(&smem[oZA + (par * 2 + f) * LB + li], (f ? a.zv_in : a.zu_in) + gz(z0, li));
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    if (tid == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (static_cast<int>(blockIdx.x) < nblk) prefetch(blockIdx.x, 0);

    // ---- roles ------------------------------------------------------------------------
    const int warp = tid / 32, lane = tid % 32;
    const int own_w = Sh::own_warps(B, W), halo_w = Sh::halo_warps(W);
    const bool is_own = warp < own_w, is_halo = !is_own && warp < own_w + halo_w;
    unsigned acc = 0;

    // role coefficients of block bb: owned: interior (3) + register 0's face-capable
    // row (9) + channel; halo: interior (3) + face 1 (9).  Loaded one block
    // ahead (block b+1's right after block b's steps, while the owned warps
    // write their outputs), so the latency of these scattered loads is hidden
    double cf[12];
    int ch = 0;
    auto load_cf = [&](int bb) {
        const int z0 = bb * B, nown = min(B, Z - z0);
        if (is_own) {
            const int wl = warp * 2 + lane / 16, sub = lane % 16;
            const int w = z0 * W + (wl < nown * W ? wl : 0);
            const WallCoef& wc = a.coef[w];
            cf[0] = wc.in.b; cf[1] = wc.in.c_su; cf[2] = wc.in.c_sv;
            // register 0's row: a face row in the face lanes, else the interior row,
            // whose face terms are 0 (hyg_coef.cuh) — picked by address, so no
            // select waits on the loads (they complete behind the outputs)
            const RowCoef& c = sub == 0 ? wc.face[0] : (sub == 15 ? wc.face[1] : wc.in);
            cf[3] = c.e; cf[4] = c.b; cf[5] = c.e_g; cf[6] = c.c_tv; cf[7] = c.c_sv; cf[8] = c.c_tu;
            cf[9] = c.c_su; cf[10] = c.c_q; cf[11] = c.c_g;
            ch = a.attach[2 * w].index;
        } else if (is_halo) {
            const int hl = (warp - own_w) * 32 + lane;
            const int hlc = hl < HW ? hl : 0;
            const int hz = hlc / W, wi = hlc - hz * W;
            const int w = gz(z0, halo_local(hz, nown)) * W + wi;
            const WallCoef& wc = a.coef[w];
            cf[0] = wc.in.b; cf[1] = wc.in.c_su; cf[2] = wc.in.c_sv;
            const RowCoef& c = wc.face[1];
            cf[3] = c.e; cf[4] = c.b; cf[5] = c.e_g; cf[6] = c.c_tv; cf[7] = c.c_sv; cf[8] = c.c_tu;
            cf[9] = c.c_su; cf[10] = c.c_q; cf[11] = c.c_g;
        }
    };
    if (static_cast<int>(blockIdx.x) < nblk) load_cf(blockIdx.x);

    for (int b = blockIdx.x, it = 0; b < nblk; b += gridDim.x, ++it) {
        const int z0 = b * B, nown = min(B, Z - z0);
        const int L = nown + 2 * S;
        const int par = it & 1;
        const bool next = b + static_cast<int>(gridDim.x) < nblk;
        RPROF(0);
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        mbar_wait(mbar, it & 1);                         // the owned walls of block b landed
        __syncthreads();                                 // staging of block b complete
        RPROF(1);
        int cur = 0;                                     // parity of the layer-k shared slots
        if (is_own) {
            // owned wall wl (two per warp), 16 lanes of NPT nodes, last lane reversed
            const int wl = warp * 2 + lane / 16, sub = lane % 16;
            const bool live = wl < nown * W;
            const int wlc = live ? wl : 0;
            const bool first = sub == 0, rev = sub == 15, mirror0 = first || rev;
            const int li = S + wlc / W;                  // local zone of face 1
            double up[NPT], uc[NPT], vp[NPT], vc[NPT];
            const int d0 = wlc * N + sub * NPT;          // this lane's NPT consecutive nodes
            // 16-byte accesses to a lane's NPT consecutive nodes (a 64-byte segment
            // at NPT = 8) would hit the same four banks for every other lane; each
            // lane starts at pair `rot` instead (conflict-free quarter warps), and
            // a select network restores the register order
            const int rot = (sub / (16 / NPT)) & (NPT / 2 - 1);
            auto shift_pairs = [&](double (&t)[NPT], int r) {   // t pair p <- t pair (p - r) mod NPT/2
#pragma unroll
                for (int bit = 1; bit < NPT / 2; bit <<= 1) {
                    const bool on = r & bit;
                    double o[NPT];
#pragma unroll
                    for (int q = 0; q < NPT; ++q) o[q] = t[q];
#pragma unroll
                    for (int q = 0; q < NPT; ++q) t[q] = on ? o[(q + NPT - 2 * bit) % NPT] : o[q];
                }
            };
            auto rd = [&](int f, double (&x)[NPT]) {     // the reversed lane by selects
                double t[NPT];
#pragma unroll
                for (int qq = 0; qq < NPT / 2; ++qq) {   // t pair qq = node pair (qq + rot) mod NPT/2
                    const int pr = (qq + rot) & (NPT / 2 - 1);
                    const double2 v = *reinterpret_cast<const double2*>(&smem[so_ix(f, d0 + 2 * pr)]);
                    t[2 * qq] = v.x;
                    t[2 * qq + 1] = v.y;
                }
                shift_pairs(t, rot);
#pragma unroll
                for (int q = 0; q < NPT; ++q) x[q] = rev ? t[NPT - 1 - q] : t[q];
            };
            rd(0, up);
            rd(1, uc);
            rd(2, vp);
            rd(3, vc);
            RPROF(2);
            __syncthreads();                             // (A) staging consumed by every role
            if (next) prefetch(b + gridDim.x, par ^ 1);
            RPROF(3);
            const double cb = cf[0], csu = cf[1], csv = cf[2];
            // register 0's face-capable row (interior coefficients, zero face terms elsewhere)
            const double fe = cf[3], fb = cf[4], feg = cf[5], fctv = cf[6], fcsv = cf[7], fctu = cf[8], fcsu = cf[9],
                         fcq = cf[10], fcg = cf[11];
            if (rev && live) {                           // layer-k surface sample (node N-1)
                smem[sf_ix(0, 0, own_slot(wl))] = uc[0];
                smem[sf_ix(0, 1, own_slot(wl))] = vc[0];
            }
            __syncthreads();                             // (B) layer-k surfaces and air published
            RPROF(4);
            const int oslot = own_slot(wlc);
            auto step = [&](double (&vP)[NPT], double (&vC)[NPT], double (&uP)[NPT], double (&uC)[NPT], int k) {
                // face inputs of register 0, branch-free (wall.cpp:162-169, 177-189;
                // coupled_node): x=0 the exterior channel, x=1 the zone's layer-k air
                const int am = oRW + k * rw + 4 * ch;
                const double ru = smem[am + 0], rv = smem[am + 1], rg = smem[am + 2], rq = smem[am + 3] + 0.0;
                const double au = smem[ar_ix(cur, 0, li)], av = smem[ar_ix(cur, 1, li)];
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
                for (int q = 0; q < NPT * !(RING_SKIP & 4); ++q) {
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
                    acc |= live ? (static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn))) : 0u;
                    vP[q] = vn;
                    uP[q] = un;
                }
                if (rev && live) {
                    smem[sf_ix(cur ^ 1, 0, oslot)] = uP[0];
                    smem[sf_ix(cur ^ 1, 1, oslot)] = vP[0];
                }
                __syncthreads();
                cur ^= 1;
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
            RPROF(5);
            if (next) load_cf(b + gridDim.x);
            RPROF(6);
            // out = (layer k+S-1, layer k+S): the warp's two walls through its
            // output scratch, two fields at a time, one bulk store (TMA engine)
            // per field — no store instructions on the warps' path
            double* out_s = &smem[oOUT + warp * 2 * 2 * N];
            const int nlive = min(2, max(0, nown * W - warp * 2));
            auto wr = [&](int f, const double (&x)[NPT]) {   // node order, then pair (qq + rot) first
                double t[NPT];
#pragma unroll
                for (int q = 0; q < NPT; ++q) t[q] = rev ? x[NPT - 1 - q] : x[q];
                shift_pairs(t, (NPT / 2 - rot) & (NPT / 2 - 1));
#pragma unroll
                for (int qq = 0; qq < NPT / 2; ++qq) {
                    const int pr = (qq + rot) & (NPT / 2 - 1);
                    *reinterpret_cast<double2*>(&out_s[f * 2 * N + (lane / 16) * N + sub * NPT + 2 * pr]) =
                        make_double2(t[2 * qq], t[2 * qq + 1]);
                }
            };
            auto flush = [&](int f0) {
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                __syncwarp();
                if (lane == 0 && nlive > 0) {
                    const unsigned bytes = static_cast<unsigned>(nlive * N * sizeof(double));
#pragma unroll
                    for (int f = 0; f < 2; ++f)
                        bulk_s2g(a.out[f0 + f] + (static_cast<size_t>(z0) * W + warp * 2) * N, &out_s[f * 2 * N], bytes);
                    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                }
            };
            auto drained = [&]() {   // the scratch may be rewritten once the last copies read it
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                __syncwarp();
            };
            if (!(RING_SKIP & 8)) {
                drained();
                wr(0, up);
                wr(1, uc);
                flush(0);
#if RING_VSTORE
                if (wl < nown * W) {   // v fields straight from registers (16-byte stores)
                    double* g2 = a.out[2] + (static_cast<size_t>(z0) * W + wl) * N + sub * NPT;
                    double* g3 = a.out[3] + (static_cast<size_t>(z0) * W + wl) * N + sub * NPT;
#pragma unroll
                    for (int q = 0; q < NPT; q += 2) {
                        *reinterpret_cast<double2*>(g2 + q) = rev ? make_double2(vp[NPT - 1 - q], vp[NPT - 2 - q]) : make_double2(vp[q], vp[q + 1]);
                        *reinterpret_cast<double2*>(g3 + q) = rev ? make_double2(vc[NPT - 1 - q], vc[NPT - 2 - q]) : make_double2(vc[q], vc[q + 1]);
                    }
                }
#else
                if (!(RING_SKIP & 64)) drained();
                wr(0, vp);
                wr(1, vc);
                flush(2);
#endif
            }
            RPROF(7);
        } else if (is_halo) {
            // halo wall: global nodes N-P .. N-1; the cut end (p = 0) mirrors
            // itself — its error moves inward one node per step and never
            // reaches the face node within S steps
            const int hl = (warp - own_w) * 32 + lane;
            const bool live = hl < HW;
            const int hlc = live ? hl : 0;
            const int hz = hlc / W, wi = hlc - hz * W;
            const int li = halo_local(hz, nown);
            const int w = gz(z0, li) * W + wi;
            double up[P], uc[P], vp[P], vc[P];
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const int d = hlc * PS + (PS - P) + p;
                up[p] = smem[oSH + 0 * HW * PS + d];
                uc[p] = smem[oSH + 1 * HW * PS + d];
                vp[p] = smem[oSH + 2 * HW * PS + d];
                vc[p] = smem[oSH + 3 * HW * PS + d];
            }
            __syncthreads();                             // (A)
            if (next) prefetch(b + gridDim.x, par ^ 1);
            const double cb = cf[0], csu = cf[1], csv = cf[2];
            RowCoef c;
            c.e = cf[3]; c.b = cf[4]; c.e_g = cf[5]; c.c_tv = cf[6]; c.c_sv = cf[7]; c.c_tu = cf[8];
            c.c_su = cf[9]; c.c_q = cf[10]; c.c_g = cf[11];
            if (live) {
                smem[sf_ix(0, 0, halo_slot(hl))] = uc[P - 1];
                smem[sf_ix(0, 1, halo_slot(hl))] = vc[P - 1];
            }
            __syncthreads();                             // (B)
            const int hslot = halo_slot(hlc);
            auto step = [&](double (&vP)[P], double (&vC)[P], double (&uP)[P], double (&uC)[P]) {
                const double u_a = smem[ar_ix(cur, 0, li)], v_a = smem[ar_ix(cur, 1, li)];
#pragma unroll
                for (int p = 0; p < P * !(RING_SKIP & 1); ++p) {
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
                    smem[sf_ix(cur ^ 1, 0, hslot)] = uP[P - 1];
                    smem[sf_ix(cur ^ 1, 1, hslot)] = vP[P - 1];
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
            if (next) load_cf(b + gridDim.x);
        } else {
            // zone thread i: zone_step_explicit (zone.cpp:69-74) of local zone i
            // (1 .. L-2 live; 0 and L-1 contribute their layer-0 air only), with
            // the staged parameter block [0] 1 + kappa, [1] g_v, [2] q_v1, [3] q_v2,
            // [4] #links, [5] #peers, [6] source, links [8 + 4q] = (wall in zone,
            // Bi_TT theta_T, Bi_TM theta_T, sign Bi_M theta_M), peers [40 + 4q] =
            // (peer zone, g_inz, q_inz1, q_inz2)
            const int i = lane;
            const bool valid = i < L;
            const bool live = i >= 1 && i < L - 1;
            const bool owned = i >= S && i < S + nown;
            const int hz = i < S ? i - 1 : (S - 1) + (i - S - nown);
            const int zp = oZS + (par * LB + (valid ? i : 0)) * ZPS;
            int nlink = 0, npeer = 0, sidx = 0;
            int ls[NL], pidx[NP];
            if (live) {
                nlink = static_cast<int>(smem[zp + 4]);
                npeer = static_cast<int>(smem[zp + 5]);
                sidx = static_cast<int>(smem[zp + 6]);
            }
#pragma unroll
            for (int q = 0; q < NL; ++q) {
                const int wi = q < nlink ? static_cast<int>(smem[zp + 8 + 4 * q]) : 0;
                ls[q] = owned ? wi * B + (i - S) : OW + wi * HZ + hz;
            }
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const int pg = q < npeer ? static_cast<int>(smem[zp + 40 + 4 * q]) : -1;
                pidx[q] = i >= 1 && gz(z0, i - 1) == pg ? i - 1 : i + 1;   // the adjacent copy
            }
            if (valid) {
                smem[ar_ix(0, 0, i)] = smem[oZA + (par * 2 + 0) * LB + i];
                smem[ar_ix(0, 1, i)] = smem[oZA + (par * 2 + 1) * LB + i];
            }
            // the parameter block in registers for the whole block (the step loop
            // then loads only states: layer-k air of the zone and peers, samples)
            const double c0 = smem[zp + 0], gv = smem[zp + 1], qv1 = smem[zp + 2], qv2 = smem[zp + 3];
            double lT[NL], lM[NL], lD[NL], pg[NP], pq1[NP], pq2[NP];
#pragma unroll
            for (int q = 0; q < NL; ++q) {
                lT[q] = smem[zp + 9 + 4 * q];
                lM[q] = smem[zp + 10 + 4 * q];
                lD[q] = smem[zp + 11 + 4 * q];
            }
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                pg[q] = smem[zp + 41 + 4 * q];
                pq1[q] = smem[zp + 42 + 4 * q];
                pq2[q] = smem[zp + 43 + 4 * q];
            }
            ZPROF(0);
            __syncthreads();                             // (A) staging consumed
            if (next) prefetch(b + gridDim.x, par ^ 1);
            __syncthreads();                             // (B) layer-k surfaces and air published
            ZPROF(1);
            for (int k = 0; k < a.steps; ++k) {
                if (live && !(RING_SKIP & 2)) {
                    const double u_a = smem[ar_ix(cur, 0, i)], v_a = smem[ar_ix(cur, 1, i)];
                    const int srow = oRW + k * rw + 4 * a.n_channels;
                    const int sz = srow + 3 * sidx;
                    const double u_inf = smem[srow + 3 * a.n_sources + 0], v_inf = smem[srow + 3 * a.n_sources + 1];
                    double du = smem[sz + 1] + smem[sz + 2] + qv1 * (u_inf * v_inf - u_a * v_a) + qv2 * (u_inf - u_a);
                    double dv = smem[sz + 0] + gv * (v_inf - v_a);
                    // branch-free over the maximum link/peer counts: the unused slots of
                    // the parameter block are zero (their terms add +0), so every load
                    // is independent and only the additions stay in order
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
            ZPROF(2);
            if (owned) {
                const int z = gz(z0, i);
                a.zu_out[z] = smem[ar_ix(cur, 0, i)];
                a.zv_out[z] = smem[ar_ix(cur, 1, i)];
            }
        }
        __syncthreads();                                 // the shared slots are reused by the next block
        RPROF(8);
    }
    if (is_own && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");   // stores drained
    // fast guard verdict of the whole launch (bit 30: |x| >= 2 or not finite)
    // (timing variants march stale staging: their verdict is dropped)
    if (__syncthreads_or((acc & 0x40000000u) != 0u) && tid == 0 && RING_SKIP < 8) atomicCAS(a.stop, 0, a.seg_index + 1);
}

}  // namespace hyg
