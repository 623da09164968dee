// k_ring_pipe.cuh — K5: the zone-ring march (configs[3]) with deeper temporal
// blocking and a per-step hand-off through mbarriers instead of a CTA barrier.
//
// Same decomposition, rows and zone arithmetic as K4r (k_ring_reg.cuh) —
// S consecutive step_explicit calls (building.cpp:152-187) per launch, a CTA
// marching B owned zones with their walls in registers plus the halo zones
// the zone cone needs — restructured for the HBM roofline:
//
//   * deeper blocks: S = 12 steps per launch, B = 3 zones per block (K4r: 8
//     and 4).  HBM per update falls from 8.98 B to 6.3 B, because the halo is
//     trimmed to what the cone uses:
//     a halo zone at distance d (1 <= d <= S-1) is consumed only through
//     layer S-d, so its walls need their last S-d nodes (rounded up to an even
//     count for 16-byte bulk copies) and S-d-1 steps (K4r: S+1 nodes, S steps);
//   * no CTA barrier per step: the walls and the zone warp hand layer-k data
//     over through two pairs of named barriers, producers arriving without
//     waiting (surface samples of layer k -> zone warp; zone air of layer k
//     -> walls), so a wall warp computes the interior rows of step k while the
//     zone warp is still producing the air its face row needs;
//   * a producer warp stages the next block while the current one marches:
//     owned walls (one bulk copy per field, on an mbarrier's transaction
//     count), halo walls and zone parameter blocks (cp.async) and zone air;
//     the row coefficients of the next block are loaded into registers
//     behind the steps;
//   * the zone warp sums every term that needs no wall sample (sources,
//     ventilation, peers) before it waits for the walls, so the per-step
//     critical path is the six wall-link terms and the division;
//   * outputs straight from registers (16-byte stores; the reversed lane
//     stores its nodes in node order), no shared-memory scratch.
//
// Every owned value is computed by the same increment-form rows (hyg_coef.cuh)
// and zone additions as K4r and the per-step path, so K5 is bitwise equal to
// both.  Guard: K1's fast guard (bit 30) over owned walls and zones; a set bit
// stops the following launches and the host replays from the flagged launch
// with K4 (exact guard).  Used for divergence_norm >= 2 and zones with <= 6
// wall links and <= 2 ring peers on 128-node walls.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "k_ring_reg.cuh"

namespace hyg {

template <int S>
struct RingPipeShape {
    static constexpr int NPT = 8, N = 128;
    static constexpr int kHaloZones = 2 * (S - 1);
    static constexpr int kZPS = kRingZP;                       // 448 B rows: whole-block bulk copies (read once per block)
    // CTA size for configs[3]'s shape, W = 6 walls per zone and B = kB owned
    // zones per block: 3 W / 2 owned + halo + zone + producer warps (16 warps
    // at S = 12: 4 per scheduler, so 128 registers per thread)
    static constexpr int kB = 3;
    static constexpr int kThreads = 32 * ((kB * 6 + 1) / 2 + (2 * (S - 1) * 6 + 31) / 32 + 2);
    // nodes kept for a halo zone at distance d: S - d, rounded up to even
    __host__ __device__ static constexpr int halo_nodes(int d) { return (S - d + 1) & ~1; }
    __host__ __device__ static int own_warps(int B, int W) { return (B * W + 1) / 2; }
    __host__ __device__ static int halo_walls(int W) { return kHaloZones * W; }
    __host__ __device__ static int halo_warps(int W) { return (halo_walls(W) + 31) / 32; }
    __host__ __device__ static int warps(int B, int W) { return own_warps(B, W) + halo_warps(W) + 2; }
    __host__ __device__ static int threads(int B, int W) { return 32 * warps(B, W); }
    __host__ __device__ static int local_zones(int B) { return B + 2 * S; }
    // doubles: owned staging [4][B W][N], halo staging [4][HW][S], zone
    // parameter blocks [2][LB][ZPS], staged zone air [2][2][LB], surfaces
    // [2][2][B W + HW], zone air [2][2][LB], forcing rows [S][rw], mbarriers
    __host__ __device__ static size_t smem_doubles(int B, int W, int rw) {
        const size_t LB = local_zones(B);
        return static_cast<size_t>(4) * B * W * N + static_cast<size_t>(4) * halo_walls(W) * S + 2 * LB * kZPS +
               4 * LB + 4 * static_cast<size_t>(B * W + halo_walls(W)) + 4 * LB +
               ((static_cast<size_t>(S) * rw + 1) & ~1ull) + 8;
    }
};

// per-step hand-off on named barriers: producers arrive (no wait), consumers
// sync (the warp sleeps, issuing nothing, until the count is reached); every
// use counts the wall warps and the zone warp (the producer warp stays out).  IDs 1-2:
// surface samples of layer g (slot g & 1); IDs 3-4: zone air of layer g.
__device__ __forceinline__ void nb_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nb_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx_only(void* mb, unsigned bytes) {   // no arrival
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(void* mb) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(mb)) : "memory");
}
__device__ __forceinline__ void mbar_wait_acq(void* mb, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n PIPE_WAIT_%=:\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra PIPE_WAIT_%=;\n}\n" ::"r"(smem_u32(mb)),
        "r"(phase)
        : "memory");
}

// timing experiments only: per-phase clock64 stamps of CTA 0 into g_ring_prof
// (k_ring_reg.cuh, RING_PROF builds): [block iteration][event]
#if RING_PROF
#define PSTAMP(e) do { if (blockIdx.x == 0 && lane == 0 && it < 32) g_ring_prof[it * 16 + (e)] = clock64(); } while (0)
#else
#define PSTAMP(e) do { } while (0)
#endif

// THREADS: the CTA size the host launches (whole roles; registers are sized for it)
template <int S, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) k_ring_pipe(const RingArgs a) {
    using Sh = RingPipeShape<S>;
    constexpr int NPT = Sh::NPT, N = Sh::N, NL = 6, NP = 2;
    constexpr int PH = S;                                // halo nodes held per thread (max over distances)
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int HZ = Sh::kHaloZones, ZPS = Sh::kZPS;
    extern __shared__ double smem[];
    if (launch_stopped(a.stop)) return;
    const int W = a.W, B = a.B, Z = a.n_zones;
    const int OW = B * W, HW = Sh::halo_walls(W), LB = Sh::local_zones(B);
    const int rw = RingShape<NPT, S>::row_width(a.n_channels, a.n_sources);
    const int oSO = 0;                                   // owned staging [4][OW][N]
    const int oSH = oSO + 4 * OW * N;                    // halo staging [4][HW][PH]
    const int oZS = oSH + 4 * HW * PH;                   // zone parameter blocks [2][LB][ZPS]
    const int oZA = oZS + 2 * LB * ZPS;                  // staged zone air [2][2][LB] (producer)
    const int oSF = oZA + 4 * LB;                        // surfaces [slot][field][OW + HW]
    const int oAR = oSF + 4 * (OW + HW);                 // zone air [slot][field][LB]
    const int oRW = oAR + 4 * LB;                        // forcing rows [S][rw]
    const int oMB = oRW + ((S * rw + 1) & ~1);           // mbarriers (8-byte each)
    double* mb_full = &smem[oMB + 0];                    // staging of the next block landed (tx)
    double* mb_free = &smem[oMB + 1];                    // staging consumed by every warp
    auto so_ix = [&](int f, int i) { return oSO + f * OW * N + i; };
    auto sf_ix = [&](int slot, int f, int i) { return oSF + (slot * 2 + f) * (OW + HW) + i; };
    auto own_slot = [&](int wl) { const int z = wl / W; return (wl - z * W) * B + z; };
    auto halo_slot = [&](int hl) { const int h = hl / W; return OW + (hl - h * W) * HZ + h; };
    auto ar_ix = [&](int slot, int f, int i) { return oAR + (slot * 2 + f) * LB + i; };
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int nblk = (Z + B - 1) / B;
    const int own_w = Sh::own_warps(B, W), halo_w = Sh::halo_warps(W);
    const int zone_warp = own_w + halo_w, producer_warp = zone_warp + 1;
    const int NT = 32 * (zone_warp + 1);                 // named-barrier count: walls + zone warp (no producer)
    const bool is_own = warp < own_w, is_halo = !is_own && warp < zone_warp;

    for (int i = tid; i < a.steps * rw; i += blockDim.x) {   // forcing rows of this launch
        const int k = i / rw, r = i - k * rw;
        cp_async8(&smem[oRW + i],
                  r < 4 * a.n_channels
                      ? reinterpret_cast<const double*>(a.table + static_cast<size_t>(k) * a.n_channels) + r
                      : a.src + static_cast<size_t>(k) * (3 * a.n_sources + 2) + (r - 4 * a.n_channels));
    }
    asm volatile("cp.async.commit_group;\n" ::);
    const bool wide = Z >= B + 3 * S;
    auto gz = [&](int z0, int i) {
        int g = z0 - S + i;
        if (wide) {
            g += g < 0 ? Z : 0;
            return g >= Z ? g - Z : g;
        }
        return (g % Z + Z) % Z;
    };
    // halo zone hz (0 .. HZ-1): local zone and distance from the owned block
    auto halo_local = [&](int hz, int nown) { return hz < S - 1 ? 1 + hz : S + nown + (hz - (S - 1)); };
    auto halo_dist = [&](int hz) { return hz < S - 1 ? S - 1 - hz : hz - (S - 1) + 1; };
    // staging of block b (run by the producer warp): owned walls (one bulk copy
    // per field) and zone parameter blocks (one per contiguous run) on
    // mb_full's tx count; halo walls (16-byte cp.async) and zone air (loads)
    // into parity `par`; then the producer's one arrival
    auto stage = [&](int b, int par) {
        const int z0 = b * B, nown = min(B, Z - z0), L = nown + 2 * S;
        const unsigned own_bytes = static_cast<unsigned>(nown * W * N * sizeof(double));
        // zone parameter blocks: the local zones are one or two contiguous runs
        // of the ring (one copy per zone for rings narrower than the block)
        const int g0 = gz(z0, 0);
        const int run1 = wide ? min(L, Z - g0) : 0;
        const unsigned zp_bytes = static_cast<unsigned>(L * kRingZP * sizeof(double));
        if (lane == 0) mbar_expect_tx_only(mb_full, 4 * own_bytes + zp_bytes);
        __syncwarp();
        if (lane < 4) bulk_g2s(&smem[so_ix(lane, 0)], a.in[lane] + static_cast<size_t>(z0) * W * N, own_bytes, mb_full);
        if (wide) {
            if (lane == 4)
                bulk_g2s(&smem[oZS + par * LB * ZPS], a.zparams + static_cast<size_t>(g0) * kRingZP,
                         static_cast<unsigned>(run1 * kRingZP * sizeof(double)), mb_full);
            if (lane == 5 && run1 < L)
                bulk_g2s(&smem[oZS + (par * LB + run1) * ZPS], a.zparams,
                         static_cast<unsigned>((L - run1) * kRingZP * sizeof(double)), mb_full);
        } else {
            for (int li = lane; li < L; li += 32)
                bulk_g2s(&smem[oZS + (par * LB + li) * ZPS], a.zparams + static_cast<size_t>(gz(z0, li)) * kRingZP,
                         static_cast<unsigned>(kRingZP * sizeof(double)), mb_full);
        }
        // halo walls: 16-byte cp.async, one (halo zone, wall, field) segment of
        // P nodes per lane and iteration — hundreds of 16-96 byte bulk copies
        // per block measured far slower on the TMA engine (profiles/)
        for (int sg = lane; sg < HZ * W * 4 && !(a.dbg_skip & 1); sg += 32) {
            const int f = sg & 3, hl = sg >> 2, hz = hl / W, wi = hl - hz * W;
            const int P = Sh::halo_nodes(halo_dist(hz));
            const double* src = a.in[f] + (static_cast<size_t>(gz(z0, halo_local(hz, nown))) * W + wi) * N + (N - P);
            double* dst = &smem[oSH + (f * HW + hl) * PH + (PH - P)];
            for (int c = 0; c < P; c += 2) cp_async16(dst + c, src + c);
        }
        asm volatile("cp.async.commit_group;\n" ::);
        for (int i = lane; i < L; i += 32) {
            const int gzi = gz(z0, i);
            smem[oZA + (par * 2 + 0) * LB + i] = a.zu_in[gzi];
            smem[oZA + (par * 2 + 1) * LB + i] = a.zv_in[gzi];
        }
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(mb_full);             // release: the parameter blocks and air above
    };
    if (tid == 0) {
        mbar_init(mb_full, 1);
        mbar_init(mb_free, own_w + halo_w + 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();                                     // rows staged, barriers initialised

    unsigned acc = 0;
    // each role marches the blocks in its own loop, with its own registers; the
    // role registers (row coefficients of the walls, zone air of the zone warp)
    // are loaded one block ahead
    if (is_own) {
        double cf[12];
        int ch = 0;
        auto load_cf = [&](int bb) {
            const int z0 = bb * B, nown = min(B, Z - z0);
            const int wl = warp * 2 + lane / 16, sub = lane % 16;
            const int w = z0 * W + (wl < nown * W ? wl : 0);
            const WallCoef& wc = a.coef[w];
            cf[0] = wc.in.b; cf[1] = wc.in.c_su; cf[2] = wc.in.c_sv;
            const RowCoef& c = sub == 0 ? wc.face[0] : (sub == 15 ? wc.face[1] : wc.in);
            cf[3] = c.e; cf[4] = c.b; cf[5] = c.e_g; cf[6] = c.c_tv; cf[7] = c.c_sv; cf[8] = c.c_tu;
            cf[9] = c.c_su; cf[10] = c.c_q; cf[11] = c.c_g;
            ch = a.attach[2 * w].index;
        };
        if (static_cast<int>(blockIdx.x) < nblk) load_cf(blockIdx.x);
        int g = 0;                                       // this role's running step index (mbarrier phases)
        for (int b = blockIdx.x, it = 0; b < nblk; b += gridDim.x, ++it) {
            const int z0 = b * B, nown = min(B, Z - z0);
            const bool next = b + static_cast<int>(gridDim.x) < nblk;
            if (warp == 0) PSTAMP(0);
            mbar_wait_acq(mb_full, it & 1);                  // block b's staging landed
            if (warp == 0) PSTAMP(1);
            const int wl = warp * 2 + lane / 16, sub = lane % 16;
            const bool live = wl < nown * W;
            const int wlc = live ? wl : 0;
            const bool first = sub == 0, rev = sub == 15, mirror0 = first || rev;
            const int li = S + wlc / W;                  // local zone of face 1
            double up[NPT], uc[NPT], vp[NPT], vc[NPT];
            const int d0 = wlc * N + sub * NPT;
            const int rot = (sub / (16 / NPT)) & (NPT / 2 - 1);
            auto shift_pairs = [&](double (&t)[NPT], int r) {
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
            auto rd = [&](int f, double (&x)[NPT]) {
                double t[NPT];
#pragma unroll
                for (int qq = 0; qq < NPT / 2; ++qq) {
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
            __syncwarp();
            if (lane == 0) mbar_arrive(mb_free);         // staging consumed by this warp
            if (warp == 0) PSTAMP(2);
            const double cb = cf[0], csu = cf[1], csv = cf[2];
            const double fe = cf[3], fb = cf[4], feg = cf[5], fctv = cf[6], fcsv = cf[7], fctu = cf[8], fcsu = cf[9],
                         fcq = cf[10], fcg = cf[11];
            const int oslot = own_slot(wlc);
            if (rev && live) {                           // layer-g surface sample
                smem[sf_ix(g & 1, 0, oslot)] = uc[0];
                smem[sf_ix(g & 1, 1, oslot)] = vc[0];
            }
            nb_arrive(1 + (g & 1), NT);                  // layer-g samples published
            auto step = [&](double (&vP)[NPT], double (&vC)[NPT], double (&uP)[NPT], double (&uC)[NPT], int k) {
                const int gg = g + k;
                const double vs = rev ? vC[NPT - 1] : vC[0], us = rev ? uC[NPT - 1] : uC[0];
                const double vup = __shfl_up_sync(FULL, vC[NPT - 1], 1, 16);
                const double uup = __shfl_up_sync(FULL, uC[NPT - 1], 1, 16);
                const double vdn = __shfl_down_sync(FULL, vs, 1, 16);
                const double udn = __shfl_down_sync(FULL, us, 1, 16);
                const double vx0 = mirror0 ? vC[1] : vup, ux0 = mirror0 ? uC[1] : uup;
                const double vx1 = rev ? vup : vdn, ux1 = rev ? uup : udn;
                // interior rows first: they need no zone air (each row reads only its own
                // layer-(k-1) node, so the new value replaces it in place)
#pragma unroll
                for (int q = 1; q < NPT; ++q) {
                    const double vl = vC[q - 1], ul = uC[q - 1];
                    const double vr = q == NPT - 1 ? vx1 : vC[q + 1], ur = q == NPT - 1 ? ux1 : uC[q + 1];
                    const double d = fma(-2.0, vP[q], vl + vr);
                    const double du = fma(-2.0, uP[q], ul + ur);
                    const double vn = fma(cb, d, vP[q]);
                    const double un = fma(csv, d, fma(csu, du, uP[q]));
                    acc |= live ? (static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn))) : 0u;
                    vP[q] = vn;
                    uP[q] = un;
                }
                // register 0: the face-capable row (wall.cpp:162-169, 177-189): x=0 the
                // exterior channel, x=1 the zone's layer-gg air (wait for it here)
                const int am = oRW + k * rw + 4 * ch;
                const double ru = smem[am + 0], rv = smem[am + 1], rg = smem[am + 2], rq = smem[am + 3] + 0.0;
                const double d = fma(-2.0, vP[0], vx0 + vC[1]);
                const double du = fma(-2.0, uP[0], ux0 + uC[1]);
                nb_sync(3 + (gg & 1), NT);               // layer-gg zone air
                const double au = smem[ar_ix(gg & 1, 0, li)], av = smem[ar_ix(gg & 1, 1, li)];
                const double u_inf = first ? ru : au, v_inf = first ? rv : av;
                const double g_inf = first ? rg : 0.0, q_inf = first ? rq : 0.0;
                {
                    const double t = v_inf - vP[0], tu = u_inf - uP[0];
                    const double vn = fma(fe, t, fma(fb, d, fma(feg, g_inf, vP[0])));
                    const double un = fma(fctv, t, fma(fcsv, d, fma(fctu, tu, fma(fcsu, du, fma(fcq, q_inf, fma(fcg, g_inf, uP[0]))))));
                    acc |= live ? (static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn))) : 0u;
                    vP[0] = vn;
                    uP[0] = un;
                }
                if (k + 1 < a.steps) {                   // layer gg+1 samples (the last layer is not consumed)
                    if (rev && live) {
                        smem[sf_ix((gg + 1) & 1, 0, oslot)] = uP[0];
                        smem[sf_ix((gg + 1) & 1, 1, oslot)] = vP[0];
                    }
                    nb_arrive(1 + ((gg + 1) & 1), NT);
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
            if (warp == 0) PSTAMP(3);
            if (next) load_cf(b + gridDim.x);
            if (warp == 0) PSTAMP(4);
            // out = (layer k+S-1, layer k+S) straight from registers, node order
            if (live) {
                const size_t o = (static_cast<size_t>(z0) * W + wl) * N + sub * NPT;
                auto st = [&](double* dst, const double (&x)[NPT]) {
#pragma unroll
                    for (int q = 0; q < NPT; q += 2)
                        *reinterpret_cast<double2*>(dst + o + q) =
                            rev ? make_double2(x[NPT - 1 - q], x[NPT - 2 - q]) : make_double2(x[q], x[q + 1]);
                };
                st(a.out[0], up);
                st(a.out[1], uc);
                st(a.out[2], vp);
                st(a.out[3], vc);
            }
            if (warp == 0) PSTAMP(5);
            g += a.steps;
        }
    } else if (is_halo) {
        double cf[12];
        auto load_cf = [&](int bb) {
            const int z0 = bb * B, nown = min(B, Z - z0);
            const int hl = (warp - own_w) * 32 + lane;
            const int hlc = hl < HW ? hl : 0;
            const int hz = hlc / W, wi = hlc - hz * W;
            const WallCoef& wc = a.coef[gz(z0, halo_local(hz, nown)) * W + wi];
            cf[0] = wc.in.b; cf[1] = wc.in.c_su; cf[2] = wc.in.c_sv;
            const RowCoef& c = wc.face[1];
            cf[3] = c.e; cf[4] = c.b; cf[5] = c.e_g; cf[6] = c.c_tv; cf[7] = c.c_sv; cf[8] = c.c_tu;
            cf[9] = c.c_su; cf[10] = c.c_q; cf[11] = c.c_g;
        };
        if (static_cast<int>(blockIdx.x) < nblk) load_cf(blockIdx.x);
        int g = 0;                                       // this role's running step index (mbarrier phases)
        for (int b = blockIdx.x, it = 0; b < nblk; b += gridDim.x, ++it) {
            const int z0 = b * B, nown = min(B, Z - z0);
            const bool next = b + static_cast<int>(gridDim.x) < nblk;
            mbar_wait_acq(mb_full, it & 1);                  // block b's staging landed
            // halo wall: its last PH nodes (the last P(d) of them real, the rest
            // stale: a cut end is wrong one more node per step and never reaches
            // the face node within the S - d - 1 steps this wall marches)
            const int hl = (warp - own_w) * 32 + lane;
            const bool live = hl < HW;
            const int hlc = live ? hl : 0;
            const int hz = hlc / W;
            const int li = halo_local(hz, nown);
            const int ks = live ? S - halo_dist(hz) - 1 : 0;   // steps this wall marches
            double up[PH], uc[PH], vp[PH], vc[PH];
#pragma unroll
            for (int p = 0; p < PH; ++p) {
                const int d = hlc * PH + p;
                up[p] = smem[oSH + 0 * HW * PH + d];
                uc[p] = smem[oSH + 1 * HW * PH + d];
                vp[p] = smem[oSH + 2 * HW * PH + d];
                vc[p] = smem[oSH + 3 * HW * PH + d];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(mb_free);
            const double cb = cf[0], csu = cf[1], csv = cf[2];
            RowCoef c;
            c.e = cf[3]; c.b = cf[4]; c.e_g = cf[5]; c.c_tv = cf[6]; c.c_sv = cf[7]; c.c_tu = cf[8];
            c.c_su = cf[9]; c.c_q = cf[10]; c.c_g = cf[11];
            const int hslot = halo_slot(hlc);
            if (live) {
                smem[sf_ix(g & 1, 0, hslot)] = uc[PH - 1];
                smem[sf_ix(g & 1, 1, hslot)] = vc[PH - 1];
            }
            nb_arrive(1 + (g & 1), NT);                  // layer-g samples published
            const int kmax = __reduce_max_sync(FULL, ks);
            auto step = [&](double (&vP)[PH], double (&vC)[PH], double (&uP)[PH], double (&uC)[PH], int k) {
                const int gg = g + k;
                if (k < kmax) {
                    // in place: node p's row reads layer k at p-1, p+1 and its own layer k-1
                    // (the cut end p = 0 mirrors itself)
                    const double d_f = fma(-2.0, vP[PH - 1], vC[PH - 2] + vC[PH - 2]);
                    const double du_f = fma(-2.0, uP[PH - 1], uC[PH - 2] + uC[PH - 2]);
#pragma unroll
                    for (int p = 0; p < PH - 1; ++p) {
                        const double vl = p == 0 ? vC[0] : vC[p - 1], ul = p == 0 ? uC[0] : uC[p - 1];
                        const double d = fma(-2.0, vP[p], vl + vC[p + 1]);
                        const double du = fma(-2.0, uP[p], ul + uC[p + 1]);
                        vP[p] = fma(cb, d, vP[p]);
                        uP[p] = fma(csv, d, fma(csu, du, uP[p]));
                    }
                    nb_sync(3 + (gg & 1), NT);
                    const double u_a = smem[ar_ix(gg & 1, 0, li)], v_a = smem[ar_ix(gg & 1, 1, li)];
                    const double t = v_a - vP[PH - 1], tu = u_a - uP[PH - 1];
                    const double vn = fma(c.e, t, fma(c.b, d_f, fma(c.e_g, 0.0, vP[PH - 1])));
                    const double un = fma(c.c_tv, t, fma(c.c_sv, d_f, fma(c.c_tu, tu, fma(c.c_su, du_f, fma(c.c_q, 0.0,
                                                                                                  fma(c.c_g, 0.0, uP[PH - 1]))))));
                    vP[PH - 1] = vn;
                    uP[PH - 1] = un;
                } else {
                    nb_sync(3 + (gg & 1), NT);           // keep the barrier phases
                }
                if (k + 1 < a.steps) {
                    if (live && k < ks) {
                        smem[sf_ix((gg + 1) & 1, 0, hslot)] = uP[PH - 1];
                        smem[sf_ix((gg + 1) & 1, 1, hslot)] = vP[PH - 1];
                    }
                    nb_arrive(1 + ((gg + 1) & 1), NT);
                }
            };
            int k = 0;
            for (; k + 1 < a.steps; k += 2) {
                step(vp, vc, up, uc, k);
                step(vc, vp, uc, up, k + 1);
            }
            if (k < a.steps) step(vp, vc, up, uc, k);
            if (next) load_cf(b + gridDim.x);
            g += a.steps;
        }
    } else if (warp == zone_warp) {
        // the zone warp: zone_step_explicit (zone.cpp:69-74) of local zone `lane`
        // (1 .. L-2 live; 0 and L-1 contribute their layer-0 air only; L <= 32).
        // Its parameter block (as K4r's) is read into registers once per block;
        // per step everything but the wall-link terms — sources, ventilation,
        // peers, which need only zone air this warp produced itself — is summed
        // before the wait for the walls' samples (the reference's order:
        // sources, ventilation, peers, walls)
        const int i = lane;
        int g = 0;                                       // this role's running step index
        for (int b = blockIdx.x, it = 0; b < nblk; b += gridDim.x, ++it) {
            const int z0 = b * B, nown = min(B, Z - z0);
            const int L = nown + 2 * S;
            const int par = it & 1;
            mbar_wait_acq(mb_full, it & 1);              // block b's staging landed
            PSTAMP(6);
            const bool valid = i < L, live = i >= 1 && i < L - 1, owned = i >= S && i < S + nown;
            const int hz = i < S ? i - 1 : (S - 1) + (i - S - nown);
            const int zp = oZS + (par * LB + (valid ? i : 0)) * ZPS;
            int nlink = 0, npeer = 0, sidx = 0;
            if (live) {
                nlink = static_cast<int>(smem[zp + 4]);
                npeer = static_cast<int>(smem[zp + 5]);
                sidx = static_cast<int>(smem[zp + 6]);
            }
            const double c0 = smem[zp + 0], gv = smem[zp + 1], qv1 = smem[zp + 2], qv2 = smem[zp + 3];
            int ls[NL], pidx[NP];
            double lT[NL], lM[NL], lD[NL], pg[NP], pq1[NP], pq2[NP];
#pragma unroll
            for (int q = 0; q < NL; ++q) {
                const int wi = q < nlink ? static_cast<int>(smem[zp + 8 + 4 * q]) : 0;
                ls[q] = owned ? wi * B + (i - S) : OW + wi * HZ + hz;
                lT[q] = smem[zp + 9 + 4 * q];
                lM[q] = smem[zp + 10 + 4 * q];
                lD[q] = smem[zp + 11 + 4 * q];
            }
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const int pgz = q < npeer ? static_cast<int>(smem[zp + 40 + 4 * q]) : -1;
                pidx[q] = i >= 1 && gz(z0, i - 1) == pgz ? i - 1 : i + 1;
                pg[q] = smem[zp + 41 + 4 * q];
                pq1[q] = smem[zp + 42 + 4 * q];
                pq2[q] = smem[zp + 43 + 4 * q];
            }
            if (valid) {                                 // layer-g air from the producer's staging
                smem[ar_ix(g & 1, 0, i)] = smem[oZA + (par * 2 + 0) * LB + i];
                smem[ar_ix(g & 1, 1, i)] = smem[oZA + (par * 2 + 1) * LB + i];
            }
            __syncwarp();
            nb_arrive(3 + (g & 1), NT);                  // layer-g air published
            if (lane == 0) mbar_arrive(mb_free);         // this block's staging consumed
            PSTAMP(7);
            for (int k = 0; k < a.steps; ++k) {
                const int gg = g + k;
                const int cs = gg & 1, ns = cs ^ 1;
                double du = 0.0, dv = 0.0, u_a = 0.0, v_a = 0.0;
                if (live) {
                    u_a = smem[ar_ix(cs, 0, i)];
                    v_a = smem[ar_ix(cs, 1, i)];
                    const int srow = oRW + k * rw + 4 * a.n_channels;
                    const int sz = srow + 3 * sidx;
                    const double u_inf = smem[srow + 3 * a.n_sources + 0], v_inf = smem[srow + 3 * a.n_sources + 1];
                    du = smem[sz + 1] + smem[sz + 2] + qv1 * (u_inf * v_inf - u_a * v_a) + qv2 * (u_inf - u_a);
                    dv = smem[sz + 0] + gv * (v_inf - v_a);
#pragma unroll
                    for (int q = 0; q < NP; ++q) {
                        const double pu = smem[ar_ix(cs, 0, pidx[q])], pv = smem[ar_ix(cs, 1, pidx[q])];
                        du += pq1[q] * (pu * pv - u_a * v_a) + pq2[q] * (pu - u_a);
                        dv += pg[q] * (pv - v_a);
                    }
                }
                nb_sync(1 + cs, NT);                     // layer-gg samples of every wall
                double nu = 0.0, nv = 0.0;
                if (live) {
#pragma unroll
                    for (int q = 0; q < NL; ++q) {
                        const double us = smem[sf_ix(cs, 0, ls[q])], vs = smem[sf_ix(cs, 1, ls[q])];
                        du += lT[q] * (us - u_a) + lM[q] * (vs - v_a);
                        dv += lD[q] * (v_a - vs);
                    }
                    nu = u_a + a.dt * (du / c0);
                    nv = v_a + a.dt * dv;
                    if (owned) acc |= static_cast<unsigned>(__double2hiint(nu)) | static_cast<unsigned>(__double2hiint(nv));
                }
                __syncwarp();                            // every lane read layer gg's air
                if (k + 1 < a.steps) {
                    if (live) {
                        smem[ar_ix(ns, 0, i)] = nu;
                        smem[ar_ix(ns, 1, i)] = nv;
                    }
                    nb_arrive(3 + ns, NT);
                } else if (owned) {
                    const int z = gz(z0, i);
                    a.zu_out[z] = nu;
                    a.zv_out[z] = nv;
                }
            }
            PSTAMP(8);
            g += a.steps;
        }
    } else if (warp == producer_warp) {
        // the producer: stages block b (after every warp consumed block b - grid)
        for (int b = blockIdx.x, it = 0; b < nblk; b += gridDim.x, ++it) {
            PSTAMP(9);
            if (it > 0) mbar_wait_acq(mb_free, (it - 1) & 1);
            PSTAMP(10);
            stage(b, it & 1);
            PSTAMP(11);
        }
    }
    // fast guard verdict of the whole launch (bit 30: |x| >= 2 or not finite)
    if (__syncthreads_or((acc & 0x40000000u) != 0u) && tid == 0) atomicCAS(a.stop, 0, a.seg_index + 1);
}

}  // namespace hyg
