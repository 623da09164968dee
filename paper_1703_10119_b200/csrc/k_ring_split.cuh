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
//     S = 8 steps — one thread per wall cone, one per zone, a CTA of LB
//     consecutive zones whose outer S on each side are halo copies (the zone
//     cone grows one zone per step along the ring).  It records the layer-k
//     air of every owned zone in `series` and writes the zone air of layer S.
//   phase 2, k_ring_walls: every wall is marched SW = m S steps (m = 1, 2, 3)
//     in registers in K1's layout (k_coupled.cuh: 16 lanes x NPT nodes, two
//     walls per warp, neighbours by shuffles, both faces in register 0), its
//     face-1 ambient read from `series`.  No shared surfaces, no barrier in the
//     step loop, no halo walls: 64 B per node per SW steps of HBM traffic (4 B
//     per update at m = 2) and K1's 7 FP64 instructions per update.
//   between the m cone launches that feed one walls launch, k_ring_stub marches
//     the walls' last 17 (25) nodes S steps with the air series just recorded:
//     the tails the next cone launch starts from, which the walls kernel has not
//     produced yet.  ~7 % of the walls' node-updates for cones and stubs.
//
// The face-1 node is computed twice (cone thread and owning lane) with the
// same instruction sequence on the same inputs, so both phases hold the same
// bits and the result equals K4r's and the per-step path's bit for bit.
// Guard: K1's fast guard (bit 30 of the high word) over walls (phase 2) and
// owned zones (phase 1); a set bit stops the following launches and the host
// replays from the flagged launch's untouched input with K4 (exact guard).
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "k_dv_warp.cuh"
#include "k_ring_reg.cuh"

// timing experiments only (tools/ring_walls_probe.cu): skip the steps (1), the
// outputs (2), the layer loads (4); minimum CTAs per SM; 0 / 3 in the library
#ifndef RW_SKIP
#define RW_SKIP 0
#endif
#ifndef RW_MINB
#define RW_MINB 3
#endif
// k_ring_cone: skip the steps (1), the staged loads (2), the zone parameter loads (4),
// the zone arithmetic (8), the cone arithmetic (16), the division (32)
#ifndef RC_SKIP
#define RC_SKIP 0
#endif

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
    // per cone warp: the 32 cones' staged tails [32][4 fields x kPS, + 2: an odd count of
    // 16-byte chunks, so the lanes' reads are conflict-free] and rows [32][12 + 1]
    static constexpr int kTail = 4 * kPS + 2, kRow = 13;
    // doubles: surfaces [parity][field][W][LB], zone air [parity][field][LB], forcing rows
    // [S][rw] (even), then per cone warp tails and rows
    __host__ __device__ static size_t smem_doubles(int LB, int W, int rw) {
        return static_cast<size_t>(4) * W * LB + 4 * LB + ((static_cast<size_t>(S) * rw + 1) & ~static_cast<size_t>(1)) +
               static_cast<size_t>(cone_warps(LB, W)) * 32 * (kTail + kRow);
    }
};

// rows of the cone threads, transposed: rowsT[k][wall], k = in.b, in.c_su, in.c_sv, face[1][0..8]
__global__ void k_ring_cone_rows(int n_walls, const WallCoef* __restrict__ coef, double* __restrict__ rowsT) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= n_walls) return;
    const double* c = reinterpret_cast<const double*>(coef + w);
#pragma unroll
    for (int k = 0; k < 12; ++k) rowsT[static_cast<size_t>(k) * n_walls + w] = c[k == 0 ? 0 : k == 1 ? 3 : k == 2 ? 5 : 15 + k];
}

// Where a cone launch finds its tails and puts its air series.  The walls kernel
// may march SW = m S steps per launch (m = 1, 2, 3): then m cone launches of S
// steps fill the slots [ser_off, ser_off + S) of a zone's SW-slot series row,
// the first from the state arrays (tails = the last nodes of every wall: stride
// n, offset n - PS), the later ones from the compact tail arrays k_ring_stub
// leaves behind (stride PS, offset 0).
struct ConeIO {
    const double* tin[4];          // up, uc, vp, vc
    int tstride, toff;             // tail of wall w: tin[f] + w tstride + toff, PS nodes
    int ser_stride, ser_off;       // series slots per zone, first slot of this launch
};

// ---- phase 1 ---------------------------------------------------------------------------
template <int S, int NL = kRingMaxLinks, int NP = kRingMaxPeers>
__global__ void __launch_bounds__(kRingConeThreads, 1) k_ring_cone(const RingArgs a, double* __restrict__ series,
                                                                  const int LB, const double* __restrict__ rowsT,
                                                                  const double* __restrict__ zpT, const ConeIO io) {
    using Sh = RingConeShape<S>;
    constexpr int P = Sh::kP, PS = Sh::kPS;
    extern __shared__ __align__(16) double smem[];
    if (launch_stopped(a.stop)) return;
    const int W = a.W, Z = a.n_zones;
    const int OB = LB - 2 * S;                          // owned zones per CTA
    const int z0 = blockIdx.x * OB, nown = min(OB, Z - z0), L = nown + 2 * S;
    const int rw = RingShape<8, S>::row_width(a.n_channels, a.n_sources);
    const int oSF = 0, oAR = oSF + 4 * W * LB, oRW = oAR + 4 * LB;
    const int oCW = oRW + ((S * rw + 1) & ~1);          // per cone warp: staged tails and rows
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
        // the warp stages its 32 cones together: tails (the last PS nodes of the four
        // layers, runs of 16-byte copies) and rows (interior b, c_su, c_sv + face[1]) by
        // cp.async, consecutive lanes on consecutive addresses of one wall
        constexpr int TS = Sh::kTail, RS = Sh::kRow, CPW = 4 * (PS / 2);   // chunks per wall
        double* tails = smem + oCW + warp * 32 * (TS + RS);
        double* rows = tails + 32 * TS;
#pragma unroll
        for (int r = 0; r < CPW * !(RC_SKIP & 2); ++r) {
            const int m = r * 32 + lane, wj = m / CPW, fc = m - wj * CPW, f = fc / (PS / 2), cc = fc - f * (PS / 2);
            const int ws = __shfl_sync(0xffffffffu, w, wj);
            cp_async16(&tails[wj * TS + f * PS + 2 * cc], io.tin[f] + static_cast<size_t>(ws) * io.tstride + io.toff + 2 * cc);
        }
        // rows: interior b, c_su, c_sv + face[1], transposed per wall (k_ring_cone_rows):
        // consecutive lanes read consecutive walls
        {
            const int n_walls = Z * W;
#pragma unroll
            for (int k = 0; k < 12 * !(RC_SKIP & 2); ++k) rows[lane * RS + k] = rowsT[static_cast<size_t>(k) * n_walls + w];
        }
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();
        const double* rw_ = rows + lane * RS;
        const double cb = rw_[0], csu = rw_[1], csv = rw_[2];
        // face[1]: b, e, e_g, c_su, c_tu, c_sv, c_tv, c_q, c_g at rw_[3 ..]; read per step
        double up[P], uc[P], vp[P], vc[P];
        {
            auto rd = [&](int f, double (&x)[P]) {
                double t[PS];
#pragma unroll
                for (int q = 0; q < PS / 2; ++q) {
                    const double2 v = *reinterpret_cast<const double2*>(&tails[lane * TS + f * PS + 2 * q]);
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
            for (int p = (RC_SKIP & 16) ? P - 1 : 0; p < P; ++p) {
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
                    const double fb = rw_[3], fe = rw_[4], feg = rw_[5], fcsu = rw_[6], fctu = rw_[7], fcsv = rw_[8],
                                 fctv = rw_[9], fcq = rw_[10], fcg = rw_[11];
                    vn = fma(fe, t, fma(fb, d, fma(feg, 0.0, vP[p])));
                    un = fma(fctv, t, fma(fcsv, d, fma(fctu, tu, fma(fcsu, du, fma(fcq, 0.0, fma(fcg, 0.0, uP[p]))))));
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
        int k = (RC_SKIP & 1) ? a.steps : 0;
        for (; k + 1 < a.steps; k += 2) {
            step(vp, vc, up, uc);
            step(vc, vp, uc, up);
        }
        if (k < a.steps) step(vp, vc, up, uc);
        if (RC_SKIP & 1) acc |= __double2hiint(up[0] + uc[1] + vp[2] + vc[3] + cb + csu + csv) & 1;
    } else {
        // zone thread i: zone_step_explicit (zone.cpp:69-74) of local zone i (1 .. L-2
        // live; 0 and L-1 contribute their layer-0 air only); parameter block as K4r's
        const int i = tid - 32 * cone_w;
        const bool valid = i < L;
        const bool live = i >= 1 && i < L - 1;
        const bool owned = i >= S && i < S + nown;
        const int zg = gz(valid ? i : 0);
        // parameter k of zone z at zpT[k Z + z]: consecutive lanes read consecutive zones
        auto zpv = [&](int k) { return zpT[static_cast<size_t>(k) * Z + ((RC_SKIP & 4) ? 0 : zg)]; };
        int nlink = 0, npeer = 0, sidx = 0;
        if (live) {
            nlink = static_cast<int>(zpv(4));
            npeer = static_cast<int>(zpv(5));
            sidx = static_cast<int>(zpv(6));
        }
        int ls[NL], pidx[NP];
        const double c0 = zpv(0), gv = zpv(1), qv1 = zpv(2), qv2 = zpv(3);
        double lT[NL], lM[NL], lD[NL], pg[NP], pq1[NP], pq2[NP];
        const int iv = valid ? i : 0;
#pragma unroll
        for (int q = 0; q < NL; ++q) {
            const int wi = q < nlink ? static_cast<int>(zpv(8 + 4 * q)) : 0;
            ls[q] = wi * LB + iv;
            lT[q] = zpv(9 + 4 * q);
            lM[q] = zpv(10 + 4 * q);
            lD[q] = zpv(11 + 4 * q);
        }
        const int zprev = gz(iv >= 1 ? iv - 1 : 0);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const int pz = q < npeer ? static_cast<int>(zpv(40 + 4 * q)) : -1;
            pidx[q] = live ? (zprev == pz ? iv - 1 : iv + 1) : 0;   // the adjacent copy
            pg[q] = zpv(41 + 4 * q);
            pq1[q] = zpv(42 + 4 * q);
            pq2[q] = zpv(43 + 4 * q);
        }
        if (valid) {
            smem[ar_ix(0, 0, i)] = a.zu_in[zg];
            smem[ar_ix(0, 1, i)] = a.zv_in[zg];
        }
        double* ser = series + (static_cast<size_t>(zg) * io.ser_stride + io.ser_off) * 2;
        __syncthreads();
        for (int k = (RC_SKIP & 1) ? a.steps : 0; k < a.steps; ++k) {
            if (live && !(RC_SKIP & 8)) {
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
                const double nu = u_a + a.dt * ((RC_SKIP & 32) ? du * c0 : du / c0);
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

// ---- tails for the later cone launches of a long walls launch ------------------------------
// k_ring_stub<DIN>: one thread per wall marches the wall's last DIN nodes (its
// tail at the start of the previous cone launch, from the state arrays or from the
// previous stub's output) S steps with the air series that cone launch recorded
// — the cone arithmetic without the zone coupling — and leaves the last DIN - S
// nodes, exact at the new time, as the next cone launch's (or stub's) tails.
// Step k only computes the nodes still needed (p > k: the cut end goes stale one
// node per step).  Bound by its scattered reads: 144-byte runs out of every 1 KB
// wall cost 56 MB of DRAM traffic per launch (ncu), ~19 us; staging them by
// coalesced cp.async through shared memory measured slower (27.6 vs 21.4 us).
template <int DIN, int S>
__global__ void __launch_bounds__(128) k_ring_stub(const RingArgs a, const double* __restrict__ series,
                                                   const double* __restrict__ rowsT, const ConeIO in,
                                                   double* __restrict__ tout0, double* __restrict__ tout1,
                                                   double* __restrict__ tout2, double* __restrict__ tout3) {
    constexpr int DS = (DIN + 1) & ~1;                  // loaded (even: 16-byte loads)
    constexpr int DOUT = DIN - S, OS = (DOUT + 1) & ~1; // kept, stored
    static_assert(S % 2 == 0 && S <= 8, "the layers end where they began; unrolled for S <= 8");
    if (launch_stopped(a.stop)) return;
    const int n_walls = a.n_zones * a.W;
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= n_walls) return;
    double up[DIN], uc[DIN], vp[DIN], vc[DIN];
    auto rd = [&](int f, double (&x)[DIN]) {
        double t[DS];
        const double* g = in.tin[f] + static_cast<size_t>(w) * in.tstride + in.toff;
#pragma unroll
        for (int q = 0; q < DS / 2; ++q) {
            const double2 v = *reinterpret_cast<const double2*>(g + 2 * q);
            t[2 * q] = v.x;
            t[2 * q + 1] = v.y;
        }
#pragma unroll
        for (int p = 0; p < DIN; ++p) x[p] = t[DS - DIN + p];
    };
    rd(0, up);
    rd(1, uc);
    rd(2, vp);
    rd(3, vc);
    double cf[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) cf[k] = rowsT[static_cast<size_t>(k) * n_walls + w];
    const double cb = cf[0], csu = cf[1], csv = cf[2];
    const double fb = cf[3], fe = cf[4], feg = cf[5], fcsu = cf[6], fctu = cf[7], fcsv = cf[8], fctv = cf[9],
                 fcq = cf[10], fcg = cf[11];
    const double* ser = series + (static_cast<size_t>(w / a.W) * in.ser_stride + in.ser_off) * 2;
    // step K (0-based) produces layer K + 1, exact at nodes p >= K + 1
    auto step = [&](auto KC, double (&vP)[DIN], double (&vC)[DIN], double (&uP)[DIN], double (&uC)[DIN]) {
        constexpr int K = decltype(KC)::value;
        const double2 air = *reinterpret_cast<const double2*>(ser + 2 * K);
        const double u_a = air.x, v_a = air.y;
#pragma unroll
        for (int p = K + 1; p < DIN; ++p) {
            const double vl = vC[p - 1], ul = uC[p - 1];
            const double vr = p == DIN - 1 ? vC[DIN - 2] : vC[p + 1], ur = p == DIN - 1 ? uC[DIN - 2] : uC[p + 1];
            const double d = fma(-2.0, vP[p], vl + vr);
            const double du = fma(-2.0, uP[p], ul + ur);
            double vn, un;
            if (p < DIN - 1) {
                vn = fma(cb, d, vP[p]);
                un = fma(csv, d, fma(csu, du, uP[p]));
            } else {
                const double t = v_a - vP[p], tu = u_a - uP[p];
                vn = fma(fe, t, fma(fb, d, fma(feg, 0.0, vP[p])));
                un = fma(fctv, t, fma(fcsv, d, fma(fctu, tu, fma(fcsu, du, fma(fcq, 0.0, fma(fcg, 0.0, uP[p]))))));
            }
            vP[p] = vn;
            uP[p] = un;
        }
    };
    auto two = [&](auto KC) {
        constexpr int K = decltype(KC)::value;
        step(std::integral_constant<int, K>{}, vp, vc, up, uc);
        step(std::integral_constant<int, K + 1>{}, vc, vp, uc, up);
    };
    two(std::integral_constant<int, 0>{});
    if constexpr (S > 2) two(std::integral_constant<int, 2>{});
    if constexpr (S > 4) two(std::integral_constant<int, 4>{});
    if constexpr (S > 6) two(std::integral_constant<int, 6>{});
    // the last OS nodes (the first may be a stale pad node, never read)
    auto wr = [&](double* t, const double (&x)[DIN]) {
        double* g = t + static_cast<size_t>(w) * OS;
#pragma unroll
        for (int q = 0; q < OS / 2; ++q) {
            const int p0 = DIN - OS + 2 * q;
            *reinterpret_cast<double2*>(g + 2 * q) = make_double2(x[p0], x[p0 + 1]);
        }
    };
    wr(tout0, up);
    wr(tout1, uc);
    wr(tout2, vp);
    wr(tout3, vc);
}

// ---- phase 2 ---------------------------------------------------------------------------
// Persistent warps: warp g of the grid marches the wall pairs g, g + G, ...
// While a pair is marched in registers, the next pair's four layers (8 KB at
// n = 128) arrive in the warp's own shared buffer by four 1-D bulk copies on
// the TMA engine (completion on the warp's mbarrier), its zones' air series and
// row coefficients by 8-byte cp.async; results leave through a per-warp scratch
// and TMA bulk stores, two fields at a time.  No per-thread global loads or
// stores of state: a lane's NPT consecutive nodes are a 64-byte segment, and
// strided 16-byte LDG/STG cost 16 L1 data-pipe passes per instruction (the
// first version of this kernel ran into that pipe at 72 %, DRAM at 50 %);
// shared reads and writes start each lane at a rotated 16-byte pair
// (conflict-free quarter warps, K4r's select network restores the order).
// Measured and not kept: walking the pairs backwards in odd launches so a launch
// starts on the data the previous one wrote last (82.7 vs 83.8 us: nothing of the
// previous output is served from L2), 4 CTAs per SM (128 registers, spills: 92 us
// vs 83 at 3), coalesced cp.async into an XOR-swizzled buffer + direct 16-byte
// stores (95 us).  tools/ring_walls_probe.cu: loads alone 39 us, stores alone 46,
// loads + stores without the steps 79 (5.1 TB/s for this eight-stream pattern).
template <int NPT>
struct RingWallShape {
    static constexpr int kN = 16 * NPT;
    static constexpr int kCoef = static_cast<int>(sizeof(WallCoef) / sizeof(double));   // 27
    // doubles per warp: the pair's four layers, the output scratch (two fields), the
    // (double-buffered) air series and row coefficients of its two walls, the mbarrier
    __host__ __device__ static int warp_doubles(int S) {
        return 4 * 2 * kN + 2 * 2 * kN + 2 * 2 * 2 * S + 2 * 2 * kCoef + 2;
    }
    __host__ __device__ static size_t smem_doubles(int S, int nch, int warps) {
        return ((static_cast<size_t>(S) * 4 * nch + 1) & ~static_cast<size_t>(1)) +
               static_cast<size_t>(warps) * warp_doubles(S);
    }
    // shared layout: the warps' staged layers and output scratch first (kBig doubles each: a
    // multiple of 512 B, the period of the tensor maps' 64-byte swizzle), then the forcing
    // rows, then the warps' small blocks; TMAP launches add 1 KB to align the base
    static constexpr int kBig = 4 * 2 * kN + 2 * 2 * kN;
    __host__ __device__ static int small_doubles(int S) { return 2 * 2 * 2 * S + 2 * 2 * kCoef + 2; }
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                     reinterpret_cast<unsigned long long>(map)),
                 "r"(c0), "r"(c1), "r"(smem_u32(src))
                 : "memory");
}

// TMAP (n = 128, an even number of walls): the pair's layers travel as 2-D TMA tiles through
// tensor maps of the state arrays (rows of 8 nodes, boxes of 32 rows = one wall pair, 64-byte
// swizzle: chunk c of row r at chunk c ^ ((r / 2) mod 4)) in both directions — UTMALDG in,
// UTMASTG out.  Lane l owns row l, so its 16-byte shared reads and writes are conflict-free
// in register order and the rotation's select network (~380 selects per pair, each reading
// two registers beside the FP64 stream) disappears.
template <int NPT, int S, bool TMAP = false>
__global__ void __launch_bounds__(32 * kRingWallWarps, RW_MINB) k_ring_walls(const RingArgs a,
                                                                      const double* __restrict__ series,
                                                                      const __grid_constant__ TiledMaps MI,
                                                                      const __grid_constant__ TiledMaps MO) {
    using Sh = RingWallShape<NPT>;
    constexpr int N = Sh::kN, NC = Sh::kCoef;
    constexpr unsigned FULL = 0xffffffffu;
    static_assert(!TMAP || NPT == 8, "a row of the tensor maps is 8 nodes");
    extern __shared__ __align__(16) double smem_raw[];
    if (launch_stopped(a.stop)) return;
    // TMAP: the swizzle pattern is a function of the shared address, so the base is 1 KB aligned
    double* smem = TMAP ? smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) / sizeof(double) : smem_raw;
    const int W = a.W, n_walls = a.n_zones * W;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int rwc = 4 * a.n_channels;
    double* rows = smem + kRingWallWarps * Sh::kBig;    // forcing rows [S][4 nch]
    for (int i = tid; i < a.steps * rwc; i += blockDim.x)
        rows[i] = reinterpret_cast<const double*>(a.table)[i];
    double* buf = smem + warp * Sh::kBig;               // [4][2 N] staged layers
    double* out_s = buf + 4 * 2 * N;                    // [2][2 N] output scratch
    double* air = rows + ((S * rwc + 1) & ~1) + warp * Sh::small_doubles(S);   // [parity][wall of the pair][S][2]
    double* cfs = air + 2 * 2 * 2 * S;                  // [parity][wall of the pair][WallCoef]
    void* mbar = cfs + 2 * 2 * NC;
    if (lane == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();                                    // rows staged, mbarriers initialised
    const int n_pairs = (n_walls + 1) / 2;
    const int stride = gridDim.x * kRingWallWarps;
    const int half = lane / 16, sub = lane % 16;
    const bool first = sub == 0, rev = sub == 15, mirror0 = first || rev;
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
    auto prefetch = [&](int pair, int par) {
        const int nw = 2 * pair + 1 < n_walls ? 2 : 1;  // the last pair of an odd wall count has one wall
        if (lane == 0) {
            const unsigned bytes = static_cast<unsigned>(nw * N * sizeof(double));
            mbar_expect_tx(mbar, (RW_SKIP & 4) ? 0u : 4 * bytes);
#pragma unroll
            for (int f = 0; f < 4 * !(RW_SKIP & 4); ++f) {
                if (TMAP) dv_tma_load_2d(&buf[f * 2 * N], &MI.m[f], 0, pair * (2 * N / 8), mbar);
                else bulk_g2s(&buf[f * 2 * N], a.in[f] + static_cast<size_t>(pair) * 2 * N, bytes, mbar);
            }
        }
        for (int i = lane; i < 2 * 2 * a.steps; i += 32) {
            const int wj = i / (2 * a.steps), r = i - wj * 2 * a.steps;
            const int w = min(2 * pair + wj, n_walls - 1);
            cp_async8(&air[(par * 2 + wj) * 2 * S + r], series + static_cast<size_t>(w / W) * S * 2 + r);
        }
        for (int i = lane; i < nw * NC; i += 32)
            cp_async8(&cfs[par * 2 * NC + i], reinterpret_cast<const double*>(a.coef + 2 * pair) + i);
        asm volatile("cp.async.commit_group;\n" ::);
    };
    int pair = blockIdx.x * kRingWallWarps + warp;
    if (pair < n_pairs) prefetch(pair, 0);
    unsigned acc = 0;
    for (int it = 0; pair < n_pairs; pair += stride, ++it) {
        const int par = it & 1;
        const int wl = 2 * pair + half;
        const bool live = wl < n_walls;
        const int nlive = min(2, n_walls - 2 * pair);
        const int ch = a.attach[2 * (live ? wl : n_walls - 1)].index;
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        mbar_wait(mbar, par);                           // the pair's layers landed
        __syncwarp();                                   // ... and every lane's air / row copies
        // rows (WallCoef = in, face[0], face[1]; RowCoef = b, e, e_g, c_su, c_tu, c_sv, c_tv, c_q, c_g).
        // Register 0's row: a face row in the face lanes, else the interior row,
        // whose face terms are 0 (hyg_coef.cuh)
        const double* wc = cfs + (par * 2 + (live ? half : 0)) * NC;
        const double cb = wc[0], csu = wc[3], csv = wc[5];
        const double* c = wc + (first ? 9 : (rev ? 18 : 0));
        const double fb = c[0], fe = c[1], feg = c[2], fcsu = c[3], fctu = c[4], fcsv = c[5], fctv = c[6],
                     fcq = c[7], fcg = c[8];
        double up[NPT], uc[NPT], vp[NPT], vc[NPT];
        const int sw = (lane >> 1) & 3;                 // TMAP: this row's chunk swizzle
        auto rd = [&](int f, double (&x)[NPT]) {        // the reversed lane by selects
            double t[NPT];
#pragma unroll
            for (int qq = 0; qq < NPT / 2; ++qq) {      // t pair qq = node pair (qq + rot) mod NPT/2; TMAP: pair qq
                const int pr = TMAP ? (qq ^ sw) : ((qq + rot) & (NPT / 2 - 1));
                const double2 v = *reinterpret_cast<const double2*>(&buf[f * 2 * N + lane * NPT + 2 * pr]);
                t[2 * qq] = v.x;
                t[2 * qq + 1] = v.y;
            }
            if (!TMAP) shift_pairs(t, rot);
#pragma unroll
            for (int q = 0; q < NPT; ++q) x[q] = rev ? t[NPT - 1 - q] : t[q];
        };
        rd(0, up);
        rd(1, uc);
        rd(2, vp);
        rd(3, vc);
        __syncwarp();                                   // the buffer is free for the next pair
        if (pair + stride < n_pairs) prefetch(pair + stride, par ^ 1);
        const double* s_air = air + (par * 2 + half) * 2 * S;
        unsigned acc_t = 0;
        auto step = [&](double (&vP)[NPT], double (&vC)[NPT], double (&uP)[NPT], double (&uC)[NPT], int k) {
            // face inputs of register 0, branch-free (wall.cpp:162-169, 177-189):
            // x = 0 the exterior channel, x = 1 the zone's layer-k air (phase 1)
            const int am = k * rwc + 4 * ch;
            const double ru = rows[am + 0], rv = rows[am + 1], rg = rows[am + 2], rq = rows[am + 3] + 0.0;
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
                acc_t |= static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn));
                vP[q] = vn;
                uP[q] = un;
            }
        };
        int k = (RW_SKIP & 1) ? a.steps : 0;
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
        if (live) acc |= acc_t;
        if (RW_SKIP & 2) {
            acc |= __double2hiint(up[0] + uc[1] + vp[2] + vc[3]) & 1;   // keep the values alive
            continue;
        }
        // out = (layer k+S-1, layer k+S): the pair through the warp's scratch, two
        // fields at a time, one bulk store (TMA engine) per field
        auto wr = [&](int f, const double (&x)[NPT]) {  // node order, then pair (qq + rot) first
            double t[NPT];
#pragma unroll
            for (int q = 0; q < NPT; ++q) t[q] = rev ? x[NPT - 1 - q] : x[q];
            if (!TMAP) shift_pairs(t, (NPT / 2 - rot) & (NPT / 2 - 1));
#pragma unroll
            for (int qq = 0; qq < NPT / 2; ++qq) {
                const int pr = TMAP ? (qq ^ sw) : ((qq + rot) & (NPT / 2 - 1));
                *reinterpret_cast<double2*>(&out_s[f * 2 * N + lane * NPT + 2 * pr]) = make_double2(t[2 * qq], t[2 * qq + 1]);
            }
        };
        auto flush = [&](int f0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                const unsigned bytes = static_cast<unsigned>(nlive * N * sizeof(double));
#pragma unroll
                for (int f = 0; f < 2; ++f) {
                    if (TMAP) tma_store_2d(&MO.m[f0 + f], 0, pair * (2 * N / 8), &out_s[f * 2 * N]);
                    else bulk_s2g(a.out[f0 + f] + static_cast<size_t>(pair) * 2 * N, &out_s[f * 2 * N], bytes);
                }
                asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            }
        };
        auto drained = [&]() {   // the scratch may be rewritten once the last copies read it
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            __syncwarp();
        };
        drained();
        wr(0, up);
        wr(1, uc);
        flush(0);
        drained();
        wr(0, vp);
        wr(1, vc);
        flush(2);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");   // stores drained
    if (__syncthreads_or((acc & 0x40000000u) != 0u) && tid == 0) atomicCAS(a.stop, 0, a.seg_index + 1);
}

}  // namespace hyg
