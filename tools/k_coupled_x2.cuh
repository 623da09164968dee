// k_coupled_x2.cuh — K1 for fp32 state (configs[2]) on packed f32x2 arithmetic.
//
// Same march, rows and guard as k_df_coupled<float> (k_coupled.cuh), which
// replaces df_step_coupled (/root/reference/proj/src/wall.cpp:144-194) per wall
// and step.  The fp32 kernel is issue-bound (one FFMA per issue slot plus the
// guard and the lane exchange); Blackwell's FFMA2/FADD2 (fma.rn.f32x2,
// add.rn.f32x2) do two fp32 operations per issue slot at the same FMA-pipe
// rate (tools/fma_probe.cu: 71.9 TFLOP/s packed vs 70.1 scalar).
//
// Packing: a lane's NPT registers (register order as K1: the last lane of a
// wall reversed, both faces in register 0) form H = NPT/2 pairs
// P[r] = (reg r, reg r+H).  The stencil neighbours of pair r are then the pairs
// r-1 and r+1, except (reg -1, reg H-1) left of pair 0 and (reg H, reg NPT)
// right of pair H-1, built from the lane exchange and one half of the opposite
// edge pair.  Pair 0 carries register 0's face-capable row with packed
// coefficients: face values in the low half, interior ones (face terms 0) in
// the high half.  Every element is the same fp32 fma/add as the scalar kernel,
// so values equal k_df_coupled<float> (up to the sign of a zero), and a fast-
// guard replay with the scalar EXACT kernel continues the same march.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_1703_10119_b200/csrc/k_coupled.cuh"

namespace hyg {

using u64 = unsigned long long;

__device__ __forceinline__ u64 pk2(float lo, float hi) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float lo2(u64 x) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x));
    return a;
}
__device__ __forceinline__ float hi2(u64 x) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x));
    return b;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
    u64 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
    u64 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

// Packed row coefficients: pair 0 (face-capable) and the interior pairs.
struct Row2 { u64 b, e, c_su, c_tu, c_sv, c_tv; };

// One step of a lane's H pairs: P holds layer n-1 on entry and n+1 on exit.
template <int LPW, int H, bool FLUX>
__device__ __forceinline__ void coupled_step_x2(u64 (&vP)[H], const u64 (&vC)[H], u64 (&uP)[H], const u64 (&uC)[H],
                                                const Row2& ci, const Row2& c0, u64 vinf2, u64 uinf2, u64 ev2, u64 eu2,
                                                bool mirror0, bool rev, unsigned& acc) {
    constexpr unsigned FULL = 0xffffffffu;
    const u64 M2 = pk2(-2.0f, -2.0f);
    const float v0 = lo2(vC[0]), u0 = lo2(uC[0]);            // register 0
    const float vN = hi2(vC[H - 1]), uN = hi2(uC[H - 1]);    // register NPT-1
    const float vs = rev ? vN : v0, us = rev ? uN : u0;
    const float vup = __shfl_up_sync(FULL, vN, 1, LPW);
    const float uup = __shfl_up_sync(FULL, uN, 1, LPW);
    const float vdn = __shfl_down_sync(FULL, vs, 1, LPW);
    const float udn = __shfl_down_sync(FULL, us, 1, LPW);
    const float vx0 = mirror0 ? lo2(vC[1]) : vup;            // outer neighbour of register 0
    const float ux0 = mirror0 ? lo2(uC[1]) : uup;
    const float vx1 = rev ? vup : vdn;                       // outer neighbour of register NPT-1
    const float ux1 = rev ? uup : udn;
    const u64 vL0 = pk2(vx0, lo2(vC[H - 1])), uL0 = pk2(ux0, lo2(uC[H - 1]));
    const u64 vRH = pk2(hi2(vC[0]), vx1), uRH = pk2(hi2(uC[0]), ux1);
#pragma unroll
    for (int r = 0; r < H; ++r) {
        const u64 sv = add2(r == 0 ? vL0 : vC[r - 1], r == H - 1 ? vRH : vC[r + 1]);
        const u64 su = add2(r == 0 ? uL0 : uC[r - 1], r == H - 1 ? uRH : uC[r + 1]);
        const u64 d = fma2(M2, vP[r], sv);
        const u64 du = fma2(M2, uP[r], su);
        u64 vn, un;
        if (r == 0) {
            const u64 t = sub2(vinf2, vP[0]);
            const u64 tu = sub2(uinf2, uP[0]);
            vn = fma2(c0.e, t, fma2(c0.b, d, FLUX ? add2(vP[0], ev2) : vP[0]));
            un = fma2(c0.c_tv, t, fma2(c0.c_sv, d, fma2(c0.c_tu, tu, fma2(c0.c_su, du, FLUX ? add2(uP[0], eu2) : uP[0]))));
        } else {
            vn = fma2(ci.b, d, vP[r]);
            un = fma2(ci.c_sv, d, fma2(ci.c_su, du, uP[r]));
        }
        acc |= static_cast<unsigned>(un) | static_cast<unsigned>(vn);
        acc |= static_cast<unsigned>(un >> 32) | static_cast<unsigned>(vn >> 32);
        vP[r] = vn;
        uP[r] = un;
    }
}

// Fast-guard march of fp32 walls (the EXACT replay runs k_df_coupled<float>).
template <int LPW, int NPT, int WARPS, int CHUNK, bool FLUX, int MINB = 0>
__global__ void __launch_bounds__(WARPS * 32, MINB) k_df_coupled_x2(const CoupledSegArgs<float> a) {
    constexpr int H = NPT / 2;
    constexpr int WALLS_PER_CTA = WARPS * 32 / LPW;
    constexpr int N = LPW * NPT;
    static_assert(NPT % 2 == 0 && H >= 2, "pairs need an even NPT >= 4");
    extern __shared__ Ambient s_tab[];   // [CHUNK][n_channels]

    if (*a.stop) return;
    const int tid = threadIdx.x;
    const int sub = tid % LPW;
    const int wall = blockIdx.x * WALLS_PER_CTA + tid / LPW;
    const bool active = wall < a.n_walls;
    const int w = active ? wall : a.n_walls - 1;
    const bool first = sub == 0, rev = sub == LPW - 1;
    const bool mirror0 = first || rev;

    const WallCoef& wc = a.coef[w];
    const float ib = float(wc.in.b), isu = float(wc.in.c_su), isv = float(wc.in.c_sv);
    Row2 ci{pk2(ib, ib), 0ull, pk2(isu, isu), 0ull, pk2(isv, isv), 0ull};
    Row2 c0 = ci;
    double e_g = 0.0, c_q = 0.0, c_g = 0.0;
    int ch = a.chan[2 * w + 0];
    if (mirror0) {
        const RowCoef& f = wc.face[first ? 0 : 1];
        c0 = Row2{pk2(float(f.b), ib), pk2(float(f.e), 0.0f), pk2(float(f.c_su), isu), pk2(float(f.c_tu), 0.0f),
                  pk2(float(f.c_sv), isv), pk2(float(f.c_tv), 0.0f)};
        e_g = f.e_g;
        c_q = f.c_q;
        c_g = f.c_g;
        ch = a.chan[2 * w + (first ? 0 : 1)];
    }

    u64 up[H], uc[H], vp[H], vc[H];
    const size_t base = static_cast<size_t>(w) * N + sub * NPT;
    auto node = [&](int j) { return base + (rev ? NPT - 1 - j : j); };
#pragma unroll
    for (int r = 0; r < H; ++r) {
        const size_t i0 = node(r), i1 = node(r + H);
        up[r] = pk2(a.in[0][i0], a.in[0][i1]);
        uc[r] = pk2(a.in[1][i0], a.in[1][i1]);
        vp[r] = pk2(a.in[2][i0], a.in[2][i1]);
        vc[r] = pk2(a.in[3][i0], a.in[3][i1]);
    }

    unsigned acc = 0;
    const int nch = a.n_channels;
    // per-step ambient of register 0 (fp32 deviations from 1; the high half is
    // an interior node: zero face terms)
    auto amb = [&](int s, u64& vinf2, u64& uinf2, u64& ev2, u64& eu2) {
        const Ambient x = s_tab[s * nch + ch];
        vinf2 = pk2(float(x.v - 1.0), 0.0f);
        uinf2 = pk2(float(x.u - 1.0), 0.0f);
        ev2 = FLUX ? pk2(float(e_g * x.g), 0.0f) : 0ull;
        eu2 = FLUX ? pk2(float(fma(c_q, x.q, c_g * x.g)), 0.0f) : 0ull;
    };
    for (int c0s = 0; c0s < a.nsteps; c0s += CHUNK) {
        const int clen = min(CHUNK, a.nsteps - c0s);
        __syncthreads();
        for (int i = tid; i < clen * nch; i += WARPS * 32) s_tab[i] = a.table[(size_t)c0s * nch + i];
        __syncthreads();
        int s = 0;
        for (; s + 1 < clen; s += 2) {
            u64 vi, ui, ev, eu;
            amb(s, vi, ui, ev, eu);
            coupled_step_x2<LPW, H, FLUX>(vp, vc, up, uc, ci, c0, vi, ui, ev, eu, mirror0, rev, acc);
            amb(s + 1, vi, ui, ev, eu);
            coupled_step_x2<LPW, H, FLUX>(vc, vp, uc, up, ci, c0, vi, ui, ev, eu, mirror0, rev, acc);
        }
        if (s < clen) {   // odd tail (last chunk only)
            u64 vi, ui, ev, eu;
            amb(s, vi, ui, ev, eu);
            coupled_step_x2<LPW, H, FLUX>(vp, vc, up, uc, ci, c0, vi, ui, ev, eu, mirror0, rev, acc);
#pragma unroll
            for (int r = 0; r < H; ++r) {
                u64 t = vp[r]; vp[r] = vc[r]; vc[r] = t;
                t = up[r]; up[r] = uc[r]; uc[r] = t;
            }
        }
    }
    const unsigned any = __reduce_or_sync(0xffffffffu, active ? acc : 0u);
    if ((any & 0x40000000u) && (tid % 32) == 0) atomicCAS(a.suspect, 0, a.seg_index + 1);
    if (!active) return;
#pragma unroll
    for (int r = 0; r < H; ++r) {
        const size_t i0 = node(r), i1 = node(r + H);
        a.out[0][i0] = lo2(up[r]); a.out[0][i1] = hi2(up[r]);
        a.out[1][i0] = lo2(uc[r]); a.out[1][i1] = hi2(uc[r]);
        a.out[2][i0] = lo2(vp[r]); a.out[2][i1] = hi2(vp[r]);
        a.out[3][i0] = lo2(vc[r]); a.out[3][i1] = hi2(vc[r]);
    }
}

}  // namespace hyg
