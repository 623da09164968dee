// k_nonlinear.cuh — K2: nonlinear DF march for walls with the analytic
// coefficient functor k_M* = d(v) (HYG_COEFF_ANALYTIC_D), one warp per wall,
// the four layers in shared memory, all steps of a segment in one launch.
//
// Replaces: df_step_nonlinear (/root/reference/proj/src/wall.cpp:196-264) with
// StarTables (wall.cpp:89-138) for the d(v) functor, called per step from
// run()/step_explicit; guard as check_bounded (building.cpp:282-300).
//
// configs[0] is one wall of 101 nodes marched 1e5 steps: the work per step is
// ~100 node-updates, so the step is latency-bound (one dependency chain:
// neighbours -> half-node d(v) (exp) -> reciprocal -> v -> u).  One warp per
// wall keeps the chain inside a warp (shared memory + __syncwarp, no block
// barrier); batches of such walls run one warp each.
//
// Rows are the reference's, rewritten in increment form around the layer
// n-1 value (exact in real arithmetic; a uniform state at ambient values is
// a fixed point bit for bit, cf. hyg_coef.cuh):
//   v (wall.cpp:213-217):  vn = vp + 2a (kp (vR - vp) + km (vL - vp)) / (c_M + a (kp + km))
//   u (wall.cpp:231-240):  with k_TT = k_TM = c_TT = c_TM = 1,
//       un = up + (2b (uR + uL - 2 up) + 2g (vR + vL - vn - vp) - gamma (vn - vp)) / (1 + 2b)
//   face rows (wall.cpp:218-229, 241-259) likewise, with the ghost-side
//   coefficient k_M at the boundary node and vg from vbar = (vn + vp)/2.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hyg_coef.cuh"
#include "k_coupled.cuh"

namespace hyg {

struct NonlinearSegArgs {
    int n_walls, n, nsteps, n_channels;
    int64_t layer0;
    int seg_index;
    double dx, dt;
    double p[4];                 // d(v) = 1 + p0 v + p1 exp(-p2 (v - p3)^2)
    const Groups* groups;
    const Biot* biot;            // [2*w + face]
    const int* chan;             // [2*w + face]
    const Ambient* table;        // [nsteps][n_channels]
    const double* in[4];
    double* out[4];
    const int* stop;
    int* suspect;
};

__device__ __forceinline__ double d_of(const double* p, double v) {
    const double e = v - p[3];
    return 1.0 + p[0] * v + p[1] * exp(-p[2] * e * e);
}

constexpr int kNlChunk = 64;   // forcing rows staged per chunk

template <int MAXN>
__global__ void __launch_bounds__(32) k_df_analytic_walls(const NonlinearSegArgs A) {
    __shared__ double s_lay[4][MAXN];            // up, uc, vp, vc (roles rotate)
    __shared__ Ambient s_amb[kNlChunk][2];       // [step][face]
    if (*A.stop) return;
    const int w = blockIdx.x, lane = threadIdx.x, n = A.n;
    const size_t o = static_cast<size_t>(w) * n;
    for (int j = lane; j < n; j += 32) {
        s_lay[0][j] = A.in[0][o + j];
        s_lay[1][j] = A.in[1][o + j];
        s_lay[2][j] = A.in[2][o + j];
        s_lay[3][j] = A.in[3][o + j];
    }
    const Groups g = A.groups[w];
    const double dx = A.dx, dt = A.dt;
    const double a = g.Fo_M * dt / (dx * dx);                  // wall.cpp:201-204
    const double b = g.Fo_TT * dt / (dx * dx);
    const double gg = g.Fo_TM * g.gamma * dt / (dx * dx);
    const double ratio = g.Fo_TT != 0.0 ? g.Fo_TM * g.gamma / g.Fo_TT : 0.0;
    const double inv_u = 1.0 / (1.0 + 2.0 * b);
    const Biot bl = A.biot[2 * w], br = A.biot[2 * w + 1];
    const int chl = A.chan[2 * w], chr = A.chan[2 * w + 1];
    double p[4] = {A.p[0], A.p[1], A.p[2], A.p[3]};
    unsigned acc = 0;
    int P = 0;    // s_lay[2*... ] roles: u_prev = s_lay[P], u_curr = s_lay[1-P], same for v (+2)
    __syncwarp();

    for (int c0 = 0; c0 < A.nsteps; c0 += kNlChunk) {
        const int clen = min(kNlChunk, A.nsteps - c0);
        for (int i = lane; i < 2 * clen; i += 32) {
            const int s = i >> 1, f = i & 1;
            s_amb[s][f] = A.table[static_cast<size_t>(c0 + s) * A.n_channels + (f ? chr : chl)];
        }
        __syncwarp();
        for (int s = 0; s < clen; ++s) {
            double* up = s_lay[P];
            const double* uc = s_lay[1 - P];
            double* vp = s_lay[2 + P];
            const double* vc = s_lay[3 - P];
            for (int j = lane; j < n; j += 32) {
                const double vpj = vp[j], upj = up[j], vcj = vc[j];
                double vn, un;
                if (j > 0 && j < n - 1) {
                    const double vL = vc[j - 1], vR = vc[j + 1], uL = uc[j - 1], uR = uc[j + 1];
                    const double kp = d_of(p, 0.5 * (vcj + vR));
                    const double km = d_of(p, 0.5 * (vL + vcj));
                    vn = vpj + 2.0 * a * (kp * (vR - vpj) + km * (vL - vpj)) / (1.0 + a * (kp + km));
                    un = upj + (2.0 * b * (uR + uL - 2.0 * upj) + 2.0 * gg * (vR + vL - vn - vpj) -
                                g.gamma * (vn - vpj)) * inv_u;
                } else {
                    const bool left = j == 0;
                    const int jn = left ? 1 : n - 2;
                    const Biot fb = left ? bl : br;
                    const Ambient am = s_amb[s][left ? 0 : 1];
                    const double vcn = vc[jn], ucn = uc[jn];
                    const double km_b = d_of(p, vcj);                  // ghost side: node value
                    const double kp_b = d_of(p, 0.5 * (vcj + vcn));    // half_front / half_back
                    const double S = kp_b + km_b;
                    const double cpl = 2.0 * a * dx * fb.Bi_M;
                    vn = vpj + (2.0 * a * S * (vcn - vpj) + 2.0 * cpl * (am.v - vpj) + 4.0 * a * dx * am.g) /
                                   (1.0 + a * S + cpl);
                    const double vbar = 0.5 * (vn + vpj);
                    const double vg = vcn - (2.0 * dx / km_b) * (fb.Bi_M * (vbar - am.v) - am.g);
                    const double cplu = 2.0 * b * dx * fb.Bi_TT;
                    un = upj + (4.0 * b * (ucn - upj) + 2.0 * cplu * (am.u - upj) - g.gamma * (vn - vpj) +
                                2.0 * b * ratio * (vcn - vg) - 4.0 * b * dx * (fb.Bi_TM * (vbar - am.v) - am.q) +
                                2.0 * gg * (vcn + vg) - 2.0 * gg * (vn + vpj)) /
                               (1.0 + 2.0 * b + cplu);
                }
                acc |= static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn));
                vp[j] = vn;     // layer n-1 slot becomes layer n+1
                up[j] = un;
            }
            __syncwarp();
            P ^= 1;
        }
    }
    // fast guard verdict (bit 30 of the high word: |x| >= 2 or not finite)
    const unsigned any = __reduce_or_sync(0xffffffffu, acc);
    if ((any & 0x40000000u) && lane == 0) atomicCAS(A.suspect, 0, A.seg_index + 1);
    const double* up = s_lay[P];
    const double* uc = s_lay[1 - P];
    const double* vp = s_lay[2 + P];
    const double* vc = s_lay[3 - P];
    for (int j = lane; j < n; j += 32) {
        A.out[0][o + j] = up[j];
        A.out[1][o + j] = uc[j];
        A.out[2][o + j] = vp[j];
        A.out[3][o + j] = vc[j];
    }
}

}  // namespace hyg
