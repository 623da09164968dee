// k_tiled.cuh — K3: temporally blocked DF march of one long wall with the
// analytic d(v) functor (configs[4]: N = 2^26 nodes).
//
// Replaces, for a single very long wall, the per-step stream of
// df_step_nonlinear (/root/reference/proj/src/wall.cpp:196-264) + StarTables
// (wall.cpp:89-138): the per-step kernel moves 48 B per node-update through
// HBM.  Here a CTA loads a tile of T nodes plus S halo nodes on each side
// (both layers of both fields) into shared memory, advances S steps there and
// writes the T owned nodes back: 64 B per node per S steps plus the halo, i.e.
// (32 (T + 2S) + 32 T) / (T S) ~ 4 B per update at T = 1024, S = 16.
//
// Exactness: at step k only nodes whose three-level stencil is still valid
// are computed — the window shrinks by one node per side and step
// ([k, W-k) in local indices; a real face node stays in the window since its
// row needs the interior neighbour only).  Every computed value is therefore
// the value the untiled march produces; the shrunk-away halo is discarded.
// Half-node coefficients d(v) are computed once per half node and step into
// shared memory (the per-step kernel evaluates each twice).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "k_nonlinear.cuh"

namespace hyg {

struct TiledArgs {
    int64_t n;                 // nodes of the wall
    int steps;                 // <= S
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
};

template <int T, int S, int THREADS>
__global__ void __launch_bounds__(THREADS) k_df_analytic_tiled(const TiledArgs A) {
    constexpr int W = T + 2 * S;
    extern __shared__ double sm[];           // lay[4][W], kp[W]
    double* lay[4] = {sm, sm + W, sm + 2 * W, sm + 3 * W};
    double* kp = sm + 4 * W;                 // kp[i]: half node between local i and i+1
    if (*A.stop) return;
    const int tid = threadIdx.x;
    const int64_t n = A.n;
    const int64_t g0 = static_cast<int64_t>(blockIdx.x) * T - S;   // global index of local 0
    for (int i = tid; i < W; i += THREADS) {
        const int64_t gi = g0 + i;
        const bool real = gi >= 0 && gi < n;
#pragma unroll
        for (int f = 0; f < 4; ++f) lay[f][i] = real ? A.in[f][gi] : 1.0;
    }
    const int lmin = static_cast<int>(g0 < 0 ? -g0 : 0);            // first real local node
    const int lmax = static_cast<int>(n - g0 < W ? n - g0 : W);      // one past the last
    const bool left_face = g0 <= 0;                                 // global node 0 is local -g0
    const bool right_face = n - 1 - g0 < W;                         // global n-1 is local n-1-g0
    const double p[4] = {A.p[0], A.p[1], A.p[2], A.p[3]};
    const AnalyticRow rc = analytic_row(A.groups, A.dx, A.dt);
    unsigned acc = 0;
    int P = 0;     // up = lay[P], uc = lay[1-P], vp = lay[2+P], vc = lay[3-P]
    __syncthreads();
    for (int k = 1; k <= A.steps; ++k) {
        double* up = lay[P];
        const double* uc = lay[1 - P];
        double* vp = lay[2 + P];
        const double* vc = lay[3 - P];
        const int lo = left_face ? lmin : k;
        const int hi = right_face ? lmax : W - k;
        const int h0 = max(lo - 1, lmin), h1 = min(hi, lmax - 1);
        for (int i = h0 + tid; i < h1; i += THREADS) kp[i] = d_of(p, 0.5 * (vc[i] + vc[i + 1]));
        __syncthreads();
        const Ambient* row = A.table + static_cast<size_t>(k - 1) * A.n_channels;
        for (int j = lo + tid; j < hi; j += THREADS) {
            const int64_t gj = g0 + j;
            double vn, un;
            if (gj == 0) {
                analytic_face(rc, A.bl, row[A.chl], vp[j], up[j], vc[j + 1], uc[j + 1], d_of(p, vc[j]), kp[j],
                              vn, un);
            } else if (gj == n - 1) {
                analytic_face(rc, A.br, row[A.chr], vp[j], up[j], vc[j - 1], uc[j - 1], d_of(p, vc[j]),
                              kp[j - 1], vn, un);
            } else {
                analytic_interior(rc, vp[j], up[j], vc[j - 1], vc[j + 1], uc[j - 1], uc[j + 1], kp[j - 1], kp[j],
                                  vn, un);
            }
            acc |= static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn));
            vp[j] = vn;
            up[j] = un;
        }
        __syncthreads();
        P ^= 1;
    }
    const unsigned any = __reduce_or_sync(0xffffffffu, acc);
    if ((any & 0x40000000u) && (tid % 32) == 0) atomicCAS(A.suspect, 0, A.seg_index + 1);
    const double* fin[4] = {lay[P], lay[1 - P], lay[2 + P], lay[3 - P]};
    for (int i = S + tid; i < S + T; i += THREADS) {
        const int64_t gi = g0 + i;
        if (gi >= n) break;
#pragma unroll
        for (int f = 0; f < 4; ++f) A.out[f][gi] = fin[f][i];
    }
}

}  // namespace hyg
