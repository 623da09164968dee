// k_tiled.cuh — K3: temporally blocked DF march of one long wall with the
// analytic d(v) functor (configs[4]: N = 2^26 nodes).
//
// Replaces, for a single very long wall, the per-step stream of
// df_step_nonlinear (/root/reference/proj/src/wall.cpp:196-264) + StarTables
// (wall.cpp:89-138): the per-step kernel moves 48 B per node-update through
// HBM.  Here a CTA loads a tile of T nodes plus S halo nodes on each side
// (both layers of both fields) into shared memory, advances S steps there and
// writes the T owned nodes back: 64 B per node per S steps plus the halo, i.e.
// (32 (T + 2S) + 32 T) / (T S) ~ 4 B per update at T = 992, S = 16.
//
// Exactness: at step k only nodes whose three-level stencil is still valid
// are computed — the window shrinks by one node per side and step
// ([k, W-k) in local indices; a real face node stays in the window since its
// row needs the interior neighbour only).  Every computed value is therefore
// the value the untiled march produces; the shrunk-away halo is discarded.
// Half-node coefficients d(v) are computed once per half node and step into
// shared memory (the per-step kernel evaluates each twice).
//
// Shape: W = T + 2S = 1024 = 4 x 256 threads, each thread owning 4 window
// slots (unrolled: independent chains interleave, no imbalance at the
// barriers); the layer roles rotate by unrolling two steps so every shared
// access has a compile-time base (a runtime-indexed pointer table would turn
// them into generic loads).
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

template <int W, int THREADS>
struct TileCtx {
    double (*lay)[W];          // [4][W] in shared memory
    double* kp;                // [W]
    const double* tab;         // [64] exp table
    int lmin, lmax, lf, rf;    // real-node range, face slots (-1 if absent)
    int tid;
};

// One step with compile-time roles: layer n-1 in (UP, VP) becomes layer n+1.
template <int W, int THREADS, int UP, int UC, int VP, int VC>
__device__ __forceinline__ void tiled_step(const TileCtx<W, THREADS>& c, const TiledArgs& A,
                                           const AnalyticRow& rc, const double (&p)[4], int k,
                                           unsigned& acc) {
    constexpr int NQ = W / THREADS;
    double* up = c.lay[UP];
    double* vp = c.lay[VP];
    const double* uc = c.lay[UC];
    const double* vc = c.lay[VC];
    const int lo = c.lf >= 0 ? c.lf : k;
    const int hi = c.rf >= 0 ? c.rf + 1 : W - k;
    const int h0 = max(lo - 1, c.lmin), h1 = min(hi, c.lmax - 1);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int i = c.tid + q * THREADS;
        const double kv = d_of(p, 0.5 * (vc[i] + vc[min(i + 1, W - 1)]), c.tab);
        if (i >= h0 && i < h1) c.kp[i] = kv;
    }
    __syncthreads();
    // interior rows, branch-free over the thread's slots (out-of-window slots
    // compute on clamped neighbours and are not stored): the slots' chains
    // interleave
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int j = c.tid + q * THREADS;
        const bool valid = j >= lo && j < hi && j != c.lf && j != c.rf;
        const int jl = max(j - 1, 0), jr = min(j + 1, W - 1);
        double vn, un;
        analytic_interior(rc, vp[j], up[j], vc[jl], vc[jr], uc[jl], uc[jr], c.kp[jl], c.kp[j], vn, un);
        if (valid) {
            acc |= static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn));
            vp[j] = vn;
            up[j] = un;
        }
    }
    if (c.lf >= 0 || c.rf >= 0) {   // the first and the last tile hold the faces
        const Ambient* row = A.table + static_cast<size_t>(k - 1) * A.n_channels;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int j = c.tid + q * THREADS;
            if (j != c.lf && j != c.rf) continue;
            const bool left = j == c.lf;
            const int jn = left ? j + 1 : j - 1;
            double vn, un;
            analytic_face(rc, left ? A.bl : A.br, row[left ? A.chl : A.chr], vp[j], up[j], vc[jn], uc[jn],
                          d_of(p, vc[j], c.tab), c.kp[left ? j : j - 1], vn, un);
            acc |= static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn));
            vp[j] = vn;
            up[j] = un;
        }
    }
    __syncthreads();
}

template <int T, int S, int THREADS>
__global__ void __launch_bounds__(THREADS) k_df_analytic_tiled(const TiledArgs A) {
    constexpr int W = T + 2 * S;
    static_assert(W % THREADS == 0, "window must split evenly over the threads");
    extern __shared__ double sm[];           // lay[4][W], kp[W]
    __shared__ double s_tab[64];
    if (*A.stop) return;
    stage_exp_table(s_tab, threadIdx.x, THREADS);
    TileCtx<W, THREADS> c;
    c.lay = reinterpret_cast<double(*)[W]>(sm);
    c.kp = sm + 4 * W;
    c.tab = s_tab;
    c.tid = threadIdx.x;
    const int64_t n = A.n;
    const int64_t g0 = static_cast<int64_t>(blockIdx.x) * T - S;   // global index of local 0
#pragma unroll
    for (int q = 0; q < W / THREADS; ++q) {
        const int i = c.tid + q * THREADS;
        const int64_t gi = g0 + i;
        const bool real = gi >= 0 && gi < n;
#pragma unroll
        for (int f = 0; f < 4; ++f) c.lay[f][i] = real ? A.in[f][gi] : 1.0;
    }
    c.lmin = static_cast<int>(g0 < 0 ? -g0 : 0);               // first real local node
    c.lmax = static_cast<int>(n - g0 < W ? n - g0 : W);         // one past the last
    c.lf = g0 <= 0 ? c.lmin : -1;                               // global node 0
    c.rf = n - 1 - g0 < W ? static_cast<int>(n - 1 - g0) : -1;  // global node n-1
    const double p[4] = {A.p[0], A.p[1], A.p[2], A.p[3]};
    const AnalyticRow rc = analytic_row(A.groups, A.dx, A.dt);
    unsigned acc = 0;
    __syncthreads();
    int k = 1;
    for (; k + 1 <= A.steps; k += 2) {
        tiled_step<W, THREADS, 0, 1, 2, 3>(c, A, rc, p, k, acc);       // prev slots 0/2 -> n+1
        tiled_step<W, THREADS, 1, 0, 3, 2>(c, A, rc, p, k + 1, acc);
    }
    const bool odd = k <= A.steps;
    if (odd) tiled_step<W, THREADS, 0, 1, 2, 3>(c, A, rc, p, k, acc);
    const unsigned any = __reduce_or_sync(0xffffffffu, acc);
    if ((any & 0x40000000u) && (c.tid % 32) == 0) atomicCAS(A.suspect, 0, A.seg_index + 1);
    // roles after an even number of steps: up = 0, uc = 1, vp = 2, vc = 3; odd: swapped
    const int ru_p = odd ? 1 : 0, rv_p = odd ? 3 : 2;
#pragma unroll
    for (int q = 0; q < W / THREADS; ++q) {
        const int i = c.tid + q * THREADS;
        const int64_t gi = g0 + i;
        if (i < S || i >= S + T || gi >= n) continue;
        A.out[0][gi] = c.lay[ru_p][i];
        A.out[1][gi] = c.lay[1 - ru_p][i];
        A.out[2][gi] = c.lay[rv_p][i];
        A.out[3][gi] = c.lay[5 - rv_p][i];
    }
}

}  // namespace hyg
