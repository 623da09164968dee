// Timing probe for K6 phase 1 (k_ring_cone, k_ring_split.cuh) on a cfg3-sized ring
// (8,192 zones x 6 walls x 128 nodes): the library's kernel compiled alone, with
// RC_SKIP bits and the CTA shape from the command line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -DRC_SKIP=0 \
//        -I paper_1703_10119_b200/csrc -o tools/_ringvar/rcp tools/ring_cone_probe.cu
//   rcp [LB]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "k_ring_split.cuh"
#ifndef PROBE_S
#define PROBE_S 8
#endif
using namespace hyg;
int main(int argc, char** argv) {
    const int Z = 8192, W = 6, N = 128, S = PROBE_S, walls = Z * W;
    const size_t cells = static_cast<size_t>(walls) * N;
    double *in[4], *series, *table, *src, *zp, *zu[2], *zv[2];
    WallCoef* coef;
    int* stop;
    std::vector<double> ones(cells, 1.0);
    for (int f = 0; f < 4; ++f) {
        cudaMalloc(&in[f], cells * 8);
        cudaMemcpy(in[f], ones.data(), cells * 8, cudaMemcpyHostToDevice);
    }
    cudaMalloc(&series, static_cast<size_t>(Z) * S * 2 * 8);
    std::vector<double> tab(S * 4, 1.0), sr(S * 5, 0.0);
    cudaMalloc(&table, tab.size() * 8);
    cudaMemcpy(table, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&src, sr.size() * 8);
    cudaMemcpy(src, sr.data(), sr.size() * 8, cudaMemcpyHostToDevice);
    std::vector<double> zpar(static_cast<size_t>(Z) * kRingZP, 0.0);
    for (int z = 0; z < Z; ++z) {
        double* b = &zpar[static_cast<size_t>(z) * kRingZP];
        b[0] = 1.5; b[1] = 0.1; b[2] = 0.1; b[3] = 0.1; b[4] = 6; b[5] = 2; b[6] = 0;
        for (int q = 0; q < 6; ++q) { b[8 + 4 * q] = q; b[9 + 4 * q] = 0.01; b[10 + 4 * q] = 0.001; b[11 + 4 * q] = 0.01; }
        b[40] = (z + 1) % Z; b[44] = (z + Z - 1) % Z;
        b[41] = b[45] = 0.01; b[42] = b[46] = 0.01; b[43] = b[47] = 0.01;
    }
    cudaMalloc(&zp, zpar.size() * 8);
    cudaMemcpy(zp, zpar.data(), zpar.size() * 8, cudaMemcpyHostToDevice);
    for (int b = 0; b < 2; ++b) {
        cudaMalloc(&zu[b], Z * 8); cudaMalloc(&zv[b], Z * 8);
        cudaMemcpy(zu[b], ones.data(), Z * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(zv[b], ones.data(), Z * 8, cudaMemcpyHostToDevice);
    }
    std::vector<WallCoef> wc(walls);
    Groups g{0.05, 0.04, 0.01, 0.1};
    Biot bb{1.0, 2.0, 0.1};
    for (auto& w : wc) coupled_coef(g, 1.0 / (N - 1), 1e-3, bb, bb, w);
    cudaMalloc(&coef, sizeof(WallCoef) * walls);
    cudaMemcpy(coef, wc.data(), sizeof(WallCoef) * walls, cudaMemcpyHostToDevice);
    double *rowsT, *zpT;
    cudaMalloc(&rowsT, sizeof(double) * 12 * walls);
    k_ring_cone_rows<<<(walls + 127) / 128, 128>>>(walls, coef, rowsT);
    std::vector<double> zt(zpar.size());
    for (int z = 0; z < Z; ++z)
        for (int k = 0; k < kRingZP; ++k) zt[static_cast<size_t>(k) * Z + z] = zpar[static_cast<size_t>(z) * kRingZP + k];
    cudaMalloc(&zpT, zt.size() * 8);
    cudaMemcpy(zpT, zt.data(), zt.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&stop, 4);
    cudaMemset(stop, 0, 4);
    RingArgs a{};
    a.n_zones = Z; a.W = W; a.n = N; a.steps = S; a.coef = coef; a.zparams = zp;
    a.table = reinterpret_cast<const Ambient*>(table); a.n_channels = 1; a.src = src; a.n_sources = 1;
    a.stop = stop; a.dt = 1e-3;
    for (int f = 0; f < 4; ++f) a.in[f] = in[f];
    using Sh = RingConeShape<PROBE_S>;
    auto k = k_ring_cone<PROBE_S, 6, 2>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    const int rw = RingShape<8, PROBE_S>::row_width(1, 1);
    int lb = argc > 1 ? atoi(argv[1]) : 72;
    const int OB = lb - 2 * S, grid = (Z + OB - 1) / OB, threads = Sh::threads(lb, W);
    const size_t smem = Sh::smem_doubles(lb, W, rw) * sizeof(double);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f, sum = 0;
    const int reps = 40;
    for (int r = 0; r < reps + 5; ++r) {
        a.zu_in = zu[r & 1]; a.zv_in = zv[r & 1]; a.zu_out = zu[1 - (r & 1)]; a.zv_out = zv[1 - (r & 1)];
        cudaEventRecord(e0);
        k<<<grid, threads, smem>>>(a, series, lb, rowsT, zpT);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 5) { best = ms < best ? ms : best; sum += ms; }
    }
    int flag = 0;
    cudaMemcpy(&flag, stop, 4, cudaMemcpyDeviceToHost);
    printf("RC_SKIP=%d S=%d LB=%d grid=%d threads=%d smem=%zu: mean %.2f us best %.2f us [%s, flag %d]\n", RC_SKIP, S, lb, grid,
           threads, smem, 1e3 * sum / reps, 1e3 * best, cudaGetErrorString(cudaGetLastError()), flag);
    return 0;
}
