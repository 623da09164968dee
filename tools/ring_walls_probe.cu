// Timing probe for K6 phase 2 (k_ring_walls, k_ring_split.cuh) on a cfg3-sized
// state (8,192 zones x 6 walls x 128 nodes): the library's kernel compiled alone
// (seconds), with RW_SKIP bits / RW_MINB / S from the command line of nvcc.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -DRW_SKIP=0 -DPROBE_S=8 \
//        -I paper_1703_10119_b200/csrc -o tools/_ringvar/rwp tools/ring_walls_probe.cu
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
    double *in[4], *out[4], *series, *table;
    WallCoef* coef;
    Attach* attach;
    int* stop;
    std::vector<double> ones(cells, 1.0);
    // argv[2]: byte skew between the eight arrays (carved from one allocation), 0: separate cudaMallocs
    const size_t skew = argc > 2 ? strtoull(argv[2], nullptr, 10) : 0;
    char* pool = nullptr;
    if (skew) cudaMalloc(&pool, 8 * (cells * 8 + skew) + (1 << 21));
    for (int f = 0; f < 4; ++f) {
        if (skew) {
            in[f] = reinterpret_cast<double*>(pool + (2 * f) * (cells * 8 + skew));
            out[f] = reinterpret_cast<double*>(pool + (2 * f + 1) * (cells * 8 + skew));
        } else {
            cudaMalloc(&in[f], cells * 8);
            cudaMalloc(&out[f], cells * 8);
        }
        cudaMemcpy(in[f], ones.data(), cells * 8, cudaMemcpyHostToDevice);
    }
    printf("in0 %p in1 %p out0 %p\n", (void*)in[0], (void*)in[1], (void*)out[0]);
    std::vector<double> ser(static_cast<size_t>(Z) * S * 2, 1.0), tab(S * 4, 1.0);
    cudaMalloc(&series, ser.size() * 8);
    cudaMemcpy(series, ser.data(), ser.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&table, tab.size() * 8);
    cudaMemcpy(table, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice);
    std::vector<WallCoef> wc(walls);
    Groups g{0.05, 0.04, 0.01, 0.1};
    Biot b{1.0, 2.0, 0.1};
    for (auto& w : wc) coupled_coef(g, 1.0 / (N - 1), 1e-3, b, b, w);
    cudaMalloc(&coef, sizeof(WallCoef) * walls);
    cudaMemcpy(coef, wc.data(), sizeof(WallCoef) * walls, cudaMemcpyHostToDevice);
    std::vector<Attach> at(2 * walls, Attach{0, 0});
    cudaMalloc(&attach, sizeof(Attach) * at.size());
    cudaMemcpy(attach, at.data(), sizeof(Attach) * at.size(), cudaMemcpyHostToDevice);
    cudaMalloc(&stop, 4);
    cudaMemset(stop, 0, 4);
    RingArgs a{};
    a.n_zones = Z; a.W = W; a.n = N; a.steps = S; a.coef = coef; a.attach = attach;
    a.table = reinterpret_cast<const Ambient*>(table); a.n_channels = 1; a.stop = stop; a.dt = 1e-3;
    auto k = k_ring_walls<8, PROBE_S>;
    const size_t smem = RingWallShape<8>::smem_doubles(S, 1, kRingWallWarps) * sizeof(double);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * kRingWallWarps, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int pairs = walls / 2, nblk = (pairs + kRingWallWarps - 1) / kRingWallWarps;
    int grid = per_sm * sms < nblk ? per_sm * sms : nblk;
    if (argc > 1) grid = atoi(argv[1]);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f, sum = 0;
    const int reps = 40;
    for (int r = 0; r < reps + 5; ++r) {
        for (int f = 0; f < 4; ++f) { a.in[f] = (r & 1) ? out[f] : in[f]; a.out[f] = (r & 1) ? in[f] : out[f]; }
        cudaEventRecord(e0);
        k<<<grid, 32 * kRingWallWarps, smem>>>(a, series, TiledMaps{}, TiledMaps{});
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 5) { best = ms < best ? ms : best; sum += ms; }
    }
    int flag = 0;
    cudaMemcpy(&flag, stop, 4, cudaMemcpyDeviceToHost);
    printf("RW_SKIP=%d MINB=%d S=%d grid=%d (%d/SM) smem=%zu: mean %.2f us best %.2f us  -> %.3e upd/s, %.2f TB/s  [%s, flag %d]\n",
           RW_SKIP, RW_MINB, S, grid, per_sm, smem, 1e3 * sum / reps, 1e3 * best, cells * double(S) / (sum / reps * 1e-3),
           cells * 64.0 / (sum / reps * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()), flag);
    return 0;
}
