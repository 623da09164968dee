// x2_variants.cu — layout/occupancy probe for the packed fp32 K1 (not product
// code): k_df_coupled_x2 variants vs the scalar k_df_coupled<float> on
// cfg2-like random walls (65,536 x 256, 4096 steps), values compared.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "k_coupled_x2.cuh"

using namespace hyg;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); std::exit(1);} } while (0)

__global__ void k_coef(int B, double dx, double dt, const Groups* g, const Biot* b, WallCoef* c) {
    int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w < B) coupled_coef(g[w], dx, dt, b[2 * w], b[2 * w + 1], c[w]);
}

template <typename Real> struct BufsT { Real* in[4]; Real* out[4]; };
using Bufs = BufsT<double>;

template <bool X2, int LPW, int NPT, int WARPS, int MINB>
float run(const char* name, CoupledSegArgs<float> a, BufsT<float>& b, int B, int steps, std::vector<float>* result) {
    constexpr int CHUNK = 128;
    void (*kern)(const CoupledSegArgs<float>);
    if constexpr (X2) kern = k_df_coupled_x2<LPW, NPT, WARPS, CHUNK, false, MINB>;
    else kern = k_df_coupled<float, LPW, NPT, WARPS, CHUNK, false, false, MINB>;
    const int smem = CHUNK * a.n_channels * sizeof(Ambient);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaFuncAttributes attr;
    cudaFuncGetAttributes(&attr, kern);
    const int wpc = WARPS * 32 / LPW;
    const int grid = (B + wpc - 1) / wpc;
    for (int k = 0; k < 4; ++k) { a.in[k] = b.in[k]; a.out[k] = b.out[k]; }
    a.nsteps = steps;
    kern<<<grid, WARPS * 32, smem>>>(a);   // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 3;
    for (int r = 0; r < reps; ++r) kern<<<grid, WARPS * 32, smem>>>(a);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double rate = (double)B * 256 * steps / (ms * 1e-3);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, WARPS * 32, smem);
    std::printf("%-26s regs %3d  warps/SM %2d  %.3f ms  %.3e upd/s\n", name, attr.numRegs, occ * WARPS, ms, rate);
    if (result) {
        result->resize((size_t)B * 256 * 4);
        for (int k = 0; k < 4; ++k)
            CK(cudaMemcpy(result->data() + (size_t)k * B * 256, b.out[k], (size_t)B * 256 * sizeof(float),
                          cudaMemcpyDeviceToHost));
    }
    return ms;
}

int main(int argc, char** argv) {
    const int B = 65536, n = 256, steps = argc > 1 ? atoi(argv[1]) : 4096;
    const double dx = 1.0 / (n - 1), dt = 1e-3;
    std::mt19937_64 rng(1);
    auto lu = [&](double lo, double hi) {
        std::uniform_real_distribution<double> d(std::log(lo), std::log(hi));
        return std::exp(d(rng));
    };
    std::vector<Groups> g(B);
    std::vector<Biot> bi(2 * B);
    for (int w = 0; w < B; ++w) {
        g[w] = Groups{lu(3.7e-5, 0.35), lu(0.018, 1.4), lu(1.1e-3, 10.4), lu(1.7e-5, 6.6e-3)};
        bi[2 * w] = Biot{lu(200, 2e4), lu(1.25, 25), lu(0.1, 2.0)};
        bi[2 * w + 1] = Biot{lu(30, 3e3), lu(0.4, 8), lu(0.01, 0.3)};
    }
    const int nch = 2;
    std::vector<Ambient> tab((size_t)steps * nch);
    double t = 0;
    for (int s = 0; s < steps; ++s) {
        tab[s * nch] = Ambient{1.0 + 0.02 * std::sin(2 * M_PI * t / 24), 1.0 + 0.2 * std::sin(2 * M_PI * t / 24), 0, 0};
        tab[s * nch + 1] = Ambient{1.0, 1.0, 0, 0};
        t += dt;
    }
    std::normal_distribution<double> nd(0.0, 0.01);
    std::vector<double> init((size_t)B * n);
    for (auto& x : init) x = 1.0 + nd(rng);
    Groups* dg; Biot* db; WallCoef* dc; Ambient* dtab; int *dchan, *dflag; unsigned long long* dkey;
    CK(cudaMalloc(&dg, B * sizeof(Groups)));
    CK(cudaMalloc(&db, 2 * B * sizeof(Biot)));
    CK(cudaMalloc(&dc, B * sizeof(WallCoef)));
    CK(cudaMalloc(&dtab, tab.size() * sizeof(Ambient)));
    CK(cudaMalloc(&dchan, 2 * B * sizeof(int)));
    CK(cudaMalloc(&dflag, 4));
    CK(cudaMalloc(&dkey, 8));
    std::vector<int> chan(2 * B);
    for (int w = 0; w < B; ++w) { chan[2 * w] = 0; chan[2 * w + 1] = 1; }
    CK(cudaMemcpy(dg, g.data(), B * sizeof(Groups), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, bi.data(), 2 * B * sizeof(Biot), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dtab, tab.data(), tab.size() * sizeof(Ambient), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dchan, chan.data(), 2 * B * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemset(dflag, 0, 4));
    k_coef<<<(B + 127) / 128, 128>>>(B, dx, dt, dg, db, dc);
    Bufs b;
    for (int k = 0; k < 4; ++k) {
        CK(cudaMalloc(&b.in[k], (size_t)B * n * 8));
        CK(cudaMalloc(&b.out[k], (size_t)B * n * 8));
        CK(cudaMemcpy(b.in[k], init.data(), (size_t)B * n * 8, cudaMemcpyHostToDevice));
    }
    CoupledSegArgs<double> a{};
    a.n_walls = B;
    a.n_channels = nch;
    a.divergence_norm = 1e3;
    a.coef = dc;
    a.chan = dchan;
    a.table = dtab;
    a.stop = dflag;
    a.suspect = dflag;
    a.fail_key = dkey;
    {
        // fp32 deviations from 1 (the cfg2 state), same walls and forcing
        BufsT<float> bf;
        std::vector<float> dev(init.size());
        for (size_t i = 0; i < init.size(); ++i) dev[i] = static_cast<float>(init[i] - 1.0);
        for (int k = 0; k < 4; ++k) {
            CK(cudaMalloc(&bf.in[k], (size_t)B * n * 4));
            CK(cudaMalloc(&bf.out[k], (size_t)B * n * 4));
            CK(cudaMemcpy(bf.in[k], dev.data(), (size_t)B * n * 4, cudaMemcpyHostToDevice));
        }
        CoupledSegArgs<float> af{};
        af.n_walls = B; af.n_channels = nch; af.divergence_norm = 1e3; af.coef = dc; af.chan = dchan;
        af.table = dtab; af.stop = dflag; af.suspect = dflag; af.fail_key = dkey;
        std::vector<float> rf, gf;
        auto checkf = [&](const char* nm) {
            double m = 0;
            for (size_t i = 0; i < rf.size(); ++i) m = std::max(m, (double)std::fabs(rf[i] - gf[i]));
            std::printf("    %s max |diff| vs prod %.3e\n", nm, m);
        };
        run<false, 8, 32, 4, 0>("scalar 8x32 (prod before)", af, bf, B, steps, &rf);
        run<true, 8, 32, 4, 0>("x2 8x32 w4", af, bf, B, steps, &gf); checkf("x2 8x32");
        run<true, 16, 16, 4, 0>("x2 16x16 w4", af, bf, B, steps, &gf); checkf("x2 16x16");
        run<true, 16, 16, 4, 3>("x2 16x16 w4 minb3", af, bf, B, steps, &gf); checkf("x2 16x16 minb3");
        run<true, 16, 16, 8, 0>("x2 16x16 w8", af, bf, B, steps, &gf); checkf("x2 16x16 w8");
        run<true, 32, 8, 4, 0>("x2 32x8 w4", af, bf, B, steps, &gf); checkf("x2 32x8");
        run<true, 32, 8, 4, 4>("x2 32x8 w4 minb4", af, bf, B, steps, &gf); checkf("x2 32x8 minb4");
        return 0;
    }
    return 0;
}
