// dv_probe.cu — dependent-chain latencies of the d(v) row pieces on the device
// (not product code): one warp, clock64 around N dependent iterations.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1703_10119_b200/csrc/k_dv_warp.cuh"

using namespace hyg;

template <int kind>
__global__ void k_probe(double* out, int iters) {
    __shared__ double s_tab[64];
    stage_exp_table(s_tab, threadIdx.x, blockDim.x);
    __syncthreads();
    const double p[4] = {0.91, 600.0, 10.0, 1.5};
    const DvParams q = dv_params(p);
    Groups g{0.1, 0.137, 3.76, 7.87e-3};
    const AnalyticRow rc = analytic_row(g, 0.01, 1e-3);
    const DvRow r = dv_row(rc);
    double x = 1.0 + threadIdx.x * 1e-9, y = 1.01, z = 0.99;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        switch (kind) {   // compile-time
            case 0: x = fma(x, 0.999999, 1e-7); break;
            case 1: x = 1.0 + 1e-4 * d_half(q, x + x, s_tab); break;               // d_half chain
            case 2: x = frcp(x + 1.0) + 0.5; break;                                  // frcp chain
            case 3: { double vn, un; dv_interior(r, x, y, z, 1.0, 1.0, 1.0, 2.0, 3.0, vn, un); x = vn; y = un; } break;
            case 4: { double vn, un; const double h = d_half(q, x + z, s_tab);
                      dv_interior(r, x, y, z, 1.0, 1.0, 1.0, h, h, vn, un); x = vn; y = un; } break;
            case 5: x = __shfl_up_sync(0xffffffffu, x, 1) * 0.999 + 1e-3; break;
            case 6: { __shared__ double sx[64]; sx[threadIdx.x] = x; __syncthreads(); x = sx[(threadIdx.x + 1) % 32] * 0.999 + 1e-3; } break;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[kind] = double(t1 - t0) / iters;
    out[16 + threadIdx.x] = x + y;
}

int main() {
    double* d;
    cudaMalloc(&d, 8192 * sizeof(double));
    const char* names[] = {"DFMA", "d_half (fexp)", "frcp + add", "dv_interior (v->v)", "d_half + dv_interior", "SHFL + FMA", "STS+bar+LDS+FMA"};
    void (*ks[])(double*, int) = {k_probe<0>, k_probe<1>, k_probe<2>, k_probe<3>, k_probe<4>, k_probe<5>, k_probe<6>};
    for (int k = 0; k < 7; ++k) {
        ks[k]<<<1, 32>>>(d, 20000);
        cudaDeviceSynchronize();
        double h;
        cudaMemcpy(&h, d + k, sizeof h, cudaMemcpyDeviceToHost);
        std::printf("%-24s %7.1f cycles per iteration\n", names[k], h);
    }
    return 0;
}
