// latency_probe.cu — dependent-chain latencies on the device (not product
// code): DFMA, DADD, exp(double), double division, __syncthreads, LDS.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_chain(double* out, int iters, int kind, double a, double b) {
    double x = 1.0 + threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        switch (kind) {
            case 0: x = fma(x, a, b); break;                       // DFMA
            case 1: x = x + b; break;                               // DADD
            case 2: x = exp(-x * a) + 0.5; break;                   // exp
            case 3: x = b / x + 0.5; break;                         // division
            case 4: { double e = x - 1.5; x = 1.0 + 0.91 * x + 600.0 * exp(-10.0 * e * e); x = 0.5 + x * 1e-3; } break;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[kind] = double(t1 - t0) / iters;
    out[8 + threadIdx.x] = x;
}

__global__ void k_sync(double* out, int iters) {
    __shared__ double s[1024];
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        s[threadIdx.x] = x;
        __syncthreads();
        x = s[(threadIdx.x + 1) % blockDim.x] * 0.999 + 1e-3;
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
    out[8 + threadIdx.x] = x;
}

int main() {
    double* d;
    cudaMalloc(&d, 8192 * sizeof(double));
    const char* names[] = {"DFMA", "DADD", "exp(double)+add", "division+add", "d(v) analytic"};
    const int iters = 100000;
    for (int k = 0; k < 5; ++k) {
        k_chain<<<1, 32>>>(d, iters, k, 0.999999, 1e-7);
        cudaDeviceSynchronize();
        double h;
        cudaMemcpy(&h, d + k, sizeof h, cudaMemcpyDeviceToHost);
        std::printf("%-18s %7.1f cycles per dependent op\n", names[k], h);
    }
    for (int t : {32, 128, 256}) {
        k_sync<<<1, t>>>(d, iters);
        cudaDeviceSynchronize();
        double h;
        cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
        std::printf("2x syncthreads + STS/LDS, %3d threads: %7.1f cycles per iteration\n", t, h);
    }
    return 0;
}
