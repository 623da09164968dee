// fma_probe.cu — FP32 FFMA (register operands) vs packed FFMA2 vs DFMA
// throughput on the device (not product code).
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void k_tp(float* out, const float* coef, int iters) {
    const float b = coef[0], c = coef[1];          // registers, not immediates
    float a[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = threadIdx.x * 1e-6f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
            if (KIND == 0) {
                a[k] = fmaf(a[k], b, c);
                a[k + 1] = fmaf(a[k + 1], b, c);
            } else {
                unsigned long long x = (static_cast<unsigned long long>(__float_as_uint(a[k + 1])) << 32) | __float_as_uint(a[k]);
                const unsigned long long bb = (static_cast<unsigned long long>(__float_as_uint(b)) << 32) | __float_as_uint(b);
                const unsigned long long cc = (static_cast<unsigned long long>(__float_as_uint(c)) << 32) | __float_as_uint(c);
                asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(bb), "l"(cc));
                a[k] = __uint_as_float(static_cast<unsigned>(x));
                a[k + 1] = __uint_as_float(static_cast<unsigned>(x >> 32));
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dp(double* out, const double* coef, int iters) {
    const double b = coef[0], c = coef[1];
    double a[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = threadIdx.x * 1e-6 + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 16; ++k) a[k] = fma(a[k], b, c);
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* o; float* cf; double* od; double* cd;
    cudaMalloc(&o, 1 << 24); cudaMalloc(&cf, 64); cudaMalloc(&od, 1 << 25); cudaMalloc(&cd, 64);
    float hc[2] = {0.9999f, 1e-4f}; double hd[2] = {0.9999, 1e-4};
    cudaMemcpy(cf, hc, 8, cudaMemcpyHostToDevice); cudaMemcpy(cd, hd, 16, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096, blocks = nsm * 8, threads = 256;
    for (int kind = 0; kind < 3; ++kind) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (kind == 0) k_tp<0><<<blocks, threads>>>(o, cf, iters);
            else if (kind == 1) k_tp<1><<<blocks, threads>>>(o, cf, iters);
            else k_dp<<<blocks, threads>>>(od, cd, iters);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double flops = 2.0 * 16 * iters * double(blocks) * threads;
            if (rep) std::printf("%s: %.1f TFLOP/s\n", kind == 0 ? "FFMA (reg operands)" : kind == 1 ? "FFMA2 (packed)" : "DFMA", flops / ms / 1e9);
        }
    }
    return 0;
}
