// dfma_operand_probe.cu — what bounds K1's FP64 pipe utilisation (not product code).
// DFMA throughput per SM as a function of resident warps, operand reuse and instruction
// mix: (A) 16 chains a = fma(a, b, c) with b, c shared by every instruction (the peak probe
// of bench.py / hyg_probe_fp64_peak), (B) the same with three distinct register operands per
// instruction, (C) K1's interior rows — 2 DADD + 5 DFMA per node-update on 16 nodes x 4 layers
// in registers — without shuffles, face row, guard or forcing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -o tools/_ringvar/dfma_probe tools/dfma_operand_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_a(double* out, const double* coef, int iters) {
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

__global__ void k_b(double* out, const double* coef, int iters) {
    double a[16], b[16], c[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        a[k] = threadIdx.x * 1e-6 + k;
        b[k] = coef[0] + 1e-9 * k;
        c[k] = coef[1] + 1e-9 * (k + threadIdx.x);
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 16; ++k) a[k] = fma(b[k], c[(k + 5) & 15], a[k]);   // three distinct registers, no reuse slot
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += a[k] + b[k] * c[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_c(double* out, const double* coef, int iters) {
    constexpr int N = 16;
    const double cb = coef[2], csu = coef[3], csv = coef[4];
    double up[N], uc[N], vp[N], vc[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        up[k] = uc[k] = 1.0 + 1e-3 * ((threadIdx.x + k) % 7);
        vp[k] = vc[k] = 1.0 + 1e-3 * ((threadIdx.x + 3 * k) % 5);
    }
    auto step = [&](double (&vP)[N], double (&vC)[N], double (&uP)[N], double (&uC)[N]) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double sv = vC[(j + N - 1) % N] + vC[(j + 1) % N];
            const double su = uC[(j + N - 1) % N] + uC[(j + 1) % N];
            const double d = fma(-2.0, vP[j], sv);
            const double du = fma(-2.0, uP[j], su);
            vP[j] = fma(cb, d, vP[j]);
            uP[j] = fma(csv, d, fma(csu, du, uP[j]));
        }
    };
    for (int i = 0; i < iters; i += 2) {
        step(vp, vc, up, uc);
        step(vc, vp, uc, up);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) s += up[k] + uc[k] + vp[k] + vc[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// (D) the same with K1's per-step extras, one bit each: 1 the neighbour exchange by shuffles
// (16-lane groups, last lane reversed), 2 the face-capable row of register 0, 4 the fast guard
// (OR of the new values' high words), 8 the per-step ambient scalars from shared memory, 16 the
// guard on the step's input layer instead (no dependency on fresh FP64 results)
template <int BITS>
__global__ void __launch_bounds__(128, 2) k_d(double* out, const double* coef, int iters) {
    constexpr int N = 16;
    constexpr unsigned FULL = 0xffffffffu;
    __shared__ double s_amb[128 * 4];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) s_amb[i] = 1.0 + 1e-6 * i;
    __syncthreads();
    const double cb = coef[2], csu = coef[3], csv = coef[4];
    const double fb = coef[2] * 0.9, fe = 0.01, fcsu = coef[3] * 0.9, fctu = 0.02, fcsv = coef[4] * 0.9, fctv = 0.001;
    const int sub = threadIdx.x % 16;
    const bool first = sub == 0, rev = sub == 15, mirror0 = first || rev;
    double up[N], uc[N], vp[N], vc[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        up[k] = uc[k] = 1.0 + 1e-3 * ((threadIdx.x + k) % 7);
        vp[k] = vc[k] = 1.0 + 1e-3 * ((threadIdx.x + 3 * k) % 5);
    }
    unsigned acc = 0;
    bool bad = false;
    auto step = [&](double (&vP)[N], double (&vC)[N], double (&uP)[N], double (&uC)[N], int k) {
        double vx0 = vC[N - 1], ux0 = uC[N - 1], vx1 = vC[0], ux1 = uC[0];
        if (BITS & 1) {
            const double vs = rev ? vC[N - 1] : vC[0], us = rev ? uC[N - 1] : uC[0];
            const double vup = __shfl_up_sync(FULL, vC[N - 1], 1, 16), uup = __shfl_up_sync(FULL, uC[N - 1], 1, 16);
            const double vdn = __shfl_down_sync(FULL, vs, 1, 16), udn = __shfl_down_sync(FULL, us, 1, 16);
            vx0 = mirror0 ? vC[1] : vup; ux0 = mirror0 ? uC[1] : uup;
            vx1 = rev ? vup : vdn; ux1 = rev ? uup : udn;
        }
        double u_inf = 1.0, v_inf = 1.0;
        if (BITS & 8) { u_inf = s_amb[(k & 127) * 4 + (first ? 0 : 2)]; v_inf = s_amb[(k & 127) * 4 + (first ? 1 : 3)]; }
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double sv = (j == 0 ? vx0 : vC[j - 1]) + (j == N - 1 ? vx1 : vC[j + 1]);
            const double su = (j == 0 ? ux0 : uC[j - 1]) + (j == N - 1 ? ux1 : uC[j + 1]);
            const double d = fma(-2.0, vP[j], sv);
            const double du = fma(-2.0, uP[j], su);
            double vn, un;
            if ((BITS & 2) && j == 0) {
                const double t = v_inf - vP[0], tu = u_inf - uP[0];
                vn = fma(fe, t, fma(fb, d, vP[0]));
                un = fma(fctv, t, fma(fcsv, d, fma(fctu, tu, fma(fcsu, du, uP[0]))));
            } else {
                vn = fma(cb, d, vP[j]);
                un = fma(csv, d, fma(csu, du, uP[j]));
            }
            if (BITS & 4) acc |= static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn));
            // 32: one value per OR (v only); 64: every other node (both fields); 128: pairs of nodes through
            // one packed word: PRMT gathers the top bytes of un, vn of two nodes, one OR per two nodes
            if (BITS & 32) acc |= static_cast<unsigned>(__double2hiint(vn));
            if ((BITS & 64) && (j & 1)) acc |= static_cast<unsigned>(__double2hiint(un)) | static_cast<unsigned>(__double2hiint(vn));
            // 256: the guard as unsigned compares into a predicate (one register read per value, no
            // accumulator read): hi >= 0x40000000 as unsigned <=> |x| >= 2, not finite, or negative
            if (BITS & 256) bad |= (static_cast<unsigned>(__double2hiint(un)) >= 0x40000000u) |
                                   (static_cast<unsigned>(__double2hiint(vn)) >= 0x40000000u);
            // 16: the guard one step late — on the step's INPUT layer, whose values are a step old
            if (BITS & 16) acc |= static_cast<unsigned>(__double2hiint(uC[j])) | static_cast<unsigned>(__double2hiint(vC[j]));
            vP[j] = vn;
            uP[j] = un;
        }
    };
    for (int i = 0; i < iters; i += 2) {
        step(vp, vc, up, uc, i);
        step(vc, vp, uc, up, i + 1);
    }
    double s = (acc & 1) + (bad ? 1.0 : 0.0);
#pragma unroll
    for (int k = 0; k < N; ++k) s += up[k] + uc[k] + vp[k] + vc[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
void run(const char* name, K kern, int threads, int warps_per_sm, int iters, double fp64_per_iter, double flop_per_iter,
         double* o, const double* cd, int nsm) {
    const int blocks = nsm * warps_per_sm * 32 / threads;
    cudaFuncAttributes at;
    cudaFuncGetAttributes(&at, kern);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, 0);
    if (occ * threads / 32 < warps_per_sm) {
        std::printf("%-34s %2d warps/SM: does not fit (%d regs)\n", name, warps_per_sm, at.numRegs);
        return;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(o, cd, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) best = ms < best ? ms : best;
    }
    const double n = double(blocks) * threads * iters;
    // one FP64 instruction of a warp occupies the SM sub-partition's pipe for 2 cycles (16 lanes)
    std::printf("%-34s %2d warps/SM %3d regs: %6.2f TFLOP/s, %5.1f %% of the FP64 issue slots (1.965 GHz)\n", name, warps_per_sm,
                at.numRegs, n * flop_per_iter / best / 1e9, 100.0 * n * fp64_per_iter / 32.0 * 2.0 / (best * 1e-3) / (nsm * 4 * 1.965e9));
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double *o, *cd;
    cudaMalloc(&o, sizeof(double) * nsm * 64 * 32);
    cudaMalloc(&cd, 64);
    const double hd[5] = {0.9999, 1e-4, 0.2, 0.3, 0.01};
    cudaMemcpy(cd, hd, sizeof hd, cudaMemcpyHostToDevice);
    for (int w : {8, 12, 16, 32, 64}) run("A: fma(a, b, c), b c shared", k_a, 256, w, 8192, 16, 32, o, cd, nsm);
    for (int w : {8, 12, 16}) run("B: fma(b[k], c[k'], a[k]) distinct", k_b, 256, w, 8192, 16, 32, o, cd, nsm);
    for (int w : {8}) run("C: K1 interior rows, 16 nodes", k_c<2>, 128, w, 4096, 16 * 7, 16 * 12, o, cd, nsm);
    for (int w : {12}) run("C: K1 interior rows, 16 nodes", k_c<3>, 128, w, 4096, 16 * 7, 16 * 12, o, cd, nsm);
    for (int w : {16}) run("C: K1 interior rows, 16 nodes", k_c<4>, 128, w, 4096, 16 * 7, 16 * 12, o, cd, nsm);
    run("D0: C in K1's loop form", k_d<0>, 128, 8, 4096, 16 * 7, 16 * 12, o, cd, nsm);
    run("D1: + shuffles", k_d<1>, 128, 8, 4096, 16 * 7, 16 * 12, o, cd, nsm);
    run("D2: + face row", k_d<2>, 128, 8, 4096, 16 * 7 + 6, 16 * 12, o, cd, nsm);
    run("D4: + guard", k_d<4>, 128, 8, 4096, 16 * 7, 16 * 12, o, cd, nsm);
    run("D8: + ambient LDS", k_d<8>, 128, 8, 4096, 16 * 7, 16 * 12, o, cd, nsm);
    run("D3: + shuffles + face", k_d<3>, 128, 8, 4096, 16 * 7 + 6, 16 * 12, o, cd, nsm);
    run("D7: + shuffles + face + guard", k_d<7>, 128, 8, 4096, 16 * 7 + 6, 16 * 12, o, cd, nsm);
    run("D15: all (K1's step)", k_d<15>, 128, 8, 4096, 16 * 7 + 6, 16 * 12, o, cd, nsm);
    run("D16: + lagged guard", k_d<16>, 128, 8, 4096, 16 * 7, 16 * 12, o, cd, nsm);
    run("D32: + guard, v only", k_d<32>, 128, 8, 4096, 16 * 7, 16 * 12, o, cd, nsm);
    run("D64: + guard, every other node", k_d<64>, 128, 8, 4096, 16 * 7, 16 * 12, o, cd, nsm);
    run("D27: all with the lagged guard", k_d<27>, 128, 8, 4096, 16 * 7 + 6, 16 * 12, o, cd, nsm);
    run("D256: + predicate guard", k_d<256>, 128, 8, 4096, 16 * 7, 16 * 12, o, cd, nsm);
    run("D267: all with the predicate guard", k_d<267>, 128, 8, 4096, 16 * 7 + 6, 16 * 12, o, cd, nsm);
    return 0;
}
