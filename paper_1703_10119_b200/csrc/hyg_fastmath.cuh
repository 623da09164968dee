// hyg_fastmath.cuh — short-latency exp and reciprocal for the d(v) rows.
//
// Measured on the B200 (tools/latency_probe.cu): a dependent DFMA is 8.3
// cycles, but libdevice exp(double) is 166 and a double division 132 — they
// set the step latency of the single-wall march (configs[0]) and most of the
// instruction count of the long-wall march (configs[4]).
//
// fexp (table-driven, 10 FP64 instructions): x = (64 k + j) ln2/64 + r with
// k, j from one FMA against the 1.5*2^52 shifter (the rounded multiple sits
// in the low word, no float->int conversion), Cody–Waite reduction with ln2/64
// split in two (kd * L_HI exact for |kd| < 2^21), |r| <= ln2/128; then
// exp(x) = 2^k T_j (1 + s), T_j = 2^(j/64) correctly rounded (64-entry table,
// staged in shared memory by the kernels), s = r + r^2/2 + ... + r^5/120
// (truncation < 3.5e-17 relative), the last step one FMA T + T s.  The scale
// 2^k goes into T_j's exponent field by an integer add.  Error <= ~1.5 ulp.
// |x| >= 708 is resolved on the integer pipe: 0 below, +inf above (glibc
// overflows at 709.78), NaN propagates.  The reference uses glibc exp; a few
// ulp in d(v) is ~1e-16 relative in a coefficient, far inside the 1e-10 parity
// tolerance.
//
// frcp: rcp.approx.ftz.f64 (~23 bits), then y (1 + e + e^2) with e = 1 - d y
// (3 FMAs; the cubic term e^3 ~ 2^-66 is far below an ulp) -> ~1 ulp.
#pragma once
#include <cuda_runtime.h>

namespace hyg {

// 2^(j/64), j = 0..63, correctly rounded (generated with 60-digit decimal arithmetic)
__device__ __constant__ const double kExp2Tab64[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0,
};

// exp(x) for -708 <= x <= 709 (no special cases; see fexp)
__device__ __forceinline__ double fexp_core(double x, const double* tab) {
    constexpr double kShift = 6755399441055744.0;                  // 1.5 * 2^52
    constexpr double kInvL = 92.332482616893658;                   // 64 / ln 2
    constexpr double kLHi = 0x1.62e42fee00000p-7;                  // ln2_hi / 64 (32 significant bits)
    constexpr double kLLo = 0x1.a39ef35793c76p-39;                 // ln2_lo / 64
    const double s = fma(x, kInvL, kShift);
    const double kd = s - kShift;
    const int k = __double2loint(s);                               // two's complement kd
    double r = fma(kd, -kLHi, x);
    r = fma(kd, -kLLo, r);
    const double r2 = r * r;
    const double c45 = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    const double c23 = fma(r, 1.0 / 6.0, 0.5);
    const double q = fma(r2, c45, c23);                            // 1/2 + r/6 + r^2/24 + r^3/120
    const double sm = fma(r2, q, r);                               // exp(r) - 1
    const double t = tab[k & 63];
    const double ts = __hiloint2double(__double2hiint(t) + static_cast<int>(static_cast<unsigned>(k >> 6) << 20),
                                       __double2loint(t));
    return fma(ts, sm, ts);
}

__device__ __forceinline__ double fexp(double x, const double* tab) {
    const double y = fexp_core(x, tab);
    // |x| >= 708, inf or NaN: integer tests and selects, no branch (a branch
    // per exp would split the caller's independent chains into basic blocks)
    const unsigned long long ax = static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7fffffffffffffffull;
    const bool big = ax >= 0x4086200000000000ull;
    const bool nan = ax > 0x7ff0000000000000ull;
    double ys = __double_as_longlong(x) < 0 ? 0.0 : __longlong_as_double(0x7ff0000000000000ll);
    ys = nan ? x : ys;
    return big ? ys : y;
}

__device__ __forceinline__ double frcp(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    const double e = fma(-d, y, 1.0);                  // |e| <= ~2^-22
    return fma(y, fma(e, e, e), y);                    // y (1 + e + e^2): error ~e^3
}

// exp(x) as a term ADDED TO A VALUE >= 2^-200 in magnitude (the d(v) half
// node: 1 + p0 v + p1 exp(x), x = -p2 (v - p3)^2 <= 0): x is clamped at -708,
// where exp is below 2^-1021 and vanishes in the sum exactly as the exact 0
// would, so the sum rounds bit for bit as with fexp.  NaN/inf states reach
// the sum through its p0 v term, so no select is needed: one DMNMX instead
// of fexp's integer tests and three selects.
__device__ __forceinline__ double fexp_addend(double x, const double* tab) {
    return fexp_core(fmax(x, -708.0), tab);
}

}  // namespace hyg
