// hyg_fastmath.cuh — short-latency exp and reciprocal for the d(v) rows.
//
// Measured on the B200 (tools/latency_probe.cu): a dependent DFMA is 8.3
// cycles, but libdevice exp(double) is 166 and a double division 132 — they
// set the step latency of the single-wall march (configs[0]) and most of the
// instruction count of the long-wall march (configs[4]).
//
// fexp: Cody–Waite reduction x = k ln2 + r (|r| <= ln2/2, ln2 split in two
// parts), exp(r) by its degree-13 Taylor polynomial (truncation < 4e-18
// relative on |r| <= 0.347) evaluated with Estrin's scheme (dependency depth
// ~5 instead of 13), scaled by 2^k through the exponent field.  Error ~1-2
// ulp; x < -708 flushes to 0 (no subnormals), x > 709 gives +inf, NaN
// propagates.  The reference uses glibc exp; a 1-2 ulp difference in d(v) is
// ~1e-16 relative in a coefficient, far inside the 1e-10 parity tolerance.
//
// frcp: rcp.approx.ftz.f64 (~23 bits) + two Newton steps -> ~1 ulp.
#pragma once
#include <cuda_runtime.h>

namespace hyg {

__device__ __forceinline__ double fexp(double x) {
    // branch-free: clamp, evaluate, then select the special results (no
    // divergent branch on the single-wall step's critical path)
    const double xc = fmin(fmax(x, -708.0), 709.0);    // NaN -> -708 here, restored below
    const double kd = rint(xc * 1.4426950408889634074);
    const double r = fma(-kd, 1.90821492927058770002e-10, fma(-kd, 6.93147180369123816490e-01, xc));
    // Taylor coefficients 1/k!, k = 0..13, in pairs (c_{2i} + c_{2i+1} r)
    const double r2 = r * r;
    const double p01 = fma(r, 1.0, 1.0);
    const double p23 = fma(r, 1.0 / 6.0, 0.5);
    const double p45 = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    const double p67 = fma(r, 1.0 / 5040.0, 1.0 / 720.0);
    const double p89 = fma(r, 1.0 / 362880.0, 1.0 / 40320.0);
    const double p1011 = fma(r, 1.0 / 39916800.0, 1.0 / 3628800.0);
    const double p1213 = fma(r, 1.0 / 6227020800.0, 1.0 / 479001600.0);
    const double r4 = r2 * r2;
    const double q03 = fma(r2, p23, p01);
    const double q47 = fma(r2, p67, p45);
    const double q811 = fma(r2, p1011, p89);
    const double q = fma(r4, fma(r4, fma(r4, p1213, q811), q47), q03);
    const long long k = static_cast<long long>(kd);
    double y = __longlong_as_double(__double_as_longlong(q) + (k << 52));
    y = x < -708.0 ? 0.0 : y;
    y = x > 709.0 ? __longlong_as_double(0x7ff0000000000000ll) : y;
    return x == x ? y : x;                              // NaN propagates
}

__device__ __forceinline__ double frcp(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double e = fma(-d, y, 1.0);
    y = fma(y, e, y);
    e = fma(-d, y, 1.0);
    return fma(y, e, y);
}

}  // namespace hyg
