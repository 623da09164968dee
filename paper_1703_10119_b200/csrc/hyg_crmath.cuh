// hyg_crmath.cuh — accurate (nearly always correctly rounded) exp, log, log10
// and pow for the parity path of the load-bearing material correlations.
//
// The reference evaluates MaterialModel (materials.cpp:11-121) with glibc's
// exp/log/pow/log10, which round correctly in all but rare cases (<= 0.52
// ulp).  The fast device path (hyg_fastmath.cuh, <= 2 ulp) differs from them
// in most evaluations, and the material wall amplifies those ulps: the
// reference's own wall_nonlinear fixture drifts 1.7e-9 relative over its 8e4
// steps (tests/test_gpu_acceptance.py).  These versions carry the result in
// double-double arithmetic (error before the final rounding ~2^-100), so they
// return the correctly rounded double except in astronomically rare cases and
// agree with glibc wherever glibc rounds correctly.
//
//   exp:  x = (64 k + j) ln2/64 + r, ln2/64 in three parts (the first with 33
//         significant bits: n * part exact for |n| < 2^20), r a double-double,
//         |r| <= ln2/128; exp(r) - 1 = r + r^2/2 (double-double) + r^3 (1/6 +
//         ... + r^5/40320) (double, its error ~2^-78); exp(x) = 2^k T_j
//         (1 + q) with T_j = 2^(j/64) a double-double table.
//   log:  x = 2^e m, m in [1, 2), j = round(64 (m - 1)), c_j ~ 1/(1 + j/64)
//         a double, r = m c_j - 1 exact as a double-double (two-product; the
//         subtraction is exact), log1p(r) to degree 10 (|r| < 2^-7),
//         log x = e ln2 + (-log c_j) + log1p(r) summed in double-double.
//   pow:  exp(y log x) with log x and the product in double-double (x > 0).
//   log10: log x times 1/ln10 in double-double.
// Domain: the material path calls these with positive, normal, bounded
// arguments (the box test runs first); overflow/underflow/NaN are handled
// only coarsely.  Constants: hyg_crmath_tables.h (tools/gen_crmath_tables.py).
#pragma once
#include <cuda_runtime.h>

#include "hyg_crmath_tables.h"

namespace hyg {
namespace cr {

struct DD {
    double h, l;
};

__device__ __forceinline__ DD two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    return DD{s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ DD fast_two_sum(double a, double b) {   // |a| >= |b| (or a == 0)
    const double s = __dadd_rn(a, b);
    return DD{s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ DD two_prod(double a, double b) {
    const double p = __dmul_rn(a, b);
    return DD{p, fma(a, b, -p)};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
    const DD s = two_sum(a.h, b.h);
    return fast_two_sum(s.h, __dadd_rn(__dadd_rn(a.l, b.l), s.l));
}
__device__ __forceinline__ DD dd_mul_d(DD a, double y) {          // (a.h + a.l) * y
    DD p = two_prod(a.h, y);
    return fast_two_sum(p.h, fma(a.l, y, p.l));
}

__device__ __constant__ const double kExpTab[64][2] = HYG_CR_EXP2_TAB;
__device__ __constant__ const double kLogTab[65][3] = HYG_CR_LOG_TAB;

// exp(zh + zl), |zl| <= ulp(zh)
__device__ __forceinline__ double exp_dd(double zh, double zl) {
    if (!(zh < 709.79)) return zh != zh ? zh : __longlong_as_double(0x7ff0000000000000ll);
    if (zh < -745.2) return 0.0;
    const double nd = rint(__dmul_rn(zh, HYG_CR_INV_LN2_64));
    const int n = static_cast<int>(nd);
    const double t1 = fma(-nd, HYG_CR_LN2_64_1, zh);               // exact
    const DD a = two_prod(nd, HYG_CR_LN2_64_2);
    const DD s = two_sum(t1, -a.h);
    double rl = __dsub_rn(s.l, a.l);
    rl = fma(-nd, HYG_CR_LN2_64_3, rl);
    rl = __dadd_rn(rl, zl);
    const DD r = fast_two_sum(s.h, rl);
    // exp(r) - 1 = r + r^2/2 + r^3 P(r)
    DD r2 = two_prod(r.h, r.h);
    r2.l = fma(2.0 * r.h, r.l, r2.l);
    const double x = r.h;
    double t = fma(x, 1.0 / 40320.0, 1.0 / 5040.0);
    t = fma(x, t, 1.0 / 720.0);
    t = fma(x, t, 1.0 / 120.0);
    t = fma(x, t, 1.0 / 24.0);
    t = fma(x, t, 1.0 / 6.0);
    const double tail = __dmul_rn(__dmul_rn(r2.h, x), t);
    DD u = two_sum(r.h, __dmul_rn(0.5, r2.h));
    u.l = __dadd_rn(__dadd_rn(u.l, r.l), fma(0.5, r2.l, tail));
    const DD q = fast_two_sum(u.h, u.l);
    const int j = n & 63, k = (n - j) / 64;
    const double Th = kExpTab[j][0], Tl = kExpTab[j][1];
    const DD m = two_prod(Th, q.h);
    const double lo = __dadd_rn(__dadd_rn(Tl, m.l), fma(Th, q.l, __dmul_rn(Tl, q.h)));
    const DD sum = two_sum(Th, m.h);
    const double res = __dadd_rn(sum.h, __dadd_rn(sum.l, lo));
    return ldexp(res, k);
}

__device__ __forceinline__ double exp(double x) { return exp_dd(x, 0.0); }

// log x as a double-double, x positive and normal
__device__ __forceinline__ DD log_dd(double x) {
    const int hi = __double2hiint(x), lo = __double2loint(x);
    const int e = ((hi >> 20) & 0x7ff) - 1023;
    const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);   // [1, 2)
    const int j = static_cast<int>(rint(__dmul_rn(__dsub_rn(m, 1.0), 64.0)));
    const double c = kLogTab[j][0];
    const DD p = two_prod(m, c);
    const DD r = fast_two_sum(__dsub_rn(p.h, 1.0), p.l);           // m c - 1, exact
    // log1p(r) = r - r^2/2 + r^3 P(r), |r| < 2^-7
    DD r2 = two_prod(r.h, r.h);
    r2.l = fma(2.0 * r.h, r.l, r2.l);
    const double x1 = r.h;
    double t = fma(x1, -1.0 / 10.0, 1.0 / 9.0);
    t = fma(x1, t, -1.0 / 8.0);
    t = fma(x1, t, 1.0 / 7.0);
    t = fma(x1, t, -1.0 / 6.0);
    t = fma(x1, t, 1.0 / 5.0);
    t = fma(x1, t, -1.0 / 4.0);
    t = fma(x1, t, 1.0 / 3.0);
    const double tail = __dmul_rn(__dmul_rn(r2.h, x1), t);
    DD u = two_sum(r.h, __dmul_rn(-0.5, r2.h));
    u.l = __dadd_rn(__dadd_rn(u.l, r.l), fma(-0.5, r2.l, tail));
    const DD l1p = fast_two_sum(u.h, u.l);
    const double ed = static_cast<double>(e);
    DD a = two_prod(ed, HYG_CR_LN2_HI);
    a.l = fma(ed, HYG_CR_LN2_LO, a.l);
    const DD b{kLogTab[j][1], kLogTab[j][2]};
    return dd_add(dd_add(a, b), l1p);
}

__device__ __forceinline__ double log(double x) {
    if (!(x > 0.0) || !(x < 1.7976931348623157e308) || x < 2.2250738585072014e-308)
        return x == 0.0 ? -__longlong_as_double(0x7ff0000000000000ll)
                        : (x > 0.0 && !(x < 1.7976931348623157e308) ? x : ::log(x));
    return log_dd(x).h;
}

__device__ __forceinline__ double log10(double x) {
    if (!(x > 0.0) || !(x < 1.7976931348623157e308) || x < 2.2250738585072014e-308) return ::log10(x);
    const DD l = log_dd(x);
    DD p = two_prod(l.h, HYG_CR_INV_LN10_HI);
    p.l = fma(l.h, HYG_CR_INV_LN10_LO, fma(l.l, HYG_CR_INV_LN10_HI, p.l));
    return __dadd_rn(p.h, p.l);
}

// pow(x, y) for x > 0 (the material's bases are positive); others: libdevice
__device__ __forceinline__ double pow(double x, double y) {
    if (!(x > 0.0) || !(x < 1.7976931348623157e308) || x < 2.2250738585072014e-308 || y != y) return ::pow(x, y);
    if (y == 0.0 || x == 1.0) return 1.0;
    const DD z = dd_mul_d(log_dd(x), y);
    return exp_dd(z.h, z.l);
}

}  // namespace cr
}  // namespace hyg
