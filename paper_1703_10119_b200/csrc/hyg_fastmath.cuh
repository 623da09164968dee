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

#include "hyg_exp256_table.h"

namespace hyg {

// 2^(j/64), j = 0..63, correctly rounded (generated with 60-digit decimal arithmetic)
#define HYG_EXP2_TAB64 { \
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0, \
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0, \
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0, \
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0, \
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0, \
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0, \
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0, \
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0, \
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0, \
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0, \
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0, \
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0, \
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0, \
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0, \
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0, \
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0 \
}
__device__ __constant__ const double kExp2Tab64[64] = HYG_EXP2_TAB64;
// the same table in global memory for callers that cannot stage it in shared
// memory (read through the read-only path: divergent indices cost a few L1
// wavefronts, where constant memory would serialise them)
__device__ const double kExp2Tab64G[64] = HYG_EXP2_TAB64;
// 2^(j/256) for fexp_addend (the d(v) half node), staged in shared memory by its kernels
__device__ const double kExp2Tab256[256] = HYG_EXP2_TAB256;


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

// The same with TWO FMAs: y (1 + e), error e^2 <= 1e-12 relative (rcp.approx is good to 2^-20), always
// towards zero.  For the d(v) v row only: there 1/den multiplies the increment
// inc = num / den, and a relative bias of 1e-12 in every increment is a relative
// change of 1e-12 in the diffusion number (the solution moves by ~1e-13 of its
// own variation), two orders inside the 1e-10 parity tolerance — one FP64
// instruction per node-update fewer than frcp.
__device__ __forceinline__ double frcp2(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    return fma(y, fma(-d, y, 1.0), y);
}

// exp(x) for the d(v) half node (1 + p0 v + p1 exp(x), x = -p2 (v - p3)^2):
// 8 FP64 instructions.  x = (256 k + j) ln2/256 + r from one FMA against the
// 1.5 * 2^52 shifter, |r| <= ln2/512 = 1.35e-3, exp(r) - 1 by its degree-4
// polynomial (truncation r^5/120 < 4e-17 relative: the 256-entry table buys the
// degree-5 term of fexp), T_j = 2^(j/256) correctly rounded from the table the
// kernels stage in shared memory, 2^k by an integer add on T_j's exponent.
// The reduction uses ln2/256 as ONE rounded constant (relative error 3.3e-17, as
// the double nearest ln 2): the result is off by |x| 3.3e-17 relative — 1 ulp at
// the edge of the d(v) range of configs[0]/[4] (|x| <= 6.4), 54 ulp at x = -180
// where the term is 1e-78; as an absolute error of the Gaussian never above
// 1.3e-17 (tests/test_gpu_fastmath.py).
// NO clamp and no special cases: valid for -700 <= x <= 0.  The host admits a
// model to the kernels that call it only if p2 (2 + |p3|)^2 <= 700 (hyg_create:
// every state inside the fast guard, |v| < 2, then keeps x above -700; a state
// outside it is flagged by the guard and the launch is replayed on the per-step
// path with the full fexp).
// STRIDE: the table's element stride (the bank-replicated copy of k_nonlinear.cuh);
// tab: entries exp_tab_biased(j) (stage_exp_table_rep)
template <int STRIDE = 1>
__device__ __forceinline__ double fexp_addend(double x, const double* tab) {
    constexpr double kShift = 6755399441055744.0;                  // 1.5 * 2^52
    constexpr double kInvL = 369.32993046757463;                   // 256 / ln 2
    constexpr double kL = 0x1.62e42fefa39efp-9;                    // ln2 / 256
    const double s = fma(x, kInvL, kShift);
    const double kd = s - kShift;
    const int k = __double2loint(s);
    const double r = fma(kd, -kL, x);
    const double r2 = r * r;
    const double c23 = fma(r, 1.0 / 6.0, 0.5);
    const double q = fma(r2, 1.0 / 24.0, c23);                     // 1/2 + r/6 + r^2/24
    const double sm = fma(r2, q, r);                               // exp(r) - 1
    // tab holds T_j with its high word lowered by j << 12 (exp_tab_biased): k << 12 =
    // ((k >> 8) << 20) + (j << 12), so ONE multiply-add puts 2^(k >> 8) into the exponent
    // field (shift, mask and add before: two integer instructions and their register
    // reads less per exp, off the FP64 pipe's register bandwidth)
    const double t = tab[(k & 255) * STRIDE];
    const double ts = __hiloint2double(__double2hiint(t) + (k << 12), __double2loint(t));
    return fma(ts, sm, ts);
}

// entry j of fexp_addend's table: 2^(j/256) with the high word lowered by j << 12
__device__ __forceinline__ double exp_tab_biased(int j) {
    const double t = kExp2Tab256[j];
    return __hiloint2double(__double2hiint(t) - (j << 12), __double2loint(t));
}

// flog_pos: ln x for positive normal finite x (the material correlations call
// it on quantities bounded by the admissible box).  x = 2^e m, m in [1, 2);
// m rounded to the nearest c_j = 1 + j/64 (j = 0..64, from the top 7 bits),
// r = m ic_j - 1 in one FMA (|r| <= 1/128) and ln x = e ln2 - ln(ic_j) +
// log1p(r), where ic_j is 1/c_j rounded and kLogC[j] = -ln(ic_j) of that
// double (so the identity is exact), log1p by its degree-7 Taylor polynomial
// (truncation < 2e-18).  j = 64 is c = 2 taken as e + 1, c = 1 (ic = 1/2,
// no table logarithm), so ln x is exact-cancellation-free on both sides of
// 1 and ln 1 = 0.  ln2 split in two (e ln2_hi exact for |e| < 2^11).  Tables
// generated with 60-digit decimal arithmetic.  Error <= ~2 ulp of
// max(|e ln2|, |ln c_j|) (tests/test_gpu_fastmath.py).
__device__ const double kLogInvC[65] = {
    0x1.0000000000000p+0, 0x1.f81f81f81f820p-1, 0x1.f07c1f07c1f08p-1, 0x1.e9131abf0b767p-1,
    0x1.e1e1e1e1e1e1ep-1, 0x1.dae6076b981dbp-1, 0x1.d41d41d41d41dp-1, 0x1.cd85689039b0bp-1,
    0x1.c71c71c71c71cp-1, 0x1.c0e070381c0e0p-1, 0x1.bacf914c1bad0p-1, 0x1.b4e81b4e81b4fp-1,
    0x1.af286bca1af28p-1, 0x1.a98ef606a63bep-1, 0x1.a41a41a41a41ap-1, 0x1.9ec8e951033d9p-1,
    0x1.999999999999ap-1, 0x1.948b0fcd6e9e0p-1, 0x1.8f9c18f9c18fap-1, 0x1.8acb90f6bf3aap-1,
    0x1.8618618618618p-1, 0x1.8181818181818p-1, 0x1.7d05f417d05f4p-1, 0x1.78a4c8178a4c8p-1,
    0x1.745d1745d1746p-1, 0x1.702e05c0b8170p-1, 0x1.6c16c16c16c17p-1, 0x1.6816816816817p-1,
    0x1.642c8590b2164p-1, 0x1.6058160581606p-1, 0x1.5c9882b931057p-1, 0x1.58ed2308158edp-1,
    0x1.5555555555555p-1, 0x1.51d07eae2f815p-1, 0x1.4e5e0a72f0539p-1, 0x1.4afd6a052bf5bp-1,
    0x1.47ae147ae147bp-1, 0x1.446f86562d9fbp-1, 0x1.4141414141414p-1, 0x1.3e22cbce4a902p-1,
    0x1.3b13b13b13b14p-1, 0x1.3813813813814p-1, 0x1.3521cfb2b78c1p-1, 0x1.323e34a2b10bfp-1,
    0x1.2f684bda12f68p-1, 0x1.2c9fb4d812ca0p-1, 0x1.29e4129e4129ep-1, 0x1.27350b8812735p-1,
    0x1.2492492492492p-1, 0x1.21fb78121fb78p-1, 0x1.1f7047dc11f70p-1, 0x1.1cf06ada2811dp-1,
    0x1.1a7b9611a7b96p-1, 0x1.1811811811812p-1, 0x1.15b1e5f75270dp-1, 0x1.135c81135c811p-1,
    0x1.1111111111111p-1, 0x1.0ecf56be69c90p-1, 0x1.0c9714fbcda3bp-1, 0x1.0a6810a6810a7p-1,
    0x1.0842108421084p-1, 0x1.0624dd2f1a9fcp-1, 0x1.0410410410410p-1, 0x1.0204081020408p-1,
    0x1.0000000000000p-1,
};
__device__ const double kLogC[65] = {
    0x0.0p+0, 0x1.fc0a8b0fc03c4p-7, 0x1.f829b0e7832f8p-6, 0x1.77458f632dcffp-5,
    0x1.f0a30c01162a8p-5, 0x1.341d7961bd1d0p-4, 0x1.6f0d28ae56b4ep-4, 0x1.a926d3a4ad562p-4,
    0x1.e27076e2af2eap-4, 0x1.0d77e7cd08e5bp-3, 0x1.29552f81ff521p-3, 0x1.44d2b6ccb7d1cp-3,
    0x1.5ff3070a793d6p-3, 0x1.7ab890210d907p-3, 0x1.9525a9cf456b6p-3, 0x1.af3c94e80bff3p-3,
    0x1.c8ff7c79a9a20p-3, 0x1.e27076e2af2e8p-3, 0x1.fb9186d5e3e29p-3, 0x1.0a324e27390e2p-2,
    0x1.1675cababa60fp-2, 0x1.22941fbcf7966p-2, 0x1.2e8e2bae11d31p-2, 0x1.3a64c556945eap-2,
    0x1.4618bc21c5ec2p-2, 0x1.51aad872df82ep-2, 0x1.5d1bdbf5809cap-2, 0x1.686c81e9b14adp-2,
    0x1.739d7f6bbd007p-2, 0x1.7eaf83b82afc2p-2, 0x1.89a3386c1425bp-2, 0x1.947941c2116fbp-2,
    0x1.9f323ecbf984dp-2, 0x1.a9cec9a9a084ap-2, 0x1.b44f77bcc8f64p-2, 0x1.beb4d9da71b7ap-2,
    0x1.c8ff7c79a9a21p-2, 0x1.d32fe7e00ebd5p-2, 0x1.dd46a04c1c4a1p-2, 0x1.e744261d68789p-2,
    0x1.f128f5faf06ecp-2, 0x1.faf588f78f31dp-2, 0x1.02552a5a5d0ffp-1, 0x1.0723e5c1cdf41p-1,
    0x1.0be72e4252a83p-1, 0x1.109f39e2d4c96p-1, 0x1.154c3d2f4d5eap-1, 0x1.19ee6b467c96fp-1,
    0x1.1e85f5e7040d1p-1, 0x1.23130d7bebf43p-1, 0x1.2795e1289b11bp-1, 0x1.2c0e9ed448e8cp-1,
    0x1.307d7334f10bep-1, 0x1.34e289d9ce1d2p-1, 0x1.393e0d3562a1ap-1, 0x1.3d9026a7156fbp-1,
    0x1.41d8fe84672afp-1, 0x1.4618bc21c5ec2p-1, 0x1.4a4f85db03ebbp-1, 0x1.4e7d811b75bb0p-1,
    0x1.52a2d265bc5abp-1, 0x1.56bf9d5b3f399p-1, 0x1.5ad404c359f2dp-1, 0x1.5ee02a9241676p-1,
    0x0.0p+0,
};

__device__ __forceinline__ double flog_pos(double x) {
    constexpr double kLn2Hi = 0x1.62e42fefa3800p-1, kLn2Lo = 0x1.ef35793c76730p-45;
    const int hi = __double2hiint(x);
    const int j = (((hi >> 13) & 127) + 1) >> 1;       // nearest c_j, 0..64
    const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(x));
    const double ed = static_cast<double>((hi >> 20) - 1023 + (j >> 6));
    const double r = fma(m, __ldg(&kLogInvC[j]), -1.0);
    double p = fma(r, 1.0 / 7.0, -1.0 / 6.0);
    p = fma(r, p, 1.0 / 5.0);
    p = fma(r, p, -0.25);
    p = fma(r, p, 1.0 / 3.0);
    p = fma(r, p, -0.5);
    p = fma(r * r, p, r);                              // log1p(r)
    return fma(ed, kLn2Hi, __ldg(&kLogC[j])) + fma(ed, kLn2Lo, p);
}

// exp for the material correlations (arguments bounded: |x| < 708), table in
// global memory
__device__ __forceinline__ double fexp_g(double x) { return fexp_core(x, kExp2Tab64G); }

// a / b to ~1 ulp (reciprocal + product), for b normal and finite
__device__ __forceinline__ double fdiv(double a, double b) { return a * frcp(b); }

}  // namespace hyg
