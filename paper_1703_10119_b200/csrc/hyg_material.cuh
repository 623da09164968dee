// hyg_material.cuh — the load-bearing material correlations
// (MaterialModel, materials.cpp:11-121) as one host/device functor.
//
// Every expression keeps the reference's operand order, so the host build
// (glibc exp/log/pow, used for setup: the reference set of a material wall,
// hyg_material_evaluate) is bit-identical to the reference, and the device
// parity build (CrMath, no FMA contraction) differs only where glibc itself
// misrounds.  Default PhysicalConstants
// (materials.hpp:7-15) — the scenario loader always uses them
// (scenario.cpp:161).
#pragma once
#include <math.h>
#if defined(__CUDACC__)
#include "hyg_crmath.cuh"
#include "hyg_fastmath.cuh"
#endif

#if defined(__CUDACC__)
#define HYG_HD __host__ __device__ __forceinline__
#else
#define HYG_HD inline
#endif

namespace hyg {
namespace mat {

constexpr double kRho0 = 790.0, kC0 = 870.0, kCw = 4180.0, kRhoL = 1000.0, kRv = 461.5, kLv = 2.5e6;
constexpr double kC1 = 1.25e-5, kC2 = 1.8e-5, kSat = 157.0;         // materials.cpp:12-14
constexpr double kBoxTMin = 274.15, kBoxTMax = 313.15;              // materials.hpp:50-53
constexpr double kBoxPhiMin = 0.01, kBoxPhiMax = 0.99;

struct Set { double c_M, k_M, c_TT, k_TT, c_TM, k_TM; };             // CoefficientSet

// The correlations are templates on the math functions: LibMath = the C
// library (the host build: glibc, bitwise the reference's setup values), CrMath
// = the accurate device versions of hyg_crmath.cuh (the device parity path:
// the reference's expressions, IEEE divisions, no FMA contraction — the
// library is built with -fmad=false — and exp/log/pow/log10 rounded like
// glibc's in all but rare cases).
struct LibMath {
    HYG_HD static double exp(double x) { return ::exp(x); }
    HYG_HD static double log(double x) { return ::log(x); }
    HYG_HD static double log10(double x) { return ::log10(x); }
    HYG_HD static double pow(double x, double y) { return ::pow(x, y); }
};
#if defined(__CUDACC__)
struct CrMath {
#if defined(__CUDA_ARCH__)
    HYG_HD static double exp(double x) { return cr::exp(x); }
    HYG_HD static double log(double x) { return cr::log(x); }
    HYG_HD static double log10(double x) { return cr::log10(x); }
    HYG_HD static double pow(double x, double y) { return cr::pow(x, y); }
#else
    HYG_HD static double exp(double x) { return ::exp(x); }
    HYG_HD static double log(double x) { return ::log(x); }
    HYG_HD static double log10(double x) { return ::log10(x); }
    HYG_HD static double pow(double x, double y) { return ::pow(x, y); }
#endif
};
#endif

template <class M = LibMath>
HYG_HD double saturation_pressure(double T) {                      // materials.cpp:33-40 (range by caller)
    return M::exp(23.5771 - 4042.9 / (T - 37.58));
}

template <class M = LibMath>
HYG_HD double plateau(double s) {                                  // materials.cpp:17-20
    return 47.1 * M::pow(1.0 + M::pow(kC1 * s, 1.65), -0.39) + 109.9 * M::pow(1.0 + M::pow(kC2 * s, 6.0), -0.83);
}

template <class M = LibMath>
HYG_HD double moisture_content(double T, double phi) {             // materials.cpp:61-63
    return plateau<M>(kRv * T * (-M::log(phi)));
}

HYG_HD double vapour_permeability(double T, double f) {            // materials.cpp:65-68
    const double z = 1.0 - f / kSat;
    return 1.88e-6 / T * z / (0.503 * z * z + 0.497);
}

HYG_HD double thermal_conductivity(double f) { return 0.2 + 0.0045 * f; }   // materials.cpp:70-72

template <class M = LibMath>
HYG_HD double moisture_transport(double P_v, double P_s) {         // materials.cpp:74-78
    const double r = 2.0 * P_v / P_s;
    return 1.97e-10 * M::pow(10.0, 1.44 - 0.07 * M::log10(r)) + 1.77e-7 * M::exp(-8.0 * (r - 2.0) * (r - 2.0));
}

template <class M = LibMath>
HYG_HD double moisture_storage(double T, double P_v, double P_s) { // materials.cpp:80-89
    const double x = -M::log(P_v / P_s);
    const double rt = kRv * T;
    const double x1 = kC1 * rt * x, x2 = kC2 * rt * x;
    const double t1 = 30.62 * (kC1 * rt / P_v) * M::pow(x1, 0.65) * M::pow(1.0 + M::pow(x1, 1.65), -1.39);
    const double t2 = 549.5 * (kC2 * rt / P_v) * M::pow(x2, 5.0) * M::pow(1.0 + M::pow(x2, 6.0), -1.83);
    return t1 + t2;
}

// MaterialModel::evaluate (materials.cpp:91-114); false where the reference
// throws domain_error (state outside the admissible box).
template <class M = LibMath>
HYG_HD bool evaluate(double T, double P_v, Set& out) {
    const double tol = 1e-9;
    const double P_s = (T >= kBoxTMin - tol && T <= kBoxTMax + tol) ? saturation_pressure<M>(T) : 0.0;
    const double phi = P_s > 0.0 ? P_v / P_s : -1.0;
    if (!(P_s > 0.0) || !(phi >= kBoxPhiMin * (1.0 - tol) && phi <= kBoxPhiMax * (1.0 + tol))) return false;
    const double f = moisture_content<M>(T, phi);
    const double c_M = moisture_storage<M>(T, P_v, P_s);
    out.c_M = c_M;
    out.k_M = moisture_transport<M>(P_v, P_s);
    out.c_TT = kRho0 * kC0 + kCw * f;
    out.k_TT = thermal_conductivity(f);
    out.c_TM = kCw * (T - 273.15) * c_M;
    out.k_TM = kLv * vapour_permeability(T, f);
    return true;
}

HYG_HD double clampd(double x, double lo, double hi) { return x < lo ? lo : (hi < x ? hi : x); }  // std::clamp

// MaterialModel::evaluate_clamped (materials.cpp:116-121)
template <class M = LibMath>
HYG_HD bool evaluate_clamped(double T, double P_v, Set& out) {
    const double Tc = clampd(T, kBoxTMin, kBoxTMax);
    const double P_s = saturation_pressure<M>(Tc);
    const double phi = clampd(P_v / P_s, kBoxPhiMin, kBoxPhiMax);
    return evaluate<M>(Tc, phi * P_s, out);
}

#if defined(__CUDACC__)
// Device evaluation with shared transcendentals.  Same box test as evaluate
// (P_s by exp, phi = P_v / P_s, identical to the reference's values up to the
// device exp's rounding); the correlations use the identities
//   x^a = exp(a ln x),  x^(a+1) = x^a * x,  (1+y)^(b-1) = (1+y)^b / (1+y),
//   x^5, x^6 by multiplication,  log10(2 P_v/P_s) = (ln 2 + ln phi) / ln 10,
//   10^(1.44 - 0.07 log10 r) = exp(1.44 ln 10 - 0.07 ln r),
// and moisture_storage's -log(P_v/P_s) is the content's -ln(phi) (the same
// quotient).  4 logs + 5 exps instead of 11 pows + 3 logs + 2 exps, all but
// the box test's P_s by the table-driven fexp/flog_pos and reciprocal-based
// quotients of hyg_fastmath.cuh; a few ulp per coefficient against the
// reference's correctly rounded glibc results (parity is asserted on whole
// runs, tests/test_gpu_material.py).
__device__ __forceinline__ bool evaluate_fast(double T, double P_v, Set& out) {
    const double tol = 1e-9;
    const double P_s = (T >= kBoxTMin - tol && T <= kBoxTMax + tol) ? saturation_pressure<LibMath>(T) : 0.0;
    const double phi = P_s > 0.0 ? P_v / P_s : -1.0;
    if (!(P_s > 0.0) || !(phi >= kBoxPhiMin * (1.0 - tol) && phi <= kBoxPhiMax * (1.0 + tol))) return false;
    // inside the box every argument below is positive, normal and bounded:
    // table-driven exp/log (hyg_fastmath.cuh) and reciprocal-based quotients
    const double lphi = flog_pos(phi);                 // < 0
    const double rt = kRv * T;
    const double s = rt * (-lphi);                     // specific capillary potential
    const double iPv = frcp(P_v);
    // first plateau: x1 = C1 s
    const double x1 = kC1 * s;
    const double l1 = flog_pos(x1);
    const double x1_165 = fexp_g(1.65 * l1);           // x1^1.65
    const double x1_065 = fdiv(x1_165, x1);            // x1^0.65
    const double B1 = 1.0 + x1_165;
    const double p1 = fexp_g(-0.39 * flog_pos(B1));    // (1 + x1^1.65)^-0.39
    const double p1m = fdiv(p1, B1);                   // (1 + x1^1.65)^-1.39
    // second plateau: x2 = C2 s
    const double x2 = kC2 * s;
    const double x2_2 = x2 * x2;
    const double x2_5 = x2_2 * x2_2 * x2;
    const double x2_6 = x2_5 * x2;
    const double B2 = 1.0 + x2_6;
    const double p2 = fexp_g(-0.83 * flog_pos(B2));    // (1 + x2^6)^-0.83
    const double p2m = fdiv(p2, B2);                   // (1 + x2^6)^-1.83
    const double f = 47.1 * p1 + 109.9 * p2;           // moisture_content
    // moisture_storage (materials.cpp:80-89)
    const double t1 = 30.62 * (kC1 * rt * iPv) * x1_065 * p1m;
    const double t2 = 549.5 * (kC2 * rt * iPv) * x2_5 * p2m;
    const double c_M = t1 + t2;
    // moisture_transport (materials.cpp:74-78): r = 2 P_v / P_s = 2 phi exactly
    const double r = 2.0 * phi;
    const double lr = 0.69314718055994530942 + lphi;
    const double k_M = 1.97e-10 * fexp_g(1.44 * 2.30258509299404568402 - 0.07 * lr) +
                       1.77e-7 * fexp_g(-8.0 * (r - 2.0) * (r - 2.0));
    out.c_M = c_M;
    out.k_M = k_M;
    out.c_TT = kRho0 * kC0 + kCw * f;
    out.k_TT = thermal_conductivity(f);
    out.c_TM = kCw * (T - 273.15) * c_M;
    const double z = 1.0 - f * (1.0 / kSat);           // vapour_permeability (materials.cpp:65-68)
    out.k_TM = kLv * (1.88e-6 * frcp(T) * z * frcp(0.503 * z * z + 0.497));
    return true;
}
#endif

// CoefficientModel::star / star_clamped (wall.cpp:50-58): the set at
// (u T_i, v P_vi) divided by the wall's reference set.  On the device `exact`
// selects the accurate path (the reference's expressions with CrMath and IEEE
// divisions, HYG_TUNE_MATERIAL_EXACT) or evaluate_fast (the default).
HYG_HD bool star(double u, double v, double T_i, double P_vi, const Set& ref, bool strict, Set& out,
                 bool exact = false) {
    Set a;
#if defined(__CUDA_ARCH__)
    bool ok;
    if (exact) {
        ok = strict ? evaluate<CrMath>(u * T_i, v * P_vi, a) : evaluate_clamped<CrMath>(u * T_i, v * P_vi, a);
    } else if (strict) {
        ok = evaluate_fast(u * T_i, v * P_vi, a);
    } else {                                            // evaluate_clamped (materials.cpp:116-121)
        const double Tc = clampd(u * T_i, kBoxTMin, kBoxTMax);
        const double P_s = saturation_pressure(Tc);
        ok = evaluate_fast(Tc, clampd(v * P_vi / P_s, kBoxPhiMin, kBoxPhiMax) * P_s, a);
    }
    if (!ok) return false;
    if (!exact) {
        out.c_M = fdiv(a.c_M, ref.c_M);
        out.k_M = fdiv(a.k_M, ref.k_M);
        out.c_TT = fdiv(a.c_TT, ref.c_TT);
        out.k_TT = fdiv(a.k_TT, ref.k_TT);
        out.c_TM = fdiv(a.c_TM, ref.c_TM);
        out.k_TM = fdiv(a.k_TM, ref.k_TM);
        return true;
    }
#else
    (void)exact;
    const bool ok = strict ? evaluate(u * T_i, v * P_vi, a) : evaluate_clamped(u * T_i, v * P_vi, a);
    if (!ok) return false;
#endif
    out.c_M = a.c_M / ref.c_M;
    out.k_M = a.k_M / ref.k_M;
    out.c_TT = a.c_TT / ref.c_TT;
    out.k_TT = a.k_TT / ref.k_TT;
    out.c_TM = a.c_TM / ref.c_TM;
    out.k_TM = a.k_TM / ref.k_TM;
    return true;
}

}  // namespace mat
}  // namespace hyg
