// hyg_scaling.cpp — host-side setup of the dimensionless groups, restating
// /root/reference/proj/src/scaling.cpp:1-115 and saturation_pressure
// (materials.cpp:33-40) behind the C ABI, so configuration builders derive
// wall/zone groups exactly as the reference's scenario loader does.
#include <cmath>

#include "../../include/hygro_b200.h"
#include "hyg_material.cuh"

namespace {
// PhysicalConstants (materials.hpp:7-15) and kPv0 (scaling.hpp:74)
constexpr double kLv = 2.5e6;
constexpr double kPv0 = 1.61e5;

bool positive(double x) { return x > 0.0 && std::isfinite(x); }  // require_positive scaling.cpp:9-16

double psat(double T) { return std::exp(23.5771 - 4042.9 / (T - 37.58)); }

// ScalingContext::from_state (scaling.cpp:20-28)
int context(double T_i, double phi_i, double t_0, double* P_vi) {
    if (!(T_i >= 273.15 && T_i <= 373.15)) return HYG_EDOMAIN;
    *P_vi = phi_i * psat(T_i);
    if (!positive(*P_vi) || !positive(t_0)) return HYG_ESCALING;
    return HYG_OK;
}

struct Zone {
    double kappa_TT0, kappa_M, kappa_a_tt1, g_v, q_v1, q_v2, g_o, q_o, q_h;
};

int zone_of(double V, double rho, double cpa, double cpv, double ach, double T_i, double P_vi,
            double t_0, Zone* z) {   // scale_zone (scaling.cpp:60-83)
    if (!positive(V) || !positive(rho) || !positive(cpa)) return HYG_ESCALING;
    z->kappa_TT0 = rho * V * cpa;
    z->kappa_M = rho * V;
    z->kappa_a_tt1 = cpv * P_vi / (cpa * kPv0);
    const double g_v = ach * V * rho / 3600.0;
    z->g_v = g_v * t_0 / z->kappa_M;
    z->q_v1 = cpv * g_v * t_0 * P_vi / (kPv0 * z->kappa_TT0);
    z->q_v2 = kLv * g_v * t_0 * P_vi / (kPv0 * z->kappa_TT0 * T_i);
    z->g_o = t_0 * kPv0 / (z->kappa_M * P_vi);
    z->q_o = kLv * t_0 / (T_i * z->kappa_TT0);
    z->q_h = t_0 / (T_i * z->kappa_TT0);
    return HYG_OK;
}
}  // namespace

extern "C" {

int hyg_saturation_pressure(double T, double* out) {
    if (!(T >= 273.15 && T <= 373.15)) return HYG_EDOMAIN;
    *out = psat(T);
    return HYG_OK;
}

int hyg_material_evaluate(double T, double P_v, int32_t clamped, hyg_coeff_set* out) {
    if (!out) return HYG_EINVAL;
    hyg::mat::Set s;
    if (clamped && !(T == T)) return HYG_EDOMAIN;     // saturation_pressure(NaN) throws
    const bool ok = clamped ? hyg::mat::evaluate_clamped(T, P_v, s) : hyg::mat::evaluate(T, P_v, s);
    if (!ok) return HYG_EDOMAIN;
    *out = hyg_coeff_set{s.c_M, s.k_M, s.c_TT, s.k_TT, s.c_TM, s.k_TM};
    return HYG_OK;
}

int hyg_scale_wall(const double r[6], double L, double h_T0, double h_M0, double h_T1, double h_M1,
                   double T_i, double phi_i, double t_0, hyg_wall_groups* g, hyg_face_biot face[2]) {
    double P_vi;
    int rc = context(T_i, phi_i, t_0, &P_vi);
    if (rc) return rc;
    if (!positive(L)) return HYG_ESCALING;
    for (int i = 0; i < 6; ++i)
        if (!positive(r[i])) return HYG_ESCALING;
    const double c_M = r[0], k_M = r[1], c_TT = r[2], k_TT = r[3], c_TM = r[4], k_TM = r[5];
    const double L2 = L * L;
    g->Fo_M = t_0 * k_M / (L2 * c_M);
    g->Fo_TT = t_0 * k_TT / (L2 * c_TT);
    g->Fo_TM = t_0 * k_TM / (L2 * c_TM);
    g->gamma = c_TM * P_vi / (c_TT * T_i);
    const double h_T[2] = {h_T0, h_T1}, h_M[2] = {h_M0, h_M1};
    for (int f = 0; f < 2; ++f) {
        face[f].Bi_M = h_M[f] * L / k_M;
        face[f].Bi_TT = h_T[f] * L / k_TT;
        face[f].Bi_TM = kLv * h_M[f] * L * P_vi / (k_TT * T_i);
    }
    return HYG_OK;
}

int hyg_scale_zone(double V, double rho, double cpa, double cpv, double ach, double T_i, double phi_i,
                   double t_0, double out[7]) {
    double P_vi;
    int rc = context(T_i, phi_i, t_0, &P_vi);
    if (rc) return rc;
    Zone z;
    rc = zone_of(V, rho, cpa, cpv, ach, T_i, P_vi, t_0, &z);
    if (rc) return rc;
    const double v[7] = {z.kappa_a_tt1, z.g_v, z.q_v1, z.q_v2, z.g_o, z.q_o, z.q_h};
    for (int i = 0; i < 7; ++i) out[i] = v[i];
    return HYG_OK;
}

int hyg_attach_wall_to_zone(const double r[6], double area, double L, double V, double rho, double cpa,
                            double T_i, double phi_i, double t_0, double out[2]) {
    double P_vi;
    int rc = context(T_i, phi_i, t_0, &P_vi);
    if (rc) return rc;
    if (!positive(area)) return HYG_ESCALING;
    Zone z;
    rc = zone_of(V, rho, cpa, 0.0, 0.0, T_i, P_vi, t_0, &z);
    if (rc) return rc;
    out[0] = r[3] * area * t_0 / (L * z.kappa_TT0);          // theta_T scaling.cpp:88
    out[1] = r[1] * area * t_0 * kPv0 / (L * z.kappa_M);     // theta_M scaling.cpp:89
    return HYG_OK;
}

int hyg_scale_interzone(double ach, double V, double rho, double cpa, double cpv, double T_i,
                        double phi_i, double t_0, double out[3]) {
    double P_vi;
    int rc = context(T_i, phi_i, t_0, &P_vi);
    if (rc) return rc;
    Zone z;
    rc = zone_of(V, rho, cpa, cpv, 0.0, T_i, P_vi, t_0, &z);
    if (rc) return rc;
    const double g = ach * V * rho / 3600.0;                 // scaling.cpp:95
    out[0] = g * t_0 / z.kappa_M;
    out[1] = cpv * g * t_0 * P_vi / (kPv0 * z.kappa_TT0);
    out[2] = kLv * g * t_0 * P_vi / (kPv0 * z.kappa_TT0 * T_i);
    return HYG_OK;
}

}  // extern "C"
