/*
 * hygro_oracle.c — TEST INFRASTRUCTURE ONLY (see hygro_oracle.h).
 *
 * Plain-C restatement of the reference DF path.  Every function follows the
 * cited reference statements in the same order and with the same expression
 * trees, so that compiled with the same flags as the reference (gcc -O2, no
 * FMA contraction: -ffp-contract=off) it reproduces the reference bit for
 * bit; tests/test_oracle_vs_ref.py checks exactly that against oracle/_ref.
 */
#define _POSIX_C_SOURCE 200809L   /* pthread_barrier_t under -std=c11 */
#include "hygro_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ---------------- signals: signal.hpp:39-50 ------------------------------ */
double orc_signal(const hyg_signal* s, double t) {
    double v = s->base;
    if (s->form == HYG_SIG_SIN) {
        v += s->amplitude * sin(2.0 * M_PI * (t - s->phase) / s->period);
    } else if (s->form == HYG_SIG_SIN2) {
        const double x = sin(2.0 * M_PI * (t - s->phase) / s->period);
        v += s->amplitude * x * x;
    }
    for (int i = 0; i < s->n_windows; ++i)
        if (t >= s->windows[i].from && t < s->windows[i].to) v += s->windows[i].value;
    return v;
}

/* ---------------- materials: materials.cpp ------------------------------- */
/* PhysicalConstants materials.hpp:7-15 */
static const double kRho0 = 790.0, kC0 = 870.0, kCw = 4180.0, kRv = 461.5, kLv = 2.5e6;
static const double kC1 = 1.25e-5, kC2 = 1.8e-5, kSat = 157.0; /* materials.cpp:14-16 */
static const double kBoxTMin = 274.15, kBoxTMax = 313.15, kBoxPhiMin = 0.01, kBoxPhiMax = 0.99;

double orc_saturation_pressure(double T) { /* materials.cpp:33-40 (range check by caller) */
    return exp(23.5771 - 4042.9 / (T - 37.58));
}

static double plateau(double s) { /* materials.cpp:19-22 */
    return 47.1 * pow(1.0 + pow(kC1 * s, 1.65), -0.39) + 109.9 * pow(1.0 + pow(kC2 * s, 6.0), -0.83);
}

int orc_material_evaluate(double T, double P_v, orc_coeffs* out) { /* materials.cpp:91-114 */
    const double tol = 1e-9;
    const double P_s = (T >= kBoxTMin - tol && T <= kBoxTMax + tol) ? orc_saturation_pressure(T) : 0.0;
    const double phi = P_s > 0.0 ? P_v / P_s : -1.0;
    if (!(P_s > 0.0) || !(phi >= kBoxPhiMin * (1.0 - tol) && phi <= kBoxPhiMax * (1.0 + tol)))
        return HYG_EDOMAIN;
    const double f = plateau(kRv * T * (-log(phi)));          /* moisture_content :61-63 */
    /* moisture_storage :80-89 */
    const double x = -log(P_v / P_s);
    const double rt = kRv * T;
    const double x1 = kC1 * rt * x, x2 = kC2 * rt * x;
    const double t1 = 30.62 * (kC1 * rt / P_v) * pow(x1, 0.65) * pow(1.0 + pow(x1, 1.65), -1.39);
    const double t2 = 549.5 * (kC2 * rt / P_v) * pow(x2, 5.0) * pow(1.0 + pow(x2, 6.0), -1.83);
    const double c_M = t1 + t2;
    out->c_M = c_M;
    /* moisture_transport :74-78 */
    const double r = 2.0 * P_v / P_s;
    out->k_M = 1.97e-10 * pow(10.0, 1.44 - 0.07 * log10(r)) + 1.77e-7 * exp(-8.0 * (r - 2.0) * (r - 2.0));
    out->c_TT = kRho0 * kC0 + kCw * f;
    out->k_TT = 0.2 + 0.0045 * f;                              /* thermal_conductivity :70-72 */
    out->c_TM = kCw * (T - 273.15) * c_M;
    const double z = 1.0 - f / kSat;                           /* vapour_permeability :65-68 */
    out->k_TM = kLv * (1.88e-6 / T * z / (0.503 * z * z + 0.497));
    return 0;
}

static double clampd(double x, double lo, double hi) { return x < lo ? lo : (hi < x ? hi : x); }

int orc_material_evaluate_clamped(double T, double P_v, orc_coeffs* out) { /* :116-121 */
    const double Tc = clampd(T, kBoxTMin, kBoxTMax);
    const double P_s = orc_saturation_pressure(Tc);
    const double phi = clampd(P_v / P_s, kBoxPhiMin, kBoxPhiMax);
    return orc_material_evaluate(Tc, phi * P_s, out);
}

static const orc_coeffs kUnit = {1.0, 1.0, 1.0, 1.0, 1.0, 1.0};

/* CoefficientModel::star / star_clamped (wall.cpp:43-58) and the analytic
 * functor passed as a StarFn to oracle::df_step (df_oracle.hpp:19). */
int orc_star(const orc_model* m, double u, double v, int strict, orc_coeffs* out) {
    if (m == NULL || m->kind == ORC_COEFF_CONSTANT) {
        *out = kUnit;
        return 0;
    }
    if (m->kind == ORC_COEFF_ANALYTIC_D) {
        *out = kUnit;
        const double d = v - m->p[3];
        out->k_M = 1.0 + m->p[0] * v + m->p[1] * exp(-m->p[2] * d * d);
        return 0;
    }
    orc_coeffs a;
    const int rc = strict ? orc_material_evaluate(u * m->T_i, v * m->P_vi, &a)
                          : orc_material_evaluate_clamped(u * m->T_i, v * m->P_vi, &a);
    if (rc) return rc;
    const orc_coeffs* b = &m->reference;
    out->c_M = a.c_M / b->c_M;
    out->k_M = a.k_M / b->k_M;
    out->c_TT = a.c_TT / b->c_TT;
    out->k_TT = a.k_TT / b->k_TT;
    out->c_TM = a.c_TM / b->c_TM;
    out->k_TM = a.k_TM / b->k_TM;
    return 0;
}

/* ---------------- wall steps: wall.cpp ----------------------------------- */
void orc_df_step_linear(int n, const double* prev, const double* curr, double lambda,
                        double* next) { /* wall.cpp:60-71 */
    next[0] = curr[0];
    next[n - 1] = curr[n - 1];
    const double a0 = (1.0 - lambda) / (1.0 + lambda);
    const double a1 = lambda / (1.0 + lambda);
    for (int j = 1; j + 1 < n; ++j) next[j] = a0 * prev[j] + a1 * (curr[j + 1] + curr[j - 1]);
}

/* rotate (wall.cpp:80-83): prev <- curr, curr <- next */
static void rotate(int n, double* prev, double* curr, const double* next) {
    memcpy(prev, curr, sizeof(double) * (size_t)n);
    memcpy(curr, next, sizeof(double) * (size_t)n);
}

void orc_df_step_coupled(orc_field* f, double dx, const hyg_wall_groups* p, const orc_face* left,
                         const orc_face* right, double dt) { /* wall.cpp:144-194 */
    const int n = f->n;
    const double lam = 2.0 * p->Fo_M * dt / (dx * dx);
    const double mu = 2.0 * p->Fo_TT * dt / (dx * dx);
    const double beta = 2.0 * p->Fo_TM * p->gamma * dt / (dx * dx);
    const double ratio = p->Fo_TT != 0.0 ? p->Fo_TM * p->gamma / p->Fo_TT : 0.0;

    double* vn = (double*)malloc(sizeof(double) * (size_t)n * 2);
    double* un = vn + n;
    const double *vp = f->vp, *vc = f->vc, *up = f->up, *uc = f->uc;

    for (int j = 1; j + 1 < n; ++j)
        vn[j] = ((1.0 - lam) * vp[j] + lam * (vc[j + 1] + vc[j - 1])) / (1.0 + lam);

    const int jb[2] = {0, n - 1}, jn[2] = {1, n - 2};
    const orc_face* bc[2] = {left, right};
    for (int k = 0; k < 2; ++k) {
        const orc_face* b = bc[k];
        const double cpl = lam * dx * b->Bi_M;
        vn[jb[k]] = ((1.0 - lam - cpl) * vp[jb[k]] + 2.0 * lam * vc[jn[k]] +
                     2.0 * lam * dx * (b->Bi_M * b->v_inf + b->g_inf)) /
                    (1.0 + lam + cpl);
    }
    for (int j = 1; j + 1 < n; ++j) {
        un[j] = ((1.0 - mu) * up[j] + mu * (uc[j + 1] + uc[j - 1]) + (p->gamma - beta) * vp[j] +
                 beta * (vc[j + 1] + vc[j - 1]) - (p->gamma + beta) * vn[j]) /
                (1.0 + mu);
    }
    for (int k = 0; k < 2; ++k) {
        const orc_face* b = bc[k];
        const double vbar = 0.5 * (vn[jb[k]] + vp[jb[k]]);
        const double vg = vc[jn[k]] - 2.0 * dx * (b->Bi_M * (vbar - b->v_inf) - b->g_inf);
        const double cplu = mu * dx * b->Bi_TT;
        un[jb[k]] = ((1.0 - mu - cplu) * up[jb[k]] + 2.0 * mu * uc[jn[k]] +
                     mu * ratio * (vc[jn[k]] - vg) +
                     2.0 * mu * dx * (b->Bi_TT * b->u_inf - b->Bi_TM * (vbar - b->v_inf) + b->q_inf) +
                     (p->gamma - beta) * vp[jb[k]] + beta * (vc[jn[k]] + vg) -
                     (p->gamma + beta) * vn[jb[k]]) /
                    (1.0 + mu + cplu);
    }
    rotate(n, f->vp, f->vc, vn);
    rotate(n, f->up, f->uc, un);
    f->t_star += dt;
    free(vn);
}

/* StarTables (wall.cpp:89-138): node[n], half[n-1]; NULL tables = unit */
typedef struct { orc_coeffs* node; orc_coeffs* half; int unit; } star_tables;

/* where the last strict evaluation left the box: node j or half node j+1/2
 * (the "[node j]" / "[half node j+1/2]" annotation of wall.cpp:105-126) */
static int g_dom_node = -1, g_dom_half = 0;
void orc_last_domain(int* node, int* half) {
    *node = g_dom_node;
    *half = g_dom_half;
}

static int build_tables(star_tables* s, const orc_model* m, int n, const double* u,
                        const double* v, int strict) {
    s->node = s->half = NULL;
    s->unit = (m == NULL || m->kind == ORC_COEFF_CONSTANT);
    if (s->unit) return 0;
    s->node = (orc_coeffs*)malloc(sizeof(orc_coeffs) * (size_t)(2 * n - 1));
    s->half = s->node + n;
    for (int j = 0; j < n; ++j) {
        const int rc = orc_star(m, u[j], v[j], strict, &s->node[j]);
        if (rc) {
            g_dom_node = j;
            g_dom_half = 0;
            return rc;
        }
    }
    for (int j = 0; j + 1 < n; ++j) {
        const double um = 0.5 * (u[j] + u[j + 1]);
        const double vm = 0.5 * (v[j] + v[j + 1]);
        const int rc = orc_star(m, um, vm, strict, &s->half[j]);
        if (rc) {
            g_dom_node = j;
            g_dom_half = 1;
            return rc;
        }
    }
    return 0;
}
static void free_tables(star_tables* s) { free(s->node); }
static const orc_coeffs* at_node(const star_tables* s, int j) { return s->unit ? &kUnit : &s->node[j]; }
static const orc_coeffs* at_half(const star_tables* s, int j) { return s->unit ? &kUnit : &s->half[j]; }

/* df_step_nonlinear (wall.cpp:196-264) in pieces over node ranges, so the
 * threaded long-wall march (orc_march_long_mt) runs the very statements the
 * serial step runs: interior v rows of [j0, j1), a face's v row, interior u
 * rows of [j0, j1) (u reads only its own node's new v), a face's u row. */
typedef struct {
    int n;
    double dx, a, b_, g_, ratio;
    const hyg_wall_groups* p;
} nl_consts;

static nl_consts nl_setup(int n, double dx, const hyg_wall_groups* p, double dt) {
    nl_consts c;
    c.n = n;
    c.dx = dx;
    c.p = p;
    c.a = p->Fo_M * dt / (dx * dx);
    c.b_ = p->Fo_TT * dt / (dx * dx);
    c.g_ = p->Fo_TM * p->gamma * dt / (dx * dx);
    c.ratio = p->Fo_TT != 0.0 ? p->Fo_TM * p->gamma / p->Fo_TT : 0.0;
    return c;
}

static void nl_v_rows(const nl_consts* c, const star_tables* s, const orc_field* f, double* vn, int j0, int j1) {
    const double a = c->a;
    const double *vp = f->vp, *vc = f->vc;
    if (j0 < 1) j0 = 1;
    if (j1 > c->n - 1) j1 = c->n - 1;
    for (int j = j0; j < j1; ++j) {
        const double kp = at_half(s, j)->k_M, km = at_half(s, j - 1)->k_M, cm = at_node(s, j)->c_M;
        vn[j] = ((cm - a * (kp + km)) * vp[j] + 2.0 * a * (kp * vc[j + 1] + km * vc[j - 1])) /
                (cm + a * (kp + km));
    }
}

static void nl_v_face(const nl_consts* c, const star_tables* s, const orc_field* f, double* vn, int k,
                      const orc_face* b) {
    const int n = c->n, jb = k == 0 ? 0 : n - 1, jn = k == 0 ? 1 : n - 2;
    const double a = c->a, dx = c->dx;
    const double km_b = at_node(s, jb)->k_M;
    const double kp_b = at_half(s, jb == 0 ? 0 : n - 2)->k_M;
    const double cm = at_node(s, jb)->c_M;
    const double cpl = 2.0 * a * dx * b->Bi_M;
    vn[jb] = ((cm - a * (kp_b + km_b) - cpl) * f->vp[jb] + 2.0 * a * (kp_b + km_b) * f->vc[jn] +
              4.0 * a * dx * (b->Bi_M * b->v_inf + b->g_inf)) /
             (cm + a * (kp_b + km_b) + cpl);
}

static void nl_u_rows(const nl_consts* c, const star_tables* s, const orc_field* f, const double* vn, double* un,
                      int j0, int j1) {
    const double b_ = c->b_, g_ = c->g_, gamma = c->p->gamma;
    const double *vp = f->vp, *vc = f->vc, *up = f->up, *uc = f->uc;
    if (j0 < 1) j0 = 1;
    if (j1 > c->n - 1) j1 = c->n - 1;
    for (int j = j0; j < j1; ++j) {
        const double ktp = at_half(s, j)->k_TT, ktm = at_half(s, j - 1)->k_TT;
        const double kmp = at_half(s, j)->k_TM, kmm = at_half(s, j - 1)->k_TM;
        const double ctt = at_node(s, j)->c_TT, ctm = at_node(s, j)->c_TM;
        un[j] = ((ctt - b_ * (ktp + ktm)) * up[j] - gamma * ctm * (vn[j] - vp[j]) +
                 2.0 * b_ * (ktp * uc[j + 1] + ktm * uc[j - 1]) +
                 2.0 * g_ * (kmp * vc[j + 1] + kmm * vc[j - 1]) - g_ * (kmp + kmm) * (vn[j] + vp[j])) /
                (ctt + b_ * (ktp + ktm));
    }
}

static void nl_u_face(const nl_consts* c, const star_tables* s, const orc_field* f, const double* vn, double* un,
                      int k, const orc_face* b) {
    const int n = c->n, jb = k == 0 ? 0 : n - 1, jn = k == 0 ? 1 : n - 2;
    const double b_ = c->b_, g_ = c->g_, dx = c->dx, ratio = c->ratio;
    const double *vp = f->vp, *vc = f->vc, *up = f->up, *uc = f->uc;
    const orc_coeffs* nb = at_node(s, jb);
    const double kt_b = nb->k_TT, kTM_b = nb->k_TM, km_b = nb->k_M;
    const orc_coeffs* hb = at_half(s, jb == 0 ? 0 : n - 2);
    const double ktp_b = hb->k_TT, kmp_b = hb->k_TM;
    const double vbar = 0.5 * (vn[jb] + vp[jb]);
    const double vg = vc[jn] - (2.0 * dx / km_b) * (b->Bi_M * (vbar - b->v_inf) - b->g_inf);
    const double cplu = 2.0 * b_ * dx * b->Bi_TT;
    un[jb] = ((nb->c_TT - b_ * (ktp_b + kt_b) - cplu) * up[jb] - c->p->gamma * nb->c_TM * (vn[jb] - vp[jb]) +
              2.0 * b_ * (ktp_b + kt_b) * uc[jn] + 2.0 * b_ * ratio * kTM_b * (vc[jn] - vg) -
              4.0 * b_ * dx * (b->Bi_TM * (vbar - b->v_inf) - b->q_inf) + 2.0 * cplu * b->u_inf +
              2.0 * g_ * (kmp_b * vc[jn] + kTM_b * vg) - g_ * (kmp_b + kTM_b) * (vn[jb] + vp[jb])) /
             (nb->c_TT + b_ * (ktp_b + kt_b) + cplu);
}

int orc_df_step_nonlinear(orc_field* f, double dx, const hyg_wall_groups* p, const orc_model* m,
                          const orc_face* left, const orc_face* right,
                          double dt) { /* wall.cpp:196-264 */
    const int n = f->n;
    const nl_consts c = nl_setup(n, dx, p, dt);
    star_tables s;
    const int rc = build_tables(&s, m, n, f->uc, f->vc, 1);
    if (rc) {
        free_tables(&s);
        return rc;
    }
    double* vn = (double*)malloc(sizeof(double) * (size_t)n * 2);
    double* un = vn + n;
    nl_v_rows(&c, &s, f, vn, 1, n - 1);                 /* wall.cpp:213-217 */
    nl_v_face(&c, &s, f, vn, 0, left);                  /* wall.cpp:218-229 */
    nl_v_face(&c, &s, f, vn, 1, right);
    nl_u_rows(&c, &s, f, vn, un, 1, n - 1);             /* wall.cpp:231-240 */
    nl_u_face(&c, &s, f, vn, un, 0, left);              /* wall.cpp:241-259 */
    nl_u_face(&c, &s, f, vn, un, 1, right);
    rotate(n, f->vp, f->vc, vn);                        /* wall.cpp:261-263 */
    rotate(n, f->up, f->uc, un);
    f->t_star += dt;
    free(vn);
    free_tables(&s);
    return 0;
}

void orc_euler_explicit_step(orc_field* f, double dx, const hyg_wall_groups* p,
                             const orc_model* m, const orc_face* left, const orc_face* right,
                             double dt) { /* wall.cpp:266-317 */
    const int n = f->n;
    star_tables s;
    build_tables(&s, m, n, f->uc, f->vc, 0);
    const double *vc = f->vc, *uc = f->uc;
    double* vn = (double*)malloc(sizeof(double) * (size_t)n * 2);
    double* un = vn + n;
    double vg[2], ug[2];
    const int jb[2] = {0, n - 1}, jn[2] = {1, n - 2};
    const orc_face* bcs[2] = {left, right};
    for (int i = 0; i < 2; ++i) {
        const orc_face* b = bcs[i];
        const orc_coeffs* nb = at_node(&s, jb[i]);
        vg[i] = vc[jn[i]] - (2.0 * dx / nb->k_M) * (b->Bi_M * (vc[jb[i]] - b->v_inf) - b->g_inf);
        ug[i] = uc[jn[i]] +
                (p->Fo_TM * p->gamma * nb->k_TM) / (p->Fo_TT * nb->k_TT) * (vc[jn[i]] - vg[i]) -
                (2.0 * dx / nb->k_TT) *
                    (b->Bi_TT * (uc[jb[i]] - b->u_inf) + b->Bi_TM * (vc[jb[i]] - b->v_inf) - b->q_inf);
    }
    const double rdt = dt / (dx * dx);
    for (int j = 0; j < n; ++j) {
        const double vL = j == 0 ? vg[0] : vc[j - 1];
        const double vR = j == n - 1 ? vg[1] : vc[j + 1];
        const double uL = j == 0 ? ug[0] : uc[j - 1];
        const double uR = j == n - 1 ? ug[1] : uc[j + 1];
        const double km = j == 0 ? at_node(&s, 0)->k_M : at_half(&s, j - 1)->k_M;
        const double kp = j == n - 1 ? at_node(&s, n - 1)->k_M : at_half(&s, j)->k_M;
        const double ktm = j == 0 ? at_node(&s, 0)->k_TT : at_half(&s, j - 1)->k_TT;
        const double ktp = j == n - 1 ? at_node(&s, n - 1)->k_TT : at_half(&s, j)->k_TT;
        const double kmm = j == 0 ? at_node(&s, 0)->k_TM : at_half(&s, j - 1)->k_TM;
        const double kmp = j == n - 1 ? at_node(&s, n - 1)->k_TM : at_half(&s, j)->k_TM;
        const double div_v = kp * (vR - vc[j]) - km * (vc[j] - vL);
        vn[j] = vc[j] + rdt * p->Fo_M * div_v / at_node(&s, j)->c_M;
        const double div_u = ktp * (uR - uc[j]) - ktm * (uc[j] - uL);
        const double div_vm = kmp * (vR - vc[j]) - kmm * (vc[j] - vL);
        un[j] = uc[j] + (rdt * (p->Fo_TT * div_u + p->Fo_TM * p->gamma * div_vm) -
                         p->gamma * at_node(&s, j)->c_TM * (vn[j] - vc[j])) /
                            at_node(&s, j)->c_TT;
    }
    rotate(n, f->vp, f->vc, vn);
    rotate(n, f->up, f->uc, un);
    f->t_star += dt;
    free(vn);
    free_tables(&s);
}

/* tridiag.hpp:11-23: overwrites rhs; modifies diag */
static void solve_tridiagonal(int n, const double* lower, double* diag, const double* upper,
                              double* rhs) {
    for (int i = 1; i < n; ++i) {
        const double m = lower[i] / diag[i - 1];
        diag[i] -= m * upper[i - 1];
        rhs[i] -= m * rhs[i - 1];
    }
    rhs[n - 1] /= diag[n - 1];
    for (int i = n - 1; i-- > 0;) rhs[i] = (rhs[i] - upper[i] * rhs[i + 1]) / diag[i];
}

/* FactoredTridiag (wall.cpp:322-346) */
static void factor_tridiag(int n, const double* lo, const double* di, const double* up, double* m,
                           double* inv) {
    for (int i = 0; i < n; ++i) m[i] = inv[i] = 0.0;
    double dp = di[0];
    inv[0] = 1.0 / dp;
    for (int i = 1; i < n; ++i) {
        m[i] = lo[i] * inv[i - 1];
        dp = di[i] - m[i] * up[i - 1];
        inv[i] = 1.0 / dp;
    }
}
static void solve_factored(int n, const double* m, const double* inv, const double* up, double* x) {
    for (int i = 1; i < n; ++i) x[i] -= m[i] * x[i - 1];
    x[n - 1] *= inv[n - 1];
    for (int i = n - 1; i-- > 0;) x[i] = (x[i] - up[i] * x[i + 1]) * inv[i];
}

/* implicit_wall_pass_unit (wall.cpp:398-429) with the factorisation of
 * cached_factors (wall.cpp:360-395) rebuilt per call (same arithmetic). */
static void implicit_pass_unit(const orc_field* base, double dx, const hyg_wall_groups* p,
                               const orc_face* left, const orc_face* right, double dt,
                               double* out_u, double* out_v) {
    const int n = base->n;
    const double r = p->Fo_M * dt / (dx * dx);
    const double rb = p->Fo_TT * dt / (dx * dx);
    const double rg = p->Fo_TM * p->gamma * dt / (dx * dx);
    double* w = (double*)calloc((size_t)n * 5, sizeof(double));
    double *lo = w, *di = w + n, *up = w + 2 * n, *mm = w + 3 * n, *inv = w + 4 * n;
    /* moisture matrix with unit coefficients (wall.cpp:370-380) */
    for (int j = 1; j + 1 < n; ++j) {
        lo[j] = -r;
        di[j] = 1.0 + 2.0 * r;
        up[j] = -r;
    }
    di[0] = 1.0 + 2.0 * r + 2.0 * r * dx * left->Bi_M;
    up[0] = -2.0 * r;
    di[n - 1] = 1.0 + 2.0 * r + 2.0 * r * dx * right->Bi_M;
    lo[n - 1] = -2.0 * r;
    factor_tridiag(n, lo, di, up, mm, inv);
    memcpy(out_v, base->vc, sizeof(double) * (size_t)n);
    out_v[0] += 2.0 * r * dx * (left->Bi_M * left->v_inf + left->g_inf);
    out_v[n - 1] += 2.0 * r * dx * (right->Bi_M * right->v_inf + right->g_inf);
    solve_factored(n, mm, inv, up, out_v);
    const double* vN = out_v;
    for (int j = 1; j + 1 < n; ++j)
        out_u[j] = base->uc[j] - p->gamma * (vN[j] - base->vc[j]) + rg * (vN[j + 1] - 2.0 * vN[j] + vN[j - 1]);
    out_u[0] = base->uc[0] - p->gamma * (vN[0] - base->vc[0]) + 2.0 * rg * (vN[1] - vN[0]) +
               2.0 * rb * dx * (left->Bi_TT * left->u_inf - left->Bi_TM * (vN[0] - left->v_inf) + left->q_inf);
    out_u[n - 1] = base->uc[n - 1] - p->gamma * (vN[n - 1] - base->vc[n - 1]) +
                   2.0 * rg * (vN[n - 2] - vN[n - 1]) +
                   2.0 * rb * dx *
                       (right->Bi_TT * right->u_inf - right->Bi_TM * (vN[n - 1] - right->v_inf) + right->q_inf);
    /* energy matrix with unit coefficients (wall.cpp:382-393) */
    for (int j = 1; j + 1 < n; ++j) {
        lo[j] = -rb;
        di[j] = 1.0 + 2.0 * rb;
        up[j] = -rb;
    }
    di[0] = 1.0 + 2.0 * rb + 2.0 * rb * dx * left->Bi_TT;
    up[0] = -2.0 * rb;
    lo[0] = 0.0;
    di[n - 1] = 1.0 + 2.0 * rb + 2.0 * rb * dx * right->Bi_TT;
    lo[n - 1] = -2.0 * rb;
    up[n - 1] = 0.0;
    factor_tridiag(n, lo, di, up, mm, inv);
    solve_factored(n, mm, inv, up, out_u);
    free(w);
}

void orc_implicit_wall_pass(const orc_field* base, double dx, const hyg_wall_groups* p,
                            const orc_model* m, const orc_face* left, const orc_face* right,
                            double dt, const double* iter_u, const double* iter_v, double* out_u,
                            double* out_v) { /* wall.cpp:433-513 */
    if (m == NULL || m->kind == ORC_COEFF_CONSTANT) {
        implicit_pass_unit(base, dx, p, left, right, dt, out_u, out_v);
        return;
    }
    const int n = base->n;
    const double r = p->Fo_M * dt / (dx * dx);
    const double rb = p->Fo_TT * dt / (dx * dx);
    const double rg = p->Fo_TM * p->gamma * dt / (dx * dx);
    star_tables s;
    build_tables(&s, m, n, iter_u, iter_v, 0);
    double* w = (double*)calloc((size_t)n * 4, sizeof(double));
    double *lo = w, *di = w + n, *up_ = w + 2 * n, *rhs = w + 3 * n;
    const int jb[2] = {0, n - 1}, jn[2] = {1, n - 2};
    const orc_face* bcs[2] = {left, right};
    for (int j = 1; j + 1 < n; ++j) {
        const double kp = at_half(&s, j)->k_M, km = at_half(&s, j - 1)->k_M;
        lo[j] = -r * km;
        di[j] = at_node(&s, j)->c_M + r * (kp + km);
        up_[j] = -r * kp;
        rhs[j] = at_node(&s, j)->c_M * base->vc[j];
    }
    for (int k = 0; k < 2; ++k) {
        const orc_face* b = bcs[k];
        const double km_b = at_node(&s, jb[k])->k_M;
        const double kp_b = at_half(&s, jb[k] == 0 ? 0 : n - 2)->k_M;
        di[jb[k]] = at_node(&s, jb[k])->c_M + r * (kp_b + km_b) + 2.0 * r * dx * b->Bi_M;
        const double off = -r * (kp_b + km_b);
        if (jb[k] == 0) up_[0] = off; else lo[n - 1] = off;
        rhs[jb[k]] = at_node(&s, jb[k])->c_M * base->vc[jb[k]] + 2.0 * r * dx * (b->Bi_M * b->v_inf + b->g_inf);
    }
    memcpy(out_v, rhs, sizeof(double) * (size_t)n);
    solve_tridiagonal(n, lo, di, up_, out_v);
    const double* vN = out_v;
    for (int j = 1; j + 1 < n; ++j) {
        const double ktp = at_half(&s, j)->k_TT, ktm = at_half(&s, j - 1)->k_TT;
        const double kmp = at_half(&s, j)->k_TM, kmm = at_half(&s, j - 1)->k_TM;
        lo[j] = -rb * ktm;
        di[j] = at_node(&s, j)->c_TT + rb * (ktp + ktm);
        up_[j] = -rb * ktp;
        rhs[j] = at_node(&s, j)->c_TT * base->uc[j] - p->gamma * at_node(&s, j)->c_TM * (vN[j] - base->vc[j]) +
                 rg * (kmp * (vN[j + 1] - vN[j]) - kmm * (vN[j] - vN[j - 1]));
    }
    for (int k = 0; k < 2; ++k) {
        const orc_face* b = bcs[k];
        const orc_coeffs* nb = at_node(&s, jb[k]);
        const double kt_b = nb->k_TT, kTM_b = nb->k_TM;
        const orc_coeffs* hb = at_half(&s, jb[k] == 0 ? 0 : n - 2);
        di[jb[k]] = nb->c_TT + rb * (hb->k_TT + kt_b) + 2.0 * rb * dx * b->Bi_TT;
        const double off = -rb * (hb->k_TT + kt_b);
        if (jb[k] == 0) up_[0] = off; else lo[n - 1] = off;
        rhs[jb[k]] = nb->c_TT * base->uc[jb[k]] - p->gamma * nb->c_TM * (vN[jb[k]] - base->vc[jb[k]]) +
                     rg * (hb->k_TM + kTM_b) * (vN[jn[k]] - vN[jb[k]]) +
                     2.0 * rb * dx * (b->Bi_TT * b->u_inf - b->Bi_TM * (vN[jb[k]] - b->v_inf) + b->q_inf);
    }
    memcpy(out_u, rhs, sizeof(double) * (size_t)n);
    solve_tridiagonal(n, lo, di, up_, out_u);
    free(w);
    free_tables(&s);
}

int orc_euler_implicit_step(orc_field* f, double dx, const hyg_wall_groups* p, const orc_model* m,
                            const orc_face* L, const orc_face* R, double dt, double eta,
                            int max_subiters, double* residual) { /* wall.cpp:515-550 */
    if (!(eta > 0.0)) return -HYG_EINVAL;
    const int n = f->n;
    double* w = (double*)malloc(sizeof(double) * (size_t)n * 4);
    double *ui = w, *vi = w + n, *uN = w + 2 * n, *vN = w + 3 * n;
    memcpy(ui, f->uc, sizeof(double) * (size_t)n);
    memcpy(vi, f->vc, sizeof(double) * (size_t)n);
    int pass = 0;
    for (;;) {
        ++pass;
        orc_implicit_wall_pass(f, dx, p, m, L, R, dt, ui, vi, uN, vN);
        double diff = 0.0;
        for (int j = 0; j < n; ++j) {
            diff = fmax(diff, fabs(uN[j] - ui[j]));
            diff = fmax(diff, fabs(vN[j] - vi[j]));
        }
        double* t = ui; ui = uN; uN = t;
        t = vi; vi = vN; vN = t;
        if (m == NULL || m->kind == ORC_COEFF_CONSTANT) break;
        if (diff < eta) break;
        if (pass >= max_subiters) {
            if (residual) *residual = diff;
            free(w);
            return -HYG_ECONVERGE;
        }
    }
    rotate(n, f->vp, f->vc, vi);
    rotate(n, f->up, f->uc, ui);
    f->t_star += dt;
    free(w);
    return pass;
}

double orc_max_abs_field(const orc_field* f) { /* wall.cpp:579-587 */
    double m = 0.0;
    for (int j = 0; j < f->n; ++j) m = fmax(m, fabs(f->uc[j]));
    for (int j = 0; j < f->n; ++j) m = fmax(m, fabs(f->vc[j]));
    for (int j = 0; j < f->n; ++j)
        if (!isfinite(f->uc[j]) || !isfinite(f->vc[j])) return INFINITY;
    return m;
}

/* ---------------- batched marches ---------------------------------------- */
static void face_of(const orc_batch* b, int w, int k, int64_t layer, orc_face* f) {
    const hyg_face_biot* bi = &b->biot[2 * w + k];
    const hyg_ambient* a = &b->table[(layer - b->layer0) * b->n_channels + b->chan[2 * w + k]];
    f->Bi_M = bi->Bi_M;
    f->Bi_TT = bi->Bi_TT;
    f->Bi_TM = bi->Bi_TM;
    f->u_inf = a->u_inf;
    f->v_inf = a->v_inf;
    f->g_inf = a->g_inf;
    f->q_inf = a->q_inf;
}

static orc_field field_of(const orc_batch* b, int w) {
    const size_t o = (size_t)w * (size_t)b->n;
    orc_field f = {b->n, b->up + o, b->uc + o, b->vp + o, b->vc + o, 0.0};
    return f;
}

typedef struct {
    const orc_batch* b;
    const orc_model* m;
    int mode;   /* 0 coupled, 1 nonlinear, 2 explicit boot, 3 implicit boot, 4 implicit march */
    int nsteps;
    double dt, eta;
    int max_subiters;
    int w0, w1;
    int64_t fail_layer;
    int fail_wall;
    int rc;
    long passes;
} job;

static void* run_job(void* arg) {
    job* J = (job*)arg;
    const orc_batch* b = J->b;
    J->fail_layer = -1;
    J->fail_wall = -1;
    J->rc = 0;
    J->passes = 0;
    for (int w = J->w0; w < J->w1; ++w) {
        orc_field f = field_of(b, w);
        orc_face L, R;
        if (J->mode == 2 || J->mode == 3) {
            const int64_t lay = b->layer0 + (J->mode == 3 ? 1 : 0);
            face_of(b, w, 0, lay, &L);
            face_of(b, w, 1, lay, &R);
            if (J->mode == 2) {
                orc_euler_explicit_step(&f, b->dx, &b->groups[w], J->m, &L, &R, J->dt);
            } else {
                double res = 0.0;
                const int rc = orc_euler_implicit_step(&f, b->dx, &b->groups[w], J->m, &L, &R, J->dt,
                                                       J->eta, J->max_subiters, &res);
                if (rc < 0) { J->rc = -rc; J->fail_wall = w; return NULL; }
                J->passes += rc;
            }
            continue;
        }
        for (int s = 0; s < J->nsteps; ++s) {
            const int64_t lay = b->layer0 + s;
            if (J->fail_layer >= 0 && lay + 1 >= J->fail_layer) break;  /* an earlier wall failed first */
            if (J->mode == 4) {
                face_of(b, w, 0, lay + 1, &L);
                face_of(b, w, 1, lay + 1, &R);
                double res = 0.0;
                const int rc = orc_euler_implicit_step(&f, b->dx, &b->groups[w], J->m, &L, &R, J->dt,
                                                       J->eta, J->max_subiters, &res);
                if (rc < 0) { J->rc = -rc; J->fail_wall = w; return NULL; }
                J->passes += rc;
                continue;
            }
            face_of(b, w, 0, lay, &L);
            face_of(b, w, 1, lay, &R);
            if (J->mode == 0) {
                orc_df_step_coupled(&f, b->dx, &b->groups[w], &L, &R, J->dt);
            } else {
                const int rc = orc_df_step_nonlinear(&f, b->dx, &b->groups[w], J->m, &L, &R, J->dt);
                if (rc) { J->rc = rc; J->fail_wall = w; J->fail_layer = lay + 1; return NULL; }
            }
            const double mx = orc_max_abs_field(&f);
            if (!(mx <= b->divergence_norm)) {
                if (J->fail_layer < 0 || lay + 1 < J->fail_layer) {
                    J->fail_layer = lay + 1;
                    J->fail_wall = w;
                }
                break;
            }
        }
    }
    return NULL;
}

static int run_jobs(const orc_batch* b, const orc_model* m, int mode, int nsteps, double dt,
                    double eta, int max_subiters, int nthreads, int64_t* fail_layer,
                    int* fail_wall, long* passes) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > b->n_walls) nthreads = b->n_walls > 0 ? b->n_walls : 1;
    job* jobs = (job*)calloc((size_t)nthreads, sizeof(job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int i = 0; i < nthreads; ++i) {
        jobs[i].b = b;
        jobs[i].m = m;
        jobs[i].mode = mode;
        jobs[i].nsteps = nsteps;
        jobs[i].dt = dt;
        jobs[i].eta = eta;
        jobs[i].max_subiters = max_subiters;
        jobs[i].w0 = (int)((int64_t)b->n_walls * i / nthreads);
        jobs[i].w1 = (int)((int64_t)b->n_walls * (i + 1) / nthreads);
        if (nthreads == 1) run_job(&jobs[i]);
        else pthread_create(&th[i], NULL, run_job, &jobs[i]);
    }
    int rc = 0;
    int64_t fl = -1;
    int fw = -1;
    long total = 0;
    for (int i = 0; i < nthreads; ++i) {
        if (nthreads > 1) pthread_join(th[i], NULL);
        total += jobs[i].passes;
        if (jobs[i].rc && !rc) { rc = jobs[i].rc; fw = jobs[i].fail_wall; fl = jobs[i].fail_layer; }
        if (jobs[i].fail_layer >= 0 && (fl < 0 || jobs[i].fail_layer < fl ||
                                        (jobs[i].fail_layer == fl && jobs[i].fail_wall < fw))) {
            fl = jobs[i].fail_layer;
            fw = jobs[i].fail_wall;
        }
    }
    if (!rc && fl >= 0) rc = HYG_EDIVERGED;
    if (fail_layer) *fail_layer = fl;
    if (fail_wall) *fail_wall = fw;
    if (passes) *passes = total;
    free(jobs);
    free(th);
    return rc;
}

int orc_march_coupled(const orc_batch* b, int nsteps, double dt, int nthreads,
                      int64_t* fail_layer, int* fail_wall) {
    return run_jobs(b, NULL, 0, nsteps, dt, 0.0, 0, nthreads, fail_layer, fail_wall, NULL);
}
int orc_march_nonlinear(const orc_batch* b, const orc_model* m, int nsteps, double dt,
                        int nthreads, int64_t* fail_layer, int* fail_wall) {
    return run_jobs(b, m, 1, nsteps, dt, 0.0, 0, nthreads, fail_layer, fail_wall, NULL);
}
int orc_bootstrap_batch(const orc_batch* b, const orc_model* m, int kind, double dt, double eta,
                        int max_subiters, int nthreads) {
    return run_jobs(b, m, kind == HYG_BOOT_EXPLICIT ? 2 : 3, 1, dt, eta, max_subiters, nthreads,
                    NULL, NULL, NULL);
}
int orc_march_implicit(const orc_batch* b, const orc_model* m, int nsteps, double dt, double eta,
                       int max_subiters, int nthreads, long* total_passes) {
    return run_jobs(b, m, 4, nsteps, dt, eta, max_subiters, nthreads, NULL, NULL, total_passes);
}

/* ---------------- zones and building: zone.cpp, building.cpp ------------- */
void orc_zone_rhs(const hyg_model_desc* m, int zi, double u_a, double v_a, const double* u_s,
                  const double* v_s, const double* zu, const double* zv, double u_inf,
                  double v_inf, double t, double* du_out, double* dv_out) { /* zone.cpp:26-53 */
    const hyg_zone_desc* z = &m->zones[zi];
    const hyg_zone_sources* src = &m->zone_sources[z->sources];
    double du = orc_signal(&src->q_o, t) + orc_signal(&src->q_h, t) +
                z->q_v1 * (u_inf * v_inf - u_a * v_a) + z->q_v2 * (u_inf - u_a);
    double dv = orc_signal(&src->g_o, t) + z->g_v * (v_inf - v_a);
    for (int i = 0; i < z->n_interzone; ++i) {
        const hyg_interzone_link* l = &z->interzone[i];
        const double pu = zu[l->peer], pv = zv[l->peer];
        du += l->q_inz1 * (pu * pv - u_a * v_a) + l->q_inz2 * (pu - u_a);
        dv += l->g_inz * (pv - v_a);
    }
    const double sign = z->moisture_sign == HYG_MOISTURE_AS_PRINTED ? 1.0 : -1.0;
    for (int i = 0; i < z->n_walls; ++i) {
        const hyg_zone_wall_link* w = &z->walls[i];
        du += w->Bi_TT * w->theta_T * (u_s[i] - u_a) + w->Bi_TM * w->theta_T * (v_s[i] - v_a);
        dv += sign * w->Bi_M * w->theta_M * (v_a - v_s[i]);
    }
    *du_out = du / (1.0 + z->kappa_a_tt1);
    *dv_out = dv;
}

/* resolve_face (building.cpp:107-126) without radiation */
/* resolve_face (building.cpp:107-126); q_rad = radiation flux of this face */
static void resolve_face(const hyg_model_desc* m, int w, int k, const double* zu, const double* zv,
                         double t, double q_rad, orc_face* f) {
    const hyg_face_biot* bi = &m->biot[2 * w + k];
    const hyg_face_attach* a = &m->attach[2 * w + k];
    f->Bi_M = bi->Bi_M;
    f->Bi_TT = bi->Bi_TT;
    f->Bi_TM = bi->Bi_TM;
    if (a->kind == HYG_FACE_EXTERIOR) {
        const hyg_channel* c = &m->channels[a->index];
        f->u_inf = orc_signal(&c->u_inf, t);
        f->v_inf = orc_signal(&c->v_inf, t);
        f->g_inf = orc_signal(&c->g_inf, t);
        f->q_inf = orc_signal(&c->q_inf, t) + q_rad;
    } else {
        f->u_inf = zu[a->index];
        f->v_inf = zv[a->index];
        f->g_inf = 0.0;
        f->q_inf = q_rad;
    }
}

/* Per-wall coefficient model of a building (BuildingWall::coeffs): constant,
 * the analytic functor, or CoefficientModel::material (wall.cpp:33-41). */
static void wall_model(const hyg_model_desc* m, int w, orc_model* out) {
    memset(out, 0, sizeof *out);
    out->kind = ORC_COEFF_CONSTANT;
    if (m->coeff_kind == HYG_COEFF_ANALYTIC_D) {
        out->kind = ORC_COEFF_ANALYTIC_D;
        memcpy(out->p, m->coeff_params, sizeof out->p);
    } else if (m->coeff_kind == HYG_COEFF_MATERIAL &&
               (m->wall_coeff == NULL || m->wall_coeff[w] == HYG_COEFF_MATERIAL)) {
        const hyg_coeff_set* r = &m->wall_reference[w];
        out->kind = ORC_COEFF_MATERIAL;
        out->T_i = m->T_i;
        out->P_vi = m->P_vi;
        out->reference.c_M = r->c_M;
        out->reference.k_M = r->k_M;
        out->reference.c_TT = r->c_TT;
        out->reference.k_TT = r->k_TT;
        out->reference.c_TM = r->c_TM;
        out->reference.k_TM = r->k_TM;
    }
}

/* radiation_fluxes (building.cpp:88-105) with zone_surface_u (:77-86) and
 * radiative_flux (zone.cpp:55-67) from the wall temperature layer u
 * ([n_walls][n]); q[2*w+face] (zeroed here). */
static void radiation_fluxes(const hyg_model_desc* m, const double* u, double* q) {
    const int n = m->n_nodes, nw = m->n_walls;
    const double sigma = 5.67e-8;                 /* PhysicalConstants materials.hpp:14 */
    for (int i = 0; i < 2 * nw; ++i) q[i] = 0.0;
    double* surf = (double*)malloc(sizeof(double) * (size_t)(nw + 1));
    for (int z = 0; z < m->n_zones; ++z) {
        const hyg_zone_desc* zd = &m->zones[z];
        if (zd->n_radiation == 0) continue;
        for (int i = 0; i < nw; ++i) surf[i] = 0.0;
        for (int i = 0; i < zd->n_walls; ++i) {
            const hyg_zone_wall_link* l = &zd->walls[i];
            surf[l->wall] = u[(size_t)l->wall * (size_t)n + (l->face == 0 ? 0 : (size_t)(n - 1))];
        }
        for (int i = 0; i < zd->n_walls; ++i) {
            const hyg_zone_wall_link* l = &zd->walls[i];
            double q_rw = 0.0;
            for (int r = 0; r < zd->n_radiation; ++r) {
                const hyg_radiation_link* rl = &zd->radiation[r];
                if (rl->receiver_wall != l->wall) continue;
                const double Te = surf[rl->emitter_wall] * m->T_i;
                const double Tr = surf[rl->receiver_wall] * m->T_i;
                q_rw += rl->view_factor * rl->emissivity * sigma * (Te * Te * Te * Te - Tr * Tr * Tr * Tr);
            }
            if (q_rw != 0.0)
                q[2 * l->wall + l->face] += m->wall_thickness[l->wall] * q_rw / (m->T_i * m->wall_k_TT0[l->wall]);
        }
    }
    free(surf);
}

static orc_field bfield(const hyg_model_desc* m, orc_building_state* s, int w) {
    const size_t o = (size_t)w * (size_t)m->n_nodes;
    orc_field f = {m->n_nodes, s->up + o, s->uc + o, s->vp + o, s->vc + o, s->t};
    return f;
}

static int face_node(const hyg_model_desc* m, int face) { return face == 0 ? 0 : m->n_nodes - 1; }

static int g_dom_wall = -1;
int orc_last_domain_wall(void) { return g_dom_wall; }

int orc_step_explicit(const hyg_model_desc* m, orc_building_state* s) { /* building.cpp:152-187 */
    const double t = s->t;
    const double dt = m->dt;
    const int nz = m->n_zones;
    double* zu0 = (double*)malloc(sizeof(double) * (size_t)(2 * nz + 1));
    double* zv0 = zu0 + nz;
    memcpy(zu0, s->zu, sizeof(double) * (size_t)nz);
    memcpy(zv0, s->zv, sizeof(double) * (size_t)nz);
    /* gather samples from layer n before any wall moves (building.cpp:162-164) */
    int total_links = 0;
    for (int z = 0; z < nz; ++z) total_links += m->zones[z].n_walls;
    double* us = (double*)malloc(sizeof(double) * (size_t)(2 * total_links + 1));
    double* vs = us + total_links;
    for (int z = 0, o = 0; z < nz; ++z) {
        for (int i = 0; i < m->zones[z].n_walls; ++i, ++o) {
            const hyg_zone_wall_link* l = &m->zones[z].walls[i];
            const size_t idx = (size_t)l->wall * (size_t)m->n_nodes + (size_t)face_node(m, l->face);
            us[o] = s->uc[idx];
            vs[o] = s->vc[idx];
        }
    }
    double* qr = (double*)malloc(sizeof(double) * (size_t)(2 * m->n_walls + 1));
    radiation_fluxes(m, s->uc, qr);                 /* from layer n (building.cpp:158) */
    for (int w = 0; w < m->n_walls; ++w) {
        orc_face L, R;
        resolve_face(m, w, 0, zu0, zv0, t, qr[2 * w], &L);
        resolve_face(m, w, 1, zu0, zv0, t, qr[2 * w + 1], &R);
        orc_field f = bfield(m, s, w);
        orc_model wm;
        wall_model(m, w, &wm);
        if (wm.kind == ORC_COEFF_CONSTANT) {
            orc_df_step_coupled(&f, m->dx, &m->groups[w], &L, &R, dt);
        } else if (orc_df_step_nonlinear(&f, m->dx, &m->groups[w], &wm, &L, &R, dt)) {
            /* domain_error propagates out of step_explicit (building.cpp:175) */
            g_dom_wall = w;
            free(qr);
            free(us);
            free(zu0);
            return HYG_EDOMAIN;
        }
    }
    free(qr);
    const double u_out = orc_signal(&m->outdoor_u, t), v_out = orc_signal(&m->outdoor_v, t);
    for (int z = 0, o = 0; z < nz; ++z) {
        double du, dv;
        orc_zone_rhs(m, z, zu0[z], zv0[z], us + o, vs + o, zu0, zv0, u_out, v_out, t, &du, &dv);
        s->zu[z] = zu0[z] + dt * du;   /* zone_step_explicit zone.cpp:69-74 */
        s->zv[z] = zv0[z] + dt * dv;
        o += m->zones[z].n_walls;
    }
    s->t += dt;
    s->layer += 1;
    free(us);
    free(zu0);
    return 0;
}

/* zone_step_implicit zone.cpp:76-115 */
static void zone_step_implicit(const hyg_model_desc* m, int zi, double u_n, double v_n,
                               const double* u_s, const double* v_s, const double* zu,
                               const double* zv, double u_inf, double v_inf, double t_next,
                               double dt, double* u1, double* v1_out) {
    const hyg_zone_desc* z = &m->zones[zi];
    const hyg_zone_sources* src = &m->zone_sources[z->sources];
    const double sign = z->moisture_sign == HYG_MOISTURE_AS_PRINTED ? 1.0 : -1.0;
    double sum_gz = 0.0, sum_gz_v = 0.0;
    for (int i = 0; i < z->n_interzone; ++i) {
        sum_gz += z->interzone[i].g_inz;
        sum_gz_v += z->interzone[i].g_inz * zv[z->interzone[i].peer];
    }
    double S_M = 0.0, W_M = 0.0;
    for (int i = 0; i < z->n_walls; ++i) {
        S_M += z->walls[i].Bi_M * z->walls[i].theta_M;
        W_M += z->walls[i].Bi_M * z->walls[i].theta_M * v_s[i];
    }
    const double v_den = 1.0 + dt * (z->g_v + sum_gz - sign * S_M);
    const double v_num = v_n + dt * (orc_signal(&src->g_o, t_next) + z->g_v * v_inf + sum_gz_v - sign * W_M);
    const double v1 = v_num / v_den;
    double u_coef = (1.0 + z->kappa_a_tt1) + dt * (z->q_v1 * v1 + z->q_v2);
    double u_rhs = (1.0 + z->kappa_a_tt1) * u_n +
                   dt * (orc_signal(&src->q_o, t_next) + orc_signal(&src->q_h, t_next) +
                         z->q_v1 * u_inf * v_inf + z->q_v2 * u_inf);
    for (int i = 0; i < z->n_interzone; ++i) {
        const hyg_interzone_link* l = &z->interzone[i];
        const double pu = zu[l->peer], pv = zv[l->peer];
        u_coef += dt * (l->q_inz1 * v1 + l->q_inz2);
        u_rhs += dt * (l->q_inz1 * pu * pv + l->q_inz2 * pu);
    }
    for (int i = 0; i < z->n_walls; ++i) {
        const hyg_zone_wall_link* w = &z->walls[i];
        u_coef += dt * w->Bi_TT * w->theta_T;
        u_rhs += dt * (w->Bi_TT * w->theta_T * u_s[i] + w->Bi_TM * w->theta_T * (v_s[i] - v1));
    }
    *u1 = u_rhs / u_coef;
    *v1_out = v1;
}

static orc_reduce_fn g_reduce = NULL;   /* shard support: see orc_set_owned */
static void* g_reduce_user = NULL;
static int g_own_w0 = 0, g_own_w1 = 0x7fffffff, g_own_z0 = 0, g_own_z1 = 0x7fffffff;

void orc_set_owned(int wall0, int wall1, int zone0, int zone1, orc_reduce_fn reduce, void* user) {
    g_own_w0 = wall0;
    g_own_w1 = wall1;
    g_own_z0 = zone0;
    g_own_z1 = zone1;
    g_reduce = reduce;
    g_reduce_user = user;
}

int orc_step_implicit(const hyg_model_desc* m, orc_building_state* s, double eta, int max_subiters,
                      int* passes, double* residual) { /* building.cpp:189-268 */
    if (!(eta > 0.0)) return HYG_EINVAL;
    const int n = m->n_nodes, nw = m->n_walls, nz = m->n_zones;
    const double t1 = s->t + m->dt;
    const double dt = m->dt;
    const size_t tot = (size_t)nw * (size_t)n;
    double* iu = (double*)malloc(sizeof(double) * (tot * 4 + 1));
    double *iv = iu + tot, *uN = iv + tot, *vN = uN + tot;
    memcpy(iu, s->uc, sizeof(double) * tot);
    memcpy(iv, s->vc, sizeof(double) * tot);
    double* izu = (double*)malloc(sizeof(double) * (size_t)(4 * nz + 1));
    double *izv = izu + nz, *snu = izv + nz, *snv = snu + nz;
    memcpy(izu, s->zu, sizeof(double) * (size_t)nz);
    memcpy(izv, s->zv, sizeof(double) * (size_t)nz);
    const double u_out = orc_signal(&m->outdoor_u, t1), v_out = orc_signal(&m->outdoor_v, t1);
    double* qr = (double*)malloc(sizeof(double) * (size_t)(2 * nw + 1));
    int pass = 0;
    double diff = 0.0;
    int rc = 0;
    for (;;) {
        ++pass;
        diff = 0.0;
        memcpy(snu, izu, sizeof(double) * (size_t)nz);
        memcpy(snv, izv, sizeof(double) * (size_t)nz);
        radiation_fluxes(m, iu, qr);          /* refreshed from the iterate (building.cpp:212) */
        for (int w = 0; w < nw; ++w) {
            orc_face L, R;
            resolve_face(m, w, 0, snu, snv, t1, qr[2 * w], &L);
            resolve_face(m, w, 1, snu, snv, t1, qr[2 * w + 1], &R);
            orc_field base = bfield(m, s, w);
            const size_t o = (size_t)w * (size_t)n;
            orc_model wm;
            wall_model(m, w, &wm);
            orc_implicit_wall_pass(&base, m->dx, &m->groups[w], &wm, &L, &R, dt, iu + o, iv + o,
                                   uN + o, vN + o);
            for (int j = 0; j < n && w >= g_own_w0 && w < g_own_w1; ++j) {
                diff = fmax(diff, fabs(uN[o + j] - iu[o + j]));
                diff = fmax(diff, fabs(vN[o + j] - iv[o + j]));
            }
            memcpy(iu + o, uN + o, sizeof(double) * (size_t)n);
            memcpy(iv + o, vN + o, sizeof(double) * (size_t)n);
        }
        for (int z = 0; z < nz; ++z) {
            const hyg_zone_desc* zd = &m->zones[z];
            double us[64], vs[64];
            for (int i = 0; i < zd->n_walls && i < 64; ++i) {
                const size_t idx = (size_t)zd->walls[i].wall * (size_t)n + (size_t)face_node(m, zd->walls[i].face);
                us[i] = iu[idx];
                vs[i] = iv[idx];
            }
            double nu, nv;
            zone_step_implicit(m, z, s->zu[z], s->zv[z], us, vs, snu, snv, u_out, v_out, t1, dt, &nu, &nv);
            if (z >= g_own_z0 && z < g_own_z1) {
                diff = fmax(diff, fabs(nu - izu[z]));
                diff = fmax(diff, fabs(nv - izv[z]));
            }
            izu[z] = nu;
            izv[z] = nv;
        }
        if (g_reduce) diff = g_reduce(g_reduce_user, diff);
        if (diff < eta) break;
        if (pass >= max_subiters) { rc = HYG_ECONVERGE; break; }
    }
    if (!rc) {
        memcpy(s->up, s->uc, sizeof(double) * tot);
        memcpy(s->uc, iu, sizeof(double) * tot);
        memcpy(s->vp, s->vc, sizeof(double) * tot);
        memcpy(s->vc, iv, sizeof(double) * tot);
        memcpy(s->zu, izu, sizeof(double) * (size_t)nz);
        memcpy(s->zv, izv, sizeof(double) * (size_t)nz);
        s->t = t1;
        s->layer += 1;
    }
    if (passes) *passes = pass;
    if (residual) *residual = diff;
    free(qr);
    free(iu);
    free(izu);
    return rc;
}

int orc_check_bounded(const hyg_model_desc* m, const orc_building_state* s, int* wall) {
    /* building.cpp:282-300 */
    for (int w = 0; w < m->n_walls; ++w) {
        const size_t o = (size_t)w * (size_t)m->n_nodes;
        orc_field f = {m->n_nodes, s->up + o, s->uc + o, s->vp + o, s->vc + o, 0.0};
        const double mx = orc_max_abs_field(&f);
        if (!(mx <= m->divergence_norm)) {
            if (wall) *wall = w;
            return HYG_EDIVERGED;
        }
    }
    for (int z = 0; z < m->n_zones; ++z) {
        if (!isfinite(s->zu[z]) || !isfinite(s->zv[z]) || fabs(s->zu[z]) > m->divergence_norm ||
            fabs(s->zv[z]) > m->divergence_norm) {
            if (wall) *wall = -1;
            return HYG_EDIVERGED;
        }
    }
    return 0;
}

int orc_run(const hyg_model_desc* m, orc_building_state* s, int64_t nsteps, int64_t* fail_layer,
            int* fail_wall, int* boot_passes) { /* building.cpp:303-356 (DF scheme) */
    int64_t done = 0;
    if (nsteps > 0) {
        int passes = 0;
        double res = 0.0;
        const int rc = orc_step_implicit(m, s, m->eta_factor * m->dt, m->max_subiters, &passes, &res);
        if (boot_passes) *boot_passes = passes;
        if (rc) return rc;
        int w;
        if (orc_check_bounded(m, s, &w)) {
            if (fail_layer) *fail_layer = s->layer;
            if (fail_wall) *fail_wall = w;
            return HYG_EDIVERGED;
        }
        ++done;
    }
    while (done < nsteps) {
        if (orc_step_explicit(m, s) == HYG_EDOMAIN) {
            if (fail_layer) *fail_layer = s->layer + 1;
            if (fail_wall) *fail_wall = g_dom_wall;
            return HYG_EDOMAIN;
        }
        int w;
        if (orc_check_bounded(m, s, &w)) {
            if (fail_layer) *fail_layer = s->layer;
            if (fail_wall) *fail_wall = w;
            return HYG_EDIVERGED;
        }
        ++done;
    }
    return 0;
}

/* ---- orc_run_mt: orc_run with the explicit steps split over threads ------
 * The same run() march (building.cpp:303-356): the implicit start serially,
 * then every step_explicit (building.cpp:152-187) with the walls and zones
 * split into contiguous ranges per thread.  Within a step every wall reads
 * only layer n of its own nodes and the layer-n zone snapshot, every zone
 * only layer-n samples and peers, so each value is computed by the same
 * statements as orc_step_explicit and the result is bitwise the serial one.
 * Three barriers per step: samples/snapshot gathered; walls and zones
 * stepped; the guard verdict (lowest failing wall, as check_bounded walks
 * walls in order, then zones).  Constant-coefficient walls without radiation
 * only (the zone-ring workloads); anything else runs orc_run. */
typedef struct {
    const hyg_model_desc* m;
    orc_building_state* s;
    int nthr, id;
    int64_t nsteps;
    double *zu0, *zv0, *us, *vs;
    const int* link0;
    pthread_barrier_t* bar;
    int* fail_wall;       /* [nthr] lowest failing wall this step (INT_MAX: none) */
    int* fail_zone;       /* [nthr] any failing zone this step */
    volatile int* stop;
    int64_t* done;
} mt_job;

static void* mt_run(void* arg) {
    mt_job* J = (mt_job*)arg;
    const hyg_model_desc* m = J->m;
    orc_building_state* s = J->s;
    const int nw = m->n_walls, nz = m->n_zones, n = m->n_nodes;
    const int w0 = (int)((int64_t)nw * J->id / J->nthr), w1 = (int)((int64_t)nw * (J->id + 1) / J->nthr);
    const int z0 = (int)((int64_t)nz * J->id / J->nthr), z1 = (int)((int64_t)nz * (J->id + 1) / J->nthr);
    for (int64_t k = 0; k < J->nsteps; ++k) {
        const double t = s->t, dt = m->dt;
        for (int z = z0; z < z1; ++z) {           /* snapshot + samples of layer n (building.cpp:157-164) */
            J->zu0[z] = s->zu[z];
            J->zv0[z] = s->zv[z];
            for (int i = 0; i < m->zones[z].n_walls; ++i) {
                const hyg_zone_wall_link* l = &m->zones[z].walls[i];
                const size_t idx = (size_t)l->wall * (size_t)n + (size_t)face_node(m, l->face);
                J->us[J->link0[z] + i] = s->uc[idx];
                J->vs[J->link0[z] + i] = s->vc[idx];
            }
        }
        pthread_barrier_wait(J->bar);
        int fw = 0x7fffffff, fz = 0;
        for (int w = w0; w < w1; ++w) {
            orc_face L, R;
            resolve_face(m, w, 0, J->zu0, J->zv0, t, 0.0, &L);
            resolve_face(m, w, 1, J->zu0, J->zv0, t, 0.0, &R);
            orc_field f = bfield(m, s, w);
            orc_df_step_coupled(&f, m->dx, &m->groups[w], &L, &R, dt);
            if (fw == 0x7fffffff && !(orc_max_abs_field(&f) <= m->divergence_norm)) fw = w;
        }
        const double u_out = orc_signal(&m->outdoor_u, t), v_out = orc_signal(&m->outdoor_v, t);
        for (int z = z0; z < z1; ++z) {
            double du, dv;
            orc_zone_rhs(m, z, J->zu0[z], J->zv0[z], J->us + J->link0[z], J->vs + J->link0[z], J->zu0, J->zv0,
                         u_out, v_out, t, &du, &dv);
            s->zu[z] = J->zu0[z] + dt * du;
            s->zv[z] = J->zv0[z] + dt * dv;
            if (!isfinite(s->zu[z]) || !isfinite(s->zv[z]) || fabs(s->zu[z]) > m->divergence_norm ||
                fabs(s->zv[z]) > m->divergence_norm)
                fz = 1;
        }
        J->fail_wall[J->id] = fw;
        J->fail_zone[J->id] = fz;
        pthread_barrier_wait(J->bar);
        if (J->id == 0) {
            s->t += dt;
            s->layer += 1;
            int any = 0;
            for (int i = 0; i < J->nthr; ++i) any |= J->fail_wall[i] != 0x7fffffff || J->fail_zone[i];
            *J->stop = any;
            *J->done = k + 1;
        }
        pthread_barrier_wait(J->bar);
        if (*J->stop) break;
    }
    return NULL;
}

int orc_run_mt(const hyg_model_desc* m, orc_building_state* s, int64_t nsteps, int nthreads,
               int64_t* fail_layer, int* fail_wall, int* boot_passes) {
    int simple = m->coeff_kind == HYG_COEFF_CONSTANT || m->coeff_kind == HYG_COEFF_MATERIAL;
    for (int w = 0; simple && w < m->n_walls; ++w) {
        orc_model wm;
        wall_model(m, w, &wm);
        simple = wm.kind == ORC_COEFF_CONSTANT;
    }
    for (int z = 0; simple && z < m->n_zones; ++z) simple = m->zones[z].n_radiation == 0;
    if (nthreads <= 1 || !simple || nsteps < 2) return orc_run(m, s, nsteps, fail_layer, fail_wall, boot_passes);
    int rc = orc_run(m, s, 1, fail_layer, fail_wall, boot_passes);   /* the implicit start (step 1) */
    if (rc) return rc;
    const int nz = m->n_zones;
    int* link0 = (int*)malloc(sizeof(int) * (size_t)(nz + 1));
    int tot = 0;
    for (int z = 0; z < nz; ++z) {
        link0[z] = tot;
        tot += m->zones[z].n_walls;
    }
    double* buf = (double*)malloc(sizeof(double) * (size_t)(2 * nz + 2 * tot + 2));
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)nthreads);
    int* fw = (int*)malloc(sizeof(int) * (size_t)nthreads * 2);
    volatile int stop = 0;
    int64_t done = 0;
    mt_job* jobs = (mt_job*)calloc((size_t)nthreads, sizeof(mt_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int i = 0; i < nthreads; ++i) {
        mt_job J = {m, s, nthreads, i, nsteps - 1, buf, buf + nz, buf + 2 * nz, buf + 2 * nz + tot, link0, &bar,
                    fw, fw + nthreads, &stop, &done};
        jobs[i] = J;
        if (i) pthread_create(&th[i], NULL, mt_run, &jobs[i]);
    }
    mt_run(&jobs[0]);
    for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
    if (stop) {
        int w = 0x7fffffff;
        for (int i = 0; i < nthreads; ++i) w = fw[i] < w ? fw[i] : w;
        if (fail_layer) *fail_layer = s->layer;
        if (fail_wall) *fail_wall = w == 0x7fffffff ? -1 : w;
        rc = HYG_EDIVERGED;
    }
    pthread_barrier_destroy(&bar);
    free(jobs);
    free(th);
    free(fw);
    free(buf);
    free(link0);
    return rc;
}

/* ---- orc_march_long_mt: one long wall, its nodes split over threads ------
 * nsteps of df_step_nonlinear (wall.cpp:196-264) on wall 0 of the batch with
 * the guard of run(), each thread owning a contiguous node range: the
 * StarTables of its nodes and half nodes, then its v rows (+ a face row),
 * then its u rows (+ the face row), then the layer rotation of its range —
 * barriers between the phases.  A node's new values are a pure function of
 * layers n and n-1 computed by the same statements as the serial step (the
 * nl_* pieces above), so the march is bitwise the serial one.  Strict
 * coefficient failures abort the march with HYG_EDOMAIN (no location). */
typedef struct {
    const orc_batch* b;
    const orc_model* m;
    int nsteps, nthr, id;
    double dt;
    star_tables* s;
    double *vn, *un;
    pthread_barrier_t* bar;
    double* mx;          /* [nthr] max |x| of the new layers */
    int* dom;            /* [nthr] strict failure */
    volatile int* stop;
    int64_t* fail_layer;
} long_job;

static void* long_run(void* arg) {
    long_job* J = (long_job*)arg;
    const orc_batch* b = J->b;
    const int n = b->n;
    const int j0 = (int)((int64_t)n * J->id / J->nthr), j1 = (int)((int64_t)n * (J->id + 1) / J->nthr);
    orc_field f = field_of(b, 0);
    const nl_consts c = nl_setup(n, b->dx, &b->groups[0], J->dt);
    star_tables* s = J->s;
    for (int k = 0; k < J->nsteps; ++k) {
        const int64_t lay = b->layer0 + k;
        int bad = 0;
        if (!s->unit) {                           /* StarTables of layer n (wall.cpp:89-138) */
            for (int j = j0; j < j1 && !bad; ++j) bad = orc_star(J->m, f.uc[j], f.vc[j], 1, &s->node[j]);
            for (int j = j0; j < j1 && j + 1 < n && !bad; ++j)
                bad = orc_star(J->m, 0.5 * (f.uc[j] + f.uc[j + 1]), 0.5 * (f.vc[j] + f.vc[j + 1]), 1, &s->half[j]);
        }
        J->dom[J->id] = bad;
        pthread_barrier_wait(J->bar);
        int any = 0;
        for (int i = 0; i < J->nthr; ++i) any |= J->dom[i];
        if (any) {
            if (J->id == 0) *J->stop = HYG_EDOMAIN;
            break;
        }
        orc_face L, R;
        face_of(b, 0, 0, lay, &L);
        face_of(b, 0, 1, lay, &R);
        nl_v_rows(&c, s, &f, J->vn, j0, j1);
        if (j0 == 0) nl_v_face(&c, s, &f, J->vn, 0, &L);
        if (j1 == n) nl_v_face(&c, s, &f, J->vn, 1, &R);
        nl_u_rows(&c, s, &f, J->vn, J->un, j0, j1);
        if (j0 == 0) nl_u_face(&c, s, &f, J->vn, J->un, 0, &L);
        if (j1 == n) nl_u_face(&c, s, &f, J->vn, J->un, 1, &R);
        pthread_barrier_wait(J->bar);             /* every row read layers n, n-1 */
        double mx = 0.0;
        int inf = 0;
        for (int j = j0; j < j1; ++j) {           /* rotate (wall.cpp:261-263), max_abs_field (:579-587) */
            f.vp[j] = f.vc[j];
            f.vc[j] = J->vn[j];
            f.up[j] = f.uc[j];
            f.uc[j] = J->un[j];
            mx = fmax(mx, fmax(fabs(f.uc[j]), fabs(f.vc[j])));
            if (!isfinite(f.uc[j]) || !isfinite(f.vc[j])) inf = 1;
        }
        J->mx[J->id] = inf ? INFINITY : mx;
        pthread_barrier_wait(J->bar);
        if (J->id == 0) {
            for (int i = 0; i < J->nthr; ++i)
                if (!(J->mx[i] <= b->divergence_norm)) *J->stop = HYG_EDIVERGED;
            if (*J->stop) *J->fail_layer = lay + 1;
        }
        pthread_barrier_wait(J->bar);
        if (*J->stop) break;
    }
    return NULL;
}

int orc_march_long_mt(const orc_batch* b, const orc_model* m, int nsteps, double dt, int nthreads,
                      int64_t* fail_layer) {
    const int n = b->n;
    if (b->n_walls != 1 || n < 3) return HYG_EINVAL;
    if (nthreads > n / 64) nthreads = n / 64 > 0 ? n / 64 : 1;
    if (nthreads < 1) nthreads = 1;
    star_tables s;
    s.unit = (m == NULL || m->kind == ORC_COEFF_CONSTANT);
    s.node = s.unit ? NULL : (orc_coeffs*)malloc(sizeof(orc_coeffs) * (size_t)(2 * n - 1));
    s.half = s.unit ? NULL : s.node + n;
    double* buf = (double*)malloc(sizeof(double) * (size_t)(2 * n + 2 * nthreads));
    int* dom = (int*)calloc((size_t)nthreads, sizeof(int));
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)nthreads);
    volatile int stop = 0;
    int64_t fl = -1;
    long_job* jobs = (long_job*)calloc((size_t)nthreads, sizeof(long_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int i = 0; i < nthreads; ++i) {
        long_job J = {b, m, nsteps, nthreads, i, dt, &s, buf, buf + n, &bar, buf + 2 * n, dom, &stop, &fl};
        jobs[i] = J;
        if (i) pthread_create(&th[i], NULL, long_run, &jobs[i]);
    }
    long_run(&jobs[0]);
    for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
    pthread_barrier_destroy(&bar);
    if (fail_layer) *fail_layer = fl;
    const int rc = stop;
    free(jobs);
    free(th);
    free(dom);
    free(buf);
    free(s.node);
    return rc;
}
