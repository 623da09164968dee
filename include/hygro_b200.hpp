// hygro_b200.hpp — C++ host layer over the C ABI (include/hygro_b200.h).
//
// 1. hygro_b200::Context: RAII owner of a hyg_ctx, errors rethrown as
//    exceptions with the reference's taxonomy (errors.hpp:8-45).
// 2. With HYGRO_B200_WITH_REFERENCE defined and the reference headers on the
//    include path: hygro::gpu::run(const hygro::BuildingModel&, double
//    cadence, hygro::SimulationResult* partial) — a drop-in for hygro::run
//    (building.hpp:101-102, building.cpp:303-356) on the DF scheme, taking the
//    reference's own model type.  Signals are opaque in the reference
//    (signal.hpp exposes only operator()(t)), so the adapter evaluates every
//    face, zone-source and outdoor Signal at the run's layer times (the
//    reference's accumulated t) and uploads them as per-layer tables.
//    Device coverage: walls on one grid with constant coefficients or the
//    load-bearing material (CoefficientModel::material with the model's
//    ScalingContext), zones, interzone links and radiation links.  Anything
//    else (another scheme, mixed grids, a material model whose starred sets
//    the device cannot reproduce bit for bit on the host) throws
//    std::invalid_argument before touching the device.
#pragma once

#include <chrono>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "hygro_b200.h"

namespace hygro_b200 {

struct error : std::runtime_error {
    int code;
    hyg_status status;
    error(int c, const hyg_status& s, const std::string& what)
        : std::runtime_error(what), code(c), status(s) {}
};

class Context {
public:
    explicit Context(const hyg_model_desc& d) {
        hyg_status st{};
        check(hyg_create(&d, &h_, &st), st, "hyg_create");
    }
    ~Context() { hyg_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    hyg_ctx* get() const { return h_; }

    // throws the mapped exception (overridable by the reference adapter)
    static void check(int rc, const hyg_status& st, const char* what) {
        if (rc == HYG_OK) return;
        throw error(rc, st, std::string(what) + ": " + (st.message[0] ? st.message : hyg_strerror(rc)));
    }

private:
    hyg_ctx* h_ = nullptr;
};

}  // namespace hygro_b200

#ifdef HYGRO_B200_WITH_REFERENCE
#include "hygro/building.hpp"
#include "hygro/errors.hpp"
#include "hygro/materials.hpp"

namespace hygro::gpu {

namespace detail {
inline hyg_signal constant(double v) {
    hyg_signal s{};
    s.form = HYG_SIG_CONSTANT;
    s.base = v;
    s.period = 1.0;
    return s;
}

// hyg status -> the reference's exception types (errors.hpp:8-45)
[[noreturn]] inline void rethrow(int rc, const hyg_status& st, double t_fail) {
    const std::string msg = st.message[0] ? st.message : hyg_strerror(rc);
    switch (rc) {
        case HYG_EDIVERGED: throw numerical_error(msg, t_fail);
        case HYG_ECONVERGE: throw convergence_error(msg, st.residual);
        case HYG_EDOMAIN: throw domain_error(msg);
        case HYG_ESCHEMA: throw schema_error(msg);
        case HYG_ESCALING: throw scaling_error(msg);
        case HYG_EINVAL: throw std::invalid_argument(msg);
        default: throw std::runtime_error(msg);
    }
}

// The reference set of a material wall.  CoefficientModel keeps it private;
// star(u, v) = evaluate(u T_i, v P_vi) / reference (wall.cpp:50-53), so at
// (1, 1) reference = evaluate(T_i, P_vi) / star(1, 1), then checked (and
// nudged by an ulp where the division rounded) against star() at sample
// states, so the device divides by exactly the reference's numbers.
inline hyg_coeff_set material_reference(const CoefficientModel& cm, const ScalingContext& ctx) {
    const MaterialModel mm;
    const CoefficientSet e = mm.evaluate(ctx.T_i, ctx.P_vi), s = cm.star(1.0, 1.0);
    double r[6] = {e.c_M / s.c_M, e.k_M / s.k_M, e.c_TT / s.c_TT, e.k_TT / s.k_TT, e.c_TM / s.c_TM, e.k_TM / s.k_TM};
    const double probes[4][2] = {{1.0, 1.0}, {1.01, 0.9}, {0.98, 1.2}, {1.03, 0.7}};
    for (int f = 0; f < 6; ++f) {
        auto field = [f](const CoefficientSet& c) {
            const double v[6] = {c.c_M, c.k_M, c.c_TT, c.k_TT, c.c_TM, c.k_TM};
            return v[f];
        };
        auto matches = [&](double ref) {
            for (const auto& p : probes) {
                CoefficientSet a, b;
                try {                     // probes outside the material box are skipped
                    a = mm.evaluate(p[0] * ctx.T_i, p[1] * ctx.P_vi);
                    b = cm.star(p[0], p[1]);
                } catch (const domain_error&) {
                    continue;
                }
                if (field(a) / ref != field(b)) return false;
            }
            return true;
        };
        const double lo1 = std::nextafter(r[f], 0.0), hi1 = std::nextafter(r[f], 1e300);
        const double cands[5] = {r[f], lo1, hi1, std::nextafter(lo1, 0.0), std::nextafter(hi1, 1e300)};
        bool ok = false;
        for (double cand : cands) {
            if (matches(cand)) {
                r[f] = cand;
                ok = true;
                break;
            }
        }
        if (!ok)
            throw std::invalid_argument(
                "hygro::gpu::run: material wall whose starred sets the device cannot reproduce "
                "(a scaling context or physical constants other than the model's)");
    }
    return hyg_coeff_set{r[0], r[1], r[2], r[3], r[4], r[5]};
}

struct Frames {
    SimulationResult* result;
    int n_walls, n_nodes, n_zones;
};

inline void on_frame(void* user, int64_t, double t, hyg_ctx* ctx) {
    auto* f = static_cast<Frames*>(user);
    std::vector<double> uc(static_cast<size_t>(f->n_walls) * f->n_nodes), vc(uc.size());
    std::vector<double> zu(f->n_zones), zv(f->n_zones);
    double tt = 0.0;
    int64_t layer = 0;
    hyg_get_state(ctx, nullptr, uc.data(), nullptr, vc.data(), f->n_zones ? zu.data() : nullptr,
                  f->n_zones ? zv.data() : nullptr, &tt, &layer);
    Frame fr;                                   // make_frame (building.cpp:271-280)
    fr.t = t;
    for (int w = 0; w < f->n_walls; ++w) {
        fr.wall_u.emplace_back(uc.begin() + static_cast<size_t>(w) * f->n_nodes,
                               uc.begin() + static_cast<size_t>(w + 1) * f->n_nodes);
        fr.wall_v.emplace_back(vc.begin() + static_cast<size_t>(w) * f->n_nodes,
                               vc.begin() + static_cast<size_t>(w + 1) * f->n_nodes);
    }
    for (int z = 0; z < f->n_zones; ++z) fr.zones.push_back(ZoneState{zu[z], zv[z]});
    f->result->frames.push_back(std::move(fr));
}
}  // namespace detail

// Drop-in for hygro::run (building.cpp:303-356) on the device, all three schemes.
inline SimulationResult run(const BuildingModel& m, double cadence, SimulationResult* partial = nullptr,
                            int device = 0) {
    m.validate();
    const auto t_start = std::chrono::steady_clock::now();
    if (m.walls.empty()) throw std::invalid_argument("hygro::gpu::run: no walls");
    const int nw = static_cast<int>(m.walls.size());
    const int nz = static_cast<int>(m.zones.size());
    const int n = m.walls[0].grid.n;
    std::vector<int32_t> wall_coeff(nw, HYG_COEFF_CONSTANT);
    std::vector<hyg_coeff_set> wall_ref(nw, hyg_coeff_set{1, 1, 1, 1, 1, 1});
    std::vector<double> thickness(nw), k_TT0(nw);
    bool any_material = false;
    for (int w = 0; w < nw; ++w) {
        const BuildingWall& bw = m.walls[w];
        if (bw.grid.n != n || bw.grid.dx != m.walls[0].grid.dx)
            throw std::invalid_argument("hygro::gpu::run: walls must share one grid");
        if (!bw.coeffs.is_constant()) {
            wall_coeff[w] = HYG_COEFF_MATERIAL;
            wall_ref[w] = detail::material_reference(bw.coeffs, m.ctx);
            any_material = true;
        }
        thickness[w] = bw.thickness;
        k_TT0[w] = bw.k_TT0;
    }

    const long nsteps = std::lround(m.horizon / m.dt);
    std::vector<double> times(static_cast<size_t>(nsteps) + 1);
    {
        double t = 0.0;   // BuildingState::t accumulation (building.cpp:185, 263)
        for (long k = 0; k <= nsteps; ++k) {
            times[k] = t;
            t += m.dt;
        }
    }
    std::vector<hyg_wall_groups> groups(nw);
    std::vector<hyg_face_biot> biot(2 * nw);
    std::vector<hyg_face_attach> attach(2 * nw);
    std::vector<std::pair<int, int>> ext;   // (wall, face) of each exterior channel
    for (int w = 0; w < nw; ++w) {
        const BuildingWall& bw = m.walls[w];
        groups[w] = hyg_wall_groups{bw.groups.Fo_M, bw.groups.Fo_TT, bw.groups.Fo_TM, bw.groups.gamma};
        for (int k = 0; k < 2; ++k) {
            biot[2 * w + k] = hyg_face_biot{bw.biot[k].Bi_M, bw.biot[k].Bi_TT, bw.biot[k].Bi_TM};
            if (bw.attach[k].kind == FaceAttachment::Kind::Exterior) {
                attach[2 * w + k] = hyg_face_attach{HYG_FACE_EXTERIOR, static_cast<int32_t>(ext.size())};
                ext.emplace_back(w, k);
            } else {
                attach[2 * w + k] = hyg_face_attach{HYG_FACE_ZONE, bw.attach[k].zone};
            }
        }
    }
    const hyg_signal c1 = detail::constant(1.0), c0 = detail::constant(0.0);
    std::vector<hyg_channel> channels(std::max<size_t>(1, ext.size()), hyg_channel{c1, c1, c0, c0});
    std::vector<std::vector<hyg_zone_wall_link>> zl(nz);
    std::vector<std::vector<hyg_interzone_link>> il(nz);
    std::vector<std::vector<hyg_radiation_link>> rl(nz);
    std::vector<hyg_zone_desc> zones(nz);
    std::vector<hyg_zone_sources> sources(std::max(1, nz), hyg_zone_sources{c0, c0, c0});
    for (int z = 0; z < nz; ++z) {
        const ZoneConfig& zc = m.zones[z];
        for (const auto& l : zc.walls)
            zl[z].push_back(hyg_zone_wall_link{l.wall, l.face, l.Bi_M, l.Bi_TT, l.Bi_TM, l.theta_T, l.theta_M});
        for (const auto& l : zc.interzone) il[z].push_back(hyg_interzone_link{l.peer, l.g_inz, l.q_inz1, l.q_inz2});
        for (const auto& r : zc.radiation)
            rl[z].push_back(hyg_radiation_link{r.emitter_wall, r.receiver_wall, r.view_factor, r.emissivity});
        zones[z] = hyg_zone_desc{zc.params.kappa_a_tt1, zc.params.g_v, zc.params.q_v1, zc.params.q_v2, z,
                                 zc.moisture_sign == MoistureWallSign::AsPrinted ? HYG_MOISTURE_AS_PRINTED
                                                                                  : HYG_MOISTURE_FLUX_CONSISTENT,
                                 static_cast<int32_t>(zl[z].size()), zl[z].data(),
                                 static_cast<int32_t>(il[z].size()), il[z].data(),
                                 static_cast<int32_t>(rl[z].size()), rl[z].data()};
    }
    hyg_model_desc d{};
    d.n_walls = nw;
    d.n_nodes = n;
    d.dx = m.walls[0].grid.dx;
    d.precision = HYG_F64;
    d.coeff_kind = any_material ? HYG_COEFF_MATERIAL : HYG_COEFF_CONSTANT;
    d.T_i = m.ctx.T_i;
    d.P_vi = m.ctx.P_vi;
    d.wall_coeff = wall_coeff.data();
    d.wall_reference = wall_ref.data();
    d.wall_thickness = thickness.data();
    d.wall_k_TT0 = k_TT0.data();
    d.groups = groups.data();
    d.biot = biot.data();
    d.attach = attach.data();
    d.n_channels = static_cast<int32_t>(channels.size());
    d.channels = channels.data();
    d.n_zones = nz;
    d.zones = zones.data();
    d.n_zone_sources = static_cast<int32_t>(sources.size());
    d.zone_sources = sources.data();
    d.outdoor_u = c1;
    d.outdoor_v = c1;
    d.dt = m.dt;
    d.divergence_norm = m.divergence_norm;
    d.eta_factor = m.eta_factor;
    d.max_subiters = m.max_subiters;
    d.device = device;

    hyg_status st{};
    hyg_ctx* ctx = nullptr;
    int rc = hyg_create(&d, &ctx, &st);
    if (rc) detail::rethrow(rc, st, 0.0);
    struct Guard { hyg_ctx* c; ~Guard() { hyg_destroy(c); } } guard{ctx};

    // forcing at the layer times, evaluated by the reference's Signal objects
    const size_t L = times.size();
    for (size_t c = 0; c < ext.size(); ++c) {
        const FaceAttachment& a = m.walls[ext[c].first].attach[ext[c].second];
        std::vector<hyg_ambient> tab(L);
        for (size_t k = 0; k < L; ++k) tab[k] = hyg_ambient{a.u_inf(times[k]), a.v_inf(times[k]),
                                                            a.g_inf(times[k]), a.q_inf(times[k])};
        hyg_set_channel_table(ctx, static_cast<int32_t>(c), 0, static_cast<int64_t>(L), tab.data());
    }
    for (int z = 0; z < nz; ++z) {
        const ZoneDimensionless& p = m.zones[z].params;
        std::vector<double> tab(3 * L);
        for (size_t k = 0; k < L; ++k) {
            tab[3 * k + 0] = p.g_o(times[k]);
            tab[3 * k + 1] = p.q_o(times[k]);
            tab[3 * k + 2] = p.q_h(times[k]);
        }
        hyg_set_source_table(ctx, z, 0, static_cast<int64_t>(L), tab.data());
    }
    {
        std::vector<double> tab(2 * L);
        for (size_t k = 0; k < L; ++k) {
            tab[2 * k + 0] = m.outdoor_u(times[k]);
            tab[2 * k + 1] = m.outdoor_v(times[k]);
        }
        hyg_set_outdoor_table(ctx, 0, static_cast<int64_t>(L), tab.data());
    }
    // initial_state (building.cpp:54-71): uniform values and study profiles
    const BuildingState s0 = initial_state(m);
    std::vector<double> up, uc, vp, vc, zu, zv;
    for (const auto& f : s0.walls) {
        up.insert(up.end(), f.u_prev.begin(), f.u_prev.end());
        uc.insert(uc.end(), f.u_curr.begin(), f.u_curr.end());
        vp.insert(vp.end(), f.v_prev.begin(), f.v_prev.end());
        vc.insert(vc.end(), f.v_curr.begin(), f.v_curr.end());
    }
    for (const auto& z : s0.zones) {
        zu.push_back(z.u_a);
        zv.push_back(z.v_a);
    }
    hyg_set_state(ctx, up.data(), uc.data(), vp.data(), vc.data(), nz ? zu.data() : nullptr,
                  nz ? zv.data() : nullptr, 0.0, 0);

    SimulationResult result;
    detail::Frames fr{&result, nw, n, nz};
    const int32_t scheme = m.scheme == Scheme::EulerImplicit   ? HYG_SCHEME_EULER_IMPLICIT
                           : m.scheme == Scheme::EulerExplicit ? HYG_SCHEME_EULER_EXPLICIT
                                                               : HYG_SCHEME_DF;
    hyg_run_report rep{};
    rc = hyg_run_scheme(ctx, scheme, m.horizon, cadence, &detail::on_frame, &fr, &rep, &st);
    result.wall_clock_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    if (rc) {
        result.steps = rep.steps;
        const double t_fail = st.layer >= 0 && st.layer < static_cast<int64_t>(L) ? times[st.layer] : st.t_star;
        if (partial) *partial = std::move(result);
        detail::rethrow(rc, st, t_fail);
    }
    result.steps = rep.steps;
    result.bootstrap_subiters = rep.bootstrap_subiters;
    result.max_subiters_seen = rep.max_subiters_seen;
    result.mean_subiters = rep.mean_subiters;
    return result;
}

}  // namespace hygro::gpu
#endif  // HYGRO_B200_WITH_REFERENCE
