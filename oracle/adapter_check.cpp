// adapter_check.cpp — TEST INFRASTRUCTURE: the reference's own run()
// (building.cpp:303-356) against the drop-in hygro::gpu::run of
// include/hygro_b200.hpp on the same hygro::BuildingModel: the one-zone
// linear building of test_building.cpp:17-78 (4 walls, frozen sets,
// schedules, sin^2 outdoor temperature), and a 3-zone ring variant.
// Built by oracle/Makefile (needs /root/reference); run on a GPU by
// tests/test_gpu_adapter.py.  Prints the relative L-inf per case; exit 0 iff
// every case is <= 1e-10 and the frame counts agree.
#define HYGRO_B200_WITH_REFERENCE
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "hygro/building.hpp"
#include "hygro/scaling.hpp"
#include "hygro_b200.hpp"

using namespace hygro;

static BuildingModel ring_model(int n_zones, double horizon) {
    const CoefficientSet sets[3] = {{1.82e-2, 5.89e-9, 7.7e5, 2.94e-1, 1.52e3, 1.59e-2},
                                    {1.18e-1, 2.92e-8, 1.28e6, 8.41e-1, 9.88e3, 2.96e-3},
                                    {6.09e-2, 5.47e-9, 8.61e5, 3.87e-1, 5.09e3, 1.53e-2}};
    struct Spec { int set; double A, hT, hM; };
    const Spec walls[4] = {{0, 18, 5, 2e-7}, {1, 18, 25, 8e-7}, {2, 9, 12, 4e-7}, {2, 9, 12, 4e-7}};
    BuildingModel m;
    m.ctx = ScalingContext::from_state(293.15, 0.5, 3600.0);
    m.outdoor_u = Signal::sin_squared(1.0, -0.02, 24.0);
    m.outdoor_v = Signal::sinusoid(1.0, 0.06, 24.0);
    ZoneAirConfig air;
    air.volume = 54.0;
    air.ventilation_ach = 0.5;
    air.moisture_source = Signal::schedule(25e-3 / 3600.0, {{6, 9, 400e-3 / 3600.0}, {30, 33, 400e-3 / 3600.0}});
    air.heat_source = Signal::sinusoid(0.0, 50.0, 24.0);
    for (int z = 0; z < n_zones; ++z) {
        ZoneConfig zc;
        zc.name = "z" + std::to_string(z);
        zc.params = scale_zone(air, m.ctx);
        for (int i = 0; i < 4; ++i) {
            BuildingWall w;
            w.name = "w";
            w.thickness = 0.1;
            w.grid = Grid1D::with_spacing(1e-2);
            WallDimensionless wd = scale_wall(sets[walls[i].set], 0.1, walls[i].hT, walls[i].hM, 8.0, 3e-8, m.ctx);
            w.groups = wd.groups;
            w.biot[0] = wd.face[0];
            w.biot[1] = wd.face[1];
            w.k_TT0 = sets[walls[i].set].k_TT;
            w.attach[0].kind = FaceAttachment::Kind::Exterior;
            w.attach[0].u_inf = m.outdoor_u;
            w.attach[0].v_inf = m.outdoor_v;
            w.attach[1].kind = FaceAttachment::Kind::Zone;
            w.attach[1].zone = z;
            w.init_profile_v = [](double x) { return 1.0 + 0.01 * std::cos(3.14159 * x); };
            attach_wall_to_zone(wd, walls[i].A, 0.1, zc.params, m.ctx);
            ZoneWallLink link;
            link.wall = static_cast<int>(m.walls.size());
            link.face = 1;
            link.Bi_M = wd.face[1].Bi_M;
            link.Bi_TT = wd.face[1].Bi_TT;
            link.Bi_TM = wd.face[1].Bi_TM;
            link.theta_T = wd.theta_T;
            link.theta_M = wd.theta_M;
            zc.walls.push_back(link);
            m.walls.push_back(std::move(w));
        }
        if (n_zones > 1) {
            const InterzoneScalars s = scale_interzone(0.5, air, zc.params, m.ctx);
            for (int d : {-1, 1}) {
                ZoneInterzoneLink l;
                l.peer = (z + d + n_zones) % n_zones;
                l.g_inz = s.g_inz;
                l.q_inz1 = s.q_inz1;
                l.q_inz2 = s.q_inz2;
                zc.interzone.push_back(l);
            }
        }
        m.zones.push_back(zc);
    }
    m.dt = 1e-3;
    m.horizon = horizon;
    m.eta_factor = 1e-6;
    return m;
}

static double compare(const SimulationResult& a, const SimulationResult& b) {
    if (a.frames.size() != b.frames.size()) return 1e30;
    double num = 0, den = 0;
    for (size_t f = 0; f < a.frames.size(); ++f) {
        if (a.frames[f].t != b.frames[f].t) return 1e30;
        for (size_t w = 0; w < a.frames[f].wall_u.size(); ++w)
            for (size_t j = 0; j < a.frames[f].wall_u[w].size(); ++j) {
                num = std::max(num, std::fabs(a.frames[f].wall_u[w][j] - b.frames[f].wall_u[w][j]));
                num = std::max(num, std::fabs(a.frames[f].wall_v[w][j] - b.frames[f].wall_v[w][j]));
                den = std::max(den, std::fabs(b.frames[f].wall_u[w][j]));
                den = std::max(den, std::fabs(b.frames[f].wall_v[w][j]));
            }
        for (size_t z = 0; z < a.frames[f].zones.size(); ++z) {
            num = std::max(num, std::fabs(a.frames[f].zones[z].u_a - b.frames[f].zones[z].u_a));
            num = std::max(num, std::fabs(a.frames[f].zones[z].v_a - b.frames[f].zones[z].v_a));
        }
    }
    return num / den;
}

int main() {
    int bad = 0;
    for (int nz : {1, 3}) {
        const BuildingModel m = ring_model(nz, 2.0);
        const SimulationResult ref = hygro::run(m, 0.25);
        const SimulationResult gpu = hygro::gpu::run(m, 0.25);
        const double e = compare(gpu, ref);
        std::printf("zones=%d frames ref=%zu gpu=%zu boot passes ref=%d gpu=%d rel_linf=%.3e\n", nz,
                    ref.frames.size(), gpu.frames.size(), ref.bootstrap_subiters, gpu.bootstrap_subiters, e);
        if (!(e <= 1e-10) || ref.bootstrap_subiters != gpu.bootstrap_subiters) ++bad;
    }
    // divergence: same exception type and t_star as the reference
    BuildingModel m = ring_model(1, 0.5);
    m.divergence_norm = 1.0005;
    double t_ref = -1, t_gpu = -2;
    SimulationResult pr, pg;
    try { hygro::run(m, 0.1, &pr); } catch (const numerical_error& e) { t_ref = e.t_star; }
    try { hygro::gpu::run(m, 0.1, &pg); } catch (const numerical_error& e) { t_gpu = e.t_star; }
    std::printf("divergence t_star ref=%.17g gpu=%.17g partial frames ref=%zu gpu=%zu\n", t_ref, t_gpu,
                pr.frames.size(), pg.frames.size());
    if (t_ref != t_gpu || t_ref < 0 || pr.frames.size() != pg.frames.size()) ++bad;
    return bad ? 1 : 0;
}
