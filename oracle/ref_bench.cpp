// ref_bench.cpp — TEST/MEASUREMENT INFRASTRUCTURE ONLY: the reference arm of
// bench.py (`--impl reference`) and the `cpu_baseline` of its GPU arm.
//
// A standalone program linked from the UNMODIFIED reference sources (see
// oracle/Makefile, target `refbench`; output only into oracle/_ref/).  It
// builds each BASELINE config's seeded synthetic workload through the
// reference's own public API — MaterialModel / saturation_pressure
// (materials.hpp), scale_wall / scale_zone / attach_wall_to_zone /
// scale_interzone (scaling.hpp), WallField, BuildingModel, Signal — and
// times the reference's own stepping functions on the host cores:
//   cfg1/cfg2  df_step_coupled (wall.cpp:144-194) + max_abs_field (the guard
//              run() applies every step, building.cpp:282-300), threads split
//              the independent walls; Euler-implicit: euler_implicit_step
//              (wall.cpp:515-550) likewise;
//   cfg3       run()'s DF loop body: step_explicit (building.cpp:152-187) —
//              serially through the public call, and with the walls and zones
//              of each step split over threads (the same reference calls,
//              df_step_coupled / zone_step_explicit, in step_explicit's
//              order; a step reads only layer n, so the split is exact);
//              Euler-implicit: step_implicit (building.cpp:189-268);
//   cfg0/cfg4  d(v) walls: the reference's CoefficientModel is a closed type
//              (wall.hpp:41-60) that cannot express d(v), so DF runs through
//              the reference's own transcription oracle with a StarFn
//              (tests/support/df_oracle.hpp:25-106) and the implicit path
//              through the C restatement of euler_implicit_step with the d(v)
//              functor (oracle/hygro_oracle.c, pinned bit-exact to the
//              reference on the coefficient models the reference has) —
//              reported as kind "port" for that figure;
//   cfg5       df_step_nonlinear with CoefficientModel::material
//              (wall.cpp:196-264), threads split walls; implicit:
//              euler_implicit_step with the same model.
// No file of the CUDA package is read, linked or loaded.  Inputs follow the
// distributions of paper_1703_10119_b200/workloads.py (same shapes, ranges and
// seeds' roles; this program's generator is std::mt19937_64, so the values
// differ while the workload is the same).  Prints one JSON object.
#include <algorithm>
#include <atomic>
#include <barrier>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "hygro/building.hpp"
#include "hygro/materials.hpp"
#include "hygro/scaling.hpp"
#include "hygro/wall.hpp"
#include "hygro/zone.hpp"
#include "support/df_oracle.hpp"

#include "hygro_oracle.h"

using namespace hygro;
using Clock = std::chrono::steady_clock;

namespace {

constexpr double kTi = 293.15, kPhi = 0.5, kT0 = 3600.0;   // wall_nonlinear.json:3 scaling block
constexpr double kCw = 4180.0, kLv = 2.5e6;                 // PhysicalConstants materials.hpp:10,13
const double kD[4] = {0.91, 600.0, 10.0, 1.5};              // d(v) = 1 + 0.91 v + 600 exp(-10 (v-1.5)^2)

struct Args {
    std::string config = "cfg1";
    int steps = 5, warmup = 3, threads = 1;
    int walls = 65536, nodes = 256, zones = 8192, material_walls = 16384;
    long long long_nodes = 1LL << 26;
    int sample_steps = 0, implicit_steps = 0;   // 0: config default
    bool implicit = true;
};

double secs(Clock::time_point a, Clock::time_point b) { return std::chrono::duration<double>(b - a).count(); }

double log_uniform(std::mt19937_64& g, double lo, double hi) {
    std::uniform_real_distribution<double> u(std::log(lo), std::log(hi));
    return std::exp(u(g));
}

// split [0, n) into nthreads contiguous ranges and run fn(i, lo, hi) on each
void parallel_for(int nthreads, long n, const std::function<void(int, long, long)>& fn) {
    nthreads = static_cast<int>(std::max<long>(1, std::min<long>(nthreads, n)));
    std::vector<std::thread> th;
    for (int i = 1; i < nthreads; ++i) th.emplace_back(fn, i, n * i / nthreads, n * (i + 1) / nthreads);
    fn(0, 0, n / nthreads);
    for (auto& t : th) t.join();
}

// ---- cfg1/cfg2: independent constant-coefficient walls -------------------------
struct Walls {
    Grid1D grid;
    std::vector<WallGroups> groups;
    std::vector<FaceBiot> face[2];
    std::vector<WallField> f;
    double P_vi = 0.0;
    FaceValues left(int w, double t) const {   // exterior: T_i (1 + 0.02 s), phi_i (1 + 0.2 s)
        const double s = std::sin(2.0 * M_PI * t / 24.0);
        const double T = kTi * (1.0 + 0.02 * s), phi = kPhi * (1.0 + 0.2 * s);
        FaceValues L;
        L.Bi_M = face[0][w].Bi_M;
        L.Bi_TT = face[0][w].Bi_TT;
        L.Bi_TM = face[0][w].Bi_TM;
        L.u_inf = T / kTi;
        L.v_inf = phi * saturation_pressure(T) / P_vi;
        return L;
    }
    FaceValues right(int w) const {
        FaceValues R;
        R.Bi_M = face[1][w].Bi_M;
        R.Bi_TT = face[1][w].Bi_TT;
        R.Bi_TM = face[1][w].Bi_TM;
        return R;
    }
};

Walls batched_walls(const Args& a) {
    Walls W;
    W.grid = Grid1D{a.nodes, 1.0 / (a.nodes - 1)};
    const ScalingContext ctx = ScalingContext::from_state(kTi, kPhi, kT0);
    W.P_vi = ctx.P_vi;
    std::mt19937_64 g(1);
    std::normal_distribution<double> noise(0.0, 0.01);
    for (int w = 0; w < a.walls; ++w) {
        const double k_tt = log_uniform(g, 0.1, 2.0), d_m = log_uniform(g, 1e-12, 1e-10);
        const double rho_c = log_uniform(g, 5e5, 2e6), c_m = log_uniform(g, 1e-4, 1e-2);
        const CoefficientSet ref{c_m, d_m, rho_c, k_tt, kCw * (kTi - 273.15) * c_m, kLv * d_m};
        const WallDimensionless d = scale_wall(ref, 0.1, 25.0, 2e-7, 8.0, 3e-8, ctx);
        W.groups.push_back(d.groups);
        W.face[0].push_back(d.face[0]);
        W.face[1].push_back(d.face[1]);
        WallField f = WallField::uniform(W.grid);
        for (int j = 0; j < a.nodes; ++j) {
            f.u_curr[j] = f.u_prev[j] = 1.0 + noise(g);
            f.v_curr[j] = f.v_prev[j] = 1.0 + noise(g);
        }
        W.f.push_back(std::move(f));
    }
    return W;
}

// ---- cfg3: the zone ring as a BuildingModel -------------------------------------
BuildingModel zone_ring(const Args& a) {
    BuildingModel m;
    m.ctx = ScalingContext::from_state(kTi, kPhi, kT0);
    m.dt = 1e-3;
    m.eta_factor = 1e-6;
    const double V = 54.0;
    ZoneAirConfig air;                             // one_zone_linear.json:44-59
    air.volume = V;
    air.rho_a = 1.0;
    air.c_pa = 1005.0;
    air.c_pv = 1960.0;
    air.ventilation_ach = 0.5;
    air.moisture_source = Signal::schedule(6.9444444444e-6, {{6.0, 9.0, 1.1111111111e-4},
                                                             {30.0, 33.0, 1.1111111111e-4},
                                                             {54.0, 57.0, 1.1111111111e-4}});
    air.heat_source = Signal::constant(0.0);
    const ZoneDimensionless zd = scale_zone(air, m.ctx);
    const InterzoneScalars inz = scale_interzone(0.5, air, zd, m.ctx);
    m.outdoor_u = Signal::sin_squared(1.0, -0.02, 24.0);
    m.outdoor_v = Signal::sinusoid(1.0, 0.06, 24.0);
    // frozen sets of one_zone_linear.json:5-7, cycled N/S/E/W/E/W (:14-43)
    const CoefficientSet north{1.82e-2, 5.89e-9, 7.70e5, 2.94e-1, 1.52e3, 1.59e-2};
    const CoefficientSet south{1.18e-1, 2.92e-8, 1.28e6, 8.41e-1, 9.88e3, 2.96e-3};
    const CoefficientSet ew{6.09e-2, 5.47e-9, 8.61e5, 3.87e-1, 5.09e3, 1.53e-2};
    struct Spec { CoefficientSet s; double area, hT, hM; };
    const Spec specs[6] = {{north, 18.0, 5.0, 2e-7}, {south, 18.0, 25.0, 8e-7}, {ew, 9.0, 12.0, 4e-7},
                           {ew, 9.0, 12.0, 4e-7},    {ew, 9.0, 12.0, 4e-7},     {ew, 9.0, 12.0, 4e-7}};
    WallDimensionless wd[6];
    for (int i = 0; i < 6; ++i) {
        wd[i] = scale_wall(specs[i].s, 0.1, specs[i].hT, specs[i].hM, 8.0, 3e-8, m.ctx);
        attach_wall_to_zone(wd[i], specs[i].area, 0.1, zd, m.ctx);
    }
    const Grid1D grid{a.nodes, 1.0 / (a.nodes - 1)};
    for (int z = 0; z < a.zones; ++z) {
        ZoneConfig zc;
        zc.name = "z" + std::to_string(z);
        zc.params = zd;
        zc.moisture_sign = MoistureWallSign::FluxConsistent;
        for (int i = 0; i < 6; ++i) {
            BuildingWall bw;
            bw.name = "w" + std::to_string(z * 6 + i);
            bw.grid = grid;
            bw.groups = wd[i].groups;
            bw.biot[0] = wd[i].face[0];
            bw.biot[1] = wd[i].face[1];
            bw.attach[0].kind = FaceAttachment::Kind::Exterior;
            bw.attach[0].u_inf = m.outdoor_u;
            bw.attach[0].v_inf = m.outdoor_v;
            bw.attach[1].kind = FaceAttachment::Kind::Zone;
            bw.attach[1].zone = z;
            m.walls.push_back(bw);
            ZoneWallLink l;
            l.wall = z * 6 + i;
            l.face = 1;
            l.Bi_M = wd[i].face[1].Bi_M;
            l.Bi_TT = wd[i].face[1].Bi_TT;
            l.Bi_TM = wd[i].face[1].Bi_TM;
            l.theta_T = wd[i].theta_T;
            l.theta_M = wd[i].theta_M;
            zc.walls.push_back(l);
        }
        if (a.zones > 1)
            for (int p : {(z + a.zones - 1) % a.zones, (z + 1) % a.zones})
                zc.interzone.push_back(ZoneInterzoneLink{p, inz.g_inz, inz.q_inz1, inz.q_inz2});
        m.zones.push_back(zc);
    }
    return m;
}

// run()'s explicit loop body with the walls and zones split over threads:
// step_explicit's statements (building.cpp:152-187, no radiation in the ring)
// around the reference's own df_step_coupled and zone_step_explicit
struct RingStepper {
    const BuildingModel& m;
    BuildingState& st;
    int nthreads;
    std::vector<ZoneState> zones_now;
    std::vector<ZoneSamples> samples;
    std::atomic<int> bad{0};
    RingStepper(const BuildingModel& model, BuildingState& s, int nt)
        : m(model), st(s), nthreads(nt), zones_now(model.zones.size()), samples(model.zones.size()) {
        for (std::size_t z = 0; z < m.zones.size(); ++z) {
            samples[z].u_s.resize(m.zones[z].walls.size());
            samples[z].v_s.resize(m.zones[z].walls.size());
        }
    }
    FaceValues face(const BuildingWall& w, int k, double t) const {   // resolve_face building.cpp:107-126
        const FaceAttachment& a = w.attach[k];
        FaceValues b;
        b.Bi_M = w.biot[k].Bi_M;
        b.Bi_TT = w.biot[k].Bi_TT;
        b.Bi_TM = w.biot[k].Bi_TM;
        if (a.kind == FaceAttachment::Kind::Exterior) {
            b.u_inf = a.u_inf(t);
            b.v_inf = a.v_inf(t);
            b.g_inf = a.g_inf(t);
            b.q_inf = a.q_inf(t);
        } else {
            b.u_inf = zones_now[a.zone].u_a;
            b.v_inf = zones_now[a.zone].v_a;
        }
        return b;
    }
    void march(long nsteps) {
        const long nw = static_cast<long>(m.walls.size()), nz = static_cast<long>(m.zones.size());
        std::barrier sync(nthreads);
        parallel_for(nthreads, nthreads, [&](int id, long, long) {
            const long w0 = nw * id / nthreads, w1 = nw * (id + 1) / nthreads;
            const long z0 = nz * id / nthreads, z1 = nz * (id + 1) / nthreads;
            for (long k = 0; k < nsteps; ++k) {
                const double t = st.t, dt = m.dt;
                for (long z = z0; z < z1; ++z) {          // layer-n snapshot and samples
                    zones_now[z] = st.zones[z];
                    const ZoneConfig& zc = m.zones[z];
                    for (std::size_t i = 0; i < zc.walls.size(); ++i) {
                        const BuildingWall& w = m.walls[zc.walls[i].wall];
                        const int j = zc.walls[i].face == 0 ? 0 : w.grid.n - 1;
                        samples[z].u_s[i] = st.walls[zc.walls[i].wall].u_curr[j];
                        samples[z].v_s[i] = st.walls[zc.walls[i].wall].v_curr[j];
                    }
                }
                sync.arrive_and_wait();
                for (long i = w0; i < w1; ++i) {
                    const BuildingWall& w = m.walls[i];
                    df_step_coupled(st.walls[i], w.grid, w.groups, face(w, 0, t), face(w, 1, t), dt);
                    if (!(max_abs_field(st.walls[i]) <= m.divergence_norm)) bad = 1;
                }
                const double u_out = m.outdoor_u(t), v_out = m.outdoor_v(t);
                for (long z = z0; z < z1; ++z)
                    st.zones[z] = zone_step_explicit(zones_now[z], m.zones[z], samples[z], zones_now, u_out, v_out,
                                                     t, dt);
                sync.arrive_and_wait();
                if (id == 0) st.t += dt;
                sync.arrive_and_wait();
            }
        });
    }
};

// ---- d(v) walls (cfg0, cfg4) -----------------------------------------------------
CoefficientSet dv_star(double, double v) {
    CoefficientSet s;
    const double d = v - kD[3];
    s.k_M = 1.0 + kD[0] * v + kD[1] * std::exp(-kD[2] * d * d);
    return s;
}

std::vector<double> long_field(long long n, std::mt19937_64& g) {
    const double dx = 1e-2, X = (n - 1) * dx;
    std::uniform_real_distribution<double> amp(-0.3 / 16, 0.3 / 16), ph(0.0, 2.0 * M_PI);
    std::uniform_int_distribution<long long> mode(1, std::max<long long>(1, (n - 1) / 1024));
    std::vector<double> f(n, 1.0);
    for (int k = 0; k < 16; ++k) {
        const double a = amp(g), p = ph(g);
        const long long mk = mode(g);
        for (long long j = 0; j < n; ++j) f[j] += a * std::sin(2.0 * M_PI * mk * (j * dx) / X + p);
    }
    return f;
}

// ---- cfg5: load-bearing material walls --------------------------------------------
struct MatWalls {
    Grid1D grid;
    CoefficientModel cm;
    std::vector<WallGroups> groups;
    std::vector<FaceBiot> face[2];
    std::vector<WallField> f;
    FaceValues fv(int w, int k, double t) const {
        FaceValues b;
        b.Bi_M = face[k][w].Bi_M;
        b.Bi_TT = face[k][w].Bi_TT;
        b.Bi_TM = face[k][w].Bi_TM;
        b.v_inf = k == 0 ? 1.0 + 0.30 * std::sin(2.0 * M_PI * t / 6.0)
                         : 1.0 + 0.24 * std::sin(2.0 * M_PI * (t - 6.0) / 24.0);
        return b;
    }
};

MatWalls material_walls(int n_walls, int n_nodes) {
    MatWalls M;
    M.grid = Grid1D{n_nodes, 1.0 / (n_nodes - 1)};
    const ScalingContext ctx = ScalingContext::from_state(kTi, kPhi, kT0);
    const MaterialModel mat;
    const CoefficientSet ref = mat.evaluate(kTi, ctx.P_vi);   // scenario.cpp:178
    M.cm = CoefficientModel::material(mat, ctx, ref);
    std::mt19937_64 g(5);
    for (int w = 0; w < n_walls; ++w) {
        const double hT0 = log_uniform(g, 15.0, 35.0), hT1 = log_uniform(g, 5.0, 12.0);
        const double hM0 = log_uniform(g, 8e-8, 2e-7), hM1 = log_uniform(g, 2e-8, 5e-8);
        const WallDimensionless d = scale_wall(ref, 0.1, hT0, hM0, hT1, hM1, ctx);
        M.groups.push_back(d.groups);
        M.face[0].push_back(d.face[0]);
        M.face[1].push_back(d.face[1]);
        M.f.push_back(WallField::uniform(M.grid));
    }
    return M;
}

// ---- the effective-core figure: a compute-bound spin on 1 and on all threads -------
double spin_cores(int nthreads) {
    auto spin = [](long iters) {
        volatile double x = 1.0;
        double y = x;
        for (long i = 0; i < iters; ++i) y = y * 1.0000000001 + 1e-12;
        x = y;
    };
    const long iters = 200'000'000;
    auto t0 = Clock::now();
    spin(iters);
    const double one = secs(t0, Clock::now());
    t0 = Clock::now();
    parallel_for(nthreads, nthreads, [&](int, long, long) { spin(iters); });
    const double all = secs(t0, Clock::now());
    return nthreads * one / all;
}

struct Timing {
    std::vector<double> rates, secs;
    std::string sample, what, kind = "reference";
    int cores = 1;
    double updates = 0;
};

void json_timing(const char* key, const Timing& t, bool last) {
    std::printf("\"%s\": {\"rates\": [", key);
    for (std::size_t i = 0; i < t.rates.size(); ++i) std::printf("%s%.6e", i ? ", " : "", t.rates[i]);
    std::printf("], \"secs\": [");
    for (std::size_t i = 0; i < t.secs.size(); ++i) std::printf("%s%.4f", i ? ", " : "", t.secs[i]);
    std::printf("], \"node_updates_per_sample\": %.6e, \"cores\": %d, \"kind\": \"%s\", \"sample\": \"%s\", "
                "\"path\": \"%s\"}%s",
                t.updates, t.cores, t.kind.c_str(), t.sample.c_str(), t.what.c_str(), last ? "" : ", ");
}

// time `reps` samples of fn (which performs `updates` node-updates each)
void timed(Timing& T, int reps, double updates, const std::function<void()>& fn) {
    T.updates = updates;
    for (int r = 0; r < reps; ++r) {
        const auto t0 = Clock::now();
        fn();
        const double s = secs(t0, Clock::now());
        T.secs.push_back(s);
        T.rates.push_back(updates / s);
    }
}

}  // namespace

int main(int argc, char** argv) {
    Args a;
    for (int i = 1; i + 1 < argc; i += 2) {
        const std::string k = argv[i], v = argv[i + 1];
        if (k == "--config") a.config = v;
        else if (k == "--steps") a.steps = std::atoi(v.c_str());
        else if (k == "--warmup") a.warmup = std::atoi(v.c_str());
        else if (k == "--threads") a.threads = std::max(1, std::atoi(v.c_str()));
        else if (k == "--walls") a.walls = std::atoi(v.c_str());
        else if (k == "--nodes") a.nodes = std::atoi(v.c_str());
        else if (k == "--zones") a.zones = std::atoi(v.c_str());
        else if (k == "--material-walls") a.material_walls = std::atoi(v.c_str());
        else if (k == "--long-nodes") a.long_nodes = std::atoll(v.c_str());
        else if (k == "--sample-steps") a.sample_steps = std::atoi(v.c_str());
        else if (k == "--implicit-steps") a.implicit_steps = std::atoi(v.c_str());
        else if (k == "--implicit") a.implicit = v != "0";
        else {
            std::fprintf(stderr, "unknown option %s\n", k.c_str());
            return 2;
        }
    }
    const int reps = a.warmup + a.steps;
    const int T = a.threads;
    Timing df, imp;
    char buf[512];
    const auto setup0 = Clock::now();
    double setup_s = 0;
    std::string workload;

    if (a.config == "cfg1" || a.config == "cfg2") {
        if (a.config == "cfg2" && a.nodes == 256 && a.walls == 65536) workload = "cfg2";
        Walls W = batched_walls(a);
        setup_s = secs(setup0, Clock::now());
        const int ns = a.sample_steps ? a.sample_steps : 200;
        const double dt = 1e-3;
        double t0 = 0.0;
        timed(df, reps, double(a.walls) * a.nodes * ns, [&] {
            parallel_for(T, a.walls, [&](int, long w0, long w1) {
                for (long w = w0; w < w1; ++w) {
                    double t = t0;
                    for (int s = 0; s < ns; ++s) {
                        df_step_coupled(W.f[w], W.grid, W.groups[w], W.left(static_cast<int>(w), t),
                                        W.right(static_cast<int>(w)), dt);
                        if (!(max_abs_field(W.f[w]) <= 1e3)) std::abort();
                        t += dt;
                    }
                }
            });
            t0 += ns * dt;
        });
        df.cores = std::min(T, a.walls);
        std::snprintf(buf, sizeof buf, "all %d walls x %d nodes x %d DF steps per sample (fp64%s)", a.walls, a.nodes,
                      ns, a.config == "cfg2" ? "; the reference has no fp32 path" : "");
        df.sample = buf;
        df.what = "df_step_coupled + max_abs_field per wall-step (wall.cpp:144-194, 579-587), threads split walls";
        if (a.implicit) {
            const int ni = a.implicit_steps ? a.implicit_steps : std::max(1, ns / 4);
            timed(imp, reps, double(a.walls) * a.nodes * ni, [&] {
                parallel_for(T, a.walls, [&](int, long w0, long w1) {
                    for (long w = w0; w < w1; ++w) {
                        double t = t0;
                        for (int s = 0; s < ni; ++s) {
                            euler_implicit_step(W.f[w], W.grid, W.groups[w], CoefficientModel::constant(),
                                                W.left(static_cast<int>(w), t + dt), W.right(static_cast<int>(w)),
                                                dt, 1e-2 * dt, 100);
                            t += dt;
                        }
                    }
                });
                t0 += ni * dt;
            });
            imp.cores = df.cores;
            std::snprintf(buf, sizeof buf, "all %d walls x %d nodes x %d Euler-implicit steps per sample", a.walls,
                          a.nodes, ni);
            imp.sample = buf;
            imp.what = "euler_implicit_step, constant coefficients: one exact pass (wall.cpp:515-550)";
        }
    } else if (a.config == "cfg3") {
        const BuildingModel m = zone_ring(a);
        BuildingState st = initial_state(m);
        std::mt19937_64 g(3);
        std::normal_distribution<double> noise(0.0, 2e-3);
        for (auto& f : st.walls)
            for (int j = 0; j < f.nodes(); ++j) {
                f.u_curr[j] = f.u_prev[j] = 1.0 + noise(g);
                f.v_curr[j] = f.v_prev[j] = 1.0 + noise(g);
            }
        step_implicit(m, st, m.eta(), m.max_subiters);   // run()'s DF start (building.cpp:317-318)
        setup_s = secs(setup0, Clock::now());
        const double cells = double(m.walls.size()) * a.nodes;
        const int ns = a.sample_steps ? a.sample_steps : 100;
        RingStepper rs(m, st, T);
        timed(df, reps, cells * ns, [&] { rs.march(ns); });
        if (rs.bad) std::abort();
        df.cores = T;
        std::snprintf(buf, sizeof buf, "all %d zones x 6 walls x %d nodes x %d DF building steps per sample", a.zones,
                      a.nodes, ns);
        df.sample = buf;
        df.what = "step_explicit's body (building.cpp:152-187) with df_step_coupled / zone_step_explicit, walls and "
                  "zones split over threads per step";
        // the serial public call, for reference (1 core)
        Timing ser;
        const int nser = std::max(5, ns / 10);
        timed(ser, 1, cells * nser, [&] {
            for (int s = 0; s < nser; ++s) step_explicit(m, st);
        });
        std::printf("{\"serial_step_explicit\": %.6e, \"serial_steps\": %d, ", ser.rates[0], nser);
        if (a.implicit) {
            const int ni = a.implicit_steps ? a.implicit_steps : 3;
            long passes = 0;
            timed(imp, reps, cells * ni, [&] {
                for (int s = 0; s < ni; ++s) passes += step_implicit(m, st, m.eta(), m.max_subiters).subiterations;
            });
            std::snprintf(buf, sizeof buf, "all %d zones x 6 walls x %d nodes x %d Euler-implicit building steps per "
                          "sample, %.2f fixed-point passes per step", a.zones, a.nodes, ni,
                          double(passes) / (double(ni) * reps));
            imp.sample = buf;
            imp.what = "step_implicit (building.cpp:189-268), the reference's serial public call";
        }
    } else if (a.config == "cfg0" || a.config == "cfg4") {
        const bool long_dom = a.config == "cfg4";
        const long long n = long_dom ? std::min<long long>(a.long_nodes, 1LL << 22) : 101;
        const double dx = long_dom ? 1e-2 : 0.01, dt = 1e-3;
        WallGroups p;
        p.Fo_M = long_dom ? 0.116 : 0.1;
        p.Fo_TT = long_dom ? 0.137 : 0.1;
        p.Fo_TM = long_dom ? 3.76 : 1.0;
        p.gamma = long_dom ? 7.87e-3 : 0.0;
        FaceValues L, R;
        L.Bi_M = 2.0;
        R.Bi_M = 1.0;
        if (long_dom) {
            L.Bi_TT = 1.7;
            L.Bi_TM = 0.678;
            R.Bi_TT = 2.72;
            R.Bi_TM = 0.101;
        }
        oracle::Layers o;
        if (long_dom) {
            std::mt19937_64 g(4);
            o.uc = long_field(n, g);
            o.vc = long_field(n, g);
        } else {
            o.uc.assign(n, 1.0);
            o.vc.assign(n, 1.0);
        }
        o.up = o.uc;
        o.vp = o.vc;
        setup_s = secs(setup0, Clock::now());
        const int ns = a.sample_steps ? a.sample_steps : (long_dom ? 5 : 20000);
        double t = 0.0;
        timed(df, reps, double(n) * ns, [&] {
            for (int s = 0; s < ns; ++s) {
                L.v_inf = 1.0 + 0.8 * std::sin(2.0 * M_PI * t / 24.0);
                oracle::df_step(o, p, L, R, dt, dx, dv_star);
                t += dt;
            }
        });
        std::snprintf(buf, sizeof buf, "1 wall x %lld nodes x %d DF steps per sample%s", n, ns,
                      long_dom ? " (the first 2^22 nodes of the 2^26-node domain)" : "");
        df.sample = buf;
        df.what = "the reference's transcription oracle oracle::df_step with the d(v) StarFn "
                  "(tests/support/df_oracle.hpp:25-106): CoefficientModel cannot express d(v)";
        if (a.implicit) {
            std::vector<double> up = o.up, uc = o.uc, vp = o.vp, vc = o.vc;
            orc_field f = {static_cast<int>(n), up.data(), uc.data(), vp.data(), vc.data(), 0.0};
            hyg_wall_groups gp = {p.Fo_M, p.Fo_TT, p.Fo_TM, p.gamma};
            orc_model om;
            std::memset(&om, 0, sizeof om);
            om.kind = ORC_COEFF_ANALYTIC_D;
            for (int i = 0; i < 4; ++i) om.p[i] = kD[i];
            const int ni = a.implicit_steps ? a.implicit_steps : (long_dom ? 2 : 2000);
            long passes = 0;
            timed(imp, reps, double(n) * ni, [&] {
                for (int s = 0; s < ni; ++s) {
                    orc_face fl = {L.Bi_M, L.Bi_TT, L.Bi_TM, 1.0, 1.0 + 0.8 * std::sin(2.0 * M_PI * (t + dt) / 24.0),
                                   0.0, 0.0};
                    orc_face fr = {R.Bi_M, R.Bi_TT, R.Bi_TM, 1.0, 1.0, 0.0, 0.0};
                    double res = 0;
                    passes += orc_euler_implicit_step(&f, dx, &gp, &om, &fl, &fr, dt, 1e-2 * dt, 100, &res);
                    t += dt;
                }
            });
            imp.kind = "port";
            std::snprintf(buf, sizeof buf, "1 wall x %lld nodes x %d Euler-implicit steps per sample, %.2f passes "
                          "per step", n, ni, double(passes) / (double(ni) * reps));
            imp.sample = buf;
            imp.what = "euler_implicit_step restated in C with the d(v) functor (oracle/hygro_oracle.c; the "
                       "reference's CoefficientModel cannot express d(v))";
        }
    } else if (a.config == "cfg5") {
        const int nw = std::min(a.material_walls, 16 * T);
        MatWalls M = material_walls(nw, 101);
        setup_s = secs(setup0, Clock::now());
        const int ns = a.sample_steps ? a.sample_steps : 100;
        const double dt = 1e-3;
        // implicit start (bootstrap_first_layer), as the GPU run does
        for (int w = 0; w < nw; ++w)
            bootstrap_first_layer(M.f[w], M.grid, M.groups[w], M.cm, M.fv(w, 0, dt), M.fv(w, 1, dt), dt, 1e-2 * dt,
                                  100);
        double t0 = dt;
        timed(df, reps, double(nw) * 101 * ns, [&] {
            parallel_for(T, nw, [&](int, long w0, long w1) {
                for (long w = w0; w < w1; ++w) {
                    double t = t0;
                    for (int s = 0; s < ns; ++s) {
                        df_step_nonlinear(M.f[w], M.grid, M.groups[w], M.cm, M.fv(static_cast<int>(w), 0, t),
                                          M.fv(static_cast<int>(w), 1, t), dt);
                        if (!(max_abs_field(M.f[w]) <= 1e3)) std::abort();
                        t += dt;
                    }
                }
            });
            t0 += ns * dt;
        });
        df.cores = std::min(T, nw);
        std::snprintf(buf, sizeof buf, "%d material walls x 101 nodes x %d DF steps per sample", nw, ns);
        df.sample = buf;
        df.what = "df_step_nonlinear with CoefficientModel::material (wall.cpp:196-264), threads split walls";
        if (a.implicit) {
            const int ni = a.implicit_steps ? a.implicit_steps : std::max(1, ns / 4);
            long passes = 0;
            std::vector<long> pp(T, 0);
            timed(imp, reps, double(nw) * 101 * ni, [&] {
                parallel_for(T, nw, [&](int id, long w0, long w1) {
                    for (long w = w0; w < w1; ++w) {
                        double t = t0;
                        for (int s = 0; s < ni; ++s) {
                            pp[id] += euler_implicit_step(M.f[w], M.grid, M.groups[w], M.cm,
                                                          M.fv(static_cast<int>(w), 0, t + dt),
                                                          M.fv(static_cast<int>(w), 1, t + dt), dt, 1e-2 * dt, 100);
                            t += dt;
                        }
                    }
                });
                t0 += ni * dt;
            });
            for (long x : pp) passes += x;
            imp.cores = df.cores;
            std::snprintf(buf, sizeof buf, "%d material walls x 101 nodes x %d Euler-implicit steps per sample, "
                          "%.2f passes per wall-step", nw, ni, double(passes) / (double(nw) * ni * reps));
            imp.sample = buf;
            imp.what = "euler_implicit_step with CoefficientModel::material (wall.cpp:515-550)";
        }
    } else {
        std::fprintf(stderr, "unknown config %s\n", a.config.c_str());
        return 2;
    }
    if (a.config != "cfg3") std::printf("{");
    std::printf("\"config\": \"%s\", \"threads\": %d, \"hardware_threads\": %u, \"effective_cores\": %.2f, "
                "\"setup_s\": %.2f, \"warmup\": %d, \"steps\": %d, ",
                a.config.c_str(), T, std::thread::hardware_concurrency(), spin_cores(T), setup_s, a.warmup, a.steps);
    json_timing("df", df, !a.implicit);
    if (a.implicit) json_timing("implicit", imp, true);
    std::printf("}\n");
    return 0;
}
