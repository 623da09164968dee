// scenario_check.cpp — TEST INFRASTRUCTURE: `hygrosim run` end to end on both
// paths.  The reference's scenario loader (load_scenario, scenario.cpp:147-413)
// builds the BuildingModel from a scenario JSON; the reference's run()
// (building.cpp:303-356) and the drop-in hygro::gpu::run (include/
// hygro_b200.hpp) march it; the reference's own CSV writer
// (write_timeseries_csv, csvio.cpp:17-41, as write_artifacts calls it,
// hygrosim.cpp:75-83) writes both results.  The two CSVs must have the same
// rows and text fields; numeric fields may differ only by the device's
// floating-point differences (relative L-inf of u, v <= 1e-10; %.12g prints
// most of them identically — the share of byte-identical rows is reported).
//
//   scenario_check <scenario.json> <out_dir> [tol]   (writes out_dir/{cpu,gpu}.csv; tol default 1e-10)
// Built by oracle/Makefile (target `scenario`); run by tests/test_gpu_scenarios.py.
#define HYGRO_B200_WITH_REFERENCE
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "hygro/csvio.hpp"
#include "hygro/errors.hpp"
#include "hygro/scenario.hpp"
#include "hygro_b200.hpp"

using namespace hygro;

static std::vector<std::string> split(const std::string& s, char c) {
    std::vector<std::string> out;
    std::string cur;
    for (char ch : s) {
        if (ch == c) {
            out.push_back(cur);
            cur.clear();
        } else {
            cur += ch;
        }
    }
    out.push_back(cur);
    return out;
}

static std::vector<std::string> lines_of(const std::string& path) {
    std::ifstream in(path);
    std::vector<std::string> out;
    for (std::string l; std::getline(in, l);) out.push_back(l);
    return out;
}

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: scenario_check <scenario.json> <out_dir>\n");
        return 2;
    }
    const Scenario sc = load_scenario(argv[1]);
    const std::string dir = argv[2];
    SimulationResult cpu, gpu, pc, pg;
    std::string cpu_err, gpu_err;
    try {
        cpu = run(sc.model, sc.cadence, &pc);
    } catch (const std::exception& e) {
        cpu_err = e.what();
        cpu = pc;
    }
    try {
        gpu = hygro::gpu::run(sc.model, sc.cadence, &pg);
    } catch (const std::exception& e) {
        gpu_err = e.what();
        gpu = pg;
    }
    {
        std::ofstream a(dir + "/cpu.csv"), b(dir + "/gpu.csv");
        write_timeseries_csv(a, sc.model, cpu);
        write_timeseries_csv(b, sc.model, gpu);
    }
    const auto A = lines_of(dir + "/cpu.csv"), B = lines_of(dir + "/gpu.csv");
    int bad = 0;
    if (cpu_err.empty() != gpu_err.empty()) {
        std::printf("error mismatch: cpu='%s' gpu='%s'\n", cpu_err.c_str(), gpu_err.c_str());
        ++bad;
    }
    if (A.size() != B.size()) {
        std::printf("row count differs: cpu %zu gpu %zu\n", A.size(), B.size());
        return 1;
    }
    size_t same = 0;
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < A.size(); ++i) {
        if (A[i] == B[i]) {
            ++same;
        }
        if (i == 0) {
            if (A[0] != B[0]) ++bad;
            continue;
        }
        const auto a = split(A[i], ','), b = split(B[i], ',');
        // t_star,entity,kind,node_or_zone,x_star,u,v,T_K,P_v_Pa,phi
        if (a.size() != 10 || b.size() != 10 || a[0] != b[0] || a[1] != b[1] || a[2] != b[2] || a[3] != b[3] ||
            a[4] != b[4]) {
            if (bad < 5) std::printf("row %zu structure differs:\n  %s\n  %s\n", i, A[i].c_str(), B[i].c_str());
            ++bad;
            continue;
        }
        for (int k = 5; k <= 6; ++k) {
            const double x = std::strtod(a[k].c_str(), nullptr), y = std::strtod(b[k].c_str(), nullptr);
            num = std::max(num, std::fabs(x - y));
            den = std::max(den, std::fabs(x));
        }
    }
    const double rel = den > 0 ? num / den : 0.0;
    std::printf("%s: rows %zu, byte-identical %zu (%.4f%%), frames cpu %zu gpu %zu, steps %ld/%ld, "
                "boot passes %d/%d, rel_linf(u,v as printed) %.3e%s%s\n",
                sc.name.c_str(), A.size(), same, 100.0 * same / A.size(), cpu.frames.size(), gpu.frames.size(),
                cpu.steps, gpu.steps, cpu.bootstrap_subiters, gpu.bootstrap_subiters, rel,
                cpu_err.empty() ? "" : (" cpu error: " + cpu_err).c_str(),
                gpu_err.empty() ? "" : (" gpu error: " + gpu_err).c_str());
    // %.12g printing bounds the visible difference by ~5e-12 relative even
    // when the underlying values agree to 1e-14
    const double tol = argc > 3 ? std::strtod(argv[3], nullptr) : 1e-10;
    if (!(rel <= tol)) ++bad;
    if (cpu.frames.size() != gpu.frames.size() || cpu.bootstrap_subiters != gpu.bootstrap_subiters) ++bad;
    // SimulationResult counters of the implicit scheme (building.cpp:327-352)
    std::printf("  steps %ld/%ld, mean subiters %.6f/%.6f, max subiters %d/%d\n", cpu.steps, gpu.steps,
                cpu.mean_subiters, gpu.mean_subiters, cpu.max_subiters_seen, gpu.max_subiters_seen);
    if (cpu.steps != gpu.steps || cpu.max_subiters_seen != gpu.max_subiters_seen ||
        cpu.mean_subiters != gpu.mean_subiters)
        ++bad;
    return bad ? 1 : 0;
}
