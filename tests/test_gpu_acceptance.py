"""The reference's own scenario fixtures (proj/scenarios/*.json, copied into
oracle/_ref/scenarios/ with the other build products of the reference) at
their own 80 h horizons, and acceptance criteria 5 and 6
(proj/tests/acceptance.cpp:165-230), through the drop-in hygro::gpu::run
(oracle/acceptance_check.cpp):

* fixtures: every frame (cadence 0.1, 801 frames) of the reference's run()
  and of hygro::gpu::run within relative L-inf 1e-10 (walls and zones) — or,
  where the fixture is worse conditioned than that, within 3x the deviation
  the reference itself shows when ONE initial value moves by one ulp
  (wall_nonlinear: ~8e-10; the reference's own FMA build differs by 7.7e-10)
  — same frame times, step counts and start passes; also the CSV rows through
  the reference's writer (scenario_check);
* criterion 5: Euler-implicit mean sub-iterations at eta = 1e-10 dt* within
  0.1 % of the CPU run's and inside the reference's windows;
* criterion 6: DF / Euler-implicit wall-clock ratio on the device <= 40 % at
  tau* = 20 and 40, drift <= 10 points."""
import json
import subprocess

import pytest

from .conftest import ROOT

pytestmark = pytest.mark.gpu

EXE = ROOT / "oracle" / "_ref" / "acceptance_check"
SCN = ROOT / "oracle" / "_ref" / "scenarios"
CHK = ROOT / "oracle" / "_ref" / "scenario_check"
FIXTURES = ["wall_nonlinear", "one_zone_linear", "two_zone_nonlinear"]

need = pytest.mark.skipif(not EXE.exists() or not SCN.exists(),
                          reason="acceptance_check / fixtures not built (need /root/reference at build time)")


def _run(*args, timeout=1800):
    r = subprocess.run([str(EXE), *map(str, args)], capture_output=True, text=True, timeout=timeout)
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    print(r.stdout, r.stderr[-2000:])
    return r.returncode, lines


@need
@pytest.mark.parametrize("name", FIXTURES)
def test_reference_fixture_full_horizon(name):
    rc, lines = _run("fixtures", SCN / f"{name}.json")
    (d,) = lines
    assert d["horizon"] == 80.0 and d["steps"][0] == d["steps"][1] == 80_000
    assert d["frames"][0] == d["frames"][1] == 801 and d["frame_t_diff"] == 0.0
    # 1e-10, or 3x the fixture's own conditioning where that is larger: the
    # reference moved by ONE ulp in one initial value (acceptance_check.cpp);
    # wall_nonlinear amplifies that to ~8e-10 over its 8e4 steps
    tol = max(1e-10, 3.0 * d["conditioning_1ulp"])
    assert d["rel_linf_walls"] <= tol and d["rel_linf_zones"] <= tol, d
    assert rc == 0 and d["ok"], d


@need
@pytest.mark.skipif(not CHK.exists(), reason="scenario_check not built")
@pytest.mark.parametrize("name", FIXTURES)
def test_reference_fixture_csv(name, tmp_path):
    """The reference's CSV writer on both results: same rows; printed u, v
    within 1e-10 (scenario_check's own bound)."""
    # wall_nonlinear: 3x its 1-ulp conditioning (~8e-10, test above)
    tol = "3e-9" if name == "wall_nonlinear" else "1e-10"
    r = subprocess.run([str(CHK), str(SCN / f"{name}.json"), str(tmp_path), tol], capture_output=True, text=True,
                       timeout=1800)
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0, r.stdout


@need
def test_criterion5_subiterations():
    rc, lines = _run("c5", SCN)
    assert len(lines) == 3
    for d in lines:
        # eta = 1e-10 dt*: a pass count can flip where a residual lands within an
        # ulp of the tolerance, so the means agree to 0.1 % (recorded: identical?)
        assert abs(d["mean_subiters"]["gpu"] - d["mean_subiters"]["cpu"]) <= 1e-3 * d["mean_subiters"]["cpu"], d
        assert d["window"][0] <= d["mean_subiters"]["gpu"] <= d["window"][1], d
    assert rc == 0


@need
def test_criterion6_df_vs_implicit_wall_clock():
    rc, lines = _run("c6", SCN)
    (d,) = lines
    print("criterion 6 on the device:", d)
    assert d["ratio_20"] <= 0.40 and d["ratio_40"] <= 0.40 and abs(d["ratio_20"] - d["ratio_40"]) <= 0.10, d
    assert rc == 0
