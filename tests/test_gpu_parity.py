"""CUDA path (through the C ABI) vs the C oracle, at the BASELINE configs.

Tolerances (north_star): relative L-inf <= 1e-10 in fp64 after the full run,
<= 1e-4 for the fp32 variant.  Relative L-inf = max|gpu - ref| / max|ref| over
both time layers of both fields.  Full-size configs are
checked on seeded strided subsets at the full horizon plus all walls on a
short horizon (SURVEY.md §8d parity procedure).
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_1703_10119_b200 import Context, NumericalError, workloads
from paper_1703_10119_b200.api import ChannelSpec, Model, Signal

from .helpers import FIELDS, gpu_run, oracle_run, random_walls, rel_linf

pytestmark = pytest.mark.gpu

TOL64, TOL32 = 1e-10, 1e-4


def _subset(w, idx):
    """Workload restricted to walls idx (same parameters, same initial rows)."""
    m = w.model
    n = m.n_nodes
    sub = Model(n, m.dx, m.groups[idx], m.biot[idx], m.attach[idx], channels=m.channels, dt=m.dt,
                precision=m.precision, divergence_norm=m.divergence_norm)
    rows = (np.asarray(idx)[:, None] * n + np.arange(n)[None, :]).reshape(-1)
    init = {k: v[rows] for k, v in w.init.items() if k in FIELDS}
    return sub, init, rows


def _extreme_walls(m, k=256):
    """Strided subset plus the walls at the extremes of lambda, mu, Bi."""
    W = m.n_walls
    idx = set(range(0, W, max(1, W // (k - 24))))
    for col in (m.groups[:, 0], m.groups[:, 1], m.groups[:, 2] * m.groups[:, 3], m.biot[:, 0, 0],
                m.biot[:, 1, 0], m.biot[:, 0, 1], m.biot[:, 0, 2]):
        order = np.argsort(col)
        idx.update(order[:2].tolist() + order[-2:].tolist())
    return np.array(sorted(idx))


@pytest.fixture(scope="module")
def cfg1():
    return workloads.batched_walls()     # 65,536 walls x 256, 1e5 steps


def test_cfg1_full_horizon_subset(cfg1):
    """All 65,536 walls on the GPU for the full 1e5 steps (implicit start);
    the oracle runs a strided + extreme-parameter subset of >= 1,024 of them
    (SURVEY.md §8(d))."""
    w = cfg1
    got = gpu_run(w.model, w.init, w.nsteps, w.boot, w.tables)
    assert got["launches"] > 0 and got["layer"] == w.nsteps
    assert abs(got["t"] - workloads.accumulate_times(np.full(w.nsteps, w.model.dt))[-1]) == 0.0
    idx = _extreme_walls(w.model, 1100)
    assert idx.size >= 1024
    sub, init, rows = _subset(w, idx)
    ref = oracle_run("oracle", sub, init, w.nsteps, w.boot, w.tables)
    err = rel_linf({k: got[k][rows] for k in FIELDS}, ref)
    assert err <= TOL64, err


def test_cfg1_all_walls_short_horizon(cfg1):
    """All 65,536 walls for 1,000 steps."""
    w = cfg1
    n = 1000
    got = gpu_run(w.model, w.init, n, w.boot, w.tables)
    ref = oracle_run("oracle", w.model, w.init, n, w.boot, w.tables)
    err = rel_linf(got, ref)
    assert err <= TOL64, err


@pytest.fixture(scope="module")
def cfg2():
    return workloads.batched_walls(precision="f32", variable_dt=True)    # 65,536 walls x 256, 1e5 steps


def test_cfg2_fp32_variable_dt(cfg2):
    """configs[2] at full size: fp32 state (deviations from 1, fp64 boundary
    flux terms) with dt doubling every 1e4 steps up to 16 dt0, all 65,536
    walls for the full 1e5 steps on the GPU, against the fp64 oracle on the
    same schedule for a strided + extreme-parameter subset of >= 1,024 walls."""
    w = cfg2
    got = gpu_run(w.model, w.init, w.nsteps, w.boot, w.tables, dt_schedule=w.dt_schedule)
    idx = _extreme_walls(w.model, 1100)
    assert idx.size >= 1024
    sub, init, rows = _subset(w, idx)
    sub.precision = "f64"
    ref = oracle_run("oracle", sub, init, w.nsteps, w.boot, w.tables, dt_schedule=w.dt_schedule)
    err = rel_linf({k: got[k][rows] for k in FIELDS}, ref)
    print("cfg2 full horizon, 1e5 steps, subset", idx.size, "rel L-inf", err)
    assert err <= TOL32, err
    assert abs(got["t"] - 1110.0) < 1e-9


def test_cfg2_all_walls_short_horizon(cfg2):
    """All 65,536 fp32 walls for 1,000 steps against the fp64 oracle."""
    w = cfg2
    n = 1000
    got = gpu_run(w.model, w.init, n, w.boot, w.tables, dt_schedule=w.dt_schedule)
    sub = Model(w.model.n_nodes, w.model.dx, w.model.groups, w.model.biot, w.model.attach, channels=w.model.channels,
                dt=w.model.dt, divergence_norm=w.model.divergence_norm)
    ref = oracle_run("oracle", sub, w.init, n, w.boot, w.tables, dt_schedule=w.dt_schedule)
    err = rel_linf(got, ref)
    print("cfg2 all walls x 1000 steps rel L-inf", err)
    assert err <= TOL32, err


def test_cfg4_n2e20_full_horizon():
    """configs[4] at N = 2^20 for the full 1e4 steps: about
    2.5 windows per warp, so the persistent, prefetching K3w runs at full
    horizon; the oracle splits the wall's nodes over the host threads
    (bitwise its serial march)."""
    w = workloads.long_domain(n_nodes=1 << 20, nsteps=10_000)
    from paper_1703_10119_b200 import Context
    with Context(w.model) as ctx:
        ctx.set_state(**w.init)
        ctx.profiling(True)
        ctx.advance(w.nsteps)
        ctx.synchronize()
        stats = {s_["name"]: s_ for s_ in ctx.kernel_stats()}
        got = ctx.get_state()
    assert stats.get("df_analytic_tiled", {}).get("launches", 0) > 0, stats.keys()
    ref = oracle_run("oracle", w.model, w.init, w.nsteps, w.boot)
    err = rel_linf(got, ref)
    print("cfg4 N=2^20 x 1e4 steps rel L-inf", err)
    assert err <= TOL64, err


def test_cfg0_single_wall_full_run():
    """configs[0]: N=101, d(v), 1 explicit start + 99,999 DF steps."""
    w = workloads.single_wall_d()
    got = gpu_run(w.model, w.init, w.nsteps, w.boot)
    ref = oracle_run("oracle", w.model, w.init, w.nsteps, w.boot)
    err = rel_linf(got, ref)
    assert err <= TOL64, err
    assert float(np.max(np.abs(got["u_curr"] - 1.0))) < 1e-12     # gamma = 0: u stays 1
    assert 0.4 < float(got["v_curr"].min()) and float(got["v_curr"].max()) < 1.9


def test_cfg4_long_domain_reduced():
    """configs[4] at N=2^16 for 2000 steps (the full N=2^26 is checked on a
    short horizon in test_cfg4_full_size_short_horizon)."""
    w = workloads.long_domain(n_nodes=1 << 16, nsteps=2000)
    got = gpu_run(w.model, w.init, w.nsteps, w.boot)
    ref = oracle_run("oracle", w.model, w.init, w.nsteps, w.boot)
    err = rel_linf(got, ref)
    assert err <= TOL64, err


@pytest.mark.parametrize("n_nodes,steps", [(1025, 37), (3000, 50), ((1 << 16) + 7, 33)])
def test_tiled_long_wall_edges(n_nodes, steps):
    """K3 (temporal blocking): tiles not dividing N, steps not dividing S,
    a face inside the first and the last tile."""
    w = workloads.long_domain(n_nodes=n_nodes, nsteps=steps)
    got = gpu_run(w.model, w.init, steps, w.boot)
    ref = oracle_run("oracle", w.model, w.init, steps, w.boot, nthreads=1)
    assert rel_linf(got, ref) <= TOL64


def test_nonlinear_fast_guard_fallback():
    """|v| >= 2 in a nonlinear wall: the fast guard of K2s/K3w fires, the
    march continues on the per-step kernel with the exact guard, same result."""
    for n in (101, 4000):
        w = workloads.long_domain(n_nodes=n, nsteps=300)
        # a mild d(v) = 1 + 0.5 v: the stiff configs[0] bump would itself diverge
        w.model.coeff_params = (0.5, 0.0, 10.0, 1.5)
        for k in FIELDS:
            w.init[k] = w.init[k].copy()
            w.init[k][n // 2: n // 2 + 5] += 1.2
        got = gpu_run(w.model, w.init, 300, "none")
        ref = oracle_run("oracle", w.model, w.init, 300, "none", nthreads=1)
        assert rel_linf(got, ref) <= TOL64, n


@pytest.mark.parametrize("n", [101, 3000])
def test_nonlinear_norm_below_two(n):
    """divergence_norm < 2: the fast guard cannot prove |x| <= norm, so d(v)
    walls take the exact per-step guard; the first failing layer and wall
    equal the oracle's check_bounded."""
    w = workloads.long_domain(n_nodes=n, nsteps=400)
    w.model.coeff_params = (0.5, 0.0, 10.0, 1.5)
    for k in FIELDS:
        w.init[k] = w.init[k].copy()
        w.init[k][n // 2: n // 2 + 5] += 0.2
    peak = max(float(np.max(np.abs(w.init[k]))) for k in FIELDS)
    w.model.divergence_norm = peak - 0.05            # crossed in the first steps, inside the wall
    wb_err = None
    try:
        oracle_run("oracle", w.model, w.init, 400, "none", nthreads=1)
    except AssertionError as e:
        wb_err = e.args[0]
    assert wb_err is not None and wb_err[0] == api_codes().HYG_EDIVERGED, wb_err
    with Context(w.model) as ctx:
        ctx.set_state(**w.init)
        with pytest.raises(NumericalError) as ei:
            ctx.advance(400)
    assert ei.value.layer == wb_err[1] and ei.value.wall == wb_err[2], (ei.value.layer, ei.value.wall, wb_err)


def api_codes():
    from paper_1703_10119_b200 import api
    return api.A


def test_cfg4_full_size_short_horizon():
    """configs[4] at the full N = 2^26.  After k DF steps node j depends only on
    nodes j-k..j+k (three-level stencil), so windows of 2^14 nodes at both
    faces and in the middle, padded by k+2 nodes of real initial data, are
    checked exactly by the oracle treating the far pad end as a face."""
    N, k, W = 1 << 26, 100, 1 << 14
    w = workloads.long_domain(n_nodes=N, nsteps=k)
    got = gpu_run(w.model, w.init, k, w.boot)
    pad = k + 2
    m = w.model
    for lo, hi, keep in ((0, W + pad, slice(0, W)), (N - W - pad, N, slice(pad, W + pad)),
                         (N // 2 - pad, N // 2 + W + pad, slice(pad, pad + W))):
        sub = Model(hi - lo, m.dx, m.groups, m.biot, m.attach, channels=m.channels, dt=m.dt,
                    coeff_kind=m.coeff_kind, coeff_params=m.coeff_params)
        init = {f: w.init[f][lo:hi] for f in FIELDS}
        ref = oracle_run("oracle", sub, init, k, w.boot)
        err = rel_linf({f: got[f][lo:hi][keep] for f in FIELDS}, {f: ref[f][keep] for f in FIELDS})
        assert err <= TOL64, (lo, err)


@pytest.mark.parametrize("n_zones,wpz,n,steps", [(1, 4, 101, 3000), (16, 6, 128, 2000)])
def test_cfg3_building_ring(n_zones, wpz, n, steps):
    """Zones: implicit building start (joint wall/zone fixed point) then
    step_explicit with zone faces and the inter-zone ring."""
    w = workloads.zone_ring(n_zones=n_zones, walls_per_zone=wpz, n_nodes=n, nsteps=steps)
    with Context(w.model) as ctx:
        ctx.set_state(**w.init)
        st = ctx.bootstrap("implicit")
        ctx.advance(steps - 1)
        got = ctx.get_state()
    b = O.Building(w.model, w.init)
    rc, _, passes = b.run("oracle", steps)
    assert rc == 0 and st.subiterations == passes
    ref = dict(b.state)
    err = rel_linf(got, ref)
    zerr = max(float(np.max(np.abs(got["zone_u"] - b.zu))), float(np.max(np.abs(got["zone_v"] - b.zv))))
    assert err <= TOL64 and zerr <= TOL64, (err, zerr)


@pytest.mark.parametrize("n_nodes", [64, 128, 256, 512, 37])
def test_fused_and_general_grids_with_flux(n_nodes):
    """Every fused grid (and a non-fused one through the general kernel), with
    imposed face fluxes g_inf/q_inf and several channels."""
    model, init = random_walls(300, n_nodes, seed=n_nodes, flux=True, channels=3)
    for boot in ("implicit", "explicit"):
        got = gpu_run(model, init, 1500, boot)
        ref = oracle_run("oracle", model, init, 1500, boot)
        assert rel_linf(got, ref) <= TOL64, (boot, rel_linf(got, ref))


def test_guard_first_failing_layer_and_wall():
    """check_bounded semantics (building.cpp:282-300): divergence_norm below the
    ambient excursion -> same first failing layer and lowest wall as the oracle."""
    model, init = random_walls(64, 256, seed=2)
    init = {k: np.ones_like(v) for k, v in init.items()}
    model.divergence_norm = 1.012     # the ambient swing (up to 1.12) crosses it later
    times = workloads.accumulate_times(np.full(3000, model.dt))
    tab = O.forcing_table(model, times, 0)
    wb = O.WallBatch(model, init, tab)
    O.bootstrap("oracle", wb, "implicit", model.dt)
    wb.set_layer0(1, tab[1:])
    rc, fl, fw = O.march("oracle", wb, 2999, model.dt, O.threads())
    assert rc == 3 and fl > 1
    with Context(model) as ctx:
        ctx.set_state(**init)
        ctx.bootstrap("implicit")
        with pytest.raises(NumericalError) as e:
            ctx.advance(2999)
    assert (e.value.layer, e.value.wall) == (fl, fw)
    assert e.value.t_star == pytest.approx(times[fl], abs=0)


def test_guard_nan_and_fast_guard_false_positive():
    model, init = random_walls(40, 128, seed=9)
    bad = {k: v.copy() for k, v in init.items()}
    bad["v_curr"][17 * 128 + 40] = math.nan          # wall 17
    with Context(model) as ctx:
        ctx.set_state(**bad)
        with pytest.raises(NumericalError) as e:
            ctx.bootstrap("implicit")
        assert (e.value.layer, e.value.wall) == (1, 17)
    # |v| >= 2 somewhere but bounded: the fast guard fires, the exact replay
    # finds no failure, and the result is unchanged
    big = {k: v.copy() for k, v in init.items()}
    for k in FIELDS:
        big[k][5 * 128: 6 * 128] += 2.5
    got = gpu_run(model, big, 2000, "implicit")
    ref = oracle_run("oracle", model, big, 2000, "implicit")
    assert rel_linf(got, ref) <= TOL64


def test_run_frames_snapshot_and_state_roundtrip():
    """hyg_run (run(), building.cpp:303-356): frames at cadence incl. the
    initial and final states; snapshot/restore; exact state round trip."""
    model, init = random_walls(48, 128, seed=4)
    frames = []
    with Context(model) as ctx:
        ctx.set_state(**init)
        back = ctx.get_state()
        for k in FIELDS:
            assert np.array_equal(back[k], init[k])
        ctx.snapshot()

        def frame(layer, t, c):
            frames.append((layer, t, c.get_state()["v_curr"].copy()))
        ctx.run(horizon=1.0, cadence=0.25, boot="implicit", frame=frame)
        final = ctx.get_state()
        ctx.restore()
        again = ctx.get_state()
        for k in FIELDS:
            assert np.array_equal(again[k], init[k])
    assert [f[0] for f in frames] == [0, 250, 500, 750, 1000]
    ref = oracle_run("oracle", model, init, 1000, "implicit")
    assert rel_linf(final, ref) <= TOL64
    mid = oracle_run("oracle", model, init, 500, "implicit")
    assert float(np.max(np.abs(frames[2][2] - mid["v_curr"]))) <= TOL64


def test_advance_with_per_call_dt_fp64():
    """dt is a per-call argument (wall.hpp:81-82): fp64 walls on cfg2's schedule."""
    model, init = random_walls(128, 256, seed=6)
    sched = [(500, 1e-3), (500, 2e-3), (500, 4e-3)]
    got = gpu_run(model, init, 1500, "implicit", dt_schedule=sched)
    ref = oracle_run("oracle", model, init, 1500, "implicit", dt_schedule=sched)
    assert rel_linf(got, ref) <= TOL64


@pytest.mark.parametrize("n_walls,n_nodes", [(1, 101), (3, 256), (5, 17), (2, 33), (300, 101), (200, 256),
                                             (160, 33), (150, 64), (170, 200), (149, 7), (1, 65), (2, 97),
                                             (1, 3), (1, 32), (4, 129), (1, 40), (1, 70), (2, 104), (1, 150)])
def test_dv_wall_batches(n_walls, n_nodes):
    """Coupled d(v) walls with random groups, Biot numbers and imposed fluxes
    through K2s (n_walls <= 148: a wall over ceil(n/32) warps; n = 33, 65,
    97, 129 put the right face in lane 0 of the last warp; K2h, the halo
    variant, where ceil(n/32) warps leave H >= 2 spare lanes a side: n = 33
    (H = 6), 40 (6, exact fit), 65 (5), 70 (4), 97, 101, 104 (3, exact fit),
    129 (3); n = 150, 256 stay on K2s) and K2w
    (one warp per wall, every NPT x reversed-lane width M), explicit start."""
    model, init = random_walls(n_walls, n_nodes, seed=n_nodes + n_walls, flux=True)
    # cfg1's Fo_M range times d(v) ~ 50 diverges in the reference arithmetic too
    # (frozen-coefficient DF with coupled u): scale Fo_M into a bounded regime
    model.groups = model.groups.copy()
    model.groups[:, :3] *= np.array([1e-3, 1e-2, 1e-2])
    model.coeff_kind = "analytic_d"
    model.coeff_params = workloads.D_PARAMS
    nsteps = 400
    with Context(model) as ctx:
        ctx.profiling(True)
        ctx.set_state(**init)
        ctx.bootstrap("explicit")
        ctx.advance(nsteps - 1)
        got = ctx.get_state()
        names = {s["name"] for s in ctx.kernel_stats() if s["launches"] > 0}
    assert "df_analytic_fused" in names, names
    assert "df_step_general" not in names, names       # no fallback to the per-step path
    ref = oracle_run("oracle", model, init, nsteps, "explicit")
    assert rel_linf(got, ref) <= TOL64
