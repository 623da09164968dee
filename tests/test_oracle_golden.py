"""Pin the C oracle against the reference's golden vectors (tests/golden/,
made by make_golden.py from the unmodified reference) and against the
reference's own known-answer and property tests (proj/tests/test_wall.cpp,
test_building.cpp), restated.  No GPU, no /root/reference needed."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_1703_10119_b200 import workloads
from paper_1703_10119_b200.api import ChannelSpec, Model

from .helpers import FIELDS, oracle_run

GOLD = Path(__file__).resolve().parent / "golden"


def load(name):
    return np.load(GOLD / f"{name}.npz", allow_pickle=False)


def model_from(g, channels):
    m = Model(int(g["n_nodes"]), float(g["dx"]), g["groups"], g["biot"], g["attach"], channels=channels,
              dt=float(g["dt"]), coeff_kind=str(g["coeff_kind"]), coeff_params=tuple(g["coeff_params"]))
    return m


def march_table(g, impl="oracle"):
    """Replay a wall fixture with its stored forcing rows."""
    m = model_from(g, [ChannelSpec()] * g["table"].shape[1])
    init = {k: g[f"init_{k}"] for k in FIELDS}
    tab = g["table"]
    dts = g["dts"]
    nsteps = int(g["nsteps"])
    wb = O.WallBatch(m, init, tab)
    assert O.bootstrap(impl, wb, str(g["boot"]), float(dts[0]), nthreads=4) == 0
    L = 1
    while L < nsteps:
        d, n = dts[L], 1
        while L + n < nsteps and dts[L + n] == d:
            n += 1
        wb.set_layer0(L, tab[L:])
        assert O.march(impl, wb, n, float(d), 4)[0] == 0
        L += n
    return wb.state


@pytest.mark.parametrize("name", ["coupled_flux_n21", "cfg1_sample16", "vardt_n64"])
def test_oracle_matches_reference_goldens_bitwise(name):
    g = load(name)
    got = march_table(g)
    for k in FIELDS:
        assert np.array_equal(got[k], g[f"ref_{k}"]), k


def test_oracle_cfg0_vs_reference_transcription_oracle_golden():
    g = load("cfg0_5000")
    got = march_table(g)
    err = max(float(np.max(np.abs(got[k] - g[f"ref_{k}"]))) for k in FIELDS)
    assert err < 1e-12


@pytest.mark.parametrize("name", ["building_one_zone", "building_ring3"])
def test_oracle_building_goldens_bitwise(name):
    g = load(name)
    w = workloads.zone_ring(n_zones=int(g["n_zones"]), walls_per_zone=int(g["walls_per_zone"]),
                            n_nodes=int(g["n_nodes"]), nsteps=int(g["nsteps"]))
    init = {k: g[f"init_{k}"] for k in FIELDS}
    init.update(zone_u=w.init["zone_u"], zone_v=w.init["zone_v"])
    b = O.Building(w.model, init)
    rc, _, passes = b.run("oracle", int(g["nsteps"]))
    assert rc == 0 and passes == int(g["passes"])
    for k in FIELDS:
        assert np.array_equal(b.state[k], g[f"ref_{k}"]), k
    assert np.array_equal(b.zu, g["ref_zone_u"]) and np.array_equal(b.zv, g["ref_zone_v"])
    assert b.s.t == float(g["ref_t"])


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def test_df_step_linear_printed_coefficients(orc):
    """test_wall.cpp:43-61 hand-evaluated values, and the golden vectors."""
    def step(prev, curr, lam):
        prev, curr = np.array(prev, float), np.array(curr, float)
        nxt = np.empty_like(curr)
        orc.orc_df_step_linear(len(curr), _p(prev), _p(curr), lam, _p(nxt))
        return nxt
    assert step([0.3, 9.9, 0.1], [0.0, 1.0, 2.0], 1.0)[1] == pytest.approx(1.0)
    assert np.allclose(step([3.25] * 5, [3.25] * 5, 0.7), 3.25, rtol=1e-15)
    assert step([0, 0, 0], [0, 1, 0], 0.5)[1] == pytest.approx(0.0)
    assert step([0.1, 0.2, 0.3], [0.4, 0.5, 0.6], 0.5)[1] == pytest.approx((1 / 3) * 0.2 + (1 / 3) * 1.0, rel=1e-15)
    g = load("df_step_linear")
    for lam in (0.1, 0.5, 1.0, 10.0, 100.0):
        assert np.array_equal(step(g["prev"], g["curr"], lam), g[f"next_{lam}"])


def _fields(n, up, uc, vp, vc):
    arrs = [np.ascontiguousarray(x, dtype=float) for x in (up, uc, vp, vc)]
    return arrs, O.Field(n, *map(_p, arrs), 0.0)


def test_coupled_step_matches_transcription_oracle(orc, ref):
    """test_wall.cpp:63-104: one coupled step vs the fixed-point transcription
    oracle (df_oracle.hpp) with unit coefficients, at 1e-12."""
    from paper_1703_10119_b200.api import Signal
    x = np.linspace(0, 1, 5)
    init = dict(u_prev=1 + 0.05 * np.sin(np.pi * x), u_curr=1 + 0.04 * np.sin(np.pi * x + 0.3),
                v_prev=1 + 0.08 * np.cos(np.pi * x), v_curr=1 + 0.07 * np.cos(np.pi * x + 0.2))
    groups = np.array([[1.0, 1.0, 0.1, 1.0]])
    biot = np.array([[[1.3, 2.0, 0.4], [0.5, 0.8, 0.1]]])
    attach = np.array([[[0, 0], [0, 1]]], dtype=np.int32)
    ch = [ChannelSpec(Signal.constant(1.02), Signal.constant(0.95), Signal.constant(0.05), Signal.constant(0.1)),
          ChannelSpec(Signal.constant(0.98), Signal.constant(1.05))]
    m = Model(5, 0.25, groups, biot, attach, channels=ch, dt=2e-3)
    tab = O.forcing_table(m, [0.0, 2e-3], 0)
    a = O.WallBatch(m, init, tab)
    assert O.march("oracle", a, 1, 2e-3)[0] == 0
    m2 = Model(5, 0.25, groups, biot, attach, channels=ch, dt=2e-3, coeff_kind="analytic_d",
               coeff_params=(0.0, 0.0, 0.0, 0.0))           # k_M* = 1: the unit StarFn
    b = O.WallBatch(m2, init, tab)
    assert O.march("ref", b, 1, 2e-3)[0] == 0
    for k in FIELDS:
        assert np.max(np.abs(a.state[k] - b.state[k])) < 1e-12


def test_uniform_equilibrium_is_fixed_point(orc):
    """test_wall.cpp:196-224 for the DF coupled/nonlinear, explicit and implicit
    steps: uniform state at the ambient stays put to 1e-12."""
    model, _ = workloads.batched_walls(n_walls=8, n_nodes=11, nsteps=3).model, None
    model.channels = [ChannelSpec(), ChannelSpec()]
    init = {k: np.ones(8 * 11) for k in FIELDS}
    for boot in ("implicit", "explicit"):
        out = oracle_run("oracle", model, init, 50, boot)
        for k in FIELDS:
            assert np.max(np.abs(out[k] - 1.0)) < 1e-12
    md = workloads.single_wall_d(nsteps=3).model
    md.channels = [ChannelSpec(), ChannelSpec()]
    out = oracle_run("oracle", md, {k: np.ones(101) for k in FIELDS}, 200, "explicit")
    for k in FIELDS:
        assert np.max(np.abs(out[k] - 1.0)) < 1e-12


def test_gamma_zero_decouples_onto_single_field_form(orc):
    """test_wall.cpp:171-194: with gamma = 0 the u update is df_step_linear."""
    rng = np.random.default_rng(7)
    n, dt, dx = 9, 3e-3, 1 / 8
    g = np.array([[0.4, 0.25, 2.0, 0.0]])
    m = Model(n, dx, g, np.zeros((1, 2, 3)), channels=[ChannelSpec()], dt=dt)
    init = {k: rng.uniform(0.9, 1.1, n) for k in FIELDS}
    tab = O.forcing_table(m, [0.0, dt], 0)
    a = O.WallBatch(m, init, tab)
    O.march("oracle", a, 1, dt)
    mu = 2.0 * 0.25 * dt / (dx * dx)
    expect = np.empty(n)
    orc.orc_df_step_linear(n, _p(init["u_prev"]), _p(init["u_curr"]), mu, _p(expect))
    assert np.allclose(a.state["u_curr"][1:-1], expect[1:-1], rtol=1e-14, atol=0)


def test_neumann_mean_conservation_and_boundedness(orc):
    """test_wall.cpp:226-272: zero Biot faces conserve the trapezoidal mean;
    DF stays inside the envelope across lambda decades."""
    n = 41
    x = np.linspace(0, 1, n)
    m = Model(n, 1 / 40, np.array([[0.1, 0.1, 1.0, 0.01]]), np.zeros((1, 2, 3)), channels=[ChannelSpec()])
    v0 = 1 + 0.1 * np.cos(np.pi * x)
    init = dict(u_prev=np.ones(n), u_curr=np.ones(n), v_prev=v0, v_curr=v0.copy())
    tab = O.forcing_table(m, np.arange(2001) * 1e-3, 0)
    a = O.WallBatch(m, init, tab)
    O.march("oracle", a, 2000, 1e-3)
    mean = lambda y: (0.5 * (y[0] + y[-1]) + y[1:-1].sum()) / (n - 1)
    assert mean(a.state["v_curr"]) == pytest.approx(mean(v0), rel=5e-3)
    assert abs(a.state["v_curr"][0] - mean(v0)) < 0.02
    for lam in (0.1, 1.0, 10.0, 100.0):
        prev = np.sin(np.pi * np.linspace(0, 1, 21))
        curr = prev.copy()
        for _ in range(10000):
            nxt = np.empty(21)
            orc.orc_df_step_linear(21, _p(prev), _p(curr), lam, _p(nxt))
            prev, curr = curr, nxt
        assert np.max(np.abs(curr)) <= 1.0 + 1e-6


def test_explicit_step_at_stability_boundary(orc):
    """test_wall.cpp:274-292: at nu dt/dx^2 = 1/2 the explicit step is the
    neighbour average."""
    n, dx = 5, 0.25
    arrs, f = _fields(n, np.zeros(n), [1.0, 2.0, 7.0, 3.0, 5.0], np.ones(n), np.ones(n))
    g = O.WallGroups if hasattr(O, "WallGroups") else None
    from paper_1703_10119_b200 import _abi as A
    p = A.WallGroups(1.0, 1.0, 0.0, 0.0)
    face = O.Face(0, 0, 0, 1, 1, 0, 0)
    orc.orc_euler_explicit_step(C.byref(f), dx, C.byref(p), None, C.byref(face), C.byref(face), 0.5 * dx * dx)
    uc = arrs[1]
    assert uc[1] == pytest.approx(4.0) and uc[2] == pytest.approx(2.5) and uc[3] == pytest.approx(6.0)
