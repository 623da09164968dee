"""Pin the C restatement (oracle/hygro_oracle.c) against the UNMODIFIED
reference compiled from /root/reference (oracle/_ref): bit-for-bit on the
coupled DF step, the nonlinear step with the reference's material model, the
explicit/implicit starting steps, the Euler-implicit march and the building
coupler (zones); within 1e-12 against the reference's own transcription
oracle (tests/support/df_oracle.hpp) for the analytic d(v) functor."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_1703_10119_b200 import workloads

from .helpers import FIELDS, random_walls


def _batch_pair(model, init, nsteps):
    times = workloads.accumulate_times(np.full(nsteps, model.dt))
    tab = O.forcing_table(model, times, 0)
    return O.WallBatch(model, init, tab), O.WallBatch(model, init, tab), tab


@pytest.mark.parametrize("n_nodes,flux", [(5, False), (21, True), (101, False), (256, True)])
def test_coupled_march_bitwise(ref, n_nodes, flux):
    model, init = random_walls(24, n_nodes, seed=n_nodes, flux=flux, channels=3)
    a, b, tab = _batch_pair(model, init, 400)
    for kind in ("implicit", "explicit"):
        a2, b2, _ = _batch_pair(model, init, 400)
        assert O.bootstrap("oracle", a2, kind, model.dt) == 0
        assert O.bootstrap("ref", b2, kind, model.dt) == 0
        for k in FIELDS:
            assert np.array_equal(a2.state[k], b2.state[k]), (kind, k)
    O.bootstrap("oracle", a, "implicit", model.dt)
    O.bootstrap("ref", b, "implicit", model.dt)
    a.set_layer0(1, tab[1:])
    b.set_layer0(1, tab[1:])
    assert O.march("oracle", a, 399, model.dt, 4) == (0, -1, -1)
    assert O.march("ref", b, 399, model.dt, 4) == (0, -1, -1)
    for k in FIELDS:
        assert np.array_equal(a.state[k], b.state[k]), k


def _material(model_T=293.15, phi=0.5):
    ref = O.Coeffs()
    lib = O.ref_lib()
    P_vi = phi * lib.ref_saturation_pressure(model_T)
    assert lib.ref_material_evaluate(model_T, P_vi, C.byref(ref)) == 0
    m = O.CoeffModel()
    m.kind = O.ORC_COEFF_MATERIAL
    m.T_i, m.P_vi, m.reference = model_T, P_vi, ref
    return m


def test_material_model_bitwise(ref, orc):
    """materials.cpp:91-121 incl. the admissible box (domain_error)."""
    P_vi = 0.5 * ref.ref_saturation_pressure(293.15)
    for T in np.linspace(270.0, 316.0, 13):
        for phi in np.linspace(0.005, 1.0, 17):
            a, b = O.Coeffs(), O.Coeffs()
            ra = orc.orc_material_evaluate(T, phi * orc.orc_saturation_pressure(T), C.byref(a))
            rb = ref.ref_material_evaluate(T, phi * orc.orc_saturation_pressure(T), C.byref(b))
            assert ra == rb
            if ra == 0:
                assert bytes(a) == bytes(b)
    m = _material()
    for u, v in [(1.0, 1.0), (1.02, 1.4), (0.95, 0.3), (1.2, 1.9), (1.0, 2.5)]:
        for strict in (1, 0):
            a, b = O.Coeffs(), O.Coeffs()
            ra = orc.orc_star(C.byref(m), u, v, strict, C.byref(a))
            rb = ref.ref_material_star(C.byref(m), u, v, strict, C.byref(b))
            assert ra == rb
            if ra == 0:
                assert bytes(a) == bytes(b)


def test_nonlinear_material_march_bitwise(ref, orc):
    """df_step_nonlinear with the load-bearing material (wall_nonlinear.json shape)."""
    m = _material()
    g, bi = [], []
    import paper_1703_10119_b200.api as api
    refset = (m.reference.c_M, m.reference.k_M, m.reference.c_TT, m.reference.k_TT, m.reference.c_TM, m.reference.k_TM)
    gg, bb = api.scale_wall(refset, 0.1, 25.0, 2e-7, 8.0, 3e-8)
    model = api.Model(101, 0.01, np.array([gg]), np.array([bb]),
                      channels=[api.ChannelSpec(v_inf=api.Signal.sinusoid(1.0, 0.4, 6.0)),
                                api.ChannelSpec(v_inf=api.Signal.sinusoid(1.0, 0.24, 24.0, 6.0))])
    model.attach[0, 1, 1] = 1
    init = {k: np.ones(101) for k in FIELDS}
    times = workloads.accumulate_times(np.full(301, 1e-3))
    tab = O.forcing_table(model, times, 0)
    a, b = O.WallBatch(model, init, tab), O.WallBatch(model, init, tab)
    fl, fw = C.c_int64(), C.c_int()
    assert orc.orc_march_nonlinear(C.byref(a.b), C.byref(m), 300, 1e-3, 1, C.byref(fl), C.byref(fw)) == 0
    assert ref.ref_march_nonlinear_material(C.byref(b.b), C.byref(m), 300, 1e-3, 1, C.byref(fl), C.byref(fw)) == 0
    for k in FIELDS:
        assert np.array_equal(a.state[k], b.state[k]), k
    # implicit march (fixed point with the material) bitwise too
    a, b = O.WallBatch(model, init, tab), O.WallBatch(model, init, tab)
    pa, pb = C.c_long(), C.c_long()
    orc.orc_march_implicit(C.byref(a.b), C.byref(m), 50, 1e-3, 1e-5, 100, 1, C.byref(pa))
    ref.ref_march_implicit(C.byref(b.b), C.byref(m), 50, 1e-3, 1e-5, 100, 1, C.byref(pb))
    assert pa.value == pb.value and pa.value > 50
    for k in FIELDS:
        assert np.array_equal(a.state[k], b.state[k]), k


def test_analytic_d_matches_reference_transcription_oracle(ref):
    """cfg0's d(v) functor: restatement of df_step_nonlinear (closed-form face
    rows) vs the reference's transcription oracle (200-iteration face fixed
    point, df_oracle.hpp:55-62,87-98)."""
    w = workloads.single_wall_d(nsteps=3000)
    a, b, tab = _batch_pair(w.model, w.init, 3000)
    O.bootstrap("oracle", a, "explicit", 1e-3)
    O.bootstrap("oracle", b, "explicit", 1e-3)
    a.set_layer0(1, tab[1:])
    b.set_layer0(1, tab[1:])
    assert O.march("oracle", a, 2999, 1e-3)[0] == 0
    assert O.march("ref", b, 2999, 1e-3)[0] == 0
    num = max(np.max(np.abs(a.state[k] - b.state[k])) for k in FIELDS)
    assert num < 1e-12


def test_implicit_march_constant_bitwise(ref):
    model, init = random_walls(16, 33, seed=5, flux=True)
    a, b, tab = _batch_pair(model, init, 60)
    pa = O.march_implicit("oracle", a, 50, model.dt)
    pb = O.march_implicit("ref", b, 50, model.dt)
    assert pa == pb == 16 * 50          # constant coefficients: one exact pass (wall.cpp:536)
    for k in FIELDS:
        assert np.array_equal(a.state[k], b.state[k]), k


def _building(n_zones, walls_per_zone, n_nodes):
    w = workloads.zone_ring(n_zones=n_zones, walls_per_zone=walls_per_zone, n_nodes=n_nodes, nsteps=10)
    return w.model, w.init


@pytest.mark.parametrize("n_zones,wpz,n", [(1, 4, 101), (5, 6, 16)])
def test_building_run_bitwise(ref, n_zones, wpz, n):
    """run(): implicit building bootstrap (step_implicit) + step_explicit loop
    + check_bounded, with zones, interzone ring and schedules."""
    model, init = _building(n_zones, wpz, n)
    init = dict(init)
    rng = np.random.default_rng(1)
    for k in FIELDS:
        init[k] = init[k] + 1e-3 * rng.standard_normal(init[k].size)
    a, b = O.Building(model, init), O.Building(model, init)
    ra = a.run("oracle", 400)
    rb = b.run("ref", 400)
    assert ra[0] == rb[0] == 0 and ra[2] == rb[2]        # same bootstrap sub-iterations
    for k in FIELDS:
        assert np.array_equal(a.state[k], b.state[k]), k
    assert np.array_equal(a.zu, b.zu) and np.array_equal(a.zv, b.zv)
    assert a.s.t == b.s.t


def test_reference_run_end_to_end(ref):
    """The reference's own run() (building.cpp:303-356) final frame equals the
    oracle's run over the same model."""
    model, init = _building(1, 4, 101)
    a = O.Building(model, init)
    assert a.run("oracle", 500)[0] == 0
    keep = []
    d = model.desc(keep)
    uc, vc = np.empty(4 * 101), np.empty(4 * 101)
    zu, zv = np.empty(1), np.empty(1)
    steps, tf = C.c_long(), C.c_double()
    p = lambda x: x.ctypes.data_as(C.POINTER(C.c_double))
    assert ref.ref_run(C.byref(d), 0.5, p(uc), p(vc), p(zu), p(zv), C.byref(steps), C.byref(tf)) == 0
    assert steps.value == 500
    assert np.array_equal(uc, a.state["u_curr"]) and np.array_equal(vc, a.state["v_curr"])
    assert np.array_equal(zu, a.zu) and np.array_equal(zv, a.zv)


def test_divergence_guard_agrees(ref):
    """check_bounded: first failing layer and lowest failing wall."""
    model, init = random_walls(8, 21, seed=2)
    model.divergence_norm = 1.012   # the ambient pushes some walls past it
    a, b, tab = _batch_pair(model, init, 3000)
    O.bootstrap("oracle", a, "implicit", model.dt)
    O.bootstrap("ref", b, "implicit", model.dt)
    a.set_layer0(1, tab[1:])
    b.set_layer0(1, tab[1:])
    ra = O.march("oracle", a, 2999, model.dt, 3)
    rb = O.march("ref", b, 2999, model.dt, 3)
    assert ra == rb and ra[0] == 3 and ra[1] > 1
