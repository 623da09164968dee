"""Material walls, mixed material/constant buildings, zone radiation and the
implicit start of nonlinear walls on the CUDA path (k_material.cuh), against
the C oracle's whole-building run (step_implicit start + step_explicit DF
steps, building.cpp:152-268; the oracle is pinned bitwise to the reference in
tests/test_oracle_material.py).

Tolerance: relative L-infinity <= 1e-10 over all fields and both layers.  The
default device evaluation uses table-driven exp/log and reciprocal quotients
(hyg_material.cuh evaluate_fast, a few ulp per coefficient); the exact mode
(HYG_TUNE_MATERIAL_EXACT) the accurate exp/log/pow of hyg_crmath.cuh with the
reference's expressions and IEEE divisions.  Neither is bit-identical to
glibc; the measured gap is ~1e-14 after 1000 steps, and both modes are
checked at the reference fixture's 8e4-step horizon below.  Domain errors
must match exactly (wall, node / half node, layer)."""
import numpy as np
import pytest

import oracle as O
from paper_1703_10119_b200 import Context, api, workloads

from .helpers import FIELDS, rel_linf

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _oracle(w, nsteps, init=None, with_bootstrap=True):
    b = O.Building(w.model, init or w.init)
    rc, fl, passes = b.run("oracle", nsteps, with_bootstrap)
    out = {k: b.state[k] for k in FIELDS}
    out.update(zone_u=b.zu[:len(w.model.zones)], zone_v=b.zv[:len(w.model.zones)])
    return rc, fl, passes, out


def _gpu(w, nsteps, init=None, boot="implicit", exact=False):
    with Context(w.model) as ctx:
        if exact:
            ctx.set_tuning("material_exact", 1)
        ctx.set_state(**(init or w.init))
        st = ctx.bootstrap(boot)
        ctx.advance(nsteps - 1)
        out = ctx.get_state()
        out["passes"] = st.subiterations if st is not None else None
    return out


@pytest.mark.parametrize("exact", [False, True])
def test_material_walls_parity(exact):
    w = workloads.material_walls(n_walls=32, n_nodes=51)
    rc, _, passes, ref = _oracle(w, 1000)
    assert rc == 0
    got = _gpu(w, 1000, exact=exact)
    err = rel_linf(got, ref)
    print("material walls exact" if exact else "material walls", "rel L-inf", err)
    assert err <= TOL
    assert np.ptp(ref["v_curr"]) > 1e-3


@pytest.mark.parametrize("exact", [False, True])
def test_material_walls_long_horizon(exact):
    """8e4 steps (the reference fixtures' 80 h) on 4 material walls, both modes."""
    w = workloads.material_walls(n_walls=4, n_nodes=101, nsteps=80_000)
    rc, _, passes, ref = _oracle(w, 80_000)
    assert rc == 0
    got = _gpu(w, 80_000, exact=exact)
    err = rel_linf(got, ref)
    print("material walls 8e4 steps", "exact" if exact else "fast", "rel L-inf", err)
    assert err <= TOL


@pytest.mark.parametrize("n_zones,mixed,radiation", [(1, False, True), (2, True, True), (3, False, False)])
def test_material_building_parity(n_zones, mixed, radiation):
    w = workloads.material_building(n_zones=n_zones, n_nodes=41, mixed=mixed, radiation=radiation)
    rc, _, passes, ref = _oracle(w, 1000)
    assert rc == 0
    got = _gpu(w, 1000, exact=n_zones == 2)
    err = rel_linf(got, ref, FIELDS + ("zone_u", "zone_v"))
    print("material building rel L-inf", err)
    assert err <= TOL


def test_radiation_moves_the_surfaces():
    """Radiation on/off must make a measurable difference (the term is live)."""
    a = _gpu(workloads.material_building(n_zones=2, n_nodes=41, radiation=True), 300)
    b = _gpu(workloads.material_building(n_zones=2, n_nodes=41, radiation=False), 300)
    assert np.abs(a["u_curr"] - b["u_curr"]).max() > 1e-9


@pytest.mark.parametrize("wall,node,field,value", [(2, 7, "v_curr", 2.1), (5, 0, "u_curr", 1.2),
                                                   (1, 40, "v_curr", 0.001)])
def test_material_domain_error(wall, node, field, value):
    w = workloads.material_building(n_zones=2, n_nodes=41)
    init = {k: np.array(v, dtype=np.float64, copy=True) for k, v in w.init.items()}
    init[field][wall * 41 + node] = value
    rc, fl, _, _ = _oracle(w, 3, init, with_bootstrap=False)
    ow, on, oh = O.Building.domain("oracle")
    assert rc == api.A.HYG_EDOMAIN
    with Context(w.model) as ctx:
        ctx.set_state(**init)
        with pytest.raises(api.DomainError) as ei:
            ctx.advance(3)
        e = ei.value
        assert (e.wall, e.node, e.half, e.layer) == (ow, on, oh, fl) == (wall, node, False, 1)
        # the failing step never ran: the state is still layer 0
        st = ctx.get_state()
        assert st["layer"] == 0
        assert np.array_equal(st["v_curr"], init["v_curr"]) and np.array_equal(st["u_curr"], init["u_curr"])


def test_material_domain_error_half_node():
    """Two neighbouring nodes inside the box whose midpoint state is outside
    it: the node table passes and the half node j+1/2 fails."""
    w = workloads.material_building(n_zones=1, n_nodes=41)
    init = {k: np.array(v, dtype=np.float64, copy=True) for k, v in w.init.items()}
    # both nodes at phi = 0.9895 but at different temperatures: P_s(T) is
    # convex, so the midpoint state (mean T, mean P_v) has phi > 0.99
    c = 3 * 41 + 20
    P_vi = w.model.P_vi
    for cell, u in ((c, 1.0), (c + 1, 0.9665)):
        init["u_curr"][cell] = u
        init["v_curr"][cell] = 0.9895 * api.saturation_pressure(u * 293.15) / P_vi
    rc, fl, _, _ = _oracle(w, 2, init, with_bootstrap=False)
    expect = O.Building.domain("oracle")
    assert rc == api.A.HYG_EDOMAIN
    with Context(w.model) as ctx:
        ctx.set_state(**init)
        with pytest.raises(api.DomainError) as ei:
            ctx.advance(2)
    assert (ei.value.wall, ei.value.node, ei.value.half) == expect == (3, 20, True)


def test_analytic_walls_implicit_start():
    """The d(v) functor through the table pass: implicit starting step + DF."""
    w = workloads.single_wall_d(nsteps=600)
    m = w.model
    rc, _, _, ref = _oracle(w, 600)
    assert rc == 0
    got = _gpu(w, 600, boot="implicit")
    err = rel_linf(got, ref)
    print("analytic implicit start rel L-inf", err)
    assert err <= TOL


def test_run_scheme_euler_implicit_matches_oracle():
    """hyg_run_scheme with the Euler-implicit scheme (step_implicit every
    step, building.cpp:327-331) on a material building with radiation: the
    state and SimulationResult's subiteration counters as the oracle's march
    of orc_step_implicit."""
    import ctypes as C
    w = workloads.material_building(n_zones=2, n_nodes=41, dt=1e-2)
    w.model.eta_factor = 1e-3
    b = O.Building(w.model, w.init)
    lib = O.oracle_lib()
    passes = []
    for _ in range(40):
        p, r = C.c_int(0), C.c_double(0)
        assert lib.orc_step_implicit(C.byref(b.desc), C.byref(b.s), w.model.eta_factor * w.model.dt,
                                     w.model.max_subiters, C.byref(p), C.byref(r)) == 0
        passes.append(p.value)
    with Context(w.model) as ctx:
        ctx.set_state(**w.init)
        rep = ctx.run_scheme("euler-implicit", horizon=40 * w.model.dt)
        got = ctx.get_state()
    assert rep.steps == 40 and rep.max_subiters_seen == max(passes)
    assert rep.mean_subiters == sum(passes) / 40
    err = rel_linf(got, dict(b.state))
    print("euler-implicit rel L-inf", err, "passes", passes[:5])
    assert err <= TOL
