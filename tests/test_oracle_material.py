"""Material walls and zone radiation in the C
restatement, pinned bit-for-bit against the UNMODIFIED reference
(oracle/_ref): MaterialModel::evaluate on the host (the product library's
setup helper and the oracle), whole-building runs with material walls, mixed
material/constant walls and radiation links (implicit start + DF steps,
building.cpp:152-268), and the location of a strict domain error
(wall.cpp:99-126)."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_1703_10119_b200 import api, workloads

from .helpers import FIELDS


def test_material_evaluate_host_bitwise(ref):
    rng = np.random.default_rng(11)
    T = rng.uniform(270.0, 316.0, 4000)
    Ps = np.array([ref.ref_saturation_pressure(min(max(t, 273.2), 373.0)) for t in T])
    Pv = Ps * rng.uniform(0.0, 1.02, T.size)
    for t, pv in zip(T, Pv):
        for clamped in (False, True):
            r = O.Coeffs()
            if clamped:    # the reference's evaluate_clamped through star_clamped at T_i = P_vi = 1
                m = O.CoeffModel(kind=O.ORC_COEFF_MATERIAL, T_i=1.0, P_vi=1.0,
                                 reference=O.Coeffs(1, 1, 1, 1, 1, 1))
                rc_ref = ref.ref_material_star(C.byref(m), t, pv, 0, C.byref(r))
            else:
                rc_ref = ref.ref_material_evaluate(t, pv, C.byref(r))
            try:
                got = api.material_evaluate(t, pv, clamped)
                rc = 0
            except api.DomainError:
                rc = 4
            assert rc == rc_ref, (t, pv, clamped)
            if rc == 0:
                assert got == (r.c_M, r.k_M, r.c_TT, r.k_TT, r.c_TM, r.k_TM)


def _run_pair(w, nsteps, with_bootstrap=True, init=None):
    init = init or w.init
    a, b = O.Building(w.model, init), O.Building(w.model, init)
    ra = a.run("oracle", nsteps, with_bootstrap)
    rb = b.run("ref", nsteps, with_bootstrap)
    return a, b, ra, rb


@pytest.mark.parametrize("n_zones,mixed,radiation", [(1, False, True), (2, False, True), (3, True, True),
                                                      (3, False, False)])
def test_material_building_bitwise(ref, n_zones, mixed, radiation):
    w = workloads.material_building(n_zones=n_zones, n_nodes=41, mixed=mixed, radiation=radiation)
    a, b, ra, rb = _run_pair(w, 300)
    assert ra == rb and ra[0] == 0, (ra, rb)
    assert ra[2] >= 2                                    # the joint fixed point iterated
    for k in FIELDS:
        assert np.array_equal(a.state[k], b.state[k]), k
    assert np.array_equal(a.zu, b.zu) and np.array_equal(a.zv, b.zv)
    # the material walls really are nonlinear and radiation moved the surfaces
    assert np.ptp(a.state["v_curr"]) > 1e-4


def test_material_walls_batch_bitwise(ref):
    w = workloads.material_walls(n_walls=6, n_nodes=31)
    times = workloads.accumulate_times(np.full(200, w.model.dt))
    tab = O.forcing_table(w.model, times, 0)
    a, b = O.WallBatch(w.model, w.init, tab), O.WallBatch(w.model, w.init, tab)
    assert O.bootstrap("oracle", a, "implicit", w.model.dt, eta=1e-5) == 0
    assert O.bootstrap("ref", b, "implicit", w.model.dt, eta=1e-5) == 0
    a.set_layer0(1, tab[1:])
    b.set_layer0(1, tab[1:])
    assert O.march("oracle", a, 199, w.model.dt, 2) == O.march("ref", b, 199, w.model.dt, 2) == (0, -1, -1)
    for k in FIELDS:
        assert np.array_equal(a.state[k], b.state[k]), k


@pytest.mark.parametrize("wall,node,field,value", [(2, 7, "v_curr", 2.1), (5, 0, "u_curr", 1.2),
                                                   (1, 40, "v_curr", 0.001)])
def test_material_domain_error_location(ref, wall, node, field, value):
    """A layer-n state outside the box fails the next DF step at the lowest
    failing wall, at the first failing node (nodes before half nodes)."""
    w = workloads.material_building(n_zones=2, n_nodes=41)
    init = {k: np.array(v, dtype=np.float64, copy=True) for k, v in w.init.items()}
    init[field][wall * 41 + node] = value
    a, b, ra, rb = _run_pair(w, 3, with_bootstrap=False, init=init)
    assert ra[0] == rb[0] == api.A.HYG_EDOMAIN
    assert ra[1] == rb[1] == 1
    assert O.Building.domain("oracle") == O.Building.domain("ref")
    dw, dn, half = O.Building.domain("ref")
    assert dw == wall and dn == node and not half


def test_material_domain_error_half_node(ref):
    """Both nodes at phi = 0.9895 at different temperatures: P_s is convex, so
    the midpoint state leaves the box and the half node j+1/2 fails."""
    w = workloads.material_building(n_zones=1, n_nodes=41)
    init = {k: np.array(v, dtype=np.float64, copy=True) for k, v in w.init.items()}
    c = 3 * 41 + 20
    for cell, u in ((c, 1.0), (c + 1, 0.9665)):
        init["u_curr"][cell] = u
        init["v_curr"][cell] = 0.9895 * api.saturation_pressure(u * 293.15) / w.model.P_vi
    _, _, ra, rb = _run_pair(w, 2, with_bootstrap=False, init=init)
    assert ra[:2] == rb[:2] == (api.A.HYG_EDOMAIN, 1)
    assert O.Building.domain("oracle") == O.Building.domain("ref") == (3, 20, True)
