"""The threaded oracle building march (orc_run_mt, test infrastructure) used
as the checker of the full-size zone ring equals the serial orc_run (the
statement-for-statement restatement of run(), building.cpp:303-356) bit for
bit, including the guard's first failing layer and lowest failing wall."""
import numpy as np
import pytest

import oracle as O
from paper_1703_10119_b200 import workloads


def _noisy(w, seed):
    rng = np.random.default_rng(seed)
    return {k: v + (2e-3 * rng.standard_normal(v.size) if k in ("u_prev", "u_curr", "v_prev", "v_curr") else 0)
            for k, v in w.init.items()}


@pytest.mark.parametrize("n_zones,threads", [(40, 3), (7, 4), (2, 5)])
def test_run_mt_bitwise_serial(n_zones, threads):
    w = workloads.zone_ring(n_zones=n_zones, walls_per_zone=6, n_nodes=128, nsteps=250)
    init = _noisy(w, n_zones)
    a, b = O.Building(w.model, init), O.Building(w.model, init)
    ra = a.run("oracle", 250)
    rb = b.run("oracle", 250, nthreads=threads)
    assert ra == rb
    for k in a.state:
        assert np.array_equal(a.state[k], b.state[k]), k
    assert np.array_equal(a.zu, b.zu) and np.array_equal(a.zv, b.zv)
    assert a.s.t == b.s.t and a.s.layer == b.s.layer


def test_run_mt_guard_matches_serial():
    w = workloads.zone_ring(n_zones=9, walls_per_zone=6, n_nodes=128, nsteps=400)
    b = O.Building(w.model, w.init)
    assert b.run("oracle", 400)[0] == 0
    peak = max(np.abs(b.state[k]).max() for k in ("u_curr", "v_curr"))
    w.model.divergence_norm = 1.0 + 0.5 * (float(peak) - 1.0)
    a, c = O.Building(w.model, w.init), O.Building(w.model, w.init)
    ra, rc = a.run("oracle", 400), c.run("oracle", 400, nthreads=4)
    assert ra[0] != 0 and ra[:2] == rc[:2] and a.fail_wall == c.fail_wall
    for k in a.state:
        assert np.array_equal(a.state[k], c.state[k]), k


@pytest.mark.parametrize("n,steps,threads", [(5000, 60, 4), (4099, 17, 7), (70001, 9, 16)])
def test_long_wall_mt_bitwise_serial(n, steps, threads):
    """orc_march_long_mt (one long d(v) wall, nodes split over threads) equals
    the serial orc_df_step_nonlinear march bit for bit."""
    w = workloads.long_domain(n_nodes=n, nsteps=steps)
    times = workloads.accumulate_times(np.full(steps, w.model.dt))
    tab = O.forcing_table(w.model, times, 0, {})
    a, b = O.WallBatch(w.model, w.init, tab), O.WallBatch(w.model, w.init, tab)
    ra = O.march("oracle", a, steps, w.model.dt, 1)
    rb = O.march_long_mt(b, steps, w.model.dt, threads)
    assert ra[0] == 0 and rb[0] == 0
    for k in a.state:
        assert np.array_equal(a.state[k], b.state[k]), k


def test_long_wall_mt_guard():
    w = workloads.long_domain(n_nodes=6000, nsteps=40)
    w.model.divergence_norm = 1.0 + 1e-3         # the initial modes already exceed it
    times = workloads.accumulate_times(np.full(40, w.model.dt))
    tab = O.forcing_table(w.model, times, 0, {})
    a, b = O.WallBatch(w.model, w.init, tab), O.WallBatch(w.model, w.init, tab)
    ra = O.march("oracle", a, 40, w.model.dt, 1)
    rb = O.march_long_mt(b, 40, w.model.dt, 5)
    assert ra[0] == rb[0] != 0 and ra[1] == rb[1] == 1
