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
