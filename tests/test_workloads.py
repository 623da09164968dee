"""Seeded synthetic inputs match the BASELINE config shapes and the ranges
SURVEY.md §8d measured for them; layer times accumulate like the reference."""
import math

import numpy as np

from paper_1703_10119_b200 import workloads


def test_cfg1_group_ranges_match_survey():
    w = workloads.batched_walls(n_walls=4096, nsteps=10)
    g, b = w.model.groups, w.model.biot
    dt, dx = w.model.dt, w.model.dx
    lam = 2 * g[:, 0] * dt / dx ** 2
    mu = 2 * g[:, 1] * dt / dx ** 2
    # Fo_M 3.7e-5-0.35, Fo_TT 0.018-1.40, Fo_TM 1.1e-3-10.4,
    # gamma 1.7e-5-6.6e-3, Bi_TT(0) 1.25-25, Bi_TM(0) 0.10-2.0, Bi_M(0) 200-2e4, Bi_M(1) 30-3e3
    for col, lo, hi in ((g[:, 0], 3.7e-5, 0.35), (g[:, 1], 0.018, 1.40), (g[:, 2], 1.1e-3, 10.4),
                        (g[:, 3], 1.7e-5, 6.6e-3), (b[:, 0, 1], 1.25, 25.0), (b[:, 0, 2], 0.10, 2.0),
                        (b[:, 0, 0], 200.0, 2e4), (b[:, 1, 0], 30.0, 3e3), (lam, 0.005, 45.0), (mu, 2.4, 182.0)):
        assert col.min() >= lo * 0.9 and col.max() <= hi * 1.1, (lo, hi, col.min(), col.max())
    assert w.model.n_nodes == 256 and w.init["u_curr"].size == 4096 * 256
    dev = w.init["v_curr"] - 1.0
    assert abs(dev.std() - 0.01) < 5e-4 and np.array_equal(w.init["v_prev"], w.init["v_curr"])
    first, tab = w.tables[0]
    assert first == 0 and tab.shape == (11, 4) and tab[0, 0] == 1.0 and tab[0, 1] == 1.0


def test_layer_times_accumulate_like_the_reference():
    t = workloads.accumulate_times(np.full(100_000, 1e-3))
    acc = 0.0
    for _ in range(100_000):
        acc += 1e-3
    assert t[-1] == acc and t[-1] != 100.0        # sequential sum, not k*dt
    w = workloads.batched_walls(n_walls=4, variable_dt=True, precision="f32")
    assert [n for n, _ in w.dt_schedule] == [10_000] * 4 + [60_000]
    assert math.isclose(sum(n * d for n, d in w.dt_schedule), 1110.0)


def test_cfg0_cfg3_cfg4_shapes():
    w0 = workloads.single_wall_d(nsteps=10)
    assert w0.model.n_nodes == 101 and w0.model.dx == 0.01 and w0.boot == "explicit"
    assert w0.model.coeff_params == (0.91, 600.0, 10.0, 1.5)
    w3 = workloads.zone_ring(n_zones=32, nsteps=10)
    assert w3.model.n_walls == 32 * 6 and len(w3.model.zones) == 32
    peers = sorted(p for p, *_ in w3.model.zones[0].interzone)
    assert peers == [1, 31]
    # theta_T = k_TT0 A t0 / (L kappa_TT0): north and south walls share A = 18 m2
    th = [l[5] for l in w3.model.zones[0].walls]
    assert math.isclose(th[0] / th[1], 0.294 / 0.841, rel_tol=1e-12)
    w4 = workloads.long_domain(n_nodes=1 << 20, nsteps=10)
    dev = w4.init["v_curr"] - 1.0
    assert abs(dev).max() < 0.3 and w4.boot == "none"
    # shortest wavelength >= 1024 nodes: the field is smooth on the grid
    assert np.abs(np.diff(w4.init["v_curr"])).max() < 0.3 * 2 * math.pi / 1024 * 1.01
