"""Edge cases of the CUDA path against the oracle (relative L-infinity <=
1e-10): the smallest grid the reference accepts (Grid1D n = 3, wall.cpp:14),
a single wall and wall counts that leave the last CTA partial on every fused
grid, step counts straddling the forcing chunk (128 rows) and the K1 segment
(4,096 steps), zero-step calls, a long general-path wall, and argument
errors that must fail loudly instead of running."""
import numpy as np
import pytest

from paper_1703_10119_b200 import Context, api, workloads

from .helpers import FIELDS, gpu_run, oracle_run, random_walls, rel_linf

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.mark.parametrize("n_walls,n_nodes,steps", [(3, 3, 500), (1, 3, 200), (1, 256, 300), (1, 64, 129),
                                                   (37, 128, 4097), (1001, 64, 260), (5, 512, 300),
                                                   (2, 1000, 400), (9, 5, 1000)])
def test_shapes_and_step_counts(n_walls, n_nodes, steps):
    model, init = random_walls(n_walls, n_nodes, seed=n_walls * 7 + n_nodes, flux=True, channels=2)
    got = gpu_run(model, init, steps, "implicit")
    ref = oracle_run("oracle", model, init, steps, "implicit")
    err = rel_linf(got, ref)
    print(n_walls, n_nodes, steps, "rel L-inf", err)
    assert err <= TOL


def test_zero_steps_and_zero_horizon():
    model, init = random_walls(4, 128, seed=1)
    with Context(model) as ctx:
        ctx.set_state(**init)
        ctx.advance(0)
        st = ctx.get_state()
        assert st["layer"] == 0 and all(np.array_equal(st[k], init[k]) for k in FIELDS)
        frames = []
        ctx.run(0.0, cadence=0.5, frame=lambda layer, t, c: frames.append((layer, t)))
        assert frames == [(0, 0.0)]          # run(): the initial frame only (building.cpp:307-310)
        assert ctx.get_state()["layer"] == 0


def test_invalid_arguments_fail_loudly():
    model, init = random_walls(2, 64, seed=2)
    with Context(model) as ctx:
        with pytest.raises(api.InvalidArgument):
            ctx.set_state(init["u_prev"][:-1], init["u_curr"], init["v_prev"], init["v_curr"])
        with pytest.raises(api.HygroError):
            ctx.advance(-1)
        with pytest.raises(api.SchemaError):
            ctx.run(-1.0)
    bad = api.Model(2, 1.0, model.groups[:1], model.biot[:1], model.attach[:1], channels=model.channels)
    with pytest.raises(api.InvalidArgument):          # Grid1D: n >= 3 (wall.cpp:14)
        Context(bad)


def test_zone_ring_long_walls_general_path():
    """Zones with walls longer than the fused grids (n = 300): the per-step
    building kernel (k_building_step) against the oracle."""
    w = workloads.zone_ring(n_zones=5, walls_per_zone=3, n_nodes=300, nsteps=400)
    rng = np.random.default_rng(5)
    init = {k: v + (1e-3 * rng.standard_normal(v.size) if k in FIELDS else 0) for k, v in w.init.items()}
    import oracle as O
    with Context(w.model) as ctx:
        ctx.set_state(**init)
        ctx.bootstrap("implicit")
        ctx.advance(399)
        got = ctx.get_state()
    b = O.Building(w.model, init)
    rc, _, _ = b.run("oracle", 400)
    assert rc == 0
    assert rel_linf(got, dict(b.state)) <= TOL
    assert float(np.max(np.abs(got["zone_u"] - b.zu[:5]))) <= TOL
