"""K6 (k_ring_split.cuh: the march split along its dependency cone — zone air
and wall cones first, then every wall in registers with no barrier per step;
the default for 64/128-node walls), K4 (k_ring.cuh), K4r (k_ring_reg.cuh:
owned walls in registers, persistent prefetching CTAs, fast guard; knob 1)
and K5 (k_ring_pipe.cuh, by the tuning knob: S = 12, trimmed halo, named-
barrier hand-off, producer warp): the zone-ring building march temporally
blocked with halo zones, against the C oracle's whole-building run
(relative L-infinity <= 1e-10, zones included): zone counts that leave the
last CTA partial, rings smaller than the halo (local copies of one zone), a
chain without the wrap-around link, grids of 64/128/256 nodes, step counts
that are not multiples of S, and a guard failure inside a launch (the host
replays that launch's steps with the exact per-step path: same first failing
layer and wall as the oracle)."""
import numpy as np
import pytest

import oracle as O
from paper_1703_10119_b200 import Context, api, workloads

from .helpers import rel_linf

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _gpu(model, init, steps, grid_cap=0, kernel=0, depth=0):
    with Context(model) as ctx:
        ctx.set_state(**init)
        if grid_cap:
            ctx.set_tuning("ring_grid", grid_cap)
        if kernel:
            ctx.set_tuning("ring_kernel", kernel)
        if depth:
            ctx.set_tuning("ring_depth", depth)   # K6: cone launches (8 steps each) per walls launch
        ctx.profiling(True)
        st = ctx.bootstrap("implicit")
        ctx.advance(steps - 1)
        ctx.synchronize()
        stats = {s["name"]: s for s in ctx.kernel_stats()}
        out = ctx.get_state()
    return out, st, stats


def _oracle(model, init, steps, nthreads=1):
    b = O.Building(model, init)
    rc, fl, passes = b.run("oracle", steps, nthreads=nthreads)
    return b, rc, fl, passes


def _noisy(w, seed, amp=2e-3):
    rng = np.random.default_rng(seed)
    return {k: v + (amp * rng.standard_normal(v.size) if k in ("u_prev", "u_curr", "v_prev", "v_curr") else 0)
            for k, v in w.init.items()}


def _compare(got, b, n_zones):
    err = rel_linf(got, dict(b.state))
    zref = max(float(np.max(np.abs(b.zu[:n_zones]))), float(np.max(np.abs(b.zv[:n_zones]))))
    zerr = max(float(np.max(np.abs(got["zone_u"] - b.zu[:n_zones]))),
               float(np.max(np.abs(got["zone_v"] - b.zv[:n_zones])))) / zref
    return err, zerr


# K4r's persistent CTAs (one per SM) walk blocks b, b + grid, ... of B = 4
# zones; the next block's bulk/cp.async prefetch into the other staging
# parity, the mbarrier phase flip, load_cf(b + grid) and the staging reuse
# run only when a CTA owns more than one block.  The grid cap forces that in
# small rings: 42 zones = 11 blocks (the last one partial, 2 zones) over 3
# CTAs walk 4/4/3 blocks; 64 zones over 2 CTAs walk 8 blocks each.
@pytest.mark.parametrize("kernel,name,depth", [(0, "ring_walls", 0), (0, "ring_walls", 1), (0, "ring_walls", 3),
                                               (1, "ring_reg", 0), (3, "ring_pipe", 0)])
@pytest.mark.parametrize("n_zones,cap,steps", [(42, 3, 203), (64, 2, 160), (42, 1, 77), (13, 2, 96)])
def test_ring_reg_multi_block_per_cta(n_zones, cap, steps, kernel, name, depth):
    w = workloads.zone_ring(n_zones=n_zones, walls_per_zone=6, n_nodes=128, nsteps=steps)
    init = _noisy(w, n_zones + cap)
    got, st, stats = _gpu(w.model, init, steps, grid_cap=cap, kernel=kernel, depth=depth)
    assert stats.get(name, {}).get("launches", 0) > 0, stats.keys()
    assert "ring_tiled" not in stats                 # no guard hand-over: the kernel marched every launch
    if kernel == 0:
        # K6: one cone launch per 8 steps, one stub between the cone launches of a walls launch
        m = depth or 2
        walls, cones = stats["ring_walls"]["launches"], stats["ring_cone"]["launches"]
        assert walls == -(-(steps - 1) // (8 * m)) and cones == sum(
            -(-min(8 * m, steps - 1 - s0) // 8) for s0 in range(0, steps - 1, 8 * m))
        assert stats.get("ring_stub", {}).get("launches", 0) == cones - walls
    b, rc, _, passes = _oracle(w.model, init, steps, nthreads=O.threads())
    assert rc == 0 and st.subiterations == passes
    err, zerr = _compare(got, b, n_zones)
    print(n_zones, cap, steps, "rel L-inf", err, "zones", zerr)
    assert err <= TOL and zerr <= TOL


def test_ring_cfg3_full_ring_1000_steps():
    """configs[3] at its BASELINE shape: 8,192 zones x 6 walls x 128 nodes
    through K6 (the default), K4r (about 14 blocks per persistent CTA) and K5
    for 1,000 steps — bitwise equal to one another — against the oracle's
    building run (threaded, bitwise the serial one): relative L-infinity <=
    1e-10 over walls and zones."""
    steps = 1000
    w = workloads.zone_ring(n_zones=8192, walls_per_zone=6, n_nodes=128, nsteps=steps)
    init = _noisy(w, 8192)
    got, st, stats = _gpu(w.model, init, steps)
    assert stats.get("ring_walls", {}).get("launches", 0) > 0, stats.keys()
    assert "ring_tiled" not in stats and "ring_reg" not in stats
    got_r, _, stats_r = _gpu(w.model, init, steps, kernel=1)          # K4r on the same input
    assert stats_r.get("ring_reg", {}).get("launches", 0) > 0 and "ring_tiled" not in stats_r
    for depth in (1, 3):                                               # K6 with 8 and 24 steps per walls launch
        got_d, _, stats_d = _gpu(w.model, init, steps, depth=depth)
        assert stats_d.get("ring_walls", {}).get("launches", 0) > 0 and "ring_tiled" not in stats_d
        for k in ("u_prev", "u_curr", "v_prev", "v_curr", "zone_u", "zone_v"):
            assert np.array_equal(got[k], got_d[k]), (depth, k)
    got_p, _, stats_p = _gpu(w.model, init, steps, kernel=3)          # K5 on the same input
    assert stats_p.get("ring_pipe", {}).get("launches", 0) > 0
    for k in ("u_prev", "u_curr", "v_prev", "v_curr", "zone_u", "zone_v"):
        assert np.array_equal(got[k], got_r[k]), k                       # K6 == K4r bit for bit
        assert np.array_equal(got[k], got_p[k]), k                       # K5 == K4r bit for bit
    b, rc, _, passes = _oracle(w.model, init, steps, nthreads=O.threads())
    assert rc == 0 and st.subiterations == passes
    err, zerr = _compare(got, b, 8192)
    print("cfg3 8192 zones x 1000 steps: rel L-inf", err, "zones", zerr)
    assert err <= TOL and zerr <= TOL


@pytest.mark.parametrize("cap,kernel,name", [(0, 0, "ring_walls"), (0, 1, "ring_reg"), (5, 1, "ring_reg")])
def test_ring_64_zones_full_horizon(cap, kernel, name):
    """A 64-zone ring at configs[3]'s full 8e4 steps (80 h) through K6 and
    through K4r with the default grid (16 CTAs, one block each) and capped at
    5 CTAs."""
    steps = 80_000
    w = workloads.zone_ring(n_zones=64, walls_per_zone=6, n_nodes=128, nsteps=steps)
    init = _noisy(w, 64)
    got, st, stats = _gpu(w.model, init, steps, grid_cap=cap, kernel=kernel)
    assert stats.get(name, {}).get("launches", 0) > 0
    b, rc, _, passes = _oracle(w.model, init, steps, nthreads=O.threads())
    assert rc == 0 and st.subiterations == passes
    err, zerr = _compare(got, b, 64)
    print("64 zones x 8e4 steps cap", cap, "rel L-inf", err, "zones", zerr)
    assert err <= TOL and zerr <= TOL


@pytest.mark.parametrize("n_zones,wpz,n,steps", [(17, 6, 128, 203), (3, 6, 128, 100), (2, 4, 64, 150),
                                                  (5, 6, 256, 120), (40, 6, 128, 1000), (1, 6, 128, 60),
                                                  (17, 5, 128, 150)])   # odd W: a one-wall store in the last block
def test_ring_matches_oracle(n_zones, wpz, n, steps):
    w = workloads.zone_ring(n_zones=n_zones, walls_per_zone=wpz, n_nodes=n, nsteps=steps)
    rng = np.random.default_rng(n_zones)
    init = {k: v + (2e-3 * rng.standard_normal(v.size) if k in ("u_prev", "u_curr", "v_prev", "v_curr") else 0)
            for k, v in w.init.items()}
    got, st, stats = _gpu(w.model, init, steps)
    kern = "ring_walls" if n <= 128 else "ring_tiled"
    assert stats.get(kern, {}).get("launches", 0) > 0, stats.keys()
    b, rc, _, passes = _oracle(w.model, init, steps)
    assert rc == 0 and st.subiterations == passes
    err = rel_linf(got, dict(b.state))
    zerr = max(float(np.max(np.abs(got["zone_u"] - b.zu[:n_zones]))),
               float(np.max(np.abs(got["zone_v"] - b.zv[:n_zones]))))
    print(n_zones, wpz, n, steps, "rel L-inf", err, "zone abs", zerr)
    assert err <= TOL and zerr <= TOL


def test_ring_chain_without_wrap():
    w = workloads.zone_ring(n_zones=12, walls_per_zone=6, n_nodes=128, nsteps=300)
    zs = w.model.zones
    zs[0].interzone = [l for l in zs[0].interzone if l[0] == 1]
    zs[-1].interzone = [l for l in zs[-1].interzone if l[0] == len(zs) - 2]
    got, st, stats = _gpu(w.model, w.init, 300)
    assert stats.get("ring_walls", {}).get("launches", 0) > 0
    b, rc, _, _ = _oracle(w.model, w.init, 300)
    assert rc == 0
    assert rel_linf(got, dict(b.state)) <= TOL
    assert float(np.max(np.abs(got["zone_u"] - b.zu[:12]))) <= TOL


def test_ring_guard_replay():
    """A norm the forced march crosses mid-run (inside a K4 launch): first
    failing layer and lowest failing wall exactly as the oracle's
    check_bounded."""
    w = workloads.zone_ring(n_zones=9, walls_per_zone=6, n_nodes=128, nsteps=400)
    b, rc, _, _ = _oracle(w.model, w.init, 400)
    assert rc == 0
    peak = max(np.abs(b.state[k]).max() for k in ("u_curr", "v_curr"))
    w.model.divergence_norm = 1.0 + 0.5 * (float(peak) - 1.0)   # the outdoor forcing lifts v steadily
    b, rc, fl, _ = _oracle(w.model, w.init, 400)
    assert rc == api.A.HYG_EDIVERGED and 20 < fl < 390, fl
    with Context(w.model) as ctx:
        ctx.set_state(**w.init)
        ctx.bootstrap("implicit")
        ctx.profiling(True)
        with pytest.raises(api.NumericalError) as ei:
            ctx.advance(399)
        ctx.synchronize()
        assert any(s["name"] == "ring_tiled" for s in ctx.kernel_stats())
    assert ei.value.layer == fl and ei.value.wall == b.fail_wall, (ei.value.layer, fl, ei.value.wall, b.fail_wall)


@pytest.mark.parametrize("kernel,name", [(0, "ring_walls"), (1, "ring_reg")])
def test_ring_reg_fast_guard_hands_over_to_k4(kernel, name):
    """Values of 2 and above (inside a norm of 1000) trip the fast guard of K6
    / K4r in the first launch; K4 replays from that launch's input with its
    exact guard and the march matches the oracle."""
    w = workloads.zone_ring(n_zones=20, walls_per_zone=6, n_nodes=128, nsteps=120)
    init = {k: v.copy() for k, v in w.init.items()}
    for k in ("u_prev", "u_curr"):
        init[k][5 * 128 + 40: 5 * 128 + 60] += 1.5          # wall 5, interior nodes
    got, st, stats = _gpu(w.model, init, 120, kernel=kernel)
    assert stats.get(name, {}).get("launches", 0) > 0 and stats.get("ring_tiled", {}).get("launches", 0) > 0
    b, rc, _, _ = _oracle(w.model, init, 120)
    assert rc == 0
    assert rel_linf(got, dict(b.state)) <= TOL
    assert float(np.max(np.abs(got["zone_u"] - b.zu[:20]))) <= TOL
