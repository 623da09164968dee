"""Shared helpers for the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

import oracle as O
from paper_1703_10119_b200 import workloads
from paper_1703_10119_b200.api import ChannelSpec, Model, Signal

FIELDS = ("u_prev", "u_curr", "v_prev", "v_curr")


def rel_linf(a: dict, b: dict, keys=FIELDS) -> float:
    """||a - b||_inf / ||b||_inf over all fields (SURVEY.md §8 definition)."""
    num = max(float(np.max(np.abs(np.asarray(a[k]) - np.asarray(b[k])))) for k in keys)
    den = max(float(np.max(np.abs(np.asarray(b[k])))) for k in keys)
    return num / den


def random_walls(n_walls, n_nodes, seed=0, flux=False, channels=2, dt=1e-3):
    """Random constant-coefficient walls spanning the cfg1 group ranges, with
    sinusoidal ambient channels (and imposed fluxes when flux=True)."""
    rng = np.random.default_rng(seed)
    lu = lambda lo, hi, n: np.exp(rng.uniform(np.log(lo), np.log(hi), n))
    groups = np.stack([lu(3.7e-5, 0.35, n_walls), lu(0.018, 1.4, n_walls), lu(1.1e-3, 10.4, n_walls),
                       lu(1.7e-5, 6.6e-3, n_walls)], axis=1)
    biot = np.empty((n_walls, 2, 3))
    biot[:, 0] = np.stack([lu(0.5, 2e4, n_walls), lu(0.5, 25, n_walls), lu(0.01, 2.0, n_walls)], axis=1)
    biot[:, 1] = np.stack([lu(0.1, 3e3, n_walls), lu(0.4, 8, n_walls), lu(0.01, 0.3, n_walls)], axis=1)
    attach = np.zeros((n_walls, 2, 2), dtype=np.int32)
    attach[:, 0, 1] = rng.integers(0, channels, n_walls)
    attach[:, 1, 1] = rng.integers(0, channels, n_walls)
    chans = []
    for c in range(channels):
        chans.append(ChannelSpec(
            u_inf=Signal.sin_squared(1.0, -0.02 * (c + 1), 24.0),
            v_inf=Signal.sinusoid(1.0, 0.06 * (c + 1), 24.0 / (c + 1), 0.5 * c),
            g_inf=Signal.sinusoid(0.0, 0.01, 6.0) if flux else Signal.constant(0.0),
            q_inf=Signal.sinusoid(0.0, 0.02, 12.0, 1.0) if flux else Signal.constant(0.0)))
    model = Model(n_nodes, 1.0 / (n_nodes - 1), groups, biot, attach, channels=chans, dt=dt)
    u0 = 1.0 + rng.normal(0, 0.01, n_walls * n_nodes)
    v0 = 1.0 + rng.normal(0, 0.01, n_walls * n_nodes)
    init = dict(u_prev=u0.copy(), u_curr=u0, v_prev=v0.copy(), v_curr=v0)
    return model, init


def oracle_run(impl, model, init, nsteps, boot, tables=None, dt=None, nthreads=None, dt_schedule=None):
    """Start step + (nsteps-1) DF steps on the CPU checker; returns the state dict."""
    dt = dt or model.dt
    nthreads = nthreads or O.threads()
    if dt_schedule:
        dts = np.concatenate([np.full(n, d) for n, d in dt_schedule])[:nsteps]
    else:
        dts = np.full(nsteps, dt)
    times = workloads.accumulate_times(dts)
    tab = O.forcing_table(model, times, 0, tables or {})
    wb = O.WallBatch(model, init, tab)
    L = 0
    if boot != "none":       # "none": DF straight from the two given layers
        rc = O.bootstrap(impl, wb, boot, dts[0], eta=model.eta_factor * dts[0], max_subiters=model.max_subiters,
                         nthreads=nthreads)
        assert rc == 0, rc
        L = 1
    # constant-dt runs of the schedule
    while L < nsteps:
        d = dts[L]
        n = 1
        while L + n < nsteps and dts[L + n] == d:
            n += 1
        wb.set_layer0(L, tab[L:])
        if impl == "oracle" and model.n_walls == 1 and model.n_nodes >= 4096 and nthreads > 1:
            rc, fl, fw = O.march_long_mt(wb, n, float(d), nthreads)    # one long wall: nodes over threads
        else:
            rc, fl, fw = O.march(impl, wb, n, float(d), nthreads)
        assert rc == 0, (rc, fl, fw)
        L += n
    return {k: wb.state[k] for k in FIELDS}


def gpu_run(model, init, nsteps, boot, tables=None, dt_schedule=None):
    """The CUDA path through the C ABI: start step + DF steps; returns state dict."""
    from paper_1703_10119_b200 import Context
    with Context(model) as ctx:
        ctx.set_state(**init)
        for ch, (first, t) in (tables or {}).items():
            ctx.set_channel_table(ch, first, t)
        if dt_schedule:
            # the start uses the model dt (= first entry of the schedule)
            ctx.bootstrap(boot)
            left = nsteps - 1
            first = True
            for n, d in dt_schedule:
                n = n - 1 if first else n
                first = False
                n = min(n, left)
                if n > 0:
                    ctx.advance(n, d)
                left -= n
        elif boot == "none":
            ctx.advance(nsteps)
        else:
            ctx.bootstrap(boot)
            ctx.advance(nsteps - 1)
        out = ctx.get_state()
        out["launches"] = ctx.launches
    return out
