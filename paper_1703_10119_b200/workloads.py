"""Seeded synthetic workloads for the five BASELINE.json configs.

No public dataset is involved: every input is generated here
from a seed with the shapes, ranges and distributions BASELINE.json states;
the parameters BASELINE leaves open are fixed as in SURVEY.md Appendix A.
The same builder output drives the CUDA library, the C oracle and the
reference (tests/, bench.py), so all three see identical inputs.

Physical groups go through the library's own scaling (scale_wall /
scale_zone / ..., restating scaling.cpp) — the same path a user takes.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import api
from .api import ChannelSpec, Model, Signal, SourceSpec, ZoneSpec

T_I, PHI_I, T0 = 293.15, 0.5, 3600.0          # wall_nonlinear.json:3 scaling block
C_W, L_V = 4180.0, 2.5e6                        # PhysicalConstants materials.hpp:10,13
D_PARAMS = (0.91, 600.0, 10.0, 1.5)             # d(v) = 1 + 0.91 v + 600 exp(-10 (v-1.5)^2)


@dataclass
class Workload:
    name: str
    model: Model
    init: dict                      # u_prev, u_curr, v_prev, v_curr (+ zone_u, zone_v)
    nsteps: int                     # total steps incl. the starting step (run() convention)
    boot: str                       # "implicit" | "explicit"
    tables: dict = field(default_factory=dict)   # channel -> (first_layer, [L,4] ambient rows)
    dt_schedule: Optional[list] = None           # [(nsteps, dt)] for variable-dt runs (cfg2)
    notes: str = ""

    @property
    def cells(self) -> int:
        return self.model.n_walls * self.model.n_nodes


def accumulate_times(dts) -> np.ndarray:
    """Layer times t_k as the reference accumulates them (state.t += dt, building.cpp:185)."""
    out = np.empty(len(dts) + 1)
    t = 0.0
    out[0] = 0.0
    for i, d in enumerate(dts):
        t = t + d
        out[i + 1] = t
    return out


def _log_uniform(rng, lo, hi, n):
    return np.exp(rng.uniform(math.log(lo), math.log(hi), n))


def batched_walls(n_walls=65536, n_nodes=256, nsteps=100_000, dt=1e-3, seed=1, precision="f64",
                  variable_dt=False, A_T=0.02, A_phi=0.2) -> Workload:
    """configs[1] (and [2] with precision='f32', variable_dt=True).

    Per wall, log-uniform k_TT in [0.1,2] W/mK, d_m in [1e-12,1e-10] s, rho c in
    [5e5,2e6], c_m in [1e-4,1e-2]; k_M = d_m, k_TM = L_v d_m (materials.cpp:112),
    c_TM = c_w (T_i - 273.15) c_M (materials.cpp:111); L = 0.1 m; faces
    h_T/h_M = 25/2e-7 (x*=0, exterior) and 8/3e-8 (x*=1, interior air at the
    reference state).  Initial u, v = 1 + N(0, 0.01^2) iid, both layers equal.
    Exterior T = T_i (1 + A_T sin(2 pi t/24)), phi = phi_i (1 + A_phi sin(2 pi t/24)),
    v_inf = phi P_s(T) / P_vi.
    """
    rng = np.random.default_rng(seed)
    k_tt = _log_uniform(rng, 0.1, 2.0, n_walls)
    d_m = _log_uniform(rng, 1e-12, 1e-10, n_walls)
    rho_c = _log_uniform(rng, 5e5, 2e6, n_walls)
    c_m = _log_uniform(rng, 1e-4, 1e-2, n_walls)
    groups = np.empty((n_walls, 4))
    biot = np.empty((n_walls, 2, 3))
    for w in range(n_walls):
        ref = (c_m[w], d_m[w], rho_c[w], k_tt[w], C_W * (T_I - 273.15) * c_m[w], L_V * d_m[w])
        g, b = api.scale_wall(ref, 0.1, 25.0, 2e-7, 8.0, 3e-8, T_I, PHI_I, T0)
        groups[w] = g
        biot[w] = b
    attach = np.zeros((n_walls, 2, 2), dtype=np.int32)
    attach[:, 1, 1] = 1                      # face 1 -> channel 1 (interior, constant 1)
    init = {}
    u0 = 1.0 + rng.normal(0.0, 0.01, n_walls * n_nodes)
    v0 = 1.0 + rng.normal(0.0, 0.01, n_walls * n_nodes)
    init = dict(u_prev=u0.copy(), u_curr=u0, v_prev=v0.copy(), v_curr=v0)
    if variable_dt:
        # dt_k = dt0 * 2^min(floor(k/1e4), 4), k = step index (step 0 = start)
        sched = [(10_000, dt), (10_000, 2 * dt), (10_000, 4 * dt), (10_000, 8 * dt), (nsteps - 40_000, 16 * dt)]
        sched = [(n, d) for n, d in sched if n > 0]
        dts = np.concatenate([np.full(n, d) for n, d in sched])[:nsteps]
    else:
        sched = None
        dts = np.full(nsteps, dt)
    times = accumulate_times(dts)            # layers 0..nsteps
    p_vi = PHI_I * api.saturation_pressure(T_I)
    s = np.sin(2.0 * math.pi * times / 24.0)
    T = T_I * (1.0 + A_T * s)
    phi = PHI_I * (1.0 + A_phi * s)
    ps = np.exp(23.5771 - 4042.9 / (T - 37.58))          # saturation_pressure materials.cpp:39
    table = np.zeros((len(times), 4))
    table[:, 0] = T / T_I
    table[:, 1] = phi * ps / p_vi
    model = Model(n_nodes, 1.0 / (n_nodes - 1), groups, biot, attach,
                  channels=[ChannelSpec(), ChannelSpec()], dt=dt, precision=precision)
    name = "cfg2_batched_fp32_vardt" if variable_dt or precision == "f32" else "cfg1_batched_fp64"
    return Workload(name, model, init, nsteps, "implicit", tables={0: (0, table)}, dt_schedule=sched,
                    notes=f"{n_walls} walls x {n_nodes} nodes, seed {seed}")


def single_wall_d(nsteps=100_000, n_nodes=101, dt=1e-3, tau=24.0) -> Workload:
    """configs[0]: the reference's 1-D nonlinear moisture wall, k_M* = d(v).

    N=101 (dx=1e-2), Fo_M=0.1, c_M*=1, gamma=0 (u decoupled, stays 1),
    Bi_M 2 (x*=0) / 1 (x*=1), v_inf = 1 + 0.8 sin(2 pi t/tau) / 1, g_inf = 0,
    both initial layers 1, explicit starting step (Euler), then DF.
    """
    groups = np.array([[0.1, 0.1, 1.0, 0.0]])
    biot = np.array([[[2.0, 0.0, 0.0], [1.0, 0.0, 0.0]]])
    attach = np.array([[[0, 0], [0, 1]]], dtype=np.int32)
    ch = [ChannelSpec(v_inf=Signal.sinusoid(1.0, 0.8, tau)), ChannelSpec()]
    model = Model(n_nodes, 0.01, groups, biot, attach, channels=ch, dt=dt, coeff_kind="analytic_d",
                  coeff_params=D_PARAMS)
    one = np.ones(n_nodes)
    init = dict(u_prev=one.copy(), u_curr=one.copy(), v_prev=one.copy(), v_curr=one.copy())
    return Workload("cfg0_single_wall_d", model, init, nsteps, "explicit", notes=f"N={n_nodes}, tau={tau}")


def long_domain(n_nodes=1 << 26, nsteps=10_000, dt=1e-3, seed=4, modes=16) -> Workload:
    """configs[4]: one very long coupled wall, Grid1D{N, 1e-2}, k_M* = d(v).

    Initial u, v = 1 + sum_k a_k sin(2 pi m_k x / X + phi_k), X = (N-1) dx,
    a_k ~ U[-0.3/16, 0.3/16], m_k ~ U{1..2^16}, phi_k ~ U[0, 2 pi); both layers equal.
    North-wall groups of test_wall.cpp:144-148; Bi_M 2/1 with cfg0's v_inf;
    Bi_TT/Bi_TM 1.7/0.678 (x*=0), 2.72/0.101 (x*=1).  The DF march starts
    directly from the two equal initial layers (as test_wall.cpp:251-272 does):
    an Euler-explicit start at Fo_M dt/dx^2 d(v) ~ 50 kicks the face nodes
    into an odd-even mode that the frozen-coefficient DF then amplifies past
    divergence_norm within ~80 steps ("cfg4 start").
    """
    rng = np.random.default_rng(seed)
    dx = 1e-2
    X = (n_nodes - 1) * dx
    x = np.arange(n_nodes) * dx
    def field_():
        a = rng.uniform(-0.3 / modes, 0.3 / modes, modes)
        # shortest wavelength >= 1024 nodes at every N (2^16 modes at N = 2^26)
        m = rng.integers(1, max(1, (n_nodes - 1) // 1024), modes, endpoint=True)
        ph = rng.uniform(0.0, 2.0 * math.pi, modes)
        f = np.ones(n_nodes)
        for k in range(modes):
            f += a[k] * np.sin(2.0 * math.pi * m[k] * x / X + ph[k])
        return f
    u0, v0 = field_(), field_()
    groups = np.array([[0.116, 0.137, 3.76, 7.87e-3]])
    biot = np.array([[[2.0, 1.7, 0.678], [1.0, 2.72, 0.101]]])
    attach = np.array([[[0, 0], [0, 1]]], dtype=np.int32)
    ch = [ChannelSpec(v_inf=Signal.sinusoid(1.0, 0.8, 24.0)), ChannelSpec()]
    model = Model(n_nodes, dx, groups, biot, attach, channels=ch, dt=dt, coeff_kind="analytic_d",
                  coeff_params=D_PARAMS)
    init = dict(u_prev=u0.copy(), u_curr=u0, v_prev=v0.copy(), v_curr=v0)
    return Workload("cfg4_long_domain", model, init, nsteps, "none", notes=f"N={n_nodes}, seed {seed}")


# frozen coefficient sets of one_zone_linear.json:5-7 / test_building.cpp:13-15
SETS = {
    "north": (1.82e-2, 5.89e-9, 7.70e5, 2.94e-1, 1.52e3, 1.59e-2),
    "south": (1.18e-1, 2.92e-8, 1.28e6, 8.41e-1, 9.88e3, 2.96e-3),
    "east_west": (6.09e-2, 5.47e-9, 8.61e5, 3.87e-1, 5.09e3, 1.53e-2),
}
# (set, area, h_T exterior, h_M exterior) cycled N/S/E/W/E/W (one_zone_linear.json:14-43)
ZONE_WALLS = [("north", 18.0, 5.0, 2e-7), ("south", 18.0, 25.0, 8e-7), ("east_west", 9.0, 12.0, 4e-7),
              ("east_west", 9.0, 12.0, 4e-7), ("east_west", 9.0, 12.0, 4e-7), ("east_west", 9.0, 12.0, 4e-7)]


def zone_ring(n_zones=8192, walls_per_zone=6, n_nodes=128, nsteps=80_000, dt=1e-3, ach=0.5,
              inz_ach=0.5) -> Workload:
    """configs[3]: zones in a ring, each with 6 walls (exterior face 0, zone face 1).

    Zone air of one_zone_linear.json:44-59 (V=54 m3, rho 1, c_pa 1005, c_pv 1960,
    0.5 ach, the fixture moisture schedule, flux-consistent sign); ring
    neighbours i+-1 exchange air at `inz_ach` (scale_interzone).  Outdoor
    u = 1 - 0.02 sin^2(2 pi t/24), v = 1 + 0.06 sin(2 pi t/24).
    """
    V = 54.0
    zd = api.scale_zone(V, 1.0, 1005.0, 1960.0, ach, T_I, PHI_I, T0)
    g_inz, q_inz1, q_inz2 = api.scale_interzone(inz_ach, V, 1.0, 1005.0, 1960.0, T_I, PHI_I, T0)
    moist = Signal.schedule(6.9444444444e-6, [(6.0, 9.0, 1.1111111111e-4), (30.0, 33.0, 1.1111111111e-4),
                                              (54.0, 57.0, 1.1111111111e-4)])
    def scaled(sig, f):
        return Signal(sig.form, sig.base * f, sig.amplitude * f, sig.period, sig.phase,
                      tuple((a, b, x * f) for a, b, x in sig.windows))
    src = SourceSpec(g_o=scaled(moist, zd["g_o_per"]), q_o=scaled(moist, zd["q_o_per"]),
                     q_h=Signal.constant(0.0))
    out_u = Signal.sin_squared(1.0, -0.02, 24.0)
    out_v = Signal.sinusoid(1.0, 0.06, 24.0)
    nw = n_zones * walls_per_zone
    groups = np.empty((nw, 4))
    biot = np.empty((nw, 2, 3))
    attach = np.zeros((nw, 2, 2), dtype=np.int32)
    per_wall = []
    for i in range(walls_per_zone):
        name, area, hT, hM = ZONE_WALLS[i % len(ZONE_WALLS)]
        g, b = api.scale_wall(SETS[name], 0.1, hT, hM, 8.0, 3e-8, T_I, PHI_I, T0)
        th = api.attach_wall_to_zone(SETS[name], area, 0.1, V, 1.0, 1005.0, T_I, PHI_I, T0)
        per_wall.append((g, b, th))
    zones = []
    for z in range(n_zones):
        links = []
        for i in range(walls_per_zone):
            w = z * walls_per_zone + i
            g, b, th = per_wall[i]
            groups[w] = g
            biot[w] = b
            attach[w, 0] = (0, 0)
            attach[w, 1] = (1, z)
            links.append((w, 1, b[1][0], b[1][1], b[1][2], th[0], th[1]))
        inz = [((z - 1) % n_zones, g_inz, q_inz1, q_inz2), ((z + 1) % n_zones, g_inz, q_inz1, q_inz2)] \
            if n_zones > 1 else []
        zones.append(ZoneSpec(zd["kappa_a_tt1"], zd["g_v"], zd["q_v1"], zd["q_v2"], 0,
                              1, links, inz))
    ch = [ChannelSpec(u_inf=out_u, v_inf=out_v)]
    model = Model(n_nodes, 1.0 / (n_nodes - 1), groups, biot, attach, channels=ch, zones=zones,
                  zone_sources=[src], outdoor_u=out_u, outdoor_v=out_v, dt=dt, eta_factor=1e-6)
    cells = nw * n_nodes
    one = np.ones(cells)
    init = dict(u_prev=one.copy(), u_curr=one.copy(), v_prev=one.copy(), v_curr=one.copy(),
                zone_u=np.ones(n_zones), zone_v=np.ones(n_zones))
    return Workload("cfg3_zone_ring", model, init, nsteps, "implicit", notes=f"{n_zones} zones x {walls_per_zone} walls x {n_nodes}")


BUILDERS = {
    "cfg0": single_wall_d,
    "cfg1": batched_walls,
    "cfg2": lambda **kw: batched_walls(precision="f32", variable_dt=True, **kw),
    "cfg3": zone_ring,
    "cfg4": long_domain,
}


# ---- load-bearing material walls -----------------------
def material_reference(T_i=T_I, phi_i=PHI_I):
    """Reference set of the built-in material: evaluate(T_i, P_vi) (scenario.cpp:178)."""
    P_vi = phi_i * api.saturation_pressure(T_i)
    return P_vi, np.array(api.material_evaluate(T_i, P_vi))


def material_walls(n_walls=4096, n_nodes=101, nsteps=2000, dt=1e-3, seed=5) -> Workload:
    """Independent load-bearing material walls (CoefficientModel::material), both
    faces exterior: a humid side v = 1 + 0.3 sin(2 pi t/6) and an outdoor side
    v = 1 + 0.24 sin(2 pi (t-6)/24), u = 1 (shapes of a single-slab scenario);
    per-wall film coefficients log-uniform around a slab's values, humid side
    h_T in [15, 35], h_M in [8e-8, 2e-7], outdoor side h_T in [5, 12], h_M in
    [2e-8, 5e-8] (larger moisture films cool the outdoor face by evaporation
    until phi leaves the material box — a domain error in the reference too);
    L = 0.1 m, dx = 1/(n-1).  Strict evaluation in every DF step; implicit start."""
    rng = np.random.default_rng(seed)
    P_vi, ref = material_reference()
    groups = np.empty((n_walls, 4))
    biot = np.empty((n_walls, 2, 3))
    hT = np.stack([_log_uniform(rng, 15.0, 35.0, n_walls), _log_uniform(rng, 5.0, 12.0, n_walls)], axis=1)
    hM = np.stack([_log_uniform(rng, 8e-8, 2e-7, n_walls), _log_uniform(rng, 2e-8, 5e-8, n_walls)], axis=1)
    for w in range(n_walls):
        g, b = api.scale_wall(ref, 0.1, hT[w, 0], hM[w, 0], hT[w, 1], hM[w, 1], T_I, PHI_I, T0)
        groups[w], biot[w] = g, b
    attach = np.zeros((n_walls, 2, 2), dtype=np.int32)
    attach[:, 1, 1] = 1
    ch = [ChannelSpec(v_inf=Signal.sinusoid(1.0, 0.30, 6.0)),
          ChannelSpec(v_inf=Signal.sinusoid(1.0, 0.24, 24.0, 6.0))]
    model = Model(n_nodes, 1.0 / (n_nodes - 1), groups, biot, attach, channels=ch, dt=dt, eta_factor=1e-2,
                  coeff_kind="material", T_i=T_I, P_vi=P_vi, wall_reference=np.tile(ref, (n_walls, 1)))
    one = np.ones(n_walls * n_nodes)
    init = dict(u_prev=one.copy(), u_curr=one.copy(), v_prev=one.copy(), v_curr=one.copy())
    return Workload("material_walls", model, init, nsteps, "implicit",
                    notes=f"{n_walls} material walls x {n_nodes}")


def material_building(n_zones=2, n_nodes=101, nsteps=2000, dt=1e-3, mixed=False, radiation=True,
                      ach=0.5, inz_ach=0.3) -> Workload:
    """Zones in a ring, each bounded by three exterior load-bearing walls
    (areas 18/18/9 m2, h_T 5/25/12, h_M 2e-7/8e-7/4e-7 outside, 8/3e-8 inside)
    and one partition shared with the next zone (face 0 -> zone z, face 1 ->
    zone z+1; exterior when n_zones == 1).  Long-wave radiation between every
    ordered pair of a zone's walls (view factor 0.2, emissivity 0.5, 0.9 for
    the partition), exterior u = 1 - 0.02 sin^2(2 pi t/24), v = 1 + 0.06
    sin(2 pi t/24), q = 0.02 sin^2(2 pi t/24).  `mixed`: every exterior wall
    of odd zones keeps constant (linearised) coefficients, so both step kinds
    meet in one building (building.cpp:172-176)."""
    V = 54.0
    P_vi, ref = material_reference()
    zd = api.scale_zone(V, 1.0, 1005.0, 1960.0, ach, T_I, PHI_I, T0)
    g_inz, q_inz1, q_inz2 = api.scale_interzone(inz_ach, V, 1.0, 1005.0, 1960.0, T_I, PHI_I, T0)
    moist = Signal.schedule(6.9e-6, [(6.0, 9.0, 1.1e-4), (30.0, 33.0, 1.1e-4)])
    src = SourceSpec(g_o=Signal("constant", moist.base * zd["g_o_per"], 0.0, 1.0, 0.0,
                                tuple((a, b, x * zd["g_o_per"]) for a, b, x in moist.windows)),
                     q_o=Signal("constant", moist.base * zd["q_o_per"], 0.0, 1.0, 0.0,
                                tuple((a, b, x * zd["q_o_per"]) for a, b, x in moist.windows)))
    out_u, out_v = Signal.sin_squared(1.0, -0.02, 24.0), Signal.sinusoid(1.0, 0.06, 24.0)
    ext = [(18.0, 5.0, 2e-7), (18.0, 25.0, 8e-7), (9.0, 12.0, 4e-7)]
    wpz = len(ext) + 1
    nw = n_zones * wpz
    groups, biot = np.empty((nw, 4)), np.empty((nw, 2, 3))
    attach = np.zeros((nw, 2, 2), dtype=np.int32)
    material = np.ones(nw, dtype=bool)
    links = [[] for _ in range(n_zones)]
    for z in range(n_zones):
        for i, (area, hT, hM) in enumerate(ext):
            w = z * wpz + i
            groups[w], biot[w] = api.scale_wall(ref, 0.1, hT, hM, 8.0, 3e-8, T_I, PHI_I, T0)
            attach[w, 0], attach[w, 1] = (0, 0), (1, z)
            th = api.attach_wall_to_zone(ref, area, 0.1, V, 1.0, 1005.0, T_I, PHI_I, T0)
            links[z].append((w, 1, *biot[w, 1], *th))
            material[w] = not (mixed and z % 2 == 1)
        p = z * wpz + len(ext)                        # partition
        groups[p], biot[p] = api.scale_wall(ref, 0.1, 8.0, 3e-8, 8.0, 3e-8, T_I, PHI_I, T0)
        th = api.attach_wall_to_zone(ref, 9.0, 0.1, V, 1.0, 1005.0, T_I, PHI_I, T0)
        attach[p, 0] = (1, z)
        links[z].append((p, 0, *biot[p, 0], *th))
        if n_zones > 1:
            zn = (z + 1) % n_zones
            attach[p, 1] = (1, zn)
            links[zn].append((p, 1, *biot[p, 1], *th))
        else:
            attach[p, 1] = (0, 0)
    zones = []
    for z in range(n_zones):
        inz = ([((z - 1) % n_zones, g_inz, q_inz1, q_inz2), ((z + 1) % n_zones, g_inz, q_inz1, q_inz2)]
               if n_zones > 2 else ([((z + 1) % 2, g_inz, q_inz1, q_inz2)] if n_zones == 2 else []))
        rad = []
        if radiation:
            ws = [l[0] for l in links[z]]
            for r in ws:
                for e in ws:
                    if e != r:
                        rad.append((e, r, 0.2, 0.9 if e % wpz == len(ext) else 0.5))
        zones.append(ZoneSpec(zd["kappa_a_tt1"], zd["g_v"], zd["q_v1"], zd["q_v2"], 0, 1, links[z], inz, rad))
    ch = [ChannelSpec(u_inf=out_u, v_inf=out_v, q_inf=Signal.sin_squared(0.0, 0.02, 24.0))]
    model = Model(n_nodes, 1.0 / (n_nodes - 1), groups, biot, attach, channels=ch, zones=zones,
                  zone_sources=[src], outdoor_u=out_u, outdoor_v=out_v, dt=dt, eta_factor=1e-2,
                  coeff_kind="material", T_i=T_I, P_vi=P_vi, wall_reference=np.tile(ref, (nw, 1)),
                  wall_material=material, wall_thickness=np.full(nw, 0.1), wall_k_TT0=np.full(nw, ref[3]))
    one = np.ones(nw * n_nodes)
    init = dict(u_prev=one.copy(), u_curr=one.copy(), v_prev=one.copy(), v_curr=one.copy(),
                zone_u=np.ones(n_zones), zone_v=np.ones(n_zones))
    return Workload("material_building", model, init, nsteps, "implicit",
                    notes=f"{n_zones} zones x {wpz} material walls x {n_nodes}, radiation={radiation}")
