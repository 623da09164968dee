"""TEST INFRASTRUCTURE ONLY — a Context-like engine over the C oracle, so the
multi-GPU decomposition (paper_1703_10119_b200/shard.py) can be exercised on
CPU ranks with the gloo backend (tests/test_shard_gloo.py)."""
from __future__ import annotations

import ctypes as C
from types import SimpleNamespace

import numpy as np

import oracle as O
from paper_1703_10119_b200 import workloads
from paper_1703_10119_b200.api import NumericalError

FIELDS = ("u_prev", "u_curr", "v_prev", "v_curr")


class OracleEngine:
    def __init__(self, model):
        self.model = model
        self.n = model.n_nodes
        self.cells = model.n_walls * model.n_nodes
        self.state = {f: np.ones(self.cells) for f in FIELDS}
        nz = max(1, len(model.zones))
        self.zu, self.zv = np.ones(nz), np.ones(nz)
        self.t, self.layer = 0.0, 0
        self.own = (0, self.cells, 0, 1 << 30)
        self._reduce = None

    # -- state -----------------------------------------------------------------
    def set_state(self, u_prev, u_curr, v_prev, v_curr, zone_u=None, zone_v=None, t=0.0, layer=0):
        for f, a in zip(FIELDS, (u_prev, u_curr, v_prev, v_curr)):
            self.state[f] = np.ascontiguousarray(a, dtype=np.float64).copy()
        if zone_u is not None:
            self.zu = np.ascontiguousarray(zone_u, dtype=np.float64).copy()
            self.zv = np.ascontiguousarray(zone_v, dtype=np.float64).copy()
        self.t, self.layer = t, layer

    def get_cells(self, c0, n):
        return {f: self.state[f][c0:c0 + n].copy() for f in FIELDS}

    def set_cells(self, c0, values):
        for f in FIELDS:
            v = np.asarray(values[f])
            self.state[f][c0:c0 + v.size] = v

    def get_zones(self, z0, n):
        return self.zu[z0:z0 + n].copy(), self.zv[z0:z0 + n].copy()

    def set_zones(self, z0, zu, zv):
        self.zu[z0:z0 + len(zu)] = zu
        self.zv[z0:z0 + len(zv)] = zv

    def set_owned(self, c0, c1, z0=0, z1=1 << 30, reduce=None):
        self.own = (c0, c1, z0, z1)
        self._reduce = reduce

    # -- marching ----------------------------------------------------------------
    def _building(self):
        b = O.Building(self.model, {**self.state, "zone_u": self.zu, "zone_v": self.zv, "t": self.t,
                                    "layer": self.layer})
        return b

    def _take(self, b):
        for f in FIELDS:
            self.state[f] = b.state[f]
        self.zu, self.zv = b.zu, b.zv
        self.t, self.layer = b.s.t, b.s.layer

    def bootstrap(self, kind="implicit"):
        lib = O.oracle_lib()
        if self.model.zones:
            c0, c1, z0, z1 = self.own
            cb = O.REDUCE_FN(lambda user, x: float(self._reduce(x))) if self._reduce else None
            lib.orc_set_owned(c0 // self.n, c1 // self.n, z0, z1, C.cast(cb, C.c_void_p) if cb else None, None)
            b = self._building()
            passes, res = C.c_int(), C.c_double()
            try:
                rc = lib.orc_step_implicit(C.byref(b.desc), C.byref(b.s), self.model.eta_factor * self.model.dt,
                                           self.model.max_subiters, C.byref(passes), C.byref(res))
            finally:
                lib.orc_set_owned(0, 1 << 30, 0, 1 << 30, None, None)
            assert rc == 0, rc
            self._take(b)
            return SimpleNamespace(subiterations=passes.value)
        raise NotImplementedError("wall-only shards start from two given layers")

    def _times(self, rows, t0):
        out = np.empty(rows)
        t = t0
        for k in range(rows):
            out[k] = t
            t = t + self.model.dt
        return out

    def advance(self, k, dt=None):
        if self.model.zones:
            b = self._building()
            lib = O.oracle_lib()
            for _ in range(k):
                lib.orc_step_explicit(C.byref(b.desc), C.byref(b.s))
            self._take(b)
            self._guard()
            return
        times = self._times(k + 1, self.t)
        tab = O.forcing_table(self.model, times, self.layer)
        wb = O.WallBatch(self.model, self.state, tab, self.layer)
        rc, fl, fw = O.march("oracle", wb, k, self.model.dt, 1)
        for f in FIELDS:
            self.state[f] = wb.state[f]
        self.t, self.layer = times[-1], self.layer + k
        self._guard()

    def _guard(self):
        c0, c1, _, _ = self.own
        for f in ("u_curr", "v_curr"):
            x = self.state[f][c0:c1]
            if not np.all(np.abs(x) <= self.model.divergence_norm):
                st = SimpleNamespace(t_star=self.t, layer=self.layer, wall=-1)
                raise NumericalError("divergence", st)
