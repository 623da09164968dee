"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the CPU checkers.

  liboracle.so          plain-C restatement of the reference DF path (hygro_oracle.c)
  _ref/libhygro_ref.so  the unmodified reference compiled from /root/reference (ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs import this package, and only as the checker or the
timed CPU baseline — never on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path
from typing import Optional

import numpy as np

from paper_1703_10119_b200 import _abi as A

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libhygro_ref.so"


class Coeffs(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("c_M", "k_M", "c_TT", "k_TT", "c_TM", "k_TM")]


class Face(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("Bi_M", "Bi_TT", "Bi_TM", "u_inf", "v_inf", "g_inf", "q_inf")]


class Field(C.Structure):
    _fields_ = [("n", C.c_int), ("up", A.dp), ("uc", A.dp), ("vp", A.dp), ("vc", A.dp), ("t_star", C.c_double)]


ORC_COEFF_CONSTANT, ORC_COEFF_ANALYTIC_D, ORC_COEFF_MATERIAL = 0, 1, 2


class CoeffModel(C.Structure):
    _fields_ = [("kind", C.c_int), ("p", C.c_double * 4), ("T_i", C.c_double), ("P_vi", C.c_double),
                ("reference", Coeffs)]


class Batch(C.Structure):
    _fields_ = [("n_walls", C.c_int), ("n", C.c_int), ("dx", C.c_double), ("groups", C.POINTER(A.WallGroups)),
                ("biot", C.POINTER(A.FaceBiot)), ("chan", C.POINTER(C.c_int32)), ("n_channels", C.c_int),
                ("table", C.POINTER(A.Ambient)), ("layer0", C.c_int64), ("divergence_norm", C.c_double),
                ("up", A.dp), ("uc", A.dp), ("vp", A.dp), ("vc", A.dp)]


class BuildingState(C.Structure):
    _fields_ = [("up", A.dp), ("uc", A.dp), ("vp", A.dp), ("vc", A.dp), ("zu", A.dp), ("zv", A.dp),
                ("t", C.c_double), ("layer", C.c_int64)]


_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)
_BP = C.POINTER(Batch)
_MP = C.POINTER(CoeffModel)

_ORACLE_PROTOS = {
    "orc_star": (C.c_int, [_MP, C.c_double, C.c_double, C.c_int, C.POINTER(Coeffs)]),
    "orc_material_evaluate": (C.c_int, [C.c_double, C.c_double, C.POINTER(Coeffs)]),
    "orc_saturation_pressure": (C.c_double, [C.c_double]),
    "orc_signal": (C.c_double, [C.POINTER(A.Signal), C.c_double]),
    "orc_df_step_linear": (None, [C.c_int, A.dp, A.dp, C.c_double, A.dp]),
    "orc_df_step_coupled": (None, [C.POINTER(Field), C.c_double, C.POINTER(A.WallGroups), C.POINTER(Face),
                                   C.POINTER(Face), C.c_double]),
    "orc_df_step_nonlinear": (C.c_int, [C.POINTER(Field), C.c_double, C.POINTER(A.WallGroups), _MP,
                                        C.POINTER(Face), C.POINTER(Face), C.c_double]),
    "orc_euler_explicit_step": (None, [C.POINTER(Field), C.c_double, C.POINTER(A.WallGroups), _MP,
                                       C.POINTER(Face), C.POINTER(Face), C.c_double]),
    "orc_euler_implicit_step": (C.c_int, [C.POINTER(Field), C.c_double, C.POINTER(A.WallGroups), _MP,
                                          C.POINTER(Face), C.POINTER(Face), C.c_double, C.c_double, C.c_int,
                                          A.dp]),
    "orc_max_abs_field": (C.c_double, [C.POINTER(Field)]),
    "orc_march_coupled": (C.c_int, [_BP, C.c_int, C.c_double, C.c_int, _i64p, _ip]),
    "orc_march_nonlinear": (C.c_int, [_BP, _MP, C.c_int, C.c_double, C.c_int, _i64p, _ip]),
    "orc_bootstrap_batch": (C.c_int, [_BP, _MP, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int]),
    "orc_march_implicit": (C.c_int, [_BP, _MP, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                     C.POINTER(C.c_long)]),
    "orc_step_explicit": (C.c_int, [C.POINTER(A.ModelDesc), C.POINTER(BuildingState)]),
    "orc_step_implicit": (C.c_int, [C.POINTER(A.ModelDesc), C.POINTER(BuildingState), C.c_double, C.c_int,
                                    _ip, A.dp]),
    "orc_run": (C.c_int, [C.POINTER(A.ModelDesc), C.POINTER(BuildingState), C.c_int64, _i64p, _ip, _ip]),
    "orc_march_long_mt": (C.c_int, [_BP, _MP, C.c_int, C.c_double, C.c_int, _i64p]),
    "orc_run_mt": (C.c_int, [C.POINTER(A.ModelDesc), C.POINTER(BuildingState), C.c_int64, C.c_int, _i64p, _ip,
                             _ip]),
    "orc_set_owned": (None, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "orc_last_domain": (None, [_ip, _ip]),
    "orc_last_domain_wall": (C.c_int, []),
}

REDUCE_FN = C.CFUNCTYPE(C.c_double, C.c_void_p, C.c_double)

_REF_PROTOS = {
    "ref_march_coupled": (C.c_int, [_BP, C.c_int, C.c_double, C.c_int, _i64p, _ip]),
    "ref_march_nonlinear_material": (C.c_int, [_BP, _MP, C.c_int, C.c_double, C.c_int, _i64p, _ip]),
    "ref_oracle_march_analytic": (C.c_int, [_BP, _MP, C.c_int, C.c_double, C.c_int, _i64p, _ip]),
    "ref_bootstrap": (C.c_int, [_BP, _MP, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int]),
    "ref_march_implicit": (C.c_int, [_BP, _MP, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                     C.POINTER(C.c_long)]),
    "ref_df_step_linear": (None, [C.c_int, A.dp, A.dp, C.c_double, A.dp]),
    "ref_material_star": (C.c_int, [_MP, C.c_double, C.c_double, C.c_int, C.POINTER(Coeffs)]),
    "ref_material_evaluate": (C.c_int, [C.c_double, C.c_double, C.POINTER(Coeffs)]),
    "ref_saturation_pressure": (C.c_double, [C.c_double]),
    "ref_scale_wall": (C.c_int, [C.POINTER(Coeffs)] + [C.c_double] * 8 + [A.dp]),
    "ref_scale_zone": (C.c_int, [C.c_double] * 9 + [A.dp]),
    "ref_attach_wall": (C.c_int, [C.POINTER(Coeffs)] + [C.c_double] * 9 + [A.dp]),
    "ref_building_march": (C.c_int, [C.POINTER(A.ModelDesc), C.POINTER(BuildingState), C.c_int64, C.c_int,
                                     _i64p, _ip]),
    "ref_run": (C.c_int, [C.POINTER(A.ModelDesc), C.c_double, A.dp, A.dp, A.dp, A.dp, C.POINTER(C.c_long), A.dp]),
    "ref_hardware_threads": (C.c_int, []),
    "ref_last_domain": (None, [_ip, _ip, _ip]),
}

_cache: dict = {}


def _load(path: Path, protos: dict) -> Optional[C.CDLL]:
    key = str(path)
    if key in _cache:
        return _cache[key]
    if not path.exists():
        return None
    lib = C.CDLL(str(path))
    for name, (res, args) in protos.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    _cache[key] = lib
    return lib


def oracle_lib() -> C.CDLL:
    lib = _load(ORACLE_SO, _ORACLE_PROTOS)
    if lib is None:
        raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle`")
    return lib


def ref_lib() -> Optional[C.CDLL]:
    """The compiled reference, or None where it was not built (no /root/reference)."""
    return _load(REF_SO, _REF_PROTOS)


def threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1


def _p(a):
    return a.ctypes.data_as(A.dp)


# ---- forcing tables from a Model (same Signal arithmetic as signal.hpp:39-50) ----
def forcing_table(model, times, layer0: int = 0, tables: Optional[dict] = None) -> np.ndarray:
    """[len(times), n_channels, 4] ambient rows; row k is layer layer0+k at time times[k]."""
    nch = max(1, len(model.channels))
    out = np.zeros((len(times), nch, 4))
    if not model.channels:
        out[:, 0, :2] = 1.0
    for c, ch in enumerate(model.channels):
        for i, sig in enumerate((ch.u_inf, ch.v_inf, ch.g_inf, ch.q_inf)):
            out[:, c, i] = [sig(t) for t in times]
    for c, (first, tab) in (tables or {}).items():
        for k in range(len(times)):
            L = layer0 + k
            if first <= L < first + len(tab):
                out[k, c, :] = tab[L - first]
    return out


class WallBatch:
    """A set of independent walls (no zones) in the layout orc_batch/ref shims take."""

    def __init__(self, model, state: dict, table: np.ndarray, layer0: int = 0):
        self.model = model
        self.n, self.W = model.n_nodes, model.n_walls
        self.state = {k: np.ascontiguousarray(state[k], dtype=np.float64).copy()
                      for k in ("u_prev", "u_curr", "v_prev", "v_curr")}
        self.groups = np.ascontiguousarray(model.groups)
        self.biot = np.ascontiguousarray(model.biot)
        ch = np.ascontiguousarray(model.attach[:, :, 1], dtype=np.int32)
        if np.any(model.attach[:, :, 0] != 0):
            raise ValueError("WallBatch: zone faces need the building path")
        self.chan = ch
        self.table = np.ascontiguousarray(table, dtype=np.float64)
        self.layer0 = layer0
        self.b = Batch(self.W, self.n, model.dx, self.groups.ctypes.data_as(C.POINTER(A.WallGroups)),
                       self.biot.ctypes.data_as(C.POINTER(A.FaceBiot)), self.chan.ctypes.data_as(C.POINTER(C.c_int32)),
                       self.table.shape[1], self.table.ctypes.data_as(C.POINTER(A.Ambient)), layer0,
                       model.divergence_norm, _p(self.state["u_prev"]), _p(self.state["u_curr"]),
                       _p(self.state["v_prev"]), _p(self.state["v_curr"]))

    def set_layer0(self, layer0: int, table: np.ndarray):
        self.table = np.ascontiguousarray(table, dtype=np.float64)
        self.b.table = self.table.ctypes.data_as(C.POINTER(A.Ambient))
        self.b.layer0 = layer0
        self.layer0 = layer0


def coeff_model(model) -> CoeffModel:
    """One coefficient model for a whole batch (material: wall 0's reference set)."""
    m = CoeffModel()
    if model.coeff_kind == "analytic_d":
        m.kind = ORC_COEFF_ANALYTIC_D
        m.p = (C.c_double * 4)(*model.coeff_params)
    elif model.coeff_kind == "material":
        m.kind = ORC_COEFF_MATERIAL
        m.T_i, m.P_vi = model.T_i, model.P_vi
        m.reference = Coeffs(*map(float, model.wall_reference[0]))
    else:
        m.kind = ORC_COEFF_CONSTANT
    return m


def march(impl: str, wb: WallBatch, nsteps: int, dt: float, nthreads: int = 1):
    """DF steps with the guard; impl 'oracle' (C restatement) or 'ref' (reference)."""
    fl, fw = C.c_int64(-1), C.c_int(-1)
    m = coeff_model(wb.model)
    if impl == "oracle":
        lib = oracle_lib()
        if m.kind == ORC_COEFF_CONSTANT:
            rc = lib.orc_march_coupled(C.byref(wb.b), nsteps, dt, nthreads, C.byref(fl), C.byref(fw))
        else:
            rc = lib.orc_march_nonlinear(C.byref(wb.b), C.byref(m), nsteps, dt, nthreads, C.byref(fl), C.byref(fw))
    else:
        lib = ref_lib()
        if m.kind == ORC_COEFF_CONSTANT:
            rc = lib.ref_march_coupled(C.byref(wb.b), nsteps, dt, nthreads, C.byref(fl), C.byref(fw))
        elif m.kind == ORC_COEFF_MATERIAL:
            rc = lib.ref_march_nonlinear_material(C.byref(wb.b), C.byref(m), nsteps, dt, nthreads, C.byref(fl),
                                                  C.byref(fw))
        else:   # d(v) is expressible only through the reference's test oracle (df_oracle.hpp)
            rc = lib.ref_oracle_march_analytic(C.byref(wb.b), C.byref(m), nsteps, dt, nthreads, C.byref(fl), C.byref(fw))
    return rc, fl.value, fw.value


def march_long_mt(wb: WallBatch, nsteps: int, dt: float, nthreads: int):
    """nsteps DF steps of a one-wall batch with its nodes split over threads
    (oracle only; bitwise the serial march)."""
    fl = C.c_int64(-1)
    m = coeff_model(wb.model)
    rc = oracle_lib().orc_march_long_mt(C.byref(wb.b), C.byref(m), nsteps, dt, nthreads, C.byref(fl))
    return rc, fl.value, 0


def bootstrap(impl: str, wb: WallBatch, kind: str, dt: float, eta: float = 1e-5, max_subiters: int = 100,
              nthreads: int = 1) -> int:
    m = coeff_model(wb.model)
    k = A.HYG_BOOT_EXPLICIT if kind == "explicit" else A.HYG_BOOT_IMPLICIT
    if impl == "oracle":
        return oracle_lib().orc_bootstrap_batch(C.byref(wb.b), C.byref(m), k, dt, eta, max_subiters, nthreads)
    return ref_lib().ref_bootstrap(C.byref(wb.b), C.byref(m), k, dt, eta, max_subiters, nthreads)


def march_implicit(impl: str, wb: WallBatch, nsteps: int, dt: float, eta: float = 1e-5, max_subiters: int = 100,
                   nthreads: int = 1) -> int:
    m = coeff_model(wb.model)
    passes = C.c_long(0)
    fn = oracle_lib().orc_march_implicit if impl == "oracle" else ref_lib().ref_march_implicit
    fn(C.byref(wb.b), C.byref(m), nsteps, dt, eta, max_subiters, nthreads, C.byref(passes))
    return passes.value


class Building:
    """Full building state for orc_step_* / ref_building_march."""

    def __init__(self, model, state: dict):
        self.model = model
        self._keep: list = []
        self.desc = model.desc(self._keep)
        self.state = {k: np.ascontiguousarray(state[k], dtype=np.float64).copy()
                      for k in ("u_prev", "u_curr", "v_prev", "v_curr")}
        nz = max(1, len(model.zones))
        self.zu = np.ascontiguousarray(state.get("zone_u", np.ones(nz)), dtype=np.float64).copy()
        self.zv = np.ascontiguousarray(state.get("zone_v", np.ones(nz)), dtype=np.float64).copy()
        if self.zu.size == 0:
            self.zu, self.zv = np.ones(1), np.ones(1)
        self.s = BuildingState(_p(self.state["u_prev"]), _p(self.state["u_curr"]), _p(self.state["v_prev"]),
                               _p(self.state["v_curr"]), _p(self.zu), _p(self.zv), state.get("t", 0.0),
                               state.get("layer", 0))

    def run(self, impl: str, nsteps: int, with_bootstrap: bool = True, nthreads: int = 1):
        """run() from the current state; nthreads > 1 (oracle, with the start):
        the explicit steps split over threads, bitwise the serial march."""
        fl, fw, bp = C.c_int64(-1), C.c_int(-1), C.c_int(0)
        if impl == "oracle":
            lib = oracle_lib()
            if with_bootstrap and nthreads > 1:
                rc = lib.orc_run_mt(C.byref(self.desc), C.byref(self.s), nsteps, nthreads, C.byref(fl), C.byref(fw),
                                    C.byref(bp))
            elif with_bootstrap:
                rc = lib.orc_run(C.byref(self.desc), C.byref(self.s), nsteps, C.byref(fl), C.byref(fw), C.byref(bp))
            else:
                rc = 0
                for _ in range(nsteps):
                    rc = lib.orc_step_explicit(C.byref(self.desc), C.byref(self.s))
                    if rc:
                        fl.value = self.s.layer + 1
                        break
        else:
            rc = ref_lib().ref_building_march(C.byref(self.desc), C.byref(self.s), nsteps, int(with_bootstrap),
                                              C.byref(fl), C.byref(bp))
        self.fail_wall = fw.value
        return rc, fl.value, bp.value

    @staticmethod
    def domain(impl: str):
        """(wall, node, half) of the last HYG_EDOMAIN of a building march."""
        w, j, h = C.c_int(-1), C.c_int(-1), C.c_int(0)
        if impl == "oracle":
            lib = oracle_lib()
            lib.orc_last_domain(C.byref(j), C.byref(h))
            w.value = lib.orc_last_domain_wall()
        else:
            ref_lib().ref_last_domain(C.byref(w), C.byref(j), C.byref(h))
        return w.value, j.value, bool(h.value)
