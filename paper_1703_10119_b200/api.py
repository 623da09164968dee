"""Python binding of the C ABI (include/hygro_b200.h).

Mirrors the reference's host interface for the DF path — BuildingModel /
BuildingState / run() (building.hpp:38-102) and the exception taxonomy of
errors.hpp:8-45 — over a device-resident batched context.  There is no CPU
fallback: importing this module without the built CUDA library raises.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Optional, Sequence

import numpy as np

from . import _abi as A

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libhygro_b200.so"
_lib: Optional[C.CDLL] = None


def load_library(path: Optional[Path] = None) -> C.CDLL:
    """Load (once) the in-tree CUDA library; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(
            f"{p} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
    _lib = A.bind(C.CDLL(str(p)))
    return _lib


# ---- exceptions (errors.hpp:8-45) -----------------------------------------------
class HygroError(RuntimeError):
    code = -1

    def __init__(self, message: str, status: Optional[A.Status] = None):
        super().__init__(message)
        self.status = status


class InvalidArgument(HygroError, ValueError):
    code = A.HYG_EINVAL


class SchemaError(HygroError):
    code = A.HYG_ESCHEMA


class NumericalError(HygroError):
    """hygro::numerical_error — carries t_star (building.cpp:282-300)."""
    code = A.HYG_EDIVERGED

    def __init__(self, message, status=None):
        super().__init__(message, status)
        self.t_star = status.t_star if status is not None else math.nan
        self.layer = status.layer if status is not None else -1
        self.wall = status.wall if status is not None else -1


class DomainError(HygroError):
    """hygro::domain_error of a strict coefficient evaluation (wall.cpp:99-126):
    the wall, the node j (half=False) or half node j+1/2 (half=True), and the
    time layer whose step failed (the state stays at the layer before it)."""
    code = A.HYG_EDOMAIN

    def __init__(self, message, status=None):
        super().__init__(message, status)
        self.wall = status.wall if status is not None else -1
        self.node = status.node if status is not None else -1
        self.half = bool(status.half) if status is not None else False
        self.layer = status.layer if status is not None else -1


class ConvergenceError(HygroError):
    code = A.HYG_ECONVERGE

    def __init__(self, message, status=None):
        super().__init__(message, status)
        self.residual = status.residual if status is not None else math.nan


class ScalingError(HygroError):
    code = A.HYG_ESCALING


class CudaError(HygroError):
    code = A.HYG_ECUDA


class NotSupported(HygroError):
    code = A.HYG_ENOTSUP


_BY_CODE = {cls.code: cls for cls in (InvalidArgument, SchemaError, NumericalError, DomainError,
                                      ConvergenceError, ScalingError, CudaError, NotSupported)}


def _check(rc: int, status: Optional[A.Status] = None, what: str = "") -> None:
    if rc == A.HYG_OK:
        return
    lib = load_library()
    msg = status.message.decode(errors="replace") if status is not None and status.message else ""
    if not msg:
        msg = lib.hyg_strerror(rc).decode()
    cls = _BY_CODE.get(rc, HygroError)
    raise cls(f"{what}: {msg}" if what else msg, status)


# ---- signals (signal.hpp:13-86) ---------------------------------------------------
@dataclass
class Signal:
    form: str = "constant"          # constant | sinusoid | sin_squared
    base: float = 0.0
    amplitude: float = 0.0
    period: float = 1.0
    phase: float = 0.0
    windows: Sequence[tuple] = ()   # (from, to, value)

    @staticmethod
    def constant(v):
        return Signal("constant", float(v))

    @staticmethod
    def sinusoid(base, amplitude, period, phase=0.0):
        return Signal("sinusoid", base, amplitude, period, phase)

    @staticmethod
    def sin_squared(base, amplitude, period, phase=0.0):
        return Signal("sin_squared", base, amplitude, period, phase)

    @staticmethod
    def schedule(base, windows):
        return Signal("constant", base, windows=tuple(windows))

    def __call__(self, t: float) -> float:        # Signal::operator() signal.hpp:39-50
        v = self.base
        if self.form == "sinusoid":
            v += self.amplitude * math.sin(2.0 * math.pi * (t - self.phase) / self.period)
        elif self.form == "sin_squared":
            s = math.sin(2.0 * math.pi * (t - self.phase) / self.period)
            v += self.amplitude * s * s
        for a, b, x in self.windows:
            if a <= t < b:
                v += x
        return v

    def to_c(self, keep: list) -> A.Signal:
        form = {"constant": A.HYG_SIG_CONSTANT, "sinusoid": A.HYG_SIG_SIN, "sin_squared": A.HYG_SIG_SIN2}[self.form]
        s = A.Signal(form=form, n_windows=len(self.windows), base=self.base, amplitude=self.amplitude,
                     period=self.period, phase=self.phase)
        if self.windows:
            arr = (A.Window * len(self.windows))(*[A.Window(a, b, x) for a, b, x in self.windows])
            keep.append(arr)
            s.windows = arr
        return s


@dataclass
class ChannelSpec:
    """Exterior forcing of a face (FaceAttachment building.hpp:13-21)."""
    u_inf: Signal = field(default_factory=lambda: Signal.constant(1.0))
    v_inf: Signal = field(default_factory=lambda: Signal.constant(1.0))
    g_inf: Signal = field(default_factory=lambda: Signal.constant(0.0))
    q_inf: Signal = field(default_factory=lambda: Signal.constant(0.0))


@dataclass
class ZoneSpec:
    """ZoneConfig (zone.hpp:47-54) with ZoneDimensionless scalars."""
    kappa_a_tt1: float
    g_v: float
    q_v1: float
    q_v2: float
    sources: int = 0
    moisture_sign: int = A.HYG_MOISTURE_FLUX_CONSISTENT
    walls: Sequence[tuple] = ()      # (wall, face, Bi_M, Bi_TT, Bi_TM, theta_T, theta_M)
    interzone: Sequence[tuple] = ()  # (peer, g_inz, q_inz1, q_inz2)
    radiation: Sequence[tuple] = ()  # (emitter_wall, receiver_wall, view_factor, emissivity)


@dataclass
class SourceSpec:
    g_o: Signal = field(default_factory=lambda: Signal.constant(0.0))
    q_o: Signal = field(default_factory=lambda: Signal.constant(0.0))
    q_h: Signal = field(default_factory=lambda: Signal.constant(0.0))


class Model:
    """A batch of walls on one grid (+ zones): the device analogue of BuildingModel.

    groups: (W,4) [Fo_M, Fo_TT, Fo_TM, gamma]; biot: (W,2,3) [Bi_M, Bi_TT, Bi_TM] per face;
    attach: (W,2,2) [kind, index] per face (kind 0 = exterior channel, 1 = zone).
    coeff_kind "material": CoefficientModel::material with ScalingContext (T_i, P_vi),
    wall_reference (W,6) [c_M, k_M, c_TT, k_TT, c_TM, k_TM] and wall_material (W,) bool
    (None = every wall); wall_thickness / wall_k_TT0 (W,) scale zone radiation fluxes.
    """

    def __init__(self, n_nodes: int, dx: float, groups, biot, attach=None, channels=(ChannelSpec(),),
                 zones=(), zone_sources=(), outdoor_u=None, outdoor_v=None, dt=1e-3,
                 divergence_norm=1e3, eta_factor=1e-2, max_subiters=100, precision="f64",
                 coeff_kind="constant", coeff_params=(0.0, 0.0, 0.0, 0.0), device=0, T_i=293.15,
                 P_vi=None, wall_reference=None, wall_material=None, wall_thickness=None, wall_k_TT0=None):
        self.groups = np.ascontiguousarray(groups, dtype=np.float64).reshape(-1, 4)
        self.n_walls = self.groups.shape[0]
        self.biot = np.ascontiguousarray(biot, dtype=np.float64).reshape(self.n_walls, 2, 3)
        if attach is None:
            attach = np.zeros((self.n_walls, 2, 2), dtype=np.int32)
        self.attach = np.ascontiguousarray(attach, dtype=np.int32).reshape(self.n_walls, 2, 2)
        self.n_nodes, self.dx = int(n_nodes), float(dx)
        self.channels = list(channels)
        self.zones = list(zones)
        self.zone_sources = list(zone_sources) or ([SourceSpec()] if zones else [])
        self.outdoor_u = outdoor_u or Signal.constant(1.0)
        self.outdoor_v = outdoor_v or Signal.constant(1.0)
        self.dt, self.divergence_norm = float(dt), float(divergence_norm)
        self.eta_factor, self.max_subiters = float(eta_factor), int(max_subiters)
        self.precision = precision
        self.coeff_kind = coeff_kind
        self.coeff_params = tuple(float(x) for x in coeff_params)
        self.device = int(device)
        self.T_i = float(T_i)
        self.P_vi = float(P_vi) if P_vi is not None else 0.0
        W = self.n_walls
        self.wall_reference = (None if wall_reference is None else
                               np.ascontiguousarray(wall_reference, dtype=np.float64).reshape(W, 6))
        self.wall_material = (None if wall_material is None else
                              np.ascontiguousarray(np.asarray(wall_material, dtype=bool).astype(np.int32)
                                                   * A.HYG_COEFF_MATERIAL).reshape(W))
        self.wall_thickness = (None if wall_thickness is None else
                               np.ascontiguousarray(wall_thickness, dtype=np.float64).reshape(W))
        self.wall_k_TT0 = (None if wall_k_TT0 is None else
                           np.ascontiguousarray(wall_k_TT0, dtype=np.float64).reshape(W))

    def desc(self, keep: list) -> A.ModelDesc:
        d = A.ModelDesc()
        d.n_walls, d.n_nodes, d.dx = self.n_walls, self.n_nodes, self.dx
        d.precision = A.HYG_F32 if self.precision == "f32" else A.HYG_F64
        d.coeff_kind = {"analytic_d": A.HYG_COEFF_ANALYTIC_D, "material": A.HYG_COEFF_MATERIAL}.get(
            self.coeff_kind, A.HYG_COEFF_CONSTANT)
        d.coeff_params = (C.c_double * 4)(*self.coeff_params)
        keep += [self.groups, self.biot, self.attach]
        d.groups = self.groups.ctypes.data_as(C.POINTER(A.WallGroups))
        d.biot = self.biot.ctypes.data_as(C.POINTER(A.FaceBiot))
        d.attach = self.attach.ctypes.data_as(C.POINTER(A.FaceAttach))
        ch = (A.Channel * max(1, len(self.channels)))()
        for i, c in enumerate(self.channels):
            ch[i] = A.Channel(c.u_inf.to_c(keep), c.v_inf.to_c(keep), c.g_inf.to_c(keep), c.q_inf.to_c(keep))
        keep.append(ch)
        d.n_channels, d.channels = len(self.channels), ch
        zs = (A.ZoneDesc * max(1, len(self.zones)))()
        for i, z in enumerate(self.zones):
            wl = (A.ZoneWallLink * max(1, len(z.walls)))(*[A.ZoneWallLink(*w) for w in z.walls])
            il = (A.InterzoneLink * max(1, len(z.interzone)))(*[A.InterzoneLink(*x) for x in z.interzone])
            rl = (A.RadiationLink * max(1, len(z.radiation)))(*[A.RadiationLink(*x) for x in z.radiation])
            keep += [wl, il, rl]
            zs[i] = A.ZoneDesc(z.kappa_a_tt1, z.g_v, z.q_v1, z.q_v2, z.sources, z.moisture_sign,
                               len(z.walls), wl, len(z.interzone), il, len(z.radiation), rl)
        keep.append(zs)
        d.n_zones, d.zones = len(self.zones), zs
        src = (A.ZoneSources * max(1, len(self.zone_sources)))()
        for i, s in enumerate(self.zone_sources):
            src[i] = A.ZoneSources(s.g_o.to_c(keep), s.q_o.to_c(keep), s.q_h.to_c(keep))
        keep.append(src)
        d.n_zone_sources, d.zone_sources = len(self.zone_sources), src
        d.outdoor_u, d.outdoor_v = self.outdoor_u.to_c(keep), self.outdoor_v.to_c(keep)
        d.dt, d.divergence_norm = self.dt, self.divergence_norm
        d.eta_factor, d.max_subiters, d.device = self.eta_factor, self.max_subiters, self.device
        d.T_i, d.P_vi = self.T_i, self.P_vi
        if self.wall_material is not None:
            keep.append(self.wall_material)
            d.wall_coeff = self.wall_material.ctypes.data_as(C.POINTER(C.c_int32))
        if self.wall_reference is not None:
            keep.append(self.wall_reference)
            d.wall_reference = self.wall_reference.ctypes.data_as(C.POINTER(A.CoeffSet))
        for name in ("wall_thickness", "wall_k_TT0"):
            a = getattr(self, name)
            if a is not None:
                keep.append(a)
                setattr(d, name, a.ctypes.data_as(A.dp))
        return d


def _ptr(a):
    return None if a is None else a.ctypes.data_as(A.dp)


def _addr(a: int):
    """A raw (host or device) address as the ABI's double*."""
    return C.cast(C.c_void_p(a), A.dp)


def _f64(a, n):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    if a.size != n:
        raise InvalidArgument(f"expected {n} values, got {a.size}")
    return a


class Context:
    """Device-resident state of one Model (BuildingState + the step/run calls)."""

    def __init__(self, model: Model):
        self.lib = load_library()
        self.model = model
        self._keep: list = []
        st = A.Status()
        h = C.c_void_p()
        _check(self.lib.hyg_create(C.byref(model.desc(self._keep)), C.byref(h), C.byref(st)), st, "hyg_create")
        self.h = h
        self.cells = model.n_walls * model.n_nodes

    # -- state ---------------------------------------------------------------------
    def set_state(self, u_prev, u_curr, v_prev, v_curr, zone_u=None, zone_v=None, t=0.0, layer=0):
        arrs = [_f64(x, self.cells) for x in (u_prev, u_curr, v_prev, v_curr)]
        nz = len(self.model.zones)
        zu = _f64(zone_u, nz) if zone_u is not None and nz else None
        zv = _f64(zone_v, nz) if zone_v is not None and nz else None
        _check(self.lib.hyg_set_state(self.h, *map(_ptr, arrs), _ptr(zu), _ptr(zv), float(t), int(layer)),
               None, "hyg_set_state")

    def get_state(self, out=None) -> dict:
        if out is None:
            out = {k: np.empty(self.cells) for k in ("u_prev", "u_curr", "v_prev", "v_curr")}
        nz = len(self.model.zones)
        zu, zv = (np.empty(nz), np.empty(nz)) if nz else (None, None)
        t, layer = C.c_double(), C.c_int64()
        _check(self.lib.hyg_get_state(self.h, _ptr(out["u_prev"]), _ptr(out["u_curr"]), _ptr(out["v_prev"]),
                                      _ptr(out["v_curr"]), _ptr(zu), _ptr(zv), C.byref(t), C.byref(layer)),
               None, "hyg_get_state")
        out.update(zone_u=zu, zone_v=zv, t=t.value, layer=layer.value)
        return out

    # -- sub-ranges (halo exchange between shards) --------------------------------
    def get_cells(self, cell0: int, count: int) -> dict:
        out = {k: np.empty(count) for k in ("u_prev", "u_curr", "v_prev", "v_curr")}
        _check(self.lib.hyg_get_cells(self.h, cell0, count, _ptr(out["u_prev"]), _ptr(out["u_curr"]),
                                      _ptr(out["v_prev"]), _ptr(out["v_curr"])), None, "hyg_get_cells")
        return out

    def set_cells(self, cell0: int, values: dict) -> None:
        arrs = [np.ascontiguousarray(values[k], dtype=np.float64) for k in ("u_prev", "u_curr", "v_prev", "v_curr")]
        count = arrs[0].size
        _check(self.lib.hyg_set_cells(self.h, cell0, count, *map(_ptr, arrs)), None, "hyg_set_cells")

    def get_cells_into(self, cell0: int, count: int, out) -> None:
        """Copy cells [cell0, cell0+count) of the four layers into `out`, a
        contiguous float64 torch tensor of shape (4, count).  A CUDA `out` is
        filled by one pack kernel on the context's stream with no host
        synchronisation (hyg_pack_cells; hand the context the stream the
        consumer runs on, set_stream); a host `out` by the synchronous copy."""
        assert out.is_contiguous() and tuple(out.shape) == (4, count) and out.element_size() == 8
        base, step = out.data_ptr(), count * 8
        if out.is_cuda:
            _check(self.lib.hyg_pack_cells(self.h, cell0, count, C.c_void_p(base)), None, "hyg_pack_cells")
            return
        _check(self.lib.hyg_get_cells(self.h, cell0, count, *[_addr(base + i * step) for i in range(4)]),
               None, "hyg_get_cells")

    def set_cells_from(self, cell0: int, src) -> None:
        """Inverse of get_cells_into (CUDA `src`: one unpack kernel, stream-ordered)."""
        assert src.is_contiguous() and src.dim() == 2 and src.shape[0] == 4 and src.element_size() == 8
        count, base = int(src.shape[1]), src.data_ptr()
        if src.is_cuda:
            _check(self.lib.hyg_unpack_cells(self.h, cell0, count, C.c_void_p(base)), None, "hyg_unpack_cells")
            return
        _check(self.lib.hyg_set_cells(self.h, cell0, count, *[_addr(base + i * count * 8) for i in range(4)]),
               None, "hyg_set_cells")

    def get_zones_into(self, zone0: int, count: int, out) -> None:
        """Zones [zone0, zone0+count) into `out`: contiguous float64 (2, count)
        (CUDA: stream-ordered device copies, no host synchronisation)."""
        assert out.is_contiguous() and tuple(out.shape) == (2, count) and out.element_size() == 8
        base = out.data_ptr()
        if out.is_cuda:
            _check(self.lib.hyg_pack_zones(self.h, zone0, count, C.c_void_p(base)), None, "hyg_pack_zones")
            return
        _check(self.lib.hyg_get_zones(self.h, zone0, count, _addr(base), _addr(base + count * 8)),
               None, "hyg_get_zones")

    def set_zones_from(self, zone0: int, src) -> None:
        assert src.is_contiguous() and src.dim() == 2 and src.shape[0] == 2 and src.element_size() == 8
        count, base = int(src.shape[1]), src.data_ptr()
        if src.is_cuda:
            _check(self.lib.hyg_unpack_zones(self.h, zone0, count, C.c_void_p(base)), None, "hyg_unpack_zones")
            return
        _check(self.lib.hyg_set_zones(self.h, zone0, count, _addr(base), _addr(base + count * 8)),
               None, "hyg_set_zones")

    def set_stream(self, stream=None) -> None:
        """Run on `stream` (a torch.cuda.Stream or a raw cudaStream_t; None: the
        context's own), ordered after the work issued so far (hyg_set_stream)."""
        ptr = getattr(stream, "cuda_stream", stream)
        _check(self.lib.hyg_set_stream(self.h, C.c_void_p(ptr) if ptr else None), None, "hyg_set_stream")

    def get_zones(self, zone0: int, count: int):
        zu, zv = np.empty(count), np.empty(count)
        _check(self.lib.hyg_get_zones(self.h, zone0, count, _ptr(zu), _ptr(zv)), None, "hyg_get_zones")
        return zu, zv

    def set_zones(self, zone0: int, zu, zv) -> None:
        zu = np.ascontiguousarray(zu, dtype=np.float64)
        zv = np.ascontiguousarray(zv, dtype=np.float64)
        _check(self.lib.hyg_set_zones(self.h, zone0, zu.size, _ptr(zu), _ptr(zv)), None, "hyg_set_zones")

    def set_owned(self, cell0: int, cell1: int, zone0: int = 0, zone1: int = 2 ** 31 - 1,
                  reduce: Optional[Callable[[float], float]] = None) -> None:
        """Guard/residual restricted to owned ranges; `reduce(local_max) -> global_max`."""
        self._reduce_cb = A.REDUCE_FN(lambda user, x: float(reduce(x))) if reduce else None
        _check(self.lib.hyg_set_owned(self.h, cell0, cell1, zone0, zone1,
                                      C.cast(self._reduce_cb, C.c_void_p) if reduce else None, None),
               None, "hyg_set_owned")

    def snapshot(self):
        """Device-side checkpoint of the full resumable state (hyg_snapshot)."""
        _check(self.lib.hyg_snapshot(self.h), None, "hyg_snapshot")

    def restore(self):
        _check(self.lib.hyg_restore(self.h), None, "hyg_restore")

    def set_channel_table(self, channel: int, first_layer: int, table) -> None:
        tab = np.ascontiguousarray(table, dtype=np.float64).reshape(-1, 4)
        self._keep_table = tab
        _check(self.lib.hyg_set_channel_table(self.h, channel, first_layer, tab.shape[0],
                                              tab.ctypes.data_as(C.POINTER(A.Ambient))), None,
               "hyg_set_channel_table")

    # -- marching --------------------------------------------------------------------
    def bootstrap(self, kind: str = "implicit") -> A.Status:
        st = A.Status()
        k = A.HYG_BOOT_EXPLICIT if kind == "explicit" else A.HYG_BOOT_IMPLICIT
        _check(self.lib.hyg_bootstrap(self.h, k, C.byref(st)), st, "hyg_bootstrap")
        return st

    def advance(self, nsteps: int, dt: Optional[float] = None, edge: Optional[tuple] = None,
                wait_event=None) -> A.Status:
        """hyg_advance; with `wait_event` (a torch.cuda.Event or a raw cudaEvent_t recorded
        behind a halo refresh of the first edge[0] / last edge[1] cells on another stream)
        hyg_advance_overlapped: the windows clear of those cells march at once."""
        st = A.Status()
        if wait_event is None:
            _check(self.lib.hyg_advance(self.h, int(nsteps), float(dt or 0.0), C.byref(st)), st, "hyg_advance")
            return st
        ev = getattr(wait_event, "cuda_event", wait_event)
        ev = getattr(ev, "value", ev)
        lo, hi = edge or (0, 0)
        _check(self.lib.hyg_advance_overlapped(self.h, int(nsteps), float(dt or 0.0), int(lo), int(hi),
                                               C.c_void_p(ev), C.byref(st)), st, "hyg_advance_overlapped")
        return st

    def set_exchange_stream(self, stream=None) -> None:
        """Pack / unpack kernels (get_cells_into, set_cells_from, get_zones_into,
        set_zones_from) run on `stream` (torch.cuda.Stream or raw cudaStream_t; None: the
        context's stream again), with no implicit ordering (hyg_set_exchange_stream)."""
        ptr = getattr(stream, "cuda_stream", stream)
        _check(self.lib.hyg_set_exchange_stream(self.h, C.c_void_p(ptr) if ptr else None), None,
               "hyg_set_exchange_stream")

    def run(self, horizon: float, cadence: float = 1e30, boot: str = "implicit",
            frame: Optional[Callable[[int, float, "Context"], None]] = None) -> A.Status:
        st = A.Status()
        cb = A.FRAME_FN((lambda u, layer, t, h: frame(layer, t, self)) if frame else (lambda *a: None))
        k = A.HYG_BOOT_EXPLICIT if boot == "explicit" else A.HYG_BOOT_IMPLICIT
        _check(self.lib.hyg_run(self.h, float(horizon), float(cadence), k, cb, None, C.byref(st)), st, "hyg_run")
        return st

    SCHEMES = {"df": A.HYG_SCHEME_DF, "euler-implicit": A.HYG_SCHEME_EULER_IMPLICIT,
               "euler-explicit": A.HYG_SCHEME_EULER_EXPLICIT}

    def run_scheme(self, scheme: str, horizon: float, cadence: float = 1e30,
                   frame: Optional[Callable[[int, float, "Context"], None]] = None) -> A.RunReport:
        """run() (building.cpp:303-356) with Scheme df | euler-implicit | euler-explicit;
        returns SimulationResult's counters (steps, bootstrap/mean/max subiterations)."""
        st, rep = A.Status(), A.RunReport()
        cb = A.FRAME_FN((lambda u, layer, t, h: frame(layer, t, self)) if frame else (lambda *a: None))
        _check(self.lib.hyg_run_scheme(self.h, self.SCHEMES[scheme], float(horizon), float(cadence), cb, None,
                                       C.byref(rep), C.byref(st)), st, "hyg_run_scheme")
        return rep

    # -- measurement -------------------------------------------------------------------
    def synchronize(self):
        _check(self.lib.hyg_synchronize(self.h))

    def record(self, slot: int):
        _check(self.lib.hyg_event_record(self.h, slot))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_double()
        _check(self.lib.hyg_event_elapsed_ms(self.h, a, b, C.byref(ms)))
        return ms.value

    def profiling(self, on: bool = True):
        _check(self.lib.hyg_set_profiling(self.h, int(on)))

    def kernel_stats(self) -> list[dict]:
        out = []
        for i in range(self.lib.hyg_kernel_stats_count(self.h)):
            name, n, ms, upd = C.c_char_p(), C.c_int64(), C.c_double(), C.c_double()
            _check(self.lib.hyg_kernel_stats(self.h, i, C.byref(name), C.byref(n), C.byref(ms), C.byref(upd)))
            out.append(dict(name=name.value.decode(), launches=n.value, ms=ms.value, node_updates=upd.value))
        return out

    TUNING = {"ring_grid": A.HYG_TUNE_RING_GRID, "ring_kernel": A.HYG_TUNE_RING_KERNEL,
              "material_exact": A.HYG_TUNE_MATERIAL_EXACT, "tiled_load": A.HYG_TUNE_TILED_LOAD,
              "ring_depth": A.HYG_TUNE_RING_DEPTH}

    def set_tuning(self, knob: str, value: int) -> None:
        """Launch-shape knob (hyg_set_tuning): ring_grid = cap on the persistent
        zone-ring grid; ring_kernel = 0 auto (K6), 1 K4r, 2 K4, 3 K5, 4 K6; material_exact = 1 for
        the accurate material evaluation (hyg_crmath.cuh) instead of the fast one."""
        _check(self.lib.hyg_set_tuning(self.h, self.TUNING[knob], int(value)), None, "hyg_set_tuning")

    def reset_kernel_stats(self):
        _check(self.lib.hyg_reset_kernel_stats(self.h))

    @property
    def launches(self) -> int:
        return int(self.lib.hyg_launch_count(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.hyg_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def df_march_linear(prev, curr, lam: float, steps: int, device: int = 0):
    """df_step_linear (wall.cpp:60-71) `steps` times with layer rotation on the
    device, for a [fields, n] batch of single fields; returns (prev, curr)."""
    p = np.array(prev, dtype=np.float64, order="C", ndmin=2)
    c = np.array(curr, dtype=np.float64, order="C", ndmin=2)
    if p.shape != c.shape:
        raise InvalidArgument("prev and curr must have the same shape")
    _check(load_library().hyg_df_march_linear(device, p.shape[0], p.shape[1], float(lam), int(steps), _ptr(p),
                                              _ptr(c)), None, "hyg_df_march_linear")
    return p, c


# ---- host-side setup (scaling.cpp) -------------------------------------------------
def saturation_pressure(T: float) -> float:
    out = C.c_double()
    _check(load_library().hyg_saturation_pressure(T, C.byref(out)), None, "saturation_pressure")
    return out.value


def material_evaluate(T: float, P_v: float, clamped: bool = False) -> tuple:
    """MaterialModel::evaluate(_clamped) (materials.cpp:91-121) on the host:
    (c_M, k_M, c_TT, k_TT, c_TM, k_TM)."""
    out = A.CoeffSet()
    _check(load_library().hyg_material_evaluate(T, P_v, int(clamped), C.byref(out)), None, "material_evaluate")
    return (out.c_M, out.k_M, out.c_TT, out.k_TT, out.c_TM, out.k_TM)


def scale_wall(reference, L, h_T0, h_M0, h_T1, h_M1, T_i=293.15, phi_i=0.5, t_0=3600.0):
    """Return (groups[4], biot[2][3]) of one wall (scaling.cpp:30-58)."""
    ref = (C.c_double * 6)(*reference)
    g, f = A.WallGroups(), (A.FaceBiot * 2)()
    _check(load_library().hyg_scale_wall(ref, L, h_T0, h_M0, h_T1, h_M1, T_i, phi_i, t_0, C.byref(g), f),
           None, "scale_wall")
    return ([g.Fo_M, g.Fo_TT, g.Fo_TM, g.gamma], [[x.Bi_M, x.Bi_TT, x.Bi_TM] for x in f])


def scale_zone(volume, rho_a=1.0, c_pa=1005.0, c_pv=1960.0, ach=0.0, T_i=293.15, phi_i=0.5, t_0=3600.0):
    out = (C.c_double * 7)()
    _check(load_library().hyg_scale_zone(volume, rho_a, c_pa, c_pv, ach, T_i, phi_i, t_0, out), None, "scale_zone")
    return dict(zip(("kappa_a_tt1", "g_v", "q_v1", "q_v2", "g_o_per", "q_o_per", "q_h_per"), list(out)))


def attach_wall_to_zone(reference, area, L, volume, rho_a=1.0, c_pa=1005.0, T_i=293.15, phi_i=0.5, t_0=3600.0):
    out = (C.c_double * 2)()
    ref = (C.c_double * 6)(*reference)
    _check(load_library().hyg_attach_wall_to_zone(ref, area, L, volume, rho_a, c_pa, T_i, phi_i, t_0, out),
           None, "attach_wall_to_zone")
    return tuple(out)


def scale_interzone(ach, volume, rho_a=1.0, c_pa=1005.0, c_pv=1960.0, T_i=293.15, phi_i=0.5, t_0=3600.0):
    out = (C.c_double * 3)()
    _check(load_library().hyg_scale_interzone(ach, volume, rho_a, c_pa, c_pv, T_i, phi_i, t_0, out), None,
           "scale_interzone")
    return tuple(out)


def probe_fp32_peak(device: int = 0) -> float:
    tf = C.c_double()
    _check(load_library().hyg_probe_fp32_peak(device, C.byref(tf)), None, "probe_fp32_peak")
    return tf.value


def probe_fp64_peak(device: int = 0) -> float:
    tf, mhz = C.c_double(), C.c_double()
    _check(load_library().hyg_probe_fp64_peak(device, C.byref(tf), C.byref(mhz)), None, "probe_fp64_peak")
    return tf.value
