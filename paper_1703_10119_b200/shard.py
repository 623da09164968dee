"""Multi-GPU decomposition of the DF path: one process per GPU, torch.distributed
for the plumbing.

  * independent walls (configs[1]/[2]): contiguous wall ranges per rank and no
    exchange at all — bench.py's weak-scaling layout;
  * the long domain (configs[4]): x-slabs with H halo nodes per side;
  * the zone ring (configs[3]): contiguous zone blocks with H halo zones per
    side (a zone travels whole with its walls).

Halo exchange is deep: every K <= H steps, not every step.  After K DF steps
node j depends only on nodes j-K..j+K of the two layers present K steps
earlier (the three-level stencil reaches one neighbour per step; a zone
reaches its ring neighbours one step at a time, walls are zone-local), so a
shard that marches its owned range plus H halo cells for K steps — treating
the far halo end as an artificial face — computes every owned cell exactly,
bit for bit as the undivided domain.  The halo copies are then refreshed
from their owners (both time layers; zones with their walls).  One exchange
moves 4 layers x H cells per side (x-slabs), i.e. K-fold fewer, larger
messages than a per-step 1-node halo, which matters when a step is a few
microseconds of GPU time.  The implicit starting step of a zoned building is
a joint fixed point: its residual is restricted to owned walls/zones and
max-reduced across ranks every pass (hyg_set_owned), and needs passes <= H.

The engine is the CUDA Context on GPUs; tests drive the same logic with the
C oracle on CPU ranks over gloo (tests/test_shard_gloo.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from .api import Model, NumericalError, ZoneSpec

FIELDS = ("u_prev", "u_curr", "v_prev", "v_curr")


@dataclass
class Slab:
    lo: int      # owned [lo, hi) in global nodes
    hi: int
    a: int       # local [a, b) = owned + halo
    b: int


def slab_bounds(n: int, world: int, rank: int, halo: int) -> Slab:
    lo, hi = n * rank // world, n * (rank + 1) // world
    if world > 1 and hi - lo < halo:
        raise ValueError(f"slab of {hi - lo} nodes is thinner than the halo ({halo})")
    return Slab(lo, hi, max(0, lo - halo), min(n, hi + halo))


class Comm:
    """Point-to-point + reductions over a torch.distributed group.

    On an NCCL group (one process per GPU, bench.py at N > 1) halo payloads
    stay on the device and in stream order: the engine runs on the current
    torch stream (Context.set_stream), packs its boundary cells into one CUDA
    buffer with one kernel (Context.get_cells_into -> hyg_pack_cells), NCCL
    moves it over NVLink behind that kernel, and the receiver's unpack kernel
    runs behind the receive — no host copies and no stream synchronisation on
    the exchange path.  On a gloo group (CPU tests, or ranks sharing one GPU)
    the same payloads travel as host tensors."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.on_device = dist.get_backend(group) == "nccl"
        self.device = torch.device("cuda", torch.cuda.current_device()) if self.on_device else torch.device("cpu")

    def tensor(self, a):
        """`a` (ndarray or tensor) as a contiguous float64 tensor on the comm device."""
        import torch
        if not isinstance(a, torch.Tensor):
            a = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        return a.to(self.device, torch.float64).contiguous()

    def exchange(self, sends: dict, recvs: dict) -> dict:
        """sends: {peer_rank: ndarray | tensor}; recvs: {peer_rank: shape};
        returns {peer_rank: tensor on the comm device}, complete and ordered
        before the host continues."""
        import torch
        reqs, out = [], {}
        for peer, shape in recvs.items():
            buf = torch.empty(shape, dtype=torch.float64, device=self.device)
            out[peer] = buf
            reqs.append(self.dist.irecv(buf, src=self._global(peer), group=self.group))
        for peer, arr in sends.items():
            reqs.append(self.dist.isend(self.tensor(arr), dst=self._global(peer), group=self.group))
        for r in reqs:
            r.wait()          # NCCL: the current stream waits for the transfers (no host block)
        return out

    def _global(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def _reduce(self, x: float, op) -> float:
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        self.dist.all_reduce(t, op=op, group=self.group)
        return float(t.item())

    def allreduce_max(self, x: float) -> float:
        return self._reduce(x, self.dist.ReduceOp.MAX)

    def allreduce_min(self, x: float) -> float:
        return self._reduce(x, self.dist.ReduceOp.MIN)


def _attach_stream(engine, comm):
    """On a device comm, run the engine on the current torch stream, so its
    pack/unpack kernels and the NCCL transfers are ordered by the stream."""
    if comm.on_device and hasattr(engine, "set_stream"):
        import torch
        engine.set_stream(torch.cuda.current_stream(comm.device))


def _get_block(engine, comm, cell0: int, count: int):
    """Cells [cell0, cell0+count) of the four layers as a (4, count) payload:
    a device tensor filled device to device when the engine and the comm are
    both on the GPU, else a host array."""
    if comm.on_device and hasattr(engine, "get_cells_into"):
        import torch
        buf = torch.empty((4, count), dtype=torch.float64, device=comm.device)
        engine.get_cells_into(cell0, count, buf)
        return buf
    c = engine.get_cells(cell0, count)
    return np.stack([c[f] for f in FIELDS])


def _set_block(engine, cell0: int, block):
    import torch
    if isinstance(block, torch.Tensor) and block.is_cuda and hasattr(engine, "set_cells_from"):
        engine.set_cells_from(cell0, block.contiguous())
        return
    a = block.cpu().numpy() if isinstance(block, torch.Tensor) else block
    engine.set_cells(cell0, dict(zip(FIELDS, a)))


class _Timer:
    """Accumulated time of the exchange and compute phases of a shard (CUDA
    events on the current stream on a device comm, host clock otherwise)."""

    def __init__(self, comm):
        self.on_device = comm.on_device
        self.ms = {"exchange": 0.0, "compute": 0.0}
        self.intervals = 0
        self._pending = []

    def phase(self, name):
        timer = self

        class _P:
            def __enter__(self_):
                if timer.on_device:
                    import torch
                    self_.e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    self_.e[0].record()
                else:
                    import time
                    self_.t0 = time.perf_counter()

            def __exit__(self_, *exc):
                if timer.on_device:
                    self_.e[1].record()
                    timer._pending.append((name, self_.e))
                else:
                    import time
                    timer.ms[name] += 1e3 * (time.perf_counter() - self_.t0)
        return _P()

    def totals(self) -> dict:
        for name, (a, b) in self._pending:
            b.synchronize()
            self.ms[name] += a.elapsed_time(b)
        self._pending.clear()
        return dict(self.ms, intervals=self.intervals)

    def reset(self):
        self.totals()
        self.ms = {"exchange": 0.0, "compute": 0.0}
        self.intervals = 0


def _advance_guarded(engine, k, comm, edge=None, wait_event=None):
    """k steps on every rank; a divergence anywhere stops all ranks with the
    earliest failing layer (check_bounded semantics across shards).  With
    `wait_event` the halo refresh of the first edge[0] / last edge[1] cells is
    still in flight on another stream (hyg_advance_overlapped)."""
    fail = float("inf")
    err = None
    try:
        if wait_event is None:
            engine.advance(k)
        else:
            engine.advance(k, edge=edge, wait_event=wait_event)
    except NumericalError as e:
        fail, err = float(e.layer), e
    first = comm.allreduce_min(fail)
    if first != float("inf"):
        if err is not None and float(err.layer) == first:
            raise err
        raise NumericalError(f"divergence on another shard at layer {int(first)}")


# ---------------------------------------------------------------------------------
class LongDomainShard:
    """configs[4]: one long wall cut into x-slabs.  `engine_factory(model)`
    returns a Context-like engine for the local slab.

    overlap (default: on a device comm with a CUDA engine): the halo refresh of
    an interval — pack, NCCL send/recv, unpack — runs on a second stream behind
    the interval's compute, and the next interval starts at once: the windows of
    its first launch that read no halo cell march while the exchange is in
    flight, the edge windows and the later launches follow behind the refresh's
    event (Context.advance(edge=, wait_event=) -> hyg_advance_overlapped)."""

    def __init__(self, model: Model, init: dict, comm, engine_factory: Callable, halo: int = 32,
                 overlap: Optional[bool] = None):
        self.comm, self.halo = comm, halo
        n = model.n_nodes
        s = self.slab = slab_bounds(n, comm.world, comm.rank, halo)
        biot = model.biot.copy()
        if s.a > 0:
            biot[0, 0] = 0.0          # artificial faces: adiabatic/impermeable (their
        if s.b < n:                   # cone never reaches the owned nodes)
            biot[0, 1] = 0.0
        local = Model(s.b - s.a, model.dx, model.groups, biot, model.attach, channels=model.channels,
                      dt=model.dt, divergence_norm=model.divergence_norm, coeff_kind=model.coeff_kind,
                      coeff_params=model.coeff_params, device=model.device)
        self.engine = engine_factory(local)
        _attach_stream(self.engine, comm)
        self.engine.set_state(**{f: init[f][s.a:s.b] for f in FIELDS})
        self.engine.set_owned(s.lo - s.a, s.hi - s.a)
        self.timer = _Timer(comm)
        can = bool(getattr(comm, "on_device", False)) and hasattr(self.engine, "set_exchange_stream")
        self.overlap = can if overlap is None else (bool(overlap) and can)
        self._xstream, self._pending = None, None
        # local cells a refresh rewrites: the left halo [0, lo - a), the right one [hi - a, b - a)
        self._edge = (s.lo - s.a, s.b - s.hi)

    def advance(self, nsteps: int):
        done = 0
        while done < nsteps:
            k = min(self.halo, nsteps - done)
            with self.timer.phase("compute"):
                _advance_guarded(self.engine, k, self.comm, edge=self._edge, wait_event=self._pending)
            self._pending = None
            if self.overlap:
                self._refresh_async()
            else:
                with self.timer.phase("exchange"):
                    self.refresh()
            self.timer.intervals += 1
            done += k
        self.join()

    def _refresh_async(self):
        """The refresh on the exchange stream, behind the compute issued so far; the
        compute stream does not wait for it (the next advance takes its event)."""
        import torch
        dev = self.comm.device
        cs = torch.cuda.current_stream(dev)
        if self._xstream is None:
            self._xstream = torch.cuda.Stream(dev)
        xs = self._xstream
        xs.wait_stream(cs)
        self.engine.set_exchange_stream(xs)
        try:
            with torch.cuda.stream(xs):
                with self.timer.phase("exchange"):
                    self.refresh()
                ev = torch.cuda.Event()
                ev.record(xs)
        finally:
            self.engine.set_exchange_stream(None)
        self._pending = ev

    def join(self):
        """The compute stream waits for a refresh still in flight."""
        if self._pending is not None:
            import torch
            torch.cuda.current_stream(self.comm.device).wait_event(self._pending)
            self._pending = None

    def refresh(self):
        s, H, r, P = self.slab, self.halo, self.comm.rank, self.comm.world
        sends, recvs = {}, {}
        if r > 0:
            sends[r - 1] = _get_block(self.engine, self.comm, s.lo - s.a, H)
            recvs[r - 1] = (4, H)
        if r < P - 1:
            sends[r + 1] = _get_block(self.engine, self.comm, s.hi - H - s.a, H)
            recvs[r + 1] = (4, H)
        got = self.comm.exchange(sends, recvs)
        if r > 0:
            _set_block(self.engine, 0, got[r - 1])
        if r < P - 1:
            _set_block(self.engine, s.hi - s.a, got[r + 1])

    def owned_state(self) -> dict:
        s = self.slab
        self.join()
        return self.engine.get_cells(s.lo - s.a, s.hi - s.lo)


# ---------------------------------------------------------------------------------
class ZoneRingShard:
    """configs[3]: zones in a ring, `walls_per_zone` consecutive walls per zone
    (zone z owns walls z*W .. z*W+W-1, face 1 on the zone), blocks of zones per
    rank with `halo` zones on each side."""

    def __init__(self, model: Model, init: dict, comm, engine_factory: Callable, walls_per_zone: int,
                 halo: int = 8):
        self.comm, self.halo, self.W = comm, halo, walls_per_zone
        Z = len(model.zones)
        P, r = comm.world, comm.rank
        self.lo, self.hi = Z * r // P, Z * (r + 1) // P
        if P > 1 and (self.hi - self.lo < halo or Z < (self.hi - self.lo) + 2 * halo):
            raise ValueError("zone block thinner than the halo")
        H = halo if P > 1 else 0
        self.gz = [(self.lo - H + i) % Z for i in range(self.hi - self.lo + 2 * H)]   # local -> global zone
        idx = {g: i for i, g in enumerate(self.gz)}
        n, W = model.n_nodes, walls_per_zone
        gw = np.concatenate([np.arange(g * W, g * W + W) for g in self.gz])            # local -> global wall
        self.gw = gw
        attach = model.attach[gw].copy()
        zones = []
        for i, g in enumerate(self.gz):
            zg = model.zones[g]
            links = [(i * W + k, l[1], *l[2:]) for k, l in enumerate(zg.walls)]
            for wl, l in zip(range(i * W, i * W + W), zg.walls):
                attach[wl, l[1]] = (1, i)
            inz = [(idx[p], *rest) for p, *rest in zg.interzone
                   if p in idx and (P == 1 or abs(idx[p] - i) == 1)]
            zones.append(ZoneSpec(zg.kappa_a_tt1, zg.g_v, zg.q_v1, zg.q_v2, zg.sources, zg.moisture_sign,
                                  links, inz))
        local = Model(n, model.dx, model.groups[gw], model.biot[gw], attach, channels=model.channels,
                      zones=zones, zone_sources=model.zone_sources, outdoor_u=model.outdoor_u,
                      outdoor_v=model.outdoor_v, dt=model.dt, divergence_norm=model.divergence_norm,
                      eta_factor=model.eta_factor, max_subiters=model.max_subiters, device=model.device)
        self.engine = engine_factory(local)
        _attach_stream(self.engine, comm)
        cells = (gw[:, None] * n + np.arange(n)[None, :]).reshape(-1)
        st = {f: init[f][cells] for f in FIELDS}
        st["zone_u"] = np.asarray(init["zone_u"])[self.gz]
        st["zone_v"] = np.asarray(init["zone_v"])[self.gz]
        self.engine.set_state(**st)
        self.H = H
        own = self.hi - self.lo
        self.engine.set_owned(H * W * n, (H + own) * W * n, H, H + own,
                              reduce=comm.allreduce_max if P > 1 else None)
        self.timer = _Timer(comm)

    def bootstrap(self, kind="implicit"):
        st = self.engine.bootstrap(kind)
        if self.H and st.subiterations > self.H:
            raise RuntimeError(f"implicit start took {st.subiterations} passes > halo {self.H}")
        self.refresh()
        return st

    def advance(self, nsteps: int):
        done = 0
        K = self.H if self.H else nsteps
        while done < nsteps:
            k = min(K, nsteps - done)
            with self.timer.phase("compute"):
                _advance_guarded(self.engine, k, self.comm)
            if self.H:
                with self.timer.phase("exchange"):
                    self.refresh()
            self.timer.intervals += 1
            done += k

    def _zone_block(self, i0, count):
        """Zones [i0, i0+count) with their walls as one flat payload:
        4 layers x cells, then zone_u, zone_v (on a device comm: one buffer,
        filled by one pack kernel and two stream-ordered copies)."""
        n, W = self.engine_model_n, self.W
        m = count * W * n
        if self.comm.on_device and hasattr(self.engine, "get_zones_into"):
            import torch
            buf = torch.empty(4 * m + 2 * count, dtype=torch.float64, device=self.comm.device)
            self.engine.get_cells_into(i0 * W * n, m, buf[:4 * m].view(4, m))
            self.engine.get_zones_into(i0, count, buf[4 * m:].view(2, count))
            return buf
        cells = _get_block(self.engine, self.comm, i0 * W * n, m)
        zu, zv = self.engine.get_zones(i0, count)
        return np.concatenate([np.asarray(cells).reshape(-1), zu, zv])

    @property
    def engine_model_n(self):
        return self.engine.model.n_nodes

    def refresh(self):
        if not self.H:
            return
        H, W, n = self.H, self.W, self.engine_model_n
        P, r = self.comm.world, self.comm.rank
        own = self.hi - self.lo
        left, right = (r - 1) % P, (r + 1) % P
        # my first H owned zones go left (they are its right halo), my last H go right
        first = self._zone_block(H, H)
        last = self._zone_block(own, H)
        size = int(first.shape[0])
        if left == right:   # two ranks: both messages go to the same peer; ship them together
            both = (self.comm.tensor(first), self.comm.tensor(last))
            import torch
            got = self.comm.exchange({left: torch.cat(both)}, {left: (2 * size,)})[left]
            from_right, from_left = got[:size], got[size:]
        else:
            got = self.comm.exchange({left: first, right: last}, {left: (size,), right: (size,)})
            from_left, from_right = got[left], got[right]
        self._set_zone_block(0, H, from_left)                   # left halo <- left's last owned
        self._set_zone_block(H + own, H, from_right)            # right halo <- right's first owned

    def _set_zone_block(self, i0, count, flat):
        n, W = self.engine_model_n, self.W
        m = count * W * n
        _set_block(self.engine, i0 * W * n, flat[:4 * m].reshape(4, m))
        z = flat[4 * m:4 * m + 2 * count].reshape(2, count)
        if getattr(z, "is_cuda", False) and hasattr(self.engine, "set_zones_from"):
            self.engine.set_zones_from(i0, z.contiguous())
        else:
            z = z.cpu().numpy() if hasattr(z, "cpu") else z
            self.engine.set_zones(i0, z[0], z[1])

    def owned_state(self) -> dict:
        n, W = self.engine_model_n, self.W
        own = self.hi - self.lo
        out = self.engine.get_cells(self.H * W * n, own * W * n)
        out["zone_u"], out["zone_v"] = self.engine.get_zones(self.H, own)
        return out
