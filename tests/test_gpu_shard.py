"""The multi-GPU decomposition (shard.py) with the CUDA engine, two ranks on
one device (the halo exchange is host-staged over gloo, so no kernel ever
waits on another rank's kernel): the sharded long wall (temporally blocked
kernel) and the sharded zone ring (joint implicit start reduced across ranks)
must equal the undivided GPU run bit for bit."""
import os
import socket
import sys
import traceback

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

FIELDS = ("u_prev", "u_curr", "v_prev", "v_curr")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1703_10119_b200 import Context, shard, workloads
        comm = shard.Comm()
        if case == "long":
            n, steps = 1 << 16, 200
            w = workloads.long_domain(n_nodes=n, nsteps=steps)
            sh = shard.LongDomainShard(w.model, w.init, comm, Context, halo=40)
            sh.advance(steps)
            got = sh.owned_state()
            with Context(w.model) as ref:
                ref.set_state(**w.init)
                ref.advance(steps)
                full = ref.get_state()
            s = sh.slab
            ok = all(np.array_equal(got[f], full[f][s.lo:s.hi]) for f in FIELDS)
        else:
            Z, W, n, steps = 16, 6, 32, 300
            wz = workloads.zone_ring(n_zones=Z, walls_per_zone=W, n_nodes=n, nsteps=steps)
            rng = np.random.default_rng(3)
            init = {f: wz.init[f] + 1e-3 * rng.standard_normal(wz.init[f].size) for f in FIELDS}
            init.update(zone_u=wz.init["zone_u"], zone_v=wz.init["zone_v"])
            sh = shard.ZoneRingShard(wz.model, init, comm, Context, walls_per_zone=W, halo=4)
            sh.bootstrap("implicit")
            sh.advance(steps - 1)
            got = sh.owned_state()
            with Context(wz.model) as ref:
                ref.set_state(**init)
                ref.bootstrap("implicit")
                ref.advance(steps - 1)
                full = ref.get_state()
            c0, c1 = sh.lo * W * n, sh.hi * W * n
            ok = all(np.array_equal(got[f], full[f][c0:c1]) for f in FIELDS)
            ok = ok and np.array_equal(got["zone_u"], full["zone_u"][sh.lo:sh.hi])
        sh.engine.close()
        dist.destroy_process_group()
        q.put((rank, bool(ok), ""))
    except Exception:
        q.put((rank, False, traceback.format_exc()))


@pytest.mark.parametrize("case", ["long", "ring"])
def test_two_ranks_one_device_bitwise(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in sorted(results):
        assert ok, f"rank {rank}: {err}"


class _LoopbackComm:
    """Device-payload comm for shards living in threads of one process: what
    an NCCL group does between GPUs (payloads stay CUDA tensors, filled and
    drained device to device by Context.get_cells_into / set_cells_from),
    with a barrier-synchronised mailbox instead of NVLink."""

    def __init__(self, rank, world, hub):
        import torch
        self.rank, self.world, self.hub = rank, world, hub
        self.on_device, self.device = True, torch.device("cuda", 0)

    def tensor(self, a):
        import torch
        if not isinstance(a, torch.Tensor):
            a = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        return a.to(self.device, torch.float64).contiguous()

    def exchange(self, sends, recvs):
        # payloads cross threads AND streams (the shards' exchange streams when the
        # refresh overlaps compute): an event per payload orders the receiver's stream
        # behind the sender's copy, as NCCL orders its transfer behind the pack kernel
        import torch
        box, bar = self.hub
        for peer, a in sends.items():
            t = self.tensor(a)
            assert t.is_cuda
            c = t.clone()
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.device))
            box[(self.rank, peer)] = (c, ev)
        bar.wait()
        out = {}
        for peer in recvs:
            c, ev = box.pop((peer, self.rank))
            torch.cuda.current_stream(self.device).wait_event(ev)
            out[peer] = c
        bar.wait()
        return out

    def _reduce(self, x, f):
        box, bar = self.hub
        box[("r", self.rank)] = x
        bar.wait()
        v = f(box[("r", r)] for r in range(self.world))
        bar.wait()
        return v

    def allreduce_max(self, x):
        return self._reduce(x, max)

    def allreduce_min(self, x):
        return self._reduce(x, min)


@pytest.mark.parametrize("case", ["long", "long_serial", "ring", "ring128", "ring128k4r", "ring128k5"])
def test_device_payload_exchange_bitwise(case):
    """Halo payloads as CUDA tensors (the NCCL path of shard.Comm: one pack
    kernel, stream-ordered, no host copies): shards in two threads equal the
    undivided run bit for bit.  long: the halo refresh runs on a second stream
    and overlaps the interior windows of the next interval's first launch
    (hyg_advance_overlapped); long_serial: the same on one stream.  ring128: 128-node walls, so each shard marches
    its zone block (a chain with halo zones) through the zone-ring kernel K4r
    (ring128k5: K5)."""
    import threading
    import torch
    from paper_1703_10119_b200 import Context, shard, workloads
    world = 2
    hub = ({}, threading.Barrier(world))
    res, errs = {}, []
    if case.startswith("long"):
        n, steps = 1 << 15, 120
        w = workloads.long_domain(n_nodes=n, nsteps=steps)
        model, init = w.model, w.init
    else:
        Z, W, n, steps = (16, 6, 32, 120) if case == "ring" else (48, 6, 128, 100)
        w = workloads.zone_ring(n_zones=Z, walls_per_zone=W, n_nodes=n, nsteps=steps)
        rng = np.random.default_rng(5)
        init = {f: w.init[f] + 1e-3 * rng.standard_normal(w.init[f].size) for f in FIELDS}
        init.update(zone_u=w.init["zone_u"], zone_v=w.init["zone_v"])
        model = w.model

    kname = {"ring128k5": "ring_pipe", "ring128k4r": "ring_reg"}.get(case, "ring_walls")   # ring128: K6, the default

    def work(rank):
        try:
            torch.cuda.set_device(0)
            comm = _LoopbackComm(rank, world, hub)
            if case.startswith("long"):
                sh = shard.LongDomainShard(model, init, comm, Context, halo=24, overlap=case == "long")
                assert sh.overlap == (case == "long")
                sh.advance(steps)
            else:
                sh = shard.ZoneRingShard(model, init, comm, Context, walls_per_zone=6, halo=4 if case == "ring" else 12)
                if case.startswith("ring128"):
                    if case == "ring128k5":
                        sh.engine.set_tuning("ring_kernel", 3)  # K5 inside the shards
                    if case == "ring128k4r":
                        sh.engine.set_tuning("ring_kernel", 1)  # K4r inside the shards
                    sh.engine.profiling(True)
                sh.bootstrap("implicit")
                sh.advance(steps - 1)
                if case.startswith("ring128"):
                    sh.engine.synchronize()
                    assert any(x["name"] == kname for x in sh.engine.kernel_stats())
            res[rank] = (sh, sh.owned_state())
        except Exception:
            errs.append(traceback.format_exc())
            hub[1].abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs[0]
    with Context(model) as ref:
        ref.set_state(**init)
        if case.startswith("long"):
            ref.advance(steps)
        else:
            ref.bootstrap("implicit")
            ref.advance(steps - 1)
        full = ref.get_state()
    for rank, (sh, got) in res.items():
        if case.startswith("long"):
            sl = slice(sh.slab.lo, sh.slab.hi)
        else:
            sl = slice(sh.lo * 6 * n, sh.hi * 6 * n)
            assert np.array_equal(got["zone_u"], full["zone_u"][sh.lo:sh.hi])
            assert np.array_equal(got["zone_v"], full["zone_v"][sh.lo:sh.hi])
        for f in FIELDS:
            assert np.array_equal(got[f], full[f][sl]), (rank, f)
        sh.engine.close()


def test_cells_into_device_roundtrip():
    """get_cells_into / set_cells_from with CUDA buffers equal the host-array calls."""
    import torch
    from paper_1703_10119_b200 import Context, workloads
    w = workloads.long_domain(n_nodes=4096, nsteps=10)
    with Context(w.model) as ctx:
        ctx.set_state(**w.init)
        ctx.advance(9)
        host = ctx.get_cells(1000, 300)
        dev = torch.empty((4, 300), dtype=torch.float64, device="cuda:0")
        ctx.get_cells_into(1000, 300, dev)
        for i, f in enumerate(FIELDS):
            assert np.array_equal(dev[i].cpu().numpy(), host[f])
        ctx.set_cells_from(2000, dev)
        back = ctx.get_cells(2000, 300)
        for f in FIELDS:
            assert np.array_equal(back[f], host[f])
