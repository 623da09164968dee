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
