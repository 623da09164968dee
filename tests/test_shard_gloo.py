"""Multi-rank decomposition (paper_1703_10119_b200/shard.py) on CPU ranks over
gloo, with the C oracle as the per-rank engine: the sharded march must equal
the undivided one bit for bit (long-domain x-slabs, zone-ring blocks with the
joint implicit start), for 2 and 3 ranks."""
import os
import socket
import sys
import traceback

import numpy as np
import pytest
import torch.multiprocessing as mp

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
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle as O
        from oracle.engine import OracleEngine
        from paper_1703_10119_b200 import shard, workloads
        comm = shard.Comm()
        if case == "long":
            n, steps, halo = 4096, 150, 16
            w = workloads.long_domain(n_nodes=n, nsteps=steps)
            sh = shard.LongDomainShard(w.model, w.init, comm, OracleEngine, halo=halo)
            sh.advance(steps)
            got = sh.owned_state()
            eng = OracleEngine(w.model)
            eng.set_state(**{f: w.init[f] for f in FIELDS})
            eng.advance(steps)
            s = sh.slab
            ok = all(np.array_equal(got[f], eng.state[f][s.lo:s.hi]) for f in FIELDS)
        else:
            Z, W, n, steps, halo = 16, 6, 16, 40, 4
            wz = workloads.zone_ring(n_zones=Z, walls_per_zone=W, n_nodes=n, nsteps=steps)
            rng = np.random.default_rng(3)
            init = {f: wz.init[f] + 1e-3 * rng.standard_normal(wz.init[f].size) for f in FIELDS}
            init.update(zone_u=wz.init["zone_u"], zone_v=wz.init["zone_v"])
            sh = shard.ZoneRingShard(wz.model, init, comm, OracleEngine, walls_per_zone=W, halo=halo)
            st = sh.bootstrap("implicit")
            sh.advance(steps - 1)
            got = sh.owned_state()
            b = O.Building(wz.model, init)
            rc, _, passes = b.run("oracle", steps)
            assert rc == 0 and passes == st.subiterations, (passes, st.subiterations)
            c0, c1 = sh.lo * W * n, sh.hi * W * n
            ok = all(np.array_equal(got[f], b.state[f][c0:c1]) for f in FIELDS)
            ok = ok and np.array_equal(got["zone_u"], b.zu[sh.lo:sh.hi]) and \
                np.array_equal(got["zone_v"], b.zv[sh.lo:sh.hi])
        dist.destroy_process_group()
        q.put((rank, bool(ok), ""))
    except Exception:
        q.put((rank, False, traceback.format_exc()))


@pytest.mark.parametrize("case,world", [("long", 2), ("long", 3), ("ring", 2), ("ring", 3)])
def test_sharded_march_is_bitwise_equal(case, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in sorted(results):
        assert ok, f"rank {rank}: {err}"
