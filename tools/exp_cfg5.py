"""Timing experiment: why is the snapshot-restore loop slower than the
set_state/get_state loop on the material path?  Alternates variants."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1703_10119_b200 import Context, workloads   # noqa: E402

w = workloads.material_walls(n_walls=16384, n_nodes=101, nsteps=1000)
ctx = Context(w.model)
ctx.set_state(**w.init)
ctx.snapshot()
host = {k: np.ascontiguousarray(v) for k, v in w.init.items()}
out = {k: np.empty_like(host[k]) for k in ("u_prev", "u_curr", "v_prev", "v_curr")}


def run(kind):
    ctx.synchronize()
    ctx.record(0)
    t = time.perf_counter()
    if kind == "restore":
        ctx.restore()
    elif kind == "set":
        ctx.set_state(**host)
    ctx.bootstrap("implicit")
    ctx.advance(w.nsteps - 1)
    if kind == "set":
        ctx.get_state(out)
    ctx.record(1)
    ctx.synchronize()
    return ctx.elapsed_ms(0, 1), 1e3 * (time.perf_counter() - t)


for rep in range(3):
    for kind in ("restore", "set", "none", "restore", "set"):
        ms, wall = run(kind)
        print(f"{kind:8s} events {ms:8.1f} ms  host {wall:8.1f} ms", flush=True)
ctx.reset_kernel_stats()
ctx.profiling(True)
run("restore")
ctx.synchronize()
ctx.profiling(False)
for s in ctx.kernel_stats():
    print(s)
