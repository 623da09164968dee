"""Where does a configs[1] run spend its time outside K1?  Per-kernel events
+ host timing of each API phase, several runs."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1703_10119_b200 import Context, workloads   # noqa: E402

w = workloads.batched_walls()
ctx = Context(w.model)
for ch, (first, tab) in w.tables.items():
    ctx.set_channel_table(ch, first, tab)
ctx.set_state(**w.init)
ctx.snapshot()
for rep in range(4):
    ctx.reset_kernel_stats()
    ctx.profiling(rep % 2 == 1)
    ctx.synchronize()
    t0 = time.perf_counter()
    ctx.record(0)
    ctx.restore()
    t1 = time.perf_counter()
    ctx.bootstrap("implicit")
    ctx.synchronize()
    t2 = time.perf_counter()
    ctx.advance(w.nsteps - 1)
    ctx.record(1)
    ctx.synchronize()
    t3 = time.perf_counter()
    print(f"run {rep}: events {ctx.elapsed_ms(0, 1):8.1f} ms | host restore {1e3*(t1-t0):6.1f} boot {1e3*(t2-t1):6.1f} "
          f"advance {1e3*(t3-t2):8.1f} ms", flush=True)
    if rep % 2 == 1:
        for s in ctx.kernel_stats():
            print("   ", s)
    ctx.profiling(False)
