"""configs[0] march time with the library or a timing variant (tools/_ringvar)."""
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1703_10119_b200 import Context, api, workloads   # noqa: E402

if len(sys.argv) > 1:
    api.load_library(sys.argv[1])
w = workloads.single_wall_d(nsteps=100_000)
with Context(w.model) as ctx:
    for ch, (first, tab) in w.tables.items():
        ctx.set_channel_table(ch, first, tab)
    ctx.set_state(**w.init)
    ctx.snapshot()
    for rep in range(3):
        ctx.restore()
        ctx.synchronize()
        t0 = time.perf_counter()
        ctx.bootstrap(w.boot)
        ctx.advance(w.nsteps - 1)
        ctx.synchronize()
        dt = time.perf_counter() - t0
    print(f"{sys.argv[1] if len(sys.argv) > 1 else 'library'}: {dt * 1e3:.1f} ms for 1e5 steps, "
          f"{dt / 1e5 * 1.965e9:.0f} cycles/step at 1965 MHz")
