"""Per-launch time of K4r (k_ring_reg) as a function of steps per launch:
t(k) - t(1) over k - 1 is the per-step cost, t(1) the per-block overhead."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1703_10119_b200 import Context, api, workloads   # noqa: E402

if len(sys.argv) > 1:          # a timing variant of the library (tools/_ringvar)
    api.load_library(sys.argv[1])
    print("library", sys.argv[1])

w = workloads.zone_ring(nsteps=100)
with Context(w.model) as ctx:
    ctx.set_state(**w.init)
    ctx.bootstrap("implicit")
    ctx.advance(64)
    ctx.synchronize()
    for k in (1, 2, 4, 8):
        ctx.reset_kernel_stats()
        ctx.profiling(True)
        for _ in range(20):
            ctx.advance(k)
        ctx.synchronize()
        st = {s["name"]: s for s in ctx.kernel_stats()}
        ctx.profiling(False)
        for name in ("ring_reg", "ring_tiled"):
            if name in st and st[name]["launches"]:
                s = st[name]
                print(f"{name} steps/launch {k}: {s['ms'] / s['launches'] * 1e3:.1f} us per launch")
