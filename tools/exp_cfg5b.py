"""Per-run kernel-time sum vs elapsed (gaps vs slow kernels) + 20 ms NVML clocks."""
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1703_10119_b200 import Context, workloads   # noqa: E402
import pynvml as N   # noqa: E402

N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def poll():
    while not stop.is_set():
        samples.append((time.time(), N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM),
                        N.nvmlDeviceGetPowerUsage(h) / 1000, N.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
        time.sleep(0.02)


threading.Thread(target=poll, daemon=True).start()
w = workloads.material_walls(n_walls=16384, n_nodes=101, nsteps=1000)
ctx = Context(w.model)
ctx.set_state(**w.init)
ctx.snapshot()
for rep in range(8):
    prof = rep % 2 == 0
    ctx.reset_kernel_stats()
    ctx.profiling(prof)
    ctx.synchronize()
    t0 = time.time()
    ctx.record(0)
    ctx.restore()
    ctx.bootstrap("implicit")
    ctx.advance(w.nsteps - 1)
    ctx.record(1)
    ctx.synchronize()
    t1 = time.time()
    ctx.profiling(False)
    ks = sum(s["ms"] for s in ctx.kernel_stats()) if prof else float("nan")
    win = [s for s in samples if t0 <= s[0] <= t1]
    clk = sorted(x[1] for x in win)
    print(f"run {rep} prof={prof} elapsed {ctx.elapsed_ms(0, 1):7.1f} ms kernel-sum {ks:7.1f} ms "
          f"sm MHz min/med {clk[0] if clk else 0}/{clk[len(clk)//2] if clk else 0} "
          f"power max {max((x[2] for x in win), default=0):.0f} W reasons {sorted({x[3] for x in win})}", flush=True)
stop.set()
