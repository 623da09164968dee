"""Minimal profiling target (no nvidia-smi child, no CPU legs): one run of a
config's hot path, for ncu launch lists and --set full captures.

  python tools/profile_target.py cfg1 [steps [ring_kernel [prof]]]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1703_10119_b200 import Context, workloads   # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4097
    if cfg == "cfg1":
        w = workloads.batched_walls(nsteps=steps)
    elif cfg == "cfg2":
        w = workloads.batched_walls(nsteps=steps, precision="f32")
    elif cfg == "cfg0":
        w = workloads.single_wall_d(nsteps=steps)
    elif cfg == "cfg3":
        w = workloads.zone_ring(nsteps=steps)
    elif cfg == "cfg5":
        w = workloads.material_walls(n_walls=16384, n_nodes=101, nsteps=steps)
    else:
        w = workloads.long_domain(nsteps=steps)
    with Context(w.model) as ctx:
        if len(sys.argv) > 3:                       # cfg3: zone-ring kernel (HYG_TUNE_RING_KERNEL)
            ctx.set_tuning("ring_kernel", int(sys.argv[3]))
        prof = len(sys.argv) > 4                    # per-kernel CUDA-event times
        if prof:
            ctx.profiling(True)
        for ch, (first, tab) in w.tables.items():
            ctx.set_channel_table(ch, first, tab)
        ctx.set_state(**w.init)
        t0 = time.perf_counter()
        if w.boot != "none":
            ctx.bootstrap(w.boot)
        ctx.advance(w.nsteps - (0 if w.boot == "none" else 1))
        ctx.synchronize()
        print(f"{cfg}: {w.nsteps} steps in {time.perf_counter() - t0:.3f} s, {ctx.launches} launches")
        if prof:
            for s in ctx.kernel_stats():
                print(f"  {s['name']:28s} {s['launches']:6d} launches  {s['ms']:10.3f} ms  "
                      f"{1e3 * s['ms'] / max(1, s['launches']):9.2f} us/launch")


if __name__ == "__main__":
    main()
