"""Smallest cases of every hand-written kernel family, for compute-sanitizer
(racecheck / synccheck / memcheck): K1, K2h, K3w (persistent + prefetch), K4r
and K5 (zone ring, grid capped so each CTA walks several blocks), the
material step.  Each case is also checked against the oracle loosely (the
sanitizer run is about hazards, the parity tests are elsewhere).

  compute-sanitizer --tool racecheck python tools/sanitize_target.py [case ...]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1703_10119_b200 import Context, workloads   # noqa: E402


def run(w, steps, tuning=(), boot=None):
    with Context(w.model) as ctx:
        for k, v in tuning:
            ctx.set_tuning(k, v)
        for ch, (first, tab) in w.tables.items():
            ctx.set_channel_table(ch, first, tab)
        ctx.set_state(**w.init)
        ctx.profiling(True)
        b = boot or w.boot
        if b != "none":
            ctx.bootstrap(b)
        ctx.advance(steps - (0 if b == "none" else 1))
        ctx.synchronize()
        names = sorted(s["name"] for s in ctx.kernel_stats())
    return names


CASES = {
    "k1": lambda: run(workloads.batched_walls(n_walls=64, n_nodes=256, nsteps=40), 40),
    "k2h": lambda: run(workloads.single_wall_d(nsteps=60), 60),
    "k3w": lambda: run(workloads.long_domain(n_nodes=1 << 15, nsteps=40), 40),
    "k5": lambda: run(workloads.zone_ring(n_zones=13, walls_per_zone=6, n_nodes=128, nsteps=40), 40,
                      (("ring_grid", 2),)),
    "k4r": lambda: run(workloads.zone_ring(n_zones=13, walls_per_zone=6, n_nodes=128, nsteps=30), 30,
                       (("ring_grid", 2), ("ring_kernel", 1))),
    "material": lambda: run(workloads.material_walls(n_walls=8, n_nodes=51, nsteps=20), 20),
}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        print(name, CASES[name](), flush=True)
