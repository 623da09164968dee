"""configs[3] at its BASELINE shape AND full horizon: 8,192 zones x 6 walls x 128 nodes x 8e4 steps
through the default zone-ring path (K6) against the C oracle's threaded building run (bitwise its
serial run, tests/test_oracle_mt.py).  Minutes of host time, so it is a one-off check whose output
is kept under profiles/, not a test of the suite.

  python tools/cfg3_full_parity.py [steps]
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import oracle as O                                         # noqa: E402
from paper_1703_10119_b200 import Context, workloads       # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 80_000
    w = workloads.zone_ring(n_zones=8192, walls_per_zone=6, n_nodes=128, nsteps=steps)
    rng = np.random.default_rng(8192)
    keys = ("u_prev", "u_curr", "v_prev", "v_curr")
    init = {k: v + (2e-3 * rng.standard_normal(v.size) if k in keys else 0) for k, v in w.init.items()}
    t0 = time.perf_counter()
    with Context(w.model) as ctx:
        ctx.set_state(**init)
        ctx.profiling(True)
        st = ctx.bootstrap("implicit")
        ctx.advance(steps - 1)
        ctx.synchronize()
        stats = {s["name"]: s["launches"] for s in ctx.kernel_stats()}
        got = ctx.get_state()
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    b = O.Building(w.model, init)
    rc, _, passes = b.run("oracle", steps, nthreads=O.threads())
    t_cpu = time.perf_counter() - t0
    assert rc == 0 and st.subiterations == passes, (rc, st.subiterations, passes)
    ref = max(float(np.max(np.abs(b.state[k]))) for k in keys)
    err = max(float(np.max(np.abs(got[k] - b.state[k]))) for k in keys) / ref
    zref = max(float(np.max(np.abs(b.zu[:8192]))), float(np.max(np.abs(b.zv[:8192]))))
    zerr = max(float(np.max(np.abs(got["zone_u"] - b.zu[:8192]))), float(np.max(np.abs(got["zone_v"] - b.zv[:8192])))) / zref
    print(f"cfg3 full shape x {steps} steps: rel L-inf walls {err:.3e}, zones {zerr:.3e} "
          f"(tolerance 1e-10); launches {stats}; GPU {t_gpu:.1f} s (profiling on), oracle {t_cpu:.1f} s on {O.threads()} threads")
    assert err <= 1e-10 and zerr <= 1e-10


if __name__ == "__main__":
    main()
