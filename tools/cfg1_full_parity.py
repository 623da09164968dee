"""configs[1] with EVERY wall at the full horizon: 65,536 walls x 256 nodes x 1e5 steps through K1
against the C oracle's threaded march (the suite checks 1,113 walls at the full horizon and all
walls at 1e3 steps).  ~10 minutes of host time on 16 threads, so it is a one-off check whose
output is kept under profiles/, not a test of the suite.   Also configs[2] (fp32, variable dt)
with every wall when called with `cfg2`.

  python tools/cfg1_full_parity.py [cfg1|cfg2]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1703_10119_b200 import workloads       # noqa: E402
from paper_1703_10119_b200.api import Model       # noqa: E402
from tests.helpers import gpu_run, oracle_run, rel_linf    # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    w = workloads.batched_walls() if cfg == "cfg1" else workloads.batched_walls(precision="f32", variable_dt=True)
    t0 = time.perf_counter()
    kw = {"dt_schedule": w.dt_schedule} if w.dt_schedule else {}
    got = gpu_run(w.model, w.init, w.nsteps, w.boot, w.tables, **kw)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    m = w.model
    ref_model = m if cfg == "cfg1" else Model(m.n_nodes, m.dx, m.groups, m.biot, m.attach, channels=m.channels,
                                              dt=m.dt, divergence_norm=m.divergence_norm)   # the fp64 oracle
    ref = oracle_run("oracle", ref_model, w.init, w.nsteps, w.boot, w.tables, **kw)
    t_cpu = time.perf_counter() - t0
    err = rel_linf(got, ref)
    tol = 1e-10 if cfg == "cfg1" else 1e-4
    print(f"{cfg} all {w.model.n_walls} walls x {w.nsteps} steps: rel L-inf {err:.3e} (tolerance {tol:g}); "
          f"GPU {t_gpu:.1f} s, oracle {t_cpu:.1f} s")
    assert err <= tol


if __name__ == "__main__":
    main()
