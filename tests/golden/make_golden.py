"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run here, where /root/reference exists:  python tests/golden/make_golden.py
The fixtures pin the C oracle (tests/test_oracle_golden.py) and the CUDA
path (tests/test_gpu_golden.py) on boxes where the reference is absent.
Every fixture stores its inputs (model parameters, forcing rows, initial
layers) and the reference's outputs.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle as O                                   # noqa: E402
from paper_1703_10119_b200 import workloads           # noqa: E402
from tests.helpers import FIELDS, oracle_run, random_walls   # noqa: E402

OUT = Path(__file__).resolve().parent


def save_walls(name, model, init, nsteps, boot, tables=None, dt_schedule=None, note=""):
    ref = oracle_run("ref", model, init, nsteps, boot, tables, nthreads=O.threads(), dt_schedule=dt_schedule)
    dts = (np.concatenate([np.full(n, d) for n, d in dt_schedule])[:nsteps] if dt_schedule
           else np.full(nsteps, model.dt))
    times = workloads.accumulate_times(dts)
    tab = O.forcing_table(model, times, 0, tables or {})
    np.savez_compressed(OUT / f"{name}.npz", n_nodes=model.n_nodes, dx=model.dx, dt=model.dt,
                        groups=model.groups, biot=model.biot, attach=model.attach, table=tab, dts=dts,
                        nsteps=nsteps, boot=boot, coeff_kind=model.coeff_kind,
                        coeff_params=np.array(model.coeff_params),
                        **{f"init_{k}": init[k] for k in FIELDS}, **{f"ref_{k}": ref[k] for k in FIELDS},
                        note=note)
    print(name, "saved", {k: float(np.abs(ref[k]).max()) for k in FIELDS})


def main():
    assert O.ref_lib() is not None, "needs oracle/_ref (make -C oracle ref)"
    # 1. coupled walls with imposed fluxes, 3 channels, N=21 (df_step_coupled)
    m, init = random_walls(12, 21, seed=11, flux=True, channels=3)
    save_walls("coupled_flux_n21", m, init, 800, "implicit", note="df_step_coupled wall.cpp:144-194")
    # 2. cfg1 sample: 16 cfg1 walls (N=256), implicit start + 1999 DF steps
    w = workloads.batched_walls(n_walls=16, nsteps=2000, seed=7)
    save_walls("cfg1_sample16", w.model, w.init, 2000, "implicit", w.tables, note="configs[1] shape")
    # 3. cfg0 through the reference's transcription oracle (df_oracle.hpp), 5000 steps
    w0 = workloads.single_wall_d(nsteps=5000)
    save_walls("cfg0_5000", w0.model, w0.init, 5000, "explicit",
               note="d(v) through tests/support/df_oracle.hpp (fixed-point face rows)")
    # 4. cfg2 schedule shape in fp64 (variable dt per call), 8 walls x 64 nodes
    m2, init2 = random_walls(8, 64, seed=12)
    save_walls("vardt_n64", m2, init2, 1200, "implicit", dt_schedule=[(400, 1e-3), (400, 2e-3), (400, 4e-3)])
    # 5. building (one zone, 4 walls, N=101; two zones ring 6 walls N=16) via run()'s loop
    for name, (nz, wpz, n, steps) in {"building_one_zone": (1, 4, 101, 600),
                                      "building_ring3": (3, 6, 16, 600)}.items():
        wz = workloads.zone_ring(n_zones=nz, walls_per_zone=wpz, n_nodes=n, nsteps=steps)
        rng = np.random.default_rng(5)
        init = {k: wz.init[k] + 1e-3 * rng.standard_normal(wz.init[k].size) for k in FIELDS}
        init.update(zone_u=wz.init["zone_u"], zone_v=wz.init["zone_v"])
        b = O.Building(wz.model, init)
        rc, fl, passes = b.run("ref", steps)
        assert rc == 0
        np.savez_compressed(OUT / f"{name}.npz", n_zones=nz, walls_per_zone=wpz, n_nodes=n, nsteps=steps,
                            passes=passes, **{f"init_{k}": init[k] for k in FIELDS},
                            **{f"ref_{k}": b.state[k] for k in FIELDS}, ref_zone_u=b.zu, ref_zone_v=b.zv,
                            ref_t=b.s.t)
        print(name, "saved, bootstrap passes", passes)
    # 6. df_step_linear hand-checkable vectors (test_wall.cpp:43-61) + random
    lib = O.ref_lib()
    import ctypes as C
    rng = np.random.default_rng(2)
    prev, curr = rng.uniform(0.9, 1.1, 33), rng.uniform(0.9, 1.1, 33)
    out = {}
    for lam in (0.1, 0.5, 1.0, 10.0, 100.0):
        nxt = np.empty(33)
        p = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
        lib.ref_df_step_linear(33, p(prev), p(curr), lam, p(nxt))
        out[f"next_{lam}"] = nxt
    np.savez_compressed(OUT / "df_step_linear.npz", prev=prev, curr=curr, **out)
    print("df_step_linear saved")


if __name__ == "__main__":
    main()
