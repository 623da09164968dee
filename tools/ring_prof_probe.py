"""K4r phase stamps (a RING_PROF=1 variant of the library): per block of CTA 0,
cycles spent in each phase of the owned warp 0 and the zone warp."""
import ctypes as C
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
from paper_1703_10119_b200 import Context, api, workloads   # noqa: E402

lib = api.load_library(sys.argv[1])
w = workloads.zone_ring(nsteps=100)
with Context(w.model) as ctx:
    ctx.set_state(**w.init)
    ctx.bootstrap("implicit")
    ctx.advance(64)
    ctx.synchronize()
    for k in (8, 1):
        ctx.advance(k)
        ctx.synchronize()
        buf = (C.c_ulonglong * 512)()
        assert lib.hyg_ring_prof_read(buf, 512) == 0
        a = np.array(buf[:], dtype=np.int64).reshape(32, 16)
        names = ["wait", "stage_rd", "A+prefetch", "B", "steps", "load_cf", "outputs", "end_sync"]
        print(f"--- {k} steps/launch: owned warp 0 (cycles per phase), zone warp")
        for it in range(32):
            r = a[it]
            if r[0] == 0 or r[8] == 0:
                continue
            d = np.diff(r[:9])
            z = [r[10] - r[1], r[11] - r[10], r[12] - r[11]]
            print(f"blk {it:2d} " + " ".join(f"{n}={x}" for n, x in zip(names, d)) + f" | total={r[8] - r[0]}"
                  f" | zone: setup={z[0]} A..B={z[1]} steps={z[2]}")
            if it < 31 and a[it + 1][0]:
                pass
