"""K5 phase stamps (a RING_PROF=1 variant of the library, tools/build_ringvar.sh
style): per block of CTA 0, cycles of owned warp 0, the zone warp and the
producer warp.

  python tools/ring_pipe_prof.py tools/_ringvar/libhygro_prof.so
"""
import ctypes as C
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
from paper_1703_10119_b200 import Context, api, workloads   # noqa: E402

lib = api.load_library(sys.argv[1])
w = workloads.zone_ring(nsteps=200)
with Context(w.model) as ctx:
    ctx.set_state(**w.init)
    ctx.bootstrap("implicit")
    ctx.advance(48)
    ctx.synchronize()
    ctx.advance(12)
    ctx.synchronize()
    buf = (C.c_ulonglong * 512)()
    assert lib.hyg_ring_prof_read(buf, 512) == 0
    a = np.array(buf[:], dtype=np.int64).reshape(32, 16)
    print("owned warp 0: wait_full stage_rd steps load_cf stores | zone: setup steps | producer: wait_free stage")
    for it in range(32):
        r = a[it]
        if r[0] == 0:
            continue
        o = np.diff(r[0:6])
        print(f"blk {it:2d} own " + " ".join(f"{x:6d}" for x in o) + f" tot={r[5] - r[0]:6d}"
              f" | zone wait_end={r[6] - r[0]:6d} setup={r[7] - r[6]:5d} steps={r[8] - r[7]:6d}"
              f" | prod wait={r[10] - r[9]:6d} stage={r[11] - r[10]:6d} (start {r[9] - r[0]:+d})")
