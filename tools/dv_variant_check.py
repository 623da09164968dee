"""configs[0] final state of a timing variant (tools/_ringvar) against the library, bitwise."""
import subprocess
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1703_10119_b200 import Context, api, workloads   # noqa: E402

if len(sys.argv) > 2:          # child: run one library, save the state
    if sys.argv[1] != "-":
        api.load_library(sys.argv[1])
    w = workloads.single_wall_d(nsteps=20_000)
    with Context(w.model) as ctx:
        for ch, (first, tab) in w.tables.items():
            ctx.set_channel_table(ch, first, tab)
        ctx.set_state(**w.init)
        ctx.bootstrap(w.boot)
        ctx.advance(w.nsteps - 1)
        st = ctx.get_state()
    np.savez(sys.argv[2], **{k: st[k] for k in ("u_prev", "u_curr", "v_prev", "v_curr")})
else:
    subprocess.run([sys.executable, __file__, "-", "/tmp/dv_lib.npz"], check=True)
    subprocess.run([sys.executable, __file__, sys.argv[1], "/tmp/dv_var.npz"], check=True)
    a, b = np.load("/tmp/dv_lib.npz"), np.load("/tmp/dv_var.npz")
    same = all(np.array_equal(a[k], b[k]) for k in a.files)
    print(f"{sys.argv[1]}: bitwise equal to the library: {same}")
