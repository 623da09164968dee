"""CUDA path vs the reference's own outputs stored in tests/golden/ (made by
make_golden.py from the unmodified reference library)."""
import numpy as np
import pytest

from paper_1703_10119_b200 import Context, workloads
from paper_1703_10119_b200.api import ChannelSpec

from .helpers import FIELDS, rel_linf
from .test_oracle_golden import load, model_from

pytestmark = pytest.mark.gpu


def _gpu_replay(g):
    nch = g["table"].shape[1]
    m = model_from(g, [ChannelSpec() for _ in range(nch)])
    init = {k: g[f"init_{k}"] for k in FIELDS}
    tab, dts, nsteps = g["table"], g["dts"], int(g["nsteps"])
    with Context(m) as ctx:
        ctx.set_state(**init)
        for c in range(nch):     # the stored forcing rows drive every channel
            ctx.set_channel_table(c, 0, tab[:, c, :])
        ctx.bootstrap(str(g["boot"]))
        L = 1
        while L < nsteps:
            d, n = dts[L], 1
            while L + n < nsteps and dts[L + n] == d:
                n += 1
            ctx.advance(n, float(d))
            L += n
        return ctx.get_state()


@pytest.mark.parametrize("name", ["coupled_flux_n21", "cfg1_sample16", "vardt_n64", "cfg0_5000"])
def test_gpu_matches_reference_goldens(name):
    g = load(name)
    got = _gpu_replay(g)
    err = rel_linf(got, {k: g[f"ref_{k}"] for k in FIELDS})
    assert err <= 1e-10, err


@pytest.mark.parametrize("name", ["building_one_zone", "building_ring3"])
def test_gpu_building_goldens(name):
    g = load(name)
    w = workloads.zone_ring(n_zones=int(g["n_zones"]), walls_per_zone=int(g["walls_per_zone"]),
                            n_nodes=int(g["n_nodes"]), nsteps=int(g["nsteps"]))
    with Context(w.model) as ctx:
        ctx.set_state(**{k: g[f"init_{k}"] for k in FIELDS}, zone_u=w.init["zone_u"], zone_v=w.init["zone_v"])
        st = ctx.bootstrap("implicit")
        ctx.advance(int(g["nsteps"]) - 1)
        got = ctx.get_state()
    assert st.subiterations == int(g["passes"])
    assert rel_linf(got, {k: g[f"ref_{k}"] for k in FIELDS}) <= 1e-10
    assert np.max(np.abs(got["zone_u"] - g["ref_zone_u"])) <= 1e-10
    assert np.max(np.abs(got["zone_v"] - g["ref_zone_v"])) <= 1e-10
    assert got["t"] == float(g["ref_t"])
