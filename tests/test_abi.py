"""The C ABI library: loads, exports every declared symbol, validates like the
reference (building.cpp:12-52), fails loudly without a device, and its host-side
scaling restates scaling.cpp bit for bit.  No GPU needed."""
import ctypes as C
import math

import numpy as np
import pytest

from paper_1703_10119_b200 import _abi as A
from paper_1703_10119_b200 import api
from paper_1703_10119_b200.api import ChannelSpec, Model, ZoneSpec

from .conftest import ROOT


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_library_exports_every_header_symbol():
    lib = api.load_library()
    declared = A.header_symbols(ROOT / "include" / "hygro_b200.h")
    assert len(declared) >= 28
    missing = [s for s in declared if not hasattr(lib, s)]
    assert missing == []
    # and the binding's prototype table covers the header exactly
    assert sorted(A.PROTOTYPES) == declared
    assert lib.hyg_abi_version() == 3
    assert lib.hyg_strerror(A.HYG_EDIVERGED).decode().startswith("numerical error")


def _model(**kw):
    groups = np.array([[0.1, 0.1, 1.0, 0.01]])
    biot = np.array([[[1.0, 1.0, 0.1], [1.0, 1.0, 0.1]]])
    return Model(11, 0.1, groups, biot, channels=[ChannelSpec()], **kw)


def test_schema_validation_precedes_device_use():
    # a face referencing a zone that does not exist (validate, building.cpp:16-27)
    m = _model()
    m.attach[0, 1] = (A.HYG_FACE_ZONE, 3)
    with pytest.raises(api.SchemaError, match="zone 3"):
        api.Context(m)
    m = _model(dt=0.0)          # building.cpp:14
    with pytest.raises(api.SchemaError):
        api.Context(m)
    m = _model()
    m.zones = [ZoneSpec(0.0, 0.0, 0.0, 0.0, 0, 1, [(5, 1, 1, 1, 1, 1, 1)], [])]
    with pytest.raises(api.SchemaError, match="wall"):
        api.Context(m)
    groups = np.array([[0.1, 0.1, 1.0, 0.01]])
    with pytest.raises(api.InvalidArgument):   # Grid1D::with_nodes needs >= 3 nodes (wall.cpp:14)
        api.Context(Model(2, 0.5, groups, np.ones((1, 2, 3)), channels=[ChannelSpec()]))


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device path")
def test_no_cpu_fallback():
    with pytest.raises(api.CudaError, match="no CPU fallback"):
        api.Context(_model())


def test_scaling_matches_reference_bitwise(ref):
    import oracle as O
    rng = np.random.default_rng(3)
    for _ in range(200):
        r = np.exp(rng.uniform(np.log(1e-12), np.log(1e6), 6))
        L, hT0, hM0, hT1, hM1 = rng.uniform(0.01, 0.5), rng.uniform(1, 30), rng.uniform(1e-8, 1e-6), \
            rng.uniform(1, 30), rng.uniform(1e-8, 1e-6)
        T_i, phi = rng.uniform(275, 320), rng.uniform(0.1, 0.9)
        g, b = api.scale_wall(tuple(r), L, hT0, hM0, hT1, hM1, T_i, phi, 3600.0)
        out = (C.c_double * 10)()
        rc = ref.ref_scale_wall(C.byref(O.Coeffs(*r)), L, hT0, hM0, hT1, hM1, T_i, phi, 3600.0, out)
        assert rc == 0
        assert g + [x for f in b for x in f] == list(out)
    # zones: scale_zone / scale_interzone / attach_wall_to_zone
    for V, ach, inz in [(54.0, 0.5, 0.5), (12.5, 2.0, 0.1), (300.0, 0.0, 3.0)]:
        z = api.scale_zone(V, 1.0, 1005.0, 1960.0, ach)
        s = api.scale_interzone(inz, V, 1.0, 1005.0, 1960.0)
        out = (C.c_double * 10)()
        assert ref.ref_scale_zone(V, 1.0, 1005.0, 1960.0, ach, inz, 293.15, 0.5, 3600.0, out) == 0
        assert [z[k] for k in ("kappa_a_tt1", "g_v", "q_v1", "q_v2", "g_o_per", "q_o_per", "q_h_per")] + list(s) \
            == list(out)
        th = api.attach_wall_to_zone((1.82e-2, 5.89e-9, 7.7e5, 0.294, 1.52e3, 1.59e-2), 18.0, 0.1, V)
        o2 = (C.c_double * 2)()
        assert ref.ref_attach_wall(C.byref(O.Coeffs(1.82e-2, 5.89e-9, 7.7e5, 0.294, 1.52e3, 1.59e-2)), 18.0, 0.1, V,
                                   1.0, 1005.0, 1960.0, 293.15, 0.5, 3600.0, o2) == 0
        assert tuple(o2) == th
    for T in (273.15, 293.15, 313.0, 373.15):
        assert api.saturation_pressure(T) == ref.ref_saturation_pressure(T)
    with pytest.raises(api.DomainError):
        api.saturation_pressure(250.0)
    with pytest.raises(api.ScalingError):   # require_positive (scaling.cpp:9-16)
        api.scale_wall((1, 1, 1, 0.0, 1, 1), 0.1, 1, 1, 1, 1)


def test_signals_match_reference_formula():
    s = api.Signal.sinusoid(1.0, 0.06, 24.0, 3.0)
    assert s(5.0) == 1.0 + 0.06 * math.sin(2.0 * math.pi * (5.0 - 3.0) / 24.0)
    q = api.Signal.schedule(0.5, [(1.0, 2.0, 0.25), (1.5, 3.0, 1.0)])
    assert q(0.5) == 0.5 and q(1.6) == 1.75 and q(2.0) == 1.5 and q(3.0) == 0.5
    import oracle as O
    lib = O.oracle_lib()
    keep = []
    for sig in (api.Signal.sin_squared(1.0, -0.02, 24.0), q, s):
        cs = sig.to_c(keep)
        for t in np.linspace(0, 80, 37):
            assert lib.orc_signal(C.byref(cs), float(t)) == sig(float(t))


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirror (_abi.py) has the same sizes and field offsets as the
    C structs of include/hygro_b200.h (compiled here with gcc)."""
    import subprocess
    import ctypes as C
    from paper_1703_10119_b200 import _abi as A
    structs = {"hyg_model_desc": A.ModelDesc, "hyg_zone_desc": A.ZoneDesc, "hyg_status": A.Status,
               "hyg_signal": A.Signal, "hyg_channel": A.Channel, "hyg_zone_wall_link": A.ZoneWallLink,
               "hyg_interzone_link": A.InterzoneLink, "hyg_radiation_link": A.RadiationLink,
               "hyg_coeff_set": A.CoeffSet, "hyg_zone_sources": A.ZoneSources}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "hygro_b200.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            cf = "from" if fname == "from_" else fname
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {cf}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)],
                   check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True, check=True)
               .stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)
