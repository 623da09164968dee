"""The C++ drop-in (include/hygro_b200.hpp: hygro::gpu::run) against the
reference's own hygro::run on the same hygro::BuildingModel (one zone and a
3-zone ring with schedules, init profiles, frames, and a divergence case),
via oracle/_ref/adapter_check built from the reference sources."""
import subprocess

import pytest

from .conftest import ROOT

pytestmark = pytest.mark.gpu

EXE = ROOT / "oracle" / "_ref" / "adapter_check"


@pytest.mark.skipif(not EXE.exists(), reason="adapter_check not built (needs /root/reference at build time)")
def test_cpp_dropin_matches_reference_run():
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
