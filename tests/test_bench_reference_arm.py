"""bench.py --impl reference (the reference arm) runs the reference's own CPU
path through oracle/_ref/ref_bench and never imports this package or loads
its CUDA library (so the driver's vs_reference ratio compares the unmodified
reference with the GPU arm)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

PROBE = r"""
import runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "{cfg}",
            "--walls", "256", "--zones", "16"]
try:
    runpy.run_path("bench.py", run_name="__main__")
except SystemExit:
    pass
maps = open("/proc/self/maps").read()
print("AUDIT", [m for m in sys.modules if m.startswith("paper_1703_10119_b200") or m == "oracle"],
      "libhygro_b200.so" in maps)
"""


@pytest.mark.parametrize("cfg", ["cfg0", "cfg1", "cfg3"])
def test_reference_arm_is_package_free(cfg):
    if not (ROOT / "oracle" / "_ref" / "ref_bench").exists():
        pytest.skip("oracle/_ref/ref_bench not built (no /root/reference)")
    r = subprocess.run([sys.executable, "-c", PROBE.format(cfg=cfg)], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    lines = r.stdout.strip().splitlines()
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["value"] > 0, line
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["implicit_value"] > 0
    assert lines[-1] == "AUDIT [] False", lines[-1]
