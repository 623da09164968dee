"""The constant tables of the device exp/log (paper_1703_10119_b200/csrc/
hyg_fastmath.cuh) checked against 60-digit decimal arithmetic on the CPU:
2^(j/64) correctly rounded; the log tables' reciprocals within half an ulp of
1/(1 + j/64) and their logarithms -ln(ic_j) correctly rounded from the stored
reciprocal (the identity flog_pos relies on), entry 64 = (1/2, 0)."""
import re
from decimal import Decimal, getcontext
from pathlib import Path

import numpy as np

SRC = Path(__file__).resolve().parents[1] / "paper_1703_10119_b200" / "csrc" / "hyg_fastmath.cuh"
getcontext().prec = 60


def _table(name_pattern):
    text = SRC.read_text()
    m = re.search(name_pattern + r"[^{]*\{(.*?)\}", text, re.S)
    assert m, name_pattern
    return [float.fromhex(x) for x in re.findall(r"0x[0-9a-fA-F.]+p[+-]\d+", m.group(1))]


def _nearest(d: Decimal) -> float:
    return float(d)   # Decimal -> float rounds to nearest


def test_exp2_table_correctly_rounded():
    tab = _table(r"#define HYG_EXP2_TAB64")
    assert len(tab) == 64
    for j, t in enumerate(tab):
        exact = (Decimal(2) ** (Decimal(j) / 64))
        assert t == _nearest(exact), j


def test_log_tables_consistent():
    ic = _table(r"kLogInvC\[65\] =")
    lc = _table(r"kLogC\[65\] =")
    assert len(ic) == 65 and len(lc) == 65
    assert ic[0] == 1.0 and lc[0] == 0.0 and ic[64] == 0.5 and lc[64] == 0.0
    for j in range(64):
        exact = Decimal(1) / (Decimal(1) + Decimal(j) / 64)
        assert abs(Decimal(ic[j]) - exact) <= Decimal(np.spacing(ic[j])) / 2, j
        if j:
            assert lc[j] == _nearest(-Decimal(ic[j]).ln()), j
