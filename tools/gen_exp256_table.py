"""Generate paper_1703_10119_b200/csrc/hyg_exp256_table.h: 2^(j/256), j = 0..255,
correctly rounded doubles from 60-digit arithmetic (mpmath)."""
from pathlib import Path

import mpmath as mp

mp.mp.dps = 60
vals = [float(mp.mpf(2) ** (mp.mpf(j) / 256)).hex() for j in range(256)]
rows = ["    " + ", ".join(vals[i:i + 4]) + ("," if i + 4 < 256 else "") + " \\" for i in range(0, 256, 4)]
out = ("// hyg_exp256_table.h — 2^(j/256), j = 0..255, correctly rounded (generated with\n"
       "// 60-digit arithmetic: tools/gen_exp256_table.py)\n#pragma once\n#define HYG_EXP2_TAB256 { \\\n"
       + "\n".join(rows) + "\n}\n")
Path(__file__).resolve().parents[1].joinpath("paper_1703_10119_b200/csrc/hyg_exp256_table.h").write_text(out)
