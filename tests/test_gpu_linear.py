"""df_step_linear (wall.cpp:60-71, the paper's single-field DF form, Eq. 8;
boundary nodes copied) on the device (hyg_df_march_linear): a batch of
fields marched with layer rotation equals the C oracle's statement-for-
statement restatement bit for bit (same IEEE operations, no contraction),
across lambda decades (the reference's boundedness test, test_wall.cpp:251-272)."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_1703_10119_b200 import api

pytestmark = pytest.mark.gpu


def _oracle(prev, curr, lam, steps):
    lib = O.oracle_lib()
    p, c = prev.copy(), curr.copy()
    nxt = np.empty(p.shape[1])
    dp = C.POINTER(C.c_double)
    for f in range(p.shape[0]):
        a, b = p[f].copy(), c[f].copy()
        for _ in range(steps):
            lib.orc_df_step_linear(a.size, a.ctypes.data_as(dp), b.ctypes.data_as(dp), lam, nxt.ctypes.data_as(dp))
            a, b = b, nxt.copy()
        p[f], c[f] = a, b
    return p, c


@pytest.mark.parametrize("lam", [0.01, 0.5, 1.0, 7.0, 100.0])
def test_df_linear_bitwise(lam):
    rng = np.random.default_rng(int(lam * 100))
    prev = 1.0 + rng.normal(0, 0.1, (6, 101))
    curr = prev + rng.normal(0, 0.01, prev.shape)
    gp, gc = api.df_march_linear(prev, curr, lam, 500)
    op, oc = _oracle(prev, curr, lam, 500)
    assert np.array_equal(gp, op) and np.array_equal(gc, oc)
    assert np.abs(gc).max() <= np.abs(curr).max() * (1 + 1e-12) + 1.0   # bounded (DF is unconditionally stable)


def test_df_linear_printed_coefficients():
    """The reference's known answers (test_wall.cpp:43-61), one device step each."""
    def step(prev, curr, lam):
        return api.df_march_linear(np.array([prev]), np.array([curr]), lam, 1)[1][0]
    assert step([0.3, 9.9, 0.1], [0.0, 1.0, 2.0], 1.0)[1] == pytest.approx(1.0)       # (0 + 2)/2
    assert np.allclose(step([3.25] * 5, [3.25] * 5, 0.7), 3.25, rtol=1e-15, atol=0)  # fixed point
    assert step([0, 0, 0], [0, 1, 0], 0.5)[1] == pytest.approx(0.0)
    assert step([0.1, 0.2, 0.3], [0.4, 0.5, 0.6], 0.5)[1] == pytest.approx((1 / 3) * 0.2 + (1 / 3) * (0.4 + 0.6),
                                                                           rel=1e-15)
