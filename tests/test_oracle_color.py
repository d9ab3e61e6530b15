"""Pin P23 of the oracle's colour conversion (P:L781-783 colour strategy; reading A35: full-range
ITU-R BT.601).  Closed forms of the standard: white/black/grey map to Cb = Cr = 1/2 and Y = the
grey level, pure red has Y = 0.299 and Cr = 1, pure blue Cb = 1; the inverse round-trips.  CPU."""
import numpy as np

import oracle as O


def test_P23_bt601_closed_forms(oracle_lib):
    cols = np.array([[1, 1, 1], [0, 0, 0], [0.25, 0.25, 0.25], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float).T
    y, cb, cr = O.rgb_to_ycbcr(cols.reshape(3, 6))
    assert np.allclose(y[:3], [1, 0, 0.25], atol=1e-15) and np.allclose(cb[:3], 0.5) and np.allclose(cr[:3], 0.5)
    assert np.allclose(y[3:], [0.299, 0.587, 0.114], atol=1e-15)
    assert abs(cr[3] - 1.0) < 1e-15 and abs(cb[5] - 1.0) < 1e-15            # R - Y = 0.701 = 1.402 / 2
    assert abs(cb[3] - (0.5 - 0.299 / 1.772)) < 1e-15
    rgb = np.random.default_rng(0).uniform(0, 1, (3, 40, 30))
    back = O.ycbcr_to_rgb(*O.rgb_to_ycbcr(rgb))
    assert np.allclose(back, rgb, rtol=0, atol=1e-14)
