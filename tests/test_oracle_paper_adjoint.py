"""Pin P25 of the oracle's paper-mode adjoint warp (P:L583 'the backward
warping function W_k^* will warp the input SAI from perspective theta_k to theta_0 using
omega_0'; reading A37).  For a constant disparity and integer shifts W_k is a translation, whose
transpose is the inverse translation -- W_k^* must equal W_k^T away from the clamped border and
invert W_k there; W_k^* keeps constants (its weights sum to one); the paper-mode A^T equals the
exact one on the interior in that setting.  CPU only."""
import numpy as np

import oracle as O


def test_P25_backward_warp(oracle_lib):
    H, W = 24, 28
    om = np.full((H, W), 1.0)
    g = np.random.default_rng(9)
    u = g.standard_normal((H, W))
    for dr, dt in ((2.0, -1.0), (-3.0, 2.0), (1.0, 1.0)):
        b = O.apply_WTb(u, om, dr, dt)
        t = O.apply_WT(u, om, dr, dt)
        inner = (slice(4, H - 4), slice(4, W - 4))
        assert np.allclose(b[inner], t[inner], rtol=0, atol=1e-14)           # = W_k^T inside
        fw = O.apply_W(u, om, dr, dt)
        assert np.allclose(O.apply_WTb(fw, om, dr, dt)[inner], u[inner], atol=1e-14)   # inverts W_k
        assert np.allclose(O.apply_WTb(np.full((H, W), 0.7), om, dr + 0.3, dt - 0.45), 0.7, atol=1e-15)
    # fractional shift and a varying map: the sample point is z - dtheta omega_0(z)
    om2 = g.uniform(-1, 1, (H, W))
    b = O.apply_WTb(u, om2, 0.6, -0.8)
    Y, X = 10, 13
    sy, sx = Y + 0.8 * om2[Y, X], X - 0.6 * om2[Y, X]
    y0, x0 = int(np.floor(sy)), int(np.floor(sx))
    a_, b_ = sy - y0, sx - x0
    ref = ((1 - a_) * (1 - b_) * u[y0, x0] + (1 - a_) * b_ * u[y0, x0 + 1] + a_ * (1 - b_) * u[y0 + 1, x0]
           + a_ * b_ * u[y0 + 1, x0 + 1])
    assert abs(b[Y, X] - ref) < 1e-14


def test_P25_paper_mode_AT(oracle_lib):
    nv, h, w, z = 4, 12, 13, 2
    vo = np.array([[1, 0], [0, 1], [-1, 0], [0, -1]], float)   # integer shifts with omega = 1 (HR px)
    om = np.ones((h * z, w * z))
    kw = dict(n_views=nv, lr_h=h, lr_w=w, scale=z, ref_view=0)
    r = np.random.default_rng(2).standard_normal((nv, h, w))
    ex = O.apply_AT(O.Params(**kw), vo, om, r)
    pa = O.apply_AT(O.Params(paper_adjoint=1, **kw), vo, om, r)
    inner = (slice(4, h * z - 4), slice(4, w * z - 4))
    assert np.allclose(ex[inner], pa[inner], rtol=0, atol=1e-13)
    assert not np.allclose(ex, pa)            # the borders differ: W_k^* is not the transpose there
