"""Input generator (lfsr_synth): shapes, noise statistics and determinism."""
import math

import numpy as np

import lfsr_synth as S


def test_noise_statistics():
    y = np.full((3, 300, 400), 0.5, dtype=np.float32)
    n = y[0].size
    out = S.add_mixed_noise(y, 0.0, 5.0, 7)
    for k in range(3):
        assert int(np.sum((out[k] == 0.0) | (out[k] == 1.0))) == math.floor(5.0 * n / 100)  # without replacement
    g = S.add_mixed_noise(y, 0.02, 0.0, 9)
    assert abs(np.std(g[0] - 0.5) - 0.02) < 0.02 * 0.02
    assert abs(np.mean(g[0] - 0.5)) < 3 * 0.02 / math.sqrt(n)
    # independent per-view streams
    c = np.corrcoef((g[0] - 0.5).ravel(), (g[1] - 0.5).ravel())[0, 1]
    assert abs(c) < 0.01


def test_lightfield_shapes_and_determinism():
    lf = S.make_lightfield("C1")
    cfg = S.CONFIGS["C1"]
    assert lf.y.shape == (9, 32, 32) and lf.y.dtype == np.float32
    assert lf.omega.shape == (64, 64) and lf.x_gt.shape == (64, 64)
    assert lf.ref_view == 4 and np.array_equal(lf.view_offsets[4], [0, 0])
    assert np.abs(lf.omega).max() <= cfg.omega_max + 1e-6
    assert lf.y.min() >= 0 and lf.y.max() <= 1
    lf2 = S.make_lightfield("C1")
    assert np.array_equal(lf.y, lf2.y) and np.array_equal(lf.omega, lf2.omega)
    assert S.CONFIGS["C4"].H == 513 and S.CONFIGS["C5"].H == 2048


def test_grid_offsets_axis_convention():
    o = S.grid_offsets(3)
    # row-major over the angular grid: row = tau, column = rho (reading A13)
    assert np.array_equal(o[0], [-1, -1]) and np.array_equal(o[1], [0, -1]) and np.array_equal(o[3], [-1, 0])


def test_misr_frames():
    """MISR configs (NEXT-1): frame 0 unshifted and the reference, 1/zeta-LR-px (1 HR px) shifts,
    constant disparity; BTV weights in the A9 offset order."""
    lf = S.make_lightfield("M1")
    assert lf.ref_view == S.CONFIGS["M1"].ref_view == 0
    assert lf.view_offsets.tolist() == [[0, 0], [1, 0], [0, 1], [1, 1]]
    assert np.all(lf.omega == 1.0)
    w = S.btv_weights(1, 0.5)
    assert w == [0.25, 0.5, 0.25, 0.5, 0.5, 0.25, 0.5, 0.25]
