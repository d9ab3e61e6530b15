"""GPU parity of the colour path (Y-channel solve, bicubic Cb/Cr; reading A35):
the BT.601 conversion kernels and LFSR_OP_BICUBIC against the oracle, and the whole
colour_super_resolve pipeline against oracle.color_sr on a C1-shaped colour light field."""
import numpy as np
import pytest
import torch

import oracle as O
import lfsr_synth as S
from test_gpu_parity import ITER_TOL, oparams, rel_l2

pytestmark = pytest.mark.gpu


def test_color_conversion_parity(lfsr_mod):
    rgb = np.random.default_rng(3).uniform(0, 1, (3, 37, 53)).astype(np.float32)
    y, cb, cr = lfsr_mod.rgb_to_ycbcr(torch.from_numpy(rgb).cuda())
    oy, ocb, ocr = O.rgb_to_ycbcr(rgb)
    for a, b in ((y, oy), (cb, ocb), (cr, ocr)):
        assert np.abs(a.cpu().numpy() - b).max() <= 2e-7
    back = lfsr_mod.ycbcr_to_rgb(y, cb, cr).cpu().numpy()
    assert np.abs(back - O.ycbcr_to_rgb(oy, ocb, ocr)).max() <= 1e-6
    assert np.abs(back - rgb).max() <= 1e-6


def colour_lf(seed=5):
    """A colour light field: the C1 luminance scene tinted per object by smooth chroma planes
    (input generator only: each view's RGB = tint * grey value of that view)."""
    lf = S.make_lightfield("C1")
    g = np.random.default_rng(seed)
    tint = g.uniform(0.7, 1.0, size=(3, 1, 1)).astype(np.float32)
    rgb = np.clip(lf.y[:, None, :, :] * tint[None], 0, 1).astype(np.float32)
    return lf, rgb


def test_color_super_resolve_parity_C1(lfsr_mod):
    lf, rgb = colour_lf()
    d = S.SolverDefaults()
    p = lfsr_mod.Params(n_views=lf.n_views, lr_height=32, lr_width=32, scale=2, ref_view=lf.ref_view,
                        nltv_radius=d.radius, lambda1=d.lambda1, lambda2=d.lambda2, lambda_reg=d.lambda_reg,
                        sigma_s=d.sigma_s, sigma_e=d.sigma_e, sigma_o1=d.sigma_o1, sigma_o2=d.sigma_o2,
                        theta=d.theta, cg_max_iters=d.cg_max_iters, cg_tol=d.cg_tol)
    n = 5
    out, stats = lfsr_mod.color_super_resolve(p, torch.from_numpy(rgb).cuda(),
                                              torch.from_numpy(lf.view_offsets).cuda(),
                                              torch.from_numpy(lf.omega).cuda(), n)
    ref = O.color_sr(oparams(p), rgb, lf.view_offsets, lf.omega, n)
    got = out.cpu().numpy()
    assert got.shape == (3, 64, 64) and len(stats) == n
    assert rel_l2(got, ref) <= ITER_TOL
    # chroma planes alone: the bicubic op
    s = lfsr_mod.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    plane = np.random.default_rng(1).uniform(0, 1, (32, 32)).astype(np.float32)
    assert rel_l2(s.op("BICUBIC", plane), O.bicubic(plane, 2)) <= 1e-6
    s.close()
