"""Small runs of every §8f mode on C1-sized inputs (development aid for compute-sanitizer,
tools/sanitize.sh): gd and gd-ls, the subgradient op, per-view maps (ADMM), a user blur kernel
at zeta = 2 and 3 (ADMM), the paper-mode adjoint (ADMM + A^T op) and the colour pipeline."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lfsr_synth as S  # noqa: E402
import paper_2206_05047_b200 as L  # noqa: E402

lf = S.make_lightfield("C1")
base = dict(n_views=9, lr_height=32, lr_width=32, scale=2, ref_view=4)


def run(name, fn):
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


def gd():
    with L.Solver(L.Params(**base)) as s:
        s.set_observations(lf.y, lf.view_offsets, lf.omega)
        s.gd_run(2, 2.0 ** -7)
        s.op("GRAD", lf.x_gt.astype(np.float32))
    with L.Solver(L.Params(**base)) as s:
        s.set_observations(lf.y, lf.view_offsets, lf.omega)
        s.gd_run(2, 1.0, line_search=True, max_trials=12)


def per_view():
    with L.Solver(L.Params(**base)) as s:
        s.set_observations(lf.y, lf.view_offsets, S.per_view_disparity(lf.omega, 9, 0.2, 1))
        s.admm_run(2)


def psf():
    with L.Solver(L.Params(**base, psf=S.motion_psf(5, 45.0))) as s:
        s.set_observations(lf.y, lf.view_offsets, lf.omega)
        s.admm_run(2)
    y, vo, om, _ = S.random_instance(3, 4, 23, 19, 3)
    with L.Solver(L.Params(n_views=4, lr_height=23, lr_width=19, scale=3, ref_view=1,
                           psf=S.motion_psf(7, 30.0))) as s:
        s.set_observations(y, vo, om)
        s.admm_run(2)


def paper():
    with L.Solver(L.Params(**base, paper_adjoint=1)) as s:
        s.set_observations(lf.y, lf.view_offsets, lf.omega)
        s.admm_run(2)
        s.op("AT", np.ones((9, 32, 32), np.float32))


def colour():
    rgb = torch.from_numpy(np.clip(lf.y[:, None] * np.array([0.9, 1.0, 0.8], np.float32)[None, :, None, None],
                                   0, 1).astype(np.float32)).cuda()
    L.color_super_resolve(L.Params(**base), rgb, torch.from_numpy(lf.view_offsets).cuda(),
                          torch.from_numpy(lf.omega).cuda(), 2)


for name, fn in (("gd", gd), ("per_view", per_view), ("psf", psf), ("paper", paper), ("colour", colour)):
    run(name, fn)
