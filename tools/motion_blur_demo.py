"""The paper's motion-blur use (Fig. sr_comp_motion_blur: x2, 25 SAIs, 45-degree motion
blur, PSNR after 1 and 10 ADMM iterations) on a synthetic C2-shaped light field (5x5 views,
256^2 -> 512^2): observations = the motion-blurred forward model of the ground truth (the
library's own A with the user kernel, LFSR_OP_A) plus C2's mixed noise, then ADMM with that
kernel as B.  Prints PSNR of x0 / x1 / x10 and the device time per iteration.
usage: python tools/motion_blur_demo.py [--length 5] [--angle 45] [--iters 10]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lfsr_synth as S  # noqa: E402
import paper_2206_05047_b200 as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--length", type=int, default=5)
ap.add_argument("--angle", type=float, default=45.0)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
cfg = S.CONFIGS[a.config]
lf = S.make_lightfield(a.config)
p = L.params_for(cfg, S.defaults_for(cfg))
p.psf = S.motion_psf(a.length, a.angle)
with L.Solver(p) as s:           # the degradation model with the motion kernel
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    y = s.op("A", lf.x_gt.astype(np.float32))
y = S.add_mixed_noise(y, cfg.sigma, cfg.nu, 2000 + 2).astype(np.float32)
ts = torch.cuda.Stream()          # a real stream (the legacy default stream's handle is NULL)
torch.cuda.set_stream(ts)
stream = ts.cuda_stream
res = {"config": a.config, "psf": "motion length %d angle %.0f" % (a.length, a.angle)}
with L.Solver(p, stream=stream) as s:
    s.set_observations(*[torch.from_numpy(v).cuda() for v in (y, lf.view_offsets, lf.omega)])
    res["psnr_x0"] = L.psnr(s.get_hr(), lf.x_gt)
    s.admm_run(1)
    res["psnr_x1"] = L.psnr(s.get_hr(), lf.x_gt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.admm_enqueue(a.iters - 1)
    e1.record()
    e1.synchronize()
    res["psnr_x%d" % a.iters] = L.psnr(s.get_hr(), lf.x_gt)
    res["ms_per_iter"] = e0.elapsed_time(e1) / max(a.iters - 1, 1)
print(json.dumps(res))
