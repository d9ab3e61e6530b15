"""PSNR sweep of the solver constants (reading A20) on a config with the GPU solver."""
import sys, os, itertools, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import lfsr_synth as S
import paper_2206_05047_b200 as L

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
lf = S.make_lightfield(cfg)
c = S.CONFIGS[cfg]
base = L.params_for(c, S.SolverDefaults())
dev = [torch.from_numpy(a).cuda() for a in (lf.y, lf.view_offsets, lf.omega)]
res = []
x0 = None
for l2, lr, th, se in itertools.product([0.05, 0.2], [0.3, 1.0, 3.0], [4.0, 16.0], [0.05, 0.2, 1.0]):
    p = L.Params(**{**base.__dict__, "lambda2": l2, "lambda_reg": lr, "theta": th, "sigma_e": se})
    s = L.Solver(p)
    s.set_observations(*dev)
    if x0 is None:
        x0 = s.get_hr()
    s.admm_run(c.n_iters, want_stats=False)
    res.append((L.psnr(s.get_hr(), lf.x_gt), l2, lr, th, se))
    s.close()
res.sort(reverse=True)
print(cfg, "x0 psnr", L.psnr(x0, lf.x_gt))
for r in res[:8]:
    print("psnr %.2f  lambda2 %g lambda_reg %g theta %g sigma_e %g" % r)
