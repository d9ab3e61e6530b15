"""Solver comparison of the paper's Fig. sr_comp_py_solvers on the GPU: cost J
against accumulated computation units (CU, reading A33) for admm-5, admm-10, gd and gd-ls on
one synthetic x2 light field (default C3: 9x9 views, 256^2 -> 512^2, the shape of the
paper's HCI 'vinyl' x2 case).  All solvers start from the same bicubic x0.

By default the weights are frozen at x0 (reweight_every_iter = 0) so that every solver
minimises the same J and the curves are comparable; --reweight uses the paper's per-iteration
re-estimation (J then changes with the weights).  gd's fixed step is the best of a sweep of
powers of two at the CU budget ("providing a good step size").  Also reports the
device time per iteration of each solver (CUDA events around the iteration graphs).

usage: python tools/convergence.py [--config C3] [--cu 240] [--reweight] [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lfsr_synth as S  # noqa: E402
import paper_2206_05047_b200 as L  # noqa: E402


_TS = None


def make(lf, reweight, K=5, tol=0.0):
    d = S.SolverDefaults()
    p = L.Params(n_views=lf.n_views, lr_height=lf.y.shape[1], lr_width=lf.y.shape[2], scale=lf.scale,
                 ref_view=lf.ref_view, nltv_radius=d.radius, lambda1=d.lambda1, lambda2=d.lambda2,
                 lambda_reg=d.lambda_reg, sigma_s=d.sigma_s, sigma_e=d.sigma_e, sigma_o1=d.sigma_o1,
                 sigma_o2=d.sigma_o2, theta=d.theta, cg_max_iters=K, cg_tol=tol,
                 reweight_every_iter=1 if reweight else 0)
    global _TS
    if _TS is None:   # a real stream: the legacy default stream's handle is NULL (=> ctx-owned stream)
        _TS = torch.cuda.Stream()
        torch.cuda.set_stream(_TS)
    s = L.Solver(p, stream=_TS.cuda_stream)
    s.set_observations(*[torch.from_numpy(a).cuda() for a in (lf.y, lf.view_offsets, lf.omega)])
    return s


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    return out, a.elapsed_time(b)


def run_admm(lf, reweight, K, cu_budget, tol=0.0):
    s = make(lf, reweight, K, tol)
    st, ms, cu = [], 0.0, 0
    while cu < cu_budget and len(st) < 400:   # with tau > 0 the CG steps per iteration vary
        r, t = timed(lambda: s.admm_run(1))
        st += r
        ms += t
        cu += 2 * (1 + r[0]["cg_iters"])
    n = len(st)
    x = s.get_hr()
    s.close()
    cu = np.concatenate([[0], np.cumsum([2 * (1 + r["cg_iters"]) for r in st])])
    return {"cu": cu[:-1].tolist(), "J": [r["J"] for r in st], "ms_per_iter": ms / n,
            "psnr_final": L.psnr(x, lf.x_gt), "iters": n}


def run_gd(lf, reweight, step, cu_budget, ls):
    s = make(lf, reweight)
    n = max(1, cu_budget // 2 + 1) if not ls else 1
    if ls:   # unknown CU per iteration: run until the budget is spent
        st, ms_tot, cu = [], 0.0, 0
        while cu < cu_budget:
            r, ms = timed(lambda: s.gd_run(1, step, line_search=True, max_trials=30))
            st += r
            ms_tot += ms
            cu += r[0]["cu"]
        n = len(st)
        ms = ms_tot
    else:
        st, ms = timed(lambda: s.gd_run(n, step))
    x = s.get_hr()
    s.close()
    cu = np.concatenate([[0], np.cumsum([r["cu"] for r in st])])
    return {"cu": cu[:-1].tolist(), "J": [r["J"] for r in st], "ms_per_iter": ms / n, "step": step,
            "psnr_final": L.psnr(x, lf.x_gt), "iters": n, "ls_evals": [r["ls_evals"] for r in st] if ls else None}


def time_solver(lf, reweight, kind, step=1.0, n=20):
    """Warm device time per iteration (graph already built, 2 warm-up iterations)."""
    s = make(lf, reweight)
    if kind == "admm":
        s.admm_run(2)
        _, ms = timed(lambda: s.admm_run(n, want_stats=False))
    else:
        ls = kind == "gd-ls"
        s.gd_run(2, step, line_search=ls, want_stats=False)
        _, ms = timed(lambda: s.gd_run(n, step, line_search=ls, want_stats=False))
    s.close()
    return ms / n


def at_cu(run, cu):
    """J of the last iterate whose cost was evaluated at or before `cu` CU."""
    js = [j for c, j in zip(run["cu"], run["J"]) if c <= cu]
    return js[-1] if js else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--cu", type=int, default=240)
    ap.add_argument("--reweight", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    L.load_library()
    lf = S.make_lightfield(a.config)
    res = {"config": a.config, "reweight_every_iter": int(a.reweight), "cu_budget": a.cu,
           "cu_rule": "reading A33: gd 2 + trials per iteration, ADMM 2(1 + CG steps)"}
    res["admm-5"] = run_admm(lf, a.reweight, 5, a.cu)
    res["admm-10"] = run_admm(lf, a.reweight, 10, a.cu)
    # with the CG early stop active (Alg.2 line 5): tau = 1e-3 of the first <r0, r0>
    s0 = make(lf, a.reweight)
    pi0 = s0.admm_run(1)[0]["cg_pi0"]
    s0.close()
    tau = 1e-3 * pi0
    res["tau"] = tau
    res["admm-5-tau"] = run_admm(lf, a.reweight, 5, a.cu, tol=tau)
    res["admm-10-tau"] = run_admm(lf, a.reweight, 10, a.cu, tol=tau)
    sweep = {}
    for k in range(2, 14):
        try:
            sweep[k] = run_gd(lf, a.reweight, 2.0 ** -k, a.cu, False)
        except L.LFSRError as e:   # too large a step: J or x overflows
            if e.status != L.LFSR_ERR_DIVERGED:
                raise
            sweep[k] = {"J": [float("inf")], "diverged": True}
    best = min(sweep, key=lambda k: sweep[k]["J"][-1] if np.isfinite(sweep[k]["J"][-1]) else np.inf)
    res["gd"] = sweep[best]
    res["gd_sweep_final_J"] = {"2^-%d" % k: sweep[k]["J"][-1] for k in sweep}
    res["gd-ls"] = run_gd(lf, a.reweight, 1.0, a.cu, True)
    res["warm_ms_per_iter"] = {"admm-5": time_solver(lf, a.reweight, "admm"),
                               "gd": time_solver(lf, a.reweight, "gd", res["gd"]["step"]),
                               "gd-ls": time_solver(lf, a.reweight, "gd-ls", 1.0)}
    marks = [c for c in (24, 48, 96, 120, 192, 240, 480) if c <= a.cu]
    names = ("admm-5", "admm-10", "admm-5-tau", "admm-10-tau", "gd", "gd-ls")
    res["J_at_cu"] = {name: {c: at_cu(res[name], c) for c in marks} for name in names}
    print(json.dumps({k: v for k, v in res.items() if k in ("config", "J_at_cu", "gd_sweep_final_J", "warm_ms_per_iter")}, indent=1))
    for name in names:
        r = res[name]
        print("%-8s iters %3d  %.3f ms/iter  final J %.6g  PSNR %.2f dB" % (name, r["iters"], r["ms_per_iter"],
                                                                        r["J"][-1], r["psnr_final"]))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1, default=float)


if __name__ == "__main__":
    main()
