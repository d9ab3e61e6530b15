"""GPU parity of the gradient-descent baselines (lfsr_gd_run, LFSR_OP_GRAD; SURVEY §8f NEXT-3,
P:L910-933, readings A30-A33) against the fp64 oracle (oracle.c or_gradient / or_gd).

Bars: the subgradient as a single operator within OP_TOL (fp32 rounding plus the fixed-point
adjoint quantum); gd / gd-ls iterates within the north-star per-iterate 1e-4,
the cost terms within 1e-4 and the line-search decisions (trials evaluated, step taken)
identical.  sgn(e) is a discrete decision taken in each side's own precision (fp32 here,
fp64 in the oracle); on these inputs no residual lies within rounding of zero, and the NLTV
signs are exact on both sides (the sign of a difference of two fp32 values never rounds
away), see DESIGN.md §3 A30."""
import numpy as np
import pytest

import oracle as O
import lfsr_synth as S
from test_gpu_parity import OP_CASES, OP_TOL, ITER_TOL, PSNR_TOL, make_solver, oparams, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", OP_CASES, ids=lambda c: "nv%d_%dx%d_z%d" % (c["nv"], c["h"], c["w"], c["z"]))
def test_grad_operator_parity(lfsr_mod, case):
    s, p, y, vo, om, x = make_solver(lfsr_mod, case)
    P = oparams(p)
    m = s.get_state()["m"]
    xin = np.random.default_rng(case["seed"] + 5).uniform(0, 1, (p.H, p.W)).astype(np.float32)
    _, _, g = O.gradient(P, y, vo, om, m, xin)
    assert rel_l2(s.op("GRAD", xin), g) < OP_TOL
    s.close()


def c1_params(lfsr_mod, lf, **over):
    d = S.SolverDefaults()
    p = lfsr_mod.Params(n_views=lf.n_views, lr_height=lf.y.shape[1], lr_width=lf.y.shape[2], scale=lf.scale,
                        ref_view=lf.ref_view, nltv_radius=d.radius, lambda1=d.lambda1, lambda2=d.lambda2,
                        lambda_reg=d.lambda_reg, sigma_s=d.sigma_s, sigma_e=d.sigma_e, sigma_o1=d.sigma_o1,
                        sigma_o2=d.sigma_o2, theta=d.theta, cg_max_iters=d.cg_max_iters, cg_tol=d.cg_tol)
    for k, v in over.items():
        setattr(p, k, v)
    return p


def run_gd_pair(lfsr_mod, lf, n, step, line_search, **over):
    """Both sides start from the same fp32 x0 (the oracle's bicubic up-sampling, rounded): the
    subgradient's sgn(0) = 0 decisions on exactly flat regions then agree (with each side's own
    bicubic, flat regions are 0 in one precision and +-1 ulp in the other)."""
    p = c1_params(lfsr_mod, lf, **over)
    x0 = O.bicubic(lf.y[p.ref_view], p.scale).astype(np.float32)
    ora = O.gd(oparams(p), lf.y, lf.view_offsets, lf.omega, n, step, line_search=line_search, max_halvings=30,
               x0=x0)
    s = lfsr_mod.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega, x0)
    xs, stats = [s.get_hr()], []
    for _ in range(n):
        stats += s.gd_run(1, step, line_search=line_search, max_trials=30)
        xs.append(s.get_hr())
    launches = s.gd_launches_per_iter()
    s.close()
    return ora, np.array(xs), stats, launches


def check_gd(ora, xs, stats, gt):
    errs = [rel_l2(xs[n], ora.x_iters[n]) for n in range(len(xs))]
    assert max(errs) <= ITER_TOL, errs
    for n, (g, o) in enumerate(zip(stats, ora.stats)):
        assert g["iter"] == n + 1
        assert g["ls_evals"] == o["ls_evals"] and g["ls_failed"] == o["ls_failed"], (n, g, o)
        assert g["step"] == pytest.approx(o["step"], rel=1e-7), n
        assert g["cu"] == 2 + o["ls_evals"]
        for k in ("J", "data_l1", "data_l2", "reg_l1", "grad_sq"):
            assert abs(g[k] - o[k]) <= ITER_TOL * abs(o[k]), (n, k, g[k], o[k])
        assert not g["nonfinite"]
    assert abs(O.psnr(xs[-1], gt) - O.psnr(ora.x_iters[-1], gt)) <= PSNR_TOL
    return errs


def test_gd_fixed_step_parity_C1(lfsr_mod):
    lf = S.make_lightfield("C1")
    ora, xs, stats, launches = run_gd_pair(lfsr_mod, lf, 10, 2.0 ** -7, False)
    errs = check_gd(ora, xs, stats, lf.x_gt)
    assert launches == 2   # k_tile<GRAD>, k_gd_update
    print("gd C1 per-iterate rel L2:", ["%.2e" % e for e in errs])


def test_gd_line_search_parity_C1(lfsr_mod):
    lf = S.make_lightfield("C1")
    ora, xs, stats, launches = run_gd_pair(lfsr_mod, lf, 6, 1.0, True)
    errs = check_gd(ora, xs, stats, lf.x_gt)
    assert launches == 2 + 1 + 30
    assert any(s["ls_evals"] > 1 for s in stats)
    print("gd-ls C1 per-iterate rel L2:", ["%.2e" % e for e in errs], [s["ls_evals"] for s in stats])


def test_gd_variants_parity(lfsr_mod):
    """Frozen weights, l1-only and l2-only data terms, zeta = 3."""
    lf = S.make_lightfield("C1")
    for over in (dict(reweight_every_iter=0), dict(lambda2=0.0), dict(lambda1=0.0)):
        ora, xs, stats, _ = run_gd_pair(lfsr_mod, lf, 4, 2.0 ** -7, False, **over)
        check_gd(ora, xs, stats, lf.x_gt)
    y, vo, om, _ = S.random_instance(8, 4, 23, 19, 3)
    p = lfsr_mod.Params(n_views=4, lr_height=23, lr_width=19, scale=3, ref_view=1)
    ora = O.gd(oparams(p), y, vo, om, 3, 0.05, line_search=True, max_halvings=12)
    s = lfsr_mod.Solver(p)
    s.set_observations(y, vo, om)
    st = s.gd_run(3, 0.05, line_search=True, max_trials=12)
    assert rel_l2(s.get_hr(), ora.x_iters[-1]) <= ITER_TOL
    assert [a["ls_evals"] for a in st] == [b["ls_evals"] for b in ora.stats]
    s.close()


def test_gd_api_rules(lfsr_mod):
    lf = S.make_lightfield("C1")
    p = c1_params(lfsr_mod, lf)
    s = lfsr_mod.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    for bad in (dict(step=0.0), dict(step=float("nan")), dict(step=1.0, line_search=True, max_trials=0),
                dict(step=1.0, line_search=True, max_trials=33), dict(step=1.0, armijo_c=-1.0)):
        with pytest.raises(lfsr_mod.LFSRError) as e:
            s.gd_run(1, **bad)
        assert e.value.status == lfsr_mod.LFSR_ERR_INVALID_ARG
    a = s.gd_run(2, 2.0 ** -7)
    b = s.gd_run(1, 2.0 ** -7)
    assert [r["iter"] for r in a + b] == [1, 2, 3]
    with pytest.raises(lfsr_mod.LFSRError) as e:      # one solver per set_observations
        s.admm_run(1)
    assert e.value.status == lfsr_mod.LFSR_ERR_STATE
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    s.admm_run(1)
    with pytest.raises(lfsr_mod.LFSRError) as e:
        s.gd_run(1, 2.0 ** -7)
    assert e.value.status == lfsr_mod.LFSR_ERR_STATE
    s.close()
    # continuation: run(2) + run(1) == run(3), bit for bit
    s1 = lfsr_mod.Solver(p)
    s1.set_observations(lf.y, lf.view_offsets, lf.omega)
    s1.gd_run(3, 1.0, line_search=True)
    x1 = s1.get_hr()
    s1.close()
    s2 = lfsr_mod.Solver(p)
    s2.set_observations(lf.y, lf.view_offsets, lf.omega)
    s2.gd_run(2, 1.0, line_search=True)
    s2.gd_run(1, 1.0, line_search=True)
    x2 = s2.get_hr()
    s2.close()
    assert rel_l2(x1, x2) <= 1e-6


def test_gd_ls_parity_full_size_C3(lfsr_mod):
    """gd-ls at BASELINE's C3 size (9x9 views, 256^2 -> 512^2) in the launch configuration of
    lfsr_gd_run, 2 iterations against the oracle.  sgn(e) is a discrete decision taken in each
    side's precision (reading A30): of the 5.3 M residuals a handful lie within fp32 rounding of
    zero, and each such flip moves x by O(eta) on the HR footprint of one LR pixel (a few dozen
    pixels).  So the bar here is: line-search decisions identical, cost terms within 1e-4, and
    every pixel within 1e-5 of the oracle except at most 0.1 % (the flip footprints)."""
    lf = S.make_lightfield("C3")
    ora, xs, stats, _ = run_gd_pair(lfsr_mod, lf, 2, 2.0 ** -5, True)
    for n, (g, o) in enumerate(zip(stats, ora.stats)):
        assert g["ls_evals"] == o["ls_evals"] and g["ls_failed"] == o["ls_failed"], (n, g, o)
        for k in ("J", "data_l1", "data_l2", "reg_l1", "grad_sq"):
            assert abs(g[k] - o[k]) <= ITER_TOL * abs(o[k]), (n, k, g[k], o[k])
    for n in range(len(xs)):
        d = np.abs(xs[n].astype(np.float64) - ora.x_iters[n])
        frac = float(np.mean(d > 1e-5))
        print("gd-ls C3 x^%d: rel L2 %.2e, pixels off by > 1e-5: %.4f %%" % (n, rel_l2(xs[n], ora.x_iters[n]),
                                                                          100 * frac))
        assert frac <= 1e-3, (n, frac)
