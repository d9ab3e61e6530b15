"""GPU parity of the paper-mode adjoint (lfsr_params.paper_adjoint; SURVEY §8f NEXT-2, P:L583
backward warp with omega_0, reading A37) against the fp64 oracle: the adjoint-side operators
(A^T, M, the gd subgradient) on several shapes and scales, and ADMM iterates on C1 with the
resulting non-symmetric CG operator; plus how the iterates compare with the exact-transpose
mode."""
import numpy as np
import pytest

import oracle as O
import lfsr_synth as S
from test_gpu_parity import OP_CASES, OP_TOL, ITER_TOL, PSNR_TOL, oparams, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", OP_CASES, ids=lambda c: "nv%d_%dx%d_z%d" % (c["nv"], c["h"], c["w"], c["z"]))
def test_paper_adjoint_operator_parity(lfsr_mod, case):
    y, vo, om, x = S.random_instance(case["seed"], case["nv"], case["h"], case["w"], case["z"], grid=case.get("grid"))
    p = lfsr_mod.Params(n_views=case["nv"], lr_height=case["h"], lr_width=case["w"], scale=case["z"],
                        ref_view=case["nv"] // 2, paper_adjoint=1)
    s = lfsr_mod.Solver(p)
    s.set_observations(y, vo, om)
    P = oparams(p)
    P.paper_adjoint = 1
    g = np.random.default_rng(case["seed"] + 23)
    xin = g.uniform(-1, 1, (p.H, p.W)).astype(np.float32)
    rin = g.uniform(-1, 1, (p.n_views, p.lr_height, p.lr_width)).astype(np.float32)
    m = s.get_state()["m"]
    assert rel_l2(s.op("A", xin), O.apply_A(P, vo, om, xin)) < OP_TOL
    assert rel_l2(s.op("AT", rin), O.apply_AT(P, vo, om, rin)) < OP_TOL
    assert rel_l2(s.op("NORMAL", xin), O.normal(P, vo, om, m, xin)) < OP_TOL
    xg = g.uniform(0, 1, (p.H, p.W)).astype(np.float32)
    assert rel_l2(s.op("GRAD", xg), O.gradient(P, y, vo, om, m, xg)[2]) < OP_TOL
    s.close()


def test_paper_adjoint_admm_parity_C1(lfsr_mod):
    lf = S.make_lightfield("C1")
    d = S.SolverDefaults()
    xs_modes = {}
    for mode in (1, 0):
        p = lfsr_mod.Params(n_views=lf.n_views, lr_height=32, lr_width=32, scale=2, ref_view=lf.ref_view,
                            nltv_radius=d.radius, lambda1=d.lambda1, lambda2=d.lambda2, lambda_reg=d.lambda_reg,
                            sigma_s=d.sigma_s, sigma_e=d.sigma_e, sigma_o1=d.sigma_o1, sigma_o2=d.sigma_o2,
                            theta=d.theta, cg_max_iters=d.cg_max_iters, cg_tol=d.cg_tol, paper_adjoint=mode)
        n = 8
        s = lfsr_mod.Solver(p)
        s.set_observations(lf.y, lf.view_offsets, lf.omega)
        xs, stats = [s.get_hr()], []
        for _ in range(n):
            stats += s.admm_run(1)
            xs.append(s.get_hr())
        s.close()
        xs_modes[mode] = xs
        if mode == 1:
            P = oparams(p)
            P.paper_adjoint = 1
            ora = O.admm(P, lf.y, lf.view_offsets, lf.omega, n)
            errs = [rel_l2(xs[i], ora.x_iters[i]) for i in range(n + 1)]
            assert max(errs) <= ITER_TOL, errs
            for g_, o in zip(stats, ora.stats):
                assert g_["cg_iters"] == o["cg_iters"] and g_["breakdown"] == o["breakdown"]
                assert abs(g_["J"] - o["J"]) <= ITER_TOL * abs(o["J"])
            assert abs(O.psnr(xs[-1], lf.x_gt) - O.psnr(ora.x_iters[-1], lf.x_gt)) <= PSNR_TOL
            print("paper-mode C1 per-iterate rel L2:", ["%.2e" % e for e in errs])
    print("paper vs exact adjoint, C1 after 8 iterations: PSNR %.2f vs %.2f dB, rel diff %.3e" % (
        O.psnr(xs_modes[1][-1], lf.x_gt), O.psnr(xs_modes[0][-1], lf.x_gt), rel_l2(xs_modes[1][-1], xs_modes[0][-1])))


def test_paper_adjoint_unsupported_combinations(lfsr_mod):
    lf = S.make_lightfield("C1")
    p = lfsr_mod.Params(n_views=9, lr_height=32, lr_width=32, scale=2, ref_view=4, paper_adjoint=1)
    s = lfsr_mod.Solver(p)
    with pytest.raises(lfsr_mod.LFSRError) as e:
        s.set_observations(lf.y, lf.view_offsets, np.stack([lf.omega] * 9))
    assert e.value.status == lfsr_mod.LFSR_ERR_UNSUPPORTED
    s.close()
