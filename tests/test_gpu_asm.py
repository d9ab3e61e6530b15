"""GPU parity of the assembled data normal operator (asm.cu): the CG operator
M p = c_A sum_k A_k^T A_k p + (th/2) S_W^T S_W p (A7) computed from the stencil of
the regular rows plus the irregular rows applied as rows, against the fp64 oracle and against the
fused tile kernel (LFSR_ASM=0) on identical inputs."""
import numpy as np
import pytest

import oracle as O
import lfsr_synth as S
from test_gpu_parity import OP_CASES, OP_TOL, ITER_TOL, rel_l2, oparams, make_solver

pytestmark = pytest.mark.gpu


def lf_solver(lfsr_mod, name, **over):
    lf = S.make_lightfield(name)
    cfg = S.get_config(name)
    d = S.defaults_for(cfg)
    p = lfsr_mod.Params(n_views=cfg.n_views, lr_height=cfg.lr_h, lr_width=cfg.lr_w, scale=cfg.scale,
                        ref_view=cfg.ref_view, nltv_radius=d.radius, lambda1=d.lambda1, lambda2=d.lambda2,
                        lambda_reg=d.lambda_reg, sigma_s=d.sigma_s, sigma_e=d.sigma_e, sigma_o1=d.sigma_o1,
                        sigma_o2=d.sigma_o2, theta=d.theta, cg_max_iters=d.cg_max_iters, cg_tol=d.cg_tol, **over)
    s = lfsr_mod.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    return s, p, lf


@pytest.mark.parametrize("case", OP_CASES, ids=lambda c: "nv%d_%dx%d_z%d" % (c["nv"], c["h"], c["w"], c["z"]))
def test_asm_normal_vs_oracle_and_tile(lfsr_mod, case, monkeypatch):
    """The operator on the six shapes of the tile-kernel parity (several tiles, ragged tails,
    zeta = 2/3/4): the assembled path is selected, matches the oracle within the operator bar and
    the tile kernel to fp32 rounding."""
    monkeypatch.setenv("LFSR_ASM", "1")
    s, p, y, vo, om, x = make_solver(lfsr_mod, case)
    info = s.normal_path
    assert info["name"] == "assembled", info
    assert 0 <= info["irregular_rows"] <= info["total_rows"] == p.n_views * p.lr_height * p.lr_width
    g = np.random.default_rng(case["seed"] + 7)
    xin = g.uniform(-1, 1, (p.H, p.W)).astype(np.float32)
    m = s.get_state()["m"]
    q_asm = s.op("NORMAL", xin)
    q_ref = O.normal(oparams(p), vo, om, m, xin)
    err_o = rel_l2(q_asm, q_ref)
    s.close()
    monkeypatch.setenv("LFSR_ASM", "0")
    s2, *_ = make_solver(lfsr_mod, case)
    assert s2.normal_path["name"] == "tile"
    q_tile = s2.op("NORMAL", xin)
    s2.close()
    err_t = rel_l2(q_asm, q_tile)
    print("asm vs oracle %.2e, vs tile kernel %.2e, irregular rows %d / %d"
          % (err_o, err_t, info["irregular_rows"], info["total_rows"]))
    assert err_o < OP_TOL
    assert err_t < OP_TOL


def test_asm_rows_all_irregular_and_all_regular(lfsr_mod, monkeypatch):
    """Degenerate splits: a disparity with a jump at every other HR column makes (almost) every
    row irregular (the stencil is ~empty, the row path carries the operator); a zero disparity
    makes every row regular (no row path)."""
    monkeypatch.setenv("LFSR_ASM", "1")
    nv, h, w, z = 9, 20, 26, 2
    y, vo, om, _ = S.random_instance(11, nv, h, w, z, grid=3)
    H, W = h * z, w * z
    stripes = (np.where((np.arange(W)[None, :] // 2) % 2 == 0, 1.5, -1.5) * np.ones((H, 1))).astype(np.float32)
    for name, omega in (("stripes", stripes), ("zero", np.zeros((H, W), np.float32))):
        if name == "zero":
            omega[0, 0] = 1e-3   # not constant: keep the MISR fast path out
        p = lfsr_mod.Params(n_views=nv, lr_height=h, lr_width=w, scale=z, ref_view=nv // 2)
        s = lfsr_mod.Solver(p)
        s.set_observations(y, vo, omega)
        info = s.normal_path
        assert info["name"] == "assembled"
        if name == "stripes":
            assert info["irregular_rows"] > 0.5 * info["total_rows"], info
        else:
            assert info["irregular_rows"] <= nv * 4, info
        xin = np.random.default_rng(3).uniform(-1, 1, (H, W)).astype(np.float32)
        m = s.get_state()["m"]
        err = rel_l2(s.op("NORMAL", xin), O.normal(oparams(p), vo, omega, m, xin))
        s.close()
        print(name, info, "%.2e" % err)
        assert err < OP_TOL


def test_asm_per_view_disparity(lfsr_mod, monkeypatch):
    """Per-view disparity maps (A34): the rows of view k use omega_k."""
    monkeypatch.setenv("LFSR_ASM", "1")
    nv, h, w, z = 9, 24, 30, 2
    y, vo, om, _ = S.random_instance(12, nv, h, w, z, grid=3)
    omk = S.per_view_disparity(om, nv, seed=5)
    p = lfsr_mod.Params(n_views=nv, lr_height=h, lr_width=w, scale=z, ref_view=nv // 2)
    s = lfsr_mod.Solver(p)
    s.set_observations(y, vo, omk)
    assert s.normal_path["name"] == "assembled"
    xin = np.random.default_rng(4).uniform(-1, 1, (p.H, p.W)).astype(np.float32)
    m = s.get_state()["m"]
    P = oparams(p)
    P.disp_per_view = 1
    err = rel_l2(s.op("NORMAL", xin), O.normal(P, vo, omk, m, xin))
    s.close()
    assert err < OP_TOL


@pytest.mark.parametrize("name,n", [("C1", 20), ("C3", 3), ("C4", 2)])
def test_asm_admm_vs_tile(lfsr_mod, name, n, monkeypatch):
    """Whole ADMM iterations (wz-step + K CG steps through the assembled operator) against the
    same solve on the tile kernel: per-iterate x within the north-star bar (both are fp32 paths of
    the same iteration; their distance bounds each one's distance to the oracle that
    test_gpu_parity checks), identical CG step counts."""
    xs = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("LFSR_ASM", flag)
        s, p, lf = lf_solver(lfsr_mod, name)
        assert s.normal_path["name"] == ("assembled" if flag == "1" else "tile")
        it = []
        for _ in range(n):
            st = s.admm_run(1)
            it.append((s.get_hr(), st[0]["cg_iters"]))
        xs[flag] = it
        s.close()
    for i, ((xa, ka), (xt, kt)) in enumerate(zip(xs["1"], xs["0"])):
        e = rel_l2(xa, xt)
        print(name, "iter", i + 1, "asm vs tile %.2e" % e)
        assert ka == kt
        assert e < ITER_TOL


def test_asm_admm_vs_oracle_C1(lfsr_mod, monkeypatch):
    """C1 (20 iterations) against the fp64 oracle, every iterate, through the assembled operator."""
    monkeypatch.setenv("LFSR_ASM", "1")
    s, p, lf = lf_solver(lfsr_mod, "C1")
    assert s.normal_path["name"] == "assembled"
    ref = O.admm(oparams(p), lf.y, lf.view_offsets, lf.omega, 20)
    for i in range(20):
        s.admm_run(1)
        e = rel_l2(s.get_hr(), ref.x_iters[i + 1])
        assert e < ITER_TOL, (i, e)
    s.close()


def test_asm_admm_variants_vs_oracle(lfsr_mod, monkeypatch):
    """C1 through the assembled operator (forced) against the oracle with every iterate checked:
    l1-only, l2-only, frozen weights, K = 1, a tau > 0 early stop (the CG-stopped path of every
    assembled kernel), BTV offset weights, per-view disparity."""
    from test_gpu_parity import run_pair, check_iterates
    monkeypatch.setenv("LFSR_ASM", "1")
    lf = S.make_lightfield("C1")
    for over in (dict(lambda2=0.0), dict(lambda1=0.0), dict(reweight_every_iter=0), dict(cg_max_iters=1),
                 dict(cg_tol=1e-3, cg_max_iters=12), dict(offset_weights=S.btv_weights(2, 0.7))):
        p, ora, xs, stats, st = run_pair(lfsr_mod, lf, 5, **over)
        check_iterates(p, ora, xs, stats, st, lf.x_gt)
    # per-view disparity maps (A34) through whole iterations
    oms = S.per_view_disparity(lf.omega, lf.n_views, amp=0.2, seed=3)
    d = S.SolverDefaults()
    p = lfsr_mod.params_for(S.CONFIGS["C1"], d)
    P = oparams(p)
    P.disp_per_view = 1
    ora = O.admm(P, lf.y, lf.view_offsets, oms, 5)
    s = lfsr_mod.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, oms)
    assert s.normal_path["name"] == "assembled"
    for i in range(5):
        s.admm_run(1)
        assert rel_l2(s.get_hr(), ora.x_iters[i + 1]) < ITER_TOL
    s.close()


@pytest.mark.parametrize("case", [dict(seed=31, nv=9, h=23, w=47, z=3), dict(seed=32, nv=9, h=17, w=33, z=4),
                                  dict(seed=33, nv=9, h=40, w=70, z=2)],
                         ids=lambda c: "%dx%d_z%d" % (c["h"], c["w"], c["z"]))
def test_asm_admm_ragged_vs_oracle(lfsr_mod, case, monkeypatch):
    """Whole ADMM iterations through the assembled operator on ragged shapes at every zeta (partial
    128-wide stencil tiles, odd widths, irregular rows at a depth edge) against the oracle."""
    from test_gpu_parity import check_iterates
    monkeypatch.setenv("LFSR_ASM", "1")
    s, p, y, vo, om, x = make_solver(lfsr_mod, case, lambda2=0.1, lambda_reg=0.5, theta=4.0, sigma_e=0.2)
    assert s.normal_path["name"] == "assembled" and s.normal_path["irregular_rows"] > 0
    n = 5
    ora = O.admm(oparams(p), y, vo, om, n)
    xs = [s.get_hr()]
    stats = []
    for _ in range(n):
        stats += s.admm_run(1)
        xs.append(s.get_hr())
    st = s.get_state()
    s.close()
    errs = check_iterates(p, ora, np.array(xs), stats, st)
    print(case, "per-iterate rel L2", ["%.1e" % e for e in errs])
