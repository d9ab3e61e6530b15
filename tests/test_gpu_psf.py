"""GPU parity of a user blur kernel (lfsr_params.psf; SURVEY §8f NEXT-4, P:L962 motion blur,
reading A36) against the fp64 oracle: A, A^T, M and the gd subgradient over several shapes and
all three scales (45-degree motion kernels and random asymmetric kernels), ADMM iterates on a
C1-shaped light field degraded by a 45-degree motion blur, and the Gaussian outer product
reproducing the default separable path."""
import numpy as np
import pytest

import oracle as O
import lfsr_synth as S
from test_gpu_parity import OP_CASES, OP_TOL, ITER_TOL, PSNR_TOL, oparams, rel_l2

pytestmark = pytest.mark.gpu


def kernel_for(case, kind):
    R = 2 if case["z"] == 2 else 3
    if kind == "motion":
        return S.motion_psf(2 * R + 1, 45.0)
    g = np.random.default_rng(case["seed"] + 3)
    r = R - (case["seed"] % 2)          # smaller-than-window kernels too
    k = g.uniform(0.0, 1.0, (2 * r + 1, 2 * r + 1)).astype(np.float32)
    return (k / k.sum()).astype(np.float32)


@pytest.mark.parametrize("kind", ["motion", "random"])
@pytest.mark.parametrize("case", OP_CASES, ids=lambda c: "nv%d_%dx%d_z%d" % (c["nv"], c["h"], c["w"], c["z"]))
def test_psf_operator_parity(lfsr_mod, case, kind):
    y, vo, om, x = S.random_instance(case["seed"], case["nv"], case["h"], case["w"], case["z"], grid=case.get("grid"))
    k = kernel_for(case, kind)
    p = lfsr_mod.Params(n_views=case["nv"], lr_height=case["h"], lr_width=case["w"], scale=case["z"],
                        ref_view=case["nv"] // 2, psf=k)
    s = lfsr_mod.Solver(p)
    s.set_observations(y, vo, om)
    P = oparams(p)
    P.psf = k.astype(np.float64)
    g = np.random.default_rng(case["seed"] + 11)
    xin = g.uniform(-1, 1, (p.H, p.W)).astype(np.float32)
    rin = g.uniform(-1, 1, (p.n_views, p.lr_height, p.lr_width)).astype(np.float32)
    m = s.get_state()["m"]
    assert rel_l2(s.op("A", xin), O.apply_A(P, vo, om, xin)) < OP_TOL
    assert rel_l2(s.op("AT", rin), O.apply_AT(P, vo, om, rin)) < OP_TOL
    assert rel_l2(s.op("NORMAL", xin), O.normal(P, vo, om, m, xin)) < OP_TOL
    xg = g.uniform(0, 1, (p.H, p.W)).astype(np.float32)
    assert rel_l2(s.op("GRAD", xg), O.gradient(P, y, vo, om, m, xg)[2]) < OP_TOL
    s.close()


def test_gaussian_kernel_matches_default(lfsr_mod):
    case = OP_CASES[1]
    y, vo, om, x = S.random_instance(case["seed"], case["nv"], case["h"], case["w"], case["z"])
    taps = O.blur_taps(case["z"])
    outs = []
    for psf in (None, np.outer(taps, taps).astype(np.float32)):
        p = lfsr_mod.Params(n_views=case["nv"], lr_height=case["h"], lr_width=case["w"], scale=case["z"],
                            ref_view=0, psf=psf)
        s = lfsr_mod.Solver(p)
        s.set_observations(y, vo, om)
        outs.append((s.op("A", x), s.op("NORMAL", x)))
        s.close()
    assert rel_l2(outs[1][0], outs[0][0]) < 1e-6 and rel_l2(outs[1][1], outs[0][1]) < 1e-5


def test_motion_blur_admm_parity_C1(lfsr_mod):
    """The paper's motion-blur use: views degraded by a 45-degree motion kernel instead
    of the Gaussian, solved with that kernel as B."""
    lf = S.make_lightfield("C1")
    k = S.motion_psf(5, 45.0)
    d = S.SolverDefaults()
    p = lfsr_mod.Params(n_views=lf.n_views, lr_height=32, lr_width=32, scale=2, ref_view=lf.ref_view,
                        nltv_radius=d.radius, lambda1=d.lambda1, lambda2=d.lambda2, lambda_reg=d.lambda_reg,
                        sigma_s=d.sigma_s, sigma_e=d.sigma_e, sigma_o1=d.sigma_o1, sigma_o2=d.sigma_o2,
                        theta=d.theta, cg_max_iters=d.cg_max_iters, cg_tol=d.cg_tol, psf=k)
    P = oparams(p)
    P.psf = k.astype(np.float64)
    # observations: the motion-blurred forward model of the ground truth plus the C1 noise
    y = O.apply_A(P, lf.view_offsets, lf.omega, lf.x_gt)
    y = S.add_mixed_noise(y.astype(np.float32), 0.02, 5.0, 2001)
    n = 6
    ora = O.admm(P, y, lf.view_offsets, lf.omega, n)
    s = lfsr_mod.Solver(p)
    s.set_observations(y, lf.view_offsets, lf.omega)
    xs, stats = [s.get_hr()], []
    for _ in range(n):
        stats += s.admm_run(1)
        xs.append(s.get_hr())
    s.close()
    errs = [rel_l2(xs[i], ora.x_iters[i]) for i in range(n + 1)]
    assert max(errs) <= ITER_TOL, errs
    for g_, o in zip(stats, ora.stats):
        assert abs(g_["J"] - o["J"]) <= ITER_TOL * abs(o["J"])
    assert abs(O.psnr(xs[-1], lf.x_gt) - O.psnr(ora.x_iters[-1], lf.x_gt)) <= PSNR_TOL
    print("motion-blur C1 per-iterate rel L2:", ["%.2e" % e for e in errs],
          "PSNR %.2f -> %.2f" % (O.psnr(xs[0], lf.x_gt), O.psnr(xs[-1], lf.x_gt)))


def test_motion_blur_admm_parity_full_size_C3(lfsr_mod):
    """User blur kernel at C3 size (9x9 views, 256^2 -> 512^2): 2 ADMM iterations vs the oracle."""
    lf = S.make_lightfield("C3")
    k = S.motion_psf(5, 45.0)
    d = S.SolverDefaults()
    p = lfsr_mod.Params(n_views=lf.n_views, lr_height=256, lr_width=256, scale=2, ref_view=lf.ref_view,
                        nltv_radius=d.radius, lambda1=d.lambda1, lambda2=d.lambda2, lambda_reg=d.lambda_reg,
                        sigma_s=d.sigma_s, sigma_e=d.sigma_e, sigma_o1=d.sigma_o1, sigma_o2=d.sigma_o2,
                        theta=d.theta, cg_max_iters=d.cg_max_iters, cg_tol=d.cg_tol, psf=k)
    P = oparams(p)
    P.psf = k.astype(np.float64)
    n = 2
    ora = O.admm(P, lf.y, lf.view_offsets, lf.omega, n)
    s = lfsr_mod.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    xs = [s.get_hr()]
    for _ in range(n):
        s.admm_run(1)
        xs.append(s.get_hr())
    s.close()
    errs = [rel_l2(xs[i], ora.x_iters[i]) for i in range(n + 1)]
    assert max(errs) <= ITER_TOL, errs


# ---- kernels larger than the Gaussian window (radius 3..7, up to 15x15): the kPsfBigR
# instances (narrower tiles, E region of radius 7).  Motion kernels of length 9 / 15 and random
# asymmetric kernels of radius 4..7 at every scale.
BIG_KERNELS = [("motion9", lambda: S.motion_psf(9, 45.0)), ("motion15", lambda: S.motion_psf(15, 45.0)),
               ("motion11_30deg", lambda: S.motion_psf(11, 30.0))]


def random_kernel(r, seed):
    g = np.random.default_rng(seed)
    k = g.uniform(0.0, 1.0, (2 * r + 1, 2 * r + 1)) * g.uniform(0.0, 1.0, (2 * r + 1, 1))
    return (k / k.sum()).astype(np.float32)


def _op_parity(lfsr_mod, case, k):
    y, vo, om, x = S.random_instance(case["seed"], case["nv"], case["h"], case["w"], case["z"], grid=case.get("grid"))
    p = lfsr_mod.Params(n_views=case["nv"], lr_height=case["h"], lr_width=case["w"], scale=case["z"],
                        ref_view=case["nv"] // 2, psf=k)
    s = lfsr_mod.Solver(p)
    s.set_observations(y, vo, om)
    P = oparams(p)
    P.psf = k.astype(np.float64)
    g = np.random.default_rng(case["seed"] + 11)
    xin = g.uniform(-1, 1, (p.H, p.W)).astype(np.float32)
    rin = g.uniform(-1, 1, (p.n_views, p.lr_height, p.lr_width)).astype(np.float32)
    m = s.get_state()["m"]
    errs = [rel_l2(s.op("A", xin), O.apply_A(P, vo, om, xin)),
            rel_l2(s.op("AT", rin), O.apply_AT(P, vo, om, rin)),
            rel_l2(s.op("NORMAL", xin), O.normal(P, vo, om, m, xin))]
    xg = g.uniform(0, 1, (p.H, p.W)).astype(np.float32)
    errs.append(rel_l2(s.op("GRAD", xg), O.gradient(P, y, vo, om, m, xg)[2]))
    # adjoint identity of the large-kernel A in fp32
    ax = s.op("A", xin)
    atr = s.op("AT", rin)
    lhs, rhs = float(np.dot(ax.ravel().astype(np.float64), rin.ravel())), float(np.dot(xin.ravel().astype(np.float64), atr.ravel()))
    assert abs(lhs - rhs) <= 1e-6 * np.linalg.norm(ax) * np.linalg.norm(rin)
    s.close()
    return errs


@pytest.mark.parametrize("kname", [n for n, _ in BIG_KERNELS])
@pytest.mark.parametrize("case", OP_CASES, ids=lambda c: "nv%d_%dx%d_z%d" % (c["nv"], c["h"], c["w"], c["z"]))
def test_big_psf_operator_parity(lfsr_mod, case, kname):
    k = dict(BIG_KERNELS)[kname]()
    errs = _op_parity(lfsr_mod, case, k)
    assert max(errs) < OP_TOL, errs


@pytest.mark.parametrize("r", [4, 5, 7])
@pytest.mark.parametrize("case", OP_CASES[:4], ids=lambda c: "nv%d_%dx%d_z%d" % (c["nv"], c["h"], c["w"], c["z"]))
def test_big_psf_random_kernel_parity(lfsr_mod, case, r):
    errs = _op_parity(lfsr_mod, case, random_kernel(r, case["seed"] + r))
    assert max(errs) < OP_TOL, errs


@pytest.mark.parametrize("z", [2, 3, 4])
def test_big_psf_motion15_admm_parity(lfsr_mod, z):
    """ADMM iterates with a 15x15 (45-degree, length 15) motion kernel as B, per scale, against
    the oracle (C1-shaped views, observations from the motion-blurred forward model + noise)."""
    lf = S.make_lightfield("C1")
    k = S.motion_psf(15, 45.0)
    d = S.SolverDefaults()
    h = 64 // z
    p = lfsr_mod.Params(n_views=lf.n_views, lr_height=h, lr_width=h, scale=z, ref_view=lf.ref_view,
                        nltv_radius=d.radius, lambda1=d.lambda1, lambda2=d.lambda2, lambda_reg=d.lambda_reg,
                        sigma_s=d.sigma_s, sigma_e=d.sigma_e, sigma_o1=d.sigma_o1, sigma_o2=d.sigma_o2,
                        theta=d.theta, cg_max_iters=d.cg_max_iters, cg_tol=d.cg_tol, psf=k)
    P = oparams(p)
    P.psf = k.astype(np.float64)
    xg = np.ascontiguousarray(lf.x_gt[:h * z, :h * z])
    om = np.ascontiguousarray(lf.omega[:h * z, :h * z])
    y = O.apply_A(P, lf.view_offsets, om, xg)
    y = S.add_mixed_noise(y.astype(np.float32), 0.02, 5.0, 2003 + z)
    n = 5
    ora = O.admm(P, y, lf.view_offsets, om, n)
    s = lfsr_mod.Solver(p)
    s.set_observations(y, lf.view_offsets, om)
    xs, stats = [s.get_hr()], []
    for _ in range(n):
        stats += s.admm_run(1)
        xs.append(s.get_hr())
    s.close()
    errs = [rel_l2(xs[i], ora.x_iters[i]) for i in range(n + 1)]
    assert max(errs) <= ITER_TOL, errs
    for g_, o in zip(stats, ora.stats):
        assert abs(g_["J"] - o["J"]) <= ITER_TOL * abs(o["J"])
    assert abs(O.psnr(xs[-1], xg) - O.psnr(ora.x_iters[-1], xg)) <= PSNR_TOL
    print("PARITY psf15 z=%d C1-shaped N=%d: per-iterate rel L2 %s; PSNR %.2f -> %.2f" % (
        z, n, " ".join("%.1e" % e for e in errs), O.psnr(xs[0], xg), O.psnr(xs[-1], xg)))


def test_big_psf_full_size_C3(lfsr_mod):
    """A 9x9 (length 9) motion kernel at C3 size: 1 ADMM iteration vs the oracle."""
    lf = S.make_lightfield("C3")
    k = S.motion_psf(9, 45.0)
    d = S.SolverDefaults()
    p = lfsr_mod.Params(n_views=lf.n_views, lr_height=256, lr_width=256, scale=2, ref_view=lf.ref_view,
                        nltv_radius=d.radius, lambda1=d.lambda1, lambda2=d.lambda2, lambda_reg=d.lambda_reg,
                        sigma_s=d.sigma_s, sigma_e=d.sigma_e, sigma_o1=d.sigma_o1, sigma_o2=d.sigma_o2,
                        theta=d.theta, cg_max_iters=d.cg_max_iters, cg_tol=d.cg_tol, psf=k)
    P = oparams(p)
    P.psf = k.astype(np.float64)
    ora = O.admm(P, lf.y, lf.view_offsets, lf.omega, 1)
    s = lfsr_mod.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    x0 = s.get_hr()
    s.admm_run(1)
    x1 = s.get_hr()
    s.close()
    errs = [rel_l2(x0, ora.x_iters[0]), rel_l2(x1, ora.x_iters[1])]
    print("PARITY psf9 C3 N=1: per-iterate rel L2 %s" % " ".join("%.1e" % e for e in errs))
    assert max(errs) <= ITER_TOL, errs


def test_big_psf_strips_unsupported(lfsr_mod):
    p = lfsr_mod.Params(n_views=9, lr_height=32, lr_width=32, scale=2, ref_view=4, psf=S.motion_psf(9, 45.0),
                        n_ranks=2, rank=-1)
    with pytest.raises(lfsr_mod.LFSRError, match="UNSUPPORTED"):
        lfsr_mod.Solver(p)
