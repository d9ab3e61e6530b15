"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on identical
seeded inputs.  Bars (BASELINE.json north_star): per-iterate relative L2 error of x^n
<= 1e-4 and final PSNR within 0.01 dB; operators within fp32 rounding (1e-5 relative
L2, derived in DESIGN.md §9)."""
import math

import numpy as np
import pytest

import oracle as O
import lfsr_synth as S

pytestmark = pytest.mark.gpu

OP_TOL = 2e-5      # relative L2, single operator application in fp32
ITER_TOL = 1e-4    # north_star per-iterate bar
PSNR_TOL = 0.01    # dB


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def oparams(gp):
    return O.Params(n_views=gp.n_views, lr_h=gp.lr_height, lr_w=gp.lr_width, scale=gp.scale, ref_view=gp.ref_view,
                    radius=gp.nltv_radius, lambda1=gp.lambda1, lambda2=gp.lambda2, lambda_reg=gp.lambda_reg,
                    sigma_s=gp.sigma_s, sigma_e=gp.sigma_e, sigma_o1=gp.sigma_o1, sigma_o2=gp.sigma_o2,
                    theta=gp.theta, cg_max_iters=gp.cg_max_iters, cg_tol=gp.cg_tol,
                    reweight_every_iter=gp.reweight_every_iter, offset_weights=gp.offset_weights)


def f32(a):
    return np.asarray(a, dtype=np.float32)


# shapes spanning several tiles and ragged tails, all three scales
OP_CASES = [
    dict(seed=1, nv=3, h=7, w=9, z=2),
    dict(seed=2, nv=5, h=40, w=70, z=2),
    dict(seed=3, nv=4, h=23, w=47, z=3),
    dict(seed=4, nv=2, h=17, w=33, z=4),
    dict(seed=5, nv=1, h=5, w=5, z=2),
    dict(seed=6, nv=9, h=33, w=31, z=2, grid=3),
]


def make_solver(lfsr_mod, case, **over):
    y, vo, om, x = S.random_instance(case["seed"], case["nv"], case["h"], case["w"], case["z"],
                                     grid=case.get("grid"))
    p = lfsr_mod.Params(n_views=case["nv"], lr_height=case["h"], lr_width=case["w"], scale=case["z"],
                        ref_view=case["nv"] // 2, **over)
    s = lfsr_mod.Solver(p)
    s.set_observations(y, vo, om)
    return s, p, y, vo, om, x


@pytest.mark.parametrize("case", OP_CASES, ids=lambda c: "nv%d_%dx%d_z%d" % (c["nv"], c["h"], c["w"], c["z"]))
def test_operator_parity(lfsr_mod, case):
    s, p, y, vo, om, x = make_solver(lfsr_mod, case)
    P = oparams(p)
    g = np.random.default_rng(case["seed"] + 99)
    xin = g.uniform(-1, 1, (p.H, p.W)).astype(np.float32)
    rin = g.uniform(-1, 1, (p.n_views, p.lr_height, p.lr_width)).astype(np.float32)
    hin = g.uniform(-1, 1, (p.s_d, p.H, p.W)).astype(np.float32)
    st = s.get_state()
    m = st["m"]
    # A, A^T, normal operator
    assert rel_l2(s.op("A", xin), O.apply_A(P, vo, om, xin)) < OP_TOL
    assert rel_l2(s.op("AT", rin), O.apply_AT(P, vo, om, rin)) < OP_TOL
    assert rel_l2(s.op("NORMAL", xin), O.normal(P, vo, om, m, xin)) < OP_TOL
    # NLTV S, S^T with the library's current weight map
    assert rel_l2(s.op("S", xin), O.apply_S(xin, m, p.nltv_radius, p.sigma_s)) < OP_TOL
    assert rel_l2(s.op("ST", hin), O.apply_ST(hin, m, p.nltv_radius, p.sigma_s)) < OP_TOL
    # setup: bicubic x0, w_o and m
    wo, _, _ = O.setup_wo(P, y, vo, om)
    x0 = O.bicubic(y[p.ref_view], p.scale)
    assert rel_l2(st["x"], x0) < 1e-6
    assert rel_l2(m, O.weights_m(x0, wo, p.lambda_reg, p.sigma_e)) < 1e-5
    assert rel_l2(s.op("WEIGHTS", xin), O.weights_m(xin, wo, p.lambda_reg, p.sigma_e)) < 1e-5
    s.close()


@pytest.mark.parametrize("case", OP_CASES[:4], ids=lambda c: "z%d" % c["z"])
def test_gpu_adjoint_identities(lfsr_mod, case):
    s, p, y, vo, om, x = make_solver(lfsr_mod, case)
    g = np.random.default_rng(7)
    for _ in range(5):
        xin = g.standard_normal((p.H, p.W)).astype(np.float32)
        rin = g.standard_normal((p.n_views, p.lr_height, p.lr_width)).astype(np.float32)
        lhs = float(np.vdot(s.op("A", xin).astype(np.float64), rin))
        rhs = float(np.vdot(xin.astype(np.float64), s.op("AT", rin)))
        # fp32 operators: |<Ax,r> - <x,A^T r>| <= eps |Ax| |r| (Cauchy-Schwarz scale)
        ax, atr = s.op("A", xin).astype(np.float64), s.op("AT", rin).astype(np.float64)
        assert abs(lhs - rhs) <= 1e-6 * max(np.linalg.norm(ax) * np.linalg.norm(rin),
                                            np.linalg.norm(xin) * np.linalg.norm(atr))
        x2 = g.standard_normal((p.H, p.W)).astype(np.float32)
        m1, m2 = s.op("NORMAL", xin).astype(np.float64), s.op("NORMAL", x2).astype(np.float64)
        a = float(np.vdot(m1, x2))
        b = float(np.vdot(xin.astype(np.float64), m2))
        assert abs(a - b) <= 1e-6 * max(np.linalg.norm(m1) * np.linalg.norm(x2), np.linalg.norm(m2) * np.linalg.norm(xin))
        assert float(np.vdot(s.op("NORMAL", xin).astype(np.float64), xin)) > 0
    s.close()


def run_pair(lfsr_mod, lf, n_iters, defaults=None, **over):
    cfg_defaults = defaults or S.SolverDefaults()
    p = lfsr_mod.Params(n_views=lf.n_views, lr_height=lf.y.shape[1], lr_width=lf.y.shape[2], scale=lf.scale,
                        ref_view=lf.ref_view, nltv_radius=cfg_defaults.radius, lambda1=cfg_defaults.lambda1,
                        lambda2=cfg_defaults.lambda2, lambda_reg=cfg_defaults.lambda_reg,
                        sigma_s=cfg_defaults.sigma_s, sigma_e=cfg_defaults.sigma_e, sigma_o1=cfg_defaults.sigma_o1,
                        sigma_o2=cfg_defaults.sigma_o2, theta=cfg_defaults.theta,
                        cg_max_iters=cfg_defaults.cg_max_iters, cg_tol=cfg_defaults.cg_tol,
                        offset_weights=getattr(cfg_defaults, "offset_weights", None))
    for k, v in over.items():
        setattr(p, k, v)
    ora = O.admm(oparams(p), lf.y, lf.view_offsets, lf.omega, n_iters)
    s = lfsr_mod.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    xs = [s.get_hr()]
    stats = []
    for n in range(n_iters):
        stats += s.admm_run(1)
        xs.append(s.get_hr())
    st = s.get_state()
    s.close()
    return p, ora, np.array(xs), stats, st


def check_iterates(p, ora, xs, stats, st, gt=None):
    errs = [rel_l2(xs[n], ora.x_iters[n]) for n in range(len(xs))]
    assert max(errs) <= ITER_TOL, errs
    for n, (g, o) in enumerate(zip(stats, ora.stats)):
        assert g["cg_iters"] == o["cg_iters"], n
        assert abs(g["J"] - o["J"]) <= ITER_TOL * abs(o["J"]), (n, g["J"], o["J"])
        assert abs(g["primal_res"] - o["primal_res"]) <= ITER_TOL * max(o["primal_res"], 1e-12), n
        assert not g["nonfinite"]
    scale = max(np.linalg.norm(ora.wA), 1e-3 * math.sqrt(ora.wA.size) / p.theta)
    assert np.linalg.norm(st["wA"] - ora.wA) <= ITER_TOL * scale
    scale = max(np.linalg.norm(ora.wS), 1e-3 * math.sqrt(ora.wS.size) / p.theta)
    assert np.linalg.norm(st["wS"] - ora.wS) <= ITER_TOL * scale
    if gt is not None:
        assert abs(O.psnr(xs[-1], gt) - O.psnr(ora.x_iters[-1], gt)) <= PSNR_TOL
        assert abs(O.psnr(xs[-1], gt, crop=0) - O.psnr(ora.x_iters[-1], gt, crop=0)) <= PSNR_TOL
    return errs


def test_admm_parity_C1(lfsr_mod):
    lf = S.make_lightfield("C1")
    p, ora, xs, stats, st = run_pair(lfsr_mod, lf, 20)
    errs = check_iterates(p, ora, xs, stats, st, lf.x_gt)
    print("C1 per-iterate rel L2:", ["%.2e" % e for e in errs])


def test_admm_parity_C1_variants(lfsr_mod):
    """l1-only, l2-only, frozen weights, K=1 and a tau > 0 early stop."""
    lf = S.make_lightfield("C1")
    for over in (dict(lambda2=0.0), dict(lambda1=0.0), dict(reweight_every_iter=0), dict(cg_max_iters=1),
                 dict(cg_tol=1e-3, cg_max_iters=12), dict(nltv_radius=1, theta=3.0)):
        p, ora, xs, stats, st = run_pair(lfsr_mod, lf, 5, **over)
        check_iterates(p, ora, xs, stats, st, lf.x_gt)


@pytest.mark.parametrize("cfg,bl,gnw", [("C1", 1, None), ("C1", 5, "3,7"), ("C2", 8, "1,12"), ("C4", 22, "2,12"),
                                        ("C2", 12, "25,1")])
def test_admm_parity_forced_tile_height(lfsr_mod, monkeypatch, cfg, bl, gnw):
    """Every tiling the per-problem tuning may pick (set_observations times a few tile heights x
    view-group / warp splits and keeps the fastest) gives the same iterates: LFSR_TILE_BL and
    LFSR_TILE_GNW force one, including degenerate 1-row tiles, heights that leave a ragged last
    band, and one view per CTA."""
    monkeypatch.setenv("LFSR_TILE_BL", str(bl))
    if gnw:
        monkeypatch.setenv("LFSR_TILE_GNW", gnw)
    lf = S.make_lightfield(cfg)
    p, ora, xs, stats, st = run_pair(lfsr_mod, lf, 2)
    check_iterates(p, ora, xs, stats, st, lf.x_gt)


def log_parity(name, p, ora, xs, stats, errs, gt):
    """One line per parity run (pytest -rP / -s shows it; profiles/ keeps the round's log)."""
    d_psnr = O.psnr(xs[-1], gt) - O.psnr(ora.x_iters[-1], gt)
    jrel = max(abs(g["J"] - o["J"]) / abs(o["J"]) for g, o in zip(stats, ora.stats))
    rrel = max(abs(g["primal_res"] - o["primal_res"]) / max(o["primal_res"], 1e-12) for g, o in zip(stats, ora.stats))
    print("PARITY %s N=%d zeta=%d: max rel L2 x^n %.2e (per n: %s); max rel J %.2e; max rel primal_res %.2e; "
          "PSNR gpu %.4f oracle %.4f delta %+.5f dB" % (name, len(xs) - 1, p.scale, max(errs),
                                                      " ".join("%.1e" % e for e in errs), jrel, rrel,
                                                      O.psnr(xs[-1], gt), O.psnr(ora.x_iters[-1], gt), d_psnr))


@pytest.mark.parametrize("cfg,n", [("C2", 10), ("C3", 10), ("C4", 10)])
def test_admm_parity_full_size(lfsr_mod, cfg, n):
    """BASELINE configs at full size, in the launch configuration bench.py times and at the bench's
    N = 10 (x^n per iterate <= 1e-4, J / primal residual, w_A / w_S, final PSNR within 0.01 dB)."""
    lf = S.make_lightfield(cfg)
    p, ora, xs, stats, st = run_pair(lfsr_mod, lf, n)
    errs = check_iterates(p, ora, xs, stats, st, lf.x_gt)
    log_parity(cfg, p, ora, xs, stats, errs, lf.x_gt)


# C5-shaped (9x9 views, zeta = 4, R = 3) at a size the oracle runs in seconds per iteration
C5R = {kind: S.Config("C5r", 9, 128, 128, 4, 0.02 if kind == "natural" else 0.05, 5.0 if kind == "natural" else 20.0,
                      1.0 if kind == "natural" else 1.5, kind, 5, "C5-shaped reduced: 9x9 views 128^2 -> 512^2")
       for kind in ("natural", "hci")}


@pytest.mark.parametrize("kind", ["natural", "hci"])
def test_admm_parity_zeta4_C5_shaped(lfsr_mod, kind):
    """The zeta = 4 wz-step (MODE_WZ of the zeta = 4 kernel instances: weights, data shrink/dual,
    NLTV shrink/dual, r = -v) and CG against the oracle iterate by iterate: 9x9 views, 128^2 -> 512^2,
    N = 5, both scene kinds (natural: C5's; hci: depth edges, severe noise)."""
    lf = S.make_lightfield(C5R[kind], seed=1505 if kind == "natural" else 1506)
    p, ora, xs, stats, st = run_pair(lfsr_mod, lf, 5)
    errs = check_iterates(p, ora, xs, stats, st, lf.x_gt)
    log_parity("C5r-" + kind, p, ora, xs, stats, errs, lf.x_gt)


def test_admm_parity_full_size_C5(lfsr_mod):
    """C5 (9x9 views, 512^2 -> 2048^2, zeta = 4) at full size, whole ADMM iterations (N = 2) against
    the oracle (about half a minute per iteration on the host cores)."""
    lf = S.make_lightfield("C5")
    p, ora, xs, stats, st = run_pair(lfsr_mod, lf, 2)
    errs = check_iterates(p, ora, xs, stats, st, lf.x_gt)
    log_parity("C5", p, ora, xs, stats, errs, lf.x_gt)


def test_continuation_and_determinism(lfsr_mod):
    lf = S.make_lightfield("C1")
    p = lfsr_mod.Params(n_views=9, lr_height=32, lr_width=32, scale=2, ref_view=4)
    a = lfsr_mod.Solver(p)
    a.set_observations(lf.y, lf.view_offsets, lf.omega)
    a.admm_run(3)
    a.admm_run(4)
    xa = a.get_hr()
    b = lfsr_mod.Solver(p)
    b.set_observations(lf.y, lf.view_offsets, lf.omega)
    st = b.admm_run(7)
    xb = b.get_hr()
    assert [r["iter"] for r in st] == list(range(1, 8))
    assert rel_l2(xa, xb) < 1e-6
    b.set_observations(lf.y, lf.view_offsets, lf.omega)   # reset: x = x0, w = 0
    b.admm_run(7)
    assert rel_l2(b.get_hr(), xb) < 1e-6


def test_device_pointer_path(lfsr_mod):
    import torch
    lf = S.make_lightfield("C1")
    p = lfsr_mod.Params(n_views=9, lr_height=32, lr_width=32, scale=2, ref_view=4)
    a = lfsr_mod.Solver(p, stream=torch.cuda.current_stream().cuda_stream)
    a.set_observations(torch.from_numpy(lf.y).cuda(), torch.from_numpy(lf.view_offsets).cuda(),
                       torch.from_numpy(lf.omega).cuda())
    a.admm_run(3)
    out = torch.empty((64, 64), device="cuda")
    a.get_hr(out)
    torch.cuda.synchronize()
    b = lfsr_mod.Solver(p)
    b.set_observations(lf.y, lf.view_offsets, lf.omega)
    b.admm_run(3)
    assert rel_l2(out.cpu().numpy(), b.get_hr()) < 1e-6


def test_device_tensors_without_stream(lfsr_mod):
    """A Solver on its own stream (no stream given) used with CUDA tensors produced by torch work on
    torch's current stream: the binding orders the ctx stream after it and torch after the ctx
    (lfsr_get_stream), so the results equal the host path."""
    import torch
    lf = S.make_lightfield("C1")
    p = lfsr_mod.Params(n_views=9, lr_height=32, lr_width=32, scale=2, ref_view=4)
    a = lfsr_mod.Solver(p)
    y = torch.from_numpy(lf.y).cuda() * 1.0          # produced by a kernel on torch's stream
    a.set_observations(y, torch.from_numpy(lf.view_offsets).cuda(), torch.from_numpy(lf.omega).cuda())
    xin = torch.linspace(-1, 1, p.H * p.W, device="cuda").reshape(p.H, p.W) * 2.0
    out = a.op("NORMAL", xin.double())               # a marshalling temporary (.float()) on the device
    got = (out * 1.0).cpu().numpy()                  # consumed by torch right away
    b = lfsr_mod.Solver(p)
    b.set_observations(lf.y, lf.view_offsets, lf.omega)
    assert rel_l2(got, b.op("NORMAL", xin.cpu().numpy())) < 1e-6
    a.admm_run(2)
    b.admm_run(2)
    xd = torch.zeros((p.H, p.W), device="cuda")
    a.get_hr(xd)
    assert rel_l2((xd + 0.0).cpu().numpy(), b.get_hr()) < 1e-6


def test_two_contexts_of_different_geometry(lfsr_mod):
    """The kernels' dynamic shared-memory limit is a per-process attribute: a ctx set up later with a
    smaller tile must not lower it below the footprint of a live ctx with a larger one."""
    big = S.make_lightfield("C2")
    pb = lfsr_mod.params_for(S.CONFIGS["C2"], S.SolverDefaults())
    a = lfsr_mod.Solver(pb)
    a.set_observations(big.y, big.view_offsets, big.omega)
    small = S.make_lightfield("C1")
    ps = lfsr_mod.params_for(S.CONFIGS["C1"], S.SolverDefaults())
    b = lfsr_mod.Solver(ps)
    b.set_observations(small.y, small.view_offsets, small.omega * 0.1)   # a thinner halo: smaller tile
    assert len(b.admm_run(1)) == 1
    assert len(a.admm_run(1)) == 1
    x = np.random.default_rng(3).uniform(-1, 1, (pb.H, pb.W)).astype(np.float32)
    assert np.isfinite(a.op("NORMAL", x)).all()
    a.close()
    b.close()


def test_error_paths(lfsr_mod):
    p = lfsr_mod.Params(n_views=9, lr_height=32, lr_width=32, scale=2, ref_view=4)
    s = lfsr_mod.Solver(p)
    with pytest.raises(lfsr_mod.LFSRError) as ei:
        s.admm_run(1)
    assert ei.value.status == 2  # LFSR_ERR_STATE
    lf = S.make_lightfield("C1")
    bad = lf.view_offsets.copy()
    bad[0, 0] = np.nan
    with pytest.raises(lfsr_mod.LFSRError) as ei:
        s.set_observations(lf.y, bad, lf.omega)
    assert ei.value.status == 1
    # non-finite disparity (inf, and NaN -- invalid pixels of real disparity maps) is rejected up front
    for bad_v in (np.inf, np.nan, -np.nan):
        om = lf.omega.copy()
        om[3, 3] = bad_v
        with pytest.raises(lfsr_mod.LFSRError) as ei:
            s.set_observations(lf.y, lf.view_offsets, om)
        assert ei.value.status == 1, bad_v
    # a shift reaching past the image is refused (UNSUPPORTED), not sampled out of the tile
    om = lf.omega.copy()
    om[5, 5] = 1e30
    with pytest.raises(lfsr_mod.LFSRError) as ei:
        s.set_observations(lf.y, lf.view_offsets, om)
    assert ei.value.status == 7
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    assert len(s.admm_run(2)) == 2
    npth = s.normal_path   # CG operator: tile kernel (1 launch) or assembled (1, + 3 with irregular rows)
    per_step = 1 if npth["name"] == "tile" else (4 if npth["irregular_rows"] else 1)
    assert s.launches_per_iter == 1 + (per_step + 1) * p.cg_max_iters


def test_divergence_guard(lfsr_mod):
    lf = S.make_lightfield("C1")
    p = lfsr_mod.Params(n_views=9, lr_height=32, lr_width=32, scale=2, ref_view=4)
    s = lfsr_mod.Solver(p)
    y = lf.y.copy()
    y[0, 0, 0] = np.nan
    s.set_observations(y, lf.view_offsets, lf.omega)
    with pytest.raises(lfsr_mod.LFSRError) as ei:
        s.admm_run(2)
    assert ei.value.status == 6  # LFSR_ERR_DIVERGED
    assert ei.value.stats[0]["nonfinite"] == 1


def test_full_size_C5_sampled(lfsr_mod):
    """C5 (9x9 views, 512^2 -> 2048^2, zeta = 4) at full size in the bench launch configuration:
    A and the normal operator are checked on interior crops the oracle can afford (an interior
    pixel only sees its neighbourhood, so a crop with a margin wider than the operator's reach
    gives the same values), plus the adjoint identity over the whole image."""
    lf = S.make_lightfield("C5")
    d = S.SolverDefaults()
    c = S.CONFIGS["C5"]
    p = lfsr_mod.params_for(c, d)
    s = lfsr_mod.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    g = np.random.default_rng(5)
    x = g.uniform(-1, 1, (c.H, c.W)).astype(np.float32)
    ax = s.op("A", x)
    mx = s.op("NORMAL", x)
    m = s.get_state()["m"]
    z = c.scale
    margin_lr = 16                                   # >= reach: (R + S_max + 1) / zeta, doubled for M
    for (i0, j0) in [(100, 140), (300, 37), (470, 420)]:
        h = w = 24
        li0, lj0 = i0 - margin_lr, j0 - margin_lr
        hh, ww = h + 2 * margin_lr, w + 2 * margin_lr
        P = O.Params(n_views=c.n_views, lr_h=hh, lr_w=ww, scale=z, ref_view=c.ref_view, radius=d.radius,
                     lambda1=d.lambda1, lambda2=d.lambda2, lambda_reg=d.lambda_reg, sigma_s=d.sigma_s,
                     sigma_e=d.sigma_e, sigma_o1=d.sigma_o1, sigma_o2=d.sigma_o2, theta=d.theta)
        sl = (slice(li0 * z, (li0 + hh) * z), slice(lj0 * z, (lj0 + ww) * z))
        a_ora = O.apply_A(P, lf.view_offsets, lf.omega[sl], x[sl])
        inner = (slice(None), slice(margin_lr, margin_lr + h), slice(margin_lr, margin_lr + w))
        got = ax[:, i0:i0 + h, j0:j0 + w]
        assert rel_l2(got, a_ora[inner]) < OP_TOL
        m_ora = O.normal(P, lf.view_offsets, lf.omega[sl], m[sl], x[sl])
        inner_hr = (slice(margin_lr * z, (margin_lr + h) * z), slice(margin_lr * z, (margin_lr + w) * z))
        got_m = mx[i0 * z:(i0 + h) * z, j0 * z:(j0 + w) * z]
        assert rel_l2(got_m, m_ora[inner_hr]) < OP_TOL
    r = g.standard_normal((c.n_views, c.lr_h, c.lr_w)).astype(np.float32)
    atr = s.op("AT", r).astype(np.float64)
    lhs, rhs = float(np.vdot(ax.astype(np.float64), r)), float(np.vdot(x.astype(np.float64), atr))
    assert abs(lhs - rhs) <= 1e-6 * np.linalg.norm(ax) * np.linalg.norm(r)
    st = s.admm_run(1)
    assert st[0]["cg_iters"] == d.cg_max_iters and not st[0]["nonfinite"]
    s.close()


# ----------------------------------------------------------------------------- MISR (NEXT-1)
def test_misr_operator_parity_btv_weights(lfsr_mod):
    """S / S^T / M with user offset weights (BTV alpha^(|dx|+|dy|)) and global-shift frames."""
    lf = S.make_lightfield("M1")
    d = S.MisrDefaults()
    p = lfsr_mod.params_for(S.CONFIGS["M1"], d)
    s = lfsr_mod.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    P = oparams(p)
    g = np.random.default_rng(17)
    xin = g.uniform(-1, 1, (p.H, p.W)).astype(np.float32)
    hin = g.uniform(-1, 1, (p.s_d, p.H, p.W)).astype(np.float32)
    m = s.get_state()["m"]
    assert np.allclose(m, d.lambda_reg)          # sigma_e = sigma_o = inf: m = lambda_R
    w = d.offset_weights
    assert rel_l2(s.op("S", xin), O.apply_S(xin, m, p.nltv_radius, p.sigma_s, weights=w)) < OP_TOL
    assert rel_l2(s.op("ST", hin), O.apply_ST(hin, m, p.nltv_radius, p.sigma_s, weights=w)) < OP_TOL
    assert rel_l2(s.op("NORMAL", xin), O.normal(P, lf.view_offsets, lf.omega, m, xin)) < OP_TOL
    s.close()


def test_misr_admm_parity(lfsr_mod):
    """The MISR use: l1 + BTV, lambda2 = 0, 4 frames x2 with global shifts."""
    lf = S.make_lightfield("M1")
    p, ora, xs, stats, st = run_pair(lfsr_mod, lf, 10, defaults=S.MisrDefaults())
    check_iterates(p, ora, xs, stats, st, lf.x_gt)


# ----------------------------------------------------------------------------- k_wz_nltv (nltv.cu)
@pytest.mark.parametrize("cfg,n", [("C1", 10), ("C4", 2)])
def test_nltv_split_kernel_parity(lfsr_mod, cfg, n, monkeypatch):
    """The NLTV rows of the wz-step in the streaming kernel (default for large images; forced here on
    small ones, C4's 513 columns exercise the ragged last float4 chunk) against the oracle."""
    monkeypatch.setenv("LFSR_NLTV_SPLIT", "1")
    lf = S.make_lightfield(cfg)
    p, ora, xs, stats, st = run_pair(lfsr_mod, lf, n)
    check_iterates(p, ora, xs, stats, st, lf.x_gt)
    errs = [rel_l2(xs[i], ora.x_iters[i]) for i in range(n + 1)]
    print("PARITY nltv-split %s N=%d: %s" % (cfg, n, " ".join("%.1e" % e for e in errs)))


def test_nltv_split_strips(lfsr_mod, monkeypatch):
    """The split kernel on each strip's own rows (virtual ranks) equals the single-strip solve."""
    monkeypatch.setenv("LFSR_NLTV_SPLIT", "1")
    lf = S.make_lightfield("C2")
    d = S.SolverDefaults()
    out = []
    for over in ({}, dict(n_ranks=3, rank=-1)):
        p = lfsr_mod.params_for(S.CONFIGS["C2"], d, **over)
        s = lfsr_mod.Solver(p)
        s.set_observations(lf.y, lf.view_offsets, lf.omega)
        s.admm_run(2)
        out.append(s.get_hr())
        s.close()
    assert rel_l2(out[1], out[0]) <= 1e-5
