"""GPU parity of the MISR / global-shift fast path (misr.cu):
with a constant disparity the CG operator's data part runs as a precomputed stencil: for a Cartesian
grid of shifts (MISR frames, a light-field grid) the separable form T_y (x) T_x with exact banded 1-D
matrices over the whole image, otherwise a zeta^2-phase stencil on the interior rectangle Z_s with the
exact tile kernel on the border tiles.  Checked against the
fp64 oracle (the operator M and ADMM iterates) and against the generic path of the same library
(LFSR_MISR_FAST=0), on MISR-shaped inputs (integer HR shifts), fractional constant shifts, and
every zeta; the gate itself (constant maps only) is checked too."""
import os

import numpy as np
import pytest

import oracle as O
import lfsr_synth as S
from test_gpu_parity import OP_TOL, ITER_TOL, PSNR_TOL, oparams, rel_l2, run_pair, check_iterates

pytestmark = pytest.mark.gpu


def _solver(lfsr_mod, p, y, vo, om, fast=True):
    old = os.environ.get("LFSR_MISR_FAST")
    os.environ["LFSR_MISR_FAST"] = "1" if fast else "0"
    try:
        s = lfsr_mod.Solver(p)
        s.set_observations(y, vo, om)
    finally:
        if old is None:
            del os.environ["LFSR_MISR_FAST"]
        else:
            os.environ["LFSR_MISR_FAST"] = old
    return s


def misr_instance(seed, grid, lr, z, c=1.0, frac=False, lw=None):
    """grid x grid frames, constant disparity c; offsets = MISR shifts (integer HR px) or generic
    fractional offsets (the 'fractional' case makes every W_k a bilinear translation); lr x lw LR."""
    g = np.random.Generator(np.random.Philox(seed))
    lw = lr if lw is None else lw
    H, W = lr * z, lw * z
    if frac == "grid":     # a light-field grid of views with one constant disparity: separable form
        vo = S.grid_offsets(grid)
    elif frac:
        vo = g.uniform(-2.5, 2.5, (grid * grid, 2)).astype(np.float32)
    else:
        vo = S.misr_offsets(grid)
    om = np.full((H, W), c, np.float32)
    y = g.uniform(0.0, 1.0, (grid * grid, lr, lw)).astype(np.float32)
    x = g.uniform(0.0, 1.0, (H, W)).astype(np.float32)
    return y, vo, om, x


CASES = [dict(seed=1, grid=2, lr=64, z=2, c=1.0, frac=False),       # M2-shaped
         dict(seed=2, grid=2, lr=128, z=2, c=1.0, frac=False),
         dict(seed=3, grid=3, lr=60, z=3, c=1.0, frac=False),       # M3-shaped
         dict(seed=4, grid=3, lr=96, z=2, c=0.37, frac=True),       # fractional constant shifts
         dict(seed=5, grid=3, lr=50, z=3, c=-0.8, frac=True),
         dict(seed=6, grid=2, lr=40, z=4, c=0.6, frac=True),
         dict(seed=7, grid=3, lr=33, z=4, c=1.0, frac=False),
         dict(seed=8, grid=3, lr=64, z=2, c=0.37, frac="grid"),     # LF grid, constant fractional disparity
         dict(seed=9, grid=5, lr=45, z=3, c=-1.3, frac="grid"),
         dict(seed=10, grid=9, lr=40, z=4, c=0.9, frac="grid"),
         dict(seed=11, grid=2, lr=37, lw=90, z=2, c=1.0, frac=False),      # non-square, ragged tiles
         dict(seed=12, grid=3, lr=70, lw=29, z=3, c=0.45, frac="grid"),
         dict(seed=13, grid=3, lr=61, lw=95, z=2, c=0.3, frac=True)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "g%d_lr%dx%d_z%d_%s" % (
    c["grid"], c["lr"], c.get("lw", c["lr"]), c["z"], c["frac"] if c["frac"] else "int"))
def test_misr_fast_normal_parity(lfsr_mod, case):
    y, vo, om, x = misr_instance(case["seed"], case["grid"], case["lr"], case["z"], case["c"], case["frac"],
                                 case.get("lw"))
    d = S.MisrDefaults()
    p = lfsr_mod.Params(n_views=len(vo), lr_height=case["lr"], lr_width=case.get("lw", case["lr"]), scale=case["z"],
                        ref_view=0,
                        nltv_radius=2, lambda1=d.lambda1, lambda2=0.7, lambda_reg=0.3, sigma_s=d.sigma_s,
                        sigma_e=0.2, sigma_o1=0.5, sigma_o2=0.2, theta=d.theta, cg_max_iters=5)
    sf = _solver(lfsr_mod, p, y, vo, om, fast=True)
    sg = _solver(lfsr_mod, p, y, vo, om, fast=False)
    fp = sf.fast_path
    assert fp["misr"], fp
    assert not sg.fast_path["misr"]
    zs = fp["zs"]
    assert zs[1] - zs[0] > 0 and zs[3] - zs[2] > 0
    # a Cartesian grid of shifts takes the separable form over the whole image (no border kernel)
    if case["frac"] in (False, "grid"):
        assert zs == (0, p.H, 0, p.W), zs
    P = oparams(p)
    g = np.random.default_rng(case["seed"] + 11)
    xin = g.uniform(-1, 1, (p.H, p.W)).astype(np.float32)
    m = sf.get_state()["m"]
    ref = O.normal(P, vo, om, m, xin)
    qf, qg = sf.op("NORMAL", xin), sg.op("NORMAL", xin)
    e_or, e_gen = rel_l2(qf, ref), rel_l2(qf, qg)
    # band and interior separately (both must hold)
    inside = np.zeros_like(ref, dtype=bool)
    inside[zs[0]:zs[1], zs[2]:zs[3]] = True
    e_in = rel_l2(qf[inside], ref[inside])
    e_band = rel_l2(qf[~inside], ref[~inside])
    print("PARITY misr-fast NORMAL %s: vs oracle %.1e (Z_s %.1e, band %.1e), vs generic %.1e" % (
        case, e_or, e_in, e_band, e_gen))
    assert e_or < OP_TOL and e_in < OP_TOL and e_band < OP_TOL and e_gen < OP_TOL
    sf.close()
    sg.close()


def test_misr_fast_gate(lfsr_mod):
    """Only constant maps take the fast path; a light field (varying disparity) does not."""
    lf = S.make_lightfield("C1")
    p = lfsr_mod.params_for(S.CONFIGS["C1"], S.SolverDefaults())
    s = lfsr_mod.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    assert not s.fast_path["misr"]
    om = np.full_like(lf.omega, 0.5)
    s.set_observations(lf.y, lf.view_offsets, om)
    assert s.fast_path["misr"]
    om[5, 7] = 0.5000001
    s.set_observations(lf.y, lf.view_offsets, om)
    assert not s.fast_path["misr"]
    s.close()


def test_misr_fast_admm_parity_M1(lfsr_mod):
    """M1 through the fast path (10 iterations, the oracle's iterates; default MISR constants)."""
    lf = S.make_lightfield("M1")
    p, ora, xs, stats, st = run_pair(lfsr_mod, lf, 10, defaults=S.MisrDefaults())
    check_iterates(p, ora, xs, stats, st, lf.x_gt)


@pytest.mark.parametrize("grid,lr,z", [(2, 128, 2), (3, 96, 3)])
def test_misr_fast_admm_parity_midsize(lfsr_mod, grid, lr, z):
    """MISR-shaped frames (M2 / M3 shifts, natural texture), N = 5 ADMM iterations: fast path vs
    the oracle (per-iterate <= 1e-4, PSNR within 0.01 dB) and vs the generic path."""
    cfg = S.Config("Mx", grid, lr, lr, z, 0.02, 5.0, 1.0, "misr", 5)
    lf = S.make_lightfield(cfg, seed=4242 + z)
    d = S.MisrDefaults()
    p = lfsr_mod.params_for(cfg, d)
    P = oparams(p)
    n = 5
    ora = O.admm(P, lf.y, lf.view_offsets, lf.omega, n)
    res = {}
    for fast in (True, False):
        s = _solver(lfsr_mod, p, lf.y, lf.view_offsets, lf.omega, fast=fast)
        assert s.fast_path["misr"] == fast
        xs, stats = [s.get_hr()], []
        for _ in range(n):
            stats += s.admm_run(1)
            xs.append(s.get_hr())
        s.close()
        res[fast] = (xs, stats)
    xs, stats = res[True]
    errs = [rel_l2(xs[i], ora.x_iters[i]) for i in range(n + 1)]
    egen = max(rel_l2(a, b) for a, b in zip(res[True][0], res[False][0]))
    print("PARITY misr-fast ADMM grid %d lr %d z %d N=%d: per-iterate %s; vs generic %.1e; PSNR %.3f vs %.3f" % (
        grid, lr, z, n, " ".join("%.1e" % e for e in errs), egen, O.psnr(xs[-1], lf.x_gt),
        O.psnr(ora.x_iters[-1], lf.x_gt)))
    assert max(errs) <= ITER_TOL, errs
    assert egen <= 1e-5
    for g_, o in zip(stats, ora.stats):
        assert abs(g_["J"] - o["J"]) <= ITER_TOL * abs(o["J"])
        assert g_["cg_iters"] == o["cg_iters"]
    assert abs(O.psnr(xs[-1], lf.x_gt) - O.psnr(ora.x_iters[-1], lf.x_gt)) <= PSNR_TOL


def test_misr_fast_full_size_M2(lfsr_mod):
    """M2 (4 frames, 1024^2 -> 2048^2): one ADMM iteration through the fast path vs the oracle."""
    lf = S.make_lightfield("M2")
    d = S.MisrDefaults()
    p = lfsr_mod.params_for(S.CONFIGS["M2"], d)
    P = oparams(p)
    ora = O.admm(P, lf.y, lf.view_offsets, lf.omega, 1)
    s = _solver(lfsr_mod, p, lf.y, lf.view_offsets, lf.omega, fast=True)
    assert s.fast_path["misr"]
    x0 = s.get_hr()
    st = s.admm_run(1)
    x1 = s.get_hr()
    s.close()
    errs = [rel_l2(x0, ora.x_iters[0]), rel_l2(x1, ora.x_iters[1])]
    print("PARITY misr-fast M2 N=1: %s, J rel %.1e" % (" ".join("%.1e" % e for e in errs),
                                                      abs(st[0]["J"] - ora.stats[0]["J"]) / abs(ora.stats[0]["J"])))
    assert max(errs) <= ITER_TOL
    assert st[0]["cg_iters"] == ora.stats[0]["cg_iters"]
