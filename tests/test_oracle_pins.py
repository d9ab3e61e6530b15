"""Pins of the fp64 oracle (oracle/oracle.c) to things other than itself.

Each test names the pin of SURVEY.md §8c.3 / DESIGN.md §3 it implements and the
PAPER.md passage it checks: closed forms, special cases that reduce to a
textbook/library routine, invariants (adjoint identities, symmetry, PSD) and
brute force on tiny inputs.  All CPU-only (no GPU marker).
"""
import math
import os

import numpy as np
import pytest

import oracle as O
from lfsr_synth import random_instance

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# "Exact" x-step: CG converges in p steps only in exact arithmetic; in fp64 on these
# tiny, moderately ill-conditioned systems (cond(A^T A) ~ 5e4) a few hundred steps reach
# machine precision (the pi == 0 guard ends the loop once r vanishes).
EXACT_K = 400


def rnd(seed, *shape):
    return np.random.default_rng(seed).standard_normal(shape)


def rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1e-300)


# ----------------------------------------------------------------------------- P1 D, D^T
def test_P1_decimation_definition(oracle_lib):
    """P:L577 'for each block of zeta x zeta pixels, one pixel at the top-left location is picked'."""
    x = np.arange(16, dtype=float).reshape(4, 4)
    d = O.apply_D(x, 2)
    assert np.array_equal(d, np.array([[0, 2], [8, 10]], dtype=float))
    # P:L578 'putting back the corresponding pixel to this location' (zero elsewhere)
    up = O.apply_DT(np.ones((2, 2)), 2)
    exp = np.zeros((4, 4))
    exp[::2, ::2] = 1
    assert np.array_equal(up, exp)
    y = rnd(1, 3, 5)
    for z in (2, 3, 4):
        y = rnd(z, 3, 5)
        assert np.array_equal(O.apply_D(O.apply_DT(y, z), z), y)  # D D^T = I
        x = rnd(10 + z, 3 * z, 5 * z)
        assert rel(np.vdot(O.apply_D(x, z), y), np.vdot(x, O.apply_DT(y, z))) < 1e-12


# ----------------------------------------------------------------------------- P2 taps
def test_P2_blur_taps_closed_form(oracle_lib):
    """sigma = 1/4 sqrt(zeta^2-1), size 3 sigma (reading A11); values from tests/golden."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "blur_taps.txt")) if l.strip() and l[0] != "#"]
    assert len(rows) == 3
    for r in rows:
        z, sigma, R = int(r[0]), float(r[1]), int(r[2])
        gold = np.array([float(v) for v in r[3:]])
        taps = O.blur_taps(z)
        assert len(taps) == 2 * R + 1
        assert abs(0.25 * math.sqrt(z * z - 1) - sigma) < 1e-7
        assert np.allclose(taps, gold, rtol=2e-7, atol=0)
        assert abs(taps.sum() - 1.0) < 1e-12
        assert np.allclose(taps, taps[::-1], rtol=0, atol=0)


# ----------------------------------------------------------------------------- P3 B
@pytest.mark.parametrize("z", [2, 3, 4])
def test_P3_blur_impulse_constant_adjoint(oracle_lib, z):
    taps = O.blur_taps(z)
    R = (len(taps) - 1) // 2
    x = np.zeros((15, 17))
    x[7, 8] = 1.0
    b = O.apply_B(x, z)
    assert np.allclose(b[7 - R:7 + R + 1, 8 - R:8 + R + 1], np.outer(taps, taps), atol=1e-15)  # impulse response
    assert abs(b.sum() - 1.0) < 1e-12
    c = O.apply_B(np.full((15, 17), 0.37), z)
    assert np.allclose(c[R:-R, R:-R], 0.37, atol=1e-14)  # constants reproduced in the interior
    for s in range(20):
        u, v = rnd(100 + s, 9, 11), rnd(200 + s, 9, 11)
        assert rel(np.vdot(O.apply_B(u, z), v), np.vdot(u, O.apply_B(v, z))) < 1e-12  # B^T = B (zero pad)


# ----------------------------------------------------------------------------- P4 W
def test_P4_warp_special_cases(oracle_lib):
    H, W = 12, 14
    Yg, Xg = np.meshgrid(np.arange(H, dtype=float), np.arange(W, dtype=float), indexing="ij")
    x = rnd(3, H, W)
    om = rnd(4, H, W)
    assert np.array_equal(O.apply_W(x, om, 0.0, 0.0), x)                 # dtheta = 0 -> identity
    ramp = Xg.copy()
    one = np.ones((H, W))
    w1 = O.apply_W(ramp, one, 1.0, 0.0)                                   # omega=1, (drho,dtau)=(1,0)
    assert np.allclose(w1[:, :-1], ramp[:, :-1] + 1.0, atol=1e-14)        # integer shift along X
    assert np.allclose(w1[:, -1], W - 1, atol=1e-14)                      # replicate clamp
    wh = O.apply_W(ramp, 0.5 * one, 1.0, 0.0)
    assert np.allclose(wh[:, :-1], ramp[:, :-1] + 0.5, atol=1e-14)       # half-pixel bilinear
    wt = O.apply_W(ramp, one, 0.0, 1.0)                                   # tau moves rows only (A13)
    assert np.allclose(wt, ramp, atol=1e-14)
    rowramp = Yg.copy()
    wr = O.apply_W(rowramp, 0.25 * one, 0.0, 2.0)
    assert np.allclose(wr[:-1], rowramp[:-1] + 0.5, atol=1e-14)
    # constant omega: W^T is the reverse translation in the interior
    t = rnd(5, H, W)
    wt_ = O.apply_WT(t, one, 2.0, -1.0)  # gather x(Y-1, X+2) -> transpose puts t(Y,X) at (Y-1, X+2)
    assert np.allclose(wt_[2:-2, 3:-3], t[3:-1, 1:-5], atol=1e-14)


def test_P4_warp_adjoint(oracle_lib):
    for s in range(120):
        H, W = 8 + s % 9, 9 + (s * 7) % 11
        x, t = rnd(s, H, W), rnd(1000 + s, H, W)
        om = 2.5 * rnd(2000 + s, H, W)
        dr, dt = np.random.default_rng(s).uniform(-3, 3, 2)
        lhs = np.vdot(O.apply_W(x, om, dr, dt), t)
        rhs = np.vdot(x, O.apply_WT(t, om, dr, dt))
        assert rel(lhs, rhs) < 1e-10


# ----------------------------------------------------------------------------- P5 A stack
def test_P5_stack_adjoint(oracle_lib):
    for s in range(100):
        z = (2, 3, 4)[s % 3]
        nv = 1 + s % 5
        h, w = 2 + s % 4, 3 + s % 3
        y, vo, om, x = random_instance(s, nv, h, w, z)
        P = O.Params(n_views=nv, lr_h=h, lr_w=w, scale=z)
        r = rnd(s + 5000, nv, h, w)
        xx = rnd(s + 6000, h * z, w * z)
        lhs = np.vdot(O.apply_A(P, vo, om, xx), r)
        rhs = np.vdot(xx, O.apply_AT(P, vo, om, r))
        assert rel(lhs, rhs) < 1e-10


def test_P5_stack_is_composition(oracle_lib):
    """A_k = D B W_k view by view."""
    y, vo, om, x = random_instance(7, 3, 5, 6, 2)
    P = O.Params(n_views=3, lr_h=5, lr_w=6, scale=2)
    a = O.apply_A(P, vo, om, x)
    for k in range(3):
        ref = O.apply_D(O.apply_B(O.apply_W(x, om, vo[k, 0], vo[k, 1]), 2), 2)
        assert np.allclose(a[k], ref, atol=1e-14)


# ----------------------------------------------------------------------------- P6 S, S^T
def test_P6_nltv_special_cases(oracle_lib):
    H, W = 9, 10
    m = np.ones((H, W))
    g = O.apply_S(np.full((H, W), 0.7), m, 2, 3.0)
    assert np.allclose(g, 0.0)                                               # constant -> 0
    offs = O.offsets(2)
    assert len(offs) == 24 and (0, 0) not in offs and len(set(offs)) == 24   # s_d = 24 for 5x5 (A9)
    assert len(O.offsets(1)) == 8                                             # s_d = 8 for 3x3
    Xg = np.meshgrid(np.arange(H, dtype=float), np.arange(W, dtype=float), indexing="ij")[1]
    g = O.apply_S(Xg, m, 1, math.inf)                                         # unit weights
    d = offs_index = O.offsets(1).index((0, 1))
    assert np.allclose(g[d][:, :-1], -1.0)                                   # x(z) - x(z+d) = -1
    assert np.allclose(g[d][:, -1], 0.0)                                     # pair leaves Omega (A10)
    wd = math.exp(-(1 + 4) / 3.0)
    mm = rnd(3, H, W) ** 2
    g = O.apply_S(Xg, mm, 2, 3.0)
    j = O.offsets(2).index((1, 2))
    assert np.allclose(g[j][:-1, :-2], wd * mm[:-1, :-2] * (-2.0))          # W_d = w_d m, w_d = e^{-|d|^2/s}


def test_P6_nltv_adjoint_and_bruteforce(oracle_lib):
    for s in range(100):
        H, W = 4 + s % 7, 5 + s % 6
        r = 1 + s % 3
        m = np.abs(rnd(s, H, W))
        x = rnd(s + 1, H, W)
        hh = rnd(s + 2, (2 * r + 1) ** 2 - 1, H, W)
        lhs = np.vdot(O.apply_S(x, m, r, 2.0), hh)
        rhs = np.vdot(x, O.apply_ST(hh, m, r, 2.0))
        assert rel(lhs, rhs) < 1e-10
    # S^T S delta equals the dense brute-force (built column by column) on 6x6
    H = W = 6
    m = np.abs(rnd(9, H, W)) + 0.1
    cols = []
    for i in range(H * W):
        e = np.zeros(H * W)
        e[i] = 1
        cols.append(O.apply_S(e.reshape(H, W), m, 2, 3.0).ravel())
    Sd = np.array(cols).T
    for i in (0, 7, 14, 35):
        e = np.zeros(H * W)
        e[i] = 1
        ref = Sd.T @ (Sd @ e)
        got = O.apply_ST(O.apply_S(e.reshape(H, W), m, 2, 3.0), m, 2, 3.0).ravel()
        assert np.allclose(got, ref, atol=1e-13)


# ----------------------------------------------------------------------------- P7 prox
def test_P7_prox_closed_form_and_clamp_identity():
    """Eq. sr_l1l2l1_prox examples; w+ = u - prox(u) = clamp(u, +-1/theta) (A5/A6)."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "prox_examples.txt")) if l.strip() and l[0] != "#"]
    for r in rows:
        th, u, z, w = map(float, r)
        soft = max(abs(u) - 1 / th, 0.0) * math.copysign(1.0, u)
        assert abs(soft - z) < 1e-12
        assert abs((u - soft) - w) < 1e-12
        assert abs(min(max(u, -1 / th), 1 / th) - w) < 1e-12
    u = np.random.default_rng(0).standard_normal(10 ** 6) * 3
    for th in (0.5, 1.0, 3.0):
        soft = np.maximum(np.abs(u) - 1 / th, 0) * np.sign(u)
        assert np.array_equal(u - soft, np.clip(u, -1 / th, 1 / th)) or np.allclose(u - soft, np.clip(u, -1 / th, 1 / th), atol=1e-15)


# ----------------------------------------------------------------------------- helpers: dense operators
def dense_ops(P, vo, om, m):
    H, W = P.H, P.W
    p = H * W
    Acols, Scols = [], []
    for i in range(p):
        e = np.zeros(p)
        e[i] = 1
        Acols.append(O.apply_A(P, vo, om, e.reshape(H, W)).ravel())
        Scols.append(O.apply_S(e.reshape(H, W), m, P.radius, P.sigma_s).ravel())
    return np.array(Acols).T, np.array(Scols).T


def tiny(seed=11, nv=2, h=4, w=4, z=2, **kw):
    y, vo, om, x = random_instance(seed, nv, h, w, z)
    P = O.Params(n_views=nv, lr_h=h, lr_w=w, scale=z, ref_view=0, **kw)
    return P, y, vo, om, x


# ----------------------------------------------------------------------------- P8 M
def test_P8_normal_operator_dense(oracle_lib):
    """M = (l2 + th/2 l1^2) A^T A + th/2 S^T S (A7) vs dense, symmetric PSD."""
    P, y, vo, om, x = tiny(lambda1=0.7, lambda2=1.3, theta=2.5)
    m = np.abs(rnd(5, P.H, P.W)) + 0.05
    Ad, Sd = dense_ops(P, vo, om, m)
    cA = P.lambda2 + 0.5 * P.theta * P.lambda1 ** 2
    Md = cA * Ad.T @ Ad + 0.5 * P.theta * Sd.T @ Sd
    p = P.H * P.W
    cols = np.array([O.normal(P, vo, om, m, np.eye(p)[i].reshape(P.H, P.W)).ravel() for i in range(p)]).T
    assert np.allclose(cols, Md, atol=1e-12 * np.abs(Md).max())
    assert np.allclose(cols, cols.T, atol=1e-12 * np.abs(Md).max())
    assert np.linalg.eigvalsh(0.5 * (cols + cols.T)).min() > -1e-10


# ----------------------------------------------------------------------------- P10 l2-only
def test_P10_l2_only_equals_lstsq(oracle_lib):
    """lambda1 = 0, lambda_R = 0, noiseless y = A x_gt: one ADMM iteration with an exact x-step
    (K = EXACT_K CG steps) is the least-squares solution (np.linalg.lstsq)."""
    nv, h, w, z = 9, 4, 4, 2
    P, _, vo, om, xgt = tiny(seed=21, nv=nv, h=h, w=w, z=z, lambda1=0.0, lambda2=1.0, lambda_reg=0.0,
                             cg_max_iters=EXACT_K, cg_tol=0.0)
    Ad, _ = dense_ops(P, vo, om, np.ones((P.H, P.W)))
    assert np.linalg.matrix_rank(Ad) == P.H * P.W
    y = (Ad @ xgt.astype(np.float64).ravel()).reshape(nv, h, w)
    x0 = np.full((P.H, P.W), 0.5)
    res = O.admm(P, y, vo, om, 1, x0=x0)
    ls = np.linalg.lstsq(Ad, y.ravel(), rcond=None)[0]
    assert np.allclose(res.x_iters[1].ravel(), ls, atol=1e-8)
    assert np.allclose(res.x_iters[1].ravel(), xgt.ravel(), atol=1e-7)


# ----------------------------------------------------------------------------- P11 Alg.1 algebra
def textbook_admm(Ad, Sd, y, l1, l2, th, x0, N):
    """Scaled ADMM on the compact problem (Eq. sr_admm_compact; steps
    P:L520-534 in the paper's z -> w -> x order, Alg.1), coded from the equations with
    dense matrices: A = sqrt(l2) Abar, b = sqrt(l2) y, F = [l1/sqrt(l2) A; S], b' = [l1/sqrt(l2) b; 0]."""
    s2 = math.sqrt(l2)
    A = s2 * Ad
    b = s2 * y
    F = np.vstack([(l1 / s2) * A, Sd])
    bp = np.concatenate([(l1 / s2) * b, np.zeros(Sd.shape[0])])
    x = x0.copy()
    w = np.zeros(F.shape[0])
    G = A.T @ A + 0.5 * th * F.T @ F  # G^T G of Eq. sr_l1l2l1_lsf (without the sqrt factors)
    xs = [x.copy()]
    ws = [w.copy()]
    for _ in range(N):
        u = F @ x - bp + w
        zz = np.maximum(np.abs(u) - 1 / th, 0) * np.sign(u)   # prox
        w = u - zz                                            # Alg.1 line 7 (scaled dual)
        rhs = A.T @ b + 0.5 * th * F.T @ (zz + bp - w)          # normal equations of
        x = np.linalg.solve(G, rhs)
        xs.append(x.copy())
        ws.append(w.copy())
    textbook_admm.ws = ws   # the scaled dual sequence w^0..w^N (block order [data rows; NLTV rows])
    return xs


def test_P11_alg1_equals_textbook_scaled_admm(oracle_lib):
    P, y, vo, om, x = tiny(seed=31, nv=3, h=4, w=4, z=2, lambda1=0.8, lambda2=2.0, theta=1.5, lambda_reg=0.4,
                           sigma_e=0.05, cg_max_iters=EXACT_K, reweight_every_iter=0)
    y = y.astype(np.float64)
    x0 = O.bicubic(y[P.ref_view], P.scale)
    wo, _, _ = O.setup_wo(P, y, vo, om)
    m = O.weights_m(x0, wo, P.lambda_reg, P.sigma_e)    # frozen weights (reweight_every_iter = 0)
    Ad, Sd = dense_ops(P, vo, om, m)
    N = 6
    xs = textbook_admm(Ad, Sd, y.ravel(), P.lambda1, P.lambda2, P.theta, x0.ravel(), N)
    res = O.admm(P, y, vo, om, N)
    for n in range(N + 1):
        assert np.allclose(res.x_iters[n].ravel(), xs[n], atol=1e-8), n


def test_P11_primal_residual_and_duals_equal_textbook(oracle_lib):
    """A27's primal residual |w^n - w^{n-1}|_2 pinned by value: the textbook scaled ADMM above tracks
    w = [w_A; w_S] on the compact F = [l1/sqrt(l2) A; S] (whose data rows are l1 (Abar x - y), so its
    scaled dual is the oracle's w_A itself, and its NLTV rows are S_w x, the oracle's w_S), so the
    oracle's reported primal_res of iteration n must equal |ws[n] - ws[n-1]| of that independent
    sequence, and its final w_A / w_S states must equal ws[N]."""
    P, y, vo, om, x = tiny(seed=37, nv=3, h=4, w=4, z=2, lambda1=0.9, lambda2=1.5, theta=2.0, lambda_reg=0.6,
                           sigma_e=0.05, cg_max_iters=EXACT_K, reweight_every_iter=0)
    y = y.astype(np.float64)
    x0 = O.bicubic(y[P.ref_view], P.scale)
    wo, _, _ = O.setup_wo(P, y, vo, om)
    m = O.weights_m(x0, wo, P.lambda_reg, P.sigma_e)
    Ad, Sd = dense_ops(P, vo, om, m)
    N = 6
    textbook_admm(Ad, Sd, y.ravel(), P.lambda1, P.lambda2, P.theta, x0.ravel(), N)
    ws = textbook_admm.ws
    res = O.admm(P, y, vo, om, N)
    for n in range(1, N + 1):
        want = float(np.linalg.norm(ws[n] - ws[n - 1]))
        assert want > 1e-6, n                       # the pin is not vacuous
        assert rel(res.stats[n - 1]["primal_res"], want) < 1e-9, (n, res.stats[n - 1]["primal_res"], want)
    nA = Ad.shape[0]
    assert np.allclose(res.wA.ravel(), ws[N][:nA], atol=1e-9)
    # dense_ops builds S_w column by column from O.apply_S, whose rows are ordered [s_d][H][W]
    assert np.allclose(res.wS.ravel(), ws[N][nA:], atol=1e-9)


def test_P11_f_identity_and_residual(oracle_lib):
    """f = 2w^n - w^{n-1} = F x^{n-1} - z - b' + w^n and primal_res = |w^n - w^{n-1}| (A27)
    are consistent with the stats the oracle reports: J at x^{n-1} equals Eq. sr_fin evaluated directly."""
    P, y, vo, om, x = tiny(seed=41, nv=2, h=4, w=5, z=2, lambda1=1.0, lambda2=3.0, lambda_reg=0.3,
                           cg_max_iters=8, reweight_every_iter=1)
    y = y.astype(np.float64)
    res = O.admm(P, y, vo, om, 3)
    wo, _, _ = O.setup_wo(P, y, vo, om)
    for n in range(3):
        m = O.weights_m(res.x_iters[n], wo, P.lambda_reg, P.sigma_e)
        J, t = O.cost(P, y, vo, om, m, res.x_iters[n])
        assert rel(res.stats[n]["J"], J) < 1e-12
        assert rel(res.stats[n]["data_l1"], t[0]) < 1e-12


# ----------------------------------------------------------------------------- P9 CG
def test_P9_cg_exact_in_p_steps_and_monotone_quadratic(oracle_lib):
    """With K >> p the x-step solves M dx = -v exactly (direct solve); with fewer steps the quadratic
    1/2 d^T M d + v^T d is non-increasing in K (textbook CG; readings A1-A4)."""
    P, y, vo, om, x = tiny(seed=51, nv=2, h=3, w=4, z=2, lambda1=0.5, lambda2=2.0, lambda_reg=0.2,
                           reweight_every_iter=0)
    y = y.astype(np.float64)
    x0 = O.bicubic(y[P.ref_view], P.scale)
    wo, _, _ = O.setup_wo(P, y, vo, om)
    m = O.weights_m(x0, wo, P.lambda_reg, P.sigma_e)
    Ad, Sd = dense_ops(P, vo, om, m)
    cA = P.lambda2 + 0.5 * P.theta * P.lambda1 ** 2
    M = cA * Ad.T @ Ad + 0.5 * P.theta * Sd.T @ Sd
    # v of the first iteration from the dense pieces (w = 0)
    e = Ad @ x0.ravel() - y.ravel()
    wA = np.clip(P.lambda1 * e, -1 / P.theta, 1 / P.theta)
    rho = P.lambda2 * e + 0.5 * P.theta * P.lambda1 * (2 * wA)
    g = Sd @ x0.ravel()
    wS = np.clip(g, -1 / P.theta, 1 / P.theta)
    v = Ad.T @ rho + 0.5 * P.theta * Sd.T @ (2 * wS)
    exact = x0.ravel() - np.linalg.solve(M, v)
    P.cg_max_iters = EXACT_K
    res = O.admm(P, y, vo, om, 1)
    assert np.allclose(res.x_iters[1].ravel(), exact, atol=1e-8)
    qs = []
    for K in range(1, 9):
        P.cg_max_iters = K
        d = O.admm(P, y, vo, om, 1).x_iters[1].ravel() - x0.ravel()
        qs.append(0.5 * d @ M @ d + v @ d)
    assert all(b <= a + 1e-12 for a, b in zip(qs, qs[1:]))


# ----------------------------------------------------------------------------- P12 convergence
def chambolle_pock(Ad, Sd, y, l1, l2, iters=40000):
    """Independent minimiser of J (Eq. sr_fin) with fixed weights: primal-dual hybrid gradient."""
    K = np.vstack([Ad, Sd])
    L = np.linalg.norm(K, 2)
    tau = sigma = 0.99 / L
    x = np.zeros(K.shape[1])
    xb = x.copy()
    nA = Ad.shape[0]
    v = np.zeros(K.shape[0])
    for _ in range(iters):
        a = v + sigma * (K @ xb)
        # prox of sigma F*: Moreau  a - sigma prox_{F/sigma}(a/sigma)
        t = 1.0 / sigma
        s = a[:nA] / sigma - y
        u1 = y + np.maximum(np.abs(s) - t * l1, 0) * np.sign(s) / (1 + 2 * t * l2)
        u2 = np.maximum(np.abs(a[nA:] / sigma) - t, 0) * np.sign(a[nA:])
        v = a - sigma * np.concatenate([u1, u2])
        xn = x - tau * (K.T @ v)
        xb = 2 * xn - x
        x = xn
    return x


def Jdense(Ad, Sd, y, l1, l2, x):
    e = Ad @ x - y
    return l1 * np.abs(e).sum() + l2 * (e ** 2).sum() + np.abs(Sd @ x).sum()


@pytest.mark.slow
def test_P12_convergence_to_independent_minimiser(oracle_lib):
    """Convex J: frozen weights + exact x-step ADMM reaches J* of an independent
    primal-dual solver within 1 %; J(x^N) <= J(x^0); primal residual decays."""
    P, y, vo, om, x = tiny(seed=61, nv=2, h=4, w=4, z=2, lambda1=1.0, lambda2=2.0, theta=4.0, lambda_reg=0.5,
                           sigma_e=math.inf, cg_max_iters=EXACT_K, reweight_every_iter=0)
    y = y.astype(np.float64)
    x0 = O.bicubic(y[P.ref_view], P.scale)
    wo, _, _ = O.setup_wo(P, y, vo, om)
    m = O.weights_m(x0, wo, P.lambda_reg, P.sigma_e)
    Ad, Sd = dense_ops(P, vo, om, m)
    xs = chambolle_pock(Ad, Sd, y.ravel(), P.lambda1, P.lambda2)
    Jstar = Jdense(Ad, Sd, y.ravel(), P.lambda1, P.lambda2, xs)
    res = O.admm(P, y, vo, om, 200)
    JN = Jdense(Ad, Sd, y.ravel(), P.lambda1, P.lambda2, res.x_iters[-1].ravel())
    J0 = Jdense(Ad, Sd, y.ravel(), P.lambda1, P.lambda2, x0.ravel())
    assert JN <= J0
    assert JN <= Jstar * 1.01 + 1e-9
    assert Jstar <= JN * 1.01 + 1e-9
    assert res.stats[19]["primal_res"] <= 0.1 * res.stats[0]["primal_res"]


# ----------------------------------------------------------------------------- P13 weights
def test_P13_weights_special_cases(oracle_lib):
    H, W = 10, 12
    x = rnd(1, H, W)
    wo = np.abs(rnd(2, H, W))
    assert np.allclose(O.weights_m(x, wo, 0.3, math.inf), 0.3 * wo)           # sigma_e -> inf: w_e = 1
    assert np.allclose(O.weights_m(np.full((H, W), 0.4), wo, 0.3, 0.01), 0.3 * wo)  # constant x
    # central differences of a ramp: |grad x|^2 = 0.25+1 interior (x = 0.5 X + Y)
    Yg, Xg = np.meshgrid(np.arange(H, dtype=float), np.arange(W, dtype=float), indexing="ij")
    mm = O.weights_m(0.5 * Xg + Yg, np.ones((H, W)), 1.0, 2.0)
    assert np.allclose(mm[1:-1, 1:-1], math.exp(-1.25 / 2.0))
    # occlusion boundary b: decreasing omega ramp slope -s per axis -> b = -2s (Eq. weight_occ)
    P = O.Params(n_views=1, lr_h=5, lr_w=6, scale=2, sigma_o1=1.0, sigma_o2=math.inf)
    s = 0.3
    Yh, Xh = np.meshgrid(np.arange(10.0), np.arange(12.0), indexing="ij")
    om = 1.0 - s * (Yh + Xh)
    y = np.random.default_rng(0).uniform(size=(1, 5, 6))
    wo_, b, p = O.setup_wo(P, y, np.zeros((1, 2)), om)
    assert np.allclose(b[:-1, :-1], -2 * s)
    assert np.allclose(O.setup_wo(P, y, np.zeros((1, 2)), 1.0 + s * (Yh + Xh))[1], 0.0)  # increasing: 0
    # b = sigma_o1 sqrt 2, p = 0 -> w_o = e^-1
    s2 = P.sigma_o1 * math.sqrt(2) / 2
    wo_, b, p = O.setup_wo(P, y, np.zeros((1, 2)), 1.0 - s2 * (Yh + Xh))
    assert np.allclose(wo_[:-1, :-1], math.exp(-1.0))
    # noiseless linear LF with constant disparity -> projection error p = 0 in the interior
    c = 0.6
    grid = np.array([(dr, dt) for dt in (-1, 0, 1) for dr in (-1, 0, 1)], dtype=float)
    P9 = O.Params(n_views=9, lr_h=8, lr_w=9, scale=2, ref_view=4)
    L = lambda Y, X: 0.01 * Y + 0.02 * X + 0.3
    ii, jj = np.meshgrid(np.arange(8.0), np.arange(9.0), indexing="ij")
    y9 = np.stack([L(2 * ii + dt * c, 2 * jj + dr * c) for dr, dt in grid])
    _, _, p = O.setup_wo(P9, y9, grid, np.full((16, 18), c))
    assert np.abs(p[2:-3, 2:-3]).max() < 1e-12


# ----------------------------------------------------------------------------- P14 sizes
def test_P14_paper_worked_sizes(oracle_lib):
    rows = [l.split() for l in open(os.path.join(GOLDEN, "paper_sizes.txt")) if l.strip() and l[0] != "#"]
    h, w, z, sk, r, rA, cA, rS = map(int, rows[0])
    P = O.Params(n_views=sk, lr_h=h, lr_w=w, scale=z, radius=r)
    assert P.s_d == len(O.offsets(r)) == 8
    assert h * w * sk == rA and P.H * P.W == cA and P.H * P.W * P.s_d == rS


# ----------------------------------------------------------------------------- bicubic x0
def test_bicubic_interpolates(oracle_lib):
    """x0 (reading A15): constants, interpolation at LR knots, linear reproduction."""
    y = np.random.default_rng(3).uniform(size=(6, 7))
    for z in (2, 3, 4):
        x0 = O.bicubic(y, z)
        assert np.allclose(x0[::z, ::z], y, atol=1e-14)
        assert np.allclose(O.bicubic(np.full((6, 7), 0.3), z), 0.3, atol=1e-14)
        ii, jj = np.meshgrid(np.arange(6.0), np.arange(7.0), indexing="ij")
        lin = O.bicubic(0.1 * ii - 0.2 * jj, z)
        Yg, Xg = np.meshgrid(np.arange(6.0 * z), np.arange(7.0 * z), indexing="ij")
        ref = 0.1 * Yg / z - 0.2 * Xg / z
        assert np.allclose(lin[z:-2 * z, z:-2 * z], ref[z:-2 * z, z:-2 * z], atol=1e-13)


# ----------------------------------------------------------------------------- determinism
def test_oracle_deterministic_across_threads(oracle_lib):
    import subprocess
    import sys
    code = ("import numpy as np, oracle as O; from lfsr_synth import random_instance as ri\n"
            "y,vo,om,x=ri(5,4,10,12,2)\nP=O.Params(n_views=4,lr_h=10,lr_w=12,scale=2,ref_view=1)\n"
            "r=O.admm(P,y,vo,om,3)\nimport sys; sys.stdout.buffer.write(r.x_iters.tobytes())")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for nt in ("1", "4"):
        env = dict(os.environ, OMP_NUM_THREADS=nt, PYTHONPATH=root)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, check=True).stdout)
    assert outs[0] == outs[1] and len(outs[0]) > 0


# ----------------------------------------------------------------------------- P15 usefulness
@pytest.mark.slow
def test_P15_admm_improves_psnr(oracle_lib):
    """Sanity (not parity): the method recovers detail — N = 10 ADMM iterations on a 3x3 light
    field with mixed noise (sigma = 10/255, 10 % impulses) raise PSNR over the bicubic x0 by
    >= 3 dB (the desk-scale analogue of P:L900-908)."""
    import lfsr_synth as S
    cfg = S.Config("P15", 3, 32, 32, 2, 10.0 / 255.0, 10.0, 1.5, "hci", 10)
    lf = S.make_lightfield(cfg, seed=77)
    d = S.SolverDefaults()
    P = O.Params(n_views=9, lr_h=32, lr_w=32, scale=2, ref_view=4, radius=d.radius, lambda1=d.lambda1,
                 lambda2=d.lambda2, lambda_reg=d.lambda_reg, sigma_s=d.sigma_s, sigma_e=d.sigma_e,
                 sigma_o1=d.sigma_o1, sigma_o2=d.sigma_o2, theta=d.theta, cg_max_iters=d.cg_max_iters)
    res = O.admm(P, lf.y, lf.view_offsets, lf.omega, 10)
    p0 = O.psnr(res.x_iters[0], lf.x_gt)
    pN = O.psnr(res.x_iters[-1], lf.x_gt)
    assert pN >= p0 + 3.0, (p0, pN)


# ----------------------------------------------------------------------------- P16/P17 MISR (NEXT-1)
def test_P16_btv_offset_weights(oracle_lib):
    """User offset weights (BTV): with m = 1, sum |S x| over all offsets equals the
    bilateral-TV value sum_{0 < |l|,|k| <= r} alpha^(|l|+|k|) sum_z |x(z) - x(z + (l, k))| over
    pairs inside the image, computed here by array slicing; and S^T is S's transpose."""
    import lfsr_synth as S
    g = np.random.default_rng(16)
    H, W, r, alpha = 13, 17, 2, 0.6
    x = g.standard_normal((H, W))
    wts = S.btv_weights(r, alpha)
    m = np.ones((H, W))
    sx = O.apply_S(x, m, r, 3.0, weights=wts)
    btv = 0.0
    for l in range(-r, r + 1):
        for k in range(-r, r + 1):
            if (l, k) == (0, 0):
                continue
            a = x[max(0, -l):H - max(0, l), max(0, -k):W - max(0, k)]
            b = x[max(0, l):H + min(0, l), max(0, k):W + min(0, k)]
            btv += alpha ** (abs(l) + abs(k)) * np.abs(a - b).sum()
    assert abs(np.abs(sx).sum() - btv) <= 1e-12 * btv
    hv = g.standard_normal(sx.shape)
    lhs = float(np.vdot(sx, hv))
    rhs = float(np.vdot(x, O.apply_ST(hv, m, r, 3.0, weights=wts)))
    assert abs(lhs - rhs) <= 1e-12 * (np.linalg.norm(sx) * np.linalg.norm(hv))
    # the Gaussian default is the same as passing its weights explicitly
    gw = [np.exp(-(dy * dy + dx * dx) / 3.0) for dy in range(-r, r + 1) for dx in range(-r, r + 1)
          if (dy, dx) != (0, 0)]
    assert np.array_equal(O.apply_S(x, m, r, 3.0), O.apply_S(x, m, r, 3.0, weights=gw))


@pytest.mark.slow
def test_P17_misr_improves_psnr(oracle_lib):
    """Sanity (not parity) for the MISR use: 4 frames x2 with 1/2-LR-px global
    shifts, l1 data term + BTV (MisrDefaults); N = 20 ADMM iterations raise PSNR over the
    bicubic x0 of frame 0 by >= 3 dB."""
    import lfsr_synth as S
    lf = S.make_lightfield("M1")
    d = S.MisrDefaults()
    P = O.Params(n_views=4, lr_h=32, lr_w=32, scale=2, ref_view=0, radius=d.radius, lambda1=d.lambda1,
                 lambda2=d.lambda2, lambda_reg=d.lambda_reg, sigma_s=d.sigma_s, sigma_e=d.sigma_e,
                 sigma_o1=d.sigma_o1, sigma_o2=d.sigma_o2, theta=d.theta, cg_max_iters=d.cg_max_iters,
                 offset_weights=d.offset_weights)
    res = O.admm(P, lf.y, lf.view_offsets, lf.omega, 20)
    p0 = O.psnr(res.x_iters[0], lf.x_gt)
    pN = O.psnr(res.x_iters[-1], lf.x_gt)
    assert pN >= p0 + 3.0, (p0, pN)
